"""GPU GMRES solve of BIE 5.4 (NEXT-2, bie_solve_porous) against the oracle's
dense LU solve of the same discrete system.  Tolerance: the
GPU iterate stops at relative residual tol = 1e-13; with the second-kind
operator's condition number O(10), the solution error bar is 1e-11 rel-L2."""
import numpy as np
import pytest

from tests.test_gpu_parity import _dev, _random_case

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bie():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1707_06551_b200 as m
    return m


def gpu_solve(bie, c, a, p, mu, uinf, eta, tol=1e-13, restart=40, precond=True):
    ctx = bie.bie_create(c, a, p, mu)
    bie.bie_set_near(ctx, eta)
    out = torch.empty((len(uinf), 3), dtype=torch.float64, device="cuda")
    it, res = bie.bie_solve_porous(ctx, _dev(uinf), out, tol=tol, max_iter=300, restart=restart,
                                   precond=precond)
    ctx.close()
    return out.cpu().numpy(), it, res


def test_single_sphere_drag(bie):
    p, a, visc = 6, 1.3, 0.8
    c = np.array([[0.2, -0.4, 1.0]])
    U = np.array([0.3, -1.1, 0.6])
    N = (p + 1) * (2 * p + 2)
    dens, it, res = gpu_solve(bie, c, np.array([a]), p, visc, np.tile(U, (N, 1)), 0.0)
    assert res <= 1e-13 and it <= 3
    assert np.abs(dens + 1.5 * visc * U / a).max() <= 1e-13


@pytest.mark.parametrize("precond", [True, False])
@pytest.mark.parametrize("p,ns,eta,restart", [(4, 2, 1.0, 40), (5, 5, 1.0, 40), (4, 6, 0.0, 10)])
def test_solution_matches_dense_oracle(bie, oracle_mod, p, ns, eta, restart, precond):
    c, a, _, _, mu = _random_case(500 + ns, ns, p, True, 1.2)
    N = ns * (p + 1) * (2 * p + 2)
    x, _, _ = oracle_mod.nodes(c, a, p)
    uinf = np.stack([np.sin(x[:, 1]), 0.3 * x[:, 0], np.cos(0.5 * x[:, 2])], 1)  # smooth imposed flow
    ref = oracle_mod.solve_porous(c, a, p, mu, uinf, eta)
    got, it, res = gpu_solve(bie, c, a, p, mu, uinf, eta, restart=restart, precond=precond)
    assert res <= 1e-13
    rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert rel <= 1e-11, (rel, it)
    again, it2, _ = gpu_solve(bie, c, a, p, mu, uinf, eta, restart=restart, precond=precond)
    assert it2 == it and np.array_equal(again, got)   # fixed-order reductions


def test_config2_porous_converges(bie, oracle_mod):
    """64 spheres (cfg 2 geometry, p = 8) in a uniform flow with the near
    correction: GMRES reaches 1e-12 and every sphere feels a drag along U
    below the isolated value 6 pi mu a U."""
    from bie_inputs import make_config
    d = make_config(2)
    N = d["n_nodes"]
    U = np.array([0.0, 0.0, 1.0])
    dens, it, res = gpu_solve(bie, d["centres"], d["radii"], d["p"], d["mu"], np.tile(U, (N, 1)),
                              1.0, tol=1e-12)
    assert res <= 1e-12 and it < 100
    dens0, it0, res0 = gpu_solve(bie, d["centres"], d["radii"], d["p"], d["mu"], np.tile(U, (N, 1)),
                                 1.0, tol=1e-12, precond=False)
    assert res0 <= 1e-12 and it <= it0         # the spectral block preconditioner never hurts here
    assert np.linalg.norm(dens - dens0) <= 1e-10 * np.linalg.norm(dens0)
    _, _, w = oracle_mod.nodes(d["centres"], d["radii"], d["p"])
    ns = (d["p"] + 1) * (2 * d["p"] + 2)
    F = -(w[:, None] * dens).reshape(64, ns, 3).sum(1)
    assert np.all(F[:, 2] > 0) and np.all(F[:, 2] < 6 * np.pi)
