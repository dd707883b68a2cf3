"""Physics pins of the whole GPU pipeline at full BASELINE scale, independent of
the oracle: for per-sphere rigid-body densities q = U_s + Omega_s x (x - c_s),
the double layer vanishes outside each sphere and equals -q inside (jump +1,
A.7 P:662), so the on-surface principal value is exactly D_pv[q] = -q/2 at every
node of every sphere.  The discrete operator reaches this only when close pairs
are handled by the near-singular correction (NEXT-1); the plain smooth rule
misses it by the quadrature error of near neighbours."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bie():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1707_06551_b200 as m
    return m


@pytest.mark.parametrize("cfg,eta,tol", [(2, 3.0, 1e-13), (4, 2.0, 1e-13)])
def test_double_layer_of_rigid_motions_at_full_scale(bie, cfg, eta, tol):
    from bie_inputs import make_config
    d = make_config(cfg, with_targets=False)
    p = d["p"]
    nsn = (p + 1) * (2 * p + 2)
    ns = len(d["radii"])
    ctx = bie.bie_create(d["centres"], d["radii"], p, 1.0)
    N = bie.bie_num_nodes(ctx)
    x = torch.empty((N, 3), dtype=torch.float64, device="cuda")
    bie.bie_get_nodes(ctx, x)
    xc = x.cpu().numpy()
    g = np.random.default_rng(cfg)
    U, Om = g.standard_normal((ns, 3)), g.standard_normal((ns, 3))
    s = np.arange(N) // nsn
    q = U[s] + np.cross(Om[s], xc - d["centres"][s])
    Q = torch.from_numpy(q).cuda()
    u = torch.empty_like(Q)
    bie.bie_apply_DL(ctx, Q, u)                      # plain smooth rule
    torch.cuda.synchronize()
    plain = np.abs(u.cpu().numpy() + 0.5 * q).max() / np.abs(q).max()
    bie.bie_set_near(ctx, eta)
    bie.bie_apply_DL(ctx, Q, u)                      # with the near correction
    torch.cuda.synchronize()
    corrected = np.abs(u.cpu().numpy() + 0.5 * q).max() / np.abs(q).max()
    ctx.close()
    assert corrected <= tol, corrected
    assert plain >= 1e-6, plain                      # the correction is what makes it exact


@pytest.mark.parametrize("gap,p,tol", [(2.0, 12, 1e-13), (1.0, 16, 1e-13), (0.5, 20, 1e-12),
                                       (0.25, 24, 1e-12), (0.1, 30, 1e-11)])
def test_two_sphere_drag_stimson_jeffery_gpu(bie, gap, p, tol):
    """NEXT-1 + NEXT-2 end to end: two fixed unit spheres in a uniform flow
    along their line of centres, BIE 5.4 solved by bie_solve_porous with the
    near-singular correction; the drag on each sphere equals the classical
    Stimson-Jeffery value 6 pi mu a U lambda_SJ, converging spectrally in p
    (measured table: profiles/r01_stimson_jeffery.jsonl)."""
    from tests.test_oracle_porous import stimson_jeffery
    c = 1.0 + gap / 2
    cen = np.array([[0.0, 0.0, -c], [0.0, 0.0, c]])
    ctx = bie.bie_create(cen, np.ones(2), p, 1.0)
    bie.bie_set_near(ctx, 10.0)
    N = bie.bie_num_nodes(ctx)
    uinf = torch.zeros((N, 3), dtype=torch.float64, device="cuda")
    uinf[:, 2] = 1.0
    mu = torch.empty_like(uinf)
    it, res = bie.bie_solve_porous(ctx, uinf, mu, tol=1e-14, max_iter=200, restart=100)
    w = torch.empty(N, dtype=torch.float64, device="cuda")
    bie.bie_get_nodes(ctx, None, None, w)
    torch.cuda.synchronize()
    ctx.close()
    lam = stimson_jeffery(c)
    nsn = N // 2
    for s in range(2):
        F = -(w[s * nsn:(s + 1) * nsn, None] * mu[s * nsn:(s + 1) * nsn]).sum(0).cpu().numpy()
        assert abs(F[2] / (6 * np.pi) - lam) <= tol * lam, (s, F[2] / (6 * np.pi), lam)
        assert np.abs(F[:2]).max() <= 1e-12
