"""Property tests of the GPU apply (SURVEY §4 tier 4), independent of the oracle:
linearity, weighted symmetry of the single-layer apply (<g, S f>_w = <S g, f>_w,
which the double layer must violate), translation invariance, sphere-permutation
equivariance, and K = D^T in the weighted inner product (reading R21)."""
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


def _apply(bie, c, a, p, mu, f, q, op="SLDL"):
    ctx = bie.bie_create(c, a, p, mu)
    N = bie.bie_num_nodes(ctx)
    u = torch.empty((N, 3), dtype=torch.float64, device="cuda")
    if op == "K":
        bie.bie_apply_K(ctx, _dev(f), u)
    else:
        bie.bie_apply_parts(ctx, _dev(f), _dev(q), u, 3)
    w = torch.empty(N, dtype=torch.float64, device="cuda")
    bie.bie_get_nodes(ctx, None, None, w)
    torch.cuda.synchronize()
    ctx.close()
    return u.cpu().numpy(), w.cpu().numpy()


def test_linearity(bie):
    c, a, f, q, mu = _random_case(1001, 6, 6, True, 1.3)
    u1, _ = _apply(bie, c, a, 6, mu, f, q)
    u2, _ = _apply(bie, c, a, 6, mu, 2.0 * f, -0.5 * q)
    uf, _ = _apply(bie, c, a, 6, mu, f, None)
    uq, _ = _apply(bie, c, a, 6, mu, None, q)
    assert np.abs(u1 - (uf + uq)).max() <= 1e-13 * np.abs(u1).max()
    assert np.abs(u2 - (2.0 * uf - 0.5 * uq)).max() <= 1e-13 * np.abs(u2).max()


def test_single_layer_weighted_symmetry_and_double_layer_asymmetry(bie):
    c, a, f, g, mu = _random_case(1002, 5, 6, True, 1.7)
    Sf, w = _apply(bie, c, a, 6, mu, f, None)
    Sg, _ = _apply(bie, c, a, 6, mu, g, None)
    l, r = np.sum(w[:, None] * g * Sf), np.sum(w[:, None] * Sg * f)
    assert abs(l - r) <= 1e-13 * abs(l)
    Df, _ = _apply(bie, c, a, 6, mu, None, f)
    Dg, _ = _apply(bie, c, a, 6, mu, None, g)
    assert abs(np.sum(w[:, None] * g * Df) - np.sum(w[:, None] * Dg * f)) > 1e-4 * abs(l)


def test_K_is_weighted_adjoint_of_D(bie):
    """<g, K f>_w = <D g, f>_w for the discrete operators: the far-field kernels are
    exact transposes (R21), and the self terms share the D_pv spectrum."""
    c, a, f, g, mu = _random_case(1003, 5, 6, True, 1.0)
    Kf, w = _apply(bie, c, a, 6, mu, f, None, op="K")
    Dg, _ = _apply(bie, c, a, 6, mu, None, g)
    l, r = np.sum(w[:, None] * g * Kf), np.sum(w[:, None] * Dg * f)
    assert abs(l - r) <= 1e-12 * max(abs(l), 1e-3)


def test_translation_and_permutation(bie):
    c, a, f, q, mu = _random_case(1004, 5, 5, True, 0.9)
    u, _ = _apply(bie, c, a, 5, mu, f, q)
    ut, _ = _apply(bie, c + np.array([17.0, -4.0, 9.5]), a, 5, mu, f, q)
    assert np.abs(u - ut).max() <= 1e-12 * np.abs(u).max()
    ns = 6 * 12
    perm = [3, 0, 4, 1, 2]
    idx = np.concatenate([np.arange(s * ns, (s + 1) * ns) for s in perm])
    up, _ = _apply(bie, c[perm], a[perm], 5, mu, f[idx], q[idx])
    assert np.abs(up - u[idx]).max() <= 1e-13 * np.abs(u).max()
