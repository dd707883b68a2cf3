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
