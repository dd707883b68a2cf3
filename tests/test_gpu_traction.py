"""GPU parity of the traction operator K (NEXT-3, bie_apply_K) against the
oracle (oracle.apply_K = far_K + D_pv-spectrum self term, reading R21)."""
import numpy as np
import pytest

from tests.test_gpu_parity import _assert_parity, _dev, _random_case

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bie():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1707_06551_b200 as m
    return m


def gpu_K(bie, c, a, p, mu, sigma, parts=3, chunks=0):
    ctx = bie.bie_create(c, a, p, mu)
    if chunks:
        bie.bie_set_source_chunks(ctx, chunks)
    u = torch.full((len(sigma), 3), np.nan, dtype=torch.float64, device="cuda")
    bie.bie_apply_K(ctx, _dev(sigma), u, parts)
    torch.cuda.synchronize()
    ctx.close()
    return u.cpu().numpy()


@pytest.mark.parametrize("p,ns,chunks", [(4, 3, 0), (6, 7, 2), (8, 5, 0), (12, 3, 1)])
def test_K_matches_oracle(bie, oracle_mod, p, ns, chunks):
    c, a, f, _, mu = _random_case(700 + p, ns, p, True, 1.3)
    _assert_parity(gpu_K(bie, c, a, p, mu, f, chunks=chunks), oracle_mod.apply_K(c, a, p, f), f"K p={p}")
    _assert_parity(gpu_K(bie, c, a, p, mu, f, parts=bie.BIE_PART_FAR), oracle_mod.far_K(c, a, p, f),
                   "K far")
    _assert_parity(gpu_K(bie, c, a, p, mu, f, parts=bie.BIE_PART_SELF),
                   oracle_mod.self_term(c, a, p, 1.0, None, f), "K self")


def test_K_translating_sphere_traction(bie):
    p, a, mu = 8, 0.9, 1.4
    c = np.array([[0.0, 0.5, 0.0]])
    U = np.array([0.2, 0.7, -0.4])
    N = (p + 1) * (2 * p + 2)
    f = np.tile(1.5 * mu * U / a, (N, 1))
    kpv = gpu_K(bie, c, np.array([a]), p, mu, f)
    assert np.abs(kpv - 0.5 * f + 1.5 * mu * U / a).max() <= 1e-13  # exterior traction K_+ = K_pv - f/2


def test_K_config3_subset(bie, oracle_mod):
    from tests.test_gpu_parity import _cfg_inputs
    d, f, _ = _cfg_inputs(oracle_mod, 3)
    sub = d["subset"][::8]
    got = gpu_K(bie, d["centres"], d["radii"], d["p"], d["mu"], f)[sub]
    _assert_parity(got, oracle_mod.apply_K(d["centres"], d["radii"], d["p"], f, sub), "cfg3 K")
