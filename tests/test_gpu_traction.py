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


@pytest.mark.parametrize("p,ns", [(3, 2), (6, 9), (12, 4), (30, 2)])
def test_completion_matches_oracle(bie, oracle_mod, p, ns):
    """Completion L of eq 5.8 (reading R22), alone and with K_pv; p = 30
    exercises nsn = 1,922 > the CTA width (strided per-thread sums)."""
    c, a, f, _, mu = _random_case(900 + p, ns, p, True, 1.3)
    L = oracle_mod.completion(c, a, p, f)
    _assert_parity(gpu_K(bie, c, a, p, mu, f, parts=bie.BIE_PART_COMPLETION), L, f"L p={p}")
    full = gpu_K(bie, c, a, p, mu, f, parts=7)
    _assert_parity(full, oracle_mod.apply_K(c, a, p, f) + L, f"K+L p={p}")


def test_completion_rigid_closed_form_and_reproducible(bie, oracle_mod):
    """L[F + W x (y - c)] = 4 pi a^2 F + (8 pi a^4/3) W x (x - c) on the device;
    two launches agree bitwise (fixed-order moment reduction)."""
    p = 10
    c = np.array([[0.2, 0.1, -0.3], [3.5, 0.0, 0.4], [-1.0, 3.0, 0.0]])
    a = np.array([1.1, 0.6, 0.9])
    x, _, _ = oracle_mod.nodes(c, a, p)
    nsn = (p + 1) * (2 * p + 2)
    rng = np.random.default_rng(11)
    F, W = rng.standard_normal((3, 3)), rng.standard_normal((3, 3))
    sig = np.concatenate([F[b] + np.cross(W[b], x[b * nsn:(b + 1) * nsn] - c[b]) for b in range(3)])
    ref = np.concatenate([4 * np.pi * a[b] ** 2 * F[b] +
                          (8 * np.pi * a[b] ** 4 / 3) * np.cross(W[b], x[b * nsn:(b + 1) * nsn] - c[b])
                          for b in range(3)])
    g1 = gpu_K(bie, c, a, p, 1.0, sig, parts=bie.BIE_PART_COMPLETION)
    g2 = gpu_K(bie, c, a, p, 1.0, sig, parts=bie.BIE_PART_COMPLETION)
    assert np.abs(g1 - ref).max() <= 1e-13 * np.abs(ref).max()
    assert np.array_equal(g1, g2)


def test_completion_part_only_for_K(bie):
    """BIE_PART_COMPLETION belongs to bie_apply_K; bie_apply_parts rejects it."""
    c = np.array([[0.0, 0.0, 0.0], [3.0, 0.0, 0.0]])
    ctx = bie.bie_create(c, np.ones(2), 4, 1.0)
    N = bie.bie_num_nodes(ctx)
    x = torch.zeros(N, 3, dtype=torch.float64, device="cuda")
    u = torch.empty_like(x)
    with pytest.raises(bie.BieError):
        bie.bie_apply_parts(ctx, x, x, u, bie.BIE_PART_COMPLETION)
    with pytest.raises(bie.BieError):
        bie.bie_apply_K(ctx, x, u, 8)
    ctx.close()


# ---------------------------------------------- near-singular correction of K
def gpu_K_near(bie, c, a, p, mu, sigma, eta, parts=3):
    ctx = bie.bie_create(c, a, p, mu)
    bie.bie_set_near(ctx, eta)
    u = torch.full((len(sigma), 3), np.nan, dtype=torch.float64, device="cuda")
    bie.bie_apply_K(ctx, _dev(sigma), u, parts)
    torch.cuda.synchronize()
    ctx.close()
    return u.cpu().numpy()


@pytest.mark.parametrize("p,ns,eta", [(4, 6, 1.0), (6, 8, 2.0), (8, 5, 0.7), (12, 4, 1.0), (3, 10, 3.0)])
def test_K_near_matches_oracle(bie, oracle_mod, p, ns, eta):
    c, a, f, _, mu = _random_case(1100 + p, ns, p, True, 0.9)
    ref = oracle_mod.apply_K_near(c, a, p, f, eta)
    _assert_parity(gpu_K_near(bie, c, a, p, mu, f, eta), ref, f"K near p={p} eta={eta}")
    if p == 6:  # with the completion operator as well
        _assert_parity(gpu_K_near(bie, c, a, p, mu, f, eta, parts=7),
                       ref + oracle_mod.completion(c, a, p, f), "K near + L")


def test_K_near_config3_subset(bie, oracle_mod):
    from tests.test_gpu_parity import _cfg_inputs
    d, f, _ = _cfg_inputs(oracle_mod, 3)
    sub = d["subset"][::8]
    got = gpu_K_near(bie, d["centres"], d["radii"], d["p"], d["mu"], f, 1.0)[sub]
    ref = oracle_mod.apply_K_near(d["centres"], d["radii"], d["p"], f, 1.0, sub)
    _assert_parity(got, ref, "cfg3 K near")


@pytest.mark.parametrize("direction", [(0.0, 0.0, 1.0), (0.3, -0.5, 0.8)])
def test_K_near_two_spheres_vs_converged_quadrature(bie, oracle_mod, direction):
    """Independent of the oracle's derivative formulas: two spheres at gap 0.5
    (axis-aligned and oblique) with band-limited densities; the near-corrected
    K_pv at sphere 0's nodes == sphere 0's self term + the converged (p = 96
    fine grid) K integral over sphere 1, to 1e-12."""
    from tests.test_oracle_near_K import _bandlimited
    p = 8
    e = np.array(direction) / np.linalg.norm(direction)
    a = np.array([1.0, 0.9])
    c = np.stack([np.zeros(3), (a[0] + a[1] + 0.5) * e])
    x, nrm, _ = oracle_mod.nodes(c, a, p)
    nsn = (p + 1) * (2 * p + 2)
    sig = np.concatenate([_bandlimited(21, p, x[:nsn], c[0], a[0]),
                          _bandlimited(22, p, x[nsn:], c[1], a[1])])
    got = gpu_K_near(bie, c, a, p, 1.0, sig, 1.0)[:nsn]
    xf, _, _ = oracle_mod.nodes(c[1:], a[1:], 96)
    sigf = _bandlimited(22, p, xf, c[1], a[1])
    ref = (oracle_mod.self_term(c, a, p, 1.0, None, sig, np.arange(nsn)) +
           oracle_mod.K_at(c[1:], a[1:], 96, sigf, x[:nsn], nrm[:nsn]))
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
