"""GPU parity of the near-singular correction (NEXT-1, bie_set_near) against
the oracle (oracle.apply_near = far + self + near), same bar as the apply:
rel-L2 <= 1e-12 and max-norm <= 1e-10."""
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


def gpu_apply_near(bie, c, a, p, mu, f, q, eta, parts=3, excl=-1):
    ctx = bie.bie_create(c, a, p, mu)
    bie.bie_set_near(ctx, eta)
    bie.bie_set_near_exclusion(ctx, excl)
    npairs = bie.bie_near_pairs(ctx)
    u = torch.full((len(a) * (p + 1) * (2 * p + 2), 3), np.nan, dtype=torch.float64, device="cuda")
    bie.bie_apply_parts(ctx, _dev(f), _dev(q), u, parts)
    torch.cuda.synchronize()
    ctx.close()
    return u.cpu().numpy(), npairs


def _count_pairs(oracle_mod, c, a, eta):
    return sum(oracle_mod.is_near(c[s], a[s], c[t], a[t], eta)
               for t in range(len(a)) for s in range(len(a)) if s != t)


def test_near_two_spheres_close(bie, oracle_mod):
    p, mu = 8, 1.3
    d = np.array([1.0, 0.13, -0.087])
    c = np.array([[0.0, 0.0, 0.0], 2.3 * d / np.linalg.norm(d)])
    a = np.ones(2)
    rng = np.random.default_rng(3)
    N = 2 * (p + 1) * (2 * p + 2)
    f, q = rng.standard_normal((N, 3)), rng.standard_normal((N, 3))
    got, npairs = gpu_apply_near(bie, c, a, p, mu, f, q, 1.0)
    assert npairs == 2
    _assert_parity(got, oracle_mod.apply_near(c, a, p, mu, f, q, 1.0), "near 2 spheres")


@pytest.mark.parametrize("excl", [0, 1])
@pytest.mark.parametrize("p,ns,eta", [(4, 6, 0.5), (6, 8, 1.0), (5, 5, 2.0), (12, 3, 1.0)])
def test_near_random_suspensions(bie, oracle_mod, p, ns, eta, excl):
    """Both treatments of the near pairs' smooth rule (bie_set_near_exclusion:
    0 subtracted by k_near, 1 skipped inside the far-field kernel)."""
    c, a, f, q, mu = _random_case(300 + p + ns, ns, p, True, 0.9)
    got, npairs = gpu_apply_near(bie, c, a, p, mu, f, q, eta, excl=excl)
    assert npairs == _count_pairs(oracle_mod, c, a, eta)
    _assert_parity(got, oracle_mod.apply_near(c, a, p, mu, f, q, eta), f"near p={p} eta={eta}")


def test_near_far_part_only_and_sl_dl(bie, oracle_mod):
    c, a, f, q, mu = _random_case(77, 5, 6, True, 1.1)
    got, _ = gpu_apply_near(bie, c, a, 6, mu, f, q, 1.0, parts=bie.BIE_PART_FAR)
    ref = oracle_mod.far(c, a, 6, mu, f, q) + oracle_mod.near(c, a, 6, mu, f, q, 1.0)
    _assert_parity(got, ref, "far+near")
    got, _ = gpu_apply_near(bie, c, a, 6, mu, f, None, 1.0)
    _assert_parity(got, oracle_mod.apply_near(c, a, 6, mu, f, None, 1.0), "SL near")
    got, _ = gpu_apply_near(bie, c, a, 6, mu, None, q, 1.0)
    _assert_parity(got, oracle_mod.apply_near(c, a, 6, mu, None, q, 1.0), "DL near")


def test_near_disabled_is_bitwise_default(bie):
    c, a, f, q, mu = _random_case(78, 4, 5, True, 1.0)
    u0, n0 = gpu_apply_near(bie, c, a, 5, mu, f, q, 0.0)
    ctx = bie.bie_create(c, a, 5, mu)
    u = torch.empty((len(f), 3), dtype=torch.float64, device="cuda")
    bie.bie_apply_SLDL(ctx, _dev(f), _dev(q), u)
    torch.cuda.synchronize()
    assert n0 == 0 and np.array_equal(u0, u.cpu().numpy())
    with pytest.raises(bie.BieError):
        bie.bie_set_near(ctx, -1.0)
    ctx.close()


def test_near_translating_sphere_neighbour(bie):
    """Physical check through the GPU path: sphere 0 translating (uniform
    traction 3 mu U/2), sphere 1 at gap 0.2 with zero density: on sphere 1 the
    near-corrected apply equals the classical Stokes flow (the plain smooth
    rule misses it by ~1e-2)."""
    p, mu = 8, 1.3
    d = np.array([1.0, 0.13, -0.087])
    c = np.array([[0.0, 0.0, 0.0], 2.2 * d / np.linalg.norm(d)])
    a = np.ones(2)
    ns = (p + 1) * (2 * p + 2)
    U = np.array([0.5, -0.3, 0.8])
    f = np.zeros((2 * ns, 3))
    f[:ns] = 3 * mu * U / 2
    got, _ = gpu_apply_near(bie, c, a, p, mu, f, None, 1.0)
    plain, _ = gpu_apply_near(bie, c, a, p, mu, f, None, 0.0)
    ctx = bie.bie_create(c, a, p, mu)
    x = torch.empty((2 * ns, 3), dtype=torch.float64, device="cuda")
    bie.bie_get_nodes(ctx, x)
    x = x.cpu().numpy()[ns:]
    ctx.close()
    dv = x - c[0]
    rr = np.linalg.norm(dv, axis=1)[:, None]
    e = dv / rr
    Ue = (e @ U)[:, None]
    ref = 0.75 * (U / rr + Ue * e / rr) + 0.25 * (U / rr ** 3 - 3 * Ue * e / rr ** 3)
    assert np.abs(got[ns:] - ref).max() <= 1e-13
    assert np.abs(plain[ns:] - ref).max() >= 1e-4


def test_near_config4_subset(bie, oracle_mod):
    """cfg 4 (jittered lattice, gaps ~1) with eta = 1: 6-ish near neighbours per sphere."""
    from tests.test_gpu_parity import _cfg_inputs
    d, f, q = _cfg_inputs(oracle_mod, 4)
    sub = d["subset"][::32]
    got, npairs = gpu_apply_near(bie, d["centres"], d["radii"], d["p"], d["mu"], f, q, 1.0)
    assert npairs > 0
    ref = oracle_mod.apply_near(d["centres"], d["radii"], d["p"], d["mu"], f, q, 1.0, sub)
    _assert_parity(got[sub], ref, "cfg4 near")


# ------------------------------------------------- off-surface targets (a7)
def _near_targets(c, a, n, seed, lo=0.1, hi=1.5):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        s = rng.integers(len(a))
        d = rng.standard_normal(3)
        x = c[s] + d / np.linalg.norm(d) * a[s] * (1.0 + rng.uniform(lo, hi))
        if np.all(np.linalg.norm(x - c, axis=1) - a > 0.05):
            out.append(x)
    return np.array(out)


@pytest.mark.parametrize("sched", [0, 1])
@pytest.mark.parametrize("p,ns,eta,use_p,m", [(5, 4, 1.0, True, 300), (8, 6, 0.5, True, 300),
                                              (6, 3, 2.0, False, 300), (4, 2, 1.0, True, 700)])
def test_offsurface_near_matches_oracle(bie, oracle_mod, p, ns, eta, use_p, m, sched):
    """Both schedules of the off-surface correction (bie_set_near_off_schedule):
    0 pairs grouped by sphere -- m = 700 targets around 2 spheres puts > 128
    pairs (one CTA chunk) on a sphere, so chunks split ragged -- and 1 one
    thread per Morton-sorted target."""
    c, a, f, q, mu = _random_case(900 + p, ns, p, True, 1.4)
    tg = _near_targets(c, a, m, p)
    tg = np.concatenate([tg, c[:2] + np.array([[0.1, -0.2, 0.15]])])  # two interior targets
    uref, pref = oracle_mod.offsurface_near(c, a, p, mu, f, q, eta, tg)
    ctx = bie.bie_create(c, a, p, mu)
    bie.bie_set_near(ctx, eta)
    bie.bie_set_near_off_schedule(ctx, sched)
    u = torch.empty((len(tg), 3), dtype=torch.float64, device="cuda")
    pr = torch.empty(len(tg), dtype=torch.float64, device="cuda") if use_p else None
    bie.bie_eval_offsurface(ctx, _dev(f), _dev(q), _dev(tg), u, pr)
    torch.cuda.synchronize()
    ctx.close()
    _assert_parity(u.cpu().numpy(), uref, "offsurface near u")
    if use_p:
        _assert_parity(pr.cpu().numpy(), pref, "offsurface near p")


def test_offsurface_near_config5_subset(bie, oracle_mod):
    """cfg 5 (targets >= 0.25 from every surface) with eta = 1."""
    from tests.test_gpu_parity import _cfg_inputs
    d, f, q = _cfg_inputs(oracle_mod, 5)
    tsub = d["target_subset"][::16]
    ctx = bie.bie_create(d["centres"], d["radii"], d["p"], d["mu"])
    bie.bie_set_near(ctx, 1.0)
    tg = _dev(d["targets"])
    M = tg.shape[0]
    u = torch.empty((M, 3), dtype=torch.float64, device="cuda")
    pr = torch.empty(M, dtype=torch.float64, device="cuda")
    bie.bie_eval_offsurface(ctx, _dev(f), _dev(q), tg, u, pr)
    torch.cuda.synchronize()
    ctx.close()
    uref, pref = oracle_mod.offsurface_near(d["centres"], d["radii"], d["p"], d["mu"], f, q, 1.0,
                                            d["targets"][tsub])
    _assert_parity(u.cpu().numpy()[tsub], uref, "cfg5 near u")
    _assert_parity(pr.cpu().numpy()[tsub], pref, "cfg5 near p")


def test_offsurface_near_schedules_agree_config5(bie, oracle_mod):
    """cfg 5, all 1e6 targets, eta = 1: the grouped schedule (0) against the
    per-target one (1) element by element (same per-pair arithmetic and the
    same ascending-sphere sum order up to list-overflow flushes), u and p."""
    from tests.test_gpu_parity import _cfg_inputs
    d, f, q = _cfg_inputs(oracle_mod, 5)
    ctx = bie.bie_create(d["centres"], d["radii"], d["p"], d["mu"])
    bie.bie_set_near(ctx, 1.0)
    tg = _dev(d["targets"])
    M = tg.shape[0]
    out = []
    for sched in (0, 1):
        bie.bie_set_near_off_schedule(ctx, sched)
        u = torch.empty((M, 3), dtype=torch.float64, device="cuda")
        pr = torch.empty(M, dtype=torch.float64, device="cuda")
        bie.bie_eval_offsurface(ctx, _dev(f), _dev(q), tg, u, pr)
        torch.cuda.synchronize()
        out.append((u.cpu().numpy(), pr.cpu().numpy()))
    with pytest.raises(bie.BieError):
        bie.bie_set_near_off_schedule(ctx, 2)
    ctx.close()
    (u0, p0), (u1, p1) = out
    assert np.abs(u0 - u1).max() <= 1e-13 * np.abs(u1).max()
    assert np.abs(p0 - p1).max() <= 1e-13 * np.abs(p1).max()


def test_offsurface_near_no_pairs_and_high_order(bie, oracle_mod):
    """Grouped schedule edge cases: targets with no near sphere (pair count 0:
    the early return) and p = 32, where a sphere's records exceed the 100 KB
    staging budget (k_noff_grp<.., STAGE = false>)."""
    c = np.array([[0.0, 0.0, 0.0], [3.0, 0.2, -0.1]])
    a = np.array([1.0, 0.8])
    for p, tg in ((6, np.array([[20.0, 0.0, 0.0], [0.0, 30.0, 1.0]])),
                  (32, _near_targets(c, a, 40, 32))):
        N = 2 * (p + 1) * (2 * p + 2)
        rng = np.random.default_rng(p)
        f, q = rng.standard_normal((N, 3)), rng.standard_normal((N, 3))
        uref, pref = oracle_mod.offsurface_near(c, a, p, 1.0, f, q, 1.0, tg)
        ctx = bie.bie_create(c, a, p, 1.0)
        bie.bie_set_near(ctx, 1.0)
        u = torch.empty((len(tg), 3), dtype=torch.float64, device="cuda")
        pr = torch.empty(len(tg), dtype=torch.float64, device="cuda")
        bie.bie_eval_offsurface(ctx, _dev(f), _dev(q), _dev(tg), u, pr)
        torch.cuda.synchronize()
        ctx.close()
        _assert_parity(u.cpu().numpy(), uref, f"offsurface near p={p} u")
        _assert_parity(pr.cpu().numpy(), pref, f"offsurface near p={p} p")


@pytest.mark.parametrize("p", [24, 30, 32])
def test_near_high_order_unstaged(bie, oracle_mod, p):
    """p >= 24: a neighbour's records + coefficients no longer fit the 160 KB
    staging budget, so k_near reads them from global memory (the STAGE = false
    instantiation).  Three spheres, sampled target nodes."""
    c = np.array([[0.0, 0.0, 0.0], [2.4, 0.3, -0.2], [-0.5, 2.3, 0.4]])
    a = np.array([1.0, 0.9, 1.1])
    N = 3 * (p + 1) * (2 * p + 2)
    rng = np.random.default_rng(p)
    f, q = rng.standard_normal((N, 3)), rng.standard_normal((N, 3))
    got, npairs = gpu_apply_near(bie, c, a, p, 1.2, f, q, 1.0)
    assert npairs == _count_pairs(oracle_mod, c, a, 1.0) > 0
    sub = np.arange(0, N, 37)
    _assert_parity(got[sub], oracle_mod.apply_near(c, a, p, 1.2, f, q, 1.0, sub), f"near p={p}")
