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


@pytest.mark.parametrize("p,ns", [(3, 2), (6, 9), (12, 4), (30, 2), (32, 2)])
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
def gpu_K_near(bie, c, a, p, mu, sigma, eta, parts=3, excl=-1):
    ctx = bie.bie_create(c, a, p, mu)
    bie.bie_set_near(ctx, eta)
    bie.bie_set_near_exclusion(ctx, excl)
    u = torch.full((len(sigma), 3), np.nan, dtype=torch.float64, device="cuda")
    bie.bie_apply_K(ctx, _dev(sigma), u, parts)
    torch.cuda.synchronize()
    ctx.close()
    return u.cpu().numpy()


@pytest.mark.parametrize("excl", [0, 1])
@pytest.mark.parametrize("p,ns,eta", [(4, 6, 1.0), (6, 8, 2.0), (8, 5, 0.7), (12, 4, 1.0), (3, 10, 3.0)])
def test_K_near_matches_oracle(bie, oracle_mod, p, ns, eta, excl):
    """Near pairs' smooth K sum subtracted (excl 0) or skipped in the far field (1)."""
    c, a, f, _, mu = _random_case(1100 + p, ns, p, True, 0.9)
    ref = oracle_mod.apply_K_near(c, a, p, f, eta)
    _assert_parity(gpu_K_near(bie, c, a, p, mu, f, eta, excl=excl), ref, f"K near p={p} eta={eta}")
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


# --------------------------------------- off-surface traction (bie_eval_traction)
def gpu_traction(bie, c, a, p, mu, sigma, tg, tn, eta=0.0, chunks=0, sched=0):
    ctx = bie.bie_create(c, a, p, mu)
    if eta > 0:
        bie.bie_set_near(ctx, eta)
        bie.bie_set_near_off_schedule(ctx, sched)
    if chunks:
        bie.bie_set_source_chunks(ctx, chunks)
    t = torch.full((len(tg), 3), np.nan, dtype=torch.float64, device="cuda")
    bie.bie_eval_traction(ctx, _dev(sigma), _dev(tg), _dev(tn), t)
    torch.cuda.synchronize()
    ctx.close()
    return t.cpu().numpy()


def _targets_around(seed, c, a, m):
    """Targets near surfaces (gaps 0.01a..1a), inside spheres, and in the bulk."""
    rng = np.random.default_rng(seed)
    s = rng.integers(0, len(a), m)
    d = rng.standard_normal((m, 3))
    d /= np.linalg.norm(d, axis=1)[:, None]
    rr = np.where(rng.uniform(size=m) < 0.15, rng.uniform(0.2, 0.9, m), 1.0 + rng.uniform(0.01, 1.0, m))
    tg = c[s] + (a[s] * rr)[:, None] * d
    nv = rng.standard_normal((m, 3))
    return tg, nv / np.linalg.norm(nv, axis=1)[:, None]


@pytest.mark.parametrize("p,ns,eta,chunks,sched", [(4, 5, 0.0, 0, 0), (6, 7, 1.0, 0, 0), (8, 4, 2.0, 3, 0),
                                                    (12, 3, 1.0, 0, 0), (6, 7, 1.0, 0, 1), (12, 3, 1.0, 0, 1)])
def test_traction_offsurface_matches_oracle(bie, oracle_mod, p, ns, eta, chunks, sched):
    """sched: bie_set_near_off_schedule (0 grouped by sphere, 1 per target)."""
    c, a, f, _, mu = _random_case(1300 + p, ns, p, True, 1.1)
    tg, nv = _targets_around(p, c, a, 700)
    got = gpu_traction(bie, c, a, p, mu, f, tg, nv, eta, chunks, sched)
    ref = oracle_mod.traction_offsurface(c, a, p, f, tg, nv, eta)
    _assert_parity(got, ref, f"traction p={p} eta={eta} sched={sched}")


def test_traction_offsurface_closed_forms_on_gpu(bie, oracle_mod):
    """eqs 3.19-3.21 (exterior) at 1.01a..1.8a from one sphere, normal e_r,
    with the near correction: the device reproduces the closed forms to 1e-12.
    Target 0 sits on the source's polar axis, where the closed forms' scipy
    harmonics divide by sin(theta): it is checked against converged
    fine-grid (p = 64) quadrature of the K kernel instead."""
    from tests import _harmonics as H
    from tests.test_oracle_traction import _K_closed_form
    p, a = 8, 1.4
    c = np.array([[0.3, -0.2, 0.5]])
    ctx = bie.bie_create(c, np.array([a]), p, 1.0)
    N = bie.bie_num_nodes(ctx)
    x = torch.empty((N, 3), dtype=torch.float64, device="cuda")
    bie.bie_get_nodes(ctx, x, None, None)
    xs = x.cpu().numpy()
    ctx.close()
    rng = np.random.default_rng(15)
    th, ph = rng.uniform(0.05, 3.1, 40), rng.uniform(-3.1, 3.1, 40)
    th[0], ph[0] = 0.0, 0.0  # a target on the source's polar axis
    er = np.stack([np.sin(th) * np.cos(ph), np.sin(th) * np.sin(ph), np.cos(th)], 1)
    rr = rng.uniform(1.01, 1.8, 40)
    rr[0] = 1.6
    pts = c[0] + a * rr[:, None] * er
    xf, _, _ = oracle_mod.nodes(c, np.array([a]), 64)
    for n, m, ch in ((1, 1, 0), (2, 0, 1), (4, -3, 2), (7, 5, 1), (8, 2, 0)):
        sig = H.vsh_density(n, m, ch, xs, c[0], a)
        got = gpu_traction(bie, c, np.array([a]), p, 1.0, sig, pts, er, eta=1.0)
        ref = np.array([_K_closed_form(n, m, ch, rr[i], th[i], ph[i]) for i in range(1, 40)])
        assert np.abs(got[1:] - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max()), (n, m, ch)
        sigf = np.nan_to_num(H.vsh_density(n, m, ch, xf, c[0], a))  # no fine node on the axis
        pole = oracle_mod.K_at(c, np.array([a]), 64, sigf, pts[:1], er[:1])
        assert np.abs(got[0] - pole[0]).max() <= 1e-12 * max(1.0, np.abs(ref).max()), (n, m, ch)


def test_traction_offsurface_batches_and_edge_cases(bie, oracle_mod):
    """m = 2^21 + 5 targets spans two internal batches; m = 0 is a no-op;
    NULL normals are rejected."""
    p = 4
    c = np.array([[0.0, 0.0, 0.0], [3.0, 0.0, 0.0]])
    a = np.ones(2)
    N = 2 * (p + 1) * (2 * p + 2)
    sig = np.random.default_rng(16).standard_normal((N, 3))
    m = (1 << 21) + 5
    g = torch.Generator(device="cuda").manual_seed(0)
    tg = torch.rand((m, 3), generator=g, dtype=torch.float64, device="cuda") * 20.0 + 5.0
    nv = torch.nn.functional.normalize(torch.randn((m, 3), generator=g, dtype=torch.float64, device="cuda"), dim=1)
    ctx = bie.bie_create(c, a, p, 1.0)
    t = torch.empty_like(tg)
    bie.bie_eval_traction(ctx, _dev(sig), tg, nv, t)
    torch.cuda.synchronize()
    sel = np.r_[0:3, (1 << 21) - 2:(1 << 21) + 5]
    ref = oracle_mod.K_at(c, a, p, sig, tg[sel].cpu().numpy(), nv[sel].cpu().numpy())
    _assert_parity(t[sel].cpu().numpy(), ref, "batched traction")
    empty = torch.empty((0, 3), dtype=torch.float64, device="cuda")
    bie.bie_eval_traction(ctx, _dev(sig), empty, empty, empty)
    with pytest.raises(bie.BieError):
        bie._abi._check(ctx, bie._abi._lib.bie_eval_traction(ctx.handle, bie._abi._ptr(_dev(sig), device=True),
                                                             tg.data_ptr(), None, m, t.data_ptr(), None))
    ctx.close()


def test_K_near_high_order_unstaged(bie, oracle_mod):
    """p = 24: k_near_K's unstaged (global-memory) instantiation; sampled nodes."""
    p = 24
    c = np.array([[0.0, 0.0, 0.0], [2.4, 0.3, -0.2], [-0.5, 2.3, 0.4]])
    a = np.array([1.0, 0.9, 1.1])
    N = 3 * (p + 1) * (2 * p + 2)
    sig = np.random.default_rng(24).standard_normal((N, 3))
    got = gpu_K_near(bie, c, a, p, 1.0, sig, 1.0)
    sub = np.arange(0, N, 37)
    _assert_parity(got[sub], oracle_mod.apply_K_near(c, a, p, sig, 1.0, sub), "K near p=24")


def test_half_plus_K_plus_L_on_rigid_density_single_sphere(bie, oracle_mod):
    """Eq 5.8's left operator on one sphere: (1/2 I + K_pv) annihilates rigid
    densities (K_pv = D_pv on the sphere, and D_pv[rigid] = -rigid/2),
    so (1/2 I + K + L)[F + W x (y - c)] = 4 pi a^2 F + (8 pi a^4/3) W x (x - c)."""
    p, a = 9, 1.3
    c = np.array([[0.4, -0.2, 0.1]])
    x, _, _ = oracle_mod.nodes(c, np.array([a]), p)
    F, W = np.array([0.3, -1.1, 0.6]), np.array([-0.7, 0.2, 0.9])
    sig = F + np.cross(W, x - c[0])
    got = 0.5 * sig + gpu_K(bie, c, np.array([a]), p, 1.0, sig, parts=7)
    ref = 4 * np.pi * a ** 2 * F + (8 * np.pi * a ** 4 / 3) * np.cross(W, x - c[0])
    assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max()
