"""GPU parity: the CUDA path (through the C-ABI) vs the CPU oracle, element by
element on the same seeded inputs.  Bar (BASELINE.json north_star): relative
L2 <= 1e-12 and max |delta| / max |u_ref| <= 1e-10 in fp64.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

REL_L2 = 1e-12
MAX_REL = 1e-10


@pytest.fixture(scope="module")
def bie():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1707_06551_b200 as m
    return m


def _err(got, ref):
    got, ref = np.asarray(got), np.asarray(ref)
    return (np.linalg.norm(got - ref) / np.linalg.norm(ref),
            np.abs(got - ref).max() / np.abs(ref).max())


def _assert_parity(got, ref, what=""):
    rel, mx = _err(got, ref)
    assert rel <= REL_L2 and mx <= MAX_REL, f"{what}: rel-L2 {rel:.3e} max {mx:.3e}"


def _dev(a):
    return None if a is None else torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def gpu_apply(bie, centres, radii, p, mu, f, q, parts=3, chunks=0):
    ctx = bie.bie_create(centres, radii, p, mu)
    if chunks:
        bie.bie_set_source_chunks(ctx, chunks)
    N = bie.bie_num_nodes(ctx)
    u = torch.full((N, 3), np.nan, dtype=torch.float64, device="cuda")
    bie.bie_apply_parts(ctx, _dev(f), _dev(q), u, parts)
    torch.cuda.synchronize()
    ctx.close()
    return u.cpu().numpy()


def _random_case(seed, ns, p, poly=True, mu=1.0):
    """Small random suspension (not a BASELINE config): RSA-like placement."""
    rng = np.random.default_rng(seed)
    radii = rng.uniform(0.5, 1.5, ns) if poly else np.ones(ns)
    c = []
    while len(c) < ns:
        x = rng.uniform(0, 4.0 * ns ** (1 / 3) + 3, 3)
        i = len(c)
        if all(np.linalg.norm(x - y) >= radii[i] + radii[j] + 0.3 for j, y in enumerate(c)):
            c.append(x)
    N = ns * (p + 1) * (2 * p + 2)
    return np.array(c), radii, rng.standard_normal((N, 3)), rng.standard_normal((N, 3)), mu


# ------------------------------------------------------------------- a1
@pytest.mark.parametrize("p", [1, 4, 12, 30, 32])
def test_nodes_match_oracle(bie, oracle_mod, p):
    c, a, _, _, _ = _random_case(p, 5, p)
    ctx = bie.bie_create(c, a, p, 1.0)
    N = bie.bie_num_nodes(ctx)
    x = torch.empty((N, 3), dtype=torch.float64, device="cuda")
    n = torch.empty_like(x)
    w = torch.empty(N, dtype=torch.float64, device="cuda")
    bie.bie_get_nodes(ctx, x, n, w)
    torch.cuda.synchronize()
    xr, nr, wr = oracle_mod.nodes(c, a, p)
    assert np.abs(x.cpu().numpy() - xr).max() <= 4e-15 * np.abs(xr).max()
    assert np.abs(n.cpu().numpy() - nr).max() <= 2e-15
    assert np.abs(w.cpu().numpy() / wr - 1).max() <= 4e-14
    ctx.close()


# --------------------------------------------------------- a4-a6 self term
@pytest.mark.parametrize("p,ns,poly,mu", [(1, 3, True, 1.0), (4, 2, False, 1.0), (8, 4, True, 1.7),
                                          (12, 2, True, 0.6), (16, 1, False, 1.0), (30, 1, True, 2.0),
                                          (31, 1, False, 1.0), (32, 2, True, 0.8)])
def test_self_term_only(bie, oracle_mod, p, ns, poly, mu):
    c, a, f, q, mu = _random_case(100 + p, ns, p, poly, mu)
    ref = oracle_mod.self_term(c, a, p, mu, f, q)
    got = gpu_apply(bie, c, a, p, mu, f, q, parts=bie.BIE_PART_SELF)
    _assert_parity(got, ref, f"self p={p}")


@pytest.mark.parametrize("variant", [0, 1, 2, 3])
@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8, 9, 12, 13, 16, 17, 24, 32])
def test_self_term_kernel_variants(bie, oracle_mod, p, variant):
    """Every self-term kernel (bie_set_self_kernel: 0 batched DMMA contractions,
    1 batched DFMA, 2 round-1 per-sphere, 3 per-sphere with two spheres per CTA) on 5 polydisperse spheres -- a
    ragged last batch for the 4- and 2-sphere batches of k_sht -- against the
    oracle's direct projection (O-4), S and D together and each alone."""
    c, a, f, q, mu = _random_case(700 + p, 5, p, True, 0.9)
    ctx = bie.bie_create(c, a, p, mu)
    P1, nphi = p + 1, 2 * p + 2
    two_sphere_smem = (2 * (6 * P1 * nphi + 12 * P1 * P1) + 2 * nphi) * 8
    if variant == 3 and two_sphere_smem > 227 * 1024:
        # include/bie.h: variant 3 stages two spheres per CTA; beyond 227 KB it
        # is refused with BIE_ERR_UNSUPPORTED and the previous kernel stays.
        with pytest.raises(bie.BieError) as e:
            bie.bie_set_self_kernel(ctx, variant)
        assert e.value.status == bie.BIE_ERR_UNSUPPORTED
        ctx.close()
        return
    bie.bie_set_self_kernel(ctx, variant)
    N = bie.bie_num_nodes(ctx)
    for fx, qx, what in ((f, q, "S+D"), (f, None, "S"), (None, q, "D")):
        u = torch.full((N, 3), np.nan, dtype=torch.float64, device="cuda")
        bie.bie_apply_parts(ctx, _dev(fx), _dev(qx), u, bie.BIE_PART_SELF)
        torch.cuda.synchronize()
        ref = oracle_mod.self_term(c, a, p, mu, fx, qx)
        _assert_parity(u.cpu().numpy(), ref, f"self variant {variant} p={p} {what}")
    ctx.close()


@pytest.mark.parametrize("p", [6, 12, 24])
def test_self_term_unaligned_views(bie, oracle_mod, p):
    """f, q, u passed as views offset by one double (8-byte, not 16-byte,
    aligned): k_self_t's TMA bulk loads of f, q and its bulk store of u need
    16-byte alignment, so it falls back to cooperative loads and direct
    stores.  Same values as the aligned call, and parity with the oracle."""
    c, a, f, q, mu = _random_case(760 + p, 3, p, True, 1.1)
    ctx = bie.bie_create(c, a, p, mu)
    N = bie.bie_num_nodes(ctx)

    def view(x):
        buf = torch.full((3 * N + 1,), np.nan, dtype=torch.float64, device="cuda")
        v = buf[1:].view(N, 3)
        if x is not None:
            v.copy_(torch.from_numpy(x))
        assert v.data_ptr() % 16 == 8
        return v
    fu, qu, uu = view(f), view(q), view(None)
    bie.bie_apply_parts(ctx, fu, qu, uu, bie.BIE_PART_SELF)
    ua = torch.full((N, 3), np.nan, dtype=torch.float64, device="cuda")
    bie.bie_apply_parts(ctx, _dev(f), _dev(q), ua, bie.BIE_PART_SELF)
    torch.cuda.synchronize()
    ctx.close()
    got = uu.cpu().numpy()
    assert np.array_equal(got, ua.cpu().numpy())
    _assert_parity(got, oracle_mod.self_term(c, a, p, mu, f, q), f"self unaligned p={p}")


# ------------------------------------------------------------- a3 far field
@pytest.mark.parametrize("p,ns,chunks", [(4, 2, 0), (4, 7, 3), (6, 9, 0), (8, 5, 1), (5, 3, 2)])
def test_far_field_only(bie, oracle_mod, p, ns, chunks):
    c, a, f, q, mu = _random_case(200 + p + ns, ns, p, True, 1.3)
    ref = oracle_mod.far(c, a, p, mu, f, q)
    got = gpu_apply(bie, c, a, p, mu, f, q, parts=bie.BIE_PART_FAR, chunks=chunks)
    _assert_parity(got, ref, f"far p={p} ns={ns} chunks={chunks}")


def test_single_sphere_far_field_is_zero(bie):
    c, a, f, q, mu = _random_case(7, 1, 6)
    got = gpu_apply(bie, c, a, 6, mu, f, q, parts=bie.BIE_PART_FAR)
    assert np.all(got == 0.0)


# ------------------------------------------------------- BASELINE configs
def _cfg_inputs(oracle_mod, cfg):
    from bie_inputs import make_config, rigid_field
    d = make_config(cfg, with_targets=(cfg == 5))
    f, q = d["f"], d["q"]
    if d["rigid"] is not None:
        x, _, _ = oracle_mod.nodes(d["centres"], d["radii"], d["p"])
        q = rigid_field(*d["rigid"], x, d["centres"], (d["p"] + 1) * (2 * d["p"] + 2))
    if d["same_fq"]:
        f = q
    return d, f, q


def test_config1_full(bie, oracle_mod):
    d, f, q = _cfg_inputs(oracle_mod, 1)
    ref = oracle_mod.apply(d["centres"], d["radii"], d["p"], d["mu"], f, q)
    got = gpu_apply(bie, d["centres"], d["radii"], d["p"], d["mu"], f, q)
    _assert_parity(got, ref, "cfg1")
    # SL only / DL only through their own entry points
    ctx = bie.bie_create(d["centres"], d["radii"], d["p"], d["mu"])
    u = torch.empty((100, 3), dtype=torch.float64, device="cuda")
    bie.bie_apply_SL(ctx, _dev(f), u)
    _assert_parity(u.cpu().numpy(), oracle_mod.apply(d["centres"], d["radii"], 4, 1.0, f, None), "SL")
    bie.bie_apply_DL(ctx, _dev(q), u)
    _assert_parity(u.cpu().numpy(), oracle_mod.apply(d["centres"], d["radii"], 4, 1.0, None, q), "DL")
    ctx.close()


def test_config2_full(bie, oracle_mod):
    d, f, q = _cfg_inputs(oracle_mod, 2)
    ref = oracle_mod.apply(d["centres"], d["radii"], d["p"], d["mu"], f, q)
    got = gpu_apply(bie, d["centres"], d["radii"], d["p"], d["mu"], f, q)
    _assert_parity(got, ref, "cfg2")


@pytest.mark.parametrize("cfg", [3, 4, 5])
def test_config_subset(bie, oracle_mod, cfg):
    """Full-size configs in the launch configuration bench.py times; the oracle
    evaluates every node of the seeded 4096-node subset (BASELINE.json configs
    3-5: "oracle on a seeded 4096-target subset")."""
    d, f, q = _cfg_inputs(oracle_mod, cfg)
    sub = d["subset"]
    assert len(sub) == 4096
    got = gpu_apply(bie, d["centres"], d["radii"], d["p"], d["mu"], f, q)[sub]
    ref = oracle_mod.apply(d["centres"], d["radii"], d["p"], d["mu"], f, q, sub)
    _assert_parity(got, ref, f"cfg{cfg}")


def test_config5_offsurface_subset(bie, oracle_mod):
    """cfg 5 off-surface velocity AND pressure at all 4096 targets of the seeded
    off-surface subset (1e6 targets evaluated on the GPU in one call)."""
    d, f, q = _cfg_inputs(oracle_mod, 5)
    tsub = d["target_subset"]
    assert len(tsub) == 4096
    ctx = bie.bie_create(d["centres"], d["radii"], d["p"], d["mu"])
    tg = _dev(d["targets"])
    M = tg.shape[0]
    u = torch.empty((M, 3), dtype=torch.float64, device="cuda")
    p = torch.empty(M, dtype=torch.float64, device="cuda")
    bie.bie_eval_offsurface(ctx, _dev(f), _dev(q), tg, u, p)
    torch.cuda.synchronize()
    uref, pref = oracle_mod.offsurface(d["centres"], d["radii"], d["p"], d["mu"], f, q,
                                       d["targets"][tsub])
    _assert_parity(u.cpu().numpy()[tsub], uref, "cfg5 offsurface u")
    _assert_parity(p.cpu().numpy()[tsub], pref, "cfg5 offsurface p")
    ctx.close()


def test_offsurface_two_batches(bie, oracle_mod):
    """m = 2^21 + 5 targets: bie_eval_offsurface splits targets into internal
    batches of 2^21 (csrc/bie.cu kOffBatch); the second batch's output offsets
    (u + 3 b0, p + b0) and its pressure partials are checked against the oracle
    at EVERY target (u and p), with the seam indices asserted separately."""
    c, a, f, q, mu = _random_case(2101, 4, 5, True, 0.9)
    m = (1 << 21) + 5
    rng = np.random.default_rng(2102)
    lo, hi = c.min(0) - 3.0, c.max(0) + 3.0
    tg = np.empty((0, 3))
    while len(tg) < m:
        x = rng.uniform(lo, hi, (m, 3))
        dmin = np.min(np.linalg.norm(x[:, None] - c[None], axis=-1) - a[None], axis=1)
        tg = np.concatenate([tg, x[np.abs(dmin) > 0.25]])
    tg = np.ascontiguousarray(tg[:m])
    ctx = bie.bie_create(c, a, 5, mu)
    u = torch.full((m, 3), np.nan, dtype=torch.float64, device="cuda")
    p = torch.full((m,), np.nan, dtype=torch.float64, device="cuda")
    bie.bie_eval_offsurface(ctx, _dev(f), _dev(q), _dev(tg), u, p)
    torch.cuda.synchronize()
    ctx.close()
    ug, pg = u.cpu().numpy(), p.cpu().numpy()
    uref, pref = oracle_mod.offsurface(c, a, 5, mu, f, q, tg)
    seam = np.arange((1 << 21) - 2, (1 << 21) + 5)
    _assert_parity(ug[seam], uref[seam], "u at the batch seam")
    _assert_parity(pg[seam], pref[seam], "p at the batch seam")
    _assert_parity(ug[:64], uref[:64], "u head")
    _assert_parity(ug, uref, "u all")
    _assert_parity(pg, pref, "p all")


# --------------------------------------------------------- a7 off-surface
@pytest.mark.parametrize("use_f,use_q,use_p", [(True, True, True), (True, False, True),
                                               (False, True, False)])
def test_offsurface_small(bie, oracle_mod, use_f, use_q, use_p):
    c, a, f, q, mu = _random_case(11, 4, 5, True, 0.8)
    rng = np.random.default_rng(12)
    tg = rng.uniform(-3, 10, (1000, 3))
    dmin = np.min(np.linalg.norm(tg[:, None] - c[None], axis=-1) - a[None], axis=1)
    tg = tg[np.abs(dmin) > 0.3]
    fx, qx = (f if use_f else None), (q if use_q else None)
    uref, pref = oracle_mod.offsurface(c, a, 5, mu, fx, qx, tg)
    ctx = bie.bie_create(c, a, 5, mu)
    M = len(tg)
    u = torch.empty((M, 3), dtype=torch.float64, device="cuda")
    p = torch.empty(M, dtype=torch.float64, device="cuda") if use_p else None
    bie.bie_eval_offsurface(ctx, _dev(fx), _dev(qx), _dev(tg), u, p)
    torch.cuda.synchronize()
    _assert_parity(u.cpu().numpy(), uref, "offsurface u")
    if use_p:
        _assert_parity(p.cpu().numpy(), pref, "offsurface p")
    # zero targets is a no-op
    bie.bie_eval_offsurface(ctx, _dev(fx), _dev(qx), torch.empty((0, 3), dtype=torch.float64,
                                                                   device="cuda"),
                            torch.empty((0, 3), dtype=torch.float64, device="cuda"))
    ctx.close()


# ---------------------------------------------------- determinism, e2e, ABI
def test_determinism_and_host_entry_point(bie, oracle_mod):
    d, f, q = _cfg_inputs(oracle_mod, 2)
    u1 = gpu_apply(bie, d["centres"], d["radii"], d["p"], d["mu"], f, q)
    u2 = gpu_apply(bie, d["centres"], d["radii"], d["p"], d["mu"], f, q)
    assert np.array_equal(u1, u2)
    ctx = bie.bie_create(d["centres"], d["radii"], d["p"], d["mu"])
    uh = np.empty_like(f)
    bie.bie_apply_SLDL_host(ctx, np.ascontiguousarray(f), np.ascontiguousarray(q), uh)
    assert np.array_equal(uh, u1)
    ctx.close()


def test_chunking_changes_only_rounding(bie, oracle_mod):
    c, a, f, q, mu = _random_case(31, 6, 7, True, 1.0)
    ref = oracle_mod.apply(c, a, 7, mu, f, q)
    for ch in (1, 2, 5, 11):
        _assert_parity(gpu_apply(bie, c, a, 7, mu, f, q, chunks=ch), ref, f"chunks={ch}")


def test_abi_errors_on_gpu(bie):
    c, a, f, q, mu = _random_case(41, 2, 4)
    ctx = bie.bie_create(c, a, 4, mu)
    fd, qd = _dev(f), _dev(q)
    with pytest.raises(bie.BieError) as e:
        bie.bie_apply_SLDL(ctx, fd, qd, fd)           # output aliases input
    assert e.value.status == bie.BIE_ERR_ARG
    from paper_1707_06551_b200 import _abi
    u = torch.empty_like(fd)
    rc = _abi._lib.bie_apply_SLDL(ctx.handle, f.ctypes.data, qd.data_ptr(), u.data_ptr(), None)
    assert rc == bie.BIE_ERR_ARG                      # host pointer where device expected
    rc = _abi._lib.bie_apply_parts(ctx.handle, fd.data_ptr(), qd.data_ptr(), u.data_ptr(), 0, None)
    assert rc == bie.BIE_ERR_ARG
    assert "parts" in bie.bie_last_error(ctx)
    ctx.close()


def test_streams_and_two_contexts(bie, oracle_mod):
    c1, a1, f1, q1, mu1 = _random_case(51, 3, 4)
    c2, a2, f2, q2, mu2 = _random_case(52, 4, 6)
    r1 = oracle_mod.apply(c1, a1, 4, mu1, f1, q1)
    r2 = oracle_mod.apply(c2, a2, 6, mu2, f2, q2)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    k1, k2 = bie.bie_create(c1, a1, 4, mu1), bie.bie_create(c2, a2, 6, mu2)
    u1 = torch.empty((len(f1), 3), dtype=torch.float64, device="cuda")
    u2 = torch.empty((len(f2), 3), dtype=torch.float64, device="cuda")
    F1, Q1, F2, Q2 = _dev(f1), _dev(q1), _dev(f2), _dev(q2)
    torch.cuda.synchronize()
    bie.bie_apply_SLDL(k1, F1, Q1, u1, stream=s1)
    bie.bie_apply_SLDL(k2, F2, Q2, u2, stream=s2)
    torch.cuda.synchronize()
    _assert_parity(u1.cpu().numpy(), r1, "ctx1")
    _assert_parity(u2.cpu().numpy(), r2, "ctx2")
    k1.close()
    k2.close()


def test_smoke_entry(bie):
    import __graft_entry__
    __graft_entry__.smoke()


# ------------------------------------------------------------ edge cases
def test_max_order_full_apply(bie, oracle_mod):
    """p = BIE_P_MAX = 32 (2178 nodes per sphere, several source tiles and a
    ragged target tile) through the whole apply, and the off-surface path."""
    p = bie.BIE_P_MAX
    c, a, f, q, mu = _random_case(1201, 2, p, True, 1.1)
    ref = oracle_mod.apply(c, a, p, mu, f, q)
    _assert_parity(gpu_apply(bie, c, a, p, mu, f, q), ref, "p=32 apply")
    rng = np.random.default_rng(1202)
    tg = rng.uniform(-4, 12, (4000, 3))
    dmin = np.min(np.linalg.norm(tg[:, None] - c[None], axis=-1) - a[None], axis=1)
    tg = tg[np.abs(dmin) > 0.2][:2000]
    uref, pref = oracle_mod.offsurface(c, a, p, mu, f, q, tg)
    ctx = bie.bie_create(c, a, p, mu)
    u = torch.empty((len(tg), 3), dtype=torch.float64, device="cuda")
    pr = torch.empty(len(tg), dtype=torch.float64, device="cuda")
    bie.bie_eval_offsurface(ctx, _dev(f), _dev(q), _dev(tg), u, pr)
    torch.cuda.synchronize()
    ctx.close()
    _assert_parity(u.cpu().numpy(), uref, "p=32 offsurface u")
    _assert_parity(pr.cpu().numpy(), pref, "p=32 offsurface p")


def test_nearly_touching_spheres_and_zero_density(bie, oracle_mod):
    """Gap 1e-3 with two nodes 1e-3 apart across the gap (touching spheres are
    rejected at create, R19): the apply stays finite and matches the oracle;
    zero densities give exactly 0."""
    p = 6
    c = np.array([[0.0, 0.0, 0.0], [1.701, 0.0, 0.0]])
    a = np.array([1.0, 0.7])
    N = 2 * (p + 1) * (2 * p + 2)
    rng = np.random.default_rng(1202)
    f, q = rng.standard_normal((N, 3)), rng.standard_normal((N, 3))
    got = gpu_apply(bie, c, a, p, 1.0, f, q)
    assert np.all(np.isfinite(got))
    _assert_parity(got, oracle_mod.apply(c, a, p, 1.0, f, q), "nearly touching")
    with pytest.raises(bie.BieError) as e:
        bie.bie_create(np.array([[0.0, 0, 0], [1.7, 0, 0]]), a, p, 1.0)
    assert e.value.status == bie.BIE_ERR_GEOMETRY
    z = np.zeros((N, 3))
    assert np.all(gpu_apply(bie, c, a, p, 1.0, z, z) == 0.0)


def test_far_schedules_agree(bie, oracle_mod):
    """cfg 5 (980,000 nodes): the far-field schedules (bie_set_far_reduction:
    1 source chunks + HBM partials + k_reduce, the default; 0 stream-K
    persistent CTAs + fix-up of split tiles; 2 clusters of 8 chunks reduced
    through distributed shared memory) agree to fp64 summation grouping for the apply,
    the off-surface u/p and the K apply, and each is deterministic run to run."""
    d, f, q = _cfg_inputs(oracle_mod, 5)
    ctx = bie.bie_create(d["centres"], d["radii"], d["p"], d["mu"])
    F, Q = _dev(f), _dev(q)
    N = F.shape[0]
    tg = _dev(d["targets"][:600000])
    out = {}
    for mode in (0, 1, 2, 5, 6, 7, 7, 0):
        bie.bie_set_far_reduction(ctx, mode)
        u = torch.empty((N, 3), dtype=torch.float64, device="cuda")
        bie.bie_apply_SLDL(ctx, F, Q, u)
        uo = torch.empty((tg.shape[0], 3), dtype=torch.float64, device="cuda")
        po = torch.empty(tg.shape[0], dtype=torch.float64, device="cuda")
        bie.bie_eval_offsurface(ctx, F, Q, tg, uo, po)
        k = torch.empty_like(u)
        bie.bie_apply_K(ctx, F, k, bie.BIE_PART_FAR | bie.BIE_PART_SELF)
        torch.cuda.synchronize()
        res = [x.cpu().numpy() for x in (u, uo, po, k)]
        if mode in out:
            assert all(np.array_equal(a, b) for a, b in zip(out[mode], res)), "not deterministic"
        out[mode] = res
    ctx.close()
    # 5 (always chained) and 6 (HBM partials + k_reduce): same sums, bit for bit; the
    # default (1) takes the constant-bank batches for the apply and the off-surface
    # sums at this size (same as 7) and the chained schedule for K
    assert all(np.array_equal(a + 0.0, b + 0.0) for a, b in zip(out[5], out[6])), "chained"
    assert all(np.array_equal(a, b) for a, b in zip(out[1][:3], out[7][:3])), "default != constant-bank at cfg 5"
    assert np.array_equal(out[1][3] + 0.0, out[5][3] + 0.0), "K: default != chained"
    for m in (1, 2, 7):  # 7: constant-bank batches (apply and off-surface; K keeps the default)
        for a, b, what in zip(out[0], out[m], ("apply", "offsurface u", "offsurface p", "K")):
            rel, mx = _err(a, b)
            assert rel <= 1e-13 and mx <= 1e-12, (m, what, rel, mx)
    sub = d["subset"][:128]
    _assert_parity(out[0][3][sub], oracle_mod.apply_K(d["centres"], d["radii"], d["p"], f, sub), "K stream-K")


@pytest.mark.parametrize("ns,p", [(1, 3), (2, 1), (3, 4), (7, 6), (40, 5)])
def test_stream_k_small_and_ragged(bie, oracle_mod, ns, p):
    """Stream-K with fewer units than CTAs (empty ranges), tiles split across
    many CTAs, and ragged last tiles: apply and off-surface vs the oracle."""
    c, a, f, q, mu = _random_case(1300 + ns + p, ns, p, True, 1.2)
    ctx = bie.bie_create(c, a, p, mu)
    bie.bie_set_far_reduction(ctx, 0)
    N = bie.bie_num_nodes(ctx)
    ua = torch.empty((N, 3), dtype=torch.float64, device="cuda")
    bie.bie_apply_SLDL(ctx, _dev(f), _dev(q), ua)
    torch.cuda.synchronize()
    _assert_parity(ua.cpu().numpy(), oracle_mod.apply(c, a, p, mu, f, q), f"sk apply {ns}")
    rng = np.random.default_rng(ns)
    tg = rng.uniform(-3, 3 + 4 * ns ** (1 / 3), (3001, 3))
    dmin = np.min(np.linalg.norm(tg[:, None] - c[None], axis=-1) - a[None], axis=1)
    tg = tg[np.abs(dmin) > 0.3]
    uref, pref = oracle_mod.offsurface(c, a, p, mu, f, q, tg)
    u = torch.empty((len(tg), 3), dtype=torch.float64, device="cuda")
    pr = torch.empty(len(tg), dtype=torch.float64, device="cuda")
    bie.bie_eval_offsurface(ctx, _dev(f), _dev(q), _dev(tg), u, pr)
    torch.cuda.synchronize()
    ctx.close()
    _assert_parity(u.cpu().numpy(), uref, "sk off u")
    _assert_parity(pr.cpu().numpy(), pref, "sk off p")


@pytest.mark.parametrize("ns,p,sub", [(1, 3, None), (2, 1, None), (3, 4, None), (7, 6, None), (40, 5, None),
                                      (12, 8, None), (5, 12, None), (7, 6, 100), (40, 5, 700), (12, 8, 1000)])
def test_constant_bank_far_field(bie, oracle_mod, ns, p, sub, monkeypatch):
    """bie_set_far_reduction(7): sources as constant-bank operands in batches of
    312 records over two streams (k_nbody_c.cuh).  Apply (self-sphere exclusion
    in batches that straddle spheres, one batch only, ragged last batch and
    target tile) and off-surface u / p against the oracle; deterministic; a
    second context used in between must not disturb the first (the constant
    buffers are shared by the process).  sub: BIE_CONST_SUB (read by bie_create)
    forces several target sub-ranges per pass on these small cases -- the path
    cfg 4 / 5 take by default -- with ranges that cut through spheres."""
    if sub is not None:
        monkeypatch.setenv("BIE_CONST_SUB", str(sub))
    else:
        monkeypatch.delenv("BIE_CONST_SUB", raising=False)
    c, a, f, q, mu = _random_case(1500 + ns + p, ns, p, True, 1.2)
    ctx = bie.bie_create(c, a, p, mu)
    ctx2 = bie.bie_create(c[:1] + 100.0, a[:1], p, mu)
    bie.bie_set_far_reduction(ctx, 7)
    bie.bie_set_far_reduction(ctx2, 7)
    N = bie.bie_num_nodes(ctx)
    n1 = bie.bie_num_nodes(ctx2)
    F, Q = _dev(f), _dev(q)
    rng = np.random.default_rng(ns + 31)
    tg = rng.uniform(-3, 3 + 4 * ns ** (1 / 3), (3001, 3))
    dmin = np.min(np.linalg.norm(tg[:, None] - c[None], axis=-1) - a[None], axis=1)
    tg = tg[np.abs(dmin) > 0.3]
    s2 = torch.cuda.Stream()
    res = []
    for rep in range(2):
        ua = torch.full((N, 3), np.nan, dtype=torch.float64, device="cuda")
        bie.bie_apply_SLDL(ctx, F, Q, ua)
        with torch.cuda.stream(s2):  # another context, another stream, same constant buffers
            u2 = torch.full((n1, 3), np.nan, dtype=torch.float64, device="cuda")
            bie.bie_apply_SLDL(ctx2, F[:n1].clone(), Q[:n1].clone(), u2)
        u = torch.full((len(tg), 3), np.nan, dtype=torch.float64, device="cuda")
        pr = torch.full((len(tg),), np.nan, dtype=torch.float64, device="cuda")
        bie.bie_eval_offsurface(ctx, F, Q, _dev(tg), u, pr)
        uv = torch.full((len(tg), 3), np.nan, dtype=torch.float64, device="cuda")
        bie.bie_eval_offsurface(ctx, F, Q, _dev(tg), uv, None)
        torch.cuda.synchronize()
        res.append([x.cpu().numpy() for x in (ua, u, pr, uv)])
    ctx.close()
    ctx2.close()
    assert all(np.array_equal(x, y) for x, y in zip(res[0], res[1])), "constant-bank: not deterministic"
    ua, u, pr, uv = res[0]
    assert np.array_equal(u, uv), "velocity depends on the pressure output"
    _assert_parity(ua, oracle_mod.apply(c, a, p, mu, f, q), f"const apply {ns}")
    uref, pref = oracle_mod.offsurface(c, a, p, mu, f, q, tg)
    _assert_parity(u, uref, "const off u")
    _assert_parity(pr, pref, "const off p")


@pytest.mark.parametrize("ns,p,chunks", [(3, 4, 2), (7, 6, 3), (40, 5, 7), (12, 8, 0), (2, 1, 2)])
def test_chained_reduction_matches_k_reduce(bie, oracle_mod, ns, p, chunks):
    """bie_set_far_reduction(5): the chunk partials are summed inside the
    far-field kernel (ticket order, chunk c waits for c - 1 of its tile) in
    k_reduce's fixed order, so every far-field output -- apply (with and without
    near exclusion), K apply, off-surface u / p, off-surface traction -- equals
    schedule 6's (HBM partials + k_reduce) bit for bit, and both match the oracle."""
    c, a, f, q, mu = _random_case(1400 + ns + p, ns, p, True, 1.1)
    ctx = bie.bie_create(c, a, p, mu)
    if chunks:
        bie.bie_set_source_chunks(ctx, chunks)
    N = bie.bie_num_nodes(ctx)
    F, Q = _dev(f), _dev(q)
    rng = np.random.default_rng(ns * 7 + p)
    tg = rng.uniform(-3, 3 + 4 * ns ** (1 / 3), (4099, 3))
    dmin = np.min(np.linalg.norm(tg[:, None] - c[None], axis=-1) - a[None], axis=1)
    tg = tg[np.abs(dmin) > 0.3]
    tn = rng.standard_normal(tg.shape)
    tn /= np.linalg.norm(tn, axis=1, keepdims=True)
    out = {}
    for mode in (6, 5, 5):
        bie.bie_set_far_reduction(ctx, mode)
        res = []
        for excl in (0, 1):
            bie.bie_set_near(ctx, 0.0 if excl == 0 else 0.8)
            bie.bie_set_near_exclusion(ctx, excl)
            u = torch.full((N, 3), np.nan, dtype=torch.float64, device="cuda")
            bie.bie_apply_SLDL(ctx, F, Q, u)
            res.append(u)
        bie.bie_set_near(ctx, 0.0)
        k = torch.full((N, 3), np.nan, dtype=torch.float64, device="cuda")
        bie.bie_apply_K(ctx, F, k, bie.BIE_PART_FAR | bie.BIE_PART_SELF)
        uo = torch.full((len(tg), 3), np.nan, dtype=torch.float64, device="cuda")
        po = torch.full((len(tg),), np.nan, dtype=torch.float64, device="cuda")
        bie.bie_eval_offsurface(ctx, F, Q, _dev(tg), uo, po)
        to = torch.full((len(tg), 3), np.nan, dtype=torch.float64, device="cuda")
        bie.bie_eval_traction(ctx, F, _dev(tg), _dev(tn), to)
        torch.cuda.synchronize()
        res += [k, uo, po, to]
        res = [x.cpu().numpy() for x in res]
        if mode in out:
            assert all(np.array_equal(x, y) for x, y in zip(out[mode], res)), "chained: not deterministic"
        out[mode] = res
    for bad in (-1, 8):
        with pytest.raises(bie.BieError) as e:
            bie.bie_set_far_reduction(ctx, bad)
        assert e.value.status == bie.BIE_ERR_ARG
    ctx.close()
    names = ("apply", "apply near-excluded", "K", "offsurface u", "offsurface p", "traction")
    for x, y, what in zip(out[6], out[5], names):
        assert np.all(np.isfinite(y)), what
        assert np.array_equal(x + 0.0, y + 0.0), f"chained != k_reduce: {what}"
    _assert_parity(out[5][0], oracle_mod.apply(c, a, p, mu, f, q), "chained apply")
    uref, pref = oracle_mod.offsurface(c, a, p, mu, f, q, tg)
    _assert_parity(out[5][3], uref, "chained off u")
    _assert_parity(out[5][4], pref, "chained off p")
