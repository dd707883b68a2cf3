"""Randomised GPU-vs-oracle sweep over the input space: sphere count 1..14,
order p = 1..14, radius spread up to 6x, gaps from 0.05, source chunking,
parts, NULL densities, near-correction eta, and the three operators (apply,
K with completion, off-surface u/p and traction).  Each case is small enough
for the oracle; together they exercise tile tails, chunk planning, masked
tiles, CSR neighbour lists and the staged / unstaged near paths on
geometries nobody hand-picked.  Same bar as every parity test."""
import numpy as np
import pytest

from tests.test_gpu_parity import _assert_parity, _dev

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bie():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1707_06551_b200 as m
    return m


def _geometry(rng):
    ns = int(rng.integers(1, 15))
    radii = rng.uniform(0.3, 1.8, ns)
    min_gap = float(rng.choice([0.05, 0.2, 1.0]))
    side = 3.0 * ns ** (1 / 3) + 4.0
    c = []
    tries = 0
    while len(c) < ns:
        x = rng.uniform(0, side, 3)
        i = len(c)
        tries += 1
        if all(np.linalg.norm(x - y) > radii[i] + radii[j] + min_gap for j, y in enumerate(c)):
            c.append(x)
        if tries > 20000:  # too dense: shrink the remaining radii
            radii[i:] *= 0.8
            tries = 0
    return np.array(c), radii


@pytest.mark.parametrize("seed", range(40))
def test_fuzz_apply_and_near(bie, oracle_mod, seed):
    rng = np.random.default_rng(5000 + seed)
    c, a = _geometry(rng)
    p = int(rng.integers(1, 15))
    mu = float(rng.uniform(0.3, 3.0))
    N = len(a) * (p + 1) * (2 * p + 2)
    f = rng.standard_normal((N, 3)) if rng.uniform() < 0.85 else None
    q = rng.standard_normal((N, 3)) if (f is None or rng.uniform() < 0.85) else None
    parts = int(rng.choice([1, 2, 3, 3, 3]))
    chunks = int(rng.choice([0, 0, 1, 2, 5]))
    eta = float(rng.choice([0.0, 0.0, 0.5, 2.0]))
    ctx = bie.bie_create(c, a, p, mu)
    if chunks:
        bie.bie_set_source_chunks(ctx, chunks)
    if eta > 0:
        bie.bie_set_near(ctx, eta)
    u = torch.full((N, 3), np.nan, dtype=torch.float64, device="cuda")
    bie.bie_apply_parts(ctx, _dev(f), _dev(q), u, parts)
    torch.cuda.synchronize()
    ctx.close()
    sub = np.arange(0, N, max(1, N // 1500))
    ref = np.zeros((len(sub), 3))
    if parts & 1:
        ref += oracle_mod.far(c, a, p, mu, f, q, sub)
        if eta > 0 and len(a) > 1:
            ref += oracle_mod.near(c, a, p, mu, f, q, eta, sub)
    if parts & 2:
        ref += oracle_mod.self_term(c, a, p, mu, f, q, sub)
    got = u.cpu().numpy()[sub]
    if np.abs(ref).max() == 0.0:  # e.g. one sphere, far part only
        assert np.abs(got).max() == 0.0
    else:
        _assert_parity(got, ref, f"seed {seed}: ns={len(a)} p={p} parts={parts} chunks={chunks} eta={eta}")


@pytest.mark.parametrize("seed", range(16))
def test_fuzz_K_completion_offsurface(bie, oracle_mod, seed):
    rng = np.random.default_rng(7000 + seed)
    c, a = _geometry(rng)
    p = int(rng.integers(1, 13))
    mu = float(rng.uniform(0.3, 3.0))
    N = len(a) * (p + 1) * (2 * p + 2)
    sig = rng.standard_normal((N, 3))
    eta = float(rng.choice([0.0, 1.0]))
    ctx = bie.bie_create(c, a, p, mu)
    if eta > 0:
        bie.bie_set_near(ctx, eta)
    # K + completion at the nodes
    u = torch.full((N, 3), np.nan, dtype=torch.float64, device="cuda")
    bie.bie_apply_K(ctx, _dev(sig), u, 7)
    # off-surface velocity/pressure and traction at random points
    m = int(rng.integers(1, 700))
    lo, hi = c.min(0) - 2.0, c.max(0) + 2.0
    tg = lo + (hi - lo) * rng.uniform(size=(m, 3))
    nv = rng.standard_normal((m, 3))
    nv /= np.linalg.norm(nv, axis=1)[:, None]
    uo = torch.empty((m, 3), dtype=torch.float64, device="cuda")
    po = torch.empty(m, dtype=torch.float64, device="cuda")
    to = torch.empty((m, 3), dtype=torch.float64, device="cuda")
    bie.bie_eval_offsurface(ctx, _dev(sig), _dev(sig), _dev(tg), uo, po)
    bie.bie_eval_traction(ctx, _dev(sig), _dev(tg), _dev(nv), to)
    torch.cuda.synchronize()
    ctx.close()
    sub = np.arange(0, N, max(1, N // 1000))
    refK = oracle_mod.apply_K(c, a, p, sig, sub) + oracle_mod.completion(c, a, p, sig)[sub]
    if eta > 0 and len(a) > 1:
        refK += oracle_mod.near_K(c, a, p, sig, eta, sub)
    _assert_parity(u.cpu().numpy()[sub], refK, f"K seed {seed}")
    if eta > 0:
        ru, rp = oracle_mod.offsurface_near(c, a, p, mu, sig, sig, eta, tg)
    else:
        ru, rp = oracle_mod.offsurface(c, a, p, mu, sig, sig, tg)
    _assert_parity(uo.cpu().numpy(), ru, f"offsurface u seed {seed}")
    _assert_parity(po.cpu().numpy(), rp, f"offsurface p seed {seed}")
    rt = oracle_mod.traction_offsurface(c, a, p, sig, tg, nv, eta)
    _assert_parity(to.cpu().numpy(), rt, f"traction seed {seed}")
