"""GPU parity of NEXT-4 (PAPER §4.2, Fig 2: rotated, pole-aligned near
evaluation with coefficient accumulation; bie_set_near_mode(ctx, 1)) against
the oracle's stage-by-stage evaluation (oracle.apply_near4 = far + self +
near4), same bar as the apply: rel-L2 <= 1e-12 and max-norm <= 1e-10.  Plus
checks that hold without the oracle: agreement with the direct NEXT-1
evaluation where the neighbour's field is (numerically) band-limited, the
rigid-body identity, and argument validation."""
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


def gpu_apply_mode(bie, c, a, p, mu, f, q, eta, mode, parts=3, variant=0, excl=-1):
    ctx = bie.bie_create(c, a, p, mu)
    bie.bie_set_self_kernel(ctx, variant)
    bie.bie_set_near(ctx, eta)
    bie.bie_set_near_exclusion(ctx, excl)
    bie.bie_set_near_mode(ctx, mode)
    N = len(a) * (p + 1) * (2 * p + 2)
    u = torch.full((N, 3), np.nan, dtype=torch.float64, device="cuda")
    bie.bie_apply_parts(ctx, _dev(f), _dev(q), u, parts)
    torch.cuda.synchronize()
    ctx.close()
    return u.cpu().numpy()


def test_next4_two_spheres_oblique(bie, oracle_mod):
    p, mu = 7, 1.3
    d = np.array([0.7, -0.45, 0.55])
    c = np.array([[0.1, 0.0, -0.2], [0.1, 0.0, -0.2] + 2.4 * d / np.linalg.norm(d)])
    a = np.array([1.0, 0.9])
    rng = np.random.default_rng(41)
    N = 2 * (p + 1) * (2 * p + 2)
    f, q = rng.standard_normal((N, 3)), rng.standard_normal((N, 3))
    got = gpu_apply_mode(bie, c, a, p, mu, f, q, 1.0, 1)
    _assert_parity(got, oracle_mod.apply_near4(c, a, p, mu, f, q, 1.0), "next4 2 spheres")


@pytest.mark.parametrize("p,ns,eta,variant,excl", [(4, 5, 1.0, 0, 1), (6, 6, 1.0, 0, 0), (5, 5, 2.0, 1, 1),
                                                   (8, 4, 1.0, 2, 0), (9, 3, 1.5, 0, 1), (12, 3, 1.0, 0, 0)])
def test_next4_random_suspensions(bie, oracle_mod, p, ns, eta, variant, excl):
    """Polydisperse random suspensions; self-kernel variants 0/1 (k_sht) and 2
    (round-1 kernel: the NEXT-4 coefficient pass then runs on k_sht); the near
    pairs' smooth rule subtracted (excl 0) or skipped in the far field (1)."""
    c, a, f, q, mu = _random_case(500 + p + ns, ns, p, True, 0.9)
    got = gpu_apply_mode(bie, c, a, p, mu, f, q, eta, 1, variant=variant, excl=excl)
    _assert_parity(got, oracle_mod.apply_near4(c, a, p, mu, f, q, eta), f"next4 p={p} eta={eta}")


@pytest.mark.parametrize("p", [16, 24, 32])
def test_next4_high_order(bie, oracle_mod, p):
    """High orders (the regime where NEXT-4 pays): three spheres with
    oblique pair axes, sampled target nodes of every sphere vs the oracle."""
    c = np.array([[0.0, 0.0, 0.0], [2.45, 0.31, -0.4], [-0.6, 2.2, 0.9]])
    a = np.array([1.0, 0.9, 1.1])
    nsn = (p + 1) * (2 * p + 2)
    rng = np.random.default_rng(p + 7)
    f, q = rng.standard_normal((3 * nsn, 3)), rng.standard_normal((3 * nsn, 3))
    got = gpu_apply_mode(bie, c, a, p, 1.1, f, q, 1.0, 1)
    sub = np.arange(0, 3 * nsn, 53)
    _assert_parity(got[sub], oracle_mod.apply_near4(c, a, p, 1.1, f, q, 1.0, sub), f"next4 p={p}")


def test_next4_parts_and_single_densities(bie, oracle_mod):
    """FAR only (= far + near4 correction), SELF only (unchanged), S only, D only."""
    p, eta = 6, 1.0
    c, a, f, q, mu = _random_case(77, 5, p, True, 1.1)
    far = gpu_apply_mode(bie, c, a, p, mu, f, q, eta, 1, parts=bie.BIE_PART_FAR)
    ref = oracle_mod.far(c, a, p, mu, f, q) + oracle_mod.near4(c, a, p, mu, f, q, eta)
    _assert_parity(far, ref, "next4 far only")
    slf = gpu_apply_mode(bie, c, a, p, mu, f, q, eta, 1, parts=bie.BIE_PART_SELF)
    _assert_parity(slf, oracle_mod.self_term(c, a, p, mu, f, q), "next4 self only")
    z = np.zeros_like(f)
    _assert_parity(gpu_apply_mode(bie, c, a, p, mu, f, z, eta, 1),
                   oracle_mod.apply_near4(c, a, p, mu, f, z, eta), "next4 S")
    _assert_parity(gpu_apply_mode(bie, c, a, p, mu, z, q, eta, 1),
                   oracle_mod.apply_near4(c, a, p, mu, z, q, eta), "next4 D")


def test_next4_lattice_with_axis_aligned_neighbours(bie, oracle_mod):
    """Jittered-free cubic lattice (cfg 4's geometry, small): every pair axis is
    a coordinate axis, and at even p target nodes lie exactly on it -- the
    rotated pipeline works in coefficient space, so this is regular."""
    p, eta = 8, 1.0
    g = np.arange(2) * 3.0
    c = np.array([[x, y, z] for x in g for y in g for z in g])
    a = np.ones(len(c))
    rng = np.random.default_rng(8)
    N = len(c) * (p + 1) * (2 * p + 2)
    f, q = rng.standard_normal((N, 3)), rng.standard_normal((N, 3))
    got = gpu_apply_mode(bie, c, a, p, 1.0, f, q, eta, 1)
    nsn = (p + 1) * (2 * p + 2)
    sub = np.concatenate([np.arange(0, nsn), np.arange(5 * nsn, 6 * nsn)])
    ref = oracle_mod.apply_near4(c, a, p, 1.0, f, q, eta, sub)
    _assert_parity(got[sub], ref, "next4 lattice")


def test_next4_converges_to_direct(bie):
    """Both modes evaluate the same exact near field, NEXT-4 through its
    degree-p re-expansion on the target sphere: the difference shrinks
    spectrally with p (two spheres at gap 2 -- rate ~ 1/3 per degree -- smooth
    band-limited densities, eta = 1.5 so that the pair is near)."""
    d = np.array([0.6, 0.3, -0.74])
    c = np.array([[0.0, 0.0, 0.0], 4.0 * d / np.linalg.norm(d)])
    a = np.ones(2)
    diffs = []
    for p in (6, 10, 14, 20):
        nsn = (p + 1) * (2 * p + 2)
        ctx = bie.bie_create(c, a, p, 1.0)
        x = torch.empty((2 * nsn, 3), dtype=torch.float64, device="cuda")
        bie.bie_get_nodes(ctx, x)
        ctx.close()
        xs = x.cpu().numpy() - np.repeat(c, nsn, 0)
        f = np.stack([xs[:, 1] * xs[:, 2], xs[:, 0] ** 2 - 0.3, xs[:, 1]], 1)  # degree <= 2
        q = np.stack([xs[:, 2], xs[:, 0] * xs[:, 1], 1.0 - xs[:, 2] ** 2], 1)
        u0 = gpu_apply_mode(bie, c, a, p, 1.0, f, q, 1.5, 0)
        u1 = gpu_apply_mode(bie, c, a, p, 1.0, f, q, 1.5, 1)
        diffs.append(np.abs(u1 - u0).max() / np.abs(u0).max())
    assert all(b < a_ for a_, b in zip(diffs, diffs[1:])), diffs
    assert diffs[-1] < 1e-8, diffs


def test_next4_rigid_density_matches_direct(bie):
    """D of a rigid-body density vanishes outside its sphere (App. B check 10):
    the exact near field is 0 in both modes, so they agree to rounding."""
    p, eta = 6, 2.0
    c, a, _, _, mu = _random_case(91, 5, p, True, 1.0)
    nsn = (p + 1) * (2 * p + 2)
    ctx = bie.bie_create(c, a, p, mu)
    x = torch.empty((len(a) * nsn, 3), dtype=torch.float64, device="cuda")
    bie.bie_get_nodes(ctx, x)
    ctx.close()
    x = x.cpu().numpy()
    rng = np.random.default_rng(92)
    q = np.empty_like(x)
    for s in range(len(a)):
        U, W = rng.standard_normal(3), rng.standard_normal(3)
        q[s * nsn:(s + 1) * nsn] = U + np.cross(W, x[s * nsn:(s + 1) * nsn] - c[s])
    z = np.zeros_like(q)
    u0 = gpu_apply_mode(bie, c, a, p, mu, z, q, eta, 0)
    u1 = gpu_apply_mode(bie, c, a, p, mu, z, q, eta, 1)
    assert np.abs(u1 - u0).max() <= 1e-13 * np.abs(u0).max()


def test_next4_mode_validation(bie):
    c, a, f, q, mu = _random_case(93, 2, 4, True, 1.0)
    ctx = bie.bie_create(c, a, 4, mu)
    for bad in (-1, 4):
        with pytest.raises(bie.BieError) as e:
            bie.bie_set_near_mode(ctx, bad)
        assert e.value.status == bie.BIE_ERR_ARG
    bie.bie_set_near_mode(ctx, 1)
    bie.bie_set_near_mode(ctx, 0)
    ctx.close()
