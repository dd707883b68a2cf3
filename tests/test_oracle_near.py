"""Pins of the NEXT-1 oracle (near-singular correction, PAPER §4.1 P:330-344,
§4.3): exact exterior evaluation of a sphere's VSH expansion (eqs
3.6-3.11 with sign reading R1, eq 4.7) and the eq 4.5 partition, checked
against classical Stokes solutions and brute-force high-order quadrature."""
import numpy as np
import pytest

from tests import _harmonics as H


def _dirs(seed, n):
    d = np.random.default_rng(seed).standard_normal((n, 3))
    return d / np.linalg.norm(d, axis=1)[:, None]


def test_exterior_eval_translating_sphere_close_range(oracle_mod):
    """S[3 mu U/(2a)] outside = classical Stokes flow of a translating sphere,
    down to r = 1.01 a where the smooth rule is useless."""
    p, a, mu = 8, 1.3, 1.7
    c = np.array([0.2, -0.1, 0.4])
    U = np.array([0.3, -1.0, 0.5])
    x, _, _ = oracle_mod.nodes(c[None], np.array([a]), p)
    f = np.tile(3 * mu * U / (2 * a), (len(x), 1))
    d = _dirs(0, 12)
    rr = np.random.default_rng(1).uniform(1.01, 1.3, (12, 1)) * a
    u = oracle_mod.exterior_eval(p, c, a, mu, f, None, c + d * rr)
    Ue = (d @ U)[:, None]
    ref = 0.75 * a * (U / rr + Ue * d / rr) + 0.25 * a ** 3 * (U / rr ** 3 - 3 * Ue * d / rr ** 3)
    assert np.abs(u - ref).max() <= 1e-14


def test_exterior_eval_double_layer_rigid_is_zero(oracle_mod):
    p, a = 8, 0.8
    c = np.array([1.0, 0.0, -1.0])
    x, _, _ = oracle_mod.nodes(c[None], np.array([a]), p)
    q = np.array([0.4, -0.2, 1.0]) + np.cross(np.array([0.3, 0.5, -0.6]), x - c)
    tg = c + _dirs(2, 12) * a * 1.02
    assert np.abs(oracle_mod.exterior_eval(p, c, a, 1.0, None, q, tg)).max() <= 1e-14


@pytest.mark.parametrize("gap", [1.0, 0.5, 0.3])
def test_exterior_eval_matches_bruteforce_quadrature(oracle_mod, gap):
    """Band-limited density (n <= 5 < p): spectral evaluation == smooth rule with
    p_src = 96 (converged at these distances)."""
    p, a, mu = 8, 1.3, 1.7
    c = np.array([0.2, -0.1, 0.4])

    def dens(y):
        return sum(H.vsh_density(n, m, ch, y, c, a)
                   for n, m, ch in [(1, 0, 0), (2, 1, 1), (3, -2, 2), (4, 3, 0), (5, 2, 1), (0, 0, 0)])

    x, _, _ = oracle_mod.nodes(c[None], np.array([a]), p)
    tg = c + _dirs(3, 10) * (a + gap)
    ue = oracle_mod.exterior_eval(p, c, a, mu, dens(x), dens(x), tg)
    xs, _, _ = oracle_mod.nodes(c[None], np.array([a]), 96)
    ub, _ = oracle_mod.offsurface(c[None], np.array([a]), 96, mu, dens(xs), dens(xs), tg)
    assert np.abs(ub - ue).max() <= 1e-13 * np.abs(ue).max()


def test_well_separation_eq_4_5(oracle_mod):
    # SPEC.md examples: unit spheres 6 apart (dist 4 >= 2): separated; 3 apart: near;
    # equality counts as separated.
    z = np.zeros(3)
    assert not oracle_mod.is_near(z, 1.0, [6.0, 0, 0], 1.0, 1.0)
    assert oracle_mod.is_near(z, 1.0, [3.0, 0, 0], 1.0, 1.0)
    assert not oracle_mod.is_near(z, 1.0, [4.0, 0, 0], 1.0, 1.0)
    assert oracle_mod.is_near(z, 1.0, [3.999, 0, 0], 1.0, 1.0)
    # the larger diameter counts (polydisperse): dist = 3 - 0.5 - 1 = 1.5, max diam = 2
    assert oracle_mod.is_near(z, 0.5, [3.0, 0, 0], 1.0, 0.8)       # 1.5 < 1.6
    assert not oracle_mod.is_near(z, 0.5, [3.0, 0, 0], 1.0, 0.7)   # 1.5 >= 1.4


def _two_spheres(gap, p):
    d = np.array([1.0, 0.13, -0.087])
    c = np.array([[0.0, 0.0, 0.0], (2.0 + gap) * d / np.linalg.norm(d)])
    a = np.ones(2)
    return c, a


def test_near_correction_recovers_the_integral(oracle_mod):
    """Two unit spheres with gap 0.3 (near for eta = 1).  Band-limited density on
    sphere 0 only: smooth sum + near correction at sphere 1's nodes equals the
    converged (p_src = 96) quadrature of sphere 0's density, while the plain
    smooth sum at p = 8 is off by orders of magnitude more."""
    p, mu, gap = 8, 1.0, 0.3
    c, a = _two_spheres(gap, p)
    ns = (p + 1) * (2 * p + 2)
    x, _, _ = oracle_mod.nodes(c, a, p)
    g = np.zeros((2 * ns, 3))
    g[:ns] = sum(H.vsh_density(n, m, ch, x[:ns], c[0], 1.0)
                 for n, m, ch in [(1, 0, 0), (2, 1, 1), (3, -2, 2), (4, 3, 0)])
    tg = np.arange(ns, 2 * ns)
    smooth = oracle_mod.far(c, a, p, mu, g, g, tg)
    corr = smooth + oracle_mod.near(c, a, p, mu, g, g, 1.0, tg)
    xs, _, _ = oracle_mod.nodes(c[:1], a[:1], 96)
    gs = sum(H.vsh_density(n, m, ch, xs, c[0], 1.0)
             for n, m, ch in [(1, 0, 0), (2, 1, 1), (3, -2, 2), (4, 3, 0)])
    ref, _ = oracle_mod.offsurface(c[:1], a[:1], 96, mu, gs, gs, x[tg])
    e_corr = np.abs(corr - ref).max() / np.abs(ref).max()
    e_smooth = np.abs(smooth - ref).max() / np.abs(ref).max()
    assert e_corr <= 1e-13
    assert e_smooth >= 1e-4


def test_near_correction_off_when_well_separated(oracle_mod):
    p = 5
    c, a = _two_spheres(0.3, p)
    N = 2 * (p + 1) * (2 * p + 2)
    rng = np.random.default_rng(9)
    f, q = rng.standard_normal((N, 3)), rng.standard_normal((N, 3))
    assert np.all(oracle_mod.near(c, a, p, 1.0, f, q, 0.0) == 0.0)   # eta = 0: nothing is near
    assert np.all(oracle_mod.near(c, a, p, 1.0, f, q, 0.14) == 0.0)  # 0.3 >= 0.14 * 2
    assert np.any(oracle_mod.near(c, a, p, 1.0, f, q, 0.16) != 0.0)


def test_near_corrected_apply_rigid_modes(oracle_mod):
    """Translating sphere 0 (S[3 mu U/2a]) next to sphere 1 (gap 0.2): with the
    correction, the field on sphere 1 is the classical Stokes flow."""
    p, mu = 8, 1.3
    c, a = _two_spheres(0.2, p)
    ns = (p + 1) * (2 * p + 2)
    x, _, _ = oracle_mod.nodes(c, a, p)
    U = np.array([0.5, -0.3, 0.8])
    f = np.zeros((2 * ns, 3))
    f[:ns] = 3 * mu * U / 2
    tg = np.arange(ns, 2 * ns)
    u = oracle_mod.apply_near(c, a, p, mu, f, None, 1.0, tg)
    dv = x[tg] - c[0]
    rr = np.linalg.norm(dv, axis=1)[:, None]
    d = dv / rr
    Ue = (d @ U)[:, None]
    ref = 0.75 * (U / rr + Ue * d / rr) + 0.25 * (U / rr ** 3 - 3 * Ue * d / rr ** 3)
    assert np.abs(u - ref).max() <= 1e-13


# ------------------------------------------------- off-surface targets (a7)
def test_exterior_pressure_translating_sphere(oracle_mod):
    """p = 3 mu a U.(x-c)/(2 r^3) outside a translating sphere (classical; P:189
    S[W_1] case) down to r = 1.01 a."""
    p, a, mu = 8, 1.3, 1.7
    c = np.array([0.2, -0.1, 0.4])
    U = np.array([0.3, -1.0, 0.5])
    x, _, _ = oracle_mod.nodes(c[None], np.array([a]), p)
    f = np.tile(3 * mu * U / (2 * a), (len(x), 1))
    d = _dirs(6, 12)
    rr = np.random.default_rng(7).uniform(1.01, 1.3, 12) * a
    pr = oracle_mod.exterior_pressure(p, c, a, mu, f, None, c + d * rr[:, None])
    assert np.abs(pr - 1.5 * mu * a * (d @ U) / rr ** 2).max() <= 1e-13


@pytest.mark.parametrize("gap", [0.5, 0.3])
def test_exterior_pressure_matches_bruteforce(oracle_mod, gap):
    """Band-limited S and D densities: spectral exterior pressure == converged
    (p_src = 96) smooth-rule pressure (whose kernels are pinned by the Stokes
    equations in test_oracle_pins.py)."""
    p, a, mu = 8, 1.3, 1.7
    c = np.array([0.2, -0.1, 0.4])

    def dens(y):
        return sum(H.vsh_density(n, m, ch, y, c, a)
                   for n, m, ch in [(1, 0, 1), (2, 1, 1), (3, -2, 1), (4, 3, 0), (2, 0, 2), (5, 2, 1)])

    x, _, _ = oracle_mod.nodes(c[None], np.array([a]), p)
    tg = c + _dirs(8, 10) * (a + gap)
    pe = oracle_mod.exterior_pressure(p, c, a, mu, dens(x), dens(x), tg)
    xs, _, _ = oracle_mod.nodes(c[None], np.array([a]), 96)
    _, pb = oracle_mod.offsurface(c[None], np.array([a]), 96, mu, dens(xs), dens(xs), tg)
    assert np.abs(pb - pe).max() <= 1e-13 * np.abs(pe).max()


def test_offsurface_near_correction_recovers_integral(oracle_mod):
    """Targets 0.1-0.6 from sphere 0's surface, band-limited densities on two
    spheres: smooth sum + near correction == converged quadrature, for u and p
    (eta = 5 so that sphere 1 is corrected too: at p = 8 the smooth rule alone
    is only ~1e-9 accurate even two radii away); the plain smooth sum is far off."""
    p, mu = 8, 1.2
    c = np.array([[0.0, 0.0, 0.0], [3.5, 0.4, -0.3]])
    a = np.array([1.0, 0.8])
    x, _, _ = oracle_mod.nodes(c, a, p)
    ns = (p + 1) * (2 * p + 2)
    mods = [(1, 0, 0), (2, 1, 1), (3, -2, 2), (4, 3, 1)]
    g = np.zeros((2 * ns, 3))
    g[:ns] = sum(H.vsh_density(n, m, ch, x[:ns], c[0], a[0]) for n, m, ch in mods)
    g[ns:] = sum(H.vsh_density(n, m, ch, x[ns:], c[1], a[1]) for n, m, ch in mods[:2])
    d = _dirs(9, 16)
    tg = c[0] + d * (1.0 + np.random.default_rng(10).uniform(0.1, 0.6, (16, 1)))
    u, pr = oracle_mod.offsurface_near(c, a, p, mu, g, g, 5.0, tg)
    u0, p0 = oracle_mod.offsurface(c, a, p, mu, g, g, tg)
    xs, _, _ = oracle_mod.nodes(c, a, 160)   # p_src = 96 is still 3e-12 off at gap 0.1
    nb = 161 * 322
    gs = np.zeros((2 * nb, 3))
    gs[:nb] = sum(H.vsh_density(n, m, ch, xs[:nb], c[0], a[0]) for n, m, ch in mods)
    gs[nb:] = sum(H.vsh_density(n, m, ch, xs[nb:], c[1], a[1]) for n, m, ch in mods[:2])
    ur, prr = oracle_mod.offsurface(c, a, 160, mu, gs, gs, tg)
    assert np.abs(u - ur).max() <= 1e-13 * np.abs(ur).max()
    assert np.abs(pr - prr).max() <= 1e-13 * np.abs(prr).max()
    assert np.abs(u0 - ur).max() >= 1e-4 * np.abs(ur).max()
