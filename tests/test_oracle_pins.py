"""Pins of the CPU oracle against what the paper and the mathematics fix.

Every test here checks oracle/ against something OTHER than itself: a library
routine (numpy leggauss, scipy sph_harm_y), a textbook value, a closed form
printed in PAPER.md, a classical Stokes-flow identity, brute-force quadrature,
or a basis-free invariant.  Citations: P:n = PAPER.md line, SURVEY = SURVEY.md,
R<k> = reading k in DESIGN.md §3.
"""
import json
import os

import numpy as np
import pytest

from tests import _harmonics as H

GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ------------------------------------------------------------- O-1 GL rule
@pytest.mark.parametrize("p", list(range(1, 33)))
def test_gl_rule_matches_numpy_leggauss(oracle_mod, p):
    t, lam = oracle_mod.gl_rule(p)
    tr, lr = np.polynomial.legendre.leggauss(p + 1)
    assert np.all(np.diff(t) > 0)
    assert np.max(np.abs(t - tr)) <= 4e-16 * 4
    # numpy's own weights are only good to ~1e-13 relative near the ends
    assert np.max(np.abs(lam - lr) / lr) <= 6e-13
    assert abs(lam.sum() - 2.0) <= 1e-14


@pytest.mark.parametrize("p", [4, 12, 24, 31])
def test_gl_rule_matches_mpmath_40_digits(oracle_mod, p):
    """40-digit Newton on P_{p+1} with mpmath (library routine) as the reference."""
    mpmath = pytest.importorskip("mpmath")
    mpmath.mp.dps = 40
    t, lam = oracle_mod.gl_rule(p)
    n = p + 1
    for j in range(n):
        x = mpmath.mpf(float(t[j]))
        for _ in range(8):
            x = x - mpmath.legendre(n, x) / mpmath.diff(lambda z: mpmath.legendre(n, z), x)
        dP = mpmath.diff(lambda z: mpmath.legendre(n, z), x)
        w = 2 / ((1 - x * x) * dP * dP)
        assert abs(t[j] - float(x)) <= 2.3e-16
        assert abs(lam[j] - float(w)) <= 2e-14 * float(w)


def test_gl_rule_textbook_5_point(oracle_mod):
    # Abramowitz & Stegun Table 25.4, n = 5
    t, lam = oracle_mod.gl_rule(4)
    ref_t = np.array([-0.9061798459386640, -0.5384693101056831, 0.0,
                      0.5384693101056831, 0.9061798459386640])
    ref_w = np.array([0.2369268850561891, 0.4786286704993665, 0.5688888888888889,
                      0.4786286704993665, 0.2369268850561891])
    assert np.max(np.abs(t - ref_t)) <= 2e-16 * 2
    assert np.max(np.abs(lam - ref_w)) <= 2e-16 * 2


# ------------------------------------------------------------- O-2 nodes
def test_nodes_weights_normals(oracle_mod):
    c = np.array([[0.5, -1.0, 2.0], [4.0, 0.0, 0.0]])
    a = np.array([1.3, 0.6])
    p = 7
    x, n, w = oracle_mod.nodes(c, a, p)
    ns = (p + 1) * (2 * p + 2)
    assert x.shape == (2 * ns, 3)
    assert np.max(np.abs(np.linalg.norm(n, axis=1) - 1.0)) <= 4e-16
    for s in range(2):
        sl = slice(s * ns, (s + 1) * ns)
        # sum of weights = area 4 pi a^2 (R4: w = a^2 lambda_j 2pi/(2p+2))
        assert abs(w[sl].sum() - 4 * np.pi * a[s] ** 2) <= 1e-14 * 4 * np.pi * a[s] ** 2
        assert np.max(np.abs(x[sl] - (c[s] + a[s] * n[sl]))) <= 1e-15 * 8
    # ordering: j major (t_j ascending), k fastest (phi_k = 2 pi k/(2p+2)), R11
    t, _ = oracle_mod.gl_rule(p)
    nn = n[:ns].reshape(p + 1, 2 * p + 2, 3)
    assert np.allclose(nn[:, 0, 2], t, atol=0)
    ph = np.arctan2(nn[3, :, 1], nn[3, :, 0]) % (2 * np.pi)
    assert np.allclose(ph, 2 * np.pi * np.arange(2 * p + 2) / (2 * p + 2), atol=1e-14)


@pytest.mark.parametrize("p", [4, 8])
def test_discrete_scalar_gram_is_identity(oracle_mod, p):
    """Exactness of the eq 4.2/4.4 rule for products of Y_n^m, n <= p (scipy Y)."""
    _, n, w = oracle_mod.nodes(np.zeros((1, 3)), np.ones(1), p)
    th, ph = H.angles(n)
    B = []
    for l in range(p + 1):
        for m in range(-l, l + 1):
            B.append(H.ylm(l, m, th, ph)[0])
    B = np.array(B)
    G = (B * w) @ B.conj().T
    assert np.max(np.abs(G - np.eye(len(B)))) <= 2e-14


@pytest.mark.parametrize("p", [4, 8])
def test_discrete_vsh_gram(oracle_mod, p):
    """Gram of {V,W,X}_nm under the grid rule = diag((n+1)(2n+1), n(2n+1), n(n+1))."""
    _, n, w = oracle_mod.nodes(np.zeros((1, 3)), np.ones(1), p)
    th, ph = H.angles(n)
    B, d = [], []
    for l in range(p + 1):
        for m in range(-l, l + 1):
            V, W, X = H.vsh(l, m, th, ph)
            for ch, Z, nn in ((0, V, (l + 1) * (2 * l + 1)), (1, W, l * (2 * l + 1)),
                              (2, X, l * (l + 1))):
                if l == 0 and ch > 0:
                    continue
                B.append(Z.reshape(-1))
                d.append(nn)
    B = np.array(B)
    w3 = np.repeat(w, 3)
    G = (B * w3) @ B.conj().T
    assert np.max(np.abs(G - np.diag(d))) <= 1e-12 * max(d)


# ------------------------------------------------------- harmonics vs scipy
@pytest.mark.parametrize("n", [0, 1, 2, 5, 9, 16])
def test_oracle_ylm_matches_scipy(oracle_mod, n):
    rng = np.random.default_rng(n)
    for _ in range(5):
        th, ph = rng.uniform(0.05, np.pi - 0.05), rng.uniform(0, 2 * np.pi)
        for m in range(-n, n + 1):
            Y, dY, dYp = oracle_mod.ylm(n, m, th, ph)
            Yr, dYr, dYpr = H.ylm(n, m, th, ph)
            scale = max(1.0, abs(Yr), abs(dYr), abs(dYpr))
            assert abs(Y - Yr) <= 1e-13 * scale
            assert abs(dY - dYr) <= 1e-13 * scale
            assert abs(dYp - dYpr) <= 1e-13 * scale
            Z = oracle_mod.vsh(n, m, th, ph)
            Zr = np.array(H.vsh(n, m, np.array(th), np.array(ph)))
            assert np.max(np.abs(Z - Zr)) <= 1e-12 * max(1.0, n)


# --------------------------------------------------- O-4 self term, pinned
def _self_single(oracle_mod, p, a, mu, c, dens, kind):
    x, _, _ = oracle_mod.nodes(c[None], np.array([a]), p)
    g = dens(x)
    if kind == "S":
        return x, oracle_mod.self_term(c[None], np.array([a]), p, mu, g, None)
    return x, oracle_mod.self_term(c[None], np.array([a]), p, mu, None, g)


@pytest.mark.parametrize("kind", ["S", "D"])
def test_self_term_single_harmonics_vs_bruteforce_quadrature(oracle_mod, kind):
    """For a band-limited density Re Z_nm (n <= p) the discrete self operator is
    the continuous on-surface operator (S, or D as principal value, R2).  The
    reference is brute-force polar quadrature of the Stokeslet/stresslet
    (eqs 2.19-2.21) about each target: this pins the eigenvalue table (Thm 2
    via eqs 3.6-3.11 at r=1, R3), the VSH projection and the a/mu scaling (R5, R6)."""
    p, a, mu = 5, 1.3, 0.7
    c = np.array([0.3, -0.2, 1.1])
    pick = [0, 17, 33, 51, 70]
    for n in range(0, p + 1):
        for m in range(-n, n + 1):
            for ch in range(3):
                if n == 0 and ch > 0:
                    continue
                dens = lambda y, n=n, m=m, ch=ch: H.vsh_density(n, m, ch, y, c, a)
                x, u = _self_single(oracle_mod, p, a, mu, c, dens, kind)
                for i in pick:
                    ref = H.onsurface_layers(x[i], c, a, mu, dens, kind)
                    scale = max(1e-3, np.abs(dens(x[:1])).max())
                    assert np.max(np.abs(u[i] - ref)) <= 2e-12 * max(1.0, scale), (n, m, ch, i)


def test_self_term_translating_sphere(oracle_mod):
    """Classical Stokes drag: uniform traction f = 3 mu U/(2a) on a sphere gives
    u = U on its surface (S[f] = U), for any a, mu (R5, R6, R16)."""
    p, a, mu = 6, 0.6, 1.7
    c = np.array([1.0, 2.0, -0.5])
    U = np.array([0.3, -1.2, 0.7])
    x, u = _self_single(oracle_mod, p, a, mu, c, lambda y: np.tile(3 * mu * U / (2 * a), (len(y), 1)), "S")
    assert np.max(np.abs(u - U)) <= 1e-14 * 10


def test_self_term_rotating_sphere(oracle_mod):
    """Rigid rotation: traction 3 mu Omega x n gives u = Omega x (x - c) on the sphere."""
    p, a, mu = 6, 1.4, 0.8
    c = np.array([0.2, 0.0, 0.4])
    Om = np.array([0.5, -0.3, 1.1])
    x, u = _self_single(oracle_mod, p, a, mu, c, lambda y: 3 * mu * np.cross(Om, (y - c) / a), "S")
    assert np.max(np.abs(u - np.cross(Om, x - c))) <= 1e-14 * 10


def test_self_term_double_layer_rigid_and_normal(oracle_mod):
    """D_pv of rigid motions = -1/2 of the motion (D = -rigid inside, 0 outside:
    jump +1, A.7 P:662); D_pv[n] = +n/2 (SURVEY §8(c) identities)."""
    p, a = 6, 0.9
    c = np.array([0.0, 1.0, 0.0])
    U = np.array([1.0, -2.0, 0.5])
    Om = np.array([-0.4, 0.9, 0.2])
    x, u = _self_single(oracle_mod, p, a, 1.0, c, lambda y: U + np.cross(Om, y - c), "D")
    assert np.max(np.abs(u + 0.5 * (U + np.cross(Om, x - c)))) <= 1e-14 * 10
    x, u = _self_single(oracle_mod, p, a, 1.0, c, lambda y: (y - c) / a, "D")
    assert np.max(np.abs(u - 0.5 * (x - c) / a)) <= 1e-14 * 10


@pytest.mark.parametrize("p", [4, 6])
def test_self_operator_trace(oracle_mod, p):
    """Basis-free invariant: trace of the discrete self operator = sum_n (2n+1)
    sum_c lambda_c(n) (each projector has rank 2n+1).  SURVEY §8(c) prints
    S: 9.696969696969697 (p=4), 13.784615384615385 (p=6);
    D_pv: -7.196969696969697, -10.284615384615385."""
    ref = {4: (9.696969696969697, -7.196969696969697), 6: (13.784615384615385, -10.284615384615385)}
    ns = (p + 1) * (2 * p + 2)
    c, a = np.zeros((1, 3)), np.ones(1)
    trS = trD = 0.0
    for k in range(ns):
        for comp in range(3):
            e = np.zeros((ns, 3))
            e[k, comp] = 1.0
            idx = np.array([k])
            trS += oracle_mod.self_term(c, a, p, 1.0, e, None, idx)[0, comp]
            trD += oracle_mod.self_term(c, a, p, 1.0, None, e, idx)[0, comp]
    assert abs(trS - ref[p][0]) <= 1e-12
    assert abs(trD - ref[p][1]) <= 1e-12


@pytest.mark.parametrize("p", [4, 8])
def test_self_projection_equals_addition_theorem(oracle_mod, p):
    """O-4 (explicit harmonics) == O-7 (addition theorem) on non-band-limited
    white noise: an internal cross-check (the value pin for white noise is
    test_self_term_on_white_noise_is_the_operator_on_the_R9_interpolant)."""
    rng = np.random.default_rng(p)
    ns = (p + 1) * (2 * p + 2)
    f, q = rng.standard_normal((ns, 3)), rng.standard_normal((ns, 3))
    a, mu = 1.2, 0.9
    u1 = oracle_mod.self_term(np.zeros((1, 3)), np.array([a]), p, mu, f, q)
    u2 = oracle_mod.self_addthm(p, mu, a, f, q)
    assert np.max(np.abs(u1 - u2)) <= 1e-13 * np.abs(u1).max()


# ----------------------------------------- O-3 far field vs closed forms
def _exterior(kind, ch, n, r, Zs):
    """Exterior branches of eqs 3.6-3.8 (S) and 3.9-3.11 (D, sign reading R1),
    PAPER.md P:175-213; Zs = (V, W, X) at the target's angles."""
    V, W, X = Zs
    if kind == "S":
        if ch == 0:
            return n / ((2 * n + 1) * (2 * n + 3)) * V * r ** (-n - 2)
        if ch == 1:
            return ((n + 1) / ((2 * n + 1) * (2 * n - 1)) * W * r ** (-n)
                    + n / (4 * n + 2) * V * (r ** (-n - 2) - r ** (-n)))
        return X * r ** (-n - 1) / (2 * n + 1)
    if ch == 0:
        return (2 * n * n + 4 * n + 3) / ((2 * n + 1) * (2 * n + 3)) * V * r ** (-n - 2)
    if ch == 1:
        return (2 * (n + 1) * (n - 1) / ((2 * n + 1) * (2 * n - 1)) * W * r ** (-n)
                + 2 * n * (n - 1) / (4 * n + 2) * V * (r ** (-n - 2) - r ** (-n)))
    return (n - 1) / (2 * n + 1) * X * r ** (-n - 1)


@pytest.mark.parametrize("kind", ["S", "D"])
def test_far_field_matches_exterior_formulas(oracle_mod, kind):
    """Smooth Nystrom sum (eq 4.4) of density Re Z_nm on sphere 1 evaluated at
    sphere 2's nodes equals the paper's exterior formulas (radius a, viscosity
    mu scaled per R5/R6) to ~1e-13 at p_src = 24."""
    p, a, mu = 24, 1.5, 2.0
    c = np.array([[0.0, 0.0, 0.0], [4.2, 0.3, -0.2]])
    radii = np.array([a, 1.0])
    x, _, _ = oracle_mod.nodes(c, radii, p)
    ns = (p + 1) * (2 * p + 2)
    tg = np.arange(ns, 2 * ns)[::7]
    th, ph = H.angles(x[tg] - c[0])
    r = np.linalg.norm(x[tg] - c[0], axis=1) / a
    for n in range(0, 5):
        for m in range(0, n + 1):
            Zs = [np.real(z) for z in H.vsh(n, m, th, ph)]
            for ch in range(3):
                if n == 0 and ch > 0:
                    continue
                g = np.zeros((2 * ns, 3))
                g[:ns] = H.vsh_density(n, m, ch, x[:ns], c[0], a)
                if kind == "S":
                    u = oracle_mod.far(c, radii, p, mu, g, None, tg)
                    ref = (a / mu) * _exterior("S", ch, n, r[:, None], Zs)
                else:
                    u = oracle_mod.far(c, radii, p, mu, None, g, tg)
                    ref = _exterior("D", ch, n, r[:, None], Zs)
                assert np.max(np.abs(u - ref)) <= 2e-13 * max(1.0, np.abs(g).max()), (n, m, ch)


def test_double_layer_constant_and_rigid_density(oracle_mod):
    """D[U + Omega x (y-c)] = 0 outside and = -(U + Omega x (x-c)) inside
    (F1 sign; jump A.7 P:662), smooth rule at p_src = 24."""
    p = 24
    c = np.array([[0.5, 0.5, 0.5]])
    U = np.array([1.0, -0.5, 2.0])
    Om = np.array([0.3, 0.7, -0.2])
    x, _, _ = oracle_mod.nodes(c, np.ones(1), p)
    q = U + np.cross(Om, x - c[0])
    rng = np.random.default_rng(1)
    dirs = rng.standard_normal((20, 3))
    dirs /= np.linalg.norm(dirs, axis=1)[:, None]
    out = c[0] + dirs * rng.uniform(3.5, 8.0, (20, 1))
    u, _ = oracle_mod.offsurface(c, np.ones(1), p, 1.0, None, q, out)
    assert np.max(np.abs(u)) <= 1e-14 * np.abs(q).max() * 10
    inn = c[0] + dirs * rng.uniform(0.0, 0.5, (20, 1))
    u, _ = oracle_mod.offsurface(c, np.ones(1), p, 1.0, None, q, inn)
    assert np.max(np.abs(u + (U + np.cross(Om, inn - c[0])))) <= 1e-13


# ----------------------------------------------- O-6 pressure / Stokes eqs
def test_translating_sphere_velocity_and_pressure(oracle_mod):
    """Classical Stokes flow past a translating sphere (radius a, viscosity mu):
    uniform traction 3 mu U/(2a) produces, outside,
      u = (3a/4)(U/r + (U.e)e/r) + (a^3/4)(U/r^3 - 3(U.e)e/r^3),
      p = 3 mu a U.(x-c)/(2 r^3)  (= P:189 S[W_1] case, reading R12)."""
    p, a, mu = 24, 1.5, 2.0
    c = np.array([[0.0, 0.2, -0.1]])
    U = np.array([0.4, -1.0, 0.6])
    x, _, _ = oracle_mod.nodes(c, np.array([a]), p)
    f = np.tile(3 * mu * U / (2 * a), (len(x), 1))
    rng = np.random.default_rng(2)
    d = rng.standard_normal((15, 3))
    d /= np.linalg.norm(d, axis=1)[:, None]
    rr = rng.uniform(3.0, 7.0, (15, 1))
    tg = c[0] + d * rr
    u, pr = oracle_mod.offsurface(c, np.array([a]), p, mu, f, None, tg)
    Ue = (d @ U)[:, None]
    uref = 0.75 * a * (U / rr + Ue * d / rr) + 0.25 * a ** 3 * (U / rr ** 3 - 3 * Ue * d / rr ** 3)
    pref = 1.5 * mu * a * (d @ U) / rr[:, 0] ** 2
    assert np.max(np.abs(u - uref)) <= 1e-13
    assert np.max(np.abs(pr - pref)) <= 1e-13


def test_double_layer_pressure_derived_formula(oracle_mod):
    """D[W_n] exterior pressure = 2n(n-1) Y_n r^{-n-1} mu/a (derived
    from Lamb's solution; PAPER P:215 prints a different value, see DESIGN R12)."""
    p, a, mu = 28, 1.5, 2.0
    c = np.zeros((1, 3))
    x, _, _ = oracle_mod.nodes(c, np.array([a]), p)
    rng = np.random.default_rng(3)
    d = rng.standard_normal((10, 3))
    d /= np.linalg.norm(d, axis=1)[:, None]
    rr = rng.uniform(2.5, 5.0, 10)
    tg = d * (a * rr)[:, None]
    th, ph = H.angles(d)
    for n, m in [(1, 0), (2, 1), (3, 2), (4, 0)]:
        q = H.vsh_density(n, m, 1, x, c[0], a)
        _, pr = oracle_mod.offsurface(c, np.array([a]), p, mu, None, q, tg)
        Y = np.real(H.ylm(n, m, th, ph)[0])
        ref = 2 * n * (n - 1) * Y * rr ** (-n - 1) * mu / a
        assert np.max(np.abs(pr - ref)) <= 1e-12, (n, m)


def test_stokes_equations_by_finite_differences(oracle_mod):
    """u and p of the smooth sums satisfy -mu Lap u + grad p = 0 and div u = 0
    (eq 5.1) away from the sources: pins the pressure kernels (R12)
    against the velocity kernels."""
    p, mu = 6, 1.7
    c = np.array([[0.0, 0.0, 0.0], [3.0, 0.5, 0.0]])
    radii = np.array([1.0, 0.7])
    N = 2 * (p + 1) * (2 * p + 2)
    rng = np.random.default_rng(4)
    f, q = rng.standard_normal((N, 3)), rng.standard_normal((N, 3))
    h = 2e-3
    for x0 in (np.array([1.5, 2.0, 1.0]), np.array([-1.0, -1.5, 2.0])):
        offs = [np.zeros(3)]
        for ax in range(3):
            for s in (1, -1):
                e = np.zeros(3)
                e[ax] = s * h
                offs.append(e)
        pts = x0 + np.array(offs)
        u, pr = oracle_mod.offsurface(c, radii, p, mu, f, q, pts)
        lap = sum(u[1 + 2 * ax] + u[2 + 2 * ax] - 2 * u[0] for ax in range(3)) / h ** 2
        gradp = np.array([(pr[1 + 2 * ax] - pr[2 + 2 * ax]) / (2 * h) for ax in range(3)])
        div = sum((u[1 + 2 * ax][ax] - u[2 + 2 * ax][ax]) / (2 * h) for ax in range(3))
        scale = np.abs(gradp).max() + np.abs(mu * lap).max()
        assert np.max(np.abs(-mu * lap + gradp)) <= 1e-5 * scale
        gscale = max(np.abs(u[1 + 2 * ax] - u[2 + 2 * ax]).max() / (2 * h) for ax in range(3))
        assert abs(div) <= 1e-5 * gscale


# ------------------------------------------------ whole-apply invariants
def _small_suspension():
    c = np.array([[0.0, 0.0, 0.0], [2.6, 0.3, -0.4], [0.4, 2.9, 0.8]])
    a = np.array([1.0, 0.6, 1.2])
    return c, a


def test_apply_single_layer_weighted_symmetry(oracle_mod):
    """<g, S f>_w = <S g, f>_w for the whole discrete SL apply (far + self);
    the DL apply is not symmetric (its adjoint is K) -- catches an S/D mix-up."""
    c, a = _small_suspension()
    p, mu = 4, 1.7
    _, _, w = oracle_mod.nodes(c, a, p)
    rng = np.random.default_rng(5)
    N = len(w)
    f, g = rng.standard_normal((N, 3)), rng.standard_normal((N, 3))
    Sf = oracle_mod.apply(c, a, p, mu, f, None)
    Sg = oracle_mod.apply(c, a, p, mu, g, None)
    lhs, rhs = np.sum(w[:, None] * g * Sf), np.sum(w[:, None] * Sg * f)
    assert abs(lhs - rhs) <= 1e-13 * abs(lhs)
    Df = oracle_mod.apply(c, a, p, mu, None, f)
    Dg = oracle_mod.apply(c, a, p, mu, None, g)
    l2, r2 = np.sum(w[:, None] * g * Df), np.sum(w[:, None] * Dg * f)
    assert abs(l2 - r2) > 1e-3 * abs(l2)


def test_apply_translation_permutation_linearity(oracle_mod):
    c, a = _small_suspension()
    p, mu = 4, 1.0
    ns = (p + 1) * (2 * p + 2)
    rng = np.random.default_rng(6)
    N = 3 * ns
    f, q = rng.standard_normal((N, 3)), rng.standard_normal((N, 3))
    u = oracle_mod.apply(c, a, p, mu, f, q)
    ut = oracle_mod.apply(c + np.array([10.0, -3.0, 7.0]), a, p, mu, f, q)
    assert np.max(np.abs(u - ut)) <= 1e-13 * np.abs(u).max()
    perm = [2, 0, 1]
    idx = np.concatenate([np.arange(s * ns, (s + 1) * ns) for s in perm])
    up = oracle_mod.apply(c[perm], a[perm], p, mu, f[idx], q[idx])
    assert np.max(np.abs(up - u[idx])) <= 1e-13 * np.abs(u).max()
    u2 = oracle_mod.apply(c, a, p, mu, 2.0 * f - q, 3.0 * q)
    ref = (2.0 * oracle_mod.apply(c, a, p, mu, f, None) - oracle_mod.apply(c, a, p, mu, q, None)
           + 3.0 * oracle_mod.apply(c, a, p, mu, None, q))
    assert np.max(np.abs(u2 - ref)) <= 1e-13 * np.abs(u2).max()


def test_far_field_spectral_convergence(oracle_mod):
    """Smooth rule on cfg-1 geometry, degree-<=4 density on sphere 1, targets =
    sphere 2's p=4 nodes: error vs p_src=64 decays spectrally."""
    c2 = np.array([[3.0, 0.0, 0.0]])
    tg, _, _ = oracle_mod.nodes(c2, np.ones(1), 4)
    c1 = np.zeros((1, 3))

    def run(ps):
        x, _, _ = oracle_mod.nodes(c1, np.ones(1), ps)
        g = sum(H.vsh_density(n, m, ch, x, c1[0], 1.0)
                for n, m, ch in [(1, 0, 0), (2, 1, 1), (3, -2, 2), (4, 3, 0), (0, 0, 0)])
        return oracle_mod.offsurface(c1, np.ones(1), ps, 1.0, g, g, tg)[0]

    ref = run(64)
    errs = [np.abs(run(ps) - ref).max() / np.abs(ref).max() for ps in (4, 8, 12, 16, 24, 32)]
    assert all(e2 < e1 for e1, e2 in zip(errs, errs[1:]))
    assert errs[-1] <= 1e-13 and errs[0] > 1e-3


# ------------------------------------------------------------ golden values
def test_survey_golden_values_cfg1(oracle_mod):
    """Cross-check of readings against SURVEY.md §8(c) 'Golden values' (printed
    by the survey's independent scratch implementation; not paper values)."""
    from bie_inputs import make_config
    d = make_config(1)
    c, a, f, q = d["centres"], d["radii"], d["f"], d["q"]
    u = oracle_mod.apply(c, a, 4, 1.0, f, q)
    assert abs(np.linalg.norm(u) - 3.426035183702123) <= 1e-13
    assert np.max(np.abs(u[0] - [-0.204571215738744, 0.035540444735914, 0.247436417796310])) <= 1e-14
    assert np.max(np.abs(u[99] - [0.008521366292125, -0.209234690265824, -0.014520019120932])) <= 1e-14
    uS = oracle_mod.apply(c, a, 4, 1.0, f, None)
    uD = oracle_mod.apply(c, a, 4, 1.0, None, q)
    assert abs(np.linalg.norm(uS) - 2.459063961864408) <= 1e-13
    assert abs(np.linalg.norm(uD) - 2.275317771005182) <= 1e-13
    assert abs(np.linalg.norm(oracle_mod.far(c, a, 4, 1.0, f, q)) - 1.005814208180684) <= 1e-13
    assert abs(np.linalg.norm(oracle_mod.self_term(c, a, 4, 1.0, f, q)) - 3.649749358202128) <= 1e-13


def test_committed_golden_fixture(oracle_mod):
    """tests/golden/cfg1_oracle.json was written by tests/golden/make_golden.py
    (calls only oracle/); regression guard for the oracle's arithmetic."""
    from bie_inputs import make_config
    with open(os.path.join(GOLD, "cfg1_oracle.json")) as fh:
        gold = json.load(fh)
    d = make_config(1)
    u = oracle_mod.apply(d["centres"], d["radii"], 4, 1.0, d["f"], d["q"])
    assert np.max(np.abs(u - np.array(gold["u"]))) <= 1e-15 * 4


# ------------------------------------- structure of the self operator (R9)
@pytest.mark.parametrize("p", [3, 5])
def test_self_operator_structure_on_white_noise(oracle_mod, p):
    """For non-band-limited input the paper pins nothing (R9); what the discrete
    projection must still satisfy: the self operator sum_nZ lam Pi_nZ is
    self-adjoint in the quadrature inner product <a,b>_w = sum w a.b (the
    projectors are w-orthogonal), for S and for D_pv separately, and its rank is
    3(p+1)^2 - 2 (W_0 = X_0 = 0; every other mode has a non-zero eigenvalue,
    except V_0 for S whose eigenvalue is 0)."""
    ns = (p + 1) * (2 * p + 2)
    c, a = np.zeros((1, 3)), np.ones(1)
    _, _, w = oracle_mod.nodes(c, a, p)
    MS = np.empty((3 * ns, 3 * ns))
    MD = np.empty((3 * ns, 3 * ns))
    for col in range(3 * ns):
        e = np.zeros((ns, 3))
        e.reshape(-1)[col] = 1.0
        MS[:, col] = oracle_mod.self_term(c, a, p, 1.0, e, None).reshape(-1)
        MD[:, col] = oracle_mod.self_term(c, a, p, 1.0, None, e).reshape(-1)
    W = np.repeat(w, 3)
    for M in (MS, MD):
        A = W[:, None] * M                          # <e_i, M e_j>_w
        assert np.abs(A - A.T).max() <= 1e-14 * np.abs(A).max()
    sv = np.linalg.svd(MD, compute_uv=False)
    assert np.sum(sv > 1e-10 * sv[0]) == 3 * (p + 1) ** 2 - 2
    sv = np.linalg.svd(MS, compute_uv=False)
    assert np.sum(sv > 1e-10 * sv[0]) == 3 * (p + 1) ** 2 - 3   # lamS_V(0) = 0


@pytest.mark.parametrize("p", [3, 5])
def test_self_term_on_white_noise_is_the_operator_on_the_R9_interpolant(oracle_mod, p):
    """Value pin for non-band-limited input.  R9 defines the forward transform
    as the discrete quadrature projection onto VSH of degree <= p; the self term
    must then be the CONTINUOUS on-surface S / D_pv (brute-force polar
    quadrature, independent of the oracle) applied to that band-limited
    interpolant.  The interpolant is built here from scipy's harmonics."""
    from tests import _harmonics as H
    rng = np.random.default_rng(40 + p)
    a, mu = 1.3, 0.8
    c = np.array([0.2, -0.1, 0.4])
    x, _, w = oracle_mod.nodes(c[None], np.array([a]), p)
    wh = w / a ** 2                       # unit-sphere weights (R4)
    g = rng.standard_normal(x.shape)      # white noise at the nodes
    th, ph = H.angles((x - c) / a)
    modes = []
    for n in range(p + 1):
        for m in range(-n, n + 1):
            Z = H.vsh(n, m, th, ph)
            for ch in range(3):
                if n == 0 and ch:
                    continue
                norm2 = np.sum(wh[:, None] * np.abs(Z[ch]) ** 2)
                alpha = np.sum(wh[:, None] * g * np.conj(Z[ch])) / norm2
                modes.append((n, m, ch, alpha))

    def interp(y):
        t2, p2 = H.angles((y - c) / a)
        out = np.zeros(y.shape, dtype=complex)
        for n, m, ch, al in modes:
            out += al * H.vsh(n, m, t2, p2)[ch]
        return np.real(out)

    uS = oracle_mod.self_term(c[None], np.array([a]), p, mu, g, None)
    uD = oracle_mod.self_term(c[None], np.array([a]), p, mu, None, g)
    for i in (0, 7, len(x) // 2, len(x) - 1):
        refS = H.onsurface_layers(x[i], c, a, mu, interp, "S")
        refD = H.onsurface_layers(x[i], c, a, mu, interp, "D")
        assert np.abs(uS[i] - refS).max() <= 1e-11 * np.abs(refS).max(), i
        assert np.abs(uD[i] - refD).max() <= 1e-11 * np.abs(refD).max(), i
