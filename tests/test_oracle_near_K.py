"""Pins of the NEXT-3 near correction for K: the traction of one
sphere's exterior single-layer expansion (eqs 3.17-3.18, reading R24) and the
corrected apply.  Pinned against (a) the paper's closed forms eqs 3.19-3.21,
(b) brute-force fine-grid quadrature of the K kernel for band-limited
densities (an independent route to the same integral), (c) finite
differences of the pinned exterior velocity/pressure (NEXT-1), and (d) a
two-sphere case where smooth + correction reproduces the converged integral."""
import numpy as np
import pytest

from tests import _harmonics as H
from tests.test_oracle_traction import _K_closed_form


def _bandlimited(seed, p, pts, c, a):
    rng = np.random.default_rng(seed)
    out = np.zeros_like(pts)
    for n in range(0, p + 1):
        for m in range(-n, n + 1):
            for ch in range(3):
                if n == 0 and ch:
                    continue
                out += rng.standard_normal() * H.vsh_density(n, m, ch, pts, c, a)
    return out


def test_exterior_traction_closed_forms(oracle_mod):
    """Unit sphere, normal e_r: eqs 3.19-3.21 exterior branches, n <= 5, all channels."""
    p = 6
    c = np.zeros(3)
    x, _, _ = oracle_mod.nodes(c[None], np.ones(1), p)
    rng = np.random.default_rng(3)
    for n in range(1, 6):
        for m in sorted({0, 1, n, -n}):
            for ch in range(3):
                sig = H.vsh_density(n, m, ch, x, c, 1.0)
                th, ph = rng.uniform(0.2, 2.9, 3), rng.uniform(-3.0, 3.0, 3)
                for r in (1.05, 1.4, 3.0):
                    er = np.stack([np.sin(th) * np.cos(ph), np.sin(th) * np.sin(ph), np.cos(th)], 1)
                    t = oracle_mod.exterior_traction(p, c, 1.0, sig, r * er, er)
                    for i in range(3):
                        ref = _K_closed_form(n, m, ch, r, th[i], ph[i])
                        assert np.abs(t[i] - ref).max() <= 1e-13, (n, m, ch, r)


@pytest.mark.parametrize("gap,P", [(2.0, 48), (1.0, 48), (0.5, 64), (0.3, 128)])
def test_exterior_traction_vs_fine_quadrature(oracle_mod, gap, P):
    """Random band-limited density (degree <= 6) on a sphere of radius 1.3:
    exterior_traction at p = 6 == the K kernel summed on a fine p = P grid
    (sigma evaluated exactly there), random points and unit normals."""
    p, a = 6, 1.3
    c = np.array([0.2, -0.1, 0.3])
    xs, _, _ = oracle_mod.nodes(c[None], np.array([a]), p)
    xf, _, _ = oracle_mod.nodes(c[None], np.array([a]), P)
    sig, sigf = _bandlimited(7, p, xs, c, a), _bandlimited(7, p, xf, c, a)
    rng = np.random.default_rng(8)
    d = rng.standard_normal((5, 3))
    d /= np.linalg.norm(d, axis=1)[:, None]
    nv = rng.standard_normal((5, 3))
    nv /= np.linalg.norm(nv, axis=1)[:, None]
    pts = c + (a + gap) * d
    t = oracle_mod.exterior_traction(p, c, a, sig, pts, nv)
    k = oracle_mod.K_at(c[None], np.array([a]), P, sigf, pts, nv)
    assert np.abs(t - k).max() <= 1e-12 * np.abs(k).max()


def test_exterior_traction_vs_finite_differences_near_surface(oracle_mod):
    """At 1.02 a .. 1.2 a, where no quadrature converges: traction == -p n +
    mu (grad u + grad u^T) n of the exterior velocity / pressure (eqs 3.6-3.8,
    P:189; pinned in test_oracle_near.py), central differences h = 1e-4 a."""
    p, a, mu = 5, 0.8, 1.9
    c = np.array([1.0, 0.5, -0.2])
    xs, _, _ = oracle_mod.nodes(c[None], np.array([a]), p)
    sig = _bandlimited(9, p, xs, c, a)
    rng = np.random.default_rng(10)
    for rr in (1.02, 1.07, 1.2):
        d = rng.standard_normal(3)
        d /= np.linalg.norm(d)
        nv = rng.standard_normal(3)
        nv /= np.linalg.norm(nv)
        x0 = c + rr * a * d
        h = 1e-4 * a
        G = np.zeros((3, 3))
        for ax in range(3):
            e = np.zeros(3)
            e[ax] = h
            up = oracle_mod.exterior_eval(p, c, a, mu, sig, None, (x0 + e)[None])[0]
            um = oracle_mod.exterior_eval(p, c, a, mu, sig, None, (x0 - e)[None])[0]
            G[:, ax] = (up - um) / (2 * h)
        pr = oracle_mod.exterior_pressure(p, c, a, mu, sig, None, x0[None])[0]
        ref = -pr * nv + mu * (G + G.T) @ nv
        t = oracle_mod.exterior_traction(p, c, a, sig, x0[None], nv[None])[0]
        assert np.abs(t - ref).max() <= 1e-7 * np.abs(ref).max(), (rr, t, ref)


def test_near_K_two_spheres_reproduces_converged_integral(oracle_mod):
    """Two spheres at gap 0.45: K_pv at sphere 0's nodes from sphere 1's
    band-limited density.  Smooth rule alone is >= 1e-5 off the converged
    integral (p = 128 fine grid); smooth + near correction matches to 1e-12."""
    p = 6
    c = np.array([[0.0, 0.0, 0.0], [2.25, 0.4, -0.3]])
    a = np.array([1.0, 0.8])
    c[1] *= (1.0 + 0.8 + 0.45) / np.linalg.norm(c[1])
    x, nrm, _ = oracle_mod.nodes(c, a, p)
    nsn = (p + 1) * (2 * p + 2)
    sig = np.zeros_like(x)
    sig[nsn:] = _bandlimited(11, p, x[nsn:], c[1], a[1])
    sub = np.arange(0, nsn, 3)
    smooth = oracle_mod.far_K(c, a, p, sig, sub)
    corr = smooth + oracle_mod.near_K(c, a, p, sig, 1.0, sub)
    xf, _, _ = oracle_mod.nodes(c[1:], a[1:], 128)
    sigf = _bandlimited(11, p, xf, c[1], a[1])
    ref = oracle_mod.K_at(c[1:], a[1:], 128, sigf, x[sub], nrm[sub])
    scale = np.abs(ref).max()
    assert np.abs(smooth - ref).max() >= 1e-5 * scale
    assert np.abs(corr - ref).max() <= 1e-12 * scale
    # eta too small to flag the pair: no correction
    assert np.abs(oracle_mod.near_K(c, a, p, sig, 0.1, sub)).max() == 0.0


def test_traction_offsurface_near_surface_closed_forms(oracle_mod):
    """Off-surface traction evaluator with the near correction: one sphere of
    radius 1.4 (scaled eqs 3.19-3.21: K is a-free, r -> |x - c|/a), targets at
    1.01 a .. 1.8 a with normal e_r, where the smooth rule alone is far off;
    with eta = 1 every target is corrected and the closed forms hold to 1e-12."""
    p, a = 6, 1.4
    c = np.array([0.3, -0.2, 0.5])
    x, _, _ = oracle_mod.nodes(c[None], np.array([a]), p)
    rng = np.random.default_rng(14)
    th, ph = rng.uniform(0.1, 3.0, 8), rng.uniform(-3.1, 3.1, 8)
    er = np.stack([np.sin(th) * np.cos(ph), np.sin(th) * np.sin(ph), np.cos(th)], 1)
    rr = np.array([1.01, 1.03, 1.1, 1.2, 1.35, 1.5, 1.65, 1.8])
    pts = c + a * rr[:, None] * er
    for n, m, ch in ((1, 0, 0), (2, 1, 1), (3, -2, 2), (5, 4, 1), (6, 3, 0)):
        sig = H.vsh_density(n, m, ch, x, c, a)
        t = oracle_mod.traction_offsurface(c[None], np.array([a]), p, sig, pts, er, eta=1.0)
        t0 = oracle_mod.traction_offsurface(c[None], np.array([a]), p, sig, pts, er, eta=0.0)
        ref = np.array([_K_closed_form(n, m, ch, rr[i], th[i], ph[i]) for i in range(8)])
        assert np.abs(t - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max()), (n, m, ch)
        assert np.abs(t0 - ref).max() >= 1e-6  # the smooth rule alone is not accurate here
