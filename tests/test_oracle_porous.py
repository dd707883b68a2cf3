"""Pins of the NEXT-2 oracle (Problem 1, porous media: BIE 5.4):
the dense solve of (1/2 I + S + D) mu = -u_inf reproduces the classical
Stokes drag and torque on a fixed sphere (independent of the paper)."""
import numpy as np
import pytest


def test_single_sphere_uniform_flow_drag(oracle_mod):
    """Fixed sphere in uniform flow U: density mu = -3 mu_visc U/(2a) (W_1 channel:
    (2/3)(a/mu) - 1/2 + 1/2), force -int mu dS = 6 pi mu a U (Stokes drag)."""
    p, a, visc = 4, 1.3, 0.8
    c = np.array([[0.2, -0.4, 1.0]])
    U = np.array([0.3, -1.1, 0.6])
    N = (p + 1) * (2 * p + 2)
    dens = oracle_mod.solve_porous(c, np.array([a]), p, visc, np.tile(U, (N, 1)))
    assert np.abs(dens + 1.5 * visc * U / a).max() <= 1e-13
    _, _, w = oracle_mod.nodes(c, np.array([a]), p)
    F = -(w[:, None] * dens).sum(0)
    assert np.abs(F - 6 * np.pi * visc * a * U).max() <= 1e-12 * np.linalg.norm(F)


def test_single_sphere_rotational_flow_torque(oracle_mod):
    """Fixed sphere in the rigid rotational flow Omega x (x - c): torque
    -int (x-c) x mu dS = 8 pi mu a^3 Omega."""
    p, a, visc = 4, 0.7, 1.6
    c = np.array([[1.0, 0.0, -0.5]])
    Om = np.array([0.4, 0.9, -0.2])
    x, _, w = oracle_mod.nodes(c, np.array([a]), p)
    uinf = np.cross(Om, x - c[0])
    dens = oracle_mod.solve_porous(c, np.array([a]), p, visc, uinf)
    T = -(w[:, None] * np.cross(x - c[0], dens)).sum(0)
    assert np.abs(T - 8 * np.pi * visc * a ** 3 * Om).max() <= 1e-12 * np.linalg.norm(T)


def test_two_spheres_mirror_symmetry(oracle_mod):
    """Two equal spheres placed symmetrically across the plane normal to the flow
    direction feel equal drags (mirror symmetry); the drag of each is reduced
    below the isolated-sphere value 6 pi mu a U (hydrodynamic shielding)."""
    p, visc = 5, 1.0
    c = np.array([[-1.6, 0.0, 0.0], [1.6, 0.0, 0.0]])
    a = np.ones(2)
    U = np.array([0.0, 0.0, 1.0])
    N = 2 * (p + 1) * (2 * p + 2)
    dens = oracle_mod.solve_porous(c, a, p, visc, np.tile(U, (N, 1)), eta=1.0)
    _, _, w = oracle_mod.nodes(c, a, p)
    ns = N // 2
    F0 = -(w[:ns, None] * dens[:ns]).sum(0)
    F1 = -(w[ns:, None] * dens[ns:]).sum(0)
    assert abs(F0[2] - F1[2]) <= 1e-12 * abs(F0[2])
    assert F0[2] < 6 * np.pi and F0[2] > 0.5 * 6 * np.pi


def stimson_jeffery(c_over_a, nterms=400):
    """Drag correction factor lambda = F / (6 pi mu a U) for two equal spheres
    translating along their line of centres (Stimson & Jeffery 1926, bipolar
    coordinates; centres at +-c, cosh(alpha) = c/a).  By linearity the same
    factor gives the drag on each of two fixed spheres in a uniform flow U
    parallel to the line of centres (Problem 1 of PAPER §5)."""
    al = np.arccosh(c_over_a)
    s = 0.0
    for n in range(1, nterms):
        if (2 * n + 1) * al > 600:  # sinh would overflow; the terms are long negligible
            break
        num = 4 * np.sinh((n + 0.5) * al) ** 2 - (2 * n + 1) ** 2 * np.sinh(al) ** 2
        den = 2 * np.sinh((2 * n + 1) * al) + (2 * n + 1) * np.sinh(2 * al)
        term = n * (n + 1) / ((2 * n - 1) * (2 * n + 3)) * (1 - num / den)
        s += term
        if n > 4 and abs(term) < 1e-18 * abs(s):
            break
    return 4.0 / 3.0 * np.sinh(al) * s


def test_stimson_jeffery_isolated_limit():
    """The series tends to 1 (Stokes drag) for far-apart spheres and matches the
    method of reflections: each sphere sits in the other's Stokeslet flow
    (3/2)(a/l) U along the axis (l = centre distance), so
    lambda = 1 / (1 + 3a/(2l)) + O((a/l)^3) = 1 - 3/(2l) + 9/(4 l^2) + O(l^-3)."""
    for ell in (20.0, 40.0, 80.0):
        lam = stimson_jeffery(ell / 2)
        approx = 1 - 3 / (2 * ell) + 9 / (4 * ell ** 2)
        assert abs(lam - approx) <= 5.0 / ell ** 3, (ell, lam, approx)


@pytest.mark.parametrize("gap,p,tol", [(2.0, 8, 1e-10), (1.0, 8, 2e-8), (0.5, 8, 2e-6)])
def test_two_sphere_drag_matches_stimson_jeffery(oracle_mod, gap, p, tol):
    """Problem 1 (eq 5.4) solved with the near-singular correction (eta large
    enough that the pair is corrected): the drag -sum w mu on each sphere of a
    pair aligned with the flow equals 6 pi mu a U lambda_SJ, converging
    spectrally in p (gap 2: 1e-14 at p = 10)."""
    c = 1.0 + gap / 2
    cen = np.array([[0.0, 0.0, -c], [0.0, 0.0, c]])
    rad = np.ones(2)
    N = 2 * (p + 1) * (2 * p + 2)
    uinf = np.tile([0.0, 0.0, 1.0], (N, 1))
    mu = oracle_mod.solve_porous(cen, rad, p, 1.0, uinf, eta=10.0)
    _, _, w = oracle_mod.nodes(cen, rad, p)
    nsn = N // 2
    lam = stimson_jeffery(c)
    for s in range(2):
        F = -(w[s * nsn:(s + 1) * nsn, None] * mu[s * nsn:(s + 1) * nsn]).sum(0)
        assert abs(F[2] / (6 * np.pi) - lam) <= tol * lam, (s, F[2] / (6 * np.pi), lam)
        assert np.abs(F[:2]).max() <= 1e-12
