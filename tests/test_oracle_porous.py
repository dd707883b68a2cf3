"""Pins of the NEXT-2 oracle (Problem 1, porous media: BIE 5.4):
the dense solve of (1/2 I + S + D) mu = -u_inf reproduces the classical
Stokes drag and torque on a fixed sphere (independent of the paper)."""
import numpy as np


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
