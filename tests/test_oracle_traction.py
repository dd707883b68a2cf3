"""Pins of the NEXT-3 oracle: the traction operator K (eq 2.22).
Reading R21: K[s](x) = -(3/4pi) int (rho.n(x))(rho.s)rho/|rho|^5,
the adjoint of the R1 double layer.  Pinned (a) on the sphere against
brute-force quadrature of this kernel, which must reproduce the spectrum
P:219 assigns to K (K_pv = D_pv), and (b) off the surface against the
traction -p n + mu (grad u + grad u^T) n of the single-layer flow computed by
finite differences of the (independently pinned) off-surface evaluator."""
import numpy as np
import pytest

from tests import _harmonics as H


def test_K_self_spectrum_is_D_pv(oracle_mod):
    """Every single harmonic n <= 4, all m, V/W/X: brute-force polar quadrature
    of the K kernel on the sphere == the D_pv self term (K_+ = D_-, K_- = D_+)."""
    p, a = 4, 1.2
    c = np.array([0.1, -0.3, 0.2])
    x, _, _ = oracle_mod.nodes(c[None], np.array([a]), p)
    for n in range(0, p + 1):
        for m in range(-n, n + 1):
            for ch in range(3):
                if n == 0 and ch > 0:
                    continue
                dens = lambda y, n=n, m=m, ch=ch: H.vsh_density(n, m, ch, y, c, a)
                u = oracle_mod.apply_K(c[None], np.array([a]), p, dens(x))
                for i in (0, 13, 27, 41):
                    ref = H.onsurface_layers(x[i], c, a, 1.0, dens, "K")
                    assert np.abs(u[i] - ref).max() <= 2e-12, (n, m, ch, i)


def test_translating_sphere_traction(oracle_mod):
    """Uniform traction density f = 3 mu U/(2a): exterior traction K_+[f] =
    K_pv[f] - f/2 = -3 mu U/(2a) (classical Stokes), interior K_-[f] = 0."""
    p, a, mu = 6, 0.9, 1.4
    c = np.array([[0.0, 0.5, 0.0]])
    U = np.array([0.2, 0.7, -0.4])
    N = (p + 1) * (2 * p + 2)
    f = np.tile(1.5 * mu * U / a, (N, 1))
    kpv = oracle_mod.apply_K(c, np.array([a]), p, f)
    assert np.abs((kpv - 0.5 * f) + 1.5 * mu * U / a).max() <= 1e-13
    assert np.abs(kpv + 0.5 * f).max() <= 1e-13


def test_K_far_field_equals_traction_of_single_layer_flow(oracle_mod):
    """At points away from two spheres, with arbitrary unit normals n:
    K[f](x; n) == -p n + mu (grad u + grad u^T) n of u = S[f] (central
    differences, h = 1e-3, of the off-surface velocity and pressure)."""
    p, mu = 8, 1.7
    c = np.array([[0.0, 0.0, 0.0], [3.0, 0.5, 0.0]])
    a = np.array([1.0, 0.7])
    N = 2 * (p + 1) * (2 * p + 2)
    f = np.random.default_rng(4).standard_normal((N, 3))
    pts = np.array([[1.5, 2.2, 1.0], [-1.0, -1.5, 2.0], [4.5, -1.0, -1.2]])
    nrm = np.random.default_rng(5).standard_normal((3, 3))
    nrm /= np.linalg.norm(nrm, axis=1)[:, None]
    K = oracle_mod.K_at(c, a, p, f, pts, nrm)
    h = 1e-3
    for t in range(3):
        G = np.zeros((3, 3))
        for ax in range(3):
            e = np.zeros(3)
            e[ax] = h
            up, _ = oracle_mod.offsurface(c, a, p, mu, f, None, (pts[t] + e)[None])
            um, _ = oracle_mod.offsurface(c, a, p, mu, f, None, (pts[t] - e)[None])
            G[:, ax] = (up[0] - um[0]) / (2 * h)          # G_ij = d u_i / d x_j
        _, p0 = oracle_mod.offsurface(c, a, p, mu, f, None, pts[t][None])
        trac = -p0[0] * nrm[t] + mu * (G + G.T) @ nrm[t]
        assert np.abs(K[t] - trac).max() <= 1e-6 * np.abs(trac).max()
