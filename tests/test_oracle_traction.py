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


# ------------------------------------------------ completion operator (eq 5.8)
def _rigid(x, c, F, W):
    return F + np.cross(W, x - c)


def test_completion_closed_forms(oracle_mod):
    """L[mu] for mu = const F: 4 pi a^2 F; for mu = W x (y - c): the moment
    int (y-c) x (W x (y-c)) dS = (8 pi a^4 / 3) W, so L = (8 pi a^4/3) W x (x - c);
    for a degree 2..4 field: 0 (orthogonal to both moments).  Two spheres with
    different radii -- each block sees only its own density (reading R22)."""
    p = 6
    c = np.array([[0.3, -0.2, 0.1], [3.1, 0.4, -0.5]])
    a = np.array([1.3, 0.8])
    x, _, _ = oracle_mod.nodes(c, a, p)
    nsn = (p + 1) * (2 * p + 2)
    F = np.array([[0.4, -1.2, 0.7], [0.0, 0.0, 0.0]])
    W = np.array([[0.0, 0.0, 0.0], [0.9, 0.3, -0.6]])
    mu = np.concatenate([_rigid(x[:nsn], c[0], F[0], W[0]), _rigid(x[nsn:], c[1], F[1], W[1])])
    L = oracle_mod.completion(c, a, p, mu)
    ref0 = np.tile(4 * np.pi * a[0] ** 2 * F[0], (nsn, 1))
    ref1 = (8 * np.pi * a[1] ** 4 / 3) * np.cross(W[1], x[nsn:] - c[1])
    assert np.abs(L[:nsn] - ref0).max() <= 1e-13 * np.abs(ref0).max()
    assert np.abs(L[nsn:] - ref1).max() <= 1e-13 * np.abs(ref1).max()
    # degree >= 2 densities on sphere 0, zero on sphere 1
    hi = np.zeros_like(x)
    for n, m, ch in ((2, 1, 0), (3, -2, 1), (4, 3, 2), (2, 0, 1)):
        hi[:nsn] += H.vsh_density(n, m, ch, x[:nsn], c[0], a[0])
    L = oracle_mod.completion(c, a, p, hi)
    assert np.abs(L).max() <= 1e-13 * np.abs(hi).max()


def test_completion_removes_the_6n_rigid_nullspace(oracle_mod):
    """1/2 I + K has a 6 n_b dimensional nullspace (per-body rigid
    motions: K = D^T (R21) and D_pv[rigid_k] = -rigid_k/2 on Gamma_k, 0
    elsewhere); adding sum_k L_k removes it.  Dense matrices, two spheres."""
    p = 3
    c = np.array([[0.0, 0.0, 0.0], [4.0, 1.0, -0.5]])
    a = np.array([1.0, 0.7])
    N = 2 * (p + 1) * (2 * p + 2)
    x, _, w = oracle_mod.nodes(c, a, p)
    M = np.empty((3 * N, 3 * N))
    ML = np.empty((3 * N, 3 * N))
    for j in range(3 * N):
        e = np.zeros(3 * N)
        e[j] = 1.0
        e = e.reshape(N, 3)
        k = 0.5 * e + oracle_mod.apply_K(c, a, p, e)
        M[:, j] = k.reshape(-1)
        ML[:, j] = (k + oracle_mod.completion(c, a, p, e)).reshape(-1)
    # symmetric form (weighted inner product) for clean singular values
    sw = np.sqrt(np.repeat(w, 3))
    s = np.linalg.svd(sw[:, None] * M / sw[None, :], compute_uv=False)
    sL = np.linalg.svd(sw[:, None] * ML / sw[None, :], compute_uv=False)
    assert np.sum(s < 1e-3 * s[0]) == 12, s[-14:]  # smooth-rule coupling error ~1e-5
    assert s[-13] > 0.1 * s[0]
    assert sL[-1] >= 0.99 * s[-13], sL[-3:]  # no new small singular values
    # the nullspace is spanned by per-body rigid motions (weighted adjoint):
    # M^T W r = 0 for every rigid field r  (since D[rigid] = -rigid/2 on-body,
    # ~0 off-body), i.e. rigid fields span the left nullspace.
    nsn = N // 2
    for b in range(2):
        for F, Wv in ((np.eye(3)[0], np.zeros(3)), (np.zeros(3), np.eye(3)[2]),
                      (np.array([0.3, -0.7, 0.2]), np.array([-0.4, 0.1, 0.9]))):
            r = np.zeros((N, 3))
            sl = slice(b * nsn, (b + 1) * nsn)
            r[sl] = _rigid(x[sl], c[b], F, Wv)
            wr = np.repeat(w, 3) * r.reshape(-1)
            lhs = (M.T @ wr).reshape(N, 3)
            # own body: exact (the self term's spectrum); other body: the
            # smooth rule's error for D[rigid] = 0 off-body at p = 3
            assert np.abs(lhs[sl]).max() <= 1e-14 * np.abs(wr).max()
            assert np.abs(lhs).max() <= 1e-4 * np.abs(wr).max()


# ------------------------------------- K off the surface: eqs 3.19-3.21
def _K_closed_form(n, m, ch, r, th, ph):
    """PAPER eqs 3.19-3.21 for the unit sphere, target normal e_r, as printed
    except the interior V coupling, whose sign is reading R23."""
    V, W, X = [np.real(z) for z in H.vsh(n, m, th, ph)]
    d1, d3 = (2 * n + 1), (2 * n + 3)
    if r > 1:
        if ch == 0:
            return -2 * n * (n + 2) / (d1 * d3) * V * r ** (-n - 3)
        if ch == 1:
            return (-(2 * n * n + 1) / (d1 * (2 * n - 1)) * W * r ** (-n - 1)
                    + n * (n + 2) / d1 * V * (r ** (-n - 1) - r ** (-n - 3)))
        return -(n + 2) / d1 * X * r ** (-n - 2)
    if ch == 0:  # R23: + (n+1)(n-1)/(2n+1) W (r^n - r^{n-2})  (printed with "-")
        return ((2 * n * n + 4 * n + 3) / (d1 * d3) * V * r ** n
                + (n + 1) * (n - 1) / d1 * W * (r ** n - r ** (n - 2)))
    if ch == 1:
        return 2 * (n + 1) * (n - 1) / (d1 * (2 * n - 1)) * W * r ** (n - 2)
    return (n - 1) / d1 * X * r ** (n - 1)


def test_K_offsurface_closed_forms(oracle_mod):
    """K[Z_n^m] at r e_r with normal e_r (unit sphere) == eqs 3.19-3.21, both
    branches, n = 1..4, V/W/X, incl. the V <-> W couplings (converged rule, p = 36)."""
    P = 36
    c, a = np.zeros((1, 3)), np.ones(1)
    x, _, _ = oracle_mod.nodes(c, a, P)
    rng = np.random.default_rng(12)
    for n in range(1, 5):
        for m in sorted({0, 1, n}):
            for ch in range(3):
                sig = H.vsh_density(n, m, ch, x, c[0], 1.0)
                for r in (0.4, 0.55, 1.7, 2.6):
                    th, ph = rng.uniform(0.2, 2.9), rng.uniform(-3.0, 3.0)
                    er = np.array([np.sin(th) * np.cos(ph), np.sin(th) * np.sin(ph), np.cos(th)])
                    K = oracle_mod.K_at(c, a, P, sig, (r * er)[None], er[None])[0]
                    ref = _K_closed_form(n, m, ch, r, th, ph)
                    assert np.abs(K - ref).max() <= 1e-12, (n, m, "VWX"[ch], r, K, ref)


def test_R23_interior_V_coupling_sign_by_finite_differences(oracle_mod):
    """Reading R23 decided without the K kernel: inside the unit sphere, the
    traction -p n + (grad u + grad u^T) n of u = S[V_2^1] (off-surface
    evaluator, central differences) matches eq 3.19 with "+ (n+1)(n-1)/(2n+1)"
    and misses the printed "-" by O(1)."""
    P, n, m = 36, 2, 1
    c, a = np.zeros((1, 3)), np.ones(1)
    x, _, _ = oracle_mod.nodes(c, a, P)
    sig = H.vsh_density(n, m, 0, x, c[0], 1.0)
    r, th, ph = 0.5, 1.1, 0.4
    er = np.array([np.sin(th) * np.cos(ph), np.sin(th) * np.sin(ph), np.cos(th)])
    pt, h = r * er, 1e-3
    G = np.zeros((3, 3))
    for ax in range(3):
        e = np.zeros(3)
        e[ax] = h
        up, _ = oracle_mod.offsurface(c, a, P, 1.0, sig, None, (pt + e)[None])
        um, _ = oracle_mod.offsurface(c, a, P, 1.0, sig, None, (pt - e)[None])
        G[:, ax] = (up[0] - um[0]) / (2 * h)
    _, p0 = oracle_mod.offsurface(c, a, P, 1.0, sig, None, pt[None])
    trac = -p0[0] * er + (G + G.T) @ er
    ref = _K_closed_form(n, m, 0, r, th, ph)
    V, W, X = [np.real(z) for z in H.vsh(n, m, th, ph)]
    printed = ref - 2 * (n + 1) * (n - 1) / (2 * n + 1) * W * (r ** n - r ** (n - 2))
    assert np.abs(trac - ref).max() <= 1e-6
    assert np.abs(trac - printed).max() >= 0.1
