"""Pins of the NEXT-4 oracle (PAPER §4.2 "FFT-accelerated near evaluation",
Fig 2; reading R25 for the rotation): stage (1) density rotation,
stage (2) evaluation at the pole-aligned target grid (the exterior formulas,
pinned in test_oracle_near.py), stage (3) forward transform on the target grid,
rotation back and evaluation.  Each pin is independent of the oracle's own
arithmetic: SciPy harmonics (tests/_harmonics.py), closed forms of rotations
about the z and x axes, invariants (per-degree norms, round trips), weighted
least squares with SciPy harmonics, and spectral convergence to the exact
exterior field."""
import numpy as np
import pytest

from tests import _harmonics as H
from tests.test_oracle_near_K import _bandlimited


def _grid(oracle_mod, p, c=np.zeros(3), a=1.0):
    x, n, w = oracle_mod.nodes(np.asarray(c, dtype=float)[None], np.array([a]), p)
    return x, n, w


def _rot_z(g):
    c, s = np.cos(g), np.sin(g)
    return np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])


def _random_rotation(rng):
    q = rng.standard_normal(4)
    q /= np.linalg.norm(q)
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                     [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                     [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]])


def test_rotation_definition(oracle_mod):
    """Q = Rz(alpha) Ry(beta) is a proper rotation with Q e_z = d (reading R25)."""
    rng = np.random.default_rng(0)
    for _ in range(20):
        cs, ct = rng.standard_normal(3), rng.standard_normal(3)
        Q = oracle_mod.next4_rotation(cs, ct)
        d = (ct - cs) / np.linalg.norm(ct - cs)
        assert np.abs(Q @ Q.T - np.eye(3)).max() < 1e-15
        assert abs(np.linalg.det(Q) - 1.0) < 1e-15
        assert np.abs(Q[:, 2] - d).max() < 1e-15


@pytest.mark.parametrize("n,m,ch", [(1, 0, 0), (1, 1, 1), (2, -1, 2), (3, 2, 0), (4, -3, 1), (5, 5, 2)])
def test_rotated_single_harmonic_equals_direct_evaluation(oracle_mod, n, m, ch):
    """Stage (1) on the density Re Z_nm: the rotated-frame coefficients,
    evaluated at random off-grid directions y, equal Q^T Re Z_nm(Q y) computed
    directly with SciPy harmonics (exactness of the grid projection for a
    band-limited field, and the orientation Q vs Q^T)."""
    p = 6
    rng = np.random.default_rng(10 * n + ch)
    _, nh, _ = _grid(oracle_mod, p)
    g = H.vsh_density(n, m, ch, nh, np.zeros(3), 1.0)
    Q = oracle_mod.next4_rotation(np.zeros(3), rng.standard_normal(3))
    gR = oracle_mod.rotate_density(p, Q, g)
    aR = oracle_mod.vsh_project(p, gR)
    y = rng.standard_normal((40, 3))
    y /= np.linalg.norm(y, axis=1)[:, None]
    got = oracle_mod.vsh_expand(p, aR, y)
    ref = H.vsh_density(n, m, ch, y @ Q.T, np.zeros(3), 1.0) @ Q  # Q^T v for each row v
    assert np.abs(got - ref).max() <= 1e-13 * max(1.0, np.abs(ref).max())


def test_rotation_about_z_multiplies_by_phase(oracle_mod):
    """Closed form: for Q = Rz(g), sigma^R(y) = Q^T sigma(Q y) has coefficients
    e^{i m g} c_nm (Y_n^m(theta, phi + g) = e^{i m g} Y_n^m)."""
    p, g = 7, 0.7318
    rng = np.random.default_rng(3)
    _, nh, _ = _grid(oracle_mod, p)
    sig = _bandlimited(4, p, nh, np.zeros(3), 1.0)
    a = oracle_mod.vsh_project(p, sig)
    aR = oracle_mod.vsh_project(p, oracle_mod.rotate_density(p, _rot_z(g), sig))
    mm = np.array([m for n in range(p + 1) for m in range(-n, n + 1)])
    assert np.abs(aR - np.exp(1j * mm * g)[:, None] * a).max() <= 1e-13 * np.abs(a).max()
    del rng


def test_rotation_by_pi_about_x_closed_form(oracle_mod):
    """Closed form: Q = Rx(pi) maps (theta, phi) -> (pi - theta, -phi); with
    P_n^m(-t) = (-1)^{n+m} P_n^m(t) and Y^{-m} = conj Y^m, c^R_{n,-m} = (-1)^{n+m} c_{n,m}."""
    p = 6
    _, nh, _ = _grid(oracle_mod, p)
    sig = _bandlimited(5, p, nh, np.zeros(3), 1.0)
    a = oracle_mod.vsh_project(p, sig)
    Q = np.diag([1.0, -1.0, -1.0])
    aR = oracle_mod.vsh_project(p, oracle_mod.rotate_density(p, Q, sig))
    for n in range(p + 1):
        for m in range(-n, n + 1):
            assert np.abs(aR[n * n + n - m] - (-1) ** (n + m) * a[n * n + n + m]).max() <= 1e-13


def test_rotation_preserves_degree_norms_and_inverts(oracle_mod):
    """Per degree and channel, sum_m |c_nm|^2 is rotation invariant (the basis
    is orthogonal and each degree is an irreducible representation); rotating
    by Q then by Q^T returns the band-limited density to 1e-14."""
    p = 9
    rng = np.random.default_rng(6)
    _, nh, _ = _grid(oracle_mod, p)
    sig = _bandlimited(6, p, nh, np.zeros(3), 1.0)
    a = oracle_mod.vsh_project(p, sig)
    for _ in range(3):
        Q = _random_rotation(rng)
        sR = oracle_mod.rotate_density(p, Q, sig)
        aR = oracle_mod.vsh_project(p, sR)
        for n in range(p + 1):
            sl = slice(n * n, n * n + 2 * n + 1)
            na, nr = np.sum(np.abs(a[sl]) ** 2, 0), np.sum(np.abs(aR[sl]) ** 2, 0)
            assert np.abs(na - nr).max() <= 1e-13 * max(1.0, na.max())
        back = oracle_mod.rotate_density(p, Q.T, sR)
        assert np.abs(back - sig).max() <= 1e-14 * 10 * np.abs(sig).max()


def test_double_layer_of_rigid_motion_gives_zero(oracle_mod):
    """D[U + W x (y - c)] = 0 outside the sphere (App. B check 10) -> every
    stage carries zero: the NEXT-4 estimate vanishes at the target nodes."""
    p = 8
    cs, ct = np.array([0.1, 0.2, -0.3]), np.array([1.9, 1.2, 0.8])
    xs, _, _ = _grid(oracle_mod, p, cs, 1.0)
    U, W = np.array([0.3, -1.2, 0.5]), np.array([0.7, 0.1, -0.4])
    q = U + np.cross(W, xs - cs)
    out = oracle_mod.next4_pair(p, cs, 1.0, ct, 0.9, 1.3, None, q)
    assert np.abs(out).max() <= 1e-13


def test_stage3_equals_weighted_least_squares_with_scipy_harmonics(oracle_mod):
    """Stages (2)-(3) re-done independently: exterior field of the rotated
    density at the pole-aligned target grid (oracle.exterior_eval, pinned in
    test_oracle_near.py), weighted least-squares fit with SciPy VSH on that
    grid (= the discrete projection of reading R9), evaluated at Q^T n_i and
    rotated back -- equals oracle.next4_pair at every target node."""
    p, mu = 5, 1.4
    cs, ct = np.array([0.0, 0.0, 0.0]), np.array([1.3, -1.7, 1.1])
    a_s, a_t = 1.1, 0.8
    xs, nh, _ = _grid(oracle_mod, p, cs, a_s)
    f = _bandlimited(11, 3, xs, cs, a_s)
    q = _bandlimited(12, 3, xs, cs, a_s)
    got = oracle_mod.next4_pair(p, cs, a_s, ct, a_t, mu, f, q)
    Q = oracle_mod.next4_rotation(cs, ct)
    fR, qR = oracle_mod.rotate_density(p, Q, f), oracle_mod.rotate_density(p, Q, q)
    Cz = np.linalg.norm(ct - cs)
    XR = np.array([0.0, 0.0, Cz]) + a_t * nh
    uR = oracle_mod.exterior_eval(p, np.zeros(3), a_s, mu, fR, qR, XR)
    # weighted least squares with SciPy VSH (unit-sphere weights lambda_j 2 pi/(2p+2))
    t, lam = np.polynomial.legendre.leggauss(p + 1)
    wu = np.repeat(lam * 2 * np.pi / (2 * p + 2), 2 * p + 2)
    th, ph = H.angles(nh)
    cols = []
    for n in range(p + 1):
        for m in range(-n, n + 1):
            for ch, Z in enumerate(H.vsh(n, m, th, ph)):
                if n == 0 and ch:
                    continue
                cols.append(Z)
    B = np.stack([c.reshape(-1) for c in cols], 1)
    sw = np.repeat(np.sqrt(wu), 3)
    coef, *_ = np.linalg.lstsq(B * sw[:, None], (uR.reshape(-1) * sw).astype(complex), rcond=None)
    thi, phi = H.angles(nh @ Q)  # Q^T n_i as rows
    cols = []
    for n in range(p + 1):
        for m in range(-n, n + 1):
            for ch, Z in enumerate(H.vsh(n, m, thi, phi)):
                if n == 0 and ch:
                    continue
                cols.append(Z)
    vR = np.real(np.stack([c.reshape(-1) for c in cols], 1) @ coef).reshape(-1, 3)
    ref = vR @ Q.T  # Q v for each row v
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()


def test_pipeline_converges_spectrally_to_exterior_field(oracle_mod):
    """As the order p grows, the NEXT-4 estimate (a degree-p re-expansion on the
    target sphere) converges spectrally to the exact exterior field of the
    (band-limited, degree 3) source density at the target nodes; the rate is
    set by the distance from the target centre to the source sphere."""
    cs, ct = np.array([0.0, 0.0, 0.0]), np.array([2.2, 2.9, -1.3])  # gap ~ 1.9
    errs = []
    for p in (6, 10, 14, 20, 26):
        xs, _, _ = _grid(oracle_mod, p, cs, 1.0)
        xt, _, _ = _grid(oracle_mod, p, ct, 1.0)
        f = _bandlimited(21, 3, xs, cs, 1.0)
        q = _bandlimited(22, 3, xs, cs, 1.0)
        got = oracle_mod.next4_pair(p, cs, 1.0, ct, 1.0, 1.0, f, q)
        ref = oracle_mod.exterior_eval(p, cs, 1.0, 1.0, f, q, xt)
        errs.append(np.abs(got - ref).max() / np.abs(ref).max())
    assert all(e2 < e1 for e1, e2 in zip(errs, errs[1:])), errs
    assert errs[-1] <= 1e-10, errs


def test_near4_correction_definition(oracle_mod):
    """oracle.near4 = sum over eq-4.5 neighbours of (next4_pair - smooth rule)
    at the subset nodes; a far-away sphere contributes nothing."""
    p, mu, eta = 5, 1.1, 1.0
    c = np.array([[0.0, 0.0, 0.0], [2.3, 0.6, -0.4], [20.0, 0.0, 0.0]])
    a = np.array([1.0, 0.9, 1.0])
    x, nrm, w = oracle_mod.nodes(c, a, p)
    nsn = (p + 1) * (2 * p + 2)
    rng = np.random.default_rng(30)
    f, q = rng.standard_normal((3 * nsn, 3)), rng.standard_normal((3 * nsn, 3))
    sub = np.arange(0, nsn)  # nodes of sphere 0; its only neighbour is sphere 1
    du = oracle_mod.near4(c, a, p, mu, f, q, eta, sub)
    est = oracle_mod.next4_pair(p, c[1], a[1], c[0], a[0], mu, f[nsn:2 * nsn], q[nsn:2 * nsn])
    # smooth rule of sphere 1 alone at sphere 0's nodes = far field of the pair minus sphere 2
    two = oracle_mod.far(c[:2], a[:2], p, mu, f[:2 * nsn], q[:2 * nsn], sub)
    assert np.abs(du - (est - two)).max() <= 1e-12 * np.abs(est).max()
    sub2 = np.arange(2 * nsn, 3 * nsn)  # sphere 2 has no neighbour
    assert np.all(oracle_mod.near4(c, a, p, mu, f, q, eta, sub2) == 0.0)


def test_vsh_evaluation_is_pole_safe(oracle_mod):
    """The stage-(3) evaluator works at directions on (or rounded onto) the polar
    axis -- at even p a target node lies exactly on an axis-aligned pair axis.
    It equals SciPy's harmonics at generic directions and is continuous at the
    poles."""
    p = 7
    rng = np.random.default_rng(40)
    a = rng.standard_normal(((p + 1) ** 2, 3)) + 1j * rng.standard_normal(((p + 1) ** 2, 3))
    d = rng.standard_normal((30, 3))
    d /= np.linalg.norm(d, axis=1)[:, None]
    th, ph = H.angles(d)
    ref = np.zeros((30, 3), complex)
    for n in range(p + 1):
        for m in range(-n, n + 1):
            Z = H.vsh(n, m, th, ph)
            for ch in range(3):
                if n == 0 and ch:
                    continue
                ref += a[n * n + n + m, ch] * Z[ch]
    assert np.abs(oracle_mod.vsh_expand(p, a, d) - ref.real).max() <= 1e-13 * np.abs(ref).max()
    for zs in (1.0, -1.0):
        pole = oracle_mod.vsh_expand(p, a, np.array([[0.0, 0.0, zs], [1e-17, 0.0, zs]]))
        near = oracle_mod.vsh_expand(p, a, np.array([[1e-7, 0.0, zs], [0.0, -1e-7, zs]]))
        assert np.all(np.isfinite(pole))
        assert np.abs(pole[0] - pole[1]).max() <= 1e-14 * np.abs(pole).max()
        assert np.abs(near - pole[0]).max() <= 1e-5 * np.abs(pole).max()
