"""Test-side harmonics built from SciPy (independent of oracle/ and of the CUDA path).

Scalar Y_n^m follows eq 2.1: |m| inside P, no Condon-Shortley
phase.  SciPy's sph_harm_y includes the phase (-1)^m for m >= 0, so
ours = (-1)^m * scipy for m >= 0 and ours = scipy for m < 0 (both then satisfy
Y_n^{-m} = conj Y_n^m).  V, W, X follow eqs 2.4-2.6.
"""
import numpy as np
from scipy.special import sph_harm_y


def ylm(n, m, th, ph):
    """Y, dY/dtheta, (1/sin theta) dY/dphi (complex arrays)."""
    th = np.asarray(th, dtype=np.float64)
    ph = np.asarray(ph, dtype=np.float64)
    y, jac = sph_harm_y(n, m, th, ph, diff_n=1)
    s = (-1.0) ** m if m >= 0 else 1.0
    return s * y, s * jac[..., 0], s * jac[..., 1] / np.sin(th)


def frames(th, ph):
    st, ct, sp, cp = np.sin(th), np.cos(th), np.sin(ph), np.cos(ph)
    er = np.stack([st * cp, st * sp, ct], -1)
    et = np.stack([ct * cp, ct * sp, -st], -1)
    ep = np.stack([-sp, cp, np.zeros_like(ph)], -1)
    return er, et, ep


def vsh(n, m, th, ph):
    """Complex Cartesian V, W, X at arrays th, ph -> three arrays [..., 3]."""
    Y, dY, dYp = ylm(n, m, th, ph)
    er, et, ep = frames(th, ph)
    grad = dY[..., None] * et + dYp[..., None] * ep
    V = grad - (n + 1) * Y[..., None] * er
    W = grad + n * Y[..., None] * er
    X = dY[..., None] * ep - dYp[..., None] * et
    return V, W, X


def angles(v):
    """(theta, phi) of direction vectors v [..., 3]."""
    r = np.linalg.norm(v, axis=-1)
    th = np.arccos(np.clip(v[..., 2] / r, -1.0, 1.0))
    ph = np.arctan2(v[..., 1], v[..., 0])
    return th, ph


def vsh_density(n, m, ch, pts, centre, a):
    """Real part of Z_nm (ch 0=V, 1=W, 2=X) at points on the sphere (centre, a)."""
    th, ph = angles((pts - centre) / a)
    return np.real(vsh(n, m, th, ph)[ch])


def onsurface_layers(xt, centre, a, mu, dens, kind, nalpha=72, nbeta=144):
    """Continuous on-surface S[f](xt) or D[q](xt) (principal value) on the sphere
    (centre, a) by brute-force quadrature in polar coordinates about xt.

    With y = c + a(cos al xh + sin al (cos be e1 + sin be e2)), dS = a^2 sin al dal dbe
    and |xt - y| = 2 a sin(al/2), the Stokeslet (eq 2.19) and the stresslet
    (eq 2.20, sign reading R1) times sin al are smooth on [0,pi]x[0,2pi), so a
    Gauss-Legendre rule in al and the trapezoid rule in be converge spectrally.
    The stresslet on a sphere has (rho . n) = -|rho|^2/(2a), so the integral is
    absolutely convergent and equals the principal value.
    """
    xh = (xt - centre) / a
    tmp = np.array([1.0, 0.0, 0.0]) if abs(xh[0]) < 0.9 else np.array([0.0, 1.0, 0.0])
    e1 = tmp - xh * (tmp @ xh)
    e1 /= np.linalg.norm(e1)
    e2 = np.cross(xh, e1)
    ga, wa = np.polynomial.legendre.leggauss(nalpha)
    al = 0.5 * np.pi * (ga + 1.0)
    wa = 0.5 * np.pi * wa
    be = 2.0 * np.pi * np.arange(nbeta) / nbeta
    AL, BE = np.meshgrid(al, be, indexing="ij")
    W = (wa[:, None] * (2.0 * np.pi / nbeta)) * a * a * np.sin(AL)
    yh = (np.cos(AL)[..., None] * xh + np.sin(AL)[..., None] *
          (np.cos(BE)[..., None] * e1 + np.sin(BE)[..., None] * e2))
    y = centre + a * yh
    g = dens(y)
    rho = xt - y
    r = np.linalg.norm(rho, axis=-1)
    if kind == "S":
        rf = np.einsum("...c,...c->...", rho, g)
        K = (g / r[..., None] + rf[..., None] * rho / r[..., None] ** 3) / (8.0 * np.pi * mu)
    elif kind == "K":
        # traction of the single layer with the TARGET normal xh (eq 2.22, reading R21)
        rn = rho @ xh
        rq = np.einsum("...c,...c->...", rho, g)
        K = -3.0 / (4.0 * np.pi) * (rn * rq)[..., None] * rho / r[..., None] ** 5
    else:
        rn = np.einsum("...c,...c->...", rho, yh)
        rq = np.einsum("...c,...c->...", rho, g)
        K = 3.0 / (4.0 * np.pi) * (rn * rq)[..., None] * rho / r[..., None] ** 5
    return np.einsum("ij,ijc->c", W, K)
