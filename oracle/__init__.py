"""CPU oracle for the discretised Stokes BIO apply (arXiv 1707.06551).

TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package; the product
package paper_1707_06551_b200 never does.  The arithmetic lives in
oracle/oracle.cpp (plain C++, fp64, -ffp-contract=off, Neumaier sums); this
file only compiles it and marshals numpy arrays through ctypes.

Functions follow SURVEY.md §8(c) O-1..O-7; each cites its PAPER.md passage in
oracle.cpp.  Parity status per function is recorded in DESIGN.md §4.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

_I64P = ctypes.POINTER(ctypes.c_int64)
_DP = ctypes.POINTER(ctypes.c_double)


def build_oracle(force: bool = False) -> str:
    """Compile oracle.cpp -> liboracle.so (g++ -O2 -ffp-contract=off -fopenmp)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = f"{_LIB}.{os.getpid()}.tmp"
        cmd = ["g++", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC",
               "-shared", "-o", tmp, _SRC]
        subprocess.run(cmd, check=True)
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build_oracle()
        lib = ctypes.CDLL(_LIB)
        i64, i32, d = ctypes.c_int64, ctypes.c_int, ctypes.c_double
        lib.oracle_gl_rule.argtypes = [i32, _DP, _DP]
        lib.oracle_nodes.argtypes = [_DP, _DP, i64, i32, _DP, _DP, _DP]
        lib.oracle_far.argtypes = [_DP, _DP, i64, i32, d, _DP, _DP, _I64P, i64, _DP]
        lib.oracle_self.argtypes = [_DP, _DP, i64, i32, d, _DP, _DP, _I64P, i64, _DP]
        lib.oracle_offsurface.argtypes = [_DP, _DP, i64, i32, d, _DP, _DP, _DP, i64, _DP, _DP]
        lib.oracle_self_addthm.argtypes = [i32, d, d, _DP, _DP, _DP]
        lib.oracle_ylm.argtypes = [i32, i32, d, d, _DP]
        lib.oracle_ylm.restype = None
        lib.oracle_vsh.argtypes = [i32, i32, d, d, _DP]
        lib.oracle_vsh.restype = None
        lib.oracle_eigen.argtypes = [i32, i32, _DP, _DP, _DP, _DP]
        lib.oracle_eigen.restype = None
        lib.oracle_num_threads.restype = i32
        lib.oracle_set_num_threads.argtypes = [i32]
        lib.oracle_set_num_threads.restype = None
        _lib = lib
    return _lib


def _dp(a):
    if a is None:
        return None
    return a.ctypes.data_as(_DP)


def _c(a, dtype=np.float64):
    return None if a is None else np.ascontiguousarray(a, dtype=dtype)


def num_threads() -> int:
    return int(_load().oracle_num_threads())


def set_num_threads(n: int) -> None:
    _load().oracle_set_num_threads(int(n))


def gl_rule(p: int):
    """O-1: (t, lambda) of the (p+1)-point Gauss-Legendre rule, t ascending."""
    t = np.empty(p + 1)
    lam = np.empty(p + 1)
    if _load().oracle_gl_rule(p, _dp(t), _dp(lam)) != 0:
        raise ValueError("gl_rule: bad p")
    return t, lam


def nodes(centres, radii, p: int):
    """O-2: x [N,3], outward normals [N,3], weights [N] in node order."""
    centres = _c(centres)
    radii = _c(radii)
    ns = len(radii)
    N = ns * (p + 1) * (2 * p + 2)
    x = np.empty((N, 3))
    n = np.empty((N, 3))
    w = np.empty(N)
    if _load().oracle_nodes(_dp(centres), _dp(radii), ns, p, _dp(x), _dp(n), _dp(w)) != 0:
        raise ValueError("nodes: bad arguments")
    return x, n, w


def _subset(idx, N):
    if idx is None:
        idx = np.arange(N, dtype=np.int64)
    return np.ascontiguousarray(idx, dtype=np.int64)


def far(centres, radii, p, mu, f, q, subset=None):
    """O-3: smooth-rule S[f] + D[q] over all other spheres at nodes `subset`."""
    centres, radii, f, q = _c(centres), _c(radii), _c(f), _c(q)
    N = len(radii) * (p + 1) * (2 * p + 2)
    idx = _subset(subset, N)
    u = np.empty((len(idx), 3))
    rc = _load().oracle_far(_dp(centres), _dp(radii), len(radii), p, mu, _dp(f), _dp(q),
                            idx.ctypes.data_as(_I64P), len(idx), _dp(u))
    if rc:
        raise ValueError("far: bad arguments")
    return u


def self_term(centres, radii, p, mu, f, q, subset=None):
    """O-4: spectral self term (a/mu) S_self[f] + D_pv,self[q] at nodes `subset`."""
    centres, radii, f, q = _c(centres), _c(radii), _c(f), _c(q)
    N = len(radii) * (p + 1) * (2 * p + 2)
    idx = _subset(subset, N)
    u = np.empty((len(idx), 3))
    rc = _load().oracle_self(_dp(centres), _dp(radii), len(radii), p, mu, _dp(f), _dp(q),
                             idx.ctypes.data_as(_I64P), len(idx), _dp(u))
    if rc:
        raise ValueError("self_term: bad arguments")
    return u


def apply(centres, radii, p, mu, f, q, subset=None):
    """O-5: u = far + self = S[f] + D_pv[q] at nodes `subset` (no 1/2 I)."""
    return far(centres, radii, p, mu, f, q, subset) + self_term(centres, radii, p, mu, f, q, subset)


def offsurface(centres, radii, p, mu, f, q, targets):
    """O-6: velocity [M,3] and pressure [M] at arbitrary targets (all sources)."""
    centres, radii, f, q, targets = _c(centres), _c(radii), _c(f), _c(q), _c(targets)
    M = 0 if targets is None else targets.shape[0]
    u = np.empty((M, 3))
    pr = np.empty(M)
    rc = _load().oracle_offsurface(_dp(centres), _dp(radii), len(radii), p, mu, _dp(f), _dp(q),
                                   _dp(targets) if M else None, M, _dp(u), _dp(pr))
    if rc:
        raise ValueError("offsurface: bad arguments")
    return u, pr


def self_addthm(p, mu, a, f, q):
    """O-7: one sphere's self operator via the addition theorem (all its nodes)."""
    f, q = _c(f), _c(q)
    ns = (p + 1) * (2 * p + 2)
    u = np.empty((ns, 3))
    if _load().oracle_self_addthm(p, mu, a, _dp(f), _dp(q), _dp(u)) != 0:
        raise ValueError("self_addthm: bad arguments")
    return u


def ylm(n, m, theta, phi):
    """Y_n^m (eq 2.1), dY/dtheta, (1/sin theta) dY/dphi as complex numbers."""
    out = np.empty(6)
    _load().oracle_ylm(n, m, theta, phi, _dp(out))
    return complex(out[0], out[1]), complex(out[2], out[3]), complex(out[4], out[5])


def vsh(n, m, theta, phi):
    """Cartesian complex V, W, X (eqs 2.4-2.6) at (theta, phi), shape [3 (V,W,X), 3]."""
    out = np.empty(18)
    _load().oracle_vsh(n, m, theta, phi, _dp(out))
    z = out[0::2] + 1j * out[1::2]
    return z.reshape(3, 3)


def eigen(n, ch):
    """(lamS, lamD_ext, lamD_int, lamD_pv) for channel ch (0=V, 1=W, 2=X), unit sphere."""
    v = [ctypes.c_double() for _ in range(4)]
    _load().oracle_eigen(n, ch, *[ctypes.byref(x) for x in v])
    return tuple(x.value for x in v)


# ---------------------------------------------------------------- NEXT-1
def _load_near():
    lib = _load()
    if not getattr(lib, "_near_ready", False):
        i64, i32, d = ctypes.c_int64, ctypes.c_int, ctypes.c_double
        lib.oracle_exterior_eval.argtypes = [i32, _DP, d, d, _DP, _DP, _DP, i64, _DP]
        lib.oracle_is_near.argtypes = [_DP, d, _DP, d, d]
        lib.oracle_near.argtypes = [_DP, _DP, i64, i32, d, _DP, _DP, d, _I64P, i64, _DP]
        lib._near_ready = True
    return lib


def exterior_eval(p, centre, a, mu, f_s, q_s, targets):
    """Exact exterior S[f_s] + D[q_s] of ONE sphere from its degree-<=p VSH
    expansion (eqs 3.6-3.11; eq 4.7) at targets [M,3]."""
    lib = _load_near()
    c = _c(np.asarray(centre, dtype=np.float64).reshape(3))
    f_s, q_s, targets = _c(f_s), _c(q_s), _c(targets)
    M = targets.shape[0]
    u = np.empty((M, 3))
    if lib.oracle_exterior_eval(p, _dp(c), a, mu, _dp(f_s), _dp(q_s), _dp(targets), M, _dp(u)):
        raise ValueError("exterior_eval: bad arguments")
    return u


def is_near(cs, a_s, ct, a_t, eta):
    """eq 4.5: True if the two spheres are NOT well separated."""
    lib = _load_near()
    cs = _c(np.asarray(cs, dtype=np.float64).reshape(3))
    ct = _c(np.asarray(ct, dtype=np.float64).reshape(3))
    return bool(lib.oracle_is_near(_dp(cs), a_s, _dp(ct), a_t, eta))


def near(centres, radii, p, mu, f, q, eta, subset=None):
    """Near-singular correction du (exact minus smooth) at nodes `subset`."""
    lib = _load_near()
    centres, radii, f, q = _c(centres), _c(radii), _c(f), _c(q)
    N = len(radii) * (p + 1) * (2 * p + 2)
    idx = _subset(subset, N)
    du = np.empty((len(idx), 3))
    if lib.oracle_near(_dp(centres), _dp(radii), len(radii), p, mu, _dp(f), _dp(q), eta,
                       idx.ctypes.data_as(_I64P), len(idx), _dp(du)):
        raise ValueError("near: bad arguments")
    return du


def apply_near(centres, radii, p, mu, f, q, eta, subset=None):
    """Composite apply with the near-singular correction: far + self + near."""
    return apply(centres, radii, p, mu, f, q, subset) + near(centres, radii, p, mu, f, q, eta, subset)


# ---------------------------------------------------------------- NEXT-2
def porous_matrix(centres, radii, p, mu, eta=0.0):
    """Dense matrix of the second-kind operator of BIE 5.4,
    A mu = (1/2) mu + sum_k (S_k + D_k)[mu] at every node, built column by
    column from the oracle apply (+ near correction when eta > 0).  Small N only."""
    N = len(radii) * (p + 1) * (2 * p + 2)
    A = np.empty((3 * N, 3 * N))
    for col in range(3 * N):
        e = np.zeros((N, 3))
        e.reshape(-1)[col] = 1.0
        col_u = apply(centres, radii, p, mu, e, e)
        if eta > 0:
            col_u = col_u + near(centres, radii, p, mu, e, e, eta)
        A[:, col] = 0.5 * e.reshape(-1) + col_u.reshape(-1)
    return A


def solve_porous(centres, radii, p, mu, uinf, eta=0.0):
    """Problem 1 (porous media, eqs 5.3-5.4): solve
    (1/2 I + sum_k (S_k + D_k)) mu = -u_inf at the nodes by dense LU (numpy)."""
    A = porous_matrix(centres, radii, p, mu, eta)
    return np.linalg.solve(A, -np.asarray(uinf, dtype=np.float64).reshape(-1)).reshape(-1, 3)


# ---------------------------------------------------------------- NEXT-3
def _load_K():
    lib = _load()
    if not getattr(lib, "_K_ready", False):
        i64, i32 = ctypes.c_int64, ctypes.c_int
        lib.oracle_far_K.argtypes = [_DP, _DP, i64, i32, _DP, _I64P, i64, _DP]
        lib.oracle_K_at.argtypes = [_DP, _DP, i64, i32, _DP, _DP, _DP, i64, _DP]
        lib._K_ready = True
    return lib


def far_K(centres, radii, p, sigma, subset=None):
    """Smooth-rule traction operator K (eq 2.22, reading R21) over all other
    spheres, at nodes `subset` (target normal = the node's outward normal)."""
    lib = _load_K()
    centres, radii, sigma = _c(centres), _c(radii), _c(sigma)
    N = len(radii) * (p + 1) * (2 * p + 2)
    idx = _subset(subset, N)
    u = np.empty((len(idx), 3))
    if lib.oracle_far_K(_dp(centres), _dp(radii), len(radii), p, _dp(sigma),
                        idx.ctypes.data_as(_I64P), len(idx), _dp(u)):
        raise ValueError("far_K: bad arguments")
    return u


def K_at(centres, radii, p, sigma, targets, normals):
    """Smooth-rule K[sigma] at arbitrary points with given unit normals (all sources)."""
    lib = _load_K()
    centres, radii, sigma, targets, normals = (_c(centres), _c(radii), _c(sigma), _c(targets),
                                               _c(normals))
    u = np.empty((targets.shape[0], 3))
    if lib.oracle_K_at(_dp(centres), _dp(radii), len(radii), p, _dp(sigma), _dp(targets),
                       _dp(normals), targets.shape[0], _dp(u)):
        raise ValueError("K_at: bad arguments")
    return u


def apply_K(centres, radii, p, sigma, subset=None):
    """Discrete K_pv[sigma] at nodes: smooth far field + self term with the
    principal-value spectrum of K, which P:219 fixes as that of D_pv
    (K_+ = D_-, K_- = D_+  =>  K_pv = D_pv)."""
    return (far_K(centres, radii, p, sigma, subset) +
            self_term(centres, radii, p, 1.0, None, sigma, subset))


def _load_near_K():
    lib = _load_K()
    if not getattr(lib, "_nearK_ready", False):
        i64, i32, d = ctypes.c_int64, ctypes.c_int, ctypes.c_double
        lib.oracle_exterior_traction.argtypes = [i32, _DP, d, _DP, _DP, _DP, i64, _DP]
        lib.oracle_near_K.argtypes = [_DP, _DP, i64, i32, _DP, d, _I64P, i64, _DP]
        lib._nearK_ready = True
    return lib


def exterior_traction(p, centre, a, sigma_s, targets, normals):
    """Traction (K) of ONE sphere's degree-<=p single-layer expansion at exterior
    points with given unit normals (eqs 3.17-3.18, reading R24)."""
    lib = _load_near_K()
    centre, sigma_s, targets, normals = _c(centre), _c(sigma_s), _c(targets), _c(normals)
    t = np.empty((targets.shape[0], 3))
    if lib.oracle_exterior_traction(p, _dp(centre), float(a), _dp(sigma_s), _dp(targets),
                                    _dp(normals), targets.shape[0], _dp(t)):
        raise ValueError("exterior_traction: bad arguments")
    return t


def near_K(centres, radii, p, sigma, eta, subset=None):
    """Near correction of K at nodes (eq 4.5 partition): exterior traction minus
    the smooth-rule K sum, over the near spheres."""
    lib = _load_near_K()
    centres, radii, sigma = _c(centres), _c(radii), _c(sigma)
    N = len(radii) * (p + 1) * (2 * p + 2)
    idx = _subset(subset, N)
    du = np.empty((len(idx), 3))
    if lib.oracle_near_K(_dp(centres), _dp(radii), len(radii), p, _dp(sigma), float(eta),
                         idx.ctypes.data_as(_I64P), len(idx), _dp(du)):
        raise ValueError("near_K: bad arguments")
    return du


def apply_K_near(centres, radii, p, sigma, eta, subset=None):
    """K_pv with the near-singular correction: apply_K + near_K."""
    return apply_K(centres, radii, p, sigma, subset) + near_K(centres, radii, p, sigma, eta, subset)


def traction_offsurface(centres, radii, p, sigma, targets, normals, eta=0.0):
    """K[sigma] at arbitrary points with given normals: smooth rule over every
    node (K_at) + the near correction for exterior targets within eta 2 a_s of
    a sphere's surface (exterior traction of its expansion, eqs 3.17-3.18)."""
    lib = _load_near_K()
    if not getattr(lib, "_nearKoff_ready", False):
        i64, i32, d = ctypes.c_int64, ctypes.c_int, ctypes.c_double
        lib.oracle_near_K_offsurface.argtypes = [_DP, _DP, i64, i32, _DP, d, _DP, _DP, i64, _DP]
        lib._nearKoff_ready = True
    t = K_at(centres, radii, p, sigma, targets, normals)
    if eta > 0:
        centres, radii, sigma, targets, normals = (_c(centres), _c(radii), _c(sigma), _c(targets),
                                                   _c(normals))
        dt = np.empty_like(t)
        if lib.oracle_near_K_offsurface(_dp(centres), _dp(radii), len(radii), p, _dp(sigma),
                                        float(eta), _dp(targets), _dp(normals), targets.shape[0],
                                        _dp(dt)):
            raise ValueError("traction_offsurface: bad arguments")
        t = t + dt
    return t


def completion(centres, radii, p, mu):
    """Completion operator sum_k L_k[mu] of the mobility BIE (eq 5.8),
    reading R22: block diagonal, one rank-6 block per sphere (all N nodes)."""
    lib = _load_K()
    if not getattr(lib, "_L_ready", False):
        lib.oracle_completion.argtypes = [_DP, _DP, ctypes.c_int64, ctypes.c_int, _DP, _DP]
        lib._L_ready = True
    centres, radii, mu = _c(centres), _c(radii), _c(mu)
    u = np.empty_like(mu)
    if lib.oracle_completion(_dp(centres), _dp(radii), len(radii), p, _dp(mu), _dp(u)):
        raise ValueError("completion: bad arguments")
    return u


def _load_near_off():
    lib = _load_near()
    if not getattr(lib, "_near_off_ready", False):
        i64, i32, d = ctypes.c_int64, ctypes.c_int, ctypes.c_double
        lib.oracle_exterior_pressure.argtypes = [i32, _DP, d, d, _DP, _DP, _DP, i64, _DP]
        lib.oracle_near_offsurface.argtypes = [_DP, _DP, i64, i32, d, _DP, _DP, d, _DP, i64, _DP, _DP]
        lib._near_off_ready = True
    return lib


def exterior_pressure(p, centre, a, mu, f_s, q_s, targets):
    """Exterior pressure of ONE sphere's expansion (D per reading R12)."""
    lib = _load_near_off()
    c = _c(np.asarray(centre, dtype=np.float64).reshape(3))
    f_s, q_s, targets = _c(f_s), _c(q_s), _c(targets)
    pr = np.empty(targets.shape[0])
    if lib.oracle_exterior_pressure(p, _dp(c), a, mu, _dp(f_s), _dp(q_s), _dp(targets),
                                    targets.shape[0], _dp(pr)):
        raise ValueError("exterior_pressure: bad arguments")
    return pr


def near_offsurface(centres, radii, p, mu, f, q, eta, targets):
    """Near correction (du, dp) at arbitrary targets (point-to-surface eq 4.5)."""
    lib = _load_near_off()
    centres, radii, f, q, targets = _c(centres), _c(radii), _c(f), _c(q), _c(targets)
    M = targets.shape[0]
    du, dp = np.empty((M, 3)), np.empty(M)
    if lib.oracle_near_offsurface(_dp(centres), _dp(radii), len(radii), p, mu, _dp(f), _dp(q), eta,
                                  _dp(targets), M, _dp(du), _dp(dp)):
        raise ValueError("near_offsurface: bad arguments")
    return du, dp


def offsurface_near(centres, radii, p, mu, f, q, eta, targets):
    """Corrected off-surface evaluator: smooth sum + near correction."""
    u, pr = offsurface(centres, radii, p, mu, f, q, targets)
    du, dp = near_offsurface(centres, radii, p, mu, f, q, eta, targets)
    return u + du, pr + dp


# ---------------------------------------------------------------- NEXT-4
def _load_next4():
    lib = _load()
    if not getattr(lib, "_next4_ready", False):
        i64, i32, d = ctypes.c_int64, ctypes.c_int, ctypes.c_double
        lib.oracle_next4_rotate_density.argtypes = [i32, _DP, _DP, _DP]
        lib.oracle_vsh_project.argtypes = [i32, _DP, _DP]
        lib.oracle_vsh_expand.argtypes = [i32, _DP, _DP, i64, _DP]
        lib.oracle_next4_pair.argtypes = [i32, _DP, d, _DP, d, d, _DP, _DP, _DP]
        lib.oracle_near4.argtypes = [_DP, _DP, i64, i32, d, _DP, _DP, d, _I64P, i64, _DP]
        lib._next4_ready = True
    return lib


def next4_rotation(cs, ct):
    """Q = Rz(alpha) Ry(beta) with Q e_z = (ct - cs)/|ct - cs| (reading R25);
    the same definition as oracle.cpp's next4_rotation, for the tests."""
    d = np.asarray(ct, dtype=np.float64) - np.asarray(cs, dtype=np.float64)
    d = d / np.linalg.norm(d)
    beta, alpha = np.arccos(np.clip(d[2], -1.0, 1.0)), np.arctan2(d[1], d[0])
    ca, sa, cb, sb = np.cos(alpha), np.sin(alpha), np.cos(beta), np.sin(beta)
    Rz = np.array([[ca, -sa, 0.0], [sa, ca, 0.0], [0.0, 0.0, 1.0]])
    Ry = np.array([[cb, 0.0, sb], [0.0, 1.0, 0.0], [-sb, 0.0, cb]])
    return Rz @ Ry


def rotate_density(p, Q, g):
    """Stage (1) of NEXT-4: gR_k = Q^T g(Q n_k) on the order-p grid, g the
    degree-<=p expansion of the nodal density g [nsn, 3]."""
    lib = _load_next4()
    Q, g = _c(np.asarray(Q).reshape(9)), _c(g)
    out = np.empty_like(g)
    if lib.oracle_next4_rotate_density(p, _dp(Q), _dp(g), _dp(out)):
        raise ValueError("rotate_density: bad arguments")
    return out


def vsh_project(p, g):
    """Discrete VSH coefficients of a nodal density: complex [(p+1)^2, 3],
    row n*n + n + m, columns (V, W, X)."""
    lib = _load_next4()
    g = _c(g)
    out = np.empty(2 * 3 * (p + 1) ** 2)
    if lib.oracle_vsh_project(p, _dp(g), _dp(out)):
        raise ValueError("vsh_project: bad arguments")
    return (out[0::2] + 1j * out[1::2]).reshape((p + 1) ** 2, 3)


def vsh_expand(p, alpha, dirs):
    """Re sum alpha Z(u) at unit directions dirs [M, 3] (pole-safe)."""
    lib = _load_next4()
    a = np.asarray(alpha, dtype=complex).reshape(-1)
    buf = _c(np.stack([a.real, a.imag], -1).reshape(-1))
    dirs = _c(dirs)
    out = np.empty((len(dirs), 3))
    if lib.oracle_vsh_expand(p, _dp(buf), _dp(dirs), len(dirs), _dp(out)):
        raise ValueError("vsh_expand: bad arguments")
    return out


def next4_pair(p, cs, a_s, ct, a_t, mu, f_s, q_s):
    """Stages (1)-(3) of PAPER §4.2 (Fig 2) for one pair: the NEXT-4 estimate
    of S[f_s] + D[q_s] of sphere (cs, a_s) at the nodes of sphere (ct, a_t)."""
    lib = _load_next4()
    cs = _c(np.asarray(cs, dtype=np.float64).reshape(3))
    ct = _c(np.asarray(ct, dtype=np.float64).reshape(3))
    f_s, q_s = _c(f_s), _c(q_s)
    nsn = (p + 1) * (2 * p + 2)
    out = np.empty((nsn, 3))
    if lib.oracle_next4_pair(p, _dp(cs), a_s, _dp(ct), a_t, mu, _dp(f_s), _dp(q_s), _dp(out)):
        raise ValueError("next4_pair: bad arguments")
    return out


def near4(centres, radii, p, mu, f, q, eta, subset=None):
    """NEXT-4 near correction du (NEXT-4 estimate minus smooth rule) at nodes `subset`."""
    lib = _load_next4()
    centres, radii, f, q = _c(centres), _c(radii), _c(f), _c(q)
    N = len(radii) * (p + 1) * (2 * p + 2)
    idx = _subset(subset, N)
    du = np.empty((len(idx), 3))
    if lib.oracle_near4(_dp(centres), _dp(radii), len(radii), p, mu, _dp(f), _dp(q), eta,
                        idx.ctypes.data_as(_I64P), len(idx), _dp(du)):
        raise ValueError("near4: bad arguments")
    return du


def apply_near4(centres, radii, p, mu, f, q, eta, subset=None):
    """Composite apply with the NEXT-4 near evaluation: far + self + near4."""
    return apply(centres, radii, p, mu, f, q, subset) + near4(centres, radii, p, mu, f, q, eta, subset)
