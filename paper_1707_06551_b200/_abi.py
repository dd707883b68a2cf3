"""ctypes binding of libbie.so (include/bie.h).  Argument marshalling only:
every arithmetic step runs in the CUDA kernels behind the C ABI.  There is no
fallback -- importing this module fails loudly when libbie.so is missing.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libbie.so")

BIE_OK, BIE_ERR_ARG, BIE_ERR_GEOMETRY, BIE_ERR_ALLOC, BIE_ERR_CUDA, BIE_ERR_UNSUPPORTED = range(6)
BIE_P_MAX = 32
BIE_PART_FAR, BIE_PART_SELF, BIE_PART_COMPLETION = 1, 2, 4
KINDS = ("setup", "self", "pack", "nbody", "reduce", "offsurface", "copy", "near", "krylov", "kfar", "complete",
         "near4")
BIE_NUM_KINDS = len(KINDS)

#: every symbol include/bie.h declares (checked by tests/test_abi_cpu.py)
SYMBOLS = (
    "bie_create", "bie_destroy", "bie_num_nodes", "bie_order", "bie_num_spheres",
    "bie_get_nodes", "bie_apply_SLDL", "bie_apply_SL", "bie_apply_DL", "bie_apply_parts",
    "bie_eval_offsurface", "bie_apply_SLDL_host", "bie_eval_offsurface_host",
    "bie_set_profiling", "bie_get_profile", "bie_reset_profile", "bie_set_source_chunks",
    "bie_set_self_kernel", "bie_set_near_mode", "bie_set_near_exclusion", "bie_set_near_off_schedule", "bie_set_far_reduction",
    "bie_near_lists",
    "bie_set_near", "bie_near_pairs", "bie_solve_porous", "bie_apply_K", "bie_eval_traction",
    "bie_status_string", "bie_last_error",
)

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libbie.so not built at {LIB_PATH}: run `python -c 'import __graft_entry__ as g; g.build()'`")

_lib = ctypes.CDLL(LIB_PATH)
_vp, _i64, _i32, _d = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
_DP = ctypes.POINTER(ctypes.c_double)

_lib.bie_create.argtypes = [_vp, _vp, _i64, _i32, _d, ctypes.POINTER(_vp)]
_lib.bie_destroy.argtypes = [_vp]
_lib.bie_destroy.restype = None
_lib.bie_num_nodes.argtypes = [_vp]
_lib.bie_num_nodes.restype = _i64
_lib.bie_order.argtypes = [_vp]
_lib.bie_num_spheres.argtypes = [_vp]
_lib.bie_num_spheres.restype = _i64
_lib.bie_get_nodes.argtypes = [_vp, _vp, _vp, _vp, _vp]
_lib.bie_apply_SLDL.argtypes = [_vp, _vp, _vp, _vp, _vp]
_lib.bie_apply_SL.argtypes = [_vp, _vp, _vp, _vp]
_lib.bie_apply_DL.argtypes = [_vp, _vp, _vp, _vp]
_lib.bie_apply_parts.argtypes = [_vp, _vp, _vp, _vp, _i32, _vp]
_lib.bie_eval_offsurface.argtypes = [_vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp]
_lib.bie_apply_SLDL_host.argtypes = [_vp, _vp, _vp, _vp, _vp]
_lib.bie_eval_offsurface_host.argtypes = [_vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp]
_lib.bie_set_profiling.argtypes = [_vp, _i32]
_lib.bie_get_profile.argtypes = [_vp, _DP, ctypes.POINTER(_i64)]
_lib.bie_reset_profile.argtypes = [_vp]
_lib.bie_set_source_chunks.argtypes = [_vp, _i32]
_lib.bie_set_self_kernel.argtypes = [_vp, _i32]
_lib.bie_set_near_mode.argtypes = [_vp, _i32]
_lib.bie_set_near_off_schedule.argtypes = [_vp, _i32]
_lib.bie_set_near_exclusion.argtypes = [_vp, _i32]
_lib.bie_near_lists.argtypes = [_vp, _vp, _i64, _d, _vp, _vp, _i64, ctypes.POINTER(_i64)]
_lib.bie_set_far_reduction.argtypes = [_vp, _i32]
_lib.bie_set_near.argtypes = [_vp, _d]
_lib.bie_near_pairs.argtypes = [_vp]
_lib.bie_near_pairs.restype = _i64
_lib.bie_apply_K.argtypes = [_vp, _vp, _vp, _i32, _vp]
_lib.bie_eval_traction.argtypes = [_vp, _vp, _vp, _vp, _i64, _vp, _vp]
_lib.bie_solve_porous.argtypes = [_vp, _vp, _vp, _d, _i32, _i32, _i32, ctypes.POINTER(_i32),
                                  ctypes.POINTER(_d), _vp]
_lib.bie_status_string.argtypes = [_i32]
_lib.bie_status_string.restype = ctypes.c_char_p
_lib.bie_last_error.argtypes = [_vp]
_lib.bie_last_error.restype = ctypes.c_char_p


class BieError(RuntimeError):
    def __init__(self, status: int, msg: str = ""):
        self.status = status
        s = _lib.bie_status_string(status).decode()
        super().__init__(f"{s} ({status}){': ' + msg if msg else ''}")


class Context:
    """Owning handle of a bie_ctx*; destroyed on close() / garbage collection."""

    def __init__(self, handle: int):
        self.handle = handle

    @property
    def _as_parameter_(self):
        return self.handle

    def close(self):
        if self.handle:
            _lib.bie_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def _ptr(x, *, device: bool, n: int | None = None):
    """Raw pointer of None / int / torch tensor / numpy array (float64, contiguous)."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):  # torch.Tensor
        import torch
        if x.dtype != torch.float64 or not x.is_contiguous():
            raise TypeError("expected a contiguous float64 tensor")
        if device != x.is_cuda:
            raise TypeError("expected a CUDA tensor" if device else "expected a CPU tensor")
        if n is not None and x.numel() != n:
            raise ValueError(f"expected {n} elements, got {x.numel()}")
        return x.data_ptr()
    import numpy as np
    if isinstance(x, np.ndarray):
        if device:
            raise TypeError("numpy arrays are host memory; use the *_host entry points")
        if x.dtype != np.float64 or not x.flags["C_CONTIGUOUS"]:
            raise TypeError("expected a C-contiguous float64 array")
        if n is not None and x.size != n:
            raise ValueError(f"expected {n} elements, got {x.size}")
        return x.ctypes.data
    raise TypeError(f"cannot pass {type(x)!r} as a buffer")


def _stream(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _check(ctx, rc):
    if rc != BIE_OK:
        raise BieError(rc, _lib.bie_last_error(ctx.handle if ctx else None).decode() if ctx else "")


# ------------------------------------------------------------ entry points
def bie_create(centres, radii, p: int, mu: float = 1.0) -> Context:
    import numpy as np
    c = np.ascontiguousarray(centres, dtype=np.float64).reshape(-1, 3)
    a = np.ascontiguousarray(radii, dtype=np.float64).reshape(-1)
    if c.shape[0] != a.shape[0]:
        raise ValueError("centres and radii disagree on the number of spheres")
    h = _vp()
    rc = _lib.bie_create(c.ctypes.data if c.size else None, a.ctypes.data if a.size else None,
                         a.shape[0], int(p), float(mu), ctypes.byref(h))
    if rc != BIE_OK:
        raise BieError(rc)
    return Context(h.value)


def bie_destroy(ctx: Context) -> None:
    ctx.close()


def bie_num_nodes(ctx: Context) -> int:
    return int(_lib.bie_num_nodes(ctx.handle))


def bie_order(ctx: Context) -> int:
    return int(_lib.bie_order(ctx.handle))


def bie_num_spheres(ctx: Context) -> int:
    return int(_lib.bie_num_spheres(ctx.handle))


def bie_get_nodes(ctx, x=None, normals=None, w=None, stream=None):
    N = bie_num_nodes(ctx)
    _check(ctx, _lib.bie_get_nodes(ctx.handle, _ptr(x, device=True, n=3 * N),
                                   _ptr(normals, device=True, n=3 * N), _ptr(w, device=True, n=N),
                                   _stream(stream)))


def bie_apply_SLDL(ctx, f, q, u, stream=None):
    N = bie_num_nodes(ctx)
    _check(ctx, _lib.bie_apply_SLDL(ctx.handle, _ptr(f, device=True, n=3 * N),
                                    _ptr(q, device=True, n=3 * N), _ptr(u, device=True, n=3 * N),
                                    _stream(stream)))


def bie_apply_SL(ctx, f, u, stream=None):
    N = bie_num_nodes(ctx)
    _check(ctx, _lib.bie_apply_SL(ctx.handle, _ptr(f, device=True, n=3 * N),
                                  _ptr(u, device=True, n=3 * N), _stream(stream)))


def bie_apply_DL(ctx, q, u, stream=None):
    N = bie_num_nodes(ctx)
    _check(ctx, _lib.bie_apply_DL(ctx.handle, _ptr(q, device=True, n=3 * N),
                                  _ptr(u, device=True, n=3 * N), _stream(stream)))


def bie_apply_parts(ctx, f, q, u, parts: int, stream=None):
    N = bie_num_nodes(ctx)
    _check(ctx, _lib.bie_apply_parts(ctx.handle, _ptr(f, device=True, n=3 * N),
                                     _ptr(q, device=True, n=3 * N), _ptr(u, device=True, n=3 * N),
                                     int(parts), _stream(stream)))


def bie_apply_K(ctx, sigma, u, parts=BIE_PART_FAR | BIE_PART_SELF, stream=None):
    """u = K_pv[sigma] (traction operator, NEXT-3); with BIE_PART_COMPLETION in
    `parts` also the completion L[sigma] of eq 5.8 (reading R22)."""
    N = bie_num_nodes(ctx)
    _check(ctx, _lib.bie_apply_K(ctx.handle, _ptr(sigma, device=True, n=3 * N),
                                 _ptr(u, device=True, n=3 * N), int(parts), _stream(stream)))


def bie_eval_traction(ctx, sigma, targets, normals, t, stream=None):
    """t = K[sigma](x; n) at arbitrary targets with normals (NEXT-3 off the surface)."""
    N = bie_num_nodes(ctx)
    m = (targets.numel() if hasattr(targets, "numel") else targets.size) // 3
    _check(ctx, _lib.bie_eval_traction(ctx.handle, _ptr(sigma, device=True, n=3 * N),
                                       _ptr(targets, device=True, n=3 * m),
                                       _ptr(normals, device=True, n=3 * m), m,
                                       _ptr(t, device=True, n=3 * m), _stream(stream)))


def bie_eval_offsurface(ctx, f, q, targets, u, p=None, stream=None):
    N = bie_num_nodes(ctx)
    m = 0 if targets is None else (targets.numel() if hasattr(targets, "numel") else targets.size) // 3
    _check(ctx, _lib.bie_eval_offsurface(ctx.handle, _ptr(f, device=True, n=3 * N),
                                         _ptr(q, device=True, n=3 * N),
                                         _ptr(targets, device=True, n=3 * m), m,
                                         _ptr(u, device=True, n=3 * m), _ptr(p, device=True, n=m),
                                         _stream(stream)))


def bie_apply_SLDL_host(ctx, f_h, q_h, u_h, stream=None):
    N = bie_num_nodes(ctx)
    _check(ctx, _lib.bie_apply_SLDL_host(ctx.handle, _ptr(f_h, device=False, n=3 * N),
                                         _ptr(q_h, device=False, n=3 * N),
                                         _ptr(u_h, device=False, n=3 * N), _stream(stream)))


def bie_eval_offsurface_host(ctx, f_h, q_h, targets_h, u_h, p_h=None, stream=None):
    N = bie_num_nodes(ctx)
    m = (targets_h.numel() if hasattr(targets_h, "numel") else targets_h.size) // 3
    _check(ctx, _lib.bie_eval_offsurface_host(ctx.handle, _ptr(f_h, device=False, n=3 * N),
                                              _ptr(q_h, device=False, n=3 * N),
                                              _ptr(targets_h, device=False, n=3 * m), m,
                                              _ptr(u_h, device=False, n=3 * m),
                                              _ptr(p_h, device=False, n=m), _stream(stream)))


def bie_set_profiling(ctx, enable: bool = True):
    _check(ctx, _lib.bie_set_profiling(ctx.handle, int(bool(enable))))


def bie_get_profile(ctx):
    """{kind: (milliseconds, launches)} since the last reset."""
    ms = (ctypes.c_double * BIE_NUM_KINDS)()
    ln = (ctypes.c_int64 * BIE_NUM_KINDS)()
    _check(ctx, _lib.bie_get_profile(ctx.handle, ms, ln))
    return {k: (ms[i], ln[i]) for i, k in enumerate(KINDS)}


def bie_reset_profile(ctx):
    _check(ctx, _lib.bie_reset_profile(ctx.handle))


def bie_set_source_chunks(ctx, chunks: int):
    _check(ctx, _lib.bie_set_source_chunks(ctx.handle, int(chunks)))


def bie_set_self_kernel(ctx, variant: int):
    """Self-term kernel: -1 auto (default), 0 DMMA contractions (k_sht), 1 DFMA,
    2 the one-CTA-per-sphere scalar kernel (include/bie.h)."""
    _check(ctx, _lib.bie_set_self_kernel(ctx.handle, int(variant)))


def bie_set_far_reduction(ctx, mode: int):
    """Far-field schedule: 1 chunk partials + k_reduce (default), 0 stream-K, 2/3/4 clusters of 8/4/16."""
    _check(ctx, _lib.bie_set_far_reduction(ctx.handle, int(mode)))


def bie_near_lists(centres, radii, eta: float):
    """Host-side CSR neighbour lists of eq 4.5 (no GPU): (off [n+1], idx)."""
    import numpy as np
    c = np.ascontiguousarray(centres, dtype=np.float64).reshape(-1, 3)
    a = np.ascontiguousarray(radii, dtype=np.float64).reshape(-1)
    n = len(a)
    off = np.zeros(n + 1, dtype=np.int64)
    total = _i64(0)
    rc = _lib.bie_near_lists(c.ctypes.data, a.ctypes.data, n, float(eta), off.ctypes.data, None, 0,
                             ctypes.byref(total))
    if rc:
        raise BieError(rc, "bie_near_lists")
    idx = np.zeros(max(total.value, 1), dtype=np.int32)
    rc = _lib.bie_near_lists(c.ctypes.data, a.ctypes.data, n, float(eta), off.ctypes.data, idx.ctypes.data,
                             len(idx), ctypes.byref(total))
    if rc:
        raise BieError(rc, "bie_near_lists")
    return off, idx[: total.value]


def bie_set_near_exclusion(ctx, mode: int):
    """Near pairs in the far field: 1 skipped, 0 subtracted, -1 auto (include/bie.h)."""
    _check(ctx, _lib.bie_set_near_exclusion(ctx.handle, int(mode)))


def bie_set_near_off_schedule(ctx, schedule: int):
    """Off-surface near correction schedule: 0 pairs grouped by sphere (default),
    1 one thread per Morton-sorted target (include/bie.h)."""
    _check(ctx, _lib.bie_set_near_off_schedule(ctx.handle, int(schedule)))


def bie_set_near_mode(ctx, mode: int):
    """Near evaluation: 0 direct (NEXT-1), 1 rotated (NEXT-4, PAPER §4.2);
    2 / 3 measurement only (exterior part alone), include/bie.h."""
    _check(ctx, _lib.bie_set_near_mode(ctx.handle, int(mode)))


def bie_set_near(ctx, eta: float):
    """Enable (eta > 0) or disable (eta = 0) the near-singular correction."""
    _check(ctx, _lib.bie_set_near(ctx.handle, float(eta)))


def bie_near_pairs(ctx) -> int:
    return int(_lib.bie_near_pairs(ctx.handle))


def bie_solve_porous(ctx, uinf, mu, tol=1e-12, max_iter=400, restart=200, precond=True, stream=None):
    """GMRES solve of BIE 5.4; returns (iterations, true relative residual)."""
    N = bie_num_nodes(ctx)
    it, res = ctypes.c_int(), ctypes.c_double()
    _check(ctx, _lib.bie_solve_porous(ctx.handle, _ptr(uinf, device=True, n=3 * N),
                                      _ptr(mu, device=True, n=3 * N), float(tol), int(max_iter),
                                      int(restart), int(bool(precond)), ctypes.byref(it),
                                      ctypes.byref(res),
                                      _stream(stream)))
    return it.value, res.value


def bie_status_string(status: int) -> str:
    return _lib.bie_status_string(int(status)).decode()


def bie_last_error(ctx) -> str:
    return _lib.bie_last_error(ctx.handle if ctx else None).decode()


def raw_create(centres_ptr, radii_ptr, n_spheres, p, mu):
    """Unchecked call for the ABI contract tests: returns (status, handle)."""
    h = _vp()
    rc = _lib.bie_create(centres_ptr, radii_ptr, n_spheres, p, mu, ctypes.byref(h))
    return rc, h.value
