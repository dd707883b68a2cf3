"""B200 (sm_100a) fp64 Stokes boundary-integral-operator apply for suspensions
of spheres -- the data-parallel hot path of Corona & Veerapaneni,
arXiv 1707.06551.  The compute lives in libbie.so (include/bie.h); this
package is its thin ctypes binding with the same entry-point names.
"""
from ._abi import (  # noqa: F401
    BIE_ERR_ALLOC, BIE_ERR_ARG, BIE_ERR_CUDA, BIE_ERR_GEOMETRY, BIE_ERR_UNSUPPORTED, BIE_OK,
    BIE_P_MAX, BIE_PART_COMPLETION, BIE_PART_FAR, BIE_PART_SELF, KINDS, LIB_PATH, SYMBOLS, BieError, Context,
    bie_apply_DL, bie_apply_K, bie_apply_parts, bie_apply_SL, bie_apply_SLDL, bie_apply_SLDL_host, bie_create,
    bie_destroy, bie_eval_offsurface, bie_eval_offsurface_host, bie_eval_traction, bie_get_nodes, bie_get_profile,
    bie_last_error, bie_near_pairs, bie_num_nodes, bie_set_near, bie_num_spheres, bie_order, bie_reset_profile,
    bie_near_lists, bie_set_far_reduction, bie_set_near_exclusion, bie_set_near_mode, bie_set_near_off_schedule, bie_set_profiling, bie_set_self_kernel, bie_set_source_chunks, bie_solve_porous, bie_status_string,
)
