"""ctypes binding of the C ABI declared in include/cpr_b200.h.

The shared library is built in-tree by build_native.py.  There is no Python
or CPU fallback for any device entry point: if the library is missing the
import of a device path raises.
"""

from __future__ import annotations

import ctypes as C
import os
import warnings
from pathlib import Path

import numpy as np

_LIB_PATH = Path(os.environ.get("CPRB_LIB") or
                 Path(__file__).resolve().parent / "_native" / "libcprb200.so")
_lib = None

OK, EINVAL, ENONFINITE, ESINGULAR, EDEVICE, ERUNTIME, EUNSUPPORTED = range(7)

i64p = C.POINTER(C.c_int64)
i32p = C.POINTER(C.c_int32)
f64p = C.POINTER(C.c_double)
u8p = C.POINTER(C.c_uint8)
vp = C.c_void_p


class Sell(C.Structure):
    _fields_ = [("nslices", C.c_int32), ("nrows", C.c_int32), ("slice_ptr", vp),
                ("lane_row", vp), ("lane_len", vp), ("lane_len_lo", vp), ("cols", vp),
                ("vals", vp), ("agg_out", vp)]


class AmgLevel(C.Structure):
    _fields_ = [("n", C.c_int32), ("ncolors", C.c_int32), ("color_slices", i32p),
                ("color_rows", i32p), ("color_snapshot", u8p), ("smoother", Sell),
                ("diag", vp), ("restrict_op", Sell), ("aggp", vp), ("b", vp), ("x", vp),
                ("tmp", vp), ("color_width", i32p), ("restrict_width", C.c_int32),
                ("pad_", C.c_int32)]


class Amg(C.Structure):
    _fields_ = [("nlevels", C.c_int32), ("levels", C.POINTER(AmgLevel)), ("n_coarse", C.c_int32),
                ("coarse_inv", vp), ("coarse_b", vp), ("coarse_x", vp), ("perm0", vp),
                ("in_stride", C.c_int32), ("cycle", C.c_int32), ("use_fcg", C.c_int32),
                ("kwork", vp), ("kwork_len", C.c_int64), ("tail_start", C.c_int32),
                ("tail_nphases", C.c_int32), ("tail_nchunks", C.c_int32), ("tail_slot", C.c_int32),
                ("tail_smem", C.c_int32), ("tail_vec_len", C.c_int32), ("tail_phases", vp),
                ("tail_chunks", vp), ("tail_stream", vp), ("tail_vec", vp),
                ("tail_stream_bytes", C.c_int64)]


class Wave(C.Structure):
    _fields_ = [("nchunks", C.c_int32), ("nsteps", C.c_int32), ("stage_max", C.c_int32),
                ("rhs_max", C.c_int32), ("chunk_step", vp), ("step_off", vp), ("step_bytes", vp),
                ("step_w", vp), ("step_k", vp), ("rhs_off", vp), ("rhs_bytes", vp),
                ("stream", vp), ("max_chunk_steps", C.c_int32), ("pad_", C.c_int32)]


class Stencil(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32), ("S", C.c_int32),
                ("D", C.c_int32), ("P", C.c_int32), ("doff", vp), ("lrec", vp), ("urec", vp)]


class Bilu(C.Structure):
    _fields_ = [("n", C.c_int32), ("b", C.c_int32), ("L", Sell), ("U", Sell), ("uinv", vp),
                ("tickets", vp), ("use_wave", C.c_int32), ("Lw", Wave), ("Uw", Wave),
                ("l_slot", vp), ("rhs_l", vp), ("rhs_u", vp), ("u_slot", vp), ("zl_step", vp),
                ("y_step", vp), ("len_l", C.c_int64), ("len_u", C.c_int64), ("St", Stencil)]


class Cpr(C.Structure):
    _fields_ = [("nb", C.c_int32), ("b", C.c_int32), ("A", Sell), ("amg", Amg), ("bilu", Bilu),
                ("zp", vp), ("r2", vp), ("zl", vp), ("y", vp)]


_SIGS = {
    "cprb_last_error": (C.c_char_p, []),
    "cprb_version": (C.c_int, []),
    "cprb_strong_connections": (C.c_int, [C.c_int64, i64p, i64p, f64p, C.c_double, i64p, i64p]),
    "cprb_vertices_grouping": (C.c_int, [C.c_int64, i64p, i64p, i64p, i64p, i64p]),
    "cprb_pairwise_aggregate": (C.c_int, [C.c_int64, i64p, i64p, f64p, C.c_double, i64p, i64p]),
    "cprb_galerkin": (C.c_int, [C.c_int64, i64p, i64p, f64p, i64p, C.c_int64, i64p, i64p, f64p,
                                i64p]),
    "cprb_is_symmetric": (C.c_int, [C.c_int64, i64p, i64p, f64p, C.c_double, i32p]),
    "cprb_bilu0_factorize": (C.c_int, [C.c_int64, C.c_int32, i64p, i64p, f64p, f64p, i64p, i64p]),
    "cprb_level_schedule": (C.c_int, [C.c_int64, i64p, i64p, i64p, i64p]),
    "cprb_dense_inverse": (C.c_int, [C.c_int64, f64p, f64p]),
    "cprb_invert_small_blocks": (C.c_int, [C.c_int64, C.c_int32, f64p, f64p]),
    "cprb_spmv": (C.c_int, [C.POINTER(Sell), C.c_int32, vp, vp, vp, vp]),
    "cprb_residual": (C.c_int, [C.POINTER(Sell), C.c_int32, vp, vp, vp, vp, vp]),
    "cprb_pgs_scm_pass": (C.c_int, [C.POINTER(AmgLevel), vp, vp, C.c_int32, C.c_int32, vp]),
    "cprb_amg_cycle": (C.c_int, [C.POINTER(Amg), vp, vp, vp]),
    "cprb_bilu_apply": (C.c_int, [C.POINTER(Bilu), vp, vp, vp, vp]),
    "cprb_cpr_apply": (C.c_int, [C.POINTER(Cpr), vp, vp, vp]),
    "cprb_wave_set_log": (C.c_int, [vp]),
    "cprb_stencil_set_log": (C.c_int, [vp]),
    "cprb_pack_bsr_sell": (C.c_int, [C.c_int64, C.c_int32, vp, vp, vp, vp, vp, vp, vp]),
    "cprb_scalar_split": (C.c_int, [C.c_int64, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "cprb_sell_fill_lanes": (C.c_int, [C.c_int64, vp, vp, vp, vp, C.c_int32, vp, vp]),
    "cprb_sell_fill_rows": (C.c_int, [C.c_int64, vp, vp, vp, vp, vp, vp, vp, vp]),
    "cprb_lower_level_schedule": (C.c_int, [C.c_int64, vp, vp, vp, vp]),
    "cprb_detect_stencil": (C.c_int, [C.c_int64, vp, vp, vp]),
    "cprb_bilu0_factorize_device": (C.c_int, [C.c_int64, C.c_int32, vp, vp, vp, vp, vp, vp,
                                              C.c_int64, vp, vp, vp]),
    "cprb_stencil_pack": (C.c_int, [C.c_int64, C.c_int32, C.c_int32, C.c_int32, vp, vp, vp, vp,
                                    vp, vp, vp, vp, vp]),
    "cprb_vtail_set_log": (C.c_int, [vp]),
    "cprb_mm_read_coord": (C.c_int, [C.c_char_p, vp, vp, vp, vp, vp]),
    "cprb_mm_write_entries": (C.c_int, [C.c_char_p, C.c_int64, vp, vp, vp]),
    "cprb_gen_row_counts": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, vp, vp]),
    "cprb_gen_assemble": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, C.c_double, vp, vp, vp, vp,
                                    vp, vp, vp]),
    "cprb_kcycle_create": (C.c_int, [vp, vp, C.c_int32, C.c_int32, vp]),
    "cprb_kcycle_destroy": (C.c_int, [vp]),
    "cprb_kcycle_correction": (C.c_int, [vp, C.c_int32, vp, vp, vp, vp]),
    "cprb_wave_solve_part": (C.c_int, [vp, C.c_int32, C.c_int32, C.c_int32, vp, vp, vp, vp, vp]),
    "cprb_l_to_u_rows": (C.c_int, [vp, C.c_int32, C.c_int32, vp, vp, vp]),
    "cprb_wave_combine_rows": (C.c_int, [vp, C.c_int32, C.c_int32, vp, vp, vp, vp]),
    "cprb_fill_sentinel_idx": (C.c_int, [C.c_int64, C.c_int32, vp, vp, vp]),
    "cprb_stage2_residual_steps": (C.c_int, [vp, vp, C.c_int32, vp, vp, vp, vp, vp, vp]),
    "cprb_stage2_residual": (C.c_int, [vp, C.c_int32, vp, vp, vp, vp]),
    "cprb_pgs_scm_color": (C.c_int, [vp, C.c_int32, vp, vp, C.c_int32, vp, C.c_int32, vp, vp, vp]),
    "cprb_seg_partials": (C.c_int, [C.c_int64, C.c_int64, vp, vp, vp, vp, vp, vp]),
    "cprb_seg_finish": (C.c_int, [C.c_int32, vp, vp, vp, C.c_int32, vp]),
    "cprb_div_if_nonzero": (C.c_int, [C.c_int64, vp, vp, vp]),
    "cprb_scatter_add": (C.c_int, [C.c_int64, vp, vp, vp, vp]),
    "cprb_gather": (C.c_int, [C.c_int64, vp, vp, C.c_int32, vp, vp]),
    "cprb_unpad": (C.c_int, [C.c_int32, C.c_int64, vp, vp, vp, vp]),
    "cprb_cpr_combine": (C.c_int, [C.c_int64, C.c_int32, vp, vp, vp, vp]),
    "cprb_amg_set_log": (C.c_int, [vp]),
    "cprb_coarse_solve": (C.c_int, [C.POINTER(Amg), vp, vp, vp]),
    "cprb_resid_restrict": (C.c_int, [C.POINTER(AmgLevel), vp, vp, vp, vp]),
    "cprb_prolong": (C.c_int, [C.POINTER(AmgLevel), vp, vp, vp]),
    "cprb_graph_cache_create": (C.c_int, [C.POINTER(C.c_void_p)]),
    "cprb_graph_cache_destroy": (C.c_int, [vp]),
    "cprb_cpr_apply_graph": (C.c_int, [vp, C.POINTER(Cpr), vp, vp, vp]),
    "cprb_amg_cycle_graph": (C.c_int, [vp, C.POINTER(Amg), vp, vp, vp]),
    "cprb_cpr_finish": (C.c_int, [C.POINTER(Cpr), vp, vp, vp]),
    "cprb_div_host": (C.c_int, [C.c_int64, vp, C.c_double, vp, vp]),
    "cprb_dot": (C.c_int, [C.c_int64, vp, vp, vp, vp, vp, vp]),
    "cprb_arnoldi_mgs": (C.c_int, [C.c_int64, C.c_int32, vp, C.c_int64, vp, vp, vp, vp]),
    "cprb_gemv_t": (C.c_int, [C.c_int64, C.c_int32, vp, C.c_int64, vp, vp, vp]),
    "cprb_add": (C.c_int, [C.c_int64, vp, vp, vp, vp]),
    "cprb_axpy": (C.c_int, [C.c_int64, C.c_double, vp, vp, vp, vp]),
    "cprb_div_scalar": (C.c_int, [C.c_int64, vp, vp, vp, vp]),
    "cprb_norm2": (C.c_int, [C.c_int64, vp, vp, vp, vp, vp]),
    "cprb_gmres_solve": (C.c_int, [vp, C.c_int32, vp, vp, C.c_int64, vp, vp, C.c_int32, C.c_int32,
                                   C.c_double, vp, vp, vp, vp]),
}

# every symbol include/cpr_b200.h declares (checked by tests/test_native_abi.py)
EXPORTS = tuple(_SIGS)


def lib():
    """Load the native library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            raise RuntimeError(
                f"native library {_LIB_PATH} is missing; build it with "
                "`python -m paper_2201_01970_b200.build_native` (no CPU fallback exists)")
        L = C.CDLL(str(_LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int, what: str = "") -> None:
    if rc == OK:
        return
    msg = lib().cprb_last_error().decode(errors="replace")
    if what and not msg:
        msg = what
    if rc == EINVAL:
        raise ValueError(msg)
    if rc == ENONFINITE:
        raise FloatingPointError(msg)
    if rc == ESINGULAR:
        raise np.linalg.LinAlgError(msg)
    if rc == EUNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(msg)


def p64(a: np.ndarray):
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(i64p)


def pf64(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(f64p)


def p32(a: np.ndarray):
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(i32p)


def warn(msg: str, category=RuntimeWarning, stacklevel: int = 3) -> None:
    warnings.warn(msg, category, stacklevel=stacklevel)
