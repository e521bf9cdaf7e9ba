"""ctypes binding of libgs2b200.so (include/gs2b200.h) and status -> exception mapping.

The library is loaded with ``ctypes.CDLL`` so every call releases the GIL,
like the reference's ``nogil`` numba kernels (_kernels.py:12).  There is no
fallback: if the library cannot be built or loaded, or no CUDA device is
present, the product path raises.
"""

from __future__ import annotations

import ctypes as C
import threading

from . import build as _build

RS_OK = 0
RS_ERR_ARG = -1
RS_ERR_CUDA = -2
RS_ERR_DIAG = -3
RS_ERR_OVERFLOW = -4
RS_ERR_NONFINITE = -5
RS_ERR_SHAPE = -6
RS_ERR_UNSUPPORTED = -7
RS_ERR_PARSE = -8

RS_F64, RS_F32 = 0, 1
DIRECTIONS = {"forward": 0, "backward": 1, "symmetric": 2}
FORMS = {"non_compact": 0, "compact": 1}
PC_KINDS = {"none": 0, "jr": 1, "gs_seq": 2, "sgs_seq": 3, "gs2": 4, "sgs2": 5, "mt_gs": 6, "mt_sgs": 7}
STENCILS = {"laplace2d": 0, "laplace3d": 1, "convdiff3d": 2}


class DivergenceError(RuntimeError):
    """Raised when a solve produces non-finite values (krylov.py:32-33)."""


class RelaxCfg(C.Structure):
    _fields_ = [("n_t", C.c_int), ("n_k", C.c_int), ("n_j", C.c_int), ("direction", C.c_int), ("form", C.c_int),
                ("omega", C.c_double), ("gamma", C.c_double)]

    @classmethod
    def of(cls, cfg) -> "RelaxCfg":
        return cls(int(cfg.n_t), int(cfg.n_k), int(cfg.n_j), DIRECTIONS[cfg.direction], FORMS[cfg.form],
                   float(cfg.omega), float(cfg.gamma))


_P = C.c_void_p
_I64 = C.c_int64
_SIGS = {
    "rs_abi_version": ([], C.c_int),
    "rs_launch_count": ([], C.c_int64),
    "rs_last_error": ([], C.c_char_p),
    "rs_last_error_index": ([], C.c_int64),
    "rs_mat_create_csr": ([C.c_int, _I64, _I64, _I64, _P, _P, _P, C.c_int, C.POINTER(_P)], C.c_int),
    "rs_mat_create_stencil": ([C.c_int, C.c_int, _I64, _I64, _I64, _P, _I64, _I64, C.c_int, C.POINTER(_P)], C.c_int),
    "rs_mat_cast": ([_P, C.c_int, C.POINTER(_P)], C.c_int),
    "rs_mat_destroy": ([_P], C.c_int),
    "rs_mat_info": ([_P, _P, C.POINTER(C.c_int)], C.c_int),
    "rs_mat_layout": ([_P, C.c_int, _P], C.c_int),
    "rs_mat_set_dia": ([_P, C.c_int], C.c_int),
    "rs_mat_export_tri": ([_P, C.c_int, _P, _P, _P, _P], C.c_int),
    "rs_mat_export_diag": ([_P, _P], C.c_int),
    "rs_mat_coloring": ([_P, _P, C.POINTER(C.c_int64)], C.c_int),
    "rs_mat_set_coloring": ([_P, _P, C.c_int64], C.c_int),
    "rs_mt_gs_sweep": ([_P, _P, _P, C.c_int, C.c_double, _P], C.c_int),
    "rs_spmv": ([_P, _P, _P, _P, _P, _P], C.c_int),
    "rs_spmv_dot": ([_P, _P, _P, _P, _P], C.c_int),
    "rs_resid_norm2": ([_P, _P, _P, _P, _P], C.c_int),
    "rs_gs_sweep": ([_P, _P, _P, C.c_int, C.c_double, _P], C.c_int),
    "rs_gs_sweep_w": ([_P, _P, _P, C.c_int, C.c_double, C.c_double, _P], C.c_int),
    "rs_mt_gs_sweep_w": ([_P, _P, _P, C.c_int, C.c_double, C.c_double, _P], C.c_int),
    "rs_jr_sweeps": ([_P, _P, _P, C.c_int, C.c_double, _P], C.c_int),
    "rs_inner_jr": ([_P, _P, _P, C.c_int, C.c_int, C.c_double, C.c_double, _P], C.c_int),
    "rs_gs2_apply": ([_P, _P, _P, C.POINTER(RelaxCfg), _P], C.c_int),
    "rs_gs2_sweep": ([_P, _P, _P, _P, C.POINTER(RelaxCfg), _P], C.c_int),
    "rs_stationary_batch": ([_P, C.c_int, C.POINTER(RelaxCfg), _P, _P, C.c_int, _P, _P], C.c_int),
    "rs_hybrid_bhat": ([_P, _P, _P, _P, _P, _P, _P], C.c_int),
    "rs_precond_apply": ([_P, C.c_int, C.POINTER(RelaxCfg), _P, _P, _P, _P], C.c_int),
    "rs_reduce_work_doubles": ([C.c_int], C.c_int64),
    "rs_gemv_t": ([_P, _I64, C.c_int, _I64, _P, _P, _P, _P, _P], C.c_int),
    "rs_gemv_n_update": ([_P, _I64, C.c_int, _I64, _P, _P, _P, _P, _P], C.c_int),
    "rs_gemv_n": ([_P, _I64, C.c_int, _I64, _P, _P, _P], C.c_int),
    "rs_cgs_pass": ([_P, _I64, C.c_int, _I64, _P, _P, _P, _P, _P, _P, _P], C.c_int),
    "rs_mgs_step": ([_I64, _P, _P, _P, _P, _P, _P, _P], C.c_int),
    "rs_scale_by_norm": ([_I64, _P, _P, _P, _P], C.c_int),
    "rs_sub_norm": ([_I64, _P, _P, _P, _P, _P, _P], C.c_int),
    "rs_dot": ([_I64, _P, _P, _P, _P, _P], C.c_int),
    "rs_axpy1": ([_I64, _P, _P, _P], C.c_int),
    "rs_dot_blas": ([_I64, _P, _P, _P, C.c_int, _P], C.c_int),
    "rs_mgs_step_blas": ([_I64, _P, _P, _P, _P, _P, _P], C.c_int),
    "rs_gemv_n_blas": ([_P, _I64, C.c_int, _I64, _P, _P, _P], C.c_int),
    "rs_host_ddot_blas": ([_I64, _P, _P], C.c_double),
    "rs_host_givens": ([_P, C.c_int, _P, _P, _P, C.c_int], C.c_double),
    "rs_graph_begin": ([_P], C.c_int),
    "rs_graph_end": ([_P, C.POINTER(_P)], C.c_int),
    "rs_graph_launch": ([_P, _P], C.c_int),
    "rs_graph_destroy": ([_P], C.c_int),
    "rs_axpy": ([_I64, C.c_double, _P, _P, _P], C.c_int),
    "rs_xpby": ([_I64, _P, C.c_double, _P, _P], C.c_int),
    "rs_cg_update": ([_I64, _P, _P, _P, _P, _P, _P, _P, _P], C.c_int),
    "rs_xpby_dev": ([_I64, _P, _P, _P, _P, _P], C.c_int),
    "rs_lcg_fill": ([C.c_uint64, _I64, _I64, _P, _P], C.c_int),
    "rs_cast_f64_f32": ([_I64, _P, _P, _P, _P], C.c_int),
    "rs_cast_f32_f64": ([_I64, _P, _P, _P], C.c_int),
    "rs_mm_parse_entries": ([_P, _I64, _I64, _I64, C.c_int, _I64, _I64, _I64, _P, _P, _P, C.POINTER(_I64),
                             C.POINTER(_I64), C.c_int], C.c_int),
    "rs_coo_sort": ([_I64, _I64, _P, _P, _P, _P, C.c_int], C.c_int),
    "rs_peer_create": ([C.c_int, C.c_int, _I64, _I64, _I64, C.POINTER(_P)], C.c_int),
    "rs_peer_ipc_handle": ([_P, _P], C.c_int),
    "rs_peer_connect": ([_P, _P], C.c_int),
    "rs_peer_connect_local": ([_P, _P], C.c_int),
    "rs_peer_set_halo": ([_P, C.c_int, _P, C.c_int, _P], C.c_int),
    "rs_peer_layout": ([_P, C.POINTER(_I64), C.POINTER(_I64)], C.c_int),
    "rs_peer_halo": ([_P, C.c_int, C.POINTER(_P), C.POINTER(_P)], C.c_int),
    "rs_halo_exchange": ([_P, _P, C.c_uint64, _P], C.c_int),
    "rs_peer_allreduce": ([_P, _P, C.c_int, _P, _P, C.c_uint64, _P], C.c_int),
    "rs_cgs_pass_peer": ([_P, _I64, C.c_int, _I64, _P, _P, _P, _P, _P, _P, _P, C.c_uint64, _P, _P, _P], C.c_int),
    "rs_peer_error": ([_P, C.POINTER(C.c_int)], C.c_int),
    "rs_dcgs2_dots": ([_P, _I64, C.c_int, _I64, _P, _P, _P, _P, _P, C.c_uint64, _P], C.c_int),
    "rs_dcgs2_dots_coef": ([_P, _I64, C.c_int, _I64, _P, _P, _P, _P, _P, C.c_uint64, _P, C.c_int, _P, _P, _P,
                            C.c_int, _P, _P, C.c_int, _P], C.c_int),
    "rs_dcgs2_coef": ([C.c_int, _P, _P, C.c_int, _P, _P, C.c_int, _P, C.c_int, _P, _P, C.c_int, _P], C.c_int),
    "rs_dcgs2_update": ([_P, _I64, C.c_int, _I64, _P, _P, _P, _P, _P, _P, _P, C.c_uint64, _P, _P, _P, _P], C.c_int),
    "rs_peer_destroy": ([_P], C.c_int),
}
RS_IPC_HANDLE_BYTES = 64

_lib = None
_lock = threading.Lock()


def lib_path():
    return _build.LIB


def load():
    """Build (if stale) and load libgs2b200.so; raises if that is impossible."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            path = _build.build()
            L = C.CDLL(str(path))
            for name, (args, res) in _SIGS.items():
                f = getattr(L, name)
                f.argtypes = args
                f.restype = res
            if L.rs_abi_version() != 1:
                raise RuntimeError("libgs2b200 ABI version mismatch")
            _lib = L
    return _lib


def exported_symbols():
    return list(_SIGS)


def check(status: int, what: str = ""):
    """Raise the reference's exception type for a non-zero status."""
    if status == RS_OK:
        return
    L = load()
    msg = L.rs_last_error().decode(errors="replace")
    idx = int(L.rs_last_error_index())
    if what:
        msg = f"{what}: {msg}"
    if status in (RS_ERR_ARG, RS_ERR_SHAPE, RS_ERR_DIAG, RS_ERR_UNSUPPORTED):
        err = ValueError(msg)
    elif status == RS_ERR_OVERFLOW:
        err = OverflowError(msg)
    elif status == RS_ERR_NONFINITE:
        err = DivergenceError(msg)
    else:
        err = RuntimeError(msg)
    err.index = idx
    raise err


def call(name: str, *args):
    check(getattr(load(), name)(*args), name)
