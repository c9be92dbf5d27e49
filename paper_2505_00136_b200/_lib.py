"""ctypes binding of the C ABI in ``include/gpb200.h`` (libgpb200.so).

The shared library is built in-tree (``make`` or ``__graft_entry__.build()``)
and loaded from this package directory.  There is no fallback: if the
library is missing, every entry point raises ``ExtensionMissing``.
ctypes releases the GIL for the duration of each foreign call, so device
work never holds the interpreter lock (the reference blocks its caller in
``run_as_root``, runtime.py:250-262, with the same effect).
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from . import errors

LIB_NAME = "libgpb200.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

_lock = threading.Lock()
_lib = None

_c_double_p = ctypes.POINTER(ctypes.c_double)
_c_i64_p = ctypes.POINTER(ctypes.c_int64)
_vp = ctypes.c_void_p

# name -> (restype, argtypes); mirrors include/gpb200.h exactly
SIGNATURES = {
    "gpb_abi_version": (ctypes.c_int, []),
    "gpb_init": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(_vp)]),
    "gpb_finalize": (ctypes.c_int, [_vp]),
    "gpb_current": (_vp, []),
    "gpb_last_error": (ctypes.c_char_p, []),
    "gpb_model_create": (ctypes.c_int, [_vp, _c_double_p, _c_double_p, ctypes.c_int64,
                                        ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(_vp)]),
    "gpb_model_create_device": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int64, ctypes.c_int64,
                                               ctypes.c_int64, ctypes.POINTER(_vp)]),
    "gpb_model_destroy": (ctypes.c_int, [_vp]),
    "gpb_model_set_train": (ctypes.c_int, [_vp, _c_double_p, _c_double_p, ctypes.c_int64,
                                           ctypes.c_int64]),
    "gpb_model_set_params": (ctypes.c_int, [_vp, ctypes.c_double, ctypes.c_double,
                                            ctypes.c_double, ctypes.POINTER(ctypes.c_uint8)]),
    "gpb_model_get_params": (ctypes.c_int, [_vp, _c_double_p]),
    "gpb_cholesky": (ctypes.c_int, [_vp, _c_double_p]),
    "gpb_last_pivot": (ctypes.c_int, [_vp, _c_i64_p]),
    "gpb_log_likelihood": (ctypes.c_int, [_vp, _c_double_p]),
    "gpb_loss_gradients": (ctypes.c_int, [_vp, _c_double_p]),
    "gpb_predict_solve_device": (ctypes.c_int, [_vp, _vp, ctypes.c_int64, ctypes.c_int64, _vp, _vp,
                                                 ctypes.c_int64]),
    "gpb_cov_block_device": (ctypes.c_int, [_vp, _vp, ctypes.c_int64, _vp, ctypes.c_int64, _vp,
                                             ctypes.c_int64, _vp, ctypes.c_int64, _vp, ctypes.c_int64]),
    "gpb_loss_gradient_terms": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_int), ctypes.c_int64,
                                               _c_double_p]),
    "gpb_optimize": (ctypes.c_int, [_vp, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                    ctypes.c_double, ctypes.c_int64, _c_double_p]),
    "gpb_predict": (ctypes.c_int, [_vp, _c_double_p, ctypes.c_int64, ctypes.c_int64,
                                   _c_double_p, _c_double_p, _c_double_p]),
    "gpb_predict_device": (ctypes.c_int, [_vp, _vp, ctypes.c_int64, ctypes.c_int64, _vp, _vp]),
    "gpb_clamp_variances": (ctypes.c_int, [_c_double_p, ctypes.c_int64]),
    "gpb_model_get_adam": (ctypes.c_int, [_vp, _c_double_p, _c_double_p, _c_i64_p]),
    "gpb_model_set_adam": (ctypes.c_int, [_vp, _c_double_p, _c_double_p, ctypes.c_int64]),
    "gpb_model_timings": (ctypes.c_int, [_vp, _c_double_p, ctypes.c_int]),
    "gpb_model_launch_count": (ctypes.c_int, [_vp, _c_i64_p]),
    "gpb_model_set_ozaki": (ctypes.c_int, [_vp, ctypes.c_int]),
    "gpb_model_get_ozaki": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_int), _c_i64_p]),
    "gpb_model_stream": (ctypes.c_int, [_vp, ctypes.POINTER(_vp)]),
    "gpb_model_set_profiling": (ctypes.c_int, [_vp, ctypes.c_int]),
    "gpb_model_kernel_stats": (ctypes.c_int, [_vp, _c_double_p, _c_double_p, _c_i64_p]),
    "gpb_model_kernel_busy": (ctypes.c_int, [_vp, _c_double_p]),
    "gpb_fp64_peak_probe": (ctypes.c_int, [_vp, ctypes.c_double, _c_double_p]),
    "gpb_int8_peak_probe": (ctypes.c_int, [_vp, ctypes.c_double, _c_double_p]),
    "gpb_layout": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int64, _c_i64_p]),
    "gpb_dev_pad": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                   ctypes.c_int64, _vp]),
    "gpb_dev_assemble": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int64, ctypes.c_int64,
                                        ctypes.c_int64, ctypes.c_int64, ctypes.c_double,
                                        ctypes.c_double, ctypes.c_double, ctypes.c_int, _vp,
                                        ctypes.c_int64]),
    "gpb_dev_potrf": (ctypes.c_int, [_vp, _vp, _vp, _vp, ctypes.c_int64, ctypes.c_int64,
                                     ctypes.c_int64, ctypes.c_int64, _vp, _vp]),
    "gpb_dev_gemm": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                    ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_double, ctypes.c_double]),
    "gpb_dev_gemm_tiled": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                          ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_int64, ctypes.c_int64, ctypes.c_double,
                                          ctypes.c_double]),
    "gpb_dev_gemm_mirror": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                           ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                           ctypes.c_int64, ctypes.c_int64, ctypes.c_double,
                                           ctypes.c_double, _vp, ctypes.c_int64]),
    "gpb_dev_ipc_alloc": (ctypes.c_int, [_vp, ctypes.c_int64, ctypes.POINTER(_vp), _vp]),
    "gpb_dev_ipc_open": (ctypes.c_int, [_vp, _vp, ctypes.POINTER(_vp)]),
    "gpb_dev_ipc_close": (ctypes.c_int, [_vp, _vp]),
    "gpb_dev_free": (ctypes.c_int, [_vp, _vp]),
    "gpb_dev_signal": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_uint64]),
    "gpb_dev_wait": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_uint64]),
    "gpb_dev_gemv": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                    ctypes.c_double, ctypes.c_int]),
    "gpb_dev_copy": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int64, ctypes.c_int64]),
    "gpb_dev_combine": (ctypes.c_int, [_vp, _vp, _vp, _vp, ctypes.c_int64, ctypes.c_int64, _vp]),
    "gpb_model_adopt_factor": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "gpb_model_factor_buffers": (ctypes.c_int, [_vp] + [ctypes.POINTER(_vp)] * 5),
    "gpb_model_mark_factored": (ctypes.c_int, [_vp]),
    "gpb_nccl_unique_id": (ctypes.c_int, [_vp]),
    "gpb_dist_init": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp,
                                     ctypes.POINTER(_vp)]),
    "gpb_dist_init_host": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp,
                                          ctypes.POINTER(_vp)]),
    "gpb_dist_init_emulate": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                             ctypes.POINTER(_vp)]),
    "gpb_dist_finalize": (ctypes.c_int, [_vp]),
    "gpb_dist_model_create": (ctypes.c_int, [_vp, _c_double_p, _c_double_p, ctypes.c_int64, ctypes.c_int64,
                                             ctypes.c_int64, ctypes.POINTER(_vp)]),
    "gpb_dist_model_destroy": (ctypes.c_int, [_vp]),
    "gpb_dist_set_params": (ctypes.c_int, [_vp, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                           ctypes.POINTER(ctypes.c_uint8)]),
    "gpb_dist_get_params": (ctypes.c_int, [_vp, _c_double_p]),
    "gpb_dist_factor": (ctypes.c_int, [_vp]),
    "gpb_dist_last_pivot": (ctypes.c_int, [_vp, _c_i64_p]),
    "gpb_dist_log_likelihood": (ctypes.c_int, [_vp, _c_double_p]),
    "gpb_dist_loss_gradients": (ctypes.c_int, [_vp, _c_double_p]),
    "gpb_dist_optimize": (ctypes.c_int, [_vp, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                         ctypes.c_double, ctypes.c_int64, _c_double_p]),
    "gpb_dist_predict": (ctypes.c_int, [_vp, _c_double_p, ctypes.c_int64, ctypes.c_int64, _c_double_p,
                                        _c_double_p, _c_double_p]),
    "gpb_dist_cholesky": (ctypes.c_int, [_vp, _c_double_p]),
    "gpb_dist_timings": (ctypes.c_int, [_vp, _c_double_p, ctypes.c_int]),
    "gpb_dist_launch_count": (ctypes.c_int, [_vp, _c_i64_p]),
    "gpb_dist_plan": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64,
                                     ctypes.c_int64, ctypes.c_int, ctypes.c_int, _vp, _c_i64_p, _vp, _c_i64_p,
                                     _c_i64_p, _c_i64_p]),
    "gpb_dist_set_exchange": (ctypes.c_int, [_vp, ctypes.c_int]),
    "gpb_msd_series_device": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_double,
                                             ctypes.c_double, ctypes.c_double, ctypes.c_double, _vp, _vp]),
    "gpb_tile_potrf": (ctypes.c_int, [_vp, _c_double_p, ctypes.c_int64, _c_double_p]),
    "gpb_tile_trsm": (ctypes.c_int, [_vp, _c_double_p, _c_double_p, ctypes.c_int64,
                                     ctypes.c_int64, _c_double_p]),
    "gpb_tile_syrk": (ctypes.c_int, [_vp, _c_double_p, _c_double_p, ctypes.c_int64,
                                     ctypes.c_int64, _c_double_p]),
    "gpb_tile_gemm": (ctypes.c_int, [_vp, _c_double_p, _c_double_p, _c_double_p,
                                     ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                     _c_double_p]),
}

_STATUS = {
    1: errors.InvalidConfig,
    2: errors.AlreadyRunning,
    3: errors.NotRunning,
    4: errors.TilingError,
    5: errors.DimensionMismatch,
    6: errors.NotPositiveDefinite,
    7: errors.SingularTriangular,
    8: errors.NumericalConsistencyError,
    9: errors.DeviceError,
    10: errors.DeviceError,
    11: errors.DeviceError,
}


class TileDesc(ctypes.Structure):
    """gpb_tile_desc"""
    _fields_ = [("i", ctypes.c_int32), ("j", ctypes.c_int32), ("ptr", ctypes.c_void_p)]


class GemmJob(ctypes.Structure):
    """gpb_gemm_job"""
    _fields_ = [("a", ctypes.c_void_p), ("b", ctypes.c_void_p), ("cin", ctypes.c_void_p),
                ("cout", ctypes.c_void_p), ("k", ctypes.c_int32), ("lower", ctypes.c_int32)]


class GemvJob(ctypes.Structure):
    """gpb_gemv_job"""
    _fields_ = [("a", ctypes.c_void_p), ("x", ctypes.c_void_p), ("y", ctypes.c_void_p)]


class CopyJob(ctypes.Structure):
    """gpb_copy_job"""
    _fields_ = [("src", ctypes.c_void_p), ("dst", ctypes.c_void_p)]


# gpb_host_coll callbacks (host-staged collectives of gpb_dist_init_host)
BCAST_FN = ctypes.CFUNCTYPE(ctypes.c_int, _vp, ctypes.c_int, _vp, ctypes.c_int64, ctypes.c_int)
REDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, _vp, ctypes.c_int, _c_double_p, ctypes.c_int64, ctypes.c_int)
ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, _vp, ctypes.c_int, _c_double_p, ctypes.c_int64)


class HostColl(ctypes.Structure):
    """gpb_host_coll"""
    _fields_ = [("bcast", BCAST_FN), ("reduce_sum", REDUCE_FN), ("allreduce_sum", ALLREDUCE_FN),
                ("user", _vp)]


NCCL_ID_BYTES = 128  # GPB_NCCL_ID_BYTES
BUFFERS = ("L", "DINV", "ROW", "COL", "VEC", "X", "KINV", "XCOL", "XROW", "LCOL")  # GPB_BUF_*
OPS = {1: "ASSEMBLE", 2: "POTRF", 3: "GEMM", 4: "COPY", 5: "GEMV", 6: "COMBINE", 7: "BCAST", 8: "REDUCE",
       9: "ALLREDUCE", 10: "RECORD", 11: "WAIT", 12: "ZERO", 13: "SOLVE_FLOW", 14: "TRACE", 15: "MIRROR",
       16: "SIGNAL", 17: "WAITFLAG", 18: "SLICE"}  # GPB_OP_*
# gpb_op / gpb_op_job as numpy records (the schedule IR of gpb_dist_plan)
OP_DTYPE = np.dtype([("kind", "<i4"), ("stream", "<i4"), ("group", "<i4"), ("root", "<i4"),
                     ("buf", "<i4", 3), ("flag", "<i4"), ("off", "<i8", 3), ("count", "<i8"),
                     ("job0", "<i8"), ("njobs", "<i8"), ("mblk", "<i4"), ("nblk", "<i4"), ("ak", "<i4"),
                     ("bk", "<i4"), ("lda", "<i8"), ("ldb", "<i8"), ("ldc", "<i8"), ("a_ktile", "<i8"),
                     ("a_kstride", "<i8"), ("b_ktile", "<i8"), ("b_kstride", "<i8"), ("alpha", "<f8"),
                     ("beta", "<f8"), ("i", "<i4"), ("j", "<i4")])
JOB_DTYPE = np.dtype([("buf", "<i4", 4), ("off", "<i8", 4), ("k", "<i4"), ("lower", "<i4"), ("i", "<i4"),
                      ("j", "<i4")])
META = ("bi", "Ti", "np", "P", "Q", "G", "nown", "nevents", "Y", "BETA", "ALPHA", "LOGDIAG", "ACC", "TMP",
        "RECV", "RED")


def dist_plan(rank: int, world: int, p: int, q: int, n: int, tiles_per_dim: int, phase: int, exchange: int = 0):
    """One rank's operation list of a phase (gpb_dist_plan; host only, no GPU):
    (ops, jobs, buffer sizes in doubles, meta dict).  exchange 1: peer-memory panels."""
    lib = load()
    nops, njobs = ctypes.c_int64(), ctypes.c_int64()
    bufsz = (ctypes.c_int64 * len(BUFFERS))()
    meta = (ctypes.c_int64 * 16)()
    check(lib.gpb_dist_plan(rank, world, p, q, n, tiles_per_dim, phase, exchange, None, ctypes.byref(nops), None,
                            ctypes.byref(njobs), bufsz, meta))
    ops = np.zeros(nops.value, dtype=OP_DTYPE)
    jobs = np.zeros(max(1, njobs.value), dtype=JOB_DTYPE)
    check(lib.gpb_dist_plan(rank, world, p, q, n, tiles_per_dim, phase, exchange, ops.ctypes.data,
                            ctypes.byref(nops), jobs.ctypes.data, ctypes.byref(njobs), bufsz, meta))
    return ops, jobs[:njobs.value], dict(zip(BUFFERS, bufsz[:])), dict(zip(META, meta[:]))


def layout(n: int, tiles_per_dim: int) -> dict:
    """The library's padded internal layout for (n, tiles_per_dim) (gpb_layout)."""
    out = (ctypes.c_int64 * 6)()
    check(load().gpb_layout(n, tiles_per_dim, out))
    return {"b": out[0], "T": out[1], "np": out[2], "pad_bp": out[3], "pad_b": out[4],
            "user_b": out[5]}


class ExtensionMissing(ImportError):
    """libgpb200.so is not built; there is deliberately no CPU fallback."""


def load():
    """Load (once) and return the CDLL with all signatures declared."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ExtensionMissing(
                f"{LIB_PATH} is missing: build it with `make` or "
                "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)"
            )
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(status: int) -> None:
    """Raise the reference-equivalent exception for a non-zero gpb_status."""
    if status == 0:
        return
    msg = load().gpb_last_error()
    msg = msg.decode("utf-8", "replace") if msg else f"gpb status {status}"
    raise _STATUS.get(status, errors.TaskGPError)(msg)


def dptr(a):
    """double* of a C-contiguous float64 ndarray (None -> NULL)."""
    if a is None:
        return None
    return a.ctypes.data_as(_c_double_p)
