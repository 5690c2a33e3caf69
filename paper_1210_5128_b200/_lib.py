"""ctypes binding of the product C-ABI (include/bnmc_gpu.h, include/bnmc_synth.h).

Loads the in-tree ``paper_1210_5128_b200/libbnmc_b200.so`` (built by
``__graft_entry__.build()`` / ``make -C paper_1210_5128_b200/csrc``). There is no
fallback: if the library is missing, or no sm_100 device is visible when a
compute entry point is called, the call raises.
"""
from __future__ import annotations

import atexit
import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BNMC_B200_LIB") or os.path.join(HERE, "libbnmc_b200.so")

_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_vp = C.c_void_p


class ScoreParams(C.Structure):
    _fields_ = [("max_parents", C.c_int), ("gamma", C.c_double), ("ess", C.c_double),
                ("alpha_mode", C.c_int), ("memory_cap_bytes", C.c_uint64), ("device", C.c_int),
                ("n_gpus", C.c_int)]


class ChainParams(C.Structure):
    _fields_ = [("iterations", C.c_uint64), ("track_top", C.c_int), ("strict", C.c_int),
                ("scan_mode", C.c_int), ("timing_sample", C.c_int), ("team_warps", C.c_int),
                ("exact_accept", C.c_int), ("accept_tol_log2", C.c_int),
                ("debug_recheck", C.c_int)]


# Every exported symbol with its ctypes signature: (restype, argtypes).
SIGNATURES = {
    "bnmc_gpu_last_error_message": (C.c_char_p, []),
    "bnmc_gpu_version": (C.c_int, []),
    "bnmc_gpu_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "bnmc_gpu_host_alloc": (C.c_int, [C.c_uint64, C.POINTER(_vp)]),
    "bnmc_gpu_host_free": (C.c_int, [_vp]),
    "bnmc_gpu_table_estimate_bytes": (C.c_uint64, [C.c_int, C.c_int]),
    "bnmc_gpu_bounded_subset_count": (C.c_uint64, [C.c_int, C.c_int]),
    "bnmc_gpu_table_build": (C.c_int, [_u8p, _i32p, C.c_uint64, C.c_int, C.POINTER(ScoreParams),
                                       _vp, C.POINTER(_vp)]),
    "bnmc_gpu_table_build_rows": (C.c_int, [_u8p, _i32p, C.c_uint64, C.c_int,
                                            C.POINTER(ScoreParams), _vp, C.c_int, C.c_int,
                                            C.POINTER(_vp)]),
    "bnmc_gpu_table_rows_buffer": (C.c_int, [_vp, C.POINTER(_vp), C.POINTER(C.c_uint64),
                                             C.POINTER(C.c_uint64)]),
    "bnmc_gpu_table_finalize": (C.c_int, [_vp]),
    "bnmc_gpu_table_upload": (C.c_int, [_f64p, C.c_int, C.POINTER(ScoreParams), _vp,
                                        C.POINTER(_vp)]),
    "bnmc_gpu_table_set_priors": (C.c_int, [_vp, _vp]),
    "bnmc_gpu_table_info": (C.c_int, [_vp, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                      C.POINTER(C.c_uint64)]),
    "bnmc_gpu_table_download": (C.c_int, [_vp, _f64p]),
    "bnmc_gpu_table_build_ms": (C.c_int, [_vp, C.POINTER(C.c_float), C.POINTER(C.c_float)]),
    "bnmc_gpu_table_free": (C.c_int, [_vp]),
    "bnmc_gpu_count_statistics": (C.c_int, [_u8p, _i32p, C.c_uint64, C.c_int, C.c_int, _i32p,
                                            _u64p, _u64p, _u32p, _u64p, C.c_int]),
    "bnmc_gpu_score_orders": (C.c_int, [_vp, _i32p, C.c_int, _vp, _vp, _vp]),
    "bnmc_gpu_score_order": (C.c_int, [_vp, _i32p, _vp, _vp, _vp]),
    "bnmc_gpu_run_chains": (C.c_int, [_vp, _u64p, C.c_int, C.POINTER(ChainParams), _vp, _vp, _vp,
                                      _vp, _vp, _vp, _vp, _vp, _vp, C.POINTER(C.c_float)]),
    "bnmc_gpu_last_scan_stats": (C.c_int, [_vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                           C.POINTER(C.c_float), C.POINTER(C.c_uint64)]),
    "bnmc_gpu_scan_slice": (C.c_int, [_vp, _i32p, C.c_int, C.c_uint64, C.c_uint64,
                                      C.POINTER(C.c_double), C.POINTER(C.c_uint64)]),
    "bnmc_gpu_table_set_scan_mode": (C.c_int, [_vp, C.c_int]),
    "bnmc_gpu_last_walk_stats": (C.c_int, [_vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                           C.POINTER(C.c_uint64), C.POINTER(C.c_float)]),
    "bnmc_gpu_table_set_walk_params": (C.c_int, [_vp, C.c_int64, C.c_int]),
    "bnmc_gpu_table_set_walk_cap": (C.c_int, [_vp, C.c_int64, C.c_int64, C.c_int]),
    "bnmc_gpu_last_replayed": (C.c_int, [_vp, C.POINTER(C.c_uint64)]),
    "bnmc_gpu_last_walk_variant": (C.c_int, [_vp, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                             C.POINTER(C.c_int)]),
    "bnmc_gpu_bench_scan": (C.c_int, [_vp, _i32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                      C.POINTER(C.c_float), C.POINTER(C.c_uint64)]),
    "bnmc_gpu_k1_partition": (C.c_int, [_i32p, C.c_uint64, C.c_int, C.c_int, C.c_int, _u64p]),
    "bnmc_gpu_table_build_part": (C.c_int, [_u8p, _i32p, C.c_uint64, C.c_int,
                                            C.POINTER(ScoreParams), _vp, C.c_int, C.c_int,
                                            C.POINTER(_vp)]),
    "bnmc_gpu_table_k1_stats": (C.c_int, [_vp, C.POINTER(C.c_float), C.POINTER(C.c_uint64),
                                          C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "bnmc_gpu_count_statistics_sparse": (C.c_int, [_u8p, _i32p, C.c_uint64, C.c_int, C.c_int,
                                                   C.c_uint64, _u64p, _u32p,
                                                   C.POINTER(C.c_uint64), C.c_int]),
    "bnmc_gpu_comm_unique_id": (C.c_int, [_u8p]),
    "bnmc_gpu_comm_init": (C.c_int, [_u8p, C.c_int, C.c_int, C.c_int, C.POINTER(_vp)]),
    "bnmc_gpu_comm_free": (C.c_int, [_vp]),
    "bnmc_gpu_table_build_comm": (C.c_int, [_u8p, _i32p, C.c_uint64, C.c_int,
                                            C.POINTER(ScoreParams), _vp, _vp, C.POINTER(_vp)]),
    "bnmc_gpu_comm_allgather": (C.c_int, [_vp, _vp, C.c_uint64, _vp]),
    "bnmc_gpu_comm_allreduce_max": (C.c_int, [_vp, _f64p, C.c_int]),
    "bnmc_gpu_table_devices": (C.c_int, [_vp, C.POINTER(C.c_int), _i32p]),
    "bnmc_synth_last_error": (C.c_char_p, []),
    "bnmc_synth_instance": (C.c_int, [C.c_int, C.c_int, C.c_double, C.c_double, C.c_uint64,
                                      _i32p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                      _u8p, _u64p]),
    "bnmc_synth_priors": (C.c_int, [C.c_int, _u64p, C.c_uint64, C.c_uint64, _f64p]),
}


class Error(RuntimeError):
    """bnmc::Error (types.hpp:16-18)."""


class UsageError(Error):
    """bnmc::UsageError — bad flags / configuration (status 2)."""


class DataError(Error):
    """bnmc::DataError — invalid input data (status 3)."""


class CapacityError(Error):
    """bnmc::CapacityError — memory estimate over the cap (status 4)."""


class CudaError(Error):
    """CUDA runtime failure or no usable sm_100 device (status 5)."""


class NcclError(Error):
    """NCCL missing or a collective failed (status 6)."""


_EXC = {2: UsageError, 3: DataError, 4: CapacityError, 5: CudaError, 6: NcclError}

_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                          "(no CPU fallback exists)")
    L = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def check(status: int):
    if status != 0:
        msg = lib().bnmc_gpu_last_error_message().decode()
        raise _EXC.get(status, Error)(msg)


def check_synth(status: int):
    if status != 0:
        raise _EXC.get(status, Error)(lib().bnmc_synth_last_error().decode())


def ptr(a):
    """Data pointer of an optional numpy array (None -> NULL)."""
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def device_count() -> int:
    n = C.c_int()
    check(lib().bnmc_gpu_device_count(C.byref(n)))
    return n.value


# ---- pinned host buffers (bnmc_gpu_host_alloc) with a small reuse pool: a
# block returns to the pool when the last numpy view of it is collected, so
# repeated run_chains calls reuse page-locked memory without staging copies.
_POOL: dict = {}
_POOL_BYTES = [0]
_POOL_CAP = 8 << 30
_EXITING = [False]


def _drain_pool():
    """At interpreter exit: return every pooled block to the driver (blocks
    still referenced are freed by their finalizers, which see _EXITING)."""
    _EXITING[0] = True
    for ptrs in _POOL.values():
        for p in ptrs:
            try:
                _lib.bnmc_gpu_host_free(p)
            except Exception:
                pass
    _POOL.clear()
    _POOL_BYTES[0] = 0


atexit.register(_drain_pool)


def _release(ptr: int, nbytes: int):
    try:
        if _EXITING[0]:
            _lib.bnmc_gpu_host_free(ptr)
        elif _POOL_BYTES[0] + nbytes <= _POOL_CAP:
            _POOL.setdefault(nbytes, []).append(ptr)
            _POOL_BYTES[0] += nbytes
        elif _lib is not None:
            _lib.bnmc_gpu_host_free(ptr)
    except Exception:  # interpreter shutdown
        pass


def pinned_empty(shape, dtype) -> np.ndarray:
    """np.empty(shape, dtype) in page-locked host memory owned by the library."""
    import weakref
    dtype = np.dtype(dtype)
    count = int(np.prod(shape)) if len(shape) else 1
    nbytes = max(8, count * dtype.itemsize)
    free = _POOL.get(nbytes)
    if free:
        ptr = free.pop()
        _POOL_BYTES[0] -= nbytes
    else:
        out = _vp()
        check(lib().bnmc_gpu_host_alloc(nbytes, C.byref(out)))
        ptr = out.value
        # a caller looping `r = run_chains(...)` holds the previous result while
        # the next call fills new buffers: keep a second block of this size
        # pooled so the steady state never allocates page-locked memory
        if _POOL_BYTES[0] + nbytes <= _POOL_CAP:
            spare = _vp()
            check(lib().bnmc_gpu_host_alloc(nbytes, C.byref(spare)))
            _POOL.setdefault(nbytes, []).append(spare.value)
            _POOL_BYTES[0] += nbytes
    buf = (C.c_char * nbytes).from_address(ptr)
    weakref.finalize(buf, _release, ptr, nbytes)
    return np.frombuffer(buf, dtype=dtype, count=count).reshape(shape)
