"""TEST INFRASTRUCTURE — ctypes binding of the plain-C restatement (oracle/bnmc_oracle.c).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` leg may
import this module. It is the parity checker, never the thing measured or shipped.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libbnmc_oracle.so")

_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


class McmcCfg(C.Structure):
    _fields_ = [("iterations", C.c_uint64), ("seed", C.c_uint64),
                ("track_top", C.c_int), ("strict", C.c_int)]


class OracleError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"[{status}] {msg}")
        self.status = status


_lib = None


def build():
    subprocess.check_call(["make", "-s", "-C", HERE, "port"])


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        build()
    L = C.CDLL(LIB_PATH)
    L.orc_last_error.restype = C.c_char_p
    L.orc_binomial.restype = C.c_uint64
    L.orc_binomial.argtypes = [C.c_int, C.c_int]
    L.orc_bounded_subset_count.restype = C.c_uint64
    L.orc_bounded_subset_count.argtypes = [C.c_int, C.c_int]
    L.orc_global_index.restype = C.c_uint64
    L.orc_global_index.argtypes = [C.c_uint64, C.c_int, C.c_int]
    L.orc_subset_at.restype = C.c_uint64
    L.orc_subset_at.argtypes = [C.c_uint64, C.c_int, C.c_int]
    L.orc_build_pst.argtypes = [C.c_int, C.c_int, _u64p]
    L.orc_index_of.restype = C.c_uint64
    L.orc_index_of.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64]
    L.orc_count_statistics.argtypes = [_u8p, _i32p, C.c_int, C.c_uint64, C.c_int, C.c_uint64,
                                       _u32p, C.c_uint64, C.POINTER(C.c_uint64)]
    L.orc_local_score.argtypes = [_u8p, _i32p, C.c_int, C.c_uint64, C.c_int, C.c_uint64,
                                  C.c_double, C.c_double, C.c_int, C.POINTER(C.c_double)]
    L.orc_ppf.restype = C.c_double
    L.orc_ppf.argtypes = [C.c_double]
    L.orc_cache_build.argtypes = [_u8p, _i32p, C.c_int, C.c_uint64, C.c_int, C.c_double,
                                  C.c_double, C.c_int, C.c_int, _f64p]
    L.orc_score_order.argtypes = [_f64p, C.c_int, C.c_int, C.c_void_p, _i32p, _u64p, _f64p,
                                  C.POINTER(C.c_double)]
    L.orc_run_mcmc.argtypes = [_f64p, C.c_int, C.c_int, C.c_void_p, C.POINTER(McmcCfg),
                               _f64p, _u8p, _f64p, _i32p, C.POINTER(C.c_double),
                               C.POINTER(C.c_uint64), C.POINTER(C.c_int), _u64p, _f64p]
    _lib = L
    return L


def _check(st):
    if st != 0:
        raise OracleError(st, lib().orc_last_error().decode())


def _prior_ptr(priors):
    if priors is None:
        return None, None
    a = np.ascontiguousarray(priors, dtype=np.float64)
    return a, a.ctypes.data_as(C.c_void_p)


def binomial(n, k):
    return int(lib().orc_binomial(n, k))


def bounded_subset_count(n, s):
    return int(lib().orc_bounded_subset_count(n, s))


def global_index(mask, c, s):
    return int(lib().orc_global_index(mask, c, s))


def subset_at(index, c, s):
    return int(lib().orc_subset_at(index, c, s))


def build_pst(c, s):
    out = np.zeros(bounded_subset_count(c, s), np.uint64)
    lib().orc_build_pst(c, s, out)
    return out


def index_of(n, s, node, pset):
    return int(lib().orc_index_of(n, s, node, pset))


def count_statistics(cells, cards, node, pset, cap=1 << 22):
    cells = np.ascontiguousarray(cells, np.uint8)
    m, n = cells.shape
    out = np.zeros(cap, np.uint32)
    r = C.c_uint64()
    _check(lib().orc_count_statistics(cells.ravel(), np.ascontiguousarray(cards, np.int32), n, m,
                                      node, pset, out, cap, C.byref(r)))
    return out[: r.value * int(cards[node])].reshape(r.value, int(cards[node]))


def local_score(cells, cards, node, pset, gamma=0.1, ess=1.0, k2=False):
    cells = np.ascontiguousarray(cells, np.uint8)
    m, n = cells.shape
    out = C.c_double()
    _check(lib().orc_local_score(cells.ravel(), np.ascontiguousarray(cards, np.int32), n, m, node,
                                 pset, gamma, ess, int(k2), C.byref(out)))
    return out.value


def ppf(r):
    return lib().orc_ppf(r)


def cache_build(cells, cards, s, gamma=0.1, ess=1.0, k2=False, threads=None):
    cells = np.ascontiguousarray(cells, np.uint8)
    m, n = cells.shape
    per = bounded_subset_count(n - 1, s)
    out = np.zeros(n * per, np.float64)
    _check(lib().orc_cache_build(cells.ravel(), np.ascontiguousarray(cards, np.int32), n, m, s,
                                 gamma, ess, int(k2), threads or os.cpu_count(), out))
    return out.reshape(n, per)


def score_order(table, s, perm, priors=None):
    """Serial restatement of score_order → (masks[n], best_by_node[n], total)."""
    table = np.ascontiguousarray(table, np.float64)
    n = table.shape[0]
    masks = np.zeros(n, np.uint64)
    best = np.zeros(n, np.float64)
    tot = C.c_double()
    keep, pp = _prior_ptr(priors)
    _check(lib().orc_score_order(table.ravel(), n, s, pp, np.ascontiguousarray(perm, np.int32),
                                 masks, best, C.byref(tot)))
    return masks, best, tot.value


def run_mcmc(table, s, iterations, seed, priors=None, track_top=10, strict=False):
    """Restatement of run_mcmc with a prebuilt cache (sampler.cpp:58-116)."""
    table = np.ascontiguousarray(table, np.float64)
    n = table.shape[0]
    cfg = McmcCfg(iterations, seed, track_top, int(strict))
    tp = np.zeros(iterations, np.float64)
    ta = np.zeros(iterations, np.uint8)
    tb = np.zeros(iterations, np.float64)
    fo = np.zeros(n, np.int32)
    fs, acc, tc = C.c_double(), C.c_uint64(), C.c_int()
    tm = np.zeros(track_top * n, np.uint64)
    tt = np.zeros(track_top, np.float64)
    keep, pp = _prior_ptr(priors)
    _check(lib().orc_run_mcmc(table.ravel(), n, s, pp, C.byref(cfg), tp, ta, tb, fo, C.byref(fs),
                              C.byref(acc), C.byref(tc), tm, tt))
    k = tc.value
    return dict(trace_proposed=tp, trace_accepted=ta.astype(bool), trace_best=tb, final_order=fo,
                final_score=fs.value, accepted=acc.value,
                tracker_masks=tm.reshape(track_top, n)[:k], tracker_totals=tt[:k])
