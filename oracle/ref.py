"""TEST INFRASTRUCTURE — ctypes binding of the reference core (oracle/_ref).

``oracle/_ref/libbnmc_ref.so`` is the UNMODIFIED reference library
(/root/reference/proj/src, canonical Release flags) plus the marshalling shim
``oracle/ref_shim.cpp``. Only tests/, ``__graft_entry__.smoke()`` and bench.py's
CPU-baseline / ``--impl reference`` legs may import this module; the product
(``paper_1210_5128_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libbnmc_ref.so")

_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


class RefError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[{status}] {msg}")
        self.status = status


_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not available():
        raise FileNotFoundError(f"{LIB_PATH} missing: run `make -C oracle ref` (needs /root/reference)")
    L = C.CDLL(LIB_PATH)
    L.ref_last_error.restype = C.c_char_p
    L.ref_max_threads.restype = C.c_int
    L.ref_generate.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_uint64, _i32p,
                               C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, _u8p, _u64p]
    L.ref_synth_priors.argtypes = [C.c_int, _u64p, C.c_uint64, C.c_uint64, _f64p]
    L.ref_binomial.restype = C.c_uint64
    L.ref_binomial.argtypes = [C.c_int, C.c_int]
    L.ref_bounded_subset_count.restype = C.c_uint64
    L.ref_bounded_subset_count.argtypes = [C.c_int, C.c_int]
    L.ref_global_index.restype = C.c_uint64
    L.ref_global_index.argtypes = [C.c_uint64, C.c_int, C.c_int]
    L.ref_subset_at.restype = C.c_uint64
    L.ref_subset_at.argtypes = [C.c_uint64, C.c_int, C.c_int]
    L.ref_build_pst.argtypes = [C.c_int, C.c_int, _u64p]
    L.ref_rng_stream.argtypes = [C.c_uint64, C.c_int64, C.c_int, C.c_uint64, C.c_uint64, _u64p]
    L.ref_shuffle_identity.argtypes = [C.c_int, C.c_uint64, C.c_int64, _i32p]
    L.ref_count_statistics.argtypes = [_u8p, _i32p, C.c_int, C.c_uint64, C.c_int, C.c_uint64,
                                       _u32p, C.c_uint64, C.POINTER(C.c_uint64)]
    L.ref_count_statistics_active.argtypes = [_u8p, _i32p, C.c_int, C.c_uint64, C.c_int,
                                              C.c_uint64, _u64p, _u32p, C.c_uint64,
                                              C.POINTER(C.c_uint64)]
    L.ref_local_score_batch.argtypes = [_u8p, _i32p, C.c_int, C.c_uint64, C.c_int, _i32p, _u64p,
                                        C.c_double, C.c_double, C.c_int, _f64p,
                                        C.POINTER(C.c_double)]
    L.ref_local_score.argtypes = [_u8p, _i32p, C.c_int, C.c_uint64, C.c_int, C.c_uint64,
                                  C.c_double, C.c_double, C.c_int, C.POINTER(C.c_double)]
    L.ref_ppf.argtypes = [C.c_double, C.POINTER(C.c_double)]
    L.ref_cache_build.restype = C.c_void_p
    L.ref_cache_build.argtypes = [_u8p, _i32p, C.c_int, C.c_uint64, C.c_int, C.c_double,
                                  C.c_double, C.c_int, C.c_int, C.c_uint64, C.POINTER(C.c_int)]
    L.ref_cache_load.restype = C.c_void_p
    L.ref_cache_load.argtypes = [C.c_char_p, C.c_int, C.c_double, C.c_double, C.c_int,
                                 C.POINTER(C.c_int)]
    L.ref_cache_save.argtypes = [C.c_void_p, C.c_char_p]
    L.ref_cache_n.argtypes = [C.c_void_p]
    L.ref_cache_per_node.restype = C.c_uint64
    L.ref_cache_per_node.argtypes = [C.c_void_p]
    L.ref_cache_table.argtypes = [C.c_void_p, _f64p]
    L.ref_cache_lookup.restype = C.c_double
    L.ref_cache_lookup.argtypes = [C.c_void_p, C.c_int, C.c_uint64]
    L.ref_estimate_bytes.restype = C.c_uint64
    L.ref_estimate_bytes.argtypes = [C.c_int, C.c_int]
    L.ref_cache_free.argtypes = [C.c_void_p]
    L.ref_scorer_new.restype = C.c_void_p
    L.ref_scorer_new.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int,
                                 C.POINTER(C.c_int)]
    L.ref_scorer_score.argtypes = [C.c_void_p, _i32p, C.c_int, _u64p, C.POINTER(C.c_double)]
    L.ref_scorer_free.argtypes = [C.c_void_p]
    L.ref_score_order.argtypes = [C.c_void_p, C.c_void_p, _i32p, C.c_int, _u64p,
                                  C.POINTER(C.c_double)]
    L.ref_score_graph.argtypes = [C.c_void_p, C.c_void_p, _u64p, C.c_int, C.POINTER(C.c_double)]
    L.ref_mh_accept.argtypes = [C.c_double, C.c_double, C.c_uint64, C.c_int64, C.c_uint64, _u8p]
    L.ref_run_mcmc.argtypes = [_u8p, _i32p, C.c_int, C.c_uint64, C.c_int, C.c_double, C.c_double,
                               C.c_int, C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int,
                               C.c_int, C.c_uint64, C.c_int, C.c_void_p, C.c_void_p,
                               _f64p, _u8p, _f64p, _i32p, C.POINTER(C.c_double),
                               C.POINTER(C.c_uint64), C.POINTER(C.c_int), _u64p, _f64p,
                               C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.ref_write_dataset_csv.argtypes = [_u8p, _i32p, C.c_int, C.c_uint64, C.c_char_p]
    L.ref_write_prior_csv.argtypes = [_f64p, C.c_int, C.c_char_p]
    L.ref_write_edge_list.argtypes = [_u64p, C.c_int, C.c_char_p]
    L.ref_learn.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_double, C.c_double, C.c_int,
                            C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_char_p]
    L.ref_eval_sweep.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_double, C.c_double,
                                 C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.c_char_p]
    _lib = L
    return L


def _check(status: int):
    if status != 0:
        raise RefError(status, lib().ref_last_error().decode())


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


# ---------------------------------------------------------------- generator
def generate(n, max_parents, m, cards, seed=7, edge_prob=0.3, concentration=1.0,
             tags=(101, 102, 103)):
    """Reference generator (evalgen.cpp:38-109) → (cells[m,n] u8, truth masks[n] u64)."""
    cards = np.ascontiguousarray(cards, dtype=np.int32)
    cells = np.zeros(m * n, dtype=np.uint8)
    truth = np.zeros(n, dtype=np.uint64)
    _check(lib().ref_generate(n, max_parents, edge_prob, concentration, m, cards, seed,
                              tags[0], tags[1], tags[2], cells, truth))
    return cells.reshape(m, n), truth


def synth_priors(n, truth, seed=7, tag=104):
    out = np.zeros(n * n, dtype=np.float64)
    _check(lib().ref_synth_priors(n, np.ascontiguousarray(truth, np.uint64), seed, tag, out))
    return out.reshape(n, n)


# ------------------------------------------------------------- combinatorics
def binomial(n, k):
    return int(lib().ref_binomial(n, k))


def bounded_subset_count(n, s):
    return int(lib().ref_bounded_subset_count(n, s))


def global_index(mask, candidates, s):
    return int(lib().ref_global_index(mask, candidates, s))


def subset_at(index, candidates, s):
    return int(lib().ref_subset_at(index, candidates, s))


def build_pst(candidates, s):
    out = np.zeros(bounded_subset_count(candidates, s), dtype=np.uint64)
    _check(lib().ref_build_pst(candidates, s, out))
    return out


def rng_stream(seed, tag, kind, count, arg=0):
    out = np.zeros(count, dtype=np.uint64)
    _check(lib().ref_rng_stream(seed, tag, kind, arg, count, out))
    return out.view(np.float64) if kind in (1, 2) else out


def shuffle_identity(n, seed, tag):
    out = np.zeros(n, dtype=np.int32)
    _check(lib().ref_shuffle_identity(n, seed, tag, out))
    return out


# ------------------------------------------------------------------ scoring
def count_statistics(cells, cards, node, pset, cap=1 << 22):
    cells = np.ascontiguousarray(cells, np.uint8)
    m, n = cells.shape
    out = np.zeros(cap, dtype=np.uint32)
    r = C.c_uint64()
    _check(lib().ref_count_statistics(cells.ravel(), np.ascontiguousarray(cards, np.int32), n, m,
                                      node, pset, out, cap, C.byref(r)))
    return out[: r.value * int(cards[node])].reshape(r.value, int(cards[node]))


def count_statistics_active(cells, cards, node, pset):
    """(configs, counts) of CountTable::for_each_active (scoring.hpp:55-67)."""
    cells = np.ascontiguousarray(cells, np.uint8)
    m, n = cells.shape
    cap = max(m, 1)
    cv = int(cards[node])
    cfg = np.zeros(cap, np.uint64)
    cnt = np.zeros(cap * cv, np.uint32)
    na = C.c_uint64()
    _check(lib().ref_count_statistics_active(cells.ravel(), np.ascontiguousarray(cards, np.int32),
                                             n, m, node, pset, cfg, cnt, cap, C.byref(na)))
    k = na.value
    return cfg[:k], cnt[:k * cv].reshape(k, cv)


def local_score(cells, cards, node, pset, gamma=0.1, ess=1.0, k2=False):
    cells = np.ascontiguousarray(cells, np.uint8)
    m, n = cells.shape
    out = C.c_double()
    _check(lib().ref_local_score(cells.ravel(), np.ascontiguousarray(cards, np.int32), n, m,
                                 node, pset, gamma, ess, int(k2), C.byref(out)))
    return out.value


def local_score_batch(cells, cards, nodes, psets, gamma=0.1, ess=1.0, k2=False):
    """(scores, seconds): local_score of many entries on one Dataset, one thread."""
    cells = np.ascontiguousarray(cells, np.uint8)
    m, n = cells.shape
    nodes = np.ascontiguousarray(nodes, np.int32)
    psets = np.ascontiguousarray(psets, np.uint64)
    out = np.zeros(nodes.size, np.float64)
    sec = C.c_double()
    _check(lib().ref_local_score_batch(cells.ravel(), np.ascontiguousarray(cards, np.int32), n, m,
                                       nodes.size, nodes, psets, gamma, ess, int(k2), out,
                                       C.byref(sec)))
    return out, sec.value


def ppf(r):
    out = C.c_double()
    _check(lib().ref_ppf(r, C.byref(out)))
    return out.value


class Cache:
    """Owning handle of a reference ScoreCache (scoring.hpp:117-161)."""

    def __init__(self, handle, n, s, gamma, ess, k2):
        self.h, self.n, self.s = handle, n, s
        self.gamma, self.ess, self.k2 = gamma, ess, k2
        self.per_node = int(lib().ref_cache_per_node(handle))

    @classmethod
    def build(cls, cells, cards, s, gamma=0.1, ess=1.0, k2=False, workers=None,
              mem_cap=(1 << 64) - 1):
        cells = np.ascontiguousarray(cells, np.uint8)
        m, n = cells.shape
        st = C.c_int()
        workers = workers or lib().ref_max_threads()
        h = lib().ref_cache_build(cells.ravel(), np.ascontiguousarray(cards, np.int32), n, m, s,
                                  gamma, ess, int(k2), workers, mem_cap, C.byref(st))
        _check(st.value)
        return cls(h, n, s, gamma, ess, k2)

    @classmethod
    def load(cls, path, s, gamma=0.1, ess=1.0, k2=False):
        st = C.c_int()
        h = lib().ref_cache_load(path.encode(), s, gamma, ess, int(k2), C.byref(st))
        _check(st.value)
        return cls(h, lib().ref_cache_n(h), s, gamma, ess, k2)

    def save(self, path):
        _check(lib().ref_cache_save(self.h, path.encode()))

    def table(self):
        out = np.zeros(self.n * self.per_node, dtype=np.float64)
        lib().ref_cache_table(self.h, out)
        return out.reshape(self.n, self.per_node)

    def lookup(self, node, pset):
        return lib().ref_cache_lookup(self.h, node, pset)

    def score_order(self, perm, priors=None):
        """Serial reference score_order (scoring.cpp:261-289)."""
        perm = np.ascontiguousarray(perm, np.int32)
        pr = _f64(priors)
        masks = np.zeros(self.n, dtype=np.uint64)
        tot = C.c_double()
        _check(lib().ref_score_order(self.h, _ptr(pr), perm, self.n, masks, C.byref(tot)))
        return masks, tot.value

    def score_graph(self, masks, priors=None):
        pr = _f64(priors)
        tot = C.c_double()
        _check(lib().ref_score_graph(self.h, _ptr(pr), np.ascontiguousarray(masks, np.uint64),
                                     self.n, C.byref(tot)))
        return tot.value

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_cache_free(self.h)
            self.h = None


class Scorer:
    """Reference OrderScorer (engine.cpp:24-98) with the given EngineConfig."""

    def __init__(self, cache: Cache, priors=None, workers=None, tasks_per_node=0, use_pst=True):
        self.cache = cache
        self._pr = _f64(priors)
        st = C.c_int()
        workers = workers or lib().ref_max_threads()
        self.h = lib().ref_scorer_new(cache.h, _ptr(self._pr), workers, tasks_per_node,
                                      int(use_pst), C.byref(st))
        _check(st.value)

    def score(self, perm):
        perm = np.ascontiguousarray(perm, np.int32)
        masks = np.zeros(self.cache.n, dtype=np.uint64)
        tot = C.c_double()
        _check(lib().ref_scorer_score(self.h, perm, self.cache.n, masks, C.byref(tot)))
        return masks, tot.value

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_scorer_free(self.h)
            self.h = None


@dataclass
class McmcResult:
    trace_proposed: np.ndarray
    trace_accepted: np.ndarray
    trace_best: np.ndarray
    final_order: np.ndarray
    final_score: float
    accepted: int
    tracker_masks: np.ndarray
    tracker_totals: np.ndarray
    preprocess_seconds: float
    sampling_seconds: float


def run_mcmc(cells, cards, s, iterations, seed, priors=None, gamma=0.1, ess=1.0, k2=False,
             workers=None, track_top=10, strict=False, use_pst=True, tasks_per_node=0,
             mem_cap=(1 << 64) - 1, debug_recheck=False, prebuilt: Cache | None = None):
    """Reference run_mcmc (sampler.cpp:58-116)."""
    cells = np.ascontiguousarray(cells, np.uint8)
    m, n = cells.shape
    workers = workers or lib().ref_max_threads()
    tp = np.zeros(iterations, np.float64)
    ta = np.zeros(iterations, np.uint8)
    tb = np.zeros(iterations, np.float64)
    fo = np.zeros(n, np.int32)
    fs, acc, tc = C.c_double(), C.c_uint64(), C.c_int()
    tm = np.zeros(track_top * n, np.uint64)
    tt = np.zeros(track_top, np.float64)
    pre, samp = C.c_double(), C.c_double()
    pr = _f64(priors)
    _check(lib().ref_run_mcmc(cells.ravel(), np.ascontiguousarray(cards, np.int32), n, m, s,
                              gamma, ess, int(k2), iterations, seed, workers, track_top,
                              int(strict), int(use_pst), tasks_per_node, mem_cap,
                              int(debug_recheck), _ptr(pr), prebuilt.h if prebuilt else None,
                              tp, ta, tb, fo, C.byref(fs), C.byref(acc), C.byref(tc), tm, tt,
                              C.byref(pre), C.byref(samp)))
    k = tc.value
    return McmcResult(tp, ta.astype(bool), tb, fo, fs.value, acc.value,
                      tm.reshape(track_top, n)[:k], tt[:k], pre.value, samp.value)


def max_threads():
    return lib().ref_max_threads()


def write_dataset_csv(cells, cards, path):
    """The reference's write_dataset_csv (io.cpp:128-141)."""
    cells = np.ascontiguousarray(cells, np.uint8)
    m, n = cells.shape
    _check(lib().ref_write_dataset_csv(cells.ravel(), np.ascontiguousarray(cards, np.int32), n, m,
                                       str(path).encode()))


def write_prior_csv(r, path):
    r = np.ascontiguousarray(r, np.float64)
    _check(lib().ref_write_prior_csv(r.ravel(), r.shape[0], str(path).encode()))


def write_edge_list(masks, path):
    masks = np.ascontiguousarray(masks, np.uint64)
    _check(lib().ref_write_edge_list(masks, masks.size, str(path).encode()))


def learn(data_path, out_prefix, s=4, iterations=1, seed=0, priors_path=None, gamma=0.1, ess=1.0,
          k2=False, workers=None, track_top=10, strict=False):
    """The reference CLI's `learn` (bnmc.cpp:100-138) through its own library."""
    _check(lib().ref_learn(str(data_path).encode(),
                           None if priors_path is None else str(priors_path).encode(), s, gamma,
                           ess, int(k2), iterations, seed, workers or max_threads(), track_top,
                           int(strict), str(out_prefix).encode()))


def eval_sweep(truth_path, data_path, out_path, s=4, iterations=1, seed=0, gamma=0.1, ess=1.0,
               workers=None, track_top=10):
    """The reference CLI's `eval --sweep` (bnmc.cpp:160-212)."""
    _check(lib().ref_eval_sweep(str(truth_path).encode(), str(data_path).encode(), s, gamma, ess,
                                iterations, seed, workers or max_threads(), track_top,
                                str(out_path).encode()))
