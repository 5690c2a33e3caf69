"""Reference-shaped host interface over the C-ABI (drop-in for the hot path).

Mirrors the reference classes a caller of the hot path uses (paths relative to
/root/reference/proj): ``RunConfig`` / ``Dataset`` / ``PriorMatrix`` / ``Order``
(include/bnmc/types.hpp), ``ScoreCache`` (include/bnmc/scoring.hpp:117-161),
``OrderScorer`` (include/bnmc/engine.hpp:77-98), ``run_mcmc`` / ``McmcResult`` /
``TraceRow`` (include/bnmc/sampler.hpp:42-68) and the error taxonomy
(types.hpp:16-30). Argument meaning and error behaviour follow the reference;
``workers``, ``tasks_per_node`` and ``use_pst`` are accepted and ignored (the
device scan has no worker knob). Every compute call goes through
``libbnmc_b200.so``; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import enum
from collections.abc import Sequence
import struct
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import CapacityError, DataError, Error, UsageError  # noqa: F401

K_MAX_NODES = 64


class AlphaMode(enum.IntEnum):
    BDEU = 0
    K2 = 1


@dataclass
class RunConfig:
    """RunConfig (types.hpp:167-183) plus the device knobs."""
    max_parents: int = 4
    gamma: float = 0.1
    ess: float = 1.0
    alpha_mode: AlphaMode = AlphaMode.BDEU
    iterations: int = 1
    seed: int = 0
    workers: int = 1
    track_top: int = 10
    strict_paper_tracker: bool = False
    use_pst: bool = True
    tasks_per_node: int = 0
    memory_cap_bytes: int = 4 << 30
    debug_recheck: bool = False
    device: int = 0
    n_gpus: int = 1  # >1: one process drives devices device..device+n_gpus-1 (split K1, replicas)
    scan_mode: int = 0  # 0 auto (= 2), 1 full-row fp32-key scan (<= 64 chains), 2 sorted walk
    team_warps: int = 0  # sorted walk: warps per chain (0 auto, 1, 2, 4, 8)
    exact_accept: int = 0  # 0 device log10 + exact replay of ambiguous chains, 1 host glibc
    accept_tol_log2: int = 0  # bound of the ambiguity test (0 = 2^-48 relative)

    def validate(self):
        """RunConfig::validate (types.cpp:111-121)."""
        if not 0 <= self.max_parents <= 8:
            raise UsageError("max-parents must lie in [0,8]")
        if not (0.0 < self.gamma <= 1.0):
            raise UsageError("gamma must lie in (0,1]")
        if not self.ess > 0.0:
            raise UsageError("ess must be positive")
        if self.iterations < 1:
            raise UsageError("iterations must be >= 1")
        if self.workers < 1:
            raise UsageError("workers must be >= 1")
        if self.track_top < 1:
            raise UsageError("track-top must be >= 1")
        if self.tasks_per_node < 0:
            raise UsageError("tasks-per-node must be >= 0")

    def score_params(self) -> _lib.ScoreParams:
        return _lib.ScoreParams(self.max_parents, self.gamma, self.ess, int(self.alpha_mode),
                                min(self.memory_cap_bytes, (1 << 64) - 1), self.device,
                                self.n_gpus)


class Dataset:
    """Complete discrete dataset, row-major uint8 m x n (types.hpp:68-90, types.cpp:8-26)."""

    def __init__(self, cardinalities, rows):
        cards = np.ascontiguousarray(cardinalities, dtype=np.int32)
        n = cards.size
        if n == 0 or n > K_MAX_NODES:
            raise DataError("dataset must have between 1 and 64 variables")
        bad = np.nonzero((cards < 2) | (cards > 256))[0]
        if bad.size:
            raise DataError(f"cardinality of variable {bad[0]} out of range [2,256]")
        cells = np.ascontiguousarray(rows, dtype=np.uint8).reshape(-1)
        if cells.size % n:
            raise DataError("row data is not a multiple of the variable count")
        cells = cells.reshape(-1, n)
        over = cells >= cards[None, :]
        if over.any():
            r, c = np.argwhere(over)[0]
            raise DataError(f"state out of range at row {r}, column {c}")
        self.cards = cards
        self.cells = cells

    @property
    def n(self) -> int:
        return int(self.cards.size)

    def rows(self) -> int:
        return int(self.cells.shape[0])

    def cardinality(self, i):
        return int(self.cards[i])

    def state(self, row, col):
        return int(self.cells[row, col])


class PriorMatrix:
    """Pairwise edge beliefs r(child, parent) in [0,1] (types.hpp:149-163)."""

    def __init__(self, n, values=None):
        self.n = n
        if values is None:
            self.values = np.full((n, n), 0.5)
        else:
            v = np.ascontiguousarray(values, dtype=np.float64)
            if v.size != n * n:
                raise DataError("prior matrix must be n x n")
            if not np.all((v >= 0.0) & (v <= 1.0)):
                raise DataError("prior matrix entries must lie in [0,1]")
            self.values = v.reshape(n, n).copy()

    @classmethod
    def neutral(cls, n):
        return cls(n)

    def r(self, child, parent):
        return float(self.values[child, parent])

    def set(self, child, parent, value):
        if not 0.0 <= value <= 1.0:
            raise DataError("prior matrix entries must lie in [0,1]")
        self.values[child, parent] = value

    def is_neutral(self):
        off = ~np.eye(self.n, dtype=bool)
        return bool(np.all(self.values[off] == 0.5))


def _prior_array(priors):
    if priors is None:
        return None
    if isinstance(priors, PriorMatrix):
        return np.ascontiguousarray(priors.values, np.float64)
    return np.ascontiguousarray(priors, np.float64)


class Order:
    """perm[pos] = node (types.hpp:93-114)."""

    def __init__(self, perm):
        p = np.ascontiguousarray(perm, dtype=np.int32)
        n = p.size
        if n > K_MAX_NODES:
            raise DataError("order exceeds 64 nodes")
        if sorted(p.tolist()) != list(range(n)):
            raise DataError("order is not a permutation of 0..n-1")
        self.perm = p

    @classmethod
    def identity(cls, n):
        return cls(np.arange(n))

    @property
    def n(self):
        return int(self.perm.size)

    def node_at(self, pos):
        return int(self.perm[pos])

    def positions(self):
        pos = np.empty(self.n, np.int32)
        pos[self.perm] = np.arange(self.n)
        return pos

    def __eq__(self, other):
        return isinstance(other, Order) and np.array_equal(self.perm, other.perm)


@dataclass
class ScoredGraph:
    """ScoredGraph (scoring.hpp:167-170): parent masks by node + total."""
    masks: np.ndarray
    total: float
    best_by_node: np.ndarray | None = None


# ----------------------------------------------------------------- BNSC file
_MAGIC = b"BNSC"


def _hyper_digest(gamma, ess):
    """hyper_digest (scoring.cpp:27-37): FNV-1a over the LE bytes of (gamma, ess)."""
    h = 0xCBF29CE484222325
    for b in struct.pack("<dd", gamma, ess):
        h ^= b
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def write_bnsc(path, table, n, s, gamma, ess, alpha_mode):
    """ScoreCache::save format (scoring.cpp:194-208)."""
    with open(path, "wb") as f:
        f.write(_MAGIC)
        f.write(bytes([1, n, s, 1 if alpha_mode == AlphaMode.K2 else 0]))
        f.write(struct.pack("<Q", _hyper_digest(gamma, ess)))
        f.write(np.ascontiguousarray(table, dtype="<f8").tobytes())


def read_bnsc(path, cfg: RunConfig):
    """ScoreCache::load checks (scoring.cpp:210-238) -> (n, s, table[n, S])."""
    try:
        f = open(path, "rb")
    except OSError:
        raise DataError(f"cannot open cache file: {path}") from None
    with f:
        magic = f.read(4)
        if magic != _MAGIC:
            raise DataError(f"not a score cache file: {path}")
        meta = f.read(4)
        if len(meta) < 4 or meta[0] != 1:
            raise DataError(f"unsupported cache version in {path}")
        mode = 1 if cfg.alpha_mode == AlphaMode.K2 else 0
        dig = f.read(8)
        if (meta[2] != cfg.max_parents or meta[3] != mode or len(dig) < 8
                or struct.unpack("<Q", dig)[0] != _hyper_digest(cfg.gamma, cfg.ess)):
            raise DataError(f"cache file {path} was built with different scoring parameters")
        n, s = meta[1], meta[2]
        per = int(_lib.lib().bnmc_gpu_bounded_subset_count(n - 1, s))
        body = f.read(8 * n * per)
        if len(body) < 8 * n * per:
            raise DataError(f"cache file truncated: {path}")
        return n, s, np.frombuffer(body, dtype="<f8").astype(np.float64).reshape(n, per)


# -------------------------------------------------------------- CountTable
_DENSE_CELLS = 1 << 22  # scoring.cpp:13


class CountTable:
    """CountTable (scoring.hpp:41-77): N_ijk of one (node, parent set), dense
    (configs x card) up to 2^22 cells, else the active configurations only —
    iteration ascending either way (for_each_active)."""

    def __init__(self, configs, card, dense=None, active=None, counts=None):
        self._r, self._card = configs, card
        self._dense = dense
        self._active = active
        self._counts = counts

    def configs(self):
        return self._r

    def child_card(self):
        return self._card

    def is_dense(self):
        return self._dense is not None

    def samples(self):
        return int(self._dense.sum() if self._dense is not None else self._counts.sum())

    def njk(self, config, state):
        if self._dense is not None:
            return int(self._dense[config, state])
        i = int(np.searchsorted(self._active, np.uint64(config)))
        if i < self._active.size and int(self._active[i]) == config:
            return int(self._counts[i, state])
        return 0

    def nk(self, config):
        return sum(self.njk(config, j) for j in range(self._card))

    def for_each_active(self):
        """(config, counts row) for every config with N_ik > 0, ascending."""
        if self._dense is not None:
            for k in np.nonzero(self._dense.sum(axis=1))[0]:
                yield int(k), self._dense[k]
        else:
            for k, row in zip(self._active, self._counts):
                yield int(k), row


def count_statistics(data, node, pset, device=0):
    """count_statistics (scoring.cpp:82-109) on the device."""
    n, m = data.n, data.rows()
    if not 0 <= node < n or (n < 64 and pset >> n):
        raise UsageError("count_statistics: bad (node, parent set)")
    if pset >> node & 1:
        raise DataError("node cannot appear in its own parent set")
    r = 1
    for p in range(n):
        if pset >> p & 1:
            r *= int(data.cards[p])
    if r >= 1 << 64:
        raise CapacityError("parent configuration space overflows 64 bits")
    card = int(data.cards[node])
    cells = np.ascontiguousarray(data.cells).reshape(-1)
    if r * card <= _DENSE_CELLS:
        out = np.zeros(r * card, np.uint32)
        cfgs = np.zeros(1, np.uint64)
        _lib.check(_lib.lib().bnmc_gpu_count_statistics(
            cells, data.cards, m, n, 1, np.array([node], np.int32), np.array([pset], np.uint64),
            np.zeros(1, np.uint64), out, cfgs, device))
        return CountTable(r, card, dense=out.reshape(r, card))
    cap = max(m, 1)
    act = np.zeros(cap, np.uint64)
    cnt = np.zeros(cap * card, np.uint32)
    na = C.c_uint64()
    _lib.check(_lib.lib().bnmc_gpu_count_statistics_sparse(cells, data.cards, m, n, node, pset,
                                                            act, cnt, C.byref(na), device))
    k = na.value
    return CountTable(r, card, active=act[:k].copy(), counts=cnt[:k * card].reshape(k, card).copy())


# -------------------------------------------------------------- ScoreCache
class ScoreCache:
    """Device-resident score table (replaces ScoreCache, scoring.hpp:117-161).

    The fp64 local scores live on the device in BNSC order; the scan keys carry
    the PPF of the priors the table was last bound to (``OrderScorer`` rebinds
    when needed). Host-side ``at``/``lookup`` use a lazily downloaded mirror.
    """

    def __init__(self, handle, n, s, cfg: RunConfig):
        self._h = C.c_void_p(handle)
        self._n, self._s = n, s
        self._cfg = cfg
        self._host = None
        self._priors_key = None
        per = C.c_uint64()
        _lib.check(_lib.lib().bnmc_gpu_table_info(self._h, None, None, C.byref(per)))
        self._per = per.value
        self.preprocess_seconds = 0.0
        self.build_ms = (0.0, 0.0)

    # -- construction
    @staticmethod
    def estimate_bytes(n, s):
        return int(_lib.lib().bnmc_gpu_table_estimate_bytes(n, s))

    @classmethod
    def build(cls, data: Dataset, cfg: RunConfig, priors=None):
        """ScoreCache::build (scoring.cpp:162-192) on the device."""
        cfg.validate()
        pr = _prior_array(priors)
        out = C.c_void_p()
        t0 = time.perf_counter()
        _lib.check(_lib.lib().bnmc_gpu_table_build(
            data.cells.reshape(-1), data.cards, data.rows(), data.n, C.byref(cfg.score_params()),
            _lib.ptr(pr), C.byref(out)))
        c = cls(out.value, data.n, cfg.max_parents, cfg)
        c.preprocess_seconds = time.perf_counter() - t0
        c._priors_key = _key(pr)
        a, b = C.c_float(), C.c_float()
        _lib.check(_lib.lib().bnmc_gpu_table_build_ms(c._h, C.byref(a), C.byref(b)))
        c.build_ms = (a.value, b.value)
        return c

    @classmethod
    def from_table(cls, table, cfg: RunConfig, priors=None):
        """Prebuilt cache (host table in BNSC body order) -> device."""
        t = np.ascontiguousarray(table, dtype=np.float64)
        n = t.shape[0]
        pr = _prior_array(priors)
        out = C.c_void_p()
        _lib.check(_lib.lib().bnmc_gpu_table_upload(t.reshape(-1), n, C.byref(cfg.score_params()),
                                                     _lib.ptr(pr), C.byref(out)))
        c = cls(out.value, n, cfg.max_parents, cfg)
        c._priors_key = _key(pr)
        return c

    @classmethod
    def load(cls, path, cfg: RunConfig, priors=None):
        """ScoreCache::load (scoring.cpp:210-238)."""
        n, s, table = read_bnsc(path, cfg)
        return cls.from_table(table, cfg, priors)

    def save(self, path):
        """ScoreCache::save (scoring.cpp:194-208)."""
        write_bnsc(path, self.table(), self._n, self._s, self._cfg.gamma, self._cfg.ess,
                   self._cfg.alpha_mode)

    # -- accessors
    def n(self):
        return self._n

    def s(self):
        return self._s

    def entries_per_node(self):
        return self._per

    def table(self):
        if self._host is None:
            out = np.empty(self._n * self._per, np.float64)
            _lib.check(_lib.lib().bnmc_gpu_table_download(self._h, out))
            self._host = out.reshape(self._n, self._per)
        return self._host

    def index_of(self, node, pset):
        """ScoreCache::index_of (scoring.hpp:133-139)."""
        low = pset & ((1 << node) - 1)
        high = (pset >> (node + 1)) << node if node + 1 < 64 else 0
        return _global_index(low | high, self._n - 1, self._s)

    def at(self, node, index):
        return float(self.table()[node, index])

    def lookup(self, node, pset):
        return self.at(node, self.index_of(node, pset))

    def bind_priors(self, priors):
        """Fold the PPF of `priors` into the device scan keys (PpfTable, scoring.cpp:150-155)."""
        pr = _prior_array(priors)
        key = _key(pr)
        if key != self._priors_key:
            _lib.check(_lib.lib().bnmc_gpu_table_set_priors(self._h, _lib.ptr(pr)))
            self._priors_key = key

    def last_walk_stats(self):
        """Statistics and kernel variant of the last sorted-walk launch on this table."""
        L = _lib.lib()
        pa, wa, en, so = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_float()
        _lib.check(L.bnmc_gpu_last_walk_stats(self._h, C.byref(pa), C.byref(wa), C.byref(en),
                                              C.byref(so)))
        tw, wu, sp, rp = C.c_int(), C.c_int(), C.c_int(), C.c_uint64()
        _lib.check(L.bnmc_gpu_last_walk_variant(self._h, C.byref(tw), C.byref(wu), C.byref(sp)))
        _lib.check(L.bnmc_gpu_last_replayed(self._h, C.byref(rp)))
        return {"pairs": pa.value, "walked": wa.value, "enumerated": en.value,
                "sort_ms": so.value, "team_warps": tw.value, "entries_per_lane": wu.value,
                "speculative": bool(sp.value), "replayed": rp.value,
                "variant": "walk_spec_kernel" if sp.value else
                           f"walk_chain_kernel<{tw.value},{wu.value}>"}

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            _lib.lib().bnmc_gpu_table_free(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _key(pr):
    return None if pr is None else pr.tobytes()


def _binom(n, k):
    from math import comb
    return comb(n, k) if 0 <= k <= n else 0


def _global_index(mask, c, s):
    """global_index (combinatorics.cpp:61-76)."""
    k = bin(mask).count("1")
    offset = sum(_binom(c, j) for j in range(k + 1, s + 1))
    rank, prev, pos, m = 0, 0, 1, mask
    while m:
        a = (m & -m).bit_length()
        rank += _binom(c - prev, k - pos + 1) - _binom(c - a + 1, k - pos + 1)
        prev = a
        pos += 1
        m &= m - 1
    return offset + rank


# ------------------------------------------------------------- OrderScorer
@dataclass
class EngineConfig:
    """EngineConfig (engine.hpp:59-68); all fields are accepted no-ops on the device."""
    workers: int = 1
    tasks_per_node: int = 0
    use_pst: bool = True


class OrderScorer:
    """OrderScorer (engine.hpp:77-98): greedy order score on the device."""

    def __init__(self, cache: ScoreCache, priors=None, cfg: EngineConfig | None = None,
                 scan_mode: int = 0):
        cfg = cfg or EngineConfig()
        self.scan_mode = scan_mode
        pr = _prior_array(priors)
        if pr is not None and pr.shape[0] != cache.n():
            raise DataError("priors and cache disagree on node count")
        if cfg.workers < 1:
            raise UsageError("workers must be >= 1")
        self.cache = cache
        self._pr = pr
        self.config = cfg

    def score_many(self, perms):
        perms = np.ascontiguousarray(perms, dtype=np.int32)
        if perms.ndim == 1:
            perms = perms[None, :]
        k, n = perms.shape
        if n != self.cache.n():
            raise DataError("order and cache disagree on node count")
        self.cache.bind_priors(self._pr)
        _lib.check(_lib.lib().bnmc_gpu_table_set_scan_mode(self.cache.handle, self.scan_mode))
        masks = np.empty((k, n), np.uint64)
        best = np.empty((k, n), np.float64)
        tot = np.empty(k, np.float64)
        _lib.check(_lib.lib().bnmc_gpu_score_orders(self.cache.handle, perms.reshape(-1), k,
                                                     _lib.ptr(masks), _lib.ptr(best),
                                                     _lib.ptr(tot)))
        return masks, best, tot

    def scan_slice(self, position, node, lo, hi, order):
        """OrderScorer::scan_slice (engine.cpp:43-58) on the device -> (score, idx);
        the identity (-inf, 2**64-1) for an empty slice."""
        perm = np.ascontiguousarray(order.perm if isinstance(order, Order) else order, np.int32)
        if perm.size != self.cache.n():
            raise DataError("order and cache disagree on node count")
        if not 0 <= position < perm.size or int(perm[position]) != node:
            raise UsageError("work slice does not match the order")
        self.cache.bind_priors(self._pr)
        sc, ix = C.c_double(), C.c_uint64()
        _lib.check(_lib.lib().bnmc_gpu_scan_slice(self.cache.handle, perm, position, lo, hi,
                                                   C.byref(sc), C.byref(ix)))
        return sc.value, ix.value

    def score(self, order) -> ScoredGraph:
        perm = order.perm if isinstance(order, Order) else order
        masks, best, tot = self.score_many(np.asarray(perm)[None, :])
        return ScoredGraph(masks[0], float(tot[0]), best[0])


def parallel_score_order(order, cache, priors, workers=1):
    """parallel_score_order (engine.hpp:99-100)."""
    return OrderScorer(cache, priors, EngineConfig(workers)).score(order)


# ---------------------------------------------------------------- sampler
@dataclass
class McmcResult:
    """McmcResult (sampler.hpp:52-60); the trace is kept as column arrays."""
    tracker_masks: np.ndarray          # [K', n] best graphs, tracker order
    tracker_totals: np.ndarray         # [K']
    trace_proposed: np.ndarray         # [iterations]
    trace_accepted: np.ndarray         # [iterations] bool
    trace_best: np.ndarray             # [iterations]
    final_order: np.ndarray
    final_score: float
    accepted: int
    preprocess_seconds: float = 0.0
    sampling_seconds: float = 0.0
    device_ms: float = 0.0
    seed: int = 0
    extra: dict = field(default_factory=dict)

    def best_score(self):
        return float(self.tracker_totals[0])


@dataclass
class ChainBatch:
    """Results of run_chains_batch as chain-major arrays (no per-chain objects)."""
    trace_proposed: np.ndarray   # [C, iterations]
    trace_accepted: np.ndarray   # [C, iterations] uint8
    trace_best: np.ndarray       # [C, iterations]
    final_order: np.ndarray      # [C, n]
    final_score: np.ndarray      # [C]
    accepted: np.ndarray         # [C]
    tracker_count: np.ndarray    # [C]
    tracker_masks: np.ndarray    # [C, K, n]
    tracker_totals: np.ndarray   # [C, K]
    device_ms: float
    wall_s: float

    @classmethod
    def allocate(cls, chains: int, iterations: int, n: int, track_top: int, pinned: bool = True):
        """Result buffers for `chains` chains; page-locked (bnmc_gpu_host_alloc,
        pooled) unless pinned=False."""
        c, i, K = chains, iterations, track_top
        shapes = [((c, i), np.float64), ((c, i), np.uint8), ((c, i), np.float64),
                  ((c, n), np.int32), ((c,), np.float64), ((c,), np.uint64),
                  ((c,), np.int32), ((c, K, n), np.uint64), ((c, K), np.float64)]
        if not pinned:
            return cls(*[np.empty(sh, dt) for sh, dt in shapes], 0.0, 0.0)
        # one page-locked block per batch (64-byte aligned views): one pool entry,
        # so a reused batch size never allocates page-locked memory again
        offs, total = [], 0
        for sh, dt in shapes:
            offs.append(total)
            total += (int(np.prod(sh)) * np.dtype(dt).itemsize + 63) // 64 * 64
        block = _lib.pinned_empty((total,), np.uint8)
        views = [block[o:o + int(np.prod(sh)) * np.dtype(dt).itemsize].view(dt).reshape(sh)
                 for o, (sh, dt) in zip(offs, shapes)]
        return cls(*views, 0.0, 0.0)

    def result(self, c: int, seed: int = 0) -> McmcResult:
        """McmcResult of chain c as views into the batch buffers (no copies)."""
        k = int(self.tracker_count[c])
        return McmcResult(
            tracker_masks=self.tracker_masks[c, :k], tracker_totals=self.tracker_totals[c, :k],
            trace_proposed=self.trace_proposed[c], trace_accepted=self.trace_accepted[c].view(np.bool_),
            trace_best=self.trace_best[c], final_order=self.final_order[c],
            final_score=float(self.final_score[c]), accepted=int(self.accepted[c]),
            sampling_seconds=self.wall_s, device_ms=self.device_ms, seed=seed)


class ChainResults(Sequence):
    """run_chains' result: a sequence of McmcResult built on access from one
    ChainBatch in pinned host memory (no per-chain staging or copies)."""

    def __init__(self, batch: ChainBatch, seeds):
        self.batch = batch
        self.seeds = np.asarray(seeds, np.uint64)

    def __len__(self):
        return int(self.seeds.size)

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(len(self)))]
        if i < 0:
            i += len(self)
        if not 0 <= i < len(self):
            raise IndexError(i)
        return self.batch.result(i, int(self.seeds[i]))


def run_chains_batch(cache: ScoreCache, priors, seeds, cfg: RunConfig, out: ChainBatch | None = None):
    """Independent chains through one bnmc_gpu_run_chains call; chain c is run_mcmc
    with seed seeds[c]. Results land in `out` (reused) or in fresh pinned buffers."""
    cfg.validate()
    pr = _prior_array(priors)
    if pr is not None and pr.shape[0] != cache.n():
        raise DataError("prior matrix does not match the dataset's node count")
    seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
    nc, n, K, it = seeds.size, cache.n(), cfg.track_top, cfg.iterations
    cache.bind_priors(pr)
    if out is None:
        out = ChainBatch.allocate(nc, it, n, K)
    ms = C.c_float()
    params = _lib.ChainParams(it, K, int(cfg.strict_paper_tracker), cfg.scan_mode, 0,
                              cfg.team_warps, cfg.exact_accept, cfg.accept_tol_log2,
                              int(cfg.debug_recheck))
    t0 = time.perf_counter()
    _lib.check(_lib.lib().bnmc_gpu_run_chains(
        cache.handle, seeds, nc, C.byref(params), _lib.ptr(out.trace_proposed),
        _lib.ptr(out.trace_accepted), _lib.ptr(out.trace_best), _lib.ptr(out.final_order),
        _lib.ptr(out.final_score), _lib.ptr(out.accepted), _lib.ptr(out.tracker_count),
        _lib.ptr(out.tracker_masks), _lib.ptr(out.tracker_totals), C.byref(ms)))
    out.wall_s = time.perf_counter() - t0
    out.device_ms = ms.value
    return out


def run_chains(cache: ScoreCache, priors, seeds, cfg: RunConfig, out: ChainBatch | None = None):
    """Independent chains (chain c == run_mcmc with seed seeds[c]) in one device
    loop -> ChainResults (McmcResult per chain, built lazily over pinned buffers)."""
    seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
    return ChainResults(run_chains_batch(cache, priors, seeds, cfg, out), seeds)


def run_mcmc(data: Dataset, cfg: RunConfig, priors=None, prebuilt: ScoreCache | None = None):
    """run_mcmc (sampler.cpp:58-116): cache build (unless prebuilt), then one chain."""
    cfg.validate()
    if data.rows() == 0:
        raise DataError("learning requires at least one row")
    pr = _prior_array(priors)
    if pr is not None and pr.shape[0] != data.n:
        raise DataError("prior matrix does not match the dataset's node count")
    if prebuilt is not None and prebuilt.n() != data.n:
        raise DataError("prebuilt cache does not match the dataset's node count")
    t0 = time.perf_counter()
    cache = prebuilt if prebuilt is not None else ScoreCache.build(data, cfg, pr)
    pre = time.perf_counter() - t0
    r = run_chains(cache, pr, [cfg.seed], cfg)[0]
    r.preprocess_seconds = pre
    return r


# ------------------------------------------------------------------ synth
def synth_instance(n, max_parents, m, cards, seed=7, edge_prob=0.3, concentration=1.0,
                   tags=(101, 102, 103)):
    """Reference-identical synthetic instance (include/bnmc_synth.h) -> (cells, truth)."""
    cards = np.ascontiguousarray(cards, np.int32)
    cells = np.empty(m * n, np.uint8)
    truth = np.empty(n, np.uint64)
    _lib.check_synth(_lib.lib().bnmc_synth_instance(n, max_parents, edge_prob, concentration, m,
                                                     cards, seed, tags[0], tags[1], tags[2],
                                                     cells, truth))
    return cells.reshape(m, n), truth


def synth_priors(n, truth, seed=7, tag=104):
    out = np.empty(n * n, np.float64)
    _lib.check_synth(_lib.lib().bnmc_synth_priors(n, np.ascontiguousarray(truth, np.uint64), seed,
                                                   tag, out))
    return out.reshape(n, n)


BASELINE_CONFIGS = {
    # SURVEY §8d / BASELINE.json configs: n, k, m, cards rule, priors
    "cfg1": dict(n=11, k=3, m=1000, cards="3", priors=False),
    "cfg2": dict(n=20, k=4, m=2000, cards="3", priors=False),
    "cfg3": dict(n=37, k=4, m=5000, cards="2+i%3", priors=True),
    "cfg4": dict(n=60, k=4, m=10000, cards="3", priors=True),
    "cfg5": dict(n=64, k=5, m=20000, cards="3", priors=True),
}


def baseline_instance(name):
    """(Dataset, priors or None, RunConfig) for a BASELINE config, seed 7."""
    c = BASELINE_CONFIGS[name]
    n = c["n"]
    cards = np.array([3] * n if c["cards"] == "3" else [2 + (i % 3) for i in range(n)], np.int32)
    cells, truth = synth_instance(n, c["k"], c["m"], cards, seed=7)
    pr = synth_priors(n, truth, seed=7) if c["priors"] else None
    cfg = RunConfig(max_parents=c["k"], gamma=0.1, ess=1.0, track_top=10,
                    memory_cap_bytes=(1 << 64) - 1)
    return Dataset(cards, cells), pr, cfg, truth
