"""Multi-GPU plumbing: one process per GPU over torch.distributed.

The path shards in two independent ways and has no per-iteration exchange:

* precompute: node ROWS of the score table are independent. Rank r builds rows
  ``row_partition(n, world)[r]`` with ``bnmc_gpu_table_build_rows`` and one
  all-gather over NCCL (NVLink) gives every GPU the full table
  (``all_gather_rows``);
* sampling: chains are independent replicas (chain id -> seed); at the end the
  fixed-size per-chain records are gathered once (``gather_chain_records``;
  NCCL has no gather, so it is an all-gather of equal-size records).

Everything here is backend-agnostic torch code so the same functions run with
``gloo`` on CPU tensors (tests/test_dist.py) and ``nccl`` on device buffers.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _lib


def env_rank_world():
    """(rank, world, local_rank) from the torchrun environment (defaults 0,1,0)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def row_partition(n: int, world: int):
    """Contiguous, balanced node-row blocks: rank r owns [r*n//w, (r+1)*n//w)."""
    return [(r * n // world, (r + 1) * n // world) for r in range(world)]


def chain_seeds(base_seed: int, rank: int, chains_per_rank: int, step: int = 0, world: int = 1):
    """Global chain id -> RunConfig.seed = base + id (seed = 1 + c)."""
    first = (step * world + rank) * chains_per_rank
    return np.arange(first, first + chains_per_rank, dtype=np.uint64) + np.uint64(base_seed)


class DeviceArray:
    """__cuda_array_interface__ view of a library-owned device buffer."""

    def __init__(self, ptr: int, count: int, typestr: str = "<f8"):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": typestr,
                                         "data": (ptr, False), "version": 3, "strides": None}


def table_rows_tensor(cache):
    """torch view (no copy) of the table's fp64 local-score rows on its device."""
    import torch
    ptr, nbytes, stride = C.c_void_p(), C.c_uint64(), C.c_uint64()
    _lib.check(_lib.lib().bnmc_gpu_table_rows_buffer(cache.handle, C.byref(ptr), C.byref(nbytes),
                                                      C.byref(stride)))
    t = torch.as_tensor(DeviceArray(ptr.value, nbytes.value // 8), device="cuda")
    return t.view(cache.n(), stride.value)


def all_gather_rows(rows, n: int, world: int, rank: int, group=None):
    """In-place all-gather of node-row shards of an (n, S) tensor.

    ``rows`` holds this rank's block (row_partition) and garbage elsewhere; on
    return every rank holds all n rows. Blocks are padded to equal size because
    all_gather_into_tensor needs equal chunks.
    """
    import torch
    import torch.distributed as dist
    parts = row_partition(n, world)
    per = max(b - a for a, b in parts)
    S = rows.shape[1]
    a, b = parts[rank]
    send = torch.zeros((per, S), dtype=rows.dtype, device=rows.device)
    send[: b - a] = rows[a:b]
    recv = torch.empty((world * per, S), dtype=rows.dtype, device=rows.device)
    dist.all_gather_into_tensor(recv, send, group=group)
    for r, (ra, rb) in enumerate(parts):
        if r != rank and rb > ra:
            rows[ra:rb] = recv[r * per: r * per + (rb - ra)]
    return rows


def build_table_sharded(data, cfg, priors, rank: int, world: int, group=None, force=False):
    """Row-sharded device precompute + NCCL all-gather -> full table on every GPU."""
    from .api import ScoreCache, _prior_array
    import time
    pr = _prior_array(priors)
    a, b = row_partition(data.n, world)[rank]
    out = C.c_void_p()
    t0 = time.perf_counter()
    _lib.check(_lib.lib().bnmc_gpu_table_build_rows(
        data.cells.reshape(-1), data.cards, data.rows(), data.n, C.byref(cfg.score_params()),
        _lib.ptr(pr), a, b, C.byref(out)))
    cache = ScoreCache(out.value, data.n, cfg.max_parents, cfg)
    if world > 1 or force:
        import torch
        rows = table_rows_tensor(cache)
        torch.cuda.synchronize()
        all_gather_rows(rows, data.n, world, rank, group)
        torch.cuda.synchronize()
    _lib.check(_lib.lib().bnmc_gpu_table_finalize(cache.handle))
    cache._priors_key = None if pr is None else pr.tobytes()
    cache.preprocess_seconds = time.perf_counter() - t0
    return cache


# Fixed-size per-chain record: [seed, accepted, best_total(bits), final_total(bits),
# best masks (n), final order (n)] as int64.
def chain_record(result, n: int) -> np.ndarray:
    rec = np.zeros(4 + 2 * n, dtype=np.int64)
    rec[0] = np.int64(np.uint64(result.seed).view(np.int64))
    rec[1] = result.accepted
    rec[2] = np.float64(result.tracker_totals[0]).view(np.int64)
    rec[3] = np.float64(result.final_score).view(np.int64)
    rec[4:4 + n] = np.asarray(result.tracker_masks[0], np.uint64).view(np.int64)
    rec[4 + n:] = np.asarray(result.final_order, np.int64)
    return rec


def chain_records_from_batch(batch, seeds, n: int) -> np.ndarray:
    """chain_record for every chain of a ChainBatch (api.run_chains_batch)."""
    seeds = np.asarray(seeds, np.uint64)
    C_ = seeds.size
    rec = np.zeros((C_, 4 + 2 * n), dtype=np.int64)
    rec[:, 0] = seeds.view(np.int64)
    rec[:, 1] = np.asarray(batch.accepted, np.uint64).view(np.int64)
    rec[:, 2] = np.ascontiguousarray(batch.tracker_totals[:, 0], np.float64).view(np.int64)
    rec[:, 3] = np.ascontiguousarray(batch.final_score, np.float64).view(np.int64)
    rec[:, 4:4 + n] = np.ascontiguousarray(batch.tracker_masks[:, 0, :], np.uint64).view(np.int64)
    rec[:, 4 + n:] = np.asarray(batch.final_order, np.int64)
    return rec


def decode_record(rec: np.ndarray, n: int) -> dict:
    return dict(seed=int(rec[0].view(np.uint64)), accepted=int(rec[1]),
                best_total=float(rec[2:3].view(np.float64)[0]),
                final_score=float(rec[3:4].view(np.float64)[0]),
                best_masks=rec[4:4 + n].view(np.uint64).copy(),
                final_order=rec[4 + n:].astype(np.int64))


def gather_chain_records(records: np.ndarray, group=None, device=None) -> np.ndarray:
    """All-gather of equal-size [chains, rec_len] int64 records (rank order)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    t = torch.from_numpy(np.ascontiguousarray(records))
    if device is not None:
        t = t.to(device)
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    return torch.cat(out).cpu().numpy()


def best_overall(records: np.ndarray, n: int) -> dict:
    """Best graph over all chains: highest best_total, ties -> lowest seed."""
    dec = [decode_record(r, n) for r in records]
    dec.sort(key=lambda d: (-d["best_total"], d["seed"]))
    return dec[0]
