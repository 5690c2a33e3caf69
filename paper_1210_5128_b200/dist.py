"""Multi-GPU plumbing: one process per GPU.

The path shards in two independent ways and has no per-iteration exchange:

* precompute: K1's unit of work is a prefix P (|P| <= s); every score-table
  entry belongs to exactly one prefix, so rank r computes the work-balanced
  prefix range ``bnmc_gpu_k1_partition(world)[r]`` into a zeroed table and one
  in-place all-reduce of the 64-bit table words (integer sum == union of the
  parts, bit-exact) completes the table on every GPU. This replaces the
  reference's OpenMP loop over node rows (src/scoring.cpp:179-190);
* sampling: chains are independent replicas (global chain id -> seed); at the
  end the fixed-size per-chain records are all-gathered once.

The data-path collectives run inside the library over its own NCCL
communicator (``bnmc_gpu_comm_*`` in include/bnmc_gpu.h: NVLink/NVSwitch);
torch.distributed (any backend — gloo on CPU in tests/test_dist.py) only ships
the NCCL unique id and provides barriers. The host-side pieces (record
packing, the int64 union) are backend-agnostic torch code so the same
functions run on CPU tensors over gloo.
"""
from __future__ import annotations

import ctypes as C
import os
import time

import numpy as np

from . import _lib


def env_rank_world():
    """(rank, world, local_rank) from the torchrun environment (defaults 0,1,0)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def k1_partition(cards, m: int, n: int, s: int, world: int) -> np.ndarray:
    """Prefix-index cuts of the work-balanced K1 split (world + 1 values)."""
    cuts = np.zeros(world + 1, np.uint64)
    _lib.check(_lib.lib().bnmc_gpu_k1_partition(np.ascontiguousarray(cards, np.int32), m, n, s,
                                                 world, cuts))
    return cuts


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


class Comm:
    """One rank of the library's NCCL communicator (bnmc_gpu_comm_init)."""

    def __init__(self, rank: int, world: int, device: int, group=None):
        import torch.distributed as dist
        self.rank, self.world, self.device = rank, world, device
        uid = np.zeros(128, np.uint8)
        if rank == 0:
            _lib.check(_lib.lib().bnmc_gpu_comm_unique_id(uid))
        if world > 1:
            box = [uid.tobytes()]
            dist.broadcast_object_list(box, src=0, group=group)
            uid = np.frombuffer(box[0], np.uint8).copy()
        h = C.c_void_p()
        _lib.check(_lib.lib().bnmc_gpu_comm_init(uid, world, rank, device, C.byref(h)))
        self.handle = h

    def allgather(self, arr: np.ndarray) -> np.ndarray:
        """All-gather of an equal-size array per rank -> [world, *arr.shape]."""
        a = np.ascontiguousarray(arr)
        out = np.empty((self.world,) + a.shape, a.dtype)
        _lib.check(_lib.lib().bnmc_gpu_comm_allgather(self.handle, _lib.ptr(a), a.nbytes,
                                                       _lib.ptr(out)))
        return out

    def max(self, values) -> list:
        v = np.ascontiguousarray(values, np.float64).copy()
        _lib.check(_lib.lib().bnmc_gpu_comm_allreduce_max(self.handle, v, v.size))
        return v.tolist()

    def close(self):
        if getattr(self, "handle", None) and self.handle.value:
            _lib.lib().bnmc_gpu_comm_free(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def build_table_comm(data, cfg, priors, comm: Comm):
    """ScoreCache::build split over the ranks of `comm`: part `rank` of the
    K1 prefix partition, NCCL all-reduce of the table words, PPF fold."""
    from .api import ScoreCache, _prior_array
    pr = _prior_array(priors)
    out = C.c_void_p()
    t0 = time.perf_counter()
    _lib.check(_lib.lib().bnmc_gpu_table_build_comm(
        data.cells.reshape(-1), data.cards, data.rows(), data.n, C.byref(cfg.score_params()),
        _lib.ptr(pr), comm.handle, C.byref(out)))
    cache = ScoreCache(out.value, data.n, cfg.max_parents, cfg)
    cache._priors_key = None if pr is None else pr.tobytes()
    cache.preprocess_seconds = time.perf_counter() - t0
    a, b = C.c_float(), C.c_float()
    _lib.check(_lib.lib().bnmc_gpu_table_build_ms(cache.handle, C.byref(a), C.byref(b)))
    cache.build_ms = (a.value, b.value)
    return cache


def union_of_parts(words, group=None):
    """In-place integer sum of part tables viewed as int64 words (torch tensor
    on any backend): each word has one writer, so the sum is the union."""
    import torch.distributed as dist
    dist.all_reduce(words, op=dist.ReduceOp.SUM, group=group)
    return words


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
    """All-gather of equal-size [chains, rec_len] int64 records (rank order)
    over torch.distributed (the CPU/gloo form of Comm.allgather)."""
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
