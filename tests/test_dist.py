"""CPU, world_size 2 over gloo: the multi-GPU host logic (the union of
disjoint part tables by an int64 sum all-reduce, the end-of-run chain-record
gather, the K1 prefix partition) on CPU tensors — the library runs the same
exchanges over its NCCL communicator on the GPU (bnmc_gpu_comm_*)."""
import os
import socket

import numpy as np
import pytest

from paper_1210_5128_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, S, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # part tables: disjoint words (every entry has one writer), zero elsewhere,
        # including -0.0 and NaN payloads that a float sum would not preserve
        rng = np.random.default_rng(0)
        full = rng.normal(size=(n, S))
        full[0, 0], full[-1, -1] = -0.0, np.nan
        owner = rng.integers(0, world, size=(n, S))
        part = np.where(owner == rank, full, 0.0)
        words = torch.from_numpy(part.view(np.int64).copy())
        D.union_of_parts(words)
        ok_rows = bool(np.array_equal(words.numpy().view(np.uint64), full.view(np.uint64)))

        class R:  # minimal chain result
            pass
        recs = []
        for c, seed in enumerate(D.chain_seeds(1, rank, 3, step=0, world=world)):
            r = R()
            r.seed = int(seed)
            r.accepted = 10 * rank + c
            r.tracker_totals = np.array([-100.0 - rank * 3 - c])
            r.final_score = -200.0
            r.tracker_masks = np.array([[c, rank, 7]], np.uint64)
            r.final_order = np.array([2, 0, 1])
            recs.append(D.chain_record(r, 3))
        allrec = D.gather_chain_records(np.stack(recs))
        q.put((rank, ok_rows, allrec))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [7, 60])
def test_gloo_world2_row_allgather_and_chain_gather(n):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, 5, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort(key=lambda x: x[0])
    for rank, ok_rows, allrec in out:
        assert ok_rows
        assert allrec.shape == (6, 4 + 2 * 3)
        dec = [D.decode_record(r, 3) for r in allrec]
        assert [d["seed"] for d in dec] == [1, 2, 3, 4, 5, 6]  # global chain ids
        best = D.best_overall(allrec, 3)
        assert best["best_total"] == -100.0 and best["seed"] == 1
        assert list(best["best_masks"]) == [0, 0, 7]
    np.testing.assert_array_equal(out[0][2], out[1][2])


def test_k1_partition_through_dist():
    cuts = D.k1_partition(np.full(60, 3, np.int32), 10000, 60, 4, 8)
    assert cuts[0] == 0 and cuts[-1] == 523686 and np.all(np.diff(cuts.astype(np.int64)) > 0)


def test_chain_seeds_are_global_ids():
    s = [D.chain_seeds(1, r, 4, step=k, world=2) for k in range(2) for r in range(2)]
    flat = np.concatenate(s)
    assert list(flat) == list(range(1, 17))


def test_chain_records_from_batch_roundtrip():
    """The bench's per-chain records (ChainBatch -> fixed-size int64 records)
    decode back to the batch's values; best_overall picks the best chain."""
    from paper_1210_5128_b200.api import ChainBatch
    n, C_, K, I = 5, 4, 3, 2
    rng = np.random.default_rng(0)
    b = ChainBatch(np.zeros((C_, I)), np.zeros((C_, I), np.uint8), np.zeros((C_, I)),
                   np.stack([rng.permutation(n) for _ in range(C_)]).astype(np.int32),
                   rng.normal(size=C_) - 10, np.arange(C_, dtype=np.uint64) * 7,
                   np.full(C_, K, np.int32), rng.integers(0, 1 << 62, (C_, K, n)).astype(np.uint64),
                   -np.sort(rng.random((C_, K)))[:, ::-1] * 0 - rng.random((C_, 1)) * 100,
                   0.0, 0.0)
    seeds = np.arange(11, 11 + C_, dtype=np.uint64)
    rec = D.chain_records_from_batch(b, seeds, n)
    for c in range(C_):
        d = D.decode_record(rec[c], n)
        assert d["seed"] == 11 + c and d["accepted"] == 7 * c
        assert d["best_total"] == b.tracker_totals[c, 0] and d["final_score"] == b.final_score[c]
        np.testing.assert_array_equal(d["best_masks"], b.tracker_masks[c, 0])
        np.testing.assert_array_equal(d["final_order"], b.final_order[c])
    assert D.best_overall(rec, n)["seed"] == 11 + int(np.argmax(b.tracker_totals[:, 0]))
