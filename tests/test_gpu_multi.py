"""GPU: multi-GPU precompute and sampling behind the C-ABI.

The box has one GPU, so the parts of a G-way build run on the same device —
sequentially (per-part K1 time and bit-exact union), as several host threads
of one process (n_gpus with BNMC_DEVICES listing device 0 G times), as a
one-rank NCCL communicator, and as two processes exchanging their parts over
gloo. Results are bit-identical to the single-GPU table and chains."""
import ctypes as C
import hashlib
import json
import os
import socket

import numpy as np
import pytest

import paper_1210_5128_b200 as P
from paper_1210_5128_b200 import _lib

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build_part(data, cfg, pri, part, nparts):
    out = C.c_void_p()
    _lib.check(_lib.lib().bnmc_gpu_table_build_part(
        data.cells.reshape(-1), data.cards, data.rows(), data.n, C.byref(cfg.score_params()),
        _lib.ptr(pri), part, nparts, C.byref(out)))
    c = P.ScoreCache(out.value, data.n, cfg.max_parents, cfg)
    k1, wide, lo, hi = C.c_float(), C.c_uint64(), C.c_uint64(), C.c_uint64()
    _lib.check(_lib.lib().bnmc_gpu_table_k1_stats(c.handle, C.byref(k1), C.byref(wide),
                                                   C.byref(lo), C.byref(hi)))
    return c, k1.value, (lo.value, hi.value)


@pytest.mark.parametrize("name", ["cfg2", "cfg3"])
@pytest.mark.parametrize("G", [2, 3, 8])
def test_parts_union_is_the_table(name, G):
    data, pri, cfg, _ = P.baseline_instance(name)
    full = P.ScoreCache.build(data, cfg, pri).table()
    acc = np.zeros(full.shape, np.uint64)
    ranges = []
    for g in range(G):
        c, _, rg = build_part(data, cfg, pri, g, G)
        t = c.table().view(np.uint64)
        assert not np.any((acc != 0) & (t != 0)), "parts overlap"
        acc += t
        ranges.append(rg)
        c.close()
    assert ranges[0][0] == 0 and all(ranges[i][1] == ranges[i + 1][0] for i in range(G - 1))
    np.testing.assert_array_equal(acc, full.view(np.uint64))


def test_part_k1_times_balance_cfg4():
    """Per-part K1 time (parts run one after another on this GPU): the slowest
    part stays within 1.3x of the single-GPU K1 time / G."""
    data, pri, cfg, _ = P.baseline_instance("cfg4")
    P.ScoreCache.build(data, cfg, pri).close()  # warm-up (module load, LUT)
    one = P.ScoreCache.build(data, cfg, pri)
    k1_one = one.build_ms[0]
    one.close()
    report = {"config": "cfg4", "k1_one_gpu_ms": k1_one, "parts": {}}
    for G in (2, 4, 8):
        times = []
        for g in range(G):
            c, ms, _ = build_part(data, cfg, pri, g, G)
            times.append(ms)
            c.close()
        report["parts"][G] = {"ms": times, "max_over_ideal": max(times) / (k1_one / G)}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "k1_parts_cfg4.json"), "w") as f:
        json.dump(report, f, indent=1)
    for G, r in report["parts"].items():
        assert r["max_over_ideal"] <= 1.3, (G, r)


def test_n_gpus_replicas_on_one_device(monkeypatch):
    """n_gpus = 3 over device 0 three times: split K1 + combine + replicas;
    chains spread over the replicas equal the single-table chains."""
    data, pri, cfg, _ = P.baseline_instance("cfg3")
    single = P.ScoreCache.build(data, cfg, pri)
    monkeypatch.setenv("BNMC_DEVICES", "0,0,0")
    cfg3 = P.RunConfig(**{**cfg.__dict__, "n_gpus": 3})
    multi = P.ScoreCache.build(data, cfg3, pri)
    cnt = C.c_int()
    devs = np.zeros(8, np.int32)
    _lib.check(_lib.lib().bnmc_gpu_table_devices(multi.handle, C.byref(cnt), devs))
    assert cnt.value == 3 and list(devs[:3]) == [0, 0, 0]
    np.testing.assert_array_equal(multi.table().view(np.uint64), single.table().view(np.uint64))
    cfg.iterations = cfg3.iterations = 150
    seeds = list(range(1, 301))
    a = P.run_chains_batch(single, pri, seeds, cfg)
    b = P.run_chains_batch(multi, pri, seeds, cfg3)
    for f in ("trace_proposed", "trace_best", "final_order", "final_score", "accepted",
              "tracker_count", "tracker_masks", "tracker_totals"):
        np.testing.assert_array_equal(np.asarray(getattr(a, f)).view(np.uint8),
                                      np.asarray(getattr(b, f)).view(np.uint8), err_msg=f)
    np.testing.assert_array_equal(a.trace_accepted, b.trace_accepted)


def test_comm_single_rank_nccl():
    """bnmc_gpu_comm_* with one rank: NCCL loads, the comm build equals the
    table, all-gather / all-reduce-max round-trip host data."""
    L = _lib.lib()
    uid = np.zeros(128, np.uint8)
    _lib.check(L.bnmc_gpu_comm_unique_id(uid))
    comm = C.c_void_p()
    _lib.check(L.bnmc_gpu_comm_init(uid, 1, 0, 0, C.byref(comm)))
    try:
        data, pri, cfg, _ = P.baseline_instance("cfg2")
        out = C.c_void_p()
        _lib.check(L.bnmc_gpu_table_build_comm(
            data.cells.reshape(-1), data.cards, data.rows(), data.n, C.byref(cfg.score_params()),
            _lib.ptr(pri), comm, C.byref(out)))
        c = P.ScoreCache(out.value, data.n, cfg.max_parents, cfg)
        ref = P.ScoreCache.build(data, cfg, pri).table()
        np.testing.assert_array_equal(c.table().view(np.uint64), ref.view(np.uint64))
        send = np.arange(37, dtype=np.uint8)
        recv = np.zeros(37, np.uint8)
        _lib.check(L.bnmc_gpu_comm_allgather(comm, _lib.ptr(send), 37, _lib.ptr(recv)))
        np.testing.assert_array_equal(send, recv)
        v = np.array([1.5, -2.0, 3.25])
        _lib.check(L.bnmc_gpu_comm_allreduce_max(comm, v, 3))
        np.testing.assert_array_equal(v, [1.5, -2.0, 3.25])
        bad = C.c_void_p()
        cfg.device = 0
        st = L.bnmc_gpu_comm_init(uid, 2, 5, 0, C.byref(bad))
        assert st == 2  # rank out of range
    finally:
        _lib.check(L.bnmc_gpu_comm_free(comm))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _part_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        data, pri, cfg, _ = P.baseline_instance("cfg3")
        c, ms, rg = build_part(data, cfg, pri, rank, world)
        words = torch.from_numpy(c.table().view(np.int64).copy())
        dist.all_reduce(words, op=dist.ReduceOp.SUM)  # int64 sum == union of the parts
        table = words.numpy().view(np.float64)
        q.put((rank, hashlib.sha256(table.tobytes()).hexdigest(), rg))
    finally:
        dist.destroy_process_group()


def test_two_processes_build_parts_and_exchange_over_gloo():
    import torch.multiprocessing as mp
    data, pri, cfg, _ = P.baseline_instance("cfg3")
    want = hashlib.sha256(P.ScoreCache.build(data, cfg, pri).table().tobytes()).hexdigest()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_part_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert res[0][2][1] == res[1][2][0]
    assert res[0][1] == res[1][1] == want
