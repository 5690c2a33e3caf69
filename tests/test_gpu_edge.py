"""GPU parity beyond the BASELINE configs: the reference's edge cases and
randomized instances through the C-ABI, checked against the plain-C oracle and
(when present) the unmodified reference in oracle/_ref. Integer/index results
and fp64 scores bit-exact."""
import itertools

import numpy as np
import pytest

import paper_1210_5128_b200 as P
from paper_1210_5128_b200 import _lib
from oracle import port, ref

pytestmark = pytest.mark.gpu
needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


def rand_instance(seed, n, m, cmax=4):
    rng = np.random.default_rng(seed)
    cards = rng.integers(2, cmax + 1, n).astype(np.int32)
    cells = (rng.integers(0, 1 << 30, (m, n)) % cards).astype(np.uint8)
    return cells, cards


@pytest.mark.parametrize("seed,n,m,s", [(1, 5, 50, 2), (2, 9, 300, 4), (3, 13, 1000, 3),
                                        (4, 8, 33, 5), (5, 16, 257, 4), (6, 6, 0, 3),
                                        (7, 2, 10, 1), (8, 1, 10, 4), (9, 10, 64, 0)])
def test_random_tables_bit_exact(seed, n, m, s):
    cells, cards = rand_instance(seed, n, m)
    cfg = P.RunConfig(max_parents=s, gamma=0.3, ess=2.0)
    t = P.ScoreCache.build(P.Dataset(cards, cells), cfg).table()
    o = port.cache_build(cells, cards, s, 0.3, 2.0)
    np.testing.assert_array_equal(t.view(np.uint64), o.view(np.uint64))


def test_k2_mode_bit_exact():
    cells, cards = rand_instance(11, 8, 400)
    cfg = P.RunConfig(max_parents=3, gamma=0.5, alpha_mode=P.AlphaMode.K2)
    t = P.ScoreCache.build(P.Dataset(cards, cells), cfg).table()
    o = port.cache_build(cells, cards, 3, 0.5, 1.0, k2=True)
    np.testing.assert_array_equal(t.view(np.uint64), o.view(np.uint64))


@needs_ref
def test_count_statistics_bit_exact():
    cells, cards = rand_instance(12, 9, 777)
    rng = np.random.default_rng(0)
    nodes, psets = [], []
    for _ in range(64):
        v = int(rng.integers(9))
        ps = int(rng.integers(1 << 9)) & ~(1 << v)
        while bin(ps).count("1") > 4:
            ps &= ps - 1
        nodes.append(v)
        psets.append(ps)
    sizes = [int(np.prod([cards[p] for p in range(9) if ps >> p & 1])) * int(cards[v])
             for v, ps in zip(nodes, psets)]
    offs = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.uint64)
    out = np.zeros(sum(sizes), np.uint32)
    cfgs = np.zeros(64, np.uint64)
    _lib.check(_lib.lib().bnmc_gpu_count_statistics(
        np.ascontiguousarray(cells).ravel(), cards, 777, 9, 64, np.array(nodes, np.int32),
        np.array(psets, np.uint64), offs, out, cfgs, 0))
    for e in range(64):
        r = ref.count_statistics(cells, cards, nodes[e], psets[e])
        assert cfgs[e] == r.shape[0]
        np.testing.assert_array_equal(out[offs[e]:offs[e] + sizes[e]], r.ravel())


def test_capacity_and_usage_errors():
    cells, cards = rand_instance(13, 10, 50)
    d = P.Dataset(cards, cells)
    with pytest.raises(P.CapacityError):  # estimate_bytes over the cap, before allocating
        P.ScoreCache.build(d, P.RunConfig(max_parents=4, memory_cap_bytes=16))
    with pytest.raises(P.UsageError):
        P.ScoreCache.build(d, P.RunConfig(max_parents=9))
    big = P.Dataset([256] * 6, np.zeros((4, 6), np.uint8))  # wide path (test_gpu_wide.py)
    assert np.all(np.isfinite(P.ScoreCache.build(big, P.RunConfig(max_parents=4)).table()))
    cache = P.ScoreCache.build(d, P.RunConfig(max_parents=2))
    with pytest.raises(P.DataError):
        P.OrderScorer(cache).score([0, 1, 2, 3, 4, 5, 6, 7, 8, 8])
    with pytest.raises(P.DataError):
        P.run_mcmc(P.Dataset(cards, np.zeros((0, 10), np.uint8)), P.RunConfig(), None)


@needs_ref
def test_exhaustive_n4_all_orders():
    """criterion 1 / test_scoring.cpp:310-338: every one of the 24 orders."""
    cells, truth = ref.generate(4, 3, 300, [2] * 4, seed=41, edge_prob=0.5, concentration=0.5,
                                tags=(11, 12, 13))
    pri = np.full((4, 4), 0.5)
    pri[1, 0], pri[3, 2] = 0.75, 0.2
    cfg = P.RunConfig(max_parents=3)
    cache = P.ScoreCache.build(P.Dataset([2] * 4, cells), cfg)
    rc = ref.Cache.build(cells, [2] * 4, 3)
    perms = np.array(list(itertools.permutations(range(4))), np.int32)
    masks, best, tot = P.OrderScorer(cache, pri).score_many(perms)
    for i, perm in enumerate(perms):
        m, t = rc.score_order(perm, pri)
        np.testing.assert_array_equal(masks[i], m)
        assert tot[i] == t
        assert rc.score_graph(masks[i], pri) == pytest.approx(t, rel=1e-13)


@needs_ref
@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("strict", [False, True])
def test_chains_vs_reference_with_priors_and_strict(strict, mode):
    cells, truth = ref.generate(12, 3, 500, [3] * 12, seed=5, tags=(1, 2, 3))
    pri = ref.synth_priors(12, truth, seed=5)
    cfg = P.RunConfig(max_parents=3, iterations=800, track_top=4, strict_paper_tracker=strict,
                      scan_mode=mode)
    cache = P.ScoreCache.build(P.Dataset([3] * 12, cells), cfg, pri)
    rc = ref.Cache.build(cells, [3] * 12, 3)
    seeds = [3, 17, 99]
    many = P.run_chains(cache, pri, seeds, cfg)
    for c, seed in enumerate(seeds):
        r = ref.run_mcmc(cells, [3] * 12, 3, 800, seed, priors=pri, track_top=4, strict=strict,
                         prebuilt=rc)
        np.testing.assert_array_equal(many[c].trace_proposed, r.trace_proposed)
        np.testing.assert_array_equal(many[c].trace_accepted, r.trace_accepted)
        np.testing.assert_array_equal(many[c].trace_best, r.trace_best)
        np.testing.assert_array_equal(many[c].tracker_masks, r.tracker_masks)
        np.testing.assert_array_equal(many[c].final_order, r.final_order)
        assert many[c].accepted == r.accepted and many[c].final_score == r.final_score


@pytest.mark.parametrize("mode", [1, 2])
def test_tie_heavy_chain_matches_oracle(mode):
    """m tiny + gamma 1: many exact ties on fp32 AND fp64 keys, every scan cell
    goes through the exact tie resolution."""
    cells, cards = rand_instance(21, 10, 3, cmax=2)
    cfg = P.RunConfig(max_parents=3, gamma=1.0, iterations=300, scan_mode=mode)
    cache = P.ScoreCache.build(P.Dataset(cards, cells), cfg)
    t = port.cache_build(cells, cards, 3, 1.0, 1.0)
    np.testing.assert_array_equal(cache.table(), t)
    r = P.run_chains(cache, None, [1, 2], cfg)
    for c, seed in enumerate([1, 2]):
        o = port.run_mcmc(t, 3, 300, seed)
        np.testing.assert_array_equal(r[c].trace_proposed, o["trace_proposed"])
        np.testing.assert_array_equal(r[c].tracker_masks, o["tracker_masks"])


@pytest.mark.parametrize("mode", [1, 2])
def test_set_priors_refold(mode):
    cells, cards = rand_instance(22, 8, 200)
    cfg = P.RunConfig(max_parents=3)
    cache = P.ScoreCache.build(P.Dataset(cards, cells), cfg)
    t = cache.table()
    rng = np.random.default_rng(2)
    perms = np.stack([rng.permutation(8) for _ in range(6)]).astype(np.int32)
    for k in range(3):
        pri = np.where(rng.random((8, 8)) < 0.3, rng.choice([0.0, 0.25, 0.75, 1.0], (8, 8)), 0.5)
        masks, best, tot = P.OrderScorer(cache, pri, scan_mode=mode).score_many(perms)
        for i in range(6):
            m, b, tt = port.score_order(t, 3, perms[i], pri)
            np.testing.assert_array_equal(masks[i], m)
            assert tot[i] == tt


def test_sharded_build_rows_plus_exchange_equals_full():
    """Row-sharded precompute (the multi-GPU path) on one device: build rows
    [a,b) on each shard, exchange rows, finalize -> identical table & scores."""
    import ctypes as C
    import torch
    from paper_1210_5128_b200 import dist as D
    data, pri, cfg, _ = P.baseline_instance("cfg2")
    full = P.ScoreCache.build(data, cfg, pri)
    shards = []
    for r, (a, b) in enumerate([(r * data.n // 3, (r + 1) * data.n // 3) for r in range(3)]):
        out = C.c_void_p()
        _lib.check(_lib.lib().bnmc_gpu_table_build_rows(
            data.cells.reshape(-1), data.cards, data.rows(), data.n, C.byref(cfg.score_params()),
            _lib.ptr(pri), a, b, C.byref(out)))
        shards.append((a, b, P.ScoreCache(out.value, data.n, cfg.max_parents, cfg)))
    dst = D.table_rows_tensor(shards[0][2])
    for a, b, sc in shards[1:]:
        dst[a:b] = D.table_rows_tensor(sc)[a:b]
    torch.cuda.synchronize()
    _lib.check(_lib.lib().bnmc_gpu_table_finalize(shards[0][2].handle))
    merged = shards[0][2]
    merged._priors_key = None if pri is None else np.asarray(pri).tobytes()
    np.testing.assert_array_equal(merged.table().view(np.uint64), full.table().view(np.uint64))
    perms = np.stack([np.random.default_rng(i).permutation(data.n) for i in range(8)]).astype(np.int32)
    a1 = P.OrderScorer(merged, pri).score_many(perms)
    a2 = P.OrderScorer(full, pri).score_many(perms)
    for x, y in zip(a1, a2):
        np.testing.assert_array_equal(x, y)


def test_bnsc_upload_download_roundtrip(tmp_path, golden):
    g = golden("cfg2")
    cfg = P.RunConfig(max_parents=4)
    path = str(tmp_path / "c.bnsc")
    P.write_bnsc(path, g["table"], 20, 4, cfg.gamma, cfg.ess, cfg.alpha_mode)
    cache = P.ScoreCache.load(path, cfg)
    np.testing.assert_array_equal(cache.table(), g["table"])
    cache.save(str(tmp_path / "d.bnsc"))
    assert open(path, "rb").read() == open(str(tmp_path / "d.bnsc"), "rb").read()
    assert cache.lookup(3, 0b101) == port.cache_build(g["cells"], g["cards"], 4)[3][
        port.index_of(20, 4, 3, 0b101)]


@pytest.mark.parametrize("mode", [1, 2])
def test_run_chains_many_chains_and_max(mode):
    data, pri, cfg, _ = P.baseline_instance("cfg1")
    cache = P.ScoreCache.build(data, cfg, pri)
    cfg.iterations = 50
    cfg.scan_mode = mode
    seeds = list(range(1, 65 if mode == 1 else 1001))
    rs = P.run_chains(cache, pri, seeds, cfg)
    t = cache.table()
    for c in (0, 31, 63, len(seeds) - 1):
        o = port.run_mcmc(t, 3, 50, seeds[c], pri)
        np.testing.assert_array_equal(rs[c].trace_proposed, o["trace_proposed"])
        np.testing.assert_array_equal(rs[c].tracker_masks, o["tracker_masks"])
    if mode == 1:
        with pytest.raises(P.UsageError):
            P.run_chains(cache, pri, list(range(65)), cfg)


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("seed,n,m,s", [(31, 1, 20, 3), (32, 2, 40, 1), (33, 7, 90, 0),
                                        (34, 12, 300, 5), (35, 17, 500, 4), (36, 24, 800, 2)])
def test_random_orders_both_scan_paths(seed, n, m, s, mode):
    """Order scores of random instances with random priors, both scan paths
    (full-row K2 and sorted walk / PST enumeration) vs the oracle's serial
    score_order: masks, per-node bests and totals bit-exact."""
    cells, cards = rand_instance(seed, n, m)
    rng = np.random.default_rng(seed)
    pri = np.where(rng.random((n, n)) < 0.3, rng.choice([0.0, 0.2, 0.8, 1.0], (n, n)), 0.5)
    cfg = P.RunConfig(max_parents=s)
    cache = P.ScoreCache.build(P.Dataset(cards, cells), cfg)
    t = cache.table()
    perms = np.stack([rng.permutation(n) for _ in range(16)]).astype(np.int32)
    masks, best, tot = P.OrderScorer(cache, pri, scan_mode=mode).score_many(perms)
    for i in range(16):
        om, ob, ot = port.score_order(t, s, perms[i], pri)
        np.testing.assert_array_equal(masks[i], om)
        np.testing.assert_array_equal(best[i].view(np.uint64), ob.view(np.uint64))
        assert tot[i] == ot


@pytest.mark.parametrize("tw", [1, 2, 4, 8])
def test_walk_team_sizes_identical(tw):
    """The walk kernel's team size (warps per chain) changes only scheduling:
    every chain's trace, tracker and final state equal the oracle's."""
    data, pri, cfg, _ = P.baseline_instance("cfg2")
    cache = P.ScoreCache.build(data, cfg, pri)
    cfg.iterations, cfg.scan_mode, cfg.team_warps = 120, 2, tw
    seeds = list(range(1, 38))  # not a multiple of the chains per CTA
    rs = P.run_chains(cache, pri, seeds, cfg)
    t = cache.table()
    for c in (0, 5, 36):
        o = port.run_mcmc(t, 4, 120, seeds[c], pri)
        np.testing.assert_array_equal(rs[c].trace_proposed, o["trace_proposed"])
        np.testing.assert_array_equal(rs[c].trace_best, o["trace_best"])
        np.testing.assert_array_equal(rs[c].tracker_masks, o["tracker_masks"])
        np.testing.assert_array_equal(rs[c].final_order, o["final_order"])
        assert rs[c].accepted == o["accepted"]


def test_device_acceptance_and_exact_replay():
    """mh_accept on the device (CUDA log10) with ambiguity flags vs host glibc
    thresholds: identical chains. A huge bound flags every chain, so every
    chain is replayed with host thresholds, and results are still identical."""
    import ctypes as C
    data, pri, cfg, _ = P.baseline_instance("cfg3")
    cache = P.ScoreCache.build(data, cfg, pri)
    cfg.iterations, cfg.scan_mode = 150, 2
    seeds = list(range(1, 41))
    ref_b = None
    for exact, tol in ((1, 0), (0, 0), (0, 30)):
        cfg.exact_accept, cfg.accept_tol_log2 = exact, tol
        b = P.run_chains_batch(cache, pri, seeds, cfg)
        rep = C.c_uint64()
        _lib.check(_lib.lib().bnmc_gpu_last_replayed(cache.handle, C.byref(rep)))
        if tol == 30:
            assert rep.value == len(seeds)
        if ref_b is None:
            ref_b = b
            continue
        for f in ("trace_proposed", "trace_accepted", "trace_best", "final_order", "final_score",
                  "accepted", "tracker_count", "tracker_masks", "tracker_totals"):
            np.testing.assert_array_equal(getattr(b, f), getattr(ref_b, f), err_msg=f)
    o = port.run_mcmc(cache.table(), 4, 150, seeds[7], pri)
    np.testing.assert_array_equal(ref_b.trace_proposed[7], o["trace_proposed"])


@pytest.mark.parametrize("enum_max,ylists,cap,budget,deep", [
    (0, 1, -1, 0, -1), (0, 0, -1, 0, 1), (-1, 1, -1, -1, -1), (1 << 40, 0, -1, -1, 0),
    (0, 1, 1 << 40, 1, 1), (0, 0, 1 << 40, 1, 0), (-1, 1, 1 << 40, 2, 1)])
def test_walk_tuning_paths_identical(enum_max, ylists, cap, budget, deep):
    """Every walk-path variant — all rows walked (with / without the delta-walk
    lists), default split, all rows enumerated, capped walks that fall back to
    enumeration for nearly every row — on tie-heavy and ordinary instances
    gives the oracle's chains and order scores bit for bit."""
    import ctypes as C
    for cells, cards, s, gamma in (rand_instance(21, 14, 3, cmax=2) + (3, 1.0),
                                   rand_instance(23, 16, 400) + (3, 0.2)):
        # one warp per chain: the team size whose deep-round width `deep` selects
        cfg = P.RunConfig(max_parents=s, gamma=gamma, iterations=200, scan_mode=2, team_warps=1)
        cache = P.ScoreCache.build(P.Dataset(cards, cells), cfg)
        _lib.check(_lib.lib().bnmc_gpu_table_set_walk_params(cache.handle, enum_max, ylists))
        _lib.check(_lib.lib().bnmc_gpu_table_set_walk_cap(cache.handle, cap, budget, deep))
        t = port.cache_build(cells, cards, s, gamma, 1.0)
        rs = P.run_chains(cache, None, [1, 2, 3], cfg)
        for c, seed in enumerate([1, 2, 3]):
            o = port.run_mcmc(t, s, 200, seed)
            np.testing.assert_array_equal(rs[c].trace_proposed, o["trace_proposed"])
            np.testing.assert_array_equal(rs[c].tracker_masks, o["tracker_masks"])
            np.testing.assert_array_equal(rs[c].final_order, o["final_order"])
        perms = np.stack([np.random.default_rng(i).permutation(cells.shape[1])
                          for i in range(6)]).astype(np.int32)
        masks, best, tot = P.OrderScorer(cache, None, scan_mode=2).score_many(perms)
        for i in range(6):
            om, ob, ot = port.score_order(t, s, perms[i])
            np.testing.assert_array_equal(masks[i], om)
            assert tot[i] == ot


def test_randomized_instances_all_paths():
    """Property test over random instances (sizes, cardinalities, s, gamma, ess,
    K2, priors incl. extremes, tiny and empty samples): device table, order
    scores and chains on both scan paths equal the oracle's bit for bit."""
    rng = np.random.default_rng(2024)
    for trial in range(14):
        n = int(rng.integers(2, 23))
        s = int(rng.integers(0, 6))
        m = int(rng.choice([0, 1, 7, 60, 400]))
        cells, cards = rand_instance(1000 + trial, n, m, cmax=int(rng.integers(2, 5)))
        gamma, ess, k2 = float(rng.choice([0.1, 0.5, 1.0])), float(rng.choice([1.0, 3.0])), bool(trial % 3 == 0)
        pri = np.where(rng.random((n, n)) < 0.3, rng.choice([0.0, 0.1, 0.9, 1.0], (n, n)), 0.5)
        cfg = P.RunConfig(max_parents=s, gamma=gamma, ess=ess,
                          alpha_mode=P.AlphaMode.K2 if k2 else P.AlphaMode.BDEU, iterations=60)
        cache = P.ScoreCache.build(P.Dataset(cards, cells), cfg)
        t = port.cache_build(cells, cards, s, gamma, ess, k2=k2)
        np.testing.assert_array_equal(cache.table().view(np.uint64), t.view(np.uint64))
        perms = np.stack([rng.permutation(n) for _ in range(4)]).astype(np.int32)
        for mode in (1, 2):
            masks, best, tot = P.OrderScorer(cache, pri, scan_mode=mode).score_many(perms)
            for i in range(4):
                om, ob, ot = port.score_order(t, s, perms[i], pri)
                np.testing.assert_array_equal(masks[i], om)
                assert tot[i] == ot
            if n >= 2 and m > 0:
                cfg.scan_mode = mode
                rs = P.run_chains(cache, pri, [trial + 1, trial + 50], cfg)
                for c, seed in enumerate([trial + 1, trial + 50]):
                    o = port.run_mcmc(t, s, 60, seed, pri)
                    np.testing.assert_array_equal(rs[c].trace_proposed, o["trace_proposed"])
                    np.testing.assert_array_equal(rs[c].tracker_masks, o["tracker_masks"])


@pytest.mark.parametrize("strict", [False, True])
@pytest.mark.parametrize("tol,exact", [(0, 0), (30, 0), (0, 1)])
def test_speculative_single_chain_kernel(strict, tol, exact):
    """Few chains and >= 1000 iterations run the speculative kernel (4
    proposals per round against the current order, committed in run_mcmc
    order). Strict and default trackers, device acceptance (with every chain
    forced through the exact replay) and host thresholds: all equal the
    oracle; plus a tie-heavy instance."""
    import ctypes as C
    data, pri, cfg, _ = P.baseline_instance("cfg2")
    rng = np.random.default_rng(3)
    pri = np.where(rng.random((20, 20)) < 0.2, rng.choice([0.1, 0.9], (20, 20)), 0.5)
    cache = P.ScoreCache.build(data, cfg, pri)
    cfg.iterations, cfg.scan_mode, cfg.strict_paper_tracker = 1200, 2, strict
    cfg.exact_accept, cfg.accept_tol_log2 = exact, tol
    seeds = [5, 6]
    rs = P.run_chains(cache, pri, seeds, cfg)
    rep = C.c_uint64()
    _lib.check(_lib.lib().bnmc_gpu_last_replayed(cache.handle, C.byref(rep)))
    if tol == 30:
        assert rep.value == len(seeds)
    t = cache.table()
    for c, seed in enumerate(seeds):
        o = port.run_mcmc(t, 4, 1200, seed, pri, strict=strict)
        np.testing.assert_array_equal(rs[c].trace_proposed, o["trace_proposed"])
        np.testing.assert_array_equal(rs[c].trace_accepted, o["trace_accepted"])
        np.testing.assert_array_equal(rs[c].trace_best, o["trace_best"])
        np.testing.assert_array_equal(rs[c].tracker_masks, o["tracker_masks"])
        np.testing.assert_array_equal(rs[c].final_order, o["final_order"])
        assert rs[c].accepted == o["accepted"] and rs[c].final_score == o["final_score"]
    if tol == 0 and exact == 0 and not strict:
        cells, cards = rand_instance(21, 14, 3, cmax=2)
        c2 = P.RunConfig(max_parents=3, gamma=1.0, iterations=1100, scan_mode=2)
        cc = P.ScoreCache.build(P.Dataset(cards, cells), c2)
        r2 = P.run_chains(cc, None, [1, 2], c2)
        t2 = port.cache_build(cells, cards, 3, 1.0, 1.0)
        for c, seed in enumerate([1, 2]):
            o = port.run_mcmc(t2, 3, 1100, seed)
            np.testing.assert_array_equal(r2[c].trace_proposed, o["trace_proposed"])
            np.testing.assert_array_equal(r2[c].tracker_masks, o["tracker_masks"])


def test_walk_cap_argument_errors():
    """set_walk_cap validates its mode and budget (usage error, table unchanged)."""
    cells, cards = rand_instance(5, 8, 50)
    cfg = P.RunConfig(max_parents=2, iterations=20, scan_mode=2)
    cache = P.ScoreCache.build(P.Dataset(cards, cells), cfg)
    L = _lib.lib()
    assert L.bnmc_gpu_table_set_walk_cap(cache.handle, -1, -1, 2) == 2
    assert L.bnmc_gpu_table_set_walk_cap(cache.handle, -1, 1 << 20, -1) == 2
    assert L.bnmc_gpu_table_set_walk_cap(cache.handle, -1, -1, -1) == 0
    t = port.cache_build(cells, cards, 2, 0.1, 1.0)
    r = P.run_chains(cache, None, [4], cfg)[0]
    np.testing.assert_array_equal(r.trace_proposed, port.run_mcmc(t, 2, 20, 4)["trace_proposed"])


def test_walk_variants_stress():
    """Random instances (n up to 30, s up to 5, priors) through every walk
    variant — team sizes 1/2/4/8/32, deep rounds off/on, capped walks off /
    budget 1 / default — against the oracle's chains bit for bit.
    BNMC_STRESS_TRIALS raises the instance count (default 8; 200 passed)."""
    import os
    trials = int(os.environ.get("BNMC_STRESS_TRIALS", "8"))
    rng = np.random.default_rng(77)
    L = _lib.lib()
    for trial in range(trials):
        n = int(rng.integers(8, 31))
        s = int(rng.integers(1, 6))
        m = int(rng.choice([30, 200, 1000]))
        cells, cards = rand_instance(3000 + trial, n, m, cmax=int(rng.integers(2, 4)))
        pri = np.where(rng.random((n, n)) < 0.2, rng.choice([0.1, 0.3, 0.7, 0.9], (n, n)), 0.5)
        iters = 80
        cfg = P.RunConfig(max_parents=s, iterations=iters, scan_mode=2)
        cache = P.ScoreCache.build(P.Dataset(cards, cells), cfg, pri)
        t = port.cache_build(cells, cards, s, 0.1, 1.0)
        seeds = [trial * 7 + 1, trial * 7 + 2]
        want = [port.run_mcmc(t, s, iters, sd, pri) for sd in seeds]
        for tw, deep, budget in ((1, 0, -1), (1, 1, 1), (2, 1, 0), (4, 0, 1), (8, -1, -1),
                                 (32, -1, 1)):
            _lib.check(L.bnmc_gpu_table_set_walk_cap(cache.handle, -1, budget, deep))
            cfg.team_warps = tw
            rs = P.run_chains(cache, pri, seeds, cfg)
            for r, o in zip(rs, want):
                np.testing.assert_array_equal(r.trace_proposed, o["trace_proposed"])
                np.testing.assert_array_equal(r.tracker_masks, o["tracker_masks"])
                np.testing.assert_array_equal(r.final_order, o["final_order"])
