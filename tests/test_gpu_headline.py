"""GPU parity of the exact kernel variants that produce the headline numbers,
against the UNMODIFIED reference (oracle/_ref) on the same GPU-built table
(BNSC export -> ScoreCache::load), plus the debug_recheck cadence and live
walk re-tuning.

* cfg4 (the bench workload) with team_warps=1: walk_chain_kernel<1,4>, the
  variant the 18,944-chain bench launch auto-selects; 64 chains x 200
  iterations, every chain's trace, tracker and final state vs the reference's
  run_mcmc with that seed (sampler.cpp:58-116).
* cfg5 with team_warps=1 on rows longer than 2^21 entries:
  walk_chain_kernel<1,8> (deep rounds), 200 iterations vs the reference.
"""
import os
import tempfile

import numpy as np
import pytest

import paper_1210_5128_b200 as P
from paper_1210_5128_b200 import _lib
from oracle import port, ref

pytestmark = pytest.mark.gpu
needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


def ref_cache_of(cache, cfg):
    """The reference's ScoreCache::load of our table (scoring.cpp:210-238)."""
    tmp = "/dev/shm" if os.path.isdir("/dev/shm") else None
    with tempfile.TemporaryDirectory(dir=tmp) as d:
        path = os.path.join(d, "t.bnsc")
        cache.save(path)
        return ref.Cache.load(path, cfg.max_parents, cfg.gamma, cfg.ess, False)


def assert_chain_equal(ours, r, what):
    np.testing.assert_array_equal(ours.trace_proposed.view(np.uint64),
                                  r.trace_proposed.view(np.uint64), err_msg=what)
    np.testing.assert_array_equal(np.asarray(ours.trace_accepted, bool), r.trace_accepted,
                                  err_msg=what)
    np.testing.assert_array_equal(ours.trace_best.view(np.uint64), r.trace_best.view(np.uint64),
                                  err_msg=what)
    np.testing.assert_array_equal(ours.tracker_masks, r.tracker_masks, err_msg=what)
    np.testing.assert_array_equal(ours.tracker_totals.view(np.uint64),
                                  r.tracker_totals.view(np.uint64), err_msg=what)
    np.testing.assert_array_equal(ours.final_order, r.final_order, err_msg=what)
    assert ours.final_score == r.final_score and ours.accepted == r.accepted, what


def ref_chain(rc, n, s, iters, seed, pri):
    return ref.run_mcmc(np.zeros((1, n), np.uint8), np.full(n, 3, np.int32), s, iters, seed,
                        priors=pri, prebuilt=rc)


@pytest.fixture(scope="module")
def cfg4():
    data, pri, cfg, _ = P.baseline_instance("cfg4")
    cache = P.ScoreCache.build(data, cfg, pri)
    return data, pri, cfg, cache


@needs_ref
def test_cfg4_one_warp_chains_vs_reference(cfg4):
    data, pri, cfg, cache = cfg4
    iters, chains = 200, 64
    seeds = [1 + 977 * c for c in range(chains)]
    c1 = P.RunConfig(max_parents=cfg.max_parents, iterations=iters, team_warps=1, scan_mode=2,
                     memory_cap_bytes=cfg.memory_cap_bytes)
    ours = P.run_chains(cache, pri, seeds, c1)
    stats = cache.last_walk_stats()
    assert stats["team_warps"] == 1 and stats["variant"] == "walk_chain_kernel<1,4>"
    rc = ref_cache_of(cache, cfg)
    for c, sd in enumerate(seeds):
        assert_chain_equal(ours[c], ref_chain(rc, data.n, cfg.max_parents, iters, sd, pri),
                           f"chain {c} seed {sd}")


@needs_ref
def test_cfg5_deep_one_warp_chains_vs_reference():
    data, pri, cfg, _ = P.baseline_instance("cfg5")
    cache = P.ScoreCache.build(data, cfg, pri)
    iters = 200
    seeds = [1, 2]
    c1 = P.RunConfig(max_parents=cfg.max_parents, iterations=iters, team_warps=1, scan_mode=2,
                     memory_cap_bytes=cfg.memory_cap_bytes)
    ours = P.run_chains(cache, pri, seeds, c1)
    stats = cache.last_walk_stats()
    assert stats["team_warps"] == 1 and stats["variant"] == "walk_chain_kernel<1,8>"
    rc = ref_cache_of(cache, cfg)
    for c, sd in enumerate(seeds):
        assert_chain_equal(ours[c], ref_chain(rc, data.n, cfg.max_parents, iters, sd, pri),
                           f"cfg5 seed {sd}")


@pytest.mark.parametrize("tw", [1, 4, 8, 32])
def test_debug_recheck_passes_and_changes_nothing(tw, golden):
    """RunConfig::debug_recheck (sampler.cpp:105-110): every 100 iterations the
    device re-scores the current order from scratch; a healthy chain passes and
    its results are those of the unchecked run (and the reference golden)."""
    data, pri, cfg, _ = P.baseline_instance("cfg2")
    cache = P.ScoreCache.build(data, cfg, pri)
    g = golden("cfg2")  # reference run_mcmc, seed 1, 2000 iterations
    it = g["trace_proposed"].size
    base = P.RunConfig(max_parents=cfg.max_parents, iterations=it, team_warps=tw, scan_mode=2)
    chk = P.RunConfig(max_parents=cfg.max_parents, iterations=it, team_warps=tw, scan_mode=2,
                      debug_recheck=True)
    seeds = [1, 2, 3]
    a = P.run_chains(cache, pri, seeds, base)
    b = P.run_chains(cache, pri, seeds, chk)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x.trace_proposed, y.trace_proposed)
        np.testing.assert_array_equal(x.tracker_masks, y.tracker_masks)
        np.testing.assert_array_equal(x.final_order, y.final_order)
    np.testing.assert_array_equal(b[0].trace_proposed, g["trace_proposed"])
    np.testing.assert_array_equal(b[0].final_order, g["final_order"])


def test_debug_recheck_needs_walk_path():
    data, pri, cfg, _ = P.baseline_instance("cfg1")
    cache = P.ScoreCache.build(data, cfg, pri)
    c1 = P.RunConfig(max_parents=cfg.max_parents, iterations=10, scan_mode=1, debug_recheck=True)
    with pytest.raises(P.UsageError):
        P.run_chains(cache, pri, [1], c1)


def test_walk_cap_retune_rebuilds_pst():
    """set_walk_cap on a table whose sorted rows already exist takes effect
    (the PST tables are rebuilt) and results stay identical."""
    data, pri, cfg, _ = P.baseline_instance("cfg3")
    cache = P.ScoreCache.build(data, cfg, pri)
    c1 = P.RunConfig(max_parents=cfg.max_parents, iterations=300, team_warps=1, scan_mode=2)
    seeds = list(range(1, 33))
    L = _lib.lib()
    a = P.run_chains(cache, pri, seeds, c1)
    sa = cache.last_walk_stats()
    _lib.check(L.bnmc_gpu_table_set_walk_cap(cache.handle, -1, 0, -1))  # no capped walks
    b = P.run_chains(cache, pri, seeds, c1)
    sb = cache.last_walk_stats()
    _lib.check(L.bnmc_gpu_table_set_walk_cap(cache.handle, 1 << 40, 1, -1))  # cap everything at 1x
    c = P.run_chains(cache, pri, seeds, c1)
    sc = cache.last_walk_stats()
    for x, y, z in zip(a, b, c):
        np.testing.assert_array_equal(x.trace_proposed, y.trace_proposed)
        np.testing.assert_array_equal(x.trace_proposed, z.trace_proposed)
    # without caps only PST(p <= pe) rows enumerate; capping every row at one
    # walk budget enumerates far more
    assert sb["enumerated"] <= sa["enumerated"] < sc["enumerated"]
    assert sc["walked"] < sb["walked"]
    t = port.cache_build(data.cells, data.cards, cfg.max_parents)
    o = port.run_mcmc(t, cfg.max_parents, 300, 1, pri)
    np.testing.assert_array_equal(a[0].trace_proposed, o["trace_proposed"])


def test_pipelined_chain_blocks_equal_single_launch(cfg4):
    """>= 16,384 chains with page-locked result buffers run as chain blocks on
    two streams with overlapped result copies (walk_launch); pageable buffers
    take the single launch. Both must give the same bytes, chain by chain, and
    sampled chains equal the plain-C oracle."""
    data, pri, cfg, cache = cfg4
    c = P.RunConfig(max_parents=cfg.max_parents, iterations=40, track_top=cfg.track_top,
                    memory_cap_bytes=cfg.memory_cap_bytes)
    seeds = np.arange(1, 16385, dtype=np.uint64)
    n = data.n
    pinned = P.run_chains_batch(cache, pri, seeds, c)  # pooled page-locked buffers
    pageable = P.run_chains_batch(cache, pri, seeds, c,
                                  P.api.ChainBatch.allocate(seeds.size, 40, n, c.track_top,
                                                            pinned=False))
    for f in ("trace_proposed", "trace_accepted", "trace_best", "final_order", "final_score",
              "accepted", "tracker_count", "tracker_masks", "tracker_totals"):
        np.testing.assert_array_equal(np.asarray(getattr(pinned, f)).view(np.uint8),
                                      np.asarray(getattr(pageable, f)).view(np.uint8), err_msg=f)
    if not ref.available():
        return
    rc = ref_cache_of(cache, cfg)
    for ci in (0, 4095, 4096, 8191, 12288, 16383):  # both sides of every block edge
        r = ref_chain(rc, n, cfg.max_parents, 40, int(seeds[ci]), pri)
        assert_chain_equal(pinned.result(ci), r, f"chain {ci}")


def test_sequential_proposal_draws_equal_batched(cfg4, monkeypatch):
    """draw_proposal_batch's sequential path (taken when a next_below draw is
    rejected, probability ~n/2^64 per draw) forced for every batch
    (BNMC_SEQ_DRAWS=1) gives the same chains as the batched path, and both
    equal the reference for a sampled chain."""
    data, pri, cfg, cache = cfg4
    c = P.RunConfig(max_parents=cfg.max_parents, iterations=100, team_warps=1, scan_mode=2,
                    memory_cap_bytes=cfg.memory_cap_bytes)
    seeds = np.arange(1, 65, dtype=np.uint64)
    batched = P.run_chains_batch(cache, pri, seeds, c, P.api.ChainBatch.allocate(64, 100, data.n,
                                                                                 c.track_top, False))
    monkeypatch.setenv("BNMC_SEQ_DRAWS", "1")
    seq = P.run_chains_batch(cache, pri, seeds, c, P.api.ChainBatch.allocate(64, 100, data.n,
                                                                             c.track_top, False))
    for f in ("trace_proposed", "trace_accepted", "trace_best", "final_order", "tracker_masks",
              "tracker_totals"):
        np.testing.assert_array_equal(np.asarray(getattr(batched, f)).view(np.uint8),
                                      np.asarray(getattr(seq, f)).view(np.uint8), err_msg=f)
    if ref.available():
        rc = ref_cache_of(cache, cfg)
        assert_chain_equal(seq.result(37), ref_chain(rc, data.n, cfg.max_parents, 100, 38, pri),
                           "sequential draws, seed 38")
