"""Small invocations of every device kernel family, for compute-sanitizer
(racecheck / memcheck / synccheck; tools/sanitize.sh). Each case is checked
against the plain-C oracle so a sanitizer run is also a parity run.

    python tools/sanitize_run.py k1|walk1|walk8|walk32|spec|scan|recheck|all
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1210_5128_b200 as P  # noqa: E402
from oracle import port  # noqa: E402


def instance(name="cfg2", m=None):
    data, pri, cfg, _ = P.baseline_instance(name)
    if m is not None:
        data = P.Dataset(data.cards, data.cells[:m])
    return data, pri, cfg


def case_k1():
    for name in ("cfg1", "cfg2", "cfg3"):
        data, pri, cfg = instance(name, m=300)
        cache = P.ScoreCache.build(data, cfg, pri)
        t = cache.table()
        cache.close()
        ref = port.cache_build(data.cells, data.cards, cfg.max_parents)
        assert np.array_equal(t.view(np.uint64), ref.view(np.uint64)), name
        print(f"k1 {name}: ok")


def chains(tw, iters, nchains, recheck=False, name="cfg2"):
    data, pri, cfg = instance(name, m=500)
    cache = P.ScoreCache.build(data, cfg, pri)
    ref = cache.table()
    cfg.iterations, cfg.team_warps, cfg.debug_recheck = iters, tw, recheck
    seeds = list(range(1, nchains + 1))
    rs = P.run_chains(cache, pri, seeds, cfg)
    for c in (0, nchains - 1):
        o = port.run_mcmc(ref, cfg.max_parents, iters, seeds[c], pri)
        assert np.array_equal(rs[c].trace_proposed, o["trace_proposed"]), (tw, c)
    print(f"walk tw={tw} iters={iters} chains={nchains} recheck={recheck}: ok "
          f"({cache.last_walk_stats()['variant']})")
    cache.close()


def case_scan():
    data, pri, cfg = instance("cfg2", m=500)
    cache = P.ScoreCache.build(data, cfg, pri)
    ref = cache.table()
    perms = np.stack([np.random.default_rng(i).permutation(data.n) for i in range(4)]).astype(np.int32)
    m, b, t = P.OrderScorer(cache, pri, scan_mode=1).score_many(perms)
    for i in range(4):
        om, ob, ot = port.score_order(ref, cfg.max_parents, perms[i], pri)
        assert np.array_equal(m[i], om) and t[i] == ot
    cfg.iterations, cfg.scan_mode = 30, 1
    rs = P.run_chains(cache, pri, [1, 2, 3], cfg)
    o = port.run_mcmc(ref, cfg.max_parents, 30, 1, pri)
    assert np.array_equal(rs[0].trace_proposed, o["trace_proposed"])
    cache.close()
    print("scan2 + step (scan_mode 1): ok")


def case_wide():
    """K1W (joint spaces beyond the dense counter) vs the plain-C oracle."""
    rng = np.random.default_rng(3)
    for cards, s_, m in (([3] * 9, 7, 200), ([3, 3, 256, 3, 2], 3, 300), ([10] * 6, 4, 250)):
        cards = np.array(cards, np.int32)
        cells = (rng.integers(0, 1 << 20, (m, cards.size)) % cards).astype(np.uint8)
        cfg = P.RunConfig(max_parents=s_, memory_cap_bytes=(1 << 64) - 1)
        cache = P.ScoreCache.build(P.Dataset(cards, cells), cfg)
        t = cache.table()
        cache.close()
        ref = port.cache_build(cells, cards, s_)
        assert np.array_equal(t.view(np.uint64), ref.view(np.uint64)), cards
    print("k1w: ok")


def case_multi():
    """n_gpus = 2 on device 0 twice: split K1, combine, chains over replicas."""
    os.environ["BNMC_DEVICES"] = "0,0"
    data, pri, cfg = instance("cfg2", m=500)
    cfg.n_gpus = 2
    cache = P.ScoreCache.build(data, cfg, pri)
    ref = cache.table()
    ref1 = port.cache_build(data.cells, data.cards, cfg.max_parents)
    assert np.array_equal(ref.view(np.uint64), ref1.view(np.uint64))
    cfg.iterations = 40
    rs = P.run_chains(cache, pri, list(range(1, 11)), cfg)
    o = port.run_mcmc(ref, cfg.max_parents, 40, 10, pri)
    assert np.array_equal(rs[9].trace_proposed, o["trace_proposed"])
    cache.close()
    print("multi (n_gpus=2 on one device): ok")


CASES = {
    "k1": case_k1,
    "walk1": lambda: chains(1, 60, 40),
    "walk8": lambda: chains(8, 60, 6),
    "walk32": lambda: chains(32, 60, 2),
    "spec": lambda: chains(32, 1000, 1),
    "scan": case_scan,
    "recheck": lambda: chains(1, 210, 9, recheck=True),
    "wide": case_wide,
    "multi": case_multi,
}

if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    for k in (CASES if which == "all" else [which]):
        CASES[k]()
