"""Generate the golden parity fixtures by running the UNMODIFIED reference.

Run in the build container (needs oracle/_ref/libbnmc_ref.so, i.e. /root/reference
at build time):  python tests/golden/make_golden.py [--cfg4]

Every array here is produced by the reference's own public API through
oracle/ref_shim.cpp (ScoreCache::build, OrderScorer::score, run_mcmc, the
evalgen generator) on the SURVEY §8d instances. The GPU parity tests and the
oracle-port tests compare against these files; nothing here is hand-written.

cfg4 (n=60, k=4, m=10000) takes ~7 min of reference precompute on 8 cores and
is only regenerated with --cfg4.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

# SURVEY §8d / BASELINE.json configs: (name, n, k, m, cards, priors, mcmc iterations)
CONFIGS = {
    "cfg1": (11, 3, 1000, "3", False, 10000),
    "cfg2": (20, 4, 2000, "3", False, 2000),
    "cfg3": (37, 4, 5000, "2+i%3", True, 200),
    "cfg4": (60, 4, 10000, "3", True, 200),
}


def cards_for(n, mode):
    return np.array([3] * n if mode == "3" else [2 + (i % 3) for i in range(n)], np.int32)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def fixed_orders(n, count=20, seed=7):
    """bench-style fixed random orders: one Rng(seed).split(7) shuffling fresh
    identities (proj/tools/bnmc.cpp:262-270)."""
    # One stream shuffles successive iotas: take its raw u64 draws from the
    # reference Rng and apply Rng::next_below's rejection + Fisher-Yates here.
    out = []
    u64 = ref.rng_stream(seed, 7, 0, count * n * 4)
    pos = 0

    def next_below(bound):
        nonlocal pos
        thr = ((1 << 64) - bound) % bound
        while True:
            x = int(u64[pos])
            pos += 1
            if x >= thr:
                return x % bound

    for _ in range(count):
        perm = list(range(n))
        for i in range(n, 1, -1):
            j = next_below(i)
            perm[i - 1], perm[j] = perm[j], perm[i - 1]
        out.append(perm)
    return np.array(out, np.int32)


def make(name, with_table_file):
    n, k, m, cmode, pri, iters = CONFIGS[name]
    cards = cards_for(n, cmode)
    t0 = time.time()
    cells, truth = ref.generate(n, k, m, cards, seed=7)
    priors = ref.synth_priors(n, truth, seed=7) if pri else None
    cache = ref.Cache.build(cells, cards, k)
    t_build = time.time() - t0
    table = cache.table()
    if os.environ.get("GOLDEN_SAVE_BNSC"):  # local scratch copy, never committed
        cache.save(os.path.join(os.environ["GOLDEN_SAVE_BNSC"], f"{name}.bnsc"))
    orders = fixed_orders(n)
    scorer = ref.Scorer(cache, priors)
    om, ot = [], []
    for perm in orders:
        mk, tt = scorer.score(perm)
        om.append(mk)
        ot.append(tt)
    t1 = time.time()
    r = ref.run_mcmc(cells, cards, k, iters, 1, priors=priors, prebuilt=cache)
    rng = np.random.default_rng(1234)
    samp_node = rng.integers(0, n, 2000)
    samp_g = rng.integers(0, cache.per_node, 2000)
    arrays = dict(
        cards=cards, truth=truth, orders=orders, order_masks=np.array(om, np.uint64),
        order_totals=np.array(ot), samp_node=samp_node, samp_g=samp_g,
        samp_val=table[samp_node, samp_g], trace_proposed=r.trace_proposed,
        trace_accepted=r.trace_accepted, trace_best=r.trace_best, final_order=r.final_order,
        tracker_masks=r.tracker_masks, tracker_totals=r.tracker_totals,
    )
    if priors is not None:
        arrays["priors"] = priors
    if with_table_file:
        arrays["cells"] = cells
        arrays["table"] = table
    np.savez_compressed(os.path.join(OUT, f"golden_{name}.npz"), **arrays)
    meta = dict(n=n, k=k, m=m, cards=cmode, priors=pri, iterations=iters, seed=1,
                cells_sha256=sha(cells), table_sha256=sha(table), per_node=cache.per_node,
                final_score=r.final_score, accepted=r.accepted,
                ref_build_seconds=t_build, ref_mcmc_sampling_seconds=r.sampling_seconds,
                ref_threads=ref.max_threads(), generated=time.strftime("%Y-%m-%dT%H:%M:%S"))
    print(name, json.dumps(meta), f"(mcmc {time.time() - t1:.1f}s)", flush=True)
    return meta


def tie_fixture():
    """m=0, gamma=1 makes every entry 0.0 → the reference picks
    the first min(p,s) predecessors of the order."""
    n, s = 7, 3
    cards = np.full(n, 3, np.int32)
    cells = np.zeros((0, n), np.uint8)
    cache = ref.Cache.build(cells, cards, s, gamma=1.0)
    perm = np.array([4, 1, 6, 0, 3, 5, 2], np.int32)
    mk, tt = ref.Scorer(cache, None, workers=3, tasks_per_node=3).score(perm)
    mk2, tt2 = cache.score_order(perm)
    assert np.array_equal(mk, mk2) and tt == tt2
    return dict(n=n, s=s, perm=perm.tolist(), masks=[int(x) for x in mk], total=tt)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg4", action="store_true")
    ap.add_argument("--only", default=None)
    a = ap.parse_args()
    path = os.path.join(OUT, "golden.json")
    meta = json.load(open(path)) if os.path.exists(path) else {}
    names = [a.only] if a.only else ["cfg1", "cfg2", "cfg3"] + (["cfg4"] if a.cfg4 else [])
    for name in names:
        meta[name] = make(name, with_table_file=name in ("cfg1", "cfg2"))
    meta["tie_fixture"] = tie_fixture()
    meta["orders_stream"] = "Rng(7).split(7) Fisher-Yates over fresh iotas (bnmc.cpp:262-270)"
    json.dump(meta, open(path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
