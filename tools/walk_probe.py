"""Dev probe: sorted-walk chain throughput at cfg4 vs chains per launch."""
import ctypes as Cc
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1210_5128_b200 as P
from paper_1210_5128_b200 import _lib

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 500
chains = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [1, 64, 148, 296, 592, 1184, 2368]
data, pri, cfg, truth = P.baseline_instance(name)
t0 = time.perf_counter()
cache = P.ScoreCache.build(data, cfg, pri)
print(f"build {time.perf_counter() - t0:.3f}s", flush=True)
cfg.iterations = iters
if os.environ.get("BNMC_DEEP") or os.environ.get("BNMC_WCAP") or os.environ.get("BNMC_WBUD"):
    # walk cap / budget / entries per lane per deep round (-1: library default)
    _lib.check(_lib.lib().bnmc_gpu_table_set_walk_cap(
        cache.handle, int(os.environ.get("BNMC_WCAP", -1)), int(os.environ.get("BNMC_WBUD", -1)),
        int(os.environ.get("BNMC_DEEP", -1))))
if os.environ.get("BNMC_ENUM_MAX"):
    _lib.check(_lib.lib().bnmc_gpu_table_set_walk_params(cache.handle, int(os.environ["BNMC_ENUM_MAX"]), -1))
tws = [int(x) for x in os.environ.get("TW", "0").split(",")]
for tw in tws:
    mode = 2
    cfg.scan_mode = mode
    cfg.team_warps = tw
    for C in chains:
        for rep in range(2):
            t0 = time.perf_counter()
            rs = P.run_chains(cache, pri, list(range(1, C + 1)), cfg)
            wall = time.perf_counter() - t0
        ms = rs[0].device_ms
        pairs, walked, enum, sort_ms = Cc.c_uint64(), Cc.c_uint64(), Cc.c_uint64(), Cc.c_float()
        _lib.check(_lib.lib().bnmc_gpu_last_walk_stats(cache.handle, Cc.byref(pairs), Cc.byref(walked),
                                                       Cc.byref(enum), Cc.byref(sort_ms)))
        best = max(r.best_score() for r in rs)
        print(f"tw {tw} C={C:5d}: dev {ms:9.2f} ms  {C * iters / ms * 1e3:12.0f} it/s  "
              f"wall {wall * 1e3:8.1f} ms ({C * iters / wall:10.0f} it/s)  pairs/it {pairs.value / (C * (iters + 1)):.1f} "
              f"walk/pair {walked.value / max(1, pairs.value):.0f} enum/pair {enum.value / max(1, pairs.value):.0f} "
              f"sort {sort_ms.value:.1f} ms best {best:.3f}", flush=True)
cfg.scan_mode = 1
cfg.iterations = iters
ms = P.run_chains(cache, pri, list(range(1, 65)), cfg)[0].device_ms
print(f"mode 1 C=64: dev {ms:.2f} ms {64 * iters / ms * 1e3:.0f} it/s", flush=True)
