"""Dev: scan-kernel phase breakdown via BNMC_DEBUG_SCAN_EXIT on bnmc_gpu_bench_scan."""
import os, sys, ctypes as Cc
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1210_5128_b200 as P
from paper_1210_5128_b200 import _lib
data, pri, cfg, truth = P.baseline_instance("cfg4")
cache = P.ScoreCache.build(data, cfg, pri)
rng = np.random.default_rng(0)
for C, lo, hi in ((1, 20, 40), (8, 20, 40), (1, 0, 59), (64, 20, 40)):
    perms = np.stack([rng.permutation(60) for _ in range(C)]).astype(np.int32)
    ms = Cc.c_float()
    _lib.check(_lib.lib().bnmc_gpu_bench_scan(cache.handle, perms.ravel(), C, lo, hi, 50, Cc.byref(ms)))
    print(os.environ.get("BNMC_DEBUG_SCAN_EXIT", "0"), f"C={C} rows {lo}..{hi}: scan {ms.value*1e3:.1f} us", flush=True)
