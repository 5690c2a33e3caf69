"""Dev: time the K2 order-scan kernel alone (cold L2 per launch):
python tools/bench_scan_one.py C lo hi reps [cfg]. Prints launch time, key bytes
streamed per launch and the achieved GB/s."""
import os, sys, ctypes as Cc
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1210_5128_b200 as P
from paper_1210_5128_b200 import _lib
C, lo, hi, reps = (int(x) for x in sys.argv[1:5])
data, pri, cfg, truth = P.baseline_instance(sys.argv[5] if len(sys.argv) > 5 else "cfg4")
cache = P.ScoreCache.build(data, cfg, pri)
rng = np.random.default_rng(0)
perms = np.stack([rng.permutation(data.n) for _ in range(C)]).astype(np.int32)
ms, kb = Cc.c_float(), Cc.c_uint64()
_lib.check(_lib.lib().bnmc_gpu_bench_scan(cache.handle, perms.ravel(), C, lo, hi, reps, 1,
                                          Cc.byref(ms), Cc.byref(kb)))
us = ms.value * 1e3
print(f"C={C} rows {lo}..{hi}: scan {us:.1f} us, {kb.value / 1e6:.1f} MB keys, "
      f"{kb.value / us / 1e3:.0f} GB/s", flush=True)
