"""Dev probe: cfg4 precompute time + parity vs golden + chain throughput sweep."""
import hashlib, json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1210_5128_b200 as P

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
g = json.load(open("tests/golden/golden.json"))[name]
gz = dict(np.load(f"tests/golden/golden_{name}.npz"))
data, pri, cfg, truth = P.baseline_instance(name)
print("cells ok", hashlib.sha256(data.cells.tobytes()).hexdigest() == g["cells_sha256"])
for rep in range(2):
    t0 = time.perf_counter()
    cache = P.ScoreCache.build(data, cfg, pri)
    print(f"build wall {time.perf_counter()-t0:.3f}s  device ms (count+score, fold) {cache.build_ms}")
t = cache.table()
print("table bit-exact vs reference:", hashlib.sha256(t.tobytes()).hexdigest() == g["table_sha256"])
masks, best, tot = P.OrderScorer(cache, pri).score_many(gz["orders"])
print("orders exact:", np.array_equal(masks, gz["order_masks"]), np.array_equal(tot, gz["order_totals"]))
cfg.iterations, cfg.seed = g["iterations"], 1
r = P.run_mcmc(data, cfg, pri, prebuilt=cache)
print("chain exact:", np.array_equal(r.trace_proposed, gz["trace_proposed"]),
      np.array_equal(r.tracker_masks, gz["tracker_masks"]), r.accepted == g["accepted"])
for mode in (1,):
    for C in (1, 2, 4, 8, 16, 32, 64):
        cfg.iterations = 2000
        cfg.scan_mode = mode
        rs = P.run_chains(cache, pri, list(range(1, C + 1)), cfg)
        ms = rs[0].device_ms
        import ctypes as Cc
        from paper_1210_5128_b200 import _lib
        a, b, c_, d = Cc.c_uint64(), Cc.c_uint64(), Cc.c_float(), Cc.c_uint64()
        _lib.lib().bnmc_gpu_last_scan_stats(cache.handle, Cc.byref(a), Cc.byref(b), Cc.byref(c_), Cc.byref(d))
        S = cache.entries_per_node()
        print(f"mode {mode} chains {C:3d}: {ms:8.1f} ms  {C*2000/ms*1e3:10.0f} it/s  "
              f"({ms/2000*1e3:.1f} us/step) scan avg {c_.value*1e3:.1f} us  rows/step {a.value/2001:.1f} "
              f"sectors/step {b.value/2001:.0f} (full rows {a.value/2001*S/8:.0f})", flush=True)
