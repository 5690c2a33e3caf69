"""Dev: short cfg4 chain run for ncu (python tools/profile_run.py CHAINS ITERS [cfg])."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1210_5128_b200 as P
C = int(sys.argv[1]) if len(sys.argv) > 1 else 1
it = int(sys.argv[2]) if len(sys.argv) > 2 else 100
name = sys.argv[3] if len(sys.argv) > 3 else "cfg4"
data, pri, cfg, truth = P.baseline_instance(name)
cache = P.ScoreCache.build(data, cfg, pri)
cfg.iterations = it
rs = P.run_chains(cache, pri, list(range(1, C + 1)), cfg)
print("done", rs[0].device_ms)
