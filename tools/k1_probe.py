"""Dev probe: K1 device time for BASELINE configs (env BNMC_K1_SMEM_KB sweeps the smem budget)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1210_5128_b200 as P
for c in sys.argv[1:] or ["cfg3", "cfg4"]:
    d, pri, cfg, t = P.baseline_instance(c)
    ca = P.ScoreCache.build(d, cfg, pri)
    print(c, os.environ.get("BNMC_K1_SMEM_KB", "56"), "KB: K1 ms", round(ca.build_ms[0], 1), flush=True)
