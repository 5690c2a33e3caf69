"""Dev: K1 on a synthetic instance: python tools/k1_synth.py n s m [cards]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1210_5128_b200 as P
n, s, m = (int(x) for x in sys.argv[1:4])
card = int(sys.argv[4]) if len(sys.argv) > 4 else 3
cells, truth = P.synth_instance(n, s, m, [card] * n)
data = P.Dataset(np.full(n, card, np.int32), cells)
cfg = P.RunConfig(max_parents=s)
ca = P.ScoreCache.build(data, cfg)
print(f"n={n} s={s} m={m}: K1 ms {ca.build_ms[0]:.1f}", flush=True)
