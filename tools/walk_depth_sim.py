"""Dev: where do sorted-row walks spend their entries? (CPU simulation on the
GPU-built cfg4 table, run on the GPU box.)

For chain states after `iters` iterations (final orders of `chains` chains)
and for every row v with p predecessors, the depth of the first admissible
entry of v's eff-sorted row (what a full walk reads) against S(p, s) (what a
PST enumeration reads). Prints a table by p.
  python tools/walk_depth_sim.py [chains] [iters]
"""
import itertools
import os
import sys
from math import comb

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1210_5128_b200 as P  # noqa: E402

chains = int(sys.argv[1]) if len(sys.argv) > 1 else 16
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 500
data, pri, cfg, truth = P.baseline_instance("cfg4")
n, s = data.n, cfg.max_parents
cache = P.ScoreCache.build(data, cfg, pri)
ls = cache.table()
c = n - 1
masks = []
for k in range(s, -1, -1):
    for comb_ in itertools.combinations(range(c), k):
        m = 0
        for j in comb_:
            m |= 1 << j
        masks.append(m)
cm = np.array(masks, dtype=np.uint64)
S = cm.size
bits = ((cm[None, :] >> np.arange(c, dtype=np.uint64)[:, None]) & np.uint64(1)).astype(bool)  # [c, S]
W = np.asarray(pri, np.float64) if pri is not None else None
w = None
if W is not None:
    d = W - 0.5
    w = 100.0 * d * d * d
    np.fill_diagonal(w, 0.0)
eff = np.empty((n, S))
order = np.empty((n, S), dtype=np.int64)
for v in range(n):
    e = ls[v].copy()
    if w is not None:
        for j in range(c):
            node = j if j < v else j + 1
            e[bits[j]] += w[v, node]  # PpfTable: w[child*n + parent]
    eff[v] = e
    order[v] = np.argsort(-e, kind="stable")

cfg.iterations = iters
b = P.run_chains_batch(cache, pri, list(range(1, chains + 1)), cfg)
rng = np.random.default_rng(0)
orders = [("final", o) for o in b.final_order] + [("random", rng.permutation(n)) for _ in range(4)]
rows = {}
for kind, perm in orders:
    pos = np.empty(n, np.int64)
    pos[np.asarray(perm)] = np.arange(n)
    for v in range(n):
        p = int(pos[v])
        preds = [int(u) for u in perm[:p]]
        cp = 0
        for u in preds:
            cp |= 1 << (u if u < v else u - 1)
        adm = (cm[order[v]] & ~np.uint64(cp)) == 0
        depth = int(np.argmax(adm)) + 1
        r = rows.setdefault((kind, p), [])
        r.append(depth)
print(f"{'kind':6s} {'p':>3s} {'rows':>5s} {'S(p,s)':>8s} {'depth med':>10s} {'mean':>10s} {'max':>8s}")
for (kind, p) in sorted(rows):
    d = np.array(rows[(kind, p)])
    sp = sum(comb(p, j) for j in range(min(p, s) + 1))
    print(f"{kind:6s} {p:3d} {d.size:5d} {sp:8d} {np.median(d):10.0f} {d.mean():10.1f} {d.max():8d}")
