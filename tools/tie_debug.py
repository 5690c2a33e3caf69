import sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_1210_5128_b200 as P
from oracle import port
rng = np.random.default_rng(21)
cards = rng.integers(2, 3, 10).astype(np.int32)
cells = (rng.integers(0, 1 << 30, (3, 10)) % cards).astype(np.uint8)
cfg = P.RunConfig(max_parents=3, gamma=1.0)
cache = P.ScoreCache.build(P.Dataset(cards, cells), cfg)
t = cache.table()
bad = 0
perms = np.stack([np.random.default_rng(i).permutation(10) for i in range(64)]).astype(np.int32)
masks, best, tot = P.OrderScorer(cache).score_many(perms)
for i in range(64):
    m, b, tt = port.score_order(t, 3, perms[i])
    if not np.array_equal(masks[i], m):
        bad += 1
        d = np.nonzero(masks[i] != m)[0]
        if bad <= 3:
            v = d[0]; perm = list(perms[i]); pos = perm.index(v)
            print("order", perm, "node", v, "pos", pos, "ours", bin(masks[i][v]), "port", bin(m[v]), best[i][v], b[v])
            pset_o, pset_p = int(masks[i][v]), int(m[v])
            print(" ours eff", t[v, port.index_of(10,3,v,pset_o)], "port eff", t[v, port.index_of(10,3,v,pset_p)])
            print(" positions ours", sorted(perm.index(x) for x in range(10) if pset_o>>x&1), "port", sorted(perm.index(x) for x in range(10) if pset_p>>x&1))
print("mismatching orders", bad)
