"""Dev: would block summaries shorten the sorted-row walks? (CPU simulation on
the GPU-built cfg4 table; run on the GPU box.)

For rows rescanned by swap proposals from chain states after `iters`
iterations: the depth of the first admissible entry of the eff-sorted row (a
plain walk reads every entry up to it) against a walk over block summaries —
the AND of the candidate masks of each block of B sorted entries. A block can
hold an admissible entry only if its AND is a subset of the predecessors, so
the walk reads summaries (32 per warp load) and opens only candidate blocks.
  python tools/block_skip_sim.py [chains] [iters] [proposals per chain]
"""
import itertools
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1210_5128_b200 as P  # noqa: E402

chains = int(sys.argv[1]) if len(sys.argv) > 1 else 32
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 500
props = int(sys.argv[3]) if len(sys.argv) > 3 else 64
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
bits = ((cm[None, :] >> np.arange(c, dtype=np.uint64)[:, None]) & np.uint64(1)).astype(bool)
d = np.asarray(pri, np.float64) - 0.5
w = 100.0 * d * d * d
np.fill_diagonal(w, 0.0)
srt = []
for v in range(n):
    e = ls[v].copy()
    for j in range(c):
        e[bits[j]] += w[v, j if j < v else j + 1]
    srt.append(cm[np.argsort(-e, kind="stable")])


def block_and(x, B):
    pad = (-x.size) % B
    y = np.concatenate([x, np.full(pad, ~np.uint64(0), np.uint64)]).reshape(-1, B)
    return np.bitwise_and.reduce(y, axis=1)


BS = (16, 32, 64)
band = {B: [block_and(r, B) for r in srt] for B in BS}
cfg.iterations = iters
b = P.run_chains_batch(cache, pri, list(range(1, chains + 1)), cfg)
rng = np.random.default_rng(0)
depths = []
cost = {B: [] for B in BS}  # (summary windows read, candidate blocks opened)
for perm in b.final_order:
    for _ in range(props):
        a_, b_ = sorted(rng.choice(n, 2, replace=False))
        pp = np.array(perm).copy()
        pp[a_], pp[b_] = pp[b_], pp[a_]
        for p in range(a_, b_ + 1):
            v = int(pp[p])
            cp = np.uint64(0)
            for u in pp[:p]:
                u = int(u)
                cp |= np.uint64(1 << (u if u < v else u - 1))
            ncp = ~cp
            adm = (srt[v] & ncp) == 0
            dep = int(np.argmax(adm)) + 1
            depths.append(dep)
            for B in BS:
                cand = (band[B][v] & ncp) == 0
                hb = (dep - 1) // B
                cost[B].append((hb // 32 + 1, int(cand[:hb + 1].sum())))
depths = np.array(depths)
print(f"rows {depths.size}: depth mean {depths.mean():.1f} median {np.median(depths):.0f} "
      f"p90 {np.percentile(depths, 90):.0f} p99 {np.percentile(depths, 99):.0f} max {depths.max()}")
# plain walk: rounds of 32, 64, 128, then 128 entries
def plain_rounds(dp):
    r, seen = 0, 0
    for sz in (32, 64, 128):
        r += 1
        seen += sz
        if dp <= seen:
            return r, seen
    extra = (dp - seen + 127) // 128
    return r + extra, seen + 128 * extra
pr = np.array([plain_rounds(x) for x in depths])
print(f"plain walk: rounds/row {pr[:, 0].mean():.2f}, entries loaded/row {pr[:, 1].mean():.1f}")
for B in BS:
    cc = np.array(cost[B])
    deep = depths > 224
    print(f"B={B:3d}: summary windows/row {cc[:, 0].mean():.2f}, candidate blocks/row "
          f"{cc[:, 1].mean():.2f} (rows deeper than 224: windows {cc[deep, 0].mean():.2f}, "
          f"blocks {cc[deep, 1].mean():.2f}, plain rounds {pr[deep, 0].mean():.2f}, "
          f"share {deep.mean():.3f})")

# Exclusion lists: row v's sorted entries WITHOUT its strongest parent t_v
# (the candidate most frequent among the top 256 entries). When t_v is not a
# predecessor, no admissible entry contains it, so the walk can use that list.
tops = []
for v in range(n):
    top = srt[v][:256]
    freq = [int(((top >> np.uint64(j)) & np.uint64(1)).sum()) for j in range(c)]
    tops.append(int(np.argmax(freq)))
excl_pos = []
for v in range(n):
    has = ((srt[v] >> np.uint64(tops[v])) & np.uint64(1)).astype(bool)
    excl_pos.append(np.cumsum(~has))  # entries without t_v up to and incl. index i
rng = np.random.default_rng(0)
newd, olddeep, hit = [], [], 0
for perm in b.final_order:
    for _ in range(props):
        a_, b_ = sorted(rng.choice(n, 2, replace=False))
        pp = np.array(perm).copy()
        pp[a_], pp[b_] = pp[b_], pp[a_]
        for p in range(a_, b_ + 1):
            v = int(pp[p])
            cp = 0
            for u in pp[:p]:
                u = int(u)
                cp |= 1 << (u if u < v else u - 1)
            adm = (srt[v] & ~np.uint64(cp)) == 0
            dep = int(np.argmax(adm)) + 1
            if (cp >> tops[v]) & 1:
                newd.append(dep)
            else:
                hit += 1
                newd.append(int(excl_pos[v][dep - 1]))
            olddeep.append(dep)
newd, olddeep = np.array(newd), np.array(olddeep)
print(f"exclusion of the top parent applies to {hit / newd.size:.3f} of rows; depth mean "
      f"{olddeep.mean():.1f} -> {newd.mean():.1f}, p90 {np.percentile(olddeep, 90):.0f} -> "
      f"{np.percentile(newd, 90):.0f}, p99 {np.percentile(olddeep, 99):.0f} -> "
      f"{np.percentile(newd, 99):.0f}; rows deeper than 224: {(olddeep > 224).mean():.3f} -> "
      f"{(newd > 224).mean():.3f}")
pr2 = np.array([plain_rounds(x) for x in newd])
print(f"plain walk on the chosen list: rounds/row {pr2[:, 0].mean():.2f} (was {pr[:, 0].mean():.2f}), "
      f"entries/row {pr2[:, 1].mean():.1f} (was {pr[:, 1].mean():.1f})")

# Two levels: lists without t1, without t2 (second most frequent), without both.
tops2 = []
for v in range(n):
    top = srt[v][:256]
    freq = np.array([int(((top >> np.uint64(j)) & np.uint64(1)).sum()) for j in range(c)])
    o = np.argsort(-freq, kind="stable")
    tops2.append((int(o[0]), int(o[1])))
rng = np.random.default_rng(0)
d1, d2 = [], []
for perm in b.final_order:
    for _ in range(props):
        a_, b_ = sorted(rng.choice(n, 2, replace=False))
        pp = np.array(perm).copy()
        pp[a_], pp[b_] = pp[b_], pp[a_]
        for p in range(a_, b_ + 1):
            v = int(pp[p])
            cp = 0
            for u in pp[:p]:
                u = int(u)
                cp |= 1 << (u if u < v else u - 1)
            adm = (srt[v] & ~np.uint64(cp)) == 0
            dep = int(np.argmax(adm))
            t1, t2 = tops2[v]
            m1, m2 = not (cp >> t1) & 1, not (cp >> t2) & 1
            has1 = ((srt[v][:dep + 1] >> np.uint64(t1)) & np.uint64(1)).astype(bool)
            has2 = ((srt[v][:dep + 1] >> np.uint64(t2)) & np.uint64(1)).astype(bool)
            # single level with two lists (t1 preferred)
            if m1:
                a = int((~has1).sum())
            elif m2:
                a = int((~has2).sum())
            else:
                a = dep + 1
            # plus the double list
            if m1 and m2:
                bb = int((~(has1 | has2)).sum())
            else:
                bb = a
            d1.append(a)
            d2.append(bb)
d1, d2 = np.array(d1), np.array(d2)
for name, dd in (("t1 | t2 lists", d1), ("+ t1&t2 list", d2)):
    pr3 = np.array([plain_rounds(x) for x in dd])
    print(f"{name}: depth mean {dd.mean():.1f}, rounds/row {pr3[:, 0].mean():.2f}, "
          f"entries/row {pr3[:, 1].mean():.1f}")

# Nested exclusion lists: without {t1..tj}, j = 1..J; the walk takes the largest
# j whose parents t1..tj are all missing from the predecessors.
topsk = []
for v in range(n):
    top = srt[v][:256]
    freq = np.array([int(((top >> np.uint64(j)) & np.uint64(1)).sum()) for j in range(c)])
    topsk.append([int(x) for x in np.argsort(-freq, kind="stable")[:4]])
for J in (1, 2, 3, 4):
    rng = np.random.default_rng(0)
    dd = []
    for perm in b.final_order:
        for _ in range(props):
            a_, b_ = sorted(rng.choice(n, 2, replace=False))
            pp = np.array(perm).copy()
            pp[a_], pp[b_] = pp[b_], pp[a_]
            for p in range(a_, b_ + 1):
                v = int(pp[p])
                cp = 0
                for u in pp[:p]:
                    u = int(u)
                    cp |= 1 << (u if u < v else u - 1)
                adm = (srt[v] & ~np.uint64(cp)) == 0
                dep = int(np.argmax(adm))
                j = 0
                while j < J and not (cp >> topsk[v][j]) & 1:
                    j += 1
                ex = np.uint64(sum(1 << t for t in topsk[v][:j]))
                dd.append(int(((srt[v][:dep + 1] & ex) == 0).sum()))
    dd = np.array(dd)
    pr3 = np.array([plain_rounds(x) for x in dd])
    print(f"nested J={J}: depth mean {dd.mean():.1f}, rounds/row {pr3[:, 0].mean():.2f}, "
          f"entries/row {pr3[:, 1].mean():.1f}")
