"""Per-source-line instruction counts of one kernel from an ncu source page.

    python tools/sass_lines.py KERNEL_MANGLED SOURCE.csv LIB.so CHAIN_ITERS [FILE]

SOURCE.csv: `ncu -i REP --page source --csv --print-source sass`; LIB.so: the
library the capture ran (line info from `nvdisasm -gi`, -lineinfo builds).
Prints executed warp instructions per chain-iteration by innermost FILE line
(default walk.cuh) and by the kernel-body line it is inlined into."""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile

name, csvf, lib, ci = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
fname = sys.argv[5] if len(sys.argv) > 5 else "walk.cuh"
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin") and "bnmc_gpu" in f][0]
    txt = subprocess.run(["nvdisasm", "-gi", os.path.join(d, cub)], capture_output=True,
                         text=True).stdout.splitlines()
start = [i for i, l in enumerate(txt) if l.startswith("\t.section") and (".text." + name) in l][0]
m, pend = {}, None
for l in txt[start + 1:]:
    if l.startswith("\t.section"):
        break
    if "## File" in l:
        locs = [(f.split("/")[-1], int(n)) for f, n in re.findall(r'"([^"]+)", line (\d+)', l)]
        if pend is None:
            pend = locs  # first annotation of a group: the innermost chain
        continue
    mi = re.search(r"/\*([0-9a-f]{4,})\*/\s+", l)
    if mi:
        if pend is not None:
            cur, pend = pend, None
        m[int(mi.group(1), 16)] = cur if "cur" in dir() else [("?", 0)]
rows = list(csv.reader(open(csvf)))
h, data = rows[1], rows[2:]
base = int(data[0][0], 16)
iex = h.index("Instructions Executed")
inner, outer = collections.Counter(), collections.Counter()
for r in data:
    ch = m.get(int(r[0], 16) - base, [("?", 0)])
    k = next((n for f, n in ch if f == fname), ("other", ch[0][0]))
    inner[k] += int(r[iex])
    outer[ch[-1]] += int(r[iex])
src = open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_1210_5128_b200", "csrc",
                        fname)).read().splitlines()
tot = sum(inner.values())
print(f"total {tot / ci:.1f} warp instructions per chain-iteration")
for k, v in sorted(inner.items(), key=lambda x: -x[1])[:60]:
    t = src[k - 1].strip()[:90] if isinstance(k, int) else ""
    print(f"{str(k):22s} {v / ci:8.1f}  {t}")
