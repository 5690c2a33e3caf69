"""Summarise a tools/walk_ab.sh log: per spec, device and wall it/s per rep and the mean."""
import re
import sys

cur, res = None, {}
chains = sys.argv[2] if len(sys.argv) > 2 else "18944"
for line in open(sys.argv[1]):
    if line.startswith("=="):
        cur = line.split()[1]
    m = re.search(r"C=\s*" + chains + r": dev\s+([\d.]+) ms\s+(\d+) it/s\s+wall\s+([\d.]+) ms \(\s*(\d+) it/s\).*walk/pair (\d+)", line)
    if m:
        res.setdefault(cur, []).append((int(m.group(2)) / 1e6, int(m.group(4)) / 1e6, int(m.group(5))))
for k, v in res.items():
    print(f"{k:28s} " + " ".join(f"{a:.1f}/{b:.1f}" for a, b, _ in v) +
          f"  walk/pair {v[0][2]}  mean dev {sum(a for a, _, _ in v) / len(v):.1f} wall {sum(b for _, b, _ in v) / len(v):.1f}")
