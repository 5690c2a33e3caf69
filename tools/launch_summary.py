"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel:
count, total, average and share of the listed device time.
  python tools/launch_summary.py gpurun_out/launches.csv [> profiles/...txt]"""
import collections
import csv
import sys

lines = [l for l in open(sys.argv[1]) if not l.startswith("==")]
rows = list(csv.DictReader(lines))
agg = collections.defaultdict(list)
for r in rows:
    if r.get("Metric Name") == "gpu__time_duration.sum":
        name = r["Kernel Name"].split("(")[0].replace("<unnamed>::", "").replace("bnmc_dev::", "")
        agg[name].append(float(r["Metric Value"]))
tot = sum(sum(v) for v in agg.values())
print(f"{'kernel':56s} {'launches':>8s} {'total ms':>10s} {'avg us':>10s} {'share':>7s}")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k[:56]:56s} {len(v):8d} {sum(v) / 1e6:10.3f} {sum(v) / len(v) / 1e3:10.1f} "
          f"{sum(v) / tot * 100:6.1f}%")
print(f"{'TOTAL':56s} {sum(len(v) for v in agg.values()):8d} {tot / 1e6:10.3f}")
