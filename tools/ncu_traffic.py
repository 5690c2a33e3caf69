"""Write profiles/ncu_traffic.json — the ncu --set full figures of the walk
kernel at the bench configuration that bench.py reports beside its own timing:
DRAM bytes, warp instructions, IPC, issue-slot use, top stalls; per launch and per
chain-iteration of the captured launch (the bench scales the latter to its step:
the library splits large calls into chain blocks, so a launch is one block).
  python tools/ncu_traffic.py REPORT.ncu-rep SUMMARY_NAME CHAINS ITERATIONS
(SUMMARY_NAME: the profiles/ text summary written by tools/ncu_summary.py;
CHAINS x ITERATIONS: the captured launch's chain-iterations)."""
import csv
import io
import json
import os
import subprocess
import sys

rep = sys.argv[1]
summary = sys.argv[2] if len(sys.argv) > 2 else "?"
chain_iters = int(sys.argv[3]) * int(sys.argv[4]) if len(sys.argv) > 4 else None
raw = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                                                 capture_output=True, text=True).stdout)))
h, u, v = raw[0], raw[1], raw[2]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "inst": 1, "%": 1,
         "msecond": 1e-3, "usecond": 1e-6, "nsecond": 1e-9, "second": 1,
         "ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1}


def get(k):
    i = h.index(k)
    return float(v[i].replace(",", "")) * scale.get(u[i], 1)


def opt(k):
    try:
        return get(k)
    except (ValueError, IndexError):
        return None


rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
st = [(float(x.replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", ""))
      for k, x in zip(h, v)
      if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")
      and x.replace(",", "").replace(".", "").isdigit()]
tot = sum(x for x, _ in st) or 1.0
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = {"walk_chain_kernel": {
    "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
    "duration_s": opt("gpu__time_duration.sum"),
    "warp_instructions": opt("smsp__inst_executed.sum"),
    "ipc": opt("sm__inst_executed.avg.per_cycle_active"),
    "issue_slots_busy": (opt("sm__instruction_throughput.avg.pct_of_peak_sustained_active") or 0)
    / 100.0,
    "top_stalls": {k: round(x / tot, 3) for x, k in sorted(st, reverse=True)[:5]},
    "chain_iterations_per_launch": chain_iters,
    "dram_bytes_per_chain_iteration": (rd + wr) / chain_iters if chain_iters else None,
    "warp_instructions_per_chain_iteration":
        (opt("smsp__inst_executed.sum") or 0) / chain_iters if chain_iters else None,
    "source": f"ncu --set full --clock-control none of one walk_chain_kernel launch (one "
              f"chain block of the bench step) of bench.py --steps 1: profiles/{summary}"}}
with open(os.path.join(root, "profiles", "ncu_traffic.json"), "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out, indent=1))
