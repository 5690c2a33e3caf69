"""Summarise an ncu --set full report: launch config, duration, throughputs,
DRAM bytes, occupancy, top stall reasons.  python tools/ncu_summary.py X.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "L1/TEX Cache Throughput", "L2 Cache Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Executed Ipc Active", "Issue Slots Busy", "Achieved Occupancy", "Theoretical Occupancy",
        "Registers Per Thread", "Dynamic Shared Memory Per Block", "Static Shared Memory Per Block",
        "Grid Size", "Block Size", "Waves Per SM"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "lts__t_bytes.sum", "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main(rep):
    det = list(csv.reader(io.StringIO(ncu(rep, "--page", "details", "--csv"))))
    hdr = det[0]
    kn = hdr.index("Kernel Name")
    mn, mu, mv = hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    print(f"report: {rep}")
    print(f"kernel: {det[1][kn]}")
    seen = set()
    for r in det[1:]:
        if r[mn] in KEYS and r[mn] not in seen:
            seen.add(r[mn])
            print(f"  {r[mn]:36s} {r[mv]:>14s} {r[mu]}")
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    h, units, vals = raw[0], raw[1], raw[2]
    print("raw:")
    for k in RAW:
        if k in h:
            i = h.index(k)
            print(f"  {k:52s} {vals[i]:>16s} {units[i]}")
    st = [(float(v.replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", ""))
          for k, v in zip(h, vals)
          if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")
          and v.replace(",", "").replace(".", "").isdigit()]
    tot = sum(x for x, _ in st) or 1.0
    print("stall samples (top 8):")
    for x, k in sorted(st, reverse=True)[:8]:
        print(f"  {k:28s} {x / tot * 100:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
