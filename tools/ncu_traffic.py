"""Write profiles/ncu_traffic.json (DRAM bytes per launch of the walk kernel)
from an ncu --set full report of bench.py --steps 1.
  python tools/ncu_traffic.py gpurun_out/ev/walk_bench.ncu-rep"""
import csv
import io
import json
import os
import subprocess
import sys

rep = sys.argv[1]
raw = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                                                 capture_output=True, text=True).stdout)))
h, u, v = raw[0], raw[1], raw[2]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def get(k):
    i = h.index(k)
    return float(v[i].replace(",", "")) * scale.get(u[i], 1)


rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
with open(os.path.join(root, "profiles", "ncu_traffic.json"), "w") as f:
    json.dump({"walk_chain_kernel": {
        "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
        "source": "ncu --set full of bench.py --steps 1 (one walk_chain_kernel<1> launch at the "
                  "bench configuration): profiles/r01_ncu_walk_bench.txt"}}, f, indent=1)
print(rd + wr)
