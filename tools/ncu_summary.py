"""Key per-launch metrics from an ncu report.  usage: python tools/ncu_summary.py rep"""
import csv
import io
import subprocess
import sys

want = ["Duration", "Registers Per Thread", "Block Size", "Grid Size", "Achieved Occupancy",
        "Executed Ipc Active", "L2 Hit Rate", "DRAM Throughput", "Active Warps Per Scheduler",
        "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction",
        "Dynamic Shared Memory Per Block"]
res = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"],
                     capture_output=True, text=True)
rows = list(csv.reader(io.StringIO(res.stdout)))
hdr = rows[0]
ki, mi, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
cur = {}
for r in rows[1:]:
    if r[mi] in want:
        cur.setdefault((r[ii], r[ki].split("(")[0][:28]), {})[r[mi]] = r[vi]
for (i, k), m in cur.items():
    print(i, k, " ".join(f"{n.split()[0][:6]}={m.get(n, '-')}" for n in want))
