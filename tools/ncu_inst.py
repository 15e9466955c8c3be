"""Top source lines by executed instructions (warp-level) from an ncu report.
usage: python tools/ncu_inst.py report.ncu-rep kernel_regex [top] [launch_skip]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
skip = sys.argv[4] if len(sys.argv) > 4 else "0"  # --launch-skip among matching kernels
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                      f"regex:{kern}", "--launch-skip", skip, "--print-source", "cuda,sass"],
                     capture_output=True,
                     text=True)
out = out.stdout or out.stderr
rows = list(csv.reader(io.StringIO(out)))
hdr, lines, fname = None, [], ""
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 3 and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0].isdigit():
        lines.append([f"{fname}:{r[0]}"] + r[1:])
idx = {n: i for i, n in enumerate(hdr)}
col = "Instructions Executed"
tot = sum(int(r[idx[col]] or 0) for r in lines)
print(f"total warp instructions {tot}")
lines.sort(key=lambda r: -int(r[idx[col]] or 0))
for r in lines[:top]:
    v = int(r[idx[col]] or 0)
    print(f"{100*v/max(tot,1):5.1f}% {r[0]:>22s} {r[1].strip()[:90]}")
