"""Top source lines by warp-stall samples from an ncu report (needs -lineinfo).
usage: python tools/ncu_hot.py report.ncu-rep kernel_regex [top]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                      f"regex:{kern}", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
lines = []
for r in rows:
    if len(r) > 3 and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0].isdigit():
        lines.append(r)
if not hdr:
    sys.exit("no source table")
idx = {n: i for i, n in enumerate(hdr)}
stall_cols = [n for n in hdr if n.startswith("stall_") and "(Not Issued)" not in n]
tot = sum(int(r[idx["Warp Stall Sampling (All Samples)"]] or 0) for r in lines)
print(f"total samples {tot}")
lines.sort(key=lambda r: -int(r[idx["Warp Stall Sampling (All Samples)"]] or 0))
for r in lines[:top]:
    smp = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    stalls = sorted(((int(r[idx[c]] or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
    st = " ".join(f"{n}:{v}" for v, n in stalls if v)
    print(f"{100*smp/max(tot,1):5.1f}% L{r[0]:>4s} {r[1].strip()[:70]:70s} {st}")
