"""Top source lines by warp-stall samples from an ncu report (needs -lineinfo and
--import-source), with each line's dominant stall reasons.
usage: python tools/ncu_hot.py report.ncu-rep kernel_regex [top] [launch_skip]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
res = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                      f"regex:{kern}", "--launch-skip", skip, "--launch-count", "1",
                      "--print-source", "cuda,sass"], capture_output=True, text=True)
rows = list(csv.reader(io.StringIO(res.stdout or res.stderr)))
hdr, lines, fname = None, [], ""
for r in rows:
    if len(r) >= 2 and r[0] in ("File Name", "File Path"):
        fname = r[1].split("/")[-1]
    elif len(r) > 3 and r[0] == "Line No":
        hdr = r
    elif hdr and len(r) == len(hdr) and r[0].isdigit():
        lines.append((f"{fname}:{r[0]}", r))
if not hdr:
    sys.exit("no source table")
idx = {}
for i, n in enumerate(hdr):
    idx.setdefault(n, i)
S = "Warp Stall Sampling (All Samples)"
stall = [n for n in hdr if n.startswith("stall_")] or \
    [n for n in hdr if "Stall" in n and n not in (S, "Warp Stall Sampling (Not-issued Samples)")]
tot = sum(int(r[idx[S]] or 0) for _, r in lines if r[idx[S]] not in ("-", ""))
print(f"total samples {tot}")
val = lambda r, c: int(r[idx[c]]) if r[idx[c]] not in ("-", "") else 0  # noqa: E731
lines.sort(key=lambda x: -val(x[1], S))
for loc, r in lines[:top]:
    reasons = sorted(((val(r, c), c) for c in stall), reverse=True)[:3]
    rs = " ".join(f"{c.replace('stall_', '')}={v}" for v, c in reasons if v)
    print(f"{100 * val(r, S) / max(tot, 1):5.1f}% {loc:>18s} {r[1].strip()[:70]:70s} {rs}")
