"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.OrderedDict()
for d in data:
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    k = d["Kernel Name"].split("(")[0].replace("void ", "")
    agg.setdefault(k, []).append(float(d["Metric Value"]) * (1e-3 if d["Metric Unit"] == "ns" else 1.0))
tot = sum(sum(v) for v in agg.values())
print(f"{'kernel':34s} {'n':>4s} {'mean_us':>9s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:34s} {len(v):4d} {sum(v)/len(v):9.2f} {100*sum(v)/tot:5.1f}%")
print(f"total {tot:.1f} us over {sum(len(v) for v in agg.values())} launches")
