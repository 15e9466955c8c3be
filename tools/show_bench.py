"""Print the key numbers of a bench.py JSON line (and its "models" sub-lines)."""
import json
import sys


def show(d):
    r = d["roofline"]
    print(f"{d['config']['model']:5s} {d['config']['system']} value {d['value']:9.0f} steps/s "
          f"({d['ms_per_step']*1e3:6.1f} us)  e2e {d['e2e']['value']:8.0f}  warm "
          f"{d.get('warm_l2_graph100', {}).get('steps_per_s', 0):8.0f}  roof {r['kernel']} "
          f"{r['frac']:.3f} traffic {r['traffic']}")
    print("   kern ", {k: round(v, 1) for k, v in d["kernels_us"].items()})
    print("   event", {k: round(v, 1) for k, v in d.get("kernels_event_us", {}).items()})


for path in sys.argv[1:]:
    d = json.loads(open(path).read().strip().splitlines()[-1])
    show(d)
    for m in d.get("models", {}).values():
        show(m)
