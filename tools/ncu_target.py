"""Short, deterministic workload for ncu: DPA3/DPA2 MD steps on a paper box.
usage: python tools/ncu_target.py [dpa3|dpa2|se_a|repformer|repflow] [1YRF|2PTC] [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_02234_b200 as P
from paper_2602_02234_b200.md import DeviceMD

name = sys.argv[1] if len(sys.argv) > 1 else "dpa3"
system = sys.argv[2] if len(sys.argv) > 2 else "1YRF"
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
fam, depth = {"dpa2": (0, 1), "dpa3": (1, 3), "se_a": (2, 1), "repformer": (3, 3),
              "repflow": (4, 3)}[name]
if fam >= 2:
    m = P.make_dp_model(P.ModelFamily(fam), depth, 0.6, 0.3, 2, 1)
else:
    m = P.make_model(P.ModelFamily(fam), depth, 0.6, 2, 8, 32, 1)
s = P.generate_synthetic_system(P.PAPER_SYSTEMS[system])
ctx = P.Context(m, max_atoms=s.n_atoms)
md = DeviceMD(ctx, s.positions, s.velocities, s.masses, s.types, s.box, steps_per_graph=1)
md.run(steps)
print("ok", md.state()[3])
