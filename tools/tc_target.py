"""ncu target for the tcgen05 embedding chain A/B: DPA3 device MD steps on a (replicated)
paper box.  usage: HMDP_TC_EMBED=0|1 python tools/tc_target.py [system] [rx,ry,rz] [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_02234_b200 as P
from paper_2602_02234_b200.md import DeviceMD

system = sys.argv[1] if len(sys.argv) > 1 else "2PTC"
reps = tuple(int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "1,1,1").split(","))
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
s = P.generate_synthetic_system(P.PAPER_SYSTEMS[system])
if reps != (1, 1, 1):
    s = P.replicate(s, reps)
m = P.make_model(P.ModelFamily.message_passing, 3, 0.6, 2, 8, 32, 1)
ctx = P.Context(m, max_atoms=s.n_atoms)
md = DeviceMD(ctx, s.positions, s.velocities, s.masses, s.types, s.box, steps_per_graph=1)
md.run(steps)
print("ok", md.state()[3])
