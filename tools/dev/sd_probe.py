"""Single-domain device MD on the 2PTC box (DPA3, FP32), for ncu launch lists beside
tools/dev/dd_compute_probe.py: `ncu ... python tools/dev/sd_probe.py [n] [steps]`."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2602_02234_b200 as P
from paper_2602_02234_b200.md import DeviceMD

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4114
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
m = P.make_model(P.ModelFamily.message_passing, 3, 0.6, 2, 8, 32, 1)
s = P.generate_synthetic_system(n)
md = DeviceMD(P.Context(m, max_atoms=n), s.positions, s.velocities, s.masses, s.types, s.box,
              precision=P.Precision.fp32, steps_per_graph=1)
md.run(steps)
md.state()
