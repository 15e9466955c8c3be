"""Small workload for compute-sanitizer: every family once through hmdp_compute (FP32 and
FP64; direct path, graph capture, replay), a few device MD steps, a device-DD evaluation."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_02234_b200 as P
from paper_2602_02234_b200.md import DeviceMD

s = P.generate_synthetic_system(64)
models = [P.make_model(P.ModelFamily.embed_fit, 1, 0.6, 2, 8, 32, 1),
          P.make_model(P.ModelFamily.message_passing, 3, 0.6, 2, 8, 32, 1),
          P.make_dp_model(P.ModelFamily.se_a, 1), P.make_dp_model(P.ModelFamily.repformer, 2),
          P.make_dp_model(P.ModelFamily.repflow, 2)]
for m in models:
    ctx = P.Context(m, max_atoms=64)
    for prec in (P.Precision.fp32, P.Precision.fp64):
        for _ in range(3):  # direct path, capture, replay
            out = ctx.compute(s.positions, s.types, s.box, prec)
    md = DeviceMD(ctx, s.positions, s.velocities, s.masses, s.types, s.box, 0.001,
                  P.Precision.fp32, steps_per_graph=2)
    md.run(4)
    print(m.family, out.energy, md.state()[3], flush=True)
from paper_2602_02234_b200.dd import DeviceDD, run_local  # noqa: E402

m = models[1]
engs = [DeviceDD(P.Context(m, max_atoms=64), 64, s.types, s.box, (2, 1, 1), r,
                 P.Precision.fp64) for r in range(2)]
for e in engs:
    e.load(s.positions)
run_local(engs)
print("dd", engs[0].result()[0])
