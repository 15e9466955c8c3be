import json, numpy as np, sys, torch
sys.path.insert(0, '/root/repo')
import paper_2602_02234_b200 as P
from paper_2602_02234_b200.dd import DeviceDD, run_local
gm = json.load(open('/root/repo/tests/golden/models.json'))
s = P.generate_synthetic_system(1231)
m = P.model_from_json(gm['dpa3'])
ref = P.Context(m).compute(s.positions, s.types, s.box, P.Precision.fp64)
# dirty the driver's free memory: a context with garbage-filled buffers, destroyed
for k in range(3):
    c = P.Context(m, max_atoms=1231)
    c.compute(s.positions + 0.01 * k, s.types, s.box, P.Precision.fp64)
    del c
A = [DeviceDD(P.Context(m, max_atoms=1231), 1231, s.types, s.box, (1,1,1), 0, P.Precision.fp64)]
A[0].load(s.positions)
run_local(A)
E, F, W, W9 = A[0].result()
print('A', E - ref.energy, np.abs(F - ref.forces).max())
c = P.Context(m, max_atoms=1231)
o = c.compute(s.positions, s.types, s.box, P.Precision.fp64)
print('normal after dirty', o.energy - ref.energy, np.abs(o.forces - ref.forces).max())
