import json, numpy as np, sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_2602_02234_b200 as P
from paper_2602_02234_b200.dd import DeviceDD, run_local
gm = json.load(open('/root/repo/tests/golden/models.json'))
s = P.generate_synthetic_system(1231)
mname = sys.argv[1] if len(sys.argv) > 1 else 'dpa3'
m = P.model_from_json(gm[mname])
ref = P.Context(m).compute(s.positions, s.types, s.box, P.Precision.fp64)
for dims in [(1,1,1),(1,1,1),(2,1,1),(2,1,1)]:
    world = dims[0]*dims[1]*dims[2]
    engs = [DeviceDD(P.Context(m, max_atoms=1231), 1231, s.types, s.box, dims, r, P.Precision.fp64) for r in range(world)]
    for e in engs: e.load(s.positions)
    run_local(engs)
    E, F, W, W9 = engs[0].result()
    err = np.abs(F - ref.forces).max(1)
    print(mname, dims, 'E', E - ref.energy, 'Ferr', err.max(), 'n_bad', (err > 1e-8).sum())
