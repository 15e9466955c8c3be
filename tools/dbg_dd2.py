import json, sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2602_02234_b200 as P
from paper_2602_02234_b200 import dd
gm = json.load(open('/root/repo/tests/golden/models.json'))
s = P.generate_synthetic_system(1231)
m = P.model_from_json(gm['dpa3'])
ref = P.Context(m).compute(s.positions, s.types, s.box, P.Precision.fp64)
for dims in [(1,1,1),(2,1,1)]:
    world = dims[0]*dims[1]*dims[2]
    inp = P.build_input_periodic(s.positions, s.types, np.arange(1231), s.box, 0.6)
    own = dd.owners(s.positions, s.box, dims)
    plans = dd.make_plans(inp.edge_offset, inp.edge_neighbor, inp.edge_dr, s.types, own, world)
    engs = [dd.GpuEngine(P.Context(m), P.Precision.fp64) for _ in range(world)]
    E, F, W, W9 = dd.evaluate_local(engs, plans, m.depth())
    Fg = np.zeros((1231, 3))
    for r in range(world): Fg[plans[r].owned] = F[r]
    print('hostDD', dims, E - ref.energy, np.abs(Fg - ref.forces).max())
