import sys, json, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, './tests')
import paper_2602_02234_b200 as P
from paper_2602_02234_b200 import dd
gm = json.load(open('./tests/golden/models.json'))
s = P.generate_synthetic_system(1231)
for mname in ['dpa2','dpa3']:
  m = P.model_from_json(gm[mname])
  for dims in [(2,1,1),(2,2,1),(1,2,1)]:
    world = dims[0]*dims[1]*dims[2]
    hub = dd.Hub(world)
    engs = [dd.HaloDD(P.Context(m, max_atoms=1231), 1231, s.types, s.box, dims, r, P.Precision.fp64) for r in range(world)]
    for e in engs: e.attach_hub(hub.handle); e.load(s.positions)
    pre = [ (e.roles()==1).sum() for e in engs]
    dd.run_hub(engs, "eval")
    R = np.array([e.roles() for e in engs])
    own = (R==1).sum(0)
    print(mname, dims, 'plan owned', pre, 'after', [(r==1).sum() for r in R], 'halo', [(r==2).sum() for r in R], 'bad', np.where(own!=1)[0][:10], [e.sync() or e.energy_virial()[0] for e in engs])
    bad = np.where(own!=1)[0]
    if len(bad): print('  roles of bad', R[:, bad[:5]].T, s.positions[bad[:5]], s.box)
