import json, numpy as np, sys, torch
sys.path.insert(0, '/root/repo')
import paper_2602_02234_b200 as P
from paper_2602_02234_b200.dd import DeviceDD, run_local
gm = json.load(open('/root/repo/tests/golden/models.json'))
s = P.generate_synthetic_system(1231)
m = P.model_from_json(gm['dpa3'])
A = [DeviceDD(P.Context(m, max_atoms=1231), 1231, s.types, s.box, (1,1,1), 0, P.Precision.fp64)]
A[0].load(s.positions)
run_local(A)
print('done', A[0].result()[0])
