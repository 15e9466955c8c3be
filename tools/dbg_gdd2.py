import json, numpy as np, sys, torch
sys.path.insert(0, '/root/repo')
import paper_2602_02234_b200 as P
from paper_2602_02234_b200.dd import DeviceDD, run_local
gm = json.load(open('/root/repo/tests/golden/models.json'))
s = P.generate_synthetic_system(1231)
m = P.model_from_json(gm['dpa3'])
ref = P.Context(m).compute(s.positions, s.types, s.box, P.Precision.fp64)
A = [DeviceDD(P.Context(m, max_atoms=1231), 1231, s.types, s.box, (1,1,1), 0, P.Precision.fp64)]
A[0].load(s.positions)
run_local(A)
print('A out', A[0].out[:2].tolist(), 'A f', float(A[0].f.abs().sum()))
B = [DeviceDD(P.Context(m, max_atoms=1231), 1231, s.types, s.box, (1,1,1), 0, P.Precision.fp64)]
print('ptrs A', [hex(t.data_ptr()) for t in (A[0].f, A[0].out)], 'B', [hex(t.data_ptr()) for t in (B[0].f, B[0].out)])
A[0].out.zero_(); A[0].f.zero_()
B[0].load(s.positions)
run_local(B)
torch.cuda.synchronize()
print('after B: A out', A[0].out[:2].tolist(), 'A f', float(A[0].f.abs().sum()), 'B out', B[0].out[:2].tolist(), 'B f', float(B[0].f.abs().sum()))
