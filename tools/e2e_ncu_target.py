"""ncu target: 30 hmdp_compute calls (graph path) of the DPA2 analog.  usage: python tools/e2e_ncu_target.py N"""
import sys, os, numpy as np
sys.path.insert(0, "/root/repo")
import paper_2602_02234_b200 as P
n = int(sys.argv[1])
m = P.make_model(P.ModelFamily.embed_fit, 1, 0.6, 2, 8, 32, 1)
s = P.generate_synthetic_system(n)
ctx = P.Context(m, max_atoms=n)
x = s.positions.copy(); t = s.types.astype(np.int32)
for _ in range(30):
    ctx.compute(x, t, s.box, P.Precision.fp32)
print("ok")
