import os, sys
sys.path.insert(0, '.')
import numpy as np
import paper_2602_02234_b200 as P
s = P.generate_synthetic_system(582)
m = P.make_model(P.ModelFamily.message_passing, 3, 0.6, 2, 8, 32, 1)
ctx = P.Context(m)
try:
    o = ctx.compute(s.positions, s.types, s.box, P.Precision.fp32)
    print("ok", o.energy)
except Exception as e:
    print("ERR", e)
