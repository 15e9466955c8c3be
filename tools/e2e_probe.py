"""Where does the host-buffer (e2e) step time go?
usage: python tools/e2e_probe.py [dpa3|dpa2] [n_atoms]"""
import ctypes
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_02234_b200 as P
from paper_2602_02234_b200._lib import lib, ptr

model = sys.argv[1] if len(sys.argv) > 1 else "dpa3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 582
fam = P.ModelFamily.message_passing if model == "dpa3" else P.ModelFamily.embed_fit
m = P.make_model(fam, 3 if model == "dpa3" else 1, 0.6, 2, 8, 32, 1)
s = P.generate_synthetic_system(n)
ctx = P.Context(m, max_atoms=n)
x = s.positions.copy()
t = s.types.astype(np.int32)
K = 2000
print(f"{model} n={n}")


def bench(name, fn):
    for _ in range(50):
        fn()
    t0 = time.perf_counter()
    for _ in range(K):
        fn()
    dt = (time.perf_counter() - t0) / K * 1e6
    print(f"{name:44s} {dt:8.1f} us")


bench("Context.compute (python API)", lambda: ctx.compute(x, t, s.box, P.Precision.fp32))
f = np.zeros((n, 3))
w9 = np.zeros(9)
e, w = ctypes.c_double(), ctypes.c_double()
px, pt, pb, pf, pw9 = ptr(x), ptr(t), ptr(np.ascontiguousarray(s.box)), ptr(f), ptr(w9)
L = lib()
bench("hmdp_compute (raw ctypes, prebuilt args)",
      lambda: L.hmdp_compute(ctx.handle, n, px, pt, pb, 0, ctypes.byref(e), None, pf, pw9,
                             ctypes.byref(w)))
v = s.velocities.copy()
im = (0.0005 / s.masses)[:, None]
tmp = np.empty_like(v)


def vv():
    global v, x
    v += f * im
    x += v * 0.001
    v += f * im


def vv_inplace():
    np.multiply(f, im, out=tmp)
    v.__iadd__(tmp)
    np.multiply(v, 0.001, out=tmp)
    x.__iadd__(tmp)
    np.multiply(f, im, out=tmp)
    v.__iadd__(tmp)


bench("numpy velocity Verlet (3 ops)", vv)
bench("numpy velocity Verlet (in place)", vv_inplace)
