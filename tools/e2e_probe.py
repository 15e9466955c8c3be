"""Where does the host-buffer (e2e) step time go?  usage: python tools/e2e_probe.py"""
import ctypes
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_02234_b200 as P
from paper_2602_02234_b200._lib import lib, ptr

m = P.make_model(P.ModelFamily.message_passing, 3, 0.6, 2, 8, 32, 1)
s = P.generate_synthetic_system(582)
ctx = P.Context(m, max_atoms=582)
x = s.positions.copy()
t = s.types.astype(np.int32)
K = 2000


def bench(name, fn):
    for _ in range(50):
        fn()
    t0 = time.perf_counter()
    for _ in range(K):
        fn()
    dt = (time.perf_counter() - t0) / K * 1e6
    print(f"{name:40s} {dt:8.1f} us")


bench("Context.compute (python API)", lambda: ctx.compute(x, t, s.box, P.Precision.fp32))
f = np.zeros((582, 3))
w9 = np.zeros(9)
e, w = ctypes.c_double(), ctypes.c_double()
px, pt, pb, pf, pw9 = ptr(x), ptr(t), ptr(np.ascontiguousarray(s.box)), ptr(f), ptr(w9)
L = lib()
bench("hmdp_compute (raw ctypes, prebuilt args)",
      lambda: L.hmdp_compute(ctx.handle, 582, px, pt, pb, 0, ctypes.byref(e), None, pf, pw9,
                             ctypes.byref(w)))
v = s.velocities.copy()
im = (0.0005 / s.masses)[:, None]


def vv():
    global v, x
    v += f * im
    x += v * 0.001
    v += f * im


bench("numpy velocity Verlet (3 ops)", vv)
