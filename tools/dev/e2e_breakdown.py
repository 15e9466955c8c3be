"""e2e step breakdown: the C++ velocity-Verlet caller over hmdp_compute (bench.py's e2e
leg) for one model on the 2PTC box; run with HMDP_E2E_PROBE=1 for the host-timer split
of the graph-replay path (printed at exit).  usage: e2e_breakdown.py dpa3|dpa2 [n]"""
import ctypes, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2602_02234_b200 as P
from paper_2602_02234_b200._lib import LIB_PATH, check, lib, ptr

name = sys.argv[1] if len(sys.argv) > 1 else "dpa3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4114
caller = ctypes.CDLL(os.path.join(os.path.dirname(LIB_PATH), "libhmdp_caller.so"))
m = (P.make_model(P.ModelFamily.message_passing, 3, 0.6, 2, 8, 32, 1) if name == "dpa3"
     else P.make_model(P.ModelFamily.embed_fit, 1, 0.6, 2, 8, 32, 1))
s = P.generate_synthetic_system(n)
ctx = P.Context(m, max_atoms=n)
x = s.positions.copy(); v = s.velocities.copy(); t = s.types.astype(np.int32)
mass = np.ascontiguousarray(s.masses, dtype=np.float64); box = np.ascontiguousarray(s.box)
f = np.ascontiguousarray(ctx.compute(x, t, box, P.Precision.fp32).forces).copy()
e = ctypes.c_double()
args = lambda k: (ctx.handle, ctypes.c_int(n), ptr(x), ptr(v), ptr(f), ptr(t), ptr(box), ptr(mass),
                  ctypes.c_double(0.001), ctypes.c_int(k), ctypes.c_int(0), ctypes.byref(e))
check(caller.hmdp_caller_velocity_verlet(*args(50)))
K = 2000
t0 = time.perf_counter()
check(caller.hmdp_caller_velocity_verlet(*args(K)))
dt = (time.perf_counter() - t0) / K * 1e6
print(f"{name} n={n}: caller {dt:.1f} us/step ({1e6/dt:.0f} steps/s)", flush=True)
