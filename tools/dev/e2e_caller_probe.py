"""Wall time per step of the C++ velocity-Verlet caller over hmdp_compute, with the
context on its own stream vs on a torch stream (dev probe for the e2e leg)."""
import ctypes, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2602_02234_b200 as P
from paper_2602_02234_b200._lib import LIB_PATH, check, lib, ptr

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4114
caller = ctypes.CDLL(os.path.join(os.path.dirname(LIB_PATH), "libhmdp_caller.so"))
m = P.make_model(P.ModelFamily.message_passing, 3, 0.6, 2, 8, 32, 1)
s = P.generate_synthetic_system(n)
for mode in ("own", "torch", "own", "torch"):
    ctx = P.Context(m, max_atoms=n)
    if mode == "torch":
        st = torch.cuda.Stream()
        check(lib().hmdp_set_stream(ctx.handle, ctypes.c_void_p(st.cuda_stream)))
    x = s.positions.copy(); v = s.velocities.copy(); t = s.types.astype(np.int32)
    mass = np.ascontiguousarray(s.masses, dtype=np.float64); box = np.ascontiguousarray(s.box)
    f = np.ascontiguousarray(ctx.compute(x, t, box, P.Precision.fp32).forces).copy()
    e = ctypes.c_double()
    args = lambda k: (ctx.handle, ctypes.c_int(n), ptr(x), ptr(v), ptr(f), ptr(t), ptr(box), ptr(mass),
                      ctypes.c_double(0.001), ctypes.c_int(k), ctypes.c_int(0), ctypes.byref(e))
    check(caller.hmdp_caller_velocity_verlet(*args(5)))
    K = 300
    t0 = time.perf_counter()
    check(caller.hmdp_caller_velocity_verlet(*args(K)))
    dt = (time.perf_counter() - t0) / K * 1e6
    t0 = time.perf_counter()
    for _ in range(K):
        check(lib().hmdp_compute(ctx.handle, n, ptr(x), ptr(t), ptr(box), 0, ctypes.byref(e), None, ptr(f), None, None))
    dc = (time.perf_counter() - t0) / K * 1e6
    print(f"{mode:6s} n={n}: caller {dt:.1f} us/step ({1e6/dt:.0f} steps/s), hmdp_compute alone {dc:.1f} us", flush=True)
