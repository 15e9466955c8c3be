"""Per-kernel times of one MD step (graph per step, events between kernels) with and
without the 256 MiB L2 flush before each step: where the flushed-L2 penalty lands.
usage: python tools/flush_probe.py [dpa3|dpa2] [1YRF|2PTC]"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_02234_b200 as P
from paper_2602_02234_b200._lib import check, lib
from paper_2602_02234_b200.md import DeviceMD

name = sys.argv[1] if len(sys.argv) > 1 else "dpa3"
system = sys.argv[2] if len(sys.argv) > 2 else "1YRF"
fam, depth = {"dpa3": (1, 3), "dpa2": (0, 1)}[name]
m = P.make_model(P.ModelFamily(fam), depth, 0.6, 2, 8, 32, 1)
s = P.generate_synthetic_system(P.PAPER_SYSTEMS[system])
L = lib()
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(dev)
torch.cuda.set_stream(stream)
ctx = P.Context(m, max_atoms=s.n_atoms)
check(L.hmdp_set_stream(ctx.handle, ctypes.c_void_p(stream.cuda_stream)))
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
buf = (ctypes.c_float * 64)()
cnt = ctypes.c_int()


def run(do_flush, K=300, prof=True):
    check(L.hmdp_profile(ctx.handle, 1 if prof else 0))
    md = DeviceMD(ctx, s.positions, s.velocities, s.masses, s.types, s.box, 0.001,
                  P.Precision.fp32, steps_per_graph=1)
    sums, counts = {}, {}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tot = 0.0
    for k in range(K + 5):
        if do_flush:
            flush.zero_()
        e0.record(stream)
        check(L.hmdp_md_enqueue(md.handle, 1))
        e1.record(stream)
        if prof:
            check(L.hmdp_profile_read(ctx.handle, buf, 64, ctypes.byref(cnt)))
        torch.cuda.synchronize()
        if k < 5:
            continue
        tot += e0.elapsed_time(e1)
        if prof:
            for i in range(cnt.value):
                nm = L.hmdp_profile_name(ctx.handle, i).decode()
                sums[nm] = sums.get(nm, 0.0) + buf[i]
                counts[nm] = counts.get(nm, 0) + 1
    md.close()
    check(L.hmdp_profile(ctx.handle, 0))
    return tot / K * 1e3, {k: sums[k] / counts[k] * 1e3 for k in sums}


for fl in (False, True):
    step, ks = run(fl, prof=False)
    stepp, ksp = run(fl, prof=True)
    print(f"flush={fl}: step {step:.1f} us (no events), {stepp:.1f} us (events)",
          {k: round(v, 2) for k, v in ksp.items()})
