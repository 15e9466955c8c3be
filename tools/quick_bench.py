"""Quick timing of the device MD loop and the host-buffer C-ABI path (dev aid)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2602_02234_b200 as P
from paper_2602_02234_b200.md import DeviceMD

for mname, fam, depth in [("dpa2", 0, 1), ("dpa3", 1, 3)]:
    m = P.make_model(P.ModelFamily(fam), depth, 0.6, 2, 8, 32, 1)
    for n in [582, 4114]:
        s = P.generate_synthetic_system(n)
        ctx = P.Context(m)
        for _ in range(3):
            ctx.compute(s.positions, s.types, s.box)
        t = time.perf_counter(); K = 50
        for _ in range(K):
            ctx.compute(s.positions, s.types, s.box)
        host_ms = (time.perf_counter() - t) / K * 1e3
        md = DeviceMD(ctx, s.positions, s.velocities, s.masses, s.types, s.box, steps_per_graph=50)
        md.run(50)
        md.state()
        t = time.perf_counter(); S = 500
        md.run(S)
        x, v, f, e = md.state()
        md_ms = (time.perf_counter() - t) / S * 1e3
        print(f"{mname} n={n}: host-path compute {host_ms:.3f} ms, device MD {md_ms:.4f} ms/step "
              f"({1e3/md_ms:.0f} steps/s, {0.0864*1e3/md_ms:.1f} ns/day), epot={e:.4f}", flush=True)
