"""Repformer NVE diagnosis: energy, kinetic energy, minimum pair distance and max force along FP64 runs at dt = 1 and 0.25 fs."""
import sys, numpy as np
sys.path.insert(0, "/root/repo")
import paper_2602_02234_b200 as P
from paper_2602_02234_b200.md import DeviceMD
import oracle as O
fam = P.ModelFamily.repformer
m = P.make_dp_model(fam, 3)
s = P.generate_synthetic_system(582, temperature=300.0)
for prec in (P.Precision.fp64,):
    for dt in (0.001, 0.00025):
        md = DeviceMD(P.Context(m), s.positions, s.velocities, s.masses, s.types, s.box, dt, prec, steps_per_graph=50)
        out = []
        for k in range(10):
            md.run(int(0.4 / dt / 10 * 1e-0) if False else int(0.0004 / dt * 1000 / 10))
            x, v, f, e = md.state()
            ke = 0.5 * float(np.sum(s.masses[:, None] * v * v))
            off, nbr, dr = O.neighbors(x, s.box, 0.6)
            rmin = float(np.sqrt((dr**2).sum(1)).min())
            fmax = float(np.abs(f).max())
            out.append((round(e, 3), round(ke, 2), round(e + ke, 3), round(rmin, 4), round(fmax, 1)))
        print(prec.name, dt, out)
