"""Static DeePMD-family forces against the FP64 oracle at neighbour capacities 64 / 96 / 128."""
import sys, numpy as np
sys.path.insert(0, "/root/repo")
import paper_2602_02234_b200 as P
import oracle as O
from oracle import dpfamily as DF
s = P.generate_synthetic_system(582)
off, nbr, dr = O.neighbors(s.positions, s.box, 0.6)
print("max nnei", np.diff(off).max())
for fam, depth in ((P.ModelFamily.se_a, 1), (P.ModelFamily.repformer, 3), (P.ModelFamily.repflow, 3)):
    m = P.make_dp_model(fam, depth)
    ref = DF.evaluate(m.as_dict(), s.types, off, nbr, dr)
    rms = np.sqrt(np.mean(np.sum(ref["forces"]**2, 1)))
    for cap in (64, 96, 128):
        ctx = P.Context(m, max_atoms=582, max_neighbors=cap)
        for prec in (P.Precision.fp64, P.Precision.fp32):
            o = ctx.compute(s.positions, s.types, s.box, prec)
            print(fam.name, cap, prec.name, abs(o.energy - ref["energy"]) / abs(ref["energy"]),
                  np.abs(o.forces - ref["forces"]).max() / rms)
