"""Long-run check of the Verlet rows: N MD steps with HMDP_SKIN = 0.1 nm (default) and
with HMDP_SKIN = 0 (full search every step) must end in bitwise the same state.
usage: python tools/verlet_long.py [steps]  (prints one line per model x box)"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_02234_b200 as P
from paper_2602_02234_b200.md import DeviceMD

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5000


def run(m, s, skin, prec):
    os.environ["HMDP_SKIN"] = str(skin)
    ctx = P.Context(m, max_atoms=s.n_atoms)
    md = DeviceMD(ctx, s.positions, s.velocities, s.masses, s.types, s.box, 0.001, prec,
                  steps_per_graph=100)
    t0 = time.perf_counter()
    md.run(steps)
    st = md.state()
    dt = time.perf_counter() - t0
    stats = md.stats()
    md.close()
    return st, stats, dt


for name, fam, depth in (("dpa3", P.ModelFamily.message_passing, 3),
                         ("dpa2", P.ModelFamily.embed_fit, 1)):
    m = P.make_model(fam, depth, 0.6, 2, 8, 32, 1)
    for system in ("1YRF", "2PTC"):
        s = P.generate_synthetic_system(P.PAPER_SYSTEMS[system])
        for prec in (P.Precision.fp32, P.Precision.fp64):
            a, sa, ta = run(m, s, 0.1, prec)
            b, sb, tb = run(m, s, 0.0, prec)
            same = all(np.array_equal(u, v) for u, v in zip(a[:3], b[:3])) and a[3] == b[3]
            print(f"{name} {system} {prec.name}: {steps} steps, bitwise equal: {same}; "
                  f"skin {sa[0]} nm, {sa[1]} row builds ({steps / max(sa[1], 1):.0f} steps per build); "
                  f"wall {ta:.2f} s vs {tb:.2f} s without rows; E_pot {a[3]:.6f}", flush=True)
