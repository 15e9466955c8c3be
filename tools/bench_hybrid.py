"""Hybrid protein-in-water MD on the device (hmdp_hybrid_*): DP model (DPA3 / DPA2
analog) on the synthetic protein group + the reference's classical force field on
every atom, velocity Verlet, CUDA-graph captured.  Prints one JSON line per box.
usage: python tools/bench_hybrid.py [dpa3|dpa2] [steps]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # topology fixture only (the synthetic system's bonded terms)
import paper_2602_02234_b200 as P
from paper_2602_02234_b200.ff import ClassicalFF, HybridMD
from paper_2602_02234_b200.hybrid import plan_group_preprocessing, synthetic_topology

name = sys.argv[1] if len(sys.argv) > 1 else "dpa3"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 500
fam, depth = {"dpa3": (1, 3), "dpa2": (0, 1)}[name]
for system, n in (("1YRF", 582), ("2PTC", 4114)):
    s = P.generate_synthetic_system(n, temperature=300.0)
    t = O.ref_synthetic_topology(n)
    # NNPot preprocessing: the group's bonded terms go to the DP model, group pairs excluded
    topo2, plan = plan_group_preprocessing(synthetic_topology(n), "protein")
    eo = np.zeros(n + 1, dtype=np.int32)
    ex = []
    for i in range(n):
        ex += topo2.exclusions[i]
        eo[i + 1] = len(ex)
    kept = set(map(tuple, topo2.bonds))
    kb = [k for k, b in enumerate(map(tuple, t["bonds"])) if b in kept]
    ff = ClassicalFF(s.types, t["charges"], O.LJ_SIGMA, O.LJ_EPS, eo, np.array(ex), t["bonds"][kb],
                     t["bond_params"][kb], coulomb_scheme=1)
    m = P.make_model(P.ModelFamily(fam), depth, 0.6, 2, 8, 32, 1)
    md = HybridMD(P.Context(m, max_atoms=n), ff, plan.atoms, s.positions, s.velocities, s.masses,
                  s.types, s.box, dt_ps=0.001, precision=P.Precision.fp32, steps_per_graph=50)
    md.run(100)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    md.run(K)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    x, v, f, e = md.state()
    print(json.dumps({"workload": f"hybrid MD {name.upper()} on the protein group + classical FF "
                                  f"(reaction field) on all atoms, {system}-shaped box",
                      "atoms": n, "group": int(len(plan.atoms)), "steps_per_s": K / dt,
                      "ns_per_day": K / dt * 0.0864, "energies_bonded_lj_coulomb_nn": e.tolist(),
                      "timing": "wall clock around graph launches (50 steps per graph), fp32"}))
