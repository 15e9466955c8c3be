"""Long NVE run on the device MD loop: total-energy drift of the DPA2 / DPA3 analogs
in FP32 and FP64 (velocity Verlet, dt = 1 fs, neighbour list rebuilt every step).
usage: python tools/nve_drift.py [dpa3|dpa2|se_a|repformer|repflow] [steps] [fp32|fp64]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_02234_b200 as P
from paper_2602_02234_b200.md import DeviceMD

name = sys.argv[1] if len(sys.argv) > 1 else "dpa3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
prec = P.Precision[sys.argv[3] if len(sys.argv) > 3 else "fp32"]
fam, depth = {"dpa3": (1, 3), "dpa2": (0, 1), "se_a": (2, 1), "repformer": (3, 3),
              "repflow": (4, 3)}[name]
if fam >= 2:  # DeePMD-style families
    m = P.make_dp_model(P.ModelFamily(fam), depth)
else:
    m = P.make_model(P.ModelFamily(fam), depth, 0.6, 2, 8, 32, 1)
s = P.generate_synthetic_system(582, temperature=300.0)
md = DeviceMD(P.Context(m), s.positions, s.velocities, s.masses, s.types, s.box, 0.001, prec,
              steps_per_graph=100)
KB = 0.0083144626  # kJ/mol/K


def totals():
    x, v, f, e = md.state()
    ke = 0.5 * float(np.sum(s.masses[:, None] * v * v))
    return e, ke, e + ke, ke * 2.0 / (3 * len(s.masses) * KB)


rows = []
e0 = totals()
t0 = time.perf_counter()
chunk = max(100, steps // 20)
done = 0
while done < steps:
    md.run(chunk)
    done += chunk
    ep, ke, et, temp = totals()
    rows.append({"step": done, "E_pot": ep, "E_kin": ke, "E_tot": et, "T_K": temp})
wall = time.perf_counter() - t0
etot = np.array([r["E_tot"] for r in rows])
drift = (etot[-1] - e0[2]) / (steps * 1e-3)  # kJ/mol per ps
print(json.dumps({"model": name, "precision": prec.name, "atoms": 582, "steps": steps,
                  "E_tot_start": e0[2], "E_tot_end": float(etot[-1]),
                  "E_tot_std": float(etot.std()), "drift_kJ_mol_per_ps": float(drift),
                  "drift_per_atom_kJ_mol_per_ns": float(drift * 1e3 / 582),
                  "T_K_mean": float(np.mean([r["T_K"] for r in rows])),
                  "wall_s": wall, "samples": rows[:: max(1, len(rows) // 5)]}))
