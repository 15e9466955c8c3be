"""Randomised parity sweep (beyond the pytest cases): random system sizes, seeds and
model seeds for every family, FP64 and FP32 through hmdp_compute against the oracles
(the C restatement for the reference families, the FP64 torch oracle for the
DeePMD-style ones).  Prints one JSON summary; usage: python tools/parity_sweep.py [cases]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O
import paper_2602_02234_b200 as P
from oracle import dpfamily as DF

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 100
rng = np.random.default_rng(2602)
fams = [("dpa2", 0, 1), ("dpa3", 1, 3), ("se_a", 2, 1), ("repformer", 3, 2), ("repflow", 4, 2)]
worst = {f[0]: {"fp64_e": 0.0, "fp64_f": 0.0, "fp32_e": 0.0, "fp32_e_norm": 0.0, "fp32_f": 0.0,
               "fp32_e_over_1e-6": 0, "reference_fp32_e_over_1e-6": 0,
               "fp32_e_vs_reference_fp32_max": 0.0, "cases": 0}
         for f in fams}
t0 = time.perf_counter()
for c in range(cases):
    name, fam, depth = fams[c % len(fams)]
    n = int(rng.integers(60, 700 if fam < 2 else 400))
    try:
        s = P.generate_synthetic_system(n, seed=int(rng.integers(1, 10_000)))
    except RuntimeError:
        continue
    mseed = int(rng.integers(1, 1000))
    if fam >= 2:
        m = P.make_dp_model(P.ModelFamily(fam), depth, seed=mseed)
        ref = DF.evaluate(m.as_dict(), s.types, *O.neighbors(s.positions, s.box, 0.6))
    else:
        m = P.make_model(P.ModelFamily(fam), depth, 0.6, 2, 8, 32, mseed)
        ref = O.evaluate(json.loads(m.to_json()), s.types, *O.neighbors(s.positions, s.box, 0.6))
    rms = float(np.sqrt(np.mean(np.sum(ref["forces"] ** 2, axis=1))))
    ctx = P.Context(m, max_atoms=n)
    w = worst[name]
    # the reference's own FP32 path beside ours (reference families): how far FP32
    # arithmetic itself lands from FP64 on this case
    ref32 = None
    if fam < 2:
        ref32 = O.evaluate(json.loads(m.to_json()), s.types, *O.neighbors(s.positions, s.box, 0.6),
                           prec="fp32")
    for prec in ("fp64", "fp32"):
        out = ctx.compute(s.positions, s.types, s.box, P.Precision[prec], per_atom=True)
        de = abs(out.energy - ref["energy"]) / abs(ref["energy"])
        df = float(np.abs(out.forces - ref["forces"]).max()) / rms
        if prec == "fp32" and de > w["fp32_e"]:
            w["fp32_e_case"] = {
                "n": n, "E": ref["energy"], "sum_abs_e_i": float(np.abs(ref["per_atom"]).sum()),
                "abs_err": abs(out.energy - ref["energy"]),
                "err_rel_sum_abs_e_i": abs(out.energy - ref["energy"]) / float(np.abs(ref["per_atom"]).sum()),
                "reference_fp32_rel_err": (abs(ref32["energy"] - ref["energy"]) / abs(ref["energy"])
                                           if ref32 is not None else None),
                "ours_vs_reference_fp32_rel": (abs(out.energy - ref32["energy"]) / abs(ref["energy"])
                                               if ref32 is not None else None)}
        w[prec + "_e"] = max(w[prec + "_e"], de)
        w[prec + "_f"] = max(w[prec + "_f"], df)
        if prec == "fp32":  # energy error relative to sum |e_i| (robust to cancellation)
            w["fp32_e_norm"] = max(w["fp32_e_norm"], abs(out.energy - ref["energy"]) /
                                   float(np.abs(ref["per_atom"]).sum()))
            w["fp32_e_over_1e-6"] += int(de > 1e-6)
            if ref32 is not None:  # ours vs the reference's own FP32 path, both against FP64
                r32 = abs(ref32["energy"] - ref["energy"])
                w["reference_fp32_e_over_1e-6"] += int(r32 / abs(ref["energy"]) > 1e-6)
                w["fp32_e_vs_reference_fp32_max"] = max(
                    w["fp32_e_vs_reference_fp32_max"],
                    abs(out.energy - ref["energy"]) / max(r32, 1e-300))
    w["cases"] += 1
    ctx.close()
# the canonical configurations of the north star (the paper boxes, the
# DPA2 / DPA3 analogs with seed-1 weights): FP32 energy relative to |E| itself
canon = {}
for name, fam, depth in fams[:2]:
    m = P.make_model(P.ModelFamily(fam), depth, 0.6, 2, 8, 32, 1)
    for system, n in P.PAPER_SYSTEMS.items():
        s = P.generate_synthetic_system(n)
        ref = O.evaluate(json.loads(m.to_json()), s.types, *O.neighbors(s.positions, s.box, 0.6))
        out = P.Context(m, max_atoms=n).compute(s.positions, s.types, s.box, P.Precision.fp32)
        canon[f"{name}_{system}"] = abs(out.energy - ref["energy"]) / abs(ref["energy"])
ok = all(w["fp64_e"] <= 1e-9 and w["fp64_f"] <= 1e-9 and w["fp32_f"] <= 1e-4
         for w in worst.values()) and max(canon.values()) <= 1e-6
print(json.dumps({"cases": cases, "wall_s": time.perf_counter() - t0, "all_within_tolerance": ok,
                  "headline": {
                      "canonical_fp32_dE_over_E": canon,
                      "canonical_fp32_dE_over_E_max": max(canon.values()),
                      "random_fp32_dE_over_E_max": {k: w["fp32_e"] for k, w in worst.items()},
                      "random_fp32_cases_over_1e-6": {k: w["fp32_e_over_1e-6"] for k, w in worst.items()},
                      "random_reference_own_fp32_cases_over_1e-6": {
                          k: worst[k]["reference_fp32_e_over_1e-6"] for k in ("dpa2", "dpa3")},
                      "random_fp32_error_vs_reference_own_fp32_max": {
                          k: worst[k]["fp32_e_vs_reference_fp32_max"] for k in ("dpa2", "dpa3")}},
                  "tolerances": {"fp64": "E, F <= 1e-9 (relative / of RMS force)",
                                 "fp32": "E <= 1e-6 relative to |E| on the canonical configs; "
                                         "random models: |dE|/|E| reported beside the "
                                         "reference's own FP32 error (cancelling per-atom "
                                         "energies make |E| small for both); F <= 1e-4 of RMS"},
                  "worst": worst}, indent=1))
