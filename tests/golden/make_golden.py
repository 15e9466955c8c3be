"""Generate the committed golden vectors from the REFERENCE itself.

Runs the reference compiled from /root/reference/proj/src (oracle/_ref, built by
oracle/Makefile) -- never our code -- and stores, per system:
  fixture  : generate_synthetic_system positions/types/masses/velocities/box
             (synthetic.cpp:36-130, seed 7, density 33.4, fraction 0.35)
  csr      : build_input_periodic edge_offset / edge_neighbor / edge_dr
  models   : make_model(embed_fit,1,...) and make_model(message_passing,3,...)
             with seed 1 (model.cpp:70-100), as JSON
  outputs  : evaluate() energy / per-atom energy / forces / virial / counters in
             fp64 and fp32, and descriptors() (inference.cpp:420-447)

Usage (in the build container, where /root/reference exists):
    python tests/golden/make_golden.py
"""
from __future__ import annotations

import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
SYSTEMS = {"n64": 64, "1YRF": 582}


def descriptors_ref(model_handle, n, x, t, off, nbr, dr, nd):
    L = O.ref()
    out = np.zeros((n, nd))
    code = L.ref_descriptors(model_handle.h, n, O._p(x), O._p(t), O._p(off), O._p(nbr), O._p(dr),
                             O._p(out))
    assert code == 0, L.ref_last_error()
    return out


def main():
    O.build(ref=True)
    models = {"dpa2": O.ref_model_json(0, 1), "dpa3": O.ref_model_json(1, 3)}
    with open(os.path.join(OUT, "models.json"), "w") as f:
        json.dump(models, f)
    for name, n in SYSTEMS.items():
        x, t, m, v, b = O.ref_synthetic(n)
        off, nbr, dr = O.ref_build_input(x, t, b, 0.6)
        arrays = dict(positions=x, types=t, masses=m, velocities=v, box=b, edge_offset=off,
                      edge_neighbor=nbr, edge_dr=dr)
        for mname, js in models.items():
            rm = O.RefModel(js)
            for prec in ("fp64", "fp32"):
                r = O.ref_evaluate_csr(rm, x, t, off, nbr, dr, prec=prec)
                p = f"{mname}_{prec}_"
                arrays[p + "energy"] = np.array(r["energy"])
                arrays[p + "per_atom"] = r["per_atom"]
                arrays[p + "forces"] = r["forces"]
                arrays[p + "virial"] = np.array(r["virial"])
                arrays[p + "counters"] = np.array([r["flops"], r["act_bytes"]], dtype=np.uint64)
            arrays[f"{mname}_descriptors"] = descriptors_ref(rm, n, x, t, off, nbr, dr, 16)
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **arrays)
        print(name, n, "edges", int(off[-1]))
    # switch function samples (inference.cpp:34-45)
    r = np.linspace(0.0, 0.7, 141)
    sv = np.array([O.ref().ref_switch_value(float(q), 0.6) for q in r])
    sd = np.array([O.ref().ref_switch_derivative(float(q), 0.6) for q in r])
    np.savez_compressed(os.path.join(OUT, "switch.npz"), r=r, value=sv, derivative=sd)


if __name__ == "__main__":
    main()
