"""The reference's own C++ call sites (build_input_periodic, evaluate,
descriptors, switch_value, ForceFunction in velocity_verlet_step) with the B200
path swapped in through include/hmdp_halomd.hpp; the program links the
reference compiled from its sources (oracle/Makefile `dropin`)."""
import os
import subprocess

import numpy as np
import pytest

from conftest import E_TOL, F_TOL, ROOT, rms

pytestmark = pytest.mark.gpu
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_test")


@pytest.mark.skipif(not os.path.exists(BIN), reason="dropin_test not built (needs /root/reference at build time)")
def test_reference_call_sites_with_b200_path():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "DROPIN PASS" in r.stdout, r.stdout + r.stderr


EXACT = os.path.join(ROOT, "oracle", "_ref", "dropin_exact")


def _load(d, name, dtype=np.float64):
    return np.fromfile(os.path.join(d, name), dtype=dtype)


@pytest.mark.skipif(not os.path.exists(EXACT),
                    reason="dropin_exact not built (needs /root/reference at build time)")
def test_exact_signature_dropin_matches_reference(tmp_path):
    """Reference call sites compiled UNCHANGED (tests/cpp/dropin_exact.cpp, halomd headers
    only) and linked with libhalomd_nn_b200.so in place of the reference's inference.o:
    CSR bit-exact, E / F / W / counters, descriptors, switch, errors and a 5-step
    velocity-Verlet ForceFunction loop, each against the reference itself."""
    import oracle as O

    r = subprocess.run([EXACT, str(tmp_path)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "DROPIN_EXACT DONE" in r.stdout, r.stdout + r.stderr
    d = str(tmp_path)
    log = open(os.path.join(d, "log.txt")).read()
    for natoms in (582, 1231):
        x, t, m, v, box = O.ref_synthetic(natoms)
        off, nbr, dr = O.ref_build_input(x, t, box, 0.6)
        tag = str(natoms)
        assert np.array_equal(_load(d, f"offset_{tag}", np.int32), off)
        assert np.array_equal(_load(d, f"nbr_{tag}", np.int32), nbr)
        assert np.array_equal(_load(d, f"dr_{tag}").reshape(-1, 3), dr)  # bit-exact FP64
        for depth, fam in ((1, 0), (3, 1)):
            model = O.RefModel(O.ref_model_json(fam, depth))
            for prec in ("fp64", "fp32"):
                ref = O.ref_evaluate_csr(model, x, t, off, nbr, dr, prec=prec)
                k = f"{tag}_d{depth}_{'f64' if prec == 'fp64' else 'f32'}"
                e, w, flops, act, inf = _load(d, f"scalars_{k}")
                f = _load(d, f"forces_{k}").reshape(-1, 3)
                sc = rms(ref["forces"])
                etol, ftol = (1e-11, 1e-10) if prec == "fp64" else (E_TOL, F_TOL)
                assert abs(e - ref["energy"]) <= etol * abs(ref["energy"]), (k, e, ref["energy"])
                assert np.abs(f - ref["forces"]).max() <= ftol * sc, k
                assert abs(w - ref["virial"]) <= ftol * max(abs(ref["virial"]), sc), k
                assert np.abs(_load(d, f"pae_{k}") - ref["per_atom"]).max() <= etol * sc + 1e-300
                assert (int(flops), int(act), int(inf)) == (ref["flops"], ref["act_bytes"], 1), k
            if natoms == 582:
                # 5 velocity-Verlet steps through the ForceFunction call site, FP64
                _, xr, vr, _ = O.ref_md(model, x, v, t, m, box, prec="fp64", steps=5)
                assert np.abs(_load(d, f"md_x_d{depth}").reshape(-1, 3) - xr).max() < 1e-11
                assert np.abs(_load(d, f"md_v_d{depth}").reshape(-1, 3) - vr).max() < 1e-8
                if depth > 1:
                    assert f"coverage_d{depth} runtime_error receptive-field error" in log
    desc = _load(d, "desc_582").reshape(582, -1)
    x, t, m, v, box = O.ref_synthetic(582)
    off, nbr, dr = O.ref_build_input(x, t, box, 0.6)
    model = O.RefModel(O.ref_model_json(0, 1))
    assert np.abs(desc - O.ref_descriptors(model, x, t, off, nbr, dr)).max() < 1e-12
    sw = _load(d, "switch").reshape(-1, 2)
    for (r_, (sv, sd)) in zip((0.1, 0.54, 0.55, 0.57, 0.59, 0.6, 0.7), sw):
        assert sv == O.ref().ref_switch_value(r_, 0.6)
        assert sd == O.ref().ref_switch_derivative(r_, 0.6)
    assert "mismatch invalid_argument positions/types/global_index size mismatch" in log
    assert "badnbr invalid_argument NnInput edge neighbor out of range" in log
    assert "halfbox invalid_argument rc+skin exceeds half the box length on axis 0" in log
