"""Device MD loop (velocity Verlet, integrators.cpp:32-47, fused into the force
kernel and captured as CUDA graphs) against a host velocity-Verlet loop driven by
the oracle, plus graph-chunking invariance and energy conservation."""
import json

import numpy as np
import pytest

import oracle as O
import paper_2602_02234_b200 as P
from paper_2602_02234_b200.md import DeviceMD

pytestmark = pytest.mark.gpu


def host_md(model_dict, s, steps, dt=0.001, prec="fp64"):
    x, v = s.positions.copy(), s.velocities.copy()
    half = 0.5 * dt
    f = O.evaluate(model_dict, s.types, *O.neighbors(x, s.box, 0.6), prec=prec)["forces"]
    e = None
    for _ in range(steps):
        v += f * (half / s.masses[:, None])
        x += v * dt
        r = O.evaluate(model_dict, s.types, *O.neighbors(x, s.box, 0.6), prec=prec)
        f, e = r["forces"], r["energy"]
        v += f * (half / s.masses[:, None])
    return x, v, f, e


@pytest.mark.parametrize("mname", ["dpa2", "dpa3"])
def test_device_md_matches_host_md_fp64(mname, golden_models):
    s = P.generate_synthetic_system(582)
    m = P.model_from_json(golden_models[mname])
    ctx = P.Context(m)
    md = DeviceMD(ctx, s.positions, s.velocities, s.masses, s.types, s.box,
                  precision=P.Precision.fp64, steps_per_graph=4)
    md.run(10)
    x, v, f, e = md.state()
    hx, hv, hf, he = host_md(json.loads(golden_models[mname]), s, 10)
    assert np.abs(x - hx).max() < 1e-10
    assert np.abs(v - hv).max() < 1e-8
    assert np.abs(f - hf).max() < 1e-7 * max(1.0, np.abs(hf).max())
    assert e == pytest.approx(he, rel=1e-11)


def test_device_md_fp32_tracks_reference(golden_models):
    s = P.generate_synthetic_system(582)
    m = P.model_from_json(golden_models["dpa3"])
    md = DeviceMD(P.Context(m), s.positions, s.velocities, s.masses, s.types, s.box,
                  precision=P.Precision.fp32, steps_per_graph=5)
    md.run(10)
    x, v, f, e = md.state()
    hx, hv, hf, he = host_md(json.loads(golden_models["dpa3"]), s, 10)
    assert np.abs(x - hx).max() < 1e-8
    assert e == pytest.approx(he, rel=1e-5)


def test_graph_chunking_is_bitwise_invariant(golden_models):
    s = P.generate_synthetic_system(582)
    m = P.model_from_json(golden_models["dpa3"])
    ctx = P.Context(m)
    a = DeviceMD(ctx, s.positions, s.velocities, s.masses, s.types, s.box, steps_per_graph=1)
    for _ in range(12):
        a.run(1)
    xa, va, fa, ea = a.state()
    b = DeviceMD(ctx, s.positions, s.velocities, s.masses, s.types, s.box, steps_per_graph=5)
    b.run(12)
    xb, vb, fb, eb = b.state()
    assert np.array_equal(xa, xb) and np.array_equal(va, vb) and np.array_equal(fa, fb)
    assert ea == eb


def test_energy_conservation_nve(golden_models):
    s = P.generate_synthetic_system(582)
    m = P.model_from_json(golden_models["dpa2"])
    md = DeviceMD(P.Context(m), s.positions, s.velocities, s.masses, s.types, s.box,
                  precision=P.Precision.fp64, steps_per_graph=50)

    def total():
        x, v, f, e = md.state()
        return e + 0.5 * np.sum(s.masses[:, None] * v * v)

    e0 = total()
    md.run(200)
    e1 = total()
    assert abs(e1 - e0) <= 1e-3 * abs(e0)


def test_md_after_host_compute_keeps_cells_consistent(golden_models):
    """Interleaving host-path calls and graph replays on one context."""
    s = P.generate_synthetic_system(582)
    m = P.model_from_json(golden_models["dpa2"])
    ctx = P.Context(m)
    md = DeviceMD(ctx, s.positions, s.velocities, s.masses, s.types, s.box,
                  precision=P.Precision.fp64, steps_per_graph=2)
    md.run(2)
    P.build_input_periodic(s.positions, s.types, np.arange(582), s.box, 0.6)
    ctx.compute(s.positions, s.types, s.box)
    md.run(2)
    x, v, f, e = md.state()
    hx, *_ = host_md(json.loads(golden_models["dpa2"]), s, 4)
    assert np.abs(x - hx).max() < 1e-10


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_caller_velocity_verlet_matches_device_md(prec, golden_models):
    """bench.py's e2e leg: the reference's velocity_verlet_step in C++ over host
    buffers with hmdp_compute as the force function (csrc/hmdp_caller_md.cpp)
    follows the same trajectory as the fused device MD loop."""
    import ctypes
    import os

    from paper_2602_02234_b200._lib import LIB_PATH, check, ptr

    caller = ctypes.CDLL(os.path.join(os.path.dirname(LIB_PATH), "libhmdp_caller.so"))
    s = P.generate_synthetic_system(582)
    m = P.model_from_json(golden_models["dpa3"])
    pr = P.Precision[prec]
    md = DeviceMD(P.Context(m), s.positions, s.velocities, s.masses, s.types, s.box,
                  precision=pr, steps_per_graph=4)
    md.run(8)
    dx, dv, df, de = md.state()
    ctx = P.Context(m, max_atoms=582)
    x = s.positions.copy()
    v = s.velocities.copy()
    t = s.types.astype(np.int32)
    mass = np.ascontiguousarray(s.masses, dtype=np.float64)
    box = np.ascontiguousarray(s.box, dtype=np.float64)
    f = np.ascontiguousarray(ctx.compute(x, t, box, pr).forces).copy()
    e = ctypes.c_double()
    check(caller.hmdp_caller_velocity_verlet(ctx.handle, ctypes.c_int(582), ptr(x), ptr(v), ptr(f),
                                             ptr(t), ptr(box), ptr(mass), ctypes.c_double(0.001),
                                             ctypes.c_int(8), ctypes.c_int(int(pr)),
                                             ctypes.byref(e)))
    tol = 1e-12 if prec == "fp64" else 1e-9
    assert np.abs(x - dx).max() < tol
    assert np.abs(v - dv).max() < 1e3 * tol
    assert e.value == pytest.approx(de, rel=1e-12 if prec == "fp64" else 1e-6)


def test_cached_compute_graph_after_other_binning(golden_models):
    """hmdp_compute's cached graph carries no cell-count memset (the network clears
    the counts after the search); operations that leave binned cells behind (an MD
    chunk, a neighbour-list build) must be followed by a clear before the replay."""
    s = P.generate_synthetic_system(582)
    m = P.model_from_json(golden_models["dpa3"])
    ref = P.Context(m).compute(s.positions, s.types, s.box, P.Precision.fp32)
    ctx = P.Context(m)
    for _ in range(3):  # direct path, capture, replay
        out = ctx.compute(s.positions, s.types, s.box, P.Precision.fp32)
        assert np.array_equal(out.forces, ref.forces)
    md = DeviceMD(ctx, s.positions, s.velocities, s.masses, s.types, s.box,
                  precision=P.Precision.fp32, steps_per_graph=2)
    for _ in range(2):  # the first round may reallocate (graph re-captured), the second
        md.run(4)       # replays the cached graph over the MD loop's binned cells
        for _ in range(2):
            out = ctx.compute(s.positions, s.types, s.box, P.Precision.fp32)
            assert np.array_equal(out.forces, ref.forces) and out.energy == ref.energy
    # a neighbour-list build on the same context bins without a network
    import ctypes

    from paper_2602_02234_b200._lib import check, lib, ptr

    x = np.ascontiguousarray(s.positions)
    box = np.ascontiguousarray(s.box, dtype=np.float64)
    off = np.zeros(583, dtype=np.int32)
    nbr = np.zeros(40000, dtype=np.int32)
    dr = np.zeros((40000, 3))
    ne = ctypes.c_int()
    for _ in range(2):
        check(lib().hmdp_build_neighbors(ctx.handle, 582, ptr(x), ptr(box), 0.6, 40000,
                                         ptr(off), ptr(nbr), ptr(dr), ctypes.byref(ne)))
        assert 0 < ne.value <= 40000
        for _ in range(2):
            out = ctx.compute(s.positions, s.types, s.box, P.Precision.fp32)
            assert np.array_equal(out.forces, ref.forces) and out.energy == ref.energy
