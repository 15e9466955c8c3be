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
