"""Domain-decomposed evaluation on the GPU phase entry points (hmdp_dd_*):
several ranks simulated in one process on cuda:0, halo rows exchanged in memory,
checked against the single-domain oracle."""
import json

import numpy as np
import pytest

import oracle as O
import paper_2602_02234_b200 as P
from conftest import E_TOL, F_TOL, load_golden, rms
from paper_2602_02234_b200 import dd

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n_ranks", [1, 2, 4, 8])
@pytest.mark.parametrize("name", ["dpa2", "dpa3"])
@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_gpu_dd_equals_single_domain(n_ranks, name, prec, golden_models):
    g = load_golden("1YRF")
    md = json.loads(golden_models[name])
    ref = O.evaluate(md, g["types"], g["edge_offset"], g["edge_neighbor"], g["edge_dr"])
    own = dd.owners(g["positions"], g["box"], dd.rank_grid(n_ranks))
    plans = dd.make_plans(g["edge_offset"], g["edge_neighbor"], g["edge_dr"], g["types"], own,
                          n_ranks)
    model = P.model_from_json(golden_models[name])
    engines = [dd.GpuEngine(P.Context(model), P.Precision[prec]) for _ in plans]
    E, F, W, W9 = dd.evaluate_local(engines, plans, model.depth())
    Fg = np.zeros_like(ref["forces"])
    for r, p in enumerate(plans):
        Fg[p.owned] = F[r]
    etol, ftol = (1e-11, 1e-10) if prec == "fp64" else (E_TOL, F_TOL)
    assert abs(E - ref["energy"]) <= etol * abs(ref["energy"])
    assert np.abs(Fg - ref["forces"]).max() <= ftol * rms(ref["forces"])
    assert abs(W - ref["virial"]) <= ftol * max(abs(ref["virial"]), rms(ref["forces"]))


# ---------------------------------------------------------------------------
# device-resident DD on the global index space (hmdp_gdd_*), simulated ranks
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("mname", ["dpa2", "dpa3"])
@pytest.mark.parametrize("dims", [(2, 1, 1), (2, 2, 1), (2, 2, 2)])
def test_device_dd_matches_single_domain(mname, dims, golden_models):
    from paper_2602_02234_b200.dd import DeviceDD, run_local

    s = P.generate_synthetic_system(1231)
    m = P.model_from_json(golden_models[mname])
    ref = P.Context(m).compute(s.positions, s.types, s.box, P.Precision.fp64)
    world = dims[0] * dims[1] * dims[2]
    engs = [DeviceDD(P.Context(m, max_atoms=1231), 1231, s.types, s.box, dims, r,
                     P.Precision.fp64) for r in range(world)]
    for e in engs:
        e.load(s.positions)
    run_local(engs)
    owned = sum(e.counts()[0] for e in engs)
    assert owned == 1231
    for e in engs:
        E, F, W, W9 = e.result()
        assert E == pytest.approx(ref.energy, rel=1e-12)
        assert np.abs(F - ref.forces).max() < 1e-10 * np.abs(ref.forces).max()
        assert np.abs(W9 - ref.virial_tensor).max() < 1e-9 * max(1.0, np.abs(W9).max())


def test_device_dd_md_matches_device_md(golden_models):
    from paper_2602_02234_b200.dd import DeviceDD, run_local
    from paper_2602_02234_b200.md import DeviceMD

    s = P.generate_synthetic_system(582, temperature=300.0)
    m = P.model_from_json(golden_models["dpa3"])
    md = DeviceMD(P.Context(m), s.positions, s.velocities, s.masses, s.types, s.box,
                  precision=P.Precision.fp64, steps_per_graph=1)
    md.run(5)
    x_ref, v_ref, f_ref, e_ref = md.state()
    engs = [DeviceDD(P.Context(m, max_atoms=582), 582, s.types, s.box, (2, 1, 1), r,
                     P.Precision.fp64, masses=s.masses) for r in range(2)]
    for e in engs:
        e.load(s.positions, s.velocities)
    run_local(engs, "eval")
    run_local(engs, "open", 0.001)  # the device MD loop's first chunk: opening kick + drift
    for _ in range(5):
        run_local(engs, "md", 0.001)
    x = engs[0].pos.cpu().numpy()
    assert np.abs(x - engs[1].pos.cpu().numpy()).max() == 0.0  # replicated state
    # DeviceMD's state is the completed step (x(t), v(t)); the DD engines hold the
    # next step's drifted positions: x(t + dt) = x(t) + dt v(t + dt/2)
    v_half = engs[0].vel.cpu().numpy()
    assert np.abs(x - 0.001 * v_half - x_ref).max() < 1e-10


def test_device_dd_fp32_within_tolerance(golden_models):
    from paper_2602_02234_b200.dd import DeviceDD, run_local

    s = P.generate_synthetic_system(2643)
    m = P.model_from_json(golden_models["dpa3"])
    ref = P.Context(m).compute(s.positions, s.types, s.box, P.Precision.fp64)
    engs = [DeviceDD(P.Context(m, max_atoms=2643), 2643, s.types, s.box, (2, 2, 1), r,
                     P.Precision.fp32) for r in range(4)]
    for e in engs:
        e.load(s.positions)
    run_local(engs)
    E, F, W, W9 = engs[3].result()
    assert abs(E - ref.energy) <= E_TOL * abs(ref.energy)
    assert np.abs(F - ref.forces).max() <= F_TOL * rms(ref.forces)


def test_device_dd_rejects_deepmd_families_and_bad_grids(golden_models):
    from paper_2602_02234_b200.dd import DeviceDD

    s = P.generate_synthetic_system(582)
    with pytest.raises(ValueError):
        DeviceDD(P.Context(P.make_dp_model(P.ModelFamily.se_a, 1)), 582, s.types, s.box,
                 (2, 1, 1), 0, P.Precision.fp32)
    m = P.model_from_json(golden_models["dpa3"])
    with pytest.raises(ValueError):
        DeviceDD(P.Context(m), 582, s.types, s.box, (2, 1, 1), 2, P.Precision.fp32)
