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
    for step in range(5):
        l0 = engs[0].launches()
        run_local(engs, "md", 0.001)
        # roles/bin/search/rev/zero, embed, (push, fwd) x2, (sums, bwd) x2, force, integrate
        assert engs[0].launches() - l0 == 16
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


def _dist_worker(rank, world, port, model_json, q):
    """One rank of a real torch.distributed job (gloo: NCCL refuses two ranks on
    one GPU, and the pool has one) running run_dist, the program bench.py captures."""
    import os
    import sys

    import torch
    import torch.distributed as tdist

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.dirname(here))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2602_02234_b200 as PP
        from paper_2602_02234_b200.dd import DeviceDD, run_dist

        s = PP.generate_synthetic_system(1231, temperature=300.0)
        m = PP.model_from_json(model_json)
        eng = DeviceDD(PP.Context(m, max_atoms=1231), 1231, s.types, s.box, (world, 1, 1), rank,
                       PP.Precision.fp64, masses=s.masses)
        eng.load(s.positions, s.velocities)
        run_dist(eng, "eval")
        torch.cuda.synchronize()
        E, F, W, W9 = eng.result()
        run_dist(eng, "open", 0.001)
        for _ in range(3):
            run_dist(eng, "md", 0.001)
        torch.cuda.synchronize()
        q.put((rank, E, F, W9, eng.pos.cpu().numpy(), eng.vel.cpu().numpy()))
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("mname", ["dpa2", "dpa3"])
def test_device_dd_two_processes_match_single_domain(mname, golden_models):
    """run_dist in two processes (torch.distributed, gloo over the GPU tensors)
    equals the single-domain evaluation and the in-process simulated ranks' MD."""
    import socket

    import torch.multiprocessing as mp

    from paper_2602_02234_b200.dd import DeviceDD, run_local

    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_dist_worker, args=(r, 2, port, golden_models[mname], q))
             for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    s = P.generate_synthetic_system(1231, temperature=300.0)
    m = P.model_from_json(golden_models[mname])
    ref = P.Context(m).compute(s.positions, s.types, s.box, P.Precision.fp64)
    engs = [DeviceDD(P.Context(m, max_atoms=1231), 1231, s.types, s.box, (2, 1, 1), r,
                     P.Precision.fp64, masses=s.masses) for r in range(2)]
    for e in engs:
        e.load(s.positions, s.velocities)
    run_local(engs, "eval")
    run_local(engs, "open", 0.001)
    for _ in range(3):
        run_local(engs, "md", 0.001)
    x_loc = engs[0].pos.cpu().numpy()
    for rank, E, F, W9, x, v in res:
        assert E == pytest.approx(ref.energy, rel=1e-12)
        assert np.abs(F - ref.forces).max() < 1e-10 * np.abs(ref.forces).max()
        assert np.abs(W9 - ref.virial_tensor).max() < 1e-9 * max(1.0, np.abs(W9).max())
        assert np.abs(x - x_loc).max() < 1e-12
    assert np.array_equal(res[0][4], res[1][4])  # replicated positions agree bitwise
