"""Halo-exchange domain decomposition (hmdp_gdd_* halo mode, dd.HaloDD): ranks own
disjoint regions, integrate only their own atoms and exchange exactly the halo with
point-to-point rounds (POS with migration, P^l, dE/dh partial sums, partial forces,
(E, W, W9)).  Ranks are simulated as contexts on cuda:0 (the in-process hub: one
host thread per rank, the same C++ step program the NCCL transport runs), and as
two real processes with a gloo callback transport.  Checked against the
single-domain evaluation and the single-GPU device MD loop.
The paper's gather-to-root strategy (strategy="gather": owned atoms to rank 0, one
single-domain evaluation, forces back to the owners) runs on the same engine and
transports and is held to the same checks."""
import numpy as np
import pytest

import paper_2602_02234_b200 as P
from conftest import E_TOL, F_TOL, rms
from paper_2602_02234_b200 import dd

pytestmark = pytest.mark.gpu


def _engines(m, s, dims, prec, masses=None, strategy="halo"):
    world = dims[0] * dims[1] * dims[2]
    hub = dd.Hub(world)
    engs = [dd.HaloDD(P.Context(m, max_atoms=s.n_atoms), s.n_atoms, s.types, s.box, dims, r, prec,
                      masses=masses, strategy=strategy) for r in range(world)]
    for e in engs:
        e.attach_hub(hub.handle)
        e.load(s.positions, s.velocities if masses is not None else None)
    return hub, engs


def _assemble(engs, n):
    F = np.full((n, 3), np.nan)
    owned = np.zeros(n, dtype=int)
    for e in engs:
        own, f = e.owned_forces()
        F[own] = f[own]
        owned += own
    return F, owned


@pytest.mark.parametrize("mname", ["dpa2", "dpa3"])
@pytest.mark.parametrize("dims", [(2, 1, 1), (2, 2, 1), (2, 2, 2)])
def test_halo_dd_matches_single_domain(mname, dims, golden_models):
    s = P.generate_synthetic_system(1231)
    m = P.model_from_json(golden_models[mname])
    ref = P.Context(m).compute(s.positions, s.types, s.box, P.Precision.fp64)
    hub, engs = _engines(m, s, dims, P.Precision.fp64)
    dd.run_hub(engs, "eval")
    F, owned = _assemble(engs, s.n_atoms)
    assert np.all(owned == 1)  # every atom owned by exactly one rank
    for e in engs:  # every rank ends with the same totals (rank-ordered sum)
        E, W, W9 = e.energy_virial()
        assert E == pytest.approx(ref.energy, rel=1e-12)
        assert np.abs(W9 - ref.virial_tensor).max() < 1e-9 * max(1.0, np.abs(W9).max())
    assert np.abs(F - ref.forces).max() < 1e-10 * np.abs(ref.forces).max()
    st = engs[0].halo_stats()
    assert st["peers"] == len(engs) - 1 and st["halo_bytes_per_step"] > 0
    assert st["rounds_per_step"] == 2 + 2 * (m.depth() - 1) + 1
    hub.close()


def test_halo_dd_fp32_within_tolerance(golden_models):
    s = P.generate_synthetic_system(2643)
    m = P.model_from_json(golden_models["dpa3"])
    ref = P.Context(m).compute(s.positions, s.types, s.box, P.Precision.fp64)
    hub, engs = _engines(m, s, (2, 2, 1), P.Precision.fp32)
    dd.run_hub(engs, "eval")
    F, owned = _assemble(engs, s.n_atoms)
    E = engs[0].energy_virial()[0]
    assert abs(E - ref.energy) <= E_TOL * abs(ref.energy)
    assert np.abs(F - ref.forces).max() <= F_TOL * rms(ref.forces)
    hub.close()


@pytest.mark.parametrize("dims", [(1, 1, 1), (2, 1, 1)])
def test_halo_dd_fp32_2ptc_kernel_shapes(dims, golden_models):
    """2PTC in FP32: one rank takes the 28-warp-CTA owned-list kernels (2 atom rounds
    instead of 3), two ranks the 20-warp ones; both within the north-star tolerances."""
    s = P.generate_synthetic_system(4114)
    m = P.model_from_json(golden_models["dpa3"])
    ref = P.Context(m).compute(s.positions, s.types, s.box, P.Precision.fp64)
    hub, engs = _engines(m, s, dims, P.Precision.fp32)
    dd.run_hub(engs, "eval")
    F, owned = _assemble(engs, s.n_atoms)
    assert np.all(owned == 1)
    E = engs[0].energy_virial()[0]
    assert abs(E - ref.energy) <= E_TOL * abs(ref.energy)
    assert np.abs(F - ref.forces).max() <= F_TOL * rms(ref.forces)
    hub.close()


@pytest.mark.parametrize("mname", ["dpa2", "dpa3"])
def test_halo_dd_md_matches_device_md(mname, golden_models):
    """60 MD steps, each rank integrating only its own atoms (atoms migrate between
    regions on the way), equal the single-GPU device MD loop in FP64."""
    from paper_2602_02234_b200.md import DeviceMD

    s = P.generate_synthetic_system(1231, temperature=300.0)
    m = P.model_from_json(golden_models[mname])
    md = DeviceMD(P.Context(m), s.positions, s.velocities, s.masses, s.types, s.box,
                  precision=P.Precision.fp64, steps_per_graph=1)
    md.run(60)
    x_ref, v_ref, f_ref, e_ref = md.state()
    hub, engs = _engines(m, s, (2, 2, 1), P.Precision.fp64, masses=s.masses)
    dd.run_hub(engs, "eval")
    dd.run_hub(engs, "open", 0.001)
    own0 = engs[0].roles() == 1
    dd.run_hub(engs, "md", 0.001, steps=60)
    x = np.full((s.n_atoms, 3), np.nan)
    v = np.full((s.n_atoms, 3), np.nan)
    owned = np.zeros(s.n_atoms, dtype=int)
    for e in engs:
        own = e.roles() == 1
        x[own] = e.pos.cpu().numpy()[own]
        v[own] = e.vel.cpu().numpy()[own]
        owned += own
    assert np.all(owned == 1)
    assert (engs[0].roles() == 1).sum() != own0.sum() or not np.array_equal(
        engs[0].roles() == 1, own0)  # ownership changed: atoms migrated
    # the engines hold the next step's drifted positions: x(t + dt) = x(t) + dt v(t + dt/2)
    assert np.abs(x - 0.001 * v - x_ref).max() < 1e-10
    assert engs[0].energy_virial()[0] == pytest.approx(e_ref, rel=1e-11)
    hub.close()


_PUSH_FORM = r"""
import json, sys
import numpy as np
import paper_2602_02234_b200 as P
from paper_2602_02234_b200 import dd
m = P.model_from_json(json.load(open(sys.argv[1]))[sys.argv[2]])
s = P.generate_synthetic_system(1231)
ref = P.Context(m).compute(s.positions, s.types, s.box, P.Precision.fp64)
dims = (2, 2, 1)
hub = dd.Hub(4)
engs = [dd.HaloDD(P.Context(m, max_atoms=s.n_atoms), s.n_atoms, s.types, s.box, dims, r,
                  P.Precision.fp64) for r in range(4)]
for e in engs:
    e.attach_hub(hub.handle)
    e.load(s.positions)
dd.run_hub(engs, "eval")
F = np.full((s.n_atoms, 3), np.nan)
for e in engs:
    own, f = e.owned_forces()
    F[own] = f[own]
print(json.dumps({"dE": abs(engs[0].energy_virial()[0] - ref.energy) / abs(ref.energy),
                  "dF": float(np.abs(F - ref.forces).max() / np.abs(ref.forces).max())}))
hub.close()
"""


@pytest.mark.parametrize("mname", ["dpa2", "dpa3"])
def test_halo_dd_push_form_matches_single_domain(mname, tmp_path):
    """The halo engine's push-form network (HMDP_DD_PULL=0: receivers push per-edge
    adjoint rows, halo sums gathered from them) stays equal to the single domain
    beside the default pull form (senders pull the owned receivers' v rows)."""
    import json
    import os
    import subprocess
    import sys

    from conftest import GOLDEN

    script = tmp_path / "push_form.py"
    script.write_text(_PUSH_FORM)
    env = dict(os.environ, HMDP_DD_PULL="0")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env["PYTHONPATH"] = root + os.pathsep + env.get("PYTHONPATH", "")
    out = subprocess.run([sys.executable, str(script), os.path.join(GOLDEN, "models.json"), mname],
                         env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert r["dE"] < 1e-12 and r["dF"] < 1e-10


def _gloo_worker(rank, world, port, model_json, q):
    import os

    import torch
    import torch.distributed as tdist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s = P.generate_synthetic_system(1231, temperature=300.0)
        m = P.model_from_json(model_json)
        eng = dd.HaloDD(P.Context(m, max_atoms=1231), 1231, s.types, s.box, (2, 1, 1), rank,
                        P.Precision.fp64, masses=s.masses)
        dd.gloo_exchange(eng)
        eng.load(s.positions, s.velocities)
        eng.step("eval")
        E = eng.energy_virial()[0]
        own, F = eng.owned_forces()
        eng.step("open", 0.001)
        for _ in range(3):
            eng.step("md", 0.001)
        torch.cuda.synchronize()
        ownx = eng.roles() == 1
        q.put((rank, E, own, F, ownx, eng.pos.cpu().numpy()))
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("mname", ["dpa2", "dpa3"])
def test_halo_dd_two_processes_gloo(mname, golden_models):
    """Two processes (torch.distributed gloo as the caller transport) run the same C++
    step program and equal the single-domain evaluation and the hub's MD."""
    import socket

    import torch.multiprocessing as mp

    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, golden_models[mname], q))
             for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=300) for _ in procs), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    s = P.generate_synthetic_system(1231, temperature=300.0)
    m = P.model_from_json(golden_models[mname])
    ref = P.Context(m).compute(s.positions, s.types, s.box, P.Precision.fp64)
    F = np.full((1231, 3), np.nan)
    for rank, E, own, f, ownx, x in res:
        assert E == pytest.approx(ref.energy, rel=1e-12)
        F[own] = f[own]
    assert np.abs(F - ref.forces).max() < 1e-10 * np.abs(ref.forces).max()
    hub, engs = _engines(m, s, (2, 1, 1), P.Precision.fp64, masses=s.masses)
    dd.run_hub(engs, "eval")
    dd.run_hub(engs, "open", 0.001)
    dd.run_hub(engs, "md", 0.001, steps=3)
    for (rank, E, own, f, ownx, x), e in zip(res, engs):
        assert np.array_equal(ownx, e.roles() == 1)
        assert np.array_equal(x[ownx], e.pos.cpu().numpy()[ownx])  # bitwise: same program
    hub.close()


@pytest.mark.parametrize("mname", ["dpa2", "dpa3"])
@pytest.mark.parametrize("dims", [(2, 1, 1), (2, 2, 1), (2, 2, 2)])
def test_gather_to_root_matches_single_domain(mname, dims, golden_models):
    """SPEC.md:505 gather_to_root: forces and (E, W) equal the single-domain result
    (FP64), every atom owned by exactly one rank, 4 rounds per step."""
    s = P.generate_synthetic_system(1231)
    m = P.model_from_json(golden_models[mname])
    ref = P.Context(m).compute(s.positions, s.types, s.box, P.Precision.fp64)
    hub, engs = _engines(m, s, dims, P.Precision.fp64, strategy="gather")
    dd.run_hub(engs, "eval")
    F, owned = _assemble(engs, s.n_atoms)
    assert np.all(owned == 1)
    for e in engs:
        E, W, W9 = e.energy_virial()
        assert E == pytest.approx(ref.energy, rel=1e-12)
        assert np.abs(W9 - ref.virial_tensor).max() < 1e-9 * max(1.0, np.abs(W9).max())
    assert np.abs(F - ref.forces).max() < 1e-10 * np.abs(ref.forces).max()
    st = [e.halo_stats() for e in engs]
    assert all(x["rounds_per_step"] == 4 for x in st)
    # the root receives (and answers) every other rank's atoms: its rows are their sum
    ov = 128 * (len(engs) - 1)
    assert st[0]["halo_bytes_per_step"] - ov == sum(x["halo_bytes_per_step"] - ov for x in st[1:])
    hub.close()


def test_gather_to_root_md_matches_halo_exchange(golden_models):
    """20 MD steps with migration: gather-to-root and halo exchange give the same
    owned positions (FP64) and energies as the single-GPU device MD loop."""
    from paper_2602_02234_b200.md import DeviceMD

    s = P.generate_synthetic_system(1231, temperature=300.0)
    m = P.model_from_json(golden_models["dpa3"])
    md = DeviceMD(P.Context(m), s.positions, s.velocities, s.masses, s.types, s.box,
                  precision=P.Precision.fp64, steps_per_graph=1)
    md.run(20)
    x_ref, v_ref, f_ref, e_ref = md.state()
    hub, engs = _engines(m, s, (2, 2, 1), P.Precision.fp64, masses=s.masses, strategy="gather")
    dd.run_hub(engs, "eval")
    dd.run_hub(engs, "open", 0.001)
    dd.run_hub(engs, "md", 0.001, steps=20)
    x = np.full((s.n_atoms, 3), np.nan)
    v = np.full((s.n_atoms, 3), np.nan)
    owned = np.zeros(s.n_atoms, dtype=int)
    for e in engs:
        own = e.roles() == 1
        x[own] = e.pos.cpu().numpy()[own]
        v[own] = e.vel.cpu().numpy()[own]
        owned += own
    assert np.all(owned == 1)
    assert np.abs(x - 0.001 * v - x_ref).max() < 1e-10
    assert engs[1].energy_virial()[0] == pytest.approx(e_ref, rel=1e-11)
    hub.close()


def test_gather_to_root_fp32_within_tolerance(golden_models):
    s = P.generate_synthetic_system(2643)
    m = P.model_from_json(golden_models["dpa3"])
    ref = P.Context(m).compute(s.positions, s.types, s.box, P.Precision.fp64)
    hub, engs = _engines(m, s, (2, 1, 1), P.Precision.fp32, strategy="gather")
    dd.run_hub(engs, "eval")
    F, owned = _assemble(engs, s.n_atoms)
    E = engs[1].energy_virial()[0]
    assert abs(E - ref.energy) <= E_TOL * abs(ref.energy)
    assert np.abs(F - ref.forces).max() <= F_TOL * rms(ref.forces)
    hub.close()
