"""Domain decomposition (paper_2602_02234_b200/dd.py) on CPU: plans, halo maps,
the phase program, the in-process transport and a 2-process gloo run, each
checked against the single-domain oracle ("decomposed ==
single-domain").  The per-rank compute is the float64 NumPy engine
(tests/dd_numpy_engine.py); the CUDA engine is covered in test_gpu_dd.py."""
import json
import os
import sys

import numpy as np
import pytest

import oracle as O
from conftest import load_golden, rms
from paper_2602_02234_b200 import dd

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from dd_numpy_engine import NumpyEngine  # noqa: E402


def single_domain(model_json, g):
    return O.evaluate(json.loads(model_json), g["types"], g["edge_offset"], g["edge_neighbor"],
                      g["edge_dr"])


def plans_for(g, n_ranks):
    own = dd.owners(g["positions"], g["box"], dd.rank_grid(n_ranks))
    return dd.make_plans(g["edge_offset"], g["edge_neighbor"], g["edge_dr"], g["types"], own,
                         n_ranks), own


@pytest.mark.parametrize("n", [1, 2, 3, 4, 6, 8])
def test_rank_grid(n):
    dims = dd.rank_grid(n)
    assert int(np.prod(dims)) == n


@pytest.mark.parametrize("n_ranks", [2, 4, 8])
def test_plans_partition_edges_and_maps(n_ranks, golden_1yrf):
    g = golden_1yrf
    plans, own = plans_for(g, n_ranks)
    n = g["types"].shape[0]
    owned = np.concatenate([p.owned for p in plans])
    assert np.array_equal(np.sort(owned), np.arange(n))  # owned sets partition the atoms
    assert sum(int(p.offset[p.n_own]) for p in plans) == int(g["edge_offset"][-1])
    for r, p in enumerate(plans):
        loc2glob = np.concatenate([p.owned, p.ghosts])
        # every local edge is the global edge (same target, bit-identical dr)
        for li, gi in enumerate(p.owned[:50]):
            a, b = g["edge_offset"][gi], g["edge_offset"][gi + 1]
            la, lb = p.offset[li], p.offset[li + 1]
            assert np.array_equal(loc2glob[p.nbr[la:lb]], g["edge_neighbor"][a:b])
            assert np.array_equal(p.dr[la:lb], g["edge_dr"][a:b])
        assert np.all(own[p.ghosts] != r)
        # halo maps are consistent in both directions
        for q, rows in p.send.items():
            assert np.array_equal(plans[q].ghosts[plans[q].recv[r] - plans[q].n_own], p.owned[rows])


def test_numpy_engine_single_domain_matches_oracle(golden_models, golden_1yrf):
    g = golden_1yrf
    for name in ("dpa2", "dpa3"):
        ref = single_domain(golden_models[name], g)
        plans, _ = plans_for(g, 1)
        eng = NumpyEngine(golden_models[name])
        depth = 1 + len(json.loads(golden_models[name])["layers"])
        E, F, W, W9 = dd.evaluate_local([eng], plans, depth)
        assert E == pytest.approx(ref["energy"], rel=1e-12)
        assert np.abs(F[0] - ref["forces"]).max() < 1e-10 * rms(ref["forces"]) * 100
        assert W == pytest.approx(ref["virial"], rel=1e-10, abs=1e-10)
        assert np.trace(W9) == pytest.approx(W, rel=1e-10)


@pytest.mark.parametrize("n_ranks", [2, 4, 8])
@pytest.mark.parametrize("name", ["dpa2", "dpa3"])
def test_decomposed_equals_single_domain(n_ranks, name, golden_models, golden_1yrf):
    g = golden_1yrf
    ref = single_domain(golden_models[name], g)
    plans, own = plans_for(g, n_ranks)
    engines = [NumpyEngine(golden_models[name]) for _ in plans]
    depth = 1 + len(json.loads(golden_models[name])["layers"])
    E, F, W, W9 = dd.evaluate_local(engines, plans, depth)
    Fg = np.zeros_like(ref["forces"])
    for r, p in enumerate(plans):
        Fg[p.owned] = F[r]
    assert E == pytest.approx(ref["energy"], rel=1e-12)
    assert np.abs(Fg - ref["forces"]).max() <= 1e-10 * rms(ref["forces"])
    assert W == pytest.approx(ref["virial"], rel=1e-10, abs=1e-10)


def test_negative_control_without_layer_exchange(golden_models, golden_1yrf):
    """dropping the per-layer halo exchange (DPA3 with an rc halo
    only) must visibly break boundary forces."""
    g = golden_1yrf
    name = "dpa3"
    ref = single_domain(golden_models[name], g)
    plans, _ = plans_for(g, 2)
    engines = [NumpyEngine(golden_models[name]) for _ in plans]
    for p in plans:  # no halo maps -> ghosts keep P = 0 and never return adjoints
        p.send.clear()
        p.recv.clear()
    E, F, W, W9 = dd.evaluate_local(engines, plans, 3)
    Fg = np.zeros_like(ref["forces"])
    for r, p in enumerate(plans):
        Fg[p.owned] = F[r]
    assert np.abs(Fg - ref["forces"]).max() > 1e-3 * rms(ref["forces"])


def _gloo_worker(rank, world, port, model_json, q):
    import torch.distributed as tdist

    sys.path.insert(0, HERE)
    sys.path.insert(0, os.path.dirname(HERE))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from conftest import load_golden as lg
        from dd_numpy_engine import NumpyEngine as NE
        from paper_2602_02234_b200 import dd as D

        g = lg("1YRF")
        own = D.owners(g["positions"], g["box"], D.rank_grid(world))
        plans = D.make_plans(g["edge_offset"], g["edge_neighbor"], g["edge_dr"], g["types"], own,
                             world)
        depth = 1 + len(json.loads(model_json)["layers"])
        E, F, W, W9 = D.evaluate_dd(NE(model_json), D.TorchDistTransport(), plans, rank, depth)
        q.put((rank, E, W, plans[rank].owned, F))
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("name", ["dpa2", "dpa3"])
def test_gloo_world2_matches_single_domain(name, golden_models, golden_1yrf):
    import socket

    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, golden_models[name], q))
             for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = single_domain(golden_models[name], golden_1yrf)
    Fg = np.zeros_like(ref["forces"])
    for rank, E, W, owned, F in res:
        assert E == pytest.approx(ref["energy"], rel=1e-12)
        assert W == pytest.approx(ref["virial"], rel=1e-10, abs=1e-10)
        Fg[owned] = F
    assert np.abs(Fg - ref["forces"]).max() <= 1e-10 * rms(ref["forces"])
