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
