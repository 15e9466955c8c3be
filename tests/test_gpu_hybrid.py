"""NNPot hybrid coupling on the GPU (hmdp_compute_group): the
provider equals the model on the extracted group, scatters only into group
atoms, conserves momentum, and a zero model leaves the classical forces alone."""
import json

import numpy as np
import pytest

import paper_2602_02234_b200 as P
from paper_2602_02234_b200.hybrid import (nn_force_provider, plan_group_preprocessing,
                                          synthetic_topology)

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mname", ["dpa2", "dpa3"])
@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_group_provider_equals_extracted_group(mname, prec, golden_models):
    s = P.generate_synthetic_system(582)
    topo = synthetic_topology(582)
    _, plan = plan_group_preprocessing(topo, "protein")
    m = P.model_from_json(golden_models[mname])
    ctx = P.Context(m)
    rng = np.random.default_rng(3)
    classical = rng.normal(size=(582, 3))  # stands in for the classical forces
    f = classical.copy()
    e = nn_force_provider(ctx, s.positions, s.types, s.box, plan, f, P.Precision[prec])
    g = plan.atoms
    ref = ctx.compute(s.positions[g], s.types[g], s.box, P.Precision[prec])
    assert e == ref.energy
    assert np.array_equal(f[g], classical[g] + ref.forces)
    other = np.setdiff1d(np.arange(582), g)
    assert np.array_equal(f[other], classical[other])
    if prec == "fp64":  # translation invariance of the model: sum of NN forces ~ 0
        assert np.abs((f[g] - classical[g]).sum(axis=0)).max() < 1e-8 * np.abs(ref.forces).max()


def test_zero_model_leaves_classical_forces(golden_models):
    md = json.loads(golden_models["dpa3"])
    for net in [md["embedding"], md["fitting"]] + [x for l in md["layers"] for x in l.values()]:
        net["weights"] = [[0.0] * len(w) for w in net["weights"]]
        net["biases"] = [[0.0] * len(b) for b in net["biases"]]
    m = P.model_from_json(json.dumps(md))
    s = P.generate_synthetic_system(582)
    _, plan = plan_group_preprocessing(synthetic_topology(582), "protein")
    f = np.ones((582, 3))
    e = nn_force_provider(P.Context(m), s.positions, s.types, s.box, plan, f, P.Precision.fp64)
    assert e == 0.0 and np.array_equal(f, np.ones((582, 3)))


def test_group_errors(golden_models):
    s = P.generate_synthetic_system(64)
    ctx = P.Context(P.model_from_json(golden_models["dpa2"]))
    _, plan = plan_group_preprocessing(synthetic_topology(64), "protein")
    plan.atoms = plan.atoms[::-1].copy()
    with pytest.raises(ValueError, match="sorted"):
        nn_force_provider(ctx, s.positions, s.types, s.box, plan, np.zeros((64, 3)))
