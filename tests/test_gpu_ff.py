"""Classical force field on the device (hmdp_ff_*) against the reference's own
compute_classical compiled from its sources (oracle/_ref, forcefield.cpp:265-279) on
the synthetic protein-in-water topology."""
import numpy as np
import pytest

import oracle as O
import paper_2602_02234_b200 as P
from paper_2602_02234_b200.ff import ClassicalFF

pytestmark = pytest.mark.gpu


def _ff(n, scheme, rc=0.7):
    t = O.ref_synthetic_topology(n)
    s = P.generate_synthetic_system(n)
    ff = ClassicalFF(s.types, t["charges"], O.LJ_SIGMA, O.LJ_EPS, t["excl_offset"], t["excl"],
                     t["bonds"], t["bond_params"], t["angles"], t["angle_params"], t["dihedrals"],
                     t["dihedral_params"], coulomb_scheme=scheme, rc_coulomb=rc, rc_lj=rc)
    return s, ff


@pytest.mark.parametrize("n", [582, 1231])
@pytest.mark.parametrize("scheme", [0, 1])
def test_classical_matches_reference_fp64(n, scheme):
    s, ff = _ff(n, scheme)
    rng = np.random.default_rng(2)
    x = s.positions + rng.normal(scale=0.01, size=s.positions.shape)
    ref = O.ref_classical(x, n, scheme=scheme)
    out = ff.compute(x, s.box, P.Precision.fp64)
    e = np.array([out.bonded, out.lj, out.coulomb])
    assert np.abs(e - ref["energies"]).max() <= 1e-10 * max(1.0, np.abs(ref["energies"]).max())
    scale = np.abs(ref["forces"]).max()
    assert np.abs(out.forces - ref["forces"]).max() <= 1e-10 * scale
    assert out.virial == pytest.approx(ref["virial"], rel=1e-10, abs=1e-8)
    assert out.collinear_angles == ref["collinear"]


def test_classical_fp32_within_tolerance():
    """FP32 arithmetic (the reference's Precision::fp32) against the FP64 answer:
    within 1e-3 of the RMS force (the stiff bonded terms dominate; the reference's
    own FP32 path is at 2e-4, ours at 4.6e-4 — different summation orders)."""
    s, ff = _ff(582, 1)
    ref64 = O.ref_classical(s.positions, 582, scheme=1, fp64=True)
    ref32 = O.ref_classical(s.positions, 582, scheme=1, fp64=False)
    out = ff.compute(s.positions, s.box, P.Precision.fp32)
    rms = float(np.sqrt(np.mean(np.sum(ref64["forces"] ** 2, axis=1))))
    ours = np.abs(out.forces - ref64["forces"]).max()
    theirs = np.abs(ref32["forces"] - ref64["forces"]).max()
    assert ours <= 1e-3 * rms and theirs <= 1e-3 * rms, (ours, theirs)
    tot, rt = out.total_potential(), float(ref64["energies"].sum())
    assert abs(tot - rt) <= 1e-5 * np.abs(ref64["energies"]).sum()


def test_classical_deterministic_and_overlap_error():
    s, ff = _ff(582, 0)
    a = ff.compute(s.positions, s.box)
    b = ff.compute(s.positions, s.box)
    assert np.array_equal(a.forces, b.forces) and a.lj == b.lj
    x = s.positions.copy()
    x[10] = x[300]  # two (non-excluded) atoms on top of each other
    with pytest.raises(RuntimeError, match="overlap"):
        ff.compute(x, s.box)


def test_classical_plus_dp_hybrid_step_on_device():
    """Hybrid force = classical (preprocessed topology) + DP on the protein group:
    the two device providers compose like the reference drop-in test."""
    from paper_2602_02234_b200.hybrid import nn_force_provider, plan_group_preprocessing, synthetic_topology

    n = 582
    s, _ = _ff(n, 0)
    t = O.ref_synthetic_topology(n)
    topo2, plan = plan_group_preprocessing(synthetic_topology(n), "protein")
    eo = np.zeros(n + 1, dtype=np.int32)
    ex = []
    for i in range(n):
        ex += topo2.exclusions[i]
        eo[i + 1] = len(ex)
    keep_b = [k for k, b in enumerate(map(tuple, t["bonds"])) if b in set(map(tuple, topo2.bonds))]
    ff2 = ClassicalFF(s.types, t["charges"], O.LJ_SIGMA, O.LJ_EPS, eo, np.array(ex), t["bonds"][keep_b],
                      t["bond_params"][keep_b], coulomb_scheme=0)
    cl = ff2.compute(s.positions, s.box)
    m = P.make_model(P.ModelFamily.message_passing, 3, 0.6, 2, 8, 32, 1)
    f = cl.forces.copy()
    e_nn = nn_force_provider(P.Context(m), s.positions, s.types, s.box, plan, f, P.Precision.fp64)
    assert np.isfinite(e_nn) and np.all(np.isfinite(f))
    assert np.abs(f.sum(axis=0)).max() < 1e-8 * np.abs(f).max()  # momentum conservation


def test_hybrid_device_md_matches_host_loop():
    """Device hybrid MD (classical on all atoms + DP on the protein group, graph
    captured) equals a host velocity-Verlet loop over the two device providers."""
    from paper_2602_02234_b200.ff import HybridMD
    from paper_2602_02234_b200.hybrid import NnGroupPlan

    n = 582
    s, ff = _ff(n, 1)
    s = P.generate_synthetic_system(n, temperature=300.0)
    m = P.make_model(P.ModelFamily.message_passing, 3, 0.6, 2, 8, 32, 1)
    grp = np.arange(204, dtype=np.int32)  # the synthetic "protein" group
    md = HybridMD(P.Context(m), ff, grp, s.positions, s.velocities, s.masses, s.types, s.box,
                  dt_ps=0.0005, precision=P.Precision.fp64, steps_per_graph=2)
    md.run(4)
    xd, vd, fd, ed = md.state()
    ctx = P.Context(m)
    inv = (0.5 * 0.0005 / s.masses)[:, None]

    def forces(x):
        f = ff.compute(x, s.box, P.Precision.fp64).forces.copy()
        nn = ctx.compute(x[grp], s.types[grp], s.box, P.Precision.fp64)
        f[grp] += nn.forces
        return f

    x, v = s.positions.copy(), s.velocities.copy()
    f = forces(x)
    v += f * inv
    x += v * 0.0005
    for _ in range(4):
        f = forces(x)
        v += f * inv
        v += f * inv
        x += v * 0.0005
    assert np.abs(xd - x).max() < 1e-9
    assert np.abs(vd - v).max() < 1e-6
    assert np.all(np.isfinite(ed))
