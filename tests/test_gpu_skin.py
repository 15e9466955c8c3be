"""Device MD loop with a Verlet skin (k_nbr_search_v): every step filters the exact
rc list out of candidate rows within rc + skin that are rebuilt only after some atom
moved more than skin/2.  The list it yields is the full search's (same pairs, order
and FP64 edge_dr, neighborlist.cpp:42-113 / inference.cpp:474-485), so trajectories
must be BITWISE identical to the skin-0 loop that searches every step."""
import numpy as np
import pytest

import paper_2602_02234_b200 as P
from paper_2602_02234_b200.md import DeviceMD

pytestmark = pytest.mark.gpu


def _model(name):
    if name == "dpa2":
        return P.make_model(P.ModelFamily.embed_fit, 1, 0.6, 2, 8, 32, 1)
    if name == "dpa3":
        return P.make_model(P.ModelFamily.message_passing, 3, 0.6, 2, 8, 32, 1)
    if name == "se_a":
        return P.make_dp_model(P.ModelFamily.se_a, 1, 0.6, 0.3, 2, 1)
    return P.make_dp_model(P.ModelFamily.repflow, 2, 0.6, 0.3, 2, 1)


def _run(monkeypatch, m, s, skin, steps, prec, spg=5, dt=0.002):
    monkeypatch.setenv("HMDP_SKIN", str(skin))
    ctx = P.Context(m, max_atoms=s.n_atoms)
    md = DeviceMD(ctx, s.positions, s.velocities, s.masses, s.types, s.box, dt_ps=dt,
                  precision=prec, steps_per_graph=spg)
    md.run(steps)
    out = md.state()
    stats = md.stats()
    md.close()
    return out, stats


def _same(a, b):
    for u, v in zip(a[:3], b[:3]):
        assert np.array_equal(u, v)
    assert a[3] == b[3]


@pytest.mark.parametrize("mname,n", [("dpa3", 582), ("dpa3", 1231), ("dpa3", 4114),
                                     ("dpa2", 582), ("dpa2", 4114)])
@pytest.mark.parametrize("prec", [P.Precision.fp32, P.Precision.fp64])
def test_skin_trajectory_bitwise_equals_full_search(monkeypatch, mname, n, prec):
    s = P.generate_synthetic_system(n)
    m = _model(mname)
    ref, st0 = _run(monkeypatch, m, s, 0.0, 40, prec)
    assert st0 == (0.0, 0)
    for skin in (0.02, 0.1):  # 0.02: a rebuild every few steps; 0.1: the default
        got, st = _run(monkeypatch, m, s, skin, 40, prec)
        assert st[0] == pytest.approx(skin)
        assert st[1] >= 1
        _same(got, ref)
    assert st[1] >= 1
    _, st_small = _run(monkeypatch, m, s, 0.02, 40, prec)
    assert st_small[1] >= 3, st_small  # the small skin really rebuilt mid-run


@pytest.mark.parametrize("mname", ["se_a", "repflow"])
def test_skin_deepmd_families(monkeypatch, mname):
    s = P.generate_synthetic_system(582)
    m = _model(mname)
    ref, _ = _run(monkeypatch, m, s, 0.0, 30, P.Precision.fp32)
    got, st = _run(monkeypatch, m, s, 0.02, 30, P.Precision.fp32)
    assert st[1] >= 2
    _same(got, ref)


def test_skin_chunking_and_interleaving(monkeypatch):
    """Graph chunk size and a foreign hmdp_compute on the same context between
    chunks (it re-bins the shared cell lists) leave the trajectory unchanged."""
    s = P.generate_synthetic_system(1231)
    m = _model("dpa3")
    ref, _ = _run(monkeypatch, m, s, 0.0, 30, P.Precision.fp32, spg=1)
    monkeypatch.setenv("HMDP_SKIN", "0.03")
    ctx = P.Context(m, max_atoms=s.n_atoms)
    md = DeviceMD(ctx, s.positions, s.velocities, s.masses, s.types, s.box, dt_ps=0.002,
                  precision=P.Precision.fp32, steps_per_graph=7)
    other = P.generate_synthetic_system(582)
    for k in (10, 3, 17):
        md.run(k)
        ctx.compute(other.positions, other.types, other.box, P.Precision.fp32)
    got = md.state()
    assert md.stats()[1] >= 2
    md.close()
    _same(got, ref)


def test_skin_disabled_when_box_too_small(monkeypatch):
    s = P.generate_synthetic_system(64)  # rc + skin > L/2: full search every step
    m = _model("dpa3")
    ref, _ = _run(monkeypatch, m, s, 0.0, 10, P.Precision.fp64)
    got, st = _run(monkeypatch, m, s, 0.5, 10, P.Precision.fp64)
    assert st == (0.0, 0)
    _same(got, ref)


def _compute_series(monkeypatch, m, s, skin, prec, calls=25, seed=3):
    """hmdp_compute (the host-buffer call e2e times) over a drifting trajectory with
    two jumps: its CUDA-graph path keeps Verlet rows across calls."""
    monkeypatch.setenv("HMDP_SKIN", str(skin))
    ctx = P.Context(m, max_atoms=s.n_atoms)
    rng = np.random.default_rng(seed)
    x = s.positions.copy()
    outs = []
    for c in range(calls):
        if c in (9, 17):  # teleport a few atoms well past skin/2
            idx = rng.choice(s.n_atoms, 5, replace=False)
            x[idx] += rng.normal(scale=0.2, size=(5, 3))
        else:
            x += rng.normal(scale=0.004, size=x.shape)
        o = ctx.compute(x, s.types, s.box, prec)
        outs.append((o.energy, o.forces.copy(), np.array(o.virial_tensor, copy=True)))
    return outs


@pytest.mark.parametrize("mname,n", [("dpa3", 582), ("dpa3", 4114), ("dpa2", 1231)])
def test_skin_compute_graph_path_bitwise(monkeypatch, mname, n):
    s = P.generate_synthetic_system(n)
    m = _model(mname)
    ref = _compute_series(monkeypatch, m, s, 0.0, P.Precision.fp32)
    got = _compute_series(monkeypatch, m, s, 0.05, P.Precision.fp32)
    for a, b in zip(ref, got):
        assert a[0] == b[0]
        assert np.array_equal(a[1], b[1])
        assert np.array_equal(a[2], b[2])


def test_compute_graph_per_atom_after_forces_only(monkeypatch):
    """The graph path's D2H copy moves the per-atom energies only when the captured call
    asked for them; a later per-atom call re-captures (large box: copy-node outputs)."""
    monkeypatch.setenv("HMDP_SKIN", "0.1")
    s = P.generate_synthetic_system(4114)
    m = _model("dpa3")
    ctx = P.Context(m, max_atoms=s.n_atoms)
    ref = ctx.compute(s.positions, s.types, s.box, P.Precision.fp32, per_atom=True)  # direct
    for _ in range(3):
        o = ctx.compute(s.positions, s.types, s.box, P.Precision.fp32)
        assert o.energy == ref.energy and np.array_equal(o.forces, ref.forces)
    for _ in range(3):
        o = ctx.compute(s.positions, s.types, s.box, P.Precision.fp32, per_atom=True)
        assert np.array_equal(o.per_atom_energy, ref.per_atom_energy)
        assert np.array_equal(o.forces, ref.forces)


@pytest.mark.parametrize("mname,prec", [("dpa2", P.Precision.fp64), ("se_a", P.Precision.fp32),
                                        ("repflow", P.Precision.fp32)])
def test_skin_compute_graph_path_other_families(monkeypatch, mname, prec):
    s = P.generate_synthetic_system(582)
    m = _model(mname)
    ref = _compute_series(monkeypatch, m, s, 0.0, prec, calls=15)
    got = _compute_series(monkeypatch, m, s, 0.05, prec, calls=15)
    for a, b in zip(ref, got):
        assert a[0] == b[0]
        assert np.array_equal(a[1], b[1])
        assert np.array_equal(a[2], b[2])
