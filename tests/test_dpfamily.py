"""DeePMD-style families (se_a, repformer): SURVEY.md §8(a'), DESIGN.md §11.

No reference function exists for these operators ("parity unpinned"): the FP64
oracle (oracle/dpfamily.py, torch autograd) is itself checked by finite
differences and by the symmetries every deep potential must have, and the
device kernels are held to the north-star tolerances against it.
"""
import json

import numpy as np
import pytest

import oracle as O
import paper_2602_02234_b200 as P
from oracle import dpfamily as DF
from conftest import E_TOL, F_TOL, rms

FAMS = [(P.ModelFamily.se_a, 1), (P.ModelFamily.repformer, 2), (P.ModelFamily.repformer, 3),
        (P.ModelFamily.repflow, 2), (P.ModelFamily.repflow, 3)]
IDS = ["se_a", "repformer_d2", "repformer_d3", "repflow_d2", "repflow_d3"]


def _system(n, seed=7):
    s = P.generate_synthetic_system(n, seed=seed)
    off, nbr, dr = O.neighbors(s.positions, s.box, 0.6)
    return s, off, nbr, dr


@pytest.fixture(scope="module")
def small():
    return _system(64)


# ---------------------------------------------------------------------------
# CPU: model files, oracle self-checks
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("fam,depth", FAMS, ids=IDS)
def test_model_json_roundtrip(fam, depth):
    m = P.make_dp_model(fam, depth, seed=3)
    d = m.as_dict()
    assert d["family"] == fam.name and m.depth() == depth
    assert P.model_from_json(m.to_json()).to_json() == m.to_json()
    assert m.receptive_radius() == pytest.approx(depth * 0.6)
    # deterministic init
    assert P.make_dp_model(fam, depth, seed=3).to_json() == m.to_json()
    assert P.make_dp_model(fam, depth, seed=4).to_json() != m.to_json()


def test_model_validation_errors():
    with pytest.raises(ValueError):
        P.make_dp_model(P.ModelFamily.se_a, 2)  # se_a is depth 1
    with pytest.raises(ValueError):
        P.make_dp_model(P.ModelFamily.repformer, 1)  # needs a layer
    with pytest.raises(ValueError):
        P.make_dp_model(P.ModelFamily.se_a, 1, rc_smooth=0.7)  # rcs >= rc
    d = P.make_dp_model(P.ModelFamily.se_a, 1).as_dict()
    d["embeddings"] = d["embeddings"][:1]
    with pytest.raises(ValueError):
        P.model_from_json(json.dumps(d))
    d = P.make_dp_model(P.ModelFamily.repformer, 2).as_dict()
    d["layers"][0]["update"]["sizes"] = [160, 32, 31]
    with pytest.raises(ValueError):
        P.model_from_json(json.dumps(d))


@pytest.mark.parametrize("fam,depth", FAMS, ids=IDS)
def test_oracle_finite_differences(fam, depth, small):
    s, off, nbr, dr = small
    d = P.make_dp_model(fam, depth).as_dict()
    out = DF.evaluate(d, s.types, off, nbr, dr)
    x = np.array(s.positions, dtype=float)
    h = 1e-5
    rng = np.random.default_rng(0)
    scale = rms(out["forces"])
    for i in rng.choice(len(x), 4, replace=False):
        for a in range(3):
            xp = x.copy()
            xp[i, a] += h
            ep = DF.energy_of_positions(d, s.types, xp, s.box, off, nbr)
            xp[i, a] -= 2 * h
            em = DF.energy_of_positions(d, s.types, xp, s.box, off, nbr)
            assert abs(-(ep - em) / (2 * h) - out["forces"][i, a]) < 1e-6 * scale
    # virial = -dE/ds under uniform scaling of positions and box
    eps = 1e-6
    eps_p = DF.energy_of_positions(d, s.types, x * (1 + eps), np.asarray(s.box) * (1 + eps), off, nbr)
    eps_m = DF.energy_of_positions(d, s.types, x * (1 - eps), np.asarray(s.box) * (1 - eps), off, nbr)
    assert out["virial"] == pytest.approx(-(eps_p - eps_m) / (2 * eps), rel=1e-6, abs=1e-8)
    assert np.abs(out["forces"].sum(0)).max() < 1e-10 * max(scale, 1.0)
    assert np.abs(out["virial9"] - out["virial9"].T).max() < 1e-9 * max(np.abs(out["virial9"]).max(), 1)


@pytest.mark.parametrize("fam,depth", FAMS, ids=IDS)
def test_oracle_rotation_permutation_invariance(fam, depth, small):
    s, off, nbr, dr = small
    d = P.make_dp_model(fam, depth).as_dict()
    out = DF.evaluate(d, s.types, off, nbr, dr)
    # rotation of every edge vector: E invariant, forces co-rotate
    th = 0.7
    Rm = np.array([[np.cos(th), -np.sin(th), 0], [np.sin(th), np.cos(th), 0], [0, 0, 1.0]])
    Rm = Rm @ np.array([[1, 0, 0], [0, np.cos(0.3), -np.sin(0.3)], [0, np.sin(0.3), np.cos(0.3)]])
    rot = DF.evaluate(d, s.types, off, nbr, np.asarray(dr) @ Rm.T)
    assert rot["energy"] == pytest.approx(out["energy"], rel=1e-12)
    assert np.abs(rot["forces"] - out["forces"] @ Rm.T).max() < 1e-10 * rms(out["forces"])
    # relabelling atoms (with the CSR rows re-sorted by neighbour index)
    n = len(s.types)
    perm = np.random.default_rng(1).permutation(n)
    inv = np.argsort(perm)
    types = np.asarray(s.types)[perm]
    rows = []
    for new_i in range(n):
        i = perm[new_i]
        a, b = off[i], off[i + 1]
        pairs = sorted((inv[nbr[e]], e) for e in range(a, b))
        rows.append(pairs)
    off2 = np.zeros(n + 1, dtype=np.int32)
    nbr2, dr2 = [], []
    for new_i, pairs in enumerate(rows):
        off2[new_i + 1] = off2[new_i] + len(pairs)
        for j, e in pairs:
            nbr2.append(j)
            dr2.append(dr[e])
    per = DF.evaluate(d, types, off2, np.array(nbr2), np.array(dr2))
    assert per["energy"] == pytest.approx(out["energy"], rel=1e-12)
    assert np.abs(per["forces"] - out["forces"][perm]).max() < 1e-10 * rms(out["forces"])


@pytest.mark.parametrize("fam", [P.ModelFamily.repformer, P.ModelFamily.repflow])
def test_oracle_smooth_at_cutoff(fam):
    """Energy is continuous as a neighbour crosses rc (the switch and the gated,
    switched attention / angle messages all vanish there)."""
    d = P.make_dp_model(fam, 2).as_dict()
    types = [0, 1, 1]
    base = np.array([[0.0, 0.0, 0.0], [0.25, 0.1, 0.0]])

    def energy(r3):
        pos = np.vstack([base, [[r3, 0.0, 0.0]]])
        box = np.array([5.0, 5.0, 5.0])
        off, nbr, dr = O.neighbors(pos + 1.0, box, 0.6)
        return DF.evaluate(d, types, off, nbr, dr)["energy"]

    inside, outside = energy(0.6 - 1e-7), energy(0.6 + 1e-7)
    assert abs(inside - outside) < 1e-6
    if fam == P.ModelFamily.repflow:  # and as it crosses the angle cutoff
        ra = d["rc_angle"]
        assert abs(energy(ra - 1e-7) - energy(ra + 1e-7)) < 1e-6


def test_counters_and_launches_cpu():
    m = P.make_dp_model(P.ModelFamily.repformer, 3)
    assert m.n_params() > 0 and m.descriptor_dim() == 128


# ---------------------------------------------------------------------------
# GPU parity (hmdp_compute through the C-ABI)
# ---------------------------------------------------------------------------
def _check(out, ref, e_tol, f_tol):
    scale = rms(ref["forces"])
    de = abs(out.energy - ref["energy"]) / abs(ref["energy"])
    df = float(np.abs(out.forces - ref["forces"]).max()) / scale
    dw = float(np.abs(out.virial_tensor - ref["virial9"]).max()) / scale
    assert de <= e_tol and df <= f_tol and dw <= f_tol * 10, (de, df, dw)
    return de, df, dw


@pytest.mark.gpu
@pytest.mark.parametrize("fam,depth", FAMS, ids=IDS)
@pytest.mark.parametrize("n", [64, 582, 1231])
def test_gpu_parity(fam, depth, n):
    s, off, nbr, dr = _system(n)
    m = P.make_dp_model(fam, depth)
    ref = DF.evaluate(m.as_dict(), s.types, off, nbr, dr)
    ctx = P.Context(m, device=0)
    out64 = ctx.compute(s.positions, s.types, s.box, P.Precision.fp64, per_atom=True)
    _check(out64, ref, 1e-11, 1e-9)
    assert np.abs(out64.per_atom_energy - ref["per_atom"]).max() < 1e-10
    assert out64.virial == pytest.approx(ref["virial"], rel=1e-9, abs=1e-9)
    out32 = ctx.compute(s.positions, s.types, s.box, P.Precision.fp32)
    _check(out32, ref, E_TOL, F_TOL)


@pytest.mark.gpu
@pytest.mark.parametrize("fam,depth", FAMS, ids=IDS)
def test_gpu_deterministic_and_capacity_growth(fam, depth):
    # a dense cluster forces neighbour-capacity growth (> 64 neighbours)
    rng = np.random.default_rng(5)
    n = 300
    box = np.array([3.0, 3.0, 3.0])
    pos = np.vstack([rng.uniform(0, 3.0, (200, 3)), 1.5 + rng.uniform(-0.25, 0.25, (100, 3))])
    types = rng.integers(0, 2, n)
    off, nbr, dr = O.neighbors(pos, box, 0.6)
    assert np.diff(off).max() > 64
    m = P.make_dp_model(fam, depth)
    ref = DF.evaluate(m.as_dict(), types, off, nbr, dr)
    ctx = P.Context(m, device=0)
    a = ctx.compute(pos, types, box, P.Precision.fp64)
    _check(a, ref, 1e-11, 1e-9)
    b = ctx.compute(pos, types, box, P.Precision.fp32)
    c = ctx.compute(pos, types, box, P.Precision.fp32)
    assert b.energy == c.energy and np.array_equal(b.forces, c.forces)


@pytest.mark.gpu
def test_gpu_se_a_csr_path_with_ghosts_free_list():
    s, off, nbr, dr = _system(582)
    m = P.make_dp_model(P.ModelFamily.se_a, 1)
    ref = DF.evaluate(m.as_dict(), s.types, off, nbr, dr)
    inp = P.NnInput(positions=np.asarray(s.positions), types=np.asarray(s.types, dtype=np.int32),
                    global_index=np.arange(582, dtype=np.int32), is_ghost=np.zeros(582, np.uint8),
                    edge_offset=off, edge_neighbor=nbr, edge_dr=dr)
    out = P.evaluate(m, inp, P.Precision.fp64)
    _check(out, ref, 1e-11, 1e-9)
    for fam in (P.ModelFamily.repformer, P.ModelFamily.repflow):
        with pytest.raises(ValueError):
            P.evaluate(P.make_dp_model(fam, 2), inp, P.Precision.fp64)


@pytest.mark.gpu
@pytest.mark.parametrize("fam,depth", FAMS[:2] + FAMS[3:4], ids=IDS[:2] + IDS[3:4])
def test_gpu_md_loop(fam, depth):
    """Device MD with a DeePMD-style model: state after 6 steps matches a host
    velocity-Verlet loop driven by the FP64 oracle."""
    from paper_2602_02234_b200.md import DeviceMD

    s = P.generate_synthetic_system(64, temperature=300.0)
    m = P.make_dp_model(fam, depth)
    md = DeviceMD(P.Context(m), s.positions, s.velocities, s.masses, s.types, s.box,
                  precision=P.Precision.fp64, steps_per_graph=3)
    md.run(6)
    x_dev, v_dev, f_dev, e_dev = md.state()
    x, v = s.positions.copy(), s.velocities.copy()
    mass = np.asarray(s.masses)[:, None]

    def evaluate(x):
        off, nbr, dr = O.neighbors(x, s.box, 0.6)
        return DF.evaluate(m.as_dict(), s.types, off, nbr, dr)

    f = evaluate(x)["forces"]
    for _ in range(6):
        v += f * (0.0005 / mass)
        x += v * 0.001
        r = evaluate(x)
        f, e = r["forces"], r["energy"]
        v += f * (0.0005 / mass)
    assert np.abs(x_dev - x).max() < 1e-10
    assert np.abs(v_dev - v).max() < 1e-8
    assert e_dev == pytest.approx(e, rel=1e-10)


@pytest.mark.gpu
@pytest.mark.parametrize("fam,depth", FAMS[:2] + FAMS[3:4], ids=IDS[:2] + IDS[3:4])
def test_gpu_group_provider(fam, depth):
    """NNPot hybrid coupling (hmdp_compute_group) with a DeePMD-style model equals
    the model on the extracted group and leaves the other atoms alone."""
    from paper_2602_02234_b200.hybrid import (nn_force_provider, plan_group_preprocessing,
                                              synthetic_topology)

    s = P.generate_synthetic_system(582)
    _, plan = plan_group_preprocessing(synthetic_topology(582), "protein")
    m = P.make_dp_model(fam, depth)
    ctx = P.Context(m)
    f = np.zeros((582, 3))
    e = nn_force_provider(ctx, s.positions, s.types, s.box, plan, f, P.Precision.fp64)
    g = plan.atoms
    off, nbr, dr = O.neighbors(s.positions[g], s.box, 0.6)
    ref = DF.evaluate(m.as_dict(), s.types[g], off, nbr, dr)
    assert e == pytest.approx(ref["energy"], rel=1e-11)
    assert np.abs(f[g] - ref["forces"]).max() < 1e-9 * rms(ref["forces"])
    assert not np.any(f[np.setdiff1d(np.arange(582), g)])


@pytest.mark.gpu
@pytest.mark.parametrize("fam,depth", [(P.ModelFamily.se_a, 1), (P.ModelFamily.repflow, 2)])
def test_gpu_four_types(fam, depth):
    s, off, nbr, dr = _system(582)
    types = (np.arange(582) * 7) % 4
    m = P.make_dp_model(fam, depth, n_types=4, seed=5)
    ref = DF.evaluate(m.as_dict(), types, off, nbr, dr)
    out = P.Context(m).compute(s.positions, types, s.box, P.Precision.fp64)
    _check(out, ref, 1e-11, 1e-9)
    with pytest.raises(ValueError):
        P.Context(m).compute(s.positions, np.full(582, 4), s.box, P.Precision.fp64)


@pytest.mark.gpu
@pytest.mark.parametrize("fam,depth", [(P.ModelFamily.se_a, 1), (P.ModelFamily.repformer, 2),
                                       (P.ModelFamily.repflow, 2)])
def test_gpu_nve_energy_conservation(fam, depth):
    """Smooth potentials conserve energy: 400 FP64 velocity-Verlet steps of 0.5 fs
    on the device keep E_kin + E_pot within a small drift."""
    from paper_2602_02234_b200.md import DeviceMD

    s = P.generate_synthetic_system(582, temperature=300.0)
    m = P.make_dp_model(fam, depth)
    md = DeviceMD(P.Context(m), s.positions, s.velocities, s.masses, s.types, s.box,
                  dt_ps=0.0005, precision=P.Precision.fp64, steps_per_graph=50)

    def etot():
        x, v, f, ep = md.state()
        return ep + 0.5 * float(np.sum(s.masses[:, None] * v * v))

    e0 = etot()
    ke0 = 0.5 * float(np.sum(s.masses[:, None] * s.velocities ** 2))
    md.run(400)
    assert abs(etot() - e0) < 2e-3 * ke0


def _sparse_system():
    """A pair, an isolated atom and a triplet in a 3 nm box: rows with 0, 1 and 2
    neighbours (empty softmax / angle lists, single-column attention)."""
    box = np.array([3.0, 3.0, 3.0])
    pos = np.array([[0.5, 0.5, 0.5], [0.8, 0.5, 0.5], [2.0, 2.0, 2.0],
                    [1.5, 0.4, 2.4], [1.5, 0.75, 2.4], [1.5, 0.6, 2.1]])
    types = np.array([0, 1, 0, 1, 0, 1], dtype=np.int32)
    return pos, types, box


@pytest.mark.gpu
@pytest.mark.parametrize("fam,depth", FAMS, ids=IDS)
def test_gpu_sparse_rows_and_tiny_systems(fam, depth):
    pos, types, box = _sparse_system()
    off, nbr, dr = O.neighbors(pos, box, 0.6)
    assert list(np.diff(off)) == [1, 1, 0, 2, 2, 2]
    m = P.make_dp_model(fam, depth)
    ref = DF.evaluate(m.as_dict(), types, off, nbr, dr)
    ctx = P.Context(m, device=0)
    out = ctx.compute(pos, types, box, P.Precision.fp64, per_atom=True)
    _check(out, ref, 1e-11, 1e-9)
    assert np.abs(out.per_atom_energy - ref["per_atom"]).max() < 1e-10
    _check(ctx.compute(pos, types, box, P.Precision.fp32), ref, E_TOL, F_TOL)
    # one isolated atom: energy = the fitting of an empty environment, no force
    one = ctx.compute(pos[2:3], types[2:3], box, P.Precision.fp64, per_atom=True)
    r1 = DF.evaluate(m.as_dict(), types[2:3], np.array([0, 0]), np.zeros(0, dtype=np.int32),
                     np.zeros((0, 3)))
    assert one.energy == pytest.approx(r1["energy"], rel=1e-12, abs=1e-12)
    assert np.abs(one.forces).max() == 0.0
    # no atoms: zero outputs
    zero = ctx.compute(np.zeros((0, 3)), np.zeros(0, dtype=np.int32), box)
    assert zero.energy == 0.0 and zero.forces.shape == (0, 3)
