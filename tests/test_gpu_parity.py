"""Parity of the CUDA path (through the C-ABI) against the oracle.

Neighbour lists: bit-exact.  Network outputs: energy <= 1e-6 relative, forces
and virial <= 1e-4 max-abs relative to the RMS force (BASELINE.json north star),
in FP32 mode; FP64 mode is held to 1e-10.  The oracle is our C restatement,
itself pinned bit-exact to the reference (tests/test_oracle.py)."""
import json
import math

import numpy as np
import pytest

import oracle as O
import paper_2602_02234_b200 as P
from conftest import E_TOL, F_TOL, load_golden, rms

pytestmark = pytest.mark.gpu

TOL = {"fp32": (E_TOL, F_TOL), "fp64": (1e-10, 1e-10)}


def model(golden_models, name):
    return P.model_from_json(golden_models[name])


def assert_close(out, ref, prec, what=""):
    etol, ftol = TOL[prec]
    scale = rms(ref["forces"])
    de = abs(out.energy - ref["energy"]) / abs(ref["energy"])
    df = np.abs(out.forces - ref["forces"]).max() / scale
    dw = abs(out.virial - ref["virial"]) / max(abs(ref["virial"]), scale)
    assert de <= etol, f"{what} energy rel err {de:.3e}"
    assert df <= ftol, f"{what} force err {df:.3e} of rms"
    assert dw <= ftol, f"{what} virial err {dw:.3e}"


@pytest.mark.parametrize("name", ["n64", "1YRF"])
def test_neighbor_list_bitexact_golden(name):
    g = load_golden(name)
    inp = P.build_input_periodic(g["positions"], g["types"], np.arange(len(g["types"])), g["box"], 0.6)
    assert np.array_equal(inp.edge_offset, g["edge_offset"])
    assert np.array_equal(inp.edge_neighbor, g["edge_neighbor"])
    assert np.array_equal(inp.edge_dr, g["edge_dr"])


@pytest.mark.parametrize("n", [1231, 2643, 4114])
def test_neighbor_list_bitexact_paper_sizes(n):
    s = P.generate_synthetic_system(n)
    inp = P.build_input_periodic(s.positions, s.types, np.arange(n), s.box, 0.6)
    off, nbr, dr = O.neighbors(s.positions, s.box, 0.6)
    assert np.array_equal(inp.edge_offset, off)
    assert np.array_equal(inp.edge_neighbor, nbr)
    assert np.array_equal(inp.edge_dr, dr)


def test_neighbor_list_random_and_edge_geometries():
    rng = np.random.default_rng(1)
    for trial in range(40):
        n = int(rng.integers(2, 400))
        L = float(rng.uniform(1.2, 4.0))
        box = np.array([L, L * rng.uniform(1, 1.6), L * rng.uniform(1, 1.6)])
        x = rng.uniform(-1.0, 2.0, size=(n, 3)) * box  # unwrapped positions too
        inp = P.build_input_periodic(x, np.zeros(n, np.int32), np.arange(n), box, 0.6)
        off, nbr, dr = O.neighbors(x, box, 0.6)
        assert np.array_equal(inp.edge_offset, off)
        assert np.array_equal(inp.edge_neighbor, nbr)
        assert np.array_equal(inp.edge_dr, dr)


def test_neighbor_list_dense_cluster_grows_capacity():
    # 300 atoms in a 0.5 nm cube: every atom sees ~all others (> default capacity 64)
    rng = np.random.default_rng(2)
    box = np.array([3.0, 3.0, 3.0])
    x = rng.uniform(0, 0.5, size=(200, 3))
    inp = P.build_input_periodic(x, np.zeros(200, np.int32), np.arange(200), box, 0.6)
    off, nbr, dr = O.neighbors(x, box, 0.6)
    assert np.array_equal(inp.edge_offset, off) and np.array_equal(inp.edge_neighbor, nbr)


@pytest.mark.parametrize("name", ["n64", "1YRF"])
@pytest.mark.parametrize("mname", ["dpa2", "dpa3"])
@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_evaluate_matches_golden(name, mname, prec, golden_models):
    g = load_golden(name)
    m = model(golden_models, mname)
    n = g["types"].shape[0]
    inp = P.NnInput(g["positions"], g["types"], np.arange(n), np.zeros(n, np.uint8),
                    g["edge_offset"], g["edge_neighbor"], g["edge_dr"])
    cnt = P.NnCounters()
    out = P.evaluate(m, inp, P.Precision[prec], cnt)
    p = f"{mname}_{prec}_"
    ref = dict(energy=float(g[f"{mname}_fp64_energy"]), forces=g[f"{mname}_fp64_forces"],
               virial=float(g[f"{mname}_fp64_virial"]))
    assert_close(out, ref, prec, f"{name}/{mname}/{prec}")
    np.testing.assert_allclose(out.per_atom_energy, g[f"{mname}_fp64_per_atom"],
                               atol=TOL[prec][0] * abs(ref["energy"]) + (1e-5 if prec == "fp32" else 1e-12))
    assert [cnt.flops, cnt.peak_activation_bytes] == [int(v) for v in g[p + "counters"]]
    # trace of the virial tensor equals the reference scalar virial
    assert np.trace(out.virial_tensor) == pytest.approx(out.virial, rel=1e-5, abs=1e-6)


@pytest.mark.parametrize("mname", ["dpa2", "dpa3"])
@pytest.mark.parametrize("n", [1231, 2643, 4114])
def test_periodic_compute_paper_sizes(mname, n, golden_models):
    s = P.generate_synthetic_system(n)
    m = model(golden_models, mname)
    ref = O.evaluate(json.loads(golden_models[mname]), s.types, *O.neighbors(s.positions, s.box, 0.6))
    ctx = P.context_for(m)
    for prec in ("fp32", "fp64"):
        out = ctx.compute(s.positions, s.types, s.box, P.Precision[prec], per_atom=True)
        assert_close(out, ref, prec, f"{n}/{mname}/{prec}")
        assert abs(out.forces.sum(axis=0)).max() < 1e-9 * n  # translation invariance


@pytest.mark.parametrize("mname", ["dpa2", "dpa3"])
def test_stage_parity(mname, golden_models, golden_1yrf):
    """Per-kernel parity: descriptor, h^m (every layer), dE/dr per edge (FP64)."""
    g = golden_1yrf
    n = g["types"].shape[0]
    m = model(golden_models, mname)
    inp = P.NnInput(g["positions"], g["types"], np.arange(n), np.zeros(n, np.uint8),
                    g["edge_offset"], g["edge_neighbor"], g["edge_dr"])
    st = {}
    P.evaluate(m, inp, P.Precision.fp64, stages=st)
    ref = O.evaluate(json.loads(golden_models[mname]), g["types"], g["edge_offset"],
                     g["edge_neighbor"], g["edge_dr"], stages=True)
    np.testing.assert_allclose(st["desc"], ref["desc"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(st["h"], ref["h"], rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(st["edge_g"], ref["edge_g"], rtol=1e-9, atol=1e-9)
    st32 = {}
    P.evaluate(m, inp, P.Precision.fp32, stages=st32)
    np.testing.assert_allclose(st32["desc"], ref["desc"], rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(st32["h"], ref["h"], rtol=1e-4, atol=1e-5)


def test_descriptors_api(golden_models, golden_1yrf):
    g = golden_1yrf
    n = g["types"].shape[0]
    inp = P.NnInput(g["positions"], g["types"], np.arange(n), np.zeros(n, np.uint8),
                    g["edge_offset"], g["edge_neighbor"], g["edge_dr"])
    d = P.descriptors(model(golden_models, "dpa2"), inp)
    np.testing.assert_allclose(d, g["dpa2_descriptors"], rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_ghost_semantics(prec, golden_models, golden_n64):
    g = golden_n64
    ghost = np.zeros(64, dtype=np.uint8)
    ghost[::3] = 1
    m = model(golden_models, "dpa3")
    inp = P.NnInput(g["positions"], g["types"], np.arange(64), ghost, g["edge_offset"],
                    g["edge_neighbor"], g["edge_dr"])
    out = P.evaluate(m, inp, P.Precision[prec])
    ref = O.evaluate(json.loads(golden_models["dpa3"]), g["types"], g["edge_offset"],
                     g["edge_neighbor"], g["edge_dr"], is_ghost=ghost)
    assert_close(out, ref, prec, "ghost")
    assert np.all(out.per_atom_energy[ghost == 1] == 0.0)


def test_asymmetric_csr_input(golden_models, golden_n64):
    """A CSR whose lists are not mirror-symmetric (edges dropped from some rows)
    goes through the generic in-edge transpose."""
    g = golden_n64
    off, nbr, dr = g["edge_offset"], g["edge_neighbor"], g["edge_dr"]
    keep = np.ones(nbr.shape[0], bool)
    keep[off[3]:off[4]] = False  # atom 3 sees nobody; others still see atom 3
    counts = np.diff(off) * 1
    counts[3] = 0
    off2 = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    m = model(golden_models, "dpa3")
    inp = P.NnInput(g["positions"], g["types"], np.arange(64), np.zeros(64, np.uint8), off2,
                    nbr[keep], dr[keep])
    out = P.evaluate(m, inp, P.Precision.fp64)
    ref = O.evaluate(json.loads(golden_models["dpa3"]), g["types"], off2, nbr[keep], dr[keep])
    assert_close(out, ref, "fp64", "asym")


def test_errors(golden_models, golden_n64):
    g = golden_n64
    m = model(golden_models, "dpa3")
    inp = P.NnInput(g["positions"], g["types"], np.arange(64), np.zeros(64, np.uint8),
                    g["edge_offset"], g["edge_neighbor"], g["edge_dr"], coverage_radius=1.0)
    with pytest.raises(RuntimeError, match=r"^receptive-field error: model needs 1.800000 nm"):
        P.evaluate(m, inp)
    inp.skip_coverage_check = True
    P.evaluate(m, inp)  # the negative-control hook
    with pytest.raises(ValueError, match="exceeds half the box length on axis 0"):
        P.build_input_periodic(g["positions"], g["types"], np.arange(64), g["box"] * [0.9, 1, 1], 0.6)
    bad = g["types"].copy()
    bad[5] = 7
    with pytest.raises(ValueError, match="out of range"):
        P.context_for(m).compute(g["positions"], bad, g["box"])
    # zero-length edge (two atoms on the same site)
    x = g["positions"].copy()
    x[1] = x[0]
    with pytest.raises(RuntimeError, match="zero-length edge in NN input"):
        P.context_for(m).compute(x, g["types"], g["box"])
    # n == 0 returns an empty output (inference.cpp:205)
    out = P.context_for(m).compute(np.zeros((0, 3)), np.zeros(0, np.int32), g["box"])
    assert out.energy == 0.0 and out.forces.shape == (0, 3)


def test_bitwise_deterministic(golden_models):
    s = P.generate_synthetic_system(1231)
    ctx = P.context_for(model(golden_models, "dpa3"))
    a = ctx.compute(s.positions, s.types, s.box, P.Precision.fp32)
    b = ctx.compute(s.positions, s.types, s.box, P.Precision.fp32)
    assert a.energy == b.energy and np.array_equal(a.forces, b.forces) and a.virial == b.virial


def test_extensivity_replicated_box(golden_models):
    """a 2x2x2 periodic replica has 8x the energy."""
    s = P.generate_synthetic_system(582)
    r = P.replicate(s, (2, 2, 2))
    for mname in ("dpa2", "dpa3"):
        ctx = P.context_for(model(golden_models, mname))
        e1 = ctx.compute(s.positions, s.types, s.box, P.Precision.fp64).energy
        e8 = ctx.compute(r.positions, r.types, r.box, P.Precision.fp64).energy
        assert e8 == pytest.approx(8 * e1, rel=1e-12)


def test_large_box_paths_agree(golden_models):
    """Two kernel paths against each other in FP32.

    The 2PTC box (4114 atoms) runs 2-warp teams, the 28-warp-CTA build and the pull
    backward with stored z rows. Its (2,1,1) periodic replica (8228 atoms) runs
    1-warp teams and the pull backward with z recomputed (hmdp_net.cu pull_mode).
    The replica's energy is twice the box's, and each copy's forces equal the box's
    (FP32 tolerances).
    """
    s = P.generate_synthetic_system(4114)
    r = P.replicate(s, (2, 1, 1))
    ctx = P.context_for(model(golden_models, "dpa3"))
    one = ctx.compute(s.positions, s.types, s.box, P.Precision.fp32)
    two = ctx.compute(r.positions, r.types, r.box, P.Precision.fp32)
    assert abs(two.energy - 2 * one.energy) <= E_TOL * abs(2 * one.energy)
    scale = rms(one.forces)
    for k in range(2):
        fk = two.forces[k * s.n_atoms:(k + 1) * s.n_atoms]
        assert np.abs(fk - one.forces).max() <= F_TOL * scale


def test_receptive_field_exactness(golden_models):
    """moving an atom beyond depth*rc of atom i leaves E_i bitwise unchanged."""
    s = P.generate_synthetic_system(2643)
    ctx = P.context_for(model(golden_models, "dpa3"))
    base = ctx.compute(s.positions, s.types, s.box, P.Precision.fp64, per_atom=True)
    x = s.positions.copy()
    d = x - x[0]
    d -= s.box * np.round(d / s.box)
    far = int(np.argmax(np.linalg.norm(d, axis=1)))
    assert np.linalg.norm(d[far]) > 1.8 + 0.1
    x[far] += [0.01, 0.0, 0.0]
    pert = ctx.compute(x, s.types, s.box, P.Precision.fp64, per_atom=True)
    assert pert.per_atom_energy[0] == base.per_atom_energy[0]


@pytest.mark.parametrize("mname", ["dpa2", "dpa3"])
def test_sparse_rows_isolated_atom(mname, golden_models):
    """Rows with 0, 1 and 2 neighbours (a pair, an isolated atom, a triplet) and a
    single isolated atom, against the oracle; message passing over empty rows."""
    box = np.array([3.0, 3.0, 3.0])
    pos = np.array([[0.5, 0.5, 0.5], [0.8, 0.5, 0.5], [2.0, 2.0, 2.0],
                    [1.5, 0.4, 2.4], [1.5, 0.75, 2.4], [1.5, 0.6, 2.1]])
    types = np.array([0, 1, 0, 1, 0, 1], dtype=np.int32)
    md = json.loads(golden_models[mname])
    ctx = P.context_for(model(golden_models, mname))
    off, nbr, dr = O.neighbors(pos, box, 0.6)
    assert list(np.diff(off)) == [1, 1, 0, 2, 2, 2]
    for prec in ("fp32", "fp64"):
        ref = O.evaluate(md, types, off, nbr, dr, prec=prec)
        out = ctx.compute(pos, types, box, P.Precision[prec], per_atom=True)
        assert out.energy == pytest.approx(ref["energy"], rel=1e-6 if prec == "fp32" else 1e-12)
        assert np.abs(out.forces - ref["forces"]).max() <= 1e-4 * rms(ref["forces"])
        assert np.abs(out.per_atom_energy - ref["per_atom"]).max() < 1e-5
    one = ctx.compute(pos[2:3], types[2:3], box, P.Precision.fp64)
    r1 = O.evaluate(md, types[2:3], np.array([0, 0], dtype=np.int32), np.zeros(0, dtype=np.int32),
                    np.zeros((0, 3)))
    assert one.energy == pytest.approx(r1["energy"], rel=1e-12)
    assert np.abs(one.forces).max() == 0.0


@pytest.mark.parametrize("n", [582, 2643])
def test_cached_graph_replays_match_direct_path(n, golden_models):
    """hmdp_compute's cached graph (second call captures, later calls replay; outputs
    through host-mapped memory below 2048 atoms, a D2H copy node above) returns
    exactly what the direct path returned, per-atom energies included."""
    s = P.generate_synthetic_system(n)
    m = model(golden_models, "dpa3")
    ctx = P.Context(m)
    first = ctx.compute(s.positions, s.types, s.box, P.Precision.fp32, per_atom=True)
    for _ in range(4):
        out = ctx.compute(s.positions, s.types, s.box, P.Precision.fp32, per_atom=True)
        assert out.energy == first.energy and out.virial == first.virial
        assert np.array_equal(out.forces, first.forces)
        assert np.array_equal(out.per_atom_energy, first.per_atom_energy)
        assert np.array_equal(out.virial_tensor, first.virial_tensor)
    ref = O.evaluate(json.loads(golden_models["dpa3"]), s.types, *O.neighbors(s.positions, s.box, 0.6))
    assert_close(out, ref, "fp32", f"graph replay {n}")


@pytest.mark.parametrize("case", range(6))
def test_random_models_and_systems(case):
    """Random model seeds and systems (tools/parity_sweep.py runs hundreds): FP64 to the
    oracle's precision; FP32 forces <= 1e-4 of the RMS force and the energy <= 1e-6 of
    sum |e_i| (random models can make |E| small by cancellation)."""
    rng = np.random.default_rng(100 + case)
    fam, depth = [(0, 1), (1, 3)][case % 2]
    n = int(rng.integers(100, 800))
    s = P.generate_synthetic_system(n, seed=int(rng.integers(1, 10_000)))
    m = P.make_model(P.ModelFamily(fam), depth, 0.6, 2, 8, 32, int(rng.integers(1, 1000)))
    ref = O.evaluate(json.loads(m.to_json()), s.types, *O.neighbors(s.positions, s.box, 0.6))
    ctx = P.Context(m, max_atoms=n)
    scale_f = rms(ref["forces"])
    scale_e = float(np.abs(ref["per_atom"]).sum())
    o64 = ctx.compute(s.positions, s.types, s.box, P.Precision.fp64)
    assert abs(o64.energy - ref["energy"]) <= 1e-12 * scale_e
    assert np.abs(o64.forces - ref["forces"]).max() <= 1e-10 * scale_f
    o32 = ctx.compute(s.positions, s.types, s.box, P.Precision.fp32)
    assert abs(o32.energy - ref["energy"]) <= 1e-6 * scale_e
    assert np.abs(o32.forces - ref["forces"]).max() <= F_TOL * scale_f
