"""oracle — TEST INFRASTRUCTURE ONLY.

ctypes access to the two CPU checkers built by oracle/Makefile:
  * _build/libhmdp_oracle.so : our plain-C restatement of the reference hot path
  * _ref/libhalomd_ref.so    : the reference itself, compiled from its own sources
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  The product never does.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORA_PATH = os.path.join(HERE, "_build", "libhmdp_oracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libhalomd_ref.so")

_ora = None
_ref = None
_vp = ctypes.c_void_p


def _p(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def build(ref: bool = True) -> None:
    """make -C oracle (restatement always; reference only if /root/reference exists)."""
    targets = ["oracle"]
    if ref and os.path.exists("/root/reference/proj/src/nn/inference.cpp"):
        targets += ["ref", "dropin"]
        # the exact-signature drop-in program needs the product's libhalomd_nn_b200.so
        lib = os.path.join(os.path.dirname(HERE), "paper_2602_02234_b200", "lib", "libhalomd_nn_b200.so")
        if os.path.exists(lib):
            targets.append("dropin_exact")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def ora():
    global _ora
    if _ora is None:
        if not os.path.exists(ORA_PATH):
            build(ref=False)
        L = ctypes.CDLL(ORA_PATH)
        L.ora_last_error.restype = ctypes.c_char_p
        for fn in ("ora_neighbor_csr", "ora_neighbor_bruteforce"):
            getattr(L, fn).argtypes = [ctypes.c_int, _vp, _vp, ctypes.c_double, ctypes.c_int, _vp,
                                       _vp, _vp]
        for fn in ("ora_evaluate_f64", "ora_evaluate_f32"):
            getattr(L, fn).argtypes = [_vp, _vp, ctypes.c_int, _vp, _vp, _vp, _vp, _vp,
                                       ctypes.c_double, ctypes.c_int, _vp, _vp, _vp, _vp, _vp, _vp,
                                       _vp, _vp]
        L.ora_descriptors.argtypes = [_vp, _vp, ctypes.c_int, _vp, _vp, _vp, _vp, _vp]
        L.ora_switch_value.restype = ctypes.c_double
        L.ora_switch_value.argtypes = [ctypes.c_double, ctypes.c_double]
        L.ora_switch_derivative.restype = ctypes.c_double
        L.ora_switch_derivative.argtypes = [ctypes.c_double, ctypes.c_double]
        _ora = L
    return _ora


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


def ref():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_PATH):
            raise FileNotFoundError(REF_PATH)
        L = ctypes.CDLL(REF_PATH)
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_make_model_json.restype = ctypes.c_long
        L.ref_make_model_json.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int,
                                          ctypes.c_int, ctypes.c_int, ctypes.c_uint64, _vp,
                                          ctypes.c_long]
        L.ref_model_load.restype = _vp
        L.ref_model_load.argtypes = [ctypes.c_char_p, ctypes.c_long]
        L.ref_model_free.argtypes = [_vp]
        L.ref_synthetic.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                    ctypes.c_uint64, ctypes.c_double, _vp, _vp, _vp, _vp, _vp]
        L.ref_input_build.restype = _vp
        L.ref_input_build.argtypes = [ctypes.c_int, _vp, _vp, _vp, ctypes.c_double]
        L.ref_input_nedges.argtypes = [_vp]
        L.ref_input_get.argtypes = [_vp, _vp, _vp, _vp]
        L.ref_input_free.argtypes = [_vp]
        L.ref_evaluate_csr.argtypes = [_vp, ctypes.c_int, _vp, _vp, _vp, _vp, _vp, _vp,
                                       ctypes.c_double, ctypes.c_int, ctypes.c_int, _vp, _vp, _vp,
                                       _vp, _vp, _vp]
        L.ref_evaluate_periodic.argtypes = [_vp, ctypes.c_int, _vp, _vp, _vp, ctypes.c_int, _vp,
                                            _vp, _vp, _vp]
        L.ref_descriptors.argtypes = [_vp, ctypes.c_int, _vp, _vp, _vp, _vp, _vp, _vp]
        L.ref_synthetic_topology.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                             ctypes.c_uint64] + [_vp] * 10
        L.ref_classical.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_uint64,
                                    _vp, _vp, _vp, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                    ctypes.c_double, ctypes.c_int, _vp, _vp, _vp, _vp]
        L.ref_switch_value.restype = ctypes.c_double
        L.ref_switch_value.argtypes = [ctypes.c_double, ctypes.c_double]
        L.ref_switch_derivative.restype = ctypes.c_double
        L.ref_switch_derivative.argtypes = [ctypes.c_double, ctypes.c_double]
        L.ref_bench_eval.restype = ctypes.c_double
        L.ref_bench_eval.argtypes = [_vp, ctypes.c_int, _vp, _vp, _vp, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_int]
        L.ref_md_run.restype = ctypes.c_double
        L.ref_md_run.argtypes = [_vp, ctypes.c_int, _vp, _vp, _vp, _vp, _vp, ctypes.c_double,
                                 ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp]
        _ref = L
    return _ref


# ---------------------------------------------------------------------------
# Model encoding for the C restatement (see hmdp_oracle.h)
# ---------------------------------------------------------------------------
def model_layout(model: dict):
    fam = 0 if model["family"] == "embed_fit" else 1
    K = len(model["basis"]["centers"])
    mlps = [model["embedding"], model["fitting"]]
    for layer in model["layers"]:
        mlps += [layer["message"], layer["update"]]
    ilay = [fam, int(model["n_types"]), K, int(model["hidden"]), len(model["layers"]), len(mlps)]
    dpar = [float(model["rc_model"]), float(model["basis"]["width"])] + [float(c) for c in model["basis"]["centers"]]
    for m in mlps:
        ilay.append(len(m["sizes"]) - 1)
        ilay += [int(s) for s in m["sizes"]]
        for w, b in zip(m["weights"], m["biases"]):
            dpar += [float(v) for v in w]
            dpar += [float(v) for v in b]
    return np.array(ilay, dtype=np.int32), np.array(dpar, dtype=np.float64)


class OracleError(Exception):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def neighbors(pos, box, rc, brute: bool = False):
    """CSR (offset, nbr, dr) from the C restatement of build_input_periodic."""
    L = ora()
    x = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 3)
    b = np.ascontiguousarray(box, dtype=np.float64)
    n = x.shape[0]
    off = np.zeros(n + 1, dtype=np.int32)
    fn = L.ora_neighbor_bruteforce if brute else L.ora_neighbor_csr
    cap = max(64, 64 * n)
    while True:
        nbr = np.zeros(cap, dtype=np.int32)
        dr = np.zeros((cap, 3))
        ne = fn(n, _p(x), _p(b), float(rc), cap, _p(off), _p(nbr), _p(dr))
        if ne < 0:
            raise OracleError(1, L.ora_last_error().decode())
        if ne <= cap:
            return off, nbr[:ne].copy(), dr[:ne].copy()
        cap = ne


def evaluate(model: dict, types, offset, nbr, dr, is_ghost=None, prec: str = "fp64",
             coverage: float = math.inf, skip_coverage: bool = False, stages: bool = False):
    """evaluate_impl<T> restated in C.  Returns a dict."""
    L = ora()
    ilay, dpar = model_layout(model)
    t = np.ascontiguousarray(types, dtype=np.int32)
    n = t.shape[0]
    off = np.ascontiguousarray(offset, dtype=np.int32)
    nb = np.ascontiguousarray(nbr, dtype=np.int32)
    d = np.ascontiguousarray(dr, dtype=np.float64).reshape(-1, 3)
    g = None if is_ghost is None else np.ascontiguousarray(is_ghost, dtype=np.uint8)
    ne = int(off[n]) if n >= 0 else 0
    e = ctypes.c_double()
    w = ctypes.c_double()
    f = np.zeros((n, 3))
    pa = np.zeros(n)
    cnt = np.zeros(2, dtype=np.uint64)
    H = int(model["hidden"])
    nd = int(model["n_types"]) * len(model["basis"]["centers"])
    desc = np.zeros((n, nd)) if stages else None
    h = np.zeros((len(model["layers"]) + 1, n, H)) if stages else None
    eg = np.zeros(max(ne, 1)) if stages else None
    fn = L.ora_evaluate_f64 if prec == "fp64" else L.ora_evaluate_f32
    code = fn(_p(ilay), _p(dpar), n, _p(t), _p(g), _p(off), _p(nb), _p(d), float(coverage),
              int(skip_coverage), ctypes.byref(e), _p(pa), _p(f), ctypes.byref(w), _p(cnt),
              _p(desc), _p(h), _p(eg))
    if code:
        raise OracleError(code, L.ora_last_error().decode())
    out = dict(energy=e.value, per_atom=pa, forces=f, virial=w.value, flops=int(cnt[0]),
               act_bytes=int(cnt[1]))
    if stages:
        out.update(desc=desc, h=h, edge_g=eg[:ne])
    return out


def switch_value(r, rc):
    return ora().ora_switch_value(float(r), float(rc))


def switch_derivative(r, rc):
    return ora().ora_switch_derivative(float(r), float(rc))


# ---------------------------------------------------------------------------
# The compiled reference (oracle/_ref)
# ---------------------------------------------------------------------------
def ref_model_json(family: int, depth: int, rc=0.6, n_types=2, n_basis=8, hidden=32, seed=1) -> str:
    L = ref()
    need = L.ref_make_model_json(family, depth, rc, n_types, n_basis, hidden, seed, None, 0)
    if need < 0:
        raise OracleError(-need, L.ref_last_error().decode())
    buf = ctypes.create_string_buffer(need + 1)
    L.ref_make_model_json(family, depth, rc, n_types, n_basis, hidden, seed, buf, need + 1)
    return buf.value.decode()


class RefModel:
    def __init__(self, text: str):
        self.h = ref().ref_model_load(text.encode(), len(text.encode()))
        if not self.h:
            raise OracleError(1, ref().ref_last_error().decode())

    def __del__(self):
        try:
            ref().ref_model_free(self.h)
        except Exception:
            pass


def ref_synthetic(n, density=33.4, fraction=0.35, seed=7, temperature=300.0):
    L = ref()
    x = np.zeros((n, 3))
    v = np.zeros((n, 3))
    t = np.zeros(n, dtype=np.int32)
    m = np.zeros(n)
    b = np.zeros(3)
    code = L.ref_synthetic(n, density, fraction, seed, temperature, _p(x), _p(t), _p(m), _p(v), _p(b))
    if code:
        raise OracleError(code, L.ref_last_error().decode())
    return x, t, m, v, b


def ref_build_input(pos, types, box, rc):
    L = ref()
    x = np.ascontiguousarray(pos, dtype=np.float64)
    t = np.ascontiguousarray(types, dtype=np.int32)
    b = np.ascontiguousarray(box, dtype=np.float64)
    n = x.shape[0]
    h = L.ref_input_build(n, _p(x), _p(t), _p(b), float(rc))
    if not h:
        raise OracleError(1, L.ref_last_error().decode())
    ne = L.ref_input_nedges(h)
    off = np.zeros(n + 1, dtype=np.int32)
    nbr = np.zeros(max(ne, 1), dtype=np.int32)
    dr = np.zeros((max(ne, 1), 3))
    L.ref_input_get(h, _p(off), _p(nbr), _p(dr))
    L.ref_input_free(h)
    return off, nbr[:ne].copy(), dr[:ne].copy()


def ref_evaluate_csr(model: RefModel, pos, types, offset, nbr, dr, is_ghost=None, prec="fp64",
                     coverage=math.inf, skip_coverage=False):
    L = ref()
    x = np.ascontiguousarray(pos, dtype=np.float64)
    t = np.ascontiguousarray(types, dtype=np.int32)
    n = t.shape[0]
    g = None if is_ghost is None else np.ascontiguousarray(is_ghost, dtype=np.uint8)
    off = np.ascontiguousarray(offset, dtype=np.int32)
    nb = np.ascontiguousarray(nbr, dtype=np.int32)
    d = np.ascontiguousarray(dr, dtype=np.float64).reshape(-1, 3)
    e = ctypes.c_double()
    w = ctypes.c_double()
    f = np.zeros((n, 3))
    pa = np.zeros(n)
    fl = ctypes.c_uint64()
    ab = ctypes.c_uint64()
    code = L.ref_evaluate_csr(model.h, n, _p(x), _p(t), _p(g), _p(off), _p(nb), _p(d),
                              float(coverage), int(skip_coverage), 0 if prec == "fp64" else 1,
                              ctypes.byref(e), _p(pa), _p(f), ctypes.byref(w), ctypes.byref(fl),
                              ctypes.byref(ab))
    if code:
        raise OracleError(code, L.ref_last_error().decode())
    return dict(energy=e.value, per_atom=pa, forces=f, virial=w.value, flops=fl.value,
                act_bytes=ab.value)


def ref_descriptors(model: RefModel, pos, types, offset, nbr, dr, nd=16):
    x = np.ascontiguousarray(pos, dtype=np.float64)
    t = np.ascontiguousarray(types, dtype=np.int32)
    out = np.zeros((t.shape[0], nd))
    _rcheck(ref().ref_descriptors(model.h, t.shape[0], _p(x), _p(t),
                                  _p(np.ascontiguousarray(offset, dtype=np.int32)),
                                  _p(np.ascontiguousarray(nbr, dtype=np.int32)),
                                  _p(np.ascontiguousarray(dr, dtype=np.float64)), _p(out)))
    return out


def ref_bench(model: RefModel, pos, types, box, prec="fp32", steps=1, threads=1) -> float:
    L = ref()
    x = np.ascontiguousarray(pos, dtype=np.float64)
    t = np.ascontiguousarray(types, dtype=np.int32)
    b = np.ascontiguousarray(box, dtype=np.float64)
    return L.ref_bench_eval(model.h, x.shape[0], _p(x), _p(t), _p(b), 0 if prec == "fp64" else 1,
                            int(steps), int(threads))


def ref_md(model: RefModel, pos, vel, types, masses, box, dt_ps=0.001, prec="fp32", steps=1,
           threads=1):
    """Velocity-Verlet MD with the reference force provider; returns (wall_s, x, v, epot)."""
    L = ref()
    x = np.ascontiguousarray(pos, dtype=np.float64).copy()
    v = np.ascontiguousarray(vel, dtype=np.float64).copy()
    t = np.ascontiguousarray(types, dtype=np.int32)
    m = np.ascontiguousarray(masses, dtype=np.float64)
    b = np.ascontiguousarray(box, dtype=np.float64)
    ep = ctypes.c_double()
    wall = L.ref_md_run(model.h, x.shape[0], _p(x), _p(v), _p(t), _p(m), _p(b), float(dt_ps),
                        0 if prec == "fp64" else 1, int(steps), int(threads), ctypes.byref(ep))
    return wall, x, v, ep.value


# ---- classical force field of the reference (forcefield.cpp) ----------------
LJ_SIGMA = (0.33, 0.30)  # SyntheticParams defaults (synthetic.hpp:30-33)
LJ_EPS = (0.40, 0.50)


def ref_synthetic_topology(n, density=33.4, fraction=0.35, seed=7) -> dict:
    """The synthetic system's topology (synthetic.cpp:36-130) as flat arrays."""
    L = ref()
    c = np.zeros(4, dtype=np.int32)
    _rcheck(L.ref_synthetic_topology(n, density, fraction, seed, _p(c), *([None] * 9)))
    nb, na, nd, ne = (int(v) for v in c)
    t = {"charges": np.zeros(n), "excl_offset": np.zeros(n + 1, dtype=np.int32),
         "excl": np.zeros(max(ne, 1), dtype=np.int32), "bonds": np.zeros((max(nb, 1), 2), dtype=np.int32),
         "bond_params": np.zeros((max(nb, 1), 2)), "angles": np.zeros((max(na, 1), 3), dtype=np.int32),
         "angle_params": np.zeros((max(na, 1), 2)), "dihedrals": np.zeros((max(nd, 1), 4), dtype=np.int32),
         "dihedral_params": np.zeros((max(nd, 1), 3))}
    _rcheck(L.ref_synthetic_topology(n, density, fraction, seed, _p(c), _p(t["charges"]),
                                     _p(t["excl_offset"]), _p(t["excl"]), _p(t["bonds"]),
                                     _p(t["bond_params"]), _p(t["angles"]), _p(t["angle_params"]),
                                     _p(t["dihedrals"]), _p(t["dihedral_params"])))
    t["excl"] = t["excl"][:ne]
    for k, m in (("bonds", nb), ("bond_params", nb), ("angles", na), ("angle_params", na),
                 ("dihedrals", nd), ("dihedral_params", nd)):
        t[k] = t[k][:m]
    return t


def ref_classical(pos, n, scheme=0, rc_c=0.7, eps_rf=78.0, rc_lj=0.7, fp64=True, density=33.4,
                  fraction=0.35, seed=7):
    """compute_classical (forcefield.cpp:265-279) on the synthetic topology."""
    L = ref()
    x = np.ascontiguousarray(pos, dtype=np.float64)
    sig = np.asarray(LJ_SIGMA)
    eps = np.asarray(LJ_EPS)
    e = np.zeros(3)
    f = np.zeros((n, 3))
    w = np.zeros(1)
    c = np.zeros(1, dtype=np.int32)
    _rcheck(L.ref_classical(n, density, fraction, seed, _p(x), _p(sig), _p(eps), scheme, rc_c,
                            eps_rf, rc_lj, int(fp64), _p(e), _p(f), _p(w), _p(c)))
    return {"energies": e, "forces": f, "virial": float(w[0]), "collinear": int(c[0])}


def _rcheck(code):
    if code:
        raise OracleError(code, ref().ref_last_error().decode())
