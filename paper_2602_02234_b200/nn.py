"""Host-side mirror of the reference's NN force-provider API, on the B200 path.

Mirrors /root/reference/proj/include/halomd/nn/{model,inference}.hpp name for
name -- ModelFamily, Precision, NnModel, make_model, model_to_json,
model_from_json, NnInput, NnOutput, NnCounters, build_input_periodic, evaluate,
descriptors, switch_value, switch_derivative -- with the same argument meaning
and the same error behaviour (std::invalid_argument -> ValueError,
std::runtime_error -> RuntimeError).  Every numerical call goes through the C-ABI
of libhmdp.so (include/hmdp.h) and runs on the GPU; there is no CPU fallback.

Divergences (documented in DESIGN.md): atom types are range-checked (the
reference writes out of bounds); the device kernels take
two-layer MLPs with H = 32, K = 8, n_types <= 4 (make_model's defaults).
"""
from __future__ import annotations

import ctypes
import enum
import hashlib
import json
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import check, lib, ptr


class ModelFamily(enum.IntEnum):
    """model.hpp:9 ``enum class ModelFamily { embed_fit, message_passing }``, plus the
    DeePMD-style families of the north star that have no reference function
    (SURVEY.md §8(a')): ``se_a`` (smooth env matrix, G^T R R^T G) and
    ``repformer`` (DPA2-style gated neighbour self-attention) and ``repflow``
    (DPA3-style edge/angle message passing)."""

    embed_fit = 0
    message_passing = 1
    se_a = 2
    repformer = 3
    repflow = 4


class Precision(enum.IntEnum):
    """forcefield.hpp:10 ``enum class Precision { fp32, fp64 }``."""

    fp32 = _lib.HMDP_FP32
    fp64 = _lib.HMDP_FP64


# ---------------------------------------------------------------------------
# Model
# ---------------------------------------------------------------------------
class NnModel:
    """Toy deep potential (model.hpp:40-56), held as its versioned JSON."""

    def __init__(self, text: str):
        code = lib().hmdp_model_validate(text.encode(), len(text.encode()))
        check(code)
        self._text = text
        self._d = json.loads(text)
        self.digest = hashlib.sha1(text.encode()).hexdigest()

    # model.hpp fields
    @property
    def family(self) -> ModelFamily:
        return ModelFamily[self._d["family"]]

    def is_dp(self) -> bool:
        return self.family >= ModelFamily.se_a

    @property
    def rc_model(self) -> float:
        return float(self._d["rc_model"])

    @property
    def n_types(self) -> int:
        return int(self._d["n_types"])

    @property
    def hidden(self) -> int:
        return int(self._d["hidden"])

    @property
    def seed(self) -> int:
        return int(self._d.get("seed", 0))

    @property
    def basis_centers(self) -> list[float]:
        return list(self._d["basis"]["centers"])

    @property
    def basis_width(self) -> float:
        return float(self._d["basis"]["width"])

    def depth(self) -> int:
        return 1 + len(self._d.get("layers", []))

    def receptive_radius(self) -> float:
        return self.depth() * self.rc_model

    def descriptor_dim(self) -> int:
        if self.is_dp():
            return int(self._d["axis"]) * self.hidden
        return self.n_types * len(self.basis_centers)

    def n_params(self) -> int:
        def mlp(m):
            return sum(len(w) for w in m["weights"]) + sum(len(b) for b in m["biases"])

        if self.is_dp():
            n = sum(mlp(e) for e in self._d["embeddings"]) + mlp(self._d["fitting"])
            n += len(self._d["energy_bias"])
            if "g1map" in self._d:
                n += mlp(self._d["g1map"])
            for layer in self._d.get("layers", []):
                n += sum(mlp(v) for v in layer.values())
            return n
        n = mlp(self._d["embedding"]) + mlp(self._d["fitting"])
        for layer in self._d["layers"]:
            n += mlp(layer["message"]) + mlp(layer["update"])
        return n

    def to_json(self) -> str:
        return self._text

    def as_dict(self) -> dict:
        return self._d


def make_model(family: ModelFamily, depth: int, rc_model: float, n_types: int, n_basis: int,
               hidden: int, seed: int) -> NnModel:
    """make_model (model.cpp:70-100): deterministic mt19937_64 random init."""
    L = lib()
    args = (int(family), int(depth), float(rc_model), int(n_types), int(n_basis), int(hidden),
            ctypes.c_uint64(seed))
    need = L.hmdp_make_model_json(*args, None, 0)
    if need < 0:
        check(-need)
    buf = ctypes.create_string_buffer(need + 1)
    L.hmdp_make_model_json(*args, buf, need + 1)
    return NnModel(buf.value.decode())


def make_dp_model(family: ModelFamily, depth: int, rc_model: float = 0.6, rc_smooth: float = 0.3,
                  n_types: int = 2, seed: int = 1, axis: int = 4) -> NnModel:
    """Random-init DeePMD-style model (se_a: depth 1; repformer / repflow: depth - 1 layers),
    same Rng / MLP init as make_model.  No reference function (parity unpinned)."""
    L = lib()
    args = (int(family), int(depth), float(rc_model), float(rc_smooth), int(n_types), int(axis),
            ctypes.c_uint64(seed))
    need = L.hmdp_make_dp_model_json(*args, None, 0)
    if need < 0:
        check(-need)
    buf = ctypes.create_string_buffer(need + 1)
    L.hmdp_make_dp_model_json(*args, buf, need + 1)
    return NnModel(buf.value.decode())


def model_to_json(model: NnModel) -> str:
    return model.to_json()


def model_from_json(text: str) -> NnModel:
    return NnModel(text)


def save_model(path: str, model: NnModel) -> None:
    with open(path, "w") as f:
        f.write(model.to_json())


def load_model(path: str) -> NnModel:
    try:
        with open(path) as f:
            return NnModel(f.read())
    except OSError as e:
        raise RuntimeError(f"cannot open model file {path}") from e


# ---------------------------------------------------------------------------
# Device contexts (one per (model, device), cached)
# ---------------------------------------------------------------------------
class Context:
    """Owns one hmdp_ctx: device weights, stream and buffers (include/hmdp.h)."""

    def __init__(self, model: NnModel | None, device: int = 0, max_atoms: int = 1024,
                 max_neighbors: int = 0):
        self.model = model
        self.device = device
        h = ctypes.c_void_p()
        text = model.to_json().encode() if model is not None else None
        check(lib().hmdp_create(text, len(text) if text else 0, device, max_atoms, max_neighbors,
                                ctypes.byref(h)))
        self.handle = h

    def close(self) -> None:
        if getattr(self, "handle", None):
            lib().hmdp_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def kernels_per_eval(self) -> int:
        return int(lib().hmdp_kernels_per_eval(self.handle))

    # ---- periodic single-domain path (positions in, E/F/W out) ----
    def compute(self, positions, types, box, precision: Precision = Precision.fp32,
                per_atom: bool = False):
        x = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1, 3)
        t = np.ascontiguousarray(types, dtype=np.int32)
        n = x.shape[0]
        if t.shape[0] != n:
            raise ValueError("positions/types/global_index size mismatch")
        b = _box3(box)
        e = ctypes.c_double()
        w = ctypes.c_double()
        f = np.zeros((n, 3))
        w9 = np.zeros(9)
        pa = np.zeros(n) if per_atom else None
        check(lib().hmdp_compute(self.handle, n, ptr(x), ptr(t), ptr(b), int(precision),
                                 ctypes.byref(e), ptr(pa), ptr(f), ptr(w9), ctypes.byref(w)))
        return NnOutput(per_atom_energy=pa if pa is not None else np.zeros(0), forces=f,
                        energy=e.value, virial=w.value, virial_tensor=w9.reshape(3, 3))


_contexts: dict[tuple, Context] = {}


def context_for(model: NnModel | None, device: int = 0) -> Context:
    key = (model.digest if model is not None else None, device)
    ctx = _contexts.get(key)
    if ctx is None:
        ctx = Context(model, device)
        _contexts[key] = ctx
    return ctx


def _box3(box) -> np.ndarray:
    if hasattr(box, "lengths"):
        box = box.lengths
    b = np.ascontiguousarray(box, dtype=np.float64).reshape(-1)
    if b.shape[0] != 3:
        raise ValueError("box must have three lengths")
    return b


# ---------------------------------------------------------------------------
# NnInput / NnOutput / NnCounters (inference.hpp:18-59)
# ---------------------------------------------------------------------------
@dataclass
class SimBox:
    """box.hpp:11-21 (orthorhombic, periodic on all axes)."""

    lx: float
    ly: float
    lz: float

    @property
    def lengths(self):
        return (self.lx, self.ly, self.lz)


@dataclass
class NnInput:
    positions: np.ndarray
    types: np.ndarray
    global_index: np.ndarray
    is_ghost: np.ndarray
    edge_offset: np.ndarray
    edge_neighbor: np.ndarray
    edge_dr: np.ndarray
    coverage_radius: float = math.inf
    skip_coverage_check: bool = False

    def n_atoms(self) -> int:
        return int(self.types.shape[0])

    def n_owned(self) -> int:
        return int(np.count_nonzero(self.is_ghost == 0))

    def check(self) -> None:
        """NnInput::check (inference.cpp:19-32)."""
        n = self.n_atoms()
        if (self.positions.shape[0] != n or self.global_index.shape[0] != n
                or self.is_ghost.shape[0] != n):
            raise ValueError("NnInput arrays disagree on atom count")
        if self.edge_offset.shape[0] != n + 1:
            raise ValueError("NnInput edge_offset has wrong size")
        if self.edge_neighbor.shape[0] != self.edge_dr.shape[0]:
            raise ValueError("NnInput edge arrays disagree")
        if self.edge_offset.shape[0] and self.edge_offset[-1] != self.edge_neighbor.shape[0]:
            raise ValueError("NnInput CSR offsets inconsistent")
        if self.edge_neighbor.size and (self.edge_neighbor.min() < 0 or self.edge_neighbor.max() >= n):
            raise ValueError("NnInput edge neighbor out of range")


@dataclass
class NnOutput:
    per_atom_energy: np.ndarray
    forces: np.ndarray
    energy: float = 0.0
    virial: float = 0.0
    virial_tensor: np.ndarray = field(default_factory=lambda: np.zeros((3, 3)))


@dataclass
class NnCounters:
    flops: int = 0
    peak_activation_bytes: int = 0
    inferences: int = 0

    def merge(self, other: "NnCounters") -> None:
        self.flops += other.flops
        self.peak_activation_bytes = max(self.peak_activation_bytes, other.peak_activation_bytes)
        self.inferences += other.inferences


def build_input_periodic(positions, types, global_index, box, rc_model: float,
                         device: int = 0) -> NnInput:
    """build_input_periodic (inference.cpp:449-487): the device cell-list
    neighbour search, exported in the reference's CSR layout (bit-exact)."""
    x = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1, 3)
    t = np.ascontiguousarray(types, dtype=np.int32)
    g = np.ascontiguousarray(global_index, dtype=np.int32)
    n = x.shape[0]
    if t.shape[0] != n or g.shape[0] != n:
        raise ValueError("positions/types/global_index size mismatch")
    b = _box3(box)
    ctx = context_for(None, device)
    offset = np.zeros(n + 1, dtype=np.int32)
    ne = ctypes.c_int()
    cap = max(64, 48 * n)
    while True:
        nbr = np.zeros(cap, dtype=np.int32)
        dr = np.zeros((cap, 3))
        check(lib().hmdp_build_neighbors(ctx.handle, n, ptr(x), ptr(b), float(rc_model), cap,
                                         ptr(offset), ptr(nbr), ptr(dr), ctypes.byref(ne)))
        if ne.value <= cap:
            break
        cap = ne.value
    m = ne.value
    return NnInput(positions=x.copy(), types=t.copy(), global_index=g.copy(),
                   is_ghost=np.zeros(n, dtype=np.uint8), edge_offset=offset,
                   edge_neighbor=nbr[:m].copy(), edge_dr=dr[:m].copy())


def evaluate(model: NnModel, input: NnInput, prec: Precision = Precision.fp64,
             counters: NnCounters | None = None, device: int = 0, stages: dict | None = None
             ) -> NnOutput:
    """evaluate (inference.cpp:420-424) on the device.  ``stages`` (optional dict)
    receives the per-stage tensors desc / h / edge_g for parity tests."""
    input.check()
    ctx = context_for(model, device)
    n = input.n_atoms()
    t = np.ascontiguousarray(input.types, dtype=np.int32)
    ghost = np.ascontiguousarray(input.is_ghost, dtype=np.uint8)
    off = np.ascontiguousarray(input.edge_offset, dtype=np.int32)
    nbr = np.ascontiguousarray(input.edge_neighbor, dtype=np.int32)
    dr = np.ascontiguousarray(input.edge_dr, dtype=np.float64).reshape(-1, 3)
    e = ctypes.c_double()
    w = ctypes.c_double()
    f = np.zeros((n, 3))
    pa = np.zeros(n)
    w9 = np.zeros(9)
    cnt = np.zeros(2, dtype=np.uint64)
    desc = hbuf = gbuf = None
    if stages is not None:
        desc = np.zeros((n, model.descriptor_dim()))
        hbuf = np.zeros((model.depth(), n, model.hidden))
        gbuf = np.zeros(nbr.shape[0])
    cov = float(input.coverage_radius)
    check(lib().hmdp_compute_csr(ctx.handle, n, ptr(t), ptr(ghost), ptr(off), ptr(nbr), ptr(dr),
                                 cov if math.isfinite(cov) else 1e300,
                                 int(bool(input.skip_coverage_check)), int(prec), ctypes.byref(e),
                                 ptr(pa), ptr(f), ptr(w9), ctypes.byref(w), ptr(desc), ptr(hbuf),
                                 ptr(gbuf), ptr(cnt)))
    if counters is not None:
        counters.merge(NnCounters(int(cnt[0]), int(cnt[1]), 1))
    if stages is not None:
        stages.update(desc=desc, h=hbuf, edge_g=gbuf)
    return NnOutput(per_atom_energy=pa, forces=f, energy=e.value, virial=w.value,
                    virial_tensor=w9.reshape(3, 3))


def descriptors(model: NnModel, input: NnInput, device: int = 0) -> np.ndarray:
    """descriptors (inference.cpp:430-447), FP64 on the device: [n, n_types*K]."""
    input.check()
    ctx = context_for(model, device)
    n = input.n_atoms()
    out = np.zeros((n, model.descriptor_dim()))
    t = np.ascontiguousarray(input.types, dtype=np.int32)
    off = np.ascontiguousarray(input.edge_offset, dtype=np.int32)
    nbr = np.ascontiguousarray(input.edge_neighbor, dtype=np.int32)
    dr = np.ascontiguousarray(input.edge_dr, dtype=np.float64).reshape(-1, 3)
    check(lib().hmdp_descriptors(ctx.handle, n, ptr(t), ptr(off), ptr(nbr), ptr(dr), ptr(out)))
    return out


def switch_value(r: float, rc: float) -> float:
    return float(lib().hmdp_switch_value(float(r), float(rc)))


def switch_derivative(r: float, rc: float) -> float:
    return float(lib().hmdp_switch_derivative(float(r), float(rc)))


# ---------------------------------------------------------------------------
# NNPot-style force provider: positions in, energy/forces/virial out
# ---------------------------------------------------------------------------
class ForceProvider:
    """The call a simulation engine makes every step: ``ForceFunction``
    (integrators.hpp:35) semantics -- recompute forces for the current positions,
    return the potential energy.  Backed by hmdp_compute (host buffers)."""

    def __init__(self, model: NnModel, device: int = 0, precision: Precision = Precision.fp32):
        self.model = model
        self.precision = precision
        self.ctx = Context(model, device)

    def __call__(self, positions, types, box) -> NnOutput:
        return self.ctx.compute(positions, types, box, self.precision)
