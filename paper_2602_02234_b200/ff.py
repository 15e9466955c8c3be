"""Classical force field on the device (include/hmdp.h hmdp_ff_*): the reference's
compute_classical (/root/reference/proj/src/forcefield.cpp:265-279) — harmonic bonds,
angles, periodic dihedrals, potential-shifted Lennard-Jones (Lorentz-Berthelot) and
Coulomb (cutoff_shifted or reaction_field) — over the device cell-list pairs minus the
topology's exclusions.  The solvent and cross-group half of the NNPot hybrid step
(SPEC.md:411-419), so protein (DP) + water (classical) stays on the GPU."""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from ._lib import check, lib, ptr
from .nn import Precision, _box3


@dataclass
class ClassicalResult:
    bonded: float
    lj: float
    coulomb: float
    forces: np.ndarray
    virial: float
    collinear_angles: int

    def total_potential(self) -> float:
        return self.bonded + self.lj + self.coulomb


class ClassicalFF:
    """Device copy of a halomd Topology + ForceFieldParams (forcefield.hpp:16-43)."""

    def __init__(self, types, charges, sigma, epsilon, excl_offset, excl, bonds=None,
                 bond_params=None, angles=None, angle_params=None, dihedrals=None,
                 dihedral_params=None, coulomb_scheme: int = 0, rc_coulomb: float = 0.7,
                 eps_rf: float = 78.0, rc_lj: float = 0.7, device: int = 0):
        t = np.ascontiguousarray(types, dtype=np.int32)
        self.n = int(t.shape[0])
        arrs = dict(
            q=np.ascontiguousarray(charges, dtype=np.float64),
            sig=np.ascontiguousarray(sigma, dtype=np.float64),
            eps=np.ascontiguousarray(epsilon, dtype=np.float64),
            eo=np.ascontiguousarray(excl_offset, dtype=np.int32),
            ex=np.ascontiguousarray(excl if excl is not None and len(excl) else [0], dtype=np.int32),
        )

        def terms(idx, par, k, m):
            a = np.ascontiguousarray(idx if idx is not None else np.zeros((0, k)), dtype=np.int32)
            b = np.ascontiguousarray(par if par is not None else np.zeros((0, m)), dtype=np.float64)
            return a.reshape(-1, k), b.reshape(-1, m)

        bi, bp = terms(bonds, bond_params, 2, 2)
        ai, ap = terms(angles, angle_params, 3, 2)
        di, dp = terms(dihedrals, dihedral_params, 4, 3)
        h = ctypes.c_void_p()
        check(lib().hmdp_ff_create(device, self.n, ptr(t), ptr(arrs["q"]), int(arrs["sig"].shape[0]),
                                   ptr(arrs["sig"]), ptr(arrs["eps"]), int(coulomb_scheme),
                                   float(rc_coulomb), float(eps_rf), float(rc_lj), ptr(arrs["eo"]),
                                   ptr(arrs["ex"]), bi.shape[0], ptr(bi), ptr(bp), ai.shape[0],
                                   ptr(ai), ptr(ap), di.shape[0], ptr(di), ptr(dp), ctypes.byref(h)))
        self.handle = h

    def compute(self, positions, box, precision: Precision = Precision.fp64) -> ClassicalResult:
        x = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1, 3)
        if x.shape[0] != self.n:
            raise ValueError("positions size mismatch")
        b = _box3(box)
        e = np.zeros(3)
        f = np.zeros((self.n, 3))
        w = ctypes.c_double()
        c = ctypes.c_int()
        check(lib().hmdp_ff_compute(self.handle, ptr(x), ptr(b), int(precision), ptr(e), ptr(f),
                                    ctypes.byref(w), ctypes.byref(c)))
        return ClassicalResult(float(e[0]), float(e[1]), float(e[2]), f, w.value, c.value)

    def close(self):
        if getattr(self, "handle", None):
            lib().hmdp_ff_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class HybridMD:
    """Hybrid device MD (include/hmdp.h hmdp_hybrid_*): classical force field on every
    atom + the DP model on one sorted atom group (the paper's NNPot coupling,
    SPEC.md:411-419), summed forces, velocity Verlet, one CUDA graph per
    ``steps_per_graph`` steps."""

    def __init__(self, ctx, ff: ClassicalFF, group, positions, velocities, masses, types, box,
                 dt_ps=0.001, precision: Precision = Precision.fp64, steps_per_graph: int = 10):
        g = np.ascontiguousarray(group, dtype=np.int32)
        x = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1, 3)
        v = np.ascontiguousarray(velocities, dtype=np.float64).reshape(-1, 3)
        m = np.ascontiguousarray(masses, dtype=np.float64)
        t = np.ascontiguousarray(types, dtype=np.int32)
        b = _box3(box)
        self.n = x.shape[0]
        self.ctx, self.ff = ctx, ff  # keep both alive
        h = ctypes.c_void_p()
        check(lib().hmdp_hybrid_create(ctx.handle, ff.handle, self.n, ptr(g), g.shape[0], ptr(x),
                                       ptr(v), ptr(m), ptr(t), ptr(b), float(dt_ps), int(precision),
                                       int(steps_per_graph), ctypes.byref(h)))
        self.handle = h

    def run(self, steps: int) -> None:
        check(lib().hmdp_hybrid_run(self.handle, int(steps)))

    def state(self):
        """(x, v, F, energies[bonded, lj, coulomb, nn]); x / v are the next step's
        drifted positions and half-kicked velocities (velocity Verlet split)."""
        x = np.zeros((self.n, 3))
        v = np.zeros((self.n, 3))
        f = np.zeros((self.n, 3))
        e = np.zeros(4)
        check(lib().hmdp_hybrid_get(self.handle, ptr(x), ptr(v), ptr(f), ptr(e)))
        return x, v, f, e

    def close(self):
        if getattr(self, "handle", None):
            lib().hmdp_hybrid_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
