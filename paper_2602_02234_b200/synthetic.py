"""Synthetic protein-in-water fixture (generate_synthetic_system,
/root/reference/proj/src/synthetic.cpp:36-130), reproduced bit-for-bit by the
host side of libhmdp (mt19937_64 + the reference's hand-rolled distributions).
Only the NN-relevant outputs are produced: positions, types, masses,
velocities (Maxwell-Boltzmann at `temperature`, COM removed) and the box."""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from ._lib import check, lib, ptr

# The paper's benchmark systems and the survey's canonical inputs
# (density 33.4 nm^-3, fraction_grouped 0.35, seed 7).
PAPER_SYSTEMS = {"1YRF": 582, "1UBQ": 1231, "3LZM": 2643, "2PTC": 4114}
DENSITY = 33.4
FRACTION_GROUPED = 0.35
SEED = 7


@dataclass
class SyntheticSystem:
    positions: np.ndarray  # [n,3] nm
    types: np.ndarray      # [n] int32, 0 = protein analog, 1 = solvent
    masses: np.ndarray     # [n] amu
    velocities: np.ndarray  # [n,3] nm/ps
    box: np.ndarray        # [3] nm

    @property
    def n_atoms(self) -> int:
        return int(self.types.shape[0])


def generate_synthetic_system(n_atoms: int = 582, density: float = DENSITY,
                              fraction_grouped: float = FRACTION_GROUPED, seed: int = SEED,
                              temperature: float = 300.0) -> SyntheticSystem:
    n = int(n_atoms)
    x = np.zeros((n, 3))
    v = np.zeros((n, 3))
    t = np.zeros(n, dtype=np.int32)
    m = np.zeros(n)
    b = np.zeros(3)
    check(lib().hmdp_synthetic_system(n, float(density), float(fraction_grouped),
                                      ctypes.c_uint64(seed), float(temperature), ptr(x), ptr(t),
                                      ptr(m), ptr(v), ptr(b)))
    return SyntheticSystem(positions=x, types=t, masses=m, velocities=v, box=b)


def replicate(sys: SyntheticSystem, reps=(2, 2, 2)) -> SyntheticSystem:
    """Periodic replica box (weak scaling; extensivity)."""
    rx, ry, rz = reps
    shifts = np.array([(i, j, k) for k in range(rz) for j in range(ry) for i in range(rx)], float)
    shifts *= sys.box
    n = sys.n_atoms
    pos = (sys.positions[None, :, :] + shifts[:, None, :]).reshape(-1, 3)
    rep = shifts.shape[0]
    return SyntheticSystem(positions=pos, types=np.tile(sys.types, rep),
                           masses=np.tile(sys.masses, rep),
                           velocities=np.tile(sys.velocities, (rep, 1)),
                           box=sys.box * np.array(reps, float))
