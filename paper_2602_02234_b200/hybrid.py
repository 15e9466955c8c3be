"""NNPot-style hybrid coupling (SPEC.md:375-383 plan_group_preprocessing,
SPEC.md:411-419 nn_force_provider; the paper's Fig. 2): the DP model runs on one
atom group (the "protein", synthetic.cpp:100-102) and its forces are scattered into
the global force array; every other term -- including all cross-group
interactions -- stays with the caller's classical force field.

The reference declares this contract but ships no code for it; the C++ drop-in
(include/hmdp_halomd.hpp) and this module follow it on the reference's Topology
shape (topology.hpp): bonded terms, symmetric sorted exclusions, named groups.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from ._lib import check, lib, ptr
from .nn import Context, Precision, _box3


@dataclass
class Topology:
    """Connectivity of halomd::Topology (topology.hpp:30-48): bonds (i, j),
    angles (i, j, k), dihedrals (i, j, k, l), exclusions[i] sorted and symmetric,
    named groups (sorted, duplicate-free)."""
    n_atoms: int
    bonds: list = field(default_factory=list)
    angles: list = field(default_factory=list)
    dihedrals: list = field(default_factory=list)
    exclusions: list = field(default_factory=list)
    groups: dict = field(default_factory=dict)

    def __post_init__(self):
        if not self.exclusions:
            self.exclusions = [[] for _ in range(self.n_atoms)]

    def excluded(self, i: int, j: int) -> bool:
        return j in self.exclusions[i]

    def add_exclusion(self, i: int, j: int) -> None:
        for a, b in ((i, j), (j, i)):
            if b not in self.exclusions[a]:
                self.exclusions[a].append(b)
                self.exclusions[a].sort()

    def copy(self) -> "Topology":
        return Topology(self.n_atoms, list(self.bonds), list(self.angles), list(self.dihedrals),
                        [list(e) for e in self.exclusions],
                        {k: list(v) for k, v in self.groups.items()})


def synthetic_topology(n_atoms: int, fraction_grouped: float = 0.35) -> Topology:
    """Connectivity of generate_synthetic_system (synthetic.cpp:52, :88-103): a
    chain over the first ceil(fraction * n) atoms (group "protein") with bonds,
    angles, dihedrals and 1-2 / 1-3 exclusions; the rest is group "solvent"."""
    ng = int(math.ceil(fraction_grouped * n_atoms))
    t = Topology(n_atoms)
    t.bonds = [(i, i + 1) for i in range(ng - 1)]
    t.angles = [(i, i + 1, i + 2) for i in range(ng - 2)]
    t.dihedrals = [(i, i + 1, i + 2, i + 3) for i in range(ng - 3)]
    for i, j in t.bonds:
        t.add_exclusion(i, j)
    for i, _, k in t.angles:
        t.add_exclusion(i, k)
    t.groups["protein"] = list(range(ng))
    t.groups["solvent"] = list(range(ng, n_atoms))
    return t


@dataclass
class NnGroupPlan:
    """What plan_group_preprocessing removed / added (reversible)."""
    group: str
    atoms: np.ndarray
    removed_bonds: list
    removed_angles: list
    removed_dihedrals: list
    added_exclusions: list


def plan_group_preprocessing(topo: Topology, group: str) -> tuple[Topology, NnGroupPlan]:
    """topo' lacks every bonded term fully inside the group; all
    in-group pairs are excluded (symmetrically); cross-group terms and pairs are
    untouched; the plan records everything (undo_group_preprocessing).  An empty
    group is a no-op.  Unknown group -> ValueError (std::invalid_argument)."""
    if group not in topo.groups:
        raise ValueError(f"unknown atom group: {group}")
    atoms = list(topo.groups[group])
    t = topo.copy()
    inside = set(atoms)
    keep = lambda terms: [x for x in terms if not set(x) <= inside]  # noqa: E731
    gone = lambda terms: [x for x in terms if set(x) <= inside]  # noqa: E731
    plan = NnGroupPlan(group, np.asarray(atoms, dtype=np.int32), gone(t.bonds), gone(t.angles),
                       gone(t.dihedrals), [])
    if not atoms:
        return t, plan
    t.bonds, t.angles, t.dihedrals = keep(t.bonds), keep(t.angles), keep(t.dihedrals)
    for p, i in enumerate(atoms):
        for j in atoms[p + 1:]:
            if not t.excluded(i, j):
                t.add_exclusion(i, j)
                plan.added_exclusions.append((i, j))
    return t, plan


def undo_group_preprocessing(topo: Topology, plan: NnGroupPlan) -> Topology:
    t = topo.copy()
    t.bonds += plan.removed_bonds
    t.angles += plan.removed_angles
    t.dihedrals += plan.removed_dihedrals
    for i, j in plan.added_exclusions:
        t.exclusions[i].remove(j)
        t.exclusions[j].remove(i)
    return t


def nn_force_provider(ctx: Context, positions, types, box, plan: NnGroupPlan, forces,
                      precision: Precision = Precision.fp32) -> float:
    """extract the group's positions (gathered on the device),
    run the DP model on them, ADD their forces into `forces` [n, 3] in place and
    return the NN energy (hmdp_compute_group)."""
    x = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1, 3)
    t = np.ascontiguousarray(types, dtype=np.int32)
    n = x.shape[0]
    if t.shape[0] != n or forces.shape != (n, 3) or forces.dtype != np.float64 \
            or not forces.flags.c_contiguous:
        raise ValueError("positions/types/forces size mismatch")
    g = np.ascontiguousarray(plan.atoms, dtype=np.int32)
    b = _box3(box)
    e = ctypes.c_double()
    check(lib().hmdp_compute_group(ctx.handle, n, ptr(x), ptr(t), ptr(g), int(g.shape[0]),
                                   ptr(b), int(precision), ctypes.byref(e), ptr(forces), None,
                                   None))
    return e.value
