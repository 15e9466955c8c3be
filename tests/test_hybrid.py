"""NNPot hybrid coupling, host side: plan_group_preprocessing against the SPEC's
known-answer examples.  CPU only."""
import math

import pytest

from paper_2602_02234_b200.hybrid import (Topology, plan_group_preprocessing, synthetic_topology,
                                          undo_group_preprocessing)


def chain(n, excl=False):
    t = Topology(n)
    t.bonds = [(i, i + 1) for i in range(n - 1)]
    t.angles = [(i, i + 1, i + 2) for i in range(n - 2)]
    t.dihedrals = [(i, i + 1, i + 2, i + 3) for i in range(n - 3)]
    if excl:
        for i, j in t.bonds:
            t.add_exclusion(i, j)
    t.groups["all"] = list(range(n))
    t.groups["none"] = []
    t.groups["head"] = list(range(5))
    return t


def n_excl(t):
    return sum(len(e) for e in t.exclusions) // 2


def test_group_all_atoms_is_total_takeover():
    t = chain(10)
    t2, plan = plan_group_preprocessing(t, "all")
    assert t2.bonds == [] and t2.angles == [] and t2.dihedrals == []
    assert n_excl(t2) == math.comb(10, 2)


def test_empty_group_is_identity():
    t = chain(10, excl=True)
    t2, plan = plan_group_preprocessing(t, "none")
    assert (t2.bonds, t2.angles, t2.dihedrals, t2.exclusions) == \
        (t.bonds, t.angles, t.dihedrals, t.exclusions)
    assert plan.added_exclusions == []


def test_ten_atom_chain_head_group():
    """bonds (0,1)..(3,4) removed; bond (4,5) retained; exclusions gain
    C(5,2) = 10 pairs."""
    t = chain(10)
    t2, plan = plan_group_preprocessing(t, "head")
    assert plan.removed_bonds == [(0, 1), (1, 2), (2, 3), (3, 4)]
    assert (4, 5) in t2.bonds and len(t2.bonds) == 5
    assert n_excl(t2) - n_excl(t) == 10
    # cross-group terms untouched: angles/dihedrals with an atom outside the group stay
    assert all(not set(a) <= set(range(5)) for a in t2.angles)
    assert (3, 4, 5) in t2.angles and (2, 3, 4, 5) in t2.dihedrals


def test_existing_exclusions_not_double_counted_and_undo():
    t = chain(10, excl=True)
    t2, plan = plan_group_preprocessing(t, "head")
    assert len(plan.added_exclusions) == 10 - 4  # (0,1)..(3,4) were already excluded
    for i in range(5):
        for j in range(5):
            if i != j:
                assert t2.excluded(i, j) and t2.excluded(j, i)
    t3 = undo_group_preprocessing(t2, plan)
    assert sorted(t3.bonds) == sorted(t.bonds) and sorted(t3.angles) == sorted(t.angles)
    assert t3.exclusions == t.exclusions


def test_unknown_group():
    with pytest.raises(ValueError, match="unknown atom group"):
        plan_group_preprocessing(chain(4), "protein")


def test_synthetic_topology_matches_generator_shape():
    t = synthetic_topology(582)
    ng = math.ceil(0.35 * 582)
    assert t.groups["protein"] == list(range(ng)) and len(t.groups["solvent"]) == 582 - ng
    t2, plan = plan_group_preprocessing(t, "protein")
    assert t2.bonds == [] and t2.angles == [] and t2.dihedrals == []  # the chain is the protein
    assert n_excl(t2) == math.comb(ng, 2)
