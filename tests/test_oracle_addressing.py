"""Pins for oracle O1 (addressing) and O2 (RCM renumbering).

O1 follows PAPER.md P:82-83 (lduAddressing: implicit DOF map, owner/neighbour)
and P:113 (per-cell face loops); O2 is reading Q12."""
import json
import os

import numpy as np
import pytest

import gen
import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_chain_addressing_golden():
    g = _load("spec_ldu_examples.json")["chain"]
    os_ = O.owner_start(g["n_cells"], g["owner"])
    lo, ls = O.losort(g["n_cells"], g["neighbour"])
    assert os_.tolist() == g["owner_start"]
    assert lo.tolist() == g["losort"]
    assert ls.tolist() == g["losort_start"]


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_addressing_invariants_random_mesh(seed):
    m = gen.permute(gen.box(6, 5, 4, jitter=0.2, seed=seed), seed=seed + 7)
    N, F = m.n_cells, m.n_faces
    assert O.check_addressing(N, m.owner, m.neighbour) == 0
    os_ = O.owner_start(N, m.owner)
    lo, ls = O.losort(N, m.neighbour)
    assert os_[0] == 0 and os_[N] == F and np.all(np.diff(os_) >= 0)
    assert ls[0] == 0 and ls[N] == F
    assert sorted(lo.tolist()) == list(range(F))  # a permutation
    # brute-force definitions on a small mesh
    for c in range(N):
        assert os_[c] == int(np.sum(m.owner < c))
        assert ls[c] == int(np.sum(m.neighbour < c))
        own = list(range(os_[c], os_[c + 1]))
        assert own == [f for f in range(F) if m.owner[f] == c]
        nb = lo[ls[c]:ls[c + 1]].tolist()
        assert nb == [f for f in range(F) if m.neighbour[f] == c]  # ascending face order (stable)


def test_addressing_validation_errors():
    own = np.array([0, 0, 1], np.int32)
    nb = np.array([1, 2, 2], np.int32)
    assert O.check_addressing(3, own, nb) == 0
    assert O.check_addressing(3, [1, 0, 1], [0, 2, 2]) == 2  # owner > neighbour
    assert O.check_addressing(3, [0, 0, 1], [2, 1, 2]) == 2  # not sorted by neighbour
    assert O.check_addressing(3, [1, 0, 1], [2, 2, 2]) == 2  # not sorted by owner
    assert O.check_addressing(3, [0, 0, 1], [1, 3, 2]) == 2  # out of range
    assert O.check_addressing(3, [0, -1, 1], [1, 2, 2]) == 2
    assert O.check_addressing(0, [], []) == 0


def _grid2d(n):
    return gen.box(n, n, 1, (1.0, 1.0, 0.1))


@pytest.mark.parametrize("key,n", [("grid2x2", 2), ("grid3x3", 3)])
def test_rcm_hand_examples(key, n):
    g = _load("rcm_hand.json")[key]
    m = _grid2d(n)
    perm = O.rcm(m.n_cells, m.owner, m.neighbour)
    assert perm.tolist() == g["perm"]


def test_rcm_two_components():
    g = _load("rcm_hand.json")["two_components"]
    perm = O.rcm(g["n_cells"], g["owner"], g["neighbour"])
    assert perm.tolist() == g["perm"]


def test_renumber_faces_hand():
    g = _load("rcm_hand.json")["renumber_faces_2x2"]
    o, n, fm, fl = O.renumber_faces(g["perm"], g["owner"], g["neighbour"])
    assert o.tolist() == g["owner_out"] and n.tolist() == g["neighbour_out"]
    assert fm.tolist() == g["face_map"] and fl.tolist() == g["flip"]


def _bandwidth(m):
    return int(np.max(m.neighbour - m.owner)) if m.n_faces else 0


def test_rcm_recovers_bandwidth_on_permuted_cube():
    """SURVEY §8(c) O2 pin: randomly permuted 30^3 cube -> RCM bandwidth <= 1.5 n^2."""
    n = 30
    m = gen.permute(gen.cube(n), seed=2)
    assert _bandwidth(m) > 10 * n * n
    perm = O.rcm(m.n_cells, m.owner, m.neighbour)
    assert sorted(perm.tolist()) == list(range(m.n_cells))  # bijection
    r = O.renumber_mesh(m, perm)
    assert O.check_addressing(r.n_cells, r.owner, r.neighbour) == 0
    assert _bandwidth(r) <= 1.5 * n * n


def test_renumber_keeps_geometry_closed():
    """Sf flipped iff the pair swapped: per-cell closure sum_out Sf = 0 still holds."""
    m = gen.permute(gen.perturbed(6, 0.3), seed=5)
    r = O.renumber_mesh(m, O.rcm(m.n_cells, m.owner, m.neighbour))
    acc = np.zeros((r.n_cells, 3))
    np.add.at(acc, r.owner, r.Sf)
    np.add.at(acc, r.neighbour, -r.Sf)
    for p in r.patches:
        np.add.at(acc, p.face_cells, p.Sf)
    assert np.abs(acc).max() < 1e-15
    # faces point from owner to neighbour: Sf . (C_N - C_P) > 0 on this mildly perturbed mesh
    d = r.C[r.neighbour] - r.C[r.owner]
    assert np.all(np.einsum("ij,ij->i", r.Sf, d) > 0)
