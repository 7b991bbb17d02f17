"""libspuma's host logic on the CPU (no device): the product's own C++ (csrc/mesh_host.cpp,
csrc/gamg_host.cpp) through the host-only C-ABI, checked against the oracle (bit-exact integer
work): RCM (Q12), the GAMG hierarchy (Q22), the DIC/DILU dependency schedules, LDU -> CSR (Q34)."""
import numpy as np
import pytest

import gen
import oracle as O
from paper_2512_22215_b200 import spuma as S

MESHES = [("cube9", lambda: gen.cube(9)), ("perturbed-permuted", lambda: gen.permute(gen.perturbed(8, 0.25), seed=3)),
          ("cavity", lambda: gen.cavity2d(13)), ("box-ragged", lambda: gen.box(11, 6, 5, (1.0, 0.7, 0.3))),
          ("cube16", lambda: gen.cube(16))]


@pytest.mark.parametrize("name,make", MESHES)
def test_host_rcm_matches_oracle(name, make):
    m = make()
    assert np.array_equal(S.host_rcm(m.n_cells, m.owner, m.neighbour), O.rcm(m.n_cells, m.owner, m.neighbour))


@pytest.mark.parametrize("params", [dict(), dict(n_coarsest=40), dict(max_levels=3)])
@pytest.mark.parametrize("name,make", MESHES)
def test_host_gamg_hierarchy_matches_oracle(name, make, params):
    m = make()
    hh = S.host_gamg_hierarchy(m.n_cells, m.owner, m.neighbour, m.magSf, params.get("n_coarsest", 10),
                               params.get("max_levels", 50))
    ho = O.gamg_hierarchy(m, O.gamg_params(n_coarsest_cells=params.get("n_coarsest", 10),
                                           max_levels=params.get("max_levels", 50)))
    assert hh["levels"] == len(ho)
    assert hh["cells"] == [lv[0] for lv in ho]
    assert hh["faces"][1:] == [int(lv[1].shape[0]) for lv in ho[1:]]
    for k in range(len(ho) - 1):
        assert np.array_equal(hh["ftc"][k], ho[k][3]), k


@pytest.mark.parametrize("name,make", MESHES)
def test_host_level_schedule_is_a_valid_topological_order(name, make):
    """Every row comes after the rows its forward (resp. backward) recurrence reads; the depth is
    the longest dependency chain (1 + max over dependencies, computed here independently)."""
    m = make()
    of, ob, df, db = S.host_level_schedule(m.n_cells, m.owner, m.neighbour)
    assert sorted(of.tolist()) == list(range(m.n_cells)) and sorted(ob.tolist()) == list(range(m.n_cells))
    pos_f, pos_b = np.empty(m.n_cells, int), np.empty(m.n_cells, int)
    pos_f[of] = np.arange(m.n_cells)
    pos_b[ob] = np.arange(m.n_cells)
    assert np.all(pos_f[m.owner] < pos_f[m.neighbour])   # forward: row neighbour reads row owner
    assert np.all(pos_b[m.neighbour] < pos_b[m.owner])   # backward: row owner reads row neighbour
    lev = np.zeros(m.n_cells, int)
    for f in np.argsort(m.neighbour, kind="stable"):
        lev[m.neighbour[f]] = max(lev[m.neighbour[f]], lev[m.owner[f]] + 1)
    assert df == lev.max() + 1


@pytest.mark.parametrize("name,make", MESHES)
def test_host_ldu_to_csr_matches_oracle(name, make):
    m = make()
    rp, col, mp = S.host_ldu_to_csr(m.n_cells, m.owner, m.neighbour)
    orp, ocol, omp = O.ldu_to_csr(m.n_cells, m.owner, m.neighbour)
    assert np.array_equal(rp, orp) and np.array_equal(col, ocol) and np.array_equal(mp, omp)


def test_host_functions_reject_bad_addressing():
    with pytest.raises(S.SpumaError):
        S.host_rcm(3, np.array([1], np.int32), np.array([0], np.int32))  # owner > neighbour
    with pytest.raises(S.SpumaError):
        S.host_ldu_to_csr(2, np.array([0, 0], np.int32), np.array([1, 1], np.int32)[::-1].copy() * 5)


def _dd_case(P, how, n=9):
    from test_oracle_decomposed import _decomposed_case
    m = gen.permute(gen.perturbed(n, 0.2), seed=4)
    part = gen.rcb_parts(m, P) if how == "rcb" else gen.block_parts(m, (P, 1, 1))
    return _decomposed_case(m, part, gen.gamma_lognormal(m), gen.rhs(m), ref=0)


@pytest.mark.parametrize("params", [dict(), dict(n_coarsest=3), dict(max_levels=3)])
@pytest.mark.parametrize("P,how", [(2, "block"), (3, "rcb"), (4, "rcb"), (8, "rcb")])
def test_host_gamg_hierarchy_dd_matches_oracle(P, how, params):
    """The decomposed hierarchy (Q36 global stop rule, Q37 coarse interfaces by first
    occurrence) of libspuma's host code -- run with one thread per rank for the collectives --
    has bitwise the decomposed oracle's per-rank level sizes and interface-face counts."""
    subs, systems = _dd_case(P, how)
    nc, ml = params.get("n_coarsest", 10), params.get("max_levels", 50)
    hh = S.host_gamg_hierarchy_dd(subs, nc, ml)
    _, po = O.gamg_decomposed(subs, systems, None, O.controls(0.0, 0.0, 0, 0),
                              O.gamg_params(n_coarsest_cells=nc, max_levels=ml))
    assert hh["levels"] == po["levels"]
    assert hh["level_cells"] == po["level_cells"]
    assert hh["level_ifaces"] == po["level_ifaces"]
    assert hh["levels"] >= (3 if ml > 3 else ml)


def _offsets_by_definition(m):
    """The lattice test written out: the distinct column offsets of the faces (at most 3) and no
    repeated (owner, neighbour) pair."""
    d = sorted(set((m.neighbour - m.owner).tolist()))
    pairs = set(zip(m.owner.tolist(), m.neighbour.tolist()))
    return d if (0 < len(d) <= 3 and len(pairs) == m.n_faces) else []


@pytest.mark.parametrize("name,make,expect", [
    ("cube5", lambda: gen.cube(5), [1, 5, 25]),
    ("cube200-like box", lambda: gen.box(7, 3, 2), [1, 7, 21]),
    ("cavity2d", lambda: gen.cavity2d(20), [1, 20]),
    ("chain", lambda: gen.box(9, 1, 1), [1]),
    ("perturbed", lambda: gen.perturbed(6, 0.3), [1, 6, 36]),
    ("weak block (rank 1 of 2x2x1)", lambda: gen.weak_block(6, (2, 2, 1), 1), [1, 6, 36]),
    ("permuted", lambda: gen.permute(gen.cube(5), seed=2), []),
])
def test_host_lattice_offsets(name, make, expect):
    """Amul variant 12 runs exactly on the meshes whose faces take <= 3 column offsets."""
    m = make()
    got = S.host_lattice_offsets(m.n_cells, m.owner, m.neighbour)
    assert got == expect == _offsets_by_definition(m)


def test_host_lattice_offsets_rejects_repeated_pairs_and_four_offsets():
    # two faces between cells 0 and 1 (legal lduAddressing, not a lattice)
    o, nb = np.array([0, 0, 1], np.int32), np.array([1, 1, 2], np.int32)
    assert S.host_lattice_offsets(3, o, nb) == []
    # offsets {1, 2, 3, 4}
    o, nb = np.array([0, 0, 0, 0], np.int32), np.array([1, 2, 3, 4], np.int32)
    assert S.host_lattice_offsets(5, o, nb) == []
    assert S.host_lattice_offsets(5, o[:3], nb[:3]) == [1, 2, 3]
    assert S.host_lattice_offsets(1, np.zeros(0, np.int32), np.zeros(0, np.int32)) == []
