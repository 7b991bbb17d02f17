"""Degenerate inputs of the §8(f) solvers on the GPU against the oracle: no cells, one cell,
no faces (every cell isolated: the agglomeration cannot coarsen, GAMG is one level; DIC/DILU
degenerate to the diagonal), two disconnected blocks, a hierarchy of two tiny levels."""
import numpy as np
import pytest

import gen
import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import paper_2512_22215_b200 as P  # noqa: E402
from paper_2512_22215_b200 import spuma as S  # noqa: E402
from gpu_helpers import dev  # noqa: E402


def _isolated(n):
    return gen.Mesh(n, np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros((0, 3)), np.zeros(0),
                    np.zeros((0, 3)), np.zeros((n, 3)), np.ones(n), [])


def _two_blocks():
    a = gen.box(5, 3, 2, (1, 1, 1))
    b = gen.box(4, 4, 3, (1, 1, 1))
    n = a.n_cells + b.n_cells
    owner = np.concatenate([a.owner, b.owner + a.n_cells]).astype(np.int32)
    nbr = np.concatenate([a.neighbour, b.neighbour + a.n_cells]).astype(np.int32)
    return gen.Mesh(n, owner, nbr, np.concatenate([a.Sf, b.Sf]), np.concatenate([a.magSf, b.magSf]),
                    np.concatenate([a.Cf, b.Cf]), np.concatenate([a.C, b.C + 5.0]), np.concatenate([a.V, b.V]), [])


def _dominant(m, seed=0):
    """negative-definite, diagonally dominant symmetric LDU system on any addressing"""
    rng = np.random.default_rng(seed)
    upper = rng.uniform(0.1, 1.0, m.n_faces)
    off = np.zeros(m.n_cells)
    np.add.at(off, m.owner, upper)
    np.add.at(off, m.neighbour, upper)
    diag = -1.1 * off - rng.uniform(0.5, 1.0, m.n_cells)
    return diag, upper, rng.standard_normal(m.n_cells)


@pytest.mark.parametrize("make", [lambda: _isolated(1), lambda: _isolated(40), _two_blocks, lambda: gen.box(4, 3, 1)],
                         ids=["one-cell", "isolated-40", "two-blocks", "two-levels"])
def test_gamg_degenerate(make):
    m = make()
    d, u, b = _dominant(m)
    h = P.Mesh.from_mesh(m)
    hg = h.gamg_hierarchy()
    ho = O.gamg_hierarchy(m)
    assert hg["cells"] == [lv[0] for lv in ho]
    for k in range(len(ho) - 1):
        assert np.array_equal(hg["ftc"][k], ho[k][3])
    sys = O.LduSystem(d, u, b, [])
    for ctl in ((0.0, 0.0, 1, 1), (1e-12, 0.0, 200, 0)):
        psi = dev(np.zeros(m.n_cells))
        pg = h.gamg_solve(dev(d), dev(u), None, dev(b), psi, *ctl)
        psi_o, po = O.gamg(m, sys, None, O.controls(*ctl))
        assert abs(pg["n_iterations"] - po["n_iterations"]) <= 2
        x = psi.cpu().numpy()
        assert np.linalg.norm(x - psi_o) <= 1e-9 * max(np.linalg.norm(psi_o), 1e-300)
    if m.n_faces == 0:
        assert hg["levels"] == 1


def test_gamg_no_cells():
    h = P.Mesh.from_mesh(_isolated(0))
    z = torch.zeros(0, dtype=torch.float64, device="cuda")
    perf = h.gamg_solve(z, z, None, z, z, 1e-6)
    assert perf["n_iterations"] == 0


@pytest.mark.parametrize("make", [lambda: _isolated(1), lambda: _isolated(33), _two_blocks], ids=["one", "iso", "two"])
def test_preconditioned_solvers_degenerate(make):
    m = make()
    d, u, b = _dominant(m, seed=3)
    rng = np.random.default_rng(4)
    lo = u * rng.uniform(0.5, 1.5, m.n_faces)
    h = P.Mesh.from_mesh(m)
    r = rng.standard_normal(m.n_cells)
    for kind, ok in ((S.PC_DIC, O.DIC), (S.PC_DILU, O.DILU), (S.PC_ADILU, O.ADILU), (S.PC_DIAGONAL, O.DIAGONAL)):
        w = dev(np.zeros(m.n_cells))
        h.precondition(dev(d), dev(u), dev(u if ok == O.DIC else lo), dev(r), w, kind, 2)
        if ok == O.DIAGONAL:
            ref = (1.0 / d) * r
        else:
            lw = u if ok == O.DIC else lo
            rD = O.ilu_factor(m.owner, m.neighbour, d, u, lw)
            ref = O.ilu_precondition(m.owner, m.neighbour, rD, u, r, lower=lw, k=2 if ok == O.ADILU else -1)
        assert np.array_equal(w.cpu().numpy(), ref), kind
        psi = dev(np.zeros(m.n_cells))
        pg = h.pcg_solve_pc(dev(d), dev(u), dev(b), psi, 1e-12, 0.0, 500, 0, kind=kind)
        psi_o, po = O.pcg_pc(m, O.LduSystem(d, u, b, []), ok, 2, None, O.controls(1e-12, 0.0, 500, 0))
        assert abs(pg["n_iterations"] - po["n_iterations"]) <= 2 and pg["converged"]
        psi = dev(np.zeros(m.n_cells))
        pg = h.pbicg_solve(dev(d), dev(u), dev(lo), dev(b), psi, 1e-12, 0.0, 500, 0, kind=kind)
        psi_o, po = O.pbicg(m.owner, m.neighbour, d, u, lo, b, ok, 2, None, O.controls(1e-12, 0.0, 500, 0))
        assert abs(pg["n_iterations"] - po["n_iterations"]) <= 2 and pg["converged"]
        assert np.allclose(psi.cpu().numpy(), psi_o, rtol=1e-9, atol=1e-12)
