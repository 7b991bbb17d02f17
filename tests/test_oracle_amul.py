"""Pins for oracle O5 (Amul, sumA): PAPER.md P:506 (SpMVM), P:519 (sumA)."""
import json
import os

import numpy as np
import pytest

import gen
import oracle as O
from cases import dense_ldu, small_random_mesh

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _chain():
    return gen.Mesh(3, np.array([0, 1], np.int32), np.array([1, 2], np.int32), np.zeros((2, 3)), np.ones(2),
                    np.zeros((2, 3)), np.zeros((3, 3)), np.ones(3))


def test_spec_chain_and_identity():
    g = json.load(open(os.path.join(GOLD, "spec_ldu_examples.json")))
    ex = g["amul_chain"]
    y = O.amul(_chain(), ex["diag"], ex["upper"], ex["x"], lower=ex["lower"])
    assert y.tolist() == ex["y"]
    ex = g["amul_identity"]
    m = gen.Mesh(4, np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros((0, 3)), np.zeros(0), np.zeros((0, 3)),
                 np.zeros((4, 3)), np.ones(4))
    assert O.amul(m, ex["diag"], np.zeros(0), ex["x"]).tolist() == ex["y"]


@pytest.mark.parametrize("seed", range(5))
def test_amul_matches_dense_matvec(seed):
    """random 50-cell mesh -> dense oracle to 1e-14 (asymmetric lower/upper too)."""
    m = small_random_mesh(seed=seed)
    rng = np.random.default_rng(seed)
    diag = rng.uniform(-3, -1, m.n_cells)
    up = rng.uniform(0.1, 1, m.n_faces)
    lo = rng.uniform(0.1, 1, m.n_faces)
    x = rng.uniform(-1, 1, m.n_cells)
    A = dense_ldu(m.n_cells, m.owner, m.neighbour, diag, up, lo)
    y = O.amul(m, diag, up, x, lower=lo)
    ref = A @ x
    assert np.max(np.abs(y - ref)) <= 1e-14 * max(1.0, np.max(np.abs(ref)))
    # transposed: swapping lower/upper multiplies by A^T
    yt = O.amul(m, diag, lo, x, lower=up)
    assert np.max(np.abs(yt - A.T @ x)) <= 1e-14 * max(1.0, np.max(np.abs(ref)))


def test_sumA_is_amul_of_ones_bitwise():
    """S:314 sumA = amul(A, 1): identical additions, so bitwise."""
    m = small_random_mesh(seed=3)
    s = O.assemble(m, gen.gamma_lognormal(m), -1)
    assert np.array_equal(O.sumA(m, s.diag, s.upper), O.amul(m, s.diag, s.upper, np.ones(m.n_cells)))


def test_amul_linear_and_symmetric():
    m = small_random_mesh(seed=4)
    s = O.assemble(m, gen.gamma_lognormal(m), -1)
    rng = np.random.default_rng(0)
    x, y = rng.standard_normal(m.n_cells), rng.standard_normal(m.n_cells)
    Ax, Ay = O.amul(m, s.diag, s.upper, x), O.amul(m, s.diag, s.upper, y)
    assert abs(Ax @ y - x @ Ay) <= 1e-12 * np.abs(Ax).sum() * np.abs(y).max()
    assert np.allclose(O.amul(m, s.diag, s.upper, 2 * x - 3 * y), 2 * Ax - 3 * Ay, rtol=0, atol=1e-13)
