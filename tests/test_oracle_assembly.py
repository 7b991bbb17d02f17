"""Pins for oracle O3 (geometry) and O4 (assembly of fvm::laplacian).

O3: "Gauss linear corrected" / linear interpolation,
reading Q6.  O4: P:736 ("P assembly"), P:520 (negSumDiag)
(pRefCell/pRefValue), readings Q7, Q9, Q15."""
import json
import os

import numpy as np
import pytest

import gen
import oracle as O
from cases import dense_ldu, dirichlet_box, small_random_mesh

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def ulp_close(a, b, k):
    a, b = np.asarray(a), np.asarray(b)
    return np.all(np.abs(a - b) <= k * np.spacing(np.maximum(np.abs(a), np.abs(b))))


# ----------------------------------------------------------------------- O3
@pytest.mark.parametrize("n", [4, 8, 16])
def test_uniform_geometry_closed_form(n):
    """h = 1/n exactly representable: delta = 1/h, w = 1/2, delta_b = 2/h to <= 2 ulp."""
    m = gen.cube(n)
    g = O.geometry(m)
    assert ulp_close(g.delta, float(n), 2)  # delta = 1/h
    assert ulp_close(g.weights, 0.5, 2)
    assert ulp_close(g.bdelta, 2.0 * n, 2)  # half-cell distance to the wall


@pytest.mark.parametrize("n", [7, 20])
def test_uniform_geometry_closed_form_rounded_vertices(n):
    """h = 1/n not representable: vertex rounding perturbs widths by ~n ulp(1)."""
    m = gen.cube(n)
    g = O.geometry(m)
    assert np.allclose(g.delta, n, rtol=n * 1e-15, atol=0)
    assert np.allclose(g.weights, 0.5, rtol=n * 1e-15, atol=0)
    assert np.allclose(g.bdelta, 2.0 * n, rtol=n * 1e-15, atol=0)


def test_geometry_bounds_perturbed():
    m = gen.perturbed(8, 0.3)
    g = O.geometry(m)
    d = np.linalg.norm(m.C[m.neighbour] - m.C[m.owner], axis=1)
    assert np.all(g.delta * d >= 1.0 - 1e-14) and np.all(g.delta * d <= 20.0 + 1e-12)
    assert np.all((g.weights >= 0) & (g.weights <= 1))
    assert np.all(g.bdelta > 0)


def test_delta_stabiliser_clamp():
    """Face normal > 87.1 deg from d: nonOrthDeltaCoeffs = 1/(0.05 |d|) (Q6)."""
    ang = np.deg2rad(89.0)
    S = np.array([[np.cos(ang), np.sin(ang), 0.0]])
    m = gen.Mesh(2, np.array([0], np.int32), np.array([1], np.int32), S, np.array([1.0]),
                 np.array([[0.5, 0.0, 0.0]]), np.array([[0.0, 0.0, 0.0], [2.0, 0.0, 0.0]]), np.ones(2))
    g = O.geometry(m)
    assert g.delta[0] == 1.0 / (0.05 * 2.0)
    ang = np.deg2rad(80.0)
    m.Sf[0] = [np.cos(ang), np.sin(ang), 0.0]
    g = O.geometry(m)
    assert abs(g.delta[0] - 1.0 / (2.0 * np.cos(ang))) < 1e-12


def test_weights_closed_form_nonuniform():
    """w = |Sf.(C_N - Cf)| / (|Sf.(Cf - C_P)| + |Sf.(C_N - Cf)|): graded 1-D cells of widths 1 and 3."""
    m = gen.Mesh(2, np.array([0], np.int32), np.array([1], np.int32), np.array([[1.0, 0, 0]]), np.array([1.0]),
                 np.array([[1.0, 0, 0]]), np.array([[0.5, 0, 0], [2.5, 0, 0]]), np.ones(2))
    g = O.geometry(m)
    assert g.weights[0] == 0.75 and g.delta[0] == 0.5


# ----------------------------------------------------------------------- O4
def test_spec_chain_negsumdiag():
    g = json.load(open(os.path.join(GOLD, "spec_ldu_examples.json")))
    ex = g["negSumDiag_chain"]
    m = gen.Mesh(3, np.array([0, 1], np.int32), np.array([1, 2], np.int32), np.zeros((2, 3)), np.ones(2),
                 np.zeros((2, 3)), np.zeros((3, 3)), np.ones(3))
    # upper = delta * (1 * magSf) with delta = -1 reproduces the SPEC chain lower = upper = -1
    geo = O.Geometry(np.array([-1.0, -1.0]), np.full(2, 0.5), np.zeros(0), np.zeros(0))
    s = O.assemble(m, None, -1, geo=geo)
    assert s.upper.tolist() == ex["upper"]
    assert s.diag.tolist() == ex["diag"]


@pytest.mark.parametrize("n", [3, 6])
def test_uniform_3d_closed_form_and_invariants(n):
    """Unit-spaced cube (h = 1): upper = |S|/h = 1, interior diag = -6, row sums exactly 0."""
    m = gen.box(n, n, n, (float(n),) * 3)
    s = O.assemble(m, None, -1)
    assert np.all(s.upper == 1.0)
    interior = np.array([c for c in range(m.n_cells)
                         if all(0 < (c // (n ** d)) % n < n - 1 for d in range(3))])
    assert np.all(s.diag[interior] == -6.0)
    rows = O.sumA(m, s.diag, s.upper)
    assert np.all(rows == 0.0)  # zero row sums with all-Neumann walls (exact: integer coefficients)
    assert s.diag.sum() == -2.0 * s.upper.sum()
    assert np.all(s.source == 0.0)


def test_uniform_2d_cavity_coefficients():
    """Cavity 0.1 x 0.1 x 0.01, 20 x 20: upper = dz = 0.01 (gamma = 1), interior diag = -4 dz."""
    m = gen.cavity2d(20)
    s = O.assemble(m, None, -1)
    # vertices 0.1 i / 20 are rounded, so widths carry ~20 ulp(0.1) of jitter
    assert np.allclose(s.upper, 0.01, rtol=1e-13, atol=0)
    i = np.arange(400)
    interior = (i % 20 > 0) & (i % 20 < 19) & (i // 20 > 0) & (i // 20 < 19)
    assert np.allclose(s.diag[interior], -0.04, rtol=1e-13, atol=0)
    rows = O.sumA(m, s.diag, s.upper)
    assert np.all(np.abs(rows) <= 4 * np.spacing(0.04))


def test_random_mesh_matches_dense_definition_and_invariants():
    m = small_random_mesh()
    gamma = gen.gamma_lognormal(m)
    s = O.assemble(m, gamma, -1)
    geo = O.geometry(m)
    # symmetric, negative diagonal, positive off-diagonals, ~zero row sums (Neumann)
    A = dense_ldu(m.n_cells, m.owner, m.neighbour, s.diag, s.upper)
    assert np.array_equal(A, A.T)
    assert np.all(s.diag < 0) and np.all(s.upper > 0)
    rows = A.sum(axis=1)
    scale = np.zeros(m.n_cells)
    np.add.at(scale, m.owner, s.upper)
    np.add.at(scale, m.neighbour, s.upper)
    assert np.all(np.abs(rows) <= 4 * np.spacing(scale))
    # coefficients follow the definition (linear interpolation of gamma, Q6)
    gf = geo.weights * (gamma[m.owner] - gamma[m.neighbour]) + gamma[m.neighbour]
    assert np.array_equal(s.upper, geo.delta * (gf * m.magSf))
    # oracle's own dense builder agrees with the definition
    assert np.array_equal(O.dense_from_ldu(m, diag=s.diag, upper=s.upper), A)


def test_fixed_value_face_adds_minus_two_S_over_h():
    n = 4
    m = gen.box(n, n, n, (float(n),) * 3)
    s0 = O.assemble(m, None, -1)
    val = np.full(n * n, 3.0)
    mf = gen.set_kind(m, "xmin", gen.FIXED_VALUE, val)
    s1 = O.assemble(mf, None, -1)
    cells = mf.patches[0].face_cells
    dd = s1.diag - s0.diag
    assert np.all(dd[cells] == -2.0)  # |S| = 1, h = 1: -|S| delta_b with delta_b = 2/h
    mask = np.ones(m.n_cells, bool)
    mask[cells] = False
    assert np.all(dd[mask] == 0.0)
    assert np.all(s1.source[cells] == -2.0 * 3.0)  # -(gamma|S|)(delta_b p_b)


def test_set_reference_doubles_one_diagonal():
    m = small_random_mesh()
    s0 = O.assemble(m, None, -1)
    src = np.linspace(-1, 1, m.n_cells)
    s1 = O.assemble(m, None, 7, 2.5, source=src)
    assert s1.diag[7] == 2.0 * s0.diag[7]
    assert s1.source[7] == src[7] + s0.diag[7] * 2.5
    k = np.arange(m.n_cells) != 7
    assert np.array_equal(s1.diag[k], s0.diag[k]) and np.array_equal(s1.source[k], src[k])


def test_empty_and_zero_gradient_add_nothing():
    m = gen.cavity2d(6)
    s = O.assemble(m, gen.gamma_lognormal(m), -1)
    rows = O.sumA(m, s.diag, s.upper)
    assert np.all(np.abs(rows) <= 8 * np.spacing(np.abs(s.diag)))
