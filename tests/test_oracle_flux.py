"""Pins for oracle O9 (the steps around the path):

- fvc::surfaceIntegrate (profile row "surfaceIntegrate")
  -- the pressure source fvc::div(phiHbyA);
- fvMatrix::flux = lduMatrix::faceH + boundary contributions --
  the SIMPLE flux correction phi = phiHbyA - pEqn.flux().

Pins: Gauss theorem on linear velocity fields (exact for planar faces), closure,
linear-solution fluxes, the SPEC faceH chain example, the discrete conservation
identity V surfaceIntegrate(flux(psi)) = A psi - (boundary source) and the
divergence-free corrected flux of a solved pressure equation."""
import json
import os

import numpy as np
import pytest

import gen
import oracle as O
from cases import dense_ldu

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _flux_of(mesh, U):
    """phi_f = U(Cf) . Sf for a velocity field U(x) (internal faces and per-patch)."""
    phi = np.einsum("ij,ij->i", U(mesh.Cf), mesh.Sf)
    pphi = [np.einsum("ij,ij->i", U(p.Cf), p.Sf) for p in mesh.patches]
    return phi, pphi


@pytest.mark.parametrize("dims,L", [((6, 5, 4), (1.0, 2.0, 0.5)), ((8, 8, 8), (1.0, 1.0, 1.0))])
def test_surface_integrate_gauss_theorem_linear_field(dims, L):
    """U = (a x + b, c y + d, e z): div U = a + c + e exactly on planar-faced hexes."""
    m = gen.box(*dims, L)
    a, c, e = 1.5, -0.25, 3.0
    U = lambda X: np.stack([a * X[:, 0] + 0.3, c * X[:, 1] - 1.0, e * X[:, 2]], axis=1)
    phi, pphi = _flux_of(m, U)
    div = O.surface_integrate(m, phi, pphi)
    assert np.allclose(div, a + c + e, rtol=1e-12, atol=1e-12)


def test_surface_integrate_closure_and_sign():
    m = gen.perturbed(6, 0.3)
    phi, pphi = _flux_of(m, lambda X: np.tile([0.7, -1.2, 0.4], (X.shape[0], 1)))
    assert np.max(np.abs(O.surface_integrate(m, phi, pphi) * m.V)) < 1e-14  # constant U: sum_out Sf = 0
    # a single internal face flux leaves its owner (+) and enters its neighbour (-)
    z = np.zeros(m.n_faces)
    z[17] = 2.5
    d = O.surface_integrate(m, z, None) * m.V
    assert d[m.owner[17]] == pytest.approx(2.5, rel=1e-15) and d[m.neighbour[17]] == pytest.approx(-2.5, rel=1e-15)
    assert np.count_nonzero(d) == 2
    # empty patches contribute nothing
    c = gen.cavity2d(5)
    pp = [np.ones(p.n_faces) for p in c.patches]
    d = O.surface_integrate(c, np.zeros(c.n_faces), pp) * c.V
    exp = np.zeros(c.n_cells)
    for p in c.patches:
        if p.kind != gen.EMPTY:
            np.add.at(exp, p.face_cells, 1.0)
    assert np.allclose(d, exp, rtol=1e-14, atol=0)


def test_spec_faceH_chain():
    """3-chain, x = [1,2,3], lower = upper = [-1,-1] -> faceH = [-1,-1]."""
    m = gen.Mesh(3, np.array([0, 1], np.int32), np.array([1, 2], np.int32), np.zeros((2, 3)), np.ones(2),
                 np.zeros((2, 3)), np.zeros((3, 3)), np.ones(3))
    geo = O.Geometry(np.ones(2), np.full(2, 0.5), np.zeros(0), np.zeros(0))
    flux, _ = O.face_flux(m, np.array([-1.0, -1.0]), np.array([1.0, 2.0, 3.0]), geo=geo)
    assert flux.tolist() == [-1.0, -1.0]
    flux, _ = O.face_flux(m, np.array([-1.0, -1.0]), np.full(3, 4.0), geo=geo)  # constant field: 0
    assert flux.tolist() == [0.0, 0.0]


def test_flux_of_linear_solution_is_face_area():
    """psi = x on a unit-spaced box (gamma = 1): x-face flux = |S| (dpsi/dx = 1), y/z faces 0;
    fixedValue x-walls with the exact values carry the same flux."""
    n = 5
    m = gen.box(n, n, n, (float(n),) * 3)
    m = gen.set_kind(m, "xmin", gen.FIXED_VALUE, np.zeros(n * n))
    m = gen.set_kind(m, "xmax", gen.FIXED_VALUE, np.full(n * n, float(n)))
    s = O.assemble(m, None, -1)
    psi = m.C[:, 0].copy()
    flux, pf = O.face_flux(m, s.upper, psi)
    xface = (m.neighbour - m.owner) == 1
    assert np.all(flux[xface] == 1.0) and np.all(flux[~xface] == 0.0)
    assert np.all(pf[0] == -1.0) and np.all(pf[1] == 1.0)  # outward: in at xmin, out at xmax
    for k in range(2, 6):
        assert np.all(pf[k] == 0.0)  # zeroGradient


def test_conservation_identity():
    """V surfaceIntegrate(flux(psi)) = A psi - source (no reference cell): the discrete divergence of
    the matrix flux is the matrix itself."""
    m = gen.permute(gen.perturbed(7, 0.25), seed=5)
    m = gen.set_kind(m, "zmax", gen.FIXED_VALUE, np.linspace(-1, 1, m.patches[5].n_faces))
    g = gen.gamma_lognormal(m)
    s = O.assemble(m, g, -1)
    psi = np.sin(np.arange(m.n_cells) * 0.21)
    flux, pf = O.face_flux(m, s.upper, psi, gamma=g)
    lhs = O.surface_integrate(m, flux, pf) * m.V
    rhs = O.amul(m, s.diag, s.upper, psi) - s.source
    assert np.allclose(lhs, rhs, rtol=0, atol=1e-12 * np.max(np.abs(rhs)))


def test_corrected_flux_is_divergence_free():
    """SIMPLE: b = V div(phiHbyA); solve A p = b; phi = phiHbyA - flux(p) has V div(phi) = b - A p,
    i.e. the linear-solver residual (Neumann walls, reference cell: the penalty row differs)."""
    m = gen.perturbed(8, 0.15)
    g = gen.gamma_lognormal(m)
    rng = np.random.default_rng(3)
    phiH = rng.standard_normal(m.n_faces) * 1e-3
    pzero = [np.zeros(p.n_faces) for p in m.patches]
    b = O.surface_integrate(m, phiH, pzero) * m.V
    s = O.assemble(m, g, 0, 0.0, source=b)
    psi, perf = O.pcg(m, s, None, O.controls(1e-12))
    flux, pf = O.face_flux(m, s.upper, psi, gamma=g)
    div = O.surface_integrate(m, phiH - flux, [a - c for a, c in zip(pzero, pf)]) * m.V
    A = dense_ldu(m.n_cells, m.owner, m.neighbour, s.diag, s.upper)
    r = s.source - A @ psi
    k = np.arange(m.n_cells) != 0  # the reference row carries the setReference penalty
    assert np.allclose(div[k], r[k], rtol=0, atol=1e-15)
    assert np.sum(np.abs(div[k])) < 1e-10 * np.sum(np.abs(b))
