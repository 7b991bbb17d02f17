"""Pins for oracle O10: the explicit non-orthogonal correction of "Gauss linear corrected"
(laplacianSchemes P:1135, snGradSchemes corrected P:1145, gradSchemes Gauss linear P:1112).

- Gauss gradient: closure (constant field -> 0), linear exactness with exact boundary values
  (SPEC S:612), on uniform and on affine (sheared) meshes;
- correction vectors are orthogonal to the face normal and vanish on orthogonal meshes;
- the corrected scheme is exact for linear fields on affine meshes (the corrected face
  gradient is n.grad p) while the uncorrected one is not;
- the correction flux and source change vanish on orthogonal meshes."""
import numpy as np
import pytest

import gen
import oracle as O

SHEAR = np.array([[1.0, 0.35, 0.0], [0.0, 1.0, 0.0], [0.0, -0.2, 1.0]])


def _linear_bc_mesh(m, a):
    """fixedValue walls carrying the exact values of p = a . x."""
    for q in m.patches:
        m = gen.set_kind(m, q.name, gen.FIXED_VALUE, q.Cf @ a)
    return m


def test_gauss_grad_constant_is_zero():
    m = gen.perturbed(6, 0.3)
    G = O.gauss_grad(m, np.full(m.n_cells, 3.7))
    assert np.max(np.abs(G)) < 1e-12


@pytest.mark.parametrize("sheared", [False, True])
def test_gauss_grad_linear_exact(sheared):
    m = gen.box(6, 5, 4, (1.0, 1.2, 0.8))
    if sheared:
        m = gen.affine(m, SHEAR)
    a = np.array([0.7, -1.3, 2.1])
    m = _linear_bc_mesh(m, a)
    G = O.gauss_grad(m, m.C @ a)
    assert np.allclose(G, a, rtol=0, atol=1e-12)


def test_gauss_grad_zero_gradient_interior_exact():
    """f(x) = x on interior cells away from the boundary -> (1, 0, 0)."""
    n = 6
    m = gen.box(n, n, n)
    G = O.gauss_grad(m, m.C[:, 0].copy())
    i = np.arange(m.n_cells)
    ii, jj, kk = i % n, (i // n) % n, i // (n * n)
    interior = (ii > 0) & (ii < n - 1)
    assert np.allclose(G[interior], [1.0, 0.0, 0.0], rtol=0, atol=1e-12)


def test_correction_vectors_and_orthogonal_meshes():
    m = gen.cube(6)
    cf, pcf, ds, _ = O.nonorth_correction(m, np.sin(np.arange(m.n_cells)), gen.gamma_lognormal(m))
    assert np.max(np.abs(cf)) < 1e-15 and np.max(np.abs(ds)) < 1e-15  # orthogonal: no correction
    for q in pcf:
        assert np.all(q == 0.0)
    # corrVec = n - delta d is orthogonal to n (checked through a unit gradient along n)
    mp = gen.perturbed(6, 0.3)
    geo = O.geometry(mp)
    nh = mp.Sf / mp.magSf[:, None]
    d = mp.C[mp.neighbour] - mp.C[mp.owner]
    cv = nh - d * geo.delta[:, None]
    assert np.max(np.abs(np.einsum("ij,ij->i", cv, nh))) < 1e-14


def test_corrected_face_flux_exact_for_linear_field_on_sheared_mesh():
    """p = a.x on an affine mesh (exact Gauss gradient): the corrected face flux
    upper (p_N - p_P) + correction = Sf . grad p exactly on every internal face (the corrected
    snGrad is n.grad p), while the uncorrected part alone is off by O(shear)."""
    m = gen.affine(gen.box(6, 6, 5, (1.0, 1.0, 1.0)), SHEAR)
    a = np.array([0.4, 1.1, -0.6])
    m = _linear_bc_mesh(m, a)
    p = m.C @ a
    s = O.assemble(m, None, -1)
    cf, _, _, _ = O.nonorth_correction(m, p)
    unc = s.upper * (p[m.neighbour] - p[m.owner])
    exact = m.Sf @ a
    assert np.max(np.abs(unc - exact)) > 1e-3
    assert np.max(np.abs(unc + cf - exact)) < 1e-13


def test_correction_source_is_minus_volume_divergence():
    """dsource = -V surfaceIntegrate(correction flux) (fvm.source() -= V fvc::div(corr))."""
    m = gen.perturbed(7, 0.3)
    p = np.cos(np.arange(m.n_cells) * 0.3)
    cf, pcf, ds, _ = O.nonorth_correction(m, p, gen.gamma_lognormal(m))
    assert np.max(np.abs(cf)) > 1e-3
    ref = np.zeros(m.n_cells)
    np.add.at(ref, m.owner, cf)
    np.add.at(ref, m.neighbour, -cf)
    assert np.allclose(ds, -ref, rtol=1e-12, atol=1e-15)
