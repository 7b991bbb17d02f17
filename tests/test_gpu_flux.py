"""GPU parity of the steps around the path: spuma_surface_integrate
(fvc::surfaceIntegrate) and spuma_face_flux (fvMatrix::flux / faceH) vs the
oracle (O9) -- bitwise, the same face-loop order -- including renumbered meshes (oriented
face fields change sign where owner/neighbour swap) and host buffers."""
import numpy as np
import pytest

import gen
import oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
import paper_2512_22215_b200 as P  # noqa: E402
from gpu_helpers import dev, gpu_assemble  # noqa: E402


def _mesh(kind):
    if kind == "cavity":
        return gen.cavity2d(12)
    m = gen.permute(gen.perturbed(9, 0.25), seed=8)
    m = gen.set_kind(m, "xmin", gen.FIXED_VALUE, np.linspace(0.0, 1.0, m.patches[0].n_faces))
    return m


@pytest.mark.parametrize("renumber", [False, True])
@pytest.mark.parametrize("kind", ["cavity", "perturbed"])
def test_surface_integrate_bitwise(kind, renumber):
    m = _mesh(kind)
    rng = np.random.default_rng(1)
    phi = rng.standard_normal(m.n_faces)
    pphi = [rng.standard_normal(p.n_faces) for p in m.patches]
    ref = O.surface_integrate(m, phi, pphi)
    h = P.Mesh.from_mesh(m, renumber=renumber)
    out = torch.empty(m.n_cells, dtype=torch.float64, device="cuda")
    h.surface_integrate(dev(phi), [dev(x) for x in pphi], dev(m.V), out)
    got = out.cpu().numpy()
    if renumber:  # internal row order changes the summation order: compare to the renumbered oracle
        perm = O.rcm(m.n_cells, m.owner, m.neighbour)
        rm = O.renumber_mesh(m, perm)
        _, _, fm, fl = O.renumber_faces(perm, m.owner, m.neighbour)
        phi_r = np.where(fl.astype(bool), -phi[fm], phi[fm])
        ref = O.surface_integrate(rm, phi_r, pphi, V=gen.permute_cell_field(m.V, perm))[perm]
    assert np.array_equal(got, ref)
    # host buffers through the same call
    out_h = np.zeros(m.n_cells)
    h.surface_integrate(phi, pphi, m.V, out_h)
    assert np.array_equal(out_h, got)


@pytest.mark.parametrize("renumber", [False, True])
@pytest.mark.parametrize("kind", ["cavity", "perturbed"])
def test_face_flux_and_correction_bitwise(kind, renumber):
    m = _mesh(kind)
    g = gen.gamma_lognormal(m)
    h = P.Mesh.from_mesh(m, renumber=renumber)
    diag, upper, src, _ = gpu_assemble(h, m, g, 0, 0.0, gen.rhs(m))
    psi = np.cos(np.arange(m.n_cells) * 0.13)
    pv = [None if p.value is None else dev(p.value) for p in m.patches]
    flux = torch.empty(m.n_faces, dtype=torch.float64, device="cuda")
    pflux = [torch.empty(p.n_faces, dtype=torch.float64, device="cuda") for p in m.patches]
    rng = np.random.default_rng(2)
    phiH = rng.standard_normal(m.n_faces)
    pphi = [rng.standard_normal(p.n_faces) for p in m.patches]
    phi_d = dev(phiH)
    pphi_d = [dev(x) for x in pphi]
    h.face_flux(dev(g), pv, upper, dev(psi), None, None, flux, pflux, phi_d, pphi_d)
    if renumber:
        perm = O.rcm(m.n_cells, m.owner, m.neighbour)
        rm = O.renumber_mesh(m, perm)
        _, _, fm, fl = O.renumber_faces(perm, m.owner, m.neighbour)
        s = O.assemble(rm, gen.permute_cell_field(g, perm), -1)
        f_r, pf_r = O.face_flux(rm, s.upper, gen.permute_cell_field(psi, perm), gamma=gen.permute_cell_field(g, perm))
        ref = np.empty(m.n_faces)
        ref[fm] = np.where(fl.astype(bool), -f_r, f_r)
        pref = pf_r
    else:
        s = O.assemble(m, g, -1)
        ref, pref = O.face_flux(m, s.upper, psi, gamma=g)
    assert np.array_equal(flux.cpu().numpy(), ref)
    for a, b in zip(pflux, pref):
        assert np.array_equal(a.cpu().numpy(), b)
    assert np.array_equal(phi_d.cpu().numpy(), phiH - ref)
    for a, b, c in zip(pphi_d, pphi, pref):
        assert np.array_equal(a.cpu().numpy(), b - c)


def test_simple_pressure_step_conserves():
    """The full pressure step through the C-ABI: source = V surfaceIntegrate(phiHbyA) -> assemble
    (+ reference) -> PCG -> phi = phiHbyA - flux: the corrected flux is divergence-free up to the
    solver residual."""
    m = gen.perturbed(20, 0.15)
    g = gen.gamma_lognormal(m)
    rng = np.random.default_rng(4)
    phiH = dev(rng.standard_normal(m.n_faces) * 1e-3)
    zeros = [dev(np.zeros(p.n_faces)) for p in m.patches]
    h = P.Mesh.from_mesh(m)
    V = dev(m.V)
    div = torch.empty(m.n_cells, dtype=torch.float64, device="cuda")
    h.surface_integrate(phiH, zeros, V, div)
    src = div * V  # fvMatrix source: V fvc::div(phiHbyA)
    diag = torch.empty(m.n_cells, dtype=torch.float64, device="cuda")
    upper = torch.empty(m.n_faces, dtype=torch.float64, device="cuda")
    gd = dev(g)
    h.assemble_laplacian(gd, None, 0, 0.0, diag, upper, src, None)
    b = src.clone()
    psi = torch.zeros(m.n_cells, dtype=torch.float64, device="cuda")
    perf = h.pcg_solve(diag, upper, None, src, psi, 1e-12, 0.0, 5000, 0)
    assert perf["converged"]
    h.face_flux(gd, None, upper, psi, None, None, None, None, phiH, zeros)
    h.surface_integrate(phiH, zeros, V, div)
    res = (div * V).cpu().numpy()
    assert np.sum(np.abs(res[1:])) < 1e-9 * np.sum(np.abs(b.cpu().numpy()))
