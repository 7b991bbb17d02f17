"""GPU parity: libspuma (sm_100a) vs the CPU oracle on the same seeded inputs.

Bar (BASELINE.json north_star): addressing and renumbering bit-exact;
coefficients within 1e-13 relative (we also require bitwise, reading Q10:
--fmad=false + the oracle's per-row order); PCG iteration count within +-2
and solution within 1e-9 relative L2 at matched iteration counts (Q11)."""
import numpy as np
import pytest

import gen
import oracle as O
from cases import dirichlet_box

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import paper_2512_22215_b200 as P  # noqa: E402
from gpu_helpers import dev, gpu_assemble, gpu_solve_case  # noqa: E402


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def meshes():
    yield "cavity20", gen.cavity2d(20)
    yield "cube7_odd", gen.cube(7)
    yield "perm_perturbed9", gen.permute(gen.perturbed(9, 0.3), seed=4)
    m = gen.perturbed(8, 0.2)
    m = gen.set_kind(m, "xmin", gen.FIXED_VALUE, np.linspace(0, 1, m.patches[0].n_faces))
    m = gen.set_kind(m, "ymax", gen.FIXED_VALUE, np.full(m.patches[3].n_faces, 0.5))
    yield "fixed_value_perturbed8", m


CASES = list(meshes())


# ------------------------------------------------------------------ A0-A2 addressing, A1 renumbering
@pytest.mark.parametrize("renumber", [False, True])
@pytest.mark.parametrize("name,mesh", CASES, ids=[c[0] for c in CASES])
def test_addressing_bit_exact(name, mesh, renumber):
    h = P.Mesh.from_mesh(mesh, renumber=renumber)
    a = h.mesh_get_addressing()
    if renumber:
        perm = O.rcm(mesh.n_cells, mesh.owner, mesh.neighbour)
        o, n, fm, _ = O.renumber_faces(perm, mesh.owner, mesh.neighbour)
    else:
        perm, o, n, fm = np.arange(mesh.n_cells), mesh.owner, mesh.neighbour, np.arange(mesh.n_faces)
    assert np.array_equal(a["perm"], perm)
    assert np.array_equal(a["owner"], o) and np.array_equal(a["neighbour"], n)
    assert np.array_equal(a["face_map"], fm)
    assert np.array_equal(a["owner_start"], O.owner_start(mesh.n_cells, o))
    lo, ls = O.losort(mesh.n_cells, n)
    assert np.array_equal(a["losort"], lo) and np.array_equal(a["losort_start"], ls)


def test_addressing_bit_exact_full_size_permuted_1M():
    """BASELINE config 2 size: 100^3 randomly permuted, RCM renumbering."""
    m = gen.permute(gen.cube(100), seed=gen.SEED_PERM)
    h = P.Mesh.from_mesh(m, renumber=True)
    a = h.mesh_get_addressing()
    perm = O.rcm(m.n_cells, m.owner, m.neighbour)
    assert np.array_equal(a["perm"], perm)
    o, n, fm, _ = O.renumber_faces(perm, m.owner, m.neighbour)
    assert np.array_equal(a["owner"], o) and np.array_equal(a["neighbour"], n) and np.array_equal(a["face_map"], fm)
    lo, ls = O.losort(m.n_cells, n)
    assert np.array_equal(a["losort"], lo) and np.array_equal(a["losort_start"], ls)


def test_invalid_addressing_rejected():
    m = gen.cube(3)
    bad = m.neighbour.copy()
    bad[0], bad[1] = bad[1], bad[0]  # unsorted
    with pytest.raises(P.SpumaError) as e:
        P.mesh_create(m.n_cells, m.owner, bad, m.Sf, m.magSf, m.C, m.Cf, m.patches)
    assert e.value.status == 2
    bad = m.owner.copy()
    bad[0] = 99
    with pytest.raises(P.SpumaError) as e:
        P.mesh_create(m.n_cells, bad, m.neighbour, m.Sf, m.magSf, m.C, m.Cf, m.patches)
    assert e.value.status == 2


# ------------------------------------------------------------------ A3 geometry
@pytest.mark.parametrize("renumber", [False, True])
@pytest.mark.parametrize("name,mesh", CASES, ids=[c[0] for c in CASES])
def test_geometry_bit_exact(name, mesh, renumber):
    h = P.Mesh.from_mesh(mesh, renumber=renumber)
    g = h.mesh_get_geometry()
    if renumber:
        perm = O.rcm(mesh.n_cells, mesh.owner, mesh.neighbour)
        rm = O.renumber_mesh(mesh, perm)
        og = O.geometry(rm)
        fm = O.renumber_faces(perm, mesh.owner, mesh.neighbour)[2]
        d = np.empty_like(og.delta)
        w = np.empty_like(og.weights)
        d[fm], w[fm] = og.delta, og.weights
    else:
        og = O.geometry(mesh)
        d, w = og.delta, og.weights
    assert np.array_equal(g["delta"], d)
    assert np.array_equal(g["weights"], w)
    nonempty = np.concatenate([np.full(p.n_faces, p.kind != gen.EMPTY) for p in mesh.patches])
    assert np.array_equal(g["bdelta"][nonempty], og.bdelta[nonempty])


# ------------------------------------------------------------------ A4-A5 assembly
@pytest.mark.parametrize("with_gamma", [False, True])
@pytest.mark.parametrize("renumber", [False, True])
@pytest.mark.parametrize("name,mesh", CASES, ids=[c[0] for c in CASES])
def test_assembly_parity(name, mesh, renumber, with_gamma):
    gamma = gen.gamma_lognormal(mesh) if with_gamma else None
    b = gen.rhs(mesh)
    ref = 3 if mesh.n_cells > 3 else 0
    h = P.Mesh.from_mesh(mesh, renumber=renumber)
    diag, upper, src, _ = gpu_assemble(h, mesh, gamma, ref, 0.7, b)
    if renumber:
        perm = O.rcm(mesh.n_cells, mesh.owner, mesh.neighbour)
        rm = O.renumber_mesh(mesh, perm)
        s = O.assemble(rm, None if gamma is None else gen.permute_cell_field(gamma, perm), int(perm[ref]), 0.7,
                       source=gen.permute_cell_field(b, perm))
        fm = O.renumber_faces(perm, mesh.owner, mesh.neighbour)[2]
        od, ou, osrc = s.diag[perm], np.empty(mesh.n_faces), s.source[perm]
        ou[fm] = s.upper
    else:
        s = O.assemble(mesh, gamma, ref, 0.7, source=b)
        od, ou, osrc = s.diag, s.upper, s.source
    gd, gu, gs = diag.cpu().numpy(), upper.cpu().numpy(), src.cpu().numpy()
    # north_star bar: 1e-13 relative ...
    assert np.max(np.abs(gu - ou)) <= 1e-13 * np.max(np.abs(ou))
    assert np.max(np.abs(gd - od)) <= 1e-13 * np.max(np.abs(od))
    assert np.max(np.abs(gs - osrc)) <= 1e-13 * max(np.max(np.abs(osrc)), 1e-300)
    # ... and bitwise under --fmad=false with the oracle's per-row order (Q10)
    assert np.array_equal(gu, ou) and np.array_equal(gd, od) and np.array_equal(gs, osrc)


# ------------------------------------------------------------------ A7 Amul
VARIANTS = list(P.spuma.AMUL_VARIANTS)


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("renumber", [False, True])
@pytest.mark.parametrize("name,mesh", CASES, ids=[c[0] for c in CASES])
def test_amul_bit_exact(name, mesh, renumber, variant):
    rng = np.random.default_rng(5)
    diag = rng.uniform(-4, -1, mesh.n_cells)
    upper = rng.uniform(0.1, 1, mesh.n_faces)
    x = rng.standard_normal(mesh.n_cells)
    h = P.Mesh.from_mesh(mesh, renumber=renumber)
    h.set_option(P.spuma.OPT_AMUL_VARIANT, variant)
    y = torch.empty(mesh.n_cells, dtype=torch.float64, device="cuda")
    h.amul(dev(diag), dev(upper), None, dev(x), y)
    ref = O.amul(mesh, diag, upper, x) if not renumber else None
    if renumber:
        perm = O.rcm(mesh.n_cells, mesh.owner, mesh.neighbour)
        rm = O.renumber_mesh(mesh, perm)
        fm = O.renumber_faces(perm, mesh.owner, mesh.neighbour)[2]
        ref = O.amul(rm, gen.permute_cell_field(diag, perm), upper[fm], gen.permute_cell_field(x, perm))[perm]
    assert np.array_equal(y.cpu().numpy(), ref)


def test_amul_host_pointers_match_device():
    m = gen.permute(gen.perturbed(6, 0.2), seed=1)
    rng = np.random.default_rng(1)
    diag, upper, x = rng.uniform(-3, -1, m.n_cells), rng.uniform(0.1, 1, m.n_faces), rng.standard_normal(m.n_cells)
    h = P.Mesh.from_mesh(m)
    y = np.zeros(m.n_cells)
    h.amul(diag, upper, None, x, y)  # numpy: host pointers staged by the library
    assert np.array_equal(y, O.amul(m, diag, upper, x))


# ------------------------------------------------------------------ A6-A12 PCG
def _pcg_parity(mesh, gamma, b, ref, tol, renumber, max_dn=2):
    ctl = (tol, 0.0, 5000, 0)
    psi_g, perf_g, _, h = gpu_solve_case(mesh, gamma, b, ref, ctl, renumber)
    if renumber:
        perm = O.rcm(mesh.n_cells, mesh.owner, mesh.neighbour)
        rm = O.renumber_mesh(mesh, perm)
        pc = lambda v: None if v is None else gen.permute_cell_field(v, perm)
        run = lambda c: O.solve_case(rm, pc(gamma), pc(b), int(perm[ref]), 0.0, c)
        back = lambda v: v[perm]
    else:
        run = lambda c: O.solve_case(mesh, gamma, b, ref, 0.0, c)
        back = lambda v: v
    psi_o, perf_o, _ = run(O.controls(*ctl))
    assert perf_g["converged"] == perf_o["converged"] == 1
    assert abs(perf_g["n_iterations"] - perf_o["n_iterations"]) <= max_dn
    assert perf_g["initial_residual"] == pytest.approx(perf_o["initial_residual"], rel=1e-12)
    n = min(perf_g["n_iterations"], perf_o["n_iterations"])
    if perf_g["n_iterations"] != perf_o["n_iterations"]:
        psi_g, perf_g, _, _ = gpu_solve_case(mesh, gamma, b, ref, (0.0, 0.0, n, n), renumber, handle=h)
        psi_o, perf_o, _ = run(O.controls(0.0, 0.0, n, n))
    err = rel_l2(psi_g, back(psi_o))
    assert err <= 1e-9, err
    return perf_g, perf_o, err


@pytest.mark.parametrize("renumber", [False, True])
@pytest.mark.parametrize("name,mesh", CASES, ids=[c[0] for c in CASES])
def test_pcg_parity(name, mesh, renumber):
    _pcg_parity(mesh, gen.gamma_lognormal(mesh), gen.rhs(mesh), 0, 1e-6, renumber)


def test_pcg_parity_config1_cavity_tol_1e6():
    """BASELINE config 1: 2-D cavity 20x20, solve to 1e-6 (Q5), gamma = 1 and log-normal."""
    m = gen.cavity2d(20)
    for gamma in (None, gen.gamma_lognormal(m)):
        _pcg_parity(m, gamma, gen.rhs(m), 0, 1e-6, False)


def test_pcg_parity_paper_controls():
    """pcgDiag controls: tol 1e-9, relTol 1e-3, maxIter 3000, minIter 1."""
    m = gen.perturbed(12, 0.15)
    g, b = gen.gamma_lognormal(m), gen.rhs(m)
    psi_g, pg, _, _ = gpu_solve_case(m, g, b, 0, (1e-9, 1e-3, 3000, 1))
    psi_o, po, _ = O.solve_case(m, g, b, 0, 0.0, O.controls(1e-9, 1e-3, 3000, 1))
    assert abs(pg["n_iterations"] - po["n_iterations"]) <= 2 and pg["converged"] and po["converged"]


def test_pcg_parity_config2_permuted_1M():
    """BASELINE config 2: 100^3 cube, random permutation, gamma log-normal, as given and renumbered."""
    m = gen.cube(100)
    g, b = gen.gamma_lognormal(m), gen.rhs(m)
    perm = gen.random_perm(m.n_cells)
    mp = gen.permute(m, perm)
    gp, bp = gen.permute_cell_field(g, perm), gen.permute_cell_field(b, perm)
    ref = int(perm[0])
    for renumber in (False, True):
        _pcg_parity(mp, gp, bp, ref, 1e-6, renumber)


def test_pcg_full_size_8M_fixed_iterations():
    """BASELINE config 3 at N = 1 (200^3, 8M cells) in bench.py's launch configuration:
    20 iterations (minIter = maxIter = 20) on both sides, solution compared element-wise."""
    m = gen.cube(200)
    b = gen.rhs(m)
    n = 20
    psi_g, pg, (dg, ug, sg), h = gpu_solve_case(m, None, b, 0, (0.0, 0.0, n, n))
    psi_o, po, s = O.solve_case(m, None, b, 0, 0.0, O.controls(0.0, 0.0, n, n))
    assert np.array_equal(ug, s.upper) and np.array_equal(dg, s.diag)
    assert pg["n_iterations"] == po["n_iterations"] == n
    assert rel_l2(psi_g, psi_o) <= 1e-9
    assert pg["final_residual"] == pytest.approx(po["final_residual"], rel=1e-9)


def test_pcg_special_cases():
    # identity, no faces: one iteration, psi = b
    n = 9
    m = gen.Mesh(n, np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros((0, 3)), np.zeros(0), np.zeros((0, 3)),
                 np.zeros((n, 3)), np.ones(n), [])
    h = P.Mesh.from_mesh(m)
    b = np.arange(1.0, n + 1)
    psi = dev(np.zeros(n))
    perf = h.pcg_solve(dev(np.ones(n)), dev(np.zeros(0)), None, dev(b), psi, 1e-9)
    assert perf["n_iterations"] == 1 and np.array_equal(psi.cpu().numpy(), b)
    # exact integer start: 0 iterations (minIter 0); singular with minIter 1 (Q3/Q4), as the oracle
    k = 5
    m = gen.box(k, k, k, (float(k),) * 3)
    s = O.assemble(m, None, 0, 0.0)
    x = np.random.default_rng(2).integers(-4, 5, m.n_cells).astype(float)
    bb = O.amul(m, s.diag, s.upper, x)
    h = P.Mesh.from_mesh(m)
    for min_iter, n_exp, sing in ((0, 0, 0), (1, 0, 1)):
        psi = dev(x)
        perf = h.pcg_solve(dev(s.diag), dev(s.upper), None, dev(bb), psi, 1e-9, 0.0, 100, min_iter)
        _, po = O.pcg(m, O.LduSystem(s.diag, s.upper, bb, []), x, O.controls(1e-9, 0.0, 100, min_iter))
        assert perf["n_iterations"] == po["n_iterations"] == n_exp and perf["singular"] == po["singular"] == sing
        assert np.array_equal(psi.cpu().numpy(), x)
    # maxIter reached without convergence
    m = gen.cube(10)
    _, perf, _, _ = gpu_solve_case(m, None, gen.rhs(m), 0, (1e-12, 0.0, 7, 0))
    assert perf["n_iterations"] == 7 and perf["converged"] == 0


def test_pcg_deterministic_and_host_pointers():
    m = gen.permute(gen.perturbed(10, 0.2), seed=9)
    g, b = gen.gamma_lognormal(m), gen.rhs(m)
    psi1, p1, _, h = gpu_solve_case(m, g, b, 0)
    psi2, p2, _, _ = gpu_solve_case(m, g, b, 0, handle=h)
    assert np.array_equal(psi1, psi2) and p1 == p2
    # host (numpy) arrays through the same C-ABI calls
    diag, upper, src = np.empty(m.n_cells), np.empty(m.n_faces), b.copy()
    h.assemble_laplacian(g, [None] * len(m.patches), 0, 0.0, diag, upper, src, None)
    psi = np.zeros(m.n_cells)
    p3 = h.pcg_solve(diag, upper, None, src, psi, 1e-6)
    assert np.array_equal(psi, psi1) and p3 == p1


def test_timing_and_stats():
    m = gen.cube(20)
    h = P.Mesh.from_mesh(m)
    h.set_option(P.spuma.OPT_PERSISTENT, 0)  # the captured graph batches (the loop: test_gpu_persistent)
    h.set_timing(True)
    _, perf, _, _ = gpu_solve_case(m, None, gen.rhs(m), 0, handle=h)
    st = h.get_stats()
    assert st["kernel_launches"] > 3 * perf["n_iterations"]
    # timing samples of the first two iterations (one even, one odd) of every executed batch
    n, B = perf["n_iterations"], st["batch_iterations"]
    expect = (n // B) * min(2, B) + min(2, n % B)
    assert st["phase_count"][1] == expect and st["phase_ms"][1] > 0
    assert st["phase_count"][3] == 1


def test_odd_sizes_and_batches():
    m = gen.box(5, 3, 7, (1, 1, 1))  # N = 105 (odd, partial warp)
    g, b = gen.gamma_lognormal(m), gen.rhs(m)
    psi_o, po, _ = O.solve_case(m, g, b, 0, 0.0, O.controls(1e-6))
    n = po["n_iterations"]
    psi_n, _, _ = O.solve_case(m, g, b, 0, 0.0, O.controls(0.0, 0.0, n, n))
    for batch in (1, 3, 16):
        h = P.Mesh.from_mesh(m)
        h.set_option(P.spuma.OPT_SMALL_SOLVE_MAX_CELLS, 0)  # graph-batched path
        h.set_batch(batch)
        psi, perf, _, _ = gpu_solve_case(m, g, b, 0, handle=h)
        assert abs(perf["n_iterations"] - n) <= 2
        psi, perf, _, _ = gpu_solve_case(m, g, b, 0, (0.0, 0.0, n, n), handle=h)  # matched count (Q11)
        assert perf["n_iterations"] == n and rel_l2(psi, psi_n) <= 1e-9


def _star_mesh(n):
    """Cell 0 is the owner of faces to every other cell, plus a chain: tiles overflow the
    shared-memory staging capacity (kTileCap), exercising the per-row fallback."""
    owner = [0] * (n - 1) + list(range(1, n - 1))
    nbr = list(range(1, n)) + list(range(2, n))
    order = np.lexsort((nbr, owner))
    owner, nbr = np.array(owner, np.int32)[order], np.array(nbr, np.int32)[order]
    F = owner.shape[0]
    C = np.stack([np.arange(n, dtype=float), np.zeros(n), np.zeros(n)], 1)
    Sf = np.tile([1.0, 0.0, 0.0], (F, 1))
    return gen.Mesh(n, owner, nbr, Sf, np.ones(F), 0.5 * (C[owner] + C[nbr]), C, np.ones(n), [])


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("n", [300, 3000])
def test_amul_bit_exact_overflowing_tiles(n, variant):
    m = _star_mesh(n)
    rng = np.random.default_rng(n)
    diag, upper, x = rng.uniform(-4, -1, n), rng.uniform(0.1, 1, m.n_faces), rng.standard_normal(n)
    h = P.Mesh.from_mesh(m)
    h.set_option(P.spuma.OPT_AMUL_VARIANT, variant)
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    h.amul(dev(diag), dev(upper), None, dev(x), y)
    assert np.array_equal(y.cpu().numpy(), O.amul(m, diag, upper, x))


def test_amul_bit_exact_full_size_8M():
    """The hot Amul kernel at BASELINE config 3 size (200^3), bench.py's launch configuration."""
    m = gen.cube(200)
    s = O.assemble(m, None, 0, 0.0)
    x = np.sin(np.arange(m.n_cells) * 1e-3)
    ref = O.amul(m, s.diag, s.upper, x)
    h = P.Mesh.from_mesh(m)
    y = torch.empty(m.n_cells, dtype=torch.float64, device="cuda")
    for v in VARIANTS:
        h.set_option(P.spuma.OPT_AMUL_VARIANT, v)
        y.zero_()
        h.amul(dev(s.diag), dev(s.upper), None, dev(x), y)
        assert np.array_equal(y.cpu().numpy(), ref), v


@pytest.mark.parametrize("variant", VARIANTS)
def test_pcg_all_amul_variants(variant):
    """Every A7 variant inside the PCG loop matches the oracle (Q11 protocol); Amul values are
    bitwise equal across variants, dots differ only by the CTA count of the reduction."""
    m = gen.permute(gen.perturbed(12, 0.2), seed=3)
    g, b = gen.gamma_lognormal(m), gen.rhs(m)
    _, po, _ = O.solve_case(m, g, b, 0, 0.0, O.controls(1e-6))
    n = po["n_iterations"]
    psi_o, _, _ = O.solve_case(m, g, b, 0, 0.0, O.controls(0.0, 0.0, n, n))
    h = P.Mesh.from_mesh(m)
    h.set_option(P.spuma.OPT_AMUL_VARIANT, variant)
    _, p, _, _ = gpu_solve_case(m, g, b, 0, handle=h)
    assert abs(p["n_iterations"] - n) <= 2
    psi, p, _, _ = gpu_solve_case(m, g, b, 0, (0.0, 0.0, n, n), handle=h)
    assert rel_l2(psi, psi_o) <= 1e-9


@pytest.mark.parametrize("name,mesh", CASES, ids=[c[0] for c in CASES])
def test_small_single_cta_path_and_graph_path(name, mesh):
    """Meshes <= 8192 cells take the single-CTA solve; both paths match the oracle (Q11)."""
    g, b = gen.gamma_lognormal(mesh), gen.rhs(mesh)
    _, po, _ = O.solve_case(mesh, g, b, 0, 0.0, O.controls(1e-6))
    n = po["n_iterations"]
    psi_o, _, _ = O.solve_case(mesh, g, b, 0, 0.0, O.controls(0.0, 0.0, n, n))
    for thr in (8192, 0):
        h = P.Mesh.from_mesh(mesh)
        h.set_option(P.spuma.OPT_SMALL_SOLVE_MAX_CELLS, thr)
        _, p, _, _ = gpu_solve_case(mesh, g, b, 0, handle=h)
        assert abs(p["n_iterations"] - n) <= 2 and p["converged"]
        psi, p, _, _ = gpu_solve_case(mesh, g, b, 0, (0.0, 0.0, n, n), handle=h)
        assert p["n_iterations"] == n and rel_l2(psi, psi_o) <= 1e-9
        st = h.get_stats()
        if thr:
            assert st["kernel_launches"] < 20  # one solve = a handful of launches


def _empty_mesh(n):
    return gen.Mesh(n, np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros((0, 3)), np.zeros(0),
                    np.zeros((0, 3)), np.zeros((n, 3)), np.ones(n), [])


@pytest.mark.parametrize("small", [8192, 0])
def test_degenerate_meshes(small):
    # no cells: nothing to solve; reported converged with zero residual, as the oracle
    m = _empty_mesh(0)
    h = P.Mesh.from_mesh(m)
    h.set_option(P.spuma.OPT_SMALL_SOLVE_MAX_CELLS, small)
    z = torch.zeros(0, dtype=torch.float64, device="cuda")
    perf = h.pcg_solve(z, z, None, z, z, 1e-6)
    _, po = O.pcg(m, O.LduSystem(np.zeros(0), np.zeros(0), np.zeros(0), []), None, O.controls(1e-6))
    assert perf["n_iterations"] == po["n_iterations"] == 0 and perf["converged"] == po["converged"] == 1
    # one cell, no faces, reference cell: diag doubled, psi = b / (2 d)
    m = _empty_mesh(1)
    m = gen.Mesh(1, m.owner, m.neighbour, m.Sf, m.magSf, m.Cf, m.C, m.V,
                 [gen.Patch("wall", gen.FIXED_VALUE, np.zeros(1, np.int32), np.array([[1.0, 0, 0]]), np.ones(1),
                            np.array([[0.5, 0, 0]]), value=np.array([2.0]))])
    m.C[0] = [0.0, 0.0, 0.0]
    h = P.Mesh.from_mesh(m)
    h.set_option(P.spuma.OPT_SMALL_SOLVE_MAX_CELLS, small)
    diag, upper, src, _ = gpu_assemble(h, m, None, 0, 0.0, np.array([3.0]))
    s = O.assemble(m, None, 0, 0.0, source=np.array([3.0]))
    assert np.array_equal(diag.cpu().numpy(), s.diag) and np.array_equal(src.cpu().numpy(), s.source)
    psi = torch.zeros(1, dtype=torch.float64, device="cuda")
    perf = h.pcg_solve(diag, upper, None, src, psi, 1e-12)
    assert perf["n_iterations"] == 1 and psi.item() == pytest.approx(s.source[0] / s.diag[0], rel=1e-15)


def test_disconnected_components_renumbered():
    """Two disconnected blocks: RCM restarts per component (Q12); both paths still bit-exact."""
    a = gen.box(3, 2, 1, (1, 1, 1))
    b = gen.box(2, 2, 2, (1, 1, 1))
    n = a.n_cells + b.n_cells
    owner = np.concatenate([a.owner, b.owner + a.n_cells]).astype(np.int32)
    nbr = np.concatenate([a.neighbour, b.neighbour + a.n_cells]).astype(np.int32)
    m = gen.Mesh(n, owner, nbr, np.concatenate([a.Sf, b.Sf]), np.concatenate([a.magSf, b.magSf]),
                 np.concatenate([a.Cf, b.Cf]), np.concatenate([a.C, b.C + 5.0]), np.concatenate([a.V, b.V]), [])
    h = P.Mesh.from_mesh(m, renumber=True)
    ad = h.mesh_get_addressing()
    assert np.array_equal(ad["perm"], O.rcm(n, owner, nbr))
    rng = np.random.default_rng(0)
    diag, upper, x = rng.uniform(-3, -1, n), rng.uniform(0.1, 1, m.n_faces), rng.standard_normal(n)
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    h.amul(dev(diag), dev(upper), None, dev(x), y)
    perm = ad["perm"]
    rm = O.renumber_mesh(m, perm)
    fm = O.renumber_faces(perm, owner, nbr)[2]
    ref = O.amul(rm, gen.permute_cell_field(diag, perm), upper[fm], gen.permute_cell_field(x, perm))[perm]
    assert np.array_equal(y.cpu().numpy(), ref)


@pytest.mark.parametrize("iters", [None, 1, 2, 7, 8])
def test_deferred_psi_updates_are_bitwise_neutral(iters):
    """SPUMA_OPT_DEFER_PSI pairs two psi updates into one pass, (psi + a1 p1) + a2 p2: the same
    roundings in the same order, so psi and perf are bitwise those of per-iteration updates
    (odd iteration counts exercise the final flush)."""
    m = gen.permute(gen.perturbed(14, 0.2), seed=12)
    g, b = gen.gamma_lognormal(m), gen.rhs(m)
    ctl = (1e-8, 0.0, 5000, 0) if iters is None else (0.0, 0.0, iters, iters)
    out = []
    for defer in (0, 1, 2):  # every iteration / pairs in the update / pairs in the direction
        h = P.Mesh.from_mesh(m)
        h.set_option(P.spuma.OPT_SMALL_SOLVE_MAX_CELLS, 0)
        h.set_option(P.spuma.OPT_PERSISTENT, 0)  # graph batches on all three (same reduction shape)
        h.set_option(P.spuma.OPT_DEFER_PSI, defer)
        out.append(gpu_solve_case(m, g, b, 0, ctl, handle=h)[:2])
    for k in (1, 2):
        assert out[0][1] == out[k][1]
        assert np.array_equal(out[0][0].view(np.uint64), out[k][0].view(np.uint64)), k


@pytest.mark.parametrize("iters", [1, 2, 3, 4, 17])
def test_deferred_psi_in_direction_lattice_and_psi0(iters):
    """SPUMA_OPT_DEFER_PSI = 2 on the lattice hot loop with a non-zero psi0: every pending-update
    count of the final flush (0, 1, 2) gives bitwise the psi of per-iteration updates."""
    m = gen.cube(24)
    g, b = gen.gamma_lognormal(m), gen.rhs(m)
    psi0 = np.cos(np.arange(m.n_cells) * 0.01)
    out = []
    for defer in (0, 2):
        h = P.Mesh.from_mesh(m)
        h.set_option(P.spuma.OPT_PERSISTENT, 0)  # graph batches on both sides (same reduction shape)
        h.set_option(P.spuma.OPT_DEFER_PSI, defer)
        out.append(gpu_solve_case(m, g, b, 0, (0.0, 0.0, iters, iters), psi0=psi0, handle=h)[:2])
        h.free()
    assert out[0][1] == out[1][1]
    assert np.array_equal(out[0][0].view(np.uint64), out[1][0].view(np.uint64))


@pytest.mark.parametrize("mode", [1, 2])
def test_fused_direction_is_bitwise_neutral(mode):
    """SPUMA_OPT_FUSE_DIRECTION: the direction formed inside the Amul gather gives bitwise the
    iterates of the separate k_direction pass (same values, same order, same reduction grid)."""
    m = gen.perturbed(24, 0.15)  # 13824 cells: above the single-CTA threshold, ELL layout
    g, b = gen.gamma_lognormal(m), gen.rhs(m)
    h = P.Mesh.from_mesh(m)
    h.set_option(P.spuma.OPT_ALT_SWEEP, 0)  # the fused kernel sweeps ascending only
    res = []
    for fm in (0, mode):
        h.set_option(P.spuma.OPT_FUSE_DIRECTION, fm)
        psi, perf, _, _ = gpu_solve_case(m, g, b, 0, (1e-8, 0.0, 5000, 0), handle=h)
        res.append((psi, perf))
    assert res[0][1] == res[1][1] and np.array_equal(res[0][0], res[1][0])


def _two_lattices():
    """two lattice blocks numbered one after the other: chunks inside a block have <= 3 column
    offsets per side (stencil-compressed), the chunk straddling the blocks has more (explicit)"""
    a = gen.box(9, 5, 3, (1, 1, 1))
    b = gen.box(7, 6, 2, (1, 1, 1))
    n = a.n_cells + b.n_cells
    owner = np.concatenate([a.owner, b.owner + a.n_cells]).astype(np.int32)
    nbr = np.concatenate([a.neighbour, b.neighbour + a.n_cells]).astype(np.int32)
    return gen.Mesh(n, owner, nbr, np.concatenate([a.Sf, b.Sf]), np.concatenate([a.magSf, b.magSf]),
                    np.concatenate([a.Cf, b.Cf]), np.concatenate([a.C, b.C + 5.0]), np.concatenate([a.V, b.V]), [])


@pytest.mark.parametrize("name,mesh", [("cube33", gen.cube(33)), ("cavity20", gen.cavity2d(20)),
                                       ("box_odd", gen.box(37, 11, 5)), ("two_lattices", _two_lattices())],
                         ids=["cube33", "cavity20", "box_odd", "two_lattices"])
def test_ell_stencil_rows_bit_exact(name, mesh):
    """SPUMA_OPT_ELL_STENCIL: the chunk-stencil rows (per-chunk column offsets + one word per
    cell) give bitwise the explicit-slot rows and the oracle's Amul, and a PCG solve is bitwise
    unchanged (same Amul values, same reduction order)."""
    rng = np.random.default_rng(9)
    diag = rng.uniform(-4, -1, mesh.n_cells)
    upper = rng.uniform(0.1, 1, mesh.n_faces)
    x = rng.standard_normal(mesh.n_cells)
    ref = O.amul(mesh, diag, upper, x)
    h = P.Mesh.from_mesh(mesh)
    out = []
    for st in (1, 0):
        h.set_option(P.spuma.OPT_ELL_STENCIL, st)
        y = torch.empty(mesh.n_cells, dtype=torch.float64, device="cuda")
        h.amul(dev(diag), dev(upper), None, dev(x), y)
        out.append(y.cpu().numpy())
        assert np.array_equal(out[-1], ref), st
    g, b = gen.gamma_lognormal(mesh), gen.rhs(mesh)
    h.set_option(P.spuma.OPT_SMALL_SOLVE_MAX_CELLS, 0)
    res = []
    for st in (1, 0):
        h.set_option(P.spuma.OPT_ELL_STENCIL, st)
        psi, perf, _, _ = gpu_solve_case(mesh, g, b, 0, (0.0, 0.0, 300, 300), handle=h)
        res.append((psi, perf))
    assert res[0][1] == res[1][1] and np.array_equal(res[0][0], res[1][0])


def test_alt_sweep_changes_only_the_dot_rounding():
    """SPUMA_OPT_ALT_SWEEP reverses the sweep of every other hot-loop kernel: the same element
    operations, per-thread partial sums in the other order -> iterates equal to rounding,
    iteration counts within 1, both within the Q11 bar of the oracle."""
    m = gen.perturbed(26, 0.15)
    g, b = gen.gamma_lognormal(m), gen.rhs(m)
    _, po, _ = O.solve_case(m, g, b, 0, 0.0, O.controls(1e-8))
    h = P.Mesh.from_mesh(m)
    res = []
    for alt in (1, 0):
        h.set_option(P.spuma.OPT_ALT_SWEEP, alt)
        psi, perf, _, _ = gpu_solve_case(m, g, b, 0, (1e-8, 0.0, 5000, 0), handle=h)
        assert abs(perf["n_iterations"] - po["n_iterations"]) <= 2
        res.append((psi, perf))
    assert abs(res[0][1]["n_iterations"] - res[1][1]["n_iterations"]) <= 1
    assert rel_l2(res[0][0], res[1][0]) <= 1e-9
