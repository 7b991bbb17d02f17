"""The persistent PCG loop (SPUMA_OPT_PERSISTENT, csrc/loop.cu) on the GPU.

Every iteration of a solve runs in one cooperative launch with the residual held on chip (tensor
memory, shared memory, HBM for the rest).  The element arithmetic is that of the graph batches
(k_direction / k_amul_dot<12> / k_update, deferred psi pairs); only the dot products are summed in
another fixed shape.  So:
- every mode (1 rA in HBM, 2 + shared memory, 3 + tensor memory) gives BITWISE the same iterates
  as the others (the residency moves bytes, not arithmetic), and the same as every L2 window;
- against the graph batches: the same iteration count and psi within 1e-12 relative;
- against the oracle: the north_star bar (iterations +-2, 1e-9 relative L2 at matched counts, Q11);
- run to run bitwise (deterministic sums), odd cell counts (the unpaired last cell), K = 1/2/3
  lattices, meshes larger than the on-chip capacity (partial residency), and the degenerate
  controls (converged at setup, max_iter = 0, min_iter > max_iter, a singular matrix)."""
import numpy as np
import pytest

import gen
import oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
import paper_2512_22215_b200 as P  # noqa: E402
from gpu_helpers import dev, gpu_solve_case  # noqa: E402

F64 = dict(dtype=torch.float64, device="cuda")
OPT = P.spuma


def _bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def _solve(h, diag, upper, src, ctl, mode, loop_l2=None, psi0=None):
    h.set_option(OPT.OPT_PERSISTENT, mode)
    if loop_l2 is not None:
        h.set_option(OPT.OPT_LOOP_L2, loop_l2)
    psi = torch.zeros_like(src) if psi0 is None else psi0.clone()
    perf = h.pcg_solve(diag, upper, None, src, psi, *ctl)
    return psi.cpu().numpy(), perf, h.get_stats()


def _assembled(m, gamma=None, ref=0, renumber=False):
    h = P.Mesh.from_mesh(m, renumber=renumber)
    h.set_option(OPT.OPT_SMALL_SOLVE_MAX_CELLS, 0)  # small meshes through the big-mesh path too
    diag, upper = torch.empty(m.n_cells, **F64), torch.empty(m.n_faces, **F64)
    src = torch.as_tensor(gen.rhs(m), **F64)
    h.assemble_laplacian(None if gamma is None else dev(gamma), None, ref, 0.0, diag, upper, src, None)
    return h, diag, upper, src


CONV = (1e-8, 0.0, 20000, 0)
MESHES = [("cube40", lambda: gen.cube(40), 3, CONV), ("box-odd", lambda: gen.box(37, 29, 13), 3, CONV),
          ("cavity2d-151", lambda: gen.cavity2d(151), 2, CONV),
          ("chain-odd", lambda: gen.box(20001, 1, 1), 1, (0.0, 0.0, 300, 300)),  # 1-D: fixed count
          ("tiny-odd", lambda: gen.box(7, 5, 3), 3, CONV)]


@pytest.mark.parametrize("name,make,K,ctl", MESHES, ids=[c[0] for c in MESHES])
def test_modes_bitwise_equal_and_match_graph_batches(name, make, K, ctl):
    m = make()
    assert len(P.spuma.host_lattice_offsets(m.n_cells, m.owner, m.neighbour)) == K
    h, diag, upper, src = _assembled(m)
    psi0, p0, s0 = _solve(h, diag, upper, src, ctl, 0)
    assert s0["loop_mode"] == 0
    outs = {}
    for mode in (1, 2, 3):
        psi, p, s = _solve(h, diag, upper, src, ctl, mode)
        assert s["loop_mode"] == mode and s["loop_grid"] > 0, s
        assert p["n_iterations"] == p0["n_iterations"], (mode, p, p0)
        assert p["converged"] == p0["converged"]
        err = np.linalg.norm(psi - psi0) / np.linalg.norm(psi0)
        assert err <= 1e-12, (mode, err)
        outs[mode] = (psi, p)
    for mode in (2, 3):  # the residency moves bytes, not arithmetic
        assert np.array_equal(_bits(outs[mode][0]), _bits(outs[1][0])), mode
        assert outs[mode][1]["final_residual"] == outs[1][1]["final_residual"]
    h.free()


@pytest.mark.parametrize("name,make", [("cube24", lambda: gen.cube(24)), ("cavity2d-100", lambda: gen.cavity2d(100)),
                                       ("gamma-box", lambda: gen.box(31, 17, 9, (1.0, 0.5, 0.3)))])
def test_persistent_loop_vs_oracle(name, make):
    """north_star bar against the oracle (Q11 protocol), through the default (persistent) path."""
    m = make()
    g, b = gen.gamma_lognormal(m), gen.rhs(m)
    ctl = (1e-8, 0.0, 5000, 0)
    h = P.Mesh.from_mesh(m)
    h.set_option(OPT.OPT_SMALL_SOLVE_MAX_CELLS, 0)
    psi_g, pg, _, _ = gpu_solve_case(m, g, b, 0, ctl, handle=h)
    assert h.get_stats()["loop_mode"] == 3
    psi_o, po, _ = O.solve_case(m, g, b, 0, 0.0, O.controls(*ctl))
    assert pg["converged"] and abs(pg["n_iterations"] - po["n_iterations"]) <= 2, (pg, po)
    n = min(pg["n_iterations"], po["n_iterations"])
    psi_g, _, _, _ = gpu_solve_case(m, g, b, 0, (0.0, 0.0, n, n), handle=h)
    psi_o, _, _ = O.solve_case(m, g, b, 0, 0.0, O.controls(0.0, 0.0, n, n))
    err = np.linalg.norm(psi_g - psi_o) / np.linalg.norm(psi_o)
    assert err <= 1e-9, err
    h.free()


def test_run_to_run_bitwise_and_l2_windows_neutral():
    m = gen.cube(50)
    h, diag, upper, src = _assembled(m)
    ctl = (1e-7, 0.0, 5000, 0)
    ref, pr, _ = _solve(h, diag, upper, src, ctl, 3, loop_l2=0)
    for ll in (0, 1, 2, 3, 4):
        psi, p, s = _solve(h, diag, upper, src, ctl, 3, loop_l2=ll)
        assert s["loop_mode"] == 3
        assert np.array_equal(_bits(psi), _bits(ref)), ll
        assert p["n_iterations"] == pr["n_iterations"] and p["final_residual"] == pr["final_residual"]
    h.free()


def test_partial_residency_beyond_on_chip_capacity():
    """252^3 = 16M cells: twice the cells the SMs hold -- the pairs beyond TMEM + shared memory stay
    in HBM; 20 fixed iterations equal the graph batches (1e-12) and the three modes bitwise."""
    m = gen.cube(252)
    h = P.Mesh.from_mesh(m)
    diag, upper = torch.empty(m.n_cells, **F64), torch.empty(m.n_faces, **F64)
    src = torch.as_tensor(gen.rhs(m), **F64)
    h.assemble_laplacian(None, None, 0, 0.0, diag, upper, src, None)
    ctl = (0.0, 0.0, 20, 20)
    psi0, p0, _ = _solve(h, diag, upper, src, ctl, 0)
    res = {}
    for mode in (1, 3):
        psi, p, s = _solve(h, diag, upper, src, ctl, mode)
        assert p["n_iterations"] == 20 and s["loop_mode"] == mode
        if mode == 3:
            T = s["loop_threads"]
            need = -(-(-(-(m.n_cells // 2) // T)) // s["loop_grid"])
            assert s["loop_tmem_pairs"] + s["loop_smem_pairs"] < need  # some pairs in HBM
            assert s["loop_tmem_pairs"] > 0 and s["loop_smem_pairs"] > 0
        assert np.linalg.norm(psi - psi0) / np.linalg.norm(psi0) <= 1e-12
        res[mode] = psi
    assert np.array_equal(_bits(res[1]), _bits(res[3]))
    h.free()


def test_degenerate_controls_match_graph_batches():
    m = gen.box(33, 21, 11)
    h, diag, upper, src = _assembled(m)
    cases = [(1e30, 0.0, 100, 0),   # converged at setup: no iteration
             (1e-8, 0.0, 0, 0),     # max_iter = 0
             (1e-8, 0.0, 3, 7),     # min_iter > max_iter: min_iter iterations (OpenFOAM loop)
             (1e-30, 0.0, 5, 0),    # max_iter reached
             (1e-8, 0.1, 1000, 0)]  # relative tolerance
    for ctl in cases:
        psi0, p0, _ = _solve(h, diag, upper, src, ctl, 0)
        psi, p, s = _solve(h, diag, upper, src, ctl, 3)
        assert s["loop_mode"] == 3
        assert p["n_iterations"] == p0["n_iterations"], (ctl, p, p0)
        assert p["converged"] == p0["converged"] and p["singular"] == p0["singular"]
        if np.linalg.norm(psi0) > 0:
            assert np.linalg.norm(psi - psi0) / np.linalg.norm(psi0) <= 1e-12, ctl
        else:
            assert not psi.any()
    h.free()


def test_singular_start_stops_like_graph_batches():
    """psi0 = the exact (integer) solution: rA = 0, so wA.pA = 0 at the first iteration -> singular
    with minIter 1, 0 iterations with minIter 0 (Q3/Q4), psi untouched -- as the graph batches."""
    k = 23
    m = gen.box(k, k, k, (float(k),) * 3)
    s = O.assemble(m, None, 0, 0.0)
    x = np.random.default_rng(2).integers(-4, 5, m.n_cells).astype(float)
    bb = O.amul(m, s.diag, s.upper, x)
    h = P.Mesh.from_mesh(m)
    h.set_option(OPT.OPT_SMALL_SOLVE_MAX_CELLS, 0)
    for min_iter, n_exp, sing in ((0, 0, 0), (1, 0, 1)):
        for mode in (0, 3):
            h.set_option(OPT.OPT_PERSISTENT, mode)
            psi = dev(x)
            perf = h.pcg_solve(dev(s.diag), dev(s.upper), None, dev(bb), psi, 1e-9, 0.0, 100, min_iter)
            assert perf["n_iterations"] == n_exp and perf["singular"] == sing, (mode, min_iter, perf)
            assert np.array_equal(psi.cpu().numpy(), x)
            assert h.get_stats()["loop_mode"] == mode
    h.free()


def test_timing_profile_is_recorded():
    m = gen.cube(64)
    h, diag, upper, src = _assembled(m)
    h.set_timing(True)
    h.set_option(OPT.OPT_LOOP_PROFILE, 1)
    h.reset_stats()
    _, p, s = _solve(h, diag, upper, src, (1e-6, 0.0, 5000, 0), 3)
    h.set_timing(False)
    assert s["loop_count"] == 1 and s["loop_ms"] > 0
    assert all(v > 0 for v in s["loop_work_ms"]) and all(v >= 0 for v in s["loop_wait_ms"])
    assert sum(s["loop_work_ms"]) + sum(s["loop_wait_ms"]) <= s["loop_ms"] * 1.05
    h.free()


@pytest.mark.parametrize("iters", [1, 2, 3, 4, 17])
def test_psi_pairs_and_final_flush_with_psi0(iters):
    """A non-zero psi0 and every pending-update count of the final flush (0, 1, 2 psi updates still
    owed when the loop stops): the loop's psi equals the graph batches' (same pairs, same flush)."""
    m = gen.cube(24)
    g, b = gen.gamma_lognormal(m), gen.rhs(m)
    psi0 = np.cos(np.arange(m.n_cells) * 0.01)
    out = []
    for mode in (0, 3):
        h = P.Mesh.from_mesh(m)
        h.set_option(OPT.OPT_PERSISTENT, mode)
        out.append(gpu_solve_case(m, g, b, 0, (0.0, 0.0, iters, iters), psi0=psi0, handle=h)[:2])
        assert h.get_stats()["loop_mode"] == mode
        h.free()
    assert out[0][1]["n_iterations"] == out[1][1]["n_iterations"] == iters
    d = np.abs(out[0][0] - out[1][0]).max() / np.abs(out[0][0]).max()
    assert d <= 1e-13, d


ELL_MESHES = [("cube30-permuted-rcm", lambda: gen.permute(gen.cube(30), seed=3), True, 10),
              ("perturbed24-permuted-rcm", lambda: gen.permute(gen.perturbed(24, 0.2), seed=5), True, 10),
              ("box-odd-permuted-rcm", lambda: gen.permute(gen.box(29, 23, 17), seed=7), True, 10),
              ("cube30-permuted-as-given", lambda: gen.permute(gen.cube(30), seed=3), False, 6),
              ("box-odd-permuted-as-given", lambda: gen.permute(gen.box(29, 23, 17), seed=7), False, 6)]


@pytest.mark.parametrize("name,make,renumber,variant", ELL_MESHES, ids=[c[0] for c in ELL_MESHES])
def test_ell_rows_loop(name, make, renumber, variant):
    """Meshes that are not lattice numberings (C2 / C4: permuted; renumbered by RCM -> the ELL rows
    of variant 10, as given -> the SELL-C rows of variant 6): modes bitwise equal, the graph batches
    within 1e-12 at the same count, the oracle within the north_star bar (Q11)."""
    m = make()
    h, diag, upper, src = _assembled(m, renumber=renumber)
    assert h.get_stats()["amul_variant"] == variant
    ctl = (1e-8, 0.0, 5000, 0)
    psi0, p0, _ = _solve(h, diag, upper, src, ctl, 0)
    outs = []
    for mode in (1, 3):
        psi, p, s = _solve(h, diag, upper, src, ctl, mode)
        assert s["loop_mode"] == mode, s
        assert p["n_iterations"] == p0["n_iterations"], (p, p0)
        assert np.linalg.norm(psi - psi0) / np.linalg.norm(psi0) <= 1e-12
        outs.append(psi)
    assert np.array_equal(_bits(outs[0]), _bits(outs[1]))
    h.free()
    # oracle (caller numbering; the handle renumbers internally)
    g, b = gen.gamma_lognormal(m), gen.rhs(m)
    hh = P.Mesh.from_mesh(m, renumber=renumber)
    hh.set_option(OPT.OPT_SMALL_SOLVE_MAX_CELLS, 0)
    psi_g, pg, _, _ = gpu_solve_case(m, g, b, 0, ctl, renumber=renumber, handle=hh)
    assert hh.get_stats()["loop_mode"] == 3
    psi_o, po, _ = O.solve_case(m, g, b, 0, 0.0, O.controls(*ctl))
    assert pg["converged"] and abs(pg["n_iterations"] - po["n_iterations"]) <= 2, (pg, po)
    n = min(pg["n_iterations"], po["n_iterations"])
    psi_g, _, _, _ = gpu_solve_case(m, g, b, 0, (0.0, 0.0, n, n), renumber=renumber, handle=hh)
    psi_o, _, _ = O.solve_case(m, g, b, 0, 0.0, O.controls(0.0, 0.0, n, n))
    assert np.linalg.norm(psi_g - psi_o) / np.linalg.norm(psi_o) <= 1e-9
    hh.free()


@pytest.mark.parametrize("n", [1, 2, 3, 5, 64, 65])
def test_tiny_chains_through_the_loop(n):
    """A few cells through the big-mesh path (small-solve threshold 0): the loop's odd-cell and
    empty-tile paths (N = 1: no pair at all) against the graph batches and the oracle."""
    m = gen.box(n, 1, 1)
    h, diag, upper, src = _assembled(m)
    ctl = (1e-12, 0.0, 200, 0)
    psi0, p0, _ = _solve(h, diag, upper, src, ctl, 0)
    psi, p, s = _solve(h, diag, upper, src, ctl, 3)
    if s["amul_variant"] in (6, 8, 10, 12, 13):  # a layout the loop runs (no faces at all: per-row fallback)
        assert s["loop_mode"] == 3, s
    assert p["n_iterations"] == p0["n_iterations"] and p["converged"] == p0["converged"]
    scale = max(np.abs(psi0).max(), 1e-300)
    assert np.abs(psi - psi0).max() / scale <= 1e-12
    g, b = None, gen.rhs(m)
    psi_o, po, _ = O.solve_case(m, g, b, 0, 0.0, O.controls(*ctl))
    assert abs(p["n_iterations"] - po["n_iterations"]) <= 2
    h.free()


@pytest.mark.parametrize("alt", [0, 1])
def test_loop_sweep_direction_option(alt):
    """SPUMA_OPT_ALT_SWEEP reaches the loop (alternating tile / chunk order): same iteration count
    and psi within 1e-12 of the graph batches either way."""
    m = gen.cube(40)
    h, diag, upper, src = _assembled(m)
    h.set_option(OPT.OPT_ALT_SWEEP, alt)
    ctl = (1e-8, 0.0, 5000, 0)
    psi0, p0, _ = _solve(h, diag, upper, src, ctl, 0)
    psi, p, s = _solve(h, diag, upper, src, ctl, 3)
    assert s["loop_mode"] == 3 and p["n_iterations"] == p0["n_iterations"]
    assert np.linalg.norm(psi - psi0) / np.linalg.norm(psi0) <= 1e-12
    h.free()


@pytest.mark.parametrize("ctas", [1, 2, 7, 32, 0])
def test_loop_grid_option(ctas):
    """SPUMA_OPT_LOOP_GRID: the loop on 1..32 CTAs (0 = automatic) -- the same element arithmetic,
    another partial-sum shape: the graph batches' iteration count and psi within 1e-12."""
    m = gen.cube(24)
    h, diag, upper, src = _assembled(m)
    ctl = (1e-8, 0.0, 5000, 0)
    psi0, p0, _ = _solve(h, diag, upper, src, ctl, 0)
    h.set_option(OPT.OPT_LOOP_GRID, ctas)
    psi, p, s = _solve(h, diag, upper, src, ctl, 3)
    assert s["loop_mode"] == 3 and (ctas == 0 or s["loop_grid"] == ctas), s
    assert p["n_iterations"] == p0["n_iterations"]
    assert np.linalg.norm(psi - psi0) / np.linalg.norm(psi0) <= 1e-12
    h.free()
