"""GPU parity of GAMG + Richardson (readings Q22-Q28) through the C-ABI
(spuma_gamg_solve / spuma_gamg_get_hierarchy) against oracle O11.

- hierarchy (agglomeration maps, level sizes): bit-exact (integer work), as given and
  RCM-renumbered (oracle run on the renumbered mesh);
- one V-cycle (minIter = maxIter = 1): relative L2 <= 1e-11 (the only differences are the
  reduction order of the scale factors and of the coarsest PCG's dots);
- full solves: iteration counts within +-2 and relative L2 <= 1e-9 at matched counts (Q11);
- parameter variants (pre-smoothing, no post-smoothing, no scaling, omega), the
  single-level hierarchy, host-pointer and renumbered entry, pGAMG controls."""
import numpy as np
import pytest

import gen
import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import paper_2512_22215_b200 as P  # noqa: E402
from gpu_helpers import dev, gpu_assemble  # noqa: E402


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _oparams(gp):
    return O.gamg_params(n_pre=gp.n_pre_sweeps, n_post=gp.n_post_sweeps, scale=bool(gp.scale_correction),
                         n_coarsest_cells=gp.n_cells_in_coarsest_level, max_levels=gp.max_levels, omega=gp.omega,
                         coarsest_tol=gp.coarsest_tolerance, coarsest_rel_tol=gp.coarsest_rel_tol,
                         coarsest_max_iter=gp.coarsest_max_iter, smoother=gp.smoother, n_inner=gp.n_inner)


class Case:
    """One system on both sides: GPU handle (+ assembled LDU) and the oracle's view of the
    same system in the handle's internal numbering."""

    def __init__(self, mesh, gamma=None, b=None, ref=0, renumber=False):
        self.mesh = mesh
        self.h = P.Mesh.from_mesh(mesh, renumber=renumber)
        b = gen.rhs(mesh) if b is None else b
        self.diag, self.upper, self.src0, _ = gpu_assemble(self.h, mesh, gamma, ref, 0.0, b)
        if renumber:
            perm = self.h.mesh_get_addressing()["perm"]
            self.om = O.renumber_mesh(mesh, perm)
            pc = lambda v: None if v is None else gen.permute_cell_field(v, perm)
            self.osys = O.assemble(self.om, pc(gamma), int(perm[ref]), 0.0, source=pc(b))
            self.back = lambda v: v[perm]
        else:
            self.om = mesh
            self.osys = O.assemble(mesh, gamma, ref, 0.0, source=b)
            self.back = lambda v: v

    def gpu(self, ctl, gp=None, psi0=None):
        psi = dev(np.zeros(self.mesh.n_cells) if psi0 is None else psi0)
        src = self.src0.clone()
        perf = self.h.gamg_solve(self.diag, self.upper, None, src, psi, *ctl, params=gp)
        return psi.cpu().numpy(), perf

    def oracle(self, ctl, gp=None):
        gp = gp or P.gamg_params()
        psi, perf = O.gamg(self.om, self.osys, None, O.controls(*ctl), _oparams(gp))
        return self.back(psi), perf


CASES = [
    ("cube12", lambda: gen.cube(12)),
    ("perturbed-permuted", lambda: gen.permute(gen.perturbed(10, 0.2), seed=7)),
    ("cavity20", lambda: gen.cavity2d(20)),
    ("box-ragged", lambda: gen.box(13, 7, 5, (1.0, 0.6, 0.4))),
    ("cube32-regular", lambda: gen.cube(32)),  # h = 2^-5: exact equal areas -> every level uniform ELL
]


@pytest.mark.parametrize("renumber", [False, True])
@pytest.mark.parametrize("name,make", CASES, ids=[c[0] for c in CASES])
def test_hierarchy_bit_exact(name, make, renumber):
    m = make()
    c = Case(m, renumber=renumber)
    hg = c.h.gamg_hierarchy()
    ho = O.gamg_hierarchy(c.om)
    assert hg["levels"] == len(ho) >= 2
    assert hg["cells"] == [lv[0] for lv in ho]
    assert hg["faces"][1:] == [int(lv[1].shape[0]) for lv in ho[1:]]
    for k in range(len(ho) - 1):
        assert np.array_equal(hg["ftc"][k], ho[k][3]), k


@pytest.mark.parametrize("name,make", CASES, ids=[c[0] for c in CASES])
def test_one_cycle_parity(name, make):
    m = make()
    c = Case(m, gen.gamma_lognormal(m))
    psi_g, pg = c.gpu((0.0, 0.0, 1, 1))
    psi_o, po = c.oracle((0.0, 0.0, 1, 1))
    assert pg["n_iterations"] == po["n_iterations"] == 1
    assert pg["initial_residual"] == pytest.approx(po["initial_residual"], rel=1e-12)
    assert pg["final_residual"] == pytest.approx(po["final_residual"], rel=1e-9)
    assert rel_l2(psi_g, psi_o) <= 1e-11


def _solve_parity(c, ctl, gp=None, max_dn=2):
    psi_g, pg = c.gpu(ctl, gp)
    psi_o, po = c.oracle(ctl, gp)
    assert pg["converged"] == po["converged"]
    assert abs(pg["n_iterations"] - po["n_iterations"]) <= max_dn
    n = min(pg["n_iterations"], po["n_iterations"])
    if pg["n_iterations"] != po["n_iterations"]:
        psi_g, pg = c.gpu((0.0, 0.0, n, n), gp)
        psi_o, po = c.oracle((0.0, 0.0, n, n), gp)
    err = rel_l2(psi_g, psi_o)
    assert err <= 1e-9, err
    return pg, po


@pytest.mark.parametrize("renumber", [False, True])
@pytest.mark.parametrize("name,make", CASES, ids=[c[0] for c in CASES])
def test_solve_parity(name, make, renumber):
    m = make()
    c = Case(m, gen.gamma_lognormal(m), renumber=renumber)
    pg, po = _solve_parity(c, (1e-9, 0.0, 300, 0))
    assert pg["converged"] and pg["n_iterations"] >= 3


def test_paper_controls_pgamg():
    """pGAMG: tolerance 1e-9, relTol 1e-3, maxIter 300, minIter 1."""
    m = gen.perturbed(14, 0.15)
    c = Case(m, gen.gamma_lognormal(m))
    pg, po = _solve_parity(c, (1e-9, 1e-3, 300, 1))
    assert pg["converged"] and pg["final_residual"] < 1e-3 * pg["initial_residual"]


@pytest.mark.parametrize("kw", [
    dict(n_pre_sweeps=1, n_post_sweeps=2),
    dict(n_pre_sweeps=2, n_post_sweeps=0),
    dict(n_post_sweeps=1, scale_correction=0),
    dict(n_post_sweeps=3, omega=0.6, n_cells_in_coarsest_level=40),
    dict(max_levels=3),
    dict(n_post_sweeps=1, omega=1.6),  # divergent Jacobi: the scale factor clamps at 0
    dict(smoother=1),                                  # two-stage Gauss-Seidel (Q30)
    dict(smoother=1, n_inner=3, n_pre_sweeps=1),
    dict(smoother=1, n_inner=0, scale_correction=0),
    dict(smoother=1, n_post_sweeps=1, n_inner=2),
], ids=["pre1", "pre2-post0", "noscale", "post3-omega", "3levels", "clamp", "gs2", "gs2-inner3-pre1",
        "gs2-inner0-noscale", "gs2-post1-inner2"])
def test_parameter_variants_one_cycle_and_solve(kw):
    m = gen.permute(gen.perturbed(9, 0.2), seed=3)
    c = Case(m, gen.gamma_lognormal(m))
    gp = P.gamg_params(**kw)
    psi_g, pg = c.gpu((0.0, 0.0, 2, 2), gp)
    psi_o, po = c.oracle((0.0, 0.0, 2, 2), gp)
    assert rel_l2(psi_g, psi_o) <= 1e-10
    if kw.get("omega", 0.75) < 1.0 or kw.get("smoother"):
        _solve_parity(c, (1e-8, 0.0, 400, 0), gp)


@pytest.mark.parametrize("renumber", [False, True])
def test_gs2_solve_parity(renumber):
    m = gen.permute(gen.perturbed(11, 0.15), seed=5)
    c = Case(m, gen.gamma_lognormal(m), renumber=renumber)
    pg, po = _solve_parity(c, (1e-9, 0.0, 300, 0), P.gamg_params(smoother=1))
    _, pr = c.oracle((1e-9, 0.0, 300, 0))
    assert pg["converged"] and po["n_iterations"] < pr["n_iterations"]


def test_single_level_hierarchy():
    """<= 10 cells: the finest level is the coarsest; one cycle = the coarsest PCG solve."""
    m = gen.box(3, 2, 1)
    c = Case(m, gen.gamma_lognormal(m))
    assert c.h.gamg_hierarchy()["levels"] == 1
    psi_g, pg = c.gpu((1e-12, 0.0, 20, 0))
    psi_o, po = c.oracle((1e-12, 0.0, 20, 0))
    assert pg["n_iterations"] == po["n_iterations"]
    assert rel_l2(psi_g, psi_o) <= 1e-10


def test_host_pointers_and_repeat_calls():
    m = gen.perturbed(8, 0.2)
    c = Case(m, gen.gamma_lognormal(m))
    psi_o, po = c.oracle((1e-9, 0.0, 300, 0))
    d, u, s = c.diag.cpu().numpy(), c.upper.cpu().numpy(), c.src0.cpu().numpy()
    for _ in range(2):  # host arrays, then again on the same handle (graph reuse)
        psi = np.zeros(m.n_cells)
        pg = c.h.gamg_solve(d, u, None, s.copy(), psi, 1e-9, 0.0, 300, 0)
        assert abs(pg["n_iterations"] - po["n_iterations"]) <= 2
        assert rel_l2(psi, psi_o) <= 1e-8
    # changed parameters on the same handle rebuild the hierarchy / graph
    gp = P.gamg_params(n_cells_in_coarsest_level=30)
    psi_g, pg = c.gpu((0.0, 0.0, 1, 1), gp)
    psi_o1, _ = c.oracle((0.0, 0.0, 1, 1), gp)
    assert rel_l2(psi_g, psi_o1) <= 1e-11


def test_gamg_beats_pcg_iterations_and_matches_dense():
    m = gen.cube(16)
    c = Case(m, gen.gamma_lognormal(m))
    psi_g, pg = c.gpu((1e-10, 0.0, 300, 0))
    from cases import dense_ldu
    A = dense_ldu(m.n_cells, m.owner, m.neighbour, c.osys.diag, c.osys.upper)
    exact = np.linalg.solve(A, c.osys.source)
    assert rel_l2(psi_g, exact) < 1e-7
    psi = dev(np.zeros(m.n_cells))
    pp = c.h.pcg_solve(c.diag, c.upper, None, c.src0.clone(), psi, 1e-10, 0.0, 5000, 0)
    assert pg["n_iterations"] * 3 < pp["n_iterations"]


def test_invalid_arguments():
    m = gen.cube(4)
    c = Case(m)
    with pytest.raises(P.SpumaError):
        c.gpu((1e-6, 0.0, 10, 0), P.gamg_params(max_levels=0))
    with pytest.raises(P.SpumaError):
        c.gpu((1e-6, 0.0, 10, 0), P.gamg_params(n_post_sweeps=-1))


@pytest.mark.parametrize("tail", [0, 4096, 100000])
@pytest.mark.parametrize("name,make", [("perturbed14", lambda: gen.perturbed(14, 0.15)),
                                       ("cube32", lambda: gen.cube(32))])
def test_single_cta_tail_on_off(name, make, tail):
    """SPUMA_OPT_GAMG_TAIL_CELLS: the small levels in one CTA (k_gamg_tail) or one launch per
    level and step; both against the oracle (one cycle and a full solve)."""
    m = make()
    c = Case(m, gen.gamma_lognormal(m))
    c.h.set_option(P.spuma.OPT_GAMG_TAIL_CELLS, tail)
    psi_g, pg = c.gpu((0.0, 0.0, 1, 1))
    psi_o, po = c.oracle((0.0, 0.0, 1, 1))
    assert rel_l2(psi_g, psi_o) <= 1e-11
    _solve_parity(c, (1e-9, 0.0, 300, 0))
    for kw in (dict(n_post_sweeps=1), dict(n_post_sweeps=3), dict(n_post_sweeps=4, omega=0.6)):
        gp = P.gamg_params(**kw)
        psi_g, _ = c.gpu((0.0, 0.0, 2, 2), gp)
        psi_o, _ = c.oracle((0.0, 0.0, 2, 2), gp)
        assert rel_l2(psi_g, psi_o) <= 1e-10, kw


def test_large_one_cycle_and_hierarchy_100cubed():
    """BASELINE-size parity (C2/C5 100^3, 1M cells, 18 levels): hierarchy bit-exact and two
    V-cycles against the oracle (relative L2 <= 1e-11), gamma log-normal."""
    m = gen.cube(100)
    c = Case(m, gen.gamma_lognormal(m))
    hg = c.h.gamg_hierarchy()
    ho = O.gamg_hierarchy(m)
    assert hg["cells"] == [lv[0] for lv in ho]
    for k in range(len(ho) - 1):
        assert np.array_equal(hg["ftc"][k], ho[k][3]), k
    psi_g, pg = c.gpu((0.0, 0.0, 2, 2))
    psi_o, po = c.oracle((0.0, 0.0, 2, 2))
    assert pg["final_residual"] == pytest.approx(po["final_residual"], rel=1e-9)
    assert rel_l2(psi_g, psi_o) <= 1e-11
