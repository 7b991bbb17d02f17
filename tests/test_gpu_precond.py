"""GPU parity of the preconditioned solvers (readings Q31-Q35) through the
C-ABI against oracle O12:

- DIC / DILU factor + exact sweeps (sync-free level-scheduled kernels), aDILU passes,
  preconditionT, asymmetric Amul / Tmul: BIT-EXACT (same per-row operation order), natural,
  permuted and RCM-renumbered numberings, and a 100^3 box (dependency depth ~300: spin-waits
  across many CTAs);
- PCG with diagonal / DIC / DILU / aDILU and PBiCG with diagonal / DILU / aDILU: iterations
  +-2 and relative L2 <= 1e-9 at matched counts (Q11);
- LDU -> CSR map bit-exact against the oracle and the value gather."""
import numpy as np
import pytest

import gen
import oracle as O
from cases import asym_system

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import paper_2512_22215_b200 as P  # noqa: E402
from paper_2512_22215_b200 import spuma as S  # noqa: E402
from gpu_helpers import dev  # noqa: E402

KINDS = {"diagonal": (S.PC_DIAGONAL, O.DIAGONAL), "DIC": (S.PC_DIC, O.DIC), "DILU": (S.PC_DILU, O.DILU),
         "aDILU": (S.PC_ADILU, O.ADILU)}


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


class Sys:
    """An asymmetric (or symmetric) system on a GPU handle and its internal-numbering view."""

    def __init__(self, mesh, renumber=False, sym=False, seed=1):
        self.m = mesh
        self.h = P.Mesh.from_mesh(mesh, renumber=renumber)
        if sym:
            s = O.assemble(mesh, gen.gamma_lognormal(mesh), 0, 0.0, source=gen.rhs(mesh))
            self.d, self.u, self.l, self.b = s.diag, s.upper, s.upper.copy(), s.source
        else:
            self.d, self.u, self.l, self.b = asym_system(mesh, seed=seed)
        if renumber:
            ad = self.h.mesh_get_addressing()
            perm, fm = ad["perm"], ad["face_map"]
            flip = perm[mesh.owner[fm]] > perm[mesh.neighbour[fm]]
            self.om = O.renumber_mesh(mesh, perm)
            self.cin = lambda v: gen.permute_cell_field(v, perm)
            self.cout = lambda v: v[perm]
            self.pair = lambda u, l: (np.where(flip, l[fm], u[fm]), np.where(flip, u[fm], l[fm]))
        else:
            self.om, self.cin, self.cout = mesh, (lambda v: v), (lambda v: v)
            self.pair = lambda u, l: (u, l)
        self.ou, self.ol = self.pair(self.u, self.l)
        self.od, self.ob = self.cin(self.d), self.cin(self.b)


def _rD(sy, okind, ou, ol):
    if okind == O.DIAGONAL:
        return 1.0 / sy.od
    return O.ilu_factor(sy.om.owner, sy.om.neighbour, sy.od, ou, ol)


@pytest.mark.parametrize("renumber", [False, True])
@pytest.mark.parametrize("name,make", [("perturbed", lambda: gen.perturbed(9, 0.2)),
                                       ("permuted", lambda: gen.permute(gen.box(11, 7, 5), seed=3)),
                                       ("cavity", lambda: gen.cavity2d(17))])
def test_precondition_bit_exact(name, make, renumber):
    sy = Sys(make(), renumber)
    r = np.sin(np.arange(sy.m.n_cells) * 0.31) + 0.2
    for kname, (gk, ok) in KINDS.items():
        for k in ((1, 2, 3) if ok == O.ADILU else (2,)):
            for tr in (False, True):
                lo = sy.u if ok == O.DIC else sy.l
                w = np.zeros(sy.m.n_cells)
                sy.h.precondition(dev(sy.d), dev(sy.u), dev(lo), dev(r), w := dev(w), gk, k, tr)
                ou, ol = sy.pair(sy.u, lo)  # DIC: the symmetric matrix (lower = upper)
                rD = _rD(sy, ok, ou, ol)
                if ok == O.DIAGONAL:
                    ref = rD * sy.cin(r)
                else:
                    ref = O.ilu_precondition(sy.om.owner, sy.om.neighbour, rD, ou, sy.cin(r), lower=ol, transpose=tr,
                                             k=k if ok == O.ADILU else -1)
                got = w.cpu().numpy()
                assert np.array_equal(got, sy.cout(ref)), (kname, k, tr)


def test_precondition_deep_dependency_chain_bit_exact():
    """100^3 box in natural order: forward/backward dependency depth 298 -> rows spin on flags
    published by other CTAs; still bitwise the sequential sweep."""
    m = gen.cube(100)
    sy = Sys(m, sym=False, seed=2)
    r = np.cos(np.arange(m.n_cells) * 0.01)
    rD = O.ilu_factor(m.owner, m.neighbour, sy.d, sy.u, sy.l)
    ref = O.ilu_precondition(m.owner, m.neighbour, rD, sy.u, r, lower=sy.l)
    w = dev(np.zeros(m.n_cells))
    sy.h.precondition(dev(sy.d), dev(sy.u), dev(sy.l), dev(r), w, S.PC_DILU)
    assert np.array_equal(w.cpu().numpy(), ref)


@pytest.mark.parametrize("renumber", [False, True])
def test_asym_amul_tmul_bit_exact(renumber):
    sy = Sys(gen.permute(gen.perturbed(8, 0.2), seed=4), renumber)
    x = np.sin(np.arange(sy.m.n_cells) * 0.7)
    for tr in (False, True):
        y = dev(np.zeros(sy.m.n_cells))
        sy.h.amul_asym(dev(sy.d), dev(sy.u), dev(sy.l), dev(x), y, tr)
        f = O.tmul if tr else O.amul_asym
        ref = f(sy.om.owner, sy.om.neighbour, sy.od, sy.ou, sy.ol, sy.cin(x))
        assert np.array_equal(y.cpu().numpy(), sy.cout(ref)), tr


def _parity(gpu_run, or_run, ctl):
    psi_g, pg = gpu_run(ctl)
    psi_o, po = or_run(ctl)
    assert pg["converged"] == po["converged"] == 1
    assert abs(pg["n_iterations"] - po["n_iterations"]) <= 2, (pg, po)
    assert pg["initial_residual"] == pytest.approx(po["initial_residual"], rel=1e-12)
    n = min(pg["n_iterations"], po["n_iterations"])
    if pg["n_iterations"] != po["n_iterations"]:
        psi_g, pg = gpu_run((0.0, 0.0, n, n))
        psi_o, po = or_run((0.0, 0.0, n, n))
    err = rel_l2(psi_g, psi_o)
    assert err <= 1e-9, err
    return pg, po


@pytest.mark.parametrize("renumber", [False, True])
@pytest.mark.parametrize("kname", list(KINDS))
def test_pcg_pc_parity(kname, renumber):
    gk, ok = KINDS[kname]
    sy = Sys(gen.permute(gen.perturbed(12, 0.15), seed=8), renumber, sym=True)

    def gpu_run(ctl):
        psi = dev(np.zeros(sy.m.n_cells))
        perf = sy.h.pcg_solve_pc(dev(sy.d), dev(sy.u), dev(sy.b), psi, *ctl, kind=gk, n_sweeps=2)
        return psi.cpu().numpy(), perf

    def or_run(ctl):
        psi, perf = O.pcg_pc(sy.om, O.LduSystem(sy.od, sy.ou, sy.ob, []), ok, 2, None, O.controls(*ctl))
        return sy.cout(psi), perf

    pg, po = _parity(gpu_run, or_run, (1e-9, 0.0, 3000, 0))
    if ok == O.DIAGONAL:  # the Jacobi kind is the O6 solver: same count as spuma_pcg_solve
        psi = dev(np.zeros(sy.m.n_cells))
        pp = sy.h.pcg_solve(dev(sy.d), dev(sy.u), None, dev(sy.b), psi, 1e-9, 0.0, 3000, 0)
        assert abs(pp["n_iterations"] - pg["n_iterations"]) <= 2


@pytest.mark.parametrize("renumber", [False, True])
@pytest.mark.parametrize("kname", ["diagonal", "DILU", "aDILU"])
def test_pbicg_parity(kname, renumber):
    gk, ok = KINDS[kname]
    sy = Sys(gen.permute(gen.perturbed(10, 0.2), seed=6), renumber, sym=False, seed=9)

    def gpu_run(ctl):
        psi = dev(np.zeros(sy.m.n_cells))
        perf = sy.h.pbicg_solve(dev(sy.d), dev(sy.u), dev(sy.l), dev(sy.b), psi, *ctl, kind=gk, n_sweeps=2)
        return psi.cpu().numpy(), perf

    def or_run(ctl):
        psi, perf = O.pbicg(sy.om.owner, sy.om.neighbour, sy.od, sy.ou, sy.ol, sy.ob, ok, 2, None, O.controls(*ctl))
        return sy.cout(psi), perf

    _parity(gpu_run, or_run, (1e-10, 0.0, 1000, 0))


def test_pbicg_paper_controls_host_arrays():
    """U/k/omega controls: PBiCG aDILU, tolerance 1e-8, relTol 1e-3; host arrays."""
    m = gen.perturbed(10, 0.15)
    d, u, l, b = asym_system(m, seed=11)
    h = P.Mesh.from_mesh(m)
    psi = np.zeros(m.n_cells)
    pg = h.pbicg_solve(d, u, l, b, psi, 1e-8, 1e-3, 1000, 0)
    po_psi, po = O.pbicg(m.owner, m.neighbour, d, u, l, b, O.ADILU, 2, None, O.controls(1e-8, 1e-3, 1000, 0))
    assert pg["converged"] and abs(pg["n_iterations"] - po["n_iterations"]) <= 2


def test_ldu_to_csr_and_values():
    m = gen.permute(gen.perturbed(7, 0.2), seed=1)
    d, u, l, _ = asym_system(m, seed=2)
    h = P.Mesh.from_mesh(m)
    rp, col, mp = h.ldu_to_csr()
    orp, ocol, omp = O.ldu_to_csr(m.n_cells, m.owner, m.neighbour)
    assert np.array_equal(rp, orp) and np.array_equal(col, ocol) and np.array_equal(mp, omp)
    vals = torch.empty(col.shape[0], dtype=torch.float64, device="cuda")
    h.csr_values(dev(d), dev(u), dev(l), vals)
    assert np.array_equal(vals.cpu().numpy(), np.concatenate([d, u, l])[omp])
    hr = P.Mesh.from_mesh(m, renumber=True)
    with pytest.raises(P.SpumaError):
        hr.ldu_to_csr()
