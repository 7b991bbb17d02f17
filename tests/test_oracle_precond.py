"""Pins for oracle O12 (readings Q31-Q34): DIC / DILU / aDILU
preconditioners, PCG with them, PBiCG, Tmul and the LDU -> CSR map.

Independent of the oracle's loops:
- SPEC examples: 3-chain DIC factor, 3-chain CSR, diagonal-only cases;
- the incomplete-factorisation identity: M = (D* + L) D*^-1 (D* + U), D* = diag(1/rD), has
  diag(M) = diag(A) and M = A on the off-diagonal pattern (hex meshes: no triangles), and
  precondition(r) = M^-1 r, preconditionT(r) = M^-T r (dense solves);
- aDILU (Q33): k = 0 is rD r, k passes equal the dense Jacobi iteration on the triangular
  factors, k >= depth is bitwise the exact sweep;
- a 1-D chain has no fill: DIC is the exact Cholesky factor, DIC-PCG converges in 1 iteration;
- PBiCG on a symmetric system reproduces PCG's iterates; on asymmetric systems it reaches
  the dense solution; Tmul = A^T x; CSR = scipy's CSR of the dense matrix."""
import json
import os

import numpy as np
import pytest
import scipy.sparse

import gen
import oracle as O
from cases import asym_system, dense_ldu

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _dense_asym(n, owner, neighbour, diag, upper, lower):
    A = np.diag(np.asarray(diag, float))
    A[owner, neighbour] = upper
    A[neighbour, owner] = lower
    return A


def test_spec_examples():
    g = json.load(open(os.path.join(GOLD, "spec_precond_csr.json")))
    ex = g["dic_chain"]
    rD = O.ilu_factor(ex["owner"], ex["neighbour"], ex["diag"], ex["upper"])
    assert np.allclose(rD, ex["rD"], rtol=1e-15)
    ex = g["csr_chain"]
    rp, col, mp = O.ldu_to_csr(3, ex["owner"], ex["neighbour"])
    assert rp.tolist() == ex["row_ptr"] and col.tolist() == ex["col"]
    # diagonal-only: rD = 1/diag; DILU precondition == diagonal preconditioner
    d = np.array([2.0, -3.0, 4.0, 0.5])
    e = np.zeros(0, np.int32)
    assert np.array_equal(O.ilu_factor(e, e, d, np.zeros(0)), 1.0 / d)
    r = np.array([1.0, 2.0, -1.0, 3.0])
    w = O.ilu_precondition(e, e, 1.0 / d, np.zeros(0), r, lower=np.zeros(0))
    assert np.array_equal(w, (1.0 / d) * r)
    rp, col, mp = O.ldu_to_csr(4, e, e)
    assert rp.tolist() == [0, 1, 2, 3, 4]


def _M(mesh, rD, upper, lower):
    Ds = np.diag(1.0 / rD)
    Lo = np.zeros((mesh.n_cells, mesh.n_cells))
    Up = np.zeros_like(Lo)
    Lo[mesh.neighbour, mesh.owner] = lower
    Up[mesh.owner, mesh.neighbour] = upper
    return (Ds + Lo) @ np.diag(rD) @ (Ds + Up)


@pytest.mark.parametrize("sym", [True, False])
@pytest.mark.parametrize("mesh", [gen.perturbed(5, 0.2), gen.permute(gen.box(6, 4, 3), seed=2), gen.cavity2d(7)],
                         ids=["perturbed", "permuted-box", "cavity"])
def test_incomplete_factorisation_identity_and_exact_apply(mesh, sym):
    if sym:
        s = O.assemble(mesh, gen.gamma_lognormal(mesh), 0, 0.0)
        diag, upper, lower = s.diag, s.upper, s.upper
    else:
        diag, upper, lower, _ = asym_system(mesh, seed=1)
    A = _dense_asym(mesh.n_cells, mesh.owner, mesh.neighbour, diag, upper, lower)
    rD = O.ilu_factor(mesh.owner, mesh.neighbour, diag, upper, None if sym else lower)
    M = _M(mesh, rD, upper, lower)
    assert np.allclose(np.diag(M), np.diag(A), rtol=1e-12, atol=0)
    pat = A != 0
    np.fill_diagonal(pat, False)
    assert np.allclose(M[pat], A[pat], rtol=1e-13, atol=0)
    r = np.sin(np.arange(mesh.n_cells) * 0.37)
    w = O.ilu_precondition(mesh.owner, mesh.neighbour, rD, upper, r, lower=lower)
    assert np.allclose(w, np.linalg.solve(M, r), rtol=1e-10, atol=1e-12 * np.max(np.abs(w)))
    wt = O.ilu_precondition(mesh.owner, mesh.neighbour, rD, upper, r, lower=lower, transpose=True)
    assert np.allclose(wt, np.linalg.solve(M.T, r), rtol=1e-10, atol=1e-12 * np.max(np.abs(wt)))


def test_adilu_jacobi_passes():
    m = gen.perturbed(5, 0.2)
    diag, upper, lower, _ = asym_system(m, seed=3)
    rD = O.ilu_factor(m.owner, m.neighbour, diag, upper, lower)
    r = np.cos(np.arange(m.n_cells) * 0.5)
    assert np.array_equal(O.ilu_precondition(m.owner, m.neighbour, rD, upper, r, lower=lower, k=0), rD * r)
    Lo = np.zeros((m.n_cells, m.n_cells))
    Up = np.zeros_like(Lo)
    Lo[m.neighbour, m.owner] = lower
    Up[m.owner, m.neighbour] = upper
    for k in (1, 2, 3):
        y = rD * r
        for _ in range(k):
            y = rD * r - rD * (Lo @ y)
        w = y.copy()
        for _ in range(k):
            w = y - rD * (Up @ w)
        got = O.ilu_precondition(m.owner, m.neighbour, rD, upper, r, lower=lower, k=k)
        assert np.allclose(got, w, rtol=1e-12, atol=1e-14 * np.max(np.abs(w))), k
    exact = O.ilu_precondition(m.owner, m.neighbour, rD, upper, r, lower=lower)
    deep = O.ilu_precondition(m.owner, m.neighbour, rD, upper, r, lower=lower, k=m.n_cells)
    assert np.array_equal(deep, exact)


def test_chain_dic_is_exact_cholesky():
    n = 32
    o, nb = np.arange(n - 1, dtype=np.int32), np.arange(1, n, dtype=np.int32)
    m = gen.Mesh(n, o, nb, np.zeros((n - 1, 3)), np.ones(n - 1), np.zeros((n - 1, 3)), np.zeros((n, 3)), np.ones(n))
    sys = O.LduSystem(np.full(n, -2.0), np.ones(n - 1), np.ones(n), [])
    sys.diag[0] = -3.0  # Dirichlet-like end: SPD (negative definite) 1-D Poisson
    psi, perf = O.pcg_pc(m, sys, O.DIC, ctl=O.controls(1e-12))
    A = _dense_asym(n, o, nb, sys.diag, sys.upper, sys.upper)
    assert perf["n_iterations"] == 1
    assert np.allclose(psi, np.linalg.solve(A, sys.source), rtol=1e-12)


def test_pcg_preconditioners_converge_to_dense_solution():
    m = gen.perturbed(8, 0.2)
    s = O.assemble(m, gen.gamma_lognormal(m), 0, 0.0, source=gen.rhs(m))
    A = dense_ldu(m.n_cells, m.owner, m.neighbour, s.diag, s.upper)
    exact = np.linalg.solve(A, s.source)
    its = {}
    for kind in (O.DIAGONAL, O.DIC, O.DILU, O.ADILU):
        psi, perf = O.pcg_pc(m, s, kind, ctl=O.controls(1e-12, 0.0, 2000, 0))
        assert perf["converged"]
        assert np.linalg.norm(psi - exact) / np.linalg.norm(exact) < 1e-8
        its[kind] = perf["n_iterations"]
    assert its[O.DIC] < 0.7 * its[O.DIAGONAL] and its[O.DILU] == its[O.DIC]
    # the diagonal kind is the O6 algorithm: same iterates as or_pcg
    psi_a, pa = O.pcg_pc(m, s, O.DIAGONAL, ctl=O.controls(1e-9))
    psi_b, pb = O.pcg(m, s, None, O.controls(1e-9))
    assert pa["n_iterations"] == pb["n_iterations"] and np.allclose(psi_a, psi_b, rtol=1e-12, atol=1e-15)


def test_tmul_and_asym_amul_are_dense_products():
    m = gen.permute(gen.perturbed(5, 0.2), seed=9)
    diag, upper, lower, _ = asym_system(m, seed=4)
    A = _dense_asym(m.n_cells, m.owner, m.neighbour, diag, upper, lower)
    x = np.sin(np.arange(m.n_cells) * 0.9)
    assert np.allclose(O.amul_asym(m.owner, m.neighbour, diag, upper, lower, x), A @ x, rtol=1e-13, atol=1e-15)
    assert np.allclose(O.tmul(m.owner, m.neighbour, diag, upper, lower, x), A.T @ x, rtol=1e-13, atol=1e-15)


@pytest.mark.parametrize("kind", [O.DIAGONAL, O.DILU, O.ADILU])
def test_pbicg_asymmetric_reaches_dense_solution(kind):
    m = gen.permute(gen.perturbed(7, 0.2), seed=6)
    diag, upper, lower, b = asym_system(m, seed=5)
    A = _dense_asym(m.n_cells, m.owner, m.neighbour, diag, upper, lower)
    psi, perf = O.pbicg(m.owner, m.neighbour, diag, upper, lower, b, kind, ctl=O.controls(1e-13, 0.0, 1000, 0))
    assert perf["converged"] and not perf["singular"]
    exact = np.linalg.solve(A, b)
    assert np.linalg.norm(psi - exact) / np.linalg.norm(exact) < 1e-9


@pytest.mark.parametrize("kind", [O.DIAGONAL, O.DIC])
def test_pbicg_on_symmetric_system_follows_pcg(kind):
    """BiCG with a symmetric preconditioner on a symmetric matrix produces the CG iterates."""
    m = gen.perturbed(7, 0.2)
    s = O.assemble(m, gen.gamma_lognormal(m), 0, 0.0, source=gen.rhs(m))
    for n in (1, 5, 20):
        pb, fb = O.pbicg(m.owner, m.neighbour, s.diag, s.upper, s.upper, s.source, kind,
                         ctl=O.controls(0.0, 0.0, n, n))
        pc, fc = O.pcg_pc(m, s, kind, ctl=O.controls(0.0, 0.0, n, n))
        assert fb["n_iterations"] == fc["n_iterations"] == n
        assert np.linalg.norm(pb - pc) / np.linalg.norm(pc) < 1e-11
        assert fb["final_residual"] == pytest.approx(fc["final_residual"], rel=1e-8)


def test_pbicg_identity_one_iteration():
    n = 10
    e = np.zeros(0, np.int32)
    b = np.arange(1.0, n + 1)
    psi, perf = O.pbicg(e, e, np.ones(n), np.zeros(0), np.zeros(0), b, O.DILU, ctl=O.controls(1e-12))
    assert perf["n_iterations"] == 1 and np.allclose(psi, b, rtol=1e-15)


@pytest.mark.parametrize("mesh", [gen.permute(gen.perturbed(5, 0.2), seed=1), gen.cavity2d(6)], ids=["perm", "cavity"])
def test_ldu_to_csr_matches_scipy(mesh):
    diag, upper, lower, _ = asym_system(mesh, seed=7)
    A = _dense_asym(mesh.n_cells, mesh.owner, mesh.neighbour, diag, upper, lower)
    S = scipy.sparse.csr_matrix(A)
    rp, col, mp = O.ldu_to_csr(mesh.n_cells, mesh.owner, mesh.neighbour)
    assert np.array_equal(rp, S.indptr) and np.array_equal(col, S.indices)
    vals = np.concatenate([diag, upper, lower])[mp]
    assert np.array_equal(vals, S.data)
    x = np.cos(np.arange(mesh.n_cells))
    y = scipy.sparse.csr_matrix((vals, col, rp), shape=A.shape) @ x
    assert np.allclose(y, O.amul_asym(mesh.owner, mesh.neighbour, diag, upper, lower, x), rtol=1e-13, atol=1e-15)


def test_normfactor_uses_row_sums_on_asymmetric_system():
    """Q1 on an asymmetric matrix: for a constant psi0, A psi0 = sumA psi0 (row sums), so
    normFactor = sum|b - A psi0| (+1e-20) and the initial residual is exactly 1 up to rounding."""
    m = gen.perturbed(6, 0.2)
    diag, upper, lower, b = asym_system(m, seed=8, skew=0.6)
    _, perf = O.pbicg(m.owner, m.neighbour, diag, upper, lower, b, O.DILU, psi0=np.full(m.n_cells, 1.5),
                      ctl=O.controls(1e-9, 0.0, 1, 1))
    assert perf["initial_residual"] == pytest.approx(1.0, rel=1e-10)


# ---- decomposed PBiCG (O8 + O12, Q31/Q32) ----
from cases import asym_decomposed  # noqa: E402


def _gather(mesh, subs, xs):
    loc = {int(g): i for i, g in enumerate(mesh.gid)}
    out = np.zeros(mesh.n_cells)
    for sm, x in zip(subs, xs):
        out[[loc[int(g)] for g in sm.gid]] = x
    return out


def test_pbicg_decomposed_single_domain_is_pbicg():
    m = gen.perturbed(6, 0.2)
    part = np.zeros(m.n_cells, np.int64)
    subs, systems, (d, u, l, b) = asym_decomposed(m, part, seed=3)
    for kind in (O.DILU, O.ADILU):
        a, pa = O.pbicg_decomposed(subs, systems, None, O.controls(1e-10, 0.0, 500, 0), kind)
        s = systems[0]
        ref, pr = O.pbicg(subs[0].owner, subs[0].neighbour, s["diag"], s["upper"], s["lower"], s["source"], kind, 2,
                          None, O.controls(1e-10, 0.0, 500, 0))
        assert pa["n_iterations"] == pr["n_iterations"] and np.array_equal(a[0], ref)


@pytest.mark.parametrize("P,how", [(2, "block"), (4, "rcb")])
def test_pbicg_decomposed_reaches_global_dense_solution(P, how):
    m = gen.permute(gen.perturbed(8, 0.2), seed=4)
    part = gen.rcb_parts(m, P) if how == "rcb" else gen.block_parts(m, (P, 1, 1))
    subs, systems, (d, u, l, b) = asym_decomposed(m, part, seed=5)
    A = _dense_asym(m.n_cells, m.owner, m.neighbour, d, u, l)
    exact = np.linalg.solve(A, b)
    for kind in (O.DIAGONAL, O.DILU, O.ADILU):
        xs, perf = O.pbicg_decomposed(subs, systems, None, O.controls(1e-13, 0.0, 2000, 0), kind)
        assert perf["converged"] and not perf["singular"]
        got = _gather(m, subs, xs)
        assert np.linalg.norm(got - exact) / np.linalg.norm(exact) < 1e-9, kind


def test_pbicg_decomposed_symmetric_follows_decomposed_pcg():
    """lower = upper, iface_t = iface: BiCG with a symmetric (processor-local DIC) preconditioner
    produces the decomposed CG iterates."""
    m = gen.perturbed(7, 0.2)
    part = gen.block_parts(m, (2, 1, 1))
    subs, systems, _ = asym_decomposed(m, part, seed=6, sym=True)
    lsys = [O.LduSystem(s["diag"], s["upper"], s["source"], s["iface"]) for s in systems]
    for n in (1, 4, 12):
        xb, pb = O.pbicg_decomposed(subs, systems, None, O.controls(0.0, 0.0, n, n), O.DIC)
        xc, pc = O.pcg_decomposed(subs, lsys, None, O.controls(0.0, 0.0, n, n), kind=O.DIC)
        gb, gc = _gather(m, subs, xb), _gather(m, subs, xc)
        assert np.linalg.norm(gb - gc) / np.linalg.norm(gc) < 1e-11, n
