"""Pins for oracle O11dd: GAMG on a decomposed mesh (readings Q36-Q38).

The paper runs GAMG decomposed over 1-8 GPUs with the coarsening unchanged (P:665, P:682,
P:708-710); OpenFOAM keeps the agglomeration processor-local and agglomerates the processor
interfaces alongside.  What pins the decomposed oracle, independently of itself:
- one domain: bitwise the single-domain O11 GAMG (already pinned in test_oracle_gamg.py);
- the decomposed hierarchy: every level's global operator (domain blocks + coarse interface
  coefficients) equals the dense Galerkin product R^T A R of the global fine matrix, with R
  the 0/1 restriction of the processor-local agglomerates; agglomerates never cross domains;
  both sides of a coarse interface face carry bitwise the same coefficient;
- one decomposed GAMG iteration equals the textbook dense V-cycle on those global operators
  (global Jacobi / two-stage Gauss-Seidel with a domain-block lower triangle, Q38);
- the level rule Q36 and convergence to the dense global solution.
"""
import numpy as np
import pytest

import gen
import oracle as O
from cases import dense_ldu
from test_oracle_decomposed import _decomposed_case


def _case(n=6, P=2, a=0.25, seed=3, how="rcb"):
    m = gen.permute(gen.perturbed(n, a), seed=seed)
    gamma = gen.gamma_lognormal(m)
    b = gen.rhs(m)
    part = gen.rcb_parts(m, P) if how == "rcb" else gen.block_parts(m, (P, 1, 1))
    subs, systems = _decomposed_case(m, part, gamma, b, ref=0)
    g = O.assemble(m, gamma, 0, 0.0, source=b)
    return m, g, subs, systems


def _domain_major(m, subs):
    """global cell index of each domain-major position"""
    loc = {int(x): i for i, x in enumerate(m.gid)}
    return np.array([loc[int(x)] for sm in subs for x in sm.gid], dtype=np.int64)


def _dense_dd(subs, systems):
    """the decomposed system as one dense matrix, cells domain-major, built in Python from each
    domain's LDU arrays and processor coefficients (the reference cell's penalty is applied to
    the domain's internal diagonal, so at a reference cell on a processor boundary this is
    not the undecomposed matrix -- the solution is the same: b has zero mean)"""
    off = np.cumsum([0] + [sm.n_cells for sm in subs])
    where = {}
    for r, sm in enumerate(subs):
        for i, x in enumerate(sm.gid):
            where[int(x)] = off[r] + i
    n = off[-1]
    A = np.zeros((n, n))
    for r, (sm, s) in enumerate(zip(subs, systems)):
        o = off[r]
        A[o:o + sm.n_cells, o:o + sm.n_cells] = dense_ldu(sm.n_cells, sm.owner, sm.neighbour, s.diag, s.upper)
        for p, c in zip(O.processor_patches(sm), s.iface):
            for fc, g, v in zip(p.face_cells, p.neighbour_gid, c):
                A[o + fc, where[int(g)]] += v
    return A


def _R(ftc, nc):
    R = np.zeros((ftc.shape[0], nc))
    R[np.arange(ftc.shape[0]), ftc] = 1.0
    return R


def _levels(subs, systems, gp):
    """dense global operators of the decomposed hierarchy + the global restriction maps"""
    As, ftcs = [], []
    l = 0
    while True:
        try:
            A, ftc = O.gamg_dd_dense_level(subs, systems, l, gp)
        except ValueError:
            break
        As.append(A)
        if l > 0:
            ftcs.append(ftc[:As[l - 1].shape[0]].copy())
        l += 1
    return As, ftcs


def test_single_domain_is_bitwise_o11():
    m = gen.permute(gen.perturbed(7, 0.2), seed=5)
    s = O.assemble(m, gen.gamma_lognormal(m), 0, 0.0, source=gen.rhs(m))
    for gp in (O.gamg_params(), O.gamg_params(n_pre=1, n_post=1, smoother=O.GS2, n_inner=2)):
        ctl = O.controls(1e-8, 0.0, 100, 0)
        psi1, perf1 = O.gamg(m, s, None, ctl, gp)
        psis, perfd = O.gamg_decomposed([m], [s], None, ctl, gp)
        assert np.array_equal(psis[0], psi1)
        assert perfd["n_iterations"] == perf1["n_iterations"]
        assert perfd["final_residual"] == perf1["final_residual"]
        assert perfd["level_cells"][0] == perf1["level_cells"]
        assert all(v == 0 for v in perfd["level_ifaces"][0])


@pytest.mark.parametrize("P,how", [(2, "block"), (3, "rcb"), (4, "rcb")])
def test_hierarchy_is_galerkin_of_global_matrix(P, how):
    m, g, subs, systems = _case(6, P, how=how)
    gp = O.gamg_params(n_coarsest_cells=4)
    As, ftcs = _levels(subs, systems, gp)
    assert len(As) >= 3
    A = _dense_dd(subs, systems)
    scale = np.max(np.abs(A))
    assert np.array_equal(As[0], A)
    sizes = [[sm.n_cells for sm in subs]]
    for l in range(1, len(As)):
        nc = As[l].shape[0]
        R = _R(ftcs[l - 1], nc)
        assert np.allclose(As[l], R.T @ As[l - 1] @ R, rtol=0, atol=1e-13 * scale)
        assert np.array_equal(As[l], As[l].T)  # both sides of every coarse interface: same bits
        # agglomerates stay inside their domain (domain-major blocks map to domain-major blocks)
        _, out = O.gamg_decomposed(subs, systems, None, O.controls(0.0, 0.0, 0, 0), gp)
        fine = out["level_cells"]
        fo = np.cumsum([0] + [fine[p][l - 1] for p in range(P)])
        co = np.cumsum([0] + [fine[p][l] for p in range(P)])
        for p in range(P):
            f = ftcs[l - 1][fo[p]:fo[p + 1]]
            assert f.min() >= co[p] and f.max() < co[p + 1]
        sizes.append([fine[p][l] for p in range(P)])
    # Q36: stop when the global count is <= P * nCellsInCoarsestLevel (or no reduction)
    tot = [sum(s) for s in sizes]
    assert all(t > P * gp.n_coarsest_cells for t in tot[:-1])
    assert tot[-1] <= P * gp.n_coarsest_cells or tot[-1] == tot[-2]


def _dense_cycle_dd(As, Rs, doms, b, gp):
    """Textbook V-cycle with dense Galerkin operators (correction form, zero initial guess);
    Richardson is global-pointwise, the two-stage Gauss-Seidel lower triangle is restricted to
    each domain's block (Q38).  doms[l][i]: the domain of global cell i of level l."""
    def smooth(l, bl, x):
        A = As[l]
        r = bl - A @ x
        if gp.smoother != O.GS2:
            return x + gp.omega * (r / np.diag(A))
        Lo, d = np.tril(A, -1) * (doms[l][:, None] == doms[l][None, :]), np.diag(A)
        z = r / d
        for _ in range(gp.n_inner):
            z = (r - Lo @ z) / d
        return x + z
    L = len(As)
    x, bl, rl = [None] * L, [None] * L, [None] * L
    bl[0] = b
    for l in range(L - 1):
        x[l] = np.zeros(As[l].shape[0])
        for _ in range(gp.n_pre):
            x[l] = smooth(l, bl[l], x[l])
        rl[l] = bl[l] - As[l] @ x[l]
        bl[l + 1] = Rs[l].T @ rl[l]
    x[L - 1] = np.linalg.solve(As[L - 1], bl[L - 1])
    for l in range(L - 2, -1, -1):
        c = Rs[l] @ x[l + 1]
        if gp.scale:
            den = c @ (As[l] @ c)
            a = np.clip((c @ rl[l]) / den, 0.0, 2.0) if abs(den) > 1e-300 else 1.0
            c = a * c
        x[l] = x[l] + c
        for _ in range(gp.n_post):
            x[l] = smooth(l, bl[l], x[l])
    return x[0]


@pytest.mark.parametrize("P,scale,n_pre,n_post,omega,smoother,n_inner", [
    (2, True, 0, 2, 0.75, O.RICHARDSON, 1), (3, False, 1, 1, 0.6, O.RICHARDSON, 1),
    (4, True, 1, 2, 0.75, O.RICHARDSON, 1), (2, True, 0, 2, 0.75, O.GS2, 1), (3, True, 1, 1, 0.75, O.GS2, 3),
])
def test_one_cycle_equals_dense_multigrid(P, scale, n_pre, n_post, omega, smoother, n_inner):
    m, g, subs, systems = _case(5, P)
    gp = O.gamg_params(n_pre=n_pre, n_post=n_post, scale=scale, n_coarsest_cells=6, omega=omega,
                       coarsest_rel_tol=1e-15, coarsest_max_iter=500, smoother=smoother, n_inner=n_inner)
    _, ftcs = _levels(subs, systems, gp)
    A = _dense_dd(subs, systems)
    As, Rs = [A], []
    doms = [np.repeat(np.arange(P), [sm.n_cells for sm in subs])]
    for f in ftcs:
        R = _R(f, int(f.max()) + 1)
        Rs.append(R)
        As.append(R.T @ As[-1] @ R)
        d = np.zeros(R.shape[1], dtype=np.int64)
        d[f] = doms[-1]
        doms.append(d)
    assert len(As) >= 3
    psi0 = [np.cos(sm.gid.astype(np.float64) * 0.7) for sm in subs]
    psis, perf = O.gamg_decomposed(subs, systems, psi0, O.controls(0.0, 0.0, 1, 1), gp)
    assert perf["n_iterations"] == 1 and perf["levels"] == len(As)
    x0 = np.concatenate(psi0)
    bb = np.concatenate([s.source for s in systems])
    ref = x0 + _dense_cycle_dd(As, Rs, doms, bb - A @ x0, gp)
    got = np.concatenate(psis)
    assert np.allclose(got, ref, rtol=0, atol=1e-10 * np.max(np.abs(ref)))


@pytest.mark.parametrize("P", [2, 4])
def test_converges_to_dense_solution(P):
    m, g, subs, systems = _case(6, P)
    psis, perf = O.gamg_decomposed(subs, systems, None, O.controls(1e-13, 0.0, 200, 0))
    assert perf["converged"]
    A = dense_ldu(m.n_cells, m.owner, m.neighbour, g.diag, g.upper)
    x = np.linalg.solve(A, g.source)
    dm = _domain_major(m, subs)
    got = np.concatenate(psis)
    assert np.linalg.norm(got - x[dm]) <= 1e-9 * np.linalg.norm(x)
    # fewer V-cycles than PCG iterations to the same tolerance
    _, pp = O.pcg_decomposed(subs, systems, None, O.controls(1e-13, 0.0, 2000, 0))
    assert perf["n_iterations"] < pp["n_iterations"]


def test_decomposition_changes_the_cycle_but_not_the_limit():
    m, g, subs, systems = _case(6, 3)
    ctl = O.controls(1e-10, 0.0, 200, 0)
    psi1, p1 = O.gamg(m, g, None, ctl)
    psis, pP = O.gamg_decomposed(subs, systems, None, ctl)
    dm = _domain_major(m, subs)
    assert np.linalg.norm(np.concatenate(psis) - psi1[dm]) <= 1e-7 * np.linalg.norm(psi1)
    assert abs(p1["n_iterations"] - pP["n_iterations"]) <= max(3, p1["n_iterations"] // 2)
