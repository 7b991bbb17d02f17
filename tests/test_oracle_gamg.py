"""Pins for oracle O11: GAMG with the Richardson smoother ("GAMG ...
Richardson smoother, diagonal at the coarsest", pGAMG controls P:1043-1052, profile rows
restrictField / prolongField / agglomerateMatrix / scale / Vcycle P:517-545; readings Q22-Q28).

Independent of the oracle's own loops:
- agglomeration: hand-derived examples of the pairing rule (Q22) and invariants (connected
  agglomerates, contiguous numbering, strict coarsening);
- coarse addressing: the distinct sparsity pattern of the dense product R^T |A| R;
- Galerkin: agglomerateMatrix equals the dense product R^T A R (R = 0/1 restriction);
- restriction = R^T r, prolongation = R x (adjoint pair);
- one GAMG iteration equals a textbook two-grid / three-grid cycle written with dense
  matrices (Galerkin coarse operator, weighted Jacobi, exact coarse solve, energy-optimal
  correction scaling clamped to [0, 2]);
- two-stage Gauss-Seidel (Q30): the same dense cycle with z = D^-1 (r - L z) inner iterations,
  and with enough inner iterations the exact forward triangular solve (scipy);
- single-level hierarchy: one cycle is the exact (dense) solve;
- fixed point and convergence to the dense solution, far fewer cycles than PCG iterations."""
import numpy as np
import pytest

import gen
import oracle as O
from cases import dense_ldu


def _chain(n):
    return np.arange(n - 1, dtype=np.int32), np.arange(1, n, dtype=np.int32)


def test_agglomerate_hand_examples():
    # 4-chain, weights [1, 3, 2]: cell 0 pairs with its only free neighbour 1; cell 2's free
    # neighbour is 3 -> [0, 0, 1, 1].
    o, nb = _chain(4)
    ftc, nc = O.agglomerate(4, o, nb, [1.0, 3.0, 2.0])
    assert ftc.tolist() == [0, 0, 1, 1] and nc == 2
    # 3-chain: cell 2 has no free neighbour -> joins cell 1's agglomerate.
    o, nb = _chain(3)
    ftc, nc = O.agglomerate(3, o, nb, [1.0, 1.0])
    assert ftc.tolist() == [0, 0, 0] and nc == 1
    # star 0-{1,2,3} with weights [1, 5, 2]: 0 pairs with 2 (largest); 1 and 3 have no free
    # neighbour and only one face each -> both join agglomerate 0.
    ftc, nc = O.agglomerate(4, np.array([0, 0, 0], np.int32), np.array([1, 2, 3], np.int32), [1.0, 5.0, 2.0])
    assert ftc.tolist() == [0, 0, 0, 0] and nc == 1
    # 2x2 grid 0-1, 0-2, 1-3, 2-3 with equal weights: ties -> first face (0-1); then 2-3.
    o = np.array([0, 0, 1, 2], np.int32)
    nb = np.array([1, 2, 3, 3], np.int32)
    ftc, nc = O.agglomerate(4, o, nb, np.ones(4))
    assert ftc.tolist() == [0, 0, 1, 1] and nc == 2
    # same grid, face 0-2 strongest -> columns {0,2}, {1,3}
    ftc, nc = O.agglomerate(4, o, nb, [1.0, 2.0, 1.0, 1.0])
    assert ftc.tolist() == [0, 1, 0, 1] and nc == 2
    # an isolated cell (no faces) is its own agglomerate
    ftc, nc = O.agglomerate(3, np.array([0], np.int32), np.array([1], np.int32), [1.0])
    assert ftc.tolist() == [0, 0, 1] and nc == 2


def _connected_within(n, owner, neighbour, ftc):
    nc = ftc.max() + 1
    adj = [[] for _ in range(n)]
    for a, b in zip(owner, neighbour):
        if ftc[a] == ftc[b]:
            adj[a].append(b)
            adj[b].append(a)
    for c in range(nc):
        mem = np.flatnonzero(ftc == c)
        seen = {mem[0]}
        st = [mem[0]]
        while st:
            x = st.pop()
            for y in adj[x]:
                if y not in seen:
                    seen.add(y)
                    st.append(y)
        if len(seen) != len(mem):
            return False
    return True


@pytest.mark.parametrize("mesh", [gen.cube(7), gen.permute(gen.perturbed(6, 0.3), seed=4), gen.cavity2d(9)],
                         ids=["cube", "perturbed-permuted", "cavity"])
def test_agglomerate_invariants(mesh):
    ftc, nc = O.agglomerate(mesh.n_cells, mesh.owner, mesh.neighbour, mesh.magSf)
    assert ftc.min() == 0 and ftc.max() == nc - 1
    assert nc <= (mesh.n_cells + 1) // 2 + 1
    first = [int(np.flatnonzero(ftc == c)[0]) for c in range(nc)]
    assert first == sorted(first)  # numbered in order of first (lowest) member
    assert _connected_within(mesh.n_cells, mesh.owner, mesh.neighbour, ftc)


def _R(ftc, nc):
    R = np.zeros((ftc.shape[0], nc))
    R[np.arange(ftc.shape[0]), ftc] = 1.0
    return R


@pytest.mark.parametrize("mesh", [gen.perturbed(6, 0.3), gen.permute(gen.box(7, 5, 4), seed=2)],
                         ids=["perturbed", "permuted-box"])
def test_coarse_addressing_and_galerkin_equal_dense_product(mesh):
    g = gen.gamma_lognormal(mesh)
    s = O.assemble(mesh, g, 0, 0.0)
    ftc, nc = O.agglomerate(mesh.n_cells, mesh.owner, mesh.neighbour, mesh.magSf)
    co, cn, fr, cw = O.coarse_addressing(mesh.owner, mesh.neighbour, ftc, mesh.magSf)
    assert O.check_addressing(nc, co, cn) == 0
    A = dense_ldu(mesh.n_cells, mesh.owner, mesh.neighbour, s.diag, s.upper)
    R = _R(ftc, nc)
    Ac = R.T @ A @ R
    pat = (R.T @ (np.abs(A) > 0) @ R) > 0
    iu = np.argwhere(np.triu(pat, 1))
    assert np.array_equal(iu[:, 0], co) and np.array_equal(iu[:, 1], cn)
    # coarse face weights: sums of fine face areas between the two agglomerates
    W = np.zeros((mesh.n_cells, mesh.n_cells))
    W[mesh.owner, mesh.neighbour] = mesh.magSf
    Wc = R.T @ (W + W.T) @ R
    assert np.allclose(cw, Wc[co, cn], rtol=1e-14)
    cd, cu = O.agglomerate_matrix(mesh.owner, ftc, fr, s.diag, s.upper, nc, co.shape[0])
    Cd = dense_ldu(nc, co, cn, cd, cu)
    assert np.allclose(Cd, Ac, rtol=0, atol=1e-13 * np.max(np.abs(Ac)))
    # fine faces inside an agglomerate map to -1, the others to the coarse face of their pair
    inside = ftc[mesh.owner] == ftc[mesh.neighbour]
    assert np.all(fr[inside] == -1) and np.all(fr[~inside] >= 0)
    lo = np.minimum(ftc[mesh.owner], ftc[mesh.neighbour])[~inside]
    assert np.array_equal(co[fr[~inside]], lo)


def test_restrict_prolong_adjoint():
    m = gen.perturbed(6, 0.2)
    ftc, nc = O.agglomerate(m.n_cells, m.owner, m.neighbour, m.magSf)
    rng = np.random.default_rng(1)
    r, xc = rng.standard_normal(m.n_cells), rng.standard_normal(nc)
    R = _R(ftc, nc)
    rc = O.restrict_field(ftc, r, nc)
    assert np.allclose(rc, R.T @ r, rtol=1e-14, atol=1e-14)
    assert np.dot(rc, xc) == pytest.approx(np.dot(r, R @ xc), rel=1e-13)


def _dense_smooth(A, b, x, gp):
    if gp.smoother == O.GS2:
        r = b - A @ x
        if gp.n_inner >= A.shape[0]:  # D^-1 L is nilpotent: the inner iteration is the exact forward solve
            import scipy.linalg
            return x + scipy.linalg.solve_triangular(np.tril(A), r, lower=True)
        Lo, d = np.tril(A, -1), np.diag(A)
        z = r / d
        for _ in range(gp.n_inner):
            z = (r - Lo @ z) / d
        return x + z
    return x + gp.omega * ((b - A @ x) / np.diag(A))


def _dense_cycle(As, Rs, b, gp):
    """Textbook V-cycle with dense Galerkin operators (correction form, zero initial guess)."""
    L = len(As)
    x = [None] * L
    bl = [None] * L
    rl = [None] * L
    bl[0] = b
    for l in range(L - 1):
        x[l] = np.zeros(As[l].shape[0])
        for _ in range(gp.n_pre):
            x[l] = _dense_smooth(As[l], bl[l], x[l], gp)
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
            x[l] = _dense_smooth(As[l], bl[l], x[l], gp)
    return x[0]


@pytest.mark.parametrize("n_coarsest,scale,n_pre,n_post,omega,smoother,n_inner", [
    (40, True, 0, 2, 0.75, 0, 1), (40, False, 1, 1, 0.6, 0, 1), (20, True, 1, 2, 0.75, 0, 1),
    (10, True, 0, 3, 0.9, 0, 1),
    (10, True, 1, 1, 1.6, 0, 1),   # omega = 1.6 (divergent Jacobi): the raw scale factor goes negative -> clamp 0
    (10, True, 0, 2, 0.75, 1, 1),  # two-stage Gauss-Seidel (Q30), one inner iteration
    (20, True, 1, 1, 0.75, 1, 3),
    (40, False, 0, 1, 0.75, 1, 0),  # zero inner iterations: a plain Jacobi step
    (40, True, 1, 2, 0.75, 1, 64),  # 64 >= cells: exact Gauss-Seidel (forward triangular solve)
])
def test_one_cycle_equals_dense_multigrid(n_coarsest, scale, n_pre, n_post, omega, smoother, n_inner):
    m = gen.perturbed(4, 0.25)  # 64 cells -> 32 -> 16 -> 8 ...
    g = gen.gamma_lognormal(m)
    s = O.assemble(m, g, 0, 0.0, source=gen.rhs(m))
    gp = O.gamg_params(n_pre=n_pre, n_post=n_post, scale=scale, n_coarsest_cells=n_coarsest, omega=omega,
                       coarsest_rel_tol=1e-15, coarsest_max_iter=500, smoother=smoother, n_inner=n_inner)
    lv = O.gamg_hierarchy(m, gp)
    A = dense_ldu(m.n_cells, m.owner, m.neighbour, s.diag, s.upper)
    As, Rs = [A], []
    for (n, _, _, ftc) in lv[:-1]:
        R = _R(ftc, int(ftc.max()) + 1)
        Rs.append(R)
        As.append(R.T @ As[-1] @ R)
    assert len(As) >= 2
    psi0 = np.cos(np.arange(m.n_cells) * 0.7)
    psi, perf = O.gamg(m, s, psi0, O.controls(0.0, 0.0, 1, 1), gp)
    assert perf["n_iterations"] == 1 and perf["levels"] == len(As)
    ref = psi0 + _dense_cycle(As, Rs, s.source - A @ psi0, gp)
    assert np.allclose(psi, ref, rtol=0, atol=1e-10 * np.max(np.abs(ref)))


def test_single_level_cycle_is_exact_solve():
    m = gen.box(3, 2, 1)  # 6 cells <= 10: the finest level is the coarsest
    s = O.assemble(m, gen.gamma_lognormal(m), 0, 0.0, source=gen.rhs(m))
    psi, perf = O.gamg(m, s, None, O.controls(0.0, 0.0, 1, 1), O.gamg_params(coarsest_rel_tol=1e-15))
    assert perf["levels"] == 1
    A = dense_ldu(m.n_cells, m.owner, m.neighbour, s.diag, s.upper)
    assert np.allclose(psi, np.linalg.solve(A, s.source), rtol=1e-12, atol=1e-14)


def test_gs2_converges_faster_than_richardson():
    """Two-stage Gauss-Seidel (Q30) is the stronger smoother: fewer cycles to the same tolerance."""
    m = gen.cube(12)
    s = O.assemble(m, gen.gamma_lognormal(m), 0, 0.0, source=gen.rhs(m))
    _, pr = O.gamg(m, s, None, O.controls(1e-9, 0.0, 300, 0))
    _, pg = O.gamg(m, s, None, O.controls(1e-9, 0.0, 300, 0), O.gamg_params(smoother=O.GS2))
    assert pr["converged"] and pg["converged"] and pg["n_iterations"] < pr["n_iterations"]


def test_fixed_point_and_convergence():
    m = gen.cube(16)
    s = O.assemble(m, gen.gamma_lognormal(m), 0, 0.0, source=gen.rhs(m))
    A = dense_ldu(m.n_cells, m.owner, m.neighbour, s.diag, s.upper)
    exact = np.linalg.solve(A, s.source)
    psi, perf = O.gamg(m, s, None, O.controls(1e-10, 0.0, 300, 0))
    _, pp = O.pcg(m, s, None, O.controls(1e-10))
    assert perf["converged"] and perf["levels"] >= 6
    assert perf["n_iterations"] * 3 < pp["n_iterations"]
    assert np.linalg.norm(psi - exact) / np.linalg.norm(exact) < 1e-7
    # starting from the exact solution: converged with no cycle
    psi2, p2 = O.gamg(m, s, exact, O.controls(1e-10, 0.0, 300, 0))
    assert p2["n_iterations"] == 0 and p2["initial_residual"] < 1e-10
    # relTol stop (pGAMG style): stops at the first cycle below relTol * initial
    _, p3 = O.gamg(m, s, None, O.controls(0.0, 1e-3, 300, 0))
    assert p3["final_residual"] < 1e-3 * p3["initial_residual"]
    _, p4 = O.gamg(m, s, None, O.controls(0.0, 1e-3, p3["n_iterations"] - 1, 0))
    assert p4["final_residual"] >= 1e-3 * p4["initial_residual"]
