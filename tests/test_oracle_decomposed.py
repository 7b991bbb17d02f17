"""Pins for oracle O8 (decomposed PCG) and the processor-patch assembly (Q9, Q13).

Domain decomposition with processor patches: PAPER.md P:87, P:110-111, P:682
("hierarchical"); interface update P:89.  P8:
the P-way solution equals the 1-way one up to round-off (the pointwise
preconditioner leaves the Krylov sequence unchanged)."""
import numpy as np
import pytest

import gen
import oracle as O


def _decomposed_case(mesh, part, gamma, b, ref=0):
    P = int(part.max()) + 1
    subs = gen.decompose(mesh, part, P)
    gs = gen.split_cell_field(gamma, part, P) if gamma is not None else [None] * P
    bs = gen.split_cell_field(b, part, P)
    halo = O.gamma_halo(subs, gs) if gamma is not None else [None] * P
    systems = []
    for r, m in enumerate(subs):
        ref_local = -1
        if ref >= 0:
            hit = np.nonzero(m.gid == mesh.gid[ref])[0]
            ref_local = int(hit[0]) if hit.size else -1
        systems.append(O.assemble(m, gs[r], ref_local, 0.0, source=bs[r], gamma_remote=halo[r]))
    return subs, systems


@pytest.mark.parametrize("P,how", [(2, "block"), (4, "rcb"), (8, "rcb")])
def test_decomposed_matrix_equals_global(P, how):
    m = gen.permute(gen.perturbed(8, 0.2), seed=3)
    gamma = gen.gamma_lognormal(m)
    part = gen.rcb_parts(m, P) if how == "rcb" else gen.block_parts(m, (2, 1, 1))
    g = O.assemble(m, gamma, -1)
    subs, systems = _decomposed_case(m, part, gamma, np.zeros(m.n_cells), ref=-1)
    # interior coefficients bitwise equal (same geometry, same formula)
    gidx = {int(f): i for i, f in enumerate(m.gface)}
    for sm, s in zip(subs, systems):
        idx = np.array([gidx[int(f)] for f in sm.gface], dtype=np.int64)
        assert np.array_equal(s.upper, g.upper[idx])
        # processor coefficients: equal to the undecomposed face's coefficient (global orientation, Q9)
        for p, c in zip(O.processor_patches(sm), s.iface):
            gi = np.array([gidx[int(f)] for f in p.global_face], dtype=np.int64)
            assert np.array_equal(c, g.upper[gi])
        # diagonal equal up to summation order
        loc = {int(x): i for i, x in enumerate(m.gid)}
        gd = g.diag[[loc[int(x)] for x in sm.gid]]
        assert np.allclose(s.diag, gd, rtol=4e-16 * 8, atol=0)
    # both sides of a processor face see the same coefficient
    seen = {}
    for sm, s in zip(subs, systems):
        for p, c in zip(O.processor_patches(sm), s.iface):
            for f, v in zip(p.global_face, c):
                if int(f) in seen:
                    assert seen[int(f)] == v
                else:
                    seen[int(f)] = v


@pytest.mark.parametrize("P", [2, 3, 4])
def test_p8_decomposition_invariance(P):
    m = gen.permute(gen.perturbed(10, 0.15), seed=2)
    gamma = gen.gamma_lognormal(m)
    b = gen.rhs(m)
    ctl = O.controls(1e-9, 0.0, 2000, 0)
    psi1, perf1, _ = O.solve_case(m, gamma, b, 0, 0.0, ctl)
    part = gen.rcb_parts(m, P)
    subs, systems = _decomposed_case(m, part, gamma, b, ref=0)
    psis, perfP = O.pcg_decomposed(subs, systems, None, ctl)
    assert abs(perfP["n_iterations"] - perf1["n_iterations"]) <= 1
    full = np.empty(m.n_cells)
    loc = {int(x): i for i, x in enumerate(m.gid)}
    for sm, ps in zip(subs, psis):
        full[[loc[int(x)] for x in sm.gid]] = ps
    # compare at equal iteration counts (Q11)
    n = min(perfP["n_iterations"], perf1["n_iterations"])
    ctl_n = O.controls(0.0, 0.0, n, n)
    psi1, _, _ = O.solve_case(m, gamma, b, 0, 0.0, ctl_n)
    psis, _ = O.pcg_decomposed(subs, systems, None, ctl_n)
    for sm, ps in zip(subs, psis):
        full[[loc[int(x)] for x in sm.gid]] = ps
    assert np.linalg.norm(full - psi1) / np.linalg.norm(psi1) < 1e-9


def test_decomposed_amul_with_exchanged_halo_equals_global():
    m = gen.perturbed(6, 0.2)
    gamma = gen.gamma_lognormal(m)
    g = O.assemble(m, gamma, -1)
    part = gen.block_parts(m, (2, 2, 1))
    subs, systems = _decomposed_case(m, part, gamma, np.zeros(m.n_cells), ref=-1)
    x = np.sin(np.arange(m.n_cells) * 0.37)
    y = O.amul(m, g.diag, g.upper, x)
    xs = gen.split_cell_field(x, part, 4)
    halo = O.gamma_halo(subs, xs)  # same lookup: value of the remote cell
    for r, (sm, s) in enumerate(zip(subs, systems)):
        yl = O.amul(sm, s.diag, s.upper, xs[r], iface=s.iface, x_remote=halo[r])
        loc = {int(v): i for i, v in enumerate(m.gid)}
        assert np.allclose(yl, y[[loc[int(v)] for v in sm.gid]], rtol=1e-14, atol=1e-14)


# ---- O8 + O12: processor-local preconditioners on decomposed meshes (Q31) ----

def _local_M(sm, s, kind):
    """dense M_p = (D* + L) D*^-1 (D* + U) of one domain's own faces (DIC), or diag (diagonal)"""
    n = sm.n_cells
    if kind == O.DIAGONAL:
        return np.diag(s.diag)
    rD = O.ilu_factor(sm.owner, sm.neighbour, s.diag, s.upper)
    Lo = np.zeros((n, n))
    Up = np.zeros((n, n))
    Lo[sm.neighbour, sm.owner] = s.upper
    Up[sm.owner, sm.neighbour] = s.upper
    Ds = np.diag(1.0 / rD)
    return (Ds + Lo) @ np.diag(rD) @ (Ds + Up)


def test_decomposed_pc_single_domain_is_pcg_pc():
    m = gen.perturbed(7, 0.2)
    s = O.assemble(m, gen.gamma_lognormal(m), 0, 0.0, source=gen.rhs(m))
    for kind in (O.DIC, O.ADILU):
        a, pa = O.pcg_decomposed([m], [s], None, O.controls(1e-9), kind=kind)
        b, pb = O.pcg_pc(m, s, kind, 2, None, O.controls(1e-9))
        assert pa["n_iterations"] == pb["n_iterations"] and np.array_equal(a[0], b)


@pytest.mark.parametrize("kind", [O.DIC, O.DIAGONAL])
def test_decomposed_pc_first_iterate_is_block_local_preconditioner(kind):
    """With processor-local preconditioning, M = blockdiag(M_1, ..., M_P) of the domains' own
    faces, and the first PCG iterate from psi = 0 is psi_1 = alpha M^-1 b with
    alpha = (b.M^-1 b) / (M^-1 b . A M^-1 b), A the GLOBAL matrix (interfaces included)."""
    m = gen.perturbed(6, 0.2)
    gamma, b = gen.gamma_lognormal(m), gen.rhs(m)
    part = gen.block_parts(m, (2, 1, 1))
    subs, systems = _decomposed_case(m, part, gamma, b, ref=0)
    psi, perf = O.pcg_decomposed(subs, systems, None, O.controls(0.0, 0.0, 1, 1), kind=kind)
    g = O.assemble(m, gamma, 0, 0.0, source=b)
    from cases import dense_ldu
    A = dense_ldu(m.n_cells, m.owner, m.neighbour, g.diag, g.upper)
    loc = {int(x): i for i, x in enumerate(m.gid)}
    Mi = np.zeros_like(A)
    for sm, s in zip(subs, systems):
        idx = np.array([loc[int(x)] for x in sm.gid])
        Mi[np.ix_(idx, idx)] = np.linalg.inv(_local_M(sm, s, kind))
    z = Mi @ g.source
    alpha = (z @ g.source) / (z @ (A @ z))
    ref = alpha * z
    got = np.zeros(m.n_cells)
    for sm, x in zip(subs, psi):
        got[[loc[int(gg)] for gg in sm.gid]] = x
    assert np.allclose(got, ref, rtol=1e-11, atol=1e-14 * np.max(np.abs(ref)))


def test_decomposed_dic_converges_to_global_solution():
    m = gen.permute(gen.perturbed(8, 0.2), seed=2)
    gamma, b = gen.gamma_lognormal(m), gen.rhs(m)
    part = gen.rcb_parts(m, 4)
    subs, systems = _decomposed_case(m, part, gamma, b, ref=0)
    psi, perf = O.pcg_decomposed(subs, systems, None, O.controls(1e-11, 0.0, 2000, 0), kind=O.DIC)
    g = O.assemble(m, gamma, 0, 0.0, source=b)
    from cases import dense_ldu
    exact = np.linalg.solve(dense_ldu(m.n_cells, m.owner, m.neighbour, g.diag, g.upper), g.source)
    loc = {int(x): i for i, x in enumerate(m.gid)}
    got = np.zeros(m.n_cells)
    for sm, x in zip(subs, psi):
        got[[loc[int(gg)] for gg in sm.gid]] = x
    assert perf["converged"] and np.linalg.norm(got - exact) / np.linalg.norm(exact) < 1e-8
    _, p1 = O.pcg_decomposed(subs, systems, None, O.controls(1e-11, 0.0, 2000, 0))
    assert perf["n_iterations"] < p1["n_iterations"]  # DIC (block-local) beats the diagonal
