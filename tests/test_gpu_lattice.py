"""Amul variant 12/13 (lattice slots) against the oracle on the GPU.

On a structured numbering every face's column offset is one of K <= 3 values, and the rows are
read from slot arrays with no index arrays: the result must still be BITWISE the oracle's face
loop (reading Q10), including the sign of zero (the absent slots are skipped, not added as 0),
the ragged tail of the last warp, K = 1 / 2 / 3, isolated cells, fixedValue walls and a
coefficient refresh per call.  Inside PCG it must meet the north_star bar (iterations +-2,
1e-9 relative L2 at matched counts, Q11), and it must be the layout the hot loop actually runs
(spuma_stats.amul_variant)."""
import numpy as np
import pytest

import gen
import oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
import paper_2512_22215_b200 as P  # noqa: E402
from gpu_helpers import dev, gpu_solve_case  # noqa: E402

F64 = dict(dtype=torch.float64, device="cuda")


def _bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def _fixed_value_cube(n):
    m = gen.perturbed(n, 0.2)
    m = gen.set_kind(m, "xmin", gen.FIXED_VALUE, np.linspace(0, 1, m.patches[0].n_faces))
    return gen.set_kind(m, "zmax", gen.FIXED_VALUE, np.full(m.patches[5].n_faces, 0.25))


LATTICE = [("cube13", lambda: gen.cube(13), 3), ("box-ragged", lambda: gen.box(37, 5, 3, (1.0, 0.2, 0.1)), 3),
           ("cavity2d", lambda: gen.cavity2d(20), 2), ("chain", lambda: gen.box(101, 1, 1), 1),
           ("perturbed", lambda: gen.perturbed(11, 0.3), 3), ("fixed-value", lambda: _fixed_value_cube(9), 3),
           ("weak-block", lambda: gen.weak_block(10, (1, 1, 1), 0), 3)]


@pytest.mark.parametrize("variant", [12, 13])
@pytest.mark.parametrize("name,make,K", LATTICE, ids=[c[0] for c in LATTICE])
def test_lattice_amul_bit_exact(name, make, K, variant):
    m = make()
    assert len(P.spuma.host_lattice_offsets(m.n_cells, m.owner, m.neighbour)) == K
    rng = np.random.default_rng(11)
    diag = rng.uniform(-4, -1, m.n_cells)
    x = rng.standard_normal(m.n_cells)
    x[rng.random(m.n_cells) < 0.2] = 0.0  # diag * 0 = -0.0: absent slots must not turn it into +0.0
    h = P.Mesh.from_mesh(m)
    h.set_option(P.spuma.OPT_AMUL_VARIANT, variant)
    y = torch.empty(m.n_cells, **F64)
    for it in range(2):  # the slot copy is refreshed per call
        upper = rng.uniform(0.1, 1, m.n_faces)
        h.amul(dev(diag), dev(upper), None, dev(x), y)
        assert np.array_equal(_bits(y.cpu().numpy()), _bits(O.amul(m, diag, upper, x))), it
    assert h.get_stats()["amul_variant"] == variant
    h.free()


def test_lattice_amul_sign_of_zero_and_isolated_cells():
    # cells 0-1-2 chained, cell 3 isolated: K = 1; x = 0 -> y = diag * 0 (+ u * 0 where a face exists)
    o, nb = np.array([0, 1], np.int32), np.array([1, 2], np.int32)
    n = 4
    C = np.stack([np.arange(n, dtype=float), np.zeros(n), np.zeros(n)], 1)
    m = gen.Mesh(n, o, nb, np.tile([1.0, 0.0, 0.0], (2, 1)), np.ones(2), 0.5 * (C[o] + C[nb]), C, np.ones(n), [])
    h = P.Mesh.from_mesh(m)
    assert h.get_stats()["amul_variant"] == 12
    diag, upper = np.array([-1.0, -2.0, -3.0, -4.0]), np.array([0.5, 0.25])
    for x in (np.zeros(n), np.array([0.0, -0.0, 1.0, -0.0])):
        y = torch.empty(n, **F64)
        h.amul(dev(diag), dev(upper), None, dev(x), y)
        ref = O.amul(m, diag, upper, x)
        assert np.array_equal(_bits(y.cpu().numpy()), _bits(ref)), (y, ref)
        if not x.any() and not np.signbit(x).any():
            assert np.signbit(ref[3])  # x = +0: the isolated cell keeps diag * 0 = -0.0
    h.free()


def test_non_lattice_meshes_fall_back():
    for m in (gen.permute(gen.cube(9), seed=2), gen.perturbed(6)):
        h = P.Mesh.from_mesh(m, renumber=True)  # RCM of a cube is not a lattice numbering
        assert h.get_stats()["amul_variant"] in (10, 6, 5)
        h.free()


@pytest.mark.parametrize("name,make", [("cube24", lambda: gen.cube(24)), ("cavity2d-100", lambda: gen.cavity2d(100)),
                                       ("fixed-value-perturbed24", lambda: _fixed_value_cube(24))])
def test_lattice_pcg_parity(name, make):
    """Graph-batched hot loop (> 8192 cells) on the lattice layout vs the oracle (Q11)."""
    m = make()
    g, b = gen.gamma_lognormal(m), gen.rhs(m)
    pv = [None if p.value is None else p.value for p in m.patches]
    has_fixed = any(v is not None for v in pv)
    ref = -1 if has_fixed else 0
    ctl = (1e-8, 0.0, 5000, 0)
    psi_g, pg, _, h = gpu_solve_case(m, g, b, ref, ctl)
    assert h.get_stats()["amul_variant"] == 12
    psi_o, po, _ = O.solve_case(m, g, b, ref, 0.0, O.controls(*ctl))
    assert pg["converged"] and abs(pg["n_iterations"] - po["n_iterations"]) <= 2, (pg, po)
    n = min(pg["n_iterations"], po["n_iterations"])
    psi_g, _, _, _ = gpu_solve_case(m, g, b, ref, (0.0, 0.0, n, n), handle=h)
    psi_o, _, _ = O.solve_case(m, g, b, ref, 0.0, O.controls(0.0, 0.0, n, n))
    err = np.linalg.norm(psi_g - psi_o) / np.linalg.norm(psi_o)
    assert err <= 1e-9, err
    # the ELL rows (variant 10) on the same handle: same iterates up to the dot rounding
    h.set_option(P.spuma.OPT_AMUL_VARIANT, 10)
    psi_e, _, _, _ = gpu_solve_case(m, g, b, ref, (0.0, 0.0, n, n), handle=h)
    assert np.linalg.norm(psi_e - psi_g) / np.linalg.norm(psi_g) <= 1e-9
    h.free()


def test_lattice_pcg_full_size_8M_fixed_iterations():
    """bench.py's workload and launch configuration (200^3, lattice slots): 20 fixed iterations
    against the oracle."""
    m = gen.cube(200)
    b = gen.rhs(m)
    s = O.assemble(m, None, 0, 0.0, b)
    psi_o, _ = O.pcg(m, s, None, O.controls(0.0, 0.0, 20, 20))
    h = P.Mesh.from_mesh(m)
    diag, upper, src = dev(s.diag), dev(s.upper), dev(s.source)
    psi = torch.zeros(m.n_cells, **F64)
    perf = h.pcg_solve(diag, upper, None, src, psi, 0.0, 0.0, 20, 20)
    assert perf["n_iterations"] == 20 and h.get_stats()["amul_variant"] == 12
    err = np.linalg.norm(psi.cpu().numpy() - psi_o) / np.linalg.norm(psi_o)
    assert err <= 1e-9, err
    h.free()

