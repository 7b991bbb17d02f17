"""BASELINE config 4 at its full size, through the C-ABI, against the oracle: the synthetic
perturbed (a = 0.15), randomly permuted 400^3 hex mesh (64M cells, 191.5M internal faces),
log-normal gamma, RCM renumbering inside libspuma, on one GPU -- the launch configuration of
`scripts/sweep.py C4`.

Checked: the RCM permutation and renumbered addressing bitwise (O2, Q12); every assembled
coefficient, diagonal and source entry within 1e-13 relative of the oracle in the caller's
numbering (the north_star bar) and bitwise equal to the oracle run on the renumbered mesh (the
library computes in its internal numbering, Q10/Q12 -- faces whose owner and neighbour swap under
RCM interpolate gamma from the other side, a different rounding); one full Amul bitwise; 20 fixed
PCG iterations within 1e-9 relative L2 (Q11).

Generation (~1 min), the library's host setup (~1 min) and the oracle's full-size assembly, Amul
and 20 iterations (single-threaded, several minutes) put this outside the round-end suite: it
runs when SPUMA_FULL_SIZE=1 (log committed under profiles/)."""
import os
import time

import numpy as np
import pytest

import gen
import oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(os.environ.get("SPUMA_FULL_SIZE") != "1",
                                                  reason="full-size C4 parity: set SPUMA_FULL_SIZE=1")]
torch = pytest.importorskip("torch")
import paper_2512_22215_b200 as P  # noqa: E402

F64 = dict(dtype=torch.float64, device="cuda")


def _bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def test_c4_full_size_parity():
    t = time.perf_counter()
    m = gen.perturbed(400, 0.15)
    g, b = gen.gamma_lognormal(m), gen.rhs(m)
    perm = gen.random_perm(m.n_cells)
    mp = gen.permute(m, perm)
    del m
    gp, bp = gen.permute_cell_field(g, perm), gen.permute_cell_field(b, perm)
    ref = int(perm[0])
    print(f"generate {time.perf_counter() - t:.1f} s; cells {mp.n_cells}, faces {mp.n_faces}", flush=True)
    t = time.perf_counter()
    h = P.Mesh.from_mesh(mp, renumber=True)
    print(f"mesh_create {time.perf_counter() - t:.1f} s; amul variant {h.get_stats()['amul_variant']}", flush=True)
    # A1-A2: the library's RCM and renumbered addressing = the oracle's
    t = time.perf_counter()
    a = h.mesh_get_addressing()
    perm = O.rcm(mp.n_cells, mp.owner, mp.neighbour)
    assert np.array_equal(a["perm"], perm)
    o, nb, fm, _ = O.renumber_faces(perm, mp.owner, mp.neighbour)
    assert np.array_equal(a["owner"], o) and np.array_equal(a["neighbour"], nb) and np.array_equal(a["face_map"], fm)
    del o, nb, a
    print(f"addressing checked {time.perf_counter() - t:.1f} s", flush=True)
    # A3-A5 on the GPU (caller numbering in and out)
    diag, upper = torch.empty(mp.n_cells, **F64), torch.empty(mp.n_faces, **F64)
    src = torch.as_tensor(bp, **F64)
    h.assemble_laplacian(torch.as_tensor(gp, **F64), None, ref, 0.0, diag, upper, src, None)
    torch.cuda.synchronize()
    gd, gu, gs = diag.cpu().numpy(), upper.cpu().numpy(), src.cpu().numpy()
    # the north_star bar against the oracle in the caller's numbering: 1e-13 relative
    t = time.perf_counter()
    s0 = O.assemble(mp, gp, ref, 0.0, source=bp)
    print(f"oracle assembly (caller numbering) {time.perf_counter() - t:.1f} s", flush=True)
    for g_, o_ in ((gu, s0.upper), (gd, s0.diag), (gs, s0.source)):
        assert np.max(np.abs(g_ - o_)) <= 1e-13 * np.max(np.abs(o_))
    nd = int(np.count_nonzero(_bits(gu) != _bits(s0.upper)))
    print(f"upper entries not bitwise the caller-orientation oracle's: {nd} of {mp.n_faces} "
          "(faces whose owner/neighbour swap under RCM interpolate gamma from the other side)", flush=True)
    del s0
    # bitwise against the oracle on the renumbered mesh (the library's internal numbering, Q10/Q12)
    t = time.perf_counter()
    rm = O.renumber_mesh(mp, perm)
    gr, br = gen.permute_cell_field(gp, perm), gen.permute_cell_field(bp, perm)
    s = O.assemble(rm, gr, int(perm[ref]), 0.0, source=br)
    print(f"oracle assembly (renumbered) {time.perf_counter() - t:.1f} s", flush=True)
    assert np.array_equal(_bits(gd), _bits(s.diag[perm]))
    assert np.array_equal(_bits(gs), _bits(s.source[perm]))
    assert np.array_equal(_bits(gu[fm]), _bits(s.upper))
    del gd, gu, gs
    # A7: one Amul of the whole mesh
    x = np.sin(np.arange(mp.n_cells) * 1e-3)
    y = torch.empty(mp.n_cells, **F64)
    h.amul(diag, upper, None, torch.as_tensor(x, **F64), y)
    t = time.perf_counter()
    yo = O.amul(rm, s.diag, s.upper, gen.permute_cell_field(x, perm))[perm]
    print(f"oracle Amul {time.perf_counter() - t:.1f} s", flush=True)
    assert np.array_equal(_bits(y.cpu().numpy()), _bits(yo))
    del y, yo
    # A6-A12: 20 fixed iterations
    psi = torch.zeros(mp.n_cells, **F64)
    perf = h.pcg_solve(diag, upper, None, src, psi, 0.0, 0.0, 20, 20)
    t = time.perf_counter()
    psi_o, perf_o = O.pcg(rm, s, None, O.controls(0.0, 0.0, 20, 20))
    print(f"oracle 20 iterations {time.perf_counter() - t:.1f} s", flush=True)
    assert perf["n_iterations"] == perf_o["n_iterations"] == 20
    assert perf["initial_residual"] == pytest.approx(perf_o["initial_residual"], rel=1e-12)
    psi_o = psi_o[perm]
    err = np.linalg.norm(psi.cpu().numpy() - psi_o) / np.linalg.norm(psi_o)
    print(f"20 iterations: rel L2 {err:.3e}; final residual gpu {perf['final_residual']:.6e} "
          f"oracle {perf_o['final_residual']:.6e}", flush=True)
    assert err <= 1e-9, err
    h.free()
