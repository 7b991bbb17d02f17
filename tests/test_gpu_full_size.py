"""BASELINE config 4 at its full size, through the C-ABI, against the oracle: the synthetic
perturbed (a = 0.15), randomly permuted 400^3 hex mesh (64M cells, 191.5M internal faces),
log-normal gamma, RCM renumbering inside libspuma, on one GPU -- the launch configuration of
`scripts/sweep.py C4`.

Checked: the RCM permutation and renumbered addressing bitwise (O2, Q12); every assembled
coefficient, diagonal and source entry bitwise (Q10) in the caller's numbering; one full Amul
bitwise; 20 fixed PCG iterations within 1e-9 relative L2 (Q11).

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
    rcm = O.rcm(mp.n_cells, mp.owner, mp.neighbour)
    assert np.array_equal(a["perm"], rcm)
    o, nb, fm, _ = O.renumber_faces(rcm, mp.owner, mp.neighbour)
    assert np.array_equal(a["owner"], o) and np.array_equal(a["neighbour"], nb) and np.array_equal(a["face_map"], fm)
    del o, nb, fm, a, rcm
    print(f"addressing checked {time.perf_counter() - t:.1f} s", flush=True)
    # A3-A5 on the GPU (caller numbering in and out)
    diag, upper = torch.empty(mp.n_cells, **F64), torch.empty(mp.n_faces, **F64)
    src = torch.as_tensor(bp, **F64)
    h.assemble_laplacian(torch.as_tensor(gp, **F64), None, ref, 0.0, diag, upper, src, None)
    torch.cuda.synchronize()
    t = time.perf_counter()
    s = O.assemble(mp, gp, ref, 0.0, source=bp)
    print(f"oracle assembly {time.perf_counter() - t:.1f} s", flush=True)
    assert np.array_equal(_bits(upper.cpu().numpy()), _bits(s.upper))
    assert np.array_equal(_bits(diag.cpu().numpy()), _bits(s.diag))
    assert np.array_equal(_bits(src.cpu().numpy()), _bits(s.source))
    # A7: one Amul of the whole mesh
    x = np.sin(np.arange(mp.n_cells) * 1e-3)
    y = torch.empty(mp.n_cells, **F64)
    h.amul(diag, upper, None, torch.as_tensor(x, **F64), y)
    t = time.perf_counter()
    yo = O.amul(mp, s.diag, s.upper, x)
    print(f"oracle Amul {time.perf_counter() - t:.1f} s", flush=True)
    assert np.array_equal(_bits(y.cpu().numpy()), _bits(yo))
    del y, yo
    # A6-A12: 20 fixed iterations
    psi = torch.zeros(mp.n_cells, **F64)
    perf = h.pcg_solve(diag, upper, None, src, psi, 0.0, 0.0, 20, 20)
    t = time.perf_counter()
    psi_o, perf_o = O.pcg(mp, s, None, O.controls(0.0, 0.0, 20, 20))
    print(f"oracle 20 iterations {time.perf_counter() - t:.1f} s", flush=True)
    assert perf["n_iterations"] == perf_o["n_iterations"] == 20
    assert perf["initial_residual"] == pytest.approx(perf_o["initial_residual"], rel=1e-12)
    err = np.linalg.norm(psi.cpu().numpy() - psi_o) / np.linalg.norm(psi_o)
    print(f"20 iterations: rel L2 {err:.3e}; final residual gpu {perf['final_residual']:.6e} "
          f"oracle {perf_o['final_residual']:.6e}", flush=True)
    assert err <= 1e-9, err
    h.free()
