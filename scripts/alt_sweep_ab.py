#!/usr/bin/env python
"""Same-box A/B of SPUMA_OPT_ALT_SWEEP (alternating sweep directions of the hot-loop kernels)
and SPUMA_OPT_ELL_STENCIL (chunk-stencil compressed ELL rows)
on the bench workload (cube n^3, gamma = 1, tol 1e-6) and a permuted/RCM case: solve time,
cells*iter/s, iteration counts, and the difference of psi between the two modes (the dots are
summed in another per-thread order, so iterates agree to rounding, not bitwise)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2512_22215_b200 as P  # noqa: E402

f64 = dict(dtype=torch.float64, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for n in [int(a) for a in sys.argv[1:]] or [200, 126, 252]:
    m = gen.cube(n)
    h = P.Mesh.from_mesh(m, stream=torch.cuda.current_stream().cuda_stream)
    diag, upper = torch.empty(m.n_cells, **f64), torch.empty(m.n_faces, **f64)
    src = torch.as_tensor(gen.rhs(m), **f64)
    h.assemble_laplacian(None, None, 0, 0.0, diag, upper, src, None)
    out = {}
    for rnd in range(2):
        for mode in ((0, 0), (1, 0), (0, 1), (1, 1)):
            h.set_option(P.spuma.OPT_ALT_SWEEP, mode[0])
            h.set_option(P.spuma.OPT_ELL_STENCIL, mode[1])
            best = None
            for _ in range(3):
                psi = torch.zeros(m.n_cells, **f64)
                torch.cuda.synchronize()
                e0.record()
                perf = h.pcg_solve(diag, upper, None, src.clone(), psi, 1e-6, 0.0, 5000, 0)
                e1.record()
                torch.cuda.synchronize()
                t = e0.elapsed_time(e1) / 1e3
                best = t if best is None else min(best, t)
            out[mode] = psi.clone()
            print(json.dumps({"n": n, "round": rnd, "alt_sweep": mode[0], "ell_stencil": mode[1], "iterations": perf["n_iterations"],
                              "solve_s": best, "cells_iter_per_s": m.n_cells * perf["n_iterations"] / best}),
                  flush=True)
    d = float((out[(0, 0)] - out[(1, 0)]).norm() / out[(0, 0)].norm())
    print(json.dumps({"n": n, "rel_l2_psi_alt0_vs_alt1": d,
                      "stencil_bitwise_neutral": bool(torch.equal(out[(0, 0)], out[(0, 1)]))}), flush=True)
    h.free()
