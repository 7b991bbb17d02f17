#!/usr/bin/env python
"""Same-box A/B of SPUMA_OPT_FUSE_DIRECTION (0 separate k_direction, 1 fused + rD read,
2 fused + 1/diag in place) on the bench workload (cube n^3, gamma = 1, tol 1e-6): solve time,
cells*iter/s, and bitwise identity of psi / iteration count across the modes."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2512_22215_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
m = gen.cube(n)
f64 = dict(dtype=torch.float64, device="cuda")
h = P.Mesh.from_mesh(m, stream=torch.cuda.current_stream().cuda_stream)
diag, upper, src = torch.empty(m.n_cells, **f64), torch.empty(m.n_faces, **f64), torch.as_tensor(gen.rhs(m), **f64)
h.assemble_laplacian(None, None, 0, 0.0, diag, upper, src, None)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ref = None
for rnd in range(2):
    for mode in (0, 1, 2):
        h.set_option(P.spuma.OPT_FUSE_DIRECTION, mode)
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
        if ref is None:
            ref = (psi.clone(), perf["n_iterations"])
        same = bool(torch.equal(psi, ref[0])) and perf["n_iterations"] == ref[1]
        print(json.dumps({"round": rnd, "fuse_direction": mode, "iterations": perf["n_iterations"], "solve_s": best,
                          "cells_iter_per_s": m.n_cells * perf["n_iterations"] / best, "bitwise_same_as_mode0": same}),
              flush=True)
