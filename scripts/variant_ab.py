#!/usr/bin/env python
"""Same-box A/B of Amul variants inside the PCG loop (cube n^3, gamma = 1, tol 1e-6):
solve time and cells*iter/s per variant, and bitwise identity of psi across variants that
share the reduction shape.  usage: variant_ab.py n [variants...]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2512_22215_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
variants = [int(v) for v in sys.argv[2:]] or [8, 10]
f64 = dict(dtype=torch.float64, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
m = gen.cube(n)
h = P.Mesh.from_mesh(m, stream=torch.cuda.current_stream().cuda_stream)
diag, upper = torch.empty(m.n_cells, **f64), torch.empty(m.n_faces, **f64)
src = torch.as_tensor(gen.rhs(m), **f64)
h.assemble_laplacian(None, None, 0, 0.0, diag, upper, src, None)
out = {}
for rnd in range(3):
    for v in variants:
        h.set_option(P.spuma.OPT_AMUL_VARIANT, v)
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
        out[v] = psi.clone()
        print(json.dumps({"n": n, "round": rnd, "variant": v, "iterations": perf["n_iterations"], "solve_s": best,
                          "cells_iter_per_s": m.n_cells * perf["n_iterations"] / best}), flush=True)
v0 = variants[0]
print(json.dumps({"n": n, "bitwise_same_as_first": {v: bool(torch.equal(out[v], out[v0])) for v in variants}}))
