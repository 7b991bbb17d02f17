#!/usr/bin/env python
"""The persistent loop's CTA count on small meshes (SPUMA_OPT_LOOP_GRID): us per iteration (best of 5
solves to 1e-6, CUDA events) for cubes of 4k..1M cells at 8..148 CTAs, single-CTA solve beside."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import torch, gen, paper_2512_22215_b200 as P
f64 = dict(dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()
for n in (16, 20, 24, 32, 40, 50, 64, 100):
    m = gen.cube(n)
    h = P.Mesh.from_mesh(m, stream=st.cuda_stream)
    diag, upper = torch.empty(m.n_cells, **f64), torch.empty(m.n_faces, **f64)
    src = torch.as_tensor(gen.rhs(m), **f64)
    h.assemble_laplacian(None, None, 0, 0.0, diag, upper, src, None)
    h.set_option(P.spuma.OPT_SMALL_SOLVE_MAX_CELLS, 0)
    for g in (0, 32, 148):  # 0 = the library's automatic choice
        h.set_option(P.spuma.OPT_LOOP_GRID, g)
        psi = torch.zeros(m.n_cells, **f64)
        h.pcg_solve(diag, upper, None, src, psi, 1e-6, 0.0, 5000, 0)
        best, it = None, 0
        for _ in range(5):
            psi.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); e0.record(st)
            perf = h.pcg_solve(diag, upper, None, src, psi, 1e-6, 0.0, 5000, 0)
            e1.record(st); torch.cuda.synchronize()
            t = e0.elapsed_time(e1)
            best = t if best is None else min(best, t)
            it = perf["n_iterations"]
        s = h.get_stats()
        print(json.dumps({"cells": m.n_cells, "ctas": s["loop_grid"], "loop_mode": s["loop_mode"], "iterations": it,
                          "us_per_iter": round(best * 1e3 / max(it, 1), 2)}), flush=True)
    h.free()
