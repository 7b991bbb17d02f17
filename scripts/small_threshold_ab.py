#!/usr/bin/env python
"""Single-CTA small solve vs the persistent loop on small meshes (SPUMA_OPT_SMALL_SOLVE_MAX_CELLS
cut-over): time to solution (assembly excluded, best of 5, CUDA events) for cubes and 2-D cavities
of 400..32k cells, each through both paths."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import torch, gen, paper_2512_22215_b200 as P
f64 = dict(dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()
cases = [("cavity20", gen.cavity2d(20)), ("cavity45", gen.cavity2d(45)), ("cavity64", gen.cavity2d(64)),
         ("cube10", gen.cube(10)), ("cube13", gen.cube(13)), ("cube16", gen.cube(16)), ("cube20", gen.cube(20)),
         ("cube24", gen.cube(24)), ("cube32", gen.cube(32))]
for name, m in cases:
    h = P.Mesh.from_mesh(m, stream=st.cuda_stream)
    diag, upper = torch.empty(m.n_cells, **f64), torch.empty(m.n_faces, **f64)
    src = torch.as_tensor(gen.rhs(m), **f64)
    h.assemble_laplacian(None, None, 0, 0.0, diag, upper, src, None)
    for thr, label in ((1 << 30, "single_cta"), (0, "loop")):
        h.set_option(P.spuma.OPT_SMALL_SOLVE_MAX_CELLS, thr)
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
        print(json.dumps({"case": name, "cells": m.n_cells, "path": label, "iterations": it, "solve_ms": round(best, 4),
                          "us_per_iter": round(best * 1e3 / max(it, 1), 2), "loop_mode": h.get_stats()["loop_mode"]}), flush=True)
    h.free()
