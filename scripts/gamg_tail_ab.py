#!/usr/bin/env python
"""Same-box A/B of SPUMA_OPT_GAMG_TAIL_CELLS (levels at or below the threshold in one single-CTA
kernel): ms per V-cycle (40 fixed cycles) at 200^3 and 100^3."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import torch, gen, paper_2512_22215_b200 as P
f64 = dict(dtype=torch.float64, device="cuda")
for n in (200, 100):
    m = gen.cube(n)
    h = P.Mesh.from_mesh(m, stream=torch.cuda.current_stream().cuda_stream)
    diag, upper = torch.empty(m.n_cells, **f64), torch.empty(m.n_faces, **f64)
    src = torch.as_tensor(gen.rhs(m), **f64)
    h.assemble_laplacian(None, None, 0, 0.0, diag, upper, src, None)
    for rnd in range(2):
        for thr in (256, 512, 1024, 2048, 4096):
            h.set_option(P.spuma.OPT_GAMG_TAIL_CELLS, thr)
            psi = torch.zeros(m.n_cells, **f64)
            h.gamg_solve(diag, upper, None, src.clone(), psi, 0.0, 0.0, 20, 20)
            best = None
            for _ in range(3):
                psi.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize(); e0.record()
                h.gamg_solve(diag, upper, None, src.clone(), psi, 0.0, 0.0, 40, 40)
                e1.record(); torch.cuda.synchronize()
                t = e0.elapsed_time(e1) / 40
                best = t if best is None else min(best, t)
            print(json.dumps({"n": n, "round": rnd, "tail_cells": thr, "ms_per_cycle": round(best, 4)}), flush=True)
