#!/usr/bin/env python
"""Same-box A/B of the GAMG small-level tail: one CTA (SPUMA_OPT_GAMG_TAIL_CLUSTER = 1) vs a
thread-block cluster of 4/8/16 CTAs, each at several tail thresholds (SPUMA_OPT_GAMG_TAIL_CELLS):
ms per V-cycle (40 fixed cycles, best of 3) at 200^3 and 100^3, and psi's relative difference to
the default configuration after 40 cycles."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import torch, gen, paper_2512_22215_b200 as P
f64 = dict(dtype=torch.float64, device="cuda")
combos = [(1, 512), (1, 1024), (8, 512), (8, 2048), (8, 4096), (8, 8192), (16, 4096), (16, 8192), (16, 16384),
          (4, 2048), (4, 4096)]
for n in (200, 100):
    m = gen.cube(n)
    h = P.Mesh.from_mesh(m, stream=torch.cuda.current_stream().cuda_stream)
    diag, upper = torch.empty(m.n_cells, **f64), torch.empty(m.n_faces, **f64)
    src = torch.as_tensor(gen.rhs(m), **f64)
    h.assemble_laplacian(None, None, 0, 0.0, diag, upper, src, None)
    ref = None
    for rnd in range(2):
        for cl, thr in combos:
            h.set_option(P.spuma.OPT_GAMG_TAIL_CLUSTER, cl)
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
            if ref is None:
                ref = psi.clone()
            rel = float(torch.linalg.norm(psi - ref) / torch.linalg.norm(ref))
            print(json.dumps({"n": n, "round": rnd, "cluster": cl, "tail_cells": thr, "ms_per_cycle": round(best, 4),
                              "rel_diff_vs_default": rel}), flush=True)
    h.free()
