#!/usr/bin/env python
"""How the in-graph CUDA-event timing of k_amul_dot (bench.py's roofline) depends on PDL:
200^3 cube, gamma = 1, tol 1e-6, timing on; PDL on / off; per-launch Amul us and solve time."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2512_22215_b200 as P  # noqa: E402

m = gen.cube(200)
f64 = dict(dtype=torch.float64, device="cuda")
h = P.Mesh.from_mesh(m, stream=torch.cuda.current_stream().cuda_stream)
diag, upper, src = torch.empty(m.n_cells, **f64), torch.empty(m.n_faces, **f64), torch.as_tensor(gen.rhs(m), **f64)
h.assemble_laplacian(None, None, 0, 0.0, diag, upper, src, None)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rnd in range(2):
    for pdl in (1, 0):
        for timing in (False, True):
            h.set_option(P.spuma.OPT_PDL, pdl)
            h.set_timing(timing)
            h.reset_stats()
            psi = torch.zeros(m.n_cells, **f64)
            e0.record()
            perf = h.pcg_solve(diag, upper, None, src.clone(), psi, 1e-6, 0.0, 5000, 0)
            e1.record()
            torch.cuda.synchronize()
            st = h.get_stats()
            amul = st["phase_ms"][1] / max(st["phase_count"][1], 1) * 1e3 if timing else None
            print(json.dumps({"pdl": pdl, "timing": timing, "solve_ms": e0.elapsed_time(e1), "its": perf["n_iterations"],
                              "amul_us": amul, "direction_us": st["phase_ms"][0] / max(st["phase_count"][0], 1) * 1e3 if timing else None,
                              "update_us": st["phase_ms"][2] / max(st["phase_count"][2], 1) * 1e3 if timing else None}))
h.set_option(P.spuma.OPT_PDL, 1)
