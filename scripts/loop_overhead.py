#!/usr/bin/env python
"""Where the PCG iteration's time goes beyond its kernels: solve the bench workload (cube n^3,
gamma = 1, tol 1e-6) with libspuma's kernel timing off (whole solve, CUDA events) and on
(per-phase averages), for several graph batch sizes, and print the per-iteration time, the sum
of the phase kernels and the difference (launch / boundary / finalisation overhead)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2512_22215_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
opts = [tuple(int(v) for v in o.split("=")) for o in sys.argv[2:]]  # option=value pairs
m = gen.cube(n)
f64 = dict(dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()
h = P.Mesh.from_mesh(m, stream=st.cuda_stream)
for o, v in opts:
    h.set_option(o, v)
diag, upper, src = torch.empty(m.n_cells, **f64), torch.empty(m.n_faces, **f64), torch.as_tensor(gen.rhs(m), **f64)
h.assemble_laplacian(None, None, 0, 0.0, diag, upper, src, None)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for batch in (16, 32, 64):
    h.set_batch(batch)
    psi = torch.zeros(m.n_cells, **f64)
    h.pcg_solve(diag, upper, None, src, psi, 1e-6, 0.0, 5000, 0)  # warm (graph capture)
    best = None
    for _ in range(3):
        psi.zero_()
        torch.cuda.synchronize()
        e0.record(st)
        perf = h.pcg_solve(diag, upper, None, src, psi, 1e-6, 0.0, 5000, 0)
        e1.record(st)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3
        best = t if best is None else min(best, t)
    it = perf["n_iterations"]
    h.reset_stats()
    h.set_timing(True)
    psi.zero_()
    h.pcg_solve(diag, upper, None, src, psi, 1e-6, 0.0, 5000, 0)
    torch.cuda.synchronize()
    s = h.get_stats()
    h.set_timing(False)
    ph = [s["phase_ms"][i] / s["phase_count"][i] * 1e3 if s["phase_count"][i] else None for i in range(3)]
    per_it = best / it * 1e6
    ksum = sum(p for p in ph if p)
    print(json.dumps({"n": n, "opts": opts, "batch": batch, "iterations": it, "solve_s": best,
                      "cells_iter_per_s": m.n_cells * it / best, "us_per_iter": per_it,
                      "phase_us": {"direction": ph[0], "amul_dot": ph[1], "update": ph[2]},
                      "kernel_sum_us": ksum, "overhead_us": per_it - ksum}), flush=True)
h.free()
