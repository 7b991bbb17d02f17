#!/usr/bin/env python
"""SPUMA_OPT_PERSISTENT A/B on one GPU: the bench workload (cube n^3, gamma = 1, tol 1e-6) solved
with the captured graph batches (mode 0) and the persistent loop (1: rA in HBM, 2: + shared
memory, 3: + tensor memory), optionally under several L2 window targets.  Prints one JSON line
per (mode, l2): iterations, best-of-3 solve time (CUDA events), us per iteration, and the
relative difference of psi to mode 0 (same handle, same inputs)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2512_22215_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
modes = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "0,1,2,3").split(",")]
l2s = [int(v) for v in (sys.argv[3] if len(sys.argv) > 3 else "2").split(",")]
loop_l2s = [int(v) for v in (sys.argv[4] if len(sys.argv) > 4 else "0").split(",")]
m = gen.cube(n)
f64 = dict(dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()
h = P.Mesh.from_mesh(m, stream=st.cuda_stream)
for kv in filter(None, os.environ.get("SPUMA_AB_OPTS", "").split(",")):  # extra option=value pairs (A/B)
    k, v = kv.split("=")
    h.set_option(int(k), int(v))
diag, upper, src = torch.empty(m.n_cells, **f64), torch.empty(m.n_faces, **f64), torch.as_tensor(gen.rhs(m), **f64)
h.assemble_laplacian(None, None, 0, 0.0, diag, upper, src, None)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ref = None
for l2, mode, ll in [(l2, mode, ll) for l2 in l2s for mode in modes for ll in (loop_l2s if mode else [0])]:
        h.set_option(P.spuma.OPT_L2_PERSIST, l2)
        h.set_option(P.spuma.OPT_LOOP_L2, ll)
        h.set_option(P.spuma.OPT_PERSISTENT, mode)
        psi = torch.zeros(m.n_cells, **f64)
        h.pcg_solve(diag, upper, None, src, psi, 1e-6, 0.0, 5000, 0)  # warm
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
        s = h.get_stats()
        prof = None
        if s["loop_mode"]:  # one more solve with the per-phase work / barrier-wait profile
            h.reset_stats()
            h.set_timing(True)
            h.set_option(P.spuma.OPT_LOOP_PROFILE, 1)
            psi.zero_()
            h.pcg_solve(diag, upper, None, src, psi, 1e-6, 0.0, 5000, 0)
            q = h.get_stats()
            h.set_timing(False)
            h.set_option(P.spuma.OPT_LOOP_PROFILE, 0)
            itq = max(q["iterations"], 1)
            prof = {"loop_us_per_iter": q["loop_ms"] * 1e3 / itq,
                    "work_us": [round(v * 1e3 / itq, 2) for v in q["loop_work_ms"]],
                    "wait_us": [round(v * 1e3 / itq, 2) for v in q["loop_wait_ms"]],
                    "work_max_us": [round(v * 1e3 / itq, 2) for v in q["loop_work_max_ms"]]}
        if ref is None:
            ref = psi.clone()
        rel = float(torch.linalg.norm(psi - ref) / torch.linalg.norm(ref))
        it = perf["n_iterations"]
        print(json.dumps({"n": n, "mode": mode, "l2": l2, "loop_l2": ll, "ran_mode": s["loop_mode"], "grid": s["loop_grid"],
                          "tmem_pairs": s["loop_tmem_pairs"], "smem_pairs": s["loop_smem_pairs"],
                          "iterations": it, "final_residual": perf["final_residual"], "solve_s": best,
                          "us_per_iter": best / it * 1e6, "cells_iter_per_s": m.n_cells * it / best,
                          "rel_diff_vs_first": rel, "prof": prof}), flush=True)
h.free()
