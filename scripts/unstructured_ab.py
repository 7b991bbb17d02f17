#!/usr/bin/env python
"""Same-box A/B of the general-mesh Amul layouts on randomly permuted, perturbed hex meshes
renumbered by RCM inside libspuma: solve time (CUDA events), cells*iter/s, Amul phase time,
equal iteration counts across the variants.  (Round 2 used it for variant 10 vs a 16-bit-index
ELL variant, profiles/r02d_ell16_ab.jsonl.)
usage: python scripts/unstructured_ab.py [--variants 10,6] n [n ...]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2512_22215_b200 as P  # noqa: E402

f64 = dict(dtype=torch.float64, device="cuda")
args = sys.argv[1:]
variants = (10, 6)
if args and args[0].startswith("--variants"):
    variants = tuple(int(v) for v in args[0].split("=")[1].split(","))
    args = args[1:]
for n in [int(a) for a in args] or [100]:
    m = gen.permute(gen.perturbed(n, 0.15), seed=2)
    g, b = gen.gamma_lognormal(m), gen.rhs(m)
    st = torch.cuda.current_stream()
    h = P.Mesh.from_mesh(m, renumber=True, stream=st.cuda_stream)
    diag, upper = torch.empty(m.n_cells, **f64), torch.empty(m.n_faces, **f64)
    src = torch.as_tensor(b, **f64)
    h.assemble_laplacian(torch.as_tensor(g, **f64), None, 0, 0.0, diag, upper, src, None)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ref = None
    for rnd in range(2):
        for v in variants:
            h.set_option(P.spuma.OPT_AMUL_VARIANT, v)
            psi = torch.zeros(m.n_cells, **f64)
            h.pcg_solve(diag, upper, None, src, psi, 1e-6, 0.0, 5000, 0)
            best = None
            for _ in range(2):
                psi.zero_()
                torch.cuda.synchronize()
                e0.record(st)
                perf = h.pcg_solve(diag, upper, None, src, psi, 1e-6, 0.0, 5000, 0)
                e1.record(st)
                torch.cuda.synchronize()
                t = e0.elapsed_time(e1) / 1e3
                best = t if best is None else min(best, t)
            h.reset_stats()
            h.set_timing(True)
            psi2 = torch.zeros(m.n_cells, **f64)
            h.pcg_solve(diag, upper, None, src, psi2, 1e-6, 0.0, 5000, 0)
            s = h.get_stats()
            h.set_timing(False)
            if ref is None:
                ref = (psi.clone(), perf["n_iterations"])
            print(json.dumps({"n": n, "cells": m.n_cells, "round": rnd, "variant": s["amul_variant"],
                              "iterations": perf["n_iterations"], "solve_s": best,
                              "cells_iter_per_s": m.n_cells * perf["n_iterations"] / best,
                              "amul_us": 1e3 * s["phase_ms"][1] / max(s["phase_count"][1], 1),
                              "same_iterations_as_first": perf["n_iterations"] == ref[1]}), flush=True)
    h.free()
