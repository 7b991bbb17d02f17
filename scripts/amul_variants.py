#!/usr/bin/env python
"""A/B the A7 Amul variants on the bench workload (200^3 cube): per-variant solve time and
the live per-launch duration of k_amul_dot (libspuma's CUDA events), parity vs variant 0."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import gen
import paper_2512_22215_b200 as P

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
perm = "--permute" in sys.argv
m = gen.cube(n)
b = gen.rhs(m)
if perm:
    pm = gen.random_perm(m.n_cells)
    m = gen.permute(m, pm)
    b = gen.permute_cell_field(b, pm)
N, F = m.n_cells, m.n_faces
f64 = dict(dtype=torch.float64, device="cuda")
h = P.Mesh.from_mesh(m, stream=torch.cuda.current_stream().cuda_stream, renumber="--renumber" in sys.argv)
diag, upper, src = torch.empty(N, **f64), torch.empty(F, **f64), torch.as_tensor(b, **f64)
h.assemble_laplacian(None, None, 0, 0.0, diag, upper, src, None)
ref = None
out = {}
for v in [int(x) for x in os.environ.get("VARIANTS", "0,5,6,7,8,9").split(",")]:
    h.set_option(P.spuma.OPT_AMUL_VARIANT, v)
    try:
        h.set_option(P.spuma.OPT_PDL, int(os.environ.get("PDL", "1")))
    except P.SpumaError:  # older library without the option (A/B runs)
        pass
    psi = torch.zeros(N, **f64)
    h.pcg_solve(diag, upper, None, src, psi, 1e-6, 0.0, 5000, 0)  # warm-up / graph capture
    h.reset_stats()
    h.set_timing(True)
    psi.zero_()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    perf = h.pcg_solve(diag, upper, None, src, psi, 1e-6, 0.0, 5000, 0)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    st = h.get_stats()
    h.set_timing(False)
    psi.zero_()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    perf2 = h.pcg_solve(diag, upper, None, src, psi, 1e-6, 0.0, 5000, 0)
    torch.cuda.synchronize()
    t_untimed = time.perf_counter() - t1
    r = psi.cpu().numpy()
    if ref is None:
        ref = r
    ph = [st["phase_ms"][i] / max(st["phase_count"][i], 1) for i in range(3)]
    out[v] = {"solve_s": t, "solve_untimed_s": t_untimed, "iters": perf["n_iterations"],
              "amul_us": 1e3 * ph[1], "dir_us": 1e3 * ph[0], "upd_us": 1e3 * ph[2],
              "amul_alg_GBps": (24 * N + 16 * F) / (ph[1] / 1e3) / 1e9,
              "cells_iter_per_s": N * perf2["n_iterations"] / t_untimed,
              "bitwise_equal_v0": bool(np.array_equal(r, ref))}
    out[v]["pdl"] = int(os.environ.get("PDL", "1"))
    print(v, json.dumps(out[v]), flush=True)
