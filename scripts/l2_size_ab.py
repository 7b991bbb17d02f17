#!/usr/bin/env python
"""L2 window A/B on large meshes (the persisting set-aside is <= 83 MB; a window over a vector of
8N bytes > that is only partly persisting): one mesh, one handle, several (persistent, l2_persist,
loop_l2) combinations, best of 2 solves each.  usage: python scripts/l2_size_ab.py C4|cube:n"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2512_22215_b200 as P  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "cube:252"
combos = [tuple(int(x) for x in c.split(",")) for c in (sys.argv[2:] or ["0,0,0", "0,2,0", "3,2,0", "3,2,4"])]
f64 = dict(dtype=torch.float64, device="cuda")
t0 = time.perf_counter()
if which == "C4" or which.startswith("perm:"):  # perturbed + randomly permuted, RCM-renumbered (ELL rows)
    m = gen.perturbed(400 if which == "C4" else int(which.split(":")[1]), 0.15)
    g, b = gen.gamma_lognormal(m), gen.rhs(m)
    perm = gen.random_perm(m.n_cells)
    m = gen.permute(m, perm)
    g, b = gen.permute_cell_field(g, perm), gen.permute_cell_field(b, perm)
    ref, ren = int(perm[0]), True
else:
    m = gen.cube(int(which.split(":")[1]))
    g, b, ref, ren = None, gen.rhs(m), 0, False
st = torch.cuda.current_stream()
h = P.Mesh.from_mesh(m, renumber=ren, stream=st.cuda_stream)
N, F = m.n_cells, m.n_faces
diag, upper = torch.empty(N, **f64), torch.empty(F, **f64)
src = torch.as_tensor(b, **f64)
h.assemble_laplacian(None if g is None else torch.as_tensor(g, **f64), None, ref, 0.0, diag, upper, src, None)
print(json.dumps({"case": which, "cells": N, "setup_s": time.perf_counter() - t0}), flush=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for pers, l2, ll in combos:
    h.set_option(P.spuma.OPT_PERSISTENT, pers)
    h.set_option(P.spuma.OPT_L2_PERSIST, l2)
    h.set_option(P.spuma.OPT_LOOP_L2, ll)
    best, it = None, 0
    for _ in range(2):
        psi = torch.zeros(N, **f64)
        torch.cuda.synchronize()
        e0.record(st)
        perf = h.pcg_solve(diag, upper, None, src, psi, 1e-6, 0.0, 5000, 0)
        e1.record(st)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3
        best = t if best is None else min(best, t)
        it = perf["n_iterations"]
    s = h.get_stats()
    print(json.dumps({"case": which, "persistent": pers, "l2_persist": l2, "loop_l2": ll, "ran_loop": s["loop_mode"],
                      "amul_variant": s["amul_variant"], "iterations": it, "us_per_iter": best / it * 1e6,
                      "cells_iter_per_s": N * it / best}), flush=True)
h.free()
