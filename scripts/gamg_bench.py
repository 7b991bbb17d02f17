#!/usr/bin/env python
"""GAMG vs PCG time to solution on one GPU.

For each case: the hierarchy, V-cycles / PCG iterations to the tolerance, solve time
(CUDA events around spuma_gamg_solve / spuma_pcg_solve, after a warm-up solve that builds
the hierarchy and captures the graphs), and GAMG's bytes per V-cycle against the measured
HBM peak.  Algorithmic bytes per cycle (defaults nPre 0, nPost 2, scale on): per level with
n cells and f faces, each row gather streams 8 B of diag + the level's ownerStart/losortStart
(8 B/cell) and losort/ownerLo/neighbour (12 B/face) + upper (8 B/face, twice) and its
vectors; we count   restrict 8n(b) + 8n_c,   scale 24n + 28f + 8n (ftc 4n),
post-sweep-1 48n + 28f + 4n(ftc), post-sweep-2 40n + 28f, residual (level 0) 40n + 28f
-> reported as 'alg_GB_per_cycle'.  One JSON line per case.
usage: python scripts/gamg_bench.py [n ...]   (default 200: the bench workload, 8M cells)
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2512_22215_b200 as P  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
f64 = dict(dtype=torch.float64, device="cuda")


def cycle_bytes(cells, faces):
    tot = 0
    for l, (n, f) in enumerate(zip(cells, faces)):
        if l == len(cells) - 1:
            break
        nc = cells[l + 1]
        tot += 8 * n + 8 * nc + 4 * n                       # restrict (b, coarse b, lists)
        tot += 24 * n + 28 * f + 12 * n                     # scale
        tot += 48 * n + 28 * f + 4 * n                      # first post-sweep (fused prolongation)
        tot += 40 * n + 28 * f                              # second post-sweep
    tot += 40 * cells[0] + 28 * faces[0]                    # outer residual
    return tot


def run(name, m, gamma, tol, rel_tol=0.0, reps=3, params=None):
    t0 = time.perf_counter()
    h = P.Mesh.from_mesh(m, renumber=False, stream=torch.cuda.current_stream().cuda_stream)
    if os.environ.get("GAMG_TAIL") is not None:  # A/B: single-CTA tail threshold (0 = off)
        h.set_option(P.spuma.OPT_GAMG_TAIL_CELLS, int(os.environ["GAMG_TAIL"]))
        name += f" [tail {os.environ['GAMG_TAIL']}]"
    if os.environ.get("AMUL_VARIANT") is not None:  # A/B: the layout of the level-0 rows (12 lattice, 10 ELL)
        h.set_option(P.spuma.OPT_AMUL_VARIANT, int(os.environ["AMUL_VARIANT"]))
        name += f" [amul variant {os.environ['AMUL_VARIANT']}]"
    if os.environ.get("GAMG_PDL") == "0":  # A/B: plain launches
        h.set_option(P.spuma.OPT_PDL, 0)
        name += " [PDL off]"
    t_create = time.perf_counter() - t0
    N, F = m.n_cells, m.n_faces
    diag, upper = torch.empty(N, **f64), torch.empty(F, **f64)
    b = torch.as_tensor(gen.rhs(m), **f64)
    g = None if gamma is None else torch.as_tensor(gamma, **f64)
    src = b.clone()
    h.assemble_laplacian(g, None, 0, 0.0, diag, upper, src, None)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def solve(kind):
        psi = torch.zeros(N, **f64)
        s = src.clone()
        torch.cuda.synchronize()
        e0.record()
        if kind == "gamg":
            perf = h.gamg_solve(diag, upper, None, s, psi, tol, rel_tol, 300, 0, params=params)
        else:
            perf = h.pcg_solve(diag, upper, None, s, psi, tol, rel_tol, 5000, 0)
        e1.record()
        torch.cuda.synchronize()
        return perf, e0.elapsed_time(e1) / 1e3

    t1 = time.perf_counter()
    solve("gamg")  # builds the hierarchy + captures the cycle
    t_hier = time.perf_counter() - t1
    hier = h.gamg_hierarchy(params, with_ftc=False)
    rg = min((solve("gamg") for _ in range(reps)), key=lambda r: r[1])
    solve("pcg")
    rp = min((solve("pcg") for _ in range(reps)), key=lambda r: r[1])
    cb = cycle_bytes(hier["cells"], hier["faces"])
    out = {"case": name, "cells": N, "faces": F, "tol": tol, "rel_tol": rel_tol,
           "levels": hier["levels"], "level_cells": hier["cells"],
           "gamg_cycles": rg[0]["n_iterations"], "gamg_converged": rg[0]["converged"],
           "gamg_final_residual": rg[0]["final_residual"], "gamg_solve_s": rg[1],
           "gamg_ms_per_cycle": 1e3 * rg[1] / max(rg[0]["n_iterations"], 1),
           "alg_GB_per_cycle": cb / 1e9,
           "gamg_cycle_GBps": cb * rg[0]["n_iterations"] / rg[1] / 1e9,
           "gamg_cycle_frac_of_peak": cb * rg[0]["n_iterations"] / rg[1] / 1e9 / PEAK,
           "pcg_iterations": rp[0]["n_iterations"], "pcg_solve_s": rp[1],
           "gamg_speedup_vs_pcg": rp[1] / rg[1],
           "mesh_create_s": t_create, "first_gamg_solve_s(incl. hierarchy)": t_hier, "peak_GBps": PEAK}
    print(json.dumps(out), flush=True)
    h.free()


if __name__ == "__main__":
    ns = [int(a) for a in sys.argv[1:]] or [200]
    for n in ns:
        m = gen.cube(n)
        run(f"cube {n}^3 gamma=1 tol 1e-6", m, None, 1e-6)
        g = gen.gamma_lognormal(m)
        run(f"cube {n}^3 gamma=lognormal pGAMG (1e-9, relTol 1e-3)", m, g, 1e-9, 1e-3)
        gs2 = P.gamg_params(smoother=P.spuma.SMOOTHER_GS2)
        run(f"cube {n}^3 gamma=1 tol 1e-6, two-stage GS", m, None, 1e-6, params=gs2)
        run(f"cube {n}^3 gamma=lognormal pGAMG, two-stage GS", m, g, 1e-9, 1e-3, params=gs2)
