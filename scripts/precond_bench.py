#!/usr/bin/env python
"""Time to solution of the preconditioned solvers on one GPU.

Symmetric: the pressure Laplacian (gamma log-normal, pRefCell 0) solved to 1e-6 by PCG with the
diagonal (the fused hot path spuma_pcg_solve, and spuma_pcg_solve_pc), DIC and aDILU(2)
preconditioners.  Asymmetric: the Laplacian's coefficients skewed like a convection-diffusion
operator (upper = u(1+e), lower = u(1-e), e ~ U(-0.4, 0.4), 5 % diagonal dominance -- the
recipe of tests/cases.py, built here with torch on the device), solved by PBiCG with the
diagonal, DILU and aDILU(2) (the paper's momentum setting).  The DIC/DILU sweeps are
sequential recurrences: their kernels' critical path is the dependency depth of the numbering
(reported).  One JSON line per case.   usage: python scripts/precond_bench.py [n ...]"""
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
from paper_2512_22215_b200 import spuma as S  # noqa: E402

f64 = dict(dtype=torch.float64, device="cuda")


def timed(fn, reps=2):
    best = None
    for _ in range(reps + 1):  # first call: warm-up (schedules, graphs)
        torch.cuda.synchronize()
        t = time.perf_counter()
        perf = fn()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        if best is None or dt < best[1]:
            best = (perf, dt)
    return best


def main(n):
    m = gen.cube(n)
    N, F = m.n_cells, m.n_faces
    h = P.Mesh.from_mesh(m)
    g = torch.as_tensor(gen.gamma_lognormal(m), **f64)
    b = torch.as_tensor(gen.rhs(m), **f64)
    diag, upper, src = torch.empty(N, **f64), torch.empty(F, **f64), b.clone()
    h.assemble_laplacian(g, None, 0, 0.0, diag, upper, src, None)
    depth = 3 * (n - 1) + 1
    rows = []

    def sym(label, fn):
        perf, dt = timed(fn)
        rows.append({"case": f"cube {n}^3 symmetric, {label}", "cells": N, "iterations": perf["n_iterations"],
                     "converged": perf["converged"], "solve_s": dt, "ms_per_iter": 1e3 * dt / max(perf["n_iterations"], 1),
                     "dependency_depth": depth})
        print(json.dumps(rows[-1]), flush=True)

    psi = torch.zeros(N, **f64)

    def run_pcg():
        psi.zero_()
        return h.pcg_solve(diag, upper, None, src.clone(), psi, 1e-6, 0.0, 5000, 0)

    sym("PCG diagonal (fused hot path)", run_pcg)
    for label, kind in (("PCG diagonal (general loop)", S.PC_DIAGONAL), ("PCG DIC", S.PC_DIC),
                        ("PCG aDILU(2)", S.PC_ADILU)):
        sym(label, lambda kind=kind: (psi.zero_(), h.pcg_solve_pc(diag, upper, src.clone(), psi, 1e-6, 0.0, 5000, 0,
                                                                   kind=kind, n_sweeps=2))[1])
    # asymmetric system (tests/cases.py recipe, on the device)
    gen_ = torch.Generator(device="cpu").manual_seed(5)
    e = (torch.rand(F, generator=gen_, dtype=torch.float64) * 0.8 - 0.4).to("cuda")
    Lap = torch.empty(F, **f64)
    d0 = torch.empty(N, **f64)
    h.assemble_laplacian(None, None, -1, 0.0, d0, Lap, torch.zeros(N, **f64), None)
    up, lo = Lap * (1 + e), Lap * (1 - e)
    own = torch.as_tensor(m.owner.astype(np.int64), device="cuda")
    nbr = torch.as_tensor(m.neighbour.astype(np.int64), device="cuda")
    off = torch.zeros(N, **f64).index_add_(0, own, up.abs()).index_add_(0, nbr, lo.abs())
    dA = -1.05 * off.clamp_min(1e-12)
    bA = torch.as_tensor(np.random.default_rng(5).standard_normal(N), **f64) * torch.as_tensor(m.V, **f64)
    for label, kind in (("PBiCG diagonal", S.PC_DIAGONAL), ("PBiCG DILU", S.PC_DILU), ("PBiCG aDILU(2)", S.PC_ADILU)):
        perf, dt = timed(lambda kind=kind: (psi.zero_(), h.pbicg_solve(dA, up, lo, bA, psi, 1e-8, 0.0, 1000, 0,
                                                                       kind=kind, n_sweeps=2))[1])
        rows.append({"case": f"cube {n}^3 asymmetric, {label}", "cells": N, "iterations": perf["n_iterations"],
                     "converged": perf["converged"], "solve_s": dt,
                     "ms_per_iter": 1e3 * dt / max(perf["n_iterations"], 1), "dependency_depth": depth})
        print(json.dumps(rows[-1]), flush=True)
    h.free()


if __name__ == "__main__":
    for a in (sys.argv[1:] or ["100", "200"]):
        main(int(a))
