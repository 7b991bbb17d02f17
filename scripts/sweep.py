#!/usr/bin/env python
"""Single-GPU measurement of the BASELINE.json configs other than the bench workload.

  C1  2-D cavity 20x20 (400 cells), gamma = 1 and log-normal: time to solution (latency-bound)
  C2  100^3 cube, random cell permutation, gamma log-normal: as given vs RCM-renumbered
  C4  perturbed (a = 0.15), randomly permuted 400^3 hex mesh (64M cells), gamma log-normal, 1 GPU
  C5  oversubscription sweep: cube n^3, n = 100/126/159/200/252/318 (1M..32M cells)

For each: cells*iter/s of the solve (CUDA events around spuma_pcg_solve), effective GB/s of
the iteration (the algorithmic bytes of the layout run: SURVEY §8(d) 112N + 16F per iteration,
or 136N on a lattice numbering with K = 3), the Amul's achieved GB/s from
libspuma's per-launch events, fraction of MEASURED_PEAKS hbm_gbs.  One JSON line per case.
usage: python scripts/sweep.py [C1] [C2] [C4] [C5] [--c5 100,126,...]
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


MODES = [None]  # --modes=0,3: every case once per SPUMA_OPT_PERSISTENT value (None: the library default)


def run_case(name, mesh, gamma, b, ref=0, renumber=False, ctl=(1e-6, 0.0, 5000, 0), reps=3, extra=None):
    out = None
    for mode in MODES:
        out = run_case1(name, mesh, gamma, b, ref, renumber, ctl, reps, dict(extra or {}), mode)
    return out


def run_case1(name, mesh, gamma, b, ref, renumber, ctl, reps, extra, mode):
    t0 = time.perf_counter()
    h = P.Mesh.from_mesh(mesh, renumber=renumber, stream=torch.cuda.current_stream().cuda_stream)
    if mode is not None:
        h.set_option(P.spuma.OPT_PERSISTENT, mode)
    t_create = time.perf_counter() - t0
    N, F = mesh.n_cells, mesh.n_faces
    diag, upper = torch.empty(N, **f64), torch.empty(F, **f64)
    b_dev = torch.as_tensor(b, **f64)
    g_dev = None if gamma is None else torch.as_tensor(gamma, **f64)
    src, psi = torch.empty(N, **f64), torch.zeros(N, **f64)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]

    def once(timing):
        h.set_timing(timing)
        src.copy_(b_dev)
        e[0].record()
        h.assemble_laplacian(g_dev, None, ref, 0.0, diag, upper, src, None)
        e[1].record()
        psi.zero_()
        e[2].record()
        perf = h.pcg_solve(diag, upper, None, src, psi, *ctl)
        e[3].record()
        torch.cuda.synchronize()
        return perf, e[0].elapsed_time(e[1]) / 1e3, e[2].elapsed_time(e[3]) / 1e3

    once(False)  # warm-up (graph capture)
    runs = [once(False) for _ in range(reps)]
    h.reset_stats()
    once(True)
    st = h.get_stats()
    perf, t_asm, t_sol = min(runs, key=lambda r: r[2])
    n_it = perf["n_iterations"]
    # algorithmic bytes of the layout the hot loop ran: lattice slots 24N + 8KN per
    # Amul, else SURVEY §8(d) 24N + 16F; the iteration adds 88N (update 56N + direction 32N)
    K = len(P.spuma.host_lattice_offsets(N, mesh.owner, mesh.neighbour)) if st["amul_variant"] in (12, 13) else 0
    B_A = 24 * N + 8 * K * N if K else 24 * N + 16 * F
    B_it = B_A + 88 * N
    amul_ms = st["phase_ms"][1] / max(st["phase_count"][1], 1)
    out = {"case": name, "cells": N, "faces": F, "renumber": renumber, "iterations": n_it,
           "converged": perf["converged"], "final_residual": perf["final_residual"],
           "solve_s": t_sol, "assembly_s": t_asm, "mesh_create_s": t_create,
           "cells_iter_per_s": N * n_it / t_sol,
           "iteration_GBps_incl_setup": B_it * n_it / t_sol / 1e9,
           "iteration_frac_of_measured_peak": B_it * n_it / t_sol / 1e9 / PEAK,
           "amul_us": 1e3 * amul_ms,
           "amul_variant": st["amul_variant"], "amul_bytes": B_A, "iteration_bytes": B_it,
           "amul_alg_GBps": B_A / (amul_ms / 1e3) / 1e9 if amul_ms else None,
           "amul_frac_of_measured_peak": B_A / (amul_ms / 1e3) / 1e9 / PEAK if amul_ms else None,
           "assembly_alg_GBps": (56 * F + 24 * N) / t_asm / 1e9,
           "peak_GBps": PEAK}
    if st["loop_mode"]:  # the persistent loop ran: its own time and bytes (bench.py loop_bytes)
        import bench
        T = st["loop_threads"]
        need = -(-(-(-(N // 2) // T)) // max(st["loop_grid"], 1))
        frac = min(1.0, (st["loop_tmem_pairs"] + st["loop_smem_pairs"]) / need) if need else 1.0
        lb = bench.loop_bytes(N, K, frac) if K else None
        loop_ms = st["loop_ms"] / max(st["loop_count"], 1)
        out.update({"loop_mode": st["loop_mode"], "loop_us_per_iter": 1e3 * loop_ms / max(n_it, 1),
                    "loop_rA_resident_frac": frac, "loop_bytes_per_iter": lb["iter"] if lb else None,
                    "loop_GBps": lb["iter"] * n_it / (loop_ms / 1e3) / 1e9 if lb and loop_ms else None})
    else:
        out["loop_mode"] = 0
    out["persistent_option"] = mode
    out.update(extra)
    print(json.dumps(out), flush=True)
    h.free()
    return out


def c1():
    m = gen.cavity2d(20)
    b = gen.rhs(m)
    for gname, g in (("gamma=1", None), ("gamma=lognormal", gen.gamma_lognormal(m))):
        r = run_case(f"C1 cavity 20x20 {gname}", m, g, b, reps=20)
        print(json.dumps({"case": f"C1 time-to-solution {gname}", "assembly_plus_solve_us":
                          1e6 * (r["solve_s"] + r["assembly_s"])}), flush=True)


def c2():
    m = gen.cube(100)
    g, b = gen.gamma_lognormal(m), gen.rhs(m)
    perm = gen.random_perm(m.n_cells)
    mp = gen.permute(m, perm)
    gp, bp = gen.permute_cell_field(g, perm), gen.permute_cell_field(b, perm)
    run_case("C2 cube 100^3 random permutation, as given", mp, gp, bp, ref=int(perm[0]))
    run_case("C2 cube 100^3 random permutation, RCM renumbered", mp, gp, bp, ref=int(perm[0]), renumber=True)
    run_case("C2 reference: cube 100^3 natural order", m, g, b)


def c4(n=400):
    t = time.perf_counter()
    m = gen.perturbed(n, 0.15)
    g, b = gen.gamma_lognormal(m), gen.rhs(m)
    perm = gen.random_perm(m.n_cells)
    mp = gen.permute(m, perm)
    del m
    gp, bp = gen.permute_cell_field(g, perm), gen.permute_cell_field(b, perm)
    tg = time.perf_counter() - t
    run_case(f"C4 perturbed {n}^3 (a=0.15) random permutation, RCM renumbered, 1 GPU", mp, gp, bp,
             ref=int(perm[0]), renumber=True, reps=1, extra={"generate_s": tg})


def c5(ns):
    for n in ns:
        m = gen.cube(n)
        run_case(f"C5 cube {n}^3", m, None, gen.rhs(m), reps=2)


if __name__ == "__main__":
    args = sys.argv[1:]
    ns = [100, 126, 159, 200, 252, 318]
    for a in args:
        if a.startswith("--c5="):
            ns = [int(x) for x in a.split("=")[1].split(",")]
        if a.startswith("--modes="):
            MODES[:] = [int(x) for x in a.split("=")[1].split(",")]
    todo = [a for a in args if not a.startswith("--")] or ["C1", "C2", "C5", "C4"]
    for t in todo:
        {"C1": c1, "C2": c2, "C4": c4, "C5": lambda: c5(ns)}[t]()
