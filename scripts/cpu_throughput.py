#!/usr/bin/env python
"""Host-throughput mode of the CPU oracle: C concurrent single-threaded oracle
processes, each on an independent cube of ~N/C cells (as an MPI CPU run would partition the
200^3 workload), each running assembly + setup + K PCG iterations.  Reports the aggregate
cells*iter/s and the paper's COE analogue against a GPU value given on the command line.
usage: python scripts/cpu_throughput.py [--n 200] [--iters 40] [--procs all] [--gpu 4.03e10]"""
import argparse
import json
import os
import sys
import time
from multiprocessing import get_context

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def work(args):
    n_local, iters, core = args
    try:
        os.sched_setaffinity(0, {core})
    except (AttributeError, OSError):
        pass
    import gen
    import oracle as O
    m = gen.cube(n_local)
    b = gen.rhs(m)
    t0 = time.perf_counter()
    O.solve_case(m, None, b, 0, 0.0, O.controls(0.0, 0.0, iters, iters))
    return m.n_cells, iters, time.perf_counter() - t0


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=200)
    ap.add_argument("--iters", type=int, default=40)
    ap.add_argument("--procs", default="all")
    ap.add_argument("--gpu", type=float, default=None)
    a = ap.parse_args()
    cores = sorted(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else list(range(os.cpu_count()))
    C = len(cores) if a.procs == "all" else int(a.procs)
    n_local = max(2, round((a.n ** 3 / C) ** (1 / 3)))
    import oracle
    oracle.build()
    with get_context("spawn").Pool(C) as pool:
        res = pool.map(work, [(n_local, a.iters, cores[i % len(cores)]) for i in range(C)])
    agg = sum(c * k / t for c, k, t in res)  # concurrent: aggregate rate
    out = {"mode": "oracle throughput", "processes": C, "cells_per_process": n_local ** 3,
           "iterations": a.iters, "aggregate_cells_iter_per_s": agg, "per_core": agg / C,
           "seconds": max(t for _, _, t in res)}
    if a.gpu:
        out["coe_cores_per_gpu"] = a.gpu / (agg / C)
        out["gpu_over_all_host_cores"] = a.gpu / agg
    print(json.dumps(out))
