#!/usr/bin/env python
"""Benchmark: pressure PCG cells*iter/s and HBM GB/s (% of peak) -- BASELINE.json metric.

Workload (config.workload): BASELINE config 3, the 3-D cavity/cube with 200^3
cells PER GPU (8M cells, 23.88M internal faces), weak scaling over
1/2/4/8 GPUs (N = 1: one 200^3 cube).  Synthetic, seeded inputs
(gen/: unit-cube lattice, six zeroGradient walls, gamma = 1, b = V(2U-1)
minus its mean, reference cell 0, psi0 = 0); solve to 1e-6 (reading Q5:
tolerance 1e-6 on the normalised residual, relTol 0, minIter 0, maxIter 5000).

One step = the whole hot path on one batch of input: assemble the Laplacian
(A4-A5: face coefficients + diagonal gather + reference) and solve it (A6
setup + A7-A11 iterations to convergence + A12).  value = global cells *
PCG iterations / step time (max over ranks).  Inputs (8M cells, ~1.3 GB per
iteration) are far larger than the 126 MB L2, so no L2 flush is needed.

Also reported: roofline of the dominant kernel (the persistent PCG loop
k_pcg_loop -- every A7-A11 iteration of a solve in one launch -- or, with the
graph batches, the Amul k_amul_dot), timed live with CUDA events over the
timed region; e2e through the C-ABI with host
buffers; clocks under load; our kernel launch count; and the CPU oracle
(cpu_baseline) on a bounded sample of the same workload.

--impl reference: the oracle (plain single-threaded C) timed on the host as
the reference arm (this tier has no reference implementation to install).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "pressure PCG cells·iter/s and HBM GB/s (% of peak) at 1/2/4/8 B200"
UNIT = "cells*iter/s"
TOL = (1e-6, 0.0, 5000, 0)


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def loop_bytes(N, lattice_k, resident_frac):
    """Bytes per iteration the persistent loop (SPUMA_OPT_PERSISTENT) must move through
    HBM, per phase: C direction rD + pA_prev + pA (24 B/cell) + the psi pair every second iteration
    (psi read + write + p_{n-2}: 12 B/cell on average) + rA where it is not on chip (8 B/cell);
    A Amul as the lattice layout (24 + 8K B/cell); B update wA + rD (16 B/cell) + rA read and write
    where it is not on chip (16 B/cell).  rA held in tensor / shared memory costs nothing per
    iteration (loaded once and written back once per solve: 16 B/cell per launch)."""
    off = 1.0 - resident_frac
    c = (24 + 12 + 8 * off) * N
    a = (24 + 8 * lattice_k) * N
    b = (16 + 16 * off) * N
    return {"C": c, "A": a, "B": b, "iter": a + b + c, "per_launch_fixed": 16 * N * resident_frac}


def algorithmic_bytes(N, F, lattice_k=0):
    """per PCG iteration, fused minimum. Phase A (Amul + dot): 24 B/cell + 16 B/face;
    B (update + dots): 56 B/cell; C (direction): 32 B/cell.

    On a lattice numbering the Amul runs over K <= 3 coefficient slots per row and no index
    arrays (variant 12): phase A is then 24 B/cell (diag, pA, wA) + 8 K B/cell
    (the owner-side slots; the neighbour-side slots and the pA gathers are L2 hits, counted
    once) -- the bytes that layout must move."""
    a = 24 * N + 8 * lattice_k * N if lattice_k else 24 * N + 16 * F
    return {"A": a, "B": 56 * N, "C": 32 * N, "iter": a + 88 * N, "A_survey": 24 * N + 16 * F,
            "iter_survey": 112 * N + 16 * F, "A_layout": "lattice slots (K = %d)" % lattice_k if lattice_k
            else "ELL rows (indices + coefficients per face)"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (FileNotFoundError, OSError):
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        mhz, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                mhz.append(float(r[1]))
                mx = float(r[2])
                for n, v in zip(names, r[5:9]):
                    if v.lower() == "active":
                        reasons.add(n)
            except (ValueError, IndexError):
                continue
        if not mhz:
            return None
        return {"sm_mhz": statistics.median(mhz), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(mhz)}


def load_traffic(workload, kernel):
    """ncu DRAM bytes per launch of the dominant kernel (profiles/ncu_traffic.json), if that capture
    is of this workload and of the kernel this run's roofline names."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    try:
        with open(p) as f:
            j = json.load(f)
        for e in j.get("kernels", [j]):
            if e.get("workload", j.get("workload")) == workload and kernel in e.get("kernel", ""):
                return e.get("dram_bytes_per_launch", e.get("amul_dram_bytes_per_launch"))
    except (OSError, ValueError):
        pass
    return None


# ---------------------------------------------------------------------------- workload
def build_workload(n, rank, world, cdev="cuda"):
    """C3: one n^3 block per rank of the global (n px, n py, n pz) cube (px,py,pz) = 1/2x1x1/2x2x1/2x2x2."""
    import gen
    wl = f"C3 cube {n}^3 per GPU (weak), gamma=1, tol 1e-6"
    if world == 1:
        m = gen.cube(n)
        b = gen.rhs(m)
        return m, b, 0, {"workload": wl, "cells_per_gpu": n ** 3}
    import torch
    import torch.distributed as dist
    nproc = gen.nproc_for(world)
    m = gen.weak_block(n, nproc, rank)
    # b = V (2U - 1) keyed by global cell id, minus the GLOBAL mean (all-reduced)
    b = m.V * (2.0 * gen.uniform(gen.SEED_RHS, 0, m.gid) - 1.0)
    t = torch.tensor([b.sum(), float(m.n_cells)], dtype=torch.float64, device=cdev)
    dist.all_reduce(t)
    b = b - float(t[0] / t[1])
    ref = 0 if rank == 0 else -1  # global cell 0 lives on rank 0, local cell 0
    return m, b, ref, {"workload": wl, "cells_per_gpu": n ** 3, "blocks": list(nproc)}


# ---------------------------------------------------------------------------- oracle legs
def oracle_sample(n, iters):
    """The oracle (as it stands) on the same workload: assembly + PCG setup + `iters` iterations."""
    import gen
    import oracle as O
    m = gen.cube(n)
    b = gen.rhs(m)
    O.build()
    t0 = time.perf_counter()
    O.solve_case(m, None, b, 0, 0.0, O.controls(0.0, 0.0, iters, iters))
    t = time.perf_counter() - t0
    return m.n_cells * iters / t, t


def cpu_baseline(n, iters):
    v, t = oracle_sample(n, iters)
    return {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"cube {n}^3 ({n ** 3} cells): assembly + PCG setup + {iters} iterations "
                      f"(minIter = maxIter = {iters}), single thread, {t:.1f} s"}


def _throughput_worker(a):
    n_local, iters, core = a
    try:
        os.sched_setaffinity(0, {core})
    except (AttributeError, OSError):
        pass
    v, t = oracle_sample(n_local, iters)
    return n_local ** 3, iters, t


def cpu_throughput(n, iters, gpu_value=None):
    """The cpu_baseline leg in host-throughput mode: C concurrent single-threaded
    oracle processes (C = the host cores), each on an independent cube of ~n^3/C cells -- the
    partition an MPI CPU run of the workload would use -- each running assembly + setup + `iters`
    PCG iterations; the aggregate cells*iter/s and the paper's COE analogue (Eq. 1)."""
    from multiprocessing import get_context
    import oracle
    oracle.build()
    cores = sorted(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else list(range(os.cpu_count()))
    C = len(cores)
    n_local = max(2, round((n ** 3 / C) ** (1 / 3)))
    with get_context("spawn").Pool(C) as pool:
        res = pool.map(_throughput_worker, [(n_local, iters, cores[i]) for i in range(C)])
    agg = sum(c * k / t for c, k, t in res)
    out = {"mode": "oracle throughput", "kind": "oracle", "cores": C, "processes": C,
           "cells_per_process": n_local ** 3, "iterations": iters, "value": agg, "unit": UNIT,
           "per_core": agg / C, "seconds": max(t for _, _, t in res)}
    if gpu_value:
        out["coe_cores_per_gpu"] = gpu_value / (agg / C)
        out["gpu_over_all_host_cores"] = gpu_value / agg
    return out


def run_reference(args, rank, world):
    if rank != 0:
        return
    n = args.n
    iters = args.ref_iters
    for _ in range(args.warmup):
        oracle_sample(n, iters)
    ts = []
    for _ in range(args.steps):
        v, t = oracle_sample(n, iters)
        ts.append(t)
    T = sum(ts)
    value = n ** 3 * iters * args.steps / T
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * T / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic",
           "config": {"workload": f"C3 cube {n}^3 per GPU (weak), gamma=1; oracle sample of {iters} iterations per step",
                      "cells": n ** 3},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                            "sample": f"per step: cube {n}^3 assembly + PCG setup + {iters} iterations, single thread"},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ---------------------------------------------------------------------------- GPU arm
def run_gpu(args, rank, world, local_rank):
    import torch
    import paper_2512_22215_b200 as P

    # SPUMA_BENCH_SHARE_GPU=1 (testing only): every rank on cuda:0, host plumbing over gloo -- runs the
    # whole N > 1 code path (peer transport) on a one-GPU box; not a scaling measurement
    share = os.environ.get("SPUMA_BENCH_SHARE_GPU") == "1"
    if share:
        local_rank = 0
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    cdev = torch.device("cpu") if share else dev  # device of the host-plumbing collectives
    if world > 1:
        import torch.distributed as dist
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    mesh, b, ref, cfg = build_workload(args.n, rank, world, cdev)
    N, F = mesh.n_cells, mesh.n_faces
    stream = torch.cuda.current_stream()
    uid = None
    transport = "none (1 rank)"
    h = None
    if world > 1 and args.transport == "peer":
        # device-side transport over peer memory (CUDA IPC over NVLink): halo stores and
        # rank-partial all-gathers inside the kernels; NCCL if any rank cannot map its peers
        h = P.Mesh.from_mesh(mesh, stream=stream.cuda_stream, rank=rank, n_ranks=world)
        err = ""
        try:
            h.enable_peer_transport()
        except Exception as e:  # noqa: BLE001
            err = str(e).splitlines()[0][:120]
        flag = torch.tensor([1.0 if err else 0.0], device=cdev)
        torch.distributed.all_reduce(flag)
        if flag.item() == 0.0:
            transport = "peer (CUDA IPC / NVLink, in-kernel halo + all-gather)"
        else:
            torch.distributed.barrier()
            h.free()
            h = None
            transport = f"nccl (peer transport unavailable: {err or 'on another rank'})"
    if world > 1 and h is None:
        obj = [P.nccl_get_unique_id() if rank == 0 else None]
        torch.distributed.broadcast_object_list(obj, src=0)
        uid = obj[0]
        if not transport.startswith("nccl"):
            transport = "nccl (send/recv halo, all-gather of rank partials)"
    if h is None:
        h = P.Mesh.from_mesh(mesh, stream=stream.cuda_stream, rank=rank, n_ranks=world, nccl_unique_id=uid)
    h.set_batch(args.batch)
    if args.amul_variant is not None:
        h.set_option(P.spuma.OPT_AMUL_VARIANT, args.amul_variant)
    if args.alt_sweep is not None:
        h.set_option(P.spuma.OPT_ALT_SWEEP, args.alt_sweep)
    if args.defer_psi is not None:
        h.set_option(P.spuma.OPT_DEFER_PSI, args.defer_psi)
    if args.l2_persist is not None:
        h.set_option(P.spuma.OPT_L2_PERSIST, args.l2_persist)
    if args.persistent is not None:
        h.set_option(P.spuma.OPT_PERSISTENT, args.persistent)
    if args.loop_l2 is not None:
        h.set_option(P.spuma.OPT_LOOP_L2, args.loop_l2)
    f64 = dict(dtype=torch.float64, device=dev)
    diag, upper = torch.empty(N, **f64), torch.empty(F, **f64)
    b_dev = torch.as_tensor(b, **f64)
    src, psi = torch.empty(N, **f64), torch.empty(N, **f64)
    iface = torch.empty(h.n_iface, **f64) if h.n_iface else None
    perfs = []

    def step():
        src.copy_(b_dev)
        h.assemble_laplacian(None, None, ref, 0.0, diag, upper, src, iface)
        psi.zero_()
        perfs.append(h.pcg_solve(diag, upper, iface, src, psi, *TOL))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    perfs.clear()
    h.reset_stats()
    h.set_timing(not args.no_kernel_timing)
    clocks = ClockSampler(local_rank)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clk = clocks.stop()
    t = e0.elapsed_time(e1) / 1000.0
    if world > 1:
        tt = torch.tensor([t], dtype=torch.float64, device=cdev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t = float(tt.item())
    st = h.get_stats()
    h.set_timing(False)
    if st["loop_mode"]:  # per-phase profile of the persistent loop: one more (untimed) step
        h.reset_stats()
        h.set_option(P.spuma.OPT_LOOP_PROFILE, 1)
        step()
        torch.cuda.synchronize()
        prof = h.get_stats()
        h.set_option(P.spuma.OPT_LOOP_PROFILE, 0)
        perfs.pop()
        for k in ("loop_work_ms", "loop_wait_ms", "loop_work_max_ms"):
            st[k] = [v * len(perfs) for v in prof[k]]  # per timed step: scaled to the timed steps
    iters = sum(p["n_iterations"] for p in perfs)
    n_global = N * world
    value = n_global * iters / t
    lat_k = len(P.spuma.host_lattice_offsets(N, mesh.owner, mesh.neighbour)) if st["amul_variant"] in (12, 13) else 0
    nb = algorithmic_bytes(N, F, lat_k)
    peak, peak_kind = peaks()
    amul_ms = st["phase_ms"][1] / max(st["phase_count"][1], 1)
    achieved = nb["A"] / (amul_ms / 1e3) / 1e9 if amul_ms > 0 else None
    phase_avg = {k: (st["phase_ms"][i] / st["phase_count"][i] if st["phase_count"][i] else None)
                 for i, k in enumerate(("direction", "amul_dot", "update", "assembly"))}
    loop = None
    if st["loop_mode"]:
        # the persistent loop ran: ONE launch per solve is the dominant kernel (CUDA events on the
        # launching stream around each launch); its bytes per launch = iterations x loop bytes
        T = st["loop_threads"]
        need = -(-(-(-(N // 2) // T)) // max(st["loop_grid"], 1))
        frac = min(1.0, (st["loop_tmem_pairs"] + st["loop_smem_pairs"]) / need) if need else 1.0
        lb = loop_bytes(N, lat_k, frac)
        launches = max(st["loop_count"], 1)
        loop_ms = st["loop_ms"] / launches
        it_per_launch = iters / launches
        bytes_launch = lb["iter"] * it_per_launch + lb["per_launch_fixed"]
        achieved = bytes_launch / (loop_ms / 1e3) / 1e9 if loop_ms > 0 else None
        itn = max(iters, 1)
        loop = {"mode": st["loop_mode"], "grid": st["loop_grid"], "threads": T,
                "rA_pairs_tmem": st["loop_tmem_pairs"], "rA_pairs_smem": st["loop_smem_pairs"],
                "rA_resident_frac": frac, "bytes_per_iter": lb, "avg_launch_ms": loop_ms,
                "us_per_iter": loop_ms * 1e3 / it_per_launch if it_per_launch else None,
                "phase_work_us": [v * 1e3 / itn for v in st["loop_work_ms"]],
                "phase_barrier_wait_us": [v * 1e3 / itn for v in st["loop_wait_ms"]],
                "phase_order": ["C direction", "A Amul + dot", "B update + dots"],
                "bytes_per_launch": bytes_launch}
    # whole-step effective bandwidth: algorithmic iteration bytes x iterations / step time
    # (assembly and setup included in the time, so this under-states the loop)
    eff_gbs = nb["iter"] * iters / t / 1e9 if t > 0 else None

    # ---- e2e: the same metric through the C-ABI with pinned host buffers (copies inside the region)
    e2e = None
    if not args.no_e2e:
        # each step's inputs (b, psi0 = 0) prepared in pinned host memory before the timed region
        # (assembly updates source in place and the solve overwrites psi, so every step has its own)
        hb = torch.as_tensor(b).pin_memory()
        bufs = [(hb.clone().pin_memory(), torch.zeros(N, dtype=torch.float64).pin_memory())
                for _ in range(args.steps + 1)]
        eperfs = []

        def estep(i):
            hsrc, hpsi = bufs[i]
            h.assemble_laplacian(None, None, ref, 0.0, diag, upper, hsrc, iface)
            eperfs.append(h.pcg_solve(diag, upper, iface, hsrc, hpsi, *TOL))

        estep(args.steps)
        eperfs.clear()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        e0.record(stream)
        for i in range(args.steps):
            estep(i)
        e1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - w0
        te = max(e0.elapsed_time(e1) / 1000.0, wall)
        if world > 1:
            tt = torch.tensor([te], dtype=torch.float64, device=cdev)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            te = float(tt.item())
        eit = sum(p["n_iterations"] for p in eperfs)
        e2e = {"value": n_global * eit / te, "unit": UNIT,
               "h2d_bytes_per_step": 8 * N * 3, "d2h_bytes_per_step": 8 * N * 2,
               "note": "pinned host source and psi0 per step (prepared before the region) through "
                       "spuma_assemble_laplacian/spuma_pcg_solve; h2d = source (assemble) + source + psi0 (solve); "
                       "d2h = source (assemble) + psi"}

    if rank != 0:
        return
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        cpu = cpu_baseline(args.n, args.cpu_iters)
        # the paper's coefficient of equivalence (Eq. 1) in its single-core form:
        # how many oracle cores one B200 is worth on this workload
        cpu["coe_cores_per_gpu"] = value / cpu["value"]
    traffic = load_traffic(cfg["workload"], "k_pcg_loop" if loop else f"k_amul_dot<{st['amul_variant']},")
    cfg.update({"global_cells": n_global, "faces_per_gpu": F, "parallelism": f"dd{world}", "transport": transport,
                "iterations_per_step": iters / max(len(perfs), 1), "l2": "inputs larger than L2 (no flush)",
                "batch_iterations": st["batch_iterations"], "grid": st["blocks_per_grid"],
                "effective_iteration_GBps": eff_gbs,
                "effective_iteration_note": "algorithmic bytes per iteration of the layout run (lattice slots: "
                                            "136N; ELL: SURVEY 8(d) 112N+16F) x iterations / whole step time "
                                            "(deferred psi updates move ~8 B/cell less than this count)",
                "amul_variant": st["amul_variant"],
                "effective_iteration_frac_of_peak": (eff_gbs / peak) if eff_gbs else None,
                "effective_iteration_frac_of_8TBps": (eff_gbs / 8000.0) if eff_gbs else None,
                "phase_avg_ms": phase_avg, "algorithmic_bytes": nb, "persistent_loop": loop})
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": 1000 * t / args.steps, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfg,
           "roofline": ({"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                         "kernel": "k_pcg_loop (persistent: every A7-A11 iteration of a solve in one launch, "
                                   "rA on chip; bytes = iterations x loop bytes per iteration)",
                         "peak_source": f"{peak_kind} hbm_gbs",
                         "bytes_per_launch": loop["bytes_per_launch"], "avg_launch_ms": loop["avg_launch_ms"]}
                        if loop else
                        {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                         "kernel": f"k_amul_dot<{st['amul_variant']}> (A7 Amul + wA.pA, {nb['A_layout']})",
                         "peak_source": f"{peak_kind} hbm_gbs",
                         "bytes_per_launch": nb["A"], "avg_launch_ms": amul_ms}),
           "cpu_baseline": cpu, "e2e": e2e, "clocks": clk, "gpu_launches": st["kernel_launches"],
           "solver": {"n_iterations": [p["n_iterations"] for p in perfs],
                      "final_residual": perfs[-1]["final_residual"] if perfs else None}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="spuma", choices=["spuma", "reference"])
    ap.add_argument("--edge", "--n", dest="n", type=int, default=200, help="cube edge per GPU (C3: 200)")
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--cpu-iters", type=int, default=150)
    ap.add_argument("--ref-iters", type=int, default=20)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-kernel-timing", action="store_true")
    ap.add_argument("--transport", default="peer", choices=["peer", "nccl"],
                    help="N > 1: device-side peer-memory transport (default) or NCCL")
    ap.add_argument("--amul-variant", type=int, default=None, help="A/B only (default: the library's)")
    ap.add_argument("--alt-sweep", type=int, default=None, help="A/B only (default: the library's)")
    ap.add_argument("--defer-psi", type=int, default=None, help="A/B only (default: the library's)")
    ap.add_argument("--l2-persist", type=int, default=None, help="A/B only (default: the library's)")
    ap.add_argument("--persistent", type=int, default=None, help="A/B only (default: the library's)")
    ap.add_argument("--loop-l2", type=int, default=None, help="A/B only (default: the library's)")
    ap.add_argument("--cpu-throughput", action="store_true",
                    help="only the cpu_baseline leg in host-throughput mode (every host core), one JSON line")
    ap.add_argument("--gpu-value", type=float, default=None, help="--cpu-throughput: GPU value for the COE analogue")
    ap.add_argument("--throughput-iters", type=int, default=40, help="--cpu-throughput: PCG iterations per process")
    args = ap.parse_args()
    if args.cpu_throughput:
        print(json.dumps(cpu_throughput(args.n, args.throughput_iters, args.gpu_value)), flush=True)
        return
    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_gpu(args, rank, world, local)


if __name__ == "__main__":
    main()
