"""Decomposed GAMG on ONE GPU (readings Q36-Q38): P processes share cuda:0, each with its own
sub-mesh handle (n_ranks = P), communicating through the external-comm callbacks over gloo
(NCCL cannot put two ranks on one device) -- the device code is the one the NCCL build runs.

Checked against the decomposed oracle O11dd (same sub-meshes, same systems): the per-rank
level sizes of the processor-local hierarchy bit-exact, V-cycle counts +-2 and the solution
within 1e-9 relative L2 at matched counts (Q11), identical decisions on every rank."""
import os

import numpy as np
import pytest

from test_gpu_multirank import _callbacks, _case, _port

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _params(S, O, name):
    """(library params, oracle params) of one configuration"""
    cfg = {
        "default": dict(),
        "gs2": dict(n_pre=1, n_post=1, smoother=1, n_inner=1),
        "noscale": dict(scale=False, n_post=1, omega=0.6, n_coarsest=4),
        "deep": dict(n_coarsest=2, n_post=3),
    }[name]
    g = S.spuma.gamg_params(n_pre_sweeps=cfg.get("n_pre", 0), n_post_sweeps=cfg.get("n_post", 2),
                      scale_correction=cfg.get("scale", True), n_cells_in_coarsest_level=cfg.get("n_coarsest", 10),
                      omega=cfg.get("omega", 0.75), smoother=cfg.get("smoother", 0), n_inner=cfg.get("n_inner", 1))
    o = O.gamg_params(n_pre=cfg.get("n_pre", 0), n_post=cfg.get("n_post", 2), scale=cfg.get("scale", True),
                      n_coarsest_cells=cfg.get("n_coarsest", 10), omega=cfg.get("omega", 0.75),
                      smoother=cfg.get("smoother", 0), n_inner=cfg.get("n_inner", 1))
    return g, o


def _global_rel_l2(P, loc, ref):
    num = np.array([np.sum((loc - ref) ** 2), np.sum(ref ** 2)])
    tot = [torch.empty(2, dtype=torch.float64) for _ in range(P)]
    dist.all_gather(tot, torch.from_numpy(num))
    return np.sqrt(sum(t[0].item() for t in tot) / sum(t[1].item() for t in tot))


def _worker(rank, P, how, configs, port, results):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import datetime
        dist.init_process_group("gloo", rank=rank, world_size=P, timeout=datetime.timedelta(seconds=300))
        import gen
        import oracle as O
        import paper_2512_22215_b200 as S
        torch.cuda.set_device(0)
        m, gamma, b, part = _case(P, how)
        subs = gen.decompose(m, part, P)
        gs, bs = gen.split_cell_field(gamma, part, P), gen.split_cell_field(b, part, P)
        halo = O.gamma_halo(subs, gs)
        ref_local = [int(np.nonzero(sm.gid == 0)[0][0]) if (sm.gid == 0).any() else -1 for sm in subs]
        systems = [O.assemble(sm, gs[r], ref_local[r], 0.0, source=bs[r], gamma_remote=halo[r])
                   for r, sm in enumerate(subs)]
        me, s = subs[rank], systems[rank]
        h = S.Mesh.from_mesh(me, rank=rank, n_ranks=P)
        h.set_comm_callbacks(*_callbacks(rank))
        f64 = dict(dtype=torch.float64, device="cuda")
        diag, upper = torch.as_tensor(s.diag, **f64), torch.as_tensor(s.upper, **f64)
        src = torch.as_tensor(s.source, **f64)
        iface = torch.as_tensor(np.concatenate(s.iface) if s.iface else np.zeros(1), **f64)
        for name in configs:
            gp, op = _params(S, O, name)
            # processor-local hierarchy: per-rank level sizes bit-exact (Q36)
            hier = h.gamg_hierarchy(gp, with_ftc=False)
            _, po = O.gamg_decomposed(subs, systems, None, O.controls(0.0, 0.0, 0, 0), op)
            assert hier["levels"] == po["levels"], (name, hier, po["level_cells"][rank])
            assert hier["cells"] == po["level_cells"][rank], (name, hier["cells"], po["level_cells"][rank])
            # solve to 1e-9: V-cycles +-2, solution at matched counts (Q11)
            psi = torch.zeros(me.n_cells, **f64)
            pf = h.gamg_solve(diag, upper, iface, src, psi, 1e-9, 0.0, 200, 0, params=gp)
            pso, po = O.gamg_decomposed(subs, systems, None, O.controls(1e-9, 0.0, 200, 0), op)
            assert pf["converged"] and abs(pf["n_iterations"] - po["n_iterations"]) <= 2, (name, pf, po)
            n = min(pf["n_iterations"], po["n_iterations"])
            psi.zero_()
            pf_n = h.gamg_solve(diag, upper, iface, src, psi, 0.0, 0.0, n, n, params=gp)
            assert pf_n["n_iterations"] == n
            pso, _ = O.gamg_decomposed(subs, systems, None, O.controls(0.0, 0.0, n, n), op)
            err = _global_rel_l2(P, psi.cpu().numpy(), pso[rank])
            assert err <= 1e-9, (name, err)
            allp = [None] * P
            dist.all_gather_object(allp, pf)
            assert all(p == allp[0] for p in allp)  # identical decisions on every rank
        h.free()
        results.put((rank, "ok"))
    except BaseException:
        import traceback
        results.put((rank, traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.parametrize("P,how,configs", [
    (2, "block", ("default", "gs2")),
    (3, "rcb", ("default", "noscale")),
    (4, "rcb", ("default", "deep")),
    (2, "lattice", ("default",)),   # un-permuted blocks: level 0 rows over ELL + interface terms
])
def test_gamg_multirank_matches_decomposed_oracle(P, how, configs):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, P, how, configs, port, q)) for r in range(P)]
    for p in ps:
        p.start()
    out = {}
    try:
        for _ in range(P):
            r, msg = q.get(timeout=900)
            out[r] = msg
            if msg != "ok":
                break
    finally:
        for p in ps:
            p.join(timeout=30)
            if p.is_alive():
                p.terminate()
    bad = {r: m for r, m in out.items() if m != "ok"}
    assert not bad and len(out) == P, bad or out
