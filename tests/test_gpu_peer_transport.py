"""The peer-memory transport on ONE GPU (spuma_peer_export / spuma_peer_import, csrc/peer.cu):
P processes share cuda:0 and map each other's mailboxes through CUDA IPC; every halo and every
all-gather of rank partials then runs as device kernels (fused pack + P2P stores, release /
acquire epoch flags) -- the code path that runs over NVLink between GPUs, no NCCL, no host
callbacks, iteration batches captured in CUDA graphs.

Checked: the decomposed PCG against the decomposed oracle (Q11 protocol) and bitwise against the
host-callback transport (same kernels, same reduction order -> same bits) and against the peer
transport with separate transport kernels (SPUMA_OPT_PEER_FUSED = 0); the decomposed GAMG
and PCG-DIC against their decomposed oracles; no poll ever timed out."""
import os

import numpy as np
import pytest

from conftest import shared_gpu_ranks  # noqa: E402

from test_gpu_multirank import _callbacks, _case, _port

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _rel(P, loc, ref):
    num = np.array([np.sum((loc - ref) ** 2), np.sum(ref ** 2)])
    tot = [torch.empty(2, dtype=torch.float64) for _ in range(P)]
    dist.all_gather(tot, torch.from_numpy(num))
    return np.sqrt(sum(t[0].item() for t in tot) / sum(t[1].item() for t in tot))


def _worker(rank, P, how, port, results):
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
        f64 = dict(dtype=torch.float64, device="cuda")
        # reference run through the host-callback transport
        hc = S.Mesh.from_mesh(me, rank=rank, n_ranks=P)
        hc.set_comm_callbacks(*_callbacks(rank))
        hc.set_option(S.spuma.OPT_SMALL_SOLVE_MAX_CELLS, 0)
        # the peer transport
        h = S.Mesh.from_mesh(me, rank=rank, n_ranks=P)
        h.enable_peer_transport()
        h.set_option(S.spuma.OPT_SMALL_SOLVE_MAX_CELLS, 0)
        # assembly through the peer halo (gamma) is bitwise the oracle's
        diag, upper = torch.zeros(me.n_cells, **f64), torch.zeros(me.n_faces, **f64)
        src = torch.as_tensor(bs[rank], **f64)
        iface = torch.zeros(max(h.n_iface, 1), **f64)
        h.assemble_laplacian(torch.as_tensor(gs[rank], **f64), None, ref_local[rank], 0.0, diag, upper, src, iface)
        assert np.array_equal(diag.cpu().numpy(), s.diag) and np.array_equal(upper.cpu().numpy(), s.upper)
        oi = np.concatenate(s.iface) if s.iface else np.zeros(0)
        assert np.array_equal(iface.cpu().numpy()[:oi.shape[0]], oi)
        # PCG: oracle (Q11) and bitwise vs the callback transport
        psi = torch.zeros(me.n_cells, **f64)
        pf = h.pcg_solve(diag, upper, iface, src, psi, 1e-9, 0.0, 3000, 0)
        _, po = O.pcg_decomposed(subs, systems, None, O.controls(1e-9, 0.0, 3000, 0))
        assert pf["converged"] and abs(pf["n_iterations"] - po["n_iterations"]) <= 2, (pf, po)
        psi_c = torch.zeros(me.n_cells, **f64)
        pc = hc.pcg_solve(diag, upper, iface, src, psi_c, 1e-9, 0.0, 3000, 0)
        assert pc == pf and torch.equal(psi, psi_c)
        # the fused loop (halo in the direction / interface-row kernels, all-gather in the
        # reductions' last CTA) vs separate transport kernels: bitwise the same
        h.set_option(S.spuma.OPT_PEER_FUSED, 0)
        psi_s = torch.zeros(me.n_cells, **f64)
        ps_ = h.pcg_solve(diag, upper, iface, src, psi_s, 1e-9, 0.0, 3000, 0)
        h.set_option(S.spuma.OPT_PEER_FUSED, 1)
        assert ps_ == pf and torch.equal(psi_s, psi)
        n = min(pf["n_iterations"], po["n_iterations"])
        psi.zero_()
        h.pcg_solve(diag, upper, iface, src, psi, 0.0, 0.0, n, n)
        pso, _ = O.pcg_decomposed(subs, systems, None, O.controls(0.0, 0.0, n, n))
        assert _rel(P, psi.cpu().numpy(), pso[rank]) <= 1e-9
        # GAMG (coarse-level interface exchanges + the hierarchy build's collectives)
        gp = S.spuma.gamg_params()
        psi.zero_()
        pg = h.gamg_solve(diag, upper, iface, src, psi, 1e-9, 0.0, 200, 0, params=gp)
        _, pgo = O.gamg_decomposed(subs, systems, None, O.controls(1e-9, 0.0, 200, 0))
        assert pg["converged"] and abs(pg["n_iterations"] - pgo["n_iterations"]) <= 2, (pg, pgo)
        ng = min(pg["n_iterations"], pgo["n_iterations"])
        psi.zero_()
        h.gamg_solve(diag, upper, iface, src, psi, 0.0, 0.0, ng, ng, params=gp)
        pso, _ = O.gamg_decomposed(subs, systems, None, O.controls(0.0, 0.0, ng, ng))
        assert _rel(P, psi.cpu().numpy(), pso[rank]) <= 1e-9
        # PCG-DIC (processor-local factorisation)
        psi.zero_()
        pk = h.pcg_solve_pc(diag, upper, src, psi, 1e-9, 0.0, 3000, 0, kind=S.spuma.PC_DIC, iface_coeffs=iface)
        _, pko = O.pcg_decomposed(subs, systems, None, O.controls(1e-9, 0.0, 3000, 0), kind=O.DIC)
        assert abs(pk["n_iterations"] - pko["n_iterations"]) <= 2, (pk, pko)
        h.peer_check()
        allp = [None] * P
        dist.all_gather_object(allp, (pf, pg, pk))
        assert all(p == allp[0] for p in allp)
        dist.barrier()  # every rank done with the peers' mailboxes before any handle is freed
        h.free()
        hc.free()
        results.put((rank, "ok"))
    except BaseException:
        import traceback
        results.put((rank, traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@shared_gpu_ranks
@pytest.mark.parametrize("P,how", [(2, "block"), (3, "rcb"), (4, "rcb"), (2, "lattice")])
def test_peer_transport_matches_oracle_and_callbacks(P, how):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, P, how, port, q)) for r in range(P)]
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
