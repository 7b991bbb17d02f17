"""Multi-rank path of libspuma on ONE GPU: P processes share cuda:0, each with its own
sub-mesh handle (n_ranks = P), communicating through the external-comm callbacks over
torch.distributed gloo (NCCL cannot put two ranks on one device).  Everything on the
device is the multi-rank code the NCCL build runs: gamma halo + processor coefficients
in global orientation (Q9), per-cell interface masks in the Amul, rank partials
finalised from the rank-ordered all-gather.

Checked against the decomposed oracle (O8, same sub-meshes): coefficients and
interface coefficients bitwise, PCG iterations +-2 and solution 1e-9 at matched counts
(Q11); and against the undecomposed oracle (P8)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _callbacks(rank):
    def exchange(peers, offsets, counts, send, recv):
        reqs = []
        for p, o, c in zip(peers, offsets, counts):
            reqs.append(dist.isend(torch.from_numpy(np.array(send[o:o + c])), p))
        bufs = []
        for p, o, c in zip(peers, offsets, counts):
            b = torch.empty(c, dtype=torch.float64)
            reqs.append(dist.irecv(b, p))
            bufs.append((o, c, b))
        for r in reqs:
            r.wait()
        for o, c, b in bufs:
            recv[o:o + c] = b.numpy()

    def allgather(send, recv):
        out = [torch.empty(send.shape[0], dtype=torch.float64) for _ in range(dist.get_world_size())]
        dist.all_gather(out, torch.from_numpy(np.array(send)))
        recv[:] = torch.cat(out).numpy()

    return exchange, allgather


def _case(P, how):
    import gen
    if how == "lattice":  # un-permuted blocks: uniform ELL widths -> the overlapped fast path
        m = gen.box(8 * P, 8, 6, (float(P), 1.0, 0.75))
        return m, gen.gamma_lognormal(m), gen.rhs(m), gen.block_parts(m, (P, 1, 1))
    m = gen.permute(gen.perturbed(10, 0.2), seed=6)
    gamma, b = gen.gamma_lognormal(m), gen.rhs(m)
    part = gen.rcb_parts(m, P) if how == "rcb" else gen.block_parts(m, (P, 1, 1))
    return m, gamma, b, part


def _worker(rank, P, how, port, results):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import datetime
        dist.init_process_group("gloo", rank=rank, world_size=P, timeout=datetime.timedelta(seconds=120))
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
        me = subs[rank]
        h = S.Mesh.from_mesh(me, rank=rank, n_ranks=P)
        h.set_comm_callbacks(*_callbacks(rank))
        h.set_option(S.spuma.OPT_SMALL_SOLVE_MAX_CELLS, 0)  # the multi-rank batch path
        f64 = dict(dtype=torch.float64, device="cuda")
        diag, upper = torch.empty(me.n_cells, **f64), torch.empty(me.n_faces, **f64)
        src = torch.as_tensor(bs[rank], **f64)
        iface = torch.empty(max(h.n_iface, 1), **f64)
        h.assemble_laplacian(torch.as_tensor(gs[rank], **f64), None, ref_local[rank], 0.0, diag, upper, src, iface)
        s = systems[rank]
        assert np.array_equal(upper.cpu().numpy(), s.upper)
        assert np.array_equal(diag.cpu().numpy(), s.diag)
        assert np.array_equal(src.cpu().numpy(), s.source)
        oi = np.concatenate(s.iface) if s.iface else np.zeros(0)
        assert np.array_equal(iface.cpu().numpy()[:oi.shape[0]], oi)
        # non-orthogonal correction with the p / gamma / gradient halos vs the decomposed oracle
        pfield = np.cos(np.arange(m.n_cells) * 0.29)
        ps = gen.split_cell_field(pfield, part, P)
        p_h = O.gamma_halo(subs, ps)
        Gs = [O.gauss_grad(sm, ps[r], p_remote=p_h[r]) for r, sm in enumerate(subs)]
        G_h = O.gamma_halo(subs, Gs)
        cf_o, pcf_o, ds_o, _ = O.nonorth_correction(me, ps[rank], gs[rank], gamma_remote=halo[rank],
                                                    p_remote=p_h[rank], G=Gs[rank], G_remote=G_h[rank])
        srcc = torch.as_tensor(bs[rank], **f64)
        cf = torch.empty(max(me.n_faces, 1), **f64)
        pcf = [torch.empty(max(pt.n_faces, 1), **f64) for pt in me.patches]
        h.laplacian_correction(torch.as_tensor(gs[rank], **f64), None, torch.as_tensor(ps[rank], **f64),
                               torch.as_tensor(me.V, **f64), srcc, cf, pcf)
        assert np.array_equal(cf.cpu().numpy()[:me.n_faces], cf_o)
        assert np.array_equal(srcc.cpu().numpy(), bs[rank] + ds_o)
        for a, pt, b in zip(pcf, me.patches, pcf_o):
            assert np.array_equal(a.cpu().numpy()[:pt.n_faces], b)
        # Amul with the halo
        x = np.cos(np.arange(m.n_cells) * 0.37)
        xs = gen.split_cell_field(x, part, P)
        y = torch.empty(me.n_cells, **f64)
        h.amul(diag, upper, iface, torch.as_tensor(xs[rank], **f64), y)
        xh = O.gamma_halo(subs, xs)[rank]
        assert np.array_equal(y.cpu().numpy(), O.amul(me, s.diag, s.upper, xs[rank], iface=s.iface, x_remote=xh))
        # PCG vs the decomposed oracle (Q11) and every rank agrees on perf
        psi = torch.zeros(me.n_cells, **f64)
        perf = h.pcg_solve(diag, upper, iface, src, psi, 1e-9, 0.0, 3000, 0)
        psis_o, po = O.pcg_decomposed(subs, systems, None, O.controls(1e-9, 0.0, 3000, 0))
        assert abs(perf["n_iterations"] - po["n_iterations"]) <= 2, (perf, po)
        n = min(perf["n_iterations"], po["n_iterations"])
        psi.zero_()
        perf_n = h.pcg_solve(diag, upper, iface, src, psi, 0.0, 0.0, n, n)
        psis_o, _ = O.pcg_decomposed(subs, systems, None, O.controls(0.0, 0.0, n, n))
        loc = psi.cpu().numpy()
        num = np.array([np.sum((loc - psis_o[rank]) ** 2), np.sum(psis_o[rank] ** 2)])
        tot = [torch.empty(2, dtype=torch.float64) for _ in range(P)]
        dist.all_gather(tot, torch.from_numpy(num))
        err = np.sqrt(sum(t[0].item() for t in tot) / sum(t[1].item() for t in tot))
        assert err <= 1e-9, err
        allp = [None] * P
        dist.all_gather_object(allp, perf)
        assert all(p == allp[0] for p in allp)  # identical decisions on every rank
        # PCG with processor-local DIC / aDILU (Q31) vs the decomposed oracle
        for kind, okind in ((S.spuma.PC_DIC, O.DIC), (S.spuma.PC_ADILU, O.ADILU)):
            psi_k = torch.zeros(me.n_cells, **f64)
            pk = h.pcg_solve_pc(diag, upper, src, psi_k, 1e-9, 0.0, 3000, 0, kind=kind, iface_coeffs=iface)
            pso, pko = O.pcg_decomposed(subs, systems, None, O.controls(1e-9, 0.0, 3000, 0), kind=okind)
            assert abs(pk["n_iterations"] - pko["n_iterations"]) <= 2, (kind, pk, pko)
            nk = min(pk["n_iterations"], pko["n_iterations"])
            psi_k.zero_()
            h.pcg_solve_pc(diag, upper, src, psi_k, 0.0, 0.0, nk, nk, kind=kind, iface_coeffs=iface)
            pso, _ = O.pcg_decomposed(subs, systems, None, O.controls(0.0, 0.0, nk, nk), kind=okind)
            lk = psi_k.cpu().numpy()
            numk = np.array([np.sum((lk - pso[rank]) ** 2), np.sum(pso[rank] ** 2)])
            totk = [torch.empty(2, dtype=torch.float64) for _ in range(P)]
            dist.all_gather(totk, torch.from_numpy(numk))
            errk = np.sqrt(sum(t[0].item() for t in totk) / sum(t[1].item() for t in totk))
            assert errk <= 1e-9, (kind, errk)
        # PBiCG on an asymmetric decomposed system: Amul / Tmul interface coefficients, pA and
        # pT halos, processor-local DILU / aDILU (Q31, Q32) vs the decomposed oracle
        from cases import asym_decomposed
        asubs, asys, _ = asym_decomposed(m, part, seed=7)
        A_ = asys[rank]
        cat = lambda xs: torch.as_tensor(np.concatenate(xs) if xs else np.zeros(1), **f64)
        for kind, okind in ((S.spuma.PC_ADILU, O.ADILU), (S.spuma.PC_DILU, O.DILU)):
            def run_gpu(ctl):
                x = torch.zeros(me.n_cells, **f64)
                pf = h.pbicg_solve(torch.as_tensor(A_["diag"], **f64), torch.as_tensor(A_["upper"], **f64),
                                   torch.as_tensor(A_["lower"], **f64), torch.as_tensor(A_["source"], **f64), x,
                                   *ctl, kind=kind, iface_coeffs=cat(A_["iface"]), iface_coeffs_t=cat(A_["iface_t"]))
                return x.cpu().numpy(), pf
            xg, pg = run_gpu((1e-10, 0.0, 1000, 0))
            xo, po = O.pbicg_decomposed(asubs, asys, None, O.controls(1e-10, 0.0, 1000, 0), okind)
            assert pg["converged"] and abs(pg["n_iterations"] - po["n_iterations"]) <= 2, (kind, pg, po)
            nb = min(pg["n_iterations"], po["n_iterations"])
            xg, _ = run_gpu((0.0, 0.0, nb, nb))
            xo, _ = O.pbicg_decomposed(asubs, asys, None, O.controls(0.0, 0.0, nb, nb), okind)
            numb = np.array([np.sum((xg - xo[rank]) ** 2), np.sum(xo[rank] ** 2)])
            totb = [torch.empty(2, dtype=torch.float64) for _ in range(P)]
            dist.all_gather(totb, torch.from_numpy(numb))
            errb = np.sqrt(sum(t[0].item() for t in totb) / sum(t[1].item() for t in totb))
            assert errb <= 1e-9, (kind, errb)
        # the inline-interface Amul (variant 0: halo before the Amul) gives the same iterates
        h.set_option(S.spuma.OPT_AMUL_VARIANT, 0)
        psi0 = torch.zeros(me.n_cells, **f64)
        p0 = h.pcg_solve(diag, upper, iface, src, psi0, 0.0, 0.0, n, n)
        assert p0["n_iterations"] == n
        assert np.max(np.abs(psi0.cpu().numpy() - loc)) <= 1e-9 * max(np.max(np.abs(loc)), 1e-300)
        h.free()
        results.put((rank, "ok"))
    except BaseException:
        import traceback
        results.put((rank, traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.parametrize("P,how", [(2, "block"), (3, "rcb"), (4, "rcb"), (2, "lattice"), (4, "lattice")])
def test_multirank_on_one_gpu_matches_decomposed_oracle(P, how):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, P, how, port, q)) for r in range(P)]
    for p in ps:
        p.start()
    import queue
    import time
    res, deadline = {}, time.time() + 600
    while len(res) < P and time.time() < deadline:
        try:
            r, msg = q.get(timeout=5)
        except queue.Empty:
            continue
        res[r] = msg
        if msg != "ok":  # a failed rank leaves the others blocked in a collective: stop them
            break
    for p in ps:
        p.join(timeout=5 if len(res) < P else 60)
        if p.is_alive():
            p.terminate()
    bad = {r: m for r, m in res.items() if m != "ok"}
    assert not bad and len(res) == P, (bad, sorted(res))
