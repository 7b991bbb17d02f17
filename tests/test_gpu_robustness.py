"""Robustness of the C-ABI calls (round-2 advisor findings), through the binding on cuda:0:

- a handle created without a stream orders its work after the caller's work on the legacy
  default stream (torch's default): the library's own stream is a blocking stream;
- caller cell arrays that are only 8-byte aligned (a torch slice at an odd offset) are staged,
  not read as double2 (a misaligned double2 access would kill the context);
- min_iter > max_iter runs min_iter iterations, as the oracle's loop (reading Q3) does, for
  PCG, PCG-pc and GAMG, instead of tripping the host-side termination guard;
- a peer-transport poll timeout makes the collective call return SPUMA_ERR_STATE (and the error
  word is cleared), instead of SPUMA_OK with stale halo / partials.
"""
import os

import numpy as np
import pytest

from conftest import shared_gpu_ranks  # noqa: E402

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import gen  # noqa: E402
import oracle as O  # noqa: E402
import paper_2512_22215_b200 as P  # noqa: E402
from gpu_helpers import dev, gpu_assemble  # noqa: E402

F64 = dict(dtype=torch.float64, device="cuda")


def _case(n=24):
    m = gen.cube(n)  # 13824 cells: above the single-CTA limit -> the graph-batched hot loop
    return m, gen.rhs(m)


def test_own_stream_is_ordered_after_default_stream_work():
    m, b = _case()
    h = P.Mesh.from_mesh(m)  # no stream: the handle's own (blocking) stream
    diag, upper, src, _ = gpu_assemble(h, m, None, 0, 0.0, b)
    psi_ref = torch.zeros(m.n_cells, **F64)
    ref = h.pcg_solve(diag, upper, None, src, psi_ref, 1e-8, 0.0, 5000, 0)
    x0h = np.linspace(-1.0, 1.0, m.n_cells)
    x0 = dev(x0h)
    for _ in range(3):
        psi = torch.full((m.n_cells,), 123.0, **F64)
        torch.cuda.synchronize()
        torch.cuda._sleep(200_000_000)  # ~0.1 s of GPU spin on the default stream, then the fill
        psi.zero_()
        perf = h.pcg_solve(diag, upper, None, src, psi, 1e-8, 0.0, 5000, 0)
        assert perf == ref and torch.equal(psi, psi_ref)
        # spuma_amul: the output zeroed and the input written on the default stream before the call
        y = torch.full((m.n_cells,), 7.0, **F64)
        x = torch.empty(m.n_cells, **F64)
        torch.cuda._sleep(200_000_000)
        x.copy_(x0)
        h.amul(diag, upper, None, x, y)
        torch.cuda.synchronize()
        assert np.array_equal(y.cpu().numpy(), O.amul(m, diag.cpu().numpy(), upper.cpu().numpy(), x0h))
    h.free()


def test_unaligned_cell_arrays_are_staged():
    m, b = _case()
    h = P.Mesh.from_mesh(m)
    diag, upper, src, _ = gpu_assemble(h, m, None, 0, 0.0, b)
    psi_a = torch.zeros(m.n_cells, **F64)
    pa = h.pcg_solve(diag, upper, None, src, psi_a, 1e-8, 0.0, 5000, 0)
    # every cell array 8-byte aligned only: slices at offset 1 of a larger buffer
    def odd(t):
        base = torch.zeros(t.numel() + 1, **F64)
        v = base[1:]
        v.copy_(t)
        assert v.data_ptr() % 16 == 8
        return base, v
    _, d_o = odd(diag)
    _, s_o = odd(src)
    _, p_o = odd(torch.zeros(m.n_cells, **F64))
    pb = h.pcg_solve(d_o, upper, None, s_o, p_o, 1e-8, 0.0, 5000, 0)
    assert pb == pa and torch.equal(p_o, psi_a)
    # assembly into unaligned diag / source, Amul into an unaligned y
    _, d2 = odd(torch.zeros(m.n_cells, **F64))
    _, s2 = odd(dev(b))
    u2 = torch.empty(m.n_faces, **F64)
    h.assemble_laplacian(None, None, 0, 0.0, d2, u2, s2, None)
    assert torch.equal(d2, diag) and torch.equal(u2, upper) and torch.equal(s2, src)
    x = dev(np.linspace(-1.0, 1.0, m.n_cells))
    _, x_o = odd(x)
    _, y_o = odd(torch.zeros(m.n_cells, **F64))
    y = torch.zeros(m.n_cells, **F64)
    h.amul(diag, upper, None, x, y)
    h.amul(d_o, upper, None, x_o, y_o)
    torch.cuda.synchronize()
    assert torch.equal(y, y_o)
    h.free()


@pytest.mark.parametrize("solver", ["pcg", "pcg_pc", "gamg"])
def test_min_iter_above_max_iter_runs_min_iter(solver):
    m, b = _case()
    sysm = O.assemble(m, None, 0, 0.0, b)
    h = P.Mesh.from_mesh(m)
    diag, upper, src, _ = gpu_assemble(h, m, None, 0, 0.0, b)
    psi = torch.zeros(m.n_cells, **F64)
    mx, mn = 5, 12
    if solver == "pcg":
        perf = h.pcg_solve(diag, upper, None, src, psi, 1e-6, 0.0, mx, mn)
        psi_o, po = O.pcg(m, sysm, None, O.controls(1e-6, 0.0, mx, mn))
    elif solver == "pcg_pc":
        perf = h.pcg_solve_pc(diag, upper, src, psi, 1e-6, 0.0, mx, mn, kind=P.spuma.PC_DIC)
        psi_o, po = O.pcg_pc(m, sysm, O.DIC, 2, None, O.controls(1e-6, 0.0, mx, mn))
    else:
        perf = h.gamg_solve(diag, upper, None, src, psi, 1e-12, 0.0, mx, mn)
        psi_o, po = O.gamg(m, sysm, None, O.controls(1e-12, 0.0, mx, mn))
    assert po["n_iterations"] == mn
    assert perf["n_iterations"] == mn
    err = np.linalg.norm(psi.cpu().numpy() - psi_o) / np.linalg.norm(psi_o)
    assert err <= 1e-9, err
    h.free()


def _peer_timeout_worker(rank, port, results):
    import datetime

    import torch.distributed as dist
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=2, timeout=datetime.timedelta(seconds=300))
        torch.cuda.set_device(0)
        m = gen.box(16, 8, 6, (2.0, 1.0, 0.75))
        subs = gen.decompose(m, gen.block_parts(m, (2, 1, 1)), 2)
        me = subs[rank]
        h = P.Mesh.from_mesh(me, rank=rank, n_ranks=2)
        h.enable_peer_transport()
        h.set_option(P.spuma.OPT_SMALL_SOLVE_MAX_CELLS, 0)
        h.set_option(P.spuma.OPT_PEER_POLL_MS, 200)
        f64 = F64
        diag, upper = torch.zeros(me.n_cells, **f64), torch.zeros(me.n_faces, **f64)
        src = dev(gen.rhs(me))
        iface = torch.zeros(h.n_iface, **f64)
        h.assemble_laplacian(None, None, 0 if rank == 0 else -1, 0.0, diag, upper, src, iface)
        dist.barrier()
        if rank == 0:  # rank 1 never joins this solve: every poll of rank 0 times out
            psi = torch.zeros(me.n_cells, **f64)
            try:
                h.pcg_solve(diag, upper, iface, src, psi, 1e-6, 0.0, 20, 0)
                results.put((rank, "pcg_solve returned OK although the neighbour never answered"))
                return
            except P.spuma.SpumaError as e:
                if e.status != 7:  # SPUMA_ERR_STATE
                    results.put((rank, f"unexpected status {e.status}: {e}"))
                    return
            h.peer_check()  # the error word was cleared by the failing call
        dist.barrier()
        h.free()
        results.put((rank, "ok"))
    except BaseException:
        import traceback
        results.put((rank, traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@shared_gpu_ranks
def test_peer_poll_timeout_returns_error_state():
    import torch.multiprocessing as mp

    from test_gpu_multirank import _port
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_peer_timeout_worker, args=(r, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = {}
    try:
        for _ in range(2):
            r, msg = q.get(timeout=600)
            out[r] = msg
            if msg != "ok":
                break
    finally:
        for p in ps:
            p.join(timeout=30)
            if p.is_alive():
                p.terminate()
    bad = {r: m for r, m in out.items() if m != "ok"}
    assert not bad and len(out) == 2, bad or out


@pytest.mark.parametrize("name,make", [("cavity20", lambda: gen.cavity2d(20)), ("cube11", lambda: gen.cube(11)),
                                       ("perm-perturbed9", lambda: gen.permute(gen.perturbed(9, 0.3), seed=4)),
                                       ("cube14-too-big", lambda: gen.cube(14))])
def test_small_solve_shared_memory_is_bitwise_global(name, make):
    """SPUMA_OPT_SMALL_SMEM: the single-CTA solve with everything staged in shared memory gives
    bitwise the iterates of the global-memory single-CTA solve (meshes that do not fit fall back)."""
    m = make()
    g, b = gen.gamma_lognormal(m), gen.rhs(m)
    out = []
    for smem in (0, 1):
        h = P.Mesh.from_mesh(m)
        h.set_option(P.spuma.OPT_SMALL_SMEM, smem)
        diag, upper, src, _ = gpu_assemble(h, m, g, 0, 0.0, b)
        psi = torch.zeros(m.n_cells, **F64)
        perf = h.pcg_solve(diag, upper, None, src, psi, 1e-8, 0.0, 5000, 0)
        out.append((psi.cpu().numpy(), perf))
        h.free()
    assert out[0][1] == out[1][1]
    assert np.array_equal(out[0][0].view(np.uint64), out[1][0].view(np.uint64))
