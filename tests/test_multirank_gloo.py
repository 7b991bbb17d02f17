"""World-size-2/4 CPU tests (torch.distributed, gloo) of the N > 1 host-side logic.

The GPU path exchanges the processor-patch halo with NCCL send/recv: each rank
packs x[face_cells] of its patch towards rank q in ascending undecomposed face
id (reading Q13) and receives the remote values in the same order.  These tests
run that exact protocol over gloo on the per-rank sub-meshes bench.py builds
(gen.weak_block) and check it against the undecomposed mesh:
- both sides of every cut list the same faces in the same order, with the same
  remote cell centres (bitwise), complementary is_owner flags and negated Sf;
- the decomposed Amul with the exchanged halo equals the undecomposed Amul
  (oracle, PAPER.md P:89/P:536 interface update);
- rank-order sums of all-gathered partials are identical on every rank, so all
  ranks take the same convergence decision.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(rank, world, port, fn, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn(rank, world)
        q.put((rank, "ok"))
    except BaseException as e:  # report to the parent
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def spawn(fn, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_run, args=(r, world, port, fn, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    bad = {r: m for r, m in res.items() if m != "ok"}
    assert not bad, bad


def _halo(mesh, x):
    """Pack x[face_cells] per processor patch, exchange with the neighbour (gloo send/recv)."""
    import gen
    out = []
    reqs = []
    for p in mesh.patches:
        if p.kind != gen.PROCESSOR:
            continue
        send = torch.from_numpy(np.ascontiguousarray(x[p.face_cells]))
        recv = torch.empty(p.n_faces, dtype=torch.float64)
        reqs.append(dist.isend(send, p.neighbour_rank))
        reqs.append(dist.irecv(recv, p.neighbour_rank))
        out.append(recv)
    for r in reqs:
        r.wait()
    return [o.numpy() for o in out]


def _check_blocks(rank, world):
    import gen
    n = 5
    nproc = gen.nproc_for(world)
    m = gen.weak_block(n, nproc, rank)
    assert m.n_cells == n ** 3
    mine = {p.neighbour_rank: p for p in m.patches if p.kind == gen.PROCESSOR}
    alls = [None] * world
    dist.all_gather_object(alls, {q: (p.global_face, p.Sf, p.neighbour_C, p.is_owner, p.neighbour_gid,
                                      m.C[p.face_cells], m.gid[p.face_cells]) for q, p in mine.items()})
    for q, p in mine.items():
        gf, Sf, nC, own, ngid, myC, mygid = alls[q][rank]
        assert np.array_equal(gf, p.global_face)
        assert np.all(np.diff(p.global_face) > 0)
        assert np.array_equal(Sf, -p.Sf)
        assert np.array_equal(nC, m.C[p.face_cells])  # their remote centre == my centre, bitwise
        assert np.array_equal(myC, p.neighbour_C)
        assert np.array_equal(own, 1 - p.is_owner)
        assert np.array_equal(mygid, p.neighbour_gid)


def _check_amul(rank, world):
    import gen
    import oracle as O
    n = 4
    nproc = gen.nproc_for(world)
    g = gen.box(n * nproc[0], n * nproc[1], n * nproc[2], tuple(float(v) for v in nproc))
    gamma_g = np.exp(np.sin(np.arange(g.n_cells) * 0.71))
    x_g = np.cos(np.arange(g.n_cells) * 0.37)
    A = O.assemble(g, gamma_g, -1)
    y_g = O.amul(g, A.diag, A.upper, x_g)
    m = gen.weak_block(n, nproc, rank)
    gamma, x = gamma_g[m.gid], x_g[m.gid]
    s = O.assemble(m, gamma, -1, gamma_remote=_halo(m, gamma))  # gamma halo, as in spuma_assemble_laplacian
    # undecomposed coefficients are reproduced bitwise on the processor faces (Q9)
    for p, c in zip(O.processor_patches(m), s.iface):
        assert np.array_equal(c, A.upper[p.global_face])
    y = O.amul(m, s.diag, s.upper, x, iface=s.iface, x_remote=_halo(m, x))
    assert np.allclose(y, y_g[m.gid], rtol=1e-13, atol=1e-15)


def _check_rank_order_sums(rank, world):
    rng = np.random.default_rng(rank)
    part = torch.from_numpy(rng.standard_normal(4) * 10.0 ** rng.integers(-8, 8, 4))
    gathered = [torch.empty(4, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(gathered, part)
    s = torch.zeros(4, dtype=torch.float64)
    for gpart in gathered:  # rank order, as k_finalize does
        s = s + gpart
    every = [torch.empty(4, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(every, s)
    for e in every:
        assert torch.equal(e, s)  # bitwise identical on all ranks


@pytest.mark.parametrize("world", [2, 4])
def test_weak_blocks_consistent_across_ranks(world):
    spawn(_check_blocks, world)


@pytest.mark.parametrize("world", [2, 4])
def test_decomposed_amul_with_exchanged_halo(world):
    spawn(_check_amul, world)


def test_rank_order_sums_identical_on_all_ranks():
    spawn(_check_rank_order_sums, 2)
