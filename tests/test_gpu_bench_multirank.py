"""The N > 1 path of bench.py (torchrun, one process per rank) on ONE GPU: SPUMA_BENCH_SHARE_GPU=1
puts every rank on cuda:0 with gloo host plumbing, so the weak-scaling workload, the peer-memory
transport, the barriers, the max-over-ranks timing and the JSON line all run as they do on an
8-GPU box (ranks time-slice one GPU, so the value is not a scaling number)."""
import json
import os
import socket
import subprocess
import sys

import pytest

from conftest import shared_gpu_ranks  # noqa: E402

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@shared_gpu_ranks
@pytest.mark.parametrize("world", [2])
def test_bench_n_ranks_peer_transport_on_one_gpu(world):
    env = dict(os.environ, SPUMA_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", str(world), "--steps", "1", "--warmup", "3", "--edge", "16", "--no-e2e"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == world and d["scaling"] == "weak" and d["value"] > 0
    assert d["config"]["transport"].startswith("peer")
    assert d["config"]["global_cells"] == world * 16 ** 3
    assert d["gpu_launches"] > 0
