import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: larger CPU cases")
    config.addinivalue_line("markers", "shared_gpu_ranks: several processes on ONE GPU whose kernels wait on "
                                       "one another (peer transport); opt-in with SPUMA_SHARED_GPU_RANKS=1")


# Ranks whose kernels poll flags another rank's kernel writes must not share one GPU as separate
# processes: nothing guarantees they run at the same time, and on this driver 2 and 4 such ranks
# raised Xid 109 (context-switch timeout, B200_PROFILING.md).  These tests ran green in rounds 1-2
# (profiles/r01m_peer_transport_pytest.log, r02h_peer_fused_pytest.log, r02ab_pytest_gpu.log); they
# now run only on request (a multi-GPU box, or a deliberate single-GPU check).
SHARED_GPU_RANKS = os.environ.get("SPUMA_SHARED_GPU_RANKS") == "1"
shared_gpu_ranks = pytest.mark.skipif(not SHARED_GPU_RANKS,
                                      reason="processes sharing one GPU with kernels that wait on one another "
                                             "(Xid 109 risk); set SPUMA_SHARED_GPU_RANKS=1")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
