#!/usr/bin/env python
"""One profiled GAMG solve (cudaProfilerStart/Stop around it) for an ncu launch list:
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/gamg_launches.csv python scripts/gamg_profile.py [n] [cycles]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2512_22215_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
cycles = int(sys.argv[2]) if len(sys.argv) > 2 else 3
m = gen.cube(n)
f64 = dict(dtype=torch.float64, device="cuda")
h = P.Mesh.from_mesh(m, renumber=False, stream=torch.cuda.current_stream().cuda_stream)
diag, upper = torch.empty(m.n_cells, **f64), torch.empty(m.n_faces, **f64)
src = torch.as_tensor(gen.rhs(m), **f64)
h.assemble_laplacian(None, None, 0, 0.0, diag, upper, src, None)
for prof in (False, True):
    psi = torch.zeros(m.n_cells, **f64)
    torch.cuda.synchronize()
    if prof:
        torch.cuda.cudart().cudaProfilerStart()
    perf = h.gamg_solve(diag, upper, None, src.clone(), psi, 0.0, 0.0, cycles, cycles)
    torch.cuda.synchronize()
    if prof:
        torch.cuda.cudart().cudaProfilerStop()
print(perf, h.gamg_hierarchy(with_ftc=False)["cells"])
