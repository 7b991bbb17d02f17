#!/usr/bin/env python
"""One DIC preconditioning (factor + forward + backward sweep) of a 100^3 Laplacian between
cudaProfilerStart/Stop, for ncu captures of the sync-free sweep kernels."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2512_22215_b200 as P  # noqa: E402
from paper_2512_22215_b200 import spuma as S  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
m = gen.cube(n)
f64 = dict(dtype=torch.float64, device="cuda")
h = P.Mesh.from_mesh(m)
diag, upper, src = torch.empty(m.n_cells, **f64), torch.empty(m.n_faces, **f64), torch.as_tensor(gen.rhs(m), **f64)
h.assemble_laplacian(None, None, 0, 0.0, diag, upper, src, None)
w = torch.empty(m.n_cells, **f64)
h.precondition(diag, upper, upper, src, w, S.PC_DIC)  # warm-up (schedules)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
h.precondition(diag, upper, upper, src, w, S.PC_DIC)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok")
