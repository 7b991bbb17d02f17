#!/usr/bin/env python
"""Same-box A/B of SPUMA_OPT_GAMG_CSR (coarse generic levels as CSR runs vs losort-addressed
rows): ms per V-cycle at n^3 (gamma = 1, tol 1e-6) and bitwise identity of psi."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2512_22215_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
perm = len(sys.argv) > 2 and sys.argv[2] == "perm"  # perturbed + permuted, RCM-renumbered (irregular level 0)
m = gen.permute(gen.perturbed(n, 0.15), seed=2) if perm else gen.cube(n)
f64 = dict(dtype=torch.float64, device="cuda")
h = P.Mesh.from_mesh(m, renumber=perm, stream=torch.cuda.current_stream().cuda_stream)
diag, upper = torch.empty(m.n_cells, **f64), torch.empty(m.n_faces, **f64)
src = torch.as_tensor(gen.rhs(m), **f64)
h.assemble_laplacian(None, None, 0, 0.0, diag, upper, src, None)
out = {}
for rnd in range(2):
    for csr in (1, 0):
        h.set_option(P.spuma.OPT_GAMG_CSR, csr)
        psi = torch.zeros(m.n_cells, **f64)
        h.gamg_solve(diag, upper, None, src.clone(), psi, 1e-6, 0.0, 300, 0)  # hierarchy + capture
        best = None
        for _ in range(3):
            psi.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            perf = h.gamg_solve(diag, upper, None, src.clone(), psi, 1e-6, 0.0, 300, 0)
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1)
            best = t if best is None else min(best, t)
        out[csr] = psi.clone()
        print(json.dumps({"n": n, "mesh": "perturbed+permuted, RCM" if perm else "cube", "round": rnd, "gamg_csr": csr, "cycles": perf["n_iterations"],
                          "ms": best, "ms_per_cycle": best / perf["n_iterations"]}), flush=True)
print(json.dumps({"bitwise_same": bool(torch.equal(out[0], out[1]))}))
