#!/usr/bin/env python
"""Small-mesh driver of every libspuma device path, run under compute-sanitizer (memcheck,
racecheck, synccheck, initcheck) by scripts/gpu_sanitize.sh (race detection /
sanitizers).  Exercises: mesh creation (natural + RCM), assembly with gamma, all Amul variants
(incl. the lattice slots), PCG (single-CTA path in shared and global memory, the captured-batch
path with the lattice / ELL rows and every psi deferral mode), the pEqn steps (surfaceIntegrate, flux,
non-orthogonal correction), GAMG (Richardson + two-stage Gauss-Seidel), PCG with DIC / DILU /
aDILU, PBiCG, LDU -> CSR values.  Prints one line per step; exits non-zero on any error."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2512_22215_b200 as P  # noqa: E402
from cases import asym_system  # noqa: E402

S = P.spuma
f64 = dict(dtype=torch.float64, device="cuda")
d = lambda x: torch.as_tensor(np.ascontiguousarray(x), **f64)  # noqa: E731


def step(name):
    print("ok", name, flush=True)


for mname, mesh, ren in (("perturbed8", gen.perturbed(8, 0.2), False), ("permuted7-rcm", gen.permute(gen.perturbed(7, 0.25), seed=3), True),
                         ("cube10", gen.cube(10), False)):
    N, F = mesh.n_cells, mesh.n_faces
    h = P.Mesh.from_mesh(mesh, renumber=ren)
    g, b = gen.gamma_lognormal(mesh), gen.rhs(mesh)
    diag, upper, src = torch.zeros(N, **f64), torch.zeros(F, **f64), d(b)
    h.assemble_laplacian(d(g), None, 0, 0.0, diag, upper, src, None)
    step(f"{mname} assemble")
    x = d(np.cos(np.arange(N) * 0.3))
    for v in S.AMUL_VARIANTS:
        h.set_option(S.OPT_AMUL_VARIANT, v)
        y = torch.zeros(N, **f64)
        h.amul(diag, upper, None, x, y)
    step(f"{mname} amul variants")
    for thr, smem in ((8192, 1), (8192, 0), (0, 1)):
        h.set_option(S.OPT_SMALL_SOLVE_MAX_CELLS, thr)
        h.set_option(S.OPT_SMALL_SMEM, smem)
        for variant, defer in ((12, 2), (10, 1), (10, 0)):  # lattice rows + psi pairs in the direction, ...
            h.set_option(S.OPT_AMUL_VARIANT, variant)
            h.set_option(S.OPT_DEFER_PSI, defer)
            psi = torch.zeros(N, **f64)
            h.pcg_solve(diag, upper, None, src.clone(), psi, 1e-8, 0.0, 2000, 0)
    # the persistent loop (one cooperative launch per solve; TMEM / shared-memory / HBM residency of
    # rA) on both Amul layouts; generous barrier limit (the tools slow every kernel down)
    h.set_option(S.OPT_SMALL_SOLVE_MAX_CELLS, 0)
    h.set_option(S.OPT_DEFER_PSI, 2)
    h.set_option(S.OPT_PEER_POLL_MS, 600000)
    for variant in (12, 10):
        h.set_option(S.OPT_AMUL_VARIANT, variant)
        for mode in (1, 2, 3):
            h.set_option(S.OPT_PERSISTENT, mode)
            psi = torch.zeros(N, **f64)
            h.pcg_solve(diag, upper, None, src.clone(), psi, 1e-8, 0.0, 2000, 0)
    h.set_option(S.OPT_PERSISTENT, 3)
    h.set_option(S.OPT_SMALL_SOLVE_MAX_CELLS, 8192)
    step(f"{mname} pcg (single-CTA in shared / global memory + batches; lattice / ELL rows; psi deferral modes; "
         f"persistent loop modes 1-3)")
    V = d(mesh.V)
    out = torch.zeros(N, **f64)
    phi = d(np.sin(np.arange(F) * 0.1))
    h.surface_integrate(phi, None, V, out)
    flux = torch.zeros(F, **f64)
    h.face_flux(d(g), None, upper, psi, flux=flux)
    src2 = src.clone()
    cf = torch.zeros(F, **f64)
    h.laplacian_correction(d(g), None, psi, V, src2, cf)
    step(f"{mname} surfaceIntegrate / flux / non-orthogonal correction")
    for sm in (S.SMOOTHER_RICHARDSON, S.SMOOTHER_GS2):
        psi = torch.zeros(N, **f64)
        h.gamg_solve(diag, upper, None, src.clone(), psi, 1e-8, 0.0, 100, 0,
                     params=S.gamg_params(smoother=sm, n_cells_in_coarsest_level=4))
    step(f"{mname} gamg")
    for kind in (S.PC_DIC, S.PC_DILU, S.PC_ADILU, S.PC_DIAGONAL):
        psi = torch.zeros(N, **f64)
        h.pcg_solve_pc(diag, upper, src.clone(), psi, 1e-8, 0.0, 2000, 0, kind=kind)
    step(f"{mname} pcg-pc")
    ad, au, al, ab = asym_system(mesh, seed=1)
    for kind in (S.PC_DILU, S.PC_ADILU):
        psi = torch.zeros(N, **f64)
        h.pbicg_solve(d(ad), d(au), d(al), d(ab), psi, 1e-8, 0.0, 500, 0, kind=kind)
    step(f"{mname} pbicg")
    if not ren:  # the CSR map is defined on the caller's numbering (renumber = 0 handles)
        h.ldu_to_csr()
        vals = torch.zeros(N + 2 * F, **f64)
        h.csr_values(d(ad), d(au), d(al), vals)
        step(f"{mname} ldu->csr")
    h.free()
torch.cuda.synchronize()
print("DRIVER DONE", flush=True)
