"""Helpers for the -m gpu parity tests: drive libspuma through the binding with torch CUDA tensors."""
import numpy as np
import torch

import paper_2512_22215_b200 as P


def dev(x, dtype=torch.float64):
    return torch.as_tensor(np.ascontiguousarray(x)).to(device="cuda", dtype=dtype).contiguous()


def patch_values(mesh):
    return [None if p.value is None else dev(p.value) for p in mesh.patches]


def n_iface(mesh):
    return sum(p.n_faces for p in mesh.patches if p.kind == P.spuma.PROCESSOR)


def gpu_assemble(h, mesh, gamma=None, ref_cell=-1, ref_value=0.0, source=None):
    N, F = mesh.n_cells, mesh.n_faces
    diag = torch.empty(N, dtype=torch.float64, device="cuda")
    upper = torch.empty(F, dtype=torch.float64, device="cuda")
    src = dev(np.zeros(N) if source is None else source)
    ni = n_iface(mesh)
    iface = torch.empty(max(ni, 1), dtype=torch.float64, device="cuda") if ni else None
    h.assemble_laplacian(None if gamma is None else dev(gamma), patch_values(mesh), ref_cell, ref_value,
                         diag, upper, src, iface)
    torch.cuda.synchronize()
    return diag, upper, src, iface


def gpu_solve_case(mesh, gamma=None, b=None, ref_cell=0, ctl=(1e-6, 0.0, 5000, 0), renumber=False, psi0=None,
                   handle=None):
    h = handle or P.Mesh.from_mesh(mesh, renumber=renumber)
    diag, upper, src, iface = gpu_assemble(h, mesh, gamma, ref_cell, 0.0, b)
    psi = dev(np.zeros(mesh.n_cells) if psi0 is None else psi0)
    perf = h.pcg_solve(diag, upper, iface, src, psi, *ctl)
    return psi.cpu().numpy(), perf, (diag.cpu().numpy(), upper.cpu().numpy(), src.cpu().numpy()), h
