"""CPU oracle for the SPUMA pressure path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product
(``paper_2512_22215_b200``) never imports it and shares no code with it; the
only common dependency is the seeded input module ``gen``.

This is a thin ctypes marshalling layer over ``oracle/oracle.c`` (plain
single-threaded C, fp64, ``-O2 -ffp-contract=off``).  All arithmetic of the
method lives in oracle.c; see its header for the paper citations per function
(O1..O7) and DESIGN.md §3 for the readings.  Parity unpinned: normFactor (Q1)
and loop/convergence semantics (Q2/Q3) are pinned only by special cases.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

import gen

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")
_lock = threading.Lock()
_lib = None

ZERO_GRADIENT, FIXED_VALUE, EMPTY, PROCESSOR = gen.ZERO_GRADIENT, gen.FIXED_VALUE, gen.EMPTY, gen.PROCESSOR


def build(force: bool = False) -> str:
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _SO)
    return _SO


class Controls(ctypes.Structure):
    """SolverControls: tolerance, relTol, maxIter, minIter."""
    _fields_ = [("tolerance", ctypes.c_double), ("rel_tol", ctypes.c_double),
                ("max_iter", ctypes.c_int), ("min_iter", ctypes.c_int)]


class Perf(ctypes.Structure):
    _fields_ = [("initial_residual", ctypes.c_double), ("final_residual", ctypes.c_double),
                ("n_iterations", ctypes.c_int), ("converged", ctypes.c_int), ("singular", ctypes.c_int)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class GamgParams(ctypes.Structure):
    """O11 GAMG parameters (readings Q22-Q28): sweeps, Richardson weight, correction scaling,
    coarsening stop, coarsest-level PCG controls."""
    _fields_ = [("n_pre", ctypes.c_int), ("n_post", ctypes.c_int), ("scale", ctypes.c_int),
                ("n_coarsest_cells", ctypes.c_int), ("max_levels", ctypes.c_int),
                ("omega", ctypes.c_double), ("coarsest_tol", ctypes.c_double),
                ("coarsest_rel_tol", ctypes.c_double), ("coarsest_max_iter", ctypes.c_int),
                ("smoother", ctypes.c_int), ("n_inner", ctypes.c_int)]


RICHARDSON, GS2 = 0, 1


def gamg_params(n_pre=0, n_post=2, scale=True, n_coarsest_cells=10, max_levels=50, omega=0.75,
                coarsest_tol=0.0, coarsest_rel_tol=1e-6, coarsest_max_iter=1000, smoother=RICHARDSON,
                n_inner=1) -> GamgParams:
    return GamgParams(n_pre, n_post, int(scale), n_coarsest_cells, max_levels, omega, coarsest_tol,
                      coarsest_rel_tol, coarsest_max_iter, smoother, n_inner)


class _Domain(ctypes.Structure):
    _fields_ = [("n_cells", ctypes.c_int), ("n_faces", ctypes.c_int),
                ("owner", ctypes.c_void_p), ("neighbour", ctypes.c_void_p),
                ("diag", ctypes.c_void_p), ("upper", ctypes.c_void_p), ("source", ctypes.c_void_p),
                ("psi", ctypes.c_void_p), ("n_iface", ctypes.c_int), ("iface_cells", ctypes.c_void_p),
                ("iface_coeffs", ctypes.c_void_p), ("iface_src_domain", ctypes.c_void_p),
                ("iface_src_cell", ctypes.c_void_p)]


def _L():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_SO)
            vp, ci, cd = ctypes.c_void_p, ctypes.c_int, ctypes.c_double
            lib.or_check_addressing.argtypes = [ci, ci, vp, vp]
            lib.or_check_addressing.restype = ci
            lib.or_owner_start.argtypes = [ci, ci, vp, vp]
            lib.or_losort.argtypes = [ci, ci, vp, vp, vp]
            lib.or_rcm.argtypes = [ci, ci, vp, vp, vp]
            lib.or_rcm.restype = ci
            lib.or_renumber_faces.argtypes = [ci, vp, vp, vp, vp, vp, vp, vp]
            lib.or_geometry.argtypes = [ci] + [vp] * 8
            lib.or_boundary_delta.argtypes = [ci] + [vp] * 6
            lib.or_processor_geometry.argtypes = [ci] + [vp] * 9
            lib.or_assemble.argtypes = [ci, ci] + [vp] * 6 + [ci] + [vp] * 8 + [ci, cd] + [vp] * 4
            lib.or_amul.argtypes = [ci, ci] + [vp] * 6 + [ci] + [vp] * 4
            lib.or_sumA.argtypes = [ci, ci] + [vp] * 5 + [ci] + [vp] * 3
            lib.or_pcg.argtypes = [ci, ctypes.POINTER(_Domain), ctypes.POINTER(Controls), ctypes.POINTER(Perf)]
            lib.or_pcg.restype = ci
            lib.or_surface_integrate.argtypes = [ci, ci, vp, vp, vp, ci] + [vp] * 5
            lib.or_face_flux.argtypes = [ci] + [vp] * 6 + [ci] + [vp] * 11
            lib.or_gauss_grad.argtypes = [ci, ci] + [vp] * 5 + [ci] + [vp] * 9
            lib.or_nonorth_flux.argtypes = [ci] + [vp] * 10 + [ci] + [vp] * 11
            lib.or_agglomerate.argtypes = [ci, ci, vp, vp, vp, vp]
            lib.or_coarse_addressing.argtypes = [ci] + [vp] * 8
            lib.or_agglomerate_matrix.argtypes = [ci, ci] + [vp] * 5 + [ci, ci, vp, vp]
            lib.or_restrict.argtypes = [ci, vp, vp, ci, vp]
            lib.or_gamg.argtypes = [ci, ci] + [vp] * 7 + [ctypes.POINTER(GamgParams), ctypes.POINTER(Controls),
                                                           ctypes.POINTER(Perf), vp, vp]
            lib.or_gamg_dd.argtypes = [ci, ctypes.POINTER(_Domain), vp, ctypes.POINTER(GamgParams),
                                       ctypes.POINTER(Controls), ctypes.POINTER(Perf), vp, vp, vp]
            lib.or_gamg_dd.restype = ci
            lib.or_gamg_dd_dense_level.argtypes = [ci, ctypes.POINTER(_Domain), vp, ctypes.POINTER(GamgParams),
                                                   ci, ci, vp, vp]
            lib.or_gamg_dd_dense_level.restype = ci
            lib.or_pcg_dd_pc.argtypes = [ci, ctypes.POINTER(_Domain), ctypes.POINTER(Controls), ci, ci,
                                         ctypes.POINTER(Perf)]
            lib.or_pbicg_dd.argtypes = [ci, ctypes.POINTER(_Domain), vp, vp, ctypes.POINTER(Controls), ci, ci,
                                        ctypes.POINTER(Perf)]
            lib.or_ilu_factor.argtypes = [ci, ci] + [vp] * 6
            lib.or_ilu_precondition.argtypes = [ci, ci] + [vp] * 7 + [ci, ci]
            lib.or_pcg_pc.argtypes = [ci, ci] + [vp] * 6 + [ctypes.POINTER(Controls), ci, ci, ctypes.POINTER(Perf)]
            lib.or_pbicg.argtypes = [ci, ci] + [vp] * 7 + [ctypes.POINTER(Controls), ci, ci, ctypes.POINTER(Perf)]
            lib.or_tmul.argtypes = [ci, ci] + [vp] * 7
            lib.or_ldu_to_csr.argtypes = [ci, ci] + [vp] * 5
            lib.or_dense_from_ldu.argtypes = [ci, ci] + [vp] * 6
            lib.or_dense_matvec.argtypes = [ci, vp, vp, vp]
            lib.or_dense_solve.argtypes = [ci, vp, vp, vp]
            lib.or_dense_solve.restype = ci
            _lib = lib
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# --------------------------------------------------------------------------- O1
def check_addressing(n_cells: int, owner, neighbour) -> int:
    owner, neighbour = _i32(owner), _i32(neighbour)
    return _L().or_check_addressing(n_cells, owner.shape[0], _p(owner), _p(neighbour))


def owner_start(n_cells: int, owner) -> np.ndarray:
    owner = _i32(owner)
    out = np.empty(n_cells + 1, np.int32)
    _L().or_owner_start(n_cells, owner.shape[0], _p(owner), _p(out))
    return out


def losort(n_cells: int, neighbour):
    neighbour = _i32(neighbour)
    lo = np.empty(neighbour.shape[0], np.int32)
    ls = np.empty(n_cells + 1, np.int32)
    _L().or_losort(n_cells, neighbour.shape[0], _p(neighbour), _p(lo), _p(ls))
    return lo, ls


# --------------------------------------------------------------------------- O2
def rcm(n_cells: int, owner, neighbour) -> np.ndarray:
    owner, neighbour = _i32(owner), _i32(neighbour)
    perm = np.empty(n_cells, np.int32)
    if _L().or_rcm(n_cells, owner.shape[0], _p(owner), _p(neighbour), _p(perm)):
        raise MemoryError("or_rcm")
    return perm


def renumber_faces(perm, owner, neighbour):
    perm, owner, neighbour = _i32(perm), _i32(owner), _i32(neighbour)
    F = owner.shape[0]
    o, n, fm = np.empty(F, np.int32), np.empty(F, np.int32), np.empty(F, np.int32)
    fl = np.empty(F, np.int8)
    _L().or_renumber_faces(F, _p(perm), _p(owner), _p(neighbour), _p(o), _p(n), _p(fm), _p(fl))
    return o, n, fm, fl


def renumber_mesh(mesh: gen.Mesh, perm) -> gen.Mesh:
    """Apply O2's face re-keying to a whole mesh (cells moved by perm[old] = new)."""
    o, n, fm, fl = renumber_faces(perm, mesh.owner, mesh.neighbour)
    sgn = np.where(fl.astype(bool), -1.0, 1.0)[:, None]
    inv = np.empty(mesh.n_cells, np.int64)
    inv[perm] = np.arange(mesh.n_cells)
    from dataclasses import replace
    patches = [replace(p, face_cells=_i32(np.asarray(perm)[p.face_cells])) for p in mesh.patches]
    return gen.Mesh(mesh.n_cells, o, n, np.ascontiguousarray(mesh.Sf[fm] * sgn), mesh.magSf[fm].copy(),
                    mesh.Cf[fm].copy(), mesh.C[inv].copy(), mesh.V[inv].copy(), patches,
                    gid=None if mesh.gid is None else mesh.gid[inv].copy(),
                    gface=None if mesh.gface is None else mesh.gface[fm].copy(), dims=mesh.dims)


# --------------------------------------------------------------------------- O3
@dataclass
class Geometry:
    delta: np.ndarray  # [F]
    weights: np.ndarray  # [F]
    bdelta: np.ndarray  # [Fb] concatenated over patches (processor: global orientation)
    bweight: np.ndarray  # [Fb] processor faces only (else 0)


def geometry(mesh: gen.Mesh) -> Geometry:
    lib = _L()
    F = mesh.n_faces
    delta, w = np.empty(F), np.empty(F)
    Sf, magSf, C, Cf = _f64(mesh.Sf), _f64(mesh.magSf), _f64(mesh.C), _f64(mesh.Cf)
    own, nbr = _i32(mesh.owner), _i32(mesh.neighbour)
    lib.or_geometry(F, _p(own), _p(nbr), _p(Sf), _p(magSf), _p(C), _p(Cf), _p(delta), _p(w))
    bd, bw = [], []
    for p in mesh.patches:
        n = p.n_faces
        d, ww = np.zeros(n), np.zeros(n)
        fc, pS, pm, pC = _i32(p.face_cells), _f64(p.Sf), _f64(p.magSf), _f64(p.Cf)
        if p.kind == PROCESSOR:
            nC, io = _f64(p.neighbour_C), np.ascontiguousarray(p.is_owner, dtype=np.int8)
            lib.or_processor_geometry(n, _p(fc), _p(pS), _p(pm), _p(pC), _p(C), _p(nC), _p(io), _p(d), _p(ww))
        elif p.kind != EMPTY:
            lib.or_boundary_delta(n, _p(fc), _p(pS), _p(pm), _p(pC), _p(C), _p(d))
        bd.append(d)
        bw.append(ww)
    cat = lambda xs: np.concatenate(xs) if xs else np.zeros(0)
    return Geometry(delta, w, cat(bd), cat(bw))


# --------------------------------------------------------------------------- O4
@dataclass
class LduSystem:
    diag: np.ndarray
    upper: np.ndarray  # lower == upper
    source: np.ndarray
    iface: List[np.ndarray]  # per processor patch (patch order), true entries A[P][remote]


def _bcat(mesh, attr, dtype, default=0):
    xs = []
    for p in mesh.patches:
        v = getattr(p, attr) if not callable(attr) else attr(p)
        xs.append(np.full(p.n_faces, default, dtype) if v is None else np.asarray(v, dtype))
    return np.ascontiguousarray(np.concatenate(xs) if xs else np.zeros(0, dtype), dtype=dtype)


def assemble(mesh: gen.Mesh, gamma=None, ref_cell: int = -1, ref_value: float = 0.0, source=None,
             geo: Optional[Geometry] = None, gamma_remote: Optional[Sequence[np.ndarray]] = None) -> LduSystem:
    """fvm::laplacian(gamma, p) + setReference + boundary coefficients (O4).

    gamma_remote: per processor patch, gamma of the remote cells (the gamma halo)."""
    lib = _L()
    geo = geo or geometry(mesh)
    N, F = mesh.n_cells, mesh.n_faces
    diag, upper = np.empty(N), np.empty(F)
    src = np.zeros(N) if source is None else _f64(source).copy()
    bkind = _i32(np.concatenate([np.full(p.n_faces, p.kind, np.int32) for p in mesh.patches]) if mesh.patches else np.zeros(0))
    bcells = _bcat(mesh, "face_cells", np.int32)
    bmag = _bcat(mesh, "magSf", np.float64)
    bval = _bcat(mesh, "value", np.float64)
    bown = _bcat(mesh, "is_owner", np.int8)
    gr = []
    k = 0
    for p in mesh.patches:
        if p.kind == PROCESSOR and gamma_remote is not None:
            gr.append(np.asarray(gamma_remote[k], np.float64))
            k += 1
        else:
            gr.append(np.zeros(p.n_faces))
    bgr = _f64(np.concatenate(gr) if gr else np.zeros(0))
    iface_all = np.zeros(bkind.shape[0])
    g = None if gamma is None else _f64(gamma)
    own, nbr, mag = _i32(mesh.owner), _i32(mesh.neighbour), _f64(mesh.magSf)
    lib.or_assemble(N, F, _p(own), _p(nbr), _p(mag), _p(geo.delta),
                    _p(geo.weights), _p(g), bkind.shape[0], _p(bkind), _p(bcells), _p(bmag), _p(geo.bdelta),
                    _p(geo.bweight), _p(bval), _p(bgr), _p(bown), int(ref_cell), float(ref_value),
                    _p(diag), _p(upper), _p(src), _p(iface_all))
    iface, off = [], 0
    for p in mesh.patches:
        if p.kind == PROCESSOR:
            iface.append(iface_all[off:off + p.n_faces].copy())
        off += p.n_faces
    return LduSystem(diag, upper, src, iface)


def processor_patches(mesh: gen.Mesh):
    return [p for p in mesh.patches if p.kind == PROCESSOR]


# --------------------------------------------------------------------------- O5
def amul(mesh: gen.Mesh, diag, upper, x, lower=None, iface=None, x_remote=None) -> np.ndarray:
    lib = _L()
    N = mesh.n_cells
    y = np.empty(N)
    lower = upper if lower is None else lower
    ic, ico, xr = _iface_arrays(mesh, iface, x_remote)
    a = [_i32(mesh.owner), _i32(mesh.neighbour), _f64(diag), _f64(lower), _f64(upper), _f64(x)]
    lib.or_amul(N, mesh.n_faces, *[_p(v) for v in a], ic.shape[0], _p(ic), _p(ico), _p(xr), _p(y))
    return y


def sumA(mesh: gen.Mesh, diag, upper, lower=None, iface=None) -> np.ndarray:
    lib = _L()
    y = np.empty(mesh.n_cells)
    lower = upper if lower is None else lower
    ic, ico, _ = _iface_arrays(mesh, iface, None)
    a = [_i32(mesh.owner), _i32(mesh.neighbour), _f64(diag), _f64(lower), _f64(upper)]
    lib.or_sumA(mesh.n_cells, mesh.n_faces, *[_p(v) for v in a], ic.shape[0], _p(ic), _p(ico), _p(y))
    return y


def _iface_arrays(mesh, iface, x_remote):
    pp = processor_patches(mesh)
    if not pp or iface is None:
        return np.zeros(0, np.int32), np.zeros(0), np.zeros(0)
    ic = _i32(np.concatenate([p.face_cells for p in pp]))
    ico = _f64(np.concatenate(iface))
    xr = np.zeros(ic.shape[0]) if x_remote is None else _f64(np.concatenate(x_remote))
    return ic, ico, xr


# --------------------------------------------------------------------------- O6 / O8
def controls(tolerance=1e-6, rel_tol=0.0, max_iter=5000, min_iter=0) -> Controls:
    return Controls(tolerance, rel_tol, max_iter, min_iter)


def pcg(mesh: gen.Mesh, sys: LduSystem, psi0=None, ctl: Optional[Controls] = None):
    """Single-domain PCG + diagonal preconditioner. Returns (psi, perf dict)."""
    psi, perf = pcg_decomposed([mesh], [sys], None if psi0 is None else [psi0], ctl)
    return psi[0], perf


def _domains(meshes: Sequence[gen.Mesh], systems, psi0=None):
    """The O8 domain table: per domain its LDU system, psi (copied), and the interface
    sources (domain, local cell) of its processor faces in (patch, face) order."""
    P = len(meshes)
    keep = []
    doms = (_Domain * P)()
    psis = []
    lut = {}
    if P > 1:
        for r, m in enumerate(meshes):
            for loc, g in enumerate(m.gid):
                lut[int(g)] = (r, loc)
    for r, (m, s) in enumerate(zip(meshes, systems)):
        psi = np.zeros(m.n_cells) if psi0 is None else _f64(psi0[r]).copy()
        psis.append(psi)
        pp = processor_patches(m)
        if pp:
            ic = _i32(np.concatenate([p.face_cells for p in pp]))
            ico = _f64(np.concatenate(s.iface))
            src = [lut[int(g)] for p in pp for g in p.neighbour_gid]
            sd = _i32([a for a, _ in src])
            sc = _i32([b for _, b in src])
        else:
            ic, ico, sd, sc = np.zeros(0, np.int32), np.zeros(0), np.zeros(0, np.int32), np.zeros(0, np.int32)
        arrs = [_i32(m.owner), _i32(m.neighbour), _f64(s.diag), _f64(s.upper), _f64(s.source), ic, ico, sd, sc]
        keep.append(arrs)
        d = doms[r]
        d.n_cells, d.n_faces = m.n_cells, m.n_faces
        d.owner, d.neighbour, d.diag, d.upper, d.source = [_p(a) for a in arrs[:5]]
        d.psi = _p(psi)
        d.n_iface = ic.shape[0]
        d.iface_cells, d.iface_coeffs, d.iface_src_domain, d.iface_src_cell = [_p(a) for a in arrs[5:]]
    return doms, psis, keep


def pcg_decomposed(meshes: Sequence[gen.Mesh], systems: Sequence[LduSystem], psi0=None,
                   ctl: Optional[Controls] = None, kind: int = 0, k: int = 2):
    """O8: PCG over P sub-domains run sequentially; x_remote copied between
    domains before every Amul; global sums in rank order.  kind != 0: the O12 preconditioner
    applied per domain on its own faces (processor-local, Q31)."""
    ctl = ctl or controls()
    P = len(meshes)
    doms, psis, keep = _domains(meshes, systems, psi0)
    perf = Perf()
    if kind:
        rc = _L().or_pcg_dd_pc(P, doms, ctypes.byref(ctl), int(kind), int(k), ctypes.byref(perf))
    else:
        rc = _L().or_pcg(P, doms, ctypes.byref(ctl), ctypes.byref(perf))
    if rc:
        raise MemoryError("or_pcg")
    return psis, perf.as_dict()


def _weights(meshes, weights):
    ws = [_f64(m.magSf if weights is None else weights[r]) for r, m in enumerate(meshes)]
    tab = (ctypes.c_void_p * len(ws))(*[_p(w) for w in ws])
    return ws, tab


def gamg_decomposed(meshes: Sequence[gen.Mesh], systems: Sequence[LduSystem], psi0=None,
                    ctl: Optional[Controls] = None, params: Optional[GamgParams] = None, weights=None):
    """O11dd: GAMG over P sub-domains (readings Q36-Q38): processor-local agglomeration,
    coarse interfaces by first occurrence, decomposed Amul / sums on every level, decomposed
    PCG on the coarsest level.  Returns (psis, perf dict incl. 'levels', 'level_cells'
    [[per level] per domain], 'level_ifaces')."""
    ctl = ctl or controls()
    gp = params or gamg_params()
    P = len(meshes)
    doms, psis, keep = _domains(meshes, systems, psi0)
    ws, tab = _weights(meshes, weights)
    nl = ctypes.c_int(0)
    cells = np.zeros(64 * P, np.int32)
    ifs = np.zeros(64 * P, np.int32)
    perf = Perf()
    rc = _L().or_gamg_dd(P, doms, ctypes.addressof(tab), ctypes.byref(gp), ctypes.byref(ctl), ctypes.byref(perf),
                         ctypes.addressof(nl), _p(cells), _p(ifs))
    if rc:
        raise ValueError("or_gamg_dd")
    out = perf.as_dict()
    out["levels"] = nl.value
    out["level_cells"] = [cells[64 * r:64 * r + nl.value].tolist() for r in range(P)]
    out["level_ifaces"] = [ifs[64 * r:64 * r + nl.value].tolist() for r in range(P)]
    return psis, out


def gamg_dd_dense_level(meshes: Sequence[gen.Mesh], systems: Sequence[LduSystem], level: int,
                        params: Optional[GamgParams] = None, weights=None, cap: int = 2048):
    """O11dd: the global operator of one level of the decomposed hierarchy (dense, cells
    domain-major) and the global fine-to-coarse map into it (level > 0), for the Galerkin pin."""
    gp = params or gamg_params()
    P = len(meshes)
    doms, _, keep = _domains(meshes, systems)
    ws, tab = _weights(meshes, weights)
    A = np.zeros(cap * cap)
    nfine = sum(m.n_cells for m in meshes)
    ftc = np.zeros(nfine + 1, np.int32)
    n = _L().or_gamg_dd_dense_level(P, doms, ctypes.addressof(tab), ctypes.byref(gp), int(level), int(cap),
                                    _p(A), _p(ftc))
    if n < 0:
        raise ValueError("no such level or capacity too small")
    return A[:n * n].reshape(n, n).copy(), ftc


def agglomerate(n_cells: int, owner, neighbour, weights):
    """O11 pairwise agglomeration (Q22). Returns (fine_to_coarse int32, n_coarse)."""
    o, nb, w = _i32(owner), _i32(neighbour), _f64(weights)
    ftc = np.zeros(n_cells + 1, np.int32)
    nc = _L().or_agglomerate(n_cells, o.shape[0], _p(o), _p(nb), _p(w), _p(ftc))
    return ftc[:n_cells], nc


def coarse_addressing(owner, neighbour, ftc, weights):
    """O11 coarse lduAddressing: (c_owner, c_neighbour, face_restrict, c_weights)."""
    o, nb, f, w = _i32(owner), _i32(neighbour), _i32(ftc), _f64(weights)
    F = o.shape[0]
    co, cn, fr = (np.zeros(F + 1, np.int32) for _ in range(3))
    cw = np.zeros(F + 1)
    ncf = _L().or_coarse_addressing(F, _p(o), _p(nb), _p(f), _p(w), _p(co), _p(cn), _p(fr), _p(cw))
    return co[:ncf], cn[:ncf], fr[:F], cw[:ncf]


def agglomerate_matrix(owner, ftc, face_restrict, diag, upper, n_coarse: int, n_coarse_faces: int):
    """O11 Galerkin coarse LDU: (c_diag, c_upper)."""
    o, f, fr, d, u = _i32(owner), _i32(ftc), _i32(face_restrict), _f64(diag), _f64(upper)
    cd, cu = np.zeros(n_coarse + 1), np.zeros(n_coarse_faces + 1)
    _L().or_agglomerate_matrix(d.shape[0], o.shape[0], _p(o), _p(f), _p(fr), _p(d), _p(u), n_coarse,
                               n_coarse_faces, _p(cd), _p(cu))
    return cd[:n_coarse], cu[:n_coarse_faces]


def restrict_field(ftc, fine, n_coarse: int):
    f, x = _i32(ftc), _f64(fine)
    out = np.zeros(n_coarse + 1)
    _L().or_restrict(x.shape[0], _p(f), _p(x), n_coarse, _p(out))
    return out[:n_coarse]


def gamg_hierarchy(mesh: gen.Mesh, params: Optional[GamgParams] = None, weights=None):
    """The level list [(n_cells, owner, neighbour, ftc-or-None)] built by the O11 rules (weights:
    face areas, faceAreaPair)."""
    gp = params or gamg_params()
    lv = []
    o, nb = _i32(mesh.owner), _i32(mesh.neighbour)
    w = _f64(mesh.magSf if weights is None else weights)
    n = mesh.n_cells
    while len(lv) + 1 < gp.max_levels and n > gp.n_coarsest_cells:
        ftc, nc = agglomerate(n, o, nb, w)
        if nc >= n:
            break
        lv.append((n, o, nb, ftc))
        o, nb, _, w = coarse_addressing(o, nb, ftc, w)
        n = nc
    lv.append((n, o, nb, None))
    return lv


def gamg(mesh: gen.Mesh, sys: LduSystem, psi0=None, ctl: Optional[Controls] = None,
         params: Optional[GamgParams] = None, weights=None):
    """O11 GAMG + Richardson smoother, single domain. Returns (psi, perf dict incl. 'levels',
    'level_cells')."""
    ctl = ctl or controls()
    gp = params or gamg_params()
    if processor_patches(mesh):
        raise ValueError("oracle GAMG is single-domain (DESIGN.md Q28)")
    o, nb, w = _i32(mesh.owner), _i32(mesh.neighbour), _f64(mesh.magSf if weights is None else weights)
    d, u, b = _f64(sys.diag), _f64(sys.upper), _f64(sys.source)
    psi = np.zeros(mesh.n_cells) if psi0 is None else _f64(psi0).copy()
    nl = ctypes.c_int(0)
    cells = np.zeros(64, np.int32)
    perf = Perf()
    _L().or_gamg(mesh.n_cells, mesh.n_faces, _p(o), _p(nb), _p(w), _p(d), _p(u), _p(b), _p(psi),
                 ctypes.byref(gp), ctypes.byref(ctl), ctypes.byref(perf), ctypes.addressof(nl), _p(cells))
    out = perf.as_dict()
    out["levels"] = nl.value
    out["level_cells"] = cells[:nl.value].tolist()
    return psi, out


# O12 preconditioner kinds (readings Q31-Q33)
DIAGONAL, DIC, DILU, ADILU = 0, 1, 2, 3


def ilu_factor(owner, neighbour, diag, upper, lower=None) -> np.ndarray:
    """[OF] DIC / DILU reciprocal diagonal (lower None: DIC, lower = upper)."""
    o, nb, d, u = _i32(owner), _i32(neighbour), _f64(diag), _f64(upper)
    lo = u if lower is None else _f64(lower)
    rD = np.zeros(d.shape[0] + 1)
    _L().or_ilu_factor(d.shape[0], o.shape[0], _p(o), _p(nb), _p(d), _p(u), _p(lo), _p(rD))
    return rD[:d.shape[0]]


def ilu_precondition(owner, neighbour, rD, upper, r, lower=None, transpose=False, k=-1) -> np.ndarray:
    """[OF] DIC/DILU precondition(T); k >= 0: aDILU with k Jacobi-style passes per sweep (Q33)."""
    o, nb, d, u, x = _i32(owner), _i32(neighbour), _f64(rD), _f64(upper), _f64(r)
    lo = u if lower is None else _f64(lower)
    w = np.zeros(d.shape[0] + 1)
    _L().or_ilu_precondition(d.shape[0], o.shape[0], _p(o), _p(nb), _p(d), _p(u), _p(lo), _p(x), _p(w),
                             int(transpose), int(k))
    return w[:d.shape[0]]


def pcg_pc(mesh: gen.Mesh, sys: LduSystem, kind=DIAGONAL, k=2, psi0=None, ctl: Optional[Controls] = None):
    """PCG with a diagonal / DIC / DILU / aDILU preconditioner, single domain (O12)."""
    ctl = ctl or controls()
    o, nb, d, u, b = _i32(mesh.owner), _i32(mesh.neighbour), _f64(sys.diag), _f64(sys.upper), _f64(sys.source)
    psi = np.zeros(mesh.n_cells) if psi0 is None else _f64(psi0).copy()
    perf = Perf()
    _L().or_pcg_pc(mesh.n_cells, mesh.n_faces, _p(o), _p(nb), _p(d), _p(u), _p(b), _p(psi), ctypes.byref(ctl),
                   int(kind), int(k), ctypes.byref(perf))
    return psi, perf.as_dict()


def pbicg(owner, neighbour, diag, upper, lower, source, kind=DILU, k=2, psi0=None,
          ctl: Optional[Controls] = None):
    """[OF] PBiCG (O12, Q32) on an asymmetric LDU system."""
    ctl = ctl or controls()
    o, nb, d, u, lo, b = (_i32(owner), _i32(neighbour), _f64(diag), _f64(upper), _f64(lower), _f64(source))
    psi = np.zeros(d.shape[0]) if psi0 is None else _f64(psi0).copy()
    perf = Perf()
    _L().or_pbicg(d.shape[0], o.shape[0], _p(o), _p(nb), _p(d), _p(u), _p(lo), _p(b), _p(psi), ctypes.byref(ctl),
                  int(kind), int(k), ctypes.byref(perf))
    return psi, perf.as_dict()


def pbicg_decomposed(meshes: Sequence[gen.Mesh], systems: Sequence[dict], psi0=None,
                     ctl: Optional[Controls] = None, kind: int = 3, k: int = 2):
    """O8 + O12: PBiCG over P sub-domains.  systems[r]: dict(diag, upper, lower, source, iface,
    iface_t) with iface / iface_t per processor patch (the Amul / Tmul coefficients, Q32)."""
    ctl = ctl or controls()
    P = len(meshes)
    keep, doms, psis = [], (_Domain * P)(), []
    lut = {}
    if P > 1:
        for r, m in enumerate(meshes):
            for loc, g in enumerate(m.gid):
                lut[int(g)] = (r, loc)
    lowers = (ctypes.c_void_p * P)()
    ifts = (ctypes.c_void_p * P)()
    for r, (m, s) in enumerate(zip(meshes, systems)):
        psi = np.zeros(m.n_cells) if psi0 is None else _f64(psi0[r]).copy()
        psis.append(psi)
        pp = processor_patches(m)
        if pp:
            ic = _i32(np.concatenate([p.face_cells for p in pp]))
            ico = _f64(np.concatenate(s["iface"]))
            ict = _f64(np.concatenate(s["iface_t"]))
            src = [lut[int(g)] for p in pp for g in p.neighbour_gid]
            sd, sc = _i32([a for a, _ in src]), _i32([b for _, b in src])
        else:
            ic, ico, ict = np.zeros(0, np.int32), np.zeros(0), np.zeros(0)
            sd, sc = np.zeros(0, np.int32), np.zeros(0, np.int32)
        arrs = [_i32(m.owner), _i32(m.neighbour), _f64(s["diag"]), _f64(s["upper"]), _f64(s["source"]), ic, ico, sd,
                sc, _f64(s["lower"]), ict]
        keep.append(arrs)
        d = doms[r]
        d.n_cells, d.n_faces = m.n_cells, m.n_faces
        d.owner, d.neighbour, d.diag, d.upper, d.source = [_p(a) for a in arrs[:5]]
        d.psi = _p(psi)
        d.n_iface = ic.shape[0]
        d.iface_cells, d.iface_coeffs, d.iface_src_domain, d.iface_src_cell = [_p(a) for a in arrs[5:9]]
        lowers[r] = _p(arrs[9])
        ifts[r] = _p(arrs[10])
    perf = Perf()
    _L().or_pbicg_dd(P, doms, ctypes.addressof(lowers), ctypes.addressof(ifts), ctypes.byref(ctl), int(kind), int(k),
                     ctypes.byref(perf))
    return psis, perf.as_dict()


def tmul(owner, neighbour, diag, upper, lower, x) -> np.ndarray:
    o, nb, d, u, lo, xx = _i32(owner), _i32(neighbour), _f64(diag), _f64(upper), _f64(lower), _f64(x)
    y = np.zeros(d.shape[0] + 1)
    _L().or_tmul(d.shape[0], o.shape[0], _p(o), _p(nb), _p(d), _p(u), _p(lo), _p(xx), _p(y))
    return y[:d.shape[0]]


def amul_asym(owner, neighbour, diag, upper, lower, x) -> np.ndarray:
    """y = A x for lower != upper (row owner: upper, row neighbour: lower)."""
    o, nb, d, u, lo, xx = _i32(owner), _i32(neighbour), _f64(diag), _f64(upper), _f64(lower), _f64(x)
    y = np.zeros(d.shape[0] + 1)
    _L().or_amul(d.shape[0], o.shape[0], _p(o), _p(nb), _p(d), _p(lo), _p(u), _p(xx), 0, None, None, None, _p(y))
    return y[:d.shape[0]]


def ldu_to_csr(n_cells: int, owner, neighbour):
    """O12 LDU -> CSR: (row_ptr, col, map) with map into [diag | upper | lower] (Q34)."""
    o, nb = _i32(owner), _i32(neighbour)
    F = o.shape[0]
    nnz = n_cells + 2 * F
    rp, col, mp = np.zeros(n_cells + 1, np.int32), np.zeros(nnz + 1, np.int32), np.zeros(nnz + 1, np.int32)
    _L().or_ldu_to_csr(n_cells, F, _p(o), _p(nb), _p(rp), _p(col), _p(mp))
    return rp, col[:nnz], mp[:nnz]


def gamma_halo(meshes: Sequence[gen.Mesh], gammas: Sequence[np.ndarray]):
    """Per domain, per processor patch: gamma of the remote cells (test plumbing)."""
    lut = {}
    for r, m in enumerate(meshes):
        for loc, g in enumerate(m.gid):
            lut[int(g)] = (r, loc)
    out = []
    for m in meshes:
        out.append([np.array([gammas[lut[int(g)][0]][lut[int(g)][1]] for g in p.neighbour_gid])
                    for p in processor_patches(m)])
    return out


# --------------------------------------------------------------------------- O9
def _patch_field(mesh, values):
    """Concatenate per-patch face values (None -> zeros) in patch order."""
    xs = []
    for i, p in enumerate(mesh.patches):
        v = None if values is None else values[i]
        xs.append(np.zeros(p.n_faces) if v is None else np.asarray(v, np.float64))
    return _f64(np.concatenate(xs) if xs else np.zeros(0))


def surface_integrate(mesh: gen.Mesh, phi, patch_phi=None, V=None) -> np.ndarray:
    """fvc::surfaceIntegrate(phi): per cell (sum of outward fluxes) / V."""
    lib = _L()
    out = np.empty(mesh.n_cells)
    own, nbr, ph = _i32(mesh.owner), _i32(mesh.neighbour), _f64(phi)
    bkind = _i32(np.concatenate([np.full(p.n_faces, p.kind, np.int32) for p in mesh.patches]) if mesh.patches else np.zeros(0))
    bcells = _bcat(mesh, "face_cells", np.int32)
    bphi = _patch_field(mesh, patch_phi)
    Vv = _f64(mesh.V if V is None else V)
    lib.or_surface_integrate(mesh.n_cells, mesh.n_faces, _p(own), _p(nbr), _p(ph), bkind.shape[0], _p(bkind),
                             _p(bcells), _p(bphi), _p(Vv), _p(out))
    return out


def face_flux(mesh: gen.Mesh, upper, psi, gamma=None, geo: Optional[Geometry] = None, gamma_remote=None,
              psi_remote=None, lower=None):
    """fvMatrix::flux of fvm::laplacian(gamma, psi) (lduMatrix::faceH) with the
    boundary contributions. Returns (internal flux [F], list of per-patch flux arrays)."""
    lib = _L()
    geo = geo or geometry(mesh)
    lower = upper if lower is None else lower
    F = mesh.n_faces
    flux = np.empty(F)
    bkind = _i32(np.concatenate([np.full(p.n_faces, p.kind, np.int32) for p in mesh.patches]) if mesh.patches else np.zeros(0))
    bcells = _bcat(mesh, "face_cells", np.int32)
    bmag = _bcat(mesh, "magSf", np.float64)
    bval = _bcat(mesh, "value", np.float64)
    bown = _bcat(mesh, "is_owner", np.int8)

    def proc_field(vals):
        xs, k = [], 0
        for p in mesh.patches:
            if p.kind == PROCESSOR and vals is not None:
                xs.append(np.asarray(vals[k], np.float64))
                k += 1
            else:
                xs.append(np.zeros(p.n_faces))
        return _f64(np.concatenate(xs) if xs else np.zeros(0))

    bgr, bpr = proc_field(gamma_remote), proc_field(psi_remote)
    bflux = np.zeros(bkind.shape[0])
    own, nbr, lo, up, ps = _i32(mesh.owner), _i32(mesh.neighbour), _f64(lower), _f64(upper), _f64(psi)
    g = None if gamma is None else _f64(gamma)
    lib.or_face_flux(F, _p(own), _p(nbr), _p(lo), _p(up), _p(ps), _p(flux), bkind.shape[0], _p(bkind), _p(bcells),
                     _p(bmag), _p(geo.bdelta), _p(geo.bweight), _p(bval), _p(bgr), _p(bown), _p(g), _p(bpr), _p(bflux))
    out, off = [], 0
    for p in mesh.patches:
        out.append(bflux[off:off + p.n_faces].copy())
        off += p.n_faces
    return flux, out


# --------------------------------------------------------------------------- O10
def _bfield(mesh, attr, dtype=np.float64, width=1):
    xs = []
    for p in mesh.patches:
        v = getattr(p, attr)
        xs.append(np.zeros((p.n_faces, width) if width > 1 else p.n_faces, dtype) if v is None else np.asarray(v, dtype))
    if not xs:
        return np.zeros(0, dtype)
    return np.ascontiguousarray(np.concatenate(xs), dtype=dtype)


def _proc_vals(mesh, vals, width=1):
    xs, k = [], 0
    for p in mesh.patches:
        if p.kind == PROCESSOR and vals is not None:
            xs.append(np.asarray(vals[k], np.float64).reshape(p.n_faces, width) if width > 1 else np.asarray(vals[k], np.float64))
            k += 1
        else:
            xs.append(np.zeros((p.n_faces, width)) if width > 1 else np.zeros(p.n_faces))
    return _f64(np.concatenate(xs) if xs else np.zeros(0))


def gauss_grad(mesh: gen.Mesh, p, geo: Optional[Geometry] = None, p_remote=None) -> np.ndarray:
    """Gauss linear cell gradient of p (gaussGrad): [N, 3]."""
    lib = _L()
    geo = geo or geometry(mesh)
    G = np.empty((mesh.n_cells, 3))
    bkind = _i32(np.concatenate([np.full(q.n_faces, q.kind, np.int32) for q in mesh.patches]) if mesh.patches else np.zeros(0))
    bcells, bSf, bval, bown = _bcat(mesh, "face_cells", np.int32), _bfield(mesh, "Sf", width=3), _bcat(mesh, "value", np.float64), _bcat(mesh, "is_owner", np.int8)
    bpr = _proc_vals(mesh, p_remote)
    own, nbr, Sf, pp, V = _i32(mesh.owner), _i32(mesh.neighbour), _f64(mesh.Sf), _f64(p), _f64(mesh.V)
    lib.or_gauss_grad(mesh.n_cells, mesh.n_faces, _p(own), _p(nbr), _p(Sf), _p(geo.weights), _p(pp), bkind.shape[0],
                      _p(bkind), _p(bcells), _p(bSf), _p(bval), _p(geo.bweight), _p(bown), _p(bpr), _p(V), _p(G))
    return G


def nonorth_correction(mesh: gen.Mesh, p, gamma=None, geo: Optional[Geometry] = None, gamma_remote=None,
                       p_remote=None, G=None, G_remote=None):
    """Explicit non-orthogonal correction of Gauss linear corrected:
    correction flux gammaMagSf * (corrVec . interpolate(grad p)) and the source change
    -V fvc::div(correction flux).  Returns (cflux [F], per-patch cflux, dsource [N], G)."""
    lib = _L()
    geo = geo or geometry(mesh)
    if G is None:
        G = gauss_grad(mesh, p, geo, p_remote)
    F = mesh.n_faces
    cflux = np.empty(F)
    bkind = _i32(np.concatenate([np.full(q.n_faces, q.kind, np.int32) for q in mesh.patches]) if mesh.patches else np.zeros(0))
    bcells, bSf, bmag = _bcat(mesh, "face_cells", np.int32), _bfield(mesh, "Sf", width=3), _bcat(mesh, "magSf", np.float64)
    bown, bnC = _bcat(mesh, "is_owner", np.int8), _bfield(mesh, "neighbour_C", width=3)
    bgr, bGr = _proc_vals(mesh, gamma_remote), _proc_vals(mesh, G_remote, width=3)
    bcf = np.zeros(bkind.shape[0])
    own, nbr, Sf, mag, C = _i32(mesh.owner), _i32(mesh.neighbour), _f64(mesh.Sf), _f64(mesh.magSf), _f64(mesh.C)
    g = None if gamma is None else _f64(gamma)
    Gc = _f64(G)
    lib.or_nonorth_flux(F, _p(own), _p(nbr), _p(Sf), _p(mag), _p(C), _p(geo.delta), _p(geo.weights), _p(g), _p(Gc),
                        _p(cflux), bkind.shape[0], _p(bkind), _p(bcells), _p(bSf), _p(bmag), _p(geo.bdelta),
                        _p(geo.bweight), _p(bown), _p(bnC), _p(bgr), _p(bGr), _p(bcf))
    pcf, off = [], 0
    for q in mesh.patches:
        pcf.append(bcf[off:off + q.n_faces].copy())
        off += q.n_faces
    div = surface_integrate(mesh, cflux, pcf)
    dsource = -(_f64(mesh.V) * div)
    return cflux, pcf, dsource, G


# --------------------------------------------------------------------------- O7
def dense_from_ldu(mesh_or_n, owner=None, neighbour=None, diag=None, upper=None, lower=None) -> np.ndarray:
    if isinstance(mesh_or_n, gen.Mesh):
        n, owner, neighbour = mesh_or_n.n_cells, mesh_or_n.owner, mesh_or_n.neighbour
    else:
        n = int(mesh_or_n)
    lower = upper if lower is None else lower
    A = np.empty((n, n))
    owner, neighbour = _i32(owner), _i32(neighbour)
    d, lo, up = _f64(diag), _f64(lower), _f64(upper)
    _L().or_dense_from_ldu(n, owner.shape[0], _p(owner), _p(neighbour), _p(d), _p(lo), _p(up), _p(A))
    return A


def dense_matvec(A, x) -> np.ndarray:
    A = _f64(A)
    y = np.empty(A.shape[0])
    x = _f64(x)
    _L().or_dense_matvec(A.shape[0], _p(A), _p(x), _p(y))
    return y


def dense_solve(A, b) -> np.ndarray:
    A = _f64(A)
    x = np.empty(A.shape[0])
    b = _f64(b)
    if _L().or_dense_solve(A.shape[0], _p(A), _p(b), _p(x)):
        raise np.linalg.LinAlgError("singular")
    return x


# --------------------------------------------------------------------------- convenience
def solve_case(mesh: gen.Mesh, gamma=None, b=None, ref_cell: int = 0, ref_value: float = 0.0,
               ctl: Optional[Controls] = None, psi0=None):
    """Assembly (O3, O4) + PCG (O6) of one case; returns (psi, perf, system)."""
    sys = assemble(mesh, gamma, ref_cell, ref_value, b)
    psi, perf = pcg(mesh, sys, psi0, ctl)
    return psi, perf, sys
