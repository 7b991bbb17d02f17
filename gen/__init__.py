"""Seeded synthetic inputs (meshes, fields, decompositions) shared by tests, bench and smoke.

This package holds NONE of the method's arithmetic: no delta coefficients,
weights, matrix coefficients or solver steps (those live, independently, in
``oracle/`` and in ``paper_2512_22215_b200``).  It produces what a mesh
generator / ``decomposePar`` / case setup hands to OpenFOAM:

* hex-lattice meshes (``box``, ``cube``, ``cavity2d``, ``perturbed``) in the
  lduAddressing convention: owner < neighbour, faces sorted by
  (owner, neighbour);
* a counter-based random cell permutation (BASELINE.json config 2/4:
  "random cell permutation to break locality");
* seeded cell fields gamma (rAU-like, log-normal) and a zero-mean RHS b;
* domain decompositions into sub-meshes with processor patches
  ("domain decomposition", "hierarchical").

The recipe (seeds, distributions) is stated in DESIGN.md §4 and SURVEY.md §8(d).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from dataclasses import dataclass, field, replace
from typing import List, Optional

import numpy as np

ZERO_GRADIENT, FIXED_VALUE, EMPTY, PROCESSOR = 0, 1, 2, 3
SEED_JITTER, SEED_PERM, SEED_GAMMA, SEED_RHS = 1, 2, 3, 4

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libgen.so")
_SRC = os.path.join(_HERE, "gen.c")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile gen.c into gen/libgen.so (plain gcc)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _SO)
    return _SO


def _L():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_SO)
            lib.gen_uniform.restype = ctypes.c_double
            lib.gen_uniform.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64]
            lib.gen_splitmix64.restype = ctypes.c_uint64
            lib.gen_splitmix64.argtypes = [ctypes.c_uint64]
            lib.gen_hex_fill.restype = ctypes.c_int
            lib.gen_hex_fill.argtypes = [ctypes.c_int] * 3 + [ctypes.c_double] * 4 + [ctypes.c_uint64] + [ctypes.c_void_p] * 11
            lib.gen_hex_counts.argtypes = [ctypes.c_int] * 3 + [ctypes.c_void_p] * 3
            lib.gen_random_perm.argtypes = [ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p]
            lib.gen_permute_faces.restype = ctypes.c_int
            lib.gen_permute_faces.argtypes = [ctypes.c_int64, ctypes.c_int64] + [ctypes.c_void_p] * 7
            lib.gen_gamma_lognormal.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p]
            lib.gen_rhs.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p]
            lib.gen_uniform_fill.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
            lib.gen_hex_window.restype = ctypes.c_int
            lib.gen_hex_window.argtypes = ([ctypes.c_int] * 3 + [ctypes.c_double] * 4 + [ctypes.c_uint64] +
                                           [ctypes.c_int] * 6 + [ctypes.c_void_p] * 15)
            _lib = lib
    return _lib


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


@dataclass
class Patch:
    """One boundary patch (OpenFOAM polyPatch + the p boundary condition kind).

    Sf points OUT of the (sub-)domain.  For ``PROCESSOR`` patches the extra
    fields describe the coupled face: the neighbouring rank, the face id in the
    undecomposed mesh (fixes order, Q13), the remote cell centre, and
    ``is_owner`` (1 if the local cell is the owner of the undecomposed face,
    i.e. the outward Sf equals the global owner->neighbour Sf)."""

    name: str
    kind: int
    face_cells: np.ndarray
    Sf: np.ndarray
    magSf: np.ndarray
    Cf: np.ndarray
    value: Optional[np.ndarray] = None  # fixedValue values (per face)
    neighbour_rank: int = -1
    global_face: Optional[np.ndarray] = None
    neighbour_C: Optional[np.ndarray] = None
    is_owner: Optional[np.ndarray] = None
    neighbour_gid: Optional[np.ndarray] = None  # global cell id of the remote cell (test plumbing)

    @property
    def n_faces(self) -> int:
        return int(self.face_cells.shape[0])


@dataclass
class Mesh:
    n_cells: int
    owner: np.ndarray  # int32 [F]
    neighbour: np.ndarray  # int32 [F]
    Sf: np.ndarray  # f64 [F,3]
    magSf: np.ndarray  # f64 [F]
    Cf: np.ndarray  # f64 [F,3]
    C: np.ndarray  # f64 [N,3]
    V: np.ndarray  # f64 [N]
    patches: List[Patch] = field(default_factory=list)
    gid: Optional[np.ndarray] = None  # int32 [N] global (lattice) cell id keying every random value
    gface: Optional[np.ndarray] = None  # int32 [F] face id in the undecomposed mesh
    dims: tuple = ()

    @property
    def n_faces(self) -> int:
        return int(self.owner.shape[0])


def uniform(seed: int, stream: int, ids: np.ndarray) -> np.ndarray:
    ids = np.ascontiguousarray(ids, dtype=np.int32)
    out = np.empty(ids.shape[0], dtype=np.float64)
    _L().gen_uniform_fill(seed, stream, ids.shape[0], _p(ids), _p(out))
    return out


def box(nx: int, ny: int, nz: int, L=(1.0, 1.0, 1.0), jitter: float = 0.0, seed: int = SEED_JITTER,
        names=("xmin", "xmax", "ymin", "ymax", "zmin", "zmax"), kinds=(ZERO_GRADIENT,) * 6) -> Mesh:
    """nx*ny*nz hex lattice on [0,Lx]x[0,Ly]x[0,Lz] with six wall patches."""
    lib = _L()
    nN = np.zeros(1, np.int64)
    nF = np.zeros(1, np.int64)
    ps = np.zeros(6, np.int64)
    lib.gen_hex_counts(nx, ny, nz, _p(nN), _p(nF), _p(ps))
    N, F, Fb = int(nN[0]), int(nF[0]), int(ps.sum())
    owner = np.empty(F, np.int32)
    nbr = np.empty(F, np.int32)
    Sf = np.empty((F, 3))
    magSf = np.empty(F)
    Cf = np.empty((F, 3))
    C = np.empty((N, 3))
    V = np.empty(N)
    bc = np.empty(Fb, np.int32)
    bSf = np.empty((Fb, 3))
    bm = np.empty(Fb)
    bCf = np.empty((Fb, 3))
    rc = lib.gen_hex_fill(nx, ny, nz, float(L[0]), float(L[1]), float(L[2]), float(jitter), seed,
                          _p(owner), _p(nbr), _p(Sf), _p(magSf), _p(Cf), _p(C), _p(V), _p(bc), _p(bSf), _p(bm), _p(bCf))
    if rc:
        raise MemoryError("gen_hex_fill")
    patches = []
    off = 0
    for k in range(6):
        n = int(ps[k])
        sl = slice(off, off + n)
        patches.append(Patch(names[k], kinds[k], bc[sl].copy(), bSf[sl].copy(), bm[sl].copy(), bCf[sl].copy()))
        off += n
    return Mesh(N, owner, nbr, Sf, magSf, Cf, C, V, patches, gid=np.arange(N, dtype=np.int32),
                gface=np.arange(F, dtype=np.int32), dims=(nx, ny, nz))


def cube(n: int, jitter: float = 0.0, seed: int = SEED_JITTER) -> Mesh:
    """G-cube(n): unit cube, h = 1/n, six zeroGradient walls."""
    return box(n, n, n, (1.0, 1.0, 1.0), jitter, seed)


def perturbed(n: int, a: float = 0.15, seed: int = SEED_JITTER) -> Mesh:
    """G-perturbed(n, a): jittered hex lattice (non-orthogonal, skewed)."""
    return box(n, n, n, (1.0, 1.0, 1.0), a, seed)


def merge_patches(mesh: Mesh, groups, kinds) -> Mesh:
    """Concatenate patches into named groups, e.g. the cavity's fixedWalls."""
    by = {p.name: p for p in mesh.patches}
    out = []
    for (name, members), kind in zip(groups, kinds):
        ps = [by[m] for m in members]
        out.append(Patch(name, kind, np.concatenate([p.face_cells for p in ps]),
                         np.concatenate([p.Sf for p in ps]), np.concatenate([p.magSf for p in ps]),
                         np.concatenate([p.Cf for p in ps])))
    return replace(mesh, patches=out)


def cavity2d(n: int = 20) -> Mesh:
    """G-cavity2D(n): the lid-driven cavity box 0.1 x 0.1 x 0.01 m, one cell deep.

    Patches: movingWall (top), fixedWalls (left, right, bottom) -- p zeroGradient --
    and frontAndBack (empty) (BASELINE.json config 1)."""
    m = box(n, n, 1, (0.1, 0.1, 0.01))
    return merge_patches(m, [("movingWall", ["ymax"]), ("fixedWalls", ["xmin", "xmax", "ymin"]),
                             ("frontAndBack", ["zmin", "zmax"])], [ZERO_GRADIENT, ZERO_GRADIENT, EMPTY])


def affine(mesh: Mesh, A, t=(0.0, 0.0, 0.0)) -> Mesh:
    """Map the geometry by x -> A x + t (an affine, e.g. sheared, mesh): centres map directly,
    vector areas by the cofactor det(A) A^-T, volumes by det(A).  Input generation only."""
    A = np.asarray(A, np.float64)
    t = np.asarray(t, np.float64)
    cof = np.linalg.det(A) * np.linalg.inv(A).T
    tr = lambda X: np.ascontiguousarray(X @ A.T + t)
    vs = lambda S: np.ascontiguousarray(S @ cof.T)
    patches = [replace(p, Sf=vs(p.Sf), magSf=np.linalg.norm(vs(p.Sf), axis=1), Cf=tr(p.Cf),
                       neighbour_C=None if p.neighbour_C is None else tr(p.neighbour_C)) for p in mesh.patches]
    Sf = vs(mesh.Sf)
    return replace(mesh, Sf=Sf, magSf=np.linalg.norm(Sf, axis=1), Cf=tr(mesh.Cf), C=tr(mesh.C),
                   V=mesh.V * np.linalg.det(A), patches=patches)


def set_kind(mesh: Mesh, name: str, kind: int, value: Optional[np.ndarray] = None) -> Mesh:
    ps = []
    for p in mesh.patches:
        if p.name == name:
            p = replace(p, kind=kind, value=None if value is None else np.ascontiguousarray(value, dtype=np.float64))
        ps.append(p)
    return replace(mesh, patches=ps)


def random_perm(n: int, seed: int = SEED_PERM) -> np.ndarray:
    perm = np.empty(n, np.int32)
    _L().gen_random_perm(n, seed, _p(perm))
    return perm


def permute(mesh: Mesh, perm: Optional[np.ndarray] = None, seed: int = SEED_PERM) -> Mesh:
    """Renumber cells by perm[old] = new (default: Fisher-Yates with ``seed``).

    Faces are re-keyed (owner = min, neighbour = max), Sf negated where the pair
    swapped, and re-sorted by (owner, neighbour), ties by old face index."""
    N, F = mesh.n_cells, mesh.n_faces
    if perm is None:
        perm = random_perm(N, seed)
    perm = np.ascontiguousarray(perm, dtype=np.int32)
    o = np.empty(F, np.int32)
    nb = np.empty(F, np.int32)
    fm = np.empty(F, np.int32)
    fl = np.empty(F, np.int8)
    if _L().gen_permute_faces(N, F, _p(perm), _p(mesh.owner), _p(mesh.neighbour), _p(o), _p(nb), _p(fm), _p(fl)):
        raise MemoryError("gen_permute_faces")
    sign = np.where(fl.astype(bool), -1.0, 1.0)[:, None]
    Sf = mesh.Sf[fm] * sign
    inv = np.empty(N, np.int64)
    inv[perm] = np.arange(N)
    patches = [replace(p, face_cells=perm[p.face_cells].astype(np.int32)) for p in mesh.patches]
    return Mesh(N, o, nb, np.ascontiguousarray(Sf), mesh.magSf[fm].copy(), mesh.Cf[fm].copy(),
                mesh.C[inv].copy(), mesh.V[inv].copy(), patches,
                gid=None if mesh.gid is None else mesh.gid[inv].copy(),
                gface=None if mesh.gface is None else mesh.gface[fm].copy(), dims=mesh.dims)


def permute_cell_field(x: np.ndarray, perm: np.ndarray) -> np.ndarray:
    out = np.empty_like(x)
    out[perm] = x
    return out


def gamma_lognormal(mesh: Mesh, seed: int = SEED_GAMMA) -> np.ndarray:
    """gamma_c = exp(0.5 xi), xi ~ N(0,1): mimics the spatial variation of rAU."""
    g = np.empty(mesh.n_cells)
    _L().gen_gamma_lognormal(mesh.n_cells, _p(np.ascontiguousarray(mesh.gid)), seed, _p(g))
    return g


def rhs(mesh: Mesh, seed: int = SEED_RHS) -> np.ndarray:
    """b_c = V_c (2U - 1), minus its mean; keyed by global cell id.

    Generate on the undecomposed, unpermuted mesh so the mean is taken in
    global-id order, then permute/decompose with the mesh."""
    b = np.empty(mesh.n_cells)
    _L().gen_rhs(mesh.n_cells, _p(np.ascontiguousarray(mesh.gid)), _p(np.ascontiguousarray(mesh.V)), seed, _p(b))
    return b


# ---------------------------------------------------------------------------
# domain decomposition (decomposePar analogue: PAPER.md P:87)
# ---------------------------------------------------------------------------

def block_parts(mesh: Mesh, nproc=(2, 1, 1)) -> np.ndarray:
    """Axis-aligned block decomposition of a lattice mesh (by cell centre)."""
    px, py, pz = nproc
    lo = mesh.C.min(axis=0)
    hi = mesh.C.max(axis=0)
    ext = np.where(hi > lo, hi - lo, 1.0)
    idx = []
    for d, p in enumerate((px, py, pz)):
        t = np.floor((mesh.C[:, d] - lo[d]) / ext[d] * p * (1 - 1e-12)).astype(np.int64)
        idx.append(np.clip(t, 0, p - 1))
    return (idx[0] + px * (idx[1] + py * idx[2])).astype(np.int32)


def rcb_parts(mesh: Mesh, nparts: int) -> np.ndarray:
    """Recursive coordinate bisection on cell centres: split x at the median
    (ties by global id), then y, then z, ... (the "hierarchical" method)."""
    part = np.zeros(mesh.n_cells, np.int32)
    gid = mesh.gid if mesh.gid is not None else np.arange(mesh.n_cells, dtype=np.int32)

    def rec(cells, p0, n, axis):
        if n == 1:
            part[cells] = p0
            return
        order = np.lexsort((gid[cells], mesh.C[cells, axis]))
        nl = n // 2
        cut = len(cells) * nl // n
        rec(cells[order[:cut]], p0, nl, (axis + 1) % 3)
        rec(cells[order[cut:]], p0 + nl, n - nl, (axis + 1) % 3)

    rec(np.arange(mesh.n_cells), 0, nparts, 0)
    return part


def decompose(mesh: Mesh, part: np.ndarray, nparts: Optional[int] = None) -> List[Mesh]:
    """Split a mesh into sub-meshes with processor patches.

    Local cells keep the global relative order; internal faces keep the global
    face order (so they stay sorted by local (owner, neighbour)); processor
    faces towards each neighbour rank are ordered by global face id (Q13) and
    carry Sf/Cf oriented out of the sub-domain, the remote cell centre and the
    ``is_owner`` flag.  Non-processor patches keep their order and come first;
    processor patches follow in ascending neighbour rank."""
    part = np.asarray(part, dtype=np.int32)
    P = int(part.max()) + 1 if nparts is None else nparts
    gid = mesh.gid if mesh.gid is not None else np.arange(mesh.n_cells, dtype=np.int32)
    gface = mesh.gface if mesh.gface is not None else np.arange(mesh.n_faces, dtype=np.int32)
    po, pn = part[mesh.owner], part[mesh.neighbour]
    out = []
    for r in range(P):
        cells = np.nonzero(part == r)[0]
        loc = np.full(mesh.n_cells, -1, np.int64)
        loc[cells] = np.arange(cells.shape[0])
        fin = np.nonzero((po == r) & (pn == r))[0]
        patches = []
        for p in mesh.patches:
            sel = np.nonzero(part[p.face_cells] == r)[0]
            patches.append(replace(p, face_cells=loc[p.face_cells[sel]].astype(np.int32), Sf=p.Sf[sel].copy(),
                                   magSf=p.magSf[sel].copy(), Cf=p.Cf[sel].copy(),
                                   value=None if p.value is None else p.value[sel].copy()))
        for q in range(P):
            if q == r:
                continue
            own = (po == r) & (pn == q)
            nei = (po == q) & (pn == r)
            fs = np.nonzero(own | nei)[0]  # ascending face index == ascending global face id
            if fs.shape[0] == 0:
                continue
            fs = fs[np.argsort(gface[fs], kind="stable")]
            is_owner = own[fs]
            lc = np.where(is_owner, mesh.owner[fs], mesh.neighbour[fs])
            rc = np.where(is_owner, mesh.neighbour[fs], mesh.owner[fs])
            sgn = np.where(is_owner, 1.0, -1.0)[:, None]
            patches.append(Patch(f"procBoundary{r}to{q}", PROCESSOR, loc[lc].astype(np.int32),
                                 np.ascontiguousarray(mesh.Sf[fs] * sgn), mesh.magSf[fs].copy(), mesh.Cf[fs].copy(),
                                 neighbour_rank=q, global_face=gface[fs].astype(np.int32),
                                 neighbour_C=np.ascontiguousarray(mesh.C[rc]), is_owner=is_owner.astype(np.int8),
                                 neighbour_gid=gid[rc].astype(np.int32)))
        out.append(Mesh(int(cells.shape[0]), loc[mesh.owner[fin]].astype(np.int32),
                        loc[mesh.neighbour[fin]].astype(np.int32), mesh.Sf[fin].copy(), mesh.magSf[fin].copy(),
                        mesh.Cf[fin].copy(), mesh.C[cells].copy(), mesh.V[cells].copy(), patches,
                        gid=gid[cells].astype(np.int32), gface=gface[fin].astype(np.int32), dims=mesh.dims))
    return out


def split_cell_field(x: np.ndarray, part: np.ndarray, nparts: Optional[int] = None) -> List[np.ndarray]:
    part = np.asarray(part)
    P = int(part.max()) + 1 if nparts is None else nparts
    return [np.ascontiguousarray(x[part == r]) for r in range(P)]


def lattice_block(gdims, L, lo, dims, rank_of, jitter: float = 0.0, seed: int = SEED_JITTER,
                  names=("xmin", "xmax", "ymin", "ymax", "zmin", "zmax")) -> Mesh:
    """One rank's window ``lo + [0, dims)`` of the global lattice ``gdims`` on box ``L``.

    Generated directly (no global mesh in memory): vertex coordinates use the
    global formula, so geometry is bitwise that of ``box(*gdims, L)`` and both
    sides of a cut agree.  Patches: the six walls (empty where the side is a
    cut), then one processor patch per cut side, to ``rank_of(side)``, in
    ascending neighbour rank (the ``decompose`` convention).  ``gface`` and
    ``gid`` are the undecomposed ids.  V of cut-side cells accumulates its
    faces in another order than ``box`` (inputs only; b is keyed by gid)."""
    lib = _L()
    NX, NY, NZ = gdims
    nx, ny, nz = dims
    nN = np.zeros(1, np.int64)
    nF = np.zeros(1, np.int64)
    ps = np.zeros(6, np.int64)
    lib.gen_hex_counts(nx, ny, nz, _p(nN), _p(nF), _p(ps))
    N, F, Fb = int(nN[0]), int(nF[0]), int(ps.sum())
    owner, nbr = np.empty(F, np.int32), np.empty(F, np.int32)
    Sf, magSf, Cf = np.empty((F, 3)), np.empty(F), np.empty((F, 3))
    C, V, gid = np.empty((N, 3)), np.empty(N), np.empty(N, np.int32)
    bc, bSf, bm, bCf = np.empty(Fb, np.int32), np.empty((Fb, 3)), np.empty(Fb), np.empty((Fb, 3))
    bnC, bng, bgf = np.empty((Fb, 3)), np.empty(Fb, np.int32), np.empty(Fb, np.int32)
    lib.gen_hex_window(NX, NY, NZ, float(L[0]), float(L[1]), float(L[2]), float(jitter), seed, lo[0], lo[1], lo[2],
                       nx, ny, nz, _p(owner), _p(nbr), _p(Sf), _p(magSf), _p(Cf), _p(C), _p(V), _p(gid), _p(bc),
                       _p(bSf), _p(bm), _p(bCf), _p(bnC), _p(bng), _p(bgf))
    walls, procs = [], []
    off = 0
    for k in range(6):
        n = int(ps[k])
        sl = slice(off, off + n)
        off += n
        cut = n > 0 and bng[sl][0] >= 0
        if not cut:
            walls.append(Patch(names[k], ZERO_GRADIENT, bc[sl].copy(), bSf[sl].copy(), bm[sl].copy(), bCf[sl].copy()))
            continue
        walls.append(Patch(names[k], ZERO_GRADIENT, np.zeros(0, np.int32), np.zeros((0, 3)), np.zeros(0), np.zeros((0, 3))))
        q = int(rank_of(k))
        procs.append((q, Patch("", PROCESSOR, bc[sl].copy(), bSf[sl].copy(), bm[sl].copy(), bCf[sl].copy(),
                               neighbour_rank=q, global_face=bgf[sl].copy(), neighbour_C=bnC[sl].copy(),
                               is_owner=np.full(n, 1 if k % 2 == 1 else 0, np.int8),
                               neighbour_gid=bng[sl].copy())))
    procs.sort(key=lambda t: t[0])
    me = None
    patches = walls + [replace(p, name=f"procBoundary{me}to{q}") for q, p in procs]
    # undecomposed face ids of the internal faces
    gi = gid[owner]
    ax = np.where(nbr - owner == 1, 0, np.where(nbr - owner == nx, 1, 2))
    gface = _lattice_face_ids(gdims, gi, ax)
    return Mesh(N, owner, nbr, Sf, magSf, Cf, C, V, patches, gid=gid, gface=gface, dims=tuple(gdims))


def _lattice_face_ids(gdims, cell, axis):
    """Face id in the undecomposed lattice of the face along ``axis`` owned by global cell ``cell``."""
    NX, NY, NZ = (np.int64(v) for v in gdims)
    c = cell.astype(np.int64)
    i, j, k = c % NX, (c // NX) % NY, c // (NX * NY)
    cx = (j + NY * k) * (NX - 1) + np.minimum(i, NX - 1)
    cy = k * NX * (NY - 1) + np.where(j < NY - 1, j * NX + i, (NY - 1) * NX)
    cz = np.where(k < NZ - 1, c, NX * NY * (NZ - 1))
    fid = cx + cy + cz + ((axis >= 1) & (i < NX - 1)) + ((axis >= 2) & (j < NY - 1))
    return fid.astype(np.int32)


def block_grid(nproc):
    """Rank of block (bx, by, bz) = bx + px (by + py bz) (matches ``block_parts``)."""
    px, py, pz = nproc
    return lambda bx, by, bz: bx + px * (by + py * bz)


def weak_block(n: int, nproc=(1, 1, 1), rank: int = 0) -> Mesh:
    """BASELINE config 3: rank ``rank``'s n^3 block of the global (n px, n py, n pz) unit-spaced
    cube (h = 1/n), generated directly from the global lattice."""
    px, py, pz = nproc
    if px * py * pz == 1:
        return cube(n)
    bx, by, bz = rank % px, (rank // px) % py, rank // (px * py)
    R = block_grid(nproc)
    nb = {0: (bx - 1, by, bz), 1: (bx + 1, by, bz), 2: (bx, by - 1, bz), 3: (bx, by + 1, bz),
          4: (bx, by, bz - 1), 5: (bx, by, bz + 1)}
    m = lattice_block((n * px, n * py, n * pz), (float(px), float(py), float(pz)), (n * bx, n * by, n * bz),
                      (n, n, n), lambda side: R(*nb[side]))
    m.patches = [replace(p, name=f"procBoundary{rank}to{p.neighbour_rank}") if p.kind == PROCESSOR else p
                 for p in m.patches]
    return m


def nproc_for(world: int):
    """Block layout of BASELINE config 3: 1 -> (1,1,1), 2 -> (2,1,1), 4 -> (2,2,1), 8 -> (2,2,2)."""
    return {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2)}.get(world) or (world, 1, 1)
