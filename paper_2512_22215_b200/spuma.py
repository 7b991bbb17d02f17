"""Thin ctypes binding of libspuma (include/spuma.h) -- argument marshalling only.

Every step of the path runs in libspuma's CUDA kernels; this module converts
numpy arrays / torch tensors to pointers and C structs.  Names follow the
C-ABI (``spuma_mesh_create`` -> ``mesh_create`` ...).  There is no CPU
fallback: if libspuma.so is missing and cannot be built, import fails; if no
CUDA device is usable, every compute call raises SpumaError(SPUMA_ERR_CUDA).

Arrays: torch CUDA tensors (device pointers, used in place), torch CPU tensors
or numpy arrays (host pointers; the library stages them).  fp64 scalars,
int32 labels; tensors/arrays must be contiguous.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

from . import _build

ZERO_GRADIENT, FIXED_VALUE, EMPTY, PROCESSOR = 0, 1, 2, 3
STATUS = {0: "SPUMA_OK", 1: "SPUMA_ERR_INVALID_ARGUMENT", 2: "SPUMA_ERR_ADDRESSING", 3: "SPUMA_ERR_LENGTH_MISMATCH",
          4: "SPUMA_ERR_CUDA", 5: "SPUMA_ERR_NCCL", 6: "SPUMA_ERR_OUT_OF_MEMORY", 7: "SPUMA_ERR_STATE"}
ABI_VERSION = 1
OPT_AMUL_VARIANT = 0
OPT_SMALL_SOLVE_MAX_CELLS = 1
OPT_PDL = 2
OPT_DEFER_PSI = 3
OPT_GAMG_TAIL_CELLS = 4
OPT_FUSE_DIRECTION = 5
OPT_ALT_SWEEP = 6
OPT_ELL_STENCIL = 7
OPT_L2_PERSIST = 8
OPT_GAMG_CSR = 9
OPT_PEER_POLL_MS = 10
OPT_SMALL_SMEM = 11
OPT_PEER_FUSED = 12
OPT_PERSISTENT = 13
OPT_LOOP_L2 = 14
OPT_LOOP_PROFILE = 15
OPT_LOOP_GRID = 16
PEER_BLOB_BYTES = 512  # SPUMA_PEER_BLOB_BYTES
AMUL_VARIANTS = (0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13)

_vp, _ci, _cd, _lab = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_int32


class SpumaError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class PatchDesc(ctypes.Structure):
    _fields_ = [("kind", _ci), ("n_faces", _lab), ("face_cells", _vp), ("Sf", _vp), ("magSf", _vp), ("Cf", _vp),
                ("neighbour_rank", _ci), ("global_face", _vp), ("neighbour_C", _vp), ("is_owner", _vp)]


class MeshDesc(ctypes.Structure):
    _fields_ = [("abi_version", _ci), ("n_cells", _lab), ("n_faces", _lab), ("owner", _vp), ("neighbour", _vp),
                ("Sf", _vp), ("magSf", _vp), ("C", _vp), ("Cf", _vp), ("n_patches", _ci),
                ("patches", ctypes.POINTER(PatchDesc)), ("renumber", _ci), ("pointers_on_device", _ci),
                ("cuda_stream", _vp), ("rank", _ci), ("n_ranks", _ci), ("nccl_unique_id", _vp)]


class SolverControls(ctypes.Structure):
    _fields_ = [("tolerance", _cd), ("rel_tol", _cd), ("max_iter", _ci), ("min_iter", _ci)]


class SolverPerf(ctypes.Structure):
    _fields_ = [("initial_residual", _cd), ("final_residual", _cd), ("n_iterations", _ci), ("converged", _ci),
                ("singular", _ci)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class GamgParams(ctypes.Structure):
    """spuma_gamg_params (include/spuma.h; readings Q22-Q28)."""
    _fields_ = [("n_pre_sweeps", _ci), ("n_post_sweeps", _ci), ("scale_correction", _ci),
                ("n_cells_in_coarsest_level", _ci), ("max_levels", _ci), ("omega", _cd),
                ("coarsest_tolerance", _cd), ("coarsest_rel_tol", _cd), ("coarsest_max_iter", _ci),
                ("smoother", _ci), ("n_inner", _ci)]


SMOOTHER_RICHARDSON, SMOOTHER_GS2 = 0, 1


def gamg_params(**kw) -> GamgParams:
    """Defaults of spuma_gamg_default_params, overridden by keyword (field names above)."""
    p = GamgParams()
    lib().spuma_gamg_default_params(ctypes.byref(p))
    for k, v in kw.items():
        if k not in dict(GamgParams._fields_):
            raise TypeError(f"unknown GAMG parameter {k}")
        setattr(p, k, v)
    return p


class Preconditioner(ctypes.Structure):
    """spuma_preconditioner (readings Q31-Q33)."""
    _fields_ = [("kind", _ci), ("n_sweeps", _ci)]


PC_DIAGONAL, PC_DIC, PC_DILU, PC_ADILU = 0, 1, 2, 3


EXCHANGE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                               ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                               ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double))
ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_double),
                                ctypes.POINTER(ctypes.c_double), ctypes.c_int)


class CommCallbacks(ctypes.Structure):
    _fields_ = [("ctx", _vp), ("exchange", EXCHANGE_FN), ("allgather", ALLGATHER_FN)]


class Stats(ctypes.Structure):
    _fields_ = [("kernel_launches", ctypes.c_uint64), ("solves", ctypes.c_uint64), ("iterations", ctypes.c_uint64),
                ("timing_enabled", _ci), ("phase_ms", _cd * 4), ("phase_count", ctypes.c_uint64 * 4),
                ("blocks_per_grid", _ci), ("threads_per_block", _ci), ("batch_iterations", _ci),
                ("amul_variant", _ci), ("loop_mode", _ci), ("loop_grid", _ci), ("loop_tmem_pairs", _ci),
                ("loop_smem_pairs", _ci), ("loop_ms", _cd), ("loop_count", ctypes.c_uint64),
                ("loop_work_ms", _cd * 3), ("loop_wait_ms", _cd * 3), ("loop_work_max_ms", _cd * 3),
                ("loop_threads", _ci)]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["phase_ms"] = list(self.phase_ms)
        d["phase_count"] = list(self.phase_count)
        for k in ("loop_work_ms", "loop_wait_ms", "loop_work_max_ms"):
            d[k] = list(getattr(self, k))
        return d


_lib = None


def lib():
    """Load libspuma.so (building it in-tree with nvcc if missing or stale)."""
    global _lib
    if _lib is None:
        path = os.environ.get("SPUMA_LIBRARY", _build.SO)  # override: an alternative in-tree build (A/B)
        if path == _build.SO and _build.stale():
            _build.build()
        L = ctypes.CDLL(path)
        L.spuma_mesh_create.argtypes = [ctypes.POINTER(MeshDesc), ctypes.POINTER(_vp)]
        L.spuma_assemble_laplacian.argtypes = [_vp, _vp, _vp, _lab, _cd, _vp, _vp, _vp, _vp]
        L.spuma_pcg_solve.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, ctypes.POINTER(SolverControls),
                                      ctypes.POINTER(SolverPerf)]
        L.spuma_free.argtypes = [_vp]
        L.spuma_free.restype = None
        L.spuma_amul.argtypes = [_vp] * 6
        if hasattr(L, "spuma_surface_integrate"):
            L.spuma_surface_integrate.argtypes = [_vp] * 5
            L.spuma_face_flux.argtypes = [_vp] * 11
        if hasattr(L, "spuma_laplacian_correction"):
            L.spuma_laplacian_correction.argtypes = [_vp] * 8
        L.spuma_mesh_get_addressing.argtypes = [_vp] * 8
        L.spuma_mesh_get_geometry.argtypes = [_vp] * 4
        L.spuma_get_stats.argtypes = [_vp, ctypes.POINTER(Stats)]
        L.spuma_reset_stats.argtypes = [_vp]
        L.spuma_set_timing.argtypes = [_vp, _ci]
        L.spuma_set_batch.argtypes = [_vp, _ci]
        L.spuma_set_option.argtypes = [_vp, _ci, _ci]
        L.spuma_nccl_get_unique_id.argtypes = [_vp]
        if hasattr(L, "spuma_set_comm_callbacks"):  # absent only in older A/B builds
            L.spuma_set_comm_callbacks.argtypes = [_vp, ctypes.POINTER(CommCallbacks)]
        if hasattr(L, "spuma_peer_export"):
            L.spuma_peer_export.argtypes = [_vp, _vp]
            L.spuma_peer_import.argtypes = [_vp, _vp, _ci]
            L.spuma_peer_check.argtypes = [_vp]
        if hasattr(L, "spuma_gamg_solve"):
            L.spuma_gamg_default_params.argtypes = [ctypes.POINTER(GamgParams)]
            L.spuma_gamg_default_params.restype = None
            L.spuma_gamg_solve.argtypes = [_vp] * 6 + [ctypes.POINTER(SolverControls), ctypes.POINTER(GamgParams),
                                                       ctypes.POINTER(SolverPerf)]
            L.spuma_gamg_get_hierarchy.argtypes = [_vp, ctypes.POINTER(GamgParams), _ci, _vp, _vp, _vp, _ci, _vp]
        if hasattr(L, "spuma_pbicg_solve"):
            L.spuma_pcg_solve_pc.argtypes = [_vp] * 6 + [ctypes.POINTER(SolverControls), ctypes.POINTER(Preconditioner),
                                                         ctypes.POINTER(SolverPerf)]
            L.spuma_pbicg_solve.argtypes = [_vp] * 8 + [ctypes.POINTER(SolverControls), ctypes.POINTER(Preconditioner),
                                                        ctypes.POINTER(SolverPerf)]
            L.spuma_precondition.argtypes = [_vp] * 4 + [ctypes.POINTER(Preconditioner), _vp, _vp, _ci]
            L.spuma_amul_asym.argtypes = [_vp] * 6 + [_ci]
            L.spuma_ldu_to_csr.argtypes = [_vp] * 4
            L.spuma_csr_values.argtypes = [_vp] * 5
        if hasattr(L, "spuma_host_gamg_hierarchy_dd"):
            L.spuma_host_gamg_hierarchy_dd.argtypes = [_ci] + [_vp] * 9 + [_ci, _ci, _vp, _vp, _vp]
        if hasattr(L, "spuma_host_rcm"):
            L.spuma_host_rcm.argtypes = [_ci, _ci, _vp, _vp, _vp]
            L.spuma_host_gamg_hierarchy.argtypes = [_ci, _ci, _vp, _vp, _vp, _ci, _ci, _ci, _vp, _vp, _vp, _vp]
            L.spuma_host_level_schedule.argtypes = [_ci, _ci, _vp, _vp, _vp, _vp, _vp, _vp]
            L.spuma_host_ldu_to_csr.argtypes = [_ci, _ci] + [_vp] * 5
        if hasattr(L, "spuma_host_lattice_offsets"):
            L.spuma_host_lattice_offsets.argtypes = [_ci, _ci, _vp, _vp, _vp, _vp]
        L.spuma_last_error.restype = ctypes.c_char_p
        L.spuma_abi_version.restype = _ci
        for name in ("spuma_mesh_create", "spuma_assemble_laplacian", "spuma_pcg_solve", "spuma_amul",
                     "spuma_mesh_get_addressing", "spuma_mesh_get_geometry", "spuma_get_stats",
                     "spuma_reset_stats", "spuma_set_timing", "spuma_set_batch", "spuma_nccl_get_unique_id",
                     "spuma_set_option", "spuma_set_comm_callbacks", "spuma_surface_integrate",
                     "spuma_face_flux", "spuma_laplacian_correction", "spuma_peer_export", "spuma_peer_import",
                     "spuma_peer_check"):
            if hasattr(L, name):
                getattr(L, name).restype = _ci
        if L.spuma_abi_version() != ABI_VERSION:
            raise SpumaError(1, "libspuma ABI version mismatch")
        _lib = L
    return _lib


def _check(st: int):
    if st != 0:
        raise SpumaError(st, lib().spuma_last_error().decode())


def _ptr(a, dtype):
    """(pointer, keep-alive) for a numpy array / torch tensor / None."""
    if a is None:
        return None, None
    try:
        import torch
        if isinstance(a, torch.Tensor):
            want = torch.float64 if dtype == np.float64 else (torch.int32 if dtype == np.int32 else torch.int8)
            if a.dtype != want:
                raise TypeError(f"expected {want}, got {a.dtype}")
            if not a.is_contiguous():
                raise ValueError("tensor must be contiguous")
            return a.data_ptr(), a
    except ImportError:  # pragma: no cover
        pass
    arr = np.ascontiguousarray(a, dtype=dtype)
    if arr is not a and isinstance(a, np.ndarray) and a.dtype == dtype and a.flags.c_contiguous:
        arr = a
    return arr.ctypes.data, arr


def nccl_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().spuma_nccl_get_unique_id(buf))
    return buf.raw


class Mesh:
    """A libspuma mesh handle (spuma_mesh)."""

    def __init__(self, handle: int, n_cells: int, n_faces: int, n_iface: int, n_bfaces: int, keep):
        self._h = handle
        self.n_cells, self.n_faces, self.n_iface, self.n_bfaces = n_cells, n_faces, n_iface, n_bfaces
        self._keep = keep

    # ---------------------------------------------------------------- create / free
    @classmethod
    def mesh_create(cls, n_cells: int, owner, neighbour, Sf, magSf, C, Cf, patches: Sequence = (),
                    renumber: bool = False, stream: Optional[int] = None, rank: int = 0, n_ranks: int = 1,
                    nccl_unique_id: Optional[bytes] = None, pointers_on_device: bool = False) -> "Mesh":
        """spuma_mesh_create.  ``patches``: objects with kind, face_cells, Sf, magSf, Cf and, for
        processor patches, neighbour_rank, global_face, neighbour_C, is_owner."""
        keep = []

        def P(a, dt):
            p, k = _ptr(a, dt)
            keep.append(k)
            return p

        n_faces = int(len(owner))
        descs = (PatchDesc * max(len(patches), 1))()
        n_iface = n_b = 0
        for i, p in enumerate(patches):
            d = descs[i]
            d.kind = int(p.kind)
            d.n_faces = int(len(p.face_cells))
            n_b += d.n_faces
            d.face_cells = P(p.face_cells, np.int32)
            d.Sf, d.magSf, d.Cf = P(p.Sf, np.float64), P(p.magSf, np.float64), P(p.Cf, np.float64)
            if d.kind == PROCESSOR:
                n_iface += d.n_faces
                d.neighbour_rank = int(p.neighbour_rank)
                d.global_face = P(p.global_face, np.int32)
                d.neighbour_C = P(p.neighbour_C, np.float64)
                d.is_owner = P(p.is_owner, np.int8)
            else:
                d.neighbour_rank = -1
        keep.append(descs)
        idbuf = None
        if nccl_unique_id is not None:
            idbuf = ctypes.create_string_buffer(bytes(nccl_unique_id), 128)
            keep.append(idbuf)
        desc = MeshDesc(ABI_VERSION, int(n_cells), n_faces, P(owner, np.int32), P(neighbour, np.int32),
                        P(Sf, np.float64), P(magSf, np.float64), P(C, np.float64), P(Cf, np.float64),
                        len(patches), descs, 1 if renumber else 0, 1 if pointers_on_device else 0,
                        stream, rank, n_ranks, ctypes.cast(idbuf, _vp) if idbuf is not None else None)
        h = _vp()
        _check(lib().spuma_mesh_create(ctypes.byref(desc), ctypes.byref(h)))
        obj = cls(h.value, int(n_cells), n_faces, n_iface, n_b, None)
        obj.rank, obj.n_ranks = int(rank), int(n_ranks)
        return obj

    @classmethod
    def from_mesh(cls, mesh, **kw) -> "Mesh":
        """Duck-typed: any object with n_cells, owner, neighbour, Sf, magSf, C, Cf, patches."""
        return cls.mesh_create(mesh.n_cells, mesh.owner, mesh.neighbour, mesh.Sf, mesh.magSf, mesh.C, mesh.Cf,
                               list(mesh.patches), **kw)

    def free(self):
        """spuma_free."""
        if self._h:
            lib().spuma_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    # ---------------------------------------------------------------- hot path
    def assemble_laplacian(self, gamma, patch_values, ref_cell: int, ref_value: float, diag, upper, source,
                           iface_coeffs=None):
        """spuma_assemble_laplacian; diag/upper/iface written, source read-modified-written in place."""
        keep = []
        arr = None
        if patch_values is not None:
            arr = (_vp * max(len(patch_values), 1))()
            for i, v in enumerate(patch_values):
                p, k = _ptr(v, np.float64)
                keep.append(k)
                arr[i] = p
        g, kg = _ptr(gamma, np.float64)
        d, kd = _ptr(diag, np.float64)
        u, ku = _ptr(upper, np.float64)
        s, ks = _ptr(source, np.float64)
        f, kf = _ptr(iface_coeffs, np.float64)
        _check(lib().spuma_assemble_laplacian(self._h, g, arr, int(ref_cell), float(ref_value), d, u, s, f))
        return kd, ku, ks, kf

    def pcg_solve(self, diag, upper, iface_coeffs, source, psi, tolerance=1e-6, rel_tol=0.0, max_iter=5000,
                  min_iter=0) -> dict:
        """spuma_pcg_solve; psi updated in place; returns the solver performance."""
        ctl = SolverControls(tolerance, rel_tol, max_iter, min_iter)
        perf = SolverPerf()
        d, kd = _ptr(diag, np.float64)
        u, ku = _ptr(upper, np.float64)
        f, kf = _ptr(iface_coeffs, np.float64)
        s, ks = _ptr(source, np.float64)
        p, kp = _ptr(psi, np.float64)
        _check(lib().spuma_pcg_solve(self._h, d, u, f, s, p, ctypes.byref(ctl), ctypes.byref(perf)))
        return perf.as_dict()

    def gamg_solve(self, diag, upper, iface_coeffs, source, psi, tolerance=1e-6, rel_tol=0.0, max_iter=1000,
                   min_iter=0, params: Optional[GamgParams] = None) -> dict:
        """spuma_gamg_solve; psi updated in place; n_iterations = V-cycles."""
        ctl = SolverControls(tolerance, rel_tol, max_iter, min_iter)
        perf = SolverPerf()
        d, kd = _ptr(diag, np.float64)
        u, ku = _ptr(upper, np.float64)
        f, kf = _ptr(iface_coeffs, np.float64)
        s, ks = _ptr(source, np.float64)
        p, kp = _ptr(psi, np.float64)
        _check(lib().spuma_gamg_solve(self._h, d, u, f, s, p, ctypes.byref(ctl),
                                      None if params is None else ctypes.byref(params), ctypes.byref(perf)))
        return perf.as_dict()

    def peer_export(self) -> bytes:
        """spuma_peer_export: this rank's peer-transport blob (CUDA IPC handle + patches)."""
        buf = ctypes.create_string_buffer(PEER_BLOB_BYTES)
        _check(lib().spuma_peer_export(self._h, buf))
        return buf.raw

    def peer_import(self, blobs) -> None:
        """spuma_peer_import: every rank's blob, rank order."""
        data = b"".join(bytes(b) for b in blobs)
        buf = ctypes.create_string_buffer(data, len(data))
        _check(lib().spuma_peer_import(self._h, buf, len(blobs)))

    def enable_peer_transport(self) -> None:
        """Switch this handle's collectives to the peer-memory transport: the blobs are
        all-gathered over the default torch.distributed process group (host plumbing only)."""
        import torch.distributed as dist
        mine = self.peer_export()
        allb = [None] * dist.get_world_size()
        dist.all_gather_object(allb, mine)
        self.peer_import(allb)

    def peer_check(self) -> None:
        _check(lib().spuma_peer_check(self._h))

    def gamg_hierarchy(self, params: Optional[GamgParams] = None, with_ftc: bool = True) -> dict:
        """spuma_gamg_get_hierarchy: level sizes and (internal-numbering) fine-to-coarse maps."""
        nl = ctypes.c_int(0)
        cells = np.zeros(64, np.int32)
        faces = np.zeros(64, np.int32)
        pp = None if params is None else ctypes.byref(params)
        _check(lib().spuma_gamg_get_hierarchy(self._h, pp, 64, ctypes.addressof(nl), cells.ctypes.data,
                                              faces.ctypes.data, -1, None))
        n = nl.value
        out = {"levels": n, "cells": cells[:n].tolist(), "faces": faces[:n].tolist(), "ftc": []}
        if with_ftc:
            for level in range(n - 1):
                ftc = np.zeros(int(cells[level]), np.int32)
                _check(lib().spuma_gamg_get_hierarchy(self._h, pp, 64, ctypes.addressof(nl), None, None, level,
                                                      ftc.ctypes.data))
                out["ftc"].append(ftc)
        return out

    # ---------------------------------------------------------------- §8(f3)/(f4)
    def pcg_solve_pc(self, diag, upper, source, psi, tolerance=1e-6, rel_tol=0.0, max_iter=5000, min_iter=0,
                     kind=PC_DIAGONAL, n_sweeps=2, iface_coeffs=None) -> dict:
        """spuma_pcg_solve_pc: PCG with a diagonal / DIC / DILU / aDILU preconditioner
        (processor-local on decomposed meshes)."""
        ctl, perf, pc = SolverControls(tolerance, rel_tol, max_iter, min_iter), SolverPerf(), Preconditioner(kind, n_sweeps)
        d, kd = _ptr(diag, np.float64)
        u, ku = _ptr(upper, np.float64)
        f, kf = _ptr(iface_coeffs, np.float64)
        s, ks = _ptr(source, np.float64)
        p, kp = _ptr(psi, np.float64)
        _check(lib().spuma_pcg_solve_pc(self._h, d, u, f, s, p, ctypes.byref(ctl), ctypes.byref(pc),
                                        ctypes.byref(perf)))
        return perf.as_dict()

    def pbicg_solve(self, diag, upper, lower, source, psi, tolerance=1e-6, rel_tol=0.0, max_iter=1000, min_iter=0,
                    kind=PC_ADILU, n_sweeps=2, iface_coeffs=None, iface_coeffs_t=None) -> dict:
        """spuma_pbicg_solve: PBiCG on an asymmetric LDU matrix (iface_*: decomposed meshes)."""
        ctl, perf, pc = SolverControls(tolerance, rel_tol, max_iter, min_iter), SolverPerf(), Preconditioner(kind, n_sweeps)
        d, kd = _ptr(diag, np.float64)
        u, ku = _ptr(upper, np.float64)
        lo, kl = _ptr(lower, np.float64)
        f, kf = _ptr(iface_coeffs, np.float64)
        ft, kft = _ptr(iface_coeffs_t, np.float64)
        s, ks = _ptr(source, np.float64)
        p, kp = _ptr(psi, np.float64)
        _check(lib().spuma_pbicg_solve(self._h, d, u, lo, f, ft, s, p, ctypes.byref(ctl), ctypes.byref(pc),
                                       ctypes.byref(perf)))
        return perf.as_dict()

    def precondition(self, diag, upper, lower, r, w, kind, n_sweeps=2, transpose=False):
        pc = Preconditioner(kind, n_sweeps)
        d, kd = _ptr(diag, np.float64)
        u, ku = _ptr(upper, np.float64)
        lo, kl = _ptr(lower, np.float64)
        rp, kr = _ptr(r, np.float64)
        wp, kw = _ptr(w, np.float64)
        _check(lib().spuma_precondition(self._h, d, u, lo, ctypes.byref(pc), rp, wp, int(transpose)))
        return kw

    def amul_asym(self, diag, upper, lower, x, y, transpose=False):
        d, kd = _ptr(diag, np.float64)
        u, ku = _ptr(upper, np.float64)
        lo, kl = _ptr(lower, np.float64)
        xp, kx = _ptr(x, np.float64)
        yp, ky = _ptr(y, np.float64)
        _check(lib().spuma_amul_asym(self._h, d, u, lo, xp, yp, int(transpose)))
        return ky

    def ldu_to_csr(self):
        N, F = self.n_cells, self.n_faces
        rp, col, mp = np.zeros(N + 1, np.int32), np.zeros(N + 2 * F, np.int32), np.zeros(N + 2 * F, np.int32)
        _check(lib().spuma_ldu_to_csr(self._h, rp.ctypes.data, col.ctypes.data, mp.ctypes.data))
        return rp, col, mp

    def csr_values(self, diag, upper, lower, values):
        _check(lib().spuma_csr_values(self._h, diag.data_ptr(), upper.data_ptr(), lower.data_ptr(), values.data_ptr()))

    def amul(self, diag, upper, iface_coeffs, x, y):
        """spuma_amul: y = A x."""
        d, kd = _ptr(diag, np.float64)
        u, ku = _ptr(upper, np.float64)
        f, kf = _ptr(iface_coeffs, np.float64)
        xp, kx = _ptr(x, np.float64)
        yp, ky = _ptr(y, np.float64)
        _check(lib().spuma_amul(self._h, d, u, f, xp, yp))
        return ky

    # ---------------------------------------------------------------- around the path (§8(f1))
    @staticmethod
    def _patch_ptrs(values, keep):
        if values is None:
            return None
        arr = (_vp * max(len(values), 1))()
        for i, v in enumerate(values):
            p, k = _ptr(v, np.float64)
            keep.append(k)
            arr[i] = p
        return arr

    def surface_integrate(self, phi, patch_phi, V, out):
        """spuma_surface_integrate: out = fvc::surfaceIntegrate(phi) (per cell, divided by V)."""
        keep = []
        pp = self._patch_ptrs(patch_phi, keep)
        a, ka = _ptr(phi, np.float64)
        v, kv = _ptr(V, np.float64)
        o, ko = _ptr(out, np.float64)
        _check(lib().spuma_surface_integrate(self._h, a, pp, v, o))
        return ko

    def face_flux(self, gamma, patch_values, upper, psi, corr_flux=None, patch_corr_flux=None, flux=None,
                  patch_flux=None, phi=None, patch_phi=None):
        """spuma_face_flux: fvMatrix::flux of the Laplacian (+ correction flux); phi -= flux in place."""
        keep = []
        pv = self._patch_ptrs(patch_values, keep)
        pc = self._patch_ptrs(patch_corr_flux, keep)
        pf = self._patch_ptrs(patch_flux, keep)
        pp = self._patch_ptrs(patch_phi, keep)
        ptrs = [_ptr(x, np.float64) for x in (gamma, upper, psi, corr_flux, flux, phi)]
        g, u, ps, cf, fl, ph = [p for p, _ in ptrs]
        _check(lib().spuma_face_flux(self._h, g, pv, u, ps, cf, pc, fl, pf, ph, pp))

    def laplacian_correction(self, gamma, patch_values, p, V, source, corr_flux=None, patch_corr_flux=None):
        """spuma_laplacian_correction: source -= V div(non-orthogonal correction flux) in place."""
        keep = []
        pv = self._patch_ptrs(patch_values, keep)
        pc = self._patch_ptrs(patch_corr_flux, keep)
        ptrs = [_ptr(x, np.float64) for x in (gamma, p, V, source, corr_flux)]
        g, pp, v, s, cf = [q for q, _ in ptrs]
        _check(lib().spuma_laplacian_correction(self._h, g, pv, pp, v, s, cf, pc))

    # ---------------------------------------------------------------- diagnostics
    def mesh_get_addressing(self) -> dict:
        N, F = self.n_cells, self.n_faces
        out = {k: np.empty(n, np.int32) for k, n in (("perm", N), ("owner", F), ("neighbour", F),
                                                      ("owner_start", N + 1), ("losort", F),
                                                      ("losort_start", N + 1), ("face_map", F))}
        _check(lib().spuma_mesh_get_addressing(self._h, *[out[k].ctypes.data for k in
                                                          ("perm", "owner", "neighbour", "owner_start", "losort",
                                                           "losort_start", "face_map")]))
        return out

    def mesh_get_geometry(self) -> dict:
        d, w, b = np.empty(self.n_faces), np.empty(self.n_faces), np.empty(max(self.n_bfaces, 1))
        _check(lib().spuma_mesh_get_geometry(self._h, d.ctypes.data, w.ctypes.data, b.ctypes.data))
        return {"delta": d, "weights": w, "bdelta": b[:self.n_bfaces]}

    def get_stats(self) -> dict:
        s = Stats()
        _check(lib().spuma_get_stats(self._h, ctypes.byref(s)))
        return s.as_dict()

    def reset_stats(self):
        _check(lib().spuma_reset_stats(self._h))

    def set_timing(self, enable: bool):
        _check(lib().spuma_set_timing(self._h, 1 if enable else 0))

    def set_batch(self, iterations: int):
        _check(lib().spuma_set_batch(self._h, int(iterations)))

    def set_comm_callbacks(self, exchange, allgather):
        """spuma_set_comm_callbacks (external-comm mode: n_ranks > 1 without an NCCL id).

        exchange(peers, offsets, counts, send, recv) and allgather(send, recv) receive numpy views
        of the library's host buffers and must fill recv; they run inside the spuma_* call."""
        def _ex(ctx, n, peers, offs, counts, send, recv):
            try:
                pe = [peers[i] for i in range(n)]
                of = [offs[i] for i in range(n)]
                co = [counts[i] for i in range(n)]
                tot = max([o + c for o, c in zip(of, co)] + [0])
                sv = np.ctypeslib.as_array(send, shape=(max(tot, 1),))
                rv = np.ctypeslib.as_array(recv, shape=(max(tot, 1),))
                exchange(pe, of, co, sv, rv)
                return 0
            except Exception:  # pragma: no cover - reported as SPUMA_ERR_NCCL
                import traceback
                traceback.print_exc()
                return 1

        def _ag(ctx, send, recv, n):
            try:
                allgather(np.ctypeslib.as_array(send, shape=(n,)),
                          np.ctypeslib.as_array(recv, shape=(n * self.n_ranks,)))
                return 0
            except Exception:  # pragma: no cover
                import traceback
                traceback.print_exc()
                return 1

        cb = CommCallbacks(None, EXCHANGE_FN(_ex), ALLGATHER_FN(_ag))
        self._cb = cb  # keep the trampolines alive with the handle
        _check(lib().spuma_set_comm_callbacks(self._h, ctypes.byref(cb)))

    def set_option(self, option: int, value: int):
        """spuma_set_option (OPT_AMUL_VARIANT: 0 per-row, 1 tile, 2 unrolled, 3 TMA pipeline)."""
        _check(lib().spuma_set_option(self._h, int(option), int(value)))


mesh_create = Mesh.mesh_create


# ---------------------------------------------------------------- host-only diagnostics (no device)
def _addr(owner, neighbour):
    return np.ascontiguousarray(owner, np.int32), np.ascontiguousarray(neighbour, np.int32)


def host_rcm(n_cells: int, owner, neighbour) -> np.ndarray:
    """spuma_host_rcm: the RCM permutation libspuma applies with renumber = 1 (perm[old] = new)."""
    o, nb = _addr(owner, neighbour)
    perm = np.zeros(max(n_cells, 1), np.int32)
    _check(lib().spuma_host_rcm(n_cells, o.shape[0], o.ctypes.data, nb.ctypes.data, perm.ctypes.data))
    return perm[:n_cells]


def host_lattice_offsets(n_cells: int, owner, neighbour) -> list:
    """spuma_host_lattice_offsets: the column offsets of Amul variant 12's lattice slots ([] if the
    numbering is not a lattice)."""
    o, nb = _addr(owner, neighbour)
    k = ctypes.c_int(0)
    d = np.zeros(3, np.int32)
    _check(lib().spuma_host_lattice_offsets(n_cells, o.shape[0], o.ctypes.data, nb.ctypes.data,
                                            ctypes.addressof(k), d.ctypes.data))
    return d[:k.value].tolist()


def host_gamg_hierarchy(n_cells: int, owner, neighbour, face_weights, n_coarsest=10, max_levels=50) -> dict:
    """spuma_host_gamg_hierarchy: level sizes and the fine-to-coarse maps libspuma builds."""
    o, nb = _addr(owner, neighbour)
    w = np.ascontiguousarray(face_weights, np.float64)
    nl = ctypes.c_int(0)
    cells, faces = np.zeros(64, np.int32), np.zeros(64, np.int32)
    _check(lib().spuma_host_gamg_hierarchy(n_cells, o.shape[0], o.ctypes.data, nb.ctypes.data, w.ctypes.data,
                                           n_coarsest, max_levels, 64, ctypes.addressof(nl), cells.ctypes.data,
                                           faces.ctypes.data, None))
    n = nl.value
    ftc = np.zeros(max(int(cells[:n - 1].sum()), 1), np.int32)
    _check(lib().spuma_host_gamg_hierarchy(n_cells, o.shape[0], o.ctypes.data, nb.ctypes.data, w.ctypes.data,
                                           n_coarsest, max_levels, 64, ctypes.addressof(nl), None, None,
                                           ftc.ctypes.data))
    maps, off = [], 0
    for k in range(n - 1):
        maps.append(ftc[off:off + cells[k]].copy())
        off += int(cells[k])
    return {"levels": n, "cells": cells[:n].tolist(), "faces": faces[:n].tolist(), "ftc": maps}


def host_gamg_hierarchy_dd(meshes, n_coarsest=10, max_levels=50) -> dict:
    """spuma_host_gamg_hierarchy_dd: the decomposed hierarchy (Q36, Q37) libspuma builds for the
    sub-meshes (duck-typed: n_cells, owner, neighbour, magSf, patches with kind / n_faces /
    face_cells / neighbour_rank), one thread per rank standing in for the collectives."""
    P = len(meshes)
    keep = []

    def arr(a, dt):
        x = np.ascontiguousarray(a, dt)
        if x.size == 0:
            x = np.zeros(1, dt)
        keep.append(x)
        return x.ctypes.data

    def tab(ptrs):
        t = (ctypes.c_void_p * P)(*ptrs)
        keep.append(t)
        return ctypes.addressof(t)

    ncell = np.array([m.n_cells for m in meshes], np.int32)
    nface = np.array([len(m.owner) for m in meshes], np.int32)
    owners, nbrs, ws, peers, counts, ifc, npat = [], [], [], [], [], [], []
    for m in meshes:
        pp = [p for p in m.patches if p.kind == PROCESSOR and p.n_faces > 0]
        owners.append(arr(m.owner, np.int32))
        nbrs.append(arr(m.neighbour, np.int32))
        ws.append(arr(m.magSf, np.float64))
        peers.append(arr([p.neighbour_rank for p in pp], np.int32))
        counts.append(arr([p.n_faces for p in pp], np.int32))
        ifc.append(arr(np.concatenate([p.face_cells for p in pp]) if pp else [], np.int32))
        npat.append(len(pp))
    npat = np.array(npat, np.int32)
    nl = ctypes.c_int(0)
    cells, ifs = np.zeros(64 * P, np.int32), np.zeros(64 * P, np.int32)
    _check(lib().spuma_host_gamg_hierarchy_dd(P, ncell.ctypes.data, nface.ctypes.data, tab(owners), tab(nbrs), tab(ws),
                                              npat.ctypes.data, tab(peers), tab(counts), tab(ifc), n_coarsest,
                                              max_levels, ctypes.addressof(nl), cells.ctypes.data, ifs.ctypes.data))
    n = nl.value
    return {"levels": n, "level_cells": [cells[64 * r:64 * r + n].tolist() for r in range(P)],
            "level_ifaces": [ifs[64 * r:64 * r + n].tolist() for r in range(P)]}


def host_level_schedule(n_cells: int, owner, neighbour):
    """spuma_host_level_schedule: (order_f, order_b, depth_f, depth_b) of the DIC/DILU sweeps."""
    o, nb = _addr(owner, neighbour)
    of, ob = np.zeros(max(n_cells, 1), np.int32), np.zeros(max(n_cells, 1), np.int32)
    df, db = ctypes.c_int(0), ctypes.c_int(0)
    _check(lib().spuma_host_level_schedule(n_cells, o.shape[0], o.ctypes.data, nb.ctypes.data, of.ctypes.data,
                                           ob.ctypes.data, ctypes.addressof(df), ctypes.addressof(db)))
    return of[:n_cells], ob[:n_cells], df.value, db.value


def host_ldu_to_csr(n_cells: int, owner, neighbour):
    """spuma_host_ldu_to_csr: (row_ptr, col, map into [diag | upper | lower])."""
    o, nb = _addr(owner, neighbour)
    nnz = n_cells + 2 * o.shape[0]
    rp, col, mp = np.zeros(n_cells + 1, np.int32), np.zeros(max(nnz, 1), np.int32), np.zeros(max(nnz, 1), np.int32)
    _check(lib().spuma_host_ldu_to_csr(n_cells, o.shape[0], o.ctypes.data, nb.ctypes.data, rp.ctypes.data,
                                       col.ctypes.data, mp.ctypes.data))
    return rp, col[:nnz], mp[:nnz]
