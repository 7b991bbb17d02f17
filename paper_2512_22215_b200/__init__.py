"""paper_2512_22215_b200 -- B200-native pressure-Laplacian assembly + Jacobi-PCG
(the hot path of SPUMA, arXiv 2512.22215), behind the C-ABI of include/spuma.h.

The product is libspuma.so (csrc/: host C++ + sm_100a CUDA kernels + NCCL);
``spuma`` is its thin ctypes binding.  This package never imports ``oracle``.
"""
from . import spuma
from .spuma import GamgParams, Mesh, Preconditioner, SpumaError, gamg_params, mesh_create, nccl_get_unique_id  # noqa: F401

__all__ = ["spuma", "Mesh", "SpumaError", "GamgParams", "gamg_params", "mesh_create", "nccl_get_unique_id"]
