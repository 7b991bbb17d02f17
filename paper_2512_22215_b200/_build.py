"""Build libspuma.so (sm_100a) in-tree with nvcc.

Flags: -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false
(--fmad=false: a*b+c stays DMUL + DADD, the rounding the oracle's
-ffp-contract=off uses -> bit-exact coefficients and Amul, reading Q10).
NCCL: the copy torch loads (nvidia/nccl in the venv), so one libnccl per process.
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libspuma.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    cands = []
    if spec and spec.submodule_search_locations:
        for loc in spec.submodule_search_locations:
            cands.append(os.path.join(loc, "nccl"))
    cands.append(os.path.join(sys.prefix, "lib", f"python{sys.version_info.major}.{sys.version_info.minor}",
                              "site-packages", "nvidia", "nccl"))
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")) and glob.glob(os.path.join(c, "lib", "libnccl.so*")):
            return os.path.join(c, "include"), os.path.join(c, "lib")
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "spuma.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out: str = None) -> str:
    """defines / out: an A/B build with -D<define> into another path (loaded via SPUMA_LIBRARY)."""
    if out is None and not force and not stale():
        return SO
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    inc, lib = nccl_dirs()
    libname = os.path.basename(sorted(glob.glob(os.path.join(lib, "libnccl.so*")))[0])
    dst = out or SO
    tmp = dst + f".tmp{os.getpid()}"
    cmd = [nvcc, *ARCH, "-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-shared",
           "-Xcompiler", "-fPIC,-ffp-contract=off,-O2", "-Xptxas", "-v" if verbose else "-O3",
           *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", inc,
           *sources(), "-o", tmp, "-L", lib, f"-l:{libname}", "-Xlinker", f"-rpath,{lib}", "-lcudart_static"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    if verbose:
        print(r.stdout + r.stderr)
    os.replace(tmp, dst)
    return dst


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
