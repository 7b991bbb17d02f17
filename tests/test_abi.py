"""CPU-side checks of the C-ABI boundary (no compute calls need a GPU here).

- libspuma.so loads and exports every function include/spuma.h declares;
- argument validation happens before any device work;
- without a CUDA device the compute path fails loudly (SPUMA_ERR_CUDA), it
  never falls back to the CPU or to the oracle;
- the product package never imports the oracle."""
import ctypes
import os
import re
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "spuma.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(spuma_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("spuma_mesh_create", "spuma_assemble_laplacian", "spuma_pcg_solve", "spuma_free"):
        assert required in names


def test_library_exports_every_declared_symbol():
    from paper_2512_22215_b200 import spuma
    L = spuma.lib()
    for name in declared_functions():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", spuma._build.SO], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (spuma_\w+)", out))
    assert set(declared_functions()) <= exported
    assert L.spuma_abi_version() == 1


def test_library_is_built_for_sm_100a():
    from paper_2512_22215_b200 import spuma
    spuma.lib()
    out = subprocess.run(["cuobjdump", "--list-elf", spuma._build.SO], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_argument_validation_without_device():
    from paper_2512_22215_b200 import spuma
    L = spuma.lib()
    h = ctypes.c_void_p()
    assert L.spuma_mesh_create(None, ctypes.byref(h)) == 1
    assert b"NULL" in L.spuma_last_error()
    d = spuma.MeshDesc()
    d.abi_version = 99
    assert L.spuma_mesh_create(ctypes.byref(d), ctypes.byref(h)) == 1
    assert h.value is None
    L.spuma_free(None)  # NULL-safe
    perf = spuma.SolverPerf()
    ctl = spuma.SolverControls(1e-6, 0, 10, 0)
    assert L.spuma_pcg_solve(None, None, None, None, None, None, ctypes.byref(ctl), ctypes.byref(perf)) == 1


def test_no_cpu_fallback_without_device():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    import gen
    import paper_2512_22215_b200 as P
    m = gen.cube(3)
    with pytest.raises(P.SpumaError) as e:
        P.Mesh.from_mesh(m)
    assert e.value.status == 4  # SPUMA_ERR_CUDA: loud failure, no CPU path


def test_product_does_not_import_oracle():
    code = ("import sys, paper_2512_22215_b200 as P; P.spuma.lib(); "
            "bad=[m for m in sys.modules if m == 'oracle' or m.startswith('oracle.') or m == 'gen']; "
            "print(bad); sys.exit(1 if bad else 0)")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    src_dir = os.path.join(ROOT, "paper_2512_22215_b200")
    for dirpath, _, files in os.walk(src_dir):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "oracle.h" not in txt and "from oracle" not in txt, f
