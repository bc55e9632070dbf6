"""CPU-side checks of the boundary: the C-ABI library builds for sm_100a, loads, and exports
every symbol include/refine.h declares (no compute calls -- there is no GPU here); the
product path refuses to run without its CUDA extension; the oracle is not imported by it."""
import ctypes
import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "refine.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(refine_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for s in ("refine_init_dense", "refine_init_csr", "refine_sweep", "refine_run", "refine_destroy"):
        assert s in syms


def test_library_builds_and_exports_every_declared_symbol():
    from paper_2602_23778_b200 import build
    path = build.build()
    L = ctypes.CDLL(path)
    for s in declared_symbols():
        assert hasattr(L, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True).stdout
    for s in declared_symbols():
        assert re.search(rf"\bT {s}\b", out), s
    import paper_2602_23778_b200 as pkg
    assert set(pkg.EXPORTED) == set(declared_symbols())


def test_library_is_sm100a_with_dmma():
    from paper_2602_23778_b200 import build
    path = build.build()
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", path], capture_output=True,
                                       text=True).stdout
    assert "DMMA.8x8x4" in sass          # FP64 tensor-core instruction in the GEMM / pass kernels


def test_status_strings_without_gpu():
    import paper_2602_23778_b200 as pkg
    assert pkg.refine_status_string(pkg.REFINE_OK) == "REFINE_OK"
    assert pkg.refine_status_string(pkg.REFINE_E_NEAR_ZERO_RQ) == "REFINE_E_NEAR_ZERO_RQ"


def test_product_path_does_not_import_the_oracle():
    code = ("import sys; sys.path.insert(0, %r); import paper_2602_23778_b200 as p; p.lib(); "
            "assert 'oracle' not in sys.modules, 'oracle imported by product path'" % ROOT)
    subprocess.check_call([sys.executable, "-c", code])
    for dirpath, _, files in os.walk(os.path.join(ROOT, "paper_2602_23778_b200")):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "liboracle" not in txt, f


def test_missing_library_fails_loudly(tmp_path):
    code = ("import sys; sys.path.insert(0, %r); import paper_2602_23778_b200 as p; "
            "p.LIB_PATH = %r; p._lib = None\n"
            "try:\n    p.lib()\nexcept ImportError as e:\n    print('raised')\n" % (ROOT, str(tmp_path / "none.so")))
    out = subprocess.check_output([sys.executable, "-c", code], text=True)
    assert "raised" in out
