"""C-ABI library checks that need no GPU: the library loads, exports every symbol the header
declares, and the host-only argument validation behaves as include/cnpint.h documents."""
import ctypes as C
import os
import re

import pytest

from paper_2401_16113_b200 import cnpint

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "cnpint.h")).read()
    return sorted(set(re.findall(r"\b(cnpint_[a-z_A-Z0-9]+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    lib = cnpint.load_library()
    syms = header_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert sorted(cnpint.EXPORTS) == syms


def op1d(n=255, toeplitz=True):
    return cnpint.Operator(1, n, 1, int(toeplitz), None, None, None, 1.0, -2.0, 1.0, 0, 0, 0, 0)


def test_workspace_bytes_validation():
    lib = cnpint.load_library()
    op = op1d()
    assert lib.cnpint_workspace_bytes(256, C.byref(op), 0) > 0
    assert lib.cnpint_workspace_bytes(255, C.byref(op), 0) == 0      # N not a power of two
    assert lib.cnpint_workspace_bytes(1, C.byref(op), 0) == 0        # N < 2
    assert lib.cnpint_workspace_bytes(256, C.byref(op), -1) == 0
    nt = op1d(toeplitz=False)                                         # variable rows need arrays
    assert lib.cnpint_workspace_bytes(256, C.byref(nt), 0) == 0
    op2 = cnpint.Operator(2, 255, 255, 1, None, None, None, 1.0, -2.0, 1.0, 1.0, -2.0, 1.0, -0.05)
    assert lib.cnpint_workspace_bytes(512, C.byref(op2), 40) > lib.cnpint_workspace_bytes(512, C.byref(op2), 0)
    bad2 = cnpint.Operator(2, 254, 255, 1, None, None, None, 1.0, -2.0, 1.0, 1.0, -2.0, 1.0, 0.0)
    assert lib.cnpint_workspace_bytes(512, C.byref(bad2), 0) == 0    # n+1 not a power of two
    sym = cnpint.Operator(2, 255, 255, 1, None, None, None, -1.0, -2.0, 1.0, 1.0, -2.0, 1.0, 0.0)
    assert lib.cnpint_workspace_bytes(512, C.byref(sym), 0) == 0     # xs*xu <= 0


def test_workspace_scales_with_restart():
    lib = cnpint.load_library()
    op = op1d(4095)
    w0 = lib.cnpint_workspace_bytes(4096, C.byref(op), 0)
    w30 = lib.cnpint_workspace_bytes(4096, C.byref(op), 30)
    vec = 4096 * 4096 * 8
    # Krylov basis (restart + 1 vectors) + the cycle's preconditioned directions z_j (restart vectors)
    assert 61 * vec <= w30 - w0 <= 61 * vec + 10 * 2**20


def test_create_rejects_before_touching_the_device():
    lib = cnpint.load_library()
    op = op1d()
    h = C.c_void_p()
    assert lib.cnpint_create(C.byref(h), 256, 1.0, 0.01, C.byref(op), 0, None, 0, None) == cnpint.EINVAL
    assert lib.cnpint_create(C.byref(h), 256, 1.0, 1.0, C.byref(op), 0, None, 0, None) == cnpint.EINVAL
    assert lib.cnpint_create(C.byref(h), 24, 1.0, 0.1, C.byref(op), 0, None, 0, None) == cnpint.EUNSUPPORTED
    assert lib.cnpint_create(C.byref(h), 256, 0.0, 0.1, C.byref(op), 0, None, 0, None) == cnpint.EINVAL


def test_product_path_does_not_import_oracle():
    """The product package must not reference the oracle (it is test infrastructure only)."""
    pkg = os.path.join(ROOT, "paper_2401_16113_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle\b", txt, re.M), f
                assert "oracle/" not in txt.replace("``oracle/``", ""), f
