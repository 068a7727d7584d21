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
    assert lib.cnpint_workspace_bytes(32768, C.byref(op2), 0) == 0   # 2D time pass limited to N <= 16384
    assert lib.cnpint_workspace_bytes(65536, C.byref(op), 0) > 0     # 1D up to N = 65536 (four-step FFT)
    tiny = cnpint.Operator(2, 1, 3, 1, None, None, None, 1.0, -2.0, 1.0, 1.0, -2.0, 1.0, 0.0)
    assert lib.cnpint_workspace_bytes(64, C.byref(tiny), 0) == 0     # 2D needs nx, ny >= 3
    # the four-step intermediate and counters are part of the workspace from 1D N = 2048 on
    assert lib.cnpint_workspace_bytes(2048, C.byref(op), 0) > 2 * lib.cnpint_workspace_bytes(1024, C.byref(op), 0)


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


def test_theorem_4_5_host_check_matches_oracle():
    """paper_2401_16113_b200.theory (host logic of NEXT #4) against the oracle's rate_bound_check on
    seeded histories, δ ∈ (0, ½), and the δ ≥ ½ refusal."""
    import math
    import numpy as np
    from oracle import gmres as og
    from paper_2401_16113_b200 import theory
    rng = np.random.default_rng(7)
    for N in (16, 256, 4096):
        for delta in (0.01, 0.25, 0.45):
            a = theory.alpha_for_delta(delta, N)
            d, r = theory.theorem_4_5_rate(a, N)
            do, ro = og.rate_bound(a, 1.0 / N, 1.0)
            assert abs(d - do) < 1e-14 and abs(r - ro) < 1e-14 * max(1.0, 1e-2 / delta)
            for _ in range(5):
                hist = list(np.cumprod(rng.uniform(0.3, 1.0, 6)) * r ** 0.5)
                c1, c2 = theory.rate_bound_check(hist, a, N), og.rate_bound_check(hist, a, 1.0 / N, 1.0)
                assert c1["holds"] == c2["holds"] and c1["holds_printed"] == c2["holds_printed"]
                assert abs(c1["worst"] - c2["worst"]) <= 1e-12 * c2["worst"]
    import pytest
    with pytest.raises(ValueError):
        theory.theorem_4_5_rate(0.5 / math.sqrt(64), 64)
