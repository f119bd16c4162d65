"""The C-ABI library loads and exports every symbol include/nlse2shoc.h declares (CPU; no
compute calls without a GPU), plus the pure-host split rule."""
import ctypes
import os
import re

import pytest

from conftest import ROOT


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "nlse2shoc.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(nlse2shoc_[a-z_0-9]+)\s*\(", txt)))


def test_library_exports_header_symbols():
    from paper_1109_1027_b200 import _lib

    L = _lib.lib()
    syms = header_symbols()
    assert len(syms) >= 16
    for s in syms:
        assert hasattr(L, s), s
    assert sorted(_lib.EXPORTS) == syms
    assert L.nlse2shoc_version().decode().startswith("nlse2shoc")


def test_strerror_and_split_rule():
    import paper_1109_1027_b200 as nl
    from paper_1109_1027_b200 import _lib

    L = _lib.lib()
    assert L.nlse2shoc_strerror(-1).decode() == "invalid argument"
    # even split, remainder to the first ranks
    parts = [nl.nlse2shoc_split(770, 8, r) for r in range(8)]
    assert parts[0] == (0, 97) and parts[1] == (97, 97) and parts[2] == (194, 96)
    assert sum(nz for _, nz in parts) == 770
    assert all(parts[i][0] + parts[i][1] == parts[i + 1][0] for i in range(7))
    with pytest.raises(nl.NLSE2SHOCError):
        nl.nlse2shoc_split(10, 0, 0)


def test_create_rejects_bad_arguments_without_touching_the_gpu():
    """Argument validation happens before any CUDA call."""
    from paper_1109_1027_b200 import _lib

    L = _lib.lib()
    H = ctypes.c_void_p()
    n = (ctypes.c_int64 * 3)(4, 1, 1)
    h = (ctypes.c_double * 3)(0.1, 1, 1)
    assert L.nlse2shoc_create(ctypes.byref(H), 1, n, h, 1.0, 1.0, None, 0, 0) == _lib.EINVAL  # N < 5
    n = (ctypes.c_int64 * 3)(8, 1, 1)
    assert L.nlse2shoc_create(ctypes.byref(H), 1, n, h, -1.0, 1.0, None, 0, 0) == _lib.EINVAL  # a <= 0
    assert L.nlse2shoc_create(ctypes.byref(H), 4, n, h, 1.0, 1.0, None, 0, 0) == _lib.EINVAL  # dims
    n2 = (ctypes.c_int64 * 3)(8, 3, 1)
    assert L.nlse2shoc_create(ctypes.byref(H), 1, n2, h, 1.0, 1.0, None, 0, 0) == _lib.EINVAL  # unused axis != 1
    assert H.value is None
    # the optional workspace / layout calls validate their handle before anything else
    assert L.nlse2shoc_set_workspace(None, None, 0) == _lib.EINVAL
    assert L.nlse2shoc_stage_workspace_bytes(None) == 0
    p3 = (ctypes.c_int64 * 3)()
    assert L.nlse2shoc_padded_layout(None, p3, p3) == _lib.EINVAL
    assert L.nlse2shoc_rk4_padded(None, None, 1e-3, 1, None) == _lib.EINVAL


def test_product_package_never_imports_oracle():
    """The product path must not route through the oracle (or any CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_1109_1027_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dp, f)).read()
                code = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
                code = re.sub(r"(#|//).*", "", code)
                code = re.sub(r'"""(.|\n)*?"""', "", code)
                assert "oracle" not in code.lower(), f
                assert "icgen" not in code, f


def test_missing_library_fails_loudly(tmp_path):
    """No fallback: with the shared library absent, the first call raises ImportError naming
    the missing file (checked in a fresh interpreter)."""
    import subprocess
    import sys

    missing = tmp_path / "libnlse2shoc.so"
    code = ("import paper_1109_1027_b200 as nl\n"
            "try:\n    nl.nlse2shoc_version()\nexcept ImportError as e:\n    print('IMPORTERROR', e)\n")
    env = dict(os.environ, NLSE_LIB=str(missing))
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True, timeout=120)
    assert "IMPORTERROR" in r.stdout and str(missing) in r.stdout, r.stdout + r.stderr
