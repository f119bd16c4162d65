"""Range-checked build (libnlse2shoc_checked.so, -DNLSE_CHECKED): every kernel family runs one
small case (scripts/checked_cases.py) and no global store of the 2D/3D stage kernels may fall
outside its buffer (output fields, neighbours' halo buffers of the fused exchange).  Stands in
for compute-sanitizer memcheck, which the GPU pool does not allow."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_checked_build_has_no_out_of_range_stores():
    so = os.path.join(ROOT, "paper_1109_1027_b200", "libnlse2shoc_checked.so")
    assert os.path.exists(so), "build() compiles the checked library"
    env = dict(os.environ, NLSE_LIB=so)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "checked_cases.py")], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "checked" in r.stdout
    assert "violations 0" in r.stdout, r.stdout[-2000:]
