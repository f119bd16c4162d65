"""GPU: a seeded random sweep of small problems (dims, sizes around tile multiples, BC,
potential kind, dtype, variant, scheme) crossed with execution-path options, the caller-owned
workspace, the padded layout, failure detection and loopback slabs, against the oracle
(scripts/fuzz_parity.py; 2100 cases over seeds 1-4 are recorded in profiles/r02/)."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_random_sweep_matches_oracle():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "fuzz_parity.py"), "200", "5"], cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    last = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else ""
    assert r.returncode == 0 and '"failed": 0' in last, (last, r.stderr[-2000:])


def test_random_sweep_under_the_range_checked_build():
    """The same sweep (another seed) on libnlse2shoc_checked.so: parity, and no out-of-buffer
    store in any of the random shapes / options (stands in for compute-sanitizer memcheck)."""
    so = os.path.join(ROOT, "paper_1109_1027_b200", "libnlse2shoc_checked.so")
    assert os.path.exists(so), "build() compiles the checked library"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "fuzz_parity.py"), "150", "6"], cwd=ROOT,
                       env=dict(os.environ, NLSE_LIB=so), capture_output=True, text=True, timeout=600)
    last = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else ""
    assert r.returncode == 0 and '"failed": 0' in last and '"checked_violations": 0' in last, (last, r.stderr[-2000:])
