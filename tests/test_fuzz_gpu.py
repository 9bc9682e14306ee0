"""Bounded run of the oracle fuzz (tools/fuzz_oracle.py): random shapes with d = 1..5,
length-1 / prime / power-of-two / long axes, every symmetry mode, nonzero padding value,
both storage modes and precisions, device multi-RHS applies and branch partitions, and 3x3
dyadic operators — each case against the CPU oracle (complex128: rel-L2 <= 1e-12,
complex64: <= 1e-5, BASELINE.json's tolerances)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("seed", [5, 17])
def test_fuzz_against_oracle(seed):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "fuzz_oracle.py"), "30", str(seed)],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "0 failure(s)" in r.stdout
