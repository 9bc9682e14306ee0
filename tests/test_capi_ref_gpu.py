"""The reference's own C-ABI suite (/root/reference/proj/tests/capi/test_capi.cpp,
compiled unmodified by tests/capi/Makefile against include/toesplit.h with a
doctest-compatible shim, linked to this repo's libtoesplit.so.1) run as a test.
The binary is built in the build container (where the reference sources are)
by __graft_entry__.build() and travels to the GPU box with the tree.
"""
import os
import subprocess
import tempfile

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
BIN = os.path.join(HERE, "capi", "_build", "test_capi")


def _run():
    if not os.path.exists(BIN):
        pytest.skip("tests/capi/_build/test_capi not built (needs /root/reference at build time)")
    with tempfile.TemporaryDirectory() as td:  # the suite writes its JSON / TSKF files to cwd
        return subprocess.run([BIN], cwd=td, capture_output=True, text=True, timeout=300)


def test_reference_capi_suite_links_this_library():
    if not os.path.exists(BIN):
        pytest.skip("tests/capi/_build/test_capi not built")
    out = subprocess.run(["ldd", BIN], capture_output=True, text=True).stdout
    line = [ln for ln in out.splitlines() if "libtoesplit.so.1" in ln]
    assert line and os.path.realpath(line[0].split("=>")[1].split("(")[0].strip()) == \
        os.path.realpath(os.path.join(HERE, "..", "paper_2406_17981_b200", "libtoesplit.so.1"))


@pytest.mark.gpu
def test_reference_capi_suite_passes():
    r = _run()
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "6 passed | 0 failed" in r.stdout
