"""The one-process multi-GPU operator (ts_operator_create_split_multi) with
P = 2, 4, 8 parts on the single GPU of a test box: NCCL is replaced by the
test-only single-process stand-in tests/nccl_mock (TSK_NCCL_LIB, and
TSK_ALLOW_SHARED_DEVICE=1 to put several parts on one device), so the
library's own orchestration runs as on P GPUs — partition operators, the x
broadcast into per-part buffers, the per-component reduce issued from the
root-level pass hooks on a second stream, the event ordering between calls,
and the host ABI path through the multi-GPU operator. Runs in a subprocess
(the NCCL loader and the switch are read once per process)."""
import os
import subprocess
import sys
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MOCK = os.path.join(ROOT, "tests", "nccl_mock", "_build", "libnccl_mock.so")

SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import paper_2406_17981_b200 as T, oracle
out = {{}}
O = oracle.Oracle()
cases = [("dyadic", [16, 16, 32], T.C64), ("dyadic", [8, 6, 16], T.C128), ("scalar", [8, 4, 8, 16], T.C64)]
for ci, (kind, levels, prec) in enumerate(cases):
    if kind == "dyadic":
        bg = T.BlockGenerator.dyadic(levels); m = 3
    else:
        g = T.Generator.random(levels, 4, 1.0, T.SYM_GENERAL); bg = T.BlockGenerator.from_scalar(g); m = 1
    s = int(np.prod(levels))
    x = O.random_vector([m] + levels, 11, 0.5) if m > 1 else O.random_vector(levels, 11, 0.5)
    ref = T.Operator.split_ex(bg, precision=prec).apply(x)
    out[f"ref{{ci}}"] = ref
    dt = torch.complex64 if prec == T.C64 else torch.complex128
    for P in (2, 4, 8):
        if P > 2 ** len(levels):
            continue
        op = T.Operator.split_multi(bg, [0] * P, precision=prec)
        assert op.info()["ndevices"] == P
        xd = torch.from_numpy(x).to(dt).cuda(); yd = torch.empty_like(xd)
        for _ in range(3):  # repeated calls: buffers reused across calls
            op.apply_device(xd, yd)
        torch.cuda.synchronize()
        out[f"dev{{ci}}_{{P}}"] = yd.cpu().numpy().astype(np.complex128)
        out[f"host{{ci}}_{{P}}"] = op.apply(x)
np.savez({path!r}, **out)
"""


def test_multi_gpu_orchestration_with_nccl_stand_in():
    if not os.path.exists(MOCK):
        pytest.skip("tests/nccl_mock not built")
    from oracle import rel_l2

    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "y.npz")
        env = dict(os.environ, TSK_NCCL_LIB=MOCK, TSK_ALLOW_SHARED_DEVICE="1")
        r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT, path=path)], env=env,
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        z = dict(np.load(path))
    n = 0
    for key, y in z.items():
        if key.startswith("ref"):
            continue
        ci = key[3] if key.startswith("dev") else key[4]
        ref = z[f"ref{ci}"]
        tol = 1e-12 if ci == "1" else 1e-6
        assert rel_l2(y, ref) <= tol, (key, rel_l2(y, ref))
        n += 1
    assert n == 2 * (3 + 3 + 3)
