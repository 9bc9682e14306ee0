"""Host wall clock of the three phases of ts_operator_apply (host -> device with
c128 -> c64 conversion, MVM, device -> host) at a config, for several transfer
worker counts. Usage: python tools/e2e_phases.py [config] [threads ...]"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if os.environ.get("TSK_E2E_CHILD") != "1":
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    for t in sys.argv[2:] or ["16"]:
        env = dict(os.environ, TSK_E2E_CHILD="1", TSK_DEBUG_TRANSFER="1", TSK_TRANSFER_THREADS=t)
        r = subprocess.run([sys.executable, __file__, name], env=env, capture_output=True, text=True)
        print(f"== {name}, {t} transfer threads")
        print("\n".join(ln for ln in (r.stdout + r.stderr).splitlines() if "ts_operator_apply" in ln or "call" in ln))
    sys.exit(0)

sys.path.insert(0, ROOT)
import time  # noqa: E402

import numpy as np  # noqa: E402

import paper_2406_17981_b200 as T  # noqa: E402
from paper_2406_17981_b200 import workloads as W  # noqa: E402

name = sys.argv[1]
op = W.make_operator(T, name)
n = op.info()["m"]
for v in W.CONFIGS[name][0]:
    n *= v
x = np.ones(n, dtype=np.complex128)
y = np.empty_like(x)
for i in range(4):
    t0 = time.perf_counter()
    op.apply(x, out=y)
    print(f"call {i}: {time.perf_counter() - t0:.4f} s", flush=True)
