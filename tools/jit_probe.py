"""error_norms at 64^2 macro x 64^2 micro (17.9 M micro DoFs) with the tapes compiled at run
time (NVRTC, jit.cu) and interpreted (TS_JIT=0): wall time per call (best of 3, after a
warm-up that includes the one-time compile) and the tape path.  Run under ncu for kernel
times (k_error_norms_jit vs k_error_norms)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_2103_17040_b200 import abi  # noqa: E402
from test_gpu_mms import MMS_INI  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
ini = MMS_INI.format(n=n, m=n)
g = abi.Context(ini, mms=True)
rng = np.random.default_rng(7)
u, w = rng.standard_normal(g.n_macro), rng.standard_normal(g.n_macro)
V = rng.standard_normal((g.n_macro, g.n_micro))
g.close()
res = {}
for mode in ("1", "0"):
    os.environ["TS_JIT"] = mode
    t0 = time.perf_counter()
    e = abi.error_norms(ini, u, w, V)
    first = time.perf_counter() - t0
    best = 1e30
    for _ in range(3):
        t0 = time.perf_counter()
        e = abi.error_norms(ini, u, w, V)
        best = min(best, time.perf_counter() - t0)
    res[mode] = e
    print(f"TS_JIT={mode}: first call {first:.3f} s, best {best:.3f} s, path: {abi.jit_status()}", flush=True)
print("bitwise equal:", bool(np.array_equal(res["0"], res["1"])))
