"""Measurement of the SURVEY.md §8f rank-1 row (error_norms + the manufactured-solution
convergence sweep) against the reference on the same box: `twoscale mms --sweep ...`
(mms.cpp:384-418) as the device pipeline (ts_mms_sweep_ini: derive_data on the host, solve and
error norms on the device) and as the unmodified reference (oracle/_ref) at all host threads;
plus error_norms alone (mms.cpp:247-377) for a given host state.  Prints one JSON line per case
and checks the numbers agree (rows: rtol 1e-8 on the norms; error_norms: rtol 1e-12)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2103_17040_b200 import abi  # noqa: E402
from oracle import ref  # noqa: E402  (CPU reference arm: measurement only)

sys.path.insert(0, os.path.join(ROOT, "tests"))
from test_gpu_mms import MMS_INI  # noqa: E402


def timed(f, *a, **k):
    t0 = time.perf_counter()
    out = f(*a, **k)
    return out, time.perf_counter() - t0


def main():
    threads = os.cpu_count() or 1
    for ns in ([8, 11, 16], [16, 32, 48]):
        ini = MMS_INI.format(n=ns[0], m=ns[0])
        abi.mms_sweep(ini, ns[:1])  # warm-up (module load, allocator)
        dev, t_dev = timed(abi.mms_sweep, ini, ns)
        rf, t_ref = timed(ref.mms_sweep, ini, ns, threads)
        ok = bool(np.array_equal(dev[:, :3], rf[:, :3]) and np.allclose(dev[:, 5:9], rf[:, 5:9], rtol=1e-8))
        print(json.dumps(dict(case="convergence_sweep", ns=ns, device_s=t_dev, reference_s=t_ref,
                              reference_threads=threads, speedup=t_ref / t_dev, parity=ok,
                              e_uw=list(dev[:, 5]), e_v=list(dev[:, 7]))), flush=True)
    n = 64
    ini = MMS_INI.format(n=n, m=n)
    g = abi.Context(ini, mms=True)
    rng = np.random.default_rng(7)
    u, w = rng.standard_normal(g.n_macro), rng.standard_normal(g.n_macro)
    V = rng.standard_normal((g.n_macro, g.n_micro))
    g.close()
    abi.error_norms(ini, u, w, V)
    e_dev, t_dev = timed(abi.error_norms, ini, u, w, V)
    e_ref, t_ref = timed(ref.error_norms, ini, u, w, V, threads)
    print(json.dumps(dict(case="error_norms", macro=n, micro=n, dofs=int(V.size), device_s=t_dev,
                          reference_s=t_ref, reference_threads=threads, speedup=t_ref / t_dev,
                          parity=bool(np.allclose(e_dev, e_ref, rtol=1e-12)),
                          note="device time includes INI parse, derive_data and the H2D of V")), flush=True)


if __name__ == "__main__":
    main()
