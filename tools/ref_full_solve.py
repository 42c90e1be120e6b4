"""End-to-end two-scale solve: the reference's fixed_point_solve (oracle/_ref, all host
threads) vs this library, on the same reference-expressible stand-in of a BASELINE config
(k = 0, D = I, symbolic config-2 map).  One-off record for profiles/.

    python tools/ref_full_solve.py c3     # the reference leg takes minutes on C3
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2103_17040_b200 import abi, configs  # noqa: E402
from oracle import ref  # noqa: E402  (CPU reference leg)


def main(name):
    cfg = configs.CONFIGS[name].reduced()
    ini = cfg.ini()
    threads = ref.hardware_threads()
    # ours: ctx build + device solve + download of u, w, V (through the C ABI)
    abi.Context(ini, cfg.ext(reference_expressible=True)).close()  # warm-up (module load, allocator)
    t0 = time.perf_counter()
    g = abi.Context(ini, cfg.ext(reference_expressible=True))
    t1 = time.perf_counter()
    out = g.solve(outer_tol=cfg.outer_tol)
    t2 = time.perf_counter()
    # reference: AssemblyContext build + fixed_point_solve at all host threads
    t3 = time.perf_counter()
    r = ref.RefContext(ini, threads)
    t4 = time.perf_counter()
    s = r.solve(outer_tol=cfg.outer_tol, workers=threads)
    t5 = time.perf_counter()
    rel = {k: float(np.linalg.norm(out[k] - s[k]) / np.linalg.norm(s[k])) for k in ("u", "V")}
    print(json.dumps(dict(config=cfg.name, threads=threads,
                          ours=dict(build_s=t1 - t0, solve_s=t2 - t1, total_s=t2 - t0, sweeps=out["sweeps"],
                                    micro_dof_iters=out["micro_dof_iters"]),
                          reference=dict(build_s=t4 - t3, solve_s=t5 - t4, total_s=t5 - t3, sweeps=s["sweeps"]),
                          speedup_total=(t5 - t3) / (t2 - t0), rel_diff=rel)), flush=True)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "c2")
