"""Wall-clock breakdown of the C-ABI end-to-end path (ctx build, solve, download, destroy)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_17040_b200 import abi, configs  # noqa: E402

cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
tab = cfg.table()
pu, pw, pV = abi.PinnedArray((cfg.n_macro,)), abi.PinnedArray((cfg.n_macro,)), abi.PinnedArray((cfg.n_macro, cfg.n_micro))
ext = cfg.ext()
for rep in range(3):
    t0 = time.perf_counter()
    c = abi.Context(cfg.ini(), ext)
    t1 = time.perf_counter()
    r = c.solve(download=False)
    t2 = time.perf_counter()
    c.state(pu.array, pw.array, pV.array)
    t3 = time.perf_counter()
    c.close()
    t4 = time.perf_counter()
    print(f"rep {rep}: create {t1-t0:.3f}s (device setup {c.info['setup_ms']:.1f} ms) solve {t2-t1:.3f}s "
          f"(device {r['total_ms']:.1f} ms) download {t3-t2:.3f}s destroy {t4-t3:.3f}s", flush=True)
