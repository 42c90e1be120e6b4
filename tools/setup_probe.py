"""Context build (setup) time per BASELINE config: ts_ctx_info.setup_ms (device events around
the build's launches) and wall time of ts_ctx_create_ini, best of 3 after a warm-up build.

    python tools/setup_probe.py [c1 c2 ...]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2103_17040_b200 import abi, configs  # noqa: E402


def main(names):
    for name in names:
        cfg = configs.CONFIGS[name]
        ini, ext = cfg.ini(), cfg.ext()
        abi.Context(ini, ext).close()
        best_dev, best_wall = 1e30, 1e30
        for _ in range(3):
            t0 = time.perf_counter()
            c = abi.Context(ini, ext)
            wall = (time.perf_counter() - t0) * 1e3
            best_dev = min(best_dev, c.info["setup_ms"])
            best_wall = min(best_wall, wall)
            c.close()
        print(f"{name}: setup device {best_dev:.2f} ms, create wall {best_wall:.2f} ms", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(configs.CONFIGS))
