"""One context build + one fixed-point solve of a BASELINE config (for ncu captures):
    python tools/ctx_solve.py c4"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2103_17040_b200 import abi, configs  # noqa: E402

cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
g = abi.Context(cfg.ini(), cfg.ext())
r = g.solve(download=False)
print(r["sweeps"], r["micro_dof_iters"], r["micro_ms"])
