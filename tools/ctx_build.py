"""One context build of a BASELINE config (for ncu captures of the setup kernels):
    python tools/ctx_build.py c5"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2103_17040_b200 import abi, configs  # noqa: E402

cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c5"]
g = abi.Context(cfg.ini(), cfg.ext())
print(g.info["setup_ms"])
