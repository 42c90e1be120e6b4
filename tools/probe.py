"""Quick device probe: build + solve a config, print timings (development aid)."""
import json
import sys
import time

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2103_17040_b200 import abi, configs  # noqa: E402

for name in sys.argv[1:] or ["c2"]:
    cfg = configs.CONFIGS[name]
    t0 = time.time()
    tab = cfg.table()
    t1 = time.time()
    ctx = abi.Context(cfg.ini(), cfg.ext())
    t2 = time.time()
    out = ctx.solve(download=False)
    t3 = time.time()
    rate = out["micro_dof_iters"] / (out["micro_ms"] * 1e-3)
    print(json.dumps(dict(cfg=name, table_s=t1 - t0, ctx_s=t2 - t1, solve_s=t3 - t2, info=ctx.info,
                          sweeps=out["sweeps"], micro_ms=out["micro_ms"], macro_ms=out["macro_ms"],
                          total_ms=out["total_ms"], dof_iters=out["micro_dof_iters"], rate=rate,
                          roof_csr=rate * cfg.csr_bytes_per_dof / 6538.9e9,
                          it_max=out["micro_iters_max"], it_min=out["micro_iters_min"],
                          hist=list(out["history"]))), flush=True)
