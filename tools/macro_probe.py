"""A/B of the macro solve paths on one config (development aid): cluster (default for macro
grids beyond one SM) vs the cooperative CSR CG (TS_MACRO_CLUSTER=0), each in its own process.
    python tools/macro_probe.py c3 [macro_n micro_n]"""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(name, mn, un, out):
    sys.path.insert(0, ROOT)
    from paper_2103_17040_b200 import abi, configs
    cfg = configs.CONFIGS[name]
    if mn:
        cfg = cfg.resized(int(mn), int(un))
    ctx = abi.Context(cfg.ini(), cfg.ext())
    ctx.solve(download=False)
    r = ctx.solve()
    np.savez(out, u=r["u"], w=r["w"], V=r["V"], hist=r["history"])
    print(json.dumps(dict(sweeps=r["sweeps"], macro_ms=r["macro_ms"], micro_ms=r["micro_ms"], total_ms=r["total_ms"])))


def main():
    if sys.argv[1] == "--child":
        child(*sys.argv[2:])
        return
    name = sys.argv[1]
    mn, un = (sys.argv[2], sys.argv[3]) if len(sys.argv) > 3 else ("", "")
    res = {}
    for tag, env in (("cluster", {}), ("coop", {"TS_MACRO_CLUSTER": "0"})):
        out = f"/tmp/macro_probe_{tag}.npz"
        p = subprocess.run([sys.executable, __file__, "--child", name, mn, un, out], env=dict(os.environ, **env),
                           capture_output=True, text=True, timeout=600)
        print(tag, p.stdout.strip(), p.stderr[-300:])
        res[tag] = np.load(out)
    a, b = res["cluster"], res["coop"]
    for k in ("u", "V"):
        print(k, "rel diff", float(np.linalg.norm(a[k] - b[k]) / max(np.linalg.norm(b[k]), 1e-300)))


if __name__ == "__main__":
    main()
