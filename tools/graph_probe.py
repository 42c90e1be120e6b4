"""Eager sweep loop vs the device-side (CUDA graph, conditional while node) loop on one
config: bitwise-equal u, w, V, histories and sweep counts expected; prints both timings.
    python tools/graph_probe.py c1 [c2 ...]      (development aid)"""
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(name):
    sys.path.insert(0, ROOT)
    from paper_2103_17040_b200 import abi, configs
    cfg = configs.CONFIGS[name]
    ctx = abi.Context(cfg.ini(), cfg.ext())
    for _ in range(3):
        ctx.solve(download=False)
    reps = [ctx.solve(download=False) for _ in range(5)]
    out = ctx.solve()
    h = {k: hashlib.sha256(out[k].tobytes()).hexdigest()[:16] for k in ("u", "w", "V", "history")}
    h.update(sweeps=out["sweeps"], dof=out["micro_dof_iters"], launches=out["gpu_launches"],
             total_ms=min(r["total_ms"] for r in reps), micro_ms=min(r["micro_ms"] for r in reps),
             macro_ms=min(r["macro_ms"] for r in reps))
    print(json.dumps(h))


def main():
    if sys.argv[1] == "--child":
        child(sys.argv[2])
        return
    bad = 0
    for name in sys.argv[1:]:
        res = {}
        for g in ("0", "1"):
            p = subprocess.run([sys.executable, __file__, "--child", name], env=dict(os.environ, TS_GRAPH=g),
                               capture_output=True, text=True, timeout=600)
            res[g] = json.loads(p.stdout.strip().splitlines()[-1]) if p.returncode == 0 else {"error": p.stderr[-500:]}
        keys = ("u", "w", "V", "history", "sweeps", "dof")
        same = all(res["0"].get(k) == res["1"].get(k) for k in keys)
        bad += not same
        print(name, "IDENTICAL" if same else "DIFFERENT", json.dumps(res))
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
