"""Bitwise A/B of two library builds: one full fixed_point_solve per config, hashes of
u, w, V, the residual history and the sweep count.  Usage (on the GPU box):

    python tools/ab_bitwise.py ab/base.so ab/new.so c1 c2 c3 ...

Each library runs in its own process (TS_B200_LIB), so the comparison is between builds,
not between runs of one build."""
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(cfg_name):
    sys.path.insert(0, ROOT)
    from paper_2103_17040_b200 import abi, configs
    cfg = configs.CONFIGS[cfg_name]
    ctx = abi.Context(cfg.ini(), cfg.ext())
    out = ctx.solve()
    h = {k: hashlib.sha256(out[k].tobytes()).hexdigest()[:16] for k in ("u", "w", "V", "history")}
    h["sweeps"] = out["sweeps"]
    h["micro_dof_iters"] = out["micro_dof_iters"]
    print(json.dumps(h))


def main():
    if sys.argv[1] == "--child":
        child(sys.argv[2])
        return
    libs = [a for a in sys.argv[1:] if a.endswith(".so")]
    cfgs = [a for a in sys.argv[1:] if not a.endswith(".so")]
    bad = 0
    for c in cfgs:
        res = []
        for lib in libs:
            env = dict(os.environ, TS_B200_LIB=os.path.abspath(lib))
            p = subprocess.run([sys.executable, __file__, "--child", c], env=env, capture_output=True, text=True)
            res.append(json.loads(p.stdout.strip().splitlines()[-1]) if p.returncode == 0 else {"error": p.stderr[-400:]})
        same = all(r == res[0] for r in res)
        bad += not same
        print(f"{c}: {'IDENTICAL' if same else 'DIFFERENT'} {res}")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
