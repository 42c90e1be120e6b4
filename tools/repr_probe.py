"""Operator representation A/B on one config (north star (2): "CSR index set with per-problem
values, or matrix-free from the coefficient tensors — choose by measured bytes per DoF"):
builds the context once per variant (environment knobs), 2 warm-up + 3 timed fixed-point
solves, prints micro PCG DoF*it/s (device events), sweeps, and the bytes the variant's
operator representation holds per DoF.

    python tools/repr_probe.py c4 "TS_GEN_Q2T=0" "TS_GEN_Q2T=1"
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2103_17040_b200 import abi, configs  # noqa: E402

KERNELS = {0: "column strips", 1: "column pairs", 2: "generic streaming", 3: "Q2 class-compact CSR",
           4: "Q2 coefficient tensors", 5: "3D cluster"}


def main(name, variants):
    cfg = configs.CONFIGS[name]
    for var in variants:
        env = dict(kv.split("=", 1) for kv in var.split(",") if kv)
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        try:
            g = abi.Context(cfg.ini(), cfg.ext())
            for _ in range(2):
                g.solve(download=False)
            reps = [g.solve(download=False) for _ in range(3)]
            dofit = sum(r["micro_dof_iters"] for r in reps)
            ms = sum(r["micro_ms"] for r in reps)
            kern = g.info["micro_kernel"]
            rep_bytes = {2: cfg.csr_bytes_per_dof, 3: None, 4: cfg.tensor_bytes_per_dof}.get(kern)
            print(json.dumps(dict(config=name, variant=var, kernel=KERNELS.get(kern, kern),
                                  dof_it_per_s=dofit / (ms * 1e-3), micro_ms_per_solve=ms / 3,
                                  total_ms_per_solve=sum(r["total_ms"] for r in reps) / 3,
                                  sweeps=reps[-1]["sweeps"], micro_dof_iters=reps[-1]["micro_dof_iters"],
                                  setup_ms=g.info["setup_ms"], device_bytes=g.info["device_bytes"],
                                  alg_bytes_per_dof=rep_bytes)), flush=True)
            g.close()
        finally:
            for k, v in old.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:] or [""])
