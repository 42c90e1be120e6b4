"""Per-config device throughput table (development record, not the driver's bench line).

For each BASELINE config: build the device context, 2 warm-up solves, 3 timed solves;
micro PCG DoF*it/s from CUDA events, two-scale solve time, CSR-roofline fraction; and
the reference cg_solve (oracle/_ref, all host threads) on a sample of the same
config's micro systems (assembled by the C oracles) for comparison.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2103_17040_b200 import abi, configs  # noqa: E402


def _hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]) * 1e9
    except Exception:
        return 6650e9  # B200_PROFILING.md fallback


HBM = _hbm()


def cpu_sample(cfg, n_sys=64):
    from oracle import port, ref
    threads = os.cpu_count() or 1
    if cfg.generic:
        o = port.GenOracleContext(cfg)
        rp, ci = o.micro_pattern()
        rhs = lambda i: 0.05 * o.rhs_parts(i)[0]  # noqa: E731
    else:
        o = port.OracleContext(cfg)
        rp, ci = o.micro_pattern()
        rhs = lambda i: 0.05 * o.rhs_parts(i)[1]  # noqa: E731
    m = cfg.macro_n
    interior = [j * (m + 1) + i for j in range(1, m) for i in range(1, m)]
    nodes = np.random.default_rng(0).choice(interior, size=min(n_sys, len(interior)), replace=False)
    vals = np.stack([o.micro_values(int(i)) for i in nodes])
    b = np.stack([rhs(int(i)) for i in nodes])
    _, it, secs = ref.batched_cg(rp, ci, vals, b, np.zeros_like(b), cfg.inner_tol, 20000, threads)
    return float(o.n_micro) * it.sum() / secs, threads


def main(names):
    rows = []
    for name in names:
        cfg = configs.CONFIGS[name]
        abi.Context(cfg.ini(), cfg.ext()).close()  # warm-up build (module load, first allocations)
        ctx = abi.Context(cfg.ini(), cfg.ext())    # setup_ms below is this second, steady build
        for _ in range(2):
            ctx.solve(download=False)
        reps = [ctx.solve(download=False) for _ in range(3)]
        dof = sum(r["micro_dof_iters"] for r in reps)
        micro_s = sum(r["micro_ms"] for r in reps) * 1e-3
        total_s = sum(r["total_ms"] for r in reps) * 1e-3 / 3
        rate = dof / micro_s
        cpu, threads = cpu_sample(cfg) if "--no-cpu" not in sys.argv else (float("nan"), 0)
        row = dict(config=name, workload=cfg.description, micro_dofs=cfg.n_micro, problems=cfg.n_macro,
                   sweeps=reps[-1]["sweeps"], rate=rate, alg_roofline=rate * cfg.alg_bytes_per_dof / HBM,
                   b_alg=cfg.alg_bytes_per_dof, micro_kernel=ctx.info["micro_kernel"],
                   two_scale_solve_s=total_s, setup_ms=ctx.info["setup_ms"], cpu_ref_rate=cpu,
                   cpu_threads=threads, speedup_vs_cpu=rate / cpu)
        rows.append(row)
        print(json.dumps(row), flush=True)
        ctx.close()
    print("\n| config | micro PCG DoF·it/s | × HBM roofline at B_alg | two-scale solve (s) | setup (ms) | ref cg_solve DoF·it/s (threads) | × |")
    print("|---|---|---|---|---|---|---|")
    for r in rows:
        print(f"| {r['config']} | {r['rate']:.3e} | {r['alg_roofline']:.2f} ({r['b_alg']:.2f} B) | {r['two_scale_solve_s']:.3f} | "
              f"{r['setup_ms']:.1f} | "
              f"{r['cpu_ref_rate']:.2e} ({r['cpu_threads']}) | {r['speedup_vs_cpu']:.0f} |")


if __name__ == "__main__":
    names = [a for a in sys.argv[1:] if not a.startswith("--")]
    main(names or ["c1", "c2", "c3", "c4", "c5"])
