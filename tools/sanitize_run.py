"""Small solves that exercise every kernel family, for compute-sanitizer
(memcheck / racecheck / initcheck / synccheck):

    compute-sanitizer --tool racecheck --error-exitcode 1 python tools/sanitize_run.py

Kernels covered: map caches + assembly (setup), column-strip micro PCG (17 wide), column-pair
micro PCG (33 wide) and its lagged-stop-test variant (65 wide), the SMEM-stencil macro solve
and the cooperative CSR macro CG, class-compact Q2 and 3D generic PCG, sweep residual, macro
rhs, VTK egress.  (compute-sanitizer is closed on this round's GPU pool — runs under it
left GPUs needing a reset — so correctness evidence here is the parity suite, the bitwise
run-to-run determinism test and tools/ab_bitwise.py; this driver is for other machines.)"""
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2103_17040_b200 import abi, configs  # noqa: E402

CASES = [("c1", 4, 16), ("c2", 3, 32), ("c3", 2, 64), ("c4", 2, 32), ("c5", 2, 16)]


def main(names):
    for name, macro_n, micro_n in CASES:
        if names and name not in names:
            continue
        cfg = configs.CONFIGS[name].resized(macro_n, micro_n)
        ctx = abi.Context(cfg.ini(), cfg.ext())
        out = ctx.solve(max_outer=3)
        print(f"{name}@{macro_n}x{micro_n}: kernel {ctx.info['micro_kernel']} sweeps {out['sweeps']} "
              f"launches {out['gpu_launches']}", flush=True)
        if name == "c1":
            with tempfile.TemporaryDirectory() as d:
                ctx.write_vtk_micro(os.path.join(d, "m.vtk"))
        ctx.close()
    # the cooperative CSR macro CG (grids beyond one SM's SMEM use it; force it here)
    os.environ["TS_MACRO_STENCIL"] = "0"
    cfg = configs.CONFIGS["c1"].resized(4, 16)
    ctx = abi.Context(cfg.ini(), cfg.ext())
    out = ctx.solve(max_outer=3)
    print(f"c1@4x16 (CSR macro CG): sweeps {out['sweeps']}", flush=True)
    ctx.close()
    print("sanitize_run done")


if __name__ == "__main__":
    main(sys.argv[1:])
