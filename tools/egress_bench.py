"""Micro-state egress timing: write_vtk_micro of a solved config.

Per config: device solve, then
  * ts_write_vtk_micro ASCII to a file and to /dev/null (formatting without the disk),
  * ts_write_vtk_micro BINARY to a file,
  * with --ref and a reference-expressible config: ts_download_state + the reference's
    write_vtk_micro (oracle/_ref, single-threaded ostream) on the same state, and a
    byte comparison of the two ASCII files when the map has no transcendental terms.
Prints one JSON line per config.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2103_17040_b200 import abi, configs  # noqa: E402


def timed(fn):
    t0 = time.perf_counter()
    fn()
    return time.perf_counter() - t0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["c2", "c3"])
    ap.add_argument("--ref", action="store_true", help="also time the reference writer (tape maps only)")
    ap.add_argument("--dir", default="/tmp/egress")
    ap.add_argument("--scale", type=float, default=0.5)
    a = ap.parse_args()
    os.makedirs(a.dir, exist_ok=True)
    for name in a.configs:
        cfg = configs.CONFIGS[name]
        ctx = abi.Context(cfg.ini(), cfg.ext())
        ctx.solve(download=False)
        n_points = ctx.n_macro * ctx.n_micro
        row = dict(config=name, points=n_points, threads=os.cpu_count())
        f_ascii = os.path.join(a.dir, f"{name}_micro.vtk")
        f_bin = os.path.join(a.dir, f"{name}_micro_bin.vtk")
        row["ascii_null_s"] = timed(lambda: ctx.write_vtk_micro("/dev/null", a.scale))
        row["ascii_file_s"] = timed(lambda: ctx.write_vtk_micro(f_ascii, a.scale))
        row["ascii_bytes"] = os.path.getsize(f_ascii)
        row["binary_file_s"] = timed(lambda: ctx.write_vtk_micro(f_bin, a.scale, binary=True))
        row["binary_bytes"] = os.path.getsize(f_bin)
        row["ascii_MB_per_s"] = row["ascii_bytes"] / row["ascii_file_s"] / 1e6
        row["binary_MB_per_s"] = row["binary_bytes"] / row["binary_file_s"] / 1e6
        if a.ref and cfg.map in ("c1", "c2"):
            from oracle import ref
            f_ref = os.path.join(a.dir, f"{name}_micro_ref.vtk")
            t0 = time.perf_counter()
            st = ctx.state()
            t1 = time.perf_counter()
            ref.write_vtk(cfg.ini(), st["u"], st["w"], st["V"], a.scale, None, f_ref)
            t2 = time.perf_counter()
            row["ref_download_s"] = t1 - t0
            row["ref_write_s"] = t2 - t1
            row["ref_total_s"] = t2 - t0
            row["speedup_ascii_vs_ref"] = row["ref_total_s"] / row["ascii_file_s"]
            with open(f_ref, "rb") as fa, open(f_ascii, "rb") as fb:
                same = True
                while True:
                    x, y = fa.read(1 << 24), fb.read(1 << 24)
                    if x != y:
                        same = False
                        break
                    if not x:
                        break
            row["ascii_identical_to_ref"] = same
            os.remove(f_ref)
        for f in (f_ascii, f_bin):
            os.remove(f)
        ctx.close()
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
