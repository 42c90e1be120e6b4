"""Regenerates tests/golden/*.npz from the REFERENCE itself (oracle/_ref, built from
/root/reference/proj/src by oracle/Makefile).  Run in the build container:

    python tests/golden/make_golden.py

The fixtures are small on purpose; they let the oracle and the B200 path be checked
against reference outputs where /root/reference (and hence oracle/_ref) is absent.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ref  # noqa: E402
from paper_2103_17040_b200 import configs  # noqa: E402

CASES = {
    "c1_ref_4x6": configs.CONFIGS["c1"].reduced().resized(4, 6),
    "c2_ref_6x8": configs.CONFIGS["c2"].reduced().resized(6, 8),
    "c1_ref_16x16": configs.CONFIGS["c1"].reduced(),
}


def main():
    for name, cfg in CASES.items():
        r = ref.RefContext(cfg.ini(), 1)
        nodes = np.array(sorted({0, 1, r.n_macro // 3, r.n_macro // 2, r.n_macro - 1}), np.int32)
        rp, ci = r.micro_pattern()
        out = dict(ini=np.array(cfg.ini()), macro_n=cfg.macro_n, micro_n=cfg.micro_n, nodes=nodes,
                   micro_row_ptr=rp, micro_col_idx=ci)
        out["micro_values"] = np.stack([r.micro_values(int(i)) for i in nodes])
        out["robin_in"] = np.stack([r.micro_rhs(int(i), 1.0, 0.0) for i in nodes])
        cache = [r.node_cache(int(i)) for i in nodes]
        out["cache_cells"] = np.stack([c for c, _ in cache])
        out["cache_faces"] = np.stack([f for _, f in cache])
        for which, tag in enumerate(("Au", "Aw", "M0")):
            mrp, mci, mv = r.macro_matrix(which)
            out[tag] = mv
        out["macro_row_ptr"], out["macro_col_idx"] = mrp, mci
        d, v = r.dirichlet(0)
        out["dirichlet_u"] = d
        s = r.solve(outer_tol=cfg.outer_tol)
        for k in ("u", "w", "V", "history"):
            out[k] = s[k]
        out["sweeps"] = s["sweeps"]
        Vs, its, _ = r.micro_sweep(np.full(r.n_macro, 0.05), np.zeros(r.n_macro))
        out["V_fixed_u"] = Vs
        out["iters_fixed_u"] = its
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
        print(name, r.n_macro, r.n_micro, s["sweeps"])
    # legacy VTK of the reference solution (vtk.cpp:36-85, tools/twoscale.cpp:139-143)
    import gzip
    import tempfile
    g = np.load(os.path.join(HERE, "c1_ref_4x6.npz"))
    with tempfile.TemporaryDirectory() as td:
        mp, up = os.path.join(td, "macro.vtk"), os.path.join(td, "micro.vtk")
        ref.write_vtk(str(g["ini"]), g["u"], g["w"], g["V"], 0.25, mp, up)
        for src, tag in ((mp, "macro"), (up, "micro")):
            with open(src, "rb") as f, gzip.GzipFile(os.path.join(HERE, f"vtk_c1_ref_4x6_{tag}.vtk.gz"), "wb", mtime=0) as o:
                o.write(f.read())
    # SPEC.md:345 known-answer CG
    rp = np.array([0, 2, 5, 7], np.int32)
    ci = np.array([0, 1, 0, 1, 2, 1, 2], np.int32)
    v = np.array([2.0, -1, -1, 2, -1, -1, 2])
    x, conv, it, res, _ = ref.cg_solve(rp, ci, v, np.ones(3), np.zeros(3), 1e-12, 50)
    np.savez_compressed(os.path.join(HERE, "cg_3x3.npz"), row_ptr=rp, col_idx=ci, vals=v, b=np.ones(3), x=x,
                        iterations=it)


if __name__ == "__main__":
    main()
