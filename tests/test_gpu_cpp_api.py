"""The host C++ mirror (include/twoscale/*.hpp) used exactly like the reference's CLI
(examples/cpp_api_demo.cpp) reproduces the reference solution."""
import json
import os
import subprocess

import numpy as np
import pytest

from paper_2103_17040_b200 import configs

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEMO = os.path.join(ROOT, "paper_2103_17040_b200", "bin", "cpp_api_demo")


def test_cpp_api_matches_reference(tmp_path, ref_mod):
    cfg = configs.CONFIGS["c2"].reduced().resized(8, 12)
    ini = tmp_path / "case.ini"
    ini.write_text(cfg.ini())
    out = tmp_path / "state.bin"
    p = subprocess.run([DEMO, str(ini), str(out), str(tmp_path)], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr
    info = json.loads(p.stdout)
    r = ref_mod.RefContext(cfg.ini(), 1)
    s = r.solve(outer_tol=cfg.outer_tol)
    raw = np.fromfile(out, dtype=np.float64)
    nM, nm = r.n_macro, r.n_micro
    u, w, V = raw[:nM], raw[nM:2 * nM], raw[2 * nM:].reshape(nM, nm)
    assert info["sweeps"] == s["sweeps"] and info["converged"] == 1 and info["cg_converged"] == 1
    assert info["micro_nnz"] == r.micro_nnz and info["w_pinned"] == 1
    for a, b in ((u, s["u"]), (V, s["V"])):
        assert np.linalg.norm(a - b) / np.linalg.norm(b) <= 1e-8
    # cmd_solve's VTK files from the C++ mirror == the reference writer on the same state
    ref_mod.write_vtk(cfg.ini(), u, w, V, 0.1, tmp_path / "ref_macro.vtk", tmp_path / "ref_micro.vtk")
    assert (tmp_path / "macro.vtk").read_bytes() == (tmp_path / "ref_macro.vtk").read_bytes()
    assert (tmp_path / "micro.vtk").read_bytes() == (tmp_path / "ref_micro.vtk").read_bytes()


def test_cpp_api_reports_degenerate_map(tmp_path):
    ini = configs.CONFIGS["c1"].resized(2, 4).ini().replace(
        configs.C1_ZETA[0], "-y0")
    f = tmp_path / "bad.ini"
    f.write_text(ini)
    p = subprocess.run([DEMO, str(f), str(tmp_path / "o.bin")], capture_output=True, text=True, timeout=120)
    assert p.returncode == 3 and "degenerate map in cache build" in p.stderr
