"""Parity of the B200 path against the C oracle for the BASELINE extensions the
reference cannot express (reaction k, tensor D, per-node tabulated A(x)).  The
oracle itself is pinned to the reference binary in tests/test_oracle_vs_ref.py."""
import os

import numpy as np
import pytest

from paper_2103_17040_b200 import abi, configs

pytestmark = pytest.mark.gpu

VAL_TOL = 1e-12
SOL_TOL = 1e-8


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def maxrel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


CASES = {
    "c1-full": configs.CONFIGS["c1"],
    "c2-small": configs.CONFIGS["c2"].resized(12, 16),
    "c3-small": configs.CONFIGS["c3"].resized(12, 16),
    "c3-ragged": configs.CONFIGS["c3"].resized(7, 11),
    "c3-bigmacro": configs.CONFIGS["c3"].resized(100, 4),   # macro CG on the cooperative grid kernel
    "c3-wide": configs.CONFIGS["c3"].resized(4, 64),        # the full 65-wide config-3 micro grid
    "c1-disc": configs.TwoScaleConfig("disc", 6, 20, "c1", reaction=("disc", 1.0, 10.0, 0.5, 0.5, 0.3)),
}


@pytest.fixture(scope="module", params=list(CASES))
def pair(request, port_mod):
    if not abi.device_ok():
        pytest.fail("no usable sm_100 device")
    cfg = CASES[request.param]
    return cfg, abi.Context(cfg.ini(), cfg.ext()), port_mod.OracleContext(cfg)


def test_caches_values_rhs(pair):
    cfg, g, o = pair
    rp, ci = g.micro_pattern()
    orp, oci = o.micro_pattern()
    assert np.array_equal(rp, orp) and np.array_equal(ci, oci)
    for node in sorted({0, 1, g.n_macro // 2, g.n_macro - 1}):
        gc, gf = g.node_cache(node)
        oc, of = o.node_cache(node)
        assert maxrel(gc, oc) <= VAL_TOL
        assert maxrel(gf, of) <= VAL_TOL
        assert maxrel(g.micro_values(node), o.micro_values(node)) <= VAL_TOL
        _, ri, ro = o.rhs_parts(node)
        assert maxrel(g.micro_rhs(node, 1.0, 0.0), ri) <= VAL_TOL
    for which in range(3):
        assert maxrel(g.macro_matrix(which)[2], o.macro_matrix(which)) <= VAL_TOL


def test_solve(pair):
    cfg, g, o = pair
    out = g.solve(outer_tol=cfg.outer_tol)
    ref = o.solve(outer_tol=cfg.outer_tol)
    assert out["sweeps"] == ref["sweeps"]
    for k in ("u", "w", "V"):
        assert rel(out[k], ref[k]) <= SOL_TOL, k
    assert out["micro_dof_iters"] == pytest.approx(ref["micro_dof_iters"], rel=0.02)


def test_validate_map_covers_every_quadrature_point(pair):
    """ts_validate_map (validate_diffeo at every point the solve uses)
    equals the min/max of det J over all nodes' cache rows."""
    cfg, g, o = pair
    ok, mn, mx, where = g.validate_map(lo=0.3 if cfg.map == "table" else 1e-6)
    dets = []
    for node in range(g.n_macro):
        c, f = o.node_cache(node)
        dets.append((c[:, :, 0].min(), c[:, :, 0].max(), f[:, :, 0].min(), f[:, :, 0].max()))
    dets = np.array(dets)
    assert mn == pytest.approx(min(dets[:, 0].min(), dets[:, 2].min()), rel=1e-12)
    assert mx == pytest.approx(max(dets[:, 1].max(), dets[:, 3].max()), rel=1e-12)
    assert ok
    if cfg.map == "table":
        assert mn >= 0.3  # the config-3 rejection sampling guarantee (BASELINE.json)


# Kernel-variant coverage: the column-pair kernel forced onto every compile-time width
# and strip height (it is the default only for 65-wide grids), and the single-column
# kernel forced onto the 65-wide grid.  Same oracle, same tolerances.
VARIANTS = [
    ("pair-33", configs.CONFIGS["c2"].resized(6, 32), {}),
    ("strips-33", configs.CONFIGS["c2"].resized(6, 32), {"TS_PCG_PAIR": "0"}),
    ("strips-17-halfwarps", configs.CONFIGS["c3"].resized(5, 16), {"TS_PCG_PAIR": "0"}),
    ("pair-17-R4", configs.CONFIGS["c3"].resized(5, 16), {"TS_PCG_PAIR": "1", "TS_PCG_ROWS": "4"}),
    ("pair-65-R5", configs.CONFIGS["c3"].resized(3, 64), {"TS_PCG_ROWS": "5"}),
    ("strips-65", configs.CONFIGS["c3"].resized(3, 64), {"TS_PCG_PAIR": "0"}),
    ("pair-65-cg1", configs.CONFIGS["c3"].resized(3, 64), {"TS_PCG_CG1": "1"}),  # single-reduction loop (opt-in)
]


@pytest.mark.parametrize("name,cfg,env", VARIANTS, ids=[v[0] for v in VARIANTS])
def test_kernel_variants(port_mod, monkeypatch, name, cfg, env):
    if not abi.device_ok():
        pytest.fail("no usable sm_100 device")
    for k in ("TS_PCG_PAIR", "TS_PCG_ROWS", "TS_PCG_CG1"):  # the case's own settings only
        monkeypatch.delenv(k, raising=False)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    g = abi.Context(cfg.ini(), cfg.ext())
    want = 0 if env.get("TS_PCG_PAIR") == "0" or (cfg.micro_n == 16 and "TS_PCG_PAIR" not in env) else 1
    assert g.info["micro_kernel"] == want
    if "TS_PCG_ROWS" in env:
        assert g.info["micro_rows"] == int(env["TS_PCG_ROWS"])
    o = port_mod.OracleContext(cfg)
    out = g.solve(outer_tol=cfg.outer_tol)
    ref = o.solve(outer_tol=cfg.outer_tol)
    assert out["sweeps"] == ref["sweeps"]
    for k in ("u", "w", "V"):
        assert rel(out[k], ref[k]) <= SOL_TOL, k


def test_bitwise_run_to_run_determinism():
    """Fixed reduction trees (warp DMMA sums, fixed-order partials, single-problem blocks):
    two solves of the same context give bitwise-identical u, w, V and histories, although
    the longest-first ticket order hands problems to blocks in a run-dependent order."""
    if not abi.device_ok():
        pytest.fail("no usable sm_100 device")
    cfg = configs.CONFIGS["c3"].resized(20, 64)
    g = abi.Context(cfg.ini(), cfg.ext())
    a = g.solve()
    b = g.solve()
    for k in ("u", "w", "V", "history"):
        assert np.array_equal(a[k], b[k]), k
    assert a["micro_dof_iters"] == b["micro_dof_iters"]


@pytest.mark.parametrize("name,macro_n,micro_n,env", [
    ("c4", 6, 32, {}),                      # Q2 2-CTA cluster kernel, block-pair mapping
    ("c4", 6, 32, {"TS_GEN_Q2B": "0"}),     # ... one class per warp
    ("c5", 6, 16, {"TS_GEN_ZFILL": "0"}),   # z-column 4-CTA cluster kernel alone
])
def test_cluster_kernels_are_deterministic(monkeypatch, name, macro_n, micro_n, env):
    """The cluster kernels' dot products are summed in a fixed order on every CTA (warp DMMA
    sums, rank-ordered exchange slots), so two solves give bitwise-identical states.  (Config
    5's default also runs the streaming kernel on the SMs 4-CTA clusters cannot use; both
    drain one ticket queue, so which kernel — which rounding — a problem gets is
    run-dependent there: equal to tolerance, not bitwise.  TS_GEN_ZFILL=0 removes that.)"""
    if not abi.device_ok():
        pytest.fail("no usable sm_100 device")
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    cfg = configs.CONFIGS[name].resized(macro_n, micro_n)
    g = abi.Context(cfg.ini(), cfg.ext())
    a = g.solve()
    b = g.solve()
    for k in ("u", "w", "V", "history"):
        assert np.array_equal(a[k], b[k]), k
    assert a["micro_dof_iters"] == b["micro_dof_iters"]


@pytest.mark.gpu
def test_pcg_control_arithmetic_is_exact(tmp_path):
    """The PCG loop's stop test (rr <= T, T from rel_threshold) and split division
    (div_recip/div_finish) are bitwise the plain sqrt(rr)/bnorm <= tol and rz_new/rz:
    tools/div_probe.cu checks 2.7e8 random divisions over the whole exponent range,
    random and special-valued (b, tol) thresholds, against the IEEE operations."""
    import subprocess
    exe = str(tmp_path / "div_probe")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                    "-I", os.path.join(root, "paper_2103_17040_b200", "csrc"), "-I", os.path.join(root, "include"),
                    os.path.join(root, "tools", "div_probe.cu"), "-o", exe], check=True, capture_output=True)
    p = subprocess.run([exe, "quick"], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0 and "div_probe OK" in p.stdout, p.stdout + p.stderr


@pytest.mark.parametrize("env", [{}, {"TS_PCG_PAIR": "0"}], ids=["pair-65-lagged", "strips-65"])
def test_indefinite_micro_systems(port_mod, monkeypatch, env):
    """A strongly negative reaction (k = -300) makes the micro operators indefinite: the
    batched PCG must stop each problem at p.Ap <= 0 (linalg.cpp:138-142) at the iteration
    the C oracle's cg_solve stops it, and report the first such system the way the
    reference does (solver.cpp:91-97).  Runs the lagged-stop-test pair kernel and the
    column-strip kernel on the 65-wide grid."""
    import dataclasses
    if not abi.device_ok():
        pytest.fail("no usable sm_100 device")
    monkeypatch.delenv("TS_PCG_PAIR", raising=False)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    cfg = dataclasses.replace(configs.CONFIGS["c3"].resized(2, 64), reaction=("const", -300.0))
    g = abi.Context(cfg.ini(), cfg.ext())
    u = np.linspace(0.02, 0.1, g.n_macro)
    w = np.zeros(g.n_macro)
    V, it, _, st = g.micro_solve(u, w, raise_on_fail=False)
    rp, ci = g.micro_pattern()
    first = None
    for i in range(g.n_macro):
        b = g.micro_rhs(i, u[i], w[i])
        _, conv, oit, _, indef = port_mod.cg_solve(rp, ci, g.micro_values(i), b, np.zeros_like(b), 1e-10, 20000)
        if indef:
            assert abs(int(it[i]) - oit) <= 1, (i, it[i], oit)
            first = i if first is None else first
        else:
            assert conv and abs(int(it[i]) - oit) <= 2, (i, it[i], oit)
    assert first is not None, "no indefinite system: raise |k|"
    assert st == abi.TS_ERR_SOLVER
    msg = abi.lib().ts_last_error().decode()
    assert msg == f"micro system {first}: CG detected negative curvature", msg


@pytest.mark.parametrize("name,macro_n,micro_n", [("c1", 16, 16), ("c2", 8, 32), ("c1", 80, 4)])
def test_device_sweep_loop_matches_eager(monkeypatch, name, macro_n, micro_n):
    """Sweeps 2.. as one CUDA graph with a conditional while node (k_sweep_control applies
    the stop test of solver.cpp:124-125 on the device) give bitwise the eager loop's u, w, V,
    residual history and sweep count — with the one-SM stencil macro solve and (80 x 80 macro
    grid) the cluster macro solve inside the graph; also with max_outer cutting the loop."""
    if not abi.device_ok():
        pytest.fail("no usable sm_100 device")
    cfg = configs.CONFIGS[name].resized(macro_n, micro_n)
    g = abi.Context(cfg.ini(), cfg.ext())
    for max_outer in (100, 4):
        outs = {}
        for mode in ("0", "1"):
            monkeypatch.setenv("TS_GRAPH", mode)
            outs[mode] = g.solve(outer_tol=cfg.outer_tol, max_outer=max_outer)
        a, b = outs["0"], outs["1"]
        assert a["sweeps"] == b["sweeps"] and a["converged"] == b["converged"]
        assert a["micro_dof_iters"] == b["micro_dof_iters"]
        for k in ("u", "w", "V", "history"):
            assert np.array_equal(a[k], b[k]), k

