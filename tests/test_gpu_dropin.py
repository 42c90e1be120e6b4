"""The drop-in claim, tested: oracle/ref_harness.cpp — a caller written against the
reference's public C++ API only (parse_config, make_problem, AssemblyContext, build_cache,
validate_diffeo, check_assumption6, cg_solve, fixed_point_solve, parallel_for,
resolve_worker_count, derive_data / convergence_sweep, write_vtk_*) — is compiled twice by
oracle/Makefile from the same source: against the reference (oracle/_ref) and, unchanged,
against this repo's include/twoscale headers linked to libtwoscale_b200.so (oracle/_mirror).
Both builds run the same calls here and must agree (values <= 1e-12, solutions <= 1e-8,
index structures and messages exactly)."""
import os

import numpy as np
import pytest

from paper_2103_17040_b200 import abi, configs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def both(ref_mod):
    if not abi.device_ok():
        pytest.fail("no usable sm_100 device")
    mir = ref_mod.mirror()
    if not os.path.exists(mir.LIB_PATH):
        pytest.fail(f"{mir.LIB_PATH} not built (make -C oracle mirror)")
    return ref_mod, mir


def maxrel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


# x-dependent Jacobian (config-2 family: A(x) y + bubble) and the config-1 map
MAPS = {"c2map": configs.CONFIGS["c2"].resized(6, 8), "c1map": configs.CONFIGS["c1"].reduced().resized(5, 6)}


@pytest.fixture(scope="module", params=list(MAPS))
def ctxs(request, both):
    ref_mod, mir = both
    cfg = MAPS[request.param].reduced() if MAPS[request.param].reaction else MAPS[request.param]
    return cfg, ref_mod.RefContext(cfg.ini(), 1), mir.RefContext(cfg.ini(), 1)


def test_build_cache_at_arbitrary_points(ctxs):
    """build_cache (mapping.cpp:79-129) at random macro points, cells and faces, through the
    mirror's build_cache -> ts_build_cache (kernel 1)."""
    cfg, r, m = ctxs
    pts = np.random.default_rng(7).random((33, 2))
    rc, rf = r.build_cache(pts)
    mc, mf = m.build_cache(pts)
    assert rc.shape == mc.shape and rf.shape == mf.shape
    assert maxrel(mc, rc) <= 1e-12 and maxrel(mf, rf) <= 1e-12
    _, rf2 = r.build_cache(pts[:5], with_cells=False)
    _, mf2 = m.build_cache(pts[:5], with_cells=False)
    assert maxrel(mf2, rf2) <= 1e-12


@pytest.mark.parametrize("lo,hi", [(1e-6, 1e6), (0.95, 1.05)], ids=["pass", "violated"])
def test_validate_diffeo(ctxs, lo, hi):
    """validate_diffeo (mapping.cpp:131-156) over a 40 x 900 lattice, on the device."""
    cfg, r, m = ctxs
    rng = np.random.default_rng(3)
    xs, ys = rng.random((40, 2)), rng.random((900, 2))
    a = r.validate_diffeo(xs, ys, lo, hi)
    b = m.validate_diffeo(xs, ys, lo, hi)
    assert a[0] == b[0]
    assert b[1] == pytest.approx(a[1], rel=1e-13) and b[2] == pytest.approx(a[2], rel=1e-13)
    assert a[3] == b[3] and a[4] == b[4]  # the same worst (x, yhat) pair
    assert a[5] == b[5]
    if lo > 1e-6 and cfg.map != "c1":
        assert not a[0] and "violated at" in a[5]
    e = m.validate_diffeo(xs[:0], ys, lo, hi)  # no pairs: pass = false, [0, 0]
    assert e[:3] == r.validate_diffeo(xs[:0], ys, lo, hi)[:3]


def test_check_assumption6(ctxs):
    """check_assumption6 (mapping.cpp:158-195): per-point Gamma^I measures summed on the device."""
    cfg, r, m = ctxs
    pts = np.random.default_rng(11).random((57, 2))
    rr, rs = r.check_assumption6(pts)
    mr, ms = m.check_assumption6(pts)
    assert maxrel(mr[:, :2], rr[:, :2]) <= 1e-13
    assert np.array_equal(mr[:, 2:], rr[:, 2:])
    assert ms[0] == rs[0] and np.array_equal(ms[3:], rs[3:])
    assert ms[1] == pytest.approx(rs[1], rel=1e-13) and ms[2] == pytest.approx(rs[2], rel=1e-13)


def test_assumption6_flags_violated(both):
    """kappa1 - kappa2 large enough that (|k1-k2|/2)|Gamma^I_x| >= 1 somewhere."""
    ref_mod, mir = both
    cfg = configs.TwoScaleConfig("a6", 4, 6, "c2", reaction=None, kappa=(3.0, 2.2, 0.0, 0.0))
    r, m = ref_mod.RefContext(cfg.ini(), 1), mir.RefContext(cfg.ini(), 1)
    pts = np.random.default_rng(5).random((64, 2))
    rr, rs = r.check_assumption6(pts)
    mr, ms = m.check_assumption6(pts)
    assert not rs[3] and rr[:, 2].min() == 0.0
    assert np.array_equal(mr[:, 2:], rr[:, 2:]) and np.array_equal(ms[3:], rs[3:])
    assert maxrel(mr[:, :2], rr[:, :2]) <= 1e-13


def test_assembly_and_solve_through_reference_api(ctxs):
    cfg, r, m = ctxs
    assert (m.n_macro, m.n_micro, m.micro_nnz, m.macro_nnz, m.n_micro_faces) == \
        (r.n_macro, r.n_micro, r.micro_nnz, r.macro_nnz, r.n_micro_faces)
    assert all(np.array_equal(a, b) for a, b in zip(m.micro_pattern(), r.micro_pattern()))
    for node in (0, m.n_macro // 2, m.n_macro - 1):
        assert maxrel(m.micro_values(node), r.micro_values(node)) <= 1e-12
        assert maxrel(m.micro_rhs(node, 0.3, 0.0), r.micro_rhs(node, 0.3, 0.0)) <= 1e-12
        mc, mf = m.node_cache(node)
        rc, rf = r.node_cache(node)
        assert maxrel(mc, rc) <= 1e-12 and maxrel(mf, rf) <= 1e-12
    for which in range(3):
        a, b = m.macro_matrix(which), r.macro_matrix(which)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and maxrel(a[2], b[2]) <= 1e-12
    for which in range(2):
        da, db = m.dirichlet(which), r.dirichlet(which)
        assert np.array_equal(da[0], db[0]) and np.array_equal(da[1], db[1])
    so = m.solve(outer_tol=1e-8)
    sr = r.solve(outer_tol=1e-8)
    assert so["sweeps"] == sr["sweeps"] and so["converged"] == sr["converged"]
    for k in ("u", "w", "V"):
        assert rel(so[k], sr[k]) <= 1e-8, k


def test_cg_solve_and_parallel_for(both):
    """cg_solve (linalg.cpp:103-161) through the mirror, alone and from parallel_for workers
    (ref_batched_cg spreads one cg_solve per system over `workers` host threads)."""
    ref_mod, mir = both
    cfg = configs.CONFIGS["c1"].reduced().resized(4, 8)
    r = ref_mod.RefContext(cfg.ini(), 1)
    rp, ci = r.micro_pattern()
    vals = np.stack([r.micro_values(i) for i in range(6, 14)])
    b = np.stack([r.micro_rhs(i, 0.05, 0.0) for i in range(6, 14)])
    x, conv, it, res, indef = mir.cg_solve(rp, ci, vals[0], b[0], np.zeros(r.n_micro), 1e-10, 2000)
    xr, convr, itr, resr, indefr = ref_mod.cg_solve(rp, ci, vals[0], b[0], np.zeros(r.n_micro), 1e-10, 2000)
    assert conv == convr and abs(it - itr) <= 1 and rel(x, xr) <= 1e-9
    for workers in (1, 4):
        xm, im, _ = mir.batched_cg(rp, ci, vals, b, np.zeros_like(b), 1e-10, 2000, workers)
        xr, ir, _ = ref_mod.batched_cg(rp, ci, vals, b, np.zeros_like(b), 1e-10, 2000, workers)
        assert np.abs(im - ir).max() <= 1 and rel(xm, xr) <= 1e-9
    assert mir.hardware_threads() == ref_mod.hardware_threads()  # resolve_worker_count(0)


def test_vtk_writers_through_reference_api(both, tmp_path):
    ref_mod, mir = both
    cfg = configs.CONFIGS["c1"].reduced().resized(3, 4)
    r = ref_mod.RefContext(cfg.ini(), 1)
    s = r.solve(outer_tol=1e-8)
    paths = {}
    for name, mod in (("ref", ref_mod), ("mir", mir)):
        mp, up = tmp_path / f"{name}_macro.vtk", tmp_path / f"{name}_micro.vtk"
        mod.write_vtk(cfg.ini(), s["u"], s["w"], s["V"], 0.5, mp, up)
        paths[name] = (mp.read_bytes(), up.read_bytes())
    assert paths["ref"][0] == paths["mir"][0] and paths["ref"][1] == paths["mir"][1]
