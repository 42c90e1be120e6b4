"""Parity of the B200 path (through the C ABI) against the reference binary
(oracle/_ref) and the C oracle (oracle/port).  Bars (BASELINE.json north_star):
index structures bit-exact, assembled values <= 1e-12 relative, u/w/V relative
L2 <= 1e-8 at CG tolerance 1e-10."""
import os

import numpy as np
import pytest

from paper_2103_17040_b200 import abi, configs

pytestmark = pytest.mark.gpu

VAL_TOL = 1e-12   # assembled values / caches, relative to the largest entry
SOL_TOL = 1e-8    # solution vectors, relative L2 (north star)


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def maxrel(a, b):
    s = np.abs(b).max()
    return np.abs(a - b).max() / (s if s > 0 else 1.0)


@pytest.fixture(scope="module")
def dev():
    if not abi.device_ok():
        pytest.fail("no usable sm_100 device: " + abi.lib().ts_last_error().decode())
    return True


# ------------------------------------------------------------------ C1 vs ref
@pytest.fixture(scope="module")
def c1_pair(dev, ref_mod):
    cfg = configs.CONFIGS["c1"].reduced()
    return abi.Context(cfg.ini(), cfg.ext(reference_expressible=True)), ref_mod.RefContext(cfg.ini(), 1)


def test_c1_index_structures_bit_exact(c1_pair):
    g, r = c1_pair
    rp, ci = g.micro_pattern()
    rrp, rci = r.micro_pattern()
    assert np.array_equal(rp, rrp) and np.array_equal(ci, rci)
    for which in range(3):
        mrp, mci, _ = g.macro_matrix(which)
        rmrp, rmci, _ = r.macro_matrix(which)
        assert np.array_equal(mrp, rmrp) and np.array_equal(mci, rmci)
    for which in range(2):
        d, v = g.dirichlet(which)
        rd, rv = r.dirichlet(which)
        assert np.array_equal(d, rd)
        assert np.array_equal(v, rv)


def test_c1_caches_values_rhs(c1_pair):
    g, r = c1_pair
    for node in (0, 5, 17, 144, 200, 288):
        gc, gf = g.node_cache(node)
        rc, rf = r.node_cache(node)
        assert maxrel(gc, rc) <= VAL_TOL
        assert maxrel(gf, rf) <= VAL_TOL
        assert maxrel(g.micro_values(node), r.micro_values(node)) <= VAL_TOL
        assert maxrel(g.micro_rhs(node, 0.37, -0.2), r.micro_rhs(node, 0.37, -0.2)) <= VAL_TOL
    for which in range(3):
        assert maxrel(g.macro_matrix(which)[2], r.macro_matrix(which)[2]) <= VAL_TOL


def test_c1_macro_rhs_and_coupling(c1_pair):
    g, r = c1_pair
    rng = np.random.default_rng(0)
    V = rng.standard_normal((g.n_macro, g.n_micro))
    for which in range(2):
        assert maxrel(g.macro_rhs(which, V), r.macro_rhs(which, V)) <= VAL_TOL
    for node in (0, 33, 288):
        for role in (0, 1):
            a, b = g.surface_coupling(V[node], node, role), r.surface_coupling(V[node], node, role)
            assert abs(a - b) <= VAL_TOL * max(1.0, abs(b))


def test_c1_fixed_point_solve_matches_reference(c1_pair):
    g, r = c1_pair
    out = g.solve(outer_tol=1e-10)
    ref = r.solve(outer_tol=1e-10)
    assert out["sweeps"] == ref["sweeps"]
    assert out["converged"] == ref["converged"]
    for k in ("u", "w", "V"):
        assert rel(out[k], ref[k]) <= SOL_TOL, k
    assert np.allclose(out["history"], ref["history"], rtol=1e-6, atol=1e-14)
    assert out["gpu_launches"] > 0


def test_c1_micro_solve_iterations(c1_pair):
    g, r = c1_pair
    u = np.full(g.n_macro, 0.05)
    w = np.zeros(g.n_macro)
    V, it, rep = g.micro_solve(u, w)
    Vr, itr, _ = r.micro_sweep(u, w)
    assert rel(V, Vr) <= SOL_TOL
    assert np.abs(it - itr).max() <= 2
    assert rep["micro_dof_iters"] == pytest.approx(float(g.n_micro * it.sum()))


# --------------------------------------------------------------- KATs (SPEC)
def test_cg_kat_3x3(dev):
    rp = np.array([0, 2, 5, 7])
    ci = np.array([0, 1, 0, 1, 2, 1, 2])
    v = np.array([2.0, -1, -1, 2, -1, -1, 2])
    x, conv, it, res, indef = abi.cg_solve(rp, ci, v, np.ones(3), np.zeros(3), 1e-12, 50)
    assert conv and not indef
    assert np.allclose(x, [1.5, 2.0, 1.5], atol=1e-12)


def test_cg_kat_identity_one_iteration(dev):
    n = 7
    rp = np.arange(n + 1)
    ci = np.arange(n)
    b = np.linspace(1, 2, n)
    x, conv, it, res, indef = abi.cg_solve(rp, ci, np.ones(n), b, np.zeros(n), 1e-10, 10)
    assert conv and it == 1 and np.allclose(x, b)


def test_cg_zero_rhs_zeroes_warm_start(dev):
    rp = np.array([0, 1, 2])
    ci = np.array([0, 1])
    x, conv, it, res, indef = abi.cg_solve(rp, ci, np.ones(2), np.zeros(2), np.array([3.0, 4.0]), 1e-10, 10)
    assert conv and it == 0 and np.all(x == 0.0)


def test_cg_indefinite_detected(dev):
    rp = np.array([0, 1, 2])
    ci = np.array([0, 1])
    x, conv, it, res, indef = abi.cg_solve(rp, ci, np.array([-1.0, -2.0]), np.ones(2), np.zeros(2), 1e-10, 10)
    assert indef and not conv and it == 1


def test_cg_random_spd_vs_reference(dev, ref_mod):
    rng = np.random.default_rng(3)
    for n in (5, 17, 50):
        M = rng.standard_normal((n, n))
        A = M @ M.T + n * np.eye(n)
        rp = np.arange(0, n * n + 1, n)
        ci = np.tile(np.arange(n), n)
        b = rng.standard_normal(n)
        x, conv, it, res, _ = abi.cg_solve(rp, ci, A.reshape(-1), b, np.zeros(n), 1e-12, 200)
        xr, convr, itr, _, _ = ref_mod.cg_solve(rp, ci, A.reshape(-1), b, np.zeros(n), 1e-12, 200)
        assert conv and convr and abs(it - itr) <= 1
        assert rel(x, np.linalg.solve(A, b)) <= 1e-10


def test_constant_compatibility_kat(dev, ref_mod):
    """f^v = 0, u_i = c kappa2/kappa1 held fixed -> every micro solution is v = c."""
    cfg = configs.CONFIGS["c1"].reduced().resized(4, 32)
    g = abi.Context(cfg.ini(), cfg.ext(reference_expressible=True))
    c = 0.7
    V, it, _ = g.micro_solve(np.full(g.n_macro, c), np.zeros(g.n_macro))
    assert np.abs(V - c).max() / c <= 1e-10 * 10


def test_surface_coupling_kats(dev):
    """v = 1 with the identity map on the left side of [-1,1]^2 -> 2;
    the manufactured map -> 2 |(-0.24,-0.216)| = 0.64578."""
    ini_id = """
[macro]
n0 = 2
n1 = 2
[micro]
n0 = 4
n1 = 4
zeta0 = y0
zeta1 = y1
[parameters]
kappa1 = 1
kappa2 = 1
kappa3 = 1
kappa4 = 1
Dv = 1
Dw = 1
"""
    g = abi.Context(ini_id)
    assert g.surface_coupling(np.ones(g.n_micro), 0, abi.TS_GAMMA_I) == pytest.approx(2.0, abs=1e-14)
    ini_m = ini_id.replace("zeta0 = y0", "zeta0 = 0.4*((x0 + 1.3)+(1.4*y0 - 0.54*y1))").replace(
        "zeta1 = y1", "zeta1 = 0.3*((x1 + 1.2)+(-0.4*y0 + 0.8*y1))")
    g2 = abi.Context(ini_m)
    expect = 2 * np.hypot(0.24, 0.216)
    assert g2.surface_coupling(np.ones(g2.n_micro), 3, abi.TS_GAMMA_I) == pytest.approx(expect, rel=1e-12)
    cells, faces = g2.node_cache(0)
    assert np.allclose(cells[:, :, 0], 0.10848, rtol=1e-12)  # det J of the manufactured map


def test_identity_map_transparency(dev):
    """identity map -> Q1 stiffness stencil (1/3)[8, -1 ...] in the interior."""
    ini = """
[macro]
n0 = 2
n1 = 2
[micro]
n0 = 6
n1 = 6
zeta0 = y0
zeta1 = y1
gamma_i = left
gamma_o = right
gamma_n = bottom,top
[parameters]
kappa1 = 1
kappa2 = 0
kappa3 = 1
kappa4 = 0
Dv = 1
Dw = 1
"""
    g = abi.Context(ini)
    assert g.info["shared_operator"] == 1
    rp, ci = g.micro_pattern()
    v = g.micro_values(0)
    row = 3 * 7 + 3
    vals = dict(zip(ci[rp[row]:rp[row + 1]], v[rp[row]:rp[row + 1]]))
    assert vals[row] == pytest.approx(8.0 / 3.0, rel=1e-14)
    for c, a in vals.items():
        if c != row:
            assert a == pytest.approx(-1.0 / 3.0, rel=1e-14)
    # kappa2 = kappa4 = 0: A 1 = 0
    ones = np.ones(g.n_micro)
    Av = np.zeros(g.n_micro)
    for r in range(g.n_micro):
        Av[r] = v[rp[r]:rp[r + 1]].sum()
    assert np.abs(Av).max() <= 1e-12


def test_degenerate_map_is_reported(dev):
    ini = """
[macro]
n0 = 2
n1 = 2
[micro]
n0 = 4
n1 = 4
zeta0 = -y0
zeta1 = y1
[parameters]
kappa1 = 1
kappa2 = 1
kappa3 = 1
kappa4 = 1
Dv = 1
Dw = 1
"""
    with pytest.raises(abi.DegenerateMapError, match="degenerate map in cache build"):
        abi.Context(ini)


def test_config_errors_are_reported(dev):
    with pytest.raises(abi.ConfigError, match="missing required keys"):
        abi.Context("[macro]\nn0 = 2\n")


# ------------------------------------------- per-problem iterations vs the reference
@pytest.mark.parametrize("name,macro_n,micro_n", [("c3", 4, 64), ("c2", 6, 32)])
def test_micro_solve_iterations_vs_reference(dev, ref_mod, name, macro_n, micro_n):
    """Reference-expressible stand-ins on the BASELINE micro widths (65 and 33: column-pair
    kernel, full warps / half warps): cold batched solve with u_i = 0.05 (SURVEY.md §8d timed region
    (ii)); per-problem iteration counts within ±2 of the reference's cg_solve (§8c)."""
    cfg = configs.CONFIGS[name].reduced().resized(macro_n, micro_n)
    g = abi.Context(cfg.ini(), cfg.ext(reference_expressible=True))
    r = ref_mod.RefContext(cfg.ini(), 8)
    if "TS_PCG_PAIR" not in os.environ:  # default kernel choice (an override changes it)
        assert g.info["micro_kernel"] == 1
    u = np.full(g.n_macro, 0.05)
    w = np.zeros(g.n_macro)
    V, it, rep = g.micro_solve(u, w)
    Vr, itr, _ = r.micro_sweep(u, w, workers=8)
    assert rel(V, Vr) <= SOL_TOL
    assert np.abs(it - itr).max() <= 2
    assert rep["micro_dof_iters"] == pytest.approx(float(g.n_micro * it.sum()))


# ------------------------------------------------------------ failure reporting
def test_solver_errors_match_reference(c1_pair):
    """SolverError messages (solver.cpp:48-57, 91-97): the macro CG failing first at a tiny
    maxit, and a micro system failing once the macro systems converge — same text, same
    failing index, as the reference at 1 worker."""
    g, r = c1_pair
    with pytest.raises(abi.SolverError) as e:
        g.solve(inner_maxit=2, outer_tol=1e-10)
    from oracle import ref as refmod
    with pytest.raises(refmod.RefError) as er:
        r.solve(inner_maxit=2, outer_tol=1e-10)
    assert str(e.value) == str(er.value).split("] ", 1)[1]
    assert str(e.value).startswith("macro u-system: CG failed to converge, relative residual ")
    # smallest maxit at which the reference fails in a micro system instead
    hit = None
    for maxit in range(5, 200):
        try:
            r.solve(inner_maxit=maxit, outer_tol=1e-10)
            break
        except refmod.RefError as ex:
            if "micro system" in str(ex):
                hit = (maxit, str(ex).split("] ", 1)[1])
                break
    assert hit is not None
    with pytest.raises(abi.SolverError) as e2:
        g.solve(inner_maxit=hit[0], outer_tol=1e-10)
    assert str(e2.value) == hit[1]
    assert e2.value.index == int(hit[1].split()[2].rstrip(":"))


# ----------------------------------------------- maxit boundary, every micro kernel
@pytest.mark.parametrize("micro_n", [64, 32, 16])
def test_micro_maxit_boundary(dev, micro_n):
    """Iteration budget exactly at / below each problem's count (linalg.cpp:134-156): with
    maxit = the median count, problems that need <= maxit iterations converge with the same
    count and bitwise the same V as an unlimited solve (including those converging exactly at
    the last allowed iteration, where the 65-wide pair kernel's lagged stop test fires after
    the loop), the others stop at maxit with status 'failed to converge' and the first of them
    is the reported system.  Covers the pair kernel with the lagged test (65 wide), the pair
    kernel (33) and column strips (17)."""
    cfg = configs.CONFIGS["c3"].resized(4, micro_n)
    g = abi.Context(cfg.ini(), cfg.ext())
    u = np.linspace(0.01, 0.1, g.n_macro)
    w = np.zeros(g.n_macro)
    V0, it0, _ = g.micro_solve(u, w)
    m = int(np.median(it0))
    assert (it0 == m).any() and (it0 > m).any()
    V, it, _, st = g.micro_solve(u, w, maxit=m, raise_on_fail=False)
    conv = it0 <= m
    assert st == abi.TS_ERR_SOLVER
    assert (it[conv] == it0[conv]).all()
    assert np.array_equal(V[conv], V0[conv])
    assert (it[~conv] == m).all()
    msg = abi.lib().ts_last_error().decode()
    first = int(np.flatnonzero(~conv)[0])
    assert msg.startswith(f"micro system {first}: CG failed to converge, relative residual "), msg
    # one more iteration of budget for the longest converged-at-m problem changes nothing for it
    V1, it1, _, _ = g.micro_solve(u, w, maxit=m + 1, raise_on_fail=False)
    assert np.array_equal(V1[conv], V0[conv]) and (it1[conv] == it0[conv]).all()


# ------------------------------------------ macro systems beyond one SM: cluster solver
@pytest.mark.parametrize("cl", ["16", "8", "0"])
def test_large_macro_grid_matches_reference(dev, ref_mod, monkeypatch, cl):
    """An 80 x 80 macro grid (6561 nodes) does not fit one SM's SMEM, so the macro u/w PCG
    runs on a thread-block cluster (mcluster.cu; 16 or 8 CTAs per system, DSMEM dot-product
    exchange and p halos) — or, with TS_MACRO_CLUSTER=0, on the cooperative CSR CG.  Whole
    fixed-point solve vs the reference binary: same sweeps, u/w/V within the north-star bar."""
    monkeypatch.setenv("TS_MACRO_CLUSTER", cl)
    cfg = configs.CONFIGS["c1"].reduced().resized(80, 4)
    g = abi.Context(cfg.ini(), cfg.ext(reference_expressible=True))
    if cl == "0":
        assert g.info["macro_solver"] == 2
    else:
        assert g.info["macro_solver"] == 1 and g.info["macro_cluster"] <= int(cl)
    r = ref_mod.RefContext(cfg.ini(), 8)
    out = g.solve(outer_tol=1e-10)
    ref = r.solve(outer_tol=1e-10, workers=8)
    assert out["sweeps"] == ref["sweeps"]
    for k in ("u", "w", "V"):
        assert rel(out[k], ref[k]) <= SOL_TOL, k
