"""Pins the C oracle (oracle/twoscale_oracle.c) to the reference library itself
(oracle/_ref, the unmodified /root/reference/proj/src compiled by oracle/Makefile)
at the reference-expressible reductions of the BASELINE configs (k = 0, D = I,
symbolic map).  CPU only."""
import numpy as np
import pytest

from paper_2103_17040_b200 import configs

CASES = [
    configs.CONFIGS["c1"].reduced(),
    configs.CONFIGS["c2"].reduced().resized(10, 12),
    configs.CONFIGS["c3"].reduced().resized(6, 20),
    configs.CONFIGS["c1"].reduced().resized(3, 5),
]


@pytest.fixture(scope="module", params=range(len(CASES)), ids=[c.name for c in CASES])
def pair(request, ref_mod, port_mod):
    cfg = CASES[request.param]
    return cfg, port_mod.OracleContext(cfg, reference_expressible=True), ref_mod.RefContext(cfg.ini(), 1)


def test_index_structures_bit_exact(pair):
    cfg, o, r = pair
    rp, ci = o.micro_pattern()
    rrp, rci = r.micro_pattern()
    assert np.array_equal(rp, rrp) and np.array_equal(ci, rci)
    _, _, mv = r.macro_matrix(0)
    assert mv.size == o.macro_nnz
    d, v = r.dirichlet(0)
    m = cfg.macro_n
    boundary = sorted({j * (m + 1) + i for j in range(m + 1) for i in range(m + 1)
                       if i in (0, m) or j in (0, m)})
    assert list(d) == boundary and np.all(v == 0.0)


def test_caches_and_values(pair):
    cfg, o, r = pair
    for node in sorted({0, 1, o.n_macro // 2, o.n_macro - 1}):
        oc, of = o.node_cache(node)
        rc, rf = r.node_cache(node)
        assert np.abs(oc - rc).max() <= 1e-14 * np.abs(rc).max()
        assert np.abs(of - rf).max() <= 1e-14 * np.abs(rf).max()
        ov, rv = o.micro_values(node), r.micro_values(node)
        assert np.abs(ov - rv).max() <= 1e-14 * np.abs(rv).max()
        _, ri, _ = o.rhs_parts(node)
        assert np.abs(ri - r.micro_rhs(node, 1.0, 0.0)).max() <= 1e-14 * np.abs(ri).max()
    for which in range(3):
        _, _, rv = r.macro_matrix(which)
        assert np.abs(o.macro_matrix(which) - rv).max() <= 1e-14 * max(np.abs(rv).max(), 1.0)


def test_fixed_point_solve(pair):
    cfg, o, r = pair
    so = o.solve(outer_tol=cfg.outer_tol)
    sr = r.solve(outer_tol=cfg.outer_tol)
    assert so["sweeps"] == sr["sweeps"] and so["converged"] == sr["converged"]
    for k in ("u", "w", "V"):
        nb = max(np.linalg.norm(sr[k]), 1e-300)
        assert np.linalg.norm(so[k] - sr[k]) / nb <= 1e-10, k
    assert np.allclose(so["history"], sr["history"], rtol=1e-8, atol=1e-15)


def test_cg_solve_matches_reference_bitwise(ref_mod, port_mod):
    rng = np.random.default_rng(7)
    n = 30
    M = rng.standard_normal((n, n))
    A = M @ M.T + n * np.eye(n)
    rp = np.arange(0, n * n + 1, n)
    ci = np.tile(np.arange(n), n)
    b = rng.standard_normal(n)
    x0 = rng.standard_normal(n)
    xo, co, io, ro, _ = port_mod.cg_solve(rp, ci, A.reshape(-1), b, x0, 1e-12, 100)
    xr, cr, ir, rr, _ = ref_mod.cg_solve(rp, ci, A.reshape(-1), b, x0, 1e-12, 100)
    assert (co, io) == (cr, ir)
    assert np.array_equal(xo, xr) and ro == rr  # same op order, no FMA: identical bits
