"""Pins the generic (Q2 / 3D) C oracle at its d = 2, p = 1 reduction to the reference
binary: a constant affine map plus the x0*x1 bubble is expressible both as a
reference INI (symbolic zeta) and as a generic-oracle table.  CPU only."""
import numpy as np
import pytest

from paper_2103_17040_b200 import configs

A0 = np.array([[1.1, 0.05], [-0.03, 0.95]])


def const_affine_cfg(macro_n, micro_n):
    cfg = configs.TwoScaleConfig("const-affine", macro_n, micro_n, "table", reaction=None)
    z0 = f"{float(A0[0,0])!r}*y0 + {float(A0[0,1])!r}*y1 + 0.15*x0*x1*16*y0*(1-y0)*y1*(1-y1)"
    z1 = f"{float(A0[1,0])!r}*y0 + {float(A0[1,1])!r}*y1 + 0.15*x0*x1*16*y0*(1-y0)*y1*(1-y1)"
    ini = cfg.ini().replace(configs.C2_ZETA[0], z0).replace(configs.C2_ZETA[1], z1)
    table = np.tile(A0.reshape(1, 4), (cfg.n_macro, 1))
    return cfg, ini, table


@pytest.mark.parametrize("sizes", [(4, 6), (6, 10), (3, 23)])
def test_generic_oracle_reduces_to_reference(sizes, ref_mod, port_mod):
    cfg, ini, table = const_affine_cfg(*sizes)
    r = ref_mod.RefContext(ini, 1)
    o = port_mod.GenOracleContext(cfg, table=table)
    rp, ci = o.micro_pattern()
    rrp, rci = r.micro_pattern()
    assert np.array_equal(rp, rrp) and np.array_equal(ci, rci)
    for node in sorted({0, o.n_macro // 2, o.n_macro - 1}):
        ov, rv = o.micro_values(node), r.micro_values(node)
        assert np.abs(ov - rv).max() <= 1e-14 * np.abs(rv).max()
        ri, _ = o.rhs_parts(node)
        assert np.abs(ri - r.micro_rhs(node, 1.0, 0.0)).max() <= 1e-14 * np.abs(ri).max()
    for which in range(3):
        _, _, rv = r.macro_matrix(which)
        assert np.abs(o.macro_matrix(which) - rv).max() <= 1e-14 * max(1.0, np.abs(rv).max())
    so = o.solve(outer_tol=cfg.outer_tol)
    sr = r.solve(outer_tol=cfg.outer_tol)
    assert so["sweeps"] == sr["sweeps"]
    for k in ("u", "V"):
        assert np.linalg.norm(so[k] - sr[k]) / np.linalg.norm(sr[k]) <= 1e-10


def test_generic_oracle_q2_and_3d_sanity(port_mod):
    """Constant compatibility holds for Q2 and 3D micro problems too: with
    u_i fixed the micro solution is the constant c (checked through a full solve's
    micro systems: A 1 = robin_in when k = 0)."""
    for cfg in (configs.CONFIGS["c4"].resized(3, 4), configs.CONFIGS["c5"].resized(3, 3)):
        cfg.reaction = None
        o = port_mod.GenOracleContext(cfg)
        rp, ci = o.micro_pattern()
        v = o.micro_values(o.n_macro // 2)
        ones = np.ones(o.n_micro)
        A1 = np.array([v[rp[r]:rp[r + 1]] @ ones[ci[rp[r]:rp[r + 1]]] for r in range(o.n_micro)])
        ri, _ = o.rhs_parts(o.n_macro // 2)
        assert np.abs(A1 - ri).max() <= 1e-12 * np.abs(ri).max()   # kappa2 = 1: Robin mass row sums
        assert np.all(np.diff(rp) > 0)
