"""Micro-state egress: legacy VTK writers.

CPU: the C++ mirror's host writers (ts_write_vtk_ini) produce files byte-identical to the
reference's write_vtk_macro / write_vtk_micro (oracle/_ref, vtk.cpp:36-85).
GPU: the streamed device writers (ts_write_vtk_macro / ts_write_vtk_micro) against the
reference writer run on the downloaded state, and the BINARY variant / tabulated maps
against the same data parsed back.
"""
import filecmp
import gzip
import os

import numpy as np
import pytest

from paper_2103_17040_b200 import abi, configs
import vtk_io

POLY_ZETA = ("y0 + 0.1*x0*x1*16*y0*(1-y0)*y1*(1-y1) + 0.05*y1", "y1 + 0.1*x0*16*y0*(1-y0)*y1*(1-y1)")


def poly_ini(macro_n, micro_n):
    ini = configs.CONFIGS["c2"].ini(macro_n=macro_n, micro_n=micro_n)
    out = []
    for ln in ini.split("\n"):
        if ln.startswith("zeta0 ="):
            ln = "zeta0 = " + POLY_ZETA[0]
        elif ln.startswith("zeta1 ="):
            ln = "zeta1 = " + POLY_ZETA[1]
        out.append(ln)
    return "\n".join(out)


def random_state(n_macro, n_micro, seed=1):
    rng = np.random.default_rng(seed)
    u, w = rng.standard_normal(n_macro), rng.standard_normal(n_macro)
    V = rng.standard_normal((n_macro, n_micro)) * 10.0 ** rng.integers(-9, 9, size=(n_macro, n_micro))
    V[0, :4] = [0.0, -0.0, 1e-300, 123456789012345678.0]
    return u, w, V


HOST_CASES = [("c1", 4, 6, 0.25), ("c2", 5, 7, 1.0), ("poly", 3, 9, 0.5), ("c1", 16, 16, 0.1)]


@pytest.mark.parametrize("name,mn,mc,scale", HOST_CASES)
def test_host_writers_byte_identical_to_reference(ref_mod, tmp_path, name, mn, mc, scale):
    ini = poly_ini(mn, mc) if name == "poly" else configs.CONFIGS[name].ini(macro_n=mn, micro_n=mc)
    u, w, V = random_state((mn + 1) ** 2, (mc + 1) ** 2)
    ref_mod.write_vtk(ini, u, w, V, scale, tmp_path / "ref_macro.vtk", tmp_path / "ref_micro.vtk")
    abi.write_vtk_ini(ini, u, w, V, scale, tmp_path / "macro.vtk", tmp_path / "micro.vtk")
    assert filecmp.cmp(tmp_path / "ref_macro.vtk", tmp_path / "macro.vtk", shallow=False)
    assert filecmp.cmp(tmp_path / "ref_micro.vtk", tmp_path / "micro.vtk", shallow=False)
    d = vtk_io.read(tmp_path / "micro.vtk")
    assert np.array_equal(d["cells"], vtk_io.lattice_cells((mc + 1, mc + 1), (mn + 1) ** 2))
    v = V.ravel()
    assert np.all(np.abs(d["scalars"]["v"] - v) <= 6e-16 * np.abs(v))   # 16 significant digits


def test_host_writer_errors_match_reference(ref_mod, tmp_path):
    ini = configs.CONFIGS["c1"].ini(macro_n=2, micro_n=2)
    u, w, V = random_state(9, 9)
    bad = str(tmp_path / "missing" / "m.vtk")
    with pytest.raises(abi.TwoScaleError) as e:
        abi.write_vtk_ini(ini, u, w, V, 1.0, bad, None)
    assert e.value.status == abi.TS_ERR_IO
    with pytest.raises(ref_mod.RefError) as r:
        ref_mod.write_vtk(ini, u, w, V, 1.0, bad, None)
    assert str(e.value) == str(r.value).split("] ", 1)[1] == f"cannot write '{bad}'"
    with pytest.raises(abi.ConfigError):
        abi.write_vtk_ini("[macro]\nn0 = 2\n", u, w, V, 1.0, str(tmp_path / "x.vtk"), None)


GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_host_writers_match_golden_reference_files(tmp_path):
    """Byte parity against VTK files written by the reference itself (tests/golden,
    make_golden.py) for the reference's own solution: holds without /root/reference."""
    g = np.load(os.path.join(GOLDEN, "c1_ref_4x6.npz"))
    abi.write_vtk_ini(str(g["ini"]), g["u"], g["w"], g["V"], 0.25, tmp_path / "macro.vtk", tmp_path / "micro.vtk")
    for tag in ("macro", "micro"):
        with gzip.open(os.path.join(GOLDEN, f"vtk_c1_ref_4x6_{tag}.vtk.gz"), "rb") as f:
            want = f.read()
        assert (tmp_path / f"{tag}.vtk").read_bytes() == want, tag


# ---------------------------------------------------------------------------- GPU
def solved(ini, ext=None):
    if not abi.device_ok():
        pytest.fail("no usable sm_100 device")
    ctx = abi.Context(ini, ext)
    ctx.solve()
    st = ctx.state()
    return ctx, st


@pytest.mark.gpu
@pytest.mark.parametrize("which", ["c1", "poly"])
def test_device_writers_vs_reference(ref_mod, tmp_path, which):
    ini = poly_ini(6, 10) if which == "poly" else configs.CONFIGS["c1"].ini(macro_n=6, micro_n=10)
    ctx, st = solved(ini)
    ctx.write_vtk_macro(tmp_path / "macro.vtk")
    ctx.write_vtk_micro(tmp_path / "micro.vtk", scale=0.3)
    ref_mod.write_vtk(ini, st["u"], st["w"], st["V"], 0.3, tmp_path / "ref_macro.vtk", tmp_path / "ref_micro.vtk")
    assert filecmp.cmp(tmp_path / "ref_macro.vtk", tmp_path / "macro.vtk", shallow=False)
    if which == "poly":  # +,-,* only: the device pushforward rounds exactly like the host
        assert filecmp.cmp(tmp_path / "ref_micro.vtk", tmp_path / "micro.vtk", shallow=False)
    a, b = vtk_io.read(tmp_path / "micro.vtk"), vtk_io.read(tmp_path / "ref_micro.vtk")
    for sec in ("CELLS", "CELL_TYPES", "SCALARS v"):
        assert a["sections"][sec] == b["sections"][sec]
    assert a["title"] == b["title"]
    # sin/cos in zeta: device libm vs host libm may differ in the last ulp
    assert np.abs(a["points"] - b["points"]).max() <= 4e-16 * np.abs(b["points"]).max()


@pytest.mark.gpu
def test_device_binary_matches_ascii(tmp_path):
    ctx, st = solved(configs.CONFIGS["c1"].ini(macro_n=5, micro_n=8))
    ctx.write_vtk_micro(tmp_path / "a.vtk", scale=0.5)
    ctx.write_vtk_micro(tmp_path / "b.vtk", scale=0.5, binary=True)
    ctx.write_vtk_macro(tmp_path / "ma.vtk")
    ctx.write_vtk_macro(tmp_path / "mb.vtk", binary=True)
    a, b = vtk_io.read(tmp_path / "a.vtk"), vtk_io.read(tmp_path / "b.vtk")
    assert b["format"] == "BINARY"
    assert np.array_equal(a["cells"], b["cells"]) and np.array_equal(a["types"], b["types"])
    assert np.array_equal(b["scalars"]["v"], st["V"].ravel())          # binary is exact
    assert np.abs(a["points"] - b["points"]).max() <= 1e-15            # ASCII keeps 16 digits
    ma, mb = vtk_io.read(tmp_path / "ma.vtk"), vtk_io.read(tmp_path / "mb.vtk")
    assert np.array_equal(mb["scalars"]["u"], st["u"]) and np.array_equal(mb["scalars"]["w"], st["w"])
    assert np.array_equal(ma["cells"], mb["cells"])


def zeta_table(cfg, x, y):
    """numpy pushforward of the tabulated families (include/twoscale_b200.h map kinds)."""
    T = cfg.table()
    if cfg.map == "fourier":
        K = [1, 1, 2, 2, 1, 3, 2, 3]
        Lm = [1, 2, 1, 2, 3, 1, 3, 2]
        c = T.reshape(-1, 2, 8)
        phi = np.stack([np.sin(np.pi * k * y[:, 0]) * np.sin(np.pi * l * y[:, 1]) for k, l in zip(K, Lm)], 1)
        return y[None, :, :2] + np.einsum("iam,pm->ipa", c, phi)
    d = 3 if cfg.map == "table3" else 2
    A = T.reshape(-1, d, d)
    beta = (16.0 if d == 2 else 64.0) * np.prod(y[:, :d] * (1 - y[:, :d]), axis=1)
    s = x[:, 0] * x[:, 1] * cfg.amp
    return np.einsum("iab,pb->ipa", A, y[:, :d]) + (s[:, None] * beta[None, :])[:, :, None]


@pytest.mark.gpu
@pytest.mark.parametrize("name,mn,mc", [("c3", 5, 8), ("c4", 4, 4), ("c5", 3, 3)])
def test_device_tabulated_maps(tmp_path, name, mn, mc):
    cfg = configs.CONFIGS[name].resized(mn, mc)
    ctx, st = solved(cfg.ini(), cfg.ext())
    scale = 0.2
    ctx.write_vtk_micro(tmp_path / "b.vtk", scale=scale, binary=True)
    ctx.write_vtk_micro(tmp_path / "a.vtk", scale=scale)
    b, a = vtk_io.read(tmp_path / "b.vtk"), vtk_io.read(tmp_path / "a.vtk")
    n1 = cfg.order * mc + 1
    nn = (n1, n1, n1) if cfg.dim == 3 else (n1, n1)
    grid1 = np.arange(n1) / (n1 - 1)
    mesh = np.meshgrid(*([grid1] * cfg.dim), indexing="ij")
    y = np.stack([m.transpose().ravel() for m in mesh], 1)            # lexicographic, y0 fastest
    xs = np.arange(mn + 1) / mn
    x = np.stack(np.meshgrid(xs, xs, indexing="xy"), -1).reshape(-1, 2)
    z = zeta_table(cfg, x, y)
    want = np.zeros((x.shape[0], y.shape[0], 3))
    want[:, :, :2] = x[:, None, :] + scale * z[:, :, :2]
    if cfg.dim == 3:
        want[:, :, 2] = scale * z[:, :, 2]
    assert np.abs(b["points"] - want.reshape(-1, 3)).max() <= 1e-14
    assert np.array_equal(b["scalars"]["v"], st["V"].ravel())
    assert np.array_equal(b["cells"], vtk_io.lattice_cells(nn, x.shape[0]))
    assert set(b["types"].tolist()) == {12 if cfg.dim == 3 else 9}
    assert np.array_equal(a["cells"], b["cells"])
    assert np.abs(a["points"] - b["points"]).max() <= 1e-15 * max(1.0, np.abs(b["points"]).max())


@pytest.mark.gpu
def test_device_writer_errors(tmp_path):
    if not abi.device_ok():
        pytest.fail("no usable sm_100 device")
    ctx = abi.Context(configs.CONFIGS["c1"].ini(macro_n=2, micro_n=2))
    with pytest.raises(abi.TwoScaleError) as e:
        ctx.write_vtk_micro(tmp_path / "m.vtk")
    assert e.value.status == abi.TS_ERR_INVALID and "ts_fixed_point_solve" in str(e.value)
    ctx.solve()
    bad = str(tmp_path / "missing" / "m.vtk")
    with pytest.raises(abi.TwoScaleError) as e:
        ctx.write_vtk_micro(bad)
    assert e.value.status == abi.TS_ERR_IO and str(e.value) == f"cannot write '{bad}'"
