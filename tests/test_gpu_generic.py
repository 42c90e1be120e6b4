"""Configs 4 (Q2 micro, Fourier map, piecewise reaction) and 5 (3D Q1 micro) on the
generic device path, against the generic C oracle (itself pinned to the reference at
its 2D Q1 reduction, tests/test_oracle_gen.py); plus the generic path run on 2D Q1
problems against the reference binary directly."""
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
    "c4-tiny": configs.CONFIGS["c4"].resized(4, 4),
    "c4-small": configs.CONFIGS["c4"].resized(8, 10),
    "c5-tiny": configs.CONFIGS["c5"].resized(4, 3),
    "c5-small": configs.CONFIGS["c5"].resized(6, 6),
}


@pytest.fixture(scope="module", params=list(CASES))
def pair(request, port_mod):
    if not abi.device_ok():
        pytest.fail("no usable sm_100 device")
    cfg = CASES[request.param]
    return cfg, abi.Context(cfg.ini(), cfg.ext()), port_mod.GenOracleContext(cfg)


def test_generic_structures_and_values(pair):
    cfg, g, o = pair
    assert g.n_micro == o.n_micro == cfg.n_micro
    rp, ci = g.micro_pattern()
    orp, oci = o.micro_pattern()
    assert np.array_equal(rp, orp) and np.array_equal(ci, oci)
    nc = 1 + cfg.dim * (cfg.dim + 1) // 2
    for node in sorted({0, g.n_macro // 2, g.n_macro - 1}):
        cells = np.zeros((o.n_cells, o.nq, nc))
        faces = np.zeros((o.n_faces, o.nqf))
        abi.check(abi.lib().ts_node_cache(g.h, node, abi._dp(cells), abi._dp(faces)))
        oc, of = o.node_cache(node)
        assert maxrel(cells, oc) <= VAL_TOL
        assert maxrel(faces, of) <= VAL_TOL
        assert maxrel(g.micro_values(node), o.micro_values(node)) <= VAL_TOL
        ri, _ = o.rhs_parts(node)
        assert maxrel(g.micro_rhs(node, 1.0, 0.0), ri) <= VAL_TOL
        v = np.random.default_rng(node).standard_normal(g.n_micro)
        assert g.surface_coupling(v, node, 0) == pytest.approx(o.surface_coupling(v, node, 0), rel=1e-12)
    for which in range(3):
        assert maxrel(g.macro_matrix(which)[2], o.macro_matrix(which)) <= VAL_TOL


def test_generic_operator_is_stored_as_its_upper_half(pair):
    """The generic (Q2 / 3D) operators keep the centre and the upper half of the direction
    planes; ts_micro_values mirrors the lower half from the neighbours' entries.  So the
    expanded CSR row set is exactly symmetric (bitwise), while still matching the oracle's
    separately assembled lower entries to VAL_TOL (test above)."""
    import scipy.sparse as sp
    cfg, g, o = pair
    rp, ci = g.micro_pattern()
    for node in (0, g.n_macro - 1):
        A = sp.csr_matrix((g.micro_values(node), ci, rp), shape=(g.n_micro, g.n_micro))
        assert (A != A.T).nnz == 0


def test_generic_solve(pair):
    cfg, g, o = pair
    out = g.solve(outer_tol=cfg.outer_tol)
    ref = o.solve(outer_tol=cfg.outer_tol)
    assert out["sweeps"] == ref["sweeps"]
    for k in ("u", "w", "V"):
        assert rel(out[k], ref[k]) <= SOL_TOL, k
    assert out["micro_dof_iters"] == pytest.approx(ref["micro_dof_iters"], rel=0.02)


def test_generic_path_2d_q1_matches_reference(ref_mod):
    """The generic kernels on the reference's own 2D Q1 problem (symbolic config-1 map)."""
    cfg = configs.CONFIGS["c1"].reduced().resized(8, 12)
    g = abi.Context(cfg.ini(), cfg.ext(reference_expressible=True, force_generic=True))
    r = ref_mod.RefContext(cfg.ini(), 1)
    rp, ci = g.micro_pattern()
    rrp, rci = r.micro_pattern()
    assert np.array_equal(rp, rrp) and np.array_equal(ci, rci)
    for node in (0, 40, g.n_macro - 1):
        assert maxrel(g.micro_values(node), r.micro_values(node)) <= VAL_TOL
        assert maxrel(g.micro_rhs(node, 1.0, 0.0), r.micro_rhs(node, 1.0, 0.0)) <= VAL_TOL
    out = g.solve(outer_tol=cfg.outer_tol)
    ref = r.solve(outer_tol=cfg.outer_tol)
    assert out["sweeps"] == ref["sweeps"]
    for k in ("u", "V"):
        assert rel(out[k], ref[k]) <= SOL_TOL


def test_3d_micro_beyond_smem_matches_oracle(port_mod):
    """3D micro 22^3 (12167 nodes): CG vectors in global scratch (generic GLOBAL variant)."""
    cfg = configs.CONFIGS["c5"].resized(2, 22)
    g = abi.Context(cfg.ini(), cfg.ext())
    o = port_mod.GenOracleContext(cfg)
    out = g.solve(outer_tol=cfg.outer_tol)
    ref = o.solve(outer_tol=cfg.outer_tol)
    assert out["sweeps"] == ref["sweeps"]
    for k in ("u", "V"):
        assert rel(out[k], ref[k]) <= SOL_TOL


@pytest.mark.parametrize("mode,macro_n,micro_n", [("auto", 4, 12), ("1", 5, 16), ("0", 4, 12)])
def test_3d_cluster_kernel_matches_oracle(port_mod, monkeypatch, mode, macro_n, micro_n):
    """3D micro problems on 4-CTA thread-block clusters (k_gen_pcg3_cluster: node ranges,
    p halos and dot products over DSMEM, split barrier around the interior SpMV) — chosen
    automatically for batches smaller than the GPU (25 problems of 13^3), forced on full
    17^3 lattices (36 problems), off — against the generic C oracle."""
    if mode == "auto":
        monkeypatch.delenv("TS_GEN_CLUSTER", raising=False)
    else:
        monkeypatch.setenv("TS_GEN_CLUSTER", mode)
    cfg = configs.CONFIGS["c5"].resized(macro_n, micro_n)
    g = abi.Context(cfg.ini(), cfg.ext())
    o = port_mod.GenOracleContext(cfg)
    out = g.solve(outer_tol=cfg.outer_tol)
    ref = o.solve(outer_tol=cfg.outer_tol)
    assert out["sweeps"] == ref["sweeps"]
    for k in ("u", "w", "V"):
        assert rel(out[k], ref[k]) <= SOL_TOL, k


@pytest.mark.parametrize("mode", ["compact", "compact-classwarps", "plain", "tensor"])
def test_q2_kernels_match_oracle(port_mod, monkeypatch, mode):
    """Config 4 through the class-compact Q2 kernel (default), the plain generic kernel
    (TS_GEN_Q2C=0) and the matrix-free coefficient-tensor kernel (TS_GEN_Q2T=1, the north
    star's second operator representation); also a micro grid whose node lattice is larger
    than the config's (21x21 -> 41x41 nodes, odd class / colour counts)."""
    if not abi.device_ok():
        pytest.fail("no usable sm_100 device")
    monkeypatch.setenv("TS_GEN_Q2C", "0" if mode == "plain" else "1")
    monkeypatch.setenv("TS_GEN_Q2T", "1" if mode == "tensor" else "0")
    # the 2-CTA cluster kernel: block-pair thread mapping (default) or one class per warp
    monkeypatch.setenv("TS_GEN_Q2B", "0" if mode == "compact-classwarps" else "1")
    cfg = configs.CONFIGS["c4"].resized(5, 20)
    g = abi.Context(cfg.ini(), cfg.ext())
    assert g.info["micro_kernel"] == {"compact": 3, "compact-classwarps": 3, "plain": 2, "tensor": 4}[mode]
    o = port_mod.GenOracleContext(cfg)
    out = g.solve(outer_tol=cfg.outer_tol)
    ref = o.solve(outer_tol=cfg.outer_tol)
    assert out["sweeps"] == ref["sweeps"]
    for k in ("u", "w", "V"):
        assert rel(out[k], ref[k]) <= SOL_TOL, k
    # one cold batched solve: per-problem iteration counts against the oracle's cg_solve
    u, w = np.full(g.n_macro, 0.05), np.zeros(g.n_macro)
    V, it, _ = g.micro_solve(u, w)
    oV, oit = o.micro_sweep(u, w)
    assert np.abs(it.astype(int) - oit).max() <= 2 and rel(V, oV) <= SOL_TOL


@pytest.mark.parametrize("name,macro_n,micro_n", [("c4", 3, 32), ("c5", 3, 16), ("c4", 2, 7), ("c5", 2, 5)])
def test_compile_time_assembly_is_bitwise_the_runtime_one(monkeypatch, name, macro_n, micro_n):
    """k_gassemble_t (element structure at compile time, row in registers) against the
    runtime-structure k_gassemble (TS_GASSEMBLE_RT=1): identical operator bits."""
    if not abi.device_ok():
        pytest.fail("no usable sm_100 device")
    cfg = configs.CONFIGS[name].resized(macro_n, micro_n)
    monkeypatch.delenv("TS_GASSEMBLE_RT", raising=False)
    a = abi.Context(cfg.ini(), cfg.ext())
    monkeypatch.setenv("TS_GASSEMBLE_RT", "1")
    b = abi.Context(cfg.ini(), cfg.ext())
    for node in range(a.n_macro):
        assert np.array_equal(a.micro_values(node), b.micro_values(node)), node


@pytest.mark.parametrize("cg1", ["0", "1"])
@pytest.mark.parametrize("macro_n,micro_n", [(4, 16), (3, 12)])
def test_3d_zcol_kernel_matches_oracle(port_mod, monkeypatch, cg1, macro_n, micro_n):
    """The z-column cluster kernel (k_gen_pcg3_zcol: SMEM-resident operator on 4-CTA
    clusters, z-window SpMV, st.async exchanges) on 17^3 and 13^3 lattices, with the standard
    two-reduction PCG and the single-reduction (Chronopoulos-Gear) loop (TS_GEN_CG1=1):
    fixed-point solve and per-problem iteration counts of a cold batched solve against the
    generic C oracle."""
    if not abi.device_ok():
        pytest.fail("no usable sm_100 device")
    monkeypatch.delenv("TS_GEN_ZCOL", raising=False)
    monkeypatch.setenv("TS_GEN_CG1", cg1)
    cfg = configs.CONFIGS["c5"].resized(macro_n, micro_n)
    g = abi.Context(cfg.ini(), cfg.ext())
    o = port_mod.GenOracleContext(cfg)
    out = g.solve(outer_tol=cfg.outer_tol)
    ref = o.solve(outer_tol=cfg.outer_tol)
    assert out["sweeps"] == ref["sweeps"]
    for k in ("u", "w", "V"):
        assert rel(out[k], ref[k]) <= SOL_TOL, k
    u, w = np.full(g.n_macro, 0.05), np.zeros(g.n_macro)
    V, it, _ = g.micro_solve(u, w)
    oV, oit = o.micro_sweep(u, w)
    assert np.abs(it.astype(int) - oit).max() <= 2 and rel(V, oV) <= SOL_TOL


@pytest.mark.parametrize("name,macro_n,micro_n", [("c4", 10, 20), ("c5", 7, 12)])
def test_cluster_kernels_reuse_a_cluster_for_many_problems(port_mod, name, macro_n, micro_n):
    """More problems than resident clusters on the smaller instantiated lattices (41 x 41 Q2:
    121 problems on <= 74 2-CTA clusters; 13^3: 64 problems on <= 33 4-CTA clusters): every
    cluster solves several problems in turn, reloading its shared-memory operator and p blocks."""
    if not abi.device_ok():
        pytest.fail("no usable sm_100 device")
    cfg = configs.CONFIGS[name].resized(macro_n, micro_n)
    g = abi.Context(cfg.ini(), cfg.ext())
    o = port_mod.GenOracleContext(cfg)
    u = np.linspace(0.02, 0.08, g.n_macro)
    w = np.linspace(-0.01, 0.03, g.n_macro)
    V, it, _ = g.micro_solve(u, w)
    oV, oit = o.micro_sweep(u, w)
    assert np.abs(it.astype(int) - oit).max() <= 2 and rel(V, oV) <= SOL_TOL
    out = g.solve(outer_tol=cfg.outer_tol)
    ref = o.solve(outer_tol=cfg.outer_tol)
    assert out["sweeps"] == ref["sweeps"]
    for k in ("u", "w", "V"):
        assert rel(out[k], ref[k]) <= SOL_TOL, k


CLUSTER_CASES = [
    ("c5-zcol-cg1", "c5", 2, 16, {"TS_GEN_CG1": "1"}),
    ("c5-zcol-2red", "c5", 2, 16, {"TS_GEN_CG1": "0"}),
    ("c4-q2cl-cg1", "c4", 2, 32, {"TS_GEN_CG1": "1"}),
    ("c4-q2cl-2red", "c4", 2, 32, {"TS_GEN_CG1": "0"}),
    ("c4-q2cl-classwarps-cg1", "c4", 2, 32, {"TS_GEN_CG1": "1", "TS_GEN_Q2B": "0"}),
    ("c4-q2cl-classwarps-2red", "c4", 2, 32, {"TS_GEN_CG1": "0", "TS_GEN_Q2B": "0"}),
]


@pytest.mark.parametrize("name,base,macro_n,micro_n,env", CLUSTER_CASES, ids=[c[0] for c in CLUSTER_CASES])
def test_cluster_kernels_failure_semantics(port_mod, monkeypatch, name, base, macro_n, micro_n, env):
    """The cluster kernels (z-column 3D, Q2 2-CTA) on the BASELINE lattices, both PCG loops:
    a strongly negative reaction makes the micro operators indefinite, and each problem must
    stop at p.Ap <= 0 (src/linalg.cpp:138-142) at the iteration the CPU cg_solve stops it
    (+-1), with the first failing system reported as the reference does (solver.cpp:91-97);
    converged problems keep their iteration counts; maxit exhaustion is reported as the
    reference's non-convergence."""
    import dataclasses
    if not abi.device_ok():
        pytest.fail("no usable sm_100 device")
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    cfg = dataclasses.replace(configs.CONFIGS[base].resized(macro_n, micro_n), reaction=("const", -300.0))
    g = abi.Context(cfg.ini(), cfg.ext())
    u = np.linspace(0.02, 0.1, g.n_macro)
    w = np.zeros(g.n_macro)
    V, it, _, st = g.micro_solve(u, w, raise_on_fail=False)
    rp, ci = g.micro_pattern()
    o = port_mod.GenOracleContext(cfg)
    first = None
    for i in range(g.n_macro):
        b = u[i] * o.rhs_parts(i)[0]
        _, conv, oit, _, indef = port_mod.cg_solve(rp, ci, g.micro_values(i), b, np.zeros_like(b), 1e-10, 20000)
        if indef:
            assert abs(int(it[i]) - oit) <= 1, (i, it[i], oit)
            first = i if first is None else first
        else:
            assert conv and abs(int(it[i]) - oit) <= max(2, 0.02 * oit), (i, it[i], oit)
    assert first is not None, "no indefinite system: raise |k|"
    assert st == abi.TS_ERR_SOLVER
    assert abi.lib().ts_last_error().decode() == f"micro system {first}: CG detected negative curvature"
    # maxit: a healthy operator stopped after 3 iterations
    cfg2 = configs.CONFIGS[base].resized(macro_n, micro_n)
    g2 = abi.Context(cfg2.ini(), cfg2.ext())
    u2 = np.full(g2.n_macro, 0.05)
    _, it2, _, st2 = g2.micro_solve(u2, np.zeros(g2.n_macro), maxit=3, raise_on_fail=False)
    interior = [i for i in range(g2.n_macro) if it2[i] > 0]
    assert st2 == abi.TS_ERR_SOLVER and all(int(it2[i]) == 3 for i in interior)
    msg = abi.lib().ts_last_error().decode()
    assert msg.startswith(f"micro system {interior[0]}: CG failed to converge"), msg
