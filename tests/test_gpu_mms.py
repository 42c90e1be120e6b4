"""The manufactured-solution pipeline on the device against the reference: the
derived problem exercises every data term of the path (f^v o zeta, g^v Robin
corrections with sqrt/division, flux functionals, Neumann g^u/g^w, Dirichlet u0+g^u1,
x-independent Jacobian -> shared micro operator), and error_norms (SURVEY.md §8f
rank 1) runs as a batched device reduction.  Case: the paper's manufactured system
(PAPER.md manu_system; SPEC.md)."""
import numpy as np
import pytest

from paper_2103_17040_b200 import abi

pytestmark = pytest.mark.gpu

MMS_INI = """
[macro]
n0 = {n}
n1 = {n}
[micro]
n0 = {m}
n1 = {m}
zeta0 = 0.4*((x0 + 1.3)+(1.4*y0 - 0.54*y1))
zeta1 = 0.3*((x1 + 1.2)+(-0.4*y0 + 0.8*y1))
[parameters]
kappa1 = 1
kappa2 = 1
kappa3 = 1
kappa4 = 1
Dv = 1
Dw = 1
[mms]
u = x1*sin(x0)
v = x0 + x1 + y0*y1*(1-y1)
w = x0*cos(x1)
[solver]
inner_tol = 1e-12
outer_tol = 1e-10
"""


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def test_mms_problem_solve_matches_reference(ref_mod):
    ini = MMS_INI.format(n=6, m=5)
    g = abi.Context(ini, mms=True)
    assert g.info["shared_operator"] == 1          # affine-in-y map: one micro matrix
    out = g.solve()
    ref = ref_mod.mms_solve(ini, g.n_macro, g.n_micro)
    assert out["sweeps"] == ref["sweeps"]
    for k in ("u", "w", "V"):
        assert rel(out[k], ref[k]) <= 1e-8, k


def test_error_norms_kernel_matches_reference(ref_mod):
    ini = MMS_INI.format(n=5, m=7)
    g = abi.Context(ini, mms=True)
    rng = np.random.default_rng(1)
    u = rng.standard_normal(g.n_macro)
    w = rng.standard_normal(g.n_macro)
    V = rng.standard_normal((g.n_macro, g.n_micro))
    np.testing.assert_allclose(abi.error_norms(ini, u, w, V), ref_mod.error_norms(ini, u, w, V), rtol=1e-12)
    s = g.solve()
    np.testing.assert_allclose(abi.error_norms(ini, s["u"], s["w"], s["V"]),
                               ref_mod.error_norms(ini, s["u"], s["w"], s["V"]), rtol=1e-10)


def test_convergence_sweep_matches_reference(ref_mod):
    ini = MMS_INI.format(n=4, m=4)
    ns = [4, 8]
    dev = abi.mms_sweep(ini, ns)
    ref = ref_mod.mms_sweep(ini, ns)
    assert np.array_equal(dev[:, :3], ref[:, :3])
    np.testing.assert_allclose(dev[:, 5:9], ref[:, 5:9], rtol=1e-8)
    np.testing.assert_allclose(dev[1, 9:], ref[1, 9:], rtol=1e-6)
    # p in [1.8, 2.3] for e_uw between n = 4 and 8 (the sweep's own check)
    assert 1.8 <= dev[1, 9] <= 2.5


def test_mms_derived_system_pieces_match_reference(ref_mod):
    """Every iterate-independent piece of the derived problem, one by one."""
    ini = MMS_INI.format(n=4, m=5)
    g = abi.Context(ini, mms=True)
    r = ref_mod.RefContext(ini, 1, mms=True)
    d, v = g.dirichlet(0)
    rd, rv = r.dirichlet(0)
    assert np.array_equal(d, rd)
    np.testing.assert_allclose(v, rv, rtol=1e-12, atol=1e-14)
    for which in range(3):
        np.testing.assert_allclose(g.macro_matrix(which)[2], r.macro_matrix(which)[2], rtol=1e-12, atol=1e-13)
    for which in range(2):
        np.testing.assert_allclose(g.macro_rhs(which), r.macro_rhs(which), rtol=1e-11, atol=1e-13)
    for node in (0, 7, g.n_macro - 1):
        np.testing.assert_allclose(g.micro_rhs(node, 0.0, 0.0), r.micro_rhs(node, 0.0, 0.0), rtol=1e-11, atol=1e-13)
        np.testing.assert_allclose(g.micro_rhs(node, 0.3, -0.7), r.micro_rhs(node, 0.3, -0.7), rtol=1e-11, atol=1e-13)
        np.testing.assert_allclose(g.micro_values(node), r.micro_values(node), rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("n,m", [(5, 7), (8, 16)])
def test_compiled_tapes_are_bitwise_the_interpreter(monkeypatch, n, m):
    """error_norms with the tapes compiled to straight-line code at run time (NVRTC, SURVEY.md
    §8f rank 4) returns the interpreter's bits: each tape instruction is the same IEEE
    operation and the kernel body is the same source."""
    ini = MMS_INI.format(n=n, m=m)
    g = abi.Context(ini, mms=True)
    rng = np.random.default_rng(n)
    u = rng.standard_normal(g.n_macro)
    w = rng.standard_normal(g.n_macro)
    V = rng.standard_normal((g.n_macro, g.n_micro))
    monkeypatch.delenv("TS_JIT", raising=False)
    a = abi.error_norms(ini, u, w, V)
    assert abi.jit_status().startswith("compiled"), abi.jit_status()
    monkeypatch.setenv("TS_JIT", "0")
    b = abi.error_norms(ini, u, w, V)
    assert abi.jit_status().startswith("interpreter (TS_JIT=0)"), abi.jit_status()
    assert np.array_equal(a, b), (a, b)
