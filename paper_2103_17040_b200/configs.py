"""BASELINE.json workloads as deterministic synthetic problems.

Each config renders (a) INI text in the reference grammar (config.cpp:126-266),
(b) the extension block for what that grammar cannot express (reaction k, tensor
D, per-node tabulated A(x)), and (c) its reference-expressible reduction (k = 0,
D = I, symbolic C2-family map) used for parity against the reference binary.
There is no public dataset on this path; all inputs are seeded synthetic data
with the shapes BASELINE.json names.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import abi

PI = 3.141592653589793
SEED = 12345  # the reference's own default seed (mms.hpp:31)

# zeta expressions (config 1 and the config-2 family), 0-based variables
C1_ZETA = ("y0 + 0.1*sin(2*pi*x0)*cos(2*pi*x1)*16*y0*(1-y0)*y1*(1-y1)",
           "y1 + 0.1*sin(2*pi*x0)*cos(2*pi*x1)*16*y0*(1-y0)*y1*(1-y1)")
C2_ZETA = ("(1+0.1*sin(2*pi*x0))*y0 + 0.1*cos(2*pi*x1)*y1 + 0.15*x0*x1*16*y0*(1-y0)*y1*(1-y1)",
           "0.1*cos(2*pi*x0)*y0 + (1+0.1*sin(2*pi*x1))*y1 + 0.15*x0*x1*16*y0*(1-y0)*y1*(1-y1)")


@dataclass
class TwoScaleConfig:
    name: str
    macro_n: int
    micro_n: int
    map: str                      # "c1" | "c2" | "table"
    reaction: tuple | None = ("const", 1.0)
    D: tuple = (1.0, 0.0, 0.0, 1.0)
    table_eps: float = 0.25
    amp: float = 0.15
    det_min: float = 0.3
    seed: int = SEED
    kappa: tuple = (1.0, 1.0, 0.0, 0.0)
    inner_tol: float = 1e-10
    outer_tol: float = 1e-10
    description: str = ""
    dim: int = 2                  # micro dimension (2 or 3)
    order: int = 1                # micro element order (1 = Q1, 2 = Q2)
    _table: np.ndarray | None = field(default=None, repr=False)

    @property
    def generic(self):
        """Q2 or 3D micro problems run on the generic (streaming-stencil) path."""
        return self.dim != 2 or self.order != 1

    # ---------------------------------------------------------------- sizes --
    @property
    def n_macro(self):
        return (self.macro_n + 1) ** 2

    @property
    def n_micro(self):
        return (self.order * self.micro_n + 1) ** self.dim

    @property
    def micro_nnz(self):
        if self.order == 1:
            return (3 * self.micro_n + 1) ** self.dim
        # Q2 1D coupling counts: vertex nodes 5, edge-interior nodes 3 (interior); boundary vertices 3
        n = self.micro_n
        per_axis = 2 * 3 + (n - 1) * 5 + n * 3
        return per_axis ** self.dim

    # ------------------------------------------------------------ rendering --
    def zeta(self):
        return C1_ZETA if self.map == "c1" else C2_ZETA

    def ini(self, macro_n=None, micro_n=None) -> str:
        z0, z1 = self.zeta()
        k1, k2, k3, k4 = self.kappa
        return f"""
[macro]
lo0 = 0
lo1 = 0
hi0 = 1
hi1 = 1
n0 = {macro_n or self.macro_n}
n1 = {macro_n or self.macro_n}
dirichlet = left,right,bottom,top
[micro]
lo0 = 0
lo1 = 0
hi0 = 1
hi1 = 1
n0 = {micro_n or self.micro_n}
n1 = {micro_n or self.micro_n}
zeta0 = {z0}
zeta1 = {z1}
gamma_i = left,right,bottom,top
gamma_o =
gamma_n =
[parameters]
kappa1 = {k1!r}
kappa2 = {k2!r}
kappa3 = {k3!r}
kappa4 = {k4!r}
Dv = 1
Dw = 1
fu = 1
u0 = 0
pi = {PI!r}
[solver]
inner_tol = {self.inner_tol!r}
outer_tol = {self.outer_tol!r}
"""

    def table(self):
        if self.map not in ("table", "fourier", "table3"):
            return None
        if self._table is None:
            if self.map == "table":
                self._table = make_table(self.macro_n, self.micro_n, self.seed, self.table_eps, self.amp, self.det_min)
            elif self.map == "fourier":
                self._table = make_fourier_table(self.macro_n, self.micro_n, self.order, self.seed, self.table_eps,
                                                 self.det_min)
            else:
                self._table = make_table3(self.macro_n, self.micro_n, self.seed, self.table_eps, self.amp,
                                          self.det_min)
        return self._table

    def ext(self, reference_expressible=False, force_generic=False):
        """Extension block for ts_ctx_create_ini.  reference_expressible drops k, D and the table;
        force_generic runs a 2D Q1 problem through the generic (Q2/3D) device path."""
        if reference_expressible and not force_generic:
            return abi.make_ext()
        if reference_expressible:
            return abi.make_ext(dim=2, order=1, force_generic=True)
        kind = {"table": abi.TS_MAP_AFFINE_BUBBLE_TABLE, "table3": abi.TS_MAP_AFFINE_BUBBLE_TABLE,
                "fourier": abi.TS_MAP_FOURIER_TABLE}.get(self.map, abi.TS_MAP_TAPE)
        return abi.make_ext(D=self.D, reaction=self.reaction, table=self.table(), map_kind=kind,
                            s_kind=abi.TS_S_PRODUCT, amp=self.amp, dim=self.dim, order=self.order,
                            micro_n=self.micro_n, force_generic=force_generic)

    def reduced(self) -> "TwoScaleConfig":
        """The reference-expressible stand-in: k = 0, D = I, symbolic map."""
        return TwoScaleConfig(self.name + "-ref", self.macro_n, self.micro_n,
                              "c2" if self.map == "table" else self.map, reaction=None,
                              kappa=self.kappa, inner_tol=self.inner_tol, outer_tol=self.outer_tol)

    def resized(self, macro_n, micro_n) -> "TwoScaleConfig":
        c = TwoScaleConfig(self.name + f"@{macro_n}x{micro_n}", macro_n, micro_n, self.map, self.reaction,
                           self.D, self.table_eps, self.amp, self.det_min, self.seed, self.kappa,
                           self.inner_tol, self.outer_tol, self.description, self.dim, self.order)
        return c

    # bytes the batched PCG's operator representation needs per micro DoF (CSR,
    # SURVEY.md §8d) — the denominator of the north-star roofline
    @property
    def csr_bytes_per_dof(self):
        return 8.0 * self.micro_nnz / self.n_micro

    # the coefficient-tensor representation: per cell quadrature point the
    # symmetric pulled-back tensor plus J k (4 doubles in 2D, 7 in 3D), per face point |nu|
    @property
    def tensor_bytes_per_dof(self):
        q1 = self.order + 1
        cells = self.micro_n ** self.dim
        faces = 2 * self.dim * self.micro_n ** (self.dim - 1)
        per_q = 4 if self.dim == 2 else 7
        return 8.0 * (cells * q1 ** self.dim * per_q + faces * q1 ** (self.dim - 1)) / self.n_micro

    @property
    def alg_bytes_per_dof(self):
        """B_alg of SURVEY.md §8d: the smaller of the two operator representations."""
        return min(self.csr_bytes_per_dof, self.tensor_bytes_per_dof)


def micro_quadrature_points(micro_n, lo=0.0, hi=1.0):
    """All Gauss-2 cell and face points of the micro grid (grid.cpp:134-141, 121-127)."""
    h = (hi - lo) / micro_n
    g = 1.0 / np.sqrt(3.0)
    gp = np.array([-g, g])
    c = lo + (np.arange(micro_n) + 0.5) * h
    cell1d = (c[:, None] + 0.5 * h * gp[None, :]).reshape(-1)
    Y0, Y1 = np.meshgrid(cell1d, cell1d, indexing="xy")
    pts = [np.stack([Y0.reshape(-1), Y1.reshape(-1)], 1)]
    edge = cell1d
    for fixed in (lo, hi):
        pts.append(np.stack([np.full_like(edge, fixed), edge], 1))
        pts.append(np.stack([edge, np.full_like(edge, fixed)], 1))
    return np.concatenate(pts, 0)


def gauss_1d(npts):
    if npts == 2:
        g = 1.0 / np.sqrt(3.0)
        return np.array([-g, g])
    g = np.sqrt(3.0 / 5.0)
    return np.array([-g, 0.0, g])


def micro_qpoints_generic(micro_n, dim, order):
    """Cell Gauss-(order+1)^dim points and face Gauss-(order+1)^(dim-1) points of the unit box."""
    h = 1.0 / micro_n
    gp = gauss_1d(order + 1)
    c = (np.arange(micro_n) + 0.5) * h
    line = (c[:, None] + 0.5 * h * gp[None, :]).reshape(-1)
    grids = np.meshgrid(*([line] * dim), indexing="ij")
    pts = [np.stack([g.reshape(-1) for g in grids], 1)]
    for a in range(dim):
        for fixed in (0.0, 1.0):
            tr = np.meshgrid(*([line] * (dim - 1)), indexing="ij")
            cols = []
            t = 0
            for k in range(dim):
                if k == a:
                    cols.append(np.full(tr[0].size, fixed))
                else:
                    cols.append(tr[t].reshape(-1))
                    t += 1
            pts.append(np.stack(cols, 1))
    return np.concatenate(pts, 0)


def _failing(min_det, idx, n_points, det_min, stride=16):
    """Mask of the draws in idx whose det J falls below det_min at some quadrature point.
    Screened first on every stride-th point: a draw failing there fails on the full set
    (a subset's minimum is >= the full minimum), so only the survivors are evaluated on all
    points.  Same decisions as evaluating every point, so the same table."""
    bad = min_det(idx, np.arange(0, n_points, stride)) < det_min
    keep = np.flatnonzero(~bad)
    if len(keep):
        bad[keep] = min_det(idx[keep], np.arange(n_points)) < det_min
    return bad


FOURIER_K = np.array([1, 1, 2, 2, 1, 3, 2, 3])
FOURIER_L = np.array([1, 2, 1, 2, 3, 1, 3, 2])


def make_fourier_table(macro_n, micro_n, order=2, seed=SEED, sigma=0.05, det_min=0.3):
    """Config 4: per node c[a][m] ~ N(0, sigma^2), zeta_a = y_a + sum_m c[a][m] sin(pi k_m y0) sin(pi l_m y1),
    nodes redrawn in order until det J >= det_min at every micro quadrature point."""
    rng = np.random.Generator(np.random.PCG64(seed))
    nodes = (macro_n + 1) ** 2
    Y = micro_qpoints_generic(micro_n, 2, order)
    pk, pl = np.pi * FOURIER_K[:, None], np.pi * FOURIER_L[:, None]
    G0 = pk * np.cos(pk * Y[None, :, 0]) * np.sin(pl * Y[None, :, 1])   # d phi_m / d y0, [8, P]
    G1 = pl * np.sin(pk * Y[None, :, 0]) * np.cos(pl * Y[None, :, 1])
    C = rng.normal(0.0, sigma, size=(nodes, 2, 8))

    def min_det(idx, pts):
        g0, g1 = G0[:, pts], G1[:, pts]
        out = np.empty(len(idx))
        for k0 in range(0, len(idx), 128):
            sl = idx[k0:k0 + 128]
            F00 = 1.0 + C[sl, 0] @ g0
            F01 = C[sl, 0] @ g1
            F10 = C[sl, 1] @ g0
            F11 = 1.0 + C[sl, 1] @ g1
            out[k0:k0 + 128] = (F00 * F11 - F01 * F10).min(1)
        return out

    todo = np.arange(nodes)
    for _ in range(1000):
        bad = todo[_failing(min_det, todo, Y.shape[0], det_min)]
        if len(bad) == 0:
            break
        C[bad] = rng.normal(0.0, sigma, size=(len(bad), 2, 8))
        todo = bad
    else:
        raise RuntimeError("rejection sampling did not converge")
    return C.reshape(nodes, 16).copy()


def make_table3(macro_n, micro_n, seed=SEED, eps=0.2, amp=0.1, det_min=0.3):
    """Config 5: A_i = I + eps R_i (3x3, U(-1,1)), zeta = A_i y + amp x0 x1 64 prod y_k(1-y_k) (1,1,1);
    nodes redrawn in order until det J >= det_min at every Gauss-2 cell / face point."""
    rng = np.random.Generator(np.random.PCG64(seed))
    nodes = (macro_n + 1) ** 2
    xs = np.arange(macro_n + 1) / macro_n
    X0, X1 = np.meshgrid(xs, xs, indexing="xy")
    s = (X0 * X1).reshape(-1)
    Y = micro_qpoints_generic(micro_n, 3, 1)
    q = Y * (1.0 - Y)
    gb = np.stack([64.0 * (1.0 - 2.0 * Y[:, 0]) * q[:, 1] * q[:, 2],
                   64.0 * (1.0 - 2.0 * Y[:, 1]) * q[:, 0] * q[:, 2],
                   64.0 * (1.0 - 2.0 * Y[:, 2]) * q[:, 0] * q[:, 1]], 1)       # [P, 3]
    A = np.eye(3)[None] + eps * rng.uniform(-1.0, 1.0, size=(nodes, 3, 3))

    def min_det(idx, pts):
        g = gb[pts]
        out = np.empty(len(idx))
        for k0 in range(0, len(idx), 256):
            sl = idx[k0:k0 + 256]
            a = amp * s[sl]
            # F = A + a (1,1,1) g^T, so det F = det A + a g . (adj(A) (1,1,1)) (matrix determinant
            # lemma); rows whose minimum lies within 1e-9 of the threshold are redone with
            # np.linalg.det on F itself, so every accept/reject decision is unchanged
            Ab = A[sl]
            adj1 = np.stack([np.cross(Ab[:, 1], Ab[:, 2]), np.cross(Ab[:, 2], Ab[:, 0]),
                             np.cross(Ab[:, 0], Ab[:, 1])], 2).sum(2)      # adj(A) @ (1,1,1)
            d = (np.linalg.det(Ab)[:, None] + a[:, None] * (adj1 @ g.T)).min(1)
            near = np.flatnonzero(np.abs(d - det_min) < 1e-9)
            for r in near:
                F = Ab[r][None] + (a[r] * g)[:, None, :]
                d[r] = np.linalg.det(F).min()
            out[k0:k0 + 256] = d
        return out

    todo = np.arange(nodes)
    for _ in range(1000):
        bad = todo[_failing(min_det, todo, Y.shape[0], det_min)]
        if len(bad) == 0:
            break
        A[bad] = np.eye(3)[None] + eps * rng.uniform(-1.0, 1.0, size=(len(bad), 3, 3))
        todo = bad
    else:
        raise RuntimeError("rejection sampling did not converge")
    return A.reshape(nodes, 9).copy()


def make_table(macro_n, micro_n, seed=SEED, eps=0.25, amp=0.15, det_min=0.3):
    """Per-node A_i = I + eps R_i, R_i ~ U(-1,1)^{2x2} i.i.d. (numpy PCG64(seed)); nodes whose
    map zeta = A_i y + amp x0 x1 beta(y)(1,1) has det J < det_min at any micro quadrature
    point are redrawn, in node order, until all pass (BASELINE.json config 3)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    nodes = (macro_n + 1) ** 2
    xs = np.arange(macro_n + 1) / macro_n
    X0, X1 = np.meshgrid(xs, xs, indexing="xy")
    s = (X0 * X1).reshape(-1)  # s(x) = x0 x1 at node i (lexicographic, j*(n+1)+i)
    Y = micro_quadrature_points(micro_n)
    g0 = 16.0 * (1.0 - 2.0 * Y[:, 0]) * Y[:, 1] * (1.0 - Y[:, 1])
    g1 = 16.0 * Y[:, 0] * (1.0 - Y[:, 0]) * (1.0 - 2.0 * Y[:, 1])
    A = np.eye(2)[None] + eps * rng.uniform(-1.0, 1.0, size=(nodes, 2, 2))

    def min_det(idx, pts):
        h0, h1 = g0[pts], g1[pts]
        out = np.empty(len(idx))
        for k0 in range(0, len(idx), 1024):
            sl = idx[k0:k0 + 1024]
            a = (amp * s[sl])[:, None]
            A00, A01, A10, A11 = (A[sl, r, c][:, None] for r, c in ((0, 0), (0, 1), (1, 0), (1, 1)))
            # F = A + a (1,1) (g0,g1): det F = det A + a (g0 (A11 - A01) + g1 (A00 - A10)) (matrix
            # determinant lemma); rows within 1e-9 of the threshold are redone on F itself
            d = (A00 * A11 - A01 * A10 + a * ((A11 - A01) * h0[None] + (A00 - A10) * h1[None])).min(1)
            for r in np.flatnonzero(np.abs(d - det_min) < 1e-9):
                F00, F01 = A00[r] + a[r] * h0, A01[r] + a[r] * h1
                F10, F11 = A10[r] + a[r] * h0, A11[r] + a[r] * h1
                d[r] = (F00 * F11 - F01 * F10).min()
            out[k0:k0 + 1024] = d
        return out

    todo = np.arange(nodes)
    for _ in range(1000):
        bad = todo[_failing(min_det, todo, Y.shape[0], det_min)]
        if len(bad) == 0:
            break
        A[bad] = np.eye(2)[None] + eps * rng.uniform(-1.0, 1.0, size=(len(bad), 2, 2))
        todo = bad
    else:
        raise RuntimeError("rejection sampling did not converge")
    return A.reshape(nodes, 4).copy()


CONFIGS = {
    "c1": TwoScaleConfig("c1-smoke", 16, 16, "c1",
                         description="2D smoke: macro Q1 16x16, micro Q1 16x16, config-1 map, D=I, k=1"),
    "c2": TwoScaleConfig("c2-mid", 64, 32, "c2",
                         description="2D mid: macro Q1 64x64 (4225 problems), micro Q1 32x32, C2 map, D=I, k=1"),
    "c3": TwoScaleConfig("c3-large", 128, 64, "table", D=(1.0, 0.0, 0.0, 0.1),
                         description="2D large: macro Q1 128x128 (16641 problems), micro Q1 64x64, "
                                     "A(x)=I+0.25R seeded table (det>=0.3), D=diag(1,0.1), k=1"),
    "c4": TwoScaleConfig("c4-q2", 64, 32, "fourier", reaction=("disc", 1.0, 10.0, 0.5, 0.5, 0.3),
                         table_eps=0.05, order=2,
                         description="2D heterogeneous Q2: macro Q1 64x64 (4225 problems), micro Q2 32x32 "
                                     "(4225 DoFs), 8-mode seeded Fourier map (det>=0.3), k=1 in r<0.3 else 10"),
    "c5": TwoScaleConfig("c5-3d", 64, 16, "table3", table_eps=0.2, amp=0.1, dim=3,
                         description="3D micro: macro Q1 64x64 (4225 problems), micro Q1 16^3 (4913 DoFs), "
                                     "A(x)=I+0.2R 3x3 seeded table (det>=0.3), 0.1 x0 x1 cubic bubble, D=I, k=1"),
}
