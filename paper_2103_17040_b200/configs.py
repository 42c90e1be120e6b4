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
    _table: np.ndarray | None = field(default=None, repr=False)

    # ---------------------------------------------------------------- sizes --
    @property
    def n_macro(self):
        return (self.macro_n + 1) ** 2

    @property
    def n_micro(self):
        return (self.micro_n + 1) ** 2

    @property
    def micro_nnz(self):
        return (3 * self.micro_n + 1) ** 2

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
        if self.map != "table":
            return None
        if self._table is None:
            self._table = make_table(self.macro_n, self.micro_n, self.seed, self.table_eps, self.amp, self.det_min)
        return self._table

    def ext(self, reference_expressible=False):
        """Extension block for ts_ctx_create_ini.  reference_expressible drops k, D and the table."""
        if reference_expressible:
            return abi.make_ext()
        return abi.make_ext(D=self.D, reaction=self.reaction, table=self.table(),
                            s_kind=abi.TS_S_PRODUCT, amp=self.amp)

    def reduced(self) -> "TwoScaleConfig":
        """The reference-expressible stand-in: k = 0, D = I, symbolic map."""
        return TwoScaleConfig(self.name + "-ref", self.macro_n, self.micro_n,
                              "c2" if self.map == "table" else self.map, reaction=None,
                              kappa=self.kappa, inner_tol=self.inner_tol, outer_tol=self.outer_tol)

    def resized(self, macro_n, micro_n) -> "TwoScaleConfig":
        c = TwoScaleConfig(self.name + f"@{macro_n}x{micro_n}", macro_n, micro_n, self.map, self.reaction,
                           self.D, self.table_eps, self.amp, self.det_min, self.seed, self.kappa,
                           self.inner_tol, self.outer_tol)
        return c

    # bytes the batched PCG's operator representation needs per micro DoF (CSR,
    # SURVEY.md §8d) — the denominator of the north-star roofline
    @property
    def csr_bytes_per_dof(self):
        return 8.0 * self.micro_nnz / self.n_micro


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

    def min_det(idx):
        out = np.empty(len(idx))
        for k0 in range(0, len(idx), 256):
            sl = idx[k0:k0 + 256]
            a = (amp * s[sl])[:, None]
            F00 = A[sl, 0, 0][:, None] + a * g0[None]
            F01 = A[sl, 0, 1][:, None] + a * g1[None]
            F10 = A[sl, 1, 0][:, None] + a * g0[None]
            F11 = A[sl, 1, 1][:, None] + a * g1[None]
            out[k0:k0 + 256] = (F00 * F11 - F01 * F10).min(1)
        return out

    todo = np.arange(nodes)
    for _ in range(1000):
        bad = todo[min_det(todo) < det_min]
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
}
