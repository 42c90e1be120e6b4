"""TEST INFRASTRUCTURE ONLY: ctypes loader for the plain-C oracle (oracle/lib/liboracle.so,
built from oracle/twoscale_oracle.c).  Only tests/, __graft_entry__.smoke() and
bench.py's CPU legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "liboracle.so")

OR_A_IDENTITY, OR_A_TRIG, OR_A_TABLE = 0, 1, 2
OR_S_NONE, OR_S_SINCOS, OR_S_PRODUCT = 0, 1, 2
OR_K_CONST, OR_K_DISC = 0, 1


class or_problem(C.Structure):
    _fields_ = [
        ("macro_lo", C.c_double * 2), ("macro_hi", C.c_double * 2), ("macro_n", C.c_int * 2),
        ("micro_lo", C.c_double * 2), ("micro_hi", C.c_double * 2), ("micro_n", C.c_int * 2),
        ("kappa", C.c_double * 4), ("Dv", C.c_double), ("D", C.c_double * 4),
        ("k_kind", C.c_int), ("k_par", C.c_double * 5),
        ("micro_role", C.c_int * 4), ("macro_dirichlet", C.c_int * 4),
        ("A_kind", C.c_int), ("A_eps", C.c_double), ("A_table", C.POINTER(C.c_double)),
        ("s_kind", C.c_int), ("amp", C.c_double),
        ("fu", C.c_double), ("fw", C.c_double), ("Dw", C.c_double), ("u0", C.c_double),
    ]


_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} not built (make -C oracle oracle)")
        L = C.CDLL(LIB_PATH)
        P, I, D = C.c_void_p, C.c_int, C.c_double
        dp, ip = C.POINTER(C.c_double), C.POINTER(C.c_int)
        L.or_last_error.restype = C.c_char_p
        L.or_create.argtypes = [C.POINTER(or_problem), C.POINTER(P)]
        L.or_destroy.argtypes = [P]
        L.or_sizes.argtypes = [P, ip]
        L.or_micro_pattern.argtypes = [P, ip, ip]
        L.or_micro_values.argtypes = [P, I, dp]
        L.or_micro_rhs_parts.argtypes = [P, I, dp, dp, dp]
        L.or_node_cache.argtypes = [P, I, dp, dp]
        L.or_jac.argtypes = [P, D, D, D, D, dp]
        L.or_macro_matrix.argtypes = [P, I, dp]
        L.or_macro_pattern.argtypes = [P, ip, ip]
        L.or_macro_fixed_rhs.argtypes = [P, dp, dp]
        L.or_surface_coupling.argtypes = [P, dp, I, I]
        L.or_surface_coupling.restype = D
        L.or_cg_solve.argtypes = [I, ip, ip, dp, dp, dp, D, I, ip, dp]
        L.or_fixed_point_solve.argtypes = [P, D, I, D, I, I, dp, dp, dp, dp, I, ip, dp]
        L.or_micro_sweep.argtypes = [P, dp, dp, D, I, I, I, ip, dp, ip]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[oracle code {code}] {msg}")
        self.code = code


def _chk(rc):
    if rc != 0:
        raise OracleError(rc, lib().or_last_error().decode())


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int))


def problem_for(cfg, reference_expressible=False):
    """or_problem for a configs.TwoScaleConfig (map family: c1 / c2 / table)."""
    p = or_problem()
    for k in range(2):
        p.macro_lo[k], p.macro_hi[k], p.macro_n[k] = 0.0, 1.0, cfg.macro_n
        p.micro_lo[k], p.micro_hi[k], p.micro_n[k] = 0.0, 1.0, cfg.micro_n
    for k in range(4):
        p.kappa[k] = cfg.kappa[k]
        p.micro_role[k] = 0  # Gamma^I on all sides
        p.macro_dirichlet[k] = 1
    p.Dv = 1.0
    keep = None
    red = reference_expressible
    D = (1.0, 0.0, 0.0, 1.0) if red else cfg.D
    for k in range(4):
        p.D[k] = D[k]
    if red or cfg.reaction is None:
        p.k_kind, p.k_par[0] = OR_K_CONST, 0.0
    elif cfg.reaction[0] == "disc":
        p.k_kind = OR_K_DISC
        for k, v in enumerate(cfg.reaction[1:]):
            p.k_par[k] = v
    else:
        p.k_kind, p.k_par[0] = OR_K_CONST, cfg.reaction[1]
    m = "c2" if (red and cfg.map == "table") else cfg.map
    if m == "c1":
        p.A_kind, p.s_kind, p.amp = OR_A_IDENTITY, OR_S_SINCOS, 0.1
    elif m == "c2":
        p.A_kind, p.A_eps, p.s_kind, p.amp = OR_A_TRIG, 0.1, OR_S_PRODUCT, 0.15
    else:
        keep = np.ascontiguousarray(cfg.table(), np.float64).reshape(-1)
        p.A_kind, p.A_table, p.s_kind, p.amp = OR_A_TABLE, _dp(keep), OR_S_PRODUCT, cfg.amp
    p.fu, p.fw, p.Dw, p.u0 = 1.0, 0.0, 1.0, 0.0
    return p, keep


class OracleContext:
    def __init__(self, cfg, reference_expressible=False):
        self.p, self._keep = problem_for(cfg, reference_expressible)
        h = C.c_void_p()
        _chk(lib().or_create(C.byref(self.p), C.byref(h)))
        self.h = h
        s = np.zeros(6, np.int32)
        lib().or_sizes(self.h, _ip(s))
        self.n_macro, self.n_micro, self.micro_nnz, self.macro_nnz, self.n_faces, self.n_cells = [int(v) for v in s]

    def close(self):
        if self.h:
            lib().or_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def micro_pattern(self):
        rp = np.zeros(self.n_micro + 1, np.int32)
        ci = np.zeros(self.micro_nnz, np.int32)
        lib().or_micro_pattern(self.h, _ip(rp), _ip(ci))
        return rp, ci

    def micro_values(self, node):
        v = np.zeros(self.micro_nnz)
        _chk(lib().or_micro_values(self.h, node, _dp(v)))
        return v

    def rhs_parts(self, node):
        f = np.zeros(self.n_micro)
        ri = np.zeros(self.n_micro)
        ro = np.zeros(self.n_micro)
        _chk(lib().or_micro_rhs_parts(self.h, node, _dp(f), _dp(ri), _dp(ro)))
        return f, ri, ro

    def node_cache(self, node):
        cells = np.zeros((self.n_cells, 4, 4))
        faces = np.zeros((self.n_faces, 2, 4))
        _chk(lib().or_node_cache(self.h, node, _dp(cells), _dp(faces)))
        return cells, faces

    def macro_matrix(self, which):
        v = np.zeros(self.macro_nnz)
        _chk(lib().or_macro_matrix(self.h, which, _dp(v)))
        return v

    def macro_fixed_rhs(self):
        bu = np.zeros(self.n_macro)
        bw = np.zeros(self.n_macro)
        lib().or_macro_fixed_rhs(self.h, _dp(bu), _dp(bw))
        return bu, bw

    def surface_coupling(self, v, node, role):
        v = np.ascontiguousarray(v, np.float64)
        return float(lib().or_surface_coupling(self.h, _dp(v), node, role))

    def solve(self, inner_tol=1e-10, inner_maxit=20000, outer_tol=1e-10, max_outer=100, threads=1):
        u = np.zeros(self.n_macro)
        w = np.zeros(self.n_macro)
        V = np.zeros((self.n_macro, self.n_micro))
        hist = np.zeros(max_outer + 1)
        info = np.zeros(4, np.int32)
        dof_it = np.zeros(1)
        _chk(lib().or_fixed_point_solve(self.h, inner_tol, inner_maxit, outer_tol, max_outer, threads, _dp(u),
                                        _dp(w), _dp(V), _dp(hist), len(hist), _ip(info), _dp(dof_it)))
        return dict(u=u, w=w, V=V, history=hist[: info[3]].copy(), sweeps=int(info[0]), converged=bool(info[1]),
                    w_pinned=bool(info[2]), micro_dof_iters=float(dof_it[0]))

    def micro_sweep(self, u, w, nodes=None, V=None, tol=1e-10, maxit=20000, threads=1):
        u = np.ascontiguousarray(u, np.float64)
        w = np.ascontiguousarray(w, np.float64)
        if nodes is None:
            n_nodes, np_nodes = self.n_macro, None
        else:
            np_nodes = np.ascontiguousarray(nodes, np.int32)
            n_nodes = len(np_nodes)
        Vout = np.zeros((n_nodes, self.n_micro)) if V is None else np.array(V, np.float64, copy=True)
        iters = np.zeros(n_nodes, np.int32)
        _chk(lib().or_micro_sweep(self.h, _dp(u), _dp(w), tol, maxit, threads, n_nodes,
                                  None if np_nodes is None else _ip(np_nodes), _dp(Vout), _ip(iters)))
        return Vout, iters


def cg_solve(row_ptr, col_idx, vals, b, x0, tol, maxit):
    row_ptr = np.ascontiguousarray(row_ptr, np.int32)
    col_idx = np.ascontiguousarray(col_idx, np.int32)
    vals = np.ascontiguousarray(vals, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    x = np.array(x0, np.float64, copy=True)
    res = np.zeros(3, np.int32)
    resid = np.zeros(1)
    _chk(lib().or_cg_solve(len(b), _ip(row_ptr), _ip(col_idx), _dp(vals), _dp(b), _dp(x), tol, maxit, _ip(res),
                           _dp(resid)))
    return x, bool(res[0]), int(res[1]), float(resid[0]), bool(res[2])


# ----------------------------------------------------------------- generic oracle (configs 4-5)
OG_MAP_AFFINE_BUBBLE, OG_MAP_FOURIER = 0, 1


class og_problem(C.Structure):
    _fields_ = [
        ("macro_lo", C.c_double * 2), ("macro_hi", C.c_double * 2), ("macro_n", C.c_int * 2),
        ("dim", C.c_int), ("order", C.c_int),
        ("micro_lo", C.c_double * 3), ("micro_hi", C.c_double * 3), ("micro_n", C.c_int * 3),
        ("kappa", C.c_double * 4), ("Dv", C.c_double), ("D", C.c_double * 9),
        ("k_kind", C.c_int), ("k_par", C.c_double * 6),
        ("micro_role", C.c_int * 6), ("macro_dirichlet", C.c_int * 4),
        ("map_kind", C.c_int), ("table", C.POINTER(C.c_double)), ("s_kind", C.c_int), ("amp", C.c_double),
        ("fu", C.c_double), ("fw", C.c_double), ("Dw", C.c_double), ("u0", C.c_double),
    ]


def _glib():
    L = lib()
    if not getattr(L, "_gen_ready", False):
        P, I, D = C.c_void_p, C.c_int, C.c_double
        dp, ip = C.POINTER(C.c_double), C.POINTER(C.c_int)
        L.og_last_error.restype = C.c_char_p
        L.og_create.argtypes = [C.POINTER(og_problem), C.POINTER(P)]
        L.og_destroy.argtypes = [P]
        L.og_sizes.argtypes = [P, ip]
        L.og_micro_pattern.argtypes = [P, ip, ip]
        L.og_micro_values.argtypes = [P, I, dp]
        L.og_rhs_parts.argtypes = [P, I, dp, dp]
        L.og_node_cache.argtypes = [P, I, dp, dp]
        L.og_macro_matrix.argtypes = [P, I, dp]
        L.og_surface_coupling.argtypes = [P, dp, I, I]
        L.og_surface_coupling.restype = D
        L.og_fixed_point_solve.argtypes = [P, D, I, D, I, I, dp, dp, dp, dp, I, ip, dp]
        L.og_micro_sweep.argtypes = [P, dp, dp, D, I, I, dp, ip]
        L._gen_ready = True
    return L


def gen_problem_for(cfg, table=None, map_kind=None):
    """og_problem for a configs.TwoScaleConfig with dim/order (c4, c5, or generic 2D)."""
    p = og_problem()
    for k in range(2):
        p.macro_lo[k], p.macro_hi[k], p.macro_n[k] = 0.0, 1.0, cfg.macro_n
        p.macro_dirichlet[k] = 1
        p.macro_dirichlet[k + 2] = 1
    p.dim, p.order = cfg.dim, cfg.order
    for k in range(cfg.dim):
        p.micro_lo[k], p.micro_hi[k], p.micro_n[k] = 0.0, 1.0, cfg.micro_n
    for k in range(4):
        p.kappa[k] = cfg.kappa[k]
    for k in range(6):
        p.micro_role[k] = 0
    p.Dv = 1.0
    d = cfg.dim
    Dm = np.eye(d).reshape(-1) if len(cfg.D) != d * d else np.asarray(cfg.D, float)
    for k in range(d * d):
        p.D[k] = Dm[k]
    if cfg.reaction is None:
        p.k_kind, p.k_par[0] = 0, 0.0
    elif cfg.reaction[0] == "disc":
        r = cfg.reaction
        p.k_kind = 1
        p.k_par[0], p.k_par[1], p.k_par[2], p.k_par[3] = r[1], r[2], r[3], r[4]
        p.k_par[4] = r[6] if len(r) > 6 else 0.0
        p.k_par[5] = r[5]
    else:
        p.k_kind, p.k_par[0] = 0, cfg.reaction[1]
    tab = cfg.table() if table is None else table
    keep = np.ascontiguousarray(tab, np.float64).reshape(-1)
    p.table = keep.ctypes.data_as(C.POINTER(C.c_double))
    if map_kind is None:
        map_kind = OG_MAP_FOURIER if cfg.map == "fourier" else OG_MAP_AFFINE_BUBBLE
    p.map_kind = map_kind
    p.s_kind = OR_S_PRODUCT
    p.amp = cfg.amp
    p.fu, p.fw, p.Dw, p.u0 = 1.0, 0.0, 1.0, 0.0
    return p, keep


class GenOracleContext:
    def __init__(self, cfg, table=None, map_kind=None):
        self.p, self._keep = gen_problem_for(cfg, table, map_kind)
        L = _glib()
        h = C.c_void_p()
        rc = L.og_create(C.byref(self.p), C.byref(h))
        if rc:
            raise OracleError(rc, L.og_last_error().decode())
        self.h = h
        s = np.zeros(9, np.int32)
        L.og_sizes(self.h, _ip(s))
        (self.n_macro, self.n_micro, self.micro_nnz, self.macro_nnz, self.n_faces, self.n_cells, self.nq,
         self.nqf, self.npf) = [int(v) for v in s]
        self.dim = cfg.dim

    def close(self):
        if self.h:
            _glib().og_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def micro_pattern(self):
        rp = np.zeros(self.n_micro + 1, np.int32)
        ci = np.zeros(self.micro_nnz, np.int32)
        _glib().og_micro_pattern(self.h, _ip(rp), _ip(ci))
        return rp, ci

    def micro_values(self, node):
        v = np.zeros(self.micro_nnz)
        rc = _glib().og_micro_values(self.h, node, _dp(v))
        if rc:
            raise OracleError(rc, _glib().og_last_error().decode())
        return v

    def rhs_parts(self, node):
        ri = np.zeros(self.n_micro)
        ro = np.zeros(self.n_micro)
        _glib().og_rhs_parts(self.h, node, _dp(ri), _dp(ro))
        return ri, ro

    def node_cache(self, node):
        nc = 1 + self.dim * (self.dim + 1) // 2
        cells = np.zeros((self.n_cells, self.nq, nc))
        faces = np.zeros((self.n_faces, self.nqf))
        _glib().og_node_cache(self.h, node, _dp(cells), _dp(faces))
        return cells, faces

    def macro_matrix(self, which):
        v = np.zeros(self.macro_nnz)
        _glib().og_macro_matrix(self.h, which, _dp(v))
        return v

    def surface_coupling(self, v, node, role):
        v = np.ascontiguousarray(v, np.float64)
        return float(_glib().og_surface_coupling(self.h, _dp(v), node, role))

    def solve(self, inner_tol=1e-10, inner_maxit=20000, outer_tol=1e-10, max_outer=100, threads=1):
        u = np.zeros(self.n_macro)
        w = np.zeros(self.n_macro)
        V = np.zeros((self.n_macro, self.n_micro))
        hist = np.zeros(max_outer + 1)
        info = np.zeros(4, np.int32)
        dof_it = np.zeros(1)
        rc = _glib().og_fixed_point_solve(self.h, inner_tol, inner_maxit, outer_tol, max_outer, threads, _dp(u),
                                          _dp(w), _dp(V), _dp(hist), len(hist), _ip(info), _dp(dof_it))
        if rc:
            raise OracleError(rc, _glib().og_last_error().decode())
        return dict(u=u, w=w, V=V, history=hist[: info[3]].copy(), sweeps=int(info[0]), converged=bool(info[1]),
                    micro_dof_iters=float(dof_it[0]))

    def micro_sweep(self, u, w, V=None, tol=1e-10, maxit=20000, threads=1):
        """One batched micro solve from V (zeros by default): (V, per-problem iterations)."""
        u = np.ascontiguousarray(u, np.float64)
        w = np.ascontiguousarray(w, np.float64)
        Vout = np.zeros((self.n_macro, self.n_micro)) if V is None else np.array(V, np.float64, copy=True)
        iters = np.zeros(self.n_macro, np.int32)
        rc = _glib().og_micro_sweep(self.h, _dp(u), _dp(w), tol, maxit, threads, _dp(Vout), _ip(iters))
        if rc:
            raise OracleError(rc, _glib().og_last_error().decode())
        return Vout, iters
