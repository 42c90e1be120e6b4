"""TEST INFRASTRUCTURE ONLY: ctypes loader for oracle/_ref/libtwoscale_ref.so.

That library is the UNMODIFIED reference (/root/reference/proj/src/*.cpp) plus the
extern "C" shim oracle/ref_harness.cpp, built by oracle/Makefile.  Only tests/,
__graft_entry__.smoke() and bench.py's CPU legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libtwoscale_ref.so")
# the same harness source compiled against include/twoscale + libtwoscale_b200.so (oracle/Makefile)
MIRROR_PATH = os.path.join(_HERE, "_mirror", "libtwoscale_refapi.so")

_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def mirror():
    """This module bound to the drop-in build (ref_harness.cpp against the B200 library's
    reference-API headers) instead of the reference: same functions, same classes."""
    import importlib.util
    import sys
    name = __name__ + "_mirror"
    if name not in sys.modules:
        spec = importlib.util.spec_from_file_location(name, __file__)
        m = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(m)
        m.LIB_PATH = MIRROR_PATH
        sys.modules[name] = m
    return sys.modules[name]


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} not built (make -C oracle ref)")
        L = C.CDLL(LIB_PATH)
        P, I, D = C.c_void_p, C.c_int, C.c_double
        dp = C.POINTER(C.c_double)
        ip = C.POINTER(C.c_int)
        L.ref_last_error.restype = C.c_char_p
        L.ref_create.argtypes = [C.c_char_p, I, C.POINTER(P)]
        L.ref_destroy.argtypes = [P]
        L.ref_build_seconds.argtypes = [P]
        L.ref_build_seconds.restype = D
        L.ref_sizes.argtypes = [P, ip]
        L.ref_micro_pattern.argtypes = [P, ip, ip]
        L.ref_micro_values.argtypes = [P, I, dp]
        L.ref_micro_rhs.argtypes = [P, I, D, D, dp]
        L.ref_node_cache.argtypes = [P, I, dp, dp]
        L.ref_jac.argtypes = [P, I, dp, dp, dp]
        L.ref_macro_matrix.argtypes = [P, I, ip, ip, dp]
        L.ref_macro_rhs.argtypes = [P, I, dp, dp]
        L.ref_dirichlet.argtypes = [P, I, ip, ip, dp]
        L.ref_surface_coupling.argtypes = [P, dp, I, I, dp]
        L.ref_solve.argtypes = [P, D, I, D, I, I, dp, dp, dp, dp, I, ip, dp]
        L.ref_cg_solve.argtypes = [I, ip, ip, dp, dp, dp, D, I, ip, dp]
        L.ref_batched_cg.argtypes = [I, ip, ip, I, dp, dp, dp, D, I, I, ip, dp]
        L.ref_micro_sweep.argtypes = [P, dp, dp, D, I, I, I, ip, dp, ip, dp]
        L.ref_hardware_threads.restype = I
        L.ref_build_cache.argtypes = [P, I, dp, dp, dp, ip]
        L.ref_validate_diffeo.argtypes = [P, I, dp, I, dp, D, D, dp, C.c_char_p, I]
        L.ref_check_assumption6.argtypes = [P, I, dp, dp, dp]
        L.ref_mms_sweep.argtypes = [C.c_char_p, ip, I, dp, I]
        L.ref_create_mms.argtypes = [C.c_char_p, I, C.POINTER(P)]
        L.ref_error_norms.argtypes = [C.c_char_p, dp, dp, dp, dp, I]
        L.ref_mms_solve.argtypes = [C.c_char_p, dp, dp, dp, ip]
        L.ref_write_vtk.argtypes = [C.c_char_p, dp, dp, dp, D, C.c_char_p, C.c_char_p]
        _lib = L
    return _lib


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[ref code {code}] {msg}")
        self.code = code


def _chk(rc):
    if rc != 0:
        raise RefError(rc, lib().ref_last_error().decode())


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int))


def cg_solve(row_ptr, col_idx, vals, b, x0, tol, maxit):
    """Reference cg_solve (linalg.cpp:103-161). Returns (x, converged, iters, residual, indefinite)."""
    row_ptr = np.ascontiguousarray(row_ptr, np.int32)
    col_idx = np.ascontiguousarray(col_idx, np.int32)
    vals = np.ascontiguousarray(vals, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    x = np.array(x0, np.float64, copy=True)
    res = np.zeros(3, np.int32)
    resd = np.zeros(1)
    _chk(lib().ref_cg_solve(len(b), _ip(row_ptr), _ip(col_idx), _dp(vals), _dp(b), _dp(x), tol, maxit,
                           _ip(res), _dp(resd)))
    return x, bool(res[0]), int(res[1]), float(resd[0]), bool(res[2])


def batched_cg(row_ptr, col_idx, vals, b, x0, tol, maxit, workers):
    """Reference cg_solve over many systems on one pattern (threads via reference parallel_for)."""
    row_ptr = np.ascontiguousarray(row_ptr, np.int32)
    col_idx = np.ascontiguousarray(col_idx, np.int32)
    vals = np.ascontiguousarray(vals, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    x = np.array(x0, np.float64, copy=True)
    n = len(row_ptr) - 1
    n_sys = b.size // n
    iters = np.zeros(n_sys, np.int32)
    secs = np.zeros(1)
    _chk(lib().ref_batched_cg(n, _ip(row_ptr), _ip(col_idx), n_sys, _dp(vals), _dp(b), _dp(x), tol, maxit,
                             workers, _ip(iters), _dp(secs)))
    return x, iters, float(secs[0])


def mms_sweep(ini, ns, workers=1):
    """Reference derive_data + convergence_sweep: rows [len(ns)][13] (SolveOptions.workers)."""
    ns = np.ascontiguousarray(ns, np.int32)
    rows = np.zeros((len(ns), 13))
    _chk(lib().ref_mms_sweep(ini.encode(), _ip(ns), len(ns), _dp(rows), workers))
    return rows


def error_norms(ini, u, w, V, workers=1):
    u, w, V = (np.ascontiguousarray(a, np.float64) for a in (u, w, V))
    out = np.zeros(4)
    _chk(lib().ref_error_norms(ini.encode(), _dp(u), _dp(w), _dp(V), _dp(out), workers))
    return out


def mms_solve(ini, n_macro, n_micro):
    u = np.zeros(n_macro)
    w = np.zeros(n_macro)
    V = np.zeros((n_macro, n_micro))
    sw = np.zeros(1, np.int32)
    _chk(lib().ref_mms_solve(ini.encode(), _dp(u), _dp(w), _dp(V), _ip(sw)))
    return dict(u=u, w=w, V=V, sweeps=int(sw[0]))


def write_vtk(ini, u, w, V, scale, macro_path=None, micro_path=None):
    """Reference write_vtk_macro / write_vtk_micro (vtk.cpp:36-85) of a host state."""
    u, w, V = (np.ascontiguousarray(a, np.float64) for a in (u, w, V))
    enc = lambda p: None if p is None else str(p).encode()  # noqa: E731
    _chk(lib().ref_write_vtk(ini.encode(), _dp(u), _dp(w), _dp(V), float(scale), enc(macro_path), enc(micro_path)))


def hardware_threads() -> int:
    return int(lib().ref_hardware_threads())


class RefContext:
    """AssemblyContext of the reference, built from INI text (config.cpp grammar)."""

    def __init__(self, ini: str, workers: int = 1, mms: bool = False):
        h = C.c_void_p()
        create = lib().ref_create_mms if mms else lib().ref_create
        _chk(create(ini.encode(), workers, C.byref(h)))
        self.h = h
        s = np.zeros(8, np.int32)
        _chk(lib().ref_sizes(self.h, _ip(s)))
        (self.n_macro, self.n_micro, self.micro_nnz, self.macro_nnz, self.n_micro_faces,
         shared, self.n_macro_cells, self.n_micro_cells) = [int(v) for v in s]
        self.shared_matrix = bool(shared)

    def close(self):
        if self.h:
            lib().ref_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def build_seconds(self):
        return lib().ref_build_seconds(self.h)

    def micro_pattern(self):
        rp = np.zeros(self.n_micro + 1, np.int32)
        ci = np.zeros(self.micro_nnz, np.int32)
        _chk(lib().ref_micro_pattern(self.h, _ip(rp), _ip(ci)))
        return rp, ci

    def micro_values(self, node):
        v = np.zeros(self.micro_nnz)
        _chk(lib().ref_micro_values(self.h, node, _dp(v)))
        return v

    def micro_rhs(self, node, u, w):
        b = np.zeros(self.n_micro)
        _chk(lib().ref_micro_rhs(self.h, node, u, w, _dp(b)))
        return b

    def node_cache(self, node):
        cells = np.zeros((self.n_micro_cells, 4, 4))
        faces = np.zeros((self.n_micro_faces, 2, 4))
        _chk(lib().ref_node_cache(self.h, node, _dp(cells), _dp(faces)))
        return cells, faces

    def jac(self, xs, ys):
        xs = np.ascontiguousarray(xs, np.float64).reshape(-1, 2)
        ys = np.ascontiguousarray(ys, np.float64).reshape(-1, 2)
        out = np.zeros((len(xs), 4))
        _chk(lib().ref_jac(self.h, len(xs), _dp(xs), _dp(ys), _dp(out)))
        return out.reshape(-1, 2, 2)

    def build_cache(self, points, with_cells=True):
        """build_cache of the context's map at macro points: (cells, faces) per cache row."""
        pts = np.ascontiguousarray(points, np.float64).reshape(-1, 2)
        n = len(pts)
        cells = np.zeros((max(n, 1), self.n_micro_cells, 4, 4)) if with_cells else None
        faces = np.zeros((max(n, 1), self.n_micro_faces, 2, 4))
        rows = C.c_int()
        _chk(lib().ref_build_cache(self.h, n, _dp(pts), None if cells is None else _dp(cells), _dp(faces),
                                   C.byref(rows)))
        r = rows.value
        return (None if cells is None else cells[:r]), faces[:r]

    def validate_diffeo(self, xs, ys, lo=1e-6, hi=1e6):
        """(pass, min_det, max_det, worst_x, worst_yhat, message)."""
        xs = np.ascontiguousarray(xs, np.float64).reshape(-1, 2)
        ys = np.ascontiguousarray(ys, np.float64).reshape(-1, 2)
        out = np.zeros(7)
        msg = C.create_string_buffer(1024)
        _chk(lib().ref_validate_diffeo(self.h, len(xs), _dp(xs), len(ys), _dp(ys), lo, hi, _dp(out), msg, 1024))
        return bool(out[0]), out[1], out[2], tuple(out[3:5]), tuple(out[5:7]), msg.value.decode()

    def check_assumption6(self, points):
        """rows [n][gamma_in, gamma_out, ok1, ok2], summary (min_dw, lhs1_max, lhs2_max, ok1, ok2)."""
        pts = np.ascontiguousarray(points, np.float64).reshape(-1, 2)
        rows = np.zeros((len(pts), 4))
        summ = np.zeros(5)
        _chk(lib().ref_check_assumption6(self.h, len(pts), _dp(pts), _dp(rows), _dp(summ)))
        return rows, summ

    def macro_matrix(self, which):
        rp = np.zeros(self.n_macro + 1, np.int32)
        ci = np.zeros(self.macro_nnz, np.int32)
        v = np.zeros(self.macro_nnz)
        _chk(lib().ref_macro_matrix(self.h, which, _ip(rp), _ip(ci), _dp(v)))
        return rp, ci, v

    def macro_rhs(self, which, V=None):
        out = np.zeros(self.n_macro)
        Vp = None
        if V is not None:
            V = np.ascontiguousarray(V, np.float64)
            Vp = _dp(V)
        _chk(lib().ref_macro_rhs(self.h, which, Vp, _dp(out)))
        return out

    def dirichlet(self, which):
        n = C.c_int()
        _chk(lib().ref_dirichlet(self.h, which, C.byref(n), None, None))
        dofs = np.zeros(n.value, np.int32)
        vals = np.zeros(n.value)
        _chk(lib().ref_dirichlet(self.h, which, C.byref(n), _ip(dofs), _dp(vals)))
        return dofs, vals

    def surface_coupling(self, v, node, role):
        v = np.ascontiguousarray(v, np.float64)
        out = np.zeros(1)
        _chk(lib().ref_surface_coupling(self.h, _dp(v), node, role, _dp(out)))
        return float(out[0])

    def solve(self, inner_tol=1e-10, inner_maxit=20000, outer_tol=1e-8, max_outer=100, workers=1):
        u = np.zeros(self.n_macro)
        w = np.zeros(self.n_macro)
        V = np.zeros((self.n_macro, self.n_micro))
        hist = np.zeros(max_outer + 1)
        info = np.zeros(4, np.int32)
        info_d = np.zeros(2)
        _chk(lib().ref_solve(self.h, inner_tol, inner_maxit, outer_tol, max_outer, workers, _dp(u), _dp(w),
                             _dp(V), _dp(hist), len(hist), _ip(info), _dp(info_d)))
        return dict(u=u, w=w, V=V, history=hist[: info[3]].copy(), sweeps=int(info[0]),
                    converged=bool(info[1]), w_pinned=bool(info[2]), final_residual=float(info_d[0]),
                    seconds=float(info_d[1]))

    def micro_sweep(self, u, w, tol=1e-10, maxit=20000, workers=1, nodes=None, V=None):
        u = np.ascontiguousarray(u, np.float64)
        w = np.ascontiguousarray(w, np.float64)
        if nodes is None:
            nodes_arr = None
            n_nodes = self.n_macro
        else:
            nodes_arr = np.ascontiguousarray(nodes, np.int32)
            n_nodes = len(nodes_arr)
        Vout = np.zeros((n_nodes, self.n_micro)) if V is None else np.array(V, np.float64, copy=True)
        iters = np.zeros(n_nodes, np.int32)
        secs = np.zeros(1)
        _chk(lib().ref_micro_sweep(self.h, _dp(u), _dp(w), tol, maxit, workers, n_nodes,
                                   None if nodes_arr is None else _ip(nodes_arr), _dp(Vout), _ip(iters),
                                   _dp(secs)))
        return Vout, iters, float(secs[0])
