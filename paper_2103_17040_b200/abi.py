"""ctypes binding of the C ABI in include/twoscale_b200.h.

This is the Python face of the drop-in boundary: every call goes straight into
lib/libtwoscale_b200.so (sm_100a kernels).  There is no CPU fallback — if the
library is missing the import fails, and without a B200 every solve returns
TS_ERR_CUDA.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TS_B200_LIB") or os.path.join(_HERE, "lib", "libtwoscale_b200.so")

TS_OK, TS_ERR_CONFIG, TS_ERR_EXPR, TS_ERR_DEGENERATE_MAP, TS_ERR_SOLVER, TS_ERR_INVALID, TS_ERR_CUDA, TS_ERR_IO = range(8)
TS_VTK_ASCII, TS_VTK_BINARY = 0, 1
TS_GAMMA_I, TS_GAMMA_O, TS_GAMMA_N = 0, 1, 2
TS_MAP_TAPE, TS_MAP_AFFINE_BUBBLE_TABLE, TS_MAP_FOURIER_TABLE = 0, 1, 2
TS_S_NONE, TS_S_SINCOS, TS_S_PRODUCT = 0, 1, 2
TS_REACTION_CONST, TS_REACTION_DISC = 0, 1


class ts_ext_desc(C.Structure):
    _fields_ = [
        ("D", C.c_double * 4),
        ("reaction_kind", C.c_int32),
        ("reaction", C.c_double * 5),
        ("map_kind", C.c_int32),
        ("A_table", C.POINTER(C.c_double)),
        ("s_kind", C.c_int32),
        ("amp", C.c_double),
        ("micro_dim", C.c_int32),
        ("micro_order", C.c_int32),
        ("micro_n2", C.c_int32),
        ("micro_lo2", C.c_double),
        ("micro_hi2", C.c_double),
        ("D3", C.c_double * 9),
        ("micro_role3", C.c_int32 * 2),
        ("reaction_cz", C.c_double),
        ("force_generic", C.c_int32),
    ]


class ts_ctx_info(C.Structure):
    _fields_ = [
        ("n_macro", C.c_int32), ("n_micro", C.c_int32), ("micro_nnz", C.c_int32), ("macro_nnz", C.c_int32),
        ("n_micro_faces", C.c_int32), ("n_micro_cells", C.c_int32), ("n_macro_cells", C.c_int32),
        ("shared_operator", C.c_int32), ("w_pinned", C.c_int32), ("n_dirichlet_u", C.c_int32),
        ("setup_ms", C.c_double), ("device_bytes", C.c_int64),
        ("micro_kernel", C.c_int32), ("micro_rows", C.c_int32), ("micro_smem_bytes", C.c_double),
        ("macro_solver", C.c_int32), ("macro_cluster", C.c_int32),
    ]


class ts_solve_opts(C.Structure):
    _fields_ = [("inner_tol", C.c_double), ("inner_maxit", C.c_int32), ("outer_tol", C.c_double),
                ("max_outer", C.c_int32)]


class ts_solve_report(C.Structure):
    _fields_ = [
        ("converged", C.c_int32), ("sweeps", C.c_int32), ("w_pinned", C.c_int32),
        ("final_residual", C.c_double), ("micro_dof_iters", C.c_double), ("micro_ms", C.c_double),
        ("macro_ms", C.c_double), ("total_ms", C.c_double), ("micro_iters_max", C.c_int32),
        ("micro_iters_min", C.c_int32), ("gpu_launches", C.c_int32),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class ts_cg_result(C.Structure):
    _fields_ = [("converged", C.c_int32), ("iterations", C.c_int32), ("indefinite", C.c_int32),
                ("residual", C.c_double)]


# Every symbol include/twoscale_b200.h declares (checked by tests/test_abi_symbols.py).
EXPORTS = [
    "ts_last_error", "ts_last_error_index", "ts_abi_version", "ts_device_ok", "ts_select_device",
    "ts_trim_device_cache",
    "ts_host_alloc", "ts_host_free", "ts_ctx_create",
    "ts_ctx_create_ini", "ts_ctx_destroy", "ts_ctx_get_info", "ts_ctx_default_opts", "ts_fixed_point_solve",
    "ts_download_state", "ts_micro_solve", "ts_micro_pattern", "ts_micro_values", "ts_micro_rhs",
    "ts_node_cache", "ts_macro_matrix", "ts_macro_rhs", "ts_dirichlet", "ts_surface_coupling", "ts_cg_solve",
    "ts_build_cache", "ts_validate_diffeo", "ts_assumption6", "ts_error_norms", "ts_jit_status", "ts_ctx_error_norms", "ts_mms_sweep_ini", "ts_ctx_create_mms_ini",
    "ts_error_norms_ini", "ts_validate_map", "ts_write_vtk_macro", "ts_write_vtk_micro", "ts_write_vtk_ini",
]

_lib = None


def lib():
    """Load the B200 library (fails loudly when it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (make -C "
                              f"paper_2103_17040_b200/csrc); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        P, I, D = C.c_void_p, C.c_int32, C.c_double
        dp, ip = C.POINTER(C.c_double), C.POINTER(C.c_int32)
        L.ts_last_error.restype = C.c_char_p
        L.ts_last_error_index.restype = I
        L.ts_abi_version.restype = I
        L.ts_device_ok.restype = I
        L.ts_select_device.argtypes = [I]
        L.ts_select_device.restype = I
        L.ts_host_alloc.argtypes = [C.c_int64]
        L.ts_host_alloc.restype = C.c_void_p
        L.ts_host_free.argtypes = [C.c_void_p]
        L.ts_ctx_create_ini.argtypes = [C.c_char_p, C.POINTER(ts_ext_desc), C.POINTER(P)]
        L.ts_ctx_destroy.argtypes = [P]
        L.ts_ctx_get_info.argtypes = [P, C.POINTER(ts_ctx_info)]
        L.ts_ctx_default_opts.argtypes = [P, C.POINTER(ts_solve_opts)]
        L.ts_fixed_point_solve.argtypes = [P, C.POINTER(ts_solve_opts), C.POINTER(ts_solve_report), dp, I]
        L.ts_download_state.argtypes = [P, dp, dp, dp]
        L.ts_micro_solve.argtypes = [P, dp, dp, dp, D, I, dp, ip, C.POINTER(ts_solve_report)]
        L.ts_micro_pattern.argtypes = [P, ip, ip]
        L.ts_micro_values.argtypes = [P, I, dp]
        L.ts_micro_rhs.argtypes = [P, I, D, D, dp]
        L.ts_node_cache.argtypes = [P, I, dp, dp]
        L.ts_macro_matrix.argtypes = [P, I, ip, ip, dp]
        L.ts_macro_rhs.argtypes = [P, I, dp, dp]
        L.ts_dirichlet.argtypes = [P, I, ip, ip, dp]
        L.ts_surface_coupling.argtypes = [P, dp, I, I, dp]
        L.ts_cg_solve.argtypes = [I, ip, ip, dp, dp, dp, D, I, C.POINTER(ts_cg_result)]
        L.ts_mms_sweep_ini.argtypes = [C.c_char_p, ip, I, dp]
        L.ts_ctx_create_mms_ini.argtypes = [C.c_char_p, C.POINTER(P)]
        L.ts_error_norms_ini.argtypes = [C.c_char_p, dp, dp, dp, dp]
        L.ts_jit_status.restype = C.c_char_p
        L.ts_validate_map.argtypes = [P, D, D, dp, ip]
        L.ts_validate_map.restype = I
        L.ts_write_vtk_macro.argtypes = [P, I, C.c_char_p]
        L.ts_write_vtk_micro.argtypes = [P, D, I, C.c_char_p]
        L.ts_write_vtk_ini.argtypes = [C.c_char_p, dp, dp, dp, D, C.c_char_p, C.c_char_p]
        for name in ("ts_write_vtk_macro", "ts_write_vtk_micro", "ts_write_vtk_ini"):
            getattr(L, name).restype = I
        for name in ("ts_error_norms_ini", "ts_mms_sweep_ini", "ts_ctx_create_mms_ini", "ts_ctx_create_ini", "ts_ctx_get_info", "ts_ctx_default_opts", "ts_fixed_point_solve",
                     "ts_download_state", "ts_micro_solve", "ts_micro_pattern", "ts_micro_values", "ts_micro_rhs",
                     "ts_node_cache", "ts_macro_matrix", "ts_macro_rhs", "ts_dirichlet", "ts_surface_coupling",
                     "ts_cg_solve"):
            getattr(L, name).restype = I
        _lib = L
    return _lib


class TwoScaleError(RuntimeError):
    """Raised for a non-zero ts_status; `.status` and `.index` mirror the ABI."""

    def __init__(self, status, message, index=-1):
        super().__init__(message)
        self.status = status
        self.index = index


class ConfigError(TwoScaleError):
    pass


class DegenerateMapError(TwoScaleError):
    pass


class SolverError(TwoScaleError):
    pass


_ERR = {TS_ERR_CONFIG: ConfigError, TS_ERR_DEGENERATE_MAP: DegenerateMapError, TS_ERR_SOLVER: SolverError}


def check(status):
    if status != TS_OK:
        L = lib()
        msg = L.ts_last_error().decode()
        raise _ERR.get(status, TwoScaleError)(status, msg, int(L.ts_last_error_index()))


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def _in(a, size, name):
    """Input array as contiguous float64 with exactly `size` elements (ValueError otherwise)."""
    a = np.ascontiguousarray(a, np.float64)
    if a.size != size:
        raise ValueError(f"{name}: expected {size} float64 values, got {a.size}")
    return a


def _out(a, shape, name):
    """Caller-supplied output array: must be C-contiguous float64 of exactly `shape`, since the
    C side writes prod(shape) doubles through its pointer."""
    shape = tuple(shape)
    if a is None:
        return np.zeros(shape)
    if not isinstance(a, np.ndarray) or a.dtype != np.float64 or not a.flags.c_contiguous or a.shape != shape:
        raise ValueError(f"{name}: expected a C-contiguous float64 array of shape {shape}, got "
                         f"{getattr(a, 'dtype', type(a))} {getattr(a, 'shape', '')}")
    if not a.flags.writeable:
        raise ValueError(f"{name}: array is read-only")
    return a


def device_ok() -> bool:
    return bool(lib().ts_device_ok())


def select_device(device: int) -> None:
    check(lib().ts_select_device(device))


class PinnedArray:
    """numpy view over page-locked host memory from ts_host_alloc (freed with the object)."""

    def __init__(self, shape, dtype=np.float64):
        self.nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
        self.ptr = lib().ts_host_alloc(self.nbytes)
        if not self.ptr:
            raise MemoryError(lib().ts_last_error().decode())
        buf = (C.c_char * self.nbytes).from_address(self.ptr)
        self.array = np.frombuffer(buf, dtype=dtype).reshape(shape)

    def __del__(self):
        try:
            if self.ptr:
                self.array = None
                lib().ts_host_free(self.ptr)
                self.ptr = None
        except Exception:
            pass


def make_ext(D=(1.0, 0.0, 0.0, 1.0), reaction=None, table=None, s_kind=TS_S_PRODUCT, amp=0.0, map_kind=None,
             dim=2, order=1, micro_n=None, force_generic=False, roles3=(TS_GAMMA_I, TS_GAMMA_I)):
    """Extension block: D tensor (4 entries in 2D, 9 in 3D), reaction ("const", k) /
    ("disc", k_in, k_out, cx, cy, r[, cz]), per-node map table, generic micro geometry."""
    e = ts_ext_desc()
    e.micro_dim = dim
    e.micro_order = order
    e.force_generic = 1 if force_generic else 0
    e.micro_role3[0], e.micro_role3[1] = roles3
    if dim == 3:
        e.micro_n2 = int(micro_n)
        e.micro_lo2, e.micro_hi2 = 0.0, 1.0
        D9 = D if len(D) == 9 else (1.0, 0, 0, 0, 1.0, 0, 0, 0, 1.0)
        for k in range(9):
            e.D3[k] = float(D9[k])
        D = (1.0, 0.0, 0.0, 1.0)
    for k in range(4):
        e.D[k] = float(D[k])
    if reaction is not None:
        kind = reaction[0]
        e.reaction_kind = TS_REACTION_DISC if kind == "disc" else TS_REACTION_CONST
        for k, v in enumerate(reaction[1:6]):
            e.reaction[k] = float(v)
        if len(reaction) > 6:
            e.reaction_cz = float(reaction[6])
    keep = None
    if table is not None:
        keep = np.ascontiguousarray(table, np.float64).reshape(-1)
        e.map_kind = TS_MAP_AFFINE_BUBBLE_TABLE if map_kind is None else map_kind
        e.A_table = _dp(keep)
        e.s_kind = s_kind
        e.amp = amp
    return e, keep


def mms_sweep(ini: str, ns):
    """Device convergence_sweep (derive_data + solves + error norms): rows [len(ns)][13]."""
    ns = np.ascontiguousarray(ns, np.int32)
    rows = np.zeros((len(ns), 13))
    check(lib().ts_mms_sweep_ini(ini.encode(), _ip(ns), len(ns), _dp(rows)))
    return rows


def error_norms(ini: str, u, w, V):
    """Device error_norms of a host state against the INI's [mms] solution: (e_uw, e_uw_grad, e_v, e_v_grad)."""
    u, w, V = (np.ascontiguousarray(a, np.float64) for a in (u, w, V))
    if len(u) != len(w) or V.ndim != 2 or V.shape[0] != len(u):
        raise ValueError(f"error_norms: u {u.shape}, w {w.shape}, V {V.shape} do not describe one state")
    out = np.zeros(4)
    check(lib().ts_error_norms_ini(ini.encode(), _dp(u), _dp(w), _dp(V), _dp(out)))
    return out


def jit_status() -> str:
    """Tape path of the last error_norms call: "compiled (...)" or "interpreter (why) (...)"."""
    return lib().ts_jit_status().decode()


def write_vtk_ini(ini: str, u, w, V, scale, macro_path=None, micro_path=None):
    """Host write_vtk_macro / write_vtk_micro of the C++ mirror for a host state (ASCII)."""
    u, w, V = (np.ascontiguousarray(a, np.float64) for a in (u, w, V))
    if len(u) != len(w) or V.ndim != 2 or V.shape[0] != len(u):
        raise ValueError(f"write_vtk_ini: u {u.shape}, w {w.shape}, V {V.shape} do not describe one state")
    enc = lambda p: None if p is None else str(p).encode()  # noqa: E731
    check(lib().ts_write_vtk_ini(ini.encode(), _dp(u), _dp(w), _dp(V), float(scale), enc(macro_path),
                                 enc(micro_path)))


class Context:
    """Device-resident AssemblyContext (ts_ctx) built from INI text + extensions
    (mms=True: the manufactured problem of the INI's [mms] section, via derive_data)."""

    def __init__(self, ini: str, ext=None, mms=False):
        self._keep = None
        self.h = C.c_void_p()
        ep = None
        if ext is not None:
            ext_struct, self._keep = ext if isinstance(ext, tuple) else (ext, None)
            self._ext = ext_struct
            ep = C.byref(ext_struct)
        if mms:
            check(lib().ts_ctx_create_mms_ini(ini.encode(), C.byref(self.h)))
        else:
            check(lib().ts_ctx_create_ini(ini.encode(), ep, C.byref(self.h)))
        info = ts_ctx_info()
        check(lib().ts_ctx_get_info(self.h, C.byref(info)))
        self.info = {k: getattr(info, k) for k, _ in info._fields_}
        self.n_macro = info.n_macro
        self.n_micro = info.n_micro

    def close(self):
        if self.h:
            lib().ts_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def default_opts(self):
        o = ts_solve_opts()
        check(lib().ts_ctx_default_opts(self.h, C.byref(o)))
        return dict(inner_tol=o.inner_tol, inner_maxit=o.inner_maxit, outer_tol=o.outer_tol, max_outer=o.max_outer)

    def solve(self, inner_tol=None, inner_maxit=None, outer_tol=None, max_outer=None, download=True):
        d = self.default_opts()
        o = ts_solve_opts(d["inner_tol"] if inner_tol is None else inner_tol,
                          d["inner_maxit"] if inner_maxit is None else inner_maxit,
                          d["outer_tol"] if outer_tol is None else outer_tol,
                          d["max_outer"] if max_outer is None else max_outer)
        rep = ts_solve_report()
        hist = np.zeros(max(o.max_outer, 1))
        check(lib().ts_fixed_point_solve(self.h, C.byref(o), C.byref(rep), _dp(hist), len(hist)))
        out = rep.as_dict()
        out["history"] = hist[: rep.sweeps].copy()
        if download:
            out.update(self.state())
        return out

    def state(self, u=None, w=None, V=None):
        """TwoScaleState download; pass (pinned) output arrays to avoid allocation."""
        u = _out(u, (self.n_macro,), "u")
        w = _out(w, (self.n_macro,), "w")
        V = _out(V, (self.n_macro, self.n_micro), "V")
        check(lib().ts_download_state(self.h, _dp(u), _dp(w), _dp(V)))
        return dict(u=u, w=w, V=V)

    def micro_solve(self, u, w, V0=None, tol=1e-10, maxit=20000, raise_on_fail=True):
        """One batched micro PCG over all problems (ts_micro_solve).  raise_on_fail=False
        returns (V, iters, report, status) instead of raising SolverError for a failed
        system, so the per-problem results stay inspectable."""
        u = _in(u, self.n_macro, "u")
        w = _in(w, self.n_macro, "w")
        Vp = None
        if V0 is not None:
            V0 = _in(V0, self.n_macro * self.n_micro, "V0")
            Vp = _dp(V0)
        V = np.zeros((self.n_macro, self.n_micro))
        it = np.zeros(self.n_macro, np.int32)
        rep = ts_solve_report()
        st = lib().ts_micro_solve(self.h, _dp(u), _dp(w), Vp, tol, maxit, _dp(V), _ip(it), C.byref(rep))
        if not raise_on_fail:
            return V, it, rep.as_dict(), st
        check(st)
        return V, it, rep.as_dict()

    def micro_pattern(self):
        rp = np.zeros(self.n_micro + 1, np.int32)
        ci = np.zeros(self.info["micro_nnz"], np.int32)
        check(lib().ts_micro_pattern(self.h, _ip(rp), _ip(ci)))
        return rp, ci

    def micro_values(self, node):
        v = np.zeros(self.info["micro_nnz"])
        check(lib().ts_micro_values(self.h, node, _dp(v)))
        return v

    def micro_rhs(self, node, u, w):
        b = np.zeros(self.n_micro)
        check(lib().ts_micro_rhs(self.h, node, u, w, _dp(b)))
        return b

    def node_cache(self, node):
        cells = np.zeros((self.info["n_micro_cells"], 4, 4))
        faces = np.zeros((self.info["n_micro_faces"], 2, 4))
        check(lib().ts_node_cache(self.h, node, _dp(cells), _dp(faces)))
        return cells, faces

    def macro_matrix(self, which):
        rp = np.zeros(self.n_macro + 1, np.int32)
        ci = np.zeros(self.info["macro_nnz"], np.int32)
        v = np.zeros(self.info["macro_nnz"])
        check(lib().ts_macro_matrix(self.h, which, _ip(rp), _ip(ci), _dp(v)))
        return rp, ci, v

    def macro_rhs(self, which, V=None):
        out = np.zeros(self.n_macro)
        Vp = None
        if V is not None:
            V = _in(V, self.n_macro * self.n_micro, "V")
            Vp = _dp(V)
        check(lib().ts_macro_rhs(self.h, which, Vp, _dp(out)))
        return out

    def dirichlet(self, which):
        n = C.c_int32()
        check(lib().ts_dirichlet(self.h, which, C.byref(n), None, None))
        dofs = np.zeros(n.value, np.int32)
        vals = np.zeros(n.value)
        check(lib().ts_dirichlet(self.h, which, C.byref(n), _ip(dofs), _dp(vals)))
        return dofs, vals

    def surface_coupling(self, v, node, role):
        v = _in(v, self.n_micro, "v")
        out = np.zeros(1)
        check(lib().ts_surface_coupling(self.h, _dp(v), node, role, _dp(out)))
        return float(out[0])

    def write_vtk_macro(self, path, binary=False):
        """write_vtk_macro of the device state u, w (vtk.cpp:36-54)."""
        check(lib().ts_write_vtk_macro(self.h, TS_VTK_BINARY if binary else TS_VTK_ASCII, str(path).encode()))

    def write_vtk_micro(self, path, scale=1.0, binary=False):
        """write_vtk_micro of the device state V, streamed in chunks (vtk.cpp:56-85)."""
        check(lib().ts_write_vtk_micro(self.h, float(scale), TS_VTK_BINARY if binary else TS_VTK_ASCII,
                                       str(path).encode()))

    def validate_map(self, lo=1e-6, hi=1e6):
        """det grad_y zeta over every node x micro quadrature point: (pass, min, max, where)."""
        out = np.zeros(6)
        ok = C.c_int32()
        check(lib().ts_validate_map(self.h, lo, hi, _dp(out), C.byref(ok)))
        return bool(ok.value), float(out[0]), float(out[1]), tuple(int(v) for v in out[2:])


def cg_solve(row_ptr, col_idx, vals, b, x0, tol, maxit):
    """Device cg_solve on a general CSR matrix: (x, converged, iterations, residual, indefinite)."""
    row_ptr = np.ascontiguousarray(row_ptr, np.int32)
    n = len(row_ptr) - 1
    if n < 0 or len(b) != n or len(x0) != n:
        raise ValueError(f"cg_solve: row_ptr has {len(row_ptr)} entries, b {len(b)}, x0 {len(x0)}")
    nnz = int(row_ptr[-1]) if n >= 0 else 0
    col_idx = np.ascontiguousarray(col_idx, np.int32)
    vals = np.ascontiguousarray(vals, np.float64)
    if len(col_idx) < nnz or len(vals) < nnz:
        raise ValueError(f"cg_solve: row_ptr[-1] = {nnz} but col_idx has {len(col_idx)}, vals {len(vals)}")
    b = np.ascontiguousarray(b, np.float64)
    x = np.array(x0, np.float64, copy=True)
    r = ts_cg_result()
    check(lib().ts_cg_solve(len(b), _ip(row_ptr), _ip(col_idx), _dp(vals), _dp(b), _dp(x), tol, maxit, C.byref(r)))
    return x, bool(r.converged), int(r.iterations), float(r.residual), bool(r.indefinite)
