"""ctypes binding of the C oracle (TEST INFRASTRUCTURE ONLY; see oracle.h)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle_mgpbd.so")
SRC = os.path.join(HERE, "oracle.c")


def build(force: bool = False) -> str:
    """Compile the oracle: serial, fp64, -O2 -ffp-contract=off, no fast-math."""
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < max(
            os.path.getmtime(SRC), os.path.getmtime(os.path.join(HERE, "oracle.h"))):
        tmp = f"{LIB_PATH}.{os.getpid()}.tmp"  # replace atomically: a running process may map the old one
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11",
                               "-fPIC", "-shared", "-o", tmp, SRC, "-lm"])
        os.replace(tmp, LIB_PATH)
    return LIB_PATH


class Config(C.Structure):
    _fields_ = [("theta", C.c_double), ("min_coarse", C.c_int32), ("max_levels", C.c_int32),
                ("stall_ratio", C.c_double), ("setup_interval", C.c_int32),
                ("bootstrap_sweeps", C.c_int32), ("power_iters", C.c_int32),
                ("lambda_min_est", C.c_double), ("lambda_safety", C.c_double), ("smoother_sweeps", C.c_int32),
                ("pcg_iters", C.c_int32), ("omega_relax", C.c_double),
                ("gravity", C.c_double * 3), ("seed", C.c_uint64), ("smoother", C.c_int32),
                ("cheb_lower", C.c_double), ("backtrack", C.c_int32), ("omega_min", C.c_double),
                ("residual_tol", C.c_double), ("pcg_tol", C.c_double), ("resetup_on_indef", C.c_int32),
                ("residual_abs", C.c_double), ("omega_refresh_iters", C.c_int32),
                ("k_nullspace", C.c_int32), ("time_budget_ms", C.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        L = _lib
        P = C.c_void_p
        i32, i64, f64, u64 = C.c_int32, C.c_int64, C.c_double, C.c_uint64
        sig = {
            "orc_config_default": (None, [P]),
            "orc_mix64": (u64, [u64]),
            "orc_key": (u64, [u64, C.c_int, C.c_int, u64]),
            "orc_uniform": (f64, [u64, C.c_int, C.c_int, u64]),
            "orc_rest_distance": (None, [i32, P, P, P]),
            "orc_rest_arap": (C.c_int, [i32, P, P, P, P]),
            "orc_eval_distance": (None, [i32, P, P, P, P, P]),
            "orc_polar": (None, [P, P]),
            "orc_eval_arap": (None, [i32, P, P, P, P, P]),
            "orc_pattern": (i64, [i32, C.c_int, P, i32, P, P]),
            "orc_assemble": (None, [i32, C.c_int, P, P, P, P, P, P, P]),
            "orc_assemble_rows": (None, [i32, P, C.c_int, P, P, P, P, P, P, P]),
            "orc_rhs": (None, [i32, P, P, P, P]),
            "orc_apply_dx": (None, [i32, C.c_int, P, i32, P, P, P, P]),
            "orc_spmv": (None, [i32, P, P, P, P, P]),
            "orc_soc": (None, [i32, P, P, P, f64, P]),
            "orc_aggregate": (i32, [i32, P, P, P, P, u64, C.c_int, P]),
            "orc_colour": (i32, [i32, P, P, u64, P]),
            "orc_gs_bootstrap": (None, [i32, P, P, P, P, i32, u64, P]),
            "orc_prolongator": (None, [i32, P, i32, P, P, P]),
            "orc_galerkin": (i64, [i32, P, P, P, P, P, i32, P, P, P]),
            "orc_power": (f64, [i32, P, P, P, i32, u64, C.c_int]),
            "orc_power_from": (f64, [i32, P, P, P, i32, P]),
            "orc_hier_refresh_omega": (None, [P, i32]),
            "orc_gs_bootstrap_k": (None, [i32, P, P, P, P, i32, u64, i32, P]),
            "orc_prolongator_qr": (i32, [i32, P, i32, i32, P, f64, P, P, P, P, P, i32]),
            "orc_galerkin_p": (i64, [i32, P, P, P, P, P, P, i32, P, P, P]),
            "orc_hier_get_P_csr": (None, [P, C.c_int, P, P, P, P]),
            "orc_cholesky": (C.c_int, [i32, P, P]),
            "orc_chol_solve": (None, [i32, P, P, P]),
            "orc_hier_build": (P, [i32, P, P, P, P]),
            "orc_hier_refresh": (C.c_int, [P, P]),
            "orc_hier_free": (None, [P]),
            "orc_hier_levels": (C.c_int, [P]),
            "orc_hier_level_size": (None, [P, C.c_int, P, P]),
            "orc_hier_get_level": (None, [P, C.c_int, P, P, P]),
            "orc_hier_get_agg": (None, [P, C.c_int, P]),
            "orc_hier_get_P": (None, [P, C.c_int, P]),
            "orc_hier_omega": (f64, [P, C.c_int]),
            "orc_hier_cheb": (None, [P, C.c_int, P, P]),
            "orc_hier_smooth": (None, [P, C.c_int, P, P, C.c_int]),
            "orc_hier_get_B0": (None, [P, P]),
            "orc_hier_n_colours": (i32, [P]),
            "orc_vcycle": (None, [P, P, P]),
            "orc_pcg": (C.c_int, [P, P, i32, P, P]),
            "orc_sim_create": (P, [C.c_int, i32, i32, P, P, P, P, P, P, P]),
            "orc_sim_step": (C.c_int, [P, f64, i32]),
            "orc_sim_mark_stale": (None, [P]),
            "orc_sim_setups": (C.c_int32, [P]),
            "orc_sim_setup_ms": (C.c_double, [P]),
            "orc_sim_indefinite_events": (i32, [P]),
            "orc_sim_iters_used": (i32, [P]),
            "orc_sim_omega": (f64, [P]),
            "orc_sim_get": (None, [P, P, P, P]),
            "orc_sim_set": (None, [P, P, P]),
            "orc_sim_hier": (P, [P]),
            "orc_sim_nnz": (i64, [P]),
            "orc_sim_get_A": (None, [P, P, P, P]),
            "orc_sim_get_b_norms": (None, [P, P, i32]),
            "orc_sim_free": (None, [P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
    return _lib


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def default_config(**kw) -> Config:
    c = Config()
    lib().orc_config_default(C.byref(c))
    for k, v in kw.items():
        if k == "gravity":
            c.gravity[:] = list(v)
        else:
            setattr(c, k, v)
    return c


# ------------------------------------------------------------------------------ hash
def mix64(z: int) -> int:
    return int(lib().orc_mix64(C.c_uint64(z & 0xFFFFFFFFFFFFFFFF)))


def key(seed: int, stream: int, level: int, i: int) -> int:
    return int(lib().orc_key(seed, stream, level, i))


def uniform(seed: int, stream: int, level: int, i: int) -> float:
    return float(lib().orc_uniform(seed, stream, level, i))


# ------------------------------------------------------------------------------ constraints
def rest_distance(verts, X):
    verts, X = _c(verts, np.int32), _c(X, np.float64)
    out = np.empty(verts.shape[0])
    lib().orc_rest_distance(verts.shape[0], _p(verts), _p(X), _p(out))
    return out


def rest_arap(verts, X):
    verts, X = _c(verts, np.int32), _c(X, np.float64)
    m = verts.shape[0]
    Dm = np.empty((m, 3, 3)); vol = np.empty(m)
    lib().orc_rest_arap(m, _p(verts), _p(X), _p(Dm), _p(vol))
    return Dm, vol


def eval_distance(verts, x, rest_len):
    verts, x, rest_len = _c(verts, np.int32), _c(x, np.float64), _c(rest_len, np.float64)
    m = verts.shape[0]
    Cv = np.empty(m); g = np.empty((m, 2, 3))
    lib().orc_eval_distance(m, _p(verts), _p(x), _p(rest_len), _p(Cv), _p(g))
    return Cv, g


def polar(F):
    F = _c(F, np.float64).reshape(3, 3)
    R = np.empty((3, 3))
    lib().orc_polar(_p(F), _p(R))
    return R


def eval_arap(verts, x, Dm_inv):
    verts, x, Dm_inv = _c(verts, np.int32), _c(x, np.float64), _c(Dm_inv, np.float64)
    m = verts.shape[0]
    Cv = np.empty(m); g = np.empty((m, 4, 3))
    lib().orc_eval_arap(m, _p(verts), _p(x), _p(Dm_inv), _p(Cv), _p(g))
    return Cv, g


def pattern(verts, n_verts):
    verts = _c(verts, np.int32)
    m, kind = verts.shape
    rowptr = np.empty(m + 1, np.int64)
    nnz = lib().orc_pattern(m, kind, _p(verts), n_verts, _p(rowptr), None)
    col = np.empty(nnz, np.int32)
    lib().orc_pattern(m, kind, _p(verts), n_verts, _p(rowptr), _p(col))
    return rowptr, col


def assemble(verts, w, g, alpha_tilde, rowptr, col):
    verts = _c(verts, np.int32)
    m, kind = verts.shape
    w, g, at = _c(w, np.float64), _c(g, np.float64), _c(alpha_tilde, np.float64)
    rowptr, col = _c(rowptr, np.int64), _c(col, np.int32)
    val = np.empty(col.shape[0])
    lib().orc_assemble(m, kind, _p(verts), _p(w), _p(g), _p(at), _p(rowptr), _p(col), _p(val))
    return val


def assemble_rows(rows, verts, w, g, alpha_tilde, rowptr, col):
    """Rows `rows` of A (values at those rows' CSR positions of a full-size array; others NaN)."""
    verts = _c(verts, np.int32)
    m, kind = verts.shape
    rows = _c(rows, np.int32)
    w, g, at = _c(w, np.float64), _c(g, np.float64), _c(alpha_tilde, np.float64)
    rowptr, col = _c(rowptr, np.int64), _c(col, np.int32)
    val = np.full(col.shape[0], np.nan)
    lib().orc_assemble_rows(rows.shape[0], _p(rows), kind, _p(verts), _p(w), _p(g), _p(at), _p(rowptr), _p(col), _p(val))
    return val


def rhs(Cv, alpha_tilde, lam):
    Cv, at, lam = _c(Cv, np.float64), _c(alpha_tilde, np.float64), _c(lam, np.float64)
    b = np.empty(Cv.shape[0])
    lib().orc_rhs(Cv.shape[0], _p(Cv), _p(at), _p(lam), _p(b))
    return b


def apply_dx(verts, n_verts, w, g, dl):
    verts = _c(verts, np.int32)
    m, kind = verts.shape
    w, g, dl = _c(w, np.float64), _c(g, np.float64), _c(dl, np.float64)
    dx = np.empty((n_verts, 3))
    lib().orc_apply_dx(m, kind, _p(verts), n_verts, _p(w), _p(g), _p(dl), _p(dx))
    return dx


def spmv(rowptr, col, val, x):
    rowptr, col, val, x = _c(rowptr, np.int64), _c(col, np.int32), _c(val, np.float64), _c(x, np.float64)
    y = np.empty(rowptr.shape[0] - 1)
    lib().orc_spmv(y.shape[0], _p(rowptr), _p(col), _p(val), _p(x), _p(y))
    return y


# ------------------------------------------------------------------------------ setup
def soc(rowptr, col, val, theta):
    rowptr, col, val = _c(rowptr, np.int64), _c(col, np.int32), _c(val, np.float64)
    s = np.empty(col.shape[0], np.uint8)
    lib().orc_soc(rowptr.shape[0] - 1, _p(rowptr), _p(col), _p(val), theta, _p(s))
    return s


def aggregate(rowptr, col, val, strong, seed=1, level=0):
    rowptr, col, val = _c(rowptr, np.int64), _c(col, np.int32), _c(val, np.float64)
    strong = _c(strong, np.uint8)
    n = rowptr.shape[0] - 1
    agg = np.empty(n, np.int32)
    na = lib().orc_aggregate(n, _p(rowptr), _p(col), _p(val), _p(strong), seed, level, _p(agg))
    return agg, int(na)


def colour(rowptr, col, seed=1):
    rowptr, col = _c(rowptr, np.int64), _c(col, np.int32)
    n = rowptr.shape[0] - 1
    c = np.empty(n, np.int32)
    nc = lib().orc_colour(n, _p(rowptr), _p(col), seed, _p(c))
    return c, int(nc)


def gs_bootstrap(rowptr, col, val, colours, sweeps=20, seed=1):
    rowptr, col, val = _c(rowptr, np.int64), _c(col, np.int32), _c(val, np.float64)
    colours = _c(colours, np.int32)
    n = rowptr.shape[0] - 1
    B = np.empty(n)
    lib().orc_gs_bootstrap(n, _p(rowptr), _p(col), _p(val), _p(colours), sweeps, seed, _p(B))
    return B


def prolongator(agg, n_agg, B):
    agg, B = _c(agg, np.int32), _c(B, np.float64)
    P = np.empty(agg.shape[0]); Bn = np.empty(n_agg)
    lib().orc_prolongator(agg.shape[0], _p(agg), n_agg, _p(B), _p(P), _p(Bn))
    return P, Bn


def gs_bootstrap_k(rowptr, col, val, colours, k, sweeps=20, seed=1):
    """k bootstrapped near-kernel columns (n x k array; reading c23)."""
    rowptr, col, val = _c(rowptr, np.int64), _c(col, np.int32), _c(val, np.float64)
    colours = _c(colours, np.int32)
    n = rowptr.shape[0] - 1
    B = np.empty(n * k)
    lib().orc_gs_bootstrap_k(n, _p(rowptr), _p(col), _p(val), _p(colours), sweeps, seed, k, _p(B))
    return B.reshape(k, n).T.copy()


def prolongator_qr(agg, n_agg, B, rank_tol=1e-10):
    """QR injection with k = B.shape[1] columns (readings c24, c25): (P as CSR (rowptr, col, val), B_next
    (n_next x k), coarse offsets per aggregate)."""
    agg = _c(agg, np.int32)
    B = np.asarray(B, np.float64)
    n, k = B.shape
    Bc = _c(B.T, np.float64)          # column-major
    coff = np.empty(n_agg + 1, np.int32); pptr = np.empty(n + 1, np.int64)
    nc = lib().orc_prolongator_qr(n, _p(agg), n_agg, k, _p(Bc), rank_tol, _p(coff), _p(pptr), None, None, None, 0)
    pcol = np.empty(int(pptr[-1]), np.int32); pval = np.empty(int(pptr[-1]))
    Bn = np.empty(nc * k)
    lib().orc_prolongator_qr(n, _p(agg), n_agg, k, _p(Bc), rank_tol, _p(coff), _p(pptr), _p(pcol), _p(pval),
                             _p(Bn), nc)
    return (pptr, pcol, pval), Bn.reshape(k, nc).T.copy(), coff


def galerkin_p(rowptr, col, val, P, nc):
    """P^T A P for a CSR prolongator P = (pptr, pcol, pval) with nc columns."""
    rowptr, col, val = _c(rowptr, np.int64), _c(col, np.int32), _c(val, np.float64)
    pptr, pcol, pval = _c(P[0], np.int64), _c(P[1], np.int32), _c(P[2], np.float64)
    n = rowptr.shape[0] - 1
    crow = np.empty(nc + 1, np.int64)
    nnz = lib().orc_galerkin_p(n, _p(rowptr), _p(col), _p(val), _p(pptr), _p(pcol), _p(pval), nc, _p(crow), None, None)
    ccol = np.empty(nnz, np.int32); cval = np.empty(nnz)
    lib().orc_galerkin_p(n, _p(rowptr), _p(col), _p(val), _p(pptr), _p(pcol), _p(pval), nc, _p(crow), _p(ccol),
                         _p(cval))
    return crow, ccol, cval


def galerkin(rowptr, col, val, agg, P, n_agg):
    rowptr, col, val = _c(rowptr, np.int64), _c(col, np.int32), _c(val, np.float64)
    agg, P = _c(agg, np.int32), _c(P, np.float64)
    n = rowptr.shape[0] - 1
    crow = np.empty(n_agg + 1, np.int64)
    nnz = lib().orc_galerkin(n, _p(rowptr), _p(col), _p(val), _p(agg), _p(P), n_agg, _p(crow), None, None)
    ccol = np.empty(nnz, np.int32); cval = np.empty(nnz)
    lib().orc_galerkin(n, _p(rowptr), _p(col), _p(val), _p(agg), _p(P), n_agg, _p(crow), _p(ccol), _p(cval))
    return crow, ccol, cval


def power(rowptr, col, val, iters=100, seed=1, level=0):
    rowptr, col, val = _c(rowptr, np.int64), _c(col, np.int32), _c(val, np.float64)
    return float(lib().orc_power(rowptr.shape[0] - 1, _p(rowptr), _p(col), _p(val), iters, seed, level))


def cholesky(A):
    A = _c(A, np.float64)
    n = A.shape[0]
    L = np.empty_like(A)
    rc = lib().orc_cholesky(n, _p(A), _p(L))
    return L, rc


def chol_solve(L, b):
    L, b = _c(L, np.float64), _c(b, np.float64)
    x = np.empty_like(b)
    lib().orc_chol_solve(b.shape[0], _p(L), _p(b), _p(x))
    return x


class Hierarchy:
    """Setup of the UA-AMG hierarchy from A_0 + V-cycle / MGPCG."""

    def __init__(self, rowptr, col, val, cfg: Config | None = None, _handle=None, _owner=None):
        self._owner = _owner
        self.cfg = cfg if cfg is not None else (getattr(_owner, "cfg", None) if _owner is not None else None)
        if _handle is not None:
            self.h = _handle
            self._own = False
        else:
            cfg = cfg or default_config()
            self.cfg = cfg
            self._keep = [_c(rowptr, np.int64), _c(col, np.int32), _c(val, np.float64)]
            r, c, v = self._keep
            self.h = lib().orc_hier_build(r.shape[0] - 1, _p(r), _p(c), _p(v), C.byref(cfg))
            self._own = True

    def __del__(self):
        if getattr(self, "_own", False) and self.h:
            lib().orc_hier_free(self.h)
            self.h = None

    @property
    def n_levels(self) -> int:
        return int(lib().orc_hier_levels(self.h))

    def level_size(self, l):
        n = C.c_int32(); nnz = C.c_int64()
        lib().orc_hier_level_size(self.h, l, C.byref(n), C.byref(nnz))
        return n.value, nnz.value

    def level(self, l):
        n, nnz = self.level_size(l)
        r = np.empty(n + 1, np.int64); c = np.empty(nnz, np.int32); v = np.empty(nnz)
        lib().orc_hier_get_level(self.h, l, _p(r), _p(c), _p(v))
        return r, c, v

    def agg(self, l):
        n, _ = self.level_size(l)
        a = np.empty(n, np.int32)
        lib().orc_hier_get_agg(self.h, l, _p(a))
        return a

    def P(self, l):
        n, _ = self.level_size(l)
        a = np.empty(n)
        lib().orc_hier_get_P(self.h, l, _p(a))
        return a

    def omega(self, l) -> float:
        return float(lib().orc_hier_omega(self.h, l))

    def cheb(self, l):
        """(theta, delta) of level l's Chebyshev interval (reading c20)."""
        t, d = C.c_double(), C.c_double()
        lib().orc_hier_cheb(self.h, l, C.byref(t), C.byref(d))
        return t.value, d.value

    def smooth(self, l, b, x0, post=False):
        """One pre (post=False) or post smoothing pass (configured smoother) at level l, from x0."""
        x = _c(x0, np.float64).copy()
        lib().orc_hier_smooth(self.h, l, _p(_c(b, np.float64)), _p(x), int(post))
        return x

    def B0(self):
        """Level-0 near kernel: n (k = 1) or n x k (k > 1)."""
        n, _ = self.level_size(0)
        k = max(int(self.cfg.k_nullspace), 1) if self.cfg is not None else 1
        a = np.empty(n * k)
        lib().orc_hier_get_B0(self.h, _p(a))
        return a if k == 1 else a.reshape(k, n).T.copy()

    def P_csr(self, l):
        """Level-l prolongator as CSR (rowptr, col, val); k = 1: one entry per row, column = aggregate."""
        nnz = C.c_int64()
        lib().orc_hier_get_P_csr(self.h, l, C.byref(nnz), None, None, None)
        n, _ = self.level_size(l)
        r = np.empty(n + 1, np.int64); c = np.empty(nnz.value, np.int32); v = np.empty(nnz.value)
        lib().orc_hier_get_P_csr(self.h, l, C.byref(nnz), _p(r), _p(c), _p(v))
        return r, c, v

    @property
    def n_colours(self) -> int:
        return int(lib().orc_hier_n_colours(self.h))

    def refresh_omega(self, iters):
        """Reading c26: omega / Chebyshev parameters from `iters` further power iterations on the current levels."""
        lib().orc_hier_refresh_omega(self.h, int(iters))

    def refresh(self, val0) -> int:
        v = _c(val0, np.float64)
        return int(lib().orc_hier_refresh(self.h, _p(v)))

    def vcycle(self, b):
        b = _c(b, np.float64)
        x = np.empty_like(b)
        lib().orc_vcycle(self.h, _p(b), _p(x))
        return x

    def pcg(self, b, iters):
        b = _c(b, np.float64)
        x = np.empty_like(b); tr = np.empty(max(iters, 1))
        rc = lib().orc_pcg(self.h, _p(b), iters, _p(x), _p(tr))
        return x, int(rc), tr[:iters]

    def operator_complexity(self) -> float:
        nnz = [self.level_size(l)[1] for l in range(self.n_levels)]
        return sum(nnz) / nnz[0]


class Sim:
    """Algorithm 1 frame loop."""

    def __init__(self, scene, cfg: Config | None = None):
        self.cfg = cfg or default_config(omega_relax=scene.omega_relax, pcg_iters=scene.pcg_iters)
        self.kind = scene.kind
        self.n = scene.n_verts
        self.m = scene.n_cons
        self._keep = [_c(scene.verts, np.int32), _c(scene.rest_pos, np.float64),
                      _c(scene.pos, np.float64), _c(scene.vel, np.float64),
                      _c(scene.inv_mass, np.float64), _c(scene.compliance, np.float64)]
        v, X, x, vel, w, a = self._keep
        self.s = lib().orc_sim_create(self.kind, self.n, self.m, _p(v), _p(X), _p(x), _p(vel),
                                      _p(w), _p(a), C.byref(self.cfg))

    def __del__(self):
        if getattr(self, "s", None):
            lib().orc_sim_free(self.s)
            self.s = None

    def step(self, dt, n_iters) -> int:
        return int(lib().orc_sim_step(self.s, dt, n_iters))

    def mark_stale(self):
        lib().orc_sim_mark_stale(self.s)

    def indefinite_events(self) -> int:
        return int(lib().orc_sim_indefinite_events(self.s))

    def setups(self) -> int:
        return int(lib().orc_sim_setups(self.s))

    def setup_ms(self) -> float:
        """Wall time of the last frame's setup (timing for bench.py; 0 if no setup ran)."""
        return float(lib().orc_sim_setup_ms(self.s))

    def iters_used(self) -> int:
        return int(lib().orc_sim_iters_used(self.s))

    def omega(self) -> float:
        return float(lib().orc_sim_omega(self.s))

    def state(self):
        x = np.empty((self.n, 3)); v = np.empty((self.n, 3)); lam = np.empty(self.m)
        lib().orc_sim_get(self.s, _p(x), _p(v), _p(lam))
        return x, v, lam

    def set_state(self, x, v):
        x, v = _c(x, np.float64), _c(v, np.float64)
        lib().orc_sim_set(self.s, _p(x), _p(v))

    def A(self):
        nnz = int(lib().orc_sim_nnz(self.s))
        r = np.empty(self.m + 1, np.int64); c = np.empty(nnz, np.int32); v = np.empty(nnz)
        lib().orc_sim_get_A(self.s, _p(r), _p(c), _p(v))
        return r, c, v

    def b_norms(self, n):
        out = np.zeros(n)
        lib().orc_sim_get_b_norms(self.s, _p(out), n)
        return out

    def hierarchy(self) -> Hierarchy:
        return Hierarchy(None, None, None, _handle=lib().orc_sim_hier(self.s), _owner=self)
