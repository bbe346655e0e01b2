"""Thin ctypes binding of libmgpbd.so (include/mgpbd.h).  Argument marshalling only: every step
of the MGPBD frame runs in the library's CUDA kernels.  There is no CPU fallback: if the library is
missing or no CUDA device is present, calls fail loudly."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmgpbd.so")

OK, E_ARG, E_CUDA, E_NCCL, E_OOM, E_INDEFINITE, E_NONFINITE, E_STALL = 0, -1, -2, -3, -4, -5, -6, -7
DISTANCE, TET_ARAP = 2, 4
MAX_LEVELS, MAX_ITERS, MAX_FRAME_ITERS = 16, 256, 1000000

SYMBOLS = ["mgpbd_config_default", "mgpbd_create", "mgpbd_setup_hierarchy", "mgpbd_step", "mgpbd_set_state",
           "mgpbd_set_profiling",
           "mgpbd_get_positions", "mgpbd_get_velocities", "mgpbd_get_lambda", "mgpbd_get_stats",
           "mgpbd_get_level_sizes", "mgpbd_get_level", "mgpbd_get_prolongator", "mgpbd_get_aggregates",
           "mgpbd_get_near_kernel", "mgpbd_debug_setup_from", "mgpbd_debug_vcycle", "mgpbd_debug_pcg",
           "mgpbd_debug_prepare", "mgpbd_get_prolongator_csr",
           "mgpbd_pass_burst",
           "mgpbd_last_error", "mgpbd_destroy", "mgpbd_nccl_unique_id", "mgpbd_vgroup_create",
           "mgpbd_vgroup_destroy", "mgpbd_partition_rows", "mgpbd_halo_plan"]


class MgpbdError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"mgpbd status {status}: {msg}")
        self.status = status


class Mesh(C.Structure):
    _fields_ = [("n_verts", C.c_int32), ("rest_pos", C.c_void_p), ("pos", C.c_void_p), ("vel", C.c_void_p)]


class Constraints(C.Structure):
    _fields_ = [("kind", C.c_int), ("n_cons", C.c_int32), ("verts", C.c_void_p)]


class Config(C.Structure):
    _fields_ = [("precision", C.c_int32), ("theta", C.c_double), ("k_nullspace", C.c_int32),
                ("min_coarse", C.c_int32), ("max_levels", C.c_int32), ("stall_ratio", C.c_double),
                ("setup_interval", C.c_int32), ("bootstrap_sweeps", C.c_int32), ("power_iters", C.c_int32),
                ("lambda_min_est", C.c_double), ("lambda_safety", C.c_double), ("smoother_sweeps", C.c_int32),
                ("pcg_iters", C.c_int32),
                ("omega_relax", C.c_double), ("gravity", C.c_double * 3), ("seed", C.c_uint64),
                ("device", C.c_int32), ("stream", C.c_void_p), ("max_dense_coarse", C.c_int32),
                ("rank", C.c_int32), ("world", C.c_int32), ("profile", C.c_int32),
                ("nccl_id", C.c_void_p), ("vgroup", C.c_void_p), ("level0_operator", C.c_int32),
                ("smoother", C.c_int32), ("cheb_lower", C.c_double), ("backtrack", C.c_int32),
                ("omega_min", C.c_double), ("residual_tol", C.c_double), ("pcg_tol", C.c_double),
                ("residual_abs", C.c_double), ("resetup_on_indef", C.c_int32),
                ("omega_refresh_iters", C.c_int32), ("time_budget_ms", C.c_double)]


class Stats(C.Structure):
    _fields_ = [("n_levels", C.c_int32), ("n", C.c_int64 * MAX_LEVELS), ("nnz", C.c_int64 * MAX_LEVELS),
                ("op_complexity", C.c_double), ("omega", C.c_double * MAX_LEVELS), ("n_colours", C.c_int32),
                ("setup_ran", C.c_int32), ("n_b", C.c_int32), ("b_norm", C.c_double * MAX_ITERS),
                ("frame", C.c_int64), ("l0_pass_ms", C.c_double), ("l0_pass_launches", C.c_int64),
                ("l0_pass_bytes", C.c_double), ("ms_setup", C.c_double), ("ms_frame", C.c_double),
                ("kernel_launches", C.c_int64), ("indefinite_events", C.c_int32),
                ("rank", C.c_int32), ("world", C.c_int32), ("row_begin", C.c_int32), ("row_end", C.c_int32),
                ("halo_rows", C.c_int64), ("omega_relax", C.c_double), ("ms_assemble", C.c_double),
                ("ms_galerkin", C.c_double), ("ms_vcycle", C.c_double), ("ms_pcg_other", C.c_double),
                ("ms_update", C.c_double), ("iters_run", C.c_int32), ("b_last", C.c_double)]


_lib = None


def lib():
    """Load libmgpbd.so (built in-tree by build.py).  Raises if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2505_13390_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        P, i32, i64, f64 = C.c_void_p, C.c_int32, C.c_int64, C.c_double
        sig = {
            "mgpbd_config_default": (C.c_int, [P]),
            "mgpbd_create": (C.c_int, [P, P, P, P, P, P]),
            "mgpbd_setup_hierarchy": (C.c_int, [P]),
            "mgpbd_step": (C.c_int, [P, f64, i32]),
            "mgpbd_set_state": (C.c_int, [P, P, P]),
            "mgpbd_set_profiling": (C.c_int, [P, i32]),
            "mgpbd_get_positions": (C.c_int, [P, P]),
            "mgpbd_get_velocities": (C.c_int, [P, P]),
            "mgpbd_get_lambda": (C.c_int, [P, P]),
            "mgpbd_get_stats": (C.c_int, [P, P]),
            "mgpbd_get_level_sizes": (C.c_int, [P, i32, P, P]),
            "mgpbd_get_level": (C.c_int, [P, i32, P, P, P]),
            "mgpbd_get_prolongator": (C.c_int, [P, i32, P]),
            "mgpbd_get_prolongator_csr": (C.c_int, [P, i32, P, P, P, P]),
            "mgpbd_get_aggregates": (C.c_int, [P, i32, P]),
            "mgpbd_get_near_kernel": (C.c_int, [P, P]),
            "mgpbd_debug_setup_from": (C.c_int, [P, P]),
            "mgpbd_debug_vcycle": (C.c_int, [P, P, P]),
            "mgpbd_debug_pcg": (C.c_int, [P, P, i32, P]),
            "mgpbd_debug_prepare": (C.c_int, [P, f64]),
            "mgpbd_pass_burst": (C.c_int, [P, i32, P, P]),
            "mgpbd_last_error": (C.c_char_p, [P]),
            "mgpbd_nccl_unique_id": (C.c_int, [P]),
            "mgpbd_vgroup_create": (C.c_int, [i32, P]),
            "mgpbd_vgroup_destroy": (None, [P]),
            "mgpbd_partition_rows": (C.c_int, [P, i32, i32, P]),
            "mgpbd_halo_plan": (C.c_int, [P, P, P, i32, P]),
            "mgpbd_destroy": (None, [P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0 creates it; broadcast it to the other ranks)."""
    buf = C.create_string_buffer(128)
    st = lib().mgpbd_nccl_unique_id(buf)
    if st != OK:
        raise MgpbdError(st, lib().mgpbd_last_error(None).decode())
    return buf.raw


class VirtualGroup:
    """W virtual ranks in one process (one thread per context, all on one GPU)."""

    def __init__(self, world: int):
        h = C.c_void_p()
        st = lib().mgpbd_vgroup_create(world, C.byref(h))
        if st != OK:
            raise MgpbdError(st, "vgroup_create")
        self.h, self.world = h, world

    def __del__(self):
        if getattr(self, "h", None):
            lib().mgpbd_vgroup_destroy(self.h)
            self.h = None


def partition_rows(rowptr, world):
    """Host-only: row blocks [bounds[p], bounds[p+1]) balanced by nonzeros (no GPU needed)."""
    rowptr = np.ascontiguousarray(rowptr, np.int64)
    out = np.empty(world + 1, np.int32)
    st = lib().mgpbd_partition_rows(_p(rowptr), rowptr.shape[0] - 1, world, _p(out))
    if st != OK:
        raise MgpbdError(st, "partition_rows")
    return out


def halo_plan(bounds, minc, maxc):
    """Host-only: recv[q, p] = [a, b) rows rank q receives from rank p."""
    bounds = np.ascontiguousarray(bounds, np.int32)
    minc, maxc = np.ascontiguousarray(minc, np.int32), np.ascontiguousarray(maxc, np.int32)
    w = bounds.shape[0] - 1
    out = np.empty((w, w, 2), np.int32)
    st = lib().mgpbd_halo_plan(_p(bounds), _p(minc), _p(maxc), w, _p(out))
    if st != OK:
        raise MgpbdError(st, "halo_plan")
    return out


def config_default(**kw) -> Config:
    c = Config()
    lib().mgpbd_config_default(C.byref(c))
    for k, v in kw.items():
        if k == "gravity":
            c.gravity[:] = list(v)
        else:
            setattr(c, k, v)
    return c


class Context:
    """One MGPBD simulation on one GPU (mgpbd_create ... mgpbd_destroy)."""

    def __init__(self, kind, verts, rest_pos, inv_mass, compliance, pos=None, vel=None, cfg: Config | None = None,
                 **cfg_kw):
        L = lib()
        nccl_id = cfg_kw.pop("nccl_id", None)
        vgroup = cfg_kw.pop("vgroup", None)
        self.cfg = cfg or config_default(**cfg_kw)
        self._keep = []
        if nccl_id is not None:
            buf = C.create_string_buffer(bytes(nccl_id), 128)
            self._keep.append(buf)
            self.cfg.nccl_id = C.cast(buf, C.c_void_p)
        if vgroup is not None:
            self._keep.append(vgroup)
            self.cfg.vgroup = vgroup.h
        self.verts = np.ascontiguousarray(verts, np.int32)
        self.m = int(self.verts.shape[0])
        self.rest = np.ascontiguousarray(rest_pos, np.float64)
        self.n = int(self.rest.shape[0])
        self._pos = None if pos is None else np.ascontiguousarray(pos, np.float64)
        self._vel = None if vel is None else np.ascontiguousarray(vel, np.float64)
        w = np.ascontiguousarray(inv_mass, np.float64)
        a = np.ascontiguousarray(compliance, np.float64)
        mesh = Mesh(self.n, _p(self.rest), _p(self._pos), _p(self._vel))
        cons = Constraints(int(kind), self.m, _p(self.verts))
        h = C.c_void_p()
        st = L.mgpbd_create(C.byref(mesh), C.byref(cons), _p(w), _p(a), C.byref(self.cfg), C.byref(h))
        if st != OK:
            raise MgpbdError(st, L.mgpbd_last_error(None).decode())
        self.h = h

    @classmethod
    def from_scene(cls, sc, **cfg_kw):
        cfg_kw.setdefault("omega_relax", sc.omega_relax)
        cfg_kw.setdefault("pcg_iters", sc.pcg_iters)
        return cls(sc.kind, sc.verts, sc.rest_pos, sc.inv_mass, sc.compliance, pos=sc.pos, vel=sc.vel, **cfg_kw)

    def _ck(self, st):
        if st != OK:
            raise MgpbdError(st, lib().mgpbd_last_error(self.h).decode())

    def close(self):
        if getattr(self, "h", None):
            lib().mgpbd_destroy(self.h)
            self.h = None

    __del__ = close

    def setup_hierarchy(self):
        self._ck(lib().mgpbd_setup_hierarchy(self.h))

    def step(self, dt, n_iters):
        self._ck(lib().mgpbd_step(self.h, float(dt), int(n_iters)))

    def set_profiling(self, on):
        """False/0 off, True/1 eager event timing, 2 events captured inside the replayed graphs."""
        self._ck(lib().mgpbd_set_profiling(self.h, int(on)))

    def set_state(self, pos, vel=None):
        pos = np.ascontiguousarray(pos, np.float64)
        vel = None if vel is None else np.ascontiguousarray(vel, np.float64)
        self._ck(lib().mgpbd_set_state(self.h, _p(pos), _p(vel)))

    def positions(self, out=None):
        out = np.empty((self.n, 3)) if out is None else out
        self._ck(lib().mgpbd_get_positions(self.h, _p(out)))
        return out

    def velocities(self, out=None):
        out = np.empty((self.n, 3)) if out is None else out
        self._ck(lib().mgpbd_get_velocities(self.h, _p(out)))
        return out

    def lambdas(self, out=None):
        out = np.empty(self.m) if out is None else out
        self._ck(lib().mgpbd_get_lambda(self.h, _p(out)))
        return out

    def stats(self) -> Stats:
        s = Stats()
        self._ck(lib().mgpbd_get_stats(self.h, C.byref(s)))
        return s

    def level_size(self, l):
        n = C.c_int64(); nnz = C.c_int64()
        self._ck(lib().mgpbd_get_level_sizes(self.h, l, C.byref(n), C.byref(nnz)))
        return n.value, nnz.value

    def level(self, l):
        n, nnz = self.level_size(l)
        r = np.empty(n + 1, np.int64); c = np.empty(nnz, np.int32); v = np.empty(nnz)
        self._ck(lib().mgpbd_get_level(self.h, l, _p(r), _p(c), _p(v)))
        return r, c, v

    def prolongator(self, l):
        n, _ = self.level_size(l)
        out = np.empty(n)
        self._ck(lib().mgpbd_get_prolongator(self.h, l, _p(out)))
        return out

    def prolongator_csr(self, l):
        """Level-l prolongator as CSR (rowptr, col, val) — k_nullspace > 1 (and k = 1 in the same form)."""
        nnz = C.c_int64()
        self._ck(lib().mgpbd_get_prolongator_csr(self.h, l, C.byref(nnz), None, None, None))
        n, _ = self.level_size(l)
        r = np.empty(n + 1, np.int64); c = np.empty(nnz.value, np.int32); v = np.empty(nnz.value)
        self._ck(lib().mgpbd_get_prolongator_csr(self.h, l, C.byref(nnz), _p(r), _p(c), _p(v)))
        return r, c, v

    def aggregates(self, l):
        n, _ = self.level_size(l)
        out = np.empty(n, np.int32)
        self._ck(lib().mgpbd_get_aggregates(self.h, l, _p(out)))
        return out

    def near_kernel(self):
        """n (k = 1) or n x k (k_nullspace > 1) bootstrapped near-kernel vectors of level 0."""
        k = max(int(self.cfg.k_nullspace), 1)
        out = np.empty(self.m * k)
        self._ck(lib().mgpbd_get_near_kernel(self.h, _p(out)))
        return out if k == 1 else out.reshape(k, self.m).T.copy()

    def debug_setup_from(self, vals):
        vals = np.ascontiguousarray(vals, np.float64)
        self._ck(lib().mgpbd_debug_setup_from(self.h, _p(vals)))

    def debug_prepare(self, dt):
        """Alg. 1 l.1-7 of the next frame without the solve (mgpbd_debug_prepare)."""
        self._ck(lib().mgpbd_debug_prepare(self.h, float(dt)))

    def debug_vcycle(self, b):
        b = np.ascontiguousarray(b, np.float64)
        x = np.empty_like(b)
        self._ck(lib().mgpbd_debug_vcycle(self.h, _p(b), _p(x)))
        return x

    def pass_burst(self, reps):
        """(device ms, algorithmic bytes) of `reps` level-0 passes replayed as one CUDA graph."""
        ms, by = C.c_double(), C.c_double()
        self._ck(lib().mgpbd_pass_burst(self.h, int(reps), C.byref(ms), C.byref(by)))
        return ms.value, by.value

    def debug_pcg(self, b, iters):
        b = np.ascontiguousarray(b, np.float64)
        x = np.empty_like(b)
        self._ck(lib().mgpbd_debug_pcg(self.h, _p(b), int(iters), _p(x)))
        return x
