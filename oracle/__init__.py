"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

Plain single-threaded fp64 C++17 implementation (``oracle/oracle.cpp``) of the
solve phase of arXiv 2006.06052's AMG-preconditioned Krylov solver, written
from PAPER.md and the SURVEY.md §8(c) readings.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product library
(``paper_2006_06052_b200``) never imports, links or calls it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")

CG, BICGSTAB, GMRES, IDRS = 0, 1, 2, 3
PC_AMG, PC_SCHUR, PC_NONE = 0, 1, 2
SPAI0, JACOBI, ILU0, ILUT = 0, 1, 2, 3
SA, PLAIN = 0, 1  # coarsening
OK, NOT_CONVERGED, EINVAL, EDIM, EZERODIAG, ESINGULAR_BLOCK, EBREAKDOWN = 0, 1, -1, -2, -3, -4, -6


def build(force: bool = False) -> str:
    srcs = [os.path.join(_HERE, f) for f in ("oracle.cpp", "oracle.h")]
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(map(os.path.getmtime, srcs)):
        subprocess.check_call(
            ["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
             "-o", _SO, srcs[0]]
        )
    return _SO


class Params(ctypes.Structure):
    _fields_ = [
        ("solver", ctypes.c_int32), ("gmres_m", ctypes.c_int32), ("precond", ctypes.c_int32),
        ("maxiter", ctypes.c_int32), ("hier_f32", ctypes.c_int32), ("vec_f32", ctypes.c_int32),
        ("smoother", ctypes.c_int32), ("jacobi_omega", ctypes.c_double), ("sa_omega", ctypes.c_double),
        ("eps_strong", ctypes.c_double), ("coarse_enough", ctypes.c_int32), ("max_levels", ctypes.c_int32),
        ("npre", ctypes.c_int32), ("npost", ctypes.c_int32), ("schur_p_component", ctypes.c_int32),
        ("nparts", ctypes.c_int32), ("idrs_s", ctypes.c_int32), ("idrs_seed", ctypes.c_int32),
        ("schur_u_scalar", ctypes.c_int32), ("coarsening", ctypes.c_int32), ("schur_shat", ctypes.c_int32),
        ("over_interp", ctypes.c_double), ("ilu_sweeps", ctypes.c_int32), ("gmres_ortho", ctypes.c_int32),
        ("ilut_tau", ctypes.c_double), ("ilut_p", ctypes.c_int32),
    ]


class Report(ctypes.Structure):
    _fields_ = [("iters", ctypes.c_int32), ("converged", ctypes.c_int32), ("levels", ctypes.c_int32),
                ("restarts", ctypes.c_int32), ("relres_true", ctypes.c_double)]


_lib = None
P = ctypes.c_void_p


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        i32, i64, dbl = ctypes.c_int32, ctypes.c_int64, ctypes.c_double
        sig = {
            "orc_params_default": (None, [P]),
            "orc_mat_new": (P, [i32, i32, i32, P, P, P]),
            "orc_mat_free": (None, [P]),
            "orc_mat_info": (None, [P, P]),
            "orc_mat_export": (None, [P, P, P, P]),
            "orc_csr_to_bsr": (P, [i32, i32, i32, P, P, P]),
            "orc_spmv": (i32, [P, dbl, P, dbl, P]),
            "orc_strength": (i64, [P, dbl, i32, P, P]),
            "orc_aggregate": (i32, [P, dbl, i32, P]),
            "orc_roots": (i32, [P, dbl, i32, P]),
            "orc_block_inverse": (i32, [i32, P, P]),
            "orc_setup": (i32, [P, P, P]),
            "orc_setup_pmask": (i32, [P, P, P, P]),
            "orc_schur_np": (i32, [P]),
            "orc_free": (None, [P]),
            "orc_levels": (i32, [P]),
            "orc_level_mat": (P, [P, i32, i32]),
            "orc_level_agg": (P, [P, i32]),
            "orc_level_M": (P, [P, i32]),
            "orc_level_smooth": (i32, [P, i32, P, P]),
            "orc_schur_Au": (P, [P]),
            "orc_schur_Au_amg": (P, [P]),
            "orc_schur_Shat_diag": (P, [P]),
            "orc_schur_mS": (P, [P]),
            "orc_vcycle": (i32, [P, P, P]),
            "orc_precond": (i32, [P, P, P]),
            "orc_solve": (i32, [P, P, P, dbl, P, P]),
            "orc_solve_timed": (i32, [P, P, P, dbl, P, P, i32]),
            "orc_idrs_shadow": (i32, [i64, i32, i64, P]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(P)


def default_params(**kw) -> Params:
    p = Params()
    lib().orc_params_default(ctypes.byref(p))
    for k, v in kw.items():
        setattr(p, k, v)
    return p


class Mat:
    """BSR matrix held by the oracle (fp64)."""

    def __init__(self, handle, owned=True):
        self.h = handle
        self.owned = owned

    @classmethod
    def from_arrays(cls, ptr, col, val, n_cols=None):
        ptr = np.ascontiguousarray(ptr, dtype=np.int32)
        col = np.ascontiguousarray(col, dtype=np.int32)
        val = np.ascontiguousarray(val, dtype=np.float64)
        n = len(ptr) - 1
        b = val.shape[-1] if val.ndim == 3 else 1
        h = lib().orc_mat_new(n, n if n_cols is None else n_cols, b, _p(ptr), _p(col), _p(val))
        if not h:
            raise ValueError("orc_mat_new rejected the matrix")
        return cls(h)

    def __del__(self):
        if getattr(self, "owned", False) and self.h:
            lib().orc_mat_free(self.h)
            self.h = None

    def info(self):
        out = np.zeros(4, dtype=np.int64)
        lib().orc_mat_info(self.h, _p(out))
        return tuple(int(v) for v in out)

    def to_arrays(self):
        n, m, b, nnz = self.info()
        ptr = np.empty(n + 1, dtype=np.int32)
        col = np.empty(nnz, dtype=np.int32)
        val = np.empty((nnz, b, b), dtype=np.float64)
        lib().orc_mat_export(self.h, _p(ptr), _p(col), _p(val))
        return ptr, col, val

    def dense(self):
        n, m, b, _ = self.info()
        ptr, col, val = self.to_arrays()
        D = np.zeros((n * b, m * b))
        for i in range(n):
            for k in range(ptr[i], ptr[i + 1]):
                D[i * b:(i + 1) * b, col[k] * b:(col[k] + 1) * b] = val[k]
        return D


def csr_to_bsr(n, m, b, ptr, col, val) -> Mat:
    ptr = np.ascontiguousarray(ptr, dtype=np.int32)
    col = np.ascontiguousarray(col, dtype=np.int32)
    val = np.ascontiguousarray(val, dtype=np.float64)
    h = lib().orc_csr_to_bsr(n, m, b, _p(ptr), _p(col), _p(val))
    if not h:
        raise ValueError("not divisible")
    return Mat(h)


def spmv(A: Mat, x, alpha=1.0, beta=0.0, y=None):
    n, m, b, _ = A.info()
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.zeros(n * b) if y is None else np.ascontiguousarray(y, dtype=np.float64).copy()
    lib().orc_spmv(A.h, alpha, _p(x), beta, _p(y))
    return y


def strength(A: Mat, eps=1e-3, nparts=1):
    n = A.info()[0]
    e = lib().orc_strength(A.h, eps, nparts, None, None)
    if e < 0:
        raise RuntimeError(f"strength failed {e}")
    ptr = np.empty(n + 1, dtype=np.int32)
    col = np.empty(max(e, 1), dtype=np.int32)
    lib().orc_strength(A.h, eps, nparts, _p(ptr), _p(col))
    return ptr, col[:e]


def aggregate(A: Mat, eps=1e-3, nparts=1):
    n = A.info()[0]
    agg = np.empty(n, dtype=np.int32)
    nc = lib().orc_aggregate(A.h, eps, nparts, _p(agg))
    if nc < 0:
        raise RuntimeError(f"aggregate failed {nc}")
    return agg, nc


def roots(A: Mat, eps=1e-3, nparts=1):
    n = A.info()[0]
    r = np.empty(n, dtype=np.int32)
    lib().orc_roots(A.h, eps, nparts, _p(r))
    return r


def idrs_shadow(n: int, s: int, base: int) -> np.ndarray:
    """IDR(s) shadow space [s][n] (counter RNG stream 6, MGS-orthonormalised)."""
    out = np.zeros((s, n))
    lib().orc_idrs_shadow(n, s, base, _p(out))
    return out


def block_inverse(blk):
    blk = np.ascontiguousarray(blk, dtype=np.float64)
    b = blk.shape[0]
    inv = np.empty_like(blk)
    rc = lib().orc_block_inverse(b, _p(blk), _p(inv))
    if rc != OK:
        raise np.linalg.LinAlgError("singular block")
    return inv


@dataclass
class SolveResult:
    x: np.ndarray
    status: int
    iters: int
    converged: bool
    relres_true: float
    levels: int
    restarts: int
    history: np.ndarray | None = field(default=None)


class Solver:
    def __init__(self, A: Mat, params: Params | None = None, pmask=None, **kw):
        """pmask (optional, n_rows*b bools): Schur split by a general scalar pressure mask (R21)."""
        self.A = A
        self.params = params if params is not None else default_params(**kw)
        h = P()
        if pmask is None:
            rc = lib().orc_setup(A.h, ctypes.byref(self.params), ctypes.byref(h))
        else:
            self._pmask = np.ascontiguousarray(pmask, dtype=np.uint8)
            rc = lib().orc_setup_pmask(A.h, self._pmask.ctypes.data_as(ctypes.c_void_p), ctypes.byref(self.params),
                                       ctypes.byref(h))
        if rc != OK:
            raise RuntimeError(f"orc_setup failed: {rc}")
        self.h = h
        self.n, _, self.b, _ = A.info()

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_free(self.h)
            self.h = None

    @property
    def levels(self) -> int:
        return lib().orc_levels(self.h)

    def level_mat(self, level: int, which: int = 0) -> Mat | None:
        h = lib().orc_level_mat(self.h, level, which)
        return Mat(h, owned=False) if h else None

    def level_agg(self, level: int) -> np.ndarray:
        A = self.level_mat(level, 0)
        n = A.info()[0]
        p = lib().orc_level_agg(self.h, level)
        return np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(ctypes.c_int32)), shape=(n,)).copy()

    def level_M(self, level: int) -> np.ndarray:
        A = self.level_mat(level, 0)
        n, _, b, _ = A.info()
        p = lib().orc_level_M(self.h, level)
        return np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(ctypes.c_double)), shape=(n, b, b)).copy()

    def level_smooth(self, level: int, f) -> np.ndarray:
        """x = S_l(f), the level's pre-smoother from zero (M f, or the sweep-solved ILU(0))."""
        f = np.ascontiguousarray(f, dtype=np.float64)
        x = np.zeros_like(f)
        assert lib().orc_level_smooth(self.h, level, _p(f), _p(x)) == 0
        return x

    def schur_Au(self) -> Mat | None:
        h = lib().orc_schur_Au(self.h)
        return Mat(h, owned=False) if h else None

    def schur_Au_amg(self) -> Mat | None:
        """The matrix the U-solver hierarchy is built on (A_u or its scalar expansion)."""
        h = lib().orc_schur_Au_amg(self.h)
        return Mat(h, owned=False) if h else None

    def schur_vectors(self):
        n = lib().orc_schur_np(self.h)
        dp = lib().orc_schur_Shat_diag(self.h)
        mp = lib().orc_schur_mS(self.h)
        if not dp:
            return None, None
        cast = lambda q: np.ctypeslib.as_array(ctypes.cast(q, ctypes.POINTER(ctypes.c_double)), shape=(n,)).copy()
        return cast(dp), cast(mp)

    def vcycle(self, f):
        A0 = self.level_mat(0, 0)
        n, _, b, _ = A0.info()
        f = np.ascontiguousarray(f, dtype=np.float64)
        x = np.zeros(n * b)
        lib().orc_vcycle(self.h, _p(f), _p(x))
        return x

    def precond(self, r):
        r = np.ascontiguousarray(r, dtype=np.float64)
        z = np.zeros_like(r)
        lib().orc_precond(self.h, _p(r), _p(z))
        return z

    def solve(self, b, x0=None, rtol=1e-8, history=False) -> SolveResult:
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.zeros_like(b) if x0 is None else np.ascontiguousarray(x0, dtype=np.float64).copy()
        rep = Report()
        hist = np.full(self.params.maxiter + 1, np.nan) if history else None
        st = lib().orc_solve(self.h, _p(b), _p(x), rtol, ctypes.byref(rep), _p(hist))
        if hist is not None:
            hist = hist[: rep.iters + 1]
        return SolveResult(x, st, rep.iters, bool(rep.converged), rep.relres_true, rep.levels,
                           rep.restarts, hist)

    def solve_timed(self, b, x0=None, rtol=1e-8):
        """solve() with per-iteration timestamps (seconds since the call; stamps[it] when
        iteration `it` completed, stamps[0] = 0).  Timing instrumentation only."""
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.zeros_like(b) if x0 is None else np.ascontiguousarray(x0, dtype=np.float64).copy()
        rep = Report()
        stamps = np.full(self.params.maxiter + 1, np.nan)
        st = lib().orc_solve_timed(self.h, _p(b), _p(x), rtol, ctypes.byref(rep), _p(stamps), len(stamps))
        return SolveResult(x, st, rep.iters, bool(rep.converged), rep.relres_true, rep.levels,
                           rep.restarts, None), stamps[: rep.iters + 1]
