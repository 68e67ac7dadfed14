"""Seeded synthetic inputs for the five BASELINE.json configs.

Test/bench input only: holds none of the method's arithmetic.  Thin ctypes
wrapper over ``gen/gen.c`` (counter-based RNG, so slabs are bit-identical to a
global generation).  Both the oracle harness and the CUDA path consume it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libgen.so")

POISSON3, RAND27, STOKES = 1, 2, 3
RHS_UNIFORM, RHS_LID, RHS_FORCE_NOISE, RHS_LID_NOISE, X_UNIFORM = 0, 1, 2, 3, 4
SEED = 200606052


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "gen.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
        os.path.getmtime(src), os.path.getmtime(os.path.join(_HERE, "gen.h"))
    ):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared",
             "-o", _SO, src, "-lm"]
        )
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        i64, i32, dbl, u64 = ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_uint64
        P = ctypes.c_void_p
        L.gen_nnzb.restype = i64
        L.gen_nnzb.argtypes = [i32, i32, i64, i64]
        L.gen_matrix.restype = i32
        L.gen_matrix.argtypes = [i32, i32, i32, i64, i64, P, P, P]
        L.gen_rhs.restype = i32
        L.gen_rhs.argtypes = [i32, i32, i32, i64, i64, P]
        L.gen_rand.restype = u64
        L.gen_rand.argtypes = [u64, u64]
        L.gen_u01.restype = dbl
        L.gen_u01.argtypes = [u64, u64]
        L.gen_n01.restype = dbl
        L.gen_n01.argtypes = [u64, u64]
        L.gen_uni.restype = dbl
        L.gen_uni.argtypes = [u64, u64, dbl, dbl]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def block_size(kind: int, b: int | None = None) -> int:
    return {POISSON3: 3, STOKES: 4}.get(kind, b if b is not None else 4)


def matrix(kind: int, n: int, b: int | None = None, row_begin: int = 0, row_end: int | None = None):
    """Return (ptr int32, col int32 [global ids], val float64 [nnzb, b, b]) for block rows
    [row_begin, row_end) of the n^3 grid."""
    b = block_size(kind, b)
    if row_end is None:
        row_end = n ** 3
    L = lib()
    nnzb = L.gen_nnzb(kind, n, row_begin, row_end)
    ptr = np.empty(row_end - row_begin + 1, dtype=np.int32)
    col = np.empty(nnzb, dtype=np.int32)
    val = np.empty((nnzb, b, b), dtype=np.float64)
    rc = L.gen_matrix(kind, n, b, row_begin, row_end, _p(ptr), _p(col), _p(val))
    if rc != 0:
        raise ValueError(f"gen_matrix({kind}, n={n}, b={b}) rejected its arguments")
    return ptr, col, val


def rhs(rhs_kind: int, n: int, b: int, row_begin: int = 0, row_end: int | None = None) -> np.ndarray:
    if row_end is None:
        row_end = n ** 3
    out = np.empty((row_end - row_begin) * b, dtype=np.float64)
    if lib().gen_rhs(rhs_kind, n, b, row_begin, row_end, _p(out)) != 0:
        raise ValueError("gen_rhs rejected its arguments")
    return out


def n01(stream: int, idx: int) -> float:
    return lib().gen_n01(stream, idx)


def u01(stream: int, idx: int) -> float:
    return lib().gen_u01(stream, idx)


# --- the five BASELINE.json configs, as (matrix kind, n, b, rhs kind, solver set-up) ---------
CONFIGS = {
    1: dict(kind=POISSON3, n=16, b=3, rhs=RHS_UNIFORM, solver="cg", precond="amg", hier="f64"),
    2: dict(kind=RAND27, n=128, b=4, rhs=X_UNIFORM, solver=None, precond=None, hier=None),
    3: dict(kind=STOKES, n=64, b=4, rhs=RHS_LID, solver="bicgstab", precond="amg", hier="f32"),
    4: dict(kind=STOKES, n=128, b=4, rhs=RHS_FORCE_NOISE, solver="gmres", precond="schur", hier="f32"),
    5: dict(kind=STOKES, n=256, b=4, rhs=RHS_LID_NOISE, solver="gmres", precond="schur", hier="f32"),
}
