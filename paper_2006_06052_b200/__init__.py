"""B200-native solve phase of the AMG-preconditioned Krylov solver for Stokes
saddle-point systems (Demidov, Mu & Wang, arXiv 2006.06052).

Thin ctypes binding over the C ABI in ``include/amg.h`` (``libamgb200.so``, built
for sm_100a by ``build.py``).  Argument marshalling only: every step of the
solve runs in the library's CUDA kernels.  PyTorch supplies device memory and
streams.  There is no CPU fallback: if the shared library is missing this module
raises at import time.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(HERE, "libamgb200.so")

# status codes / enums (include/amg.h)
OK, NOT_CONVERGED = 0, 1
EINVAL, EDIM, EZERODIAG, ESINGULAR_BLOCK, EINDEX_OVERFLOW, EBREAKDOWN, ECUDA, ENCCL, ENOMEM = (
    -1, -2, -3, -4, -5, -6, -7, -8, -9)
F64, F32 = 0, 1
CG, BICGSTAB, GMRES, IDRS = 0, 1, 2, 3
PC_AMG, PC_SCHUR, PC_NONE = 0, 1, 2
SPAI0, JACOBI, ILU0, ILUT = 0, 1, 2, 3
SA, PLAIN_AGG = 0, 1  # coarsening


class AmgError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: {status_string(status)} ({status}) {last_error()}")


class amg_bsr(ctypes.Structure):
    _fields_ = [("n_block_rows", ctypes.c_int32), ("n_block_cols", ctypes.c_int32),
                ("block_size", ctypes.c_int32), ("_pad", ctypes.c_int32), ("nnzb", ctypes.c_int64),
                ("row_ptr", ctypes.c_void_p), ("col_idx", ctypes.c_void_p), ("values", ctypes.c_void_p),
                ("dtype", ctypes.c_int32), ("_pad2", ctypes.c_int32)]


class amg_params(ctypes.Structure):
    _fields_ = [("solver", ctypes.c_int32), ("gmres_m", ctypes.c_int32), ("precond", ctypes.c_int32),
                ("maxiter", ctypes.c_int32), ("hier_dtype", ctypes.c_int32),
                ("vcycle_vec_dtype", ctypes.c_int32), ("smoother", ctypes.c_int32),
                ("coarse_enough", ctypes.c_int32), ("jacobi_omega", ctypes.c_double),
                ("sa_omega", ctypes.c_double), ("eps_strong", ctypes.c_double),
                ("max_levels", ctypes.c_int32), ("npre", ctypes.c_int32), ("npost", ctypes.c_int32),
                ("schur_p_component", ctypes.c_int32), ("use_graphs", ctypes.c_int32),
                ("idrs_s", ctypes.c_int32), ("idrs_seed", ctypes.c_int32), ("schur_u_scalar", ctypes.c_int32),
                ("coarsening", ctypes.c_int32), ("schur_shat", ctypes.c_int32), ("over_interp", ctypes.c_double),
                ("ilu_sweeps", ctypes.c_int32), ("gmres_ortho", ctypes.c_int32),
                ("fused_presmooth", ctypes.c_int32), ("ilut_p", ctypes.c_int32), ("ilut_tau", ctypes.c_double)]


class amg_report(ctypes.Structure):
    _fields_ = [("iters", ctypes.c_int32), ("converged", ctypes.c_int32), ("levels", ctypes.c_int32),
                ("restarts", ctypes.c_int32), ("relres_true", ctypes.c_double), ("setup_s", ctypes.c_double),
                ("solve_s", ctypes.c_double), ("alg_bytes", ctypes.c_double)]


# every symbol include/amg.h declares (checked by tests/test_capi.py)
EXPORTS = ["amg_params_default", "amg_status_string", "amg_setup", "amg_solve", "amg_solve_host",
           "amg_apply_precond", "bsr_spmv", "amg_destroy", "amg_level_info", "amg_level_export",
           "amg_level_aggregates", "amg_schur_export", "amg_vcycle", "amg_device_bytes",
           "amg_comm_unique_id", "amg_comm_init", "amg_setup_dist", "amg_comm_destroy",
           "amg_kernel_launches", "amg_profile_begin", "amg_profile_end", "amg_last_error",
           "bsr_plan_create", "bsr_plan_spmv", "bsr_plan_destroy", "amg_csr_to_bsr", "amg_memory_report",
           "amg_local_group_create", "amg_local_group_destroy", "amg_comm_init_local", "amg_setup_pmask",
           "amg_solve_counters", "amg_setup_dist_pmask", "amg_comm_init_host"]

_lib = None


def lib():
    """Load libamgb200.so (fails loudly when the CUDA library was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(SO_PATH):
            raise ImportError(f"{SO_PATH} missing: run `python -m paper_2006_06052_b200.build` "
                              "(no CPU fallback exists)")
        L = ctypes.CDLL(SO_PATH)
        P, i32, i64, dbl = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
        sig = {
            "amg_params_default": (i32, [P]),
            "amg_status_string": (ctypes.c_char_p, [i32]),
            "amg_last_error": (ctypes.c_char_p, []),
            "amg_setup": (i32, [P, P, P, P]),
            "amg_setup_pmask": (i32, [P, P, P, P, P]),
            "amg_solve": (i32, [P, P, P, dbl, P, P]),
            "amg_solve_host": (i32, [P, P, P, dbl, P, P]),
            "amg_apply_precond": (i32, [P, P, P, P]),
            "bsr_spmv": (i32, [P, dbl, P, i32, dbl, P, i32, P]),
            "amg_destroy": (None, [P]),
            "amg_level_info": (i32, [P, i32, P]),
            "amg_level_export": (i32, [P, i32, i32, P, P, P]),
            "amg_level_aggregates": (i32, [P, i32, P]),
            "amg_schur_export": (i32, [P, P, P]),
            "amg_vcycle": (i32, [P, P, P, P]),
            "amg_device_bytes": (i64, [P]),
            "amg_memory_report": (i32, [P, P, i32]),
            "amg_solve_counters": (i32, [P, P, i32]),
            "amg_comm_unique_id": (i32, [P]),
            "amg_comm_init": (i32, [P, i32, i32, P]),
            "amg_setup_dist": (i32, [P, i64, i64, P, P, P, P]),
            "amg_setup_dist_pmask": (i32, [P, P, i64, i64, P, P, P, P]),
            "amg_comm_init_host": (i32, [P, i32, i32, i32, P]),
            "amg_comm_destroy": (None, [P]),
            "amg_kernel_launches": (i64, []),
            "amg_local_group_create": (i32, [i32, P]),
            "amg_local_group_destroy": (None, [P]),
            "amg_comm_init_local": (i32, [P, i32, P]),
            "bsr_plan_create": (i32, [P, P, P]),
            "bsr_plan_spmv": (i32, [P, dbl, P, i32, dbl, P, i32, P]),
            "bsr_plan_destroy": (None, [P]),
            "amg_profile_begin": (i32, []),
            "amg_profile_end": (i64, [P, i64]),
            "amg_csr_to_bsr": (i32, [i32, i32, i32, i64, P, P, P, i32, P, P, P, P, P]),
        }
        for name, (res, args) in sig.items():
            if not hasattr(L, name):
                continue  # tests/test_capi.py checks that every declared symbol exists
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def kernel_launches() -> int:
    """Library kernels launched by this process so far."""
    return int(lib().amg_kernel_launches())


def profile_begin():
    _check(lib().amg_profile_begin(), "amg_profile_begin")


def profile_end() -> list:
    """Per-(kernel, bytes/launch) CUDA-event timings recorded since profile_begin()."""
    import json
    cap = 1 << 22
    buf = ctypes.create_string_buffer(cap)
    n = lib().amg_profile_end(buf, cap)
    if n >= cap:
        raise RuntimeError("profile record larger than the buffer")
    return json.loads(buf.value.decode())


def status_string(status: int) -> str:
    return lib().amg_status_string(status).decode()


def last_error() -> str:
    return lib().amg_last_error().decode()


def _check(rc: int, where: str, allow=(OK,)):
    if rc not in allow:
        raise AmgError(rc, where)
    return rc


def _torch():
    import torch
    return torch


def _stream_ptr(stream=None):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _dt(t) -> int:
    torch = _torch()
    if t.dtype == torch.float64:
        return F64
    if t.dtype == torch.float32:
        return F32
    raise TypeError(f"unsupported dtype {t.dtype}")


class BSR:
    """Device BSR matrix: int32 row_ptr [n+1], int32 col [nnzb], values [nnzb, b, b]
    (fp32 or fp64), row-major blocks."""

    def __init__(self, row_ptr, col, values, n_block_cols=None):
        self.row_ptr, self.col, self.values = row_ptr, col, values
        self.n = row_ptr.numel() - 1
        self.b = values.shape[-1]
        self.m = self.n if n_block_cols is None else n_block_cols

    @classmethod
    def from_numpy(cls, ptr, col, val, device="cuda", dtype=None, n_block_cols=None):
        torch = _torch()
        v = torch.as_tensor(val)
        if dtype is not None:
            v = v.to(dtype)
        return cls(torch.as_tensor(ptr, dtype=torch.int32).to(device),
                   torch.as_tensor(col, dtype=torch.int32).to(device), v.to(device).contiguous(),
                   n_block_cols)

    def desc(self) -> amg_bsr:
        d = amg_bsr()
        d.n_block_rows, d.n_block_cols, d.block_size = self.n, self.m, self.b
        d.nnzb = self.col.numel()
        d.row_ptr, d.col_idx, d.values = self.row_ptr.data_ptr(), self.col.data_ptr(), self.values.data_ptr()
        d.dtype = _dt(self.values)
        return d


def bsr_spmv(A: BSR, x, y, alpha: float = 1.0, beta: float = 0.0, stream=None):
    """y = alpha A x + beta y on the device (fp64 accumulation)."""
    d = A.desc()
    _check(lib().bsr_spmv(ctypes.byref(d), alpha, ctypes.c_void_p(x.data_ptr()), _dt(x), beta,
                          ctypes.c_void_p(y.data_ptr()), _dt(y), _stream_ptr(stream)), "bsr_spmv")
    return y


def csr_to_bsr(n: int, m: int, b: int, ptr, col, val, stream=None):
    """amg_csr_to_bsr: scalar CSR (device tensors) -> BSR (ptr, col, val[nnzb, b, b])."""
    import torch
    dt = _dt(val)
    nnzb = ctypes.c_int64()
    nnz = int(col.numel())
    args = (n, m, b, nnz, ctypes.c_void_p(ptr.data_ptr()), ctypes.c_void_p(col.data_ptr() if nnz else 0),
            ctypes.c_void_p(val.data_ptr() if nnz else 0), dt)
    _check(lib().amg_csr_to_bsr(*args, None, None, None, ctypes.byref(nnzb), _stream_ptr(stream)), "amg_csr_to_bsr")
    nb = nnzb.value
    bptr = torch.zeros(n // b + 1, dtype=torch.int32, device=ptr.device)
    bcol = torch.zeros(max(nb, 1), dtype=torch.int32, device=ptr.device)
    bval = torch.zeros((max(nb, 1), b, b), dtype=val.dtype, device=ptr.device)
    _check(lib().amg_csr_to_bsr(*args, ctypes.c_void_p(bptr.data_ptr()), ctypes.c_void_p(bcol.data_ptr()),
                                ctypes.c_void_p(bval.data_ptr()), ctypes.byref(nnzb), _stream_ptr(stream)),
           "amg_csr_to_bsr")
    return bptr, bcol[:nb], bval[:nb]


class SpmvPlan:
    """bsr_plan_create / bsr_plan_spmv: repeated products with A on the kernel the plan picks
    (interleaved row-per-lane or sliced copy for long rows, owned by the plan; A's tensors must
    stay alive and unchanged)."""

    def __init__(self, A: BSR, stream=None):
        self.A = A
        self.d = A.desc()
        h = ctypes.c_void_p()
        _check(lib().bsr_plan_create(ctypes.byref(self.d), _stream_ptr(stream), ctypes.byref(h)), "bsr_plan_create")
        self.h = h

    def __call__(self, x, y, alpha: float = 1.0, beta: float = 0.0, stream=None):
        _check(lib().bsr_plan_spmv(self.h, alpha, ctypes.c_void_p(x.data_ptr()), _dt(x), beta,
                                   ctypes.c_void_p(y.data_ptr()), _dt(y), _stream_ptr(stream)), "bsr_plan_spmv")
        return y

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.bsr_plan_destroy(self.h)
            self.h = None


def default_params(**kw) -> amg_params:
    p = amg_params()
    _check(lib().amg_params_default(ctypes.byref(p)), "amg_params_default")
    for k, v in kw.items():
        if not hasattr(p, k):
            raise AttributeError(k)
        setattr(p, k, v)
    return p


@dataclass
class Report:
    status: int
    iters: int
    converged: bool
    levels: int
    restarts: int
    relres_true: float
    setup_s: float
    solve_s: float
    alg_bytes: float


class Solver:
    """amg_setup / amg_solve on a device BSR matrix (Listing 3: ``Solver S(A, prm)``)."""

    def __init__(self, A: BSR, params: amg_params | None = None, stream=None, comm=None,
                 row_begin: int = 0, n_global: int | None = None, pmask=None, **kw):
        """pmask: optional device uint8 tensor [n*b] (non-zero = pressure unknown) -> amg_setup_pmask
        (with comm: this rank's rows -> amg_setup_dist_pmask)."""
        self.params = params if params is not None else default_params(**kw)
        self.A = A
        self.comm = comm  # the handle keeps the communicator's pointer: it must outlive the solver
        d = A.desc()
        h = ctypes.c_void_p()
        self.n_pressure = None
        if pmask is not None and comm is not None:  # this rank's rows of the mask (R27)
            rc = lib().amg_setup_dist_pmask(ctypes.byref(d), ctypes.c_void_p(pmask.data_ptr()), row_begin,
                                            A.m if n_global is None else n_global, comm.h, ctypes.byref(self.params),
                                            _stream_ptr(stream), ctypes.byref(h))
            self.n_pressure = int((pmask != 0).sum().item())
        elif pmask is not None:
            rc = lib().amg_setup_pmask(ctypes.byref(d), ctypes.c_void_p(pmask.data_ptr()), ctypes.byref(self.params),
                                       _stream_ptr(stream), ctypes.byref(h))
            self.n_pressure = int((pmask != 0).sum().item())
        elif comm is None:
            rc = lib().amg_setup(ctypes.byref(d), ctypes.byref(self.params), _stream_ptr(stream), ctypes.byref(h))
        else:
            rc = lib().amg_setup_dist(ctypes.byref(d), row_begin, A.m if n_global is None else n_global,
                                      comm.h, ctypes.byref(self.params), _stream_ptr(stream), ctypes.byref(h))
        _check(rc, "amg_setup")
        self.h = h
        self.setup_s = None

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.amg_destroy(self.h)
            self.h = None

    def solve(self, b, x, rtol: float = 1e-8, stream=None, allow_not_converged=True) -> Report:
        rep = amg_report()
        rc = lib().amg_solve(self.h, ctypes.c_void_p(b.data_ptr()), ctypes.c_void_p(x.data_ptr()), rtol,
                             _stream_ptr(stream), ctypes.byref(rep))
        _check(rc, "amg_solve", (OK, NOT_CONVERGED) if allow_not_converged else (OK,))
        return Report(rc, rep.iters, bool(rep.converged), rep.levels, rep.restarts, rep.relres_true,
                      rep.setup_s, rep.solve_s, rep.alg_bytes)

    def solve_host(self, b, x, rtol: float = 1e-8, stream=None) -> Report:
        """b, x: host (CPU) fp64 tensors; copies happen inside the C-ABI call."""
        rep = amg_report()
        rc = lib().amg_solve_host(self.h, ctypes.c_void_p(b.data_ptr()), ctypes.c_void_p(x.data_ptr()), rtol,
                                  _stream_ptr(stream), ctypes.byref(rep))
        _check(rc, "amg_solve_host", (OK, NOT_CONVERGED))
        return Report(rc, rep.iters, bool(rep.converged), rep.levels, rep.restarts, rep.relres_true,
                      rep.setup_s, rep.solve_s, rep.alg_bytes)

    def apply_precond(self, r, z, stream=None):
        _check(lib().amg_apply_precond(self.h, ctypes.c_void_p(r.data_ptr()), ctypes.c_void_p(z.data_ptr()),
                                       _stream_ptr(stream)), "amg_apply_precond")
        return z

    def vcycle(self, f, x, stream=None):
        _check(lib().amg_vcycle(self.h, ctypes.c_void_p(f.data_ptr()), ctypes.c_void_p(x.data_ptr()),
                                _stream_ptr(stream)), "amg_vcycle")
        return x

    def level_info(self, level: int):
        import numpy as np
        out = np.zeros(5, dtype=np.int64)
        _check(lib().amg_level_info(self.h, level, out.ctypes.data_as(ctypes.c_void_p)), "amg_level_info")
        return tuple(int(v) for v in out)

    @property
    def levels(self) -> int:
        n = 0
        while lib().amg_level_info(self.h, n, (ctypes.c_int64 * 5)()) == OK:
            n += 1
        return n

    def level_export(self, level: int, which: int):
        """which 0/1/2: (ptr, col, val[nnz,b,b]) of A_l/P_l/R_l; 3: M_l [n,b,b] (fp64 host numpy);
        4/5: the ILU strictly lower / upper factors (AMG_ILU0 / AMG_ILUT)."""
        import numpy as np
        n, b, nnzA, nnzP, nc = self.level_info(level)
        if which == 3:
            val = np.zeros((n, b, b))
            _check(lib().amg_level_export(self.h, level, 3, None, None, val.ctypes.data_as(ctypes.c_void_p)),
                   "amg_level_export")
            return val
        rows = {0: n, 1: n, 2: nc, 4: n, 5: n}[which]
        nnz = nnzA if which in (0, 4, 5) else nnzP  # ILU(0) factors: at most nnz(A) - n blocks
        if which in (4, 5) and self.params.smoother == ILUT:
            nnz += self.params.ilut_p * n  # ILUT: + p fill blocks per row on each side
        ptr = np.zeros(rows + 1, dtype=np.int32)
        col = np.zeros(max(nnz, 1), dtype=np.int32)
        val = np.zeros((max(nnz, 1), b, b))
        _check(lib().amg_level_export(self.h, level, which, ptr.ctypes.data_as(ctypes.c_void_p),
                                      col.ctypes.data_as(ctypes.c_void_p), val.ctypes.data_as(ctypes.c_void_p)),
               "amg_level_export")
        nnz = int(ptr[-1])
        return ptr, col[:nnz], val[:nnz]

    def level_aggregates(self, level: int):
        import numpy as np
        n = self.level_info(level)[0]
        agg = np.zeros(n, dtype=np.int32)
        _check(lib().amg_level_aggregates(self.h, level, agg.ctypes.data_as(ctypes.c_void_p)),
               "amg_level_aggregates")
        return agg

    def schur_export(self):
        import numpy as np
        n = self.A.n if self.n_pressure is None else self.n_pressure
        d, m = np.zeros(n), np.zeros(n)
        _check(lib().amg_schur_export(self.h, d.ctypes.data_as(ctypes.c_void_p), m.ctypes.data_as(ctypes.c_void_p)),
               "amg_schur_export")
        return d, m

    def memory_report(self) -> dict:
        """amg_memory_report: device bytes per component."""
        import numpy as np
        out = np.zeros(8, dtype=np.int64)
        _check(lib().amg_memory_report(self.h, out.ctypes.data_as(ctypes.c_void_p), 8), "amg_memory_report")
        keys = ["outer_A", "hierarchy", "sliced_copies", "smoothers", "schur", "coarse_inverse", "krylov", "total"]
        return dict(zip(keys, (int(v) for v in out)))

    def counters(self) -> dict:
        """amg_solve_counters: GMRES reorthogonalisation passes taken, CUDA graphs built."""
        import numpy as np
        out = np.zeros(2, dtype=np.int64)
        _check(lib().amg_solve_counters(self.h, out.ctypes.data_as(ctypes.c_void_p), 2), "amg_solve_counters")
        return {"reorth_passes": int(out[0]), "graphs": int(out[1])}

    @property
    def device_bytes(self) -> int:
        return int(lib().amg_device_bytes(self.h))


def broadcast_unique_id(rank: int, nranks: int, pg=None, make=None) -> bytes:
    """Rank 0 creates the 128-byte NCCL unique id (amg_comm_unique_id), torch.distributed
    broadcasts it (any backend: nccl, or gloo on CPU)."""
    if rank == 0:
        if make is not None:
            raw = make()
        else:
            uid = (ctypes.c_ubyte * 128)()
            _check(lib().amg_comm_unique_id(uid), "amg_comm_unique_id")
            raw = bytes(uid)
    else:
        raw = None
    if nranks > 1:
        import torch.distributed as dist
        obj = [raw]
        dist.broadcast_object_list(obj, src=0, group=pg)
        raw = obj[0]
    assert isinstance(raw, bytes) and len(raw) == 128
    return raw


def slab_bounds(n_rows: int, nranks: int):
    """Contiguous block-row slabs (z-slabs for the x-fastest grid ordering)."""
    return [r * n_rows // nranks for r in range(nranks + 1)]


class LocalGroup:
    """amg_local_group_create: P ranks as P threads of this process on one device."""

    def __init__(self, nranks: int):
        h = ctypes.c_void_p()
        _check(lib().amg_local_group_create(nranks, ctypes.byref(h)), "amg_local_group_create")
        self.h = h
        self.nranks = nranks

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.amg_local_group_destroy(self.h)
            self.h = None


_AR = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.c_int32)
_AG = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64), ctypes.c_int32,
                       ctypes.POINTER(ctypes.c_int64))
_EX = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32),
                       ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_int64), ctypes.c_int32,
                       ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_int64))
_BA = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p)


class amg_host_comm_ops(ctypes.Structure):
    _fields_ = [("ctx", ctypes.c_void_p), ("allreduce_sum", _AR), ("allgather_i64", _AG), ("exchange", _EX),
                ("barrier", _BA)]


def _host_ops(pg=None):
    """amg_host_comm_ops over a torch.distributed (CPU / gloo) process group: marshalling only
    -- every buffer is a host array the library owns for the duration of the call."""
    import numpy as np
    import torch
    import torch.distributed as dist

    def guard(fn):
        def run(*a):
            try:
                fn(*a)
                return 0
            except Exception:  # reported as AMG_ENCCL by the library
                return 1
        return run

    def allreduce(_, vals, n):
        t = torch.from_numpy(np.ctypeslib.as_array(vals, (n,)))
        dist.all_reduce(t, group=pg)

    def allgather(_, mine, n_each, out):
        world = dist.get_world_size(pg)
        src = torch.from_numpy(np.ctypeslib.as_array(mine, (n_each,)).copy())
        dst = torch.from_numpy(np.ctypeslib.as_array(out, (world * n_each,)))
        dist.all_gather(list(dst.view(world, n_each).unbind(0)), src, group=pg)

    def as_bytes(ptr, n):
        return torch.from_numpy(np.ctypeslib.as_array(ctypes.cast(ptr, ctypes.POINTER(ctypes.c_uint8)), (max(n, 1),)))

    def exchange(_, ns, sp, sb, sz, nr, rp, rb, rz):
        reqs = [dist.isend(as_bytes(sb[i], sz[i])[:sz[i]], sp[i], group=pg) for i in range(ns) if sz[i]]
        reqs += [dist.irecv(as_bytes(rb[i], rz[i])[:rz[i]], rp[i], group=pg) for i in range(nr) if rz[i]]
        for r in reqs:
            r.wait()

    def barrier(_):
        dist.barrier(group=pg)

    cbs = (_AR(guard(allreduce)), _AG(guard(allgather)), _EX(guard(exchange)), _BA(guard(barrier)))
    ops = amg_host_comm_ops(None, *cbs)
    ops._keep = cbs  # the C function pointers live as long as these objects
    return ops


class Comm:
    """NCCL communicator for amg_setup_dist (one process per GPU); ``Comm.local(group, rank)``
    the thread-emulated one; ``Comm.host(pg)`` the host-staged one over a torch.distributed
    (gloo) group -- separate processes, e.g. several on one GPU in the multi-process tests."""

    @classmethod
    def host(cls, pg=None, ordered: bool = False):
        """ordered: stream-ordered mode (copies + host functions on the stream, graph-capturable)."""
        import torch.distributed as dist
        self = cls.__new__(cls)
        self.ops = _host_ops(pg)  # the callbacks must outlive the communicator
        h = ctypes.c_void_p()
        _check(lib().amg_comm_init_host(ctypes.byref(self.ops), dist.get_world_size(pg), dist.get_rank(pg),
                                        1 if ordered else 0, ctypes.byref(h)), "amg_comm_init_host")
        self.h = h
        return self

    @classmethod
    def local(cls, group: "LocalGroup", rank: int):
        self = cls.__new__(cls)
        h = ctypes.c_void_p()
        _check(lib().amg_comm_init_local(group.h, rank, ctypes.byref(h)), "amg_comm_init_local")
        self.h = h
        self.group = group
        return self

    def __init__(self, rank: int, nranks: int, pg=None):
        raw = broadcast_unique_id(rank, nranks, pg)
        uid = (ctypes.c_ubyte * 128).from_buffer_copy(raw)
        h = ctypes.c_void_p()
        _check(lib().amg_comm_init(uid, nranks, rank, ctypes.byref(h)), "amg_comm_init")
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.amg_comm_destroy(self.h)
            self.h = None
