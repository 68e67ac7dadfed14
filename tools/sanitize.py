"""Reduced cfg 3 / 4 / 5 solves for compute-sanitizer (SURVEY.md §5 race detection):

  compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck} python tools/sanitize.py [case]

Cases: cfg3 (BiCGStab + monolithic SA-AMG, graphed step), cfg4 (FGMRES + Schur, Gram/Cholesky),
cfg5 (FGMRES + Schur with the fp32 shadow basis), idrs, dist2 (two thread-emulated ranks on
one device: the concurrent launches of the emulated ranks), spmv (every SpMV kernel variant
via the forced-copy switches).  Small grids: the tools slow kernels down by 10-1000x.
"""
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2006_06052_b200 as amg  # noqa: E402


def solve(kind, n, rk, **kw):
    ptr, col, val = gen.matrix(kind, n)
    b = torch.as_tensor(gen.rhs(rk, n, val.shape[-1]), device="cuda")
    S = amg.Solver(amg.BSR.from_numpy(ptr, col, val), amg.default_params(**kw))
    for _ in range(2):  # the second solve replays the cached graphs
        x = torch.zeros_like(b)
        rep = S.solve(b, x, 1e-8)
    torch.cuda.synchronize()
    print(kw, rep.iters, rep.converged, rep.relres_true, flush=True)
    assert rep.converged


def dist2(n=8):
    P, N = 2, n ** 3
    group = amg.LocalGroup(P)
    bvec = gen.rhs(gen.RHS_LID_NOISE, n, 4)
    bd = amg.slab_bounds(N, P)
    errs = []

    def w(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            lp, lc, lv = gen.matrix(gen.STOKES, n, None, bd[r], bd[r + 1])
            S = amg.Solver(amg.BSR.from_numpy(lp, lc, lv, n_block_cols=N), amg.default_params(solver=2, precond=1),
                           stream=st, comm=amg.Comm.local(group, r), row_begin=bd[r], n_global=N)
            with torch.cuda.stream(st):
                b = torch.as_tensor(bvec[bd[r] * 4:bd[r + 1] * 4], device="cuda")
                x = torch.zeros_like(b)
            rep = S.solve(b, x, 1e-8, stream=st)
            st.synchronize()
            assert rep.converged
        except Exception as e:
            errs.append(repr(e))

    th = [threading.Thread(target=w, args=(r,)) for r in range(P)]
    [t.start() for t in th]
    [t.join() for t in th]
    assert not errs, errs
    print("dist2 ok", flush=True)


CASES = {
    "cfg3": lambda: solve(gen.STOKES, 12, gen.RHS_LID, solver=1, precond=0),
    "cfg4": lambda: solve(gen.STOKES, 12, gen.RHS_FORCE_NOISE, solver=2, precond=1),
    "cfg5": lambda: solve(gen.STOKES, 12, gen.RHS_LID_NOISE, solver=2, precond=1, gmres_ortho=2),
    "cg": lambda: solve(gen.POISSON3, 10, gen.RHS_UNIFORM, solver=0, precond=0, hier_dtype=0, vcycle_vec_dtype=0,
                        coarse_enough=100),
    "idrs": lambda: solve(gen.STOKES, 10, gen.RHS_LID_NOISE, solver=3, precond=1),
    "dist2": dist2,
}

if __name__ == "__main__":
    torch.cuda.set_device(0)
    names = sys.argv[1:] or list(CASES)
    for c in names:
        CASES[c]()
