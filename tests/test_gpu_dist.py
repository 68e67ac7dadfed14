"""Distributed (row-slab) setup + solve through amg_setup_dist, on ONE device: P ranks
are P host threads with the thread-emulated communicator (amg_comm_init_local), the same
code path as NCCL except the transport.  Parity against the oracle in its multi-rank
mode (nparts = P: rank-local aggregation): aggregates per slab
bit-exact, every rank reports the same iteration count within +-2 of the oracle, and the
assembled solution has true relres <= 1e-8."""
import threading

import numpy as np
import pytest

import gen
import oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def amg():
    import paper_2006_06052_b200 as m
    assert torch.cuda.is_available()
    return m


def run_dist(amg, P, kind, n, rk, **kw):
    N = n ** 3
    ptr, col, val = gen.matrix(kind, n)
    b = val.shape[-1]
    bvec = gen.rhs(rk, n, b)
    group = amg.LocalGroup(P)
    out = [None] * P
    errs = []
    bounds = [r * N // P for r in range(P + 1)]

    def worker(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            r0, r1 = bounds[r], bounds[r + 1]
            lp, lc, lv = gen.matrix(kind, n, None, r0, r1)
            A = amg.BSR.from_numpy(lp, lc, lv, n_block_cols=N)
            comm = amg.Comm.local(group, r)
            S = amg.Solver(A, amg.default_params(**kw), stream=st, comm=comm, row_begin=r0, n_global=N)
            with torch.cuda.stream(st):
                bl = torch.as_tensor(bvec[r0 * b:r1 * b], device="cuda")
                x = torch.zeros_like(bl)
            rep = S.solve(bl, x, 1e-8, stream=st)
            st.synchronize()
            aggs = [S.level_aggregates(l) for l in range(S.levels - 1)]
            out[r] = (rep, x.cpu().numpy(), aggs, S)
        except Exception as e:  # surfaced below
            errs.append((r, repr(e)))

    th = [threading.Thread(target=worker, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    x = np.concatenate([o[1] for o in out])
    A = oracle.Mat.from_arrays(ptr, col, val)
    relres = np.linalg.norm(bvec - oracle.spmv(A, x)) / np.linalg.norm(bvec)
    return out, x, relres, (ptr, col, val, bvec)


CASES = [
    ("schur-gmres", gen.STOKES, 16, gen.RHS_LID_NOISE, dict(solver=2, precond=1)),
    ("amg-bicgstab", gen.STOKES, 16, gen.RHS_LID, dict(solver=1, precond=0)),
    ("amg-cg-f64", gen.POISSON3, 16, gen.RHS_UNIFORM, dict(solver=0, precond=0, hier_dtype=0, vcycle_vec_dtype=0,
                                                            coarse_enough=200)),
    ("schur-idrs", gen.STOKES, 16, gen.RHS_LID_NOISE, dict(solver=3, precond=1)),
    # slab-local ILU factors (reading R26): ILU(0) and the paper's ILUT U-solver smoother
    ("schur-ilu0-idrs", gen.STOKES, 16, gen.RHS_LID_NOISE, dict(solver=3, precond=1, smoother=2)),
    ("schur-ilut-gmres", gen.STOKES, 16, gen.RHS_LID_NOISE, dict(solver=2, precond=1, smoother=3)),
    ("amg-ilut-cg-f64", gen.POISSON3, 16, gen.RHS_UNIFORM, dict(solver=1, precond=0, smoother=3, hier_dtype=0,
                                                                 vcycle_vec_dtype=0, coarse_enough=200)),
    # the paper's V2: the U-solver hierarchy on the scalar expansion of A_u, slabs of 3 scalar rows per cell
    ("schur-v2-scalar-idrs", gen.STOKES, 16, gen.RHS_LID_NOISE, dict(solver=3, precond=1, schur_u_scalar=1)),
    ("schur-v2-scalar-f64", gen.STOKES, 12, gen.RHS_FORCE_NOISE, dict(solver=2, precond=1, schur_u_scalar=1,
                                                                      hier_dtype=0, vcycle_vec_dtype=0)),
    # SURVEY §8(f) #4 on several ranks: the explicit PETSc-style S_hat and plain aggregation
    ("schur-shat-full-gmres", gen.STOKES, 12, gen.RHS_LID_NOISE, dict(solver=2, precond=1, schur_shat=2)),
    ("schur-plain-agg-idrs", gen.STOKES, 16, gen.RHS_LID_NOISE, dict(solver=3, precond=1, coarsening=1)),
]


@pytest.mark.parametrize("P", [1, 2, 4, 8])
@pytest.mark.parametrize("name,kind,n,rk,kw", CASES, ids=[c[0] for c in CASES])
def test_dist_solve_parity(amg, P, name, kind, n, rk, kw):
    out, x, relres, (ptr, col, val, bvec) = run_dist(amg, P, kind, n, rk, **kw)
    its = {o[0].iters for o in out}
    assert len(its) == 1, its  # identical control flow on every rank
    assert all(o[0].converged for o in out)
    assert relres <= 1e-8
    ok = {"solver": "solver", "precond": "precond", "coarse_enough": "coarse_enough", "smoother": "smoother",
          "ilut_tau": "ilut_tau", "ilut_p": "ilut_p", "ilu_sweeps": "ilu_sweeps", "schur_u_scalar": "schur_u_scalar",
          "schur_shat": "schur_shat", "coarsening": "coarsening"}
    op = oracle.default_params(nparts=P, hier_f32=int(kw.get("hier_dtype", 1) == 1),
                               vec_f32=int(kw.get("vcycle_vec_dtype", 1) == 1),
                               **{ok[k]: v for k, v in kw.items() if k in ok})
    O = oracle.Solver(oracle.Mat.from_arrays(ptr, col, val), op)
    ro = O.solve(bvec, rtol=1e-8)
    assert abs(out[0][0].iters - ro.iters) <= 2, (out[0][0].iters, ro.iters)
    # slab-local aggregates equal the oracle's rank-local aggregation, level by level
    assert out[0][0].levels == O.levels
    for l in range(O.levels - 1):
        oagg = O.level_agg(l)
        if len(out[0][2][l]) == len(oagg) and P > 1:  # a replicated level: whole on every rank
            assert all(np.array_equal(o[2][l], out[0][2][l]) for o in out)
            agg = out[0][2][l]
        else:
            agg = np.concatenate([o[2][l] for o in out])
        assert np.array_equal(agg, oagg), f"level {l}"


def test_dist_p1_equals_single(amg):
    n = 12
    ptr, col, val = gen.matrix(gen.STOKES, n)
    bvec = gen.rhs(gen.RHS_LID_NOISE, n, 4)
    S = amg.Solver(amg.BSR.from_numpy(ptr, col, val), amg.default_params(solver=2, precond=1))
    x1 = torch.zeros(len(bvec), dtype=torch.float64, device="cuda")
    r1 = S.solve(torch.as_tensor(bvec, device="cuda"), x1)
    out, x, relres, _ = run_dist(amg, 1, gen.STOKES, n, gen.RHS_LID_NOISE, solver=2, precond=1)
    assert out[0][0].iters == r1.iters
    assert np.array_equal(x, x1.cpu().numpy())


def test_nccl_communicator_single_rank(amg):
    # the NCCL communicator itself (ncclCommInitRank from amg_comm_unique_id) on one rank:
    # amg_setup_dist + solve through it equals the single-device solve
    n = 12
    ptr, col, val = gen.matrix(gen.STOKES, n)
    bvec = gen.rhs(gen.RHS_LID_NOISE, n, 4)
    N = n ** 3
    comm = amg.Comm(0, 1)
    A = amg.BSR.from_numpy(ptr, col, val, n_block_cols=N)
    S = amg.Solver(A, amg.default_params(solver=2, precond=1), comm=comm, row_begin=0, n_global=N)
    b = torch.as_tensor(bvec, device="cuda")
    x = torch.zeros_like(b)
    rep = S.solve(b, x, 1e-8)
    S1 = amg.Solver(amg.BSR.from_numpy(ptr, col, val), amg.default_params(solver=2, precond=1))
    x1 = torch.zeros_like(b)
    rep1 = S1.solve(b, x1, 1e-8)
    assert rep.converged and rep.iters == rep1.iters
    assert torch.allclose(x, x1, rtol=0, atol=1e-12 * float(x1.abs().max()))


@pytest.mark.parametrize("P", [2, 4, 8])
def test_replicated_coarse_levels_are_exact(amg, envvars, P):
    # levels below AMG_REPLICATE_ROWS block rows per rank are held whole on every rank (no
    # halos, one allgather of their right-hand side); the same arithmetic row by row as the
    # slab-distributed levels -> the same iterates
    runs = []
    for rep_rows in (0, 10 ** 9):  # 0: only the coarsest replicated; 1e9: every level >= 1
        envvars(AMG_REPLICATE_ROWS=rep_rows)
        out, x, relres, _ = run_dist(amg, P, gen.STOKES, 16, gen.RHS_LID_NOISE, solver=2, precond=1)
        assert relres <= 1e-8
        runs.append((x, out[0][0].iters))
    assert runs[0][1] == runs[1][1]
    assert np.array_equal(runs[0][0], runs[1][0])


def test_nccl_single_rank_graphs_bit_identical(amg):
    # graph capture under an NCCL communicator (the preconditioner apply replayed from a CUDA
    # graph, NCCL calls captured with the kernels): bit-identical to the eager apply
    n = 12
    ptr, col, val = gen.matrix(gen.STOKES, n)
    bvec = gen.rhs(gen.RHS_LID_NOISE, n, 4)
    N = n ** 3
    comm = amg.Comm(0, 1)
    xs = []
    for graphs in (0, 1):
        A = amg.BSR.from_numpy(ptr, col, val, n_block_cols=N)
        S = amg.Solver(A, amg.default_params(solver=2, precond=1, use_graphs=graphs), comm=comm, row_begin=0,
                       n_global=N)
        b = torch.as_tensor(bvec, device="cuda")
        x = torch.zeros_like(b)
        rep = S.solve(b, x, 1e-8)
        assert rep.converged
        assert (S.counters()["graphs"] >= 1) == bool(graphs)
        xs.append((x.cpu().numpy(), rep.iters))
        del S
    assert xs[0][1] == xs[1][1]
    assert np.array_equal(xs[0][0], xs[1][0])


def test_halo_overlap_is_exact(amg, envvars):
    # the interior rows computed while the exchange is in flight, then the boundary rows:
    # the same per-row arithmetic as exchange-then-compute -> bit-identical iterates
    runs = []
    for off in (False, True):
        if off:
            envvars(AMG_NO_OVERLAP=1)
        out, x, relres, _ = run_dist(amg, 2, gen.STOKES, 16, gen.RHS_LID_NOISE, solver=2, precond=1)
        runs.append((x, out[0][0].iters))
    assert runs[0][1] == runs[1][1]
    assert np.array_equal(runs[0][0], runs[1][0])


def test_halo_overlap_interleaved_copy_is_exact(amg, envvars):
    # the same with the interleaved row-per-lane copy on every fp32 level (whole 32-row
    # slices: the interior rounded inward), unsorted slices so row ranges apply
    envvars(AMG_SELLR_MIN_SLICES=1, AMG_SELL_NO_SORT=1)
    runs = []
    for off in (False, True):
        if off:
            envvars(AMG_NO_OVERLAP=1)
        out, x, relres, _ = run_dist(amg, 2, gen.STOKES, 16, gen.RHS_LID_NOISE, solver=2, precond=1)
        runs.append((x, out[0][0].iters))
    assert runs[0][1] == runs[1][1]
    assert np.array_equal(runs[0][0], runs[1][0])


def _dist_arrays(amg, P, ptr, col, val, bvec, mask, kw):
    """P thread-emulated ranks on row slabs of the given global BSR arrays, with the rows'
    slice of a scalar pressure mask (amg_setup_dist_pmask)."""
    n, b = len(ptr) - 1, val.shape[-1]
    group = amg.LocalGroup(P)
    bounds = [r * n // P for r in range(P + 1)]
    out, errs = [None] * P, []

    def worker(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            r0, r1 = bounds[r], bounds[r + 1]
            lp = (ptr[r0:r1 + 1] - ptr[r0]).astype(np.int32)
            lc, lv = col[ptr[r0]:ptr[r1]], val[ptr[r0]:ptr[r1]]
            A = amg.BSR.from_numpy(lp, lc, lv, n_block_cols=n)
            pm = torch.as_tensor(mask[r0 * b:r1 * b].astype(np.uint8), device="cuda")
            S = amg.Solver(A, amg.default_params(precond=1, **kw), stream=st, comm=amg.Comm.local(group, r),
                           row_begin=r0, n_global=n, pmask=pm)
            with torch.cuda.stream(st):
                bl = torch.as_tensor(bvec[r0 * b:r1 * b], device="cuda")
                x = torch.zeros_like(bl)
            rep = S.solve(bl, x, 1e-8, stream=st)
            st.synchronize()
            out[r] = (rep, x.cpu().numpy(), [S.level_aggregates(l) for l in range(S.levels - 1)])
        except Exception as e:  # surfaced below
            errs.append((r, repr(e)))

    th = [threading.Thread(target=worker, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    return out


def _cellwise_scrambled_stokes(n, seed=7):
    """4x4 Stokes blocks with the (u, v, w, p) order of every cell permuted at random: the
    pressure sits at a different component in each cell (a general mask on a block matrix
    whose slabs stay whole cells)."""
    ptr, col, val = gen.matrix(gen.STOKES, n)
    perm = np.array([np.random.default_rng(seed + i).permutation(4) for i in range(n ** 3)])
    rows = np.repeat(np.arange(n ** 3), np.diff(ptr))
    val2 = np.stack([val[k][np.ix_(perm[rows[k]], perm[col[k]])] for k in range(len(col))])
    mask = (perm == 3).ravel()
    return ptr, col, val2, mask


@pytest.mark.parametrize("P", [1, 2, 4])
@pytest.mark.parametrize("case", ["interleaved-f32-idrs", "cellwise-scrambled-f64-gmres"])
def test_dist_pmask_parity(amg, P, case):
    # reading R27: the general scalar pressure mask on P ranks -- each rank owns contiguous
    # ranges of the velocity and of the pressure unknowns, the scalar U-solver hierarchy is
    # slab-distributed by the velocity ranges; the oracle's P-slab pmask mode is the reference
    if case.startswith("interleaved"):
        n = 12
        ptr, col, val = gen.matrix(gen.STOKES, n)
        mask = np.arange(4 * n ** 3) % 4 == 3
        kw = dict(solver=3)
    else:
        ptr, col, val, mask = _cellwise_scrambled_stokes(8)
        kw = dict(solver=2, coarse_enough=100, hier_dtype=0, vcycle_vec_dtype=0)
    N = len(mask)
    bvec = np.random.default_rng(3).standard_normal(N)
    out = _dist_arrays(amg, P, ptr, col, val, bvec, mask, kw)
    its = {o[0].iters for o in out}
    assert len(its) == 1, its
    x = np.concatenate([o[1] for o in out])
    A = oracle.Mat.from_arrays(ptr, col, val)
    relres = np.linalg.norm(bvec - oracle.spmv(A, x)) / np.linalg.norm(bvec)
    assert all(o[0].converged for o in out) and relres <= 1e-8
    h32 = int(kw.get("hier_dtype", 1) == 1)
    O = oracle.Solver(A, oracle.default_params(nparts=P, precond=oracle.PC_SCHUR, solver=kw["solver"], hier_f32=h32,
                                               vec_f32=h32, coarse_enough=kw.get("coarse_enough", 3000)), pmask=mask)
    ro = O.solve(bvec, rtol=1e-8)
    assert abs(out[0][0].iters - ro.iters) <= 2, (out[0][0].iters, ro.iters)
    assert out[0][0].levels == O.levels
    for l in range(O.levels - 1):
        oagg = O.level_agg(l)
        agg = out[0][2][l] if (len(out[0][2][l]) == len(oagg) and P > 1) else np.concatenate([o[2][l] for o in out])
        assert np.array_equal(agg, oagg), f"level {l}"
