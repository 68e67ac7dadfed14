"""GPU setup / V-cycle / Schur / Krylov parity against the CPU oracle, through the C ABI.

Bars (BASELINE.json north_star): aggregates and sparsity patterns
bit-exact; level values bit-exact in fp64 (== after fp32 rounding for the fp32
hierarchy); V-cycle / preconditioner outputs norm-wise 1e-10 (fp64; the coarse
solve is an explicit Gauss-Jordan inverse on the GPU vs LU in the oracle) and 1e-5
(fp32); solves within +-2 iterations of the oracle with true relres <= 1e-8."""
import numpy as np
import pytest

import gen
import oracle
from conftest import random_bsr

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def amg():
    import paper_2006_06052_b200 as m
    assert torch.cuda.is_available()
    return m


ORC_OF = {"solver": "solver", "gmres_m": "gmres_m", "precond": "precond", "maxiter": "maxiter",
          "smoother": "smoother", "sa_omega": "sa_omega", "eps_strong": "eps_strong",
          "coarse_enough": "coarse_enough", "npre": "npre", "npost": "npost", "max_levels": "max_levels",
          "jacobi_omega": "jacobi_omega", "idrs_s": "idrs_s", "idrs_seed": "idrs_seed",
          "schur_u_scalar": "schur_u_scalar", "coarsening": "coarsening", "schur_shat": "schur_shat",
          "over_interp": "over_interp", "ilu_sweeps": "ilu_sweeps", "ilut_tau": "ilut_tau", "ilut_p": "ilut_p"}
# gmres_ortho is deliberately NOT forwarded: the oracle always runs its default CGS2
# (SURVEY.md C11), so every GPU GMRES case -- whatever orthogonalisation the GPU uses --
# is checked against the plain reading (VERDICT r01 "What's weak" #2).


def make_pair(amg, ptr, col, val, hier32=True, **kw):
    """Build the GPU solver and the oracle with the same parameters."""
    A = amg.BSR.from_numpy(ptr, col, val)
    gp = amg.default_params(hier_dtype=amg.F32 if hier32 else amg.F64,
                            vcycle_vec_dtype=amg.F32 if hier32 else amg.F64, **kw)
    S = amg.Solver(A, gp)
    op = oracle.default_params(hier_f32=int(hier32), vec_f32=int(hier32),
                               **{ORC_OF[k]: v for k, v in kw.items() if k in ORC_OF})
    O = oracle.Solver(oracle.Mat.from_arrays(ptr, col, val), op)
    return A, S, O


def r32(a):
    return a.astype(np.float32).astype(np.float64)


def relerr(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def check_hierarchy(S, O, hier32):
    assert S.levels == O.levels
    for l in range(O.levels):
        n, b, nnzA, nnzP, nc = S.level_info(l)
        oA = O.level_mat(l, 0)
        optr, ocol, oval = oA.to_arrays()
        ptr, col, val = S.level_export(l, 0)
        assert np.array_equal(ptr, optr) and np.array_equal(col, ocol), f"A pattern level {l}"
        assert np.array_equal(val, r32(oval) if hier32 else oval), f"A values level {l}"
        if l == O.levels - 1:
            break
        assert np.array_equal(S.level_aggregates(l), O.level_agg(l)), f"aggregates level {l}"
        for which in (1, 2):
            optr, ocol, oval = O.level_mat(l, which).to_arrays()
            ptr, col, val = S.level_export(l, which)
            assert np.array_equal(ptr, optr) and np.array_equal(col, ocol), f"pattern {which} level {l}"
            assert np.array_equal(val, r32(oval) if hier32 else oval), f"values {which} level {l}"
        M = S.level_export(l, 3)
        oM = O.level_M(l)
        assert np.array_equal(M, r32(oM) if hier32 else oM), f"smoother level {l}"
        for which in (4, 5):  # ILU factors (AMG_ILU0 / AMG_ILUT)
            oF = O.level_mat(l, which)
            if oF is None:
                continue
            optr, ocol, oval = oF.to_arrays()
            ptr, col, val = S.level_export(l, which)
            assert np.array_equal(ptr, optr) and np.array_equal(col, ocol), f"ILU pattern {which} level {l}"
            assert np.array_equal(val, r32(oval) if hier32 else oval), f"ILU values {which} level {l}"


CASES = [
    ("cfg1-16", gen.POISSON3, 16, dict(precond=0, solver=0), False),
    ("cfg3-16", gen.STOKES, 16, dict(precond=0, solver=1), True),
    ("cfg3-24", gen.STOKES, 24, dict(precond=0, solver=1), True),
    ("cfg4-16", gen.STOKES, 16, dict(precond=1, solver=2), True),
    ("poisson-lowce", gen.POISSON3, 10, dict(precond=0, solver=0, coarse_enough=40), False),
    ("stokes-lowce-f64", gen.STOKES, 10, dict(precond=1, solver=2, coarse_enough=40), False),
    # V2 of the paper's ladder: the U-solver hierarchy on the scalar expansion of A_u
    ("stokes-v2-scalar-f64", gen.STOKES, 10, dict(precond=1, solver=3, schur_u_scalar=1, coarse_enough=40), False),
    ("stokes-v2-scalar-16", gen.STOKES, 16, dict(precond=1, solver=3, schur_u_scalar=1), True),
    # plain aggregation (Listings V2-V4) and the S_hat variants
    ("plain-agg-poisson", gen.POISSON3, 10, dict(precond=0, solver=0, coarsening=1, coarse_enough=40), False),
    ("plain-agg-stokes-16", gen.STOKES, 16, dict(precond=1, solver=3, coarsening=1), True),
    ("plain-agg-alpha1-f64", gen.STOKES, 10, dict(precond=1, solver=2, coarsening=1, over_interp=1.0,
                                                  coarse_enough=40), False),
    ("shat-C-f64", gen.STOKES, 10, dict(precond=1, solver=2, schur_shat=0, coarse_enough=40), False),
    ("shat-full-f64", gen.STOKES, 12, dict(precond=1, solver=2, schur_shat=2, coarse_enough=40), False),
    ("shat-full-plain-16", gen.STOKES, 16, dict(precond=1, solver=3, schur_shat=2, coarsening=1), True),
    # block ILU(0) smoothing (R20); plain aggregation + ILU = the paper's V3/V4 U-solver shape
    ("ilu0-poisson-f64", gen.POISSON3, 10, dict(precond=0, solver=1, smoother=2, coarse_enough=40), False),
    ("ilu0-stokes-schur-16", gen.STOKES, 16, dict(precond=1, solver=3, smoother=2), True),
    ("ilu0-plain-agg-f64", gen.STOKES, 12, dict(precond=1, solver=3, smoother=2, coarsening=1, coarse_enough=40),
     False),
    ("ilu0-monolithic-4x4-16", gen.STOKES, 16, dict(precond=0, solver=1, smoother=2, ilu_sweeps=3), True),
    # block ILUT(tau, p) (reading R25): the paper's U-solver smoother, Listing V2 = plain aggregation + ILUT
    ("ilut-stokes-schur-16", gen.STOKES, 16, dict(precond=1, solver=3, smoother=3), True),
    ("ilut-plain-agg-f64", gen.STOKES, 12, dict(precond=1, solver=3, smoother=3, coarsening=1, coarse_enough=40),
     False),
    ("ilut-p0-tau0-poisson-f64", gen.POISSON3, 10, dict(precond=0, solver=1, smoother=3, ilut_p=0, ilut_tau=0.0,
                                                         coarse_enough=40), False),
    ("ilut-monolithic-4x4-16", gen.STOKES, 16, dict(precond=0, solver=1, smoother=3, ilut_p=4, ilut_tau=1e-3), True),
]


@pytest.mark.parametrize("name,kind,n,kw,h32", CASES, ids=[c[0] for c in CASES])
def test_hierarchy_bit_exact(amg, name, kind, n, kw, h32):
    ptr, col, val = gen.matrix(kind, n)
    A, S, O = make_pair(amg, ptr, col, val, hier32=h32, **kw)
    check_hierarchy(S, O, h32)
    if kw.get("precond") == 1:
        d, m = S.schur_export()
        od, om = O.schur_vectors()
        assert np.array_equal(d, od) and np.array_equal(m, om)


def test_hierarchy_random_matrices(amg, rng):
    for b in (1, 2, 3, 4):
        for trial in range(2):
            ptr, col, val = random_bsr(rng, 400, b, density=0.012, symmetric_pattern=(trial == 0), dom=6)
            for h32 in (False, True):
                A, S, O = make_pair(amg, ptr, col, val, hier32=h32, precond=0, coarse_enough=20 * b)
                check_hierarchy(S, O, h32)


def _weak_mix(rng, ptr, col, val, share=0.3, scale=1e-4):
    """Scale a random share of the off-diagonal block pairs by 1e-4 so that they are weak at
    eps = 1e-3 (GPU hierarchies with >= 10 % weak edges at level 0)."""
    val = val.copy()
    n = len(ptr) - 1
    pos = {(i, int(col[k])): k for i in range(n) for k in range(ptr[i], ptr[i + 1])}
    for (i, j), k in pos.items():
        if i < j and rng.random() < share:
            val[k] *= scale
            if (j, i) in pos and rng.random() < 0.8:
                val[pos[(j, i)]] *= scale
    return val


def _weak_share(S_or_O_strength, ptr, col):
    sp, sc = S_or_O_strength
    offd = sum(1 for i in range(len(ptr) - 1) for k in range(ptr[i], ptr[i + 1]) if col[k] != i)
    return 1.0 - len(sc) / offd


@pytest.mark.parametrize("b", [1, 2, 3, 4])
def test_hierarchy_weak_edges_random(amg, rng, b):
    # weak blocks exercise A_F lumping and the filtered D (k_filtered_diag, k_p_cand, k_p_fill)
    ptr, col, val = random_bsr(rng, 500, b, density=0.012, symmetric_pattern=True, dom=6)
    val = _weak_mix(rng, ptr, col, val)
    share = _weak_share(oracle.strength(oracle.Mat.from_arrays(ptr, col, val), 1e-3), ptr, col)
    assert share >= 0.1, share
    for h32 in (False, True):
        A, S, O = make_pair(amg, ptr, col, val, hier32=h32, precond=0, coarse_enough=20 * b)
        assert O.levels >= 3
        check_hierarchy(S, O, h32)


@pytest.mark.parametrize("kind,n,kw,h32", [
    (gen.STOKES, 12, dict(precond=1, solver=2, coarse_enough=40), False),
    (gen.STOKES, 16, dict(precond=1, solver=2), True),
    (gen.STOKES, 12, dict(precond=0, solver=1, coarse_enough=40), True),
    (gen.POISSON3, 12, dict(precond=0, solver=0, coarse_enough=40), False),
], ids=["schur-f64", "schur-f32", "mono-f32", "poisson-f64"])
def test_hierarchy_and_solve_weak_edges_stencil(amg, kind, n, kw, h32):
    rng = np.random.default_rng(17 + n)
    ptr, col, val = gen.matrix(kind, n)
    val = _weak_mix(rng, ptr, col, val, share=0.2)
    A, S, O = make_pair(amg, ptr, col, val, hier32=h32, **kw)
    check_hierarchy(S, O, h32)
    if kw.get("precond") == 1:
        d, m = S.schur_export()
        od, om = O.schur_vectors()
        assert np.array_equal(d, od) and np.array_equal(m, om)
    bvec = np.random.default_rng(5).uniform(-1, 1, len(val) * 0 + (len(ptr) - 1) * val.shape[-1])
    ro = O.solve(bvec, rtol=1e-8)
    x, rep = _solve(amg, S, bvec)
    true = np.linalg.norm(bvec - oracle.spmv(oracle.Mat.from_arrays(ptr, col, val), x)) / np.linalg.norm(bvec)
    assert ro.converged and rep.converged and true <= 1e-8 and abs(rep.iters - ro.iters) <= 2, (rep.iters, ro.iters)


def test_aggregation_pass2_hand_graph(amg):
    # the oracle pin's hand-built graph (tests/test_oracle_pins.py): pass-2 node 3 touches
    # aggregates 0 and 1 and must join its lowest-index assigned neighbour's (2 -> 1)
    n = 6
    Dn = 4.0 * np.eye(n)
    for i, j in [(0, 4), (0, 5), (1, 2), (2, 3), (3, 5)]:
        Dn[i, j] = Dn[j, i] = -1.0
    nz = [(i, j) for i in range(n) for j in range(n) if Dn[i, j] != 0]
    ptr = np.searchsorted([i for i, _ in nz], np.arange(n + 1)).astype(np.int32)
    col = np.array([j for _, j in nz], np.int32)
    val = np.array([Dn[i, j] for i, j in nz]).reshape(-1, 1, 1)
    A, S, O = make_pair(amg, ptr, col, val, hier32=False, precond=0, coarse_enough=2, max_levels=2)
    assert S.level_aggregates(0).tolist() == [0, 1, 1, 1, 0, 0]
    check_hierarchy(S, O, False)


def test_ilu0_random_matrices(amg, rng):
    # block ILU(0) factors bit-exact with the oracle for b = 1..4, fp64 and fp32 hierarchies
    for b in (1, 2, 3, 4):
        ptr, col, val = random_bsr(rng, 300, b, density=0.015, dom=6)
        for h32 in (False, True):
            A, S, O = make_pair(amg, ptr, col, val, hier32=h32, precond=0, solver=1, smoother=2,
                                coarse_enough=20 * b)
            check_hierarchy(S, O, h32)


@pytest.mark.parametrize("tau,p", [(1e-2, 2), (0.0, 0), (0.05, 1), (0.0, 40), (1e-3, 6)])
def test_ilut_random_matrices(amg, rng, tau, p):
    # block ILUT factors (patterns and fp64 values) bit-exact with the oracle for b = 1..4
    # (R25: the same elimination order, threshold and fill-ranking decisions in fp64)
    for b in (1, 2, 3, 4):
        ptr, col, val = random_bsr(rng, 300, b, density=0.015, dom=3 * b)
        for h32 in (False, True):
            A, S, O = make_pair(amg, ptr, col, val, hier32=h32, precond=0, solver=1, smoother=3, ilut_tau=tau,
                                ilut_p=p, coarse_enough=20 * b)
            check_hierarchy(S, O, h32)


def test_ilut_overflow_fails_cleanly(amg, rng):
    # a row beyond the factorisation's working-row capacity (512 blocks) fails the setup with
    # AMG_EINVAL -- and every row waiting on it is released (no hang)
    n, b = 700, 1
    rows = [np.arange(n)] + [np.array([0, i]) for i in range(1, n)]  # arrow matrix
    ptr = np.zeros(n + 1, np.int32)
    ptr[1:] = np.cumsum([len(r) for r in rows])
    col = np.concatenate(rows).astype(np.int32)
    val = rng.standard_normal((len(col), b, b)) * 0.1
    for i in range(n):
        val[ptr[i] + (0 if i == 0 else 1)] = 4.0
    A = amg.BSR.from_numpy(ptr, col, val)
    with pytest.raises(amg.AmgError) as e:
        amg.Solver(A, amg.default_params(precond=0, solver=1, smoother=3, hier_dtype=0, vcycle_vec_dtype=0,
                                         coarse_enough=10))
    assert "ILUT" in str(e.value) or "-1" in str(e.value)
    # the library is still usable afterwards
    S = amg.Solver(A, amg.default_params(precond=0, solver=1, hier_dtype=0, vcycle_vec_dtype=0, coarse_enough=10))
    assert S.levels >= 2


def test_ilut_stencil_levels(amg):
    # every level of a 3x3 SA hierarchy (7-point stencil rows, then aggregated rows with 20-60
    # blocks and their fill) factorised on the GPU equals the oracle's factorisation
    ptr, col, val = gen.matrix(gen.POISSON3, 16)
    for tau, p in ((1e-2, 2), (1e-4, 8)):
        A, S, O = make_pair(amg, ptr, col, val, hier32=False, precond=0, solver=0, smoother=3, ilut_tau=tau, ilut_p=p,
                            coarse_enough=100)
        assert S.levels >= 3
        check_hierarchy(S, O, False)


def test_smoother_jacobi_and_omega(amg):
    ptr, col, val = gen.matrix(gen.POISSON3, 10)
    A, S, O = make_pair(amg, ptr, col, val, hier32=False, precond=0, smoother=1, sa_omega=0.5,
                        coarse_enough=100)
    check_hierarchy(S, O, False)


@pytest.mark.parametrize("name,kind,n,kw,h32", CASES, ids=[c[0] for c in CASES])
def test_precond_parity(amg, rng, name, kind, n, kw, h32):
    ptr, col, val = gen.matrix(kind, n)
    A, S, O = make_pair(amg, ptr, col, val, hier32=h32, **kw)
    N = len(ptr) * 0 + (len(ptr) - 1) * val.shape[-1]
    for _ in range(2):
        r = rng.standard_normal(N)
        z = S.apply_precond(torch.as_tensor(r, device="cuda"), torch.zeros(N, dtype=torch.float64, device="cuda"))
        torch.cuda.synchronize()
        assert relerr(z.cpu().numpy(), O.precond(r)) <= (1e-5 if h32 else 1e-10)


def _solve(amg, S, bvec, rtol=1e-8):
    b = torch.as_tensor(bvec, device="cuda")
    x = torch.zeros_like(b)
    rep = S.solve(b, x, rtol)
    return x.cpu().numpy(), rep


SOLVE_CASES = [
    ("cfg1", gen.POISSON3, 16, gen.RHS_UNIFORM, dict(precond=0, solver=0), False),
    ("cfg1-f32", gen.POISSON3, 16, gen.RHS_UNIFORM, dict(precond=0, solver=0), True),
    ("cfg3-32", gen.STOKES, 32, gen.RHS_LID, dict(precond=0, solver=1), True),
    ("cfg4-16", gen.STOKES, 16, gen.RHS_FORCE_NOISE, dict(precond=1, solver=2), True),
    ("cfg4-32", gen.STOKES, 32, gen.RHS_FORCE_NOISE, dict(precond=1, solver=2), True),
    ("cfg5-24", gen.STOKES, 24, gen.RHS_LID_NOISE, dict(precond=1, solver=2), True),
    ("gmres-m10-f64", gen.STOKES, 12, gen.RHS_LID_NOISE, dict(precond=1, solver=2, gmres_m=10), False),
    # IDR(s): the paper's outer solver (Table 1), V4 = Schur PC + fp32 hierarchy
    ("idrs5-cfg4-16", gen.STOKES, 16, gen.RHS_FORCE_NOISE, dict(precond=1, solver=3), True),
    ("idrs5-cfg5-24", gen.STOKES, 24, gen.RHS_LID_NOISE, dict(precond=1, solver=3), True),
    ("idrs5-cfg3-16", gen.STOKES, 16, gen.RHS_LID, dict(precond=0, solver=3), True),
    ("idrs2-poisson-f64", gen.POISSON3, 12, gen.RHS_UNIFORM, dict(precond=0, solver=3, idrs_s=2), False),
    ("idrs8-stokes-f64", gen.STOKES, 10, gen.RHS_LID_NOISE, dict(precond=1, solver=3, idrs_s=8, idrs_seed=7), False),
    # the paper's ladder: V2 (scalar fp64 U-solver), V3 (3x3 fp64), V4 (3x3 fp32), IDR(5) outer
    ("ladder-v2", gen.STOKES, 16, gen.RHS_FORCE_NOISE, dict(precond=1, solver=3, schur_u_scalar=1), False),
    ("ladder-v3", gen.STOKES, 16, gen.RHS_FORCE_NOISE, dict(precond=1, solver=3), False),
    # plain aggregation + the S_hat variants
    ("plain-agg-idrs5-cfg4-16", gen.STOKES, 16, gen.RHS_FORCE_NOISE, dict(precond=1, solver=3, coarsening=1), True),
    ("plain-agg-cg-poisson", gen.POISSON3, 16, gen.RHS_UNIFORM, dict(precond=0, solver=0, coarsening=1), False),
    ("plain-agg-bicgstab-cfg3", gen.STOKES, 16, gen.RHS_LID, dict(precond=0, solver=1, coarsening=1), True),
    ("shat-full-gmres-cfg5-16", gen.STOKES, 16, gen.RHS_LID_NOISE, dict(precond=1, solver=2, schur_shat=2), True),
    ("shat-C-gmres-f64", gen.STOKES, 12, gen.RHS_FORCE_NOISE, dict(precond=1, solver=2, schur_shat=0), False),
    # block ILU(0) smoothing
    ("ilu0-idrs5-cfg4-16", gen.STOKES, 16, gen.RHS_FORCE_NOISE, dict(precond=1, solver=3, smoother=2), True),
    ("ilu0-plain-gmres-cfg5-16", gen.STOKES, 16, gen.RHS_LID_NOISE,
     dict(precond=1, solver=2, smoother=2, coarsening=1), True),
    ("ilu0-bicgstab-cfg3-16", gen.STOKES, 16, gen.RHS_LID, dict(precond=0, solver=1, smoother=2), True),
    ("ilu0-sweeps3-f64", gen.STOKES, 12, gen.RHS_FORCE_NOISE, dict(precond=1, solver=2, smoother=2, ilu_sweeps=3),
     False),
    # block ILUT (reading R25): Listing V2's U-solver (plain aggregation + ILUT) and SA + ILUT
    ("ilut-idrs5-cfg4-16", gen.STOKES, 16, gen.RHS_FORCE_NOISE, dict(precond=1, solver=3, smoother=3), True),
    ("ilut-plain-idrs5-cfg5-16", gen.STOKES, 16, gen.RHS_LID_NOISE, dict(precond=1, solver=3, smoother=3,
                                                                         coarsening=1), True),
    ("ilut-gmres-f64", gen.STOKES, 12, gen.RHS_FORCE_NOISE, dict(precond=1, solver=2, smoother=3, ilut_p=3,
                                                                  ilut_tau=3e-3), False),
    ("ilut-bicgstab-cfg3-16", gen.STOKES, 16, gen.RHS_LID, dict(precond=0, solver=1, smoother=3), True),
    # GPU orthogonalisation variants of flexible GMRES, each against the oracle's CGS2:
    # two-pass Gram/Cholesky (R22), its fp32-shadow first pass (R23) and the GPU's CGS2 (every
    # case above without gmres_ortho runs the GPU default, R28: the fp16-shadow first pass)
    ("gram-gmres-cfg4-16", gen.STOKES, 16, gen.RHS_FORCE_NOISE, dict(precond=1, solver=2, gmres_ortho=1), True),
    ("gram-gmres-cfg5-24", gen.STOKES, 24, gen.RHS_LID_NOISE, dict(precond=1, solver=2, gmres_ortho=1), True),
    ("gram-gmres-m10-f64", gen.STOKES, 12, gen.RHS_LID_NOISE, dict(precond=1, solver=2, gmres_m=10, gmres_ortho=1),
     False),
    ("gram-gmres-poisson", gen.POISSON3, 16, gen.RHS_UNIFORM, dict(precond=0, solver=2, gmres_ortho=1), False),
    ("cgs2-gmres-cfg4-16", gen.STOKES, 16, gen.RHS_FORCE_NOISE, dict(precond=1, solver=2, gmres_ortho=0), True),
    ("cgs2-gmres-cfg5-24", gen.STOKES, 24, gen.RHS_LID_NOISE, dict(precond=1, solver=2, gmres_ortho=0), True),
    ("cgs2-gmres-m10-f64", gen.STOKES, 12, gen.RHS_LID_NOISE, dict(precond=1, solver=2, gmres_m=10, gmres_ortho=0),
     False),
    ("f32-gmres-cfg4-16", gen.STOKES, 16, gen.RHS_FORCE_NOISE, dict(precond=1, solver=2, gmres_ortho=2), True),
    ("f32-gmres-cfg5-24", gen.STOKES, 24, gen.RHS_LID_NOISE, dict(precond=1, solver=2, gmres_ortho=2), True),
    ("f32-gmres-m10-f64", gen.STOKES, 12, gen.RHS_LID_NOISE, dict(precond=1, solver=2, gmres_m=10, gmres_ortho=2),
     False),
    ("f32-gmres-poisson", gen.POISSON3, 16, gen.RHS_UNIFORM, dict(precond=0, solver=2, gmres_ortho=2), False),
]


@pytest.mark.parametrize("name,kind,n,rk,kw,h32", SOLVE_CASES, ids=[c[0] for c in SOLVE_CASES])
def test_solve_parity(amg, name, kind, n, rk, kw, h32):
    ptr, col, val = gen.matrix(kind, n)
    bvec = gen.rhs(rk, n, val.shape[-1])
    A, S, O = make_pair(amg, ptr, col, val, hier32=h32, **kw)
    ro = O.solve(bvec, rtol=1e-8)
    x, rep = _solve(amg, S, bvec)
    assert rep.status == amg.OK and rep.converged
    assert rep.relres_true <= 1e-8
    # independent check of the reported relres with the oracle's SpMV
    true = np.linalg.norm(bvec - oracle.spmv(oracle.Mat.from_arrays(ptr, col, val), x)) / np.linalg.norm(bvec)
    assert true <= 1e-8 and abs(true - rep.relres_true) <= 1e-10
    assert abs(rep.iters - ro.iters) <= 2, (rep.iters, ro.iters)
    assert rep.levels == O.levels


def test_cfg3_full_size(amg):
    # BASELINE configs[2] at its full size (64^3, 1.05M unknowns)
    n = 64
    ptr, col, val = gen.matrix(gen.STOKES, n)
    bvec = gen.rhs(gen.RHS_LID, n, 4)
    A, S, O = make_pair(amg, ptr, col, val, hier32=True, precond=0, solver=1)
    check_hierarchy(S, O, True)
    ro = O.solve(bvec, rtol=1e-8)
    x, rep = _solve(amg, S, bvec)
    assert rep.converged and rep.relres_true <= 1e-8 and abs(rep.iters - ro.iters) <= 2


def test_zero_rhs_and_x0(amg, rng):
    ptr, col, val = gen.matrix(gen.POISSON3, 8)
    A = amg.BSR.from_numpy(ptr, col, val)
    S = amg.Solver(A, amg.default_params(solver=amg.CG, coarse_enough=100))
    b = torch.zeros(512 * 3, dtype=torch.float64, device="cuda")
    x = torch.as_tensor(rng.standard_normal(512 * 3), device="cuda")
    rep = S.solve(b, x)
    assert rep.converged and rep.iters == 0 and rep.relres_true == 0 and not x.any()
    # nonzero x0 is honoured: starting at the solution converges immediately
    bv = gen.rhs(gen.RHS_UNIFORM, 8, 3)
    xs = np.linalg.solve(oracle.Mat.from_arrays(ptr, col, val).dense(), bv)
    rep = S.solve(torch.as_tensor(bv, device="cuda"), torch.as_tensor(xs, device="cuda"))
    assert rep.converged and rep.iters == 0


def test_single_level_exact(amg, rng):
    ptr, col, val = gen.matrix(gen.POISSON3, 6)  # 648 unknowns <= coarse_enough
    A = amg.BSR.from_numpy(ptr, col, val)
    for solver in (amg.CG, amg.BICGSTAB, amg.GMRES):
        S = amg.Solver(A, amg.default_params(solver=solver, hier_dtype=amg.F64, vcycle_vec_dtype=amg.F64))
        assert S.levels == 1
        x, rep = _solve(amg, S, rng.standard_normal(648))
        assert rep.converged and rep.iters == 1


def test_identity_no_precond(amg, rng):
    n = 100
    A = amg.BSR.from_numpy(np.arange(n + 1, dtype=np.int32), np.arange(n, dtype=np.int32), np.tile(np.eye(3), (n, 1, 1)))
    for solver in (amg.CG, amg.BICGSTAB, amg.GMRES, amg.IDRS):
        S = amg.Solver(A, amg.default_params(solver=solver, precond=amg.PC_NONE))
        b = rng.standard_normal(3 * n)
        x, rep = _solve(amg, S, b)
        assert rep.converged and rep.iters == 1 and np.allclose(x, b)


def test_error_codes(amg):
    ptr, col, val = gen.matrix(gen.POISSON3, 4)
    # non-square
    A = amg.BSR.from_numpy(ptr, col, val, n_block_cols=65)
    with pytest.raises(amg.AmgError) as e:
        amg.Solver(A)
    assert e.value.status == amg.EDIM
    # missing diagonal block
    p2 = np.array([0, 1, 2], np.int32)
    c2 = np.array([1, 0], np.int32)
    with pytest.raises(amg.AmgError) as e:
        amg.Solver(amg.BSR.from_numpy(p2, c2, np.ones((2, 3, 3))), coarse_enough=1)
    assert e.value.status == amg.EZERODIAG
    # singular diagonal block
    v = val.copy()
    for i in range(64):
        for k in range(ptr[i], ptr[i + 1]):
            if col[k] == i and i == 5:
                v[k] = np.array([[1, 2, 3], [2, 4, 6], [0, 0, 1.0]])
    with pytest.raises(amg.AmgError) as e:
        amg.Solver(amg.BSR.from_numpy(ptr, col, v), coarse_enough=30)
    assert e.value.status == amg.ESINGULAR_BLOCK
    # bad params
    for bad in (dict(gmres_m=40), dict(coarsening=2), dict(schur_shat=3), dict(over_interp=0.0), dict(gmres_ortho=4)):
        with pytest.raises(amg.AmgError) as e:
            amg.Solver(amg.BSR.from_numpy(ptr, col, val), **bad)
        assert e.value.status == amg.EINVAL, bad


def test_fp32_vs_fp64_iteration_parity(amg):
    # mixed precision "does not increase the number of iterations"
    n = 24
    ptr, col, val = gen.matrix(gen.STOKES, n)
    bvec = gen.rhs(gen.RHS_LID_NOISE, n, 4)
    its = []
    for h32 in (False, True):
        A = amg.BSR.from_numpy(ptr, col, val)
        dt = amg.F32 if h32 else amg.F64
        S = amg.Solver(A, amg.default_params(solver=amg.GMRES, precond=amg.PC_SCHUR, hier_dtype=dt,
                                             vcycle_vec_dtype=dt))
        x, rep = _solve(amg, S, bvec)
        assert rep.converged
        its.append(rep.iters)
    assert abs(its[0] - its[1]) <= 1


@pytest.mark.parametrize("ortho", [1, 2, 3])
@pytest.mark.parametrize("wide", [1, 99])
def test_gram_gmres_kernel_paths(amg, envvars, wide, ortho):
    # the update + dots + norm pass (and, ortho = 2 / 3, the fp32 / fp16-shadow multi-dot) on
    # the wide (wide=1) and K-templated (wide=99) kernels
    envvars(AMG_CGS_WIDE=wide)
    n = 16
    ptr, col, val = gen.matrix(gen.STOKES, n)
    bvec = gen.rhs(gen.RHS_LID_NOISE, n, 4)
    A, S, O = make_pair(amg, ptr, col, val, hier32=True, precond=1, solver=2, gmres_ortho=ortho)
    ro = O.solve(bvec, rtol=1e-8)
    x, rep = _solve(amg, S, bvec)
    true = np.linalg.norm(bvec - oracle.spmv(oracle.Mat.from_arrays(ptr, col, val), x)) / np.linalg.norm(bvec)
    assert rep.converged and true <= 1e-8 and abs(rep.iters - ro.iters) <= 2, (rep.iters, ro.iters, true)


@pytest.mark.parametrize("wide,copy", [(1, "sell"), (99, "sell"), (1, "sellr")])
def test_solve_forced_kernel_paths(amg, envvars, wide, copy):
    # sliced (SELL-C) or interleaved row-per-lane copies on every level they apply to (small
    # grid: lower the slice-count gates) and the wide (wide=1) or K-templated (wide=99) CGS2
    # kernels at every k
    if copy == "sell":
        envvars(AMG_SELL_MIN_SLICES=1, AMG_SELLR=0, AMG_CGS_WIDE=wide)
    else:
        envvars(AMG_SELLR_MIN_SLICES=1, AMG_CGS_WIDE=wide)
    n = 24
    ptr, col, val = gen.matrix(gen.STOKES, n)
    bvec = gen.rhs(gen.RHS_LID_NOISE, n, 4)
    A, S, O = make_pair(amg, ptr, col, val, hier32=True, precond=1, solver=2)
    if copy == "sellr":  # the outer operator's BSR values (fp64) are released once its copy exists
        envvars(AMG_KEEP_VALUES=1)
        S_keep = amg.Solver(A, S.params)
        assert S_keep.memory_report()["outer_A"] - S.memory_report()["outer_A"] == len(col) * 16 * 8
        del S_keep
    ro = O.solve(bvec, rtol=1e-8)
    x, rep = _solve(amg, S, bvec)
    true = np.linalg.norm(bvec - oracle.spmv(oracle.Mat.from_arrays(ptr, col, val), x)) / np.linalg.norm(bvec)
    assert rep.converged and true <= 1e-8 and abs(rep.iters - ro.iters) <= 2, (rep.iters, ro.iters, true)


@pytest.mark.parametrize("solver", [1, 2])
def test_solve_interleaved_copies_everywhere(amg, envvars, solver):
    # every square-block matrix of the handle (outer operator: fused SpMV+dot and
    # residual+norm; hierarchy A, P, R) on the interleaved row-per-lane copy
    envvars(AMG_LANE_VAR=8)
    n = 20
    ptr, col, val = gen.matrix(gen.STOKES, n)
    bvec = gen.rhs(gen.RHS_LID_NOISE, n, 4)
    A, S, O = make_pair(amg, ptr, col, val, hier32=True, precond=1, solver=solver)
    ro = O.solve(bvec, rtol=1e-8)
    x, rep = _solve(amg, S, bvec)
    true = np.linalg.norm(bvec - oracle.spmv(oracle.Mat.from_arrays(ptr, col, val), x)) / np.linalg.norm(bvec)
    assert rep.converged and true <= 1e-8 and abs(rep.iters - ro.iters) <= 2, (rep.iters, ro.iters, true)


# ---- Schur split by a general scalar pressure mask (amg_setup_pmask, R21) ----
def _csr_from_dense(D):
    ptr = np.zeros(D.shape[0] + 1, np.int32)
    cols, vals = [], []
    for i in range(D.shape[0]):
        nz = np.flatnonzero(D[i])
        if i not in nz:
            nz = np.sort(np.append(nz, i))
        cols.extend(nz.tolist())
        vals.extend(D[i, nz].tolist())
        ptr[i + 1] = len(cols)
    return ptr, np.array(cols, np.int32), np.array(vals).reshape(-1, 1, 1)


def _pmask_pair(amg, ptr, col, val, mask, hier32, **kw):
    A = amg.BSR.from_numpy(ptr, col, val)
    gp = amg.default_params(hier_dtype=amg.F32 if hier32 else amg.F64,
                            vcycle_vec_dtype=amg.F32 if hier32 else amg.F64, precond=1, **kw)
    S = amg.Solver(A, gp, pmask=torch.as_tensor(mask.astype(np.uint8), device="cuda"))
    op = oracle.default_params(hier_f32=int(hier32), vec_f32=int(hier32), precond=oracle.PC_SCHUR,
                               **{ORC_OF[k]: v for k, v in kw.items() if k in ORC_OF})
    O = oracle.Solver(oracle.Mat.from_arrays(ptr, col, val), op, pmask=mask)
    return A, S, O


def _scrambled_stokes(n, seed=5):
    ptr, col, val = gen.matrix(gen.STOKES, n)
    Ad0 = oracle.Mat.from_arrays(ptr, col, val).dense()
    perm = np.random.default_rng(seed).permutation(Ad0.shape[0])
    Ad = Ad0[np.ix_(perm, perm)]
    return (*_csr_from_dense(Ad), perm % 4 == 3)


PMASK_CASES = [
    ("interleaved-f64", False, 10, dict(solver=2, coarse_enough=40)),
    ("interleaved-f32-idrs", True, 16, dict(solver=3)),
    ("scrambled-f64", False, 8, dict(solver=2, coarse_enough=60, scrambled=True)),
    ("scrambled-f32-ilu0", True, 10, dict(solver=3, smoother=2, scrambled=True)),
]


@pytest.mark.parametrize("name,h32,n,kw", PMASK_CASES, ids=[c[0] for c in PMASK_CASES])
def test_pmask_parity(amg, rng, name, h32, n, kw):
    kw = dict(kw)
    if kw.pop("scrambled", False):
        ptr, col, val, mask = _scrambled_stokes(n)
    else:
        ptr, col, val = gen.matrix(gen.STOKES, n)
        mask = np.arange(4 * n ** 3) % 4 == 3
    A, S, O = _pmask_pair(amg, ptr, col, val, mask, h32, **kw)
    check_hierarchy(S, O, h32)
    d, m = S.schur_export()
    od, om = O.schur_vectors()
    assert np.array_equal(d, od) and np.array_equal(m, om)
    N = len(mask)
    for _ in range(2):
        r = rng.standard_normal(N)
        z = S.apply_precond(torch.as_tensor(r, device="cuda"), torch.zeros(N, dtype=torch.float64, device="cuda"))
        torch.cuda.synchronize()
        assert relerr(z.cpu().numpy(), O.precond(r)) <= (1e-5 if h32 else 1e-10)
    bvec = rng.standard_normal(N)
    ro = O.solve(bvec, rtol=1e-8)
    x, rep = _solve(amg, S, bvec)
    true = np.linalg.norm(bvec - oracle.spmv(oracle.Mat.from_arrays(ptr, col, val), x)) / np.linalg.norm(bvec)
    assert rep.converged and true <= 1e-8 and abs(rep.iters - ro.iters) <= 2, (rep.iters, ro.iters, true)


def test_pmask_errors(amg):
    ptr, col, val = gen.matrix(gen.STOKES, 4)
    A = amg.BSR.from_numpy(ptr, col, val)
    N = 4 * 64
    for mask, kw in ((np.zeros(N), {}), (np.ones(N), {}), (np.arange(N) % 4 == 3, dict(schur_shat=2)),
                     (np.arange(N) % 4 == 3, dict(precond=0))):
        gp = amg.default_params(**({"precond": 1} | kw))
        with pytest.raises(amg.AmgError) as e:
            amg.Solver(A, gp, pmask=torch.as_tensor(mask.astype(np.uint8), device="cuda"))
        assert e.value.status == amg.EINVAL


@pytest.mark.parametrize("solver", [0, 1, 2, 3])
def test_maxiter_not_converged(amg, solver):
    # maxiter reached: AMG_NOT_CONVERGED, the report filled, x the last iterate -- the same
    # iteration count and (to the precision bar) the same residual as the oracle
    n = 12
    kind = gen.POISSON3 if solver == 0 else gen.STOKES
    ptr, col, val = gen.matrix(kind, n)
    bvec = gen.rhs(gen.RHS_UNIFORM if solver == 0 else gen.RHS_LID_NOISE, n, val.shape[-1])
    pc = 1 if solver in (2, 3) else 0
    A, S, O = make_pair(amg, ptr, col, val, hier32=False, precond=pc, solver=solver, maxiter=3, coarse_enough=100)
    ro = O.solve(bvec, rtol=1e-12)
    x, rep = _solve(amg, S, bvec, rtol=1e-12)
    assert rep.status == amg.NOT_CONVERGED and not rep.converged
    assert rep.iters == ro.iters == 3
    true = np.linalg.norm(bvec - oracle.spmv(oracle.Mat.from_arrays(ptr, col, val), x)) / np.linalg.norm(bvec)
    assert abs(true - rep.relres_true) <= 1e-10 * max(true, 1.0)
    assert abs(rep.relres_true - ro.relres_true) <= 1e-6 * ro.relres_true


def test_memory_report(amg):
    ptr, col, val = gen.matrix(gen.STOKES, 16)
    S = amg.Solver(amg.BSR.from_numpy(ptr, col, val), amg.default_params(solver=2, precond=1))
    m = S.memory_report()
    nnz = len(col)
    assert m["outer_A"] >= nnz * (4 + 16 * 8)  # 4x4 fp64 library copy
    assert m["hierarchy"] > 0 and m["smoothers"] > 0 and m["schur"] > 0 and m["krylov"] > 0
    assert sum(v for k, v in m.items() if k != "total") <= m["total"] == S.device_bytes


def _block_diag_matrix(eigs, n, b, rng):
    """n diagonal b x b blocks Q_i diag(e) Q_i^T with eigenvalues drawn from `eigs`."""
    ptr = np.arange(n + 1, dtype=np.int32)
    col = np.arange(n, dtype=np.int32)
    val = np.zeros((n, b, b))
    for i in range(n):
        q, _ = np.linalg.qr(rng.standard_normal((b, b)))
        val[i] = q @ np.diag(rng.choice(eigs, b)) @ q.T
    return ptr, col, val


@pytest.mark.parametrize("force", [0, 1], ids=["guarded", "forced"])
@pytest.mark.parametrize("eigs", [(1.0, 2.0, 3.0, 5.0, 8.0), tuple(np.logspace(0, 2, 400))],
                         ids=["near-invariant", "ill-conditioned"])
def test_gram_gmres_reorthogonalisation_safeguard(amg, envvars, eigs, force):
    # the Gram/Cholesky orthogonalisation must not trust 1 - |R(:,k)|^2
    # when the new direction is (nearly) in span(V).  A spectrum of five values makes the
    # Krylov space invariant after five steps (w in span(V) up to rounding); a wide spectrum
    # without preconditioner drives a long Arnoldi sequence.  Both compared against CGS2.
    # forced: AMG_REORTH_ALWAYS=1 takes the extra pass at every step (exercises it on the GPU)
    if force:
        envvars(AMG_REORTH_ALWAYS=1)
    rng = np.random.default_rng(11)
    ptr, col, val = _block_diag_matrix(np.array(eigs), 2000, 3, rng)
    bvec = rng.standard_normal(6000)
    res = {}
    for ortho in (0, 1, 2, 3):
        A = amg.BSR.from_numpy(ptr, col, val)
        S = amg.Solver(A, amg.default_params(solver=amg.GMRES, precond=amg.PC_NONE, gmres_ortho=ortho,
                                             maxiter=1000))
        x, rep = _solve(amg, S, bvec)
        true = np.linalg.norm(bvec - oracle.spmv(oracle.Mat.from_arrays(ptr, col, val), x)) / np.linalg.norm(bvec)
        res[ortho] = (rep, true, S.counters()["reorth_passes"])
    r0, t0, _ = res[0]
    for o in (1, 2, 3):
        r1, t1, reorth = res[o]
        assert r0.converged and r1.converged and t0 <= 1e-8 and t1 <= 1e-8, (o, t0, t1)
        assert abs(r0.iters - r1.iters) <= 2, (o, r0.iters, r1.iters)
        if force:
            assert reorth >= r1.iters
    O = oracle.Solver(oracle.Mat.from_arrays(ptr, col, val), oracle.default_params(
        solver=oracle.GMRES, precond=oracle.PC_NONE, maxiter=1000))
    assert abs(O.solve(bvec, rtol=1e-8).iters - r1.iters) <= 2


@pytest.mark.parametrize("copy,kw", [("sellr", dict(precond=1, solver=2)), ("sell", dict(precond=1, solver=2)),
                                     ("sellr", dict(precond=0, solver=1)), ("sell", dict(precond=0, solver=1))],
                         ids=["sellr-schur", "sell-schur", "sellr-monolithic", "sell-monolithic"])
def test_released_values_rematerialised_from_copies(amg, envvars, copy, kw):
    # a single-device handle frees the BSR values of every matrix whose
    # interleaved / sliced copy carries its products; the export re-materialises them from the
    # copy (bit-exact with the oracle), and the solve is unchanged
    if copy == "sellr":
        envvars(AMG_SELLR_MIN_SLICES=1)
    else:
        envvars(AMG_SELL_MIN_SLICES=1, AMG_SELLR=0)
    n = 24
    ptr, col, val = gen.matrix(gen.STOKES, n)
    bvec = gen.rhs(gen.RHS_LID_NOISE, n, 4)
    res = []
    for keep in (0, 1):
        if keep:
            envvars(AMG_KEEP_VALUES=1)
        A, S, O = make_pair(amg, ptr, col, val, hier32=True, **kw)
        check_hierarchy(S, O, True)  # values and column indices re-materialised from the copies
        x, rep = _solve(amg, S, bvec)
        res.append((S.memory_report(), x, rep.iters))
    (m0, x0, i0), (m1, x1, i1) = res
    assert m0["hierarchy"] < m1["hierarchy"]
    if copy == "sellr":  # the outer 4x4 operator (7 blocks per row) has only the interleaved copy
        assert m0["outer_A"] < m1["outer_A"]
    assert i0 == i1 and np.array_equal(x0, x1)


@pytest.mark.parametrize("kind,n,rk,kw", [
    (gen.STOKES, 24, gen.RHS_LID, dict(precond=0, solver=1)),
    (gen.STOKES, 12, gen.RHS_LID_NOISE, dict(precond=1, solver=1)),
    (gen.POISSON3, 12, gen.RHS_UNIFORM, dict(precond=0, solver=1, smoother=2, coarse_enough=40)),
    (gen.POISSON3, 16, gen.RHS_UNIFORM, dict(precond=0, solver=0, hier_dtype=0, vcycle_vec_dtype=0)),
    (gen.POISSON3, 12, gen.RHS_UNIFORM, dict(precond=0, solver=0, coarse_enough=40)),
], ids=["cfg3-24", "schur-12", "ilu0-poisson", "cg-cfg1", "cg-f32"])
def test_step_graph_bit_identical(amg, envvars, kind, n, rk, kw):
    # reading R24: one CUDA graph per BiCGStab / CG step with alpha / beta / omega formed on
    # the device -- the same iterates as the host-driven loop, bit for bit
    ptr, col, val = gen.matrix(kind, n)
    bvec = gen.rhs(rk, n, val.shape[-1])
    runs = []
    for eager in (0, 1):
        if eager:
            envvars(AMG_NO_STEP_GRAPH=1)
        A = amg.BSR.from_numpy(ptr, col, val)
        S = amg.Solver(A, amg.default_params(**kw))
        x, rep = _solve(amg, S, bvec)
        x2, rep2 = _solve(amg, S, bvec)  # the cached step graph replayed by a second solve
        assert np.array_equal(x, x2) and rep.iters == rep2.iters
        runs.append((x, rep.iters, rep.relres_true, S.counters()["graphs"]))
    (xg, ig, rg, ng), (xe, ie, re_, ne) = runs
    assert ig == ie and rg == re_ and np.array_equal(xg, xe)
    assert ng >= 1 and ne >= 1  # graphed: the step graph; host-driven: the preconditioner graphs


@pytest.mark.parametrize("kind,n,kw,h32,env", [
    (gen.STOKES, 16, dict(precond=1, solver=2), True, {}),                      # split4 + B^T (TMA) + R fused
    (gen.STOKES, 24, dict(precond=1, solver=2), True, dict(AMG_NO_TMA_SCHUR=1)),  # B^T on the lane kernels
    (gen.STOKES, 24, dict(precond=1, solver=2), True, dict(AMG_SELLR_MIN_SLICES=1)),  # interleaved R copies
    (gen.STOKES, 24, dict(precond=1, solver=2), True, dict(AMG_SELL_MIN_SLICES=1, AMG_SELLR=0)),  # sliced copies
    (gen.STOKES, 10, dict(precond=1, solver=2, coarse_enough=40), False, {}),   # fp64: generic split, R fused
    (gen.STOKES, 16, dict(precond=0, solver=1), True, {}),                      # monolithic 4x4: convert_M
    (gen.POISSON3, 12, dict(precond=0, solver=0, coarse_enough=40), False, {}),  # monolithic 3x3 fp64
    (gen.STOKES, 16, dict(precond=1, solver=3, schur_u_scalar=1, coarse_enough=300), True, {}),  # V2 (b = 1)
], ids=["schur-f32", "schur-lane-BT", "schur-sellr", "schur-sell", "schur-f64", "mono-4x4", "mono-3x3-f64", "v2"])
def test_fused_presmooth_bit_identical(amg, envvars, rng, kind, n, kw, h32, env):
    # x = M f formed in the epilogue of the kernel producing f (split,
    # B^T update, restriction, narrowing) -- the same preconditioner output and the same solve
    # bit for bit as the separate K4a pass, with fewer kernels per application
    envvars(**env)
    ptr, col, val = gen.matrix(kind, n)
    N = (len(ptr) - 1) * val.shape[-1]
    r = torch.as_tensor(rng.standard_normal(N), device="cuda")
    bvec = gen.rhs(gen.RHS_LID_NOISE if kind == gen.STOKES else gen.RHS_UNIFORM, n, val.shape[-1])
    out = []
    for fused in (1, 0):
        A = amg.BSR.from_numpy(ptr, col, val)
        dt = amg.F32 if h32 else amg.F64
        S = amg.Solver(A, amg.default_params(hier_dtype=dt, vcycle_vec_dtype=dt, fused_presmooth=fused, **kw))
        z = torch.zeros(N, dtype=torch.float64, device="cuda")
        k0 = amg.kernel_launches()
        S.apply_precond(r, z)
        torch.cuda.synchronize()
        k = amg.kernel_launches() - k0
        x, rep = _solve(amg, S, bvec)
        out.append((z.cpu().numpy(), k, x, rep.iters))
    (z1, k1, x1, i1), (z0, k0_, x0, i0) = out
    assert np.array_equal(z1, z0)
    assert np.array_equal(x1, x0) and i1 == i0
    assert k1 < k0_, (k1, k0_)


@pytest.mark.parametrize("n,kw,env", [
    (16, dict(precond=1, solver=2), {}),                                # GMRES: z stored fp32
    (24, dict(precond=1, solver=2), dict(AMG_SELLR_MIN_SLICES=1)),      # level 0 on the interleaved copy
    (24, dict(precond=1, solver=2), dict(AMG_SELLR=0)),                 # level 0 on the row lanes
    (16, dict(precond=1, solver=1), {}),                                # BiCGStab: z fp64
    (16, dict(precond=1, solver=2, npost=2), {}),                       # the last of two post-smoothing steps
], ids=["gmres", "sellr", "lanes", "bicgstab", "npost2"])
def test_fused_join_bit_identical(amg, envvars, rng, n, kw, env):
    # the Schur preconditioner's join z = (u, p) written by the second
    # U-solve's last post-smoothing step -- the same output and solve bit for bit as the
    # separate K9' pass, one kernel fewer per application
    envvars(**env)
    ptr, col, val = gen.matrix(gen.STOKES, n)
    N = (len(ptr) - 1) * 4
    r = torch.as_tensor(rng.standard_normal(N), device="cuda")
    bvec = gen.rhs(gen.RHS_LID_NOISE, n, 4)
    out = []
    for off in (0, 1):
        envvars(AMG_NO_JOIN_FUSE=off)
        A = amg.BSR.from_numpy(ptr, col, val)
        S = amg.Solver(A, amg.default_params(hier_dtype=amg.F32, vcycle_vec_dtype=amg.F32, **kw))
        z = torch.zeros(N, dtype=torch.float64, device="cuda")
        k0 = amg.kernel_launches()
        S.apply_precond(r, z)
        torch.cuda.synchronize()
        k = amg.kernel_launches() - k0
        x, rep = _solve(amg, S, bvec)
        out.append((z.cpu().numpy(), k, x, rep.iters, rep.alg_bytes))
    (z1, k1, x1, i1, b1), (z0, k0_, x0, i0, b0) = out
    assert np.array_equal(z1, z0)
    assert np.array_equal(x1, x0) and i1 == i0
    assert k1 == k0_ - 1, (k1, k0_)
    assert b1 < b0


@pytest.mark.parametrize("kind,n,rhs,kw,env", [
    (gen.STOKES, 16, gen.RHS_LID, dict(solver=1, hier_dtype=1, vcycle_vec_dtype=1), {}),      # cfg 3 shape: 4x4 fp32 -> fp64 z
    (gen.STOKES, 24, gen.RHS_LID, dict(solver=1, hier_dtype=1, vcycle_vec_dtype=1),
     dict(AMG_SELLR_MIN_SLICES=1)),                                                           # level 0 on the interleaved copy
    (gen.STOKES, 24, gen.RHS_LID, dict(solver=1, hier_dtype=1, vcycle_vec_dtype=1), dict(AMG_SELLR=0)),  # row lanes
    (gen.POISSON3, 16, gen.RHS_UNIFORM, dict(solver=0), {}),                                  # cfg 1: 3x3 fp64, z of the same dtype
    (gen.POISSON3, 16, gen.RHS_UNIFORM, dict(solver=0, hier_dtype=1, vcycle_vec_dtype=1), {}),  # 3x3 fp32 -> fp64
    (gen.STOKES, 16, gen.RHS_LID, dict(solver=2, hier_dtype=1, vcycle_vec_dtype=1), {}),      # GMRES: z fp32 (same dtype)
    (gen.STOKES, 16, gen.RHS_LID, dict(solver=1, hier_dtype=1, vcycle_vec_dtype=1, npost=2), {}),  # last of two steps
], ids=["cfg3", "sellr", "lanes", "cfg1-f64", "b3-f32", "gmres-f32z", "npost2"])
def test_fused_widen_bit_identical(amg, envvars, rng, kind, n, rhs, kw, env):
    # the monolithic preconditioner's output conversion (the fp32
    # V-cycle result widened into the outer z, C9) written by level 0's last post-smoothing
    # step -- the same output and solve bit for bit as the separate conversion pass, one kernel
    # fewer per application
    envvars(**env)
    ptr, col, val = gen.matrix(kind, n)
    b = gen.block_size(kind)
    N = (len(ptr) - 1) * b
    r = torch.as_tensor(rng.standard_normal(N), device="cuda")
    bvec = gen.rhs(rhs, n, b)
    out = []
    for off in (0, 1):
        envvars(AMG_NO_WIDEN_FUSE=off)
        A = amg.BSR.from_numpy(ptr, col, val)
        S = amg.Solver(A, amg.default_params(precond=amg.PC_AMG, **kw))
        z = torch.zeros(N, dtype=torch.float64, device="cuda")
        k0 = amg.kernel_launches()
        S.apply_precond(r, z)
        torch.cuda.synchronize()
        k = amg.kernel_launches() - k0
        x, rep = _solve(amg, S, bvec)
        out.append((z.cpu().numpy(), k, x, rep.iters, rep.alg_bytes))
    (z1, k1, x1, i1, b1), (z0, k0_, x0, i0, b0) = out
    assert np.array_equal(z1, z0)
    assert np.array_equal(x1, x0) and i1 == i0
    assert k1 == k0_ - 1, (k1, k0_)
    assert b1 < b0


@pytest.mark.parametrize("kind,n,rhs,kw", [
    (gen.STOKES, 16, gen.RHS_LID, dict(hier_dtype=1, vcycle_vec_dtype=1)),   # cfg 3 shape: 4x4 fp32
    (gen.STOKES, 24, gen.RHS_LID, dict(hier_dtype=1, vcycle_vec_dtype=1)),
    (gen.POISSON3, 16, gen.RHS_UNIFORM, dict()),                             # 3x3 fp64
], ids=["stokes16", "stokes24", "poisson-f64"])
def test_fused_bicg_p_bit_identical(amg, envvars, kind, n, rhs, kw):
    # BiCGStab's direction update p = r + beta (p - omega v) formed
    # in the monolithic apply's narrowing pass -- the same iterates bit for bit as the separate
    # k_bicg_p, fewer bytes and kernels per step
    ptr, col, val = gen.matrix(kind, n)
    bvec = gen.rhs(rhs, n, gen.block_size(kind))
    out = []
    for off in (0, 1):
        envvars(AMG_NO_BICGP_FUSE=off)
        S = amg.Solver(amg.BSR.from_numpy(ptr, col, val), amg.default_params(precond=amg.PC_AMG, solver=1, **kw))
        k0 = amg.kernel_launches()
        x, rep = _solve(amg, S, bvec)
        out.append((x, rep.iters, rep.alg_bytes, amg.kernel_launches() - k0))
    (x1, i1, b1, k1), (x0, i0, b0, k0_) = out
    assert np.array_equal(x1, x0) and i1 == i0
    assert b1 < b0 and k1 < k0_, (b1, b0, k1, k0_)


def test_f16_shadow_wide_dynamic_range(amg):
    # reading R28: the fp16 shadow is scaled to about unit rms by a power of two, so basis
    # vectors whose entries span 12 orders of magnitude neither overflow nor lose the dots that
    # matter (the smallest entries underflow): a right-hand side scaled by 10^[-6, 6] block by
    # block, no preconditioner; the fp16-shadow GMRES converges like the GPU's CGS2 and the
    # fp32-shadow form
    rng = np.random.default_rng(28)
    ptr, col, val = _block_diag_matrix(np.logspace(0, 1.5, 50), 3000, 3, rng)
    sc = 10.0 ** rng.uniform(-6, 6, 3000)
    bvec = rng.standard_normal(9000) * np.repeat(sc, 3)
    res = {}
    for ortho in (0, 2, 3):
        S = amg.Solver(amg.BSR.from_numpy(ptr, col, val), amg.default_params(
            solver=amg.GMRES, precond=amg.PC_NONE, gmres_ortho=ortho, maxiter=2000))
        x, rep = _solve(amg, S, bvec)
        assert np.all(np.isfinite(x))
        true = np.linalg.norm(bvec - oracle.spmv(oracle.Mat.from_arrays(ptr, col, val), x)) / np.linalg.norm(bvec)
        res[ortho] = (rep.converged, rep.iters, true)
    for o in (0, 2, 3):
        assert res[o][0] and res[o][2] <= 1e-8, (o, res[o])
    assert abs(res[3][1] - res[0][1]) <= 2 and abs(res[2][1] - res[0][1]) <= 2, res
