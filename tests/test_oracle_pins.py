"""Pins of the CPU oracle against what the paper and the mathematics fix
(SURVEY.md §8(c) C0-C12).  None of these re-types an oracle formula: each
check is a printed value, a closed form, an invariant, a library routine
(numpy dense linear algebra) or brute force on a tiny input."""
import numpy as np
import pytest

import gen
import oracle
from conftest import bsr_dense, golden, laplace3_blocks, poisson1d, random_bsr

pytestmark = pytest.mark.filterwarnings("ignore")


# ---------------------------------------------------------------- C0 / C1
def test_worked_example_csr_to_bsr():
    g = golden("worked_example.json")
    A = oracle.csr_to_bsr(6, 6, 2, g["csr_ptr"], g["csr_col"], g["csr_val"])
    ptr, col, val = A.to_arrays()
    assert ptr.tolist() == g["bsr_ptr"]
    assert col.tolist() == g["bsr_col"]
    assert np.array_equal(val, np.array(g["bsr_val"]))
    # ptr halves, col shrinks 4x
    assert len(ptr) - 1 == (len(g["csr_ptr"]) - 1) // 2
    assert len(col) * 4 == len(g["csr_col"])


def test_worked_example_spmv():
    g = golden("worked_example.json")
    A = oracle.Mat.from_arrays(g["bsr_ptr"], g["bsr_col"], np.array(g["bsr_val"]))
    y = oracle.spmv(A, np.ones(6))
    assert np.allclose(y, g["y_ones"], rtol=0, atol=1e-14)


def test_csr_to_bsr_explicit_zeros_and_not_divisible(rng):
    # a tile with one scalar becomes a full block with explicit zeros
    A = oracle.csr_to_bsr(4, 4, 2, [0, 1, 1, 2, 3], [1, 3, 2], [5.0, 7.0, 9.0])
    ptr, col, val = A.to_arrays()
    assert ptr.tolist() == [0, 1, 2] and col.tolist() == [0, 1]
    assert val[0].tolist() == [[0, 5], [0, 0]] and val[1].tolist() == [[0, 7], [9, 0]]
    with pytest.raises(ValueError):
        oracle.csr_to_bsr(3, 3, 2, [0, 0, 0, 0], [], [])


@pytest.mark.parametrize("b", [1, 2, 3, 4])
def test_spmv_dense(rng, b):
    for n in (1, 7, 40):
        ptr, col, val = random_bsr(rng, n, b, density=0.2)
        A = oracle.Mat.from_arrays(ptr, col, val)
        x = rng.standard_normal(n * b)
        y0 = rng.standard_normal(n * b)
        D = bsr_dense(ptr, col, val)
        for alpha, beta in ((1.0, 0.0), (-0.5, 2.0), (2.0, 1.0)):
            y = oracle.spmv(A, x, alpha, beta, y0)
            ref = alpha * (D @ x) + beta * y0
            assert np.linalg.norm(y - ref) <= 1e-13 * max(1.0, np.linalg.norm(ref))


def test_spmv_beta0_ignores_nan(rng):
    ptr, col, val = random_bsr(rng, 10, 3)
    A = oracle.Mat.from_arrays(ptr, col, val)
    y = oracle.spmv(A, np.ones(30), 1.0, 0.0, np.full(30, np.nan))
    assert np.all(np.isfinite(y))


def test_spmv_block_vs_scalar_expansion(rng):
    # b-blocked vs scalar-expanded equivalence
    ptr, col, val = random_bsr(rng, 12, 3, density=0.3)
    D = bsr_dense(ptr, col, val)
    rows, cols = np.nonzero(D != 0)
    sptr = np.searchsorted(rows, np.arange(D.shape[0] + 1)).astype(np.int32)
    As = oracle.Mat.from_arrays(sptr, cols.astype(np.int32), D[rows, cols].reshape(-1, 1, 1))
    Ab = oracle.Mat.from_arrays(ptr, col, val)
    x = rng.standard_normal(36)
    assert np.allclose(oracle.spmv(As, x), oracle.spmv(Ab, x), rtol=0, atol=1e-13)


# ---------------------------------------------------------------- block inverse
def test_block_inverse(rng):
    assert np.array_equal(oracle.block_inverse(np.diag([2.0, 4.0])), np.diag([0.5, 0.25]))
    assert np.array_equal(oracle.block_inverse(np.eye(3)), np.eye(3))
    for b in (1, 2, 3, 4):
        for _ in range(20):
            X = rng.standard_normal((b, b)) + 3 * np.eye(b)
            Xi = oracle.block_inverse(X)
            assert np.linalg.norm(Xi @ X - np.eye(b)) < 1e-12
    # a permutation needs pivoting
    Pm = np.array([[0.0, 1.0], [1.0, 0.0]])
    assert np.array_equal(oracle.block_inverse(Pm), Pm)
    with pytest.raises(np.linalg.LinAlgError):
        oracle.block_inverse(np.array([[1.0, 2.0], [2.0, 4.0]]))


# ---------------------------------------------------------------- C2 strength
def test_strength_eps0_keeps_all_and_diagonal_has_none(rng):
    ptr, col, val = random_bsr(rng, 30, 3, density=0.2, symmetric_pattern=True, dom=5)
    A = oracle.Mat.from_arrays(ptr, col, val)
    sp, sc = oracle.strength(A, eps=0.0)
    offdiag = sum(1 for i in range(30) for k in range(ptr[i], ptr[i + 1]) if col[k] != i)
    assert len(sc) == offdiag
    d = np.array([np.eye(3) * (i + 1) for i in range(30)])
    Ad = oracle.Mat.from_arrays(np.arange(31, dtype=np.int32), np.arange(30, dtype=np.int32), d)
    sp, sc = oracle.strength(Ad, 1e-3)
    assert len(sc) == 0
    agg, nc = oracle.aggregate(Ad)
    assert nc == 0 and np.all(agg == -1)


def test_strength_constructed_strong_weak(rng):
    # off-diagonal blocks are either O(1) ("strong") or O(1e-9) ("weak"): the graph must be
    # exactly the symmetrised set of O(1) blocks, whatever the exact threshold arithmetic.
    n, b = 25, 2
    ptr, col, val = random_bsr(rng, n, b, density=0.25, dom=4)
    strong_set = set()
    for i in range(n):
        for k in range(ptr[i], ptr[i + 1]):
            j = col[k]
            if j == i:
                continue
            if rng.random() < 0.5:
                val[k] *= 1e-9
            else:
                strong_set.add((i, j))
                strong_set.add((j, i))
    A = oracle.Mat.from_arrays(ptr, col, val)
    sp, sc = oracle.strength(A, 1e-3)
    got = {(i, int(sc[k])) for i in range(n) for k in range(sp[i], sp[i + 1])}
    assert got == strong_set


def test_strength_1d_poisson_all_strong():
    A = oracle.Mat.from_arrays(*poisson1d(9))
    sp, sc = oracle.strength(A, 1e-3)  # |-1|^2 > 1e-6*2*2
    assert len(sc) == 16


def test_strength_slabs_drop_cross_edges():
    A = oracle.Mat.from_arrays(*poisson1d(10))
    sp, sc = oracle.strength(A, 1e-3, nparts=2)
    assert len(sc) == 16  # the edge 4-5 is dropped both ways


# ---------------------------------------------------------------- C3 aggregation
def test_aggregation_1d_hand_trace():
    g = golden("aggregation_1d.json")
    agg, nc = oracle.aggregate(oracle.Mat.from_arrays(*poisson1d(9)))
    assert agg.tolist() == g["n9_agg"] and nc == 3
    agg, nc = oracle.aggregate(oracle.Mat.from_arrays(*poisson1d(729)))
    assert nc == g["n729_count"]


def test_aggregation_pass2_lowest_index_neighbour():
    # Hand-built graph where pass-2 node 3 touches two pass-1 aggregates (
    # SURVEY.md C3 "lowest-index strong neighbour that was assigned in pass 1").
    # Edges 0-4, 0-5, 1-2, 2-3, 3-5.  Pass 1: root 0 takes {0,4,5}; root 1 takes {1,2};
    # node 3 is blocked (neighbours 2 and 5 assigned).  Pass 2: its lowest-index assigned
    # neighbour is 2 (aggregate 1) -- not 5 (the last neighbour, aggregate 0) and not the
    # lowest aggregate id (0).
    n = 6
    edges = {(0, 4), (0, 5), (1, 2), (2, 3), (3, 5)}
    Dn = 4.0 * np.eye(n)
    for i, j in edges:
        Dn[i, j] = Dn[j, i] = -1.0
    ptr, col, val = [0], [], []
    for i in range(n):
        for j in range(n):
            if Dn[i, j] != 0:
                col.append(j)
                val.append(Dn[i, j])
        ptr.append(len(col))
    A = oracle.Mat.from_arrays(np.array(ptr, np.int32), np.array(col, np.int32),
                               np.array(val).reshape(-1, 1, 1))
    agg, nc = oracle.aggregate(A)
    assert nc == 2
    assert agg.tolist() == [0, 1, 1, 1, 0, 0]
    assert oracle.roots(A).tolist() == [1, 1, 0, 0, 0, 0]


def _graph(sp, sc, n):
    return [set(sc[sp[i]:sp[i + 1]].tolist()) for i in range(n)]


def _dist2(adj, i):
    d1 = adj[i]
    d2 = set()
    for j in d1:
        d2 |= adj[j]
    return (d1 | d2) - {i}


def _parallel_rounds_roots(adj):
    """Independent formulation: lexicographically-first MIS of the distance-2 graph by
    parallel rounds: an undecided node becomes a root when every
    lower-index node within distance 2 is decided non-root; it is removed when any node
    within distance 2 is a root."""
    n = len(adj)
    UND, ROOT, NOT = 0, 1, 2
    st = [NOT if not adj[i] else UND for i in range(n)]
    nb2 = [_dist2(adj, i) for i in range(n)]
    rounds = 0
    while UND in st:
        rounds += 1
        new = list(st)
        for i in range(n):
            if st[i] != UND:
                continue
            if any(st[j] == ROOT for j in nb2[i]):
                new[i] = NOT
            elif all(st[j] == NOT for j in nb2[i] if j < i):
                new[i] = ROOT
        st = new
    return [1 if s == ROOT else 0 for s in st], rounds


def _check_aggregation_invariants(A, adj, agg, nc, roots):
    n = len(adj)
    root_ids = [i for i in range(n) if roots[i]]
    assert len(root_ids) == nc
    # coarse ids in ascending root order
    assert [agg[r] for r in root_ids] == list(range(nc))
    for a in root_ids:  # roots pairwise at distance >= 3
        assert not (_dist2(adj, a) & set(root_ids))
    for i in range(n):
        if not adj[i]:
            assert agg[i] == -1
            continue
        assert 0 <= agg[i] < nc
        r = root_ids[agg[i]]
        assert i == r or r in _dist2(adj, i)  # every member within distance 2 of its root


def test_aggregation_invariants_and_rounds(rng):
    for trial in range(6):
        n = 60
        ptr, col, val = random_bsr(rng, n, 2, density=0.06, symmetric_pattern=True, dom=3)
        for i in range(n):  # make a few nodes isolated (weak rows)
            if rng.random() < 0.1:
                for k in range(ptr[i], ptr[i + 1]):
                    if col[k] != i:
                        val[k] *= 1e-12
                        # symmetric partner
                        for kk in range(ptr[col[k]], ptr[col[k] + 1]):
                            if col[kk] == i:
                                val[kk] *= 1e-12
        A = oracle.Mat.from_arrays(ptr, col, val)
        sp, sc = oracle.strength(A, 1e-3)
        adj = _graph(sp, sc, n)
        agg, nc = oracle.aggregate(A)
        roots = oracle.roots(A)
        _check_aggregation_invariants(A, adj, agg, nc, roots)
        pr, _ = _parallel_rounds_roots(adj)
        assert pr == roots.tolist()


def test_aggregation_probe_counts_7pt():
    # 16^3 7-point -> 514 aggregates
    ptr, col, val = laplace3_blocks(16)
    agg, nc = oracle.aggregate(oracle.Mat.from_arrays(ptr, col, val))
    assert nc == 514


def test_aggregation_parallel_rounds_7pt_8():
    ptr, col, val = laplace3_blocks(8)
    A = oracle.Mat.from_arrays(ptr, col, val)
    sp, sc = oracle.strength(A, 1e-3)
    adj = _graph(sp, sc, 512)
    pr, rounds = _parallel_rounds_roots(adj)
    assert pr == oracle.roots(A).tolist()
    assert rounds > 1


# ---------------------------------------------------------------- C4-C6 hierarchy
def _solver(ptr, col, val, **kw):
    A = oracle.Mat.from_arrays(ptr, col, val)
    return A, oracle.Solver(A, **kw)


def test_tentative_prolongator_omega0():
    ptr, col, val = laplace3_blocks(6)
    A, S = _solver(ptr, col, val, sa_omega=0.0, coarse_enough=64, hier_f32=0, vec_f32=0)
    P = S.level_mat(0, 1).dense()
    agg = S.level_agg(0)
    nc = agg.max() + 1
    sizes = np.bincount(agg[agg >= 0], minlength=nc)
    assert np.array_equal(P.T @ P, np.kron(np.diag(sizes), np.eye(3)))
    assert set(np.unique(P)) <= {0.0, 1.0}


def test_smoothed_prolongator_partition_of_unity():
    # interior rows of the 7-point Laplacian tensor I3 have zero row sums; all edges are
    # strong, so A_F = A and P's row sums equal P_tent's
    n = 6
    ptr, col, val = laplace3_blocks(n)
    A, S = _solver(ptr, col, val, coarse_enough=64, hier_f32=0, vec_f32=0)
    P = S.level_mat(0, 1).dense()
    rs = P.reshape(n ** 3, 3, -1, 3).sum(axis=2)  # block row sums
    for i in range(n ** 3):
        x, y, z = i % n, (i // n) % n, i // (n * n)
        if 0 < x < n - 1 and 0 < y < n - 1 and 0 < z < n - 1:
            assert np.allclose(rs[i], np.eye(3), atol=1e-14)


def test_smoothed_prolongator_1d_closed_form():
    # 1-D Poisson (2,-1), omega = 2/3, aggregates {0,1},{2,3,4},{5,6,7,8} (C3 hand trace).
    # P = (I - omega D^-1 A) P_tent written out by hand for this stencil (D = 2, all edges
    # strong): a row whose both neighbours share its aggregate keeps 1; a row with one
    # neighbour in another aggregate gets 1 - omega/2 = 2/3 at home and +omega/2 = 1/3 at
    # the neighbour's aggregate; an end row (one neighbour, same aggregate) keeps 1 - 1/3.
    ptr, col, val = poisson1d(9)
    A, S = _solver(ptr, col, val, coarse_enough=2, hier_f32=0, vec_f32=0, max_levels=2)
    P = S.level_mat(0, 1).dense()
    t, h = 1.0 / 3.0, 2.0 / 3.0
    expect = np.array([
        [1 - t, 0, 0],   # node 0: end row, neighbour 1 in agg 0
        [h, t, 0],       # node 1: neighbour 2 in agg 1
        [t, h, 0],       # node 2: neighbour 1 in agg 0
        [0, 1, 0],       # node 3
        [0, h, t],       # node 4: neighbour 5 in agg 2
        [0, t, h],       # node 5: neighbour 4 in agg 1
        [0, 0, 1],       # node 6
        [0, 0, 1],       # node 7
        [0, 0, 1 - t],   # node 8: end row
    ])
    assert np.allclose(P, expect, rtol=0, atol=1e-15)


def _weak_mix_bsr(rng, n, b, density, scale_share=0.35, scale=1e-4):
    """Random symmetric-pattern BSR where a share of the off-diagonal block pairs is scaled
    down so that they are weak at eps = 1e-3 (test input only)."""
    ptr, col, val = random_bsr(rng, n, b, density=density, symmetric_pattern=True, dom=3 * b)
    pos = {(i, int(col[k])): k for i in range(n) for k in range(ptr[i], ptr[i + 1])}
    for (i, j), k in pos.items():
        if i < j and rng.random() < scale_share:
            val[k] *= scale
            if rng.random() < 0.8:  # most pairs weak both ways, some only one way
                val[pos[(j, i)]] *= scale
    return ptr, col, val


def _brute_strong(ptr, col, val, eps):
    """Strength by brute force on the dense blocks: ||A_IJ||_F^2 > eps^2 ||A_II||_F ||A_JJ||_F,
    then symmetric closure."""
    n = len(ptr) - 1
    blk = {(i, int(col[k])): val[k] for i in range(n) for k in range(ptr[i], ptr[i + 1])}
    fro = lambda m: np.sqrt((m * m).sum())
    s = set()
    for (i, j), m in blk.items():
        if i != j and (m * m).sum() > eps * eps * fro(blk[(i, i)]) * fro(blk[(j, j)]):
            s.add((i, j))
            s.add((j, i))
    return blk, s


@pytest.mark.parametrize("b", [1, 2, 3])
def test_smoothed_prolongator_dense_with_weak_blocks(rng, b):
    # SURVEY.md C5's own pin: a dense (I - omega D_F^-1 A_F) P_tent on random <= 64-row
    # inputs, with >= 10 % weak blocks so that the lumping of weak blocks into D and the
    # sign of the smoothing term both change P.
    n, eps, omega = 48, 1e-3, 2.0 / 3.0
    ptr, col, val = _weak_mix_bsr(rng, n, b, density=0.12)
    blk, strong = _brute_strong(ptr, col, val, eps)
    offd = [(i, j) for (i, j) in blk if i != j]
    weak = [e for e in offd if e not in strong]
    assert len(weak) >= 0.1 * len(offd)
    A, S = _solver(ptr, col, val, coarse_enough=b * 8, hier_f32=0, vec_f32=0, eps_strong=eps,
                   sa_omega=omega)
    agg = S.level_agg(0)
    nc = int(agg.max()) + 1
    # dense A_F: strong and diagonal blocks kept, weak ones added to the diagonal
    AF = np.zeros((n * b, n * b))
    for (i, j), m in blk.items():
        if i == j or (i, j) in strong:
            AF[i * b:(i + 1) * b, j * b:(j + 1) * b] += m
        else:
            AF[i * b:(i + 1) * b, i * b:(i + 1) * b] += m
    Dinv = np.zeros_like(AF)
    for i in range(n):
        Dinv[i * b:(i + 1) * b, i * b:(i + 1) * b] = np.linalg.inv(AF[i * b:(i + 1) * b, i * b:(i + 1) * b])
    Pt = np.zeros((n * b, nc * b))
    for i in range(n):
        if agg[i] >= 0:
            Pt[i * b:(i + 1) * b, agg[i] * b:(agg[i] + 1) * b] = np.eye(b)
    expect = (np.eye(n * b) - omega * Dinv @ AF) @ Pt
    P = S.level_mat(0, 1).dense()
    assert P.shape == expect.shape
    assert np.abs(P - expect).max() <= 1e-12 * np.abs(expect).max()
    # and the lumping is visible: without it P would differ by far more than rounding
    AF_nolump = AF.copy()
    for (i, j) in weak:
        AF_nolump[i * b:(i + 1) * b, i * b:(i + 1) * b] -= blk[(i, j)]
    assert not np.allclose(AF, AF_nolump, rtol=0, atol=1e-9)


def test_smoothed_prolongator_partition_of_unity_with_weak_edges(rng):
    # A zero-row-sum operator (a graph Laplacian) with weak couplings: lumping the weak
    # blocks into the diagonal keeps A_F's row sums zero, so P's row sums equal P_tent's on
    # EVERY row.  Dropping weak blocks without lumping breaks this.
    n = 40
    W = np.zeros((n, n))
    for i in range(n):
        for j in range(i + 1, n):
            if rng.random() < 0.15 or j == i + 1:
                W[i, j] = W[j, i] = (1e-5 if rng.random() < 0.3 else 1.0) * rng.uniform(0.5, 1.5)
    L = np.diag(W.sum(axis=1)) - W
    ptr = [0]
    cols, vals = [], []
    for i in range(n):
        for j in range(n):
            if i == j or W[i, j] != 0:
                cols.append(j)
                vals.append(L[i, j])
        ptr.append(len(cols))
    ptr, col, val = np.array(ptr, np.int32), np.array(cols, np.int32), np.array(vals).reshape(-1, 1, 1)
    _, strong = _brute_strong(ptr, col, val, 1e-3)
    assert sum(1 for i in range(n) for j in range(n) if W[i, j] != 0 and (i, j) not in strong) > 0
    A, S = _solver(ptr, col, val, coarse_enough=8, hier_f32=0, vec_f32=0)
    P = S.level_mat(0, 1).dense()
    agg = S.level_agg(0)
    assert np.allclose(P.sum(axis=1), (agg >= 0).astype(float), rtol=0, atol=1e-13)


def test_galerkin_identity_and_symmetry(rng):
    # P^T (A (P u)) = A_c u (north_star) and symmetry preservation
    ptr, col, val = gen.matrix(gen.POISSON3, 8)
    A, S = _solver(ptr, col, val, coarse_enough=64, hier_f32=0, vec_f32=0)
    assert S.levels >= 3
    for l in range(S.levels - 1):
        Al, Pl, Rl, Ac = (S.level_mat(l, 0), S.level_mat(l, 1), S.level_mat(l, 2), S.level_mat(l + 1, 0))
        u = rng.standard_normal(Ac.info()[0] * 3)
        lhs = oracle.spmv(Rl, oracle.spmv(Al, oracle.spmv(Pl, u)))
        rhs = oracle.spmv(Ac, u)
        assert np.linalg.norm(lhs - rhs) <= 1e-12 * np.linalg.norm(rhs)
        D = Ac.dense()
        assert np.linalg.norm(D - D.T) <= 1e-12 * np.linalg.norm(D)
        assert np.array_equal(Rl.dense(), Pl.dense().T)


def test_galerkin_dense_triple_product(rng):
    ptr, col, val = random_bsr(rng, 150, 2, density=0.03, symmetric_pattern=True, dom=6)
    A, S = _solver(ptr, col, val, coarse_enough=40, hier_f32=0, vec_f32=0)
    assert S.levels >= 2
    Ad = A.dense()
    P = S.level_mat(0, 1).dense()
    Ac = S.level_mat(1, 0).dense()
    assert np.linalg.norm(P.T @ Ad @ P - Ac) <= 1e-12 * np.linalg.norm(Ac)


@pytest.mark.parametrize("alpha", [1.0, 1.5])
def test_plain_aggregation_is_tentative_with_scaled_galerkin(rng, alpha):
    # plain aggregation (Listings V2-V4 "coarsening::aggregation"): P = P_tent exactly (one
    # identity block per aggregated row, at its aggregate), A_c = (1/alpha) P^T A P
    # (over-interpolation, reading R19) -- numpy dense triple product, every level
    ptr, col, val = random_bsr(rng, 300, 3, density=0.02, symmetric_pattern=True, dom=6)
    A, S = _solver(ptr, col, val, coarse_enough=60, coarsening=oracle.PLAIN, over_interp=alpha,
                   hier_f32=0, vec_f32=0)
    assert S.levels >= 2
    for l in range(S.levels - 1):
        Al, P, Ac = S.level_mat(l, 0).dense(), S.level_mat(l, 1).dense(), S.level_mat(l + 1, 0).dense()
        agg = S.level_agg(l)
        Pt = np.zeros_like(P)
        for i, a in enumerate(agg):
            if a >= 0:
                Pt[3 * i:3 * i + 3, 3 * a:3 * a + 3] = np.eye(3)
        assert np.array_equal(P, Pt)
        assert np.array_equal(S.level_mat(l, 2).dense(), P.T)
        assert np.linalg.norm(P.T @ Al @ P / alpha - Ac) <= 1e-13 * np.linalg.norm(Ac)


def test_plain_aggregation_solves_to_dense_solution(rng):
    for kind, pc, solver in ((gen.POISSON3, oracle.PC_AMG, oracle.CG), (gen.STOKES, oracle.PC_SCHUR, oracle.GMRES)):
        ptr, col, val = gen.matrix(kind, 8)
        A = oracle.Mat.from_arrays(ptr, col, val)
        S = oracle.Solver(A, precond=pc, solver=solver, coarsening=oracle.PLAIN, coarse_enough=60,
                          hier_f32=0, vec_f32=0)
        assert S.levels >= 2
        b = rng.standard_normal(len(ptr) * 0 + (len(ptr) - 1) * val.shape[-1])
        r = S.solve(b, rtol=1e-10)
        xd = np.linalg.solve(A.dense(), b)
        assert r.converged and np.linalg.norm(r.x - xd) <= 1e-6 * np.linalg.norm(xd)


def test_level_sizes_strictly_decrease():
    ptr, col, val = gen.matrix(gen.STOKES, 12)
    A, S = _solver(ptr, col, val, coarse_enough=50)
    sizes = [S.level_mat(l, 0).info()[0] for l in range(S.levels)]
    assert all(a > b for a, b in zip(sizes, sizes[1:]))


# ---------------------------------------------------------------- C8 smoother
def test_spai0_is_scaled_block_inverse(rng):
    # M_I A_II = theta_I I with 0 < theta_I <= 1; with vanishing couplings theta -> 1,
    # i.e. a diagonal A gets its exact inverse
    n, b = 40, 3
    blocks = [rng.standard_normal((b, b)) + 4 * np.eye(b) for _ in range(n)]
    for scale in (0.5, 1e-2):
        pp, cc, vv = [0], [], []
        for i in range(n):
            for j in (i - 1, i, i + 1):
                if 0 <= j < n:
                    cc.append(j)
                    vv.append(blocks[i] if j == i else -scale * np.eye(b))
            pp.append(len(cc))
        A, S = _solver(np.array(pp, np.int32), np.array(cc, np.int32), np.array(vv), coarse_enough=30,
                       hier_f32=0, vec_f32=0)
        M = S.level_M(0)
        for i in range(n):
            T = M[i] @ blocks[i]
            theta = T[0, 0]
            assert np.allclose(T, theta * np.eye(b), atol=1e-13)
            assert 0 < theta <= 1
            if scale == 1e-2:
                assert abs(theta - 1) < 1e-4


def test_spai0_closed_form_7pt():
    # 7-point Laplacian tensor I3: interior theta = 108 / (108 + 6*3) = 6/7
    n = 6
    ptr, col, val = laplace3_blocks(n)
    A, S = _solver(ptr, col, val, coarse_enough=64, hier_f32=0, vec_f32=0)
    M = S.level_M(0)
    i = 2 + n * (2 + n * 2)
    assert np.allclose(M[i], (6.0 / 7.0) * np.eye(3) / 6.0, rtol=1e-15)
    c = 0  # corner: 3 neighbours -> 108 / (108 + 9)
    assert np.allclose(M[c], (108.0 / 117.0) * np.eye(3) / 6.0, rtol=1e-15)


def test_spai0_scalar_minimiser(rng):
    # b = 1: m_i = a_ii / sum_j a_ij^2 minimises ||I - M A||_F over diagonal M
    n = 80
    ptr, col, val = random_bsr(rng, n, 1, density=0.1, symmetric_pattern=True, dom=3)
    A, S = _solver(ptr, col, val, coarse_enough=20, hier_f32=0, vec_f32=0)
    m = S.level_M(0).reshape(-1)
    Ad = A.dense()
    best = np.linalg.norm(np.eye(n) - np.diag(m) @ Ad)
    for _ in range(100):
        D = m * (1 + 0.05 * rng.standard_normal(n))
        assert best <= np.linalg.norm(np.eye(n) - np.diag(D) @ Ad) + 1e-12


# ---- C8b block ILU(0) smoother (reading R20) ----
def _ilu_dense(S, level=0):
    """L = I + L_s, U = blockdiag(pivots) + U_s as dense arrays (pivots = inverse of D^-1)."""
    Ls, Us = S.level_mat(level, 4), S.level_mat(level, 5)
    Dinv = S.level_M(level)
    n, _, b, _ = Ls.info()
    L = np.eye(n * b) + Ls.dense()
    U = Us.dense()
    for i in range(n):
        U[i * b:(i + 1) * b, i * b:(i + 1) * b] = np.linalg.inv(Dinv[i])
    return L, U


def _ilu_solver(ptr, col, val, **kw):
    kw.setdefault("hier_f32", 0)
    kw.setdefault("vec_f32", 0)
    return _solver(ptr, col, val, smoother=oracle.ILU0, precond=oracle.PC_AMG, **kw)


def test_ilu0_factors_reproduce_A_on_its_pattern(rng):
    # the defining property of ILU(0) (Saad §10.3): (L U)_ij = a_ij for every stored (i, j)
    for b, dom in ((3, 6), (2, 3), (1, 4)):
        ptr, col, val = random_bsr(rng, 200, b, density=0.03, dom=dom)
        A, S = _ilu_solver(ptr, col, val, coarse_enough=30 * b)
        assert S.levels >= 2
        L, U = _ilu_dense(S)
        Ad = A.dense()
        mask = bsr_dense(ptr, col, np.ones_like(val)) != 0
        LU = L @ U
        assert np.abs(LU[mask] - Ad[mask]).max() <= 1e-12 * np.abs(Ad).max()
        for which, side in ((4, -1), (5, 1)):  # no fill: strictly lower / upper blocks of A's pattern
            fp, fc, _ = S.level_mat(0, which).to_arrays()
            rows = np.repeat(np.arange(200), np.diff(fp))
            assert np.all(np.sign(fc - rows) == side)
            assert not (S.level_mat(0, which).dense() != 0)[~mask].any()


def test_ilu0_without_fill_is_exact_lu(rng):
    # a block-tridiagonal chain has no fill: ILU(0) = LU, and with sweeps >= the chain depth
    # the sweep-solved smoother is A^-1 (numpy dense solve)
    n, b = 40, 3
    ptr = np.zeros(n + 1, np.int32)
    cols = []
    for i in range(n):
        c = [j for j in (i - 1, i, i + 1) if 0 <= j < n]
        cols.extend(c)
        ptr[i + 1] = len(cols)
    col = np.array(cols, np.int32)
    val = rng.standard_normal((len(col), b, b))
    for i in range(n):
        for k in range(ptr[i], ptr[i + 1]):
            if col[k] == i:
                val[k] += 8.0 * np.eye(b)
    A, S = _ilu_solver(ptr, col, val, coarse_enough=30, ilu_sweeps=n)
    assert S.levels >= 2
    L, U = _ilu_dense(S)
    Ad = A.dense()
    assert np.linalg.norm(L @ U - Ad) <= 1e-12 * np.linalg.norm(Ad)
    f = rng.standard_normal(n * b)
    x = S.level_smooth(0, f)
    xd = np.linalg.solve(Ad, f)
    assert np.linalg.norm(x - xd) <= 1e-10 * np.linalg.norm(xd)


def test_ilu0_sweeps_converge_to_triangular_solves(rng):
    # k >= the dependency depth: the Jacobi sweeps equal the exact forward / backward
    # substitutions with the dense factors (numpy); k = 1 is a different, coarser operator
    n, b = 120, 3
    ptr, col, val = random_bsr(rng, n, b, density=0.04, dom=6)
    f = rng.standard_normal(n * b)
    A, S = _ilu_solver(ptr, col, val, coarse_enough=60, ilu_sweeps=n)
    L, U = _ilu_dense(S)
    want = np.linalg.solve(U, np.linalg.solve(L, f))
    x = S.level_smooth(0, f)
    assert np.linalg.norm(x - want) <= 1e-10 * np.linalg.norm(want)
    _, S1 = _ilu_solver(ptr, col, val, coarse_enough=60, ilu_sweeps=1)
    x1 = S1.level_smooth(0, f)
    assert np.linalg.norm(x1 - want) > 1e-6 * np.linalg.norm(want)


def test_ilu0_smoothed_solves_reach_dense_solution(rng):
    for kind, pc, solver in ((gen.STOKES, oracle.PC_SCHUR, oracle.GMRES), (gen.STOKES, oracle.PC_AMG, oracle.BICGSTAB),
                             (gen.POISSON3, oracle.PC_AMG, oracle.IDRS)):
        ptr, col, val = gen.matrix(kind, 8)
        A = oracle.Mat.from_arrays(ptr, col, val)
        S = oracle.Solver(A, precond=pc, solver=solver, smoother=oracle.ILU0, coarse_enough=60,
                          hier_f32=0, vec_f32=0)
        assert S.levels >= 2
        b = rng.standard_normal((len(ptr) - 1) * val.shape[-1])
        r = S.solve(b, rtol=1e-10)
        xd = np.linalg.solve(A.dense(), b)
        assert r.converged and np.linalg.norm(r.x - xd) <= 1e-6 * np.linalg.norm(xd), (kind, solver)


# ---- C8c block ILUT(tau, p) smoother (Listing V2 "relaxation::ilut"; reading R25) ----
def _ilut(ptr, col, val, tau, p, **kw):
    kw.setdefault("coarse_enough", 1)
    kw.setdefault("max_levels", 2)
    A, S = _solver(ptr, col, val, smoother=oracle.ILUT, precond=oracle.PC_AMG, ilut_tau=tau, ilut_p=p,
                   hier_f32=0, vec_f32=0, **kw)
    assert S.levels >= 2
    return A, S


def _factors(S):
    """(L_s, U_s, D) at level 0 as dicts {(i, j): block} and the list of pivot blocks."""
    out = []
    for which in (4, 5):
        fp, fc, fv = S.level_mat(0, which).to_arrays()
        out.append({(i, int(fc[k])): fv[k] for i in range(len(fp) - 1) for k in range(fp[i], fp[i + 1])})
    D = [np.linalg.inv(m) for m in S.level_M(0)]
    return out[0], out[1], D


def _csr3(rows):
    ptr, col, val = [0], [], []
    for r in rows:
        for j, v in enumerate(r):
            if v != 0:
                col.append(j)
                val.append([[v]])
        ptr.append(len(col))
    return np.array(ptr, np.int32), np.array(col, np.int32), np.array(val, float)


def test_ilut_fill_limit_hand_example():
    # worked by hand: A = [[1,1,1],[1,3,0],[1,0,3]], tau = 0.  Row 1 eliminates (1,0) with
    # multiplier 1 and creates fill (1,2) = -1; row 2 creates fill (2,1) = -1, whose multiplier
    # -1/2 updates (2,2) through U(1,2) only if that fill was kept.
    #   p = 0: L = {(1,0): 1, (2,0): 1}, U = {(0,1): 1, (0,2): 1}, D = (1, 2, 2)
    #   p = 1: + L(2,1) = -1/2, U(1,2) = -1, D = (1, 2, 3/2)  (= the exact LU)
    ptr, col, val = _csr3([[1, 1, 1], [1, 3, 0], [1, 0, 3]])
    _, S = _ilut(ptr, col, val, 0.0, 0)
    L, U, D = _factors(S)
    assert {k: float(v[0, 0]) for k, v in L.items()} == {(1, 0): 1.0, (2, 0): 1.0}
    assert {k: float(v[0, 0]) for k, v in U.items()} == {(0, 1): 1.0, (0, 2): 1.0}
    assert np.allclose([d[0, 0] for d in D], [1, 2, 2], rtol=0, atol=1e-15)
    _, S = _ilut(ptr, col, val, 0.0, 1)
    L, U, D = _factors(S)
    assert {k: float(v[0, 0]) for k, v in L.items()} == {(1, 0): 1.0, (2, 0): 1.0, (2, 1): -0.5}
    assert {k: float(v[0, 0]) for k, v in U.items()} == {(0, 1): 1.0, (0, 2): 1.0, (1, 2): -1.0}
    assert np.allclose([d[0, 0] for d in D], [1, 2, 1.5], rtol=0, atol=1e-15)


def test_ilut_keeps_largest_fill_hand_example():
    # row 1 of [[1,0,1,3],[1,5,0,0],[0,0,4,0],[0,0,0,4]] eliminates (1,0) (multiplier 1) and
    # creates two U fills, (1,2) = -1 and (1,3) = -3: p = 1 keeps the larger, (1,3).  With a
    # tie ((1,2) = (1,3) = -2) the lower column is kept.
    ptr, col, val = _csr3([[1, 0, 1, 3], [1, 5, 0, 0], [0, 0, 4, 0], [0, 0, 0, 4]])
    _, S = _ilut(ptr, col, val, 0.0, 1)
    _, U, _ = _factors(S)
    assert {k: float(v[0, 0]) for k, v in U.items() if k[0] == 1} == {(1, 3): -3.0}
    ptr, col, val = _csr3([[1, 0, 2, 2], [1, 5, 0, 0], [0, 0, 4, 0], [0, 0, 0, 4]])
    _, S = _ilut(ptr, col, val, 0.0, 1)
    _, U, _ = _factors(S)
    assert {k: float(v[0, 0]) for k, v in U.items() if k[0] == 1} == {(1, 2): -2.0}


def test_ilut_threshold_hand_example():
    # worked by hand: A = [[10,1,0],[3,10,5],[0,6,10]], tau = 0.05, p = 2.
    #   row 0: tau_0 = 0.05 sqrt(101) = 0.5025: U(0,1) = 1 kept
    #   row 1: tau_1 = 0.05 sqrt(134) = 0.5788: multiplier 3/10 = 0.3 dropped, with no update
    #          (so D_1 = 10, not 10 - 0.3 * 1 = 9.7); U(1,2) = 5 kept
    #   row 2: tau_2 = 0.05 sqrt(136) = 0.5831: multiplier 6/10 = 0.6 kept, D_2 = 10 - 0.6 * 5 = 7
    # (a threshold not scaled by the row norm, a drop test on the unscaled w_k, or an update
    # applied for a dropped multiplier each give D_1 = 9.7)
    ptr, col, val = _csr3([[10, 1, 0], [3, 10, 5], [0, 6, 10]])
    _, S = _ilut(ptr, col, val, 0.05, 2)
    L, U, D = _factors(S)
    assert set(L) == {(2, 1)} and abs(L[(2, 1)][0, 0] - 0.6) <= 1e-15
    assert set(U) == {(0, 1), (1, 2)} and U[(0, 1)][0, 0] == 1.0 and U[(1, 2)][0, 0] == 5.0
    assert np.allclose([d[0, 0] for d in D], [10, 10, 7], rtol=0, atol=1e-13)


@pytest.mark.parametrize("b", [1, 2, 3])
def test_ilut_without_dropping_is_exact_lu(rng, b):
    # tau = 0 and p >= n: nothing is dropped, ILUT = the exact LU (numpy dense)
    n = 24
    ptr, col, val = random_bsr(rng, n, b, density=0.2, dom=4 * b)
    A, S = _ilut(ptr, col, val, 0.0, n)
    Ls, Us, D = _factors(S)
    L = np.eye(n * b)
    U = np.zeros((n * b, n * b))
    for (i, j), v in Ls.items():
        L[i * b:(i + 1) * b, j * b:(j + 1) * b] = v
    for (i, j), v in Us.items():
        U[i * b:(i + 1) * b, j * b:(j + 1) * b] = v
    for i in range(n):
        U[i * b:(i + 1) * b, i * b:(i + 1) * b] = D[i]
    Ad = A.dense()
    assert np.linalg.norm(L @ U - Ad) <= 1e-12 * np.linalg.norm(Ad)
    # and the sweep-solved smoother with sweeps >= the depth is A^-1
    _, S2 = _ilut(ptr, col, val, 0.0, n, ilu_sweeps=n)
    f = rng.standard_normal(n * b)
    assert np.linalg.norm(S2.level_smooth(0, f) - np.linalg.solve(Ad, f)) <= 1e-10 * np.linalg.norm(f)


def test_ilut_limits(rng):
    # tau = inf: everything off the diagonal is dropped, D_i = A_ii
    n, b = 30, 3
    ptr, col, val = random_bsr(rng, n, b, density=0.2, dom=10)
    A, S = _ilut(ptr, col, val, 1e300, 2)
    L, U, D = _factors(S)
    assert not L and not U
    for i in range(n):
        k = ptr[i] + int(np.nonzero(col[ptr[i]:ptr[i + 1]] == i)[0][0])
        assert np.allclose(D[i], val[k], rtol=1e-12)


def test_ilut_row_bounds(rng):
    # every kept off-diagonal block has ||.||_F >= tau ||a_i||_2, and each of L and U keeps at
    # most p entries outside A's pattern
    n, b, tau, p = 80, 3, 0.01, 2
    ptr, col, val = random_bsr(rng, n, b, density=0.08, dom=4)
    A, S = _ilut(ptr, col, val, tau, p)
    L, U, _ = _factors(S)
    pat = {(i, int(col[k])) for i in range(n) for k in range(ptr[i], ptr[i + 1])}
    rown = [np.sqrt(sum(np.sum(val[k] ** 2) for k in range(ptr[i], ptr[i + 1]))) for i in range(n)]
    nfill = 0
    for F in (L, U):
        for i in range(n):
            ent = [(j, v) for (r, j), v in F.items() if r == i]
            assert all(np.linalg.norm(v) >= tau * rown[i] for _, v in ent)
            fill = [j for j, _ in ent if (i, j) not in pat]
            assert len(fill) <= p
            nfill += len(fill)
    assert nfill > 0  # the case exercises the fill limit


@pytest.mark.parametrize("smoother", [oracle.ILU0, oracle.ILUT])
def test_ilu_slab_local_factors(rng, smoother):
    # reading R26: with nparts slabs the factors are those of the slabs' diagonal blocks --
    # no block couples two slabs, and with tau = 0, p >= n (ILUT) they are the exact LU of
    # the block-diagonal part (numpy); ILU(0) keeps (LU)_ij = a_ij on that part's pattern
    n, b, P = 60, 2, 3
    ptr, col, val = random_bsr(rng, n, b, density=0.12, dom=10, symmetric_pattern=True)
    kw = dict(ilut_tau=0.0, ilut_p=n) if smoother == oracle.ILUT else {}
    A, S = _solver(ptr, col, val, smoother=smoother, precond=oracle.PC_AMG, nparts=P, coarse_enough=10 * b,
                   hier_f32=0, vec_f32=0, **kw)
    assert S.levels >= 2
    bd = [r * n // P for r in range(P + 1)]
    part = np.repeat(np.arange(P), np.diff(bd))
    L, U = _ilu_dense(S)
    Ad = A.dense()
    mask = np.kron(part[:, None] == part[None, :], np.ones((b, b), bool))
    Abar = np.where(mask, Ad, 0.0)
    assert not L[~mask].any() and not U[~mask].any()
    LU = L @ U
    if smoother == oracle.ILUT:
        assert np.linalg.norm(LU - Abar) <= 1e-12 * np.linalg.norm(Abar)
    else:
        pat = (bsr_dense(ptr, col, np.ones_like(val)) != 0) & mask
        assert np.abs(LU[pat] - Abar[pat]).max() <= 1e-12 * np.abs(Abar).max()
        assert np.linalg.norm(LU - Abar) > 1e-6 * np.linalg.norm(Abar)  # a real incomplete factorisation


def test_ilut_smoothed_solves_reach_dense_solution(rng):
    for kind, pc, solver in ((gen.STOKES, oracle.PC_SCHUR, oracle.GMRES), (gen.POISSON3, oracle.PC_AMG, oracle.IDRS)):
        ptr, col, val = gen.matrix(kind, 8)
        A = oracle.Mat.from_arrays(ptr, col, val)
        S = oracle.Solver(A, precond=pc, solver=solver, smoother=oracle.ILUT, coarse_enough=60,
                          hier_f32=0, vec_f32=0)
        assert S.levels >= 2
        b = rng.standard_normal((len(ptr) - 1) * val.shape[-1])
        r = S.solve(b, rtol=1e-10)
        xd = np.linalg.solve(A.dense(), b)
        assert r.converged and np.linalg.norm(r.x - xd) <= 1e-6 * np.linalg.norm(xd), (kind, solver)


def test_jacobi_smoother_closed_form():
    n = 6
    ptr, col, val = laplace3_blocks(n)
    A, S = _solver(ptr, col, val, coarse_enough=64, smoother=oracle.JACOBI, jacobi_omega=2.0 / 3.0,
                   hier_f32=0, vec_f32=0)
    assert np.allclose(S.level_M(0), (2.0 / 3.0) * np.eye(3) / 6.0, rtol=1e-15)


# ---------------------------------------------------------------- C9 V-cycle
def test_vcycle_linear_and_symmetric(rng):
    ptr, col, val = gen.matrix(gen.POISSON3, 8)
    A, S = _solver(ptr, col, val, coarse_enough=100, hier_f32=0, vec_f32=0)
    assert S.levels >= 2
    N = 512 * 3
    u, w = rng.standard_normal(N), rng.standard_normal(N)
    Vu, Vw = S.vcycle(u), S.vcycle(w)
    assert np.allclose(S.vcycle(2.5 * u), 2.5 * Vu, rtol=0, atol=1e-12 * np.abs(Vu).max())
    assert abs(Vu @ w - u @ Vw) <= 1e-13 * abs(Vu @ w)  # symmetric on SPD (probe 2e-16)


def test_vcycle_single_level_is_exact(rng):
    ptr, col, val = gen.matrix(gen.POISSON3, 6)
    A, S = _solver(ptr, col, val, hier_f32=0, vec_f32=0)  # 648 unknowns <= 3000
    assert S.levels == 1
    f = rng.standard_normal(648)
    x = S.vcycle(f)
    assert np.allclose(x, np.linalg.solve(A.dense(), f), rtol=0, atol=1e-10)


def test_vcycle_two_level_dense_replay(rng):
    ptr, col, val = random_bsr(rng, 60, 2, density=0.06, symmetric_pattern=True, dom=5)
    A, S = _solver(ptr, col, val, coarse_enough=100, hier_f32=0, vec_f32=0)
    assert S.levels == 2
    Ad = A.dense()
    P, R, Ac = S.level_mat(0, 1).dense(), S.level_mat(0, 2).dense(), S.level_mat(1, 0).dense()
    M = S.level_M(0)
    Md = np.zeros_like(Ad)
    for i in range(60):
        Md[2 * i:2 * i + 2, 2 * i:2 * i + 2] = M[i]
    f = rng.standard_normal(120)
    x = Md @ f
    r = f - Ad @ x
    xc = np.linalg.solve(Ac, R @ r)
    x = x + P @ xc
    x = x + Md @ (f - Ad @ x)
    assert np.allclose(S.vcycle(f), x, rtol=0, atol=1e-11 * np.abs(x).max())


# ---------------------------------------------------------------- C10 Schur
def test_schur_eq10_hand_value():
    g = golden("schur_eq10_hand.json")
    blk = np.array(g["block"])[None]
    A = oracle.Mat.from_arrays(np.array([0, 1], np.int32), np.array([0], np.int32), blk)
    S = oracle.Solver(A, precond=oracle.PC_SCHUR, schur_p_component=g["p_component"], hier_f32=0, vec_f32=0)
    d, m = S.schur_vectors()
    assert d[0] == g["Shat"]
    assert m[0] == 1.0 / g["Shat"]  # SPAI0 of a 1x1 matrix is its inverse


def _stokes_split(n):
    ptr, col, val = gen.matrix(gen.STOKES, n)
    A = oracle.Mat.from_arrays(ptr, col, val)
    Ad = A.dense()
    vel = np.array([q for q in range(4 * n ** 3) if q % 4 != 3])
    pre = np.array([q for q in range(4 * n ** 3) if q % 4 == 3])
    return A, Ad[np.ix_(vel, vel)], Ad[np.ix_(vel, pre)], Ad[np.ix_(pre, vel)], Ad[np.ix_(pre, pre)]


def test_schur_shat_variants_dense():
    # schur_shat = 0: S_hat = C; 1: Eq. 10 C - diag(B diag(A_u)^-1 B^T); 2: the explicitly
    # assembled C - B diag(A_u)^-1 B^T (PETSc variant).  m_S = SPAI0:
    # m_i = S_ii / sum_j S_ij^2 -- all three from numpy dense products
    n = 4
    A, Au, Bt, B, C = _stokes_split(n)
    X = B @ np.diag(1.0 / np.diag(Au)) @ Bt
    want = {0: C, 1: C - np.diag(np.diag(X)), 2: C - X}
    diags = {}
    for mode, Sh in want.items():
        S = oracle.Solver(A, precond=oracle.PC_SCHUR, schur_shat=mode, hier_f32=0, vec_f32=0)
        d, m = S.schur_vectors()
        assert np.allclose(d, np.diag(Sh), rtol=1e-14, atol=0), mode
        assert np.allclose(m, np.diag(Sh) / (Sh ** 2).sum(axis=1), rtol=1e-13, atol=0), mode
        diags[mode] = d
    assert np.array_equal(diags[1], diags[2])  # same diagonal terms, same order
    assert not np.allclose(want[2], np.diag(np.diag(want[2])))  # the full S_hat has off-diagonal fill


# ---- C10b Schur split by a general scalar pressure mask (R21) ----
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


@pytest.mark.parametrize("h32", [0, 1])
def test_pmask_interleaved_is_the_v2_split(rng, h32):
    # mask = component 3 of every (u,v,w,p) block: the scalar split is V2's term for term
    # (same A_u, same S_hat / m_S, same preconditioner bits)
    n = 6
    ptr, col, val = gen.matrix(gen.STOKES, n)
    A = oracle.Mat.from_arrays(ptr, col, val)
    mask = (np.arange(4 * n ** 3) % 4 == 3)
    kw = dict(precond=oracle.PC_SCHUR, solver=oracle.GMRES, coarse_enough=60, hier_f32=h32, vec_f32=h32)
    Sm = oracle.Solver(A, pmask=mask, **kw)
    S2 = oracle.Solver(A, schur_u_scalar=1, **kw)
    assert Sm.levels == S2.levels >= 2
    for a, b in zip(Sm.schur_vectors(), S2.schur_vectors()):
        assert np.array_equal(a, b)
    assert np.array_equal(Sm.schur_Au_amg().dense(), S2.schur_Au_amg().dense())
    for _ in range(2):
        r = rng.standard_normal(4 * n ** 3)
        assert np.array_equal(Sm.precond(r), S2.precond(r))


def test_pmask_scrambled_ordering_exact_schur_identity(rng):
    # a scalar matrix whose pressure unknowns sit at random positions: with an exact
    # (single-level) U-solve the PC satisfies (A z)_u = r_u and
    # (A z)_p - r_p = (S m_S - I)(r_p - B A_u^-1 r_u), S = C - B A_u^-1 B^T (numpy dense);
    # m_S is SPAI0 of Eq. 10's S_hat on the scrambled split
    n = 3
    ptr, col, val = gen.matrix(gen.STOKES, n)
    Ad0 = oracle.Mat.from_arrays(ptr, col, val).dense()
    N = Ad0.shape[0]
    perm = rng.permutation(N)
    Ad = Ad0[np.ix_(perm, perm)]
    mask = (perm % 4 == 3)
    A = oracle.Mat.from_arrays(*_csr_from_dense(Ad))
    S = oracle.Solver(A, pmask=mask, precond=oracle.PC_SCHUR, hier_f32=0, vec_f32=0)
    assert S.levels == 1
    vel, pre = np.flatnonzero(~mask), np.flatnonzero(mask)
    Au, Bt, B, C = Ad[np.ix_(vel, vel)], Ad[np.ix_(vel, pre)], Ad[np.ix_(pre, vel)], Ad[np.ix_(pre, pre)]
    X = B @ np.diag(1.0 / np.diag(Au)) @ Bt
    Sh = C - np.diag(np.diag(X))
    d, mS = S.schur_vectors()
    assert np.allclose(d, np.diag(Sh), rtol=1e-14, atol=0)
    assert np.allclose(mS, np.diag(Sh) / (Sh ** 2).sum(axis=1), rtol=1e-13, atol=0)
    Sx = C - B @ np.linalg.solve(Au, Bt)
    for _ in range(3):
        r = rng.standard_normal(N)
        z = S.precond(r)
        Az = Ad @ z
        assert np.allclose(Az[vel], r[vel], atol=1e-10 * np.abs(r).max())
        expect = (Sx @ np.diag(mS) - np.eye(len(pre))) @ (r[pre] - B @ np.linalg.solve(Au, r[vel]))
        assert np.allclose(Az[pre] - r[pre], expect, atol=1e-10 * np.abs(r).max())


def test_pmask_scrambled_solve_reaches_dense_solution(rng):
    n = 6
    ptr, col, val = gen.matrix(gen.STOKES, n)
    Ad0 = oracle.Mat.from_arrays(ptr, col, val).dense()
    perm = rng.permutation(Ad0.shape[0])
    Ad = Ad0[np.ix_(perm, perm)]
    A = oracle.Mat.from_arrays(*_csr_from_dense(Ad))
    for solver in (oracle.GMRES, oracle.IDRS):
        S = oracle.Solver(A, pmask=(perm % 4 == 3), precond=oracle.PC_SCHUR, solver=solver, coarse_enough=60,
                          hier_f32=0, vec_f32=0)
        assert S.levels >= 2
        b = rng.standard_normal(Ad.shape[0])
        r = S.solve(b, rtol=1e-10)
        xd = np.linalg.solve(Ad, b)
        assert r.converged and np.linalg.norm(r.x - xd) <= 1e-6 * np.linalg.norm(xd)


def test_schur_shat_interior_closed_form():
    # Stokes generator: Shat_ii = -6 - (#neighbours) (1/(2h))^2 / (6/h^2) = -6 - k/24
    n = 6
    ptr, col, val = gen.matrix(gen.STOKES, n)
    A = oracle.Mat.from_arrays(ptr, col, val)
    S = oracle.Solver(A, precond=oracle.PC_SCHUR, hier_f32=0, vec_f32=0)
    d, m = S.schur_vectors()
    k = np.diff(ptr) - 1
    assert np.allclose(d, -6.0 - k / 24.0, rtol=1e-15)
    i = 2 + n * (2 + n * 2)
    assert d[i] == -6.25


def test_schur_block_lu_identity(rng):
    # exact U-solve (single level): z = apply(r) satisfies (A z)_u = r_u and
    # (A z)_p - r_p = (S m_S - I)(r_p - B A_u^-1 r_u), S = C - B A_u^-1 B^T (Eq. 9)
    n = 3
    ptr, col, val = gen.matrix(gen.STOKES, n)
    A = oracle.Mat.from_arrays(ptr, col, val)
    S = oracle.Solver(A, precond=oracle.PC_SCHUR, hier_f32=0, vec_f32=0)
    Ad = A.dense()
    vel = np.array([q for q in range(4 * n ** 3) if q % 4 != 3])
    pre = np.array([q for q in range(4 * n ** 3) if q % 4 == 3])
    Au, Bt, B, C = Ad[np.ix_(vel, vel)], Ad[np.ix_(vel, pre)], Ad[np.ix_(pre, vel)], Ad[np.ix_(pre, pre)]
    _, mS = S.schur_vectors()
    Sx = C - B @ np.linalg.solve(Au, Bt)
    for _ in range(3):
        r = rng.standard_normal(4 * n ** 3)
        z = S.precond(r)
        Az = Ad @ z
        assert np.allclose(Az[vel], r[vel], atol=1e-10 * np.abs(r).max())
        expect = (Sx @ np.diag(mS) - np.eye(len(pre))) @ (r[pre] - B @ np.linalg.solve(Au, r[vel]))
        assert np.allclose(Az[pre] - r[pre], expect, atol=1e-10 * np.abs(r).max())


def test_schur_decoupled_exact_one_iteration(rng):
    # B = 0, C diagonal: Shat = C, m_S = C^-1 exactly, single-level U-solve is exact ->
    # the preconditioner is A^-1 and GMRES converges in 1 iteration (SURVEY.md C10 pin).
    n = 3
    ptr, col, val = gen.matrix(gen.STOKES, n)
    val = val.copy()
    for i in range(n ** 3):
        for k in range(ptr[i], ptr[i + 1]):
            val[k][3, :3] = 0
            val[k][:3, 3] = 0
            val[k][3, 3] = -6.0 - 0.1 * i if col[k] == i else 0.0
    A = oracle.Mat.from_arrays(ptr, col, val)
    S = oracle.Solver(A, precond=oracle.PC_SCHUR, solver=oracle.GMRES, hier_f32=0, vec_f32=0)
    res = S.solve(rng.standard_normal(4 * n ** 3), rtol=1e-10)
    assert res.converged and res.iters == 1


def test_schur_scalar_u_solver_expansion(rng):
    # V2 (Listing V2): the U-solver hierarchy on the scalar expansion of A_u -- the same
    # operator (dense equality), zero entries inside stored blocks not stored (R18), and
    # the V2 / V3 preconditioned solves both reach the dense solution
    n = 5
    ptr, col, val = gen.matrix(gen.STOKES, n)
    A = oracle.Mat.from_arrays(ptr, col, val)
    S2 = oracle.Solver(A, precond=oracle.PC_SCHUR, solver=oracle.GMRES, schur_u_scalar=1, coarse_enough=40,
                       hier_f32=0, vec_f32=0)
    Au, As = S2.schur_Au(), S2.schur_Au_amg()
    assert As.info()[2] == 1 and As.info()[0] == 3 * n ** 3
    assert np.array_equal(As.dense(), Au.dense())
    sp, sc, sv = As.to_arrays()
    assert np.count_nonzero(sv.reshape(-1) == 0.0) == 0  # Laplacian x I3: only the diagonal couplings
    assert S2.levels >= 2
    b = rng.standard_normal(4 * n ** 3)
    xd = np.linalg.solve(A.dense(), b)
    for S in (S2, oracle.Solver(A, precond=oracle.PC_SCHUR, solver=oracle.GMRES, coarse_enough=40,
                                hier_f32=0, vec_f32=0)):
        r = S.solve(b, rtol=1e-10)
        assert r.converged and np.linalg.norm(r.x - xd) <= 1e-6 * np.linalg.norm(xd)


# ---------------------------------------------------------------- C11 Krylov
@pytest.mark.parametrize("solver", [oracle.CG, oracle.BICGSTAB, oracle.GMRES, oracle.IDRS])
def test_identity_one_iteration(rng, solver):
    n = 50
    A = oracle.Mat.from_arrays(np.arange(n + 1, dtype=np.int32), np.arange(n, dtype=np.int32),
                               np.tile(np.eye(2), (n, 1, 1)))
    S = oracle.Solver(A, solver=solver, precond=oracle.PC_NONE)
    b = rng.standard_normal(2 * n)
    r = S.solve(b, rtol=1e-10)
    assert r.converged and r.iters == 1 and np.allclose(r.x, b)


def test_zero_rhs(rng):
    ptr, col, val = gen.matrix(gen.POISSON3, 4)
    A, S = _solver(ptr, col, val, solver=oracle.CG)
    r = S.solve(np.zeros(192), x0=rng.standard_normal(192))
    assert r.converged and r.iters == 0 and r.relres_true == 0 and not r.x.any()


@pytest.mark.parametrize("solver,kind", [(oracle.CG, gen.POISSON3), (oracle.BICGSTAB, gen.STOKES),
                                         (oracle.GMRES, gen.STOKES), (oracle.IDRS, gen.STOKES)])
def test_dense_solve_small(rng, solver, kind):
    # <= 2000 unknowns, coarse_enough lowered so that a real hierarchy is exercised (C7 caveat)
    n = 7 if kind == gen.POISSON3 else 6
    ptr, col, val = gen.matrix(kind, n)
    A = oracle.Mat.from_arrays(ptr, col, val)
    pc = oracle.PC_SCHUR if solver in (oracle.GMRES, oracle.IDRS) else oracle.PC_AMG
    S = oracle.Solver(A, solver=solver, precond=pc, coarse_enough=64)
    assert S.levels >= 2
    b = rng.standard_normal(len(ptr) * 0 + (len(ptr) - 1) * val.shape[-1])
    r = S.solve(b, rtol=1e-10)
    xd = np.linalg.solve(A.dense(), b)
    assert r.converged and r.relres_true <= 1e-10
    assert np.linalg.norm(r.x - xd) <= 1e-6 * np.linalg.norm(xd)


def _dense_bsr(M):
    n = M.shape[0]
    ptr = np.arange(0, n * n + 1, n, dtype=np.int32)
    col = np.tile(np.arange(n, dtype=np.int32), n)
    return ptr, col, M.reshape(n * n, 1, 1).copy()


@pytest.mark.parametrize("solver", ["cg", "bicgstab"])
def test_krylov_iterates_match_scipy(rng, solver):
    # unpreconditioned CG (SPD) and BiCGStab (nonsymmetric): the oracle's iterate after k
    # steps equals scipy.sparse.linalg's textbook iterate after k steps (an independent
    # implementation of Hestenes-Stiefel CG and van der Vorst's BiCGStab, shadow r^ = r_0)
    import scipy.sparse.linalg as sla
    n = 30
    G = rng.standard_normal((n, n))
    M = G @ G.T + n * np.eye(n) if solver == "cg" else G + 2.0 * np.sqrt(n) * np.eye(n)
    b = rng.standard_normal(n)
    ptr, col, val = _dense_bsr(M)
    for k in range(1, 7):
        A = oracle.Mat.from_arrays(ptr, col, val)
        S = oracle.Solver(A, solver=oracle.CG if solver == "cg" else oracle.BICGSTAB, precond=oracle.PC_NONE,
                          maxiter=k)
        r = S.solve(b, rtol=1e-14)
        assert r.iters == k
        fn = sla.cg if solver == "cg" else sla.bicgstab
        xs, _ = fn(M, b, x0=np.zeros(n), rtol=1e-300, atol=0.0, maxiter=k)
        assert np.linalg.norm(r.x - xs) <= 1e-11 * np.linalg.norm(xs), (solver, k)


def test_cg_terminates_in_distinct_eigenvalue_count():
    # CG's minimal polynomial property: an SPD matrix with 3 distinct eigenvalues is solved in
    # exactly 3 iterations (to rounding)
    n = 24
    Q, _ = np.linalg.qr(np.random.default_rng(5).standard_normal((n, n)))
    M = Q @ np.diag(np.repeat([1.0, 4.0, 9.0], n // 3)) @ Q.T
    ptr, col, val = _dense_bsr(M)
    S = oracle.Solver(oracle.Mat.from_arrays(ptr, col, val), solver=oracle.CG, precond=oracle.PC_NONE)
    r = S.solve(np.ones(n), rtol=1e-10)
    assert r.converged and r.iters == 3


def test_fp32_emulation_rounds_every_stored_vector(rng):
    # C9 / R10: with vec_f32 the V-cycle's stored vectors are fp32, so the preconditioner
    # output (widened exactly) is fp32-representable; with fp64 vectors it is not
    ptr, col, val = gen.matrix(gen.STOKES, 6)
    A = oracle.Mat.from_arrays(ptr, col, val)
    r = rng.standard_normal((len(ptr) - 1) * 4)
    for pc in (oracle.PC_AMG, oracle.PC_SCHUR):
        z32 = oracle.Solver(A, precond=pc, coarse_enough=64).precond(r)
        assert np.array_equal(z32, z32.astype(np.float32).astype(np.float64))
        z64 = oracle.Solver(A, precond=pc, coarse_enough=64, hier_f32=0, vec_f32=0).precond(r)
        assert not np.array_equal(z64, z64.astype(np.float32).astype(np.float64))
        assert 0 < np.linalg.norm(z32 - z64) <= 1e-4 * np.linalg.norm(z64)


@pytest.mark.parametrize("ortho", [0, 1, 2, 3])
def test_gmres_finite_termination(rng, ortho):
    n = 20
    ptr, col, val = random_bsr(rng, n, 1, density=1.0, dom=10)
    A = oracle.Mat.from_arrays(ptr, col, val)
    S = oracle.Solver(A, solver=oracle.GMRES, gmres_m=n, precond=oracle.PC_NONE, gmres_ortho=ortho)
    b = rng.standard_normal(n)
    r = S.solve(b, rtol=1e-12)
    assert r.converged and r.iters <= n
    xd = np.linalg.solve(A.dense(), b)
    assert np.linalg.norm(r.x - xd) <= 1e-9 * np.linalg.norm(xd)


def test_gmres_two_pass_orthogonalisation_is_arnoldi(rng):
    # the Gram/Cholesky two-pass orthogonalisation (R22) and CGS2 build the same Arnoldi
    # process: on a non-normal operator without preconditioning the residual history (the
    # GMRES minimal residuals, unique in exact arithmetic) agrees step by step, and with the
    # AMG preconditioners the iteration counts and solutions agree
    n = 60
    ptr, col, val = random_bsr(rng, n, 1, density=0.2, dom=3)
    A = oracle.Mat.from_arrays(ptr, col, val)
    b = rng.standard_normal(n)
    # (R23, gmres_ortho = 2: the first pass's dots on the fp32-rounded basis; R28, 3: on the
    # fp16-rounded basis -- only the projection coefficients change, the Arnoldi relation and
    # R stay exact, so the minimal residuals agree step by step as well)
    hs = []
    for ortho in (0, 1, 2, 3):
        S = oracle.Solver(A, solver=oracle.GMRES, gmres_m=40, precond=oracle.PC_NONE, gmres_ortho=ortho)
        hs.append(np.array(S.solve(b, rtol=1e-10, history=True).history))
    for o in (1, 2, 3):
        k = min(len(hs[0]), len(hs[o]))
        assert abs(len(hs[0]) - len(hs[o])) <= 1
        if o < 3:
            assert np.allclose(hs[0][:k], hs[o][:k], rtol=1e-6, atol=1e-14)
        else:  # fp16 coefficients: the same history to 1e-6 down to 1e-8, within 1e-4 below it
            hi = hs[0][:k] > 1e-8
            assert np.allclose(hs[0][:k][hi], hs[o][:k][hi], rtol=1e-6, atol=0)
            assert np.allclose(hs[0][:k], hs[o][:k], rtol=1e-4, atol=1e-14)
    for kind, pc in ((gen.STOKES, oracle.PC_SCHUR), (gen.POISSON3, oracle.PC_AMG)):
        ptr, col, val = gen.matrix(kind, 8)
        A = oracle.Mat.from_arrays(ptr, col, val)
        b = rng.standard_normal((len(ptr) - 1) * val.shape[-1])
        rs = [oracle.Solver(A, solver=oracle.GMRES, precond=pc, gmres_ortho=o, coarse_enough=60).solve(b, rtol=1e-10)
              for o in (0, 1, 2, 3)]
        for o in (1, 2, 3):
            assert rs[0].iters == rs[o].iters and rs[0].converged and rs[o].converged
            assert np.linalg.norm(rs[0].x - rs[o].x) <= 1e-8 * np.linalg.norm(rs[0].x)


# ---- IDR(s) (Table 1: the paper's outer solver; reading R17) ----
def test_idrs_shadow_space_rng_and_orthonormal():
    # the oracle's own counter RNG equals gen/'s (same formula, written twice) and the
    # shadow space is orthonormal; P_0 is the normalised draw vector
    n, s, base = 300, 5, 64 * 1234
    P = oracle.idrs_shadow(n, s, base)
    assert np.abs(P @ P.T - np.eye(s)).max() <= 1e-14
    d0 = np.array([gen.n01(6, base * n + i) for i in range(n)])
    assert np.allclose(P[0], d0 / np.linalg.norm(d0), rtol=0, atol=1e-15)
    d1 = np.array([gen.n01(6, (base + 1) * n + i) for i in range(n)])
    q = d1 - (P[0] @ d1) * P[0]
    assert np.allclose(P[1], q / np.linalg.norm(q), rtol=0, atol=1e-14)


@pytest.mark.parametrize("s", [1, 2, 4, 8])
def test_idrs_finite_termination(rng, s):
    # IDR(s) reaches the exact solution in at most N + N/s products with A (Sonneveld &
    # van Gijzen 2008, Theorem 2.2 / the dimension argument); nonsymmetric dense A
    n = 16
    ptr, col, val = random_bsr(rng, n, 1, density=1.0, dom=6)
    A = oracle.Mat.from_arrays(ptr, col, val)
    S = oracle.Solver(A, solver=oracle.IDRS, idrs_s=s, precond=oracle.PC_NONE)
    b = rng.standard_normal(n)
    r = S.solve(b, rtol=1e-11)
    assert r.converged and r.iters <= n + n // s
    assert np.allclose(r.x, np.linalg.solve(A.dense(), b), rtol=0, atol=1e-9 * np.abs(r.x).max())


def test_idrs_1d_poisson_dense(rng):
    # SPEC.md:325 example: 1-D Poisson n = 50, no preconditioner, vs a dense solve
    ptr, col, val = poisson1d(50)
    A = oracle.Mat.from_arrays(ptr, col, val)
    S = oracle.Solver(A, solver=oracle.IDRS, precond=oracle.PC_NONE)
    b = rng.standard_normal(50)
    r = S.solve(b, rtol=1e-10)
    xd = np.linalg.solve(A.dense(), b)
    assert r.converged and np.linalg.norm(r.x - xd) <= 1e-6 * np.linalg.norm(xd)


def test_idrs_deterministic_and_seeded(rng):
    ptr, col, val = gen.matrix(gen.STOKES, 6)
    A = oracle.Mat.from_arrays(ptr, col, val)
    b = gen.rhs(gen.RHS_LID_NOISE, 6, 4)
    runs = [oracle.Solver(A, solver=oracle.IDRS, precond=oracle.PC_SCHUR, coarse_enough=100, idrs_seed=sd).solve(b)
            for sd in (1234, 1234, 99)]
    assert np.array_equal(runs[0].x, runs[1].x) and runs[0].iters == runs[1].iters
    assert not np.array_equal(runs[0].x, runs[2].x) and all(r.converged for r in runs)


def test_gmres_true_residual_monotone(rng):
    ptr, col, val = gen.matrix(gen.STOKES, 8)
    A = oracle.Mat.from_arrays(ptr, col, val)
    S = oracle.Solver(A, solver=oracle.GMRES, precond=oracle.PC_SCHUR, gmres_m=10, coarse_enough=100)
    r = S.solve(gen.rhs(gen.RHS_LID_NOISE, 8, 4), rtol=1e-8, history=True)
    h = r.history
    assert r.converged and r.iters > 10  # crosses a restart
    assert np.all(np.diff(h) <= 1e-12 * h[:-1] + 1e-15)
    assert h[-1] <= 1e-8


@pytest.mark.parametrize("kind,solver,pc,rhs", [
    (gen.POISSON3, oracle.CG, oracle.PC_AMG, gen.RHS_UNIFORM),
    (gen.STOKES, oracle.BICGSTAB, oracle.PC_AMG, gen.RHS_LID),
    (gen.STOKES, oracle.GMRES, oracle.PC_SCHUR, gen.RHS_FORCE_NOISE),
    (gen.STOKES, oracle.IDRS, oracle.PC_SCHUR, gen.RHS_FORCE_NOISE),  # V3 -> V4 of Table 1
])
def test_fp32_hierarchy_iteration_parity(kind, solver, pc, rhs):
    # mixed precision "does not increase the number of iterations"
    n = 12
    ptr, col, val = gen.matrix(kind, n)
    A = oracle.Mat.from_arrays(ptr, col, val)
    b = gen.rhs(rhs, n, val.shape[-1])
    its = []
    for h32 in (0, 1):
        S = oracle.Solver(A, solver=solver, precond=pc, hier_f32=h32, vec_f32=h32, coarse_enough=200)
        r = S.solve(b, rtol=1e-8)
        assert r.converged and r.relres_true <= 1e-8
        its.append(r.iters)
    assert abs(its[0] - its[1]) <= 1


# ---------------------------------------------------------------- C12 multi-rank
def test_multirank_aggregates_are_slab_local():
    n = 8
    ptr, col, val = gen.matrix(gen.STOKES, n)
    A = oracle.Mat.from_arrays(ptr, col, val)
    for P in (2, 4):
        agg, nc = oracle.aggregate(A, nparts=P)
        rows = n ** 3 // P
        for r in range(P):
            a = agg[r * rows:(r + 1) * rows]
            others = np.concatenate([agg[:r * rows], agg[(r + 1) * rows:]])
            assert not (set(a.tolist()) & set(others.tolist()))
        S = oracle.Solver(A, solver=oracle.GMRES, precond=oracle.PC_SCHUR, nparts=P, coarse_enough=100)
        res = S.solve(gen.rhs(gen.RHS_LID_NOISE, n, 4), rtol=1e-8)
        assert res.converged and res.relres_true <= 1e-8
    a1, n1 = oracle.aggregate(A, nparts=1)
    a0, n0 = oracle.aggregate(A)
    assert np.array_equal(a1, a0)


@pytest.mark.parametrize("ortho", [1, 2])
def test_gmres_gram_near_invariant_subspace(rng, ortho):
    # a spectrum of five values: the Krylov space is invariant after five steps, the new
    # direction lies in span(V) up to rounding and 1 - |R(:,k)|^2 cancels -- the Gram/
    # Cholesky variants' reorthogonalisation safeguard must keep them on CGS2's track (the
    # minimal residual after <= 5 steps reaches rounding level, x equals the dense solution)
    n = 300
    d = rng.choice([1.0, 2.0, 3.0, 5.0, 8.0], n)
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    D = Q @ np.diag(d) @ Q.T
    ptr = (np.arange(n + 1) * n).astype(np.int32)
    col = np.tile(np.arange(n, dtype=np.int32), n)
    A = oracle.Mat.from_arrays(ptr, col, D.reshape(-1, 1, 1))
    b = rng.standard_normal(n)
    xs = np.linalg.solve(D, b)
    for o in (0, ortho):
        r = oracle.Solver(A, solver=oracle.GMRES, precond=oracle.PC_NONE, gmres_ortho=o).solve(b, rtol=1e-12)
        assert r.converged and r.iters <= 6
        assert np.linalg.norm(r.x - xs) <= 1e-10 * np.linalg.norm(xs)
