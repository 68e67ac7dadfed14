"""K1 BSR SpMV parity: CUDA path (through the C ABI) vs the CPU oracle on the same
seeded inputs.  Norm-wise relative error: <= 1e-12 when the
oracle sees the same (fp32-rounded) values, <= 1e-5 for fp32 values vs the fp64
oracle (north_star); fp32 outputs add one fp32 rounding (<= 1e-7)."""
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


def _relerr(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def _r32(a):
    return a.astype(np.float32).astype(np.float64)


def _run(amg, ptr, col, val, x, vt, xt, yt, alpha=1.0, beta=0.0, y0=None):
    tdt = {amg.F32: torch.float32, amg.F64: torch.float64}
    A = amg.BSR.from_numpy(ptr, col, val, dtype=tdt[vt])
    xd = torch.as_tensor(x).to("cuda", tdt[xt])
    n, b = len(ptr) - 1, val.shape[-1]
    yd = (torch.zeros(n * b, dtype=tdt[yt], device="cuda") if y0 is None
          else torch.as_tensor(y0).to("cuda", tdt[yt]))
    amg.bsr_spmv(A, xd, yd, alpha, beta)
    torch.cuda.synchronize()
    return yd.double().cpu().numpy()


@pytest.mark.parametrize("b", [1, 2, 3, 4])
@pytest.mark.parametrize("vt,xt,yt", [(0, 0, 0), (1, 0, 0), (1, 1, 1), (1, 1, 0), (0, 1, 0), (1, 0, 1)])
def test_spmv_random(amg, rng, b, vt, xt, yt):
    for n, dens in ((1, 1.0), (37, 0.2), (300, 0.02), (1000, 0.05)):  # several tiles + ragged tail
        ptr, col, val = random_bsr(rng, n, b, density=dens)
        x = rng.uniform(-1, 1, n * b)
        y0 = rng.standard_normal(n * b)
        for alpha, beta in ((1.0, 0.0), (-0.7, 1.3)):
            y = _run(amg, ptr, col, val, x, vt, xt, yt, alpha, beta, y0)
            vv = _r32(val) if vt == amg.F32 else val
            xx = _r32(x) if xt == amg.F32 else x
            yy = _r32(y0) if yt == amg.F32 else y0
            ref_same = oracle.spmv(oracle.Mat.from_arrays(ptr, col, vv), xx, alpha, beta, yy)
            tol = 1e-12 if yt == amg.F64 else 2e-7
            assert _relerr(y, ref_same) <= tol
            if vt == amg.F32:
                ref64 = oracle.spmv(oracle.Mat.from_arrays(ptr, col, val), x, alpha, beta, y0)
                assert _relerr(y, ref64) <= 1e-5


def test_spmv_beta0_overwrites_nan(amg, rng):
    ptr, col, val = random_bsr(rng, 50, 3, density=0.1)
    y = _run(amg, ptr, col, val, np.ones(150), 0, 0, 0, 1.0, 0.0, np.full(150, np.nan))
    assert np.all(np.isfinite(y))


def test_spmv_empty_rows_and_empty_matrix(amg, rng):
    # rows without blocks produce 0 (beta = 0); n = 0 is a no-op
    ptr = np.array([0, 0, 2, 2, 3], np.int32)
    col = np.array([0, 3, 1], np.int32)
    val = rng.standard_normal((3, 4, 4))
    x = rng.standard_normal(16)
    y = _run(amg, ptr, col, val, x, 0, 0, 0)
    ref = oracle.spmv(oracle.Mat.from_arrays(ptr, col, val), x)
    assert _relerr(y, ref) <= 1e-14 and not y[:4].any() and not y[8:12].any()
    A = amg.BSR.from_numpy(np.zeros(1, np.int32), np.zeros(0, np.int32), np.zeros((0, 3, 3)))
    amg.bsr_spmv(A, torch.zeros(0, dtype=torch.float64, device="cuda"),
                 torch.zeros(0, dtype=torch.float64, device="cuda"))


def test_spmv_worked_example(amg):
    from conftest import golden
    g = golden("worked_example.json")
    y = _run(amg, np.array(g["bsr_ptr"]), np.array(g["bsr_col"]), np.array(g["bsr_val"]), np.ones(6), 0, 0, 0)
    assert np.allclose(y, g["y_ones"], rtol=0, atol=1e-14)


def test_spmv_bad_args(amg):
    A = amg.BSR.from_numpy(np.array([0, 1], np.int32), np.array([0], np.int32), np.ones((1, 5, 5)))
    with pytest.raises(amg.AmgError) as e:
        amg.bsr_spmv(A, torch.ones(5, dtype=torch.float64, device="cuda"),
                     torch.ones(5, dtype=torch.float64, device="cuda"))
    assert e.value.status == amg.EINVAL


@pytest.mark.parametrize("b", [3, 4])
@pytest.mark.parametrize("n", [16, 24])
def test_spmv_cfg2_pattern(amg, b, n):
    # cfg 2 distribution (27-point, N(0,1) + 30 I) at reduced n: f64/f64 and f32-values/f64-x
    ptr, col, val = gen.matrix(gen.RAND27, n, b)
    x = gen.rhs(gen.X_UNIFORM, n, b)
    ref = oracle.spmv(oracle.Mat.from_arrays(ptr, col, val), x)
    assert _relerr(_run(amg, ptr, col, val, x, 0, 0, 0), ref) <= 1e-12
    y32 = _run(amg, ptr, col, val, x, 1, 0, 0)
    assert _relerr(y32, ref) <= 1e-5
    ref32 = oracle.spmv(oracle.Mat.from_arrays(ptr, col, _r32(val)), x)
    assert _relerr(y32, ref32) <= 1e-12


@pytest.mark.parametrize("b", [4])
def test_spmv_cfg2_full_size(amg, b):
    # BASELINE configs[1] at its full size (128^3, 55.7M blocks), in the bench's launch
    # configuration (fp32 values x fp64 x); the oracle computes every row
    n = 128
    ptr, col, val = gen.matrix(gen.RAND27, n, b)
    x = gen.rhs(gen.X_UNIFORM, n, b)
    ref = oracle.spmv(oracle.Mat.from_arrays(ptr, col, val), x)
    y = _run(amg, ptr, col, val, x, 1, 0, 0)
    assert _relerr(y, ref) <= 1e-5
    y = _run(amg, ptr, col, val, x, 0, 0, 0)
    assert _relerr(y, ref) <= 1e-12


# ---- TMA-staged plan path (bsr_plan_create / bsr_plan_spmv) ----
def _run_plan(amg, ptr, col, val, x, vt, xt, yt, alpha=1.0, beta=0.0, y0=None):
    tdt = {amg.F32: torch.float32, amg.F64: torch.float64}
    A = amg.BSR.from_numpy(ptr, col, val, dtype=tdt[vt])
    P = amg.SpmvPlan(A)
    xd = torch.as_tensor(x).to("cuda", tdt[xt])
    n, b = len(ptr) - 1, val.shape[-1]
    yd = (torch.zeros(n * b, dtype=tdt[yt], device="cuda") if y0 is None
          else torch.as_tensor(y0).to("cuda", tdt[yt]))
    P(xd, yd, alpha, beta)
    torch.cuda.synchronize()
    return yd.double().cpu().numpy()


@pytest.mark.parametrize("b", [1, 2, 3, 4])
@pytest.mark.parametrize("vt,xt,yt", [(0, 0, 0), (1, 0, 0), (1, 1, 1)])
def test_plan_spmv_random(amg, rng, b, vt, xt, yt):
    # n >= 2048 so the TMA tiles are used; ragged last tile, empty rows, long rows
    for n, dens in ((2049, 0.002), (5000, 0.004)):
        ptr, col, val = random_bsr(rng, n, b, density=dens)
        x = rng.uniform(-1, 1, n * b)
        y0 = rng.standard_normal(n * b)
        for alpha, beta in ((1.0, 0.0), (0.5, -2.0)):
            y = _run_plan(amg, ptr, col, val, x, vt, xt, yt, alpha, beta, y0)
            vv = _r32(val) if vt == amg.F32 else val
            xx = _r32(x) if xt == amg.F32 else x
            yy = _r32(y0) if yt == amg.F32 else y0
            ref = oracle.spmv(oracle.Mat.from_arrays(ptr, col, vv), xx, alpha, beta, yy)
            assert _relerr(y, ref) <= (1e-12 if yt == amg.F64 else 2e-7)


def test_plan_spmv_empty_rows(amg, rng):
    n = 4096
    ptr = np.zeros(n + 1, np.int32)
    cols = []
    for i in range(n):
        c = [] if i % 7 == 3 else sorted(set(rng.integers(0, n, 3).tolist()))
        cols.extend(c)
        ptr[i + 1] = ptr[i] + len(c)
    col = np.array(cols, np.int32)
    val = rng.standard_normal((len(col), 3, 3))
    x = rng.standard_normal(3 * n)
    y = _run_plan(amg, ptr, col, val, x, 1, 0, 0, 1.0, 0.0, np.full(3 * n, np.nan))
    ref = oracle.spmv(oracle.Mat.from_arrays(ptr, col, _r32(val)), x)
    assert _relerr(y, ref) <= 1e-12


@pytest.mark.parametrize("b", [3, 4])
def test_plan_spmv_cfg2(amg, b):
    for n in (16, 24):
        ptr, col, val = gen.matrix(gen.RAND27, n, b)
        x = gen.rhs(gen.X_UNIFORM, n, b)
        ref = oracle.spmv(oracle.Mat.from_arrays(ptr, col, val), x)
        assert _relerr(_run_plan(amg, ptr, col, val, x, 0, 0, 0), ref) <= 1e-12
        assert _relerr(_run_plan(amg, ptr, col, val, x, 1, 0, 0), ref) <= 1e-5


@pytest.mark.parametrize("b", [3, 4])
def test_plan_spmv_cfg2_full_size(amg, b):
    # BASELINE configs[1] at full size, the bench's launch configuration (plan: the sliced
    # copy), fp32 values x fp64 x and fp64 x fp64, both block sizes the config names
    n = 128
    ptr, col, val = gen.matrix(gen.RAND27, n, b)
    x = gen.rhs(gen.X_UNIFORM, n, b)
    ref = oracle.spmv(oracle.Mat.from_arrays(ptr, col, val), x)
    assert _relerr(_run_plan(amg, ptr, col, val, x, 1, 0, 0), ref) <= 1e-5
    assert _relerr(_run_plan(amg, ptr, col, val, x, 0, 0, 0), ref) <= 1e-12


# ---- every kernel variant of bsr_lane.cuh, forced (the plan picks one per shape) ----
def _ragged_bsr(rng, n, b):
    """rows of 0, 1..5 and 20..90 blocks (empty, short and long rows in one matrix)"""
    ptr = np.zeros(n + 1, np.int32)
    cols = []
    for i in range(n):
        r = i % 9
        L = 0 if r == 4 else (int(rng.integers(1, 6)) if r < 6 else int(rng.integers(20, 91)))
        c = np.unique(np.concatenate([[i], rng.integers(0, n, L)]))[:max(L, 0)] if L else np.zeros(0, int)
        cols.append(np.sort(c))
        ptr[i + 1] = ptr[i] + len(c)
    col = np.concatenate(cols).astype(np.int32)
    return ptr, col, rng.standard_normal((len(col), b, b))


@pytest.mark.parametrize("var", [0, 1, 2, 3, 4, 5, 6])
@pytest.mark.parametrize("b", [1, 2, 3, 4])
def test_spmv_lane_variants(amg, rng, envvars, var, b):
    envvars(AMG_LANE_VAR=var)
    ptr, col, val = _ragged_bsr(rng, 700, b)
    x = rng.uniform(-1, 1, 700 * b)
    y0 = rng.standard_normal(700 * b)
    for vt, xt, yt in ((0, 0, 0), (1, 0, 0), (1, 1, 1)):
        y = _run(amg, ptr, col, val, x, vt, xt, yt, -0.5, 2.0, y0)
        vv = _r32(val) if vt == amg.F32 else val
        xx = _r32(x) if xt == amg.F32 else x
        yy = _r32(y0) if yt == amg.F32 else y0
        ref = oracle.spmv(oracle.Mat.from_arrays(ptr, col, vv), xx, -0.5, 2.0, yy)
        assert _relerr(y, ref) <= (1e-12 if yt == amg.F64 else 2e-7), (var, b, vt, xt, yt)


def _long_rows_bsr(rng, n, b):
    """a few hundred rows of 0..300 blocks (the coarse restrictions' shape: R_l rows of
    150-240 blocks on a few hundred coarse rows), empty rows included"""
    ptr = np.zeros(n + 1, np.int32)
    cols = []
    for i in range(n):
        L = 0 if i % 11 == 5 else int(rng.integers(1, 301))
        c = np.sort(rng.choice(4 * n, size=L, replace=False)) if L else np.zeros(0, int)
        cols.append(c)
        ptr[i + 1] = ptr[i] + L
    col = np.concatenate(cols).astype(np.int32)
    return ptr, col, rng.standard_normal((len(col), b, b))


@pytest.mark.parametrize("g", [1, 2, 4, 8])
@pytest.mark.parametrize("b", [1, 2, 3, 4])
def test_spmv_warps_per_row(amg, rng, envvars, g, b):
    # warp-per-row kernel with G warps per block row (k_bsr_warps): G partial sums per row
    # meet in shared memory; a ragged last CTA (n not a multiple of 8 / G rows)
    envvars(AMG_LANE_VAR=6, AMG_WARP_G=g)
    n = 301
    ptr, col, val = _long_rows_bsr(rng, n, b)
    m = 4 * n
    x = rng.uniform(-1, 1, m * b)
    y0 = rng.standard_normal(n * b)
    tdt = {amg.F32: torch.float32, amg.F64: torch.float64}
    for vt, xt, yt in ((0, 0, 0), (1, 0, 0), (1, 1, 1)):
        A = amg.BSR.from_numpy(ptr, col, val, dtype=tdt[vt], n_block_cols=m)
        xd = torch.as_tensor(x).to("cuda", tdt[xt])
        yd = torch.as_tensor(y0).to("cuda", tdt[yt])
        amg.bsr_spmv(A, xd, yd, -0.5, 2.0)
        y = yd.double().cpu().numpy()
        vv = _r32(val) if vt == amg.F32 else val
        xx = _r32(x) if xt == amg.F32 else x
        yy = _r32(y0) if yt == amg.F32 else y0
        ref = oracle.spmv(oracle.Mat.from_arrays(ptr, col, vv, n_cols=m), xx, -0.5, 2.0, yy)
        assert _relerr(y, ref) <= (1e-12 if yt == amg.F64 else 2e-7), (g, b, vt, xt, yt)


@pytest.mark.parametrize("b", [2, 3, 4])
def test_spmv_sliced_copy(amg, rng, envvars, b):
    # force the sliced copy (k_bsr_sell) on a small ragged matrix: empty, short and long
    # rows in one slice, ragged last slice
    envvars(AMG_SELL_MIN_ROW=0, AMG_SELL_MAX_ROW=100000, AMG_SELL_MIN_SLICES=1)
    n = 1003
    ptr, col, val = _ragged_bsr(rng, n, b)
    x = rng.uniform(-1, 1, n * b)
    y0 = rng.standard_normal(n * b)
    for vt, xt, yt in ((0, 0, 0), (1, 0, 0), (1, 1, 1)):
        y = _run_plan(amg, ptr, col, val, x, vt, xt, yt, 0.75, -1.0, y0)
        vv = _r32(val) if vt == amg.F32 else val
        xx = _r32(x) if xt == amg.F32 else x
        yy = _r32(y0) if yt == amg.F32 else y0
        ref = oracle.spmv(oracle.Mat.from_arrays(ptr, col, vv), xx, 0.75, -1.0, yy)
        assert _relerr(y, ref) <= (1e-12 if yt == amg.F64 else 2e-7), (b, vt, xt, yt)


@pytest.mark.parametrize("b", [2, 3, 4])
@pytest.mark.parametrize("w,nosort", [(4, 0), (2, 0), (4, 1)])
def test_spmv_interleaved_copy(amg, rng, envvars, b, w, nosort):
    # force the interleaved row-per-lane copy (k_bsr_sellr): empty, short and long rows
    # in one slice, ragged last slice, tail steps of every length, sorted windows or not
    envvars(AMG_LANE_VAR=8, AMG_SELLR_W=w, AMG_SELL_NO_SORT=nosort)
    n = 1003
    ptr, col, val = _ragged_bsr(rng, n, b)
    x = rng.uniform(-1, 1, n * b)
    y0 = rng.standard_normal(n * b)
    for vt, xt, yt in ((0, 0, 0), (1, 0, 0), (1, 1, 1), (0, 1, 0)):
        if vt == amg.F64 and w == 4:
            continue  # fp64 values: 2-wide vectors only
        y = _run_plan(amg, ptr, col, val, x, vt, xt, yt, 0.75, -1.0, y0)
        vv = _r32(val) if vt == amg.F32 else val
        xx = _r32(x) if xt == amg.F32 else x
        yy = _r32(y0) if yt == amg.F32 else y0
        ref = oracle.spmv(oracle.Mat.from_arrays(ptr, col, vv), xx, 0.75, -1.0, yy)
        assert _relerr(y, ref) <= (1e-12 if yt == amg.F64 else 2e-7), (b, vt, xt, yt)


@pytest.mark.parametrize("b", [3, 4])
def test_spmv_interleaved_matches_row_lanes_bitwise(amg, rng, envvars, b):
    # same block-row dots in the same block order as the ROWS lane kernel: identical bits
    n = 777
    ptr, col, val = _ragged_bsr(rng, n, b)
    x = rng.uniform(-1, 1, n * b)
    out = []
    for var in (2, 8):
        envvars(AMG_LANE_VAR=var)
        out.append(_run_plan(amg, ptr, col, val, x, 1, 0, 0))
    assert np.array_equal(out[0], out[1])


# ---- S1: scalar CSR -> BSR on the device (amg_csr_to_bsr) vs the oracle: bit-exact ----
def _rand_csr(rng, n, m, dens, dup=True):
    ptr = [0]
    cols, vals = [], []
    for i in range(n):
        k = rng.binomial(m, dens)
        c = rng.integers(0, m, k)  # unsorted, duplicates allowed (summed in CSR order)
        if not dup:
            c = np.unique(c)
            rng.shuffle(c)
        cols.extend(c.tolist())
        vals.extend(rng.standard_normal(len(c)).tolist())
        ptr.append(len(cols))
    return np.array(ptr, np.int32), np.array(cols, np.int32), np.array(vals)


@pytest.mark.parametrize("b", [1, 2, 3, 4])
@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_csr_to_bsr_parity(amg, rng, b, dt):
    for nb_rows, dens in ((1, 0.5), (7, 0.3), (333, 0.01)):
        n = m = nb_rows * b
        ptr, col, val = _rand_csr(rng, n, m, dens)
        tdt = torch.float64 if dt == "f64" else torch.float32
        vv = val if dt == "f64" else _r32(val)
        bp, bc, bv = amg.csr_to_bsr(n, m, b, torch.as_tensor(ptr, device="cuda"), torch.as_tensor(col, device="cuda"),
                                    torch.as_tensor(vv, device="cuda", dtype=tdt))
        O = oracle.csr_to_bsr(n, m, b, ptr, col, vv)
        op, oc, ov = O.to_arrays()
        assert np.array_equal(bp.cpu().numpy(), op) and np.array_equal(bc.cpu().numpy(), oc)
        if dt == "f64":
            assert np.array_equal(bv.cpu().numpy(), ov)  # same summation order: bit-exact
        else:  # fp32 sums of duplicates (the oracle sums in fp64): equal to 1 ulp-level
            assert np.allclose(bv.double().cpu().numpy(), ov, rtol=1e-6, atol=1e-6)


def test_csr_to_bsr_worked_example_and_errors(amg):
    from conftest import golden
    g = golden("worked_example.json")
    bp, bc, bv = amg.csr_to_bsr(6, 6, 2, torch.as_tensor(np.array(g["csr_ptr"], np.int32), device="cuda"),
                                torch.as_tensor(np.array(g["csr_col"], np.int32), device="cuda"),
                                torch.as_tensor(np.array(g["csr_val"], np.float64), device="cuda"))
    assert bp.cpu().tolist() == g["bsr_ptr"] and bc.cpu().tolist() == g["bsr_col"]
    assert np.array_equal(bv.cpu().numpy(), np.array(g["bsr_val"]))
    with pytest.raises(amg.AmgError) as e:  # not divisible
        amg.csr_to_bsr(3, 3, 2, torch.zeros(4, dtype=torch.int32, device="cuda"),
                       torch.zeros(0, dtype=torch.int32, device="cuda"), torch.zeros(0, dtype=torch.float64, device="cuda"))
    assert e.value.status == amg.EINVAL
    with pytest.raises(amg.AmgError) as e:  # column out of range
        amg.csr_to_bsr(2, 2, 1, torch.as_tensor(np.array([0, 1, 1], np.int32), device="cuda"),
                       torch.as_tensor(np.array([5], np.int32), device="cuda"),
                       torch.ones(1, dtype=torch.float64, device="cuda"))
    assert e.value.status == amg.EINVAL
