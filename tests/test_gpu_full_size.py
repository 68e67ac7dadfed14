"""Full-size solve parity (BASELINE.json configs[3], configs[4]) in the launch
configuration bench.py times (bench.params_for).  At these sizes the oracle's own
solve takes minutes to tens of minutes on one core, so:
  * the true relative residual of the GPU solution is recomputed by the ORACLE's SpMV
    on the full matrix (CPU, fp64) -- the north_star bar relres <= 1e-8 at any size;
  * the iteration count is compared (+-2) with the oracle's count at the same size,
    stored in tests/golden/oracle_full_size.json by tools/oracle_reference_runs.py (a
    committed script that calls only gen/ and oracle/);
  * the hierarchy (depth, rows and blocks of every level) matches the oracle's.
"""
import json
import os

import numpy as np
import pytest

import gen
import oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

GOLD = os.path.join(os.path.dirname(__file__), "golden", "oracle_full_size.json")


@pytest.fixture(scope="module")
def amg():
    import paper_2006_06052_b200 as m
    assert torch.cuda.is_available()
    return m


def _golden(cfg):
    if not os.path.exists(GOLD):
        return None
    return json.load(open(GOLD)).get(f"cfg{cfg}")


@pytest.mark.parametrize("cfg", [4, 5])
def test_full_size_solve(amg, cfg):
    import bench
    n = gen.CONFIGS[cfg]["n"]
    g = _golden(cfg)
    if g is None:
        pytest.skip(f"no oracle reference for cfg{cfg} (run tools/oracle_reference_runs.py {cfg})")
    ptr, col, val, bvec = bench.make_problem(cfg, n, 0, n ** 3)
    A = amg.BSR.from_numpy(ptr, col, val)
    S = amg.Solver(A, bench.params_for(amg, cfg))
    del A
    torch.cuda.empty_cache()
    bd = torch.as_tensor(bvec, device="cuda")
    xd = torch.zeros_like(bd)
    rep = S.solve(bd, xd, 1e-8)
    x = xd.cpu().numpy()
    # the hierarchy the oracle built at this size: rows and nnzb of every level (aggregates
    # are deterministic), so equal sizes mean the same coarsening
    sizes = [list(S.level_info(l)[:1]) + [S.level_info(l)[2]] for l in range(rep.levels)]
    assert sizes == [list(v) for v in g["level_sizes"]], (sizes, g["level_sizes"])
    del S, bd, xd
    torch.cuda.empty_cache()
    assert rep.converged
    Ao = oracle.Mat.from_arrays(ptr, col, val)
    del val
    true = np.linalg.norm(bvec - oracle.spmv(Ao, x)) / np.linalg.norm(bvec)
    assert true <= 1e-8, true
    assert abs(true - rep.relres_true) <= 1e-10
    assert abs(rep.iters - g["iters"]) <= 2, (rep.iters, g["iters"])
    assert rep.levels == g["levels"], (rep.levels, g["levels"])
