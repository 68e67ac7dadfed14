"""Worker of tests/test_gpu_multiprocess.py (launched by torch.distributed.run, one process
per rank, all on cuda:0): the distributed setup + solve through amg_setup_dist with the
host-staged communicator over a gloo process group (Comm.host) -- real separate processes
exchanging the halos, allgathers and allreduces.  Rank 0 prints one JSON line with the
assembled solution checked against the oracle's P-slab mode (test infrastructure)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import gen  # noqa: E402
import paper_2006_06052_b200 as amg  # noqa: E402

CASES = {
    "schur-gmres": (gen.STOKES, 16, gen.RHS_LID_NOISE, dict(solver=2, precond=1)),
    "amg-bicgstab": (gen.STOKES, 12, gen.RHS_LID, dict(solver=1, precond=0)),
    "schur-idrs-ilut": (gen.STOKES, 12, gen.RHS_LID_NOISE, dict(solver=3, precond=1, smoother=3)),
}


def main():
    case = sys.argv[1]
    dist.init_process_group("gloo")
    rank, P = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    kind, n, rk, kw = CASES[case]
    N = n ** 3
    bd = amg.slab_bounds(N, P)
    lp, lc, lv = gen.matrix(kind, n, None, bd[rank], bd[rank + 1])
    b = lv.shape[-1]
    bvec = gen.rhs(rk, n, b)
    ordered = os.environ.get("MP_ORDERED", "0") == "1"  # stream-ordered host comm: CUDA graphs capture it
    S = amg.Solver(amg.BSR.from_numpy(lp, lc, lv, n_block_cols=N), amg.default_params(**kw),
                   comm=amg.Comm.host(ordered=ordered), row_begin=bd[rank], n_global=N)
    bl = torch.as_tensor(bvec[bd[rank] * b:bd[rank + 1] * b], device="cuda")
    x = torch.zeros_like(bl)
    rep = S.solve(bl, x, 1e-8)
    x2 = torch.zeros_like(bl)
    rep2 = S.solve(bl, x2, 1e-8)  # a second solve replays the captured graphs (ordered mode)
    same = bool(torch.equal(x, x2)) and rep2.iters == rep.iters
    graphs = S.counters()["graphs"]
    parts = [None] * P
    dist.all_gather_object(parts, (rep.iters, rep.converged, x.cpu().numpy(),
                                   [S.level_aggregates(l).tolist() for l in range(S.levels - 1)]))
    if rank == 0:
        import oracle
        ptr, col, val = gen.matrix(kind, n)
        A = oracle.Mat.from_arrays(ptr, col, val)
        xs = np.concatenate([p[2] for p in parts])
        relres = float(np.linalg.norm(bvec - oracle.spmv(A, xs)) / np.linalg.norm(bvec))
        ok = {k: v for k, v in kw.items() if k in ("solver", "precond", "smoother")}
        O = oracle.Solver(A, oracle.default_params(nparts=P, **ok))
        ro = O.solve(bvec, rtol=1e-8)
        aggs_ok = True
        for l in range(O.levels - 1):
            oagg = O.level_agg(l)
            mine = [np.array(p[3][l]) for p in parts]
            agg = mine[0] if len(mine[0]) == len(oagg) and P > 1 else np.concatenate(mine)
            aggs_ok &= bool(np.array_equal(agg, oagg))
        print(json.dumps({"case": case, "P": P, "iters": [p[0] for p in parts], "converged": [p[1] for p in parts],
                          "relres": relres, "oracle_iters": ro.iters, "levels": S.levels, "oracle_levels": O.levels,
                          "aggregates_equal": aggs_ok, "graphs": graphs, "replay_identical": same}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
