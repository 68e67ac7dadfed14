"""Oracle-only reference solves at the BASELINE.json full sizes (test infrastructure).

Writes tests/golden/oracle_full_size.json: for each requested config, the CPU oracle's
iteration count, true relative residual and level sizes at the full grid, so that the
GPU full-size parity tests (tests/test_gpu_full_size.py) can check "+-2 iterations of
the oracle" without re-running a multi-minute single-threaded solve.  Calls only
gen/ (inputs) and oracle/ -- nothing from the CUDA path.

  python tools/oracle_reference_runs.py 4          # cfg 4 at 128^3 (~10 GB host RAM)
  python tools/oracle_reference_runs.py 5          # cfg 5 at 256^3 (~60-100 GB host RAM)
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import gen  # noqa: E402
import oracle  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "oracle_full_size.json")
CFG = {  # BASELINE configs -> generator, rhs, oracle solver / preconditioner, hierarchy precision
    1: (gen.POISSON3, gen.RHS_UNIFORM, oracle.CG, oracle.PC_AMG, 0),
    3: (gen.STOKES, gen.RHS_LID, oracle.BICGSTAB, oracle.PC_AMG, 1),
    4: (gen.STOKES, gen.RHS_FORCE_NOISE, oracle.GMRES, oracle.PC_SCHUR, 1),
    5: (gen.STOKES, gen.RHS_LID_NOISE, oracle.GMRES, oracle.PC_SCHUR, 1),
}


def run(cfg: int, n: int):
    kind, rk, solver, pc, h32 = CFG[cfg]
    t0 = time.time()
    ptr, col, val = gen.matrix(kind, n)
    b = gen.rhs(rk, n, val.shape[-1])
    A = oracle.Mat.from_arrays(ptr, col, val)
    del val
    t1 = time.time()
    S = oracle.Solver(A, oracle.default_params(solver=solver, precond=pc, hier_f32=h32, vec_f32=h32))
    t2 = time.time()
    r = S.solve(b, rtol=1e-8)
    t3 = time.time()
    lv = []
    for l in range(S.levels):
        M = S.level_mat(l, 0)
        lv.append((M.info()[0], M.info()[3]) if M is not None else None)
    return {"cfg": cfg, "n": n, "iters": r.iters, "converged": bool(r.converged), "relres_true": r.relres_true,
            "levels": S.levels, "level_sizes": [list(map(int, v)) if v else None for v in lv],
            "gen_s": t1 - t0, "setup_s": t2 - t1, "solve_s": t3 - t2, "threads": 1,
            "script": "tools/oracle_reference_runs.py"}


if __name__ == "__main__":
    cfgs = [int(a) for a in sys.argv[1:]] or [4]
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for c in cfgs:
        n = gen.CONFIGS[c]["n"]
        res = run(c, n)
        print(json.dumps(res), flush=True)
        data[f"cfg{c}"] = res
        with open(OUT, "w") as f:
            json.dump(data, f, indent=1)
