"""The paper's V2 -> V3 -> V4 ladder on B200.

Same outer solver and Schur pressure correction, only the U-solver changes:
  V2  scalar fp64 U-solver hierarchy (Listing V2: builtin<double>)
  V3  3x3-block fp64 hierarchy      (Listing V3: static_matrix<3,3,double>)
  V4  3x3-block fp32 hierarchy      (Listing V4: static_matrix<3,3,float>, fp32 P-solver)
The paper's outer solver is IDR(5) (Table 1); GMRES(30) (the BASELINE cfg 4/5 solver) is
reported beside it.  Prints one JSON line per (cfg, solver, variant) and a table.

  python tools/ladder.py [n ...] [--extra]   (default 128; --extra: the §8(f) #3/#4 variants of V4)
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import gen  # noqa: E402
import paper_2006_06052_b200 as amg  # noqa: E402

VARIANTS = {
    "V2": dict(schur_u_scalar=1, hier_dtype=amg.F64, vcycle_vec_dtype=amg.F64),
    "V3": dict(schur_u_scalar=0, hier_dtype=amg.F64, vcycle_vec_dtype=amg.F64),
    "V4": dict(schur_u_scalar=0, hier_dtype=amg.F32, vcycle_vec_dtype=amg.F32),
}
# SURVEY.md §8(f) #3/#4 variants of the V4 U-solver / P-solver (--extra)
EXTRA = {
    "V4-plain": dict(hier_dtype=amg.F32, vcycle_vec_dtype=amg.F32, coarsening=amg.PLAIN_AGG),
    "V4-ilu0": dict(hier_dtype=amg.F32, vcycle_vec_dtype=amg.F32, smoother=amg.ILU0),
    "V4-plain-ilu0": dict(hier_dtype=amg.F32, vcycle_vec_dtype=amg.F32, coarsening=amg.PLAIN_AGG, smoother=amg.ILU0),
    "V4-shat-full": dict(hier_dtype=amg.F32, vcycle_vec_dtype=amg.F32, schur_shat=2),
    # block ILUT(1e-2, 2) (R25): the paper's U-solver smoother; plain aggregation + ILUT = Listings V2-V4
    "V4-ilut": dict(hier_dtype=amg.F32, vcycle_vec_dtype=amg.F32, smoother=amg.ILUT),
    "V4-plain-ilut": dict(hier_dtype=amg.F32, vcycle_vec_dtype=amg.F32, coarsening=amg.PLAIN_AGG, smoother=amg.ILUT),
}
SOLVERS = {"idrs5": amg.IDRS, "gmres30": amg.GMRES}


def main():
    sizes = [int(a) for a in sys.argv[1:] if not a.startswith("--")] or [128]
    variants = ({"V4": VARIANTS["V4"], **EXTRA} if "--extra" in sys.argv else VARIANTS)
    rows = []
    for n in sizes:
        cfg = 5 if n == 256 else 4
        ptr, col, val, bvec = bench.make_problem(cfg, n, 0, n ** 3)
        A = amg.BSR.from_numpy(ptr, col, val)
        b = torch.as_tensor(bvec, device="cuda")
        for sname, solver in SOLVERS.items():
            for vname, kw in variants.items():
                torch.cuda.synchronize()
                torch.cuda.empty_cache()
                t0 = time.perf_counter()
                S = amg.Solver(A, amg.default_params(solver=solver, precond=amg.PC_SCHUR, **kw))
                torch.cuda.synchronize()
                setup_s = time.perf_counter() - t0
                x = torch.zeros_like(b)
                S.solve(b, x, 1e-8)  # warm-up (graph capture)
                ts = []
                for _ in range(3):
                    x.zero_()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    rep = S.solve(b, x, 1e-8)
                    e1.record()
                    torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1) / 1e3)
                r = {"n": n, "cfg": cfg, "solver": sname, "variant": vname, "setup_s": setup_s,
                     "solve_s": sorted(ts)[1], "iters": rep.iters, "relres_true": rep.relres_true,
                     "converged": bool(rep.converged), "levels": rep.levels, "device_bytes": S.device_bytes, "memory": S.memory_report(),
                     "alg_bytes": rep.alg_bytes}
                rows.append(r)
                print(json.dumps(r), flush=True)
                del S
        del A, b
    print(f"\n{'n':>4s} {'solver':8s} {'var':3s} {'setup s':>8s} {'solve s':>8s} {'its':>4s} {'GB dev':>7s} "
          f"{'solve vs prev':>13s} {'setup vs prev':>13s} {'mem vs prev':>11s}")
    prev = {}
    for r in rows:
        key = (r["n"], r["solver"])
        p = prev.get(key)
        rel = (f"{p['solve_s'] / r['solve_s']:13.2f} {p['setup_s'] / r['setup_s']:13.2f} "
               f"{r['device_bytes'] / p['device_bytes']:11.2f}") if p else ""
        print(f"{r['n']:4d} {r['solver']:8s} {r['variant']:3s} {r['setup_s']:8.3f} {r['solve_s']:8.3f} "
              f"{r['iters']:4d} {r['device_bytes'] / 1e9:7.2f} {rel}")
        prev[key] = r


if __name__ == "__main__":
    main()
