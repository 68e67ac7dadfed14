"""A/B timing of solver variants on one workload (CUDA events, median of 3 solves after one
warm-up; not a bench line).

  python tools/ab_solve.py [cfg] [n] "field=value,field=value" ["..."] ...
  e.g. python tools/ab_solve.py 5 256 "" "gmres_ortho=2"
Each quoted argument is one variant (amg_params fields, comma-separated; "" = defaults);
ENV:NAME=value items set an environment switch for that variant only.
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import gen  # noqa: E402
import paper_2006_06052_b200 as amg  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
n = int(sys.argv[2]) if len(sys.argv) > 2 else gen.CONFIGS[cfg]["n"]
variants = sys.argv[3:] or [""]
ptr, col, val, bvec = bench.make_problem(cfg, n, 0, n ** 3)
A = amg.BSR.from_numpy(ptr, col, val)
del val
b = torch.as_tensor(bvec, device="cuda")
x = torch.zeros_like(b)
stream = torch.cuda.current_stream()
for var in variants:
    prm = bench.params_for(amg, cfg)
    env = {}
    for item in filter(None, var.split(",")):
        k, v = item.split("=")
        if k.startswith("ENV:"):
            env[k[4:]] = v
            continue
        setattr(prm, k, float(v) if isinstance(getattr(prm, k), float) else int(v))
    saved = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    S = amg.Solver(A, prm)
    x.zero_()
    S.solve(b, x, 1e-8)
    ts = []
    for _ in range(3):
        x.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        rep = S.solve(b, x, 1e-8)
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    mem = S.memory_report()
    print(json.dumps({"variant": var or "default", "ms": statistics.median(ts), "all_ms": ts, "iters": rep.iters,
                      "relres": rep.relres_true, "converged": rep.converged,
                      "alg_GBs": rep.alg_bytes / statistics.median(ts) / 1e6, "device_GB": mem["total"] / 1e9,
                      "counters": S.counters()}), flush=True)
    del S
    torch.cuda.empty_cache()
    for k, v in saved.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v
