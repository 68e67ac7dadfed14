"""Time the SpMV-type kernel variants on a REAL hierarchy matrix (export of level l's A/P/R
of a cfg-4/5 Schur hierarchy), fp32 values x fp32 vectors, y = A x and y += A x.

  python tools/level_probe.py <n> <level> <which 0=A 1=P 2=R> [reps]
Prints one line per AMG_LANE_VAR variant (and the default plan; 7 sliced, 8 interleaved w4/w2): ms, GB/s.
"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2006_06052_b200 as amg  # noqa: E402

n, level, which = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 20
cfg = 5 if n == 256 else 4
ptr, col, val, _ = bench.make_problem(cfg, n, 0, n ** 3)
S = amg.Solver(amg.BSR.from_numpy(ptr, col, val), bench.params_for(amg, cfg))
del val
p, c, v = S.level_export(level, which)
ncol = S.level_info(level + 1)[0] if which == 1 else S.level_info(level)[0]
del S
torch.cuda.empty_cache()
nr, b = len(p) - 1, v.shape[-1]
print(f"level {level} which {which}: rows {nr} blocks {len(c)} ({len(c) / nr:.2f}/row) b {b}")
x = torch.rand(ncol * b, dtype=torch.float32, device="cuda")
for var in [None, 0, 1, 2, 3, 4, 5, 6, 7, "8w4", "8w2"]:
    os.environ.pop("AMG_SELLR_W", None)
    if var is None:
        os.environ.pop("AMG_LANE_VAR", None)
    elif isinstance(var, str):
        os.environ["AMG_LANE_VAR"] = "8"
        os.environ["AMG_SELLR_W"] = var[2:]
    else:
        os.environ["AMG_LANE_VAR"] = str(var)
    A = amg.BSR.from_numpy(p, c, v, dtype=torch.float32, n_block_cols=ncol)
    plan = amg.SpmvPlan(A)
    y = torch.zeros(nr * b, dtype=torch.float32, device="cuda")
    for beta in (0.0, 1.0):
        for _ in range(3):
            plan(x, y, 1.0, beta)
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                plan(x, y, 1.0, beta)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / reps)
        ms = statistics.median(ts)
        byts = 4 * (nr + 1) + len(c) * (4 + b * b * 4) + ncol * b * 4 + nr * b * 4 * (2 if beta else 1)
        print(f"  var {str(var):>4s} beta {beta:.0f}: {ms:.4f} ms {byts / ms / 1e6:7.0f} GB/s")
    del A, plan, y
