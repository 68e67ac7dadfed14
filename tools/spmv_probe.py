"""Quick cfg-2 SpMV timing (CUDA events, median of reps) for all variants."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/", 2)[0])
import gen  # noqa: E402
import paper_2006_06052_b200 as amg  # noqa: E402


def main(n=128, reps=30, bs=(4, 3), variants=((1, 0), (0, 0), (1, 1))):
    out = []
    for b in bs:
        t0 = time.time()
        if os.environ.get("PROBE_7PT"):  # 7-point 3x3 (velocity block of the Stokes configs)
            n7 = int(os.environ["PROBE_7PT"])
            ptr, col, val = gen.matrix(gen.POISSON3, n7)
            x = gen.rhs(gen.RHS_UNIFORM, n7, 3)
            n = n7
        else:
            ptr, col, val = gen.matrix(gen.RAND27, n, b)
            x = gen.rhs(gen.X_UNIFORM, n, b)
        tg = time.time() - t0
        for vt, xt in variants:
            tdt = {amg.F32: torch.float32, amg.F64: torch.float64}
            A = amg.BSR.from_numpy(ptr, col, val, dtype=tdt[vt])
            xd = torch.as_tensor(x).to("cuda", tdt[xt])
            yd = torch.zeros(len(x), dtype=tdt[xt] if xt == amg.F32 else torch.float64, device="cuda")
            plan = amg.SpmvPlan(A) if not os.environ.get("PROBE_DIRECT") else None
            run = (lambda: plan(xd, yd)) if plan else (lambda: amg.bsr_spmv(A, xd, yd))
            for _ in range(5):
                run()
            ts = []
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            for _ in range(5):
                s.record()
                for _ in range(reps):
                    run()
                e.record(); e.synchronize()
                ts.append(s.elapsed_time(e) / reps)
            t = float(np.median(ts))
            nrows, Z = n ** 3, len(col)
            sv, sx = (4 if vt == amg.F32 else 8), (4 if xt == amg.F32 else 8)
            byts = 4 * (nrows + 1) + Z * (4 + b * b * sv) + nrows * b * sx + nrows * b * (4 if xt == amg.F32 else 8)
            out.append(dict(b=b, vt=vt, xt=xt, ms=t, GBs=byts / t / 1e6, bytes=byts, gen_s=tg))
            print(json.dumps(out[-1]), flush=True)
            del A, xd, yd, plan
            torch.cuda.empty_cache()


if __name__ == "__main__":
    if len(sys.argv) > 1:  # b vt xt reps
        b, vt, xt, reps = map(int, sys.argv[1:5])
        main(reps=reps, bs=(b,), variants=((vt, xt),))
    else:
        main()
