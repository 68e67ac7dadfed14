"""Time one config's solve (CUDA events, graphs warm) and optionally bracket one solve with
cudaProfilerStart/Stop for `ncu --profile-from-start off` (gap analysis: the solve's event
time against the sum of its kernels' serialised durations).

  python tools/cfg_solve.py cfg [n] [--reps R] [--profile] [field=value ...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import gen  # noqa: E402
import paper_2006_06052_b200 as amg  # noqa: E402

argv = sys.argv[1:]
if "--reps" in argv:
    i = argv.index("--reps")
    argv = argv[:i] + argv[i + 2:]
args = [a for a in argv if not a.startswith("--")]
cfg = int(args[0]) if args else 3
n = int(args[1]) if len(args) > 1 and "=" not in args[1] else gen.CONFIGS[cfg]["n"]
reps = 10
if "--reps" in sys.argv:
    reps = int(sys.argv[sys.argv.index("--reps") + 1])
ptr, col, val, bvec = bench.make_problem(cfg, n, 0, n ** 3)
A = amg.BSR.from_numpy(ptr, col, val)
prm = bench.params_for(amg, cfg)
for a in args[1:]:
    if "=" in a:
        k, v = a.split("=")
        setattr(prm, k, type(getattr(prm, k))(float(v)) if isinstance(getattr(prm, k), float) else int(v))
S = amg.Solver(A, prm)
b = torch.as_tensor(bvec, device="cuda")
x = torch.zeros_like(b)
s = torch.cuda.current_stream()
for _ in range(3):
    x.zero_()
    S.solve(b, x, 1e-8)
ts = []
for _ in range(reps):
    x.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    rep = S.solve(b, x, 1e-8)
    e1.record(s)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts.sort()
l0 = amg.kernel_launches()
x.zero_()
S.solve(b, x, 1e-8)
nk = amg.kernel_launches() - l0
print(f"cfg{cfg} n={n}: median {ts[len(ts) // 2]:.3f} ms min {ts[0]:.3f} ms, {rep.iters} its, "
      f"relres {rep.relres_true:.2e}, {nk} kernels/solve, alg {rep.alg_bytes / 1e9:.3f} GB")
if "--profile" in sys.argv:
    x.zero_()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    S.solve(b, x, 1e-8)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
