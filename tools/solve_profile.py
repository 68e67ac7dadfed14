"""Per-kernel breakdown of one solve (library CUDA-event profiler, not a bench number).

  python tools/solve_profile.py [cfg] [n] [idrs] [field=value ...]     e.g. 5 256 | 4 128 | 3 64 | 5 256 idrs
Prints every (kernel, bytes/launch) record: launches, total ms, GB/s, share of the solve.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import gen  # noqa: E402
import paper_2006_06052_b200 as amg  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
n = int(sys.argv[2]) if len(sys.argv) > 2 else gen.CONFIGS[cfg]["n"]
ptr, col, val, bvec = bench.make_problem(cfg, n, 0, n ** 3)
A = amg.BSR.from_numpy(ptr, col, val)
del val
prm = bench.params_for(amg, cfg)
for a in sys.argv[3:]:
    if a == "idrs":
        prm.solver = amg.IDRS  # the paper's outer solver (Table 1), s = 5
    elif "=" in a:  # any amg_params field, e.g. gmres_ortho=1
        k, v = a.split("=")
        setattr(prm, k, type(getattr(prm, k))(float(v)) if isinstance(getattr(prm, k), float) else int(v))
S = amg.Solver(A, prm)
del A
for l in range(S.levels):
    nb, bs, za, zp, nc = S.level_info(l)
    print(f"level {l}: n {nb} b {bs} A {za} ({za / max(nb, 1):.1f}/row) P {zp} ({zp / max(nb, 1):.2f}/row) "
          f"R rows {nc} ({zp / max(nc, 1):.1f}/row)")
b = torch.as_tensor(bvec, device="cuda")
x = torch.zeros_like(b)
for _ in range(2):
    x.zero_()
    rep = S.solve(b, x, 1e-8)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
x.zero_()
e0.record()
rep = S.solve(b, x, 1e-8)
e1.record()
torch.cuda.synchronize()
t = e0.elapsed_time(e1)
x.zero_()
amg.profile_begin()
rep = S.solve(b, x, 1e-8)
prof = amg.profile_end()
tot = sum(p["total_ms"] for p in prof)
peak = bench.peaks()[0]
print(f"cfg{cfg} n={n}: solve {t:.2f} ms, {rep.iters} its, relres {rep.relres_true:.2e}, "
      f"alg {rep.alg_bytes / 1e9:.1f} GB -> {rep.alg_bytes / t / 1e6:.0f} GB/s ({rep.alg_bytes / t / 1e6 / peak:.3f} of peak); "
      f"profiled kernels sum {tot:.2f} ms")
print(f"{'kernel':34s} {'MB/launch':>10s} {'launches':>8s} {'ms':>9s} {'us/launch':>9s} {'GB/s':>7s} {'share':>6s}")
for p in sorted(prof, key=lambda p: -p["total_ms"]):
    us = p["total_ms"] / p["launches"] * 1e3
    print(f"{p['kernel']:34s} {p['bytes'] / 1e6:10.2f} {p['launches']:8d} {p['total_ms']:9.3f} {us:9.1f} "
          f"{p['bytes'] / us / 1e3:7.0f} {p['total_ms'] / tot:6.3f}")
