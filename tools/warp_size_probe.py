"""Warp-per-row kernel throughput against matrix size (cfg 3 level-1 shape: 30 blocks per row,
4x4 fp32 values, fp32 x): is the level-1 rate a size (wave / ramp) effect?
  AMG_LANE_VAR=6 python tools/warp_size_probe.py
"""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/", 2)[0])
import paper_2006_06052_b200 as amg  # noqa: E402

rng = np.random.default_rng(0)
for n in (8192, 32768, 131072, 524288):
    L = 30
    base = np.arange(n)[:, None]
    col = np.sort((base + rng.integers(-2000, 2000, (n, L))) % n, axis=1).astype(np.int32)
    col = np.array([np.unique(r)[:L] for r in col], dtype=object)
    ptr = np.zeros(n + 1, np.int32)
    ptr[1:] = np.cumsum([len(r) for r in col])
    col = np.concatenate(col).astype(np.int32)
    val = rng.standard_normal((len(col), 4, 4)).astype(np.float32)
    A = amg.BSR.from_numpy(ptr, col, val, dtype=torch.float32)
    x = torch.rand(4 * n, device="cuda", dtype=torch.float32)
    y = torch.zeros(4 * n, device="cuda", dtype=torch.float32)
    for _ in range(5):
        amg.bsr_spmv(A, x, y)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(20):
        s.record()
        amg.bsr_spmv(A, x, y)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    us = sorted(ts)[len(ts) // 2]
    by = len(col) * 68 + n * 16 * 2
    print(f"n {n:7d} nnzb {len(col):9d}: {us:8.1f} us  {by / us / 1e3:7.0f} GB/s")
