"""Build the sm_100a shared library in-tree (paper_2006_06052_b200/libamgb200.so).

nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo, one shared object with a
plain C ABI (include/amg.h).  Setup kernels (setup*.cu) are compiled with
--fmad=false so that their fp64 arithmetic rounds every product and sum
separately, in the oracle's order (bit-exact aggregates).
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "libamgb200.so")
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl():
    try:
        import nvidia.nccl as nn  # torch's bundled NCCL: the same libnccl.so.2 torch loads
        base = list(nn.__path__)[0]
        return os.path.join(base, "include"), os.path.join(base, "lib")
    except Exception:
        return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def _stale(obj, deps):
    return not os.path.exists(obj) or os.path.getmtime(obj) < max(os.path.getmtime(d) for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    inc_nccl, lib_nccl = _nccl()
    headers = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + [
        os.path.join(ROOT, "include", "amg.h")]
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    jobs = []
    for src in srcs:
        obj = os.path.join(OBJ, os.path.basename(src)[:-3] + ".o")
        flags = ["nvcc", *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                 "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", inc_nccl,
                 "--expt-relaxed-constexpr", "-c", src, "-o", obj]
        if os.path.basename(src).startswith("setup"):
            flags[1:1] = ["--fmad=false"]
        if force or _stale(obj, [src] + headers):
            jobs.append((src, flags))
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
            futs = {ex.submit(subprocess.run, f, capture_output=True, text=True): s for s, f in jobs}
            for fu in cf.as_completed(futs):
                r = fu.result()
                if r.returncode != 0:
                    sys.stderr.write(r.stdout + r.stderr)
                    raise RuntimeError(f"nvcc failed on {futs[fu]}")
                if verbose:
                    sys.stderr.write(r.stderr)
    objs = [os.path.join(OBJ, os.path.basename(s)[:-3] + ".o") for s in srcs]
    if force or jobs or _stale(SO, objs):
        cmd = ["nvcc", *ARCH, "-shared", "-o", SO, *objs, "-L", lib_nccl, "-l:libnccl.so.2",
               "-Xlinker", f"-rpath={lib_nccl}", "-lcudart"]
        subprocess.check_call(cmd)
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
