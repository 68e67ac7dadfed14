"""The distributed path with real separate processes: P ranks launched by
torch.distributed.run, each its own process and CUDA context on cuda:0, exchanging through
the host-staged communicator over a gloo group (amg_comm_init_host).  NCCL itself cannot
run two ranks on one GPU; the data plane here -- distributed setup (allgathers), halo
exchanges, Krylov allreduces -- is the library's, only the transport differs.  Every rank
must take the same iteration count, within +-2 of the oracle's P-slab mode, with the same
slab-local aggregates and true relres <= 1e-8."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("ordered", [0, 1], ids=["sync", "graphs"])
@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("case", ["schur-gmres", "amg-bicgstab", "schur-idrs-ilut"])
def test_multiprocess_solve(P, case, ordered):
    # ordered = 1: the stream-ordered host communicator -- the preconditioner and Krylov-step
    # CUDA graphs capture every halo exchange and allreduce, as with NCCL
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(P),
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "mp_worker.py"), case]
    env = dict(os.environ, MP_ORDERED=str(ordered))
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("{")][-1]
    d = json.loads(line)
    assert d["P"] == P and len(set(d["iters"])) == 1 and all(d["converged"])
    assert d["relres"] <= 1e-8
    assert abs(d["iters"][0] - d["oracle_iters"]) <= 2, d
    assert d["levels"] == d["oracle_levels"] and d["aggregates_equal"], d
    assert d["replay_identical"], d
    assert (d["graphs"] > 0) == bool(ordered), d  # graphs exist exactly when the transport is capturable


def test_bench_two_ranks_host_comm():
    # bench.py's N > 1 path (self-launch under torch.distributed.run, slabs, barrier, max over
    # ranks, rank-0 line, whole-job e2e bytes) with 2 processes on the one GPU through the
    # host-staged communicator -- a check of the multi-rank bench code, not a scaling number
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "3",
           "--cfg", "4", "--n", "24", "--comm", "host"]
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]  # rank 0 only
    d = lines[0]
    assert d["n_gpus"] == 2 and d["converged"] and d["relres_true"] <= 1e-8 and "host-staged" in d["comm"]
    assert d["e2e"]["h2d_bytes_per_step"] == 2 * 4 * 24 ** 3 * 8 and "cpu_baseline" not in d
