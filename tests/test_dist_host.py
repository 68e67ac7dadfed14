"""Host-side logic of the multi-GPU path on CPU with the gloo backend (world_size 2):
slab partition, per-rank slab generation == global generation, the NCCL unique-id
broadcast through torch.distributed, and max-over-ranks timing reduction."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import gen
        import paper_2006_06052_b200 as amg
        n = 8
        bd = amg.slab_bounds(n ** 3, world)
        lp, lc, lv = gen.matrix(gen.STOKES, n, None, bd[rank], bd[rank + 1])
        b = gen.rhs(gen.RHS_LID_NOISE, n, 4, bd[rank], bd[rank + 1])
        # unique id: rank 0 makes it, everybody gets the same 128 bytes
        raw = amg.broadcast_unique_id(rank, world, make=lambda: bytes(range(128)))
        # max over ranks of a per-rank "time"
        t = torch.tensor([float(rank + 1)])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        parts = [None] * world
        dist.all_gather_object(parts, (lp.tolist(), lc.tolist(), lv.ravel().tolist(), b.tolist()))
        q.put((rank, raw, float(t.item()), parts if rank == 0 else None, bd))
    finally:
        dist.destroy_process_group()


def test_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert res[0][1] == res[1][1] == bytes(range(128))
    assert res[0][2] == res[1][2] == 2.0
    import gen
    n = 8
    ptr, col, val = gen.matrix(gen.STOKES, n)
    bfull = gen.rhs(gen.RHS_LID_NOISE, n, 4)
    parts = res[0][3]
    bd = res[0][4]
    assert bd == [0, 256, 512]
    cols = np.concatenate([np.array(p[1]) for p in parts])
    vals = np.concatenate([np.array(p[2]) for p in parts])
    assert np.array_equal(cols, col) and np.array_equal(vals, val.ravel())
    assert np.array_equal(np.concatenate([np.array(p[3]) for p in parts]), bfull)
    # local row pointers rebase to the global ones
    off = 0
    for r, p in enumerate(parts):
        lp = np.array(p[0])
        assert np.array_equal(lp + ptr[bd[r]], ptr[bd[r]:bd[r + 1] + 1])


def _ops_worker(rank, world, port, q):
    # the host-staged communicator's callbacks (amg_host_comm_ops over gloo) called the way
    # the library calls them: host buffers behind raw pointers
    import ctypes
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from paper_2006_06052_b200 import _host_ops
        ops = _host_ops()
        vals = (ctypes.c_double * 3)(1.0 + rank, 2.0, -rank)
        assert ops.allreduce_sum(None, vals, 3) == 0
        mine = (ctypes.c_int64 * 2)(10 * rank, 10 * rank + 1)
        allv = (ctypes.c_int64 * (2 * world))()
        assert ops.allgather_i64(None, mine, 2, allv) == 0
        # ring exchange: send rank-stamped bytes to the next rank, receive from the previous
        nxt, prv = (rank + 1) % world, (rank - 1) % world
        sbuf = (ctypes.c_uint8 * 5)(*[rank * 10 + i for i in range(5)])
        rbuf = (ctypes.c_uint8 * 5)()
        sp, rp = (ctypes.c_int32 * 1)(nxt), (ctypes.c_int32 * 1)(prv)
        sb = (ctypes.c_void_p * 1)(ctypes.addressof(sbuf))
        rb = (ctypes.c_void_p * 1)(ctypes.addressof(rbuf))
        sz = (ctypes.c_int64 * 1)(5)
        assert ops.exchange(None, 1, sp, sb, sz, 1, rp, rb, sz) == 0
        assert ops.barrier(None) == 0
        q.put((rank, list(vals), list(allv), list(rbuf)))
    finally:
        dist.destroy_process_group()


def test_host_comm_ops_gloo():
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30500 + (os.getpid() % 1000)
    ps = [ctx.Process(target=_ops_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, vals, allv, rbuf in res:
        assert vals == [1.0 + 2.0 + 3.0, 6.0, -3.0]
        assert allv == [0, 1, 10, 11, 20, 21]
        prv = (rank - 1) % world
        assert rbuf == [prv * 10 + i for i in range(5)]
