"""Multi-process host logic on CPU (gloo, world_size 2): every rank draws
the identical full partner schedule from the reference streams (each GPU
needs the whole map for its RAW/WAR flag waits), handle blobs are gathered
in node order, the NCCL id is broadcast, and max-over-ranks timing works."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch
        from paper_1611_04581_b200 import _native as N
        from paper_1611_04581_b200.engine import (Stream, broadcast_nccl_id, draw_pull_partners,
                                                  exchange_blobs)
        p = 8
        streams = [Stream.make(1, "run/trial0", i, "partner-choice") for i in range(p)]
        sched = np.array([draw_pull_partners(streams) for _ in range(30)])
        gathered = [None] * world
        dist.all_gather_object(gathered, sched.tolist())
        blob = bytes([rank]) * N.HANDLE_BYTES
        blobs = exchange_blobs(blob, rank, world)
        uid = broadcast_nccl_id(rank, world, make=lambda: b"\x07" * N.NCCL_ID_BYTES)
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        q.put((rank, gathered, [b[0] for b in blobs], uid, float(t.item())))
    finally:
        dist.destroy_process_group()


def test_two_rank_host_logic():
    import oracle as O
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    ref = O.pull_schedule(1, "run/trial0", 8, 1, 31)[1:].tolist()
    for rank, gathered, blob_order, uid, tmax in res:
        assert gathered[0] == gathered[1] == ref
        assert blob_order == [0, 1]
        assert uid == b"\x07" * 128
        assert tmax == 2.0
