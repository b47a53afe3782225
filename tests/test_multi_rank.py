"""World-size-2 gloo tests of the multi-GPU host logic (CPU, -m "not gpu"):
weak-scaling shards are disjoint, cover the stream, regenerate bit-identically
on each rank, solve identically to a single-process run (oracle as the
stand-in solver), and the max-over-ranks timing reduction works."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
import scengen


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import oracle
    s0, s1 = bench.shard(rank, n)
    pd, sc, _ = scengen.config("C3", s0, s1)
    out = oracle.solve_batch(pd, sc, nthreads=2)
    t = bench.max_over_ranks(float(rank + 1) * 0.5, dist, "cpu")
    obj = [None] * ws
    dist.all_gather_object(obj, (rank, s0, s1, out["lat"], out["batch_end"], sc["I"]))
    if rank == 0:
        q.put((t, obj))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shards_gloo():
    import oracle
    oracle.build()
    n = 24
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    t, obj = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert t == 1.0                                   # max over ranks of 0.5, 1.0
    obj.sort(key=lambda x: x[0])
    assert [(o[1], o[2]) for o in obj] == [(0, n), (n, 2 * n)]
    pd, sc, _ = scengen.config("C3", 0, 2 * n)
    ref = oracle.solve_batch(pd, sc, nthreads=4)
    lat = np.concatenate([o[3] for o in obj])
    be = np.concatenate([o[4] for o in obj])
    I = np.concatenate([o[5] for o in obj])
    assert np.array_equal(I, sc["I"])
    assert np.array_equal(lat, ref["lat"]) and np.array_equal(be, ref["batch_end"])
