"""World-size-2 gloo tests of the multi-GPU host logic (CPU, -m "not gpu"):
the strong-scaling shards (paper_2510_11331_b200/shard.py) are contiguous,
disjoint and cover the sweep (also for a ragged n), regenerate bit-identically
on each rank, and -- placed at their rows of the one-buffer GatherLayout that
rank 0 exports to the other GPUs -- reproduce a single-process solve (the
oracle stands in for the GPU solver on CPU); the max-over-ranks timing
reduction works."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
import scengen
from paper_2510_11331_b200.shard import GatherLayout, shard_range


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
    s0, s1 = shard_range(n, ws, rank)
    pd, sc, _ = scengen.config("C3", s0, s1)
    out = oracle.solve_batch(pd, sc, nthreads=2)
    t = bench.max_over_ranks(float(rank + 1) * 0.5, dist, "cpu")
    obj = [None] * ws
    dist.all_gather_object(obj, (rank, s0, s1, {k: out[k] for k in ("lat", "gamma", "M", "batch_end", "order",
                                                                   "w", "status")}, sc["I"]))
    if rank == 0:
        q.put((t, obj))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_ranges():
    for n, ws in ((10, 3), (1_000_000, 8), (7, 8), (0, 2)):
        rs = [shard_range(n, ws, r) for r in range(ws)]
        assert rs[0][0] == 0 and rs[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(rs, rs[1:])) and all(a <= b for a, b in rs)


def test_two_rank_shards_gloo():
    import oracle
    oracle.build()
    n = 47                                            # ragged: shards of 24 and 23
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
    assert [(o[1], o[2]) for o in obj] == [(0, 24), (24, 47)]
    pd, sc, _ = scengen.config("C3", 0, n)
    ref = oracle.solve_batch(pd, sc, nthreads=4)
    # rank 0's gather buffer: every shard's rows at their offsets of the one-buffer layout
    lay = GatherLayout(n, pd["K"], True)
    buf = torch.zeros(lay.nbytes, dtype=torch.uint8)
    views = lay.views(torch, buf)
    for _, s0, s1, out, _ in obj:
        for k, v in out.items():
            views[k][s0:s1] = torch.from_numpy(np.ascontiguousarray(v)).view(views[k].dtype)
    I = np.concatenate([o[4] for o in obj])
    assert np.array_equal(I, sc["I"])
    for k in ("lat", "gamma", "M", "batch_end", "order", "w", "status"):
        assert np.array_equal(views[k].numpy(), ref[k]), k
