#!/usr/bin/env python
"""Multi-GPU byte-identity check of the fused gather.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \\
        --master-port P tools/multi_gpu_check.py [--config C4] [--n 1000000]

Every rank solves its contiguous shard (paper_2510_11331_b200/shard.py) with
its outputs stored straight into cuda:0's arrays over NVLink (CUDA IPC); rank 0
then solves ALL n scenarios alone on its own GPU and compares every output
array byte for byte.  Prints one JSON line; exits 1 on any difference."""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import scengen  # noqa: E402
import paper_2510_11331_b200 as sd  # noqa: E402
from paper_2510_11331_b200.shard import GatherLayout, shard_range  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--pair", default=None)
    ap.add_argument("--scenarios", type=int, default=1_000_000)
    ap.add_argument("--precision", type=int, default=0)
    ap.add_argument("--gather", choices=["fused", "chunked"], default="fused")
    ap.add_argument("--chunks", type=int, default=4)
    a = ap.parse_args()
    ws, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    pd, _, _ = scengen.config(a.config, 0, 1, pair=a.pair)
    K = pd["K"]
    s0, s1 = shard_range(a.scenarios, ws, rank)
    _, sc, _ = scengen.config(a.config, s0, s1, pair=a.pair)
    t = {k: torch.from_numpy(np.ascontiguousarray(sc[k])).to(dev) for k in ("I", "p", "g", "alpha")}
    lay = GatherLayout(a.scenarios, K, True)
    if rank == 0:
        buf = torch.full((lay.nbytes,), 0xAB, dtype=torch.uint8, device=dev)   # poison: unwritten rows show
        h = [sd.ipc_export(buf)]
    else:
        h = [None]
    dist.broadcast_object_list(h, src=0, device=dev)
    peer = None
    if rank == 0:
        out = lay.rows(buf.data_ptr(), s0)
    else:
        peer = (sd.ipc_open(*h[0]), h[0][1])
        out = lay.rows(peer[0], s0)
    dist.barrier()
    if a.gather == "fused" or rank == 0:
        sd.solve(pd, t["I"], t["p"], t["g"], t["alpha"], None, out=out, precision=a.precision)
    else:                                   # chunked solves, copy engines move each chunk to cuda:0
        n = s1 - s0
        loc = GatherLayout(n, K, True)
        lbuf = torch.empty(loc.nbytes, dtype=torch.uint8, device=dev)
        lv = loc.views(torch, lbuf)
        st, cs = torch.cuda.current_stream(dev), torch.cuda.Stream(dev)
        for c in range(a.chunks):
            c0, c1 = n * c // a.chunks, n * (c + 1) // a.chunks
            if c1 <= c0:
                continue
            sd.solve(pd, t["I"][c0:c1], t["p"][c0:c1], t["g"][c0:c1], t["alpha"][c0:c1], None,
                     out={k: v[c0:c1] for k, v in lv.items() if v is not None}, precision=a.precision)
            ev = torch.cuda.Event()
            ev.record(st)
            cs.wait_event(ev)
            for dst, src, nb in lay.chunk_copies(peer[0], s0, loc, lbuf.data_ptr(), c0, c1):
                sd.copy_async(dst, src, nb, cs)
        st.wait_stream(cs)
    torch.cuda.synchronize()
    dist.barrier()
    ok, res = True, {}
    if rank == 0:
        g = lay.views(torch, buf)
        _, full, _ = scengen.config(a.config, 0, a.scenarios, pair=a.pair)
        f = {k: torch.from_numpy(np.ascontiguousarray(full[k])).to(dev) for k in ("I", "p", "g", "alpha")}
        ref = sd.solve(pd, f["I"], f["p"], f["g"], f["alpha"], None, precision=a.precision)
        torch.cuda.synchronize()
        for k in ("lat", "gamma", "M", "batch_end", "order", "w", "status"):
            same = bool(torch.equal(g[k].view(torch.uint8) if g[k].dtype != torch.uint8 else g[k],
                                    ref[k].view(torch.uint8)))
            res[k] = same
            ok &= same
        print(json.dumps({"check": "multi_gpu_gather_byte_identity", "world_size": ws, "n": a.scenarios,
                          "config": a.config, "pair": a.pair or "default", "precision": a.precision,
                          "gather": a.gather,
                          "arrays_identical": res, "ok": ok,
                          "shards": [list(shard_range(a.scenarios, ws, r)) for r in range(ws)]}), flush=True)
    dist.barrier()
    if peer is not None:
        sd.ipc_close(*peer)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
