"""Multi-GPU plumbing: contiguous scenario shards, one
process per GPU, and the final gather of every output array to cuda:0.

Scenarios are independent, so the only exchange is the gather.  It is fused
into the solve: rank 0 allocates the full output arrays in ONE device buffer
(`GatherLayout`), exports it once through CUDA IPC (`ipc_export`), every other
rank maps it (`ipc_open`) and passes pointers at its shard's rows as the
solve's output arrays, so the kernel epilogue stores each finished scenario
straight into cuda:0's memory over NVLink.  Host logic only: the shard
arithmetic and the layout are tested on CPU with gloo (tests/test_multi_rank.py).
"""
from __future__ import annotations

from dataclasses import dataclass

# (name, element bytes, elements per scenario given K) of the solve outputs, in buffer order
_ARRAYS = (("lat", 8, lambda K: 3), ("gamma", 4, lambda K: 1), ("M", 4, lambda K: 1),
           ("batch_end", 4, lambda K: K), ("order", 4, lambda K: K), ("w", 8, lambda K: K),
           ("status", 4, lambda K: 1))


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Rank r owns scenarios [r c, min(n, (r+1) c)) with c = ceil(n / world)
    (strong scaling: the total n is fixed)."""
    c = -(-n // world)
    return min(n, rank * c), min(n, (rank + 1) * c)


@dataclass
class GatherLayout:
    """Byte offsets of the output arrays of n scenarios in one buffer (each
    array 256-byte aligned, row-major [n][width])."""
    n: int
    K: int
    want_w: bool = True

    def arrays(self):
        off = 0
        for name, item, width in _ARRAYS:
            if name == "w" and not self.want_w:
                continue
            wd = width(self.K)
            yield name, off, item, wd
            off += (self.n * wd * item + 255) // 256 * 256

    @property
    def nbytes(self) -> int:
        return sum(-(-self.n * wd * item // 256) * 256 for _, _, item, wd in self.arrays())

    def views(self, torch, buf):
        """Typed torch views of a uint8 device buffer of nbytes."""
        dt = {8: {"lat": torch.float64, "w": torch.float64}, 4: {}}
        out = {}
        for name, off, item, wd in self.arrays():
            t = dt[item].get(name, torch.int32)
            v = buf[off: off + self.n * wd * item].view(t)
            out[name] = v.view(self.n, wd) if wd > 1 or name == "lat" else v
        if not self.want_w:
            out["w"] = None
        return out

    def chunk_copies(self, base: int, s0: int, local: "GatherLayout", base_local: int, c0: int, c1: int):
        """(dst, src, bytes) of every array for scenarios [c0, c1) of a rank whose shard starts at
        s0 of this (cuda:0) layout and lives in `local` at base_local -- one contiguous block
        per array, for the copy engines."""
        for (name, off_g, item, wd), (name_l, off_l, _, _) in zip(self.arrays(), local.arrays()):
            assert name == name_l
            yield (base + off_g + (s0 + c0) * wd * item, base_local + off_l + c0 * wd * item, (c1 - c0) * wd * item)

    def rows(self, base: int, s0: int):
        """Raw-address outputs starting at scenario s0 of a (peer-mapped) buffer."""
        from . import Rows
        out = {name: Rows(base + off, wd, item, s0) for name, off, item, wd in self.arrays()}
        if not self.want_w:
            out["w"] = None
        return out
