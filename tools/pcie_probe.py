#!/usr/bin/env python
"""PCIe probe (run on the GPU box): pinned H2D / D2H bandwidth alone and together, and the bound the
end-to-end byte mix (2568 B in, 2084 B out per C4 scenario) puts on sdedge_solve_batch_host."""
import torch, time
dev = torch.device("cuda:0")
n = 1 << 30
h_in = torch.empty(n, dtype=torch.uint8).pin_memory(); h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_in = torch.empty(n, dtype=torch.uint8, device=dev); d_out = torch.empty(n, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f, reps=5):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps
def h2d():
    with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
def both():
    h2d(); d2h()
a = t(h2d); b = t(d2h); c = t(both)
print(f"H2D alone {n/a/1e9:.1f} GB/s; D2H alone {n/b/1e9:.1f} GB/s; both at once: {n/c/1e9:.1f} GB/s each direction")
# the e2e mix: 2568 B in, 2084 B out per scenario
m_in, m_out = int(n * 2568 / 2568), int(n * 2084 / 2568)
def mix():
    with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2): h_out[:m_out].copy_(d_out[:m_out], non_blocking=True)
e = t(mix)
print(f"e2e byte mix (2568 in : 2084 out): {m_in/e/1e9:.1f} GB/s in -> {m_in/e/2568/1e6:.1f} M scenarios/s bound")
