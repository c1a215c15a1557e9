"""Pinned host <-> device copy bandwidth: H2D alone, D2H alone, both concurrently (two streams)."""
import time
import torch

n = 1 << 29  # 4 GiB of fp64
h_in = torch.empty(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.zeros(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d_a.copy_(h_in, non_blocking=True); h_out.copy_(d_b, non_blocking=True)
torch.cuda.synchronize()
def timed(fn):
    torch.cuda.synchronize(); t = time.perf_counter(); fn(); torch.cuda.synchronize(); return time.perf_counter() - t
gb = n * 8 / 1e9
t1 = timed(lambda: d_a.copy_(h_in, non_blocking=True))
t2 = timed(lambda: h_out.copy_(d_b, non_blocking=True))
def both():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
t3 = timed(both)
print(f"H2D {gb/t1:.1f} GB/s, D2H {gb/t2:.1f} GB/s, concurrent {2*gb/t3:.1f} GB/s total ({t3*1e3:.0f} ms for {gb:.1f}+{gb:.1f} GB)")
