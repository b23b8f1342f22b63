"""Pinned host <-> device copy bandwidth of 12.6 MB buffers: H2D alone, D2H alone, both
at once on two streams (the e2e leg's ceiling)."""
import torch, time
n = 8192 * 768
x = torch.empty(n, dtype=torch.bfloat16).pin_memory()
y = torch.empty(n, dtype=torch.bfloat16).pin_memory()
d1 = torch.empty(n, dtype=torch.bfloat16, device="cuda")
d2 = torch.empty(n, dtype=torch.bfloat16, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=50):
    for _ in range(5): fn()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps * 1e6
def h2d():
    with torch.cuda.stream(s1): d1.copy_(x, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): y.copy_(d2, non_blocking=True)
def both():
    h2d(); d2h()
b = n * 2
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    us = t(fn)
    print(f"{name}: {us:.1f} us per 12.6 MB step -> {b / us / 1e3:.1f} GB/s per direction")
