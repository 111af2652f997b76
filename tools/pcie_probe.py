"""Pinned host <-> device copy rates (the ceiling of bench.py's e2e leg)."""
import torch
n = 5 * 1023 * 1023
h = [torch.empty(n // 5, dtype=torch.float64).pin_memory() for _ in range(5)]
o = [torch.empty(n // 5, dtype=torch.float64).pin_memory() for _ in range(5)]
d = [torch.empty(n // 5, dtype=torch.float64, device="cuda") for _ in range(5)]
e = [torch.empty(n // 5, dtype=torch.float64, device="cuda") for _ in range(5)]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=10):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
def h2d():
    for x, y in zip(h, d): y.copy_(x, non_blocking=True)
def d2h():
    for x, y in zip(e, o): y.copy_(x, non_blocking=True)
def both():
    with torch.cuda.stream(s1): h2d()
    with torch.cuda.stream(s2): d2h()
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
mb = n * 8 / 1e6
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    ms = t(fn)
    print(f"{name}: {ms:.3f} ms for {mb:.1f} MB each way -> {mb / ms:.1f} GB/s per direction")
