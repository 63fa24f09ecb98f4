"""Pinned host <-> device copy bandwidth (H2D, D2H, and both at once on two
streams): the PCIe bound of bench.py's e2e number (development aid)."""
import torch, time
n = 256 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory(); h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda"); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps
h2d = t(lambda: d.copy_(h, non_blocking=True)); print("H2D GB/s", n / h2d / 1e9)
d2h = t(lambda: h.copy_(d, non_blocking=True)); print("D2H GB/s", n / d2h / 1e9)
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
bt = t(both); print("duplex GB/s each", n / bt / 1e9)
