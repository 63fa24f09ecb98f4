"""Achievable read bandwidth on a 4096 x 4096 bf16 tensor (32 MB), HBM-cold
(8 distinct tensors cycled), torch reductions vs our absmax pass."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
xs = [torch.randn(n, n, device="cuda").to(torch.bfloat16) for _ in range(8)]
def t(fn, reps=48):
    g = torch.cuda.CUDAGraph()
    fn(xs[0]); torch.cuda.synchronize()
    with torch.cuda.graph(g):
        for i in range(reps): fn(xs[i % 8])
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3
o = torch.empty(1, device="cuda", dtype=torch.bfloat16)
for name, fn in [("amax", lambda x: torch.amax(x, dim=None, out=o) if False else torch.amax(x)),
                 ("sum", lambda x: x.sum()),
                 ("copy", lambda x: xs[0].copy_(x))]:
    us = t(fn)
    print(f"{name:6s} {us:7.2f} us  {n*n*2/us/1e3:7.0f} GB/s read", flush=True)
