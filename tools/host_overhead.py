"""Host-side cost per public-API call (development aid): wall time of N eager
calls (no graph) vs the device time of the same launches in a CUDA graph."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_08713_b200 as M

V = M.Variant
g = torch.Generator(device="cuda").manual_seed(0)
for (m, k, n) in ((16, 2880, 5760), (4096, 4096, 4096)):
    a = torch.randn(m, k, device="cuda", generator=g).to(torch.bfloat16)
    w = M.quantize_tensor((torch.randn(n, k, device="cuda", generator=g) * 0.02).to(torch.bfloat16), M.SchemeConfig(V.MBS_D))
    out = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    cfg = M.SchemeConfig(V.MBS_S)
    def q(): return M.quantize_tensor(a, cfg, check=False)
    aq = q()
    def mm(): return M.matmul_quantized(aq, w, out=out, out_dtype=torch.bfloat16, check=False)
    def both(): return M.matmul_quantized(q(), w, out=out, out_dtype=torch.bfloat16, check=False)
    for name, fn in (("quantize_tensor", q), ("matmul_quantized", mm), ("quantize+matmul", both)):
        for _ in range(20): fn()
        torch.cuda.synchronize()
        n_it = 200
        t0 = time.perf_counter()
        for _ in range(n_it): fn()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            for _ in range(20): fn()
        gr.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); gr.replay(); e1.record(); torch.cuda.synchronize()
        dev_us = e0.elapsed_time(e1) / 20 * 1e3
        print(f"{m}x{k}x{n} {name:18s} host {1e6*(t1-t0)/n_it:7.1f} us/call  eager wall {1e6*(t2-t0)/n_it:7.1f}  device {dev_us:7.1f} us", flush=True)
