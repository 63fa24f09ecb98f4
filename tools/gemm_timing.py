"""Quick device timing of the tcgen05 GEMM variants (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2603_08713_b200 as M

def run(m, n, k, va, vb, iters=20):
    g = torch.Generator(device="cuda").manual_seed(0)
    a = torch.randn(m, k, device="cuda", generator=g).to(torch.bfloat16)
    b = (torch.randn(n, k, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    aq = M.quantize_tensor(a, M.SchemeConfig(M.Variant(va)))
    bq = M.quantize_tensor(b, M.SchemeConfig(M.Variant(vb)))
    out = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        M.matmul_quantized(aq, bq, out=out, out_dtype=torch.bfloat16)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(iters):
        M.matmul_quantized(aq, bq, out=out, out_dtype=torch.bfloat16)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    print(f"{va}x{vb} {m}x{n}x{k}: {ms*1e3:.1f} us  {2*m*n*k/ms/1e9:.1f} TFLOP/s", flush=True)

for s in (4096, 8192):
    for va, vb in (("ocp32", "ocp32"), ("mx16_oas", "mx16_oas"), ("nvfp4", "nvfp4"), ("mbs_s", "mbs_d")):
        run(s, s, s, va, vb)
