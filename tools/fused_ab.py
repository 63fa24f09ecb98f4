"""A/B device timing of the activation side of a quantized linear layer
(development aid): MBS-S quantize_tensor + matmul_quantized (two launches)
against quantize_matmul (the quantizer fused into the MBS GEMM launch), on the
Llama-3-8B layer shapes at M = 4096, bf16 out, 8 rotating bf16 activations
(HBM-cold), each variant captured in one CUDA graph."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_08713_b200 as M

V = M.Variant
SHAPES = [("qkv", 4096, 6144, 4096), ("o", 4096, 4096, 4096), ("gate_up", 4096, 28672, 4096),
          ("down", 4096, 4096, 14336)]


def graph_ms(fn, reps=16):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for i in range(3):
            fn(i)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(reps):
            fn(i)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


gen = torch.Generator(device="cuda").manual_seed(0)
tot = {"two": 0.0, "fused": 0.0}
flops = 0.0
for name, m, n, k in SHAPES:
    xs = [torch.randn(m, k, device="cuda", generator=gen).to(torch.bfloat16) for _ in range(8)]
    wq = M.quantize_tensor((torch.randn(n, k, device="cuda", generator=gen) * 0.02).to(torch.bfloat16),
                           M.SchemeConfig(V.MBS_D))
    out = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    cfg = M.SchemeConfig(V.MBS_S)

    def two(i):
        aq = M.quantize_tensor(xs[i % 8], cfg, check=False)
        M.matmul_quantized(aq, wq, out=out, out_dtype=torch.bfloat16, check=False)

    def fused(i):
        M.quantize_matmul(xs[i % 8], wq, cfg, out=out, out_dtype=torch.bfloat16, check=False)

    t2, tf = graph_ms(two), graph_ms(fused)
    tot["two"] += t2
    tot["fused"] += tf
    flops += 2.0 * m * n * k
    print(f"{name:8s} {m}x{n}x{k}: two launches {t2*1e3:8.1f} us   fused {tf*1e3:8.1f} us   "
          f"({2.0*m*n*k/(tf*1e-3)/1e12:.0f} TF/s fused)")
print(f"step: two launches {tot['two']*1e3:.1f} us ({flops/(tot['two']*1e-3)/1e12:.0f} TF/s), "
      f"fused {tot['fused']*1e3:.1f} us ({flops/(tot['fused']*1e-3)/1e12:.0f} TF/s)")
