"""MBS GEMM time vs macro size (chunk = macro/64 MMAs per accumulator switch)."""
import torch, paper_2603_08713_b200 as M
V = M.Variant
n = 8192
g = torch.Generator(device="cuda").manual_seed(0)
a = torch.randn(n, n, device="cuda", generator=g).to(torch.bfloat16)
w = (torch.randn(n, n, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
out = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
for macro in (64, 128, 256, 512):
    aq = M.quantize_tensor(a, M.SchemeConfig(V.MBS_S, macro_size=macro))
    wq = M.quantize_tensor(w, M.SchemeConfig(V.MBS_S, macro_size=macro))
    for _ in range(3): M.matmul_quantized(aq, wq, M.TileConfig(128, 128, macro), out=out, out_dtype=torch.bfloat16)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5): M.matmul_quantized(aq, wq, M.TileConfig(128, 128, macro), out=out, out_dtype=torch.bfloat16)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"macro {macro}: {ms*1e3:.1f} us {2*n**3/ms/1e9:.0f} TFLOP/s", flush=True)
