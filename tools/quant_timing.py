"""Device timing of the streaming quantizers (development aid): a CUDA graph
of launches cycling over 8 distinct 4096 x 4096 bf16 activations (256 MB,
twice the L2), so every launch streams from HBM; algorithmic bytes
(2 read + 0.5 codes + 1/bs scales + 1/128 MBS bytes) per launch."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_08713_b200 as M

V = M.Variant
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
ncol = int(sys.argv[2]) if len(sys.argv) > 2 else n
g = torch.Generator(device="cuda").manual_seed(0)
xs = [torch.randn(n, ncol, device="cuda", generator=g).to(torch.bfloat16) for _ in range(8)]
for v, bpe in ((V.OCP32, 2.53125), (V.MX16, 2.5625), (V.MX16_OAS, 2.5625), (V.MBS_S, 2.5703125), (V.NVFP4, 2.5625)):
    cfg = M.SchemeConfig(v)
    for x in xs:
        M.quantize_tensor(x, cfg, check=False, gemm_layout=True)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    reps = 48
    with torch.cuda.graph(graph):
        for i in range(reps):
            M.quantize_tensor(xs[i % 8], cfg, check=False, gemm_layout=True)
    graph.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    graph.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{v.value:9s} {n}x{ncol} {ms*1e3:7.2f} us  {n*ncol*bpe/ms/1e6:7.0f} GB/s (HBM-cold inputs)", flush=True)
# reference: a device copy of the same bf16 tensor (read + write 2 B/elem each)
dst = torch.empty_like(xs[0])
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph):
    for i in range(48):
        dst.copy_(xs[i % 8])
graph.replay(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record(); graph.replay(); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 48
print(f"copy      {n}x{ncol} {ms*1e3:7.2f} us  {n*ncol*4/ms/1e6:7.0f} GB/s (torch copy_, read+write)", flush=True)
