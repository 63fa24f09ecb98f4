"""One fused quantize+GEMM launch and one plain MBS GEMM launch on the
Llama-3-8B gate_up shape, for an ncu capture of both (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_08713_b200 as M

V = M.Variant
m, n, k = 4096, int(sys.argv[1]) if len(sys.argv) > 1 else 28672, 4096
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(m, k, device="cuda", generator=g).to(torch.bfloat16)
wq = M.quantize_tensor((torch.randn(n, k, device="cuda", generator=g) * 0.02).to(torch.bfloat16), M.SchemeConfig(V.MBS_D))
out = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
aq = M.quantize_tensor(x, M.SchemeConfig(V.MBS_S))
for _ in range(2):
    M.quantize_matmul(x, wq, out=out, out_dtype=torch.bfloat16)
    M.matmul_quantized(aq, wq, out=out, out_dtype=torch.bfloat16)
torch.cuda.synchronize()
print("done")
