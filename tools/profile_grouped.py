"""One grouped expert-GEMM launch (64 GPT-OSS gate_up experts, 8 tokens each,
MBS-H) after a warm-up launch, for an ncu capture (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_08713_b200 as M

V = M.Variant
g = torch.Generator(device="cuda").manual_seed(0)
m = int(sys.argv[1]) if len(sys.argv) > 1 else 8
n, k, E = 5760, 2880, 64
wq = [M.quantize_tensor((torch.randn(n, k, device="cuda", generator=g) * 0.02).to(torch.bfloat16),
                        M.SchemeConfig(V.MBS_D)) for _ in range(E)]
aq = [M.quantize_tensor(torch.randn(m, k, device="cuda", generator=g).to(torch.bfloat16), M.SchemeConfig(V.MBS_S))
      for _ in range(E)]
for _ in range(2):
    M.matmul_quantized_grouped(aq, wq, out_dtype=torch.bfloat16)
torch.cuda.synchronize()
print("done")
