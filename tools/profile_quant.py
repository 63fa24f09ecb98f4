"""Warm launches of the streaming quantizers on a 4096 x 4096 bf16 activation
for ncu captures (development aid): MBS_S, MX16_OAS, OCP32, NVFP4."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_08713_b200 as M

V = M.Variant
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
g = torch.Generator(device="cuda").manual_seed(0)
a = torch.randn(n, n, device="cuda", generator=g).to(torch.bfloat16)
for v in (V.MBS_S, V.MX16_OAS, V.OCP32, V.NVFP4):
    for _ in range(2):
        q = M.quantize_tensor(a, M.SchemeConfig(v), check=False)
torch.cuda.synchronize()
print("done")
