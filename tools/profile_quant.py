"""Warm launches of the streaming quantizers on a 4096 x 4096 bf16 tensor for
ncu (development aid): 4 launches per variant, variants in argv order."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_08713_b200 as M

n = 4096
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(n, n, device="cuda", generator=g).to(torch.bfloat16)
for v in (sys.argv[1:] or ["mx16", "mbs_s", "nvfp4"]):
    for _ in range(4):
        M.quantize_tensor(x, M.SchemeConfig(M.Variant(v)), check=False)
torch.cuda.synchronize()
print("done")
