"""Warm grouped expert launches (GPT-OSS gate_up, 64 experts, 8 tokens) for
ncu: MBS-H then NVFP4 (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_08713_b200 as M
V = M.Variant
g = torch.Generator(device="cuda").manual_seed(0)
wd = [(torch.randn(5760, 2880, device="cuda", generator=g) * 0.02).to(torch.bfloat16) for _ in range(64)]
for av, wv in ((V.MBS_S, V.MBS_D), (V.NVFP4, V.NVFP4)):
    wq = [M.quantize_tensor(w, M.SchemeConfig(wv), check=False) for w in wd]
    toks = [M.quantize_tensor(torch.randn(8, 2880, device="cuda", generator=g).to(torch.bfloat16), M.SchemeConfig(av)) for _ in range(64)]
    for _ in range(3):
        M.matmul_quantized_grouped(toks, wq, out_dtype=torch.bfloat16, check=False)
    torch.cuda.synchronize()
print("done")
