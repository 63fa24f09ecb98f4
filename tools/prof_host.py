import os, sys, cProfile, pstats
sys.path.insert(0, "/root/repo")
import torch
import paper_2603_08713_b200 as M
V = M.Variant
a = torch.randn(16, 2880, device="cuda").to(torch.bfloat16)
cfg = M.SchemeConfig(V.MBS_S)
w = M.quantize_tensor((torch.randn(5760, 2880, device="cuda") * 0.02).to(torch.bfloat16), M.SchemeConfig(V.MBS_D))
out = torch.empty(16, 5760, device="cuda", dtype=torch.bfloat16)
for _ in range(50): M.matmul_quantized(M.quantize_tensor(a, cfg, check=False), w, out=out, out_dtype=torch.bfloat16, check=False)
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for _ in range(500): M.matmul_quantized(M.quantize_tensor(a, cfg, check=False), w, out=out, out_dtype=torch.bfloat16, check=False)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
