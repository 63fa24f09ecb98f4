"""One small call of every product kernel (for compute-sanitizer runs):
quantizers (6 variants + MBS-D LUT), dequantizer, QSNR evaluator, the plain /
NVFP4 / MBS tcgen05 GEMMs (direct, swap-AB + split-K, grouped MBS and NVFP4,
fused quantize+GEMM), the exact GEMM."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_08713_b200 as M

V = M.Variant
g = torch.Generator(device="cuda").manual_seed(0)
a = torch.randn(256, 512, device="cuda", generator=g).to(torch.bfloat16)
w = (torch.randn(384, 512, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
qs = {}
for v in ("ocp32", "mx16", "mx16_oas", "mbs_s", "mbs_d", "nvfp4"):
    qs[v] = (M.quantize_tensor(a, M.SchemeConfig(V(v))), M.quantize_tensor(w, M.SchemeConfig(V(v))))
    M.dequantize_tensor(qs[v][0])
    M.qsnr_quantized(a, qs[v][0])
M.quantize_tensor(w, M.SchemeConfig(V.MBS_D, mbs_mode="lut"))
for va, vb in (("ocp32", "ocp32"), ("mx16_oas", "mx16_oas"), ("nvfp4", "nvfp4"), ("mbs_s", "mbs_d")):
    M.matmul_quantized(qs[va][0], qs[vb][1])
    M.matmul_quantized(qs[va][0], qs[vb][1], out_dtype=torch.bfloat16)
M.matmul_quantized(qs["mbs_d"][0], qs["nvfp4"][1])  # exact CUDA-core path
small = M.quantize_tensor(a[:5], M.SchemeConfig(V.MBS_S))
M.matmul_quantized(small, M.quantize_tensor(torch.randn(1280, 512, device="cuda").to(torch.bfloat16), M.SchemeConfig(V.MBS_D)))
M.matmul_quantized_grouped([small, small], [qs["mbs_d"][1], qs["mbs_d"][1]])
nv_small = M.quantize_tensor(a[:3], M.SchemeConfig(V.NVFP4))
M.matmul_quantized_grouped([nv_small, nv_small], [qs["nvfp4"][1], qs["nvfp4"][1]])
M.quantize_matmul(a, qs["mbs_d"][1])
torch.cuda.synchronize()
print("sanitize smoke ok")
