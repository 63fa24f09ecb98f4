"""One warm launch of each hot kernel for ncu captures (development aid):
quantize (MBS_S, MX16_OAS, NVFP4) on a 4096x4096 bf16 activation and the
tcgen05 GEMM (MBS-H, OCP32, MX16_OAS) at the given size."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_08713_b200 as M

V = M.Variant
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
arms = sys.argv[2].split(",") if len(sys.argv) > 2 else ["mbs_h", "ocp32", "mx16_oas"]
g = torch.Generator(device="cuda").manual_seed(0)
a = torch.randn(n, n, device="cuda", generator=g).to(torch.bfloat16)
w = (torch.randn(n, n, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
pairs = {"mbs_h": (V.MBS_S, V.MBS_D), "ocp32": (V.OCP32, V.OCP32), "mx16_oas": (V.MX16_OAS, V.MX16_OAS),
         "nvfp4": (V.NVFP4, V.NVFP4)}
for arm in arms:
    va, vw = pairs[arm]
    wq = M.quantize_tensor(w, M.SchemeConfig(vw))
    for _ in range(2):
        aq = M.quantize_tensor(a, M.SchemeConfig(va), check=False)
        c = M.matmul_quantized(aq, wq, out_dtype=torch.bfloat16)
    torch.cuda.synchronize()
print("done")
