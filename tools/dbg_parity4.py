import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_08713_b200 as M
dev = torch.device("cuda", 0)
V = M.Variant
def run(m, n, k, va, vb, seed=1):
    g = torch.Generator(device=dev).manual_seed(seed)
    a = torch.randn(m, k, device=dev, generator=g).to(torch.bfloat16)
    w = (torch.randn(n, k, device=dev, generator=g) * 0.02).to(torch.bfloat16)
    wq = M.quantize_tensor(w, M.SchemeConfig(vb))
    aq = M.quantize_tensor(a, M.SchemeConfig(va))
    ex = M.matmul_quantized(aq, wq, exact=True).double()
    c = M.matmul_quantized(aq, wq).double()
    err = (c - ex).abs() > 1e-4 * ex.abs().max()
    print(f"  {va.value}x{vb.value} {m}x{n}x{k}: relfro {float((c-ex).norm()/ex.norm()):.2e} bad {int(err.sum())}", flush=True)
for va, vb in [(V.MBS_S, V.MBS_D), (V.MX16_OAS, V.MBS_D), (V.MBS_S, V.MX16_OAS)]:
    run(4096, 6144, 1024, va, vb)
