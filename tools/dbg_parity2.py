import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import paper_2603_08713_b200 as M
from test_gpu_bench_parity import bench_inputs, M_TOK
dev = torch.device("cuda", 0)
n, k = int(sys.argv[1]), int(sys.argv[2])
mode = sys.argv[3] if len(sys.argv) > 3 else "outliers"
a, w = bench_inputs(dev, k, n, 77)
if mode == "plain":
    a = torch.randn(M_TOK, k, device=dev).to(torch.bfloat16)
wq = M.quantize_tensor(w, M.SchemeConfig(M.Variant.MBS_D))
aq = M.quantize_tensor(a, M.SchemeConfig(M.Variant.MBS_S))
ex = M.matmul_quantized(aq, wq, exact=True).double()
for it in range(3):
    c = M.matmul_quantized(aq, wq).double()
    rel = ((c - ex).norm(dim=1) / ex.norm(dim=1))
    bad_rows = (rel > 1e-5).nonzero().flatten()
    colrel = ((c - ex).norm(dim=0) / ex.norm(dim=0))
    bad_cols = (colrel > 1e-5).nonzero().flatten()
    print(f"it{it}: relfro {float((c-ex).norm()/ex.norm()):.3e} bad rows {len(bad_rows)} {bad_rows[:12].tolist()} bad cols {len(bad_cols)} {bad_cols[:16].tolist()}")
    if len(bad_cols):
        print("   cols mod 192:", sorted(set((bad_cols % 192).tolist()))[:40], " rows mod 128:", sorted(set((bad_rows % 128).tolist()))[:40])
