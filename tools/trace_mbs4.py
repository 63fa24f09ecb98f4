"""Per-warp release / fold-end clock64 trace of k_gemm_mbs2 in CTA 0
(MXQ_LIB_PATH=tools/_bin/libmxq200_trace2.so, built with -DMXQ_GEMM_TRACE=2)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2603_08713_b200 as M
from paper_2603_08713_b200 import _lib

V = M.Variant
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
g = torch.Generator(device="cuda").manual_seed(0)
a = torch.randn(n, n, device="cuda", generator=g).to(torch.bfloat16)
w = (torch.randn(n, n, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
aq = M.quantize_tensor(a, M.SchemeConfig(V.MBS_S))
wq = M.quantize_tensor(w, M.SchemeConfig(V.MBS_D))
M.matmul_quantized(aq, wq, out_dtype=torch.bfloat16)
tr = torch.zeros(512 * 16, dtype=torch.int64, device="cuda")
_lib.lib().mxq_debug_set_trace(tr.data_ptr())
M.matmul_quantized(aq, wq, out_dtype=torch.bfloat16)
torch.cuda.synchronize()
_lib.lib().mxq_debug_set_trace(None)
t = tr.cpu().numpy().reshape(512, 16).astype(np.int64)
nw = int(sys.argv[2]) if len(sys.argv) > 2 else 8
t0 = t[100, 0]
t = t - t0
sl = slice(100, 400)
print("fold START relative to warp 0 (median over chunks 100-400), per warp:")
print([float(np.median(t[sl, w] - t[sl, 0])) for w in range(nw)])
print("fold end relative to warp 0 fold end:")
print([float(np.median(t[sl, 8 + w] - t[sl, 8])) for w in range(nw)])
print("period per warp (release):", [float(np.median(np.diff(t[sl, w]))) for w in range(nw)])
print("fold duration per warp:", [float(np.median(t[sl, 8 + w] - t[sl, w])) for w in range(nw)])
for c in range(200, 206):
    print(c, list(t[c, :nw]), list(t[c, 8:8 + nw]))
