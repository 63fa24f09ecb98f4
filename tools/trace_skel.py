"""Stage-level clock64 trace of CTA 0 of k_gemm_mbs2 (MXQ_GEMM_TRACE=1 build):
producer empty-wait, MMA tempty / full waits (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2603_08713_b200 as M
from paper_2603_08713_b200 import _lib

V = M.Variant
n = 8192
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
sl = slice(100, 400, 2)
med = lambda x: float(np.median(x))
print("MMA: period", med(np.diff(t[100:400, 1])), " tempty wait", med(t[100:400, 1] - t[100:400, 0]),
      " full wait (stage chunks)", med(t[sl, 10] - t[sl, 1]), " go->commit", med(t[100:400, 2] - t[100:400, 1]))
print("TMA: stage period", med(np.diff(t[sl, 12])), " empty wait", med(t[sl, 13] - t[sl, 12]),
      " lead of TMA issue over MMA full-ok (cycles)", med(t[sl, 10] - t[sl, 13]))
print("epi: tfull wait", med(t[100:400, 4] - t[100:400, 3]), " commit->epi go", med(t[100:400, 4] - t[100:400, 2]))
