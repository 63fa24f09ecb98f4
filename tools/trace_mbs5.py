"""Step-level clock64 trace of epilogue warps 0 and 2 of k_gemm_mbs2, CTA 0
(MXQ_LIB_PATH=tools/_bin/libmxq200_tr2.so, -DMXQ_GEMM_TRACE=2).  Per chunk:
0 release, 1 after tfull wait, 2 after TMEM load issue, 3 after sigma wait,
4 after barrier tests, 5 fold end (warp 2: +8)."""
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
sl = slice(100, 400)
med = lambda x: float(np.median(x))
for w, o in ((0, 0), (2, 8)):
    d = [med(t[sl, o + k + 1] - t[sl, o + k]) for k in range(5)]
    nxt = med(t[101:401, o] - t[sl, o + 5])
    print(f"warp {w}: period {med(np.diff(t[sl, o])):.0f}  tfull-wait {d[0]:.0f}  ldtm-issue {d[1]:.0f}  "
          f"sig-wait {d[2]:.0f}  tests {d[3]:.0f}  fold {d[4]:.0f}  fold-end->next-release {nxt:.0f}")
print("warp2 release - warp0 release:", med(t[sl, 8] - t[sl, 0]))
