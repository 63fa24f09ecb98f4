"""clock64 trace of the MBS GEMM's MMA/epilogue hand-offs (CTA 0)."""
import numpy as np
import torch
import paper_2603_08713_b200 as M
from paper_2603_08713_b200 import _lib

V = M.Variant
n = 4096
g = torch.Generator(device="cuda").manual_seed(0)
a = torch.randn(n, n, device="cuda", generator=g).to(torch.bfloat16)
w = (torch.randn(n, n, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
aq = M.quantize_tensor(a, M.SchemeConfig(V.MBS_S))
wq = M.quantize_tensor(w, M.SchemeConfig(V.MBS_D))
M.matmul_quantized(aq, wq, out_dtype=torch.bfloat16)
tr = torch.zeros(512 * 4, dtype=torch.int64, device="cuda")
_lib.lib().mxq_debug_set_trace(tr.data_ptr())
M.matmul_quantized(aq, wq, out_dtype=torch.bfloat16)
torch.cuda.synchronize()
_lib.lib().mxq_debug_set_trace(None)
t = tr.cpu().numpy().reshape(512, 4)
t0 = t[0, 0]
t = t - t0
print("chunk  mma_start  mma_go(tempty ok)  epi_wait  epi_go(tfull ok)")
for c in list(range(0, 40)) + list(range(64, 72)) + list(range(200, 210)):
    print(c, *t[c])
d = np.diff(t[:, 1])
print("median cycles between MMA chunk issues:", np.median(d[d > 0]))
d = np.diff(t[:, 3])
print("median cycles between epilogue chunk starts:", np.median(d[d > 0]))
print("median MMA wait for tempty:", np.median((t[:, 1] - t[:, 0])[:200]))
print("median epi wait for tfull:", np.median((t[:, 3] - t[:, 2])[:200]))
