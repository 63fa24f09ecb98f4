"""clock64 trace of the 192-column MBS GEMM's hand-offs in CTA 0 (development
aid; needs a build with MXQ_NVCC_EXTRA=-DMXQ_GEMM_TRACE=1).  Slots per chunk:
0/1 MMA before/after tempty wait, 2 MMA after tfull commit, 10 MMA after
sf_ready wait, 3/4 epilogue warp 0 before/after tfull wait, 5 after release,
6 after sfull wait, 7 end of chunk, 8/9 warp 15 after tfull / end of chunk,
11 TMA sigma issued, 12 TMA stage issued (first chunk of the stage)."""
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
t0 = t[0, 0]
t = np.where(t > 0, t - t0, -1)
names = ["mma_pre", "mma_go", "mma_commit", "epi_pre", "epi_go", "epi_rel", "epi_sig", "epi_end", "w15_go", "w15_end",
         "mma_sf", "tma_sig", "tma_stage"]
print("chunk " + " ".join(names))
for c in list(range(0, 12)) + list(range(100, 112)):
    print(c, " ".join(str(x) for x in t[c, :13]))
sl = slice(100, 400)
def med(x): return float(np.median(x))
print("median chunk period (epi_go):", med(np.diff(t[sl, 4])))
print("median MMA wait tempty:", med(t[sl, 1] - t[sl, 0]))
print("median MMA go->commit:", med(t[sl, 2] - t[sl, 1]))
print("median epi wait tfull:", med(t[sl, 4] - t[sl, 3]))
print("median epi go->release:", med(t[sl, 5] - t[sl, 4]))
print("median epi release->sig ok:", med(t[sl, 6] - t[sl, 5]))
print("median epi sig->end (compute):", med(t[sl, 7] - t[sl, 6]))
print("median release(c) -> MMA go(c+2):", med(t[102:402, 1] - t[100:400, 5]))
print("median MMA commit(c) -> epi go(c):", med(t[sl, 4] - t[sl, 2]))
print("median w15 go - w0 go:", med(t[sl, 8] - t[sl, 4]))
print("median w15 end - w0 end:", med(t[sl, 9] - t[sl, 7]))
print("median tma sigma issue lead (epi_sig - tma_sig):", med(t[sl, 6] - t[sl, 11]))
