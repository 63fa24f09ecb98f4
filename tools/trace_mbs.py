"""clock64 trace of the MBS GEMM's hand-offs in CTA 0 (development aid).
Slots per chunk: 0/1 MMA before/after tempty wait, 4/5 MMA before/after
sf_ready wait (stage containing the chunk), 2 epilogue warp 0 before sfull
wait, 3 after tfull wait, 6 after releasing the buffer, 7 last epilogue warp
after tfull wait."""
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
tr = torch.zeros(512 * 8, dtype=torch.int64, device="cuda")
_lib.lib().mxq_debug_set_trace(tr.data_ptr())
M.matmul_quantized(aq, wq, out_dtype=torch.bfloat16)
torch.cuda.synchronize()
_lib.lib().mxq_debug_set_trace(None)
t = tr.cpu().numpy().reshape(512, 8).astype(np.int64)
t0 = t[0, 0]
t = np.where(t > 0, t - t0, -1)
print("chunk mma_pre mma_go(tempty) epi_pre epi_go(tfull) sf_pre sf_go epi_rel epi_last_go")
for c in list(range(0, 24)) + list(range(100, 116)) + list(range(300, 310)):
    r = t[c]
    print(c, r[0], r[1], r[2], r[3], r[4], r[5], r[6], r[7])
sl = slice(100, 500)
def med(x): return float(np.median(x))
print("median MMA chunk period:", med(np.diff(t[sl, 1])))
print("median epi chunk period:", med(np.diff(t[sl, 3])))
print("median MMA wait tempty:", med(t[sl, 1] - t[sl, 0]))
print("median epi0 wait (sfull+tfull):", med(t[sl, 3] - t[sl, 2]))
print("median epi0 go->release:", med(t[sl, 6] - t[sl, 3]))
print("median release(c) -> MMA go(c+3):", med(t[103:503, 1] - t[100:500, 6]))
print("median MMA go(c) -> epi go(c):", med(t[sl, 3] - t[sl, 1]))
print("median epi last - epi0 go:", med(t[sl, 7] - t[sl, 3]))
