"""clock64 trace of the MBS GEMM (k_gemm_mbs, 128x192 tiles, two TMEM partial
buffers) hand-offs in CTA 0 (development aid; run with
MXQ_LIB_PATH=tools/_bin/libmxq200_trace.so, built by
tools/build_variant.sh trace -DMXQ_GEMM_TRACE=1; profiles/r02_trace_mbs_8192.txt).  Slots per chunk q:
0/1 MMA before/after tempty wait, 10 MMA after stage-full wait, 2 MMA after
tfull commit; 3/4 epilogue warp 0 before/after tfull wait (then LDTM issue),
5 after release (arrive tempty), 6 after sigma wait, 7 fold end; 8/9 last
epilogue warp after tfull wait / release; 11 TMA sigma issued, 12/13 TMA
before/after stage-empty wait (first chunk of the stage)."""
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
names = ["mma_pre", "mma_go", "mma_commit", "epi_pre", "epi_go", "epi_rel", "epi_sig", "epi_end", "w7_go", "w7_rel",
         "mma_sf", "tma_sig", "tma_st0", "tma_st1"]
print("chunk " + " ".join(names))
for c in list(range(0, 8)) + list(range(200, 212)):
    print(c, " ".join(str(x) for x in t[c, :14]))
sl = slice(100, 400)
def med(x): return float(np.median(x))
print("median chunk period (epi_go):", med(np.diff(t[sl, 4])), " mma_go:", med(np.diff(t[sl, 1])))
print("MMA wait tempty:", med(t[sl, 1] - t[sl, 0]), " MMA go->commit:", med(t[sl, 2] - t[sl, 1]))
print("epi wait tfull:", med(t[sl, 4] - t[sl, 3]), " epi go(c)->release(c) [LDTM + fold(c-1)]:", med(t[sl, 5] - t[sl, 4]))
print("epi release->sig ok:", med(t[sl, 6] - t[sl, 5]), " fold:", med(t[sl, 7] - t[sl, 6]))
print("release(c) -> MMA go(c+2):", med(t[102:402, 1] - t[100:400, 5]), " w15:", med(t[102:402, 1] - t[100:400, 9]))
print("MMA commit(c) -> epi go(c):", med(t[sl, 4] - t[sl, 2]), " w7:", med(t[sl, 8] - t[sl, 2]))
print("w7 rel - w0 rel:", med(t[sl, 9] - t[sl, 5]))
st = t[100:400, 12]; st = st[st > 0]
print("TMA empty wait:", med((t[100:400, 13] - t[100:400, 12])[t[100:400, 12] > 0]))
sf = t[sl, 10]
print("MMA sf-wait gaps (stage full - mma_go):", med((t[sl, 10] - t[sl, 1])[t[sl, 10] > 0]))
