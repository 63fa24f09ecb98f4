"""clock64 trace of CTA 0 of the grouped decode kernel (GPT-OSS gate_up, 64
experts x 8 tokens; MXQ_LIB_PATH=tools/_bin/libmxq200_trg.so built with
-DMXQ_GEMM_TRACE=1).  Per chunk: MMA 0/1 around the TMEM-empty wait, 10 after
the stage-full wait, 2 after the commit; epilogue warp 0: 3/4 around the
TMEM-full wait, 5 after release, 6 after the sigma wait, 7 fold end; producer:
11/12 around the sigma-slot wait (per chunk), 13/14 around the stage-empty wait
(per stage)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2603_08713_b200 as M
from paper_2603_08713_b200 import _lib

V = M.Variant
av, wv = (V.NVFP4, V.NVFP4) if "nv" in sys.argv else (V.MBS_S, V.MBS_D)
g = torch.Generator(device="cuda").manual_seed(0)
wd = [(torch.randn(5760, 2880, device="cuda", generator=g) * 0.02).to(torch.bfloat16) for _ in range(64)]
wq = [M.quantize_tensor(w, M.SchemeConfig(wv), check=False) for w in wd]
toks = [M.quantize_tensor(torch.randn(8, 2880, device="cuda", generator=g).to(torch.bfloat16), M.SchemeConfig(av)) for _ in range(64)]
for _ in range(3):
    M.matmul_quantized_grouped(toks, wq, out_dtype=torch.bfloat16, check=False)
tr = torch.zeros(512 * 16, dtype=torch.int64, device="cuda")
_lib.lib().mxq_debug_set_trace(tr.data_ptr())
M.matmul_quantized_grouped(toks, wq, out_dtype=torch.bfloat16, check=False)
torch.cuda.synchronize()
_lib.lib().mxq_debug_set_trace(None)
t = tr.cpu().numpy().reshape(512, 16).astype(np.int64)
nq = int((t[:, 2] != 0).sum())
sl = slice(20, nq - 20)
med = lambda x: float(np.median(x))
print("chunks traced", nq)
print(f"MMA: period {med(np.diff(t[sl, 2])):.0f}  tempty-wait {med(t[sl,1]-t[sl,0]):.0f}  issue {med(t[sl,2]-t[sl,1]):.0f}")
m = t[sl, 10] != 0
print(f"MMA stage-start chunks: sffree-wait {med((t[sl,15]-t[sl,1])[m]):.0f}  full-wait {med((t[sl,10]-t[sl,15])[m]):.0f}  "
      f"cp+mma+commit {med((t[sl,2]-t[sl,10])[m]):.0f};  other chunks issue {med((t[sl,2]-t[sl,1])[~m]):.0f}")
print(f"EPI: period {med(np.diff(t[sl, 3])):.0f}  tfull-wait {med(t[sl,4]-t[sl,3]):.0f}  ld+release {med(t[sl,5]-t[sl,4]):.0f}  "
      f"sig-wait {med(t[sl,6]-t[sl,5]):.0f}  fold {med(t[sl,7]-t[sl,6]):.0f}  next {med(t[21:nq-19,3]-t[sl,7]):.0f}")
print(f"   mean tfull-wait {np.mean(t[sl,4]-t[sl,3]):.0f}  mean sig-wait {np.mean(t[sl,6]-t[sl,5]):.0f}  mean period {np.mean(np.diff(t[sl,3])):.0f}")
ns = int((t[:, 14] != 0).sum())
ss = slice(10, ns - 10)
print(f"TMA: sig-slot wait mean {np.mean(t[sl,12]-t[sl,11]):.0f}  stage wait mean {np.mean(t[ss,14]-t[ss,13]):.0f}  stage period {med(np.diff(t[ss,13])):.0f}")
# lead of the producer over the epilogue (chunks)
lead = [int(np.searchsorted(t[:nq, 3], t[i, 12])) for i in range(20, nq - 20, 40)]
print("epilogue chunk index at producer sigma issue, i - idx:", [i - l for i, l in zip(range(20, nq - 20, 40), lead)])
