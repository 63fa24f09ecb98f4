#!/bin/bash
# MBS GEMM timing under ablation flags and cluster sizes (dev only).
export PYTHONPATH=$PWD
for cl in ${CLS:-2 1}; do
for f in ${FLAGS:-0 32}; do for ss in ${SSIG:-1}; do export MXQ_GEMM_STAGE_SIG=$ss
  echo "== MXQ_GEMM_DBG=$f MXQ_GEMM_CL=$cl STAGE_SIG=$ss"
  MXQ_GEMM_CL=$cl MXQ_GEMM_DBG=$f timeout 60 python - <<'PY'
import torch, paper_2603_08713_b200 as M
V = M.Variant
for n in (8192,):
    g = torch.Generator(device="cuda").manual_seed(0)
    a = torch.randn(n, n, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(n, n, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    for va, vw in ((V.MBS_S, V.MBS_D), (V.MX16_OAS, V.MX16_OAS)):
        aq = M.quantize_tensor(a, M.SchemeConfig(va)); wq = M.quantize_tensor(w, M.SchemeConfig(vw))
        out = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
        for _ in range(3): M.matmul_quantized(aq, wq, out=out, out_dtype=torch.bfloat16)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(10): M.matmul_quantized(aq, wq, out=out, out_dtype=torch.bfloat16)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(f"  {va.value}x{vw.value} {n}: {ms*1e3:.1f} us {2*n**3/ms/1e9:.0f} TFLOP/s", flush=True)
PY
done
done; done
