"""A/B device timing of the MBS-H GEMM (MBS_S x MBS_D) on the Llama-3-8B
layer shapes and 8192^3, against the plain MX16_OAS / OCP32 kernels
(development aid; MXQ_LIB_PATH selects a tools/build_variant.sh build, see
tools/probe_ab.sh)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_08713_b200 as M

V = M.Variant
SHAPES = [("qkv", 4096, 6144, 4096), ("o", 4096, 4096, 4096), ("gate_up", 4096, 28672, 4096),
          ("down", 4096, 4096, 14336), ("sq8192", 8192, 8192, 8192)]
PAIRS = [(V.MBS_S, V.MBS_D), (V.MX16_OAS, V.MX16_OAS), (V.OCP32, V.OCP32)]
if os.environ.get("AB_SHAPES"):
    SHAPES = [x for x in SHAPES if x[0] in os.environ["AB_SHAPES"].split(",")]
if len(sys.argv) > 1:
    PAIRS = [p for p in PAIRS if p[0].value in sys.argv[1].split(",")]


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


for name, m, n, k in SHAPES:
    g = torch.Generator(device="cuda").manual_seed(0)
    a = torch.randn(m, k, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(n, k, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    line = f"{name:8s} {m}x{n}x{k}:"
    for va, vw in PAIRS:
        aq = M.quantize_tensor(a, M.SchemeConfig(va))
        wq = M.quantize_tensor(w, M.SchemeConfig(vw))
        out = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
        ms = timeit(lambda: M.matmul_quantized(aq, wq, out=out, out_dtype=torch.bfloat16))
        line += f"  {va.value}x{vw.value} {ms*1e3:7.1f} us {2*m*n*k/ms/1e9:6.0f} TF/s"
    print(line, flush=True)
