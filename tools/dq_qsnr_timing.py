"""Device timing of the dequantizer (K5) and the QSNR evaluator (K6) on
4096 x 4096 MBS-S tensors (development aid): graphs of launches cycling over
8 distinct inputs (HBM-cold), algorithmic bytes per element
K5: 0.5 codes + 1/16 scales + 1/128 m8 in, 4 (f32) out; K6 (fused dequant):
2 (bf16 ref) + 0.5 + 1/16 + 1/128 in."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_08713_b200 as M

V = M.Variant
g = torch.Generator(device="cuda").manual_seed(0)
xs = [torch.randn(4096, 4096, device="cuda", generator=g).to(torch.bfloat16) for _ in range(8)]
qs = [M.quantize_tensor(x, M.SchemeConfig(V.MBS_S)) for x in xs]
n = xs[0].numel()


def graph_us(fn, reps=16):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn(0)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for i in range(reps):
            fn(i)
    gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    gr.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


import ctypes
from paper_2603_08713_b200 import _lib
L = _lib.lib()
ws = torch.empty(int(L.mxq_qsnr_workspace_bytes(n)), dtype=torch.uint8, device="cuda")
out = torch.empty(4, dtype=torch.float64, device="cuda")
status = torch.zeros(4, dtype=torch.int32, device="cuda")
qts = [q.qt() for q in qs]


def k6(i):
    x = xs[i % 8]
    _lib.check(L.mxq_qsnr(x.data_ptr(), _lib.MXQ_BF16, x.stride(0), ctypes.byref(qts[i % 8]), None, 0, 4096, 4096,
                          ws.data_ptr(), out.data_ptr(), status.data_ptr(), _lib.stream_handle()), "qsnr")


dq = torch.empty(4096, 4096, device="cuda", dtype=torch.float32)


def k5(i):
    _lib.check(L.mxq_dequantize(ctypes.byref(qts[i % 8]), dq.data_ptr(), 4096, status.data_ptr(),
                                _lib.stream_handle()), "dequantize")


t5 = graph_us(k5)
b5 = n * (0.5 + 1 / 16 + 1 / 128 + 4)
print(f"K5 dequantize 4096x4096 MBS-S: {t5:.2f} us, {b5 / (t5 * 1e-6) / 1e9:.0f} GB/s")
t6 = graph_us(k6)
b6 = n * (2 + 0.5 + 1 / 16 + 1 / 128)
print(f"K6 qsnr (fused dequant, bf16 ref) 4096x4096 MBS-S: {t6:.2f} us, {b6 / (t6 * 1e-6) / 1e9:.0f} GB/s")
