"""Device timing of the MBS-D weight quantizer (K3, exact and LUT modes) on a
4096 x 4096 bf16 tensor (development aid; compute-bound, so one warm tensor)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_08713_b200 as M

V = M.Variant
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
g = torch.Generator(device="cuda").manual_seed(0)
x = (torch.randn(n, n, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
for mode in ("exact", "lut"):
    cfg = M.SchemeConfig(V.MBS_D, mbs_mode=mode)
    for _ in range(2):
        M.quantize_tensor(x, cfg, check=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5):
        M.quantize_tensor(x, cfg, check=False)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"mbs_d {mode:5s} {n}x{n} {ms*1e3:8.1f} us  {n*n/ms/1e6:7.1f} Gelem/s", flush=True)
