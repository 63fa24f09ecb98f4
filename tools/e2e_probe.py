"""bench.py's e2e leg alone (development aid): the same run_e2e on the
Llama-3-8B step, in a fresh process, repeated, to separate its own rate from
whatever ran before it in the full bench."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2603_08713_b200 as M
from paper_2603_08713_b200 import parallel as P

dev = torch.device("cuda", 0)
torch.cuda.set_device(0)
layers = bench.WORKLOADS["llama8b"]
g = torch.Generator(device=dev).manual_seed(1234)
acts = [bench.synth_activation(torch, dev, bench.M_TOK, k, g) for _, n, k in layers]
gw = torch.Generator(device=dev).manual_seed(4321)
wq = [M.quantize_tensor((torch.randn(n, k, device=dev, generator=gw) * 0.02).to(torch.bfloat16),
                        M.SchemeConfig(M.Variant.MBS_D)) for _, n, k in layers]
outs = [torch.empty(bench.M_TOK, n, device=dev, dtype=torch.bfloat16) for _, n, _ in layers]
flops = sum(2.0 * bench.M_TOK * n * k for _, n, k in layers)
args = argparse.Namespace(warmup=3, steps=10)
if os.environ.get("PREPIN"):  # pinned blocks of the e2e sizes allocated, used once and returned to torch's host cache
    t0 = time.perf_counter()
    pre = [a.cpu().pin_memory() for a in acts] + [torch.empty(o.shape, dtype=torch.bfloat16).pin_memory() for o in outs]
    for h, d in zip(pre, acts + outs):
        d.copy_(h, non_blocking=True) if h.shape == d.shape else None
    torch.cuda.synchronize()
    del pre
    print("prepin s", round(time.perf_counter() - t0, 3))
if os.environ.get("SLEEP"):
    time.sleep(float(os.environ["SLEEP"]))
for rep in range(int(os.environ.get("REPS", "3"))):
    r = bench.run_e2e(torch, M, P, dev, 1, args, acts, outs, wq, flops, torch.cuda.synchronize, len(layers), False)
    print(rep, round(r["value"], 1), "TF/s", round(r["ms_per_step"], 2), "ms/step", flush=True)
