"""Single-GPU measurements of BASELINE.json configs 3-5 (SURVEY §8 d rows
C3-C5), next to bench.py's configs 1-2.  Device time with CUDA events, inputs
larger than L2 or rotated across distinct buffers; writes one JSON object.

  C3  Qwen3-8B whole-model weight quantization (MBS-D exact, 36 layers x 7
      projections, random N(0, 0.02) weights) + prefill MBS-H GEMMs at M=4096;
      per-GPU share at 2/4/8 GPUs = layers / G (layer sharding, no exchange).
  C4  Llama-3-70B FFN (K=8192, N=28672) column-sharded over 8: one rank's GEMM
      (M=4096, N=3584) MBS-H, plus the bf16 all_gather volume it implies.
  C5  GPT-OSS-120B expert GEMMs (gate_up 5760x2880, down 2880x2880; K=2880
      leaves a 64-wide last macro), M in {1, 8, 32, 128} tokens per expert,
      MBS-H vs NVFP4, as weight-streaming GB/s (HBM-bound) and TFLOP/s.

  python tools/configs_bench.py [--out profiles/configs_r01.json]
"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_08713_b200 as M

V = M.Variant
dev = torch.device("cuda", 0)
bf16 = torch.bfloat16


def events_ms(fn, reps, graph=True):
    """Device time per call: the calls are captured in one CUDA graph so the
    host-side wrapper cost (tens of us per call) does not leave the GPU idle."""
    torch.cuda.synchronize()
    g = None
    if graph:
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            fn(0)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for i in range(reps):
                fn(i)
        g.replay()
        torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    if g is not None:
        g.replay()
    else:
        for i in range(reps):
            fn(i)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def c3():
    hidden, inter, layers = 4096, 12288, 36
    projs = [("q", 4096, hidden), ("k", 1024, hidden), ("v", 1024, hidden), ("o", hidden, 4096),
             ("gate", inter, hidden), ("up", inter, hidden), ("down", hidden, inter)]
    g = torch.Generator(device=dev).manual_seed(7)
    params = 0
    t_quant = 0.0
    wq_layer0 = []
    torch.cuda.synchronize()
    for layer in range(layers):
        for name, n, k in projs:
            w = (torch.randn(n, k, device=dev, generator=g) * 0.02).to(bf16)
            params += n * k
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            q = M.quantize_tensor(w, M.SchemeConfig(V.MBS_D), check=False)
            e1.record()
            torch.cuda.synchronize()
            t_quant += e0.elapsed_time(e1)
            if layer == 0:
                wq_layer0.append(q)
            del w
    # prefill GEMMs of one layer at M = 4096 (every layer has the same shapes)
    acts = {k: (torch.randn(4096, k, device=dev, generator=g)).to(bf16) for _, _, k in projs}
    outs = [torch.empty(4096, n, device=dev, dtype=bf16) for _, n, _ in projs]

    def layer_step(_):
        for (name, n, k), wq, o in zip(projs, wq_layer0, outs):
            aq = M.quantize_tensor(acts[k], M.SchemeConfig(V.MBS_S), check=False)
            M.matmul_quantized(aq, wq, out=o, out_dtype=bf16, check=False)
    layer_step(0)
    ms_layer = events_ms(layer_step, 5)
    flops_layer = sum(2.0 * 4096 * n * k for _, n, k in projs)
    return {"config": "C3 Qwen3-8B whole-model weight quantization (MBS-D exact) + prefill MBS-H GEMMs, M=4096",
            "params": params, "weight_quant_s": t_quant / 1e3,
            "weight_quant_gelem_s": params / (t_quant * 1e-3) / 1e9,
            "prefill_ms_per_layer": ms_layer, "prefill_ms_model": ms_layer * layers,
            "prefill_tflops": flops_layer / (ms_layer * 1e-3) / 1e12,
            "layer_sharded_ms_per_gpu": {str(gp): round(ms_layer * ((layers + gp - 1) // gp) +
                                                        t_quant / gp, 3) for gp in (1, 2, 4, 8)},
            "note": "layer sharding: each GPU quantizes and runs ceil(36/G) layers, no data-path exchange; "
                    "per-GPU time = its prefill share + its share of the weight quantization"}


def c4():
    m, n, k, world = 4096, 28672, 8192, 8
    ns = n // world
    g = torch.Generator(device=dev).manual_seed(11)
    xs = [torch.randn(m, k, device=dev, generator=g).to(bf16) for _ in range(2)]
    w = (torch.randn(ns, k, device=dev, generator=g) * 0.02).to(bf16)
    wq = M.quantize_tensor(w, M.SchemeConfig(V.MBS_D))
    aqs = [M.quantize_tensor(x, M.SchemeConfig(V.MBS_S)) for x in xs]
    out = torch.empty(m, ns, device=dev, dtype=bf16)
    fn = lambda i: M.matmul_quantized(aqs[i % 2], wq, out=out, out_dtype=bf16, check=False)
    fn(0)
    ms = events_ms(fn, 10)
    gather_bytes = m * n * 2 * (world - 1) // world
    return {"config": "C4 Llama-3-70B FFN K=8192 N=28672 column-sharded x8: one rank's MBS-H GEMM (M=4096, N=3584)",
            "gemm_ms": ms, "gemm_tflops": 2.0 * m * ns * k / (ms * 1e-3) / 1e12,
            "all_gather_bytes_in_per_rank": gather_bytes,
            "all_gather_ms_at_770GBs": gather_bytes / 770e9 * 1e3,
            "note": "NVLink time estimated from the measured 770 GB/s per-direction peer copy (B200_PROFILING.md); "
                    "the exchange itself is exercised by bench.py --mode columns"}


def c5():
    g = torch.Generator(device=dev).manual_seed(13)
    res = []
    for lname, n, k in (("gate_up", 5760, 2880), ("down", 2880, 2880)):
        ws = [(torch.randn(n, k, device=dev, generator=g) * 0.02).to(bf16) for _ in range(16)]  # 16 experts > L2
        for arm, (va, vw) in (("mbs_h", (V.MBS_S, V.MBS_D)), ("nvfp4", (V.NVFP4, V.NVFP4))):
            wqs = [M.quantize_tensor(w, M.SchemeConfig(vw)) for w in ws]
            wbytes = n * k * (0.5 + 1 / 16) + (n * ((k + 127) // 128) * 4 if arm == "mbs_h" else 0)
            for m in (1, 8, 32, 128):
                a = torch.randn(m, k, device=dev, generator=g).to(bf16)
                aq = M.quantize_tensor(a, M.SchemeConfig(va))
                out = torch.empty(m, n, device=dev, dtype=bf16)
                fn = lambda i: M.matmul_quantized(aq, wqs[i % 16], out=out, out_dtype=bf16, check=False)
                fn(0)
                ms = events_ms(fn, 32)
                res.append({"layer": lname, "arm": arm, "m": m, "n": n, "k": k, "us": round(ms * 1e3, 2),
                            "weight_gbs": round(wbytes / (ms * 1e-3) / 1e9, 1),
                            "tflops": round(2.0 * m * n * k / (ms * 1e-3) / 1e12, 2)})
    # grouped: all 64 experts of a layer in one launch (tokens per expert <= 128)
    grouped = []
    for lname, n, k in (("gate_up", 5760, 2880), ("down", 2880, 2880)):
        E = 64
        wq = [M.quantize_tensor((torch.randn(n, k, device=dev, generator=g) * 0.02).to(bf16),
                                M.SchemeConfig(V.MBS_D)) for _ in range(E)]
        wbytes = E * (n * k * (0.5 + 1 / 16) + n * ((k + 127) // 128) * 4)
        for m in (1, 8, 32, 64, 128):
            aq = [M.quantize_tensor(torch.randn(m, k, device=dev, generator=g).to(bf16), M.SchemeConfig(V.MBS_S))
                  for _ in range(E)]
            fn = lambda i: M.matmul_quantized_grouped(aq, wq, out_dtype=bf16, check=False)
            fn(0)
            ms = events_ms(fn, 8)
            grouped.append({"layer": lname, "arm": "mbs_h", "experts": E, "m_per_expert": m, "us_per_launch": round(ms * 1e3, 2),
                            "us_per_expert": round(ms * 1e3 / E, 3), "weight_gbs": round(wbytes / (ms * 1e-3) / 1e9, 1),
                            "tflops": round(2.0 * E * m * n * k / (ms * 1e-3) / 1e12, 2)})
        del wq
    return {"config": "C5 GPT-OSS-120B expert GEMMs, one expert per launch cycling over 16 experts (weights > L2)",
            "rows": res, "grouped_rows": grouped,
            "grouped_note": "matmul_quantized_grouped: the 64 experts' GEMMs in one launch of the MBS kernel -- swap-AB "
                            "(one CTA pair per 128 weight rows of an expert) up to 64 tokens, direct 128x192 tiles "
                            "up to 128 -- weights streamed from HBM once",
            "note": "HBM-bound on weights: compare weight_gbs with the measured 6.55 TB/s copy bandwidth; "
                    "one 128-row M tile per launch leaves most SMs idle at these N (no split-K yet)"}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    out = {"c4": c4(), "c5": c5(), "c3": c3(), "device": torch.cuda.get_device_name(0)}
    txt = json.dumps(out, indent=1)
    print(txt)
    if args.out:
        open(args.out, "w").write(txt + "\n")
