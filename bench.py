#!/usr/bin/env python
"""Benchmark of the B200 MXFP4 quantize-and-GEMM path (BASELINE.json configs[1]).

Workload (one "step"): the four Llama-3-8B linear layers at M = 4096 tokens --
QKV (N 6144, K 4096), O (4096, 4096), gate_up (28672, 4096), down (4096, 14336)
-- each = quantize the bf16 activation on the fly (MBS-S) and run the tcgen05
block-scaled GEMM against resident MBS-D weights (MBS-H, the paper's default),
bf16 output.  Synthetic data: activations student-t dof 4 (activation-like),
random-init weights N(0, 0.02).  Headline `value` = step TFLOP/s (device-timed,
inputs resident in HBM); `e2e` = the same step through the public API with
pinned host activations in and bf16 products out.  Comparison arms on the
same shapes: plain MXFP4 (OCP32 block-32, kind::mxf4), MX16+OAS and NVFP4.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (torchrun, default --mode columns): every layer is column-sharded
(weight rows) across ranks (parallel.column_parallel_forward) and the bf16
outputs are all-gathered over NVLink into the (M, N) product, the gather of
row block i overlapped with the GEMM of block i+1 (strong scaling, SURVEY
section 8 e).  --mode replicas: own tokens per rank, no collective (weak);
--mode layers: C3, Qwen3-8B weight quantization + prefill with the layers
sharded; --workload llama70b-ffn: C4's 70B FFN GEMM.
`--impl reference` times the reference algorithm (the CPU oracle port,
oracle/mxq_oracle.py) on the host cores on a bounded row sample of the same
workload; under torchrun only rank 0 runs it.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "OAS+MBS MXFP4 GEMM TFLOPS & overhead vs plain MXFP4/NVFP4; quant GB/s; QSNR"
LAYERS = (("qkv", 6144, 4096), ("o", 4096, 4096), ("gate_up", 28672, 4096), ("down", 4096, 14336))
M_TOK = 4096
WORKLOAD = ("llama3-8b linear layers QKV 6144x4096, O 4096x4096, gate_up 28672x4096, down 4096x14336; "
            "M=4096 tokens; A quantized per step (MBS_S) x resident W (MBS_D) = MBS-H; bf16 out")


def flops_per_step(m=M_TOK, n_scale=1.0):
    return sum(2.0 * m * n * k for _, n, k in LAYERS) * n_scale


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class Clocks:
    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi takes up to a second to print its first line: start the
            # timed work only once sampling runs, so the whole region is covered
            t0 = time.perf_counter()
            while not self.lines and time.perf_counter() - t0 < 5.0 and self.proc.poll() is None:
                time.sleep(0.01)
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# workloads (SURVEY section 8 d; Appendix B shapes)
# ---------------------------------------------------------------------------
WORKLOADS = {
    # C2 (and the N>1 column-sharded form of it): the four Llama-3-8B linears
    "llama8b": LAYERS,
    # C4: the Llama-3-70B FFN gate/up GEMM, K = 8192, N = 28672
    "llama70b-ffn": (("ffn_gate_up", 28672, 8192),),
}
# C3: Qwen3-8B, 36 layers x 7 projections (name, N, K)
QWEN3_8B = (("q", 4096, 4096), ("k", 1024, 4096), ("v", 1024, 4096), ("o", 4096, 4096),
            ("gate", 12288, 4096), ("up", 12288, 4096), ("down", 4096, 12288))
QWEN3_LAYERS = 36


def synth_activation(torch, dev, rows, k, gen):
    """Student-t, dof 4 -- the reference's activation-like generator
    (src/metrics.py:103-105; SURVEY section 8 d, C2) -- drawn on the device as
    Z / sqrt(chi2_4 / 4), chi2_4 the sum of four squared standard normals; bf16."""
    z = torch.randn(rows, k, device=dev, generator=gen)
    chi2 = torch.zeros_like(z)
    for _ in range(4):
        e = torch.randn(rows, k, device=dev, generator=gen)
        chi2.addcmul_(e, e)
    return (z * torch.rsqrt(chi2 * 0.25)).to(torch.bfloat16)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2603_08713_b200 as M
    from paper_2603_08713_b200 import parallel as P

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    # one process per GPU; MXQ_DIST_BACKEND=gloo lets a single-GPU box run the
    # multi-rank code path (ranks share the device) for testing
    backend = os.environ.get("MXQ_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    mode = args.mode
    if mode == "auto":
        mode = "columns" if world > 1 else "single"
    if mode == "layers":
        return run_layers(args, world, rank, local, dev, backend)
    layers = WORKLOADS[args.workload]
    V = M.Variant
    bf16 = torch.bfloat16

    def barrier():
        if world > 1:
            if backend == "nccl":
                dist.barrier(device_ids=[local])
            else:
                dist.barrier()
        torch.cuda.synchronize()

    # ---- synthetic inputs: activations replicated (same seed on every rank
    # in columns mode, own tokens per rank in replicas mode); weights random
    # init N(0, 0.02), row-sharded in columns mode -----------------------------
    cols = mode == "columns" and world > 1
    g = torch.Generator(device=dev).manual_seed(1234 + (rank if mode == "replicas" else 0))
    acts = [synth_activation(torch, dev, M_TOK, k, g) for _, n, k in layers]
    gw = torch.Generator(device=dev).manual_seed(4321)
    wdense, bounds = [], []
    for _, n, k in layers:
        full = (torch.randn(n, k, device=dev, generator=gw) * 0.02).to(bf16)
        lo, hi = P.shard_bounds(n, world, rank) if cols else (0, n)
        bounds.append((lo, hi))
        wdense.append(full[lo:hi].contiguous())
        del full

    arms = {  # name -> (activation variant, weight variant)
        "mbs_h": (V.MBS_S, V.MBS_D),
        "ocp32": (V.OCP32, V.OCP32),
        "mx16_oas": (V.MX16_OAS, V.MX16_OAS),
        "nvfp4": (V.NVFP4, V.NVFP4),
    }
    weights = {name: [M.quantize_tensor(w, M.SchemeConfig(wv)) for w in wdense] for name, (_, wv) in arms.items()}
    del wdense
    outs = [torch.empty(M_TOK, hi - lo, device=dev, dtype=bf16) for lo, hi in bounds]   # local products
    full_outs = [torch.empty(M_TOK, n, device=dev, dtype=bf16) for _, n, _ in layers] if cols else None
    n_local = sum(2.0 * M_TOK * (hi - lo) * k for (lo, hi), (_, _, k) in zip(bounds, layers))
    step_flops_global = sum(2.0 * M_TOK * n * k for _, n, k in layers) * (1 if cols else world)
    comm = torch.cuda.Stream() if cols else None

    def local_step(arm, li, x, dst):
        av, _ = arms[arm]
        aq = M.quantize_tensor(x, M.SchemeConfig(av), check=False)
        M.matmul_quantized(aq, weights[arm][li], out=dst, out_dtype=bf16, check=False)

    def step(arm):
        for li in range(len(layers)):
            if cols:
                # column shards + overlapped all_gather into the (M, N) product
                P.column_parallel_forward(acts[li], weights[arm][li], full_outs[li], world,
                                          lambda x, wq, dst, li=li: local_step(arm, li, x, dst),
                                          chunks=args.chunks, comm_stream=comm)
            else:
                local_step(arm, li, acts[li], outs[li])

    def gemm_only(arm, aqs):
        for li in range(len(layers)):
            M.matmul_quantized(aqs[li], weights[arm][li], out=outs[li], out_dtype=bf16, check=False)

    def capture(fn):
        """fn() as one CUDA graph (warmed once on a side stream)."""
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            fn()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            fn()
        return gr

    def timed(fn, k, w):
        for _ in range(w):
            fn()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(k):
            fn()
        e1.record()
        barrier()
        return P.max_over_ranks(e0.elapsed_time(e1) / k, device=dev)

    K, W = args.steps, args.warmup
    results = {}
    with Clocks(local) as clocks:
        for arm in ("mbs_h", "ocp32", "mx16_oas", "nvfp4"):
            if args.graphs and not cols:
                gs = capture(lambda: step(arm))
                ms = timed(gs.replay, K, W)
            else:  # NCCL collectives and the comm stream run eagerly
                ms = timed(lambda: step(arm), K, W)
            # the dominant kernel alone: the step's GEMM launches (operands
            # quantized beforehand) replayed as one graph, device time per step
            aqs = [M.quantize_tensor(a, M.SchemeConfig(arms[arm][0]), check=False) for a in acts]
            if args.graphs:
                gg = capture(lambda: gemm_only(arm, aqs))
                gemm_ms = timed(gg.replay, K, W)
            else:
                gemm_ms = timed(lambda: gemm_only(arm, aqs), K, W)
            results[arm] = {
                "ms_per_step": ms,
                "tflops_step": step_flops_global / (ms * 1e-3) / 1e12,
                "gemm_ms": gemm_ms,
                "gemm_tflops": n_local * world / (gemm_ms * 1e-3) / 1e12,  # all ranks' GEMM work / max per-rank time
            }
            del aqs
    head = results["mbs_h"]

    # ---- e2e: public API, pinned host activations in, bf16 products out ----
    e2e = run_e2e(torch, M, P, dev, world, args, acts, outs, weights["mbs_h"], step_flops_global, barrier,
                  len(layers), cols)
    if world > 1:
        barrier()

    # ---- quantizer bandwidth (4096x4096 bf16 activations, HBM-cold) -------
    # the timed launches cycle over 8 distinct activations (256 MB, twice the
    # L2), so every launch streams its input from HBM
    # (the clock sampler also covers the quantizer and C5 timed regions)
    with Clocks(local) as clocks2:
        qbw = quantizer_bandwidth(torch, M, dev, args)
        experts = grouped_experts(torch, M, P, dev, args, world, rank, barrier) if args.experts else None
    clocks.lines += clocks2.lines

    out = None
    if rank == 0:
        out = {}
        # ---- C1: QSNR of config 1 (4096x4096 gaussian+outliers, bf16), seeds
        # 0..7, each value against the reference's (tests/golden/qsnr_seeds.json,
        # made by tests/golden/make_qsnr_seeds.py from the reference package);
        # the mean is the reference's mean_qsnr (running sum / n) ----
        ref_seeds = json.load(open(os.path.join(ROOT, "tests", "golden", "qsnr_seeds.json")))
        vnames = ("ocp32", "mx16", "mx16_oas", "mbs_s", "mbs_d", "nvfp4")
        per = {v: [] for v in vnames}
        for seed in range(8):
            t1 = M.generate_tensor(M.GeneratorSpec("gaussian_with_outliers", (4096, 4096), seed=seed))
            t1b = torch.from_numpy(t1).to(dev).to(bf16)
            for vname in vnames:
                q = M.quantize_tensor(t1b, M.SchemeConfig(V(vname)))
                rep, fl = M.qsnr_quantized(t1b, q)
                ref = ref_seeds["seeds"][str(seed)][vname]
                per[vname].append((rep.qsnr_db, fl, rep.qsnr_db == ref["qsnr_db"] and fl == ref["flush"]))
        qs = {}
        for vname in vnames:
            db_sum = fl_sum = 0.0
            for db, fl, _ in per[vname]:
                db_sum += db
                fl_sum += fl
            qs[vname] = {"qsnr_db_seed0": round(per[vname][0][0], 6), "mean_qsnr_db": round(db_sum / 8, 6),
                         "mean_flush": round(fl_sum / 8, 6),
                         "equals_reference": all(e for _, _, e in per[vname]),
                         "mean_equals_reference": db_sum / 8 == ref_seeds["mean_qsnr_db"][vname]}
        qs["seeds"] = "0..7"
        out["qsnr"] = qs


    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel (tcgen05 MBS GEMM) -----------------
    clk = clocks.summary()
    roofline = gemm_roofline(head["gemm_tflops"] / world, clk)

    # ---- CPU baseline: the reference algorithm (oracle port) on a sample ---
    cpu = cpu_baseline_sample(weights_from_gpu=[weights["mbs_h"][li] for li in range(len(layers))],
                              acts=acts, rows=args.cpu_rows) if (world == 1 and args.workload == "llama8b") else None

    ocp = results["ocp32"]
    par = {"single": "single", "replicas": f"replicas x{world} (own tokens per rank, no collective)",
           "columns": f"column-shard x{world} (weight rows) + overlapped NCCL all_gather of the bf16 outputs "
                      f"into (M, N), {args.chunks} row blocks"}[mode if world > 1 else "single"]
    wl_desc = WORKLOAD if args.workload == "llama8b" else (
        "llama3-70b FFN gate/up N=28672 K=8192; M=4096 tokens; A quantized per step (MBS_S) x resident W (MBS_D); bf16 out")
    line = {
        "metric": METRIC, "value": round(head["tflops_step"], 2), "unit": "TFLOP/s", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": round(head["ms_per_step"], 4), "higher_is_better": True,
        "scaling": "strong" if cols else "weak", "vs_baseline": None,
        "dtype": "fp4_e2m1 (UE8M0 block-16 scales, MBS sigma f32, f32 accum)",
        "data": "synthetic (activations student-t dof 4, the reference's activation_like; random-init N(0,0.02) weights)",
        "config": {"workload": wl_desc, "global_batch": M_TOK * (1 if cols else world), "seq_len": None,
                   "parallelism": par,
                   "l2": "inputs larger than L2 (218 MB bf16 activations + 121 MB fp4 weights per step)"},
        "gemm_only_tflops": round(head["gemm_tflops"], 2),
        "arms": {k: {kk: (round(vv, 4) if isinstance(vv, float) else vv) for kk, vv in v.items()}
                 for k, v in results.items()},
        "mbs_h_overhead_vs_ocp32": round(1.0 - head["tflops_step"] / ocp["tflops_step"], 4),
        "mbs_h_gemm_overhead_vs_ocp32": round(1.0 - head["gemm_tflops"] / ocp["gemm_tflops"], 4),
        "mbs_h_overhead_vs_nvfp4": round(1.0 - head["tflops_step"] / results["nvfp4"]["tflops_step"], 4),
        "quantizer": {k: {kk: round(vv, 2) for kk, vv in v.items()} for k, v in qbw.items()},
        "quantizer_hbm_frac_mbs_s": round(qbw["mbs_s"]["gbs"] / hbm_peak(), 4),
        "moe_experts_c5": experts,
        "qsnr_config1": out["qsnr"],
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": 8 * K,
        "clocks": clk,
    }
    if cols:
        line["gather_overhead"] = round(1.0 - head["gemm_ms"] / head["ms_per_step"], 4)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def hbm_peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6550.0


def gemm_roofline(achieved_per_gpu, clk):
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    bf16_peak = peaks.get("bf16_tflops")
    basis = "4 x measured dense bf16 (MEASURED_PEAKS.json bf16_tflops, burst): FP4 dense = 4x bf16 on B200"
    if not bf16_peak:
        bf16_peak, basis = 1590.0, "4 x fallback dense bf16 1.59 PF (B200_PROFILING.md)"
    fp4_peak = 4.0 * bf16_peak
    traffic, tbasis = None, "no ncu capture committed"
    prof = os.path.join(ROOT, "profiles", "gemm_traffic.json")
    if os.path.exists(prof):
        try:
            tj = json.load(open(prof))
            traffic, tbasis = tj.get("mbs_h_bytes_per_launch"), tj.get("basis", tbasis)
        except Exception:
            pass
    # MBS-specific ceiling: the epilogue folds every
    # 128-K macro partial with two FP32 ops per output, 128 FP32 lanes/clk/SM
    # -> 64 output-macros x 128 K x 2 flop per clock per SM
    f_mhz = clk.get("sm_mhz") or clk.get("sm_max_mhz") or 1965.0
    fp32_bound = 148 * 64 * 128 * 2 * f_mhz * 1e6 / 1e12
    return {"bound": "tensor", "achieved": round(achieved_per_gpu, 1), "peak": round(fp4_peak, 1), "unit": "TFLOP/s",
            "frac": round(achieved_per_gpu / fp4_peak, 4), "traffic": traffic, "peak_basis": basis,
            "kernel": "mbs::k_gemm_mbs<BN=192,NB=2,bf16,CL=2> (kind::mxf4nvf4.block16 UE8M0, N=192 MMAs, "
                      "tcgen05.cp scale factors, 16 FP32 epilogue warps)",
            "mbs_fp32_epilogue_bound": round(fp32_bound, 1),
            "frac_of_mbs_fp32_bound": round(achieved_per_gpu / fp32_bound, 4),
            "mbs_bound_basis": f"2 FP32 ops per output per 128-K macro at 128 FP32 lanes/clk/SM, {f_mhz:.0f} MHz",
            "traffic_basis": tbasis,
            "algorithmic": "2*M*N*K summed over the step's GEMM launches / device time of a CUDA graph holding "
                           "exactly those launches (operands quantized beforehand), CUDA events on the launch stream"}


def quantizer_bandwidth(torch, M, dev, args):
    V = M.Variant
    gq = torch.Generator(device=dev).manual_seed(1234)
    xq = [torch.randn(M_TOK, 4096, device=dev, generator=gq).to(torch.bfloat16) for _ in range(8)]
    # algorithmic bytes / element: bf16 read + packed codes + scale bytes
    # (+ MBS mantissa byte per 128 elements); the GEMM-layout copies the
    # kernels also write (row-major + MMA-atom scales, f32 sigma) are not
    # counted, so the GB/s is conservative.
    bytes_per_el = {"ocp32": 2 + 0.5 + 1 / 32, "mx16": 2 + 0.5 + 1 / 16, "mx16_oas": 2 + 0.5 + 1 / 16,
                    "mbs_s": 2 + 0.5 + 1 / 16 + 1 / 128, "mbs_d": 2 + 0.5 + 1 / 16 + 1 / 128,
                    "nvfp4": 2 + 0.5 + 1 / 16, "mbs_d_lut": 2 + 0.5 + 1 / 16 + 1 / 128}
    qbw = {}
    for vname in ("ocp32", "mx16", "mx16_oas", "mbs_s", "nvfp4", "mbs_d", "mbs_d_lut"):
        cfg = M.SchemeConfig(V.MBS_D, mbs_mode="lut") if vname == "mbs_d_lut" else M.SchemeConfig(V(vname))
        reps = 8 if vname.startswith("mbs_d") else 48
        for x in xq:
            M.quantize_tensor(x, cfg, check=False, gemm_layout=True)
        torch.cuda.synchronize()
        g = None
        if args.graphs:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for i in range(reps):
                    M.quantize_tensor(xq[i % 8], cfg, check=False, gemm_layout=True)
            g.replay()
            torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if g is not None:
            g.replay()
        else:
            for i in range(reps):
                M.quantize_tensor(xq[i % 8], cfg, check=False, gemm_layout=True)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        qbw[vname] = {"us": ms * 1e3, "gbs": xq[0].numel() * bytes_per_el[vname] / (ms * 1e-3) / 1e9,
                      "melem_s": xq[0].numel() / (ms * 1e-3) / 1e6}
    del xq
    # the same kernels on the down-projection's activation (4096 x 14336, 117 MB
    # bf16): at 32 MB a pure-read kernel reaches only ~4.1 TB/s on this part
    # (tools/microbench_read.cu: ~3 us of per-launch ramp), so the config-size
    # fraction is reported beside the 4096^2 one
    xl = [torch.randn(M_TOK, 14336, device=dev, generator=gq).to(torch.bfloat16) for _ in range(3)]
    for vname in ("mx16_oas", "mbs_s", "nvfp4"):
        cfg = M.SchemeConfig(V(vname))
        for x in xl:
            M.quantize_tensor(x, cfg, check=False, gemm_layout=True)
        torch.cuda.synchronize()
        reps = 12
        g = torch.cuda.CUDAGraph()  # device time of the launches alone (no host gaps)
        with torch.cuda.graph(g):
            for i in range(reps):
                M.quantize_tensor(xl[i % 3], cfg, check=False, gemm_layout=True)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        qbw[vname + "@4096x14336"] = {"us": ms * 1e3, "gbs": xl[0].numel() * bytes_per_el[vname] / (ms * 1e-3) / 1e9,
                                      "melem_s": xl[0].numel() / (ms * 1e-3) / 1e6}
    del xl
    return qbw


def grouped_experts(torch, M, P, dev, args, world=1, rank=0, barrier=None):
    """C5: GPT-OSS-120B MoE expert GEMMs (decode-sized token groups), one MoE
    layer's 128 experts, MBS-H (MBS_S tokens x MBS_D weights) vs NVFP4 x
    NVFP4, both on the grouped tcgen05 kernel (matmul_quantized_grouped, up
    to 64 experts per launch).  Expert-parallel over the ranks (SURVEY §8 e:
    128/N experts per GPU, replicas only -- the per-expert GEMMs exchange
    nothing; 16 experts per GPU at N = 8), timed as the max over ranks of the
    device time of one layer's launches.  Per GPU the weights (gate_up
    5760 x 2880: 1.2 GB in MBS at N = 1) exceed the L2 at N <= 4, so every
    launch streams its weights from HBM; reported as whole-job weight GB/s
    (algorithmic weight bytes: codes + scales + MBS mantissa bytes), the
    fraction of N x HBM, and microseconds per layer and per expert."""
    V = M.Variant
    n_total, k = 128, 2880
    n_exp = n_total // world
    first = rank * n_exp
    out = {"experts_per_layer": n_total, "experts_per_gpu": n_exp, "n_gpus": world}
    hbm = hbm_peak()
    for proj, n in (("gate_up", 5760), ("down", 2880)):
        for arm, (av, wv) in (("mbs_h", (V.MBS_S, V.MBS_D)), ("nvfp4", (V.NVFP4, V.NVFP4))):
            wq = []
            for e in range(first, first + n_exp):  # (this rank's experts; quantized one at a time)
                gw = torch.Generator(device=dev).manual_seed(777 + e)
                w = (torch.randn(n, k, device=dev, generator=gw) * 0.02).to(torch.bfloat16)
                wq.append(M.quantize_tensor(w, M.SchemeConfig(wv), check=False))
                del w
            wbytes = n * k * (0.5 + 1 / 16 + (1 / 128 if arm == "mbs_h" else 0.0))
            for mtok in (1, 2, 4, 8, 16, 32, 64, 128):
                gt = torch.Generator(device=dev).manual_seed(mtok * 1000 + rank)
                toks = [M.quantize_tensor(torch.randn(mtok, k, device=dev, generator=gt).to(torch.bfloat16),
                                          M.SchemeConfig(av), check=False) for _ in range(n_exp)]

                def layer():
                    for g0 in range(0, n_exp, 64):
                        M.matmul_quantized_grouped(toks[g0:g0 + 64], wq[g0:g0 + 64], out_dtype=torch.bfloat16,
                                                   check=False)

                layer()
                torch.cuda.synchronize()
                reps = 10
                g = torch.cuda.CUDAGraph()  # device time of the launches (the expert table is a kernel parameter)
                with torch.cuda.graph(g):
                    for _ in range(reps):
                        layer()
                g.replay()
                if barrier is not None:
                    barrier()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                torch.cuda.synchronize()
                us = P.max_over_ranks(e0.elapsed_time(e1) / reps * 1e3, device=dev)
                gbs = n_total * wbytes / (us * 1e-6) / 1e9
                out[f"{proj}.{arm}.m{mtok}"] = {"us_per_layer": round(us, 2), "us_per_expert": round(us / n_exp, 3),
                                                "weight_gbs": round(gbs, 1), "hbm_frac": round(gbs / (hbm * world), 3)}
                del g, toks
            del wq
    return out


def run_e2e(torch, M, P, dev, world, args, acts, outs, wq, step_flops_global, barrier, n_layers, cols):
    """The headline step through the public API from pinned HOST bf16
    activations to HOST bf16 products.  Every rank uploads the (replicated or
    own) activations and downloads its own products (columns mode: its column
    shard -- the host holds the whole product across ranks); the time is the
    max over ranks."""
    bf16 = torch.bfloat16
    V = M.Variant
    host_in = [a.cpu().pin_memory() for a in acts]
    host_out = [torch.empty(o.shape, dtype=bf16).pin_memory() for o in outs]
    # two device buffer sets: step i+1's uploads and GEMMs run while step i's
    # products are still being read back (steps pipelined as a server would
    # run them; every step still moves all its bytes)
    dev_in = [[torch.empty_like(a) for a in acts] for _ in range(2)]
    dev_out = [[torch.empty_like(o) for o in outs] for _ in range(2)]
    cfg_a = M.SchemeConfig(V.MBS_S)
    s_h2d, s_d2h = torch.cuda.Stream(), torch.cuda.Stream()
    comp = torch.cuda.current_stream()
    consumed = [[None] * n_layers for _ in range(2)]   # compute done reading dev_in[b][li]
    drained = [[None] * n_layers for _ in range(2)]    # D2H done reading dev_out[b][li]
    status_acc = torch.zeros(1, dtype=torch.int32, device=dev)   # non-finite flags of every step

    def e2e_step(it):
        # H2D on one copy engine, D2H on the other, compute in between: layer
        # li's input lands while li-1 computes, its product leaves while li+1
        # computes (PCIe is full duplex)
        b = it % 2
        landed = []
        for li in range(n_layers):
            with torch.cuda.stream(s_h2d):
                if consumed[b][li] is not None:
                    s_h2d.wait_event(consumed[b][li])
                dev_in[b][li].copy_(host_in[li], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(s_h2d)
            landed.append(ev)
        for li in range(n_layers):
            comp.wait_event(landed[li])
            if drained[b][li] is not None:
                comp.wait_event(drained[b][li])
            # public API; the non-finite status is checked after the timed region
            aq = M.quantize_tensor(dev_in[b][li], cfg_a, check=False)
            # OR the status word into one accumulator: holding the status view
            # itself would keep the call's whole output allocation alive, and
            # every later quantize call would then cudaMalloc (2-3 ms of host
            # time each: the e2e leg ran host-bound at 20-60 ms per step)
            status_acc.bitwise_or_(aq._cache["status"][:1])
            M.matmul_quantized(aq, wq[li], out=dev_out[b][li], out_dtype=bf16, check=False)
            done = torch.cuda.Event()
            done.record(comp)
            consumed[b][li] = done
            with torch.cuda.stream(s_d2h):
                s_d2h.wait_event(done)
                host_out[li].copy_(dev_out[b][li], non_blocking=True)
                dr = torch.cuda.Event()
                dr.record(s_d2h)
                drained[b][li] = dr

    W, K = args.warmup, args.steps
    for it in range(max(env_int("MXQ_E2E_WARMUP", 8), W)):
        e2e_step(it)
    torch.cuda.synchronize()
    ke = max(8, K)
    barrier()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t_enq = 0.0
    for it in range(ke):
        tq = time.perf_counter()
        e2e_step(it)
        t_enq += time.perf_counter() - tq
    comp.wait_stream(s_d2h)   # the last step's products are on the host
    e1.record()
    torch.cuda.synchronize()
    ms_e2e = P.max_over_ranks(e0.elapsed_time(e1) / ke, device=dev)
    wall = P.max_over_ranks((time.perf_counter() - t0) * 1e3 / ke, device=dev)
    M._lib.raise_on_status(status_acc)
    host_ok = bool(torch.equal(host_out[0], dev_out[(ke - 1) % 2][0].cpu()))
    # the link's rate in the same run, both directions at once on the two copy
    # streams (the e2e step is bound by it; it varies between runs of one box)
    nb = 256 << 20
    hb = [torch.empty(nb, dtype=torch.uint8).pin_memory() for _ in range(2)]
    db = [torch.empty(nb, dtype=torch.uint8, device=dev) for _ in range(2)]
    for rep in range(2):
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        s_h2d.wait_event(f0)
        s_d2h.wait_event(f0)
        with torch.cuda.stream(s_h2d):
            db[0].copy_(hb[0], non_blocking=True)
        with torch.cuda.stream(s_d2h):
            hb[1].copy_(db[1], non_blocking=True)
        comp.wait_stream(s_h2d)
        comp.wait_stream(s_d2h)
        f1.record()
        torch.cuda.synchronize()
    duplex = nb / (f0.elapsed_time(f1) * 1e-3) / 1e9
    bound_ms = max(sum(a.numel() * 2 for a in acts), sum(o.numel() * 2 for o in outs)) / (duplex * 1e9) * 1e3
    return {"value": step_flops_global / (ms_e2e * 1e-3) / 1e12, "unit": "TFLOP/s",
            "pcie_duplex_gbs_each_way": round(duplex, 1), "host_enqueue_ms_per_step": round(t_enq * 1e3 / ke, 3), "pcie_bound_ms_per_step": round(bound_ms, 3),
            "h2d_bytes_per_step": int(sum(a.numel() * 2 for a in acts)) * world,
            "d2h_bytes_per_step": int(sum(o.numel() * 2 for o in outs)) * world,
            "ms_per_step": ms_e2e, "wall_ms_per_step": wall, "steps": ke,
            "pipelined": "step i+1's uploads and GEMMs overlap step i's downloads (double-buffered); "
                         "the timed region ends when the last step's products are in host memory",
            "host_copy_matches_device": host_ok}


def run_layers(args, world, rank, local, dev, backend):
    """C3: Qwen3-8B whole-model weight quantization (MBS-D exact) + prefill
    GEMMs (MBS-H, M = 4096), the 36 layers sharded over the ranks
    (parallel.layer_owner); no exchange.  A step = quantize every owned
    layer's 7 weight matrices from bf16 + run their prefill GEMMs (activation
    quantization included).  value = all ranks' prefill GEMM FLOPs / the
    max-over-ranks step time."""
    import torch
    import torch.distributed as dist

    import paper_2603_08713_b200 as M
    from paper_2603_08713_b200 import parallel as P

    V = M.Variant
    bf16 = torch.bfloat16
    owner = P.layer_owner(QWEN3_LAYERS, world)
    mine = [l for l in range(QWEN3_LAYERS) if owner[l] == rank]
    # weights of the owned layers, seeded per (layer, projection)
    wdense = {}
    for l in mine:
        for pi, (name, n, k) in enumerate(QWEN3_8B):
            gw = torch.Generator(device=dev).manual_seed(10_000 * l + pi)
            wdense[(l, pi)] = (torch.randn(n, k, device=dev, generator=gw) * 0.02).to(bf16)
    g = torch.Generator(device=dev).manual_seed(99)
    acts = {k: synth_activation(torch, dev, M_TOK, k, g) for k in sorted({k for _, _, k in QWEN3_8B})}
    outs = {pi: torch.empty(M_TOK, n, device=dev, dtype=bf16) for pi, (_, n, _) in enumerate(QWEN3_8B)}
    wcfg, acfg = M.SchemeConfig(V.MBS_D), M.SchemeConfig(V.MBS_S)

    def quantize_weights():
        return {key: M.quantize_tensor(w, wcfg, check=False) for key, w in wdense.items()}

    def prefill(wq):
        for (l, pi), q in wq.items():
            _, n, k = QWEN3_8B[pi]
            aq = M.quantize_tensor(acts[k], acfg, check=False)
            M.matmul_quantized(aq, q, out=outs[pi], out_dtype=bf16, check=False)

    def barrier():
        if world > 1:
            if backend == "nccl":
                dist.barrier(device_ids=[local])
            else:
                dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        prefill(quantize_weights())
    barrier()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    tq = tp = 0.0
    with Clocks(local) as clocks:
        for _ in range(args.steps):
            e[0].record()
            wq = quantize_weights()
            e[1].record()
            prefill(wq)
            e[2].record()
            torch.cuda.synchronize()
            tq += e[0].elapsed_time(e[1])
            tp += e[1].elapsed_time(e[2])
    barrier()
    tq, tp = tq / args.steps, tp / args.steps
    t_step = P.max_over_ranks(tq + tp, device=dev)
    tq_max, tp_max = P.max_over_ranks(tq, device=dev), P.max_over_ranks(tp, device=dev)
    params = sum(n * k for _, n, k in QWEN3_8B) * QWEN3_LAYERS
    flops = 2.0 * M_TOK * params
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(flops / (t_step * 1e-3) / 1e12, 2), "unit": "TFLOP/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_step, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "fp4_e2m1 (UE8M0 block-16 scales, MBS sigma f32, f32 accum)",
            "data": "synthetic (random-init N(0,0.02) bf16 weights per (layer, projection); activations "
                    "student-t dof 4)",
            "config": {"workload": "qwen3-8b: 36 layers x {q,k,v,o,gate,up,down} (6.95 B params) MBS-D exact "
                                   "weight quantization + MBS-H prefill GEMMs at M=4096, per step",
                       "global_batch": M_TOK, "seq_len": None,
                       "parallelism": f"layer-shard x{world} (parallel.layer_owner, no collective)"},
            "weight_quant_ms": round(tq_max, 3),
            "weight_quant_gelem_s": round(params / world / (tq_max * 1e-3) / 1e9, 2),
            "prefill_ms": round(tp_max, 3),
            "prefill_tflops": round(flops / (tp_max * 1e-3) / 1e12, 2),
            "layers_per_rank": len(mine),
            "gpu_launches": args.steps * len(wdense) * 3,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def cpu_baseline_sample(weights_from_gpu, acts, rows: int):
    """Reference algorithm on the host cores: quantize a row sample of every
    layer's activation with the CPU oracle (MBS-S), dequantize, f64 GEMM
    against the dequantized MBS-D weights (weights prepared outside the
    timed region, as on the GPU)."""
    import torch

    from oracle import mxq_oracle as O

    wdq = []
    for q in weights_from_gpu:
        h = q.to_host()
        oq = O.OracleQ("mbs_d", h["shape"], 16, 128, h["codes"], h["block_scales"], None, h["mbs_mantissas"], None)
        wdq.append(O.dequantize(oq).astype(np.float64))
    samples = [a[:rows].float().cpu().numpy() for a in acts]
    t0 = time.perf_counter()
    flops = 0.0
    for x, w in zip(samples, wdq):
        q = O.quantize(x, "mbs_s")
        xd = O.dequantize(q).astype(np.float64)
        c = (xd @ w.T).astype(np.float32)
        flops += 2.0 * x.shape[0] * w.shape[0] * w.shape[1]
    dt = time.perf_counter() - t0
    return {"value": round(flops / dt / 1e12, 6), "unit": "TFLOP/s", "cores": os.cpu_count(), "kind": "port",
            "sample": f"{rows} of 4096 token rows per layer, all 4 layers (MBS_S quantize + dequant + f64 BLAS "
                      f"GEMM vs pre-dequantized MBS_D weights); {dt:.2f} s"}


# ---------------------------------------------------------------------------
# reference arm: the reference algorithm (oracle port) on the host cores
# ---------------------------------------------------------------------------
def run_reference(args):
    rank = env_int("RANK", 0)
    if rank != 0:
        return
    from concurrent.futures import ProcessPoolExecutor

    from oracle import mxq_oracle as O

    cores = os.cpu_count() or 1
    rows = args.ref_rows
    rng = np.random.Generator(np.random.PCG64(1234))
    wrng = np.random.Generator(np.random.PCG64(4321))
    # weights: MBS-D on a column sample (prepared outside the timed region)
    ncols_sample = args.ref_wrows
    with ProcessPoolExecutor(max_workers=cores) as pool:
        wdq = []
        for _, n, k in LAYERS:
            w = (wrng.standard_normal((min(n, ncols_sample), k)) * 0.02).astype(np.float32)
            wdq.append(O.dequantize(O.quantize_sharded(w, "mbs_d", cores, pool)).astype(np.float64))
        acts = []
        for _, n, k in LAYERS:
            x = rng.standard_t(4, (rows, k)).astype(np.float32)  # the reference's activation_like
            acts.append(O.bf16_round(x))

        def step():
            fl = 0.0
            for x, w in zip(acts, wdq):
                q = O.quantize_sharded(x, "mbs_s", cores, pool)
                xd = O.dequantize(q).astype(np.float64)
                _ = (xd @ w.T).astype(np.float32)
                fl += 2.0 * x.shape[0] * w.shape[0] * w.shape[1]
            return fl

        for _ in range(args.warmup):
            step()
        t0 = time.perf_counter()
        fl = 0.0
        for _ in range(args.steps):
            fl += step()
        dt = (time.perf_counter() - t0) / args.steps
    val = fl / args.steps / dt / 1e12
    line = {
        "metric": METRIC, "value": round(val, 6), "unit": "TFLOP/s", "n_gpus": env_int("WORLD_SIZE", 1),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True,
        # (labelled like our arm's line for the same launch: columns mode at N > 1)
        "scaling": "strong" if env_int("WORLD_SIZE", 1) > 1 and args.mode in ("auto", "columns") else "weak",
        "vs_baseline": None, "dtype": "fp64 reference arithmetic (numpy)",
        "data": "synthetic", "impl": "reference",
        "config": {"workload": WORKLOAD, "global_batch": M_TOK, "seq_len": None, "parallelism": "host cores"},
        "cpu_baseline": {"value": round(val, 6), "unit": "TFLOP/s", "cores": cores, "kind": "port",
                         "sample": f"{rows} token rows x {ncols_sample} weight rows per layer (4 layers): "
                                   f"row-sharded MBS_S quantize over {cores} processes + dequant + f64 BLAS GEMM"},
        "e2e": {"value": round(val, 6), "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--mode", default="auto", choices=("auto", "replicas", "columns", "layers"),
                    help="auto: N=1 single GPU, N>1 columns (column shards + overlapped all_gather, strong); "
                         "replicas: every rank its own tokens (weak, no collective); layers: C3 Qwen3-8B "
                         "whole-model weight quantization + prefill, layers sharded")
    ap.add_argument("--workload", default="llama8b", choices=tuple(WORKLOADS),
                    help="llama8b: the four Llama-3-8B linears (C2); llama70b-ffn: the 70B FFN gate/up (C4)")
    ap.add_argument("--chunks", type=int, default=4, help="columns mode: row blocks of the gather overlap")
    ap.add_argument("--no-experts", dest="experts", action="store_false",
                    help="skip the C5 grouped expert-GEMM block (MBS-H vs NVFP4)")
    ap.add_argument("--cpu-rows", type=int, default=256)
    ap.add_argument("--ref-rows", type=int, default=256)
    ap.add_argument("--ref-wrows", type=int, default=2048)
    ap.add_argument("--no-graphs", dest="graphs", action="store_false",
                    help="launch every kernel eagerly instead of replaying a captured CUDA graph")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
