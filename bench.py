#!/usr/bin/env python
"""Benchmark of the B200 MXFP4 quantize-and-GEMM path (BASELINE.json configs[1]).

Workload (one "step"): the four Llama-3-8B linear layers at M = 4096 tokens --
QKV (N 6144, K 4096), O (4096, 4096), gate_up (28672, 4096), down (4096, 14336)
-- each = quantize the bf16 activation on the fly (MBS-S) and run the tcgen05
block-scaled GEMM against resident MBS-D weights (MBS-H, the paper's default),
bf16 output.  Synthetic data: activations gaussian with 1% x100 outliers,
random-init weights N(0, 0.02).  Headline `value` = step TFLOP/s (device-timed,
inputs resident in HBM); `e2e` = the same step through the public API with
pinned host activations in and bf16 products out.  Comparison arms on the
same shapes: plain MXFP4 (OCP32 block-32, kind::mxf4), MX16+OAS and NVFP4.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (torchrun): every layer is column-sharded (weight rows) across ranks and
the bf16 outputs are all-gathered over NVLink (strong scaling, SURVEY §8 e).
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
    V = M.Variant
    bf16 = torch.bfloat16

    # ---- synthetic inputs (activations replicated, weights sharded) --------
    g = torch.Generator(device=dev).manual_seed(1234)
    acts = []
    for _, n, k in LAYERS:
        x = torch.randn(M_TOK, k, device=dev, generator=g)
        hit = torch.rand(M_TOK, k, device=dev, generator=g) < 0.01
        acts.append(torch.where(hit, x * 100.0, x).to(bf16))
    gw = torch.Generator(device=dev).manual_seed(4321 + rank)
    wdense, bounds = [], []
    cols = args.mode == "columns" and world > 1  # tensor-parallel column shards + all_gather
    for _, n, k in LAYERS:
        lo, hi = P.shard_bounds(n, world, rank) if cols else (0, n)
        bounds.append((lo, hi))
        wdense.append((torch.randn(hi - lo, k, device=dev, generator=gw) * 0.02).to(bf16))

    arms = {  # name -> (activation variant, weight variant)
        "mbs_h": (V.MBS_S, V.MBS_D),
        "ocp32": (V.OCP32, V.OCP32),
        "mx16_oas": (V.MX16_OAS, V.MX16_OAS),
        "nvfp4": (V.NVFP4, V.NVFP4),
    }
    weights = {name: [M.quantize_tensor(w, M.SchemeConfig(wv)) for w in wdense] for name, (_, wv) in arms.items()}
    del wdense
    outs = [torch.empty(M_TOK, hi - lo, device=dev, dtype=bf16) for lo, hi in bounds]
    gathered = [torch.empty(world * M_TOK, max(P.shard_bounds(n, world, r)[1] - P.shard_bounds(n, world, r)[0]
                                               for r in range(world)), device=dev, dtype=bf16)
                if cols else None for _, n, _ in LAYERS]
    n_local_frac = sum(2.0 * M_TOK * (hi - lo) * k for (lo, hi), (_, _, k) in zip(bounds, LAYERS))
    # replicas (default): every rank runs the whole step on its own M tokens,
    # no data-path collective, weak scaling; columns: one step split by output
    # column across ranks plus the bf16 all_gather (config 4's pattern)
    step_flops_global = flops_per_step() * (1 if cols else world)

    def step(arm, gemm_events=None):
        av, _ = arms[arm]
        for li in range(len(LAYERS)):
            aq = M.quantize_tensor(acts[li], M.SchemeConfig(av), check=False)
            if gemm_events is not None:
                gemm_events[li][0].record()
            M.matmul_quantized(aq, weights[arm][li], out=outs[li], out_dtype=bf16, check=False)
            if gemm_events is not None:
                gemm_events[li][1].record()
            if cols:
                send = outs[li]
                if send.shape[1] != gathered[li].shape[1]:
                    pad = torch.zeros(M_TOK, gathered[li].shape[1], device=dev, dtype=bf16)
                    pad[:, : send.shape[1]] = send
                    send = pad
                dist.all_gather_into_tensor(gathered[li], send)

    def barrier():
        if world > 1:
            if backend == "nccl":
                dist.barrier(device_ids=[local])
            else:
                dist.barrier()
        torch.cuda.synchronize()

    graphs = {}

    def capture(arm):
        """The whole step (4 x quantize + GEMM [+ all_gather]) as one CUDA graph."""
        if cols:
            return None  # NCCL collectives are replayed eagerly
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            step(arm)  # warm (allocations, attributes, descriptors)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step(arm)
        return g

    def run_step(arm):
        g = graphs.get(arm)
        if g is not None:
            g.replay()
        else:
            step(arm)

    def time_steps(arm, k, w):
        if args.graphs and arm not in graphs:
            graphs[arm] = capture(arm)
        for _ in range(w):
            run_step(arm)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(k):
            run_step(arm)
        e1.record()
        barrier()
        ms = e0.elapsed_time(e1) / k
        return P.max_over_ranks(ms, device=dev)

    def time_gemms(arm, k):
        """Per-launch device time of the dominant kernel (the GEMM)."""
        evs = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                for _ in LAYERS] for _ in range(k)]
        barrier()
        for i in range(k):
            step(arm, evs[i])
        barrier()
        per_layer = [float(np.mean([evs[i][li][0].elapsed_time(evs[i][li][1]) for i in range(k)]))
                     for li in range(len(LAYERS))]
        return per_layer

    K, W = args.steps, args.warmup
    results = {}
    with Clocks(local) as clocks:
        for arm in ("mbs_h", "ocp32", "mx16_oas", "nvfp4"):
            ms = time_steps(arm, K, W)
            gl = time_gemms(arm, max(3, K // 2))
            gemm_ms = sum(gl)
            results[arm] = {
                "ms_per_step": ms,
                "tflops_step": step_flops_global / (ms * 1e-3) / 1e12,
                "gemm_ms": gemm_ms,
                "gemm_tflops": n_local_frac / (gemm_ms * 1e-3) / 1e12 * world,  # all ranks' GEMM work / per-rank time
                "gemm_ms_per_layer": {name: t for (name, _, _), t in zip(LAYERS, gl)},
            }
    head = results["mbs_h"]

    # ---- quantizer bandwidth (4096x4096 bf16 activations, HBM-cold) -------
    # the timed launches cycle over 8 distinct activations (256 MB, twice the
    # L2), so every launch streams its input from HBM
    qbw = {}
    gq = torch.Generator(device=dev).manual_seed(1234)
    xq = [torch.randn(M_TOK, 4096, device=dev, generator=gq).to(bf16) for _ in range(8)]
    # algorithmic bytes / element: bf16 read + packed codes + scale bytes
    # (+ MBS mantissa byte per 128 elements); the GEMM-layout copies the
    # kernels also write (row-major + MMA-atom scales, f32 sigma) are not
    # counted, so the GB/s is conservative.
    bytes_per_el = {"ocp32": 2 + 0.5 + 1 / 32, "mx16": 2 + 0.5 + 1 / 16, "mx16_oas": 2 + 0.5 + 1 / 16,
                    "mbs_s": 2 + 0.5 + 1 / 16 + 1 / 128, "mbs_d": 2 + 0.5 + 1 / 16 + 1 / 128,
                    "nvfp4": 2 + 0.5 + 1 / 16}
    for vname in ("ocp32", "mx16", "mx16_oas", "mbs_s", "nvfp4", "mbs_d"):
        cfg = M.SchemeConfig(V(vname))
        reps = 8 if vname == "mbs_d" else 48
        for x in xq:
            M.quantize_tensor(x, cfg, check=False, gemm_layout=True)
        torch.cuda.synchronize()
        g = None
        if args.graphs and vname != "mbs_d":  # MBS-D uploads its candidate table per call
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

    out = None
    if rank == 0:
        out = {}
        # ---- QSNR on config 1 (4096x4096 gaussian+outliers seed 0, bf16) ----
        t1 = M.generate_tensor(M.GeneratorSpec("gaussian_with_outliers", (4096, 4096), seed=0))
        t1b = torch.from_numpy(t1).to(dev).to(bf16)
        meta = json.load(open(os.path.join(ROOT, "tests", "golden", "golden_meta.json")))
        qs = {}
        for vname in ("ocp32", "mx16", "mx16_oas", "mbs_s", "mbs_d", "nvfp4"):
            q = M.quantize_tensor(t1b, M.SchemeConfig(V(vname)))
            rep, fl = M.qsnr_quantized(t1b, q)
            ref = meta["config1"][vname]
            qs[vname] = {"qsnr_db": round(rep.qsnr_db, 6), "flush": round(fl, 6),
                         "equals_reference": rep.qsnr_db == ref["qsnr_db"] and fl == ref["flush"]}
        out["qsnr"] = qs

    # ---- e2e: public API, pinned host activations in, bf16 out -------------
    # every rank (replicas) runs its own step from its own pinned host buffers;
    # the time is the max over ranks
    e2e = None
    if not cols:
        host_in = [a.cpu().pin_memory() for a in acts]
        host_out = [torch.empty(o.shape, dtype=bf16).pin_memory() for o in outs]
        # two device buffer sets: step i+1's uploads and GEMMs run while step
        # i's products are still being read back (steps pipelined as a server
        # would run them; every step still moves all its bytes)
        dev_in = [[torch.empty_like(a) for a in acts] for _ in range(2)]
        dev_out = [[torch.empty_like(o) for o in outs] for _ in range(2)]
        cfg_a = M.SchemeConfig(V.MBS_S)
        s_h2d, s_d2h = torch.cuda.Stream(), torch.cuda.Stream()
        comp = torch.cuda.current_stream()
        consumed = [[None] * len(LAYERS) for _ in range(2)]   # compute done reading dev_in[b][li]
        drained = [[None] * len(LAYERS) for _ in range(2)]    # D2H done reading dev_out[b][li]
        statuses = []

        def e2e_step(it):
            # H2D on one copy engine, D2H on the other, compute in between:
            # layer li's input lands while li-1 computes, its product leaves
            # while li+1 computes (PCIe is full duplex)
            b = it % 2
            landed = []
            for li in range(len(LAYERS)):
                with torch.cuda.stream(s_h2d):
                    if consumed[b][li] is not None:
                        s_h2d.wait_event(consumed[b][li])
                    dev_in[b][li].copy_(host_in[li], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(s_h2d)
                landed.append(ev)
            for li in range(len(LAYERS)):
                comp.wait_event(landed[li])
                if drained[b][li] is not None:
                    comp.wait_event(drained[b][li])
                # public API; the non-finite status is checked after the timed region
                aq = M.quantize_tensor(dev_in[b][li], cfg_a, check=False)
                statuses.append(aq._cache["status"])
                M.matmul_quantized(aq, weights["mbs_h"][li], out=dev_out[b][li], out_dtype=bf16, check=False)
                done = torch.cuda.Event()
                done.record(comp)
                consumed[b][li] = done
                with torch.cuda.stream(s_d2h):
                    s_d2h.wait_event(done)
                    host_out[li].copy_(dev_out[b][li], non_blocking=True)
                    dr = torch.cuda.Event()
                    dr.record(s_d2h)
                    drained[b][li] = dr

        for it in range(max(2, W // 2)):
            e2e_step(it)
        torch.cuda.synchronize()
        ke = max(4, K // 2)
        barrier()
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for it in range(ke):
            e2e_step(it)
        comp.wait_stream(s_d2h)   # the last step's products are on the host
        e1.record()
        torch.cuda.synchronize()
        ms_e2e = P.max_over_ranks(e0.elapsed_time(e1) / ke, device=dev)
        wall = P.max_over_ranks((time.perf_counter() - t0) * 1e3 / ke, device=dev)
        for st in statuses:
            M._lib.raise_on_status(st)
        host_ok = bool(torch.equal(host_out[0], dev_out[(ke - 1) % 2][0].cpu()))
        e2e = {"value": step_flops_global / (ms_e2e * 1e-3) / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": int(sum(a.numel() * 2 for a in acts)) * world,
               "d2h_bytes_per_step": int(sum(o.numel() * 2 for o in outs)) * world,
               "ms_per_step": ms_e2e, "wall_ms_per_step": wall, "steps": ke,
               "pipelined": "step i+1's uploads and GEMMs overlap step i's downloads (double-buffered); "
                            "the timed region ends when the last step's products are in host memory",
               "host_copy_matches_device": host_ok}
    if world > 1:
        barrier()

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel (tcgen05 GEMM, MBS-H) -------------
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
    achieved = head["gemm_tflops"]
    traffic = None
    prof = os.path.join(ROOT, "profiles", "gemm_traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get("mbs_h_bytes_per_launch")
        except Exception:
            traffic = None
    # MBS-specific ceiling: the epilogue folds every
    # 128-K macro partial with two FP32 ops per output, 128 FP32 lanes/clk/SM
    # -> 64 output-macros x 128 K x 2 flop per clock per SM
    clk = clocks.summary()
    f_mhz = clk.get("sm_mhz") or clk.get("sm_max_mhz") or 1965.0
    fp32_bound = 148 * 64 * 128 * 2 * f_mhz * 1e6 / 1e12
    roofline = {"bound": "tensor", "achieved": round(achieved, 1), "peak": round(fp4_peak, 1), "unit": "TFLOP/s",
                "frac": round(achieved / fp4_peak, 4), "traffic": traffic, "peak_basis": basis,
                "kernel": "mbs::k_gemm_mbs<BN=192,NB=2,bf16,CL=2> (kind::mxf4nvf4.block16 UE8M0, N=192 MMAs, "
                          "tcgen05.cp scale factors, 16 FP32 epilogue warps)",
                "mbs_fp32_epilogue_bound": round(fp32_bound, 1),
                "frac_of_mbs_fp32_bound": round(achieved / fp32_bound, 4),
                "mbs_bound_basis": f"2 FP32 ops per output per 128-K macro at 128 FP32 lanes/clk/SM, {f_mhz:.0f} MHz",
                "traffic_basis": "profiles/gemm_traffic.json: ncu --set full DRAM bytes per launch, mean of the same 4 layer launches",
                "algorithmic": "2*M*N*K per launch over the 4 layer launches, CUDA events on the launch stream"}

    # ---- CPU baseline: the reference algorithm (oracle port) on a sample ---
    cpu = cpu_baseline_sample(weights_from_gpu=[weights["mbs_h"][li] for li in range(len(LAYERS))],
                              acts=acts, rows=args.cpu_rows)

    ocp = results["ocp32"]
    line = {
        "metric": METRIC, "value": round(head["tflops_step"], 2), "unit": "TFLOP/s", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": round(head["ms_per_step"], 4), "higher_is_better": True,
        "scaling": "strong" if cols else "weak", "vs_baseline": None,
        "dtype": "fp4_e2m1 (UE8M0 block-16 scales, MBS sigma f32, f32 accum)",
        "data": "synthetic (activations N(0,1) with 1% x100 outliers; random-init N(0,0.02) weights)",
        "config": {"workload": WORKLOAD, "global_batch": M_TOK * (1 if cols else world), "seq_len": None,
                   "parallelism": (f"column-shard x{world} + all_gather" if cols else
                                   f"replicas x{world} (token-parallel, no collective)") if world > 1 else "single",
                   "l2": "inputs larger than L2 (218 MB bf16 activations + 121 MB fp4 weights per step)"},
        "gemm_only_tflops": round(head["gemm_tflops"], 2),
        "arms": {k: {kk: (round(vv, 4) if isinstance(vv, float) else vv) for kk, vv in v.items()}
                 for k, v in results.items()},
        "mbs_h_overhead_vs_ocp32": round(1.0 - head["tflops_step"] / ocp["tflops_step"], 4),
        "mbs_h_gemm_overhead_vs_ocp32": round(1.0 - head["gemm_tflops"] / ocp["gemm_tflops"], 4),
        "mbs_h_overhead_vs_nvfp4": round(1.0 - head["tflops_step"] / results["nvfp4"]["tflops_step"], 4),
        "quantizer": {k: {kk: round(vv, 2) for kk, vv in v.items()} for k, v in qbw.items()},
        "quantizer_hbm_frac_mbs_s": round(qbw["mbs_s"]["gbs"] / peaks.get("hbm_gbs", 6650.0), 4),
        "qsnr_config1": out["qsnr"],
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": 8 * K,
        "clocks": clk,
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
            x = rng.standard_normal((rows, k))
            x = np.where(rng.random((rows, k)) < 0.01, x * 100, x).astype(np.float32)
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
        "scaling": "weak", "vs_baseline": None, "dtype": "fp64 reference arithmetic (numpy)",
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
    ap.add_argument("--mode", default="replicas", choices=("replicas", "columns"),
                    help="N>1: independent replicas on their own tokens (weak) or column shards + all_gather (strong)")
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
