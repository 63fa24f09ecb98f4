"""Quantized GEMM on the B200 (drop-in for src/gemm.py).

``matmul_quantized`` runs the tcgen05 block-scaled kernel (csrc/gemm_tc.cu)
for every operand pair the tensor cores can take natively (any two
E8M0-scaled variants, NVFP4 x NVFP4), applying the MBS factor per 128-K macro
chunk in the epilogue; its output matches the reference dequantize-then-f64
matmul within the tolerance stated in DESIGN.md.  E8M0 x NVFP4 pairs
run on the tensor cores too when the E8M0 operand's block exponents span at
most 17 (its scales re-expressed exactly as UE4M3 powers of two);
``exact=True`` (and mixed pairs outside that span) use the CUDA-core f64
kernel (csrc/gemm_exact.cu), which is bit-identical to the reference's
``matmul_quantized`` / ``matmul_reference``.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .quantize import QuantizedTensor, SchemeConfig, Variant, quantize_tensor

__all__ = ["TileConfig", "OverheadReport", "matmul_reference", "matmul_quantized", "matmul_quantized_grouped",
           "quantize_matmul",
           "roofline_overhead", "max_ulp_divergence", "tc_supported"]


@dataclass(frozen=True)
class TileConfig:
    """Output tile (t_m x t_n) and k-chunk t_k (src/gemm.py:33-43).  Tiles
    never change results; t_k is validated exactly like the reference and
    otherwise unused (the kernels chunk K at the macro size)."""

    t_m: int = 128
    t_n: int = 128
    t_k: int = 128

    def __post_init__(self) -> None:
        if self.t_m <= 0 or self.t_n <= 0 or self.t_k <= 0:
            raise ValueError(f"tile dims must be positive, got {self}")


@dataclass(frozen=True)
class OverheadReport:
    compute_ratio: float
    traffic_ratio: float


def _dense_f32(t, name: str) -> torch.Tensor:
    dev = _lib.require_device()
    x = t if isinstance(t, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(t, dtype=np.float32))
    x = x.to(device=dev, dtype=torch.float32)
    if x.ndim != 2:
        raise ValueError(f"{name} must be 2-D, got shape {tuple(x.shape)}")
    return x.contiguous()


def matmul_reference(a, b) -> torch.Tensor:
    """C = A @ B.T with f64 products summed in ascending k, one f32 rounding
    (src/gemm.py:68-90), on CUDA cores; bit-identical to the reference."""
    a32, b32 = _dense_f32(a, "a"), _dense_f32(b, "b")
    if a32.shape[1] != b32.shape[1]:
        raise ValueError(f"inner dimensions differ: {tuple(a32.shape)} vs {tuple(b32.shape)}")
    m, k = a32.shape
    n = b32.shape[0]
    c = torch.empty((m, n), dtype=torch.float32, device=a32.device)
    _lib.check(_lib.lib().mxq_matmul_reference(a32.data_ptr(), k, b32.data_ptr(), k, m, n, k, c.data_ptr(), n,
                                               _lib.stream_handle()), "matmul_reference")
    return c


def _validate_chunking(q: QuantizedTensor, t_k: int, name: str) -> None:
    """src/gemm.py:126-134."""
    if t_k % q.block_size != 0:
        raise ValueError(f"t_k {t_k} is not a multiple of operand {name}'s block size {q.block_size}")
    if q.mbs_mantissas is not None and t_k % q.macro_size != 0:
        raise ValueError(f"t_k {t_k} is not a multiple of operand {name}'s macro size {q.macro_size}")


def tc_supported(aq: QuantizedTensor, bq: QuantizedTensor) -> bool:
    """Whether the pair runs on the tcgen05 block-scaled path."""
    nva, nvb = aq.variant is Variant.NVFP4, bq.variant is Variant.NVFP4
    if nva != nvb:
        return False  # UE8M0 x UE4M3: no single MMA scale format
    for q in (aq, bq):
        if q.mbs_mantissas is not None and q.macro_size % 64:
            return False  # sigma chunks must align with the 64-K MMA step
    if aq.mbs_mantissas is not None and bq.mbs_mantissas is not None and aq.macro_size != bq.macro_size:
        return False
    return True


def _e4m3_pow2_code(k: int) -> int:
    """E4M3 byte of 2**k, k in [-9, 8] (subnormals 2^-9..2^-7 = codes 1, 2, 4)."""
    return (k + 7) << 3 if k >= -6 else 1 << (k + 9)


def _ue4m3_view(q: QuantizedTensor):
    """The UE8M0 operand's tcgen05 scale atoms re-expressed as UE4M3 powers of
    two, or None: 2^(b - 127) -> 2^(b - 127 - off) is exact in E4M3 (2^-9 ..
    2^8) when the block exponents span at most 17 (hard part
    8, option A; the span the reference measures in within_e4m3_span_fraction,
    src/metrics.py:185-207).  Returns (scales_mma bytes, off); the power of two
    2^off is folded into the NVFP4 side's tensor scale.  Cached per tensor."""
    c = q._cache
    if "ue4m3" in c:
        return c["ue4m3"]
    lo, hi = (int(v) for v in torch.aminmax(q.block_scales))
    res = None
    if hi - lo <= 17:
        off = hi - 127 - 8
        lut = torch.zeros(256, dtype=torch.uint8)
        for b in range(lo, hi + 1):
            lut[b] = _e4m3_pow2_code(b - 127 - off)
        q.gemm_qt(16)
        mma = c[("mma", 16)]
        # (padding bytes hold 0: they map to lut[0], finite, against zero data)
        res = (lut.to(mma.device)[mma.long()].contiguous(), off)
    c["ue4m3"] = res
    return res


def _mixed_pair_qts(aq: QuantizedTensor, bq: QuantizedTensor):
    """Descriptors for a UE8M0 x NVFP4 pair on the tcgen05 path (the UE8M0
    side's scales re-expressed as UE4M3, its 2^off folded into the NVFP4
    tensor scale), or None when the span does not fit (exact path)."""
    if (aq.variant is Variant.NVFP4) == (bq.variant is Variant.NVFP4):
        return None
    e8, nv = (aq, bq) if bq.variant is Variant.NVFP4 else (bq, aq)
    if e8.mbs_mantissas is not None and e8.macro_size % 64:
        return None
    view = _ue4m3_view(e8)
    if view is None:
        return None
    sf, off = view
    q8 = _lib.QT.from_buffer_copy(e8.gemm_qt(16))
    q8.scales_mma, q8.sf_format = sf.data_ptr(), 1
    ts = nv._ts_device() * (2.0 ** off)
    qn = _lib.QT.from_buffer_copy(nv.gemm_qt(16))
    qn.tensor_scale = ts.data_ptr()
    keep = (sf, ts)
    return ((q8, qn) if e8 is aq else (qn, q8)), keep


def _sf_block(aq: QuantizedTensor, bq: QuantizedTensor) -> int:
    return 32 if (aq.block_size == 32 and bq.block_size == 32) else 16


def matmul_quantized(aq: QuantizedTensor, bq: QuantizedTensor, cfg: TileConfig = TileConfig(), *,
                     exact: bool = False, out_dtype: torch.dtype = torch.float32, out: torch.Tensor = None,
                     check: bool = True) -> torch.Tensor:
    """C = dequant(aq) @ dequant(bq).T (src/gemm.py:137-172) as a CUDA tensor.

    Operand variants may be mixed (e.g. MBS-H = MBS_S activations x MBS_D
    weights).  ``exact=True`` gives the reference's bit-exact f64 result.
    """
    if aq.shape[1] != bq.shape[1]:
        raise ValueError(f"operands disagree on K: {aq.shape} vs {bq.shape}")
    _validate_chunking(aq, cfg.t_k, "a")
    _validate_chunking(bq, cfg.t_k, "b")
    m, n = aq.shape[0], bq.shape[0]
    dev = aq.codes.device
    if out_dtype not in (torch.float32, torch.bfloat16):
        raise ValueError("out_dtype must be float32 or bfloat16")
    if out is not None:
        _check_out(out, m, n, out_dtype, dev)
    stream = _lib.stream_handle()
    L = _lib.lib()
    mixed = None if (exact or tc_supported(aq, bq)) else _mixed_pair_qts(aq, bq)
    if mixed is not None:
        # UE8M0 x NVFP4 on tensor cores: both scale sets as UE4M3 (exact re-expression)
        if check:
            _check_scale_codes(aq)
            _check_scale_codes(bq)
        (qa, qb), keep = mixed
        c = out if out is not None else torch.empty((m, n), dtype=out_dtype, device=dev)
        dt = _lib.MXQ_BF16 if out_dtype == torch.bfloat16 else _lib.MXQ_F32
        _lib.check(L.mxq_gemm(ctypes.byref(qa), ctypes.byref(qb), c.data_ptr(), dt, c.stride(0), None, stream),
                   "matmul_quantized")
        c._mxq_keep = keep  # the re-expressed scales / folded tensor scale outlive the async launch
        return c
    if exact or not tc_supported(aq, bq):
        c = torch.empty((m, n), dtype=torch.float32, device=dev)
        status = torch.zeros(4, dtype=torch.int32, device=dev)
        qa, qb = aq.qt(), bq.qt()
        _lib.check(L.mxq_gemm_exact(ctypes.byref(qa), ctypes.byref(qb), c.data_ptr(), n, status.data_ptr(), stream),
                   "matmul_quantized(exact)")
        if check:
            _lib.raise_on_status(status)
        if out is not None:
            out.copy_(c)
            return out
        return c if out_dtype == torch.float32 else c.to(out_dtype)
    if check:
        _check_scale_codes(aq)
        _check_scale_codes(bq)
    c = out if out is not None else torch.empty((m, n), dtype=out_dtype, device=dev)
    sfb = _sf_block(aq, bq)
    qa, qb = aq.gemm_qt(sfb), bq.gemm_qt(sfb)
    dt = _lib.MXQ_BF16 if out_dtype == torch.bfloat16 else _lib.MXQ_F32
    # (the tcgen05 kernels report nothing through the status word: no buffer)
    _lib.check(L.mxq_gemm(ctypes.byref(qa), ctypes.byref(qb), c.data_ptr(), dt, c.stride(0), None, stream),
               "matmul_quantized")
    return c


def _check_out(out: torch.Tensor, m: int, n: int, out_dtype: torch.dtype, dev) -> None:
    """``out=`` must be exactly the result tensor the call would allocate
    (shape, dtype, device, unit column stride): the kernels write through
    its pointer and row pitch."""
    if not isinstance(out, torch.Tensor) or tuple(out.shape) != (m, n):
        raise ValueError(f"out must have shape {(m, n)}, got {getattr(out, 'shape', None)}")
    if out.dtype != out_dtype:
        raise ValueError(f"out has dtype {out.dtype} but out_dtype is {out_dtype}")
    if out.device != dev:
        raise ValueError(f"out is on {out.device}, the operands on {dev}")
    if out.stride(1) != 1 or out.stride(0) < n:
        raise ValueError("out must have unit column stride and a row pitch >= n")


def _check_scale_codes(q: QuantizedTensor) -> None:
    """The reference's corrupt-scale ValueError (src/quantize.py:228-241),
    checked once per tensor: the quantizers never write an E8M0 255 or an
    E4M3 NaN byte, so only tensors built or edited by the caller are scanned."""
    c = q._cache
    if c.get("scales_ok") or "status" in c:
        return
    if q.variant is Variant.NVFP4:
        if bool(((q.e4m3_scales & 0x7F) == 0x7F).any()):
            raise ValueError("corrupt block scale: E4M3 NaN code")
    elif bool((q.block_scales == 255).any()):
        raise ValueError("corrupt block scale: E8M0 code 255 is reserved")
    c["scales_ok"] = True


def matmul_quantized_grouped(aqs, bqs, cfg: TileConfig = TileConfig(), *, out_dtype: torch.dtype = torch.float32,
                             check: bool = True) -> list:
    """``[matmul_quantized(a, b) for a, b in zip(aqs, bqs)]`` for MoE-style
    expert GEMMs (SURVEY section 8 d config 5): ``aqs[g]`` the tokens routed
    to expert g (at most 128 rows for the grouped kernel), ``bqs[g]`` that
    expert's weights, all of one shape.  MBS pairs (MBS-H: MBS_S tokens x
    MBS_D weights, or an MBS side against E8M0) and NVFP4 x NVFP4 pairs run
    as one launch per 64 experts (swap-AB up to 64 tokens, direct 128-row
    tiles up to 128) (csrc/gemm_mbs.cu ``k_gemm_mbs_grouped``; NVFP4 groups
    use UE4M3 scales, one K chunk and the s_tA s_tB epilogue); other pairs
    fall back to one launch per expert.  Tolerance parity as
    ``matmul_quantized``."""
    aqs, bqs = list(aqs), list(bqs)
    if len(aqs) != len(bqs) or not aqs:
        raise ValueError("need one weight per token group")
    n = bqs[0].shape[0]
    for aq, bq in zip(aqs, bqs):
        if aq.shape[1] != bq.shape[1]:
            raise ValueError(f"operands disagree on K: {aq.shape} vs {bq.shape}")
        if bq.shape != bqs[0].shape:
            raise ValueError("every expert's weights must have one shape")
        _validate_chunking(aq, cfg.t_k, "a")
        _validate_chunking(bq, cfg.t_k, "b")
    if out_dtype not in (torch.float32, torch.bfloat16):
        raise ValueError("out_dtype must be float32 or bfloat16")
    # the grouped kernel takes MBS pairs and NVFP4 x NVFP4 pairs (block-16 scale
    # layouts); anything else runs expert by expert through matmul_quantized
    def grouped_pair(aq, bq):
        if aq.variant is Variant.NVFP4 or bq.variant is Variant.NVFP4:
            return aq.variant is Variant.NVFP4 and bq.variant is Variant.NVFP4
        return tc_supported(aq, bq) and (aq.mbs_mantissas is not None or bq.mbs_mantissas is not None)

    if not all(grouped_pair(aq, bq) for aq, bq in zip(aqs, bqs)):
        return [matmul_quantized(aq, bq, cfg, out_dtype=out_dtype, check=check) for aq, bq in zip(aqs, bqs)]
    if check:
        for q in (*aqs, *bqs):
            _check_scale_codes(q)
    dev = aqs[0].codes.device
    outs = [torch.empty((aq.shape[0], n), dtype=out_dtype, device=dev) for aq in aqs]
    sfb = 16  # (an MBS operand makes every pair block-16)
    qa = (_lib.QT * len(aqs))(*[aq.gemm_qt(sfb) for aq in aqs])
    qb = (_lib.QT * len(bqs))(*[bq.gemm_qt(sfb) for bq in bqs])
    cp = (ctypes.c_void_p * len(outs))(*[o.data_ptr() for o in outs])
    status = torch.zeros(4, dtype=torch.int32, device=dev)
    dt = _lib.MXQ_BF16 if out_dtype == torch.bfloat16 else _lib.MXQ_F32
    _lib.check(_lib.lib().mxq_gemm_grouped(qa, qb, len(aqs), ctypes.cast(cp, ctypes.c_void_p), dt, n,
                                           status.data_ptr(), _lib.stream_handle()), "matmul_quantized_grouped")
    return outs


def quantize_matmul(a, bq: QuantizedTensor, cfg: SchemeConfig = SchemeConfig(Variant.MBS_S),
                    tile: TileConfig = TileConfig(), *, out_dtype: torch.dtype = torch.float32,
                    out: torch.Tensor = None, check: bool = True, fused: bool = False):
    """``(matmul_quantized(aq, bq), aq)`` with ``aq = quantize_tensor(a, cfg)``
    (src/quantize.py:709-725, src/gemm.py:137-172) -- the activation side of
    a quantized linear layer.

    By default the two calls run back to back (quantizer launch + GEMM
    launch).  ``fused=True`` (an MBS-S bf16 activation of more than 64 rows
    against an MBS / E8M0 weight) runs the quantization inside the GEMM
    launch instead (csrc/gemm_mbs.cu ``fused_quant_a``: the running CTAs
    claim 8-row slices of A, quantize them with the standalone kernel's
    arithmetic and publish them before the first tile loads) -- one launch,
    no co-residency assumption, but measured slower than the two launches
    (DESIGN.md section 7).  The result and ``aq`` are bit-identical either way.
    """
    from . import quantize as _q

    cfg = cfg if isinstance(cfg, SchemeConfig) else SchemeConfig(cfg)
    fusable = (fused and cfg.variant is Variant.MBS_S and bq.variant in (Variant.MBS_S, Variant.MBS_D, Variant.MX16,
                                                                Variant.MX16_OAS, Variant.OCP32)
               and isinstance(a, torch.Tensor) and a.dtype == torch.bfloat16 and a.is_cuda
               # the pair must be one the tcgen05 MBS kernel takes (else: two calls,
               # and matmul_quantized picks the path, as for any other pair)
               and cfg.macro_size in (64, 128, 256)
               and (bq.mbs_mantissas is None or bq.macro_size == cfg.macro_size))
    if not fusable:
        aq = quantize_tensor(a, cfg, check=check)
        return matmul_quantized(aq, bq, tile, out_dtype=out_dtype, out=out, check=check), aq
    x, dt = _q._as_device_2d(a, 16)
    rows, cols = x.shape
    if cols != bq.shape[1]:
        raise ValueError(f"operands disagree on K: {(rows, cols)} vs {bq.shape}")
    macro = cfg.macro_size
    if tile.t_k % 16 != 0:  # _validate_chunking for the operand not yet quantized
        raise ValueError(f"t_k {tile.t_k} is not a multiple of operand a's block size 16")
    if tile.t_k % macro != 0:
        raise ValueError(f"t_k {tile.t_k} is not a multiple of operand a's macro size {macro}")
    _validate_chunking(bq, tile.t_k, "b")
    if out_dtype not in (torch.float32, torch.bfloat16):
        raise ValueError("out_dtype must be float32 or bfloat16")
    bufs = _q._Outputs(Variant.MBS_S, rows, cols, 16, macro, x.device, True)
    qa = bufs.qt(Variant.MBS_S, rows, cols, 16, macro)
    n = bq.shape[0]
    if out is not None:
        _check_out(out, rows, n, out_dtype, x.device)
    c = out if out is not None else torch.empty((rows, n), dtype=out_dtype, device=x.device)
    qb = bq.gemm_qt(16)  # (an MBS-S A makes the pair block-16)
    dtc = _lib.MXQ_BF16 if out_dtype == torch.bfloat16 else _lib.MXQ_F32
    _lib.check(_lib.lib().mxq_quantize_gemm(x.data_ptr(), dt, x.stride(0), ctypes.byref(qa), ctypes.byref(qb),
                                            c.data_ptr(), dtc, c.stride(0), bufs.status.data_ptr(),
                                            _lib.stream_handle()), "quantize_matmul")
    aq = _q._result(bufs, Variant.MBS_S, rows, cols, 16, macro, check)
    return c, aq


def roofline_overhead(cfg: TileConfig, sigma_bytes: int = 2, out_bytes: int = 4) -> OverheadReport:
    """Per-chunk scale-application cost vs the 4-bit tensor work
    (src/gemm.py:175-193, Appendix B)."""
    if sigma_bytes <= 0 or out_bytes <= 0:
        raise ValueError("byte widths must be positive")
    return OverheadReport(compute_ratio=2.0 / cfg.t_k,
                          traffic_ratio=((cfg.t_m + cfg.t_n) * sigma_bytes) / (cfg.t_m * cfg.t_n * out_bytes))


def max_ulp_divergence(a, b) -> int:
    """Largest ulp distance between two float32 arrays (src/gemm.py:196-214)."""
    to_np = lambda t: t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else t
    x = np.ascontiguousarray(to_np(a), dtype=np.float32)
    y = np.ascontiguousarray(to_np(b), dtype=np.float32)
    if x.shape != y.shape:
        raise ValueError(f"shape mismatch: {x.shape} vs {y.shape}")
    if x.size == 0:
        return 0

    def key(v: np.ndarray) -> np.ndarray:
        bits = v.view(np.uint32).astype(np.int64)
        return np.where(bits & 0x80000000, 0x80000000 - bits, bits)

    return int(np.max(np.abs(key(x) - key(y))))
