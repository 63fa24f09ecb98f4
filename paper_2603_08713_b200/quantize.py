"""Block and macro-block 4-bit quantization on the B200.

Drop-in for the reference's ``mxq.quantize`` (src/quantize.py): the same
names, dataclasses, defaults and ``ValueError`` messages.  Tensor-level work
runs in the sm_100a kernels of ``csrc/quantize.cu`` through the C ABI
(``include/mxq200.h``); results live in CUDA memory as ``torch`` tensors.

Variants (src/quantize.py:1-28): OCP32 (block-32 E8M0, D = 2^(floor(log2
alpha)-2)), MX16 (block-16, SF = 2^floor(log2(6/alpha))), MX16_OAS (MX16 +
overflow-aware doubling when alpha*SF <= 3.5), MBS_S / MBS_D (per-macro
8-bit mantissa factor then OAS blocks; static or SSE-optimal), NVFP4 (global
s_t plus per-block E4M3).  Outputs are bit-identical to the reference.
"""

from __future__ import annotations

import ctypes
import dataclasses
from dataclasses import dataclass, field
from enum import Enum
from typing import Any, Optional

import numpy as np
import torch

from . import _lib
from .formats import (
    E4M3_TABLE, E8M0_BIAS, E8M0Scale, Mantissa8, decode_e2m1_array, encode_e2m1_array,
)

__all__ = [
    "Variant", "CandidateSet", "ErrorLut", "SchemeConfig", "QuantizedTensor", "default_candidates",
    "block_scale_ocp", "block_scale_16", "quantize_block", "mbs_static_mantissa", "mbs_dynamic_exact",
    "build_error_lut", "mbs_dynamic_lut", "quantize_tensor", "quantize_nvfp4", "dequantize_tensor",
    "macro_segments",
]


class Variant(str, Enum):
    OCP32 = "ocp32"
    MX16 = "mx16"
    MX16_OAS = "mx16_oas"
    MBS_S = "mbs_s"
    MBS_D = "mbs_d"
    NVFP4 = "nvfp4"


MBS_VARIANTS = (Variant.MBS_S, Variant.MBS_D)
MACRO_SIZES = (32, 64, 128, 256, 512)


@dataclass(frozen=True)
class CandidateSet:
    """Ordered MBS-D candidate mantissa bytes (src/quantize.py:85-100)."""

    mantissas: tuple

    def __post_init__(self) -> None:
        if len(self.mantissas) == 0:
            raise ValueError("candidate set is empty")
        if len(set(self.mantissas)) != len(self.mantissas):
            raise ValueError("candidate set contains duplicates")
        if 0 not in self.mantissas:
            raise ValueError("candidate set must contain the identity factor m8=0")
        for m in self.mantissas:
            if not 0 <= m <= 255:
                raise ValueError(f"mantissa byte out of range: {m}")


def default_candidates() -> CandidateSet:
    """{0, 16, ..., 240} (src/quantize.py:103-105)."""
    return CandidateSet(tuple(range(0, 256, 16)))


LUT_BINS = 64
LUT_SUBNORMAL_EDGES = np.arange(LUT_BINS) / LUT_BINS
LUT_NORMAL_EDGES = 1.0 + np.arange(LUT_BINS) * 7.0 / LUT_BINS


@dataclass(frozen=True)
class ErrorLut:
    """[regime 2][candidate 16][bin 64] fp16 squared relative errors
    (src/quantize.py:114-125)."""

    entries: np.ndarray
    candidates: tuple
    subnormal_edges: np.ndarray = field(default_factory=lambda: LUT_SUBNORMAL_EDGES)
    normal_edges: np.ndarray = field(default_factory=lambda: LUT_NORMAL_EDGES)

    def __post_init__(self) -> None:
        if self.entries.shape != (2, 16, LUT_BINS) or self.entries.dtype != np.float16:
            raise ValueError("ErrorLut entries must be float16 of shape (2, 16, 64)")


@dataclass(frozen=True)
class SchemeConfig:
    """Scheme selection and knobs (src/quantize.py:128-170)."""

    variant: Variant
    block_size: Optional[int] = None
    macro_size: int = 128
    mbs_mode: str = "exact"
    candidates: Optional[CandidateSet] = None
    augment_static: bool = True

    def __post_init__(self) -> None:
        object.__setattr__(self, "variant", Variant(self.variant))
        expected = 32 if self.variant is Variant.OCP32 else 16
        if self.block_size is None:
            object.__setattr__(self, "block_size", expected)
        elif self.block_size != expected:
            raise ValueError(f"{self.variant.value} requires block_size {expected}, got {self.block_size}")
        if self.macro_size <= 0 or self.macro_size % self.block_size != 0:
            raise ValueError(
                f"macro_size {self.macro_size} is not a positive multiple of block_size {self.block_size}")
        if self.mbs_mode not in ("exact", "lut"):
            raise ValueError(f"unknown mbs_mode: {self.mbs_mode}")
        if self.candidates is None:
            object.__setattr__(self, "candidates", default_candidates())


def macro_segments(cols: int, macro_size: int) -> list:
    """Full macros plus one trailing partial (src/quantize.py:250-254)."""
    edges = list(range(0, cols, macro_size)) + [cols]
    return [(edges[i], edges[i + 1]) for i in range(len(edges) - 1)]


def _round_up(x: int, m: int) -> int:
    return (x + m - 1) // m * m


def _to_device_u8(a, dev) -> Optional[torch.Tensor]:
    if a is None:
        return None
    if isinstance(a, torch.Tensor):
        return a.to(device=dev, dtype=torch.uint8)
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint8)).to(dev)


@dataclass(frozen=True, eq=False)
class QuantizedTensor:
    """A quantized 2-D tensor in CUDA memory (src/quantize.py:173-247).

    Field meaning and layouts are the reference's: ``codes`` (rows, cols/2)
    two E2M1 codes per byte (even column low nibble); ``block_scales``
    (rows, cols/bs) E8M0 biased exponents of the dequant multiplier D;
    ``e4m3_scales`` (rows, cols/16) for NVFP4; ``mbs_mantissas``
    (rows, n_macros); ``tensor_scale`` the NVFP4 s_t.  Array fields are
    ``torch.uint8`` CUDA tensors (numpy inputs are uploaded).  The tcgen05
    GEMM operand layouts are cached privately (built by the quantizer, or on
    first use for user-constructed tensors).
    """

    variant: Variant
    shape: tuple
    block_size: int
    macro_size: int
    codes: Any
    block_scales: Any
    e4m3_scales: Any
    mbs_mantissas: Any
    tensor_scale: Any
    _cache: dict = field(default=None, init=False, repr=False, compare=False)

    def __post_init__(self) -> None:
        dev = _lib.require_device()
        object.__setattr__(self, "variant", Variant(self.variant))
        object.__setattr__(self, "shape", tuple(int(s) for s in self.shape))
        for f in ("codes", "block_scales", "e4m3_scales", "mbs_mantissas"):
            a = getattr(self, f)
            if not (a is None or (isinstance(a, torch.Tensor) and a.dtype == torch.uint8 and a.device == dev)):
                object.__setattr__(self, f, _to_device_u8(a, dev))
        object.__setattr__(self, "_cache", {})

    # ---- reference accessors ------------------------------------------------
    @property
    def n_macros(self) -> int:
        return -(-self.shape[1] // self.macro_size)

    def __eq__(self, other: object) -> bool:
        if not isinstance(other, QuantizedTensor):
            return NotImplemented

        def same(a, b) -> bool:
            if a is None or b is None:
                return a is None and b is None
            return a.shape == b.shape and bool(torch.equal(a, b.to(a.device)))

        ts = lambda q: None if q.tensor_scale is None else float(q.tensor_scale)
        return (self.variant == other.variant and self.shape == other.shape
                and self.block_size == other.block_size and self.macro_size == other.macro_size
                and same(self.codes, other.codes) and same(self.block_scales, other.block_scales)
                and same(self.e4m3_scales, other.e4m3_scales)
                and same(self.mbs_mantissas, other.mbs_mantissas) and ts(self) == ts(other))

    def unpack_codes(self) -> torch.Tensor:
        """One uint8 code per element, (rows, cols)."""
        rows, cols = self.shape
        out = torch.empty((rows, cols), dtype=torch.uint8, device=self.codes.device)
        out[:, 0::2] = self.codes & 15
        out[:, 1::2] = self.codes >> 4
        return out

    def block_dequant_values(self) -> torch.Tensor:
        """Per-block D as float64, (rows, n_blocks) (src/quantize.py:220-240)."""
        if self.variant is Variant.NVFP4:
            tab = torch.from_numpy(E4M3_TABLE).to(self.codes.device)
            vals = tab[self.e4m3_scales.long()]
            if bool(torch.isnan(vals).any()):
                raise ValueError("corrupt block scale: E4M3 NaN code")
            return vals
        if bool((self.block_scales == 255).any()):
            raise ValueError("corrupt block scale: E8M0 code 255 is reserved")
        # 2^(b-127) built from its f64 bit pattern (exact for b in 0..254)
        bits = (self.block_scales.to(torch.int64) + (1023 - E8M0_BIAS)) << 52
        return bits.view(torch.float64)

    def macro_factors(self) -> Optional[torch.Tensor]:
        if self.mbs_mantissas is None:
            return None
        return 1.0 + self.mbs_mantissas.to(torch.float64) / 256.0

    def to_host(self) -> dict:
        """Numpy copy of the reference fields (for parity checks / storage)."""
        c = lambda t: None if t is None else t.cpu().numpy()
        return {"variant": self.variant.value, "shape": self.shape, "block_size": self.block_size,
                "macro_size": self.macro_size, "codes": c(self.codes), "block_scales": c(self.block_scales),
                "e4m3_scales": c(self.e4m3_scales), "mbs_mantissas": c(self.mbs_mantissas),
                "tensor_scale": None if self.tensor_scale is None else float(self.tensor_scale)}

    # ---- C-ABI views --------------------------------------------------------
    def _scales_tensor(self) -> torch.Tensor:
        return self.e4m3_scales if self.variant is Variant.NVFP4 else self.block_scales

    def _ts_device(self) -> Optional[torch.Tensor]:
        if self.variant is not Variant.NVFP4:
            return None
        ts = self.tensor_scale
        if isinstance(ts, torch.Tensor):
            return ts.to(device=self.codes.device, dtype=torch.float64).reshape(1)
        t = self._cache.get("ts")
        if t is None:
            t = torch.tensor([float(ts)], dtype=torch.float64, device=self.codes.device)
            self._cache["ts"] = t
        return t

    def qt(self) -> _lib.QT:
        """Reference-layout descriptor (row-major scales, mantissas)."""
        rows, cols = self.shape
        s = self._scales_tensor()
        if self.codes.stride(1) != 1 or s.stride(1) != 1:
            raise ValueError("codes / scales must have unit column stride")
        q = _lib.QT()
        q.variant = _lib.VARIANT_CODE[self.variant.value]
        q.block_size, q.macro_size = self.block_size, self.macro_size
        q.rows, q.cols = rows, cols
        q.codes, q.codes_ld = self.codes.data_ptr(), self.codes.stride(0)
        q.scales, q.scales_ld = s.data_ptr(), s.stride(0)
        if self.mbs_mantissas is not None:
            m = self.mbs_mantissas
            q.mant, q.mant_ld = m.data_ptr(), m.stride(0)
        ts = self._ts_device()
        q.tensor_scale = None if ts is None else ts.data_ptr()
        return q

    def gemm_qt(self, sf_block: Optional[int] = None) -> _lib.QT:
        """Descriptor with the tcgen05 operand layouts: 16-byte code pitch,
        scale-factor atoms for `sf_block` (16, or 32 for OCP32 pairs) and the
        transposed mantissas.  Built once and cached."""
        sf_block = sf_block or self.block_size
        key = ("gemm", sf_block)
        hit = self._cache.get(key)
        if hit is not None:
            return hit[0]
        rows, cols = self.shape
        dev = self.codes.device
        stream = _lib.stream_handle()
        keep = []
        codes = self.codes
        if codes.stride(0) % 16 or codes.data_ptr() % 16:
            pitch = _round_up(cols // 2, 16)
            buf = torch.zeros((rows, pitch), dtype=torch.uint8, device=dev)
            buf[:, : cols // 2] = codes
            codes = buf[:, : cols // 2]
        keep.append(codes)
        q = self.qt()
        q.codes, q.codes_ld = codes.data_ptr(), codes.stride(0)
        pre = self._cache.get(("mma", sf_block))
        rows_pad = _round_up(rows, 256)
        kpad = _round_up(cols, 256) // sf_block
        if pre is not None:
            sf = pre
        else:
            sf = torch.empty(rows_pad * kpad, dtype=torch.uint8, device=dev)
        q.scales_mma, q.sf_kpad = sf.data_ptr(), kpad
        keep.append(sf)
        mt = None
        if self.mbs_mantissas is not None:
            mt = self._cache.get("sig_t")
            if mt is None:
                mt = torch.empty((self.n_macros, rows_pad), dtype=torch.float32, device=dev)
            q.sig_t, q.sig_t_ld = mt.data_ptr(), mt.stride(0)
            keep.append(mt)
        need_sf = pre is None
        need_mt = self.mbs_mantissas is not None and self._cache.get("sig_t") is None
        if need_sf or need_mt:
            qb = _lib.QT.from_buffer_copy(q)
            if not need_sf:
                qb.scales_mma = None
            if not need_mt:
                qb.sig_t = None
            _lib.check(_lib.lib().mxq_build_gemm_layout(ctypes.byref(qb), sf_block, stream), "build_gemm_layout")
            self._cache[("mma", sf_block)] = sf
            if mt is not None:
                self._cache["sig_t"] = mt
        ts = self._ts_device()
        if ts is not None:
            keep.append(ts)
        self._cache[key] = (q, keep)
        return q


# ---------------------------------------------------------------------------
# Scalar / per-block helpers (host, same arithmetic header as the kernels)
# ---------------------------------------------------------------------------

def _validate_block(block, size: int) -> np.ndarray:
    arr = np.asarray(block, dtype=np.float64)
    if arr.shape != (size,):
        raise ValueError(f"expected a block of {size} elements, got shape {arr.shape}")
    if not np.all(np.isfinite(arr)):
        raise ValueError("block contains non-finite elements")
    return np.ascontiguousarray(arr)


def _block_scale(block, size: int, kind: int) -> E8M0Scale:
    arr = _validate_block(block, size)
    b, c = ctypes.c_uint8(), ctypes.c_int32()
    _lib.check(_lib.lib().mxq_host_block_scale(arr.ctypes.data, size, kind, ctypes.byref(b), ctypes.byref(c)),
               "block_scale")
    return E8M0Scale(b.value, clamped=bool(c.value))


def block_scale_ocp(block) -> E8M0Scale:
    """D = 2^(floor(log2 alpha) - 2) for a 32-block (src/quantize.py:301-311)."""
    return _block_scale(block, 32, 0)


def block_scale_16(block, oas: bool = False) -> E8M0Scale:
    """D = 1/SF for a 16-block, optional OAS (src/quantize.py:314-334)."""
    return _block_scale(block, 16, 2 if oas else 1)


def quantize_block(block, sf: float, factor: Optional[Mantissa8] = None) -> np.ndarray:
    """Codes of encode(x * factor * sf), saturating (src/quantize.py:337-361)."""
    if not sf > 0:
        raise ValueError(f"sf must be positive, got {sf}")
    arr = np.asarray(block, dtype=np.float32)
    if not np.all(np.isfinite(arr)):
        raise ValueError("block contains non-finite elements")
    if factor is not None:
        arr = (arr * np.float32(factor.factor)).astype(np.float32)
    return encode_e2m1_array(arr.astype(np.float64) * float(sf), saturate=True)


def mbs_static_mantissa(alpha_max_128: float) -> Mantissa8:
    """Top 8 fraction bits of f32(6)/f32(alpha) (src/quantize.py:369-380)."""
    if alpha_max_128 == 0:
        return Mantissa8(0)
    if not (np.isfinite(alpha_max_128) and alpha_max_128 > 0):
        raise ValueError(f"macro maximum must be positive finite, got {alpha_max_128}")
    m = ctypes.c_uint8()
    _lib.check(_lib.lib().mxq_host_static_m8(float(alpha_max_128), ctypes.byref(m)), "static_m8")
    return Mantissa8(m.value)


def _choose(macro, candidates: CandidateSet, augment: bool, lut: Optional[np.ndarray]) -> Mantissa8:
    arr = np.ascontiguousarray(macro, dtype=np.float32)
    if arr.ndim != 1:
        raise ValueError("macro must be one-dimensional")
    if arr.size == 0 or arr.size % 16 != 0:
        raise ValueError(f"macro length must be a positive multiple of 16, got {arr.size}")
    if not np.all(np.isfinite(arr)):
        raise ValueError("macro contains non-finite elements")
    cand = np.asarray(candidates.mantissas, dtype=np.uint8)
    m = ctypes.c_uint8()
    lut_p = None if lut is None else lut.ctypes.data
    _lib.check(_lib.lib().mxq_host_mbs_choose(arr.ctypes.data, arr.size, cand.ctypes.data, len(cand),
                                              int(augment), lut_p, ctypes.byref(m)), "mbs_choose")
    return Mantissa8(m.value)


def mbs_dynamic_exact(macro, candidates: CandidateSet) -> Mantissa8:
    """SSE-optimal mantissa for one macro, ties to the smaller byte
    (src/quantize.py:464-479)."""
    return _choose(macro, candidates, False, None)


def build_error_lut(candidates: CandidateSet) -> ErrorLut:
    """Squared relative error of the saturating E2M1 grid at bin centres
    (src/quantize.py:482-504)."""
    if len(candidates.mantissas) != 16:
        raise ValueError(
            f"the lookup table holds exactly 16 candidates, got {len(candidates.mantissas)}")
    sub_c = LUT_SUBNORMAL_EDGES + 0.5 / LUT_BINS
    nor_c = LUT_NORMAL_EDGES + 0.5 * 7.0 / LUT_BINS
    ent = np.empty((2, 16, LUT_BINS))
    for j, m in enumerate(candidates.mantissas):
        f = 1.0 + m / 256.0
        for r, c in enumerate((sub_c, nor_c)):
            u = c * f
            q = decode_e2m1_array(encode_e2m1_array(u, saturate=True))
            ent[r, j] = ((q - u) / u) ** 2
    return ErrorLut(ent.astype(np.float16), tuple(candidates.mantissas))


def mbs_dynamic_lut(macro, lut: ErrorLut, candidates: CandidateSet) -> Mantissa8:
    """LUT-estimated mantissa for one macro (src/quantize.py:545-560)."""
    if tuple(candidates.mantissas) != lut.candidates:
        raise ValueError("lookup table was built from a different candidate set")
    return _choose(macro, candidates, False, np.ascontiguousarray(lut.entries, dtype=np.float32))


# ---------------------------------------------------------------------------
# Tensor level (GPU)
# ---------------------------------------------------------------------------

def _as_device_2d(t, bs: int):
    """(tensor, dtype code) ready for the kernels, with the reference's
    validation messages (src/quantize.py:573-583).  Finiteness is checked on
    the device."""
    dev = _lib.require_device()
    if isinstance(t, torch.Tensor):
        x = t
        if x.dtype not in (torch.float32, torch.bfloat16):
            x = x.to(torch.float32)
    else:
        arr = np.asarray(t, dtype=np.float32)
        x = torch.from_numpy(np.ascontiguousarray(arr))
    if x.ndim != 2 or x.shape[0] == 0 or x.shape[1] == 0:
        raise ValueError(f"expected a non-empty 2-D tensor, got shape {tuple(x.shape)}")
    if x.shape[1] % bs != 0:
        raise ValueError(f"row length {x.shape[1]} is not divisible by block_size {bs}")
    if x.device != dev:
        x = x.to(dev, non_blocking=True)
    esz = x.element_size()
    # the streaming kernels read 32-byte units: 32-byte aligned base and row pitch
    if x.stride(1) != 1 or (x.stride(0) * esz) % 32 or x.data_ptr() % 32:
        x = x.contiguous()
        if (x.stride(0) * esz) % 32 or x.data_ptr() % 32:
            pitch = _round_up(x.shape[1], 32 // esz)
            buf = torch.empty((x.shape[0], pitch), dtype=x.dtype, device=dev)
            buf[:, : x.shape[1]] = x
            x = buf[:, : x.shape[1]]
    code = _lib.MXQ_BF16 if x.dtype == torch.bfloat16 else _lib.MXQ_F32
    return x, code


class _Outputs:
    """Device buffers one quantize call writes, carved out of ONE allocation
    (16-byte aligned views): codes, row-major scales, tcgen05 scale atoms,
    mantissas, transposed sigma, the NVFP4 tensor scale and the 4-word status
    (zeroed by the C call itself)."""

    def __init__(self, variant: Variant, rows: int, cols: int, bs: int, macro: int, dev, gemm_layout: bool):
        mbs = variant in MBS_VARIANTS
        nmac = -(-cols // macro)
        self.rows_pad = _round_up(rows, 256)
        self.kpad = _round_up(cols, 256) // bs
        pitch = _round_up(cols // 2, 16)
        sizes = [("codes", rows * pitch), ("scales", rows * (cols // bs)),
                 ("sf", self.rows_pad * self.kpad if gemm_layout else 0),
                 ("mant", rows * nmac if mbs else 0),
                 ("sig", 4 * nmac * self.rows_pad if (mbs and gemm_layout) else 0),
                 ("ts", 8 if variant is Variant.NVFP4 else 0), ("status", 16)]
        offs, total = {}, 0
        for name, n in sizes:
            offs[name] = total
            total += _round_up(n, 16)
        buf = torch.empty(total, dtype=torch.uint8, device=dev)
        part = lambda name, n: buf[offs[name]:offs[name] + n]
        self.keep = buf
        self.codes_buf = part("codes", rows * pitch).view(rows, pitch)
        self.codes = self.codes_buf[:, : cols // 2]
        self.scales = part("scales", rows * (cols // bs)).view(rows, cols // bs)
        self.sf_mma = part("sf", self.rows_pad * self.kpad) if gemm_layout else None
        self.mant = part("mant", rows * nmac).view(rows, nmac) if mbs else None
        self.sig_t = (part("sig", 4 * nmac * self.rows_pad).view(torch.float32).view(nmac, self.rows_pad)
                      if (mbs and gemm_layout) else None)
        self.ts = part("ts", 8).view(torch.float64) if variant is Variant.NVFP4 else None
        self.status = part("status", 16).view(torch.int32)

    def qt(self, variant: Variant, rows: int, cols: int, bs: int, macro: int) -> _lib.QT:
        q = _lib.QT()
        q.variant = _lib.VARIANT_CODE[variant.value]
        q.block_size, q.macro_size, q.rows, q.cols = bs, macro, rows, cols
        q.codes, q.codes_ld = self.codes.data_ptr(), self.codes.stride(0)
        q.scales, q.scales_ld = self.scales.data_ptr(), self.scales.stride(0)
        if self.sf_mma is not None:
            q.scales_mma, q.sf_kpad = self.sf_mma.data_ptr(), self.kpad
        if self.mant is not None:
            q.mant, q.mant_ld = self.mant.data_ptr(), self.mant.stride(0)
        if self.sig_t is not None:
            q.sig_t, q.sig_t_ld = self.sig_t.data_ptr(), self.sig_t.stride(0)
        if self.ts is not None:
            q.tensor_scale = self.ts.data_ptr()
        return q


_CAND_CACHE: dict = {}


def _cand_array(candidates) -> np.ndarray:
    """Candidate bytes as a uint8 host array, built once per candidate set."""
    key = tuple(candidates.mantissas)
    arr = _CAND_CACHE.get(key)
    if arr is None:
        arr = _CAND_CACHE[key] = np.asarray(key, dtype=np.uint8)
    return arr


def quantize_tensor(t, cfg: SchemeConfig, *, check: bool = True, gemm_layout: bool = True) -> QuantizedTensor:
    """Quantize a 2-D tensor under ``cfg`` on the GPU (src/quantize.py:709-725).

    ``t`` may be a numpy array (uploaded) or a float32 / bfloat16 torch tensor
    (CUDA tensors are used in place).  With ``check`` (the default, the
    reference's semantics) the call synchronises once to raise ValueError on
    non-finite input; ``check=False`` keeps the call fully asynchronous (the
    status word is kept on the result: ``_raise_status(q)`` checks it later).
    ``gemm_layout`` also writes the tcgen05 scale-factor atoms and transposed
    mantissas in the same pass.
    """
    cfg = cfg if isinstance(cfg, SchemeConfig) else SchemeConfig(cfg)
    bs = 32 if cfg.variant is Variant.OCP32 else 16
    x, dt = _as_device_2d(t, bs)
    rows, cols = x.shape
    macro = cfg.macro_size
    if cfg.variant is Variant.NVFP4:
        macro = 128  # the reference records 128 for NVFP4 (src/quantize.py:677, :700)
    out = _Outputs(cfg.variant, rows, cols, bs, macro, x.device, gemm_layout)
    q = out.qt(cfg.variant, rows, cols, bs, macro)
    stream = _lib.stream_handle()
    L = _lib.lib()
    cand = _cand_array(cfg.candidates)
    if cfg.variant is Variant.MBS_D and cfg.mbs_mode == "lut":
        lut = np.ascontiguousarray(build_error_lut(cfg.candidates).entries, dtype=np.float32)
        rc = L.mxq_quantize_mbs_lut(x.data_ptr(), dt, x.stride(0), ctypes.byref(q), cand.ctypes.data, len(cand),
                                    lut.ctypes.data, out.status.data_ptr(), stream)
    else:
        rc = L.mxq_quantize(x.data_ptr(), dt, x.stride(0), ctypes.byref(q), 0, cand.ctypes.data, len(cand),
                            int(cfg.augment_static), out.status.data_ptr(), stream)
    _lib.check(rc, "quantize_tensor")
    return _result(out, cfg.variant, rows, cols, bs, macro, check)


def _result(out: "_Outputs", variant: Variant, rows: int, cols: int, bs: int, macro: int,
            check: bool) -> QuantizedTensor:
    """QuantizedTensor over the buffers a quantize call wrote (the status word
    is checked now with ``check``, else kept for ``_raise_status``)."""
    nv = variant is Variant.NVFP4
    ts: Any = None
    if check:
        _lib.raise_on_status(out.status)
        if nv:
            ts = float(out.ts.item())
    elif nv:
        ts = out.ts
    res = QuantizedTensor(
        variant=variant, shape=(rows, cols), block_size=bs, macro_size=macro, codes=out.codes,
        block_scales=None if nv else out.scales, e4m3_scales=out.scales if nv else None,
        mbs_mantissas=out.mant, tensor_scale=ts)
    c = res._cache
    c["keep"] = out.keep
    c["status"] = out.status
    if out.sf_mma is not None:
        c[("mma", bs)] = out.sf_mma
    if out.sig_t is not None:
        c["sig_t"] = out.sig_t
    if nv:
        c["ts"] = out.ts
    return res


def _raise_status(q: QuantizedTensor) -> None:
    st = q._cache.get("status")
    if st is not None:
        _lib.raise_on_status(st)


def quantize_nvfp4(t) -> QuantizedTensor:
    """NVFP4: s_t = amax/(448*6), E4M3 block scales (src/quantize.py:662-706)."""
    return quantize_tensor(t, SchemeConfig(Variant.NVFP4))


def dequantize_tensor(q: QuantizedTensor) -> torch.Tensor:
    """f32(decode * D / f * s_t) on the GPU (src/quantize.py:728-746);
    returns a (rows, cols) float32 CUDA tensor."""
    rows, cols = q.shape
    out = torch.empty((rows, cols), dtype=torch.float32, device=q.codes.device)
    status = torch.zeros(4, dtype=torch.int32, device=q.codes.device)
    qt = q.qt()
    _lib.check(_lib.lib().mxq_dequantize(ctypes.byref(qt), out.data_ptr(), out.stride(0), status.data_ptr(),
                                         _lib.stream_handle()), "dequantize_tensor")
    _lib.raise_on_status(status)
    return out
