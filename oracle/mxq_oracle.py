"""CPU oracle for the MXFP4 quantize-and-GEMM path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference package's hot path
(``/root/reference/pkg/src/mxq``).  It exists to *check* the CUDA product,
never to *be* it: only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import it.
The product package (``paper_2603_08713_b200``) never imports this file and
fails loudly when its CUDA extension is missing.

Parity is pinned: ``tests/golden/make_golden.py`` runs the real reference
(imported from ``/root/reference/pkg/src`` in the build container) on seeded
inputs and commits its outputs as ``tests/golden/*.npz``;
``tests/test_oracle_golden.py`` checks every function here against them.

Each function cites the reference file:line it restates.  The mechanics are
deliberately different from the reference where that is natural (counting
midpoint crossings instead of ``searchsorted``, an explicit ``e_floor``
helper, a one-pass NVFP4 formulation) while the *arithmetic contract* is the
same: float32 factor multiply, exact power-of-two scaling in float64, one
final rounding to float32, float64 SSE in numpy pairwise order.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

# --------------------------------------------------------------------------
# Codec constants (src/formats.py:46-56, :235-257)
# --------------------------------------------------------------------------

GRID = np.array([0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0])
MIDS = np.array([0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0])
BIAS = 127
VARIANTS = ("ocp32", "mx16", "mx16_oas", "mbs_s", "mbs_d", "nvfp4")


def e4m3_table() -> np.ndarray:
    """All 256 E4M3 codes decoded (src/formats.py:235-252); NaN codes -> nan."""
    out = np.empty(256)
    for c in range(256):
        e, m = (c >> 3) & 15, c & 7
        if e == 0:
            v = m * 2.0 ** -9
        elif e == 15 and m == 7:
            v = math.nan
        else:
            v = (8 + m) * 2.0 ** (e - 10)
        out[c] = -v if c & 0x80 else v
    return out


E4M3 = e4m3_table()


# --------------------------------------------------------------------------
# E2M1 (src/formats.py:141-207)
# --------------------------------------------------------------------------

def e2m1_index(mag: np.ndarray) -> np.ndarray:
    """Nearest grid index for magnitudes in [0, 6]; ties go to the even index.

    Restates ``_nearest_magnitude_index`` (src/formats.py:141-151): the index
    is the number of midpoints strictly below ``mag``; a value sitting exactly
    on a midpoint is between index k and k+1 and takes whichever is even.
    """
    mag = np.asarray(mag, dtype=np.float64)
    idx = np.zeros(mag.shape, dtype=np.int64)
    tie = np.zeros(mag.shape, dtype=bool)
    for k, m in enumerate(MIDS):
        idx += mag > m
        tie |= mag == m
    return np.where(tie & (idx % 2 == 1), idx + 1, idx)


def e2m1_encode(values: np.ndarray) -> np.ndarray:
    """Saturating E2M1 encode (src/formats.py:185-200, saturate=True).

    bit 3 = sign (only when the magnitude index is non-zero: -0 and negative
    flushes normalise to code 0, src/formats.py:176/:199), bits 0..2 = index.
    """
    v = np.asarray(values, dtype=np.float64)
    if not np.all(np.isfinite(v)):
        raise ValueError("cannot encode non-finite values")
    idx = e2m1_index(np.minimum(np.abs(v), 6.0))
    neg = (v < 0) & (idx > 0)
    return (idx | (neg.astype(np.int64) << 3)).astype(np.uint8)


def e2m1_decode(codes: np.ndarray) -> np.ndarray:
    """uint8 codes -> float64 grid values (src/formats.py:203-207)."""
    c = np.asarray(codes).astype(np.int64)
    mag = GRID[c & 7]
    return np.where(c & 8, -mag, mag)


# --------------------------------------------------------------------------
# E4M3 (src/formats.py:260-292)
# --------------------------------------------------------------------------

_POS = E4M3[:127]
_POS_MID = (_POS[:-1] + _POS[1:]) * 0.5


def e4m3_encode(values: np.ndarray) -> np.ndarray:
    """Nearest finite E4M3 byte, ties to the even code, clamp at 448."""
    v = np.asarray(values, dtype=np.float64)
    if not np.all(np.isfinite(v)):
        raise ValueError("cannot encode non-finite values")
    mag = np.minimum(np.abs(v), 448.0)
    idx = np.zeros(mag.shape, dtype=np.int64)
    tie = np.zeros(mag.shape, dtype=bool)
    # 126 midpoints; accumulate crossings in chunks to bound memory.
    for m in _POS_MID:
        idx += mag > m
        tie |= mag == m
    idx = np.where(tie & (idx % 2 == 1), idx + 1, idx)
    sign = np.where((v < 0) & (idx > 0), 0x80, 0)
    return (idx | sign).astype(np.uint8)


# --------------------------------------------------------------------------
# E8M0 block scales (src/quantize.py:262-289)
# --------------------------------------------------------------------------

def e_floor(x: np.ndarray) -> np.ndarray:
    """floor(log2 x) for positive finite float64 (frexp exponent - 1)."""
    return np.frexp(np.asarray(x, dtype=np.float64))[1].astype(np.int64) - 1


def scale_exp_16(alpha: np.ndarray, oas: bool) -> np.ndarray:
    """Biased E8M0 exponent of D for 16-blocks (src/quantize.py:268-281).

    SF = 2^floor(log2(6/alpha)); OAS doubles SF when alpha*SF <= 3.5;
    stored byte = clip(127 - log2 SF, 0, 254); alpha == 0 stores 127.
    """
    alpha = np.asarray(alpha, dtype=np.float64)
    pos = alpha > 0
    a = np.where(pos, alpha, 1.0)
    k = e_floor(6.0 / a)
    if oas:
        k = k + (np.ldexp(a, k) <= 3.5)
    return np.where(pos, np.clip(BIAS - k, 0, 254), BIAS).astype(np.uint8)


def scale_exp_ocp(alpha: np.ndarray) -> np.ndarray:
    """Biased exponent of D = 2^(floor(log2 alpha) - 2) (src/quantize.py:284-289)."""
    alpha = np.asarray(alpha, dtype=np.float64)
    pos = alpha > 0
    k = e_floor(np.where(pos, alpha, 1.0)) - 2
    return np.where(pos, np.clip(k + BIAS, 0, 254), BIAS).astype(np.uint8)


def static_m8(alpha: np.ndarray) -> np.ndarray:
    """MBS-S mantissa byte: top 8 fraction bits of f32(6)/f32(alpha).

    Restates ``_static_mantissas`` (src/quantize.py:383-389); alpha == 0 -> 0.
    """
    alpha = np.asarray(alpha, dtype=np.float64)
    a32 = np.where(alpha > 0, alpha, 6.0).astype(np.float32)
    with np.errstate(over="ignore", divide="ignore"):
        r = np.float32(6.0) / a32
    m8 = (r.view(np.uint32) >> np.uint32(15)) & np.uint32(0xFF)
    return np.where(alpha > 0, m8, 0).astype(np.uint8)


# --------------------------------------------------------------------------
# Quantized tensor container (src/quantize.py:173-247)
# --------------------------------------------------------------------------

@dataclass
class OracleQ:
    variant: str
    shape: tuple
    block_size: int
    macro_size: int
    codes: np.ndarray                 # (rows, cols//2) u8, even col -> low nibble
    block_scales: Optional[np.ndarray]  # (rows, cols//bs) u8 E8M0 biased
    e4m3_scales: Optional[np.ndarray]   # (rows, cols//16) u8 (NVFP4)
    mbs_mantissas: Optional[np.ndarray]  # (rows, n_macros) u8 (MBS)
    tensor_scale: Optional[float]       # NVFP4


def pack(codes: np.ndarray) -> np.ndarray:
    """Even column -> low nibble (src/quantize.py:568-570)."""
    c = codes.astype(np.uint8)
    return (c[:, 0::2] | (c[:, 1::2] << 4)).astype(np.uint8)


def unpack(packed: np.ndarray, cols: int) -> np.ndarray:
    p = np.asarray(packed, dtype=np.uint8)
    out = np.empty((p.shape[0], cols), dtype=np.uint8)
    out[:, 0::2] = p & 15
    out[:, 1::2] = p >> 4
    return out


def segments(cols: int, macro: int) -> list:
    """Macro column ranges incl. a trailing partial one (src/quantize.py:250-254)."""
    return [(s, min(s + macro, cols)) for s in range(0, cols, macro)]


def _check(t: np.ndarray, bs: int) -> np.ndarray:
    """src/quantize.py:573-583."""
    a = np.ascontiguousarray(t, dtype=np.float32)
    if a.ndim != 2 or a.shape[0] == 0 or a.shape[1] == 0:
        raise ValueError(f"expected a non-empty 2-D tensor, got shape {a.shape}")
    if a.shape[1] % bs:
        raise ValueError(f"row length {a.shape[1]} is not divisible by block_size {bs}")
    if not np.all(np.isfinite(a)):
        raise ValueError("tensor contains non-finite elements")
    return a


def _blocks_quantize(y: np.ndarray, oas: bool, ocp: bool = False):
    """Quantize (n, L) f32 rows in blocks of 16 (or 32 for OCP); returns
    (codes (n, L), biased (n, L/bs)).  Scaling by 2^(127-biased) is exact in
    float64 (src/quantize.py:586-609, :392-406)."""
    bs = 32 if ocp else 16
    n, L = y.shape
    b = y.astype(np.float64).reshape(n, L // bs, bs)
    alpha = np.abs(b).max(axis=2)
    biased = scale_exp_ocp(alpha) if ocp else scale_exp_16(alpha, oas)
    scaled = np.ldexp(b, (BIAS - biased.astype(np.int64))[:, :, None])
    return e2m1_encode(scaled.reshape(n, L)), biased


def _deq(codes, d_el, fac_el=None, ts=None) -> np.ndarray:
    """Pinned element formula f32(g*D/f*s_t) in float64 (src/quantize.py:409-423)."""
    v = e2m1_decode(codes) * d_el
    if fac_el is not None:
        v = v / fac_el
    if ts is not None:
        v = v * ts
    return v.astype(np.float32)


def _factor32(m8: np.ndarray) -> np.ndarray:
    return (1.0 + m8.astype(np.float64) / 256.0).astype(np.float32)


def macro_sse(x: np.ndarray, m8: np.ndarray) -> np.ndarray:
    """Round-trip SSE per macro row (src/quantize.py:426-435).

    The f64 diff^2 row sums go through np.sum(axis=1) so the summation order
    is numpy's pairwise order -- the same order the CUDA kernel emulates.
    """
    f = _factor32(m8)
    y = (x * f[:, None]).astype(np.float32)
    codes, biased = _blocks_quantize(y, oas=True)
    n, L = x.shape
    d = np.repeat(np.ldexp(1.0, biased.astype(np.int64) - BIAS), 16, axis=1)
    fac = np.broadcast_to((1.0 + m8.astype(np.float64) / 256.0)[:, None], (n, L))
    dq = _deq(codes, d, fac)
    diff = dq.astype(np.float64) - x.astype(np.float64)
    return np.sum(diff * diff, axis=1)


def choose_exact(x: np.ndarray, cands: Sequence[int], augment: bool) -> np.ndarray:
    """Argmin-SSE mantissa per macro row, ties to the smaller byte
    (src/quantize.py:438-461)."""
    n = x.shape[0]
    trials = [np.full(n, c, dtype=np.uint8) for c in cands]
    if augment:
        trials.append(static_m8(np.abs(x.astype(np.float64)).max(axis=1)))
    m8s = np.stack(trials).astype(np.int64)
    sses = np.stack([macro_sse(x, t) for t in trials])
    best = sses.min(axis=0)
    cand = np.where(sses == best[None, :], m8s, 1 << 20)
    return cand.min(axis=0).astype(np.uint8)


# ---- LUT mode (src/quantize.py:108-125, :482-542) -------------------------

LUT_BINS = 64


def build_lut(cands: Sequence[int]) -> np.ndarray:
    """(2, 16, 64) fp16 squared-relative-error table (src/quantize.py:482-504)."""
    if len(cands) != 16:
        raise ValueError("the lookup table holds exactly 16 candidates")
    sub_c = np.arange(LUT_BINS) / LUT_BINS + 0.5 / LUT_BINS
    nor_c = 1.0 + np.arange(LUT_BINS) * 7.0 / LUT_BINS + 0.5 * 7.0 / LUT_BINS
    ent = np.empty((2, 16, LUT_BINS))
    for j, m in enumerate(cands):
        f = 1.0 + m / 256.0
        for r, c in enumerate((sub_c, nor_c)):
            u = c * f
            q = e2m1_decode(e2m1_encode(u))
            ent[r, j] = ((q - u) / u) ** 2
    return ent.astype(np.float16)


def choose_lut(x: np.ndarray, lut: np.ndarray, cands: Sequence[int]) -> np.ndarray:
    """LUT-estimated argmin (src/quantize.py:507-542)."""
    n, L = x.shape
    x64 = x.astype(np.float64)
    w = (x64 * x64).reshape(n, L // 16, 16)
    ent = lut.astype(np.float64)
    best_c = np.full(n, np.inf)
    best_m = np.zeros(n, dtype=np.uint8)
    for j, m in enumerate(cands):
        y = (x * np.float32(1.0 + m / 256.0)).astype(np.float32)
        _, biased = _blocks_quantize(y, oas=True)
        sf = np.ldexp(1.0, BIAS - biased.astype(np.int64))
        v = np.abs(x64.reshape(n, L // 16, 16)) * sf[:, :, None]
        bs = np.clip((v * LUT_BINS).astype(np.int64), 0, LUT_BINS - 1)
        bn = np.clip(((v - 1.0) * LUT_BINS / 7.0).astype(np.int64), 0, LUT_BINS - 1)
        t = np.where(v < 1.0, ent[0, j][bs], ent[1, j][bn])
        cost = np.sum(w * t, axis=(1, 2))
        if j == 0:
            better = np.ones(n, dtype=bool)
        else:
            better = (cost < best_c) | ((cost == best_c) & (m < best_m))
        best_c = np.where(better, cost, best_c)
        best_m = np.where(better, np.uint8(m), best_m)
    return best_m


# ---- tensor-level quantizers ----------------------------------------------

def quantize(t: np.ndarray, variant: str, macro_size: int = 128,
             mbs_mode: str = "exact", candidates: Sequence[int] = tuple(range(0, 256, 16)),
             augment_static: bool = True) -> OracleQ:
    """Tensor quantizer dispatch (src/quantize.py:709-725)."""
    bs = 32 if variant == "ocp32" else 16
    a = _check(t, bs)
    rows, cols = a.shape
    if variant == "nvfp4":
        return quantize_nvfp4(a)
    if variant in ("ocp32", "mx16", "mx16_oas"):
        codes, biased = _blocks_quantize(a, oas=variant == "mx16_oas", ocp=variant == "ocp32")
        return OracleQ(variant, (rows, cols), bs, macro_size, pack(codes), biased, None, None, None)
    # MBS (src/quantize.py:612-659): every macro row is independent, so the
    # tensor is processed one segment column-range at a time.
    segs = segments(cols, macro_size)
    codes = np.empty((rows, cols), dtype=np.uint8)
    biased = np.empty((rows, cols // 16), dtype=np.uint8)
    m8all = np.empty((rows, len(segs)), dtype=np.uint8)
    lut = build_lut(candidates) if (variant == "mbs_d" and mbs_mode == "lut") else None
    for i, (s, e) in enumerate(segs):
        x = np.ascontiguousarray(a[:, s:e])
        if variant == "mbs_s":
            m8 = static_m8(np.abs(x.astype(np.float64)).max(axis=1))
        elif mbs_mode == "exact":
            m8 = choose_exact(x, candidates, augment_static)
        else:
            m8 = choose_lut(x, lut, candidates)
        y = (x * _factor32(m8)[:, None]).astype(np.float32)
        c, b = _blocks_quantize(y, oas=True)
        codes[:, s:e] = c
        biased[:, s // 16:e // 16] = b
        m8all[:, i] = m8
    return OracleQ(variant, (rows, cols), 16, macro_size, pack(codes), biased, None, m8all, None)


def quantize_nvfp4(t: np.ndarray) -> OracleQ:
    """NVFP4: s_t = amax/2688, E4M3 block scale of alpha/(6 s_t), codes of
    x/(s_t d) in float64; d == 0 blocks flush (src/quantize.py:662-706)."""
    a = _check(t, 16)
    rows, cols = a.shape
    x = a.astype(np.float64)
    amax = float(np.abs(x).max())
    if amax == 0.0:
        return OracleQ("nvfp4", (rows, cols), 16, 128, np.zeros((rows, cols // 2), np.uint8),
                       None, np.zeros((rows, cols // 16), np.uint8), None, 1.0)
    st = amax / 2688.0
    b = x.reshape(rows, cols // 16, 16)
    alpha = np.abs(b).max(axis=2)
    sb = e4m3_encode(alpha / (6.0 * st))
    den = st * E4M3[sb]
    with np.errstate(divide="ignore", invalid="ignore"):
        sc = np.where(den[:, :, None] > 0, b / np.where(den > 0, den, 1.0)[:, :, None], 0.0)
    codes = e2m1_encode(sc.reshape(rows, cols))
    return OracleQ("nvfp4", (rows, cols), 16, 128, pack(codes), None, sb, None, st)


def block_d(q: OracleQ) -> np.ndarray:
    """Per-block D in float64 (src/quantize.py:220-240), validating codes."""
    if q.variant == "nvfp4":
        v = E4M3[q.e4m3_scales]
        if np.any(np.isnan(v)):
            raise ValueError("corrupt block scale: E4M3 NaN code")
        return v
    if np.any(q.block_scales == 255):
        raise ValueError("corrupt block scale: E8M0 code 255 is reserved")
    return np.ldexp(1.0, q.block_scales.astype(np.int64) - BIAS)


def factor_el(q: OracleQ) -> Optional[np.ndarray]:
    if q.mbs_mantissas is None:
        return None
    rows, cols = q.shape
    out = np.empty((rows, cols))
    f = 1.0 + q.mbs_mantissas.astype(np.float64) / 256.0
    for i, (s, e) in enumerate(segments(cols, q.macro_size)):
        out[:, s:e] = f[:, i:i + 1]
    return out


def dequantize(q: OracleQ) -> np.ndarray:
    """src/quantize.py:728-746."""
    rows, cols = q.shape
    d = np.repeat(block_d(q), q.block_size, axis=1)
    return _deq(unpack(q.codes, cols), d, factor_el(q), q.tensor_scale)


# --------------------------------------------------------------------------
# GEMM oracle (src/gemm.py:68-90, :137-172)
# --------------------------------------------------------------------------

def matmul_ref(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """C = f32(sum_k f64(a)f64(b)), k ascending (src/gemm.py:68-90).

    Each step adds a rounded f64 product (no FMA), exactly like the
    reference's outer-product loop.
    """
    a64 = np.asarray(a, dtype=np.float32).astype(np.float64)
    b64 = np.asarray(b, dtype=np.float32).astype(np.float64)
    if a64.ndim != 2 or b64.ndim != 2 or a64.shape[1] != b64.shape[1]:
        raise ValueError("inner dimensions differ")
    c = np.zeros((a64.shape[0], b64.shape[0]))
    for k in range(a64.shape[1]):
        c += a64[:, k:k + 1] * b64[None, :, k]
    return c.astype(np.float32)


def matmul_blas(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Large-shape GEMM oracle: f64 BLAS then one f32 rounding.  Not the
    ascending-k order, so used only with a tolerance."""
    return (np.asarray(a, np.float64) @ np.asarray(b, np.float64).T).astype(np.float32)


def matmul_quantized(aq: OracleQ, bq: OracleQ) -> np.ndarray:
    """Reference quantized GEMM == dequantize-then-matmul_ref, bit-exact
    (src/gemm.py:137-172, tests/test_gemm.py:73-93)."""
    if aq.shape[1] != bq.shape[1]:
        raise ValueError("operands disagree on K")
    return matmul_ref(dequantize(aq), dequantize(bq))


def ulp_distance(a: np.ndarray, b: np.ndarray) -> int:
    """src/gemm.py:196-214."""
    x = np.ascontiguousarray(a, np.float32).view(np.int32).astype(np.int64)
    y = np.ascontiguousarray(b, np.float32).view(np.int32).astype(np.int64)
    kx = np.where(x < 0, -(x & 0x7FFFFFFF), x)
    ky = np.where(y < 0, -(y & 0x7FFFFFFF), y)
    return int(np.max(np.abs(kx - ky))) if x.size else 0


# --------------------------------------------------------------------------
# Evaluator (src/metrics.py:127-182, :210-227)
# --------------------------------------------------------------------------

def qsnr(ref: np.ndarray, x: np.ndarray) -> tuple[float, float, float]:
    """(qsnr_db, mse, signal) with f64 numpy sums and a +inf sentinel."""
    r = np.asarray(ref, np.float32).astype(np.float64)
    d = r - np.asarray(x, np.float32).astype(np.float64)
    sig = float(np.sum(r * r))
    if sig == 0.0:
        raise ValueError("reference tensor is all zero")
    mse = float(np.sum(d * d))
    if mse == 0.0:
        return math.inf, 0.0, sig
    return 10.0 * math.log10(sig / mse), mse, sig


def flush_rate(ref: np.ndarray, q: OracleQ) -> float:
    r = np.asarray(ref, np.float32)
    nz = r != 0
    tot = int(nz.sum())
    if tot == 0:
        return 0.0
    mag = unpack(q.codes, q.shape[1]) & 7
    return int((nz & (mag == 0)).sum()) / tot


def generate(distribution: str, shape: tuple, seed: int, dof: float = 4.0,
             rate: float = 0.01, magnitude: float = 100.0) -> np.ndarray:
    """Seeded PCG64 tensors (src/metrics.py:210-227): the draw order is part
    of the contract, so the calls mirror the reference's."""
    g = np.random.Generator(np.random.PCG64(seed))
    if distribution == "gaussian":
        t = g.standard_normal(shape)
    elif distribution == "lognormal":
        t = g.lognormal(0.0, 1.0, shape)
    elif distribution == "student_t":
        t = g.standard_t(dof, shape)
    elif distribution == "gaussian_with_outliers":
        t = g.standard_normal(shape)
        t = np.where(g.random(shape) < rate, t * magnitude, t)
    else:
        raise ValueError(f"unknown distribution: {distribution}")
    return np.ascontiguousarray(t, dtype=np.float32)


def bf16_round(t: np.ndarray) -> np.ndarray:
    """Round f32 to the nearest bf16 (RNE), returned as f32 values."""
    u = np.ascontiguousarray(t, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


# --------------------------------------------------------------------------
# Row-sharded multi-process driver (bit-identical by
# tests/test_quantize.py:371-387) -- used only for the CPU baseline timing.
# --------------------------------------------------------------------------

def _q_worker(args):
    t, variant, kw = args
    q = quantize(t, variant, **kw)
    return q


def quantize_sharded(t: np.ndarray, variant: str, workers: int, pool=None, **kw) -> OracleQ:
    if variant == "nvfp4" or workers <= 1:
        return quantize(t, variant, **kw)
    parts = np.array_split(t, workers, axis=0)
    parts = [p for p in parts if p.shape[0]]
    res = list(pool.map(_q_worker, [(p, variant, kw) for p in parts]))
    cat = lambda f: None if getattr(res[0], f) is None else np.vstack([getattr(r, f) for r in res])
    return OracleQ(variant, t.shape, res[0].block_size, res[0].macro_size, cat("codes"),
                   cat("block_scales"), None, cat("mbs_mantissas"), None)
