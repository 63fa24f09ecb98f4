// sq_dev.cuh -- device side of the streaming quantizers, shared by
// quantize.cu (k_stream_quant, K1/K2) and gemm_mbs.cu (the fused MBS-S
// activation quantization in front of the MBS GEMM):
// 16-element unit loads, absmax, E2M1 encode of a unit, and sq_unit (one unit
// of OCP32 / MX16 / MX16_OAS / MBS-S with its scale / mantissa stores).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "mxq_arith.cuh"
#include "mxq_internal.h"

namespace mxq {

// Clear the sign bit of every nibble whose magnitude is 0 (the reference maps
// -0 / negative flushes to code 0): mag + 7 carries into bit 3 iff mag != 0.
__device__ __forceinline__ uint32_t fix_neg_zero(uint32_t w) {
  const uint32_t nz = ((w & 0x77777777u) + 0x77777777u) & 0x88888888u;
  return w & (0x77777777u | nz);
}

__device__ __forceinline__ uint32_t cvt_e2m1x2(float lo, float hi) {
  uint16_t r;
  asm("{\n\t.reg .b8 t;\n\tcvt.rn.satfinite.e2m1x2.f32 t, %1, %2;\n\tcvt.u16.u8 %0, t;\n\t}" : "=h"(r) : "f"(hi), "f"(lo));
  return r;
}

__device__ __forceinline__ void fmul2(float& o0, float& o1, float a0, float a1, float s) {
  asm("{\n\t.reg .b64 x, y;\n\tmov.b64 x, {%2, %3};\n\tmov.b64 y, {%4, %4};\n\t"
      "mul.rn.f32x2 x, x, y;\n\tmov.b64 {%0, %1}, x;\n\t}"
      : "=f"(o0), "=f"(o1) : "f"(a0), "f"(a1), "f"(s));
}

// 16 raw elements of one block.
template <int DT>
struct Blk16 {
  uint32_t w[DT == DT_BF16 ? 8 : 16];
};

template <int DT>
__device__ __forceinline__ void ld_blk(const void* __restrict__ x, int64_t off, Blk16<DT>& b) {
  if constexpr (DT == DT_BF16) {
    // one 256-bit load per 16-element block (sm_100 LDG.256): a warp reads 1 KB
    // contiguous per instruction; no L1 allocation for the streamed input
    const uint16_t* p = reinterpret_cast<const uint16_t*>(x) + off;
    asm volatile("ld.global.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(b.w[0]), "=r"(b.w[1]), "=r"(b.w[2]), "=r"(b.w[3]), "=r"(b.w[4]), "=r"(b.w[5]),
                   "=r"(b.w[6]), "=r"(b.w[7])
                 : "l"(p));
  } else {
    const uint4* p = reinterpret_cast<const uint4*>(reinterpret_cast<const float*>(x) + off);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint4 a = __ldcs(p + q);
      b.w[4 * q] = a.x; b.w[4 * q + 1] = a.y; b.w[4 * q + 2] = a.z; b.w[4 * q + 3] = a.w;
    }
  }
}

template <int DT>
__device__ __forceinline__ void zero_blk(Blk16<DT>& b) {
#pragma unroll
  for (int i = 0; i < (DT == DT_BF16 ? 8 : 16); ++i) b.w[i] = 0u;
}

// |x| max as f32 (exact), and the non-finite flag: integer max of the
// sign-cleared bit patterns (ordering of non-negative floats; NaN/Inf sort
// above every finite value).
template <int DT>
__device__ __forceinline__ float blk_absmax(const Blk16<DT>& b, uint32_t& bad) {
  if constexpr (DT == DT_BF16) {
    uint32_t m = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) m = __vmaxu2(m, b.w[j] & 0x7FFF7FFFu);
    const uint32_t top = max(m & 0xFFFFu, m >> 16);
    bad |= (top >= 0x7F80u) ? 1u : 0u;
    return __uint_as_float(top << 16);
  } else {
    uint32_t m = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) m = max(m, b.w[j] & 0x7FFFFFFFu);
    bad |= (m >= 0x7F800000u) ? 1u : 0u;
    return __uint_as_float(m);
  }
}

template <int DT>
__device__ __forceinline__ void blk_f32(const Blk16<DT>& b, float (&v)[16]) {
  if constexpr (DT == DT_BF16) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      v[2 * j] = __uint_as_float(b.w[j] << 16);
      v[2 * j + 1] = __uint_as_float(b.w[j] & 0xFFFF0000u);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(b.w[j]);
  }
}

// 16 codes of v * sf (exact power-of-two scaling) -> two packed words.
__device__ __forceinline__ void enc16(const float (&v)[16], float sf, uint32_t (&out)[2]) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    uint32_t word = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float lo, hi;
      fmul2(lo, hi, v[8 * h + 2 * j], v[8 * h + 2 * j + 1], sf);
      word |= cvt_e2m1x2(lo, hi) << (8 * j);
    }
    out[h] = fix_neg_zero(word);
  }
}

__device__ __forceinline__ float group_max(float v, int G) {
  for (int o = G / 2; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

constexpr int SQ_FOLD_LO = 27, SQ_FOLD_HI = 227;  // biased range where x*(f*SF) == RN(x*f)*SF for every code

enum { SQ_OCP32 = 0, SQ_MX16 = 1, SQ_OAS = 2, SQ_MBS_S = 3 };

// Output row pointers of one row tile, computed once per tile: the row index
// is CTA-uniform, so these live in uniform registers and every per-unit store
// address is one 32-bit offset from them.
struct RowOut {
  uint8_t* codes;   // codes of row r
  uint8_t* scales;  // row-major scales of row r (or null)
  uint8_t* sfm;     // SF-atom layout: the row part of sf_mma_offset (or null)
  uint8_t* mant;    // mantissa bytes of row r (or null)
  float* sig;       // sig_t column r (or null)
};

__device__ __forceinline__ RowOut row_out(const QDesc& q, uint32_t r) {
  RowOut o;
  o.codes = q.codes + (int64_t)r * q.codes_ld;
  o.scales = q.scales ? q.scales + (int64_t)r * q.scales_ld : nullptr;
  o.sfm = q.scales_mma ? q.scales_mma + sf_mma_offset(r, 0, q.sf_kpad) : nullptr;
  o.mant = q.mant ? q.mant + (int64_t)r * q.mant_ld : nullptr;
  o.sig = q.sig_t ? q.sig_t + r : nullptr;
  return o;
}

// one scale byte at block kbs of the row (both layouts)
__device__ __forceinline__ void store_scale_row(const RowOut& o, uint32_t kbs, uint8_t s) {
  if (o.scales) o.scales[kbs] = s;
  if (o.sfm) o.sfm[(kbs >> 2) * 512u + (kbs & 3u)] = s;
}

template <int DT, int VAR, int G>
__device__ __forceinline__ void sq_unit(const Blk16<DT>& xb, bool active, const RowOut& o, int64_t sig_ld,
                                        uint32_t kb, uint32_t lane, const float* sig_tab, uint32_t& bad,
                                        uint32_t& ovf_any) {
  float a = blk_absmax<DT>(xb, bad);
  float v[16];
  blk_f32<DT>(xb, v);
  uint32_t codes[2];
  if constexpr (VAR == SQ_MBS_S) {
    // src/quantize.py:383-406: m8 from the macro max, y = RN(x*f), OAS on y
    const float amac = G > 1 ? group_max(a, G) : a;
    const uint8_t m8 = static_m8(amac);
    const float f = mbs_factor(m8);
    const float af = __fmul_rn(a, f);
    const uint8_t biased = e8m0_biased_16(af, true);
    if (active && !(af <= 3.402823466e38f)) ovf_any = 1u;
    const float sf = exp2i_f32(127 - (int)biased);
    if (__all_sync(0xffffffffu, biased >= SQ_FOLD_LO && biased <= SQ_FOLD_HI)) {
      // f*SF is exact and RN(x*f)*SF == RN(x*(f*SF)) for every element that
      // can reach a nonzero code (quantizer section)
      enc16(v, __fmul_rn(f, sf), codes);
    } else {
      float y[16];
#pragma unroll
      for (int i = 0; i < 16; i += 2) fmul2(y[i], y[i + 1], v[i], v[i + 1], f);
      enc16(y, sf, codes);
    }
    if (active) {
      *reinterpret_cast<uint2*>(o.codes + kb * 8u) = make_uint2(codes[0], codes[1]);
      store_scale_row(o, kb, biased);
      if ((lane & (G - 1)) == 0) {
        const uint32_t mac = kb / G;
        if (o.mant) o.mant[mac] = m8;
        if (o.sig) o.sig[(int64_t)mac * sig_ld] = sig_tab[m8];
      }
    }
  } else {
    if constexpr (VAR == SQ_OCP32) a = group_max(a, 2);
    const uint8_t biased = VAR == SQ_OCP32 ? e8m0_biased_ocp(a) : e8m0_biased_16(a, VAR == SQ_OAS);
    enc16(v, exp2i_f32(127 - (int)biased), codes);
    if (active) {
      *reinterpret_cast<uint2*>(o.codes + kb * 8u) = make_uint2(codes[0], codes[1]);
      if (VAR != SQ_OCP32) store_scale_row(o, kb, biased);
      else if ((lane & 1) == 0) store_scale_row(o, kb >> 1, biased);
    }
  }
}

}  // namespace mxq
