// mxq_arith.cuh -- the arithmetic core of the MXFP4 (OCP / MX16 / OAS / MBS /
// NVFP4) path, shared by the sm_100a kernels and the host-compiled scalar
// C-ABI helpers.  Every routine restates a reference function bit-exactly;
// the citations point at /root/reference/pkg/src/mxq (written src/...).
//
// Pinned arithmetic (src/quantize.py:22-27): the MBS factor multiply is an
// f32 RN multiply (no FMA contraction), power-of-two scaling is exact, the
// dequantised element is rounded to f32 once.  Compile WITHOUT fast-math and
// without FTZ: f32-subnormal block maxima legitimately produce non-zero codes
// once the E8M0 exponent clamps at biased 0.
#pragma once
#include <stdint.h>
#include <math.h>
#include <string.h>

#if defined(__CUDACC__)
#define MXQ_HD __host__ __device__ __forceinline__
#else
#define MXQ_HD inline
#endif

namespace mxq {

enum Variant : int32_t { OCP32 = 0, MX16 = 1, MX16_OAS = 2, MBS_S = 3, MBS_D = 4, NVFP4 = 5 };

// Device status word bits (the Python wrapper raises the reference's
// ValueError text for each).
enum StatusBits : uint32_t {
  ST_NONFINITE = 1u,     // src/quantize.py:581-582
  ST_BAD_E8M0 = 2u,      // src/quantize.py:239-240
  ST_BAD_E4M3 = 4u,      // src/quantize.py:235-236
  ST_OVERFLOW = 8u,      // f32 factor multiply overflowed (reference raises in encode)
};

MXQ_HD uint32_t f2u(float f) {
#if defined(__CUDA_ARCH__)
  return __float_as_uint(f);
#else
  uint32_t u; memcpy(&u, &f, 4); return u;
#endif
}
MXQ_HD float u2f(uint32_t u) {
#if defined(__CUDA_ARCH__)
  return __uint_as_float(u);
#else
  float f; memcpy(&f, &u, 4); return f;
#endif
}

// IEEE RN f32 multiply / divide that the compiler may not contract or
// approximate.
MXQ_HD float mul_rn(float a, float b) {
#if defined(__CUDA_ARCH__)
  return __fmul_rn(a, b);
#else
  volatile float r = a * b; return r;
#endif
}
MXQ_HD float div_rn(float a, float b) {
#if defined(__CUDA_ARCH__)
  return __fdiv_rn(a, b);
#else
  volatile float r = a / b; return r;
#endif
}
MXQ_HD double dmul_rn(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dmul_rn(a, b);
#else
  volatile double r = a * b; return r;
#endif
}
MXQ_HD double dadd_rn(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dadd_rn(a, b);
#else
  volatile double r = a + b; return r;
#endif
}

// ---------------------------------------------------------------------------
// floor(log2 a) and the 23-bit fraction of a positive finite f32, with f32
// subnormals normalised (the reference works on the exact f64 value).
// ---------------------------------------------------------------------------
MXQ_HD void f32_exp_frac(float a, int& e, uint32_t& frac) {
  uint32_t u = f2u(a) & 0x7fffffffu;
  uint32_t ex = u >> 23;
  if (ex != 0) {
    e = (int)ex - 127;
    frac = u & 0x7fffffu;
  } else {  // subnormal: value = m * 2^-149
    uint32_t m = u;
#if defined(__CUDA_ARCH__)
    int msb = 31 - __clz(m);
#else
    int msb = 31 - __builtin_clz(m);
#endif
    e = msb - 149;
    frac = (m << (23 - msb)) & 0x7fffffu;
  }
}

// E8M0 biased dequant exponent for 16-blocks, MX16 / OAS
// (src/quantize.py:268-281).  SF = 2^floor(log2(6/alpha)); with alpha =
// 1.f * 2^e that is 2-e when 1.f <= 1.5 and 1-e otherwise; OAS doubles SF
// when alpha*SF <= 3.5, i.e. exactly when 1.f <= 1.75.
MXQ_HD uint8_t e8m0_biased_16(float alpha, bool oas) {
  if (!(alpha > 0.0f)) return 127;
  int e; uint32_t f;
  f32_exp_frac(alpha, e, f);
  int sf_exp = (f <= (oas ? 0x600000u : 0x400000u)) ? 2 - e : 1 - e;
  int b = 127 - sf_exp;
  return (uint8_t)(b < 0 ? 0 : (b > 254 ? 254 : b));
}

// OCP32: D = 2^(floor(log2 alpha) - 2) (src/quantize.py:284-289).
MXQ_HD uint8_t e8m0_biased_ocp(float alpha) {
  if (!(alpha > 0.0f)) return 127;
  int e; uint32_t f;
  f32_exp_frac(alpha, e, f);
  int b = e - 2 + 127;
  return (uint8_t)(b < 0 ? 0 : (b > 254 ? 254 : b));
}

// f64 forms for the host scalar API (the reference's block helpers take
// float64 blocks, src/quantize.py:292-334): floor(log2(6/alpha)) via frexp on
// the f64 quotient, OAS trigger on the exact alpha*SF, OCP floor(log2 alpha)-2.
// kind: 0 = OCP32, 1 = MX16, 2 = MX16 + OAS.  Returns the biased byte and
// whether the exponent was clamped into [0, 254].
MXQ_HD int e8m0_block_f64(double alpha, int kind, int* clamped) {
  *clamped = 0;
  if (!(alpha > 0.0)) return 127;
  int e, want;
  if (kind == 0) {
    frexp(alpha, &e);
    want = (e - 1) - 2 + 127;
  } else {
    frexp(6.0 / alpha, &e);
    int sf_exp = e - 1;
    if (kind == 2 && ldexp(alpha, sf_exp) <= 3.5) sf_exp += 1;
    want = 127 - sf_exp;
  }
  int b = want < 0 ? 0 : (want > 254 ? 254 : want);
  *clamped = (b != want);
  return b;
}

// 2^k as an f32 for k in [-127, 127] (2^-127 is the subnormal 0x00400000).
MXQ_HD float exp2i_f32(int k) {
  return k >= -126 ? u2f((uint32_t)(k + 127) << 23) : u2f(0x00400000u >> (-127 - k));
}

// MBS-S mantissa byte (src/quantize.py:369-389, eq. 3 of the paper):
// bits(f32(6)/f32(alpha)) >> 15 & 0xFF; alpha == 0 -> 0.  An overflowing
// quotient (alpha tiny) is +inf whose fraction bits are 0.
MXQ_HD uint8_t static_m8(float alpha) {
  if (!(alpha > 0.0f)) return 0;
  float r = div_rn(6.0f, alpha);
  return (uint8_t)((f2u(r) >> 15) & 0xFFu);
}

// 1 + m8/256 as the f32 the reference multiplies by (exact: 9 bits).
MXQ_HD float mbs_factor(uint32_t m8) { return 1.0f + (float)m8 * (1.0f / 256.0f); }

// ---------------------------------------------------------------------------
// E2M1 (src/formats.py:141-207)
// ---------------------------------------------------------------------------
// Grid magnitudes by index, and their midpoints.
MXQ_HD float e2m1_grid(int i) {
  // 0, 0.5, 1, 1.5, 2, 3, 4, 6
  return i < 4 ? 0.5f * (float)i : (i == 4 ? 2.0f : (i == 5 ? 3.0f : (i == 6 ? 4.0f : 6.0f)));
}

// Nearest index for a magnitude in f64, ties to the even index, saturating.
MXQ_HD uint32_t e2m1_index_f64(double mag) {
  const double mids[7] = {0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0};
  uint32_t idx = 0;
  bool tie = false;
#pragma unroll
  for (int k = 0; k < 7; ++k) {
    idx += (mag > mids[k]) ? 1u : 0u;
    tie |= (mag == mids[k]);
  }
  return (tie && (idx & 1u)) ? idx + 1u : idx;
}

// Signed code from an f64 value (sign only when the index is non-zero).
MXQ_HD uint32_t e2m1_code_f64(double v) {
  double mag = v < 0 ? -v : v;
  if (mag > 6.0) mag = 6.0;
  uint32_t idx = e2m1_index_f64(mag);
  return (v < 0 && idx) ? (idx | 8u) : idx;
}

// Same for an f32 scaled value (host path / reference for the cvt path).
MXQ_HD uint32_t e2m1_code_f32_soft(float v) { return e2m1_code_f64((double)v); }

#if defined(__CUDACC__)
// Two codes via the sm_100 converter: cvt.rn.satfinite.e2m1x2.f32 rounds to
// nearest-even (E2M1 mantissa bit == index & 1, so ties-to-even-mantissa ==
// the reference's ties-to-even-index) and saturates at +-6.  The hardware
// keeps the sign of a zero result; the reference maps -0 to code 0, so a
// nibble whose magnitude is 0 is cleared.  lo -> bits 0-3, hi -> bits 4-7.
__device__ __forceinline__ uint32_t e2m1x2(float lo, float hi) {
  uint16_t r;
  asm("{\n\t.reg .b8 t;\n\tcvt.rn.satfinite.e2m1x2.f32 t, %1, %2;\n\tcvt.u16.u8 %0, t;\n\t}"
      : "=h"(r) : "f"(hi), "f"(lo));
  uint32_t b = r;
  if ((b & 0x7u) == 0) b &= 0xF0u;
  if ((b & 0x70u) == 0) b &= 0x0Fu;
  return b;
}
#endif

// ---------------------------------------------------------------------------
// E4M3 (src/formats.py:235-292): decode table and RNE encode from f64.
// ---------------------------------------------------------------------------
MXQ_HD double e4m3_decode(uint32_t c) {
  uint32_t e = (c >> 3) & 15u, m = c & 7u;
  double v;
  if (e == 0) {
    v = (double)m * 0.001953125;  // m * 2^-9
  } else if (e == 15 && m == 7) {
    v = NAN;
  } else {  // (8 + m) * 2^(e - 10) = 1.m * 2^(e - 7), built from its bit pattern (exact)
    const uint64_t bits = ((uint64_t)(e - 7 + 1023) << 52) | ((uint64_t)m << 49);
    memcpy(&v, &bits, sizeof(v));
  }
  return (c & 0x80u) ? -v : v;
}

// Nearest finite E4M3 magnitude code (0..0x7E) for r >= 0 in f64, ties to
// the even code, clamp at 448.  The reference's searchsorted over exact
// midpoints + odd-tie bump (src/formats.py:278-292) is RNE on the 3-bit
// mantissa, computed here on the exact f64 value.
MXQ_HD uint32_t e4m3_code_f64(double r) {
  if (!(r > 0.0)) return 0;
  if (r >= 448.0) return 0x7Eu;
  if (r < 0.015625) {  // subnormal range: multiples of 2^-9 (code 8 == 2^-6)
    double q = rint(r * 512.0);
    return (uint32_t)q;
  }
  // normal range [2^-6, 448): RNE of the 52-bit fraction to 3 bits on the f64
  // bit pattern (== rint((fr * 2 - 1) * 8) with frexp, without the library calls)
  uint64_t bits;
  memcpy(&bits, &r, sizeof(bits));
  const int e = (int)((bits >> 52) & 0x7ffu) - 1023;  // r = 1.f * 2^e, e in [-6, 8]
  const uint64_t frac = bits & ((1ull << 52) - 1);
  uint32_t m = (uint32_t)(frac >> 49);
  const uint64_t rem = frac & ((1ull << 49) - 1), half = 1ull << 48;
  if (rem > half || (rem == half && (m & 1u))) ++m;
  int E = e + 7;
  if (m >= 8u) { m = 0u; E += 1; }
  const uint32_t code = ((uint32_t)E << 3) | m;
  return code > 0x7Eu ? 0x7Eu : code;
}

// ---------------------------------------------------------------------------
// Dequantised element (src/quantize.py:409-423): f32(g * D / f * s_t) with
// the reference's f64 internal arithmetic.
// ---------------------------------------------------------------------------
// Power-of-two variants: g*D is exact in f64 and its f32 rounding is the
// f32 product (exact or +-inf) computed directly.
MXQ_HD float deq_pow2(uint32_t code, uint32_t biased) {
  double v = (double)e2m1_grid(code & 7) * ldexp(1.0, (int)biased - 127);
  float r = (float)v;
  return (code & 8u) ? -r : r;
}

// MBS: f32(f64(g*D) / f64(f)).  For 4 <= biased <= 250 the quotient and
// g*D are f32-normal and the single f32 division is the same correctly
// rounded value (re-verified exhaustively by
// tests/test_capi_host.py); outside that window the f64 formula is used
// verbatim.
MXQ_HD float deq_mbs(uint32_t code, uint32_t biased, uint32_t m8) {
  uint32_t idx = code & 7u;
  float r;
  if (idx == 0) {
    r = 0.0f;
  } else if (biased >= 4 && biased <= 250) {
    float gd = e2m1_grid((int)idx) * exp2i_f32((int)biased - 127);
    r = div_rn(gd, mbs_factor(m8));
  } else {
    double gd = (double)e2m1_grid((int)idx) * ldexp(1.0, (int)biased - 127);
    r = (float)(gd / (1.0 + (double)m8 / 256.0));
  }
  return (code & 8u) ? -r : r;
}

// NVFP4: f32((g*d) * s_t), g*d exact in f64, one f64 rounding then f32.
MXQ_HD float deq_nvfp4(uint32_t code, uint32_t e4m3, double st) {
  double v = (double)e2m1_grid(code & 7) * e4m3_decode(e4m3);
  v = dmul_rn(v, st);
  float r = (float)v;
  return (code & 8u) ? -r : r;
}

// ---------------------------------------------------------------------------
// tcgen05 scale-factor atom layout (K-major): 128 rows x 4 blocks = 512 B,
// byte (r%32)*16 + ((r%128)/32)*4 + kb%4; atoms ordered [row/128][kb/4].
// Third-party cross-check: CUTLASS cutlass/detail/sm100_blockscaled_layout.hpp
// (SfKMajorAtom).
// ---------------------------------------------------------------------------
MXQ_HD int64_t sf_mma_offset(int64_t r, int64_t kb, int64_t kb_pad) {
  return ((r >> 7) * (kb_pad >> 2) + (kb >> 2)) * 512 + (r & 31) * 16 + ((r >> 5) & 3) * 4 + (kb & 3);
}

// ---------------------------------------------------------------------------
// numpy pairwise summation (numpy/core/src/umath/loops_utils.h.src
// pairwise_sum, PW_BLOCKSIZE 128).  The reference's f64 sums
// (np.sum(axis=1) in _macro_sse, np.sum in qsnr_tensor) use it, so the GPU
// reproduces the exact tree: leaves of <= 128 elements reduced with 8
// strided accumulators, split points n/2 rounded down to a multiple of 8.
// ---------------------------------------------------------------------------
MXQ_HD double pw_leaf(const double* a, int64_t n) {
  if (n < 8) {
    double s = 0.0;  // numpy starts this branch at 0.
    for (int64_t i = 0; i < n; ++i) s = dadd_rn(s, a[i]);
    return s;
  }
  double r[8];
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8)
    for (int j = 0; j < 8; ++j) r[j] = dadd_rn(r[j], a[i + j]);
  double res = dadd_rn(dadd_rn(dadd_rn(r[0], r[1]), dadd_rn(r[2], r[3])),
                       dadd_rn(dadd_rn(r[4], r[5]), dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = dadd_rn(res, a[i]);
  return res;
}

MXQ_HD int64_t pw_split(int64_t n) {
  int64_t n2 = n / 2;
  return n2 - (n2 % 8);
}

}  // namespace mxq
