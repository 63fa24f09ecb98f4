// quantize.cu -- sm_100a quantizer kernels (K1-K4) and the dequantiser (K5).
//
// K1 quantize_pow2   OCP32 / MX16 / MX16_OAS   src/quantize.py:586-609
// K2 quantize_mbs_s  MBS-Static                src/quantize.py:612-659, :383-406
// K3 quantize_mbs_d  MBS-Dynamic (exact)       src/quantize.py:426-461
// K4 quantize_nvfp4  two passes (amax, encode) src/quantize.py:662-706
// K5 dequantize                                src/quantize.py:728-746
//
// All quantizers are HBM-bound streaming kernels except MBS-D (17 candidate
// trials per macro, compute-bound).  One thread owns one 16-element block
// (32 for OCP32): 128-bit loads of bf16/f32, warp-shuffle macro maxima, the
// integer E8M0 closed form, hardware E2M1 pair conversion, one 8/16-byte code
// store.  Scales are written row-major (the reference layout) and/or in the
// tcgen05 SF-atom layout the GEMM's TMA reads directly.
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>

#include "mxq_arith.cuh"
#include "mxq_internal.h"
#include "sq_dev.cuh"

namespace mxq {

// ---------------------------------------------------------------------------
// Loading one block of `N` elements as f32 (bf16 widened exactly).
// ---------------------------------------------------------------------------
template <int N>
__device__ __forceinline__ void load_block(const void* __restrict__ x, int dtype, int64_t off, float (&v)[N]) {
  if (dtype == DT_BF16) {
    const uint4* p = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(x) + off);
#pragma unroll
    for (int q = 0; q < N / 8; ++q) {
      uint4 w = __ldcs(p + q);
      uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        v[q * 8 + 2 * j] = __uint_as_float(ws[j] << 16);
        v[q * 8 + 2 * j + 1] = __uint_as_float(ws[j] & 0xffff0000u);
      }
    }
  } else {
    const float4* p = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(x) + off);
#pragma unroll
    for (int q = 0; q < N / 4; ++q) {
      float4 w = __ldcs(p + q);
      v[q * 4 + 0] = w.x; v[q * 4 + 1] = w.y; v[q * 4 + 2] = w.z; v[q * 4 + 3] = w.w;
    }
  }
}

template <int N>
__device__ __forceinline__ float block_absmax(const float (&v)[N], bool& finite) {
  float a = 0.0f;
  uint32_t bad = 0;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    uint32_t u = __float_as_uint(v[i]) & 0x7fffffffu;
    bad |= (u >= 0x7f800000u);
    a = fmaxf(a, __uint_as_float(u));
  }
  finite = !bad;
  return a;
}

// ---------------------------------------------------------------------------
// Streaming fast path (K1, K2).  Index math uses a precomputed 32-bit
// division (the 64-bit integer division the first version used cost ~100
// instructions per block); the -0 fix-up, absmax and scaling run on packed
// words; every thread keeps two blocks of loads in flight.
// ---------------------------------------------------------------------------
struct FastDiv {
  uint32_t d, m, s;
};

static FastDiv make_fastdiv(uint32_t d) {
  FastDiv f;
  f.d = d;
  f.s = 0;
  while ((1ull << f.s) < d) ++f.s;
  f.m = (uint32_t)((((1ull << 32) * ((1ull << f.s) - d)) / d) + 1);
  return f;
}

__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) {
  return (uint32_t)(((uint64_t)__umulhi(n, f.m) + n) >> f.s);
}

__device__ __forceinline__ void store_scale(const QDesc& q, uint32_t r, uint32_t kb, uint8_t s) {
  if (q.scales) q.scales[(int64_t)r * q.scales_ld + kb] = s;
  if (q.scales_mma) q.scales_mma[sf_mma_offset(r, kb, q.sf_kpad)] = s;
}

// ---------------------------------------------------------------------------
// Macro-group geometry for MBS: G lanes (a power of two <= 32) own one macro
// of up to 32 blocks (macro_size <= 512); a trailing partial macro simply has
// fewer active lanes.
// ---------------------------------------------------------------------------
struct MacroGeom {
  int G;          // lanes per macro group
  int64_t nmac;   // macros per row
  int macro;      // macro width (elements)
};

__device__ __forceinline__ void store_m8(const QDesc& q, int64_t r, int64_t mac, uint8_t m8) {
  if (q.mant) q.mant[r * q.mant_ld + mac] = m8;
  if (q.sig_t) q.sig_t[mac * q.sig_t_ld + r] = 1.0f / mbs_factor(m8);
}

// Quantise one block (v, scaled by the f32 factor f) with OAS: the shared
// second half of MBS-S and MBS-D (src/quantize.py:392-406).  y = RN(x*f);
// max|y| = RN(max|x| * f) because rounding is monotone.
__device__ __forceinline__ uint8_t mbs_block(const float (&v)[16], float alpha, float f, uint32_t (&packed)[2],
                                             bool& ovf) {
  float y[16];
#pragma unroll
  for (int i = 0; i < 16; i += 2) fmul2(y[i], y[i + 1], v[i], v[i + 1], f);
  const float a = __fmul_rn(alpha, f);
  ovf = !(a <= 3.402823466e38f);
  const uint8_t biased = e8m0_biased_16(a, true);
  enc16(y, exp2i_f32(127 - (int)biased), packed);
  return biased;
}

// K2: MBS-Static.  The CTA-uniform `base` loop keeps every warp converged
// for the group shuffles.
template <int DT>
__global__ void __launch_bounds__(256) k_quantize_mbs_s(const void* __restrict__ x, int64_t x_ld, QDesc q,
                                                        MacroGeom g, FastDiv fd_nmac, uint32_t ngroups,
                                                        uint32_t* __restrict__ status) {
  const int lane = threadIdx.x & 31;
  const int sub = lane & (g.G - 1);
  const uint32_t gpb = blockDim.x / g.G;  // groups per CTA pass
  uint32_t bad = 0, ovf_any = 0;
  for (uint32_t base = blockIdx.x * gpb; base < ngroups; base += gridDim.x * gpb) {
    const uint32_t gi = base + threadIdx.x / g.G;
    const bool live_group = gi < ngroups;
    const uint32_t r = live_group ? fdiv(gi, fd_nmac) : 0u;
    const uint32_t mac = live_group ? gi - r * fd_nmac.d : 0u;
    const int64_t c0 = (int64_t)mac * g.macro + (int64_t)sub * 16;
    const int64_t width = live_group ? min((int64_t)g.macro, q.cols - (int64_t)mac * g.macro) : 0;
    const bool active = live_group && sub * 16 < width;
    Blk16<DT> xb;
    if (active) ld_blk<DT>(x, (int64_t)r * x_ld + c0, xb);
    else zero_blk<DT>(xb);
    const float a16 = blk_absmax<DT>(xb, bad);
    const float amac = group_max(a16, g.G);
    const uint8_t m8 = static_m8(amac);
    float v[16];
    blk_f32<DT>(xb, v);
    uint32_t packed[2];
    bool ovf;
    const uint8_t biased = mbs_block(v, a16, mbs_factor(m8), packed, ovf);
    if (active) {
      ovf_any |= ovf ? 1u : 0u;
      const uint32_t kb = (uint32_t)(c0 >> 4);
      *reinterpret_cast<uint2*>(q.codes + (int64_t)r * q.codes_ld + kb * 8) = make_uint2(packed[0], packed[1]);
      store_scale(q, r, kb, biased);
      if (sub == 0) store_m8(q, r, mac, m8);
    }
  }
  if (bad) atomicOr(status, ST_NONFINITE);
  if (ovf_any) atomicOr(status, ST_OVERFLOW);
}

// ---------------------------------------------------------------------------
// Row-tiled streaming path (K1, K2 and K4 pass 2).  A CTA takes a tile of 256
// consecutive 16-element units of one row (4096 elements); unit kb of the row
// belongs to lane kb % 32, so loads and code stores are coalesced and all row /
// tile index math is CTA-uniform.  G consecutive lanes share one scale (OCP32:
// G = 2) or one MBS macro (G = macro/16, a power of two); SQ_UNROLL tiles are
// in flight per thread.
// ---------------------------------------------------------------------------
constexpr int SQ_THREADS = 256;
#ifndef MXQ_SQ_UNROLL
#define MXQ_SQ_UNROLL 4
#endif
constexpr int SQ_UNROLL = MXQ_SQ_UNROLL;  // tiles per thread in flight


__device__ __forceinline__ void store_scale_u(const QDesc& q, uint32_t r, uint32_t kbs, uint8_t s) {
  if (q.scales) q.scales[(int64_t)r * q.scales_ld + kbs] = s;
  if (q.scales_mma) q.scales_mma[sf_mma_offset(r, kbs, q.sf_kpad)] = s;
}

template <int DT, int VAR, int G>
__global__ void __launch_bounds__(SQ_THREADS) k_stream_quant(const void* __restrict__ x, int64_t x_ld, QDesc q,
                                                             uint32_t nblk, FastDiv tpr, uint32_t ntiles,
                                                             uint32_t* __restrict__ status) {
  const uint32_t tid = threadIdx.x, lane = tid & 31;
  uint32_t bad = 0, ovf_any = 0;
  // sigma = 1/(1+m8/256) for every m8 (IEEE f32 division, as the GEMM layout
  // expects), one entry per thread, instead of a division per macro
  __shared__ float sig_tab[256];
  if constexpr (VAR == SQ_MBS_S) {
    sig_tab[tid] = 1.0f / mbs_factor(tid);
    __syncthreads();
  }
  for (uint32_t t0 = blockIdx.x; t0 < ntiles; t0 += SQ_UNROLL * gridDim.x) {
    // all SQ_UNROLL tiles' loads first: a 4096 x 4096 tensor is in flight at once
    Blk16<DT> xb[SQ_UNROLL];
    uint32_t rr[SQ_UNROLL], kk[SQ_UNROLL];
#pragma unroll
    for (int u = 0; u < SQ_UNROLL; ++u) {
      const uint32_t t = t0 + u * gridDim.x;
      rr[u] = fdiv(t, tpr);
      kk[u] = (t - rr[u] * tpr.d) * SQ_THREADS + tid;
      if (t < ntiles && kk[u] < nblk) ld_blk<DT>(x, (int64_t)rr[u] * x_ld + kk[u] * 16, xb[u]);
      else zero_blk<DT>(xb[u]);
    }
#pragma unroll
    for (int u = 0; u < SQ_UNROLL; ++u) {
      const uint32_t t = t0 + u * gridDim.x;
      if (t < ntiles)
        sq_unit<DT, VAR, G>(xb[u], kk[u] < nblk, row_out(q, rr[u]), q.sig_t_ld, kk[u], lane, sig_tab, bad, ovf_any);
    }
  }
  if (bad) atomicOr(status, ST_NONFINITE);
  if (ovf_any) atomicOr(status, ST_OVERFLOW);
}

// ---------------------------------------------------------------------------
// Row-RUN streaming quantizer (K1 / K2 / K4 pass 2, the standalone launches).
// A thread owns RUN = 4 consecutive 16-element units of one row (64
// elements): one row pointer per run, four 256-bit loads in flight, and the
// outputs leave as whole words -- 32 B of codes, the run's 4 scale bytes as
// one 32-bit store in each layout (row-major and the tcgen05 SF atom, whose 4
// bytes of a 128-row x 4-block atom row are contiguous), one mantissa byte and
// one sigma per MBS macro.  Lane j of a warp takes run j of a row, so a warp
// reads 4 KB contiguous and the per-unit index math of the unit-per-thread
// form (one unit per lane, ~190 instructions per unit measured) is paid once
// per run.  MBS macros: UPM = macro/16 units; UPM <= 4 -> RUN/UPM macros per
// thread, else GL = UPM/4 lanes per macro (max over a lane group); runs per
// row are padded to a multiple of GL so lane groups never straddle rows.
// ---------------------------------------------------------------------------
constexpr int RUN = 4;

template <int DT, int VAR, int UPM>
__global__ void __launch_bounds__(256) k_quant_runs(const void* __restrict__ x, int64_t x_ld, QDesc q,
                                                    uint32_t nblk, FastDiv rpr, uint32_t nruns,
                                                    uint32_t* __restrict__ status) {
  constexpr int GL = (VAR == SQ_MBS_S && UPM > RUN) ? UPM / RUN : 1;   // lanes per macro
  constexpr int MPT = (VAR == SQ_MBS_S && UPM <= RUN) ? RUN / UPM : 1;  // macros per thread
  const uint32_t lane = threadIdx.x & 31;
  uint32_t bad = 0, ovf_any = 0;
  __shared__ float sig_tab[256];
  if constexpr (VAR == SQ_MBS_S) {
    sig_tab[threadIdx.x] = 1.0f / mbs_factor(threadIdx.x);
    __syncthreads();
  }
  const bool words_ok = ((q.scales_ld & 3) == 0) && (((uintptr_t)q.scales & 3) == 0);
  const uint32_t step = gridDim.x * blockDim.x;
  const uint32_t total = (nruns + 31u) & ~31u;  // whole warps (GL lane groups stay converged)
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < total; j += step) {
    const bool live = j < nruns;
    const uint32_t r = live ? fdiv(j, rpr) : 0u;
    const uint32_t kb0 = live ? (j - r * rpr.d) * RUN : nblk;
    const uint32_t nu = kb0 < nblk ? min((uint32_t)RUN, nblk - kb0) : 0u;  // valid units of the run
    Blk16<DT> xb[RUN];
    const int64_t off = (int64_t)r * x_ld + (int64_t)kb0 * 16;
#pragma unroll
    for (int i = 0; i < RUN; ++i) {
      if ((uint32_t)i < nu) ld_blk<DT>(x, off + i * 16, xb[i]);
      else zero_blk<DT>(xb[i]);
    }
    float a[RUN];
#pragma unroll
    for (int i = 0; i < RUN; ++i) a[i] = blk_absmax<DT>(xb[i], bad);
    uint32_t codes[RUN][2];
    uint8_t sc[RUN];
    uint8_t m8s[MPT];
    if constexpr (VAR == SQ_MBS_S) {
      // src/quantize.py:383-406: m8 from the macro max, y = RN(x*f), OAS on y
#pragma unroll
      for (int mi = 0; mi < MPT; ++mi) {
        constexpr int UM = MPT > 1 ? UPM : RUN;  // units of this thread in the macro
        float am = a[mi * UM];
#pragma unroll
        for (int i = 1; i < UM; ++i) am = fmaxf(am, a[mi * UM + i]);
        if constexpr (GL > 1) am = group_max(am, GL);
        m8s[mi] = static_m8(am);
        const float f = mbs_factor(m8s[mi]);
#pragma unroll
        for (int i = mi * UM; i < (mi + 1) * UM; ++i) {
          const float af = __fmul_rn(a[i], f);
          if ((uint32_t)i < nu && !(af <= 3.402823466e38f)) ovf_any = 1u;
          const uint8_t biased = e8m0_biased_16(af, true);
          sc[i] = biased;
          const float sf = exp2i_f32(127 - (int)biased);
          float v[16];
          blk_f32<DT>(xb[i], v);
          if (biased >= SQ_FOLD_LO && biased <= SQ_FOLD_HI) {
            // f*SF exact and RN(x*f)*SF == RN(x*(f*SF)) for every element that
            // can reach a nonzero code (quantizer section)
            enc16(v, __fmul_rn(f, sf), codes[i]);
          } else {
            float y[16];
#pragma unroll
            for (int e = 0; e < 16; e += 2) fmul2(y[e], y[e + 1], v[e], v[e + 1], f);
            enc16(y, sf, codes[i]);
          }
        }
      }
    } else if constexpr (VAR == SQ_OCP32) {
#pragma unroll
      for (int bb = 0; bb < RUN / 2; ++bb) {
        const uint8_t biased = e8m0_biased_ocp(fmaxf(a[2 * bb], a[2 * bb + 1]));
        sc[2 * bb] = sc[2 * bb + 1] = biased;
        const float sf = exp2i_f32(127 - (int)biased);
#pragma unroll
        for (int i = 2 * bb; i < 2 * bb + 2; ++i) {
          float v[16];
          blk_f32<DT>(xb[i], v);
          enc16(v, sf, codes[i]);
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < RUN; ++i) {
        const uint8_t biased = e8m0_biased_16(a[i], VAR == SQ_OAS);
        sc[i] = biased;
        float v[16];
        blk_f32<DT>(xb[i], v);
        enc16(v, exp2i_f32(127 - (int)biased), codes[i]);
      }
    }
    if (nu == 0) continue;
    // ---- stores -------------------------------------------------------------
    uint8_t* crow = q.codes + (int64_t)r * q.codes_ld + kb0 * 8;
    if (nu == RUN) {
      reinterpret_cast<uint4*>(crow)[0] = make_uint4(codes[0][0], codes[0][1], codes[1][0], codes[1][1]);
      reinterpret_cast<uint4*>(crow)[1] = make_uint4(codes[2][0], codes[2][1], codes[3][0], codes[3][1]);
    } else {
#pragma unroll
      for (int i = 0; i < RUN; ++i)
        if ((uint32_t)i < nu) reinterpret_cast<uint2*>(crow)[i] = make_uint2(codes[i][0], codes[i][1]);
    }
    if constexpr (VAR == SQ_OCP32) {
      // two 32-element blocks per run: scale bytes kb0/2, kb0/2 + 1
      const uint32_t kbs = kb0 >> 1, ns = (nu + 1) >> 1;
      if (q.scales) {
        uint8_t* sp = q.scales + (int64_t)r * q.scales_ld + kbs;
        for (uint32_t i = 0; i < ns; ++i) sp[i] = sc[2 * i];
      }
      if (q.scales_mma) {
        uint8_t* sp = q.scales_mma + sf_mma_offset(r, kbs, q.sf_kpad);
        for (uint32_t i = 0; i < ns; ++i) sp[i] = sc[2 * i];
      }
    } else {
      const uint32_t w = (uint32_t)sc[0] | ((uint32_t)sc[1] << 8) | ((uint32_t)sc[2] << 16) | ((uint32_t)sc[3] << 24);
      if (q.scales) {
        uint8_t* sp = q.scales + (int64_t)r * q.scales_ld + kb0;
        if (nu == RUN && words_ok) *reinterpret_cast<uint32_t*>(sp) = w;
        else for (uint32_t i = 0; i < nu; ++i) sp[i] = sc[i];
      }
      if (q.scales_mma) {  // kb0 % 4 == 0: the 4 bytes of one atom row are contiguous
        uint8_t* sp = q.scales_mma + sf_mma_offset(r, kb0, q.sf_kpad);
        if (nu == RUN) *reinterpret_cast<uint32_t*>(sp) = w;
        else for (uint32_t i = 0; i < nu; ++i) sp[i] = sc[i];
      }
      if constexpr (VAR == SQ_MBS_S) {
#pragma unroll
        for (int mi = 0; mi < MPT; ++mi) {
          const uint32_t ufirst = kb0 + mi * (MPT > 1 ? UPM : RUN);
          if (ufirst >= nblk || (GL > 1 && (lane & (GL - 1)) != 0)) continue;
          const uint32_t mac = ufirst / UPM;
          if (q.mant) q.mant[(int64_t)r * q.mant_ld + mac] = m8s[mi];
          if (q.sig_t) q.sig_t[(int64_t)mac * q.sig_t_ld + r] = sig_tab[m8s[mi]];
        }
      }
    }
  }
  if (bad) atomicOr(status, ST_NONFINITE);
  if (ovf_any) atomicOr(status, ST_OVERFLOW);
}

// ---------------------------------------------------------------------------
// K4 NVFP4 in the run form (src/quantize.py:662-706): pass 1 |x| max, pass 2
// E4M3 block scale + element codes, four 16-element units per thread.
// Block scale: the E4M3 RNE code of the f64 ratio alpha / (6 s_t) is taken from
// the hardware converter on an f32 estimate (relative error < 2^-22) at
// r(1 - 2^-19), r and r(1 + 2^-19); when the three codes agree they equal the
// code of the exact ratio (E4M3 RNE is monotone), else the f64 division runs.
// Elements: as nvfp4_unit (f32 estimate, three E2M1 encodes, f64 fallback).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t cvt_e4m3x2(float lo, float hi) {
  uint16_t r;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
  return r;
}

// Warp CHUNKS: a warp takes 128 consecutive units of one row (lane: units
// base + lane + 32 i), so every 256-bit load instruction reads 1 KB contiguous
// (a run of four units per lane reads a 4 KB span per instruction: 4x the L1
// tag work per byte) and the row pointer is computed once per chunk.
constexpr int CHUNK = 128;

template <int DT>
__global__ void __launch_bounds__(256) k_absmax_runs(const void* __restrict__ x, int64_t x_ld, uint32_t nblk,
                                                     FastDiv cpr, uint32_t nchunks, uint32_t* __restrict__ status) {
  uint32_t bad = 0;
  float m = 0.0f;
  const uint32_t lane = threadIdx.x & 31, wstep = gridDim.x * (blockDim.x / 32);
  for (uint32_t ch = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); ch < nchunks; ch += wstep) {
    const uint32_t r = fdiv(ch, cpr), kb0 = (ch - r * cpr.d) * CHUNK;
    Blk16<DT> xb[CHUNK / 32];
#pragma unroll
    for (int i = 0; i < CHUNK / 32; ++i) {
      const uint32_t kb = kb0 + lane + 32 * i;
      if (kb < nblk) ld_blk<DT>(x, (int64_t)r * x_ld + (int64_t)kb * 16, xb[i]);
      else zero_blk<DT>(xb[i]);
    }
#pragma unroll
    for (int i = 0; i < CHUNK / 32; ++i) m = fmaxf(m, blk_absmax<DT>(xb[i], bad));
  }
  // one atomic per CTA, and only when it can raise the running maximum
  // (same-address atomics of one per warp serialize at the L2 slice)
  __shared__ uint32_t s_m, s_bad;
  if (threadIdx.x == 0) { s_m = 0u; s_bad = 0u; }
  __syncthreads();
  for (int o = 16; o > 0; o >>= 1) {
    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  if (lane == 0) {
    atomicMax(&s_m, __float_as_uint(m));
    if (bad) atomicOr(&s_bad, 1u);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t mb = s_m;
    if (mb != 0u && mb > *reinterpret_cast<volatile uint32_t*>(status + 1)) atomicMax(status + 1, mb);
    if (s_bad) atomicOr(status, ST_NONFINITE);
  }
}

// Rare exact paths, out of line so the hot loop stays small (an inlined f64
// division per call site overflowed the instruction cache: 44 % of the stall
// samples were no_instructions).
__device__ __noinline__ uint32_t nvfp4_scale_exact(float alpha, double six_st) {
  return e4m3_code_f64((double)alpha / six_st);
}
__device__ __noinline__ uint32_t nvfp4_pair_exact(float v0, float v1, double st, uint32_t sb) {
  const double den = st * e4m3_decode(sb);
  return e2m1_code_f64(__ddiv_rn((double)v0, den)) | (e2m1_code_f64(__ddiv_rn((double)v1, den)) << 4);
}
// E4M3 value of a code (0..0x7E) as an exact f32.
__device__ __forceinline__ float e4m3_f32(uint32_t c) {
  const uint32_t e = c >> 3, m = c & 7u;
  return e ? __uint_as_float(((e + 120u) << 23) | (m << 20)) : (float)m * 0.001953125f;  // subnormal: m * 2^-9
}

template <int DT>
__global__ void __launch_bounds__(256) k_nvfp4_runs(const void* __restrict__ x, int64_t x_ld, QDesc q, uint32_t nblk,
                                                    FastDiv cpr, uint32_t nchunks,
                                                    const uint32_t* __restrict__ amax_bits) {
  const float amax = __uint_as_float(*amax_bits);
  const bool nz = amax > 0.0f;
  const double st = nz ? (double)amax / 2688.0 : 1.0;
  const double six_st = 6.0 * st;
  const float inv6 = (float)(1.0 / six_st);
  const bool est_ok = inv6 >= 1.17549435e-38f && inv6 <= 3.0e38f;  // f32-normal reciprocal (else f64 scales)
  const float st32 = (float)st;
  if (blockIdx.x == 0 && threadIdx.x == 0 && q.tensor_scale) *q.tensor_scale = st;
  const uint32_t lane = threadIdx.x & 31, wstep = gridDim.x * (blockDim.x / 32);
  for (uint32_t ch = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); ch < nchunks; ch += wstep) {
    const uint32_t r = fdiv(ch, cpr), kb0 = (ch - r * cpr.d) * CHUNK;
    constexpr int NU = CHUNK / 32;
    Blk16<DT> xb[NU];
#pragma unroll
    for (int i = 0; i < NU; ++i) {
      const uint32_t kb = kb0 + lane + 32 * i;
      if (kb < nblk) ld_blk<DT>(x, (int64_t)r * x_ld + (int64_t)kb * 16, xb[i]);
      else zero_blk<DT>(xb[i]);
    }
    uint32_t codes[NU][2];
    uint32_t scw = 0;
#pragma unroll
    for (int i = 0; i < NU; ++i) {
      uint32_t unused = 0;
      const float alpha = blk_absmax<DT>(xb[i], unused);
      uint32_t sb = 0;
      if (nz) {
        const float rr = alpha * inv6;
        const uint32_t c2 = cvt_e4m3x2(rr * 0.99999809265136719f, rr * 1.00000190734863281f);  // r (1 -+ 2^-19)
        const uint32_t cm = cvt_e4m3x2(rr, rr) & 0xFFu;
        sb = (est_ok && (c2 & 0xFFu) == cm && (c2 >> 8) == cm) ? cm : nvfp4_scale_exact(alpha, six_st);
      }
      scw |= sb << (8 * i);
      codes[i][0] = codes[i][1] = 0u;
      if (sb != 0) {
        // quotient estimate x / den in f32: den32 = RN(RN(st) * E4M3(sb)), relative
        // error < 2^-21 after the reciprocal and the product
        const float den32 = st32 * e4m3_f32(sb);
        const bool f32_ok = den32 > 1e-30f && den32 < 1e30f;
        const float inv = __frcp_rn(den32);
        // the exact quotient lies between x*inv_lo and x*inv_hi (relative error
        // of the estimate < 2^-21 << 2^-17); E2M1 RNE is monotone, so equal
        // codes at both ends are the code of the exact quotient
        const float inv_lo = inv * 0.99999237060546875f, inv_hi = inv * 1.00000762939453125f;  // 1 -+ 2^-17
        float v[16];
        blk_f32<DT>(xb[i], v);
        uint32_t word[2] = {0u, 0u}, mism = 0;  // mism: pairs whose two ends disagree
#pragma unroll
        for (int pr = 0; pr < 8; ++pr) {
          float l0, l1, u0, u1;
          fmul2(l0, l1, v[2 * pr], v[2 * pr + 1], inv_lo);
          fmul2(u0, u1, v[2 * pr], v[2 * pr + 1], inv_hi);
          const uint32_t c = cvt_e2m1x2(l0, l1);
          mism |= (cvt_e2m1x2(u0, u1) != c) ? (1u << pr) : 0u;
          word[pr >> 2] |= c << (8 * (pr & 3));
        }
        if (!f32_ok) mism = 0xFFu;
        // straddling pairs (f64 quotient, out of line).  On bf16 data about 0.4 %
        // of the elements sit EXACTLY on an E2M1 midpoint after the f64 division
        // (x, amax and the E4M3 scale have few significand bits), so most warps
        // take this branch for a pair or two per unit -- it is the main cost of
        // the pass (NVFP4).
        if (mism) {
          for (int pr = 0; pr < 8; ++pr)
            if (mism & (1u << pr)) {
              const uint32_t c = nvfp4_pair_exact(v[2 * pr], v[2 * pr + 1], st, sb);
              word[pr >> 2] = (word[pr >> 2] & ~(0xFFu << (8 * (pr & 3)))) | (c << (8 * (pr & 3)));
            }
        }
        codes[i][0] = fix_neg_zero(word[0]);
        codes[i][1] = fix_neg_zero(word[1]);
      }
    }
    uint8_t* crow = q.codes + (int64_t)r * q.codes_ld;
    uint8_t* srow = q.scales ? q.scales + (int64_t)r * q.scales_ld : nullptr;
    uint8_t* mrow = q.scales_mma ? q.scales_mma + sf_mma_offset(r, 0, q.sf_kpad) : nullptr;
#pragma unroll
    for (int i = 0; i < NU; ++i) {
      const uint32_t kb = kb0 + lane + 32 * i;
      if (kb < nblk) {
        *reinterpret_cast<uint2*>(crow + kb * 8) = make_uint2(codes[i][0], codes[i][1]);
        const uint8_t sb = (uint8_t)(scw >> (8 * i));
        if (srow) srow[kb] = sb;
        if (mrow) mrow[(kb >> 2) * 512u + (kb & 3u)] = sb;
      }
    }
  }
}

// K4 pass 1: |x| max of the whole tensor (uint ordering of non-negative
// floats) and the non-finite check, same tiling, one atomic per warp.
template <int DT>
__global__ void __launch_bounds__(SQ_THREADS) k_stream_absmax(const void* __restrict__ x, int64_t x_ld,
                                                              uint32_t nblk, FastDiv tpr, uint32_t ntiles,
                                                              uint32_t* __restrict__ status) {
  const uint32_t tid = threadIdx.x;
  uint32_t bad = 0;
  float m = 0.0f;
  for (uint32_t t0 = blockIdx.x; t0 < ntiles; t0 += SQ_UNROLL * gridDim.x) {
    Blk16<DT> xb[SQ_UNROLL];
#pragma unroll
    for (int u = 0; u < SQ_UNROLL; ++u) {
      const uint32_t t = t0 + u * gridDim.x;
      const uint32_t r = fdiv(t, tpr), kb = (t - r * tpr.d) * SQ_THREADS + tid;
      if (t < ntiles && kb < nblk) ld_blk<DT>(x, (int64_t)r * x_ld + kb * 16, xb[u]);
      else zero_blk<DT>(xb[u]);
    }
#pragma unroll
    for (int u = 0; u < SQ_UNROLL; ++u) m = fmaxf(m, blk_absmax<DT>(xb[u], bad));
  }
  for (int o = 16; o > 0; o >>= 1) {
    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  if ((tid & 31) == 0) {
    if (m > 0.0f) atomicMax(status + 1, __float_as_uint(m));
    if (bad) atomicOr(status, ST_NONFINITE);
  }
}

// K4 pass 2.  The element code is E2M1-RN of the f64 quotient x/(s_t*d)
// (src/quantize.py:684-700).  The quotient is estimated in f32 (relative error
// < 2^-21) and encoded at t*(1-2^-17), t and t*(1+2^-17); E2M1 rounding is
// monotone, so when all three codes agree they equal the code of the exact
// f64 quotient.  Only pairs that straddle a rounding boundary (or an
// out-of-range denominator) take the f64 division.
template <int DT>
__device__ __forceinline__ void nvfp4_unit(const Blk16<DT>& xb, bool active, const QDesc& q, uint32_t r, uint32_t kb,
                                           double st, double six_st, bool nz) {
  uint32_t bad_unused = 0;
  const float alpha = blk_absmax<DT>(xb, bad_unused);
  const uint32_t sb = nz ? e4m3_code_f64((double)alpha / six_st) : 0u;
  const double den = st * e4m3_decode(sb);
  float v[16];
  blk_f32<DT>(xb, v);
  uint32_t packed[2] = {0u, 0u};
  if (den > 0.0) {
    const bool f32_ok = den > 1e-30 && den < 1e30;
    const float inv = f32_ok ? __frcp_rn(__double2float_rn(den)) : 0.0f;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint32_t word = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int i = 8 * h + 2 * j;
        float t0, t1, l0, l1, u0, u1;
        fmul2(t0, t1, v[i], v[i + 1], inv);
        fmul2(l0, l1, t0, t1, 0.99999237060546875f);   // 1 - 2^-17
        fmul2(u0, u1, t0, t1, 1.00000762939453125f);   // 1 + 2^-17
        uint32_t c = cvt_e2m1x2(t0, t1);
        const uint32_t cl = cvt_e2m1x2(l0, l1), cu = cvt_e2m1x2(u0, u1);
        if (!f32_ok || cl != c || cu != c)
          c = e2m1_code_f64(__ddiv_rn((double)v[i], den)) | (e2m1_code_f64(__ddiv_rn((double)v[i + 1], den)) << 4);
        word |= c << (8 * j);
      }
      packed[h] = fix_neg_zero(word);
    }
  }
  if (active) {
    *reinterpret_cast<uint2*>(q.codes + (int64_t)r * q.codes_ld + kb * 8) = make_uint2(packed[0], packed[1]);
    store_scale_u(q, r, kb, (uint8_t)sb);
  }
}

template <int DT>
__global__ void __launch_bounds__(SQ_THREADS) k_stream_nvfp4(const void* __restrict__ x, int64_t x_ld, QDesc q,
                                                             uint32_t nblk, FastDiv tpr, uint32_t ntiles,
                                                             const uint32_t* __restrict__ amax_bits) {
  const float amax = __uint_as_float(*amax_bits);
  const bool nz = amax > 0.0f;
  const double st = nz ? (double)amax / 2688.0 : 1.0;
  const double six_st = 6.0 * st;
  if (blockIdx.x == 0 && threadIdx.x == 0 && q.tensor_scale) *q.tensor_scale = st;
  constexpr int NV_UNROLL = 2;  // (the f64 fallback path needs the registers)
  const uint32_t tid = threadIdx.x;
  for (uint32_t t0 = blockIdx.x; t0 < ntiles; t0 += NV_UNROLL * gridDim.x) {
    Blk16<DT> xb[NV_UNROLL];
    uint32_t rr[NV_UNROLL], kk[NV_UNROLL];
#pragma unroll
    for (int u = 0; u < NV_UNROLL; ++u) {
      const uint32_t t = t0 + u * gridDim.x;
      rr[u] = fdiv(t, tpr);
      kk[u] = (t - rr[u] * tpr.d) * SQ_THREADS + tid;
      if (t < ntiles && kk[u] < nblk) ld_blk<DT>(x, (int64_t)rr[u] * x_ld + kk[u] * 16, xb[u]);
      else zero_blk<DT>(xb[u]);
    }
#pragma unroll
    for (int u = 0; u < NV_UNROLL; ++u) {
      const uint32_t t = t0 + u * gridDim.x;
      if (t < ntiles) nvfp4_unit<DT>(xb[u], kk[u] < nblk, q, rr[u], kk[u], st, six_st, nz);
    }
  }
}

// ---------------------------------------------------------------------------
// K3: MBS-Dynamic, exact mode.  For every candidate m8 (plus the static one
// when augmenting) the macro is quantised and dequantised exactly as the
// reference does, the f64 squared errors are staged in shared memory and one
// lane per group reduces them in numpy's pairwise order, so the argmin (ties
// to the smaller byte) is bit-identical to src/quantize.py:438-461.
// ---------------------------------------------------------------------------
constexpr int MBSD_THREADS = 128;
constexpr int MBSD_STRIDE = 17;  // doubles per lane slot (16 + 1 pad)
constexpr int MBSD_BUF = MBSD_THREADS * MBSD_STRIDE;  // one trial's staged errors
#ifndef MXQ_MBSD_PAIR
#define MXQ_MBSD_PAIR 1
#endif

// Element p of a macro lives in lane p/16, slot p%16.
__device__ __forceinline__ double sq_at(const double* base, int64_t p) {
  return base[(p >> 4) * MBSD_STRIDE + (p & 15)];
}

__device__ __forceinline__ double pw_leaf_smem(const double* base, int64_t s, int64_t n) {
  if (n < 8) {
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) acc = __dadd_rn(acc, sq_at(base, s + i));
    return acc;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = sq_at(base, s + j);
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], sq_at(base, s + i + j));
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, sq_at(base, s + i));
  return res;
}

// numpy's split recursion, unrolled at compile time (no device recursion):
// macro widths <= 512 need at most 2 split levels, D = 3 covers <= 1024.
template <int D>
__device__ __forceinline__ double pw_sum_smem_t(const double* base, int64_t s, int64_t n) {
  if constexpr (D == 0) {
    return pw_leaf_smem(base, s, n);
  } else {
    if (n <= 128) return pw_leaf_smem(base, s, n);
    const int64_t n2 = pw_split(n);
    return __dadd_rn(pw_sum_smem_t<D - 1>(base, s, n2), pw_sum_smem_t<D - 1>(base, s + n2, n - n2));
  }
}

__device__ __noinline__ double pw_sum_smem(const double* base, int64_t s, int64_t n) { return pw_sum_smem_t<3>(base, s, n); }

// MBS-D candidate bytes and (LUT mode) the error table (src/quantize.py:482-504:
// [regime][candidate][bin] fp16 values widened to f32, exact), passed BY VALUE
// as a __grid_constant__ kernel parameter: every launch carries its own copy,
// so concurrent quantize calls on different streams cannot see each other's
// candidates (no process-global __constant__ symbol is written).
struct MbsdTables {
  uint8_t cands[256];
  float lut[2][16][64];
};

// LUT bin of v = |x| * SF (src/quantize.py:507-542) as a byte: bit 7 the
// regime (v >= 1), bits 0-5 the bin -- floor(v * 64) below 1,
// floor((v - 1) * 64 / 7) above.  v is exact in f32 wherever a bin can be
// nonzero (an f32 x times a power of two; an f32-subnormal v is below 2^-126
// and lands in bin 0 either way), v - 1 and the products by 64 and 7 are
// exact, and floor(RN64(t / 7)) == floor(t / 7) (t has a 24-bit significand,
// so t / 7 is never within an f64 half-ulp of an integer from below) -- the
// reference's f64 division per element becomes an f32 estimate with an exact
// integer correction.
__device__ __forceinline__ uint32_t lut_bin_byte(float x, float sf) {
  const float vf = fabsf(x) * sf;
  if (vf < 1.0f) {
    const int b = (int)(vf * 64.0f);
    return (uint32_t)(b > 63 ? 63 : b);
  }
  const float tt = (vf - 1.0f) * 64.0f;
  int b = (int)(tt * 0.142857142857142857f);
  if (7.0f * (float)(b + 1) <= tt) ++b;
  else if (7.0f * (float)b > tt) --b;
  b = b < 0 ? 0 : (b > 63 ? 63 : b);
  return 0x80u | (uint32_t)b;
}

// LUT=false: exact SSE search (src/quantize.py:438-461).
// LUT=true : table-estimated cost sum(x^2 * T[v]) (src/quantize.py:507-542),
//            v = |x| * SF(OAS scale of the candidate-scaled block).
template <bool LUT>
__global__ void __launch_bounds__(MBSD_THREADS, LUT ? 5 : 4) k_quantize_mbs_d(const void* __restrict__ x, int dtype, int64_t x_ld,
                                                                 QDesc q, MacroGeom g, int n_cand, int augment,
                                                                 uint32_t* __restrict__ status,
                                                                 const __grid_constant__ MbsdTables tab) {
  __shared__ double s_sq[((!LUT && MXQ_MBSD_PAIR) ? 2 : 1) * MBSD_BUF];
  // the LUT in shared memory: a dynamically indexed kernel parameter would be
  // copied to local memory per thread
  __shared__ float s_lut[LUT ? 2 * 16 * 64 : 1];
  // (RN(1/f), RN(1.5/f)) per mantissa byte: every dequantised magnitude
  // RN(g/f) of the E2M1 grid g = {0.5,1,1.5,2,3,4,6} is one of the two times a
  // power of two (exact: g/f lies in [0.25, 12], f32-normal), so a trial's
  // eight levels need no division
  __shared__ float2 s_uv[LUT ? 1 : 256];
#ifndef MXQ_MBSD_SMEM_TQ
#define MXQ_MBSD_SMEM_TQ 1
#endif
  // per-lane signed dequantisation levels of the current trial as f64 (code
  // 0..15 -> value): one shared load per element instead of a select chain
  // over a dynamically indexed register array and a conversion
  using tq_t = typename std::conditional<MXQ_MBSD_PAIR != 0, float, double>::type;  // (48 KB static limit)
  __shared__ tq_t s_tq[(LUT || !MXQ_MBSD_SMEM_TQ) ? 1 : MBSD_THREADS * 17];
  __shared__ double s_x2[LUT ? MBSD_THREADS * 17 : 1];
  if constexpr (LUT) {
    for (int i = threadIdx.x; i < 2 * 16 * 64; i += MBSD_THREADS) s_lut[i] = (&tab.lut[0][0][0])[i];
  } else {
    for (int i = threadIdx.x; i < 256; i += MBSD_THREADS) {
      const float f = mbs_factor((uint32_t)i);
      s_uv[i] = make_float2(__fdiv_rn(1.0f, f), __fdiv_rn(1.5f, f));
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int sub = lane & (g.G - 1);
  double* gbase = s_sq + (threadIdx.x - sub) * MBSD_STRIDE;  // this group's slots
  double* mine = s_sq + threadIdx.x * MBSD_STRIDE;
  const int64_t ngroups = q.rows * g.nmac;
  const int64_t gpb = MBSD_THREADS / g.G;
  uint32_t bad = 0;
  for (int64_t base = (int64_t)blockIdx.x * gpb; base < ngroups; base += (int64_t)gridDim.x * gpb) {
    const int64_t gi = base + threadIdx.x / g.G;
    const bool live_group = gi < ngroups;
    const int64_t r = live_group ? gi / g.nmac : 0;
    const int64_t mac = live_group ? gi - r * g.nmac : 0;
    const int64_t c0 = mac * g.macro + (int64_t)sub * 16;
    const int64_t width = live_group ? min((int64_t)g.macro, q.cols - mac * g.macro) : 0;
    const bool active = live_group && sub * 16 < width;
    float v[16];
    if (active) load_block<16>(x, dtype, r * x_ld + c0, v);
    else {
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = 0.0f;
    }
    bool fin;
    float a16 = block_absmax<16>(v, fin);
    bad |= !fin;
    const float amac = group_max(a16, g.G);
    const uint32_t m8_static = static_m8(amac);
    const int n_trials = n_cand + (augment ? 1 : 0);
    double best_sse = 0.0;
    uint32_t best_m8 = 0;
    // LUT mode: x^2 (f64, the reference's first product) and the bin bytes of
    // |x| * SF for the two scale exponents a trial can take, once per macro
    uint32_t lut_b0 = 0, lut_bins[2][4] = {{0u, 0u, 0u, 0u}, {0u, 0u, 0u, 0u}};
    double* x2s = s_x2 + threadIdx.x * 17;
    if constexpr (LUT) {
      lut_b0 = e8m0_biased_16(a16, true);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const float sfe = exp2i_f32(127 - (int)(lut_b0 + e));
#pragma unroll
        for (int i = 0; i < 16; ++i) lut_bins[e][i >> 2] |= lut_bin_byte(v[i], sfe) << (8 * (i & 3));
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const double x64 = (double)v[i];
        x2s[i] = __dmul_rn(x64, x64);
      }
    }
    // One trial's per-element pass: the quantise-dequantise (or LUT) squared
    // errors of this lane's 16 elements into mb (this lane's slots of a buffer).
    auto elem_pass = [&](int t, double* mb) -> uint32_t {
        const uint32_t m8 = t < n_cand ? (uint32_t)tab.cands[t] : m8_static;
        const float f = mbs_factor(m8);
        // quantise: y = x*f, OAS scale, codes.  max|RN(x f)| = RN(max|x| f)
        // (RN is monotone), so the block maximum needs no pass over y
        const float a = __fmul_rn(a16, f);
        const uint32_t biased = e8m0_biased_16(a, true);
        const float sf = exp2i_f32(127 - (int)biased);
        if constexpr (LUT) {
          // f < 2, so the trial's scale exponent is b0 or b0 + 1: the bins of
          // both were taken once per macro (lut_bins); other exponents (none
          // expected) take the per-element computation below
          const uint32_t e = biased - lut_b0;
          if (e <= 1u) {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const uint32_t word = e ? lut_bins[1][i >> 2] : lut_bins[0][i >> 2];
              const uint32_t byte = (word >> (8 * (i & 3))) & 0xFFu;
              const float tv = s_lut[((byte >> 7) * 16 + t) * 64 + (byte & 63u)];
              mb[i] = active ? __dmul_rn(x2s[i], (double)tv) : 0.0;
            }
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const uint32_t byte = lut_bin_byte(v[i], sf);
              const float tv = s_lut[((byte >> 7) * 16 + t) * 64 + (byte & 63u)];
              mb[i] = active ? __dmul_rn(x2s[i], (double)tv) : 0.0;
            }
          }
        }
        if constexpr (!LUT) {
          float y[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) y[i] = __fmul_rn(v[i], f);
          const bool fast = biased >= 4 && biased <= 250;
          float tq[8];
          if (fast) {
            const float d = exp2i_f32((int)biased - 127);
            const float2 uv = s_uv[m8];
            const float u = uv.x * d, w = uv.y * d;  // (exact: d is a power of two in the normal range)
            tq[0] = 0.0f;
            tq[1] = 0.5f * u;
            tq[2] = u;
            tq[3] = w;
            tq[4] = 2.0f * u;
            tq[5] = 2.0f * w;
            tq[6] = 4.0f * u;
            tq[7] = 4.0f * w;
          }
          if (MXQ_MBSD_SMEM_TQ && fast) {
            tq_t* tqd = s_tq + threadIdx.x * 17;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              tqd[k] = (tq_t)tq[k];
              tqd[8 + k] = -(tq_t)tq[k];
            }
#pragma unroll
            for (int i = 0; i < 16; i += 2) {
              const uint32_t c2 = e2m1x2(__fmul_rn(y[i], sf), __fmul_rn(y[i + 1], sf));
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const double diff = __dsub_rn((double)tqd[(c2 >> (4 * h)) & 15u], (double)v[i + h]);
                mb[i + h] = active ? __dmul_rn(diff, diff) : 0.0;
              }
            }
          } else {
#pragma unroll
          for (int i = 0; i < 16; i += 2) {
            uint32_t c2 = e2m1x2(__fmul_rn(y[i], sf), __fmul_rn(y[i + 1], sf));
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const uint32_t c = (c2 >> (4 * h)) & 15u;
              float dq;
              if (fast) {
                dq = tq[c & 7];
                dq = (c & 8u) ? -dq : dq;
              } else {
                dq = deq_mbs(c, biased, m8);
              }
              const double diff = __dsub_rn((double)dq, (double)v[i + h]);
              mb[i + h] = active ? __dmul_rn(diff, diff) : 0.0;
            }
          }
          }
        }
        return m8;
    };
    // A full 128-element macro's eight strided accumulators (numpy's leaf
    // order): r_j = sq[j] + sq[j+8] + ... in ascending order, one per lane of
    // the group (element sub + 8k sits in lane slot k/2, position sub + 8 (k % 2)).
    auto lane_chain = [&](const double* gb) -> double {
      const double* cb = gb + sub;
      double r = cb[0];
#pragma unroll
      for (int k = 1; k < 16; ++k) r = __dadd_rn(r, cb[(k >> 1) * MBSD_STRIDE + 8 * (k & 1)]);
      return r;
    };
    auto take = [&](int t, uint32_t m8, double sse) {
      if (sub == 0) {
        const bool better = (t == 0) || (sse < best_sse) || (sse == best_sse && m8 < best_m8);
        if (better) { best_sse = sse; best_m8 = m8; }
      }
    };
    // Trials in pairs (exact mode): both trials' errors are staged in two
    // buffers and their accumulator chains and shuffle trees run interleaved --
    // each is a dependent f64 chain, and the kernel was latency-bound on them.
    // The argmin is taken in trial order, as before.
    constexpr int PAIR = (!LUT && MXQ_MBSD_PAIR) ? 2 : 1;
    for (int t0 = 0; t0 < n_trials; t0 += PAIR) {
      const bool two = PAIR == 2 && t0 + 1 < n_trials;
      const uint32_t m8a = elem_pass(t0, mine);
      uint32_t m8b = 0;
      if (two) m8b = elem_pass(t0 + 1, mine + MBSD_BUF);
      __syncwarp();
      double sa = 0.0, sb = 0.0;
      if (g.G == 8) {
        // ... then ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) by shuffles -- the same
        // operations in the same order as pw_leaf
        double ra = lane_chain(gbase), rb = two ? lane_chain(gbase + MBSD_BUF) : 0.0;
        ra = __dadd_rn(ra, __shfl_down_sync(0xffffffffu, ra, 1));  // r0+r1, r2+r3, ...
        rb = __dadd_rn(rb, __shfl_down_sync(0xffffffffu, rb, 1));
        ra = __dadd_rn(ra, __shfl_down_sync(0xffffffffu, ra, 2));  // (r0+r1)+(r2+r3), ...
        rb = __dadd_rn(rb, __shfl_down_sync(0xffffffffu, rb, 2));
        ra = __dadd_rn(ra, __shfl_down_sync(0xffffffffu, ra, 4));  // the macro's sum at sub 0
        rb = __dadd_rn(rb, __shfl_down_sync(0xffffffffu, rb, 4));
        if (sub == 0 && live_group) {
          sa = width == 128 ? ra : pw_sum_smem(gbase, 0, width);
          if (two) sb = width == 128 ? rb : pw_sum_smem(gbase + MBSD_BUF, 0, width);
        }
      } else if (sub == 0 && live_group) {
        sa = pw_sum_smem(gbase, 0, width);
        if (two) sb = pw_sum_smem(gbase + MBSD_BUF, 0, width);
      }
      __syncwarp();
      take(t0, m8a, sa);
      if (two) take(t0 + 1, m8b, sb);
    }
    const uint32_t m8 = __shfl_sync(0xffffffffu, best_m8, lane & ~(g.G - 1));
    uint32_t packed[2];
    bool ovf;
    const uint8_t biased = mbs_block(v, a16, mbs_factor(m8), packed, ovf);
    if (active) {
      bad |= ovf ? 2u : 0u;
      *reinterpret_cast<uint2*>(q.codes + r * q.codes_ld + (c0 / 16) * 8) = make_uint2(packed[0], packed[1]);
      store_scale(q, (uint32_t)r, (uint32_t)(c0 / 16), biased);
      if (sub == 0) store_m8(q, r, mac, (uint8_t)m8);
    }
  }
  if (bad & 1u) atomicOr(status, ST_NONFINITE);
  if (bad & 2u) atomicOr(status, ST_OVERFLOW);
}

// ---------------------------------------------------------------------------
// K5: dequantise to f32 (src/quantize.py:728-746).  Thread == block.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_dequantize(QDesc q, float* __restrict__ out, int64_t out_ld,
                                                    FastDiv fd_nbr, uint32_t nb, uint32_t* __restrict__ status) {
  const int bs = q.block_size;
  const uint32_t nbr = fd_nbr.d;
  const double st = (q.variant == NVFP4 && q.tensor_scale) ? *q.tensor_scale : 1.0;
  // (RN(1/f), RN(1.5/f)) per mantissa byte, shared by the CTA (two f32
  // divisions per block otherwise)
  __shared__ float2 s_uv[256];
  if (q.mant) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
      const float f = mbs_factor((uint32_t)i);
      s_uv[i] = make_float2(__fdiv_rn(1.0f, f), __fdiv_rn(1.5f, f));
    }
    __syncthreads();
  }
  const uint32_t umac = (uint32_t)q.macro_size;
  const bool mac_pow2 = (umac & (umac - 1)) == 0;
  const int mac_shift = __ffs((int)umac) - 1;
  uint32_t bad = 0;
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += gridDim.x * blockDim.x) {
    const uint32_t r = fdiv(b, fd_nbr), kb = b - r * nbr;
    const uint32_t s = q.scales[(int64_t)r * q.scales_ld + kb];
    uint32_t m8 = 0;
    if (q.mant) {
      const uint32_t col = kb * (uint32_t)bs;
      m8 = q.mant[(int64_t)r * q.mant_ld + (mac_pow2 ? (col >> mac_shift) : col / umac)];
    }
    if (q.variant == NVFP4) bad |= ((s & 0x7fu) == 0x7fu) ? ST_BAD_E4M3 : 0u;
    else bad |= (s == 255u) ? ST_BAD_E8M0 : 0u;
    // Fast path (E8M0 variants, 4 <= biased <= 250, every value f32-normal):
    // the grid is {0.5, 1, 2, 4} x 1 and {1, 2, 4} x 1.5, so with
    // u = RN(1/f), v = RN(1.5/f) (f = 1+m8/256, or 1) every magnitude is
    // u or v times 2^((idx>>1) - 1 + biased - 127) -- an exact power-of-two
    // scaling of the same correctly rounded quotient deq_mbs computes.
    const bool fast = q.variant != NVFP4 && s >= 4u && s <= 250u;
    float u = 1.0f, v = 1.5f;
    if (fast && q.mant) {
      const float2 uv = s_uv[m8];
      u = uv.x;
      v = uv.y;
    }
    const uint8_t* cp = q.codes + (int64_t)r * q.codes_ld + kb * (bs / 2);
    float* op = out + (int64_t)r * out_ld + (int64_t)kb * bs;
    for (int w = 0; w < bs / 8; ++w) {
      const uint32_t word = *reinterpret_cast<const uint32_t*>(cp + 4 * w);
      float o[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t c = (word >> (4 * j)) & 15u;
        if (fast) {
          const uint32_t idx = c & 7u;
          const float base = ((idx & 1u) && idx > 1u) ? v : u;
          const float mag = idx ? base * __uint_as_float((uint32_t)((int)(idx >> 1) - 1 + (int)s) << 23) : 0.0f;
          o[j] = (c & 8u) ? -mag : mag;
        } else if (q.variant == NVFP4) {
          o[j] = deq_nvfp4(c, s, st);
        } else if (q.mant) {
          o[j] = deq_mbs(c, s, m8);
        } else {
          o[j] = deq_pow2(c, s);
        }
      }
      float4* o4 = reinterpret_cast<float4*>(op + 8 * w);
      __stcs(o4, make_float4(o[0], o[1], o[2], o[3]));
      __stcs(o4 + 1, make_float4(o[4], o[5], o[6], o[7]));
    }
  }
  if (bad) atomicOr(status, bad);
}

// ---------------------------------------------------------------------------
// Host launchers
// ---------------------------------------------------------------------------
static int grid_for(int64_t work, int threads) {
  int64_t g = (work + threads - 1) / threads;
  int64_t cap = (int64_t)num_sms() * 16;
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

static int macro_lanes(int macro) {
  int nblk = macro / 16, G = 1;
  while (G < nblk) G <<= 1;
  return G;
}

int launch_quantize(const void* x, int dtype, int64_t x_ld, const QDesc& q, int mbs_mode, const uint8_t* cand,
                    int n_cand, int augment, uint32_t* status, cudaStream_t st) {
  const int64_t rows = q.rows, cols = q.cols;
  const int64_t nbr16 = cols / 16;
  if (rows * nbr16 >= (int64_t)1 << 31) return set_error(ERR_UNSUPPORTED, "tensor too large (>= 2^31 blocks)");
  const bool bf = dtype == DT_BF16;
  // Row-tiled streaming grid (see k_stream_quant)
  const uint32_t nblk = (uint32_t)nbr16;
  const uint32_t tpr_n = (uint32_t)((nbr16 + SQ_THREADS - 1) / SQ_THREADS);
  const FastDiv tpr = make_fastdiv(tpr_n);  // tiles per row (row index = tile / tpr)
  const int64_t ntiles64 = rows * (int64_t)tpr_n;
  if (ntiles64 >= (int64_t)1 << 31) return set_error(ERR_UNSUPPORTED, "tensor too large");
  const uint32_t ntiles = (uint32_t)ntiles64;
#ifndef MXQ_SQ_CTAS
#define MXQ_SQ_CTAS 8
#endif
  const int sq_grid = (int)std::min<int64_t>((ntiles + SQ_UNROLL - 1) / SQ_UNROLL, (int64_t)num_sms() * MXQ_SQ_CTAS);
  // row-run launches: runs per row padded to a multiple of the MBS lane group
  const uint32_t runs_raw = (nblk + RUN - 1) / RUN;
#define UNIT_LAUNCH(VAR, G)                                                                                     \
  do {                                                                                                          \
    if (bf) k_stream_quant<DT_BF16, VAR, G><<<sq_grid, SQ_THREADS, 0, st>>>(x, x_ld, q, nblk, tpr, ntiles, status); \
    else k_stream_quant<DT_F32, VAR, G><<<sq_grid, SQ_THREADS, 0, st>>>(x, x_ld, q, nblk, tpr, ntiles, status);     \
  } while (0)
#define RUN_LAUNCH(VAR, UPM)                                                                                     \
  do {                                                                                                          \
    constexpr uint32_t GLV = (VAR == SQ_MBS_S && UPM > RUN) ? UPM / RUN : 1;                                    \
    const uint32_t rpr_n = (runs_raw + GLV - 1) / GLV * GLV;                                                    \
    const int64_t nr = rows * (int64_t)rpr_n;                                                                   \
    if (nr >= ((int64_t)1 << 31) - 32) return set_error(ERR_UNSUPPORTED, "tensor too large");                   \
    const int grid = (int)std::min<int64_t>((nr + 255) / 256, (int64_t)num_sms() * MXQ_SQ_CTAS);                \
    if (bf) k_quant_runs<DT_BF16, VAR, UPM><<<grid, 256, 0, st>>>(x, x_ld, q, nblk, make_fastdiv(rpr_n),       \
                                                                  (uint32_t)nr, status);                        \
    else k_quant_runs<DT_F32, VAR, UPM><<<grid, 256, 0, st>>>(x, x_ld, q, nblk, make_fastdiv(rpr_n),           \
                                                              (uint32_t)nr, status);                            \
  } while (0)
  switch (q.variant) {
    // OCP32 / MX16 / OAS: one 16-element unit per lane (k_stream_quant); MBS-S:
    // a run of four units per thread (k_quant_runs) -- the faster form of each
    // (quantizer section: measured unit / run / TMA-staged forms)
    case OCP32:
      UNIT_LAUNCH(SQ_OCP32, 2);
      break;
    case MX16:
      UNIT_LAUNCH(SQ_MX16, 1);
      break;
    case MX16_OAS:
      UNIT_LAUNCH(SQ_OAS, 1);
      break;
    case MBS_S:
    case MBS_D: {
      MacroGeom g;
      g.macro = q.macro_size;
      g.G = macro_lanes(q.macro_size);
      g.nmac = (cols + q.macro_size - 1) / q.macro_size;
      const int64_t ngroups = rows * g.nmac;
      if (q.variant == MBS_S && g.G * 16 == g.macro && g.G <= 128) {
        switch (g.G) {  // power-of-two macro of G units (runs of 4 units: up to 32 lanes per macro, 2048 elements)
          case 1: RUN_LAUNCH(SQ_MBS_S, 1); break;
          case 2: RUN_LAUNCH(SQ_MBS_S, 2); break;
          case 4: RUN_LAUNCH(SQ_MBS_S, 4); break;
          case 8: RUN_LAUNCH(SQ_MBS_S, 8); break;
          case 16: RUN_LAUNCH(SQ_MBS_S, 16); break;
          case 32: RUN_LAUNCH(SQ_MBS_S, 32); break;
          case 64: RUN_LAUNCH(SQ_MBS_S, 64); break;
          default: RUN_LAUNCH(SQ_MBS_S, 128); break;
        }
      } else if (g.G > 32) {
        return set_error(ERR_UNSUPPORTED, "this macro_size is not supported by the CUDA quantizer (MBS-S: powers of two up to 2048; otherwise up to 512)");
      } else if (q.variant == MBS_S) {
        const FastDiv fd = make_fastdiv((uint32_t)g.nmac);
        const int grid = grid_for(ngroups * g.G, 256);
        if (bf) k_quantize_mbs_s<DT_BF16><<<grid, 256, 0, st>>>(x, x_ld, q, g, fd, (uint32_t)ngroups, status);
        else k_quantize_mbs_s<DT_F32><<<grid, 256, 0, st>>>(x, x_ld, q, g, fd, (uint32_t)ngroups, status);
      } else {
        if (mbs_mode != 0) return set_error(ERR_INVALID, "mbs_mode='lut' runs through mxq_quantize_mbs_lut");
        if (n_cand < 1 || n_cand > 256) return set_error(ERR_INVALID, "candidate count out of range");
        if (!cand) return set_error(ERR_INVALID, "null candidate list");
        std::unique_ptr<MbsdTables> tab(new MbsdTables());
        memcpy(tab->cands, cand, (size_t)n_cand);
        const int64_t gpb = MBSD_THREADS / g.G;
        int64_t blocks = (ngroups + gpb - 1) / gpb;
        int64_t cap = (int64_t)num_sms() * 16;
        k_quantize_mbs_d<false><<<(int)(blocks < cap ? blocks : cap), MBSD_THREADS, 0, st>>>(
            x, dtype, x_ld, q, g, n_cand, augment, status, *tab);
      }
      break;
    }
    case NVFP4: {
      // pass 1 |x| max into status[1], pass 2 scales and codes (run form)
      cudaError_t e = cudaMemsetAsync(status + 1, 0, sizeof(uint32_t), st);
      if (e != cudaSuccess) return set_cuda_error(e);
      const uint32_t cpr_n = (nblk + CHUNK - 1) / CHUNK;
      const int64_t nch = rows * (int64_t)cpr_n;
      if (nch >= ((int64_t)1 << 31)) return set_error(ERR_UNSUPPORTED, "tensor too large");
      const int grid = (int)std::min<int64_t>((nch + 7) / 8, (int64_t)num_sms() * MXQ_SQ_CTAS);
      const FastDiv fr = make_fastdiv(cpr_n);
      const uint32_t nr = (uint32_t)nch;
      if (bf) {
        k_absmax_runs<DT_BF16><<<grid, 256, 0, st>>>(x, x_ld, nblk, fr, (uint32_t)nr, status);
        k_nvfp4_runs<DT_BF16><<<grid, 256, 0, st>>>(x, x_ld, q, nblk, fr, (uint32_t)nr, status + 1);
      } else {
        k_absmax_runs<DT_F32><<<grid, 256, 0, st>>>(x, x_ld, nblk, fr, (uint32_t)nr, status);
        k_nvfp4_runs<DT_F32><<<grid, 256, 0, st>>>(x, x_ld, q, nblk, fr, (uint32_t)nr, status + 1);
      }
      break;
    }
    default:
      return set_error(ERR_INVALID, "unknown variant");
  }
  return check_launch();
}

int launch_quantize_lut(const void* x, int dtype, int64_t x_ld, const QDesc& q, const uint8_t* cand, int n_cand,
                        const float* lut, uint32_t* status, cudaStream_t st) {
  if (q.variant != MBS_D) return set_error(ERR_INVALID, "lut mode applies to MBS_D only");
  if (n_cand != 16) return set_error(ERR_INVALID, "the lookup table holds exactly 16 candidates");
  MacroGeom g;
  g.macro = q.macro_size;
  g.G = macro_lanes(q.macro_size);
  g.nmac = (q.cols + q.macro_size - 1) / q.macro_size;
  if (g.G > 32) return set_error(ERR_UNSUPPORTED, "macro_size > 512 is not supported by the CUDA quantizer");
  std::unique_ptr<MbsdTables> tab(new MbsdTables());
  memcpy(tab->cands, cand, 16);
  memcpy(tab->lut, lut, sizeof(tab->lut));
  const int64_t ngroups = q.rows * g.nmac;
  const int64_t gpb = MBSD_THREADS / g.G;
  int64_t blocks = (ngroups + gpb - 1) / gpb;
  int64_t cap = (int64_t)num_sms() * 16;
  k_quantize_mbs_d<true><<<(int)(blocks < cap ? blocks : cap), MBSD_THREADS, 0, st>>>(x, dtype, x_ld, q, g, 16, 0,
                                                                                     status, *tab);
  return check_launch();
}

int launch_dequantize(const QDesc& q, float* out, int64_t out_ld, uint32_t* status, cudaStream_t st) {
  const int64_t nb = q.rows * (q.cols / q.block_size);
  if (nb >= ((int64_t)1 << 31)) return set_error(ERR_UNSUPPORTED, "tensor too large (>= 2^31 blocks)");
  k_dequantize<<<grid_for(nb, 256), 256, 0, st>>>(q, out, out_ld, make_fastdiv((uint32_t)(q.cols / q.block_size)),
                                                  (uint32_t)nb, status);
  return check_launch();
}

}  // namespace mxq
