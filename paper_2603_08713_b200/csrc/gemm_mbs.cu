// gemm_mbs.cu -- tcgen05 MBS GEMM (K8) for sm_100a.   C[M,N] = A[M,K] . B[N,K]^T
//
// Replaces matmul_quantized (src/gemm.py:137-172) for operand pairs where at
// least one side carries the MBS macro factor sigma = 1/(1+m8/256) per (row,
// macro of 128 K) (src/quantize.py:383-406; per-chunk semantics SPEC.md:325;
// the paper's Appendix E epilogue).  sigma is not a power of
// two, so it cannot ride in the UE8M0 block scales of the block-scaled MMA:
// every macro chunk is MMA'd (kind::mxf4nvf4.block16, UE8M0) into its own
// TMEM partial buffer P and the epilogue folds acc += (sigmaA_i*sigmaB_j) * P_ij
// in registers, two FP32 operations per output per chunk.
//
// That FP32 work bounds the kernel: 128 FP32 lanes/clk/SM against 16384 FP4
// MACs/clk/SM means 2*BM*BN/128 cycles of FP32 per chunk versus BM*BN*128/16384
// of MMA -- the tensor pipe can be at most 50 % busy:
//   * 128 x 192 tiles, N=192 MMAs (96 cycles each, long enough to hide the
//     issuing thread's ~70-cycle per-MMA cost that made N=128 MMAs issue-bound),
//     two 192-column TMEM partial buffers and two 64-column-aligned
//     scale-factor buffers (384 + 2*64 columns <= 512);
//   * scale factors reach TMEM by tcgen05.cp from the MMA warp, in order with
//     the MMAs: the tensor pipe has the slack, the epilogue does not;
//   * 16 epilogue warps (4 per TMEM lane quadrant, 48 columns each) hold the
//     48 f32 accumulators and load a chunk's whole partial before releasing its
//     TMEM buffer; setmaxnreg gives them 112 registers and the 4 control warps
//     32 (the pool is the 96 x 640 registers allocated at launch);
//   * clusters of 2 CTAs share the B tile by TMA multicast;
//   * few-tile shapes (small M: decode / expert GEMMs) split K over CTAs at
//     stage boundaries, write f32 partials and sum them in a fixed order
//     (k_splitk_reduce), so every SM streams weights.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <type_traits>

#include "mxq_arith.cuh"
#include "mxq_internal.h"
#include "sq_dev.cuh"
#include "tc_ptx.cuh"

namespace mxq {
constexpr int KSTEP_MBS = 64;
namespace mbs {

using namespace tc;

constexpr int BM = 128;
constexpr int KSTAGE = 256, KSTEP = 64;     // K elements per pipeline stage / per MMA
#ifndef MXQ_NSIG
#define MXQ_NSIG 8
#endif
constexpr int NSFB = 2, NSIG = MXQ_NSIG;
constexpr int ATOM = 512;                   // SF atom: 128 rows x 4 blocks of 16
constexpr int STAGE_A = BM * KSTAGE / 2;    // 16 KB of A codes per stage
constexpr int SFA_BYTES = 4 * ATOM;         // 4 k-steps
// Tile shape (BN output columns, NB TMEM partial buffers, EPIW epilogue
// warps).  The product path is <192, 2, 16> (DESIGN.md section 3.4 lists the
// measured alternatives).
template <int BN_, int NB_, int EPIW_>
struct MbsCfg {
  static constexpr int BN = BN_, NB = NB_;
  static constexpr int EPIW = EPIW_;                    // epilogue warps (EPIW/4 per TMEM lane quadrant)
  static constexpr int W_TMA = EPIW, W_MMA = EPIW + 1;  // control warpgroup after them
  static constexpr int THREADS = (EPIW + 4) * 32;
  static constexpr int COLS = BN / (EPIW / 4);          // output columns per epilogue thread
  static constexpr int NRB = BN / 128 + (BN % 128 ? 1 : 0);  // 128-row SF atoms a tile can touch
  static constexpr int STAGES = BN > 128 ? 4 : (BN > 64 ? 5 : (BN > 16 ? 7 : 10));  // narrow (decode) tiles: deeper weight prefetch
  static constexpr int STAGE_B = BN * KSTAGE / 2;
  static constexpr int SFB_BYTES = NRB * 4 * ATOM;     // NRB row blocks x 4 k-steps
  static constexpr int SIG_SLOT = (BM + BN) * 4;       // sigmaA[128] + sigmaB[BN], f32
  static constexpr int OFF_A = 0;
  static constexpr int OFF_B = OFF_A + STAGES * STAGE_A;
  static constexpr int OFF_SFA = OFF_B + STAGES * STAGE_B;
  static constexpr int OFF_SFB = OFF_SFA + STAGES * SFA_BYTES;
  static constexpr int OFF_SIG = OFF_SFB + STAGES * SFB_BYTES;
  static constexpr int OFF_BAR = OFF_SIG + NSIG * SIG_SLOT;
  static constexpr int NUM_BARS = 2 * STAGES + 2 * NB + 2 * NSIG + NSFB;
  static constexpr int SMEM = OFF_BAR + NUM_BARS * 8 + 16 + 1024;  // + alignment slack
  // TMEM: partial buffers [0, NB*BN), SF buffers 64-aligned after them
  // (misaligned SF addresses slow the MMA, tools/microbench_mma3.cu).  Within
  // an SF buffer: SFA of k-step j at +4j, SFB (NRB 128-row atoms) at +16+4*NRB*j.
  static constexpr int COL_SF0 = (NB * BN + 63) / 64 * 64;
  static constexpr int SF_STRIDE = 64;
  // EPIW*32*EPI + 4*32*CTRL must fit the registers allocated at launch
  // (ptxas' per-thread count x THREADS: 96 x 640 for 16 epilogue warps,
  // 168 x 384 for 8) -- setmaxnreg.inc blocks forever otherwise
#ifndef MXQ_NO_SETMAXNREG
  static constexpr bool SETMAXNREG = COLS > 32 && EPIW > 4;
#else
  static constexpr bool SETMAXNREG = false;
#endif
  static constexpr int EPI_REGS = EPIW == 16 ? 112 : 208, CTRL_REGS = EPIW == 16 ? 32 : 48;
  // per-thread register cap at launch: the whole file fits 64K registers
  static constexpr int MAXNREG = EPIW == 16 ? 96 : (THREADS * 168 <= 65536 ? 168 : (65536 / THREADS) & ~7);
  static_assert(!SETMAXNREG || EPIW * 32 * EPI_REGS + 4 * 32 * CTRL_REGS <= MAXNREG * THREADS, "register pool");
  static_assert(SMEM <= 232448, "shared memory budget");
  static_assert(OFF_B % 1024 == 0 && STAGE_B % 1024 == 0 && (BN / 2) * 128 % 1024 == 0, "128B-swizzle alignment");
  static_assert(COL_SF0 + NSFB * SF_STRIDE <= 512, "TMEM budget");
  static_assert(16 + 4 * NRB * 4 <= SF_STRIDE, "SF buffer");
};

struct Params {
  const uint8_t* sfa;  // scale-factor atoms [rows/128][sf_kg][512]
  const uint8_t* sfb;
  int64_t sfa_kg, sfb_kg;
  int sfb_rb;          // allocated 128-row blocks of B's SF atoms
  const float* sga;    // sigma^T (n_macros, ld) f32; a non-MBS side points at a ones row with ld 0
  const float* sgb;
  int64_t sga_ld, sgb_ld;
  void* c;
  int64_t ldc;
  int M, N, K;
  int mac_steps;       // macro size / 64 (1, 2 or 4: chunks never straddle a 256-K stage)
  int n_chunks;        // macros per row
  int ksplit;          // K splits (stage-aligned); > 1: f32 partials to ws[split][M][ws_ld]
  const double* tsa;   // NVFP4 tensor scales (UE4M3 pairs): C *= s_tA s_tB at the store, else null
  const double* tsb;
  float* ws;
  int64_t ws_ld;
  uint32_t idesc;
  long long* trace;    // clock64 trace of CTA 0 (MXQ_GEMM_TRACE builds only)
  // FUSED: the bf16 activation xa (M x K, row pitch xa_ld elements) is
  // quantized (MBS-S) inside the launch into qa -- the buffers sfa / sga / the
  // A tensor map point at -- and ready[mb] is set once 128-row block mb is out.
  const void* xa;
  int64_t xa_ld;
  QDesc qa;
  uint32_t* ready;     // slices published (zeroed before the launch)
  uint32_t* status;
};

// Grouped launch (GPT-OSS-style expert GEMMs, SURVEY section 8 d config 5): up
// to MAXG independent decode-sized GEMMs of one shape in ONE launch, swap-AB
// form (weights on the MMA's M side).  Per group: the two tensor maps and the
// operand / output pointers; everything else is shared (GroupTable::p).  The
// table travels as a __grid_constant__ kernel parameter (param space, no
// device allocation, graph-capturable).
constexpr int MAXG = 64;
struct GroupDesc {
  CUtensorMap tmA, tmB;  // weights (kernel A), tokens (kernel B)
  const uint8_t* sfa;
  const uint8_t* sfb;
  const float* sga;
  const float* sgb;
  int64_t sgb_ld;
  void* c;
  int n;                 // kernel N of this group (tokens, swap-AB form)
  int m;                 // kernel M of this group (tokens, direct form)
  const double* tsa;     // NVFP4 groups: the two tensor scales (s_t of each operand), else null
  const double* tsb;
};
struct GroupTable {
  Params p;
  int n_groups;
  GroupDesc g[MAXG];
};

#ifndef MXQ_GEMM_TRACE
#define MXQ_GEMM_TRACE 0
#endif
// 16 clock64 slots per chunk of CTA 0, first 512 chunks (tools/trace_mbs.py).
__device__ __forceinline__ void trace_at(const Params& p, uint32_t chunk, int slot) {
  if constexpr (MXQ_GEMM_TRACE != 0) {
    if (p.trace != nullptr && blockIdx.x == 0 && chunk < 512 && (threadIdx.x & 31) == 0)
      p.trace[chunk * 16 + slot] = clock64();
  }
}
template <int R>
__device__ __forceinline__ void setmaxnreg_inc() { asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(R)); }
template <int R>
__device__ __forceinline__ void setmaxnreg_dec() { asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(R)); }

__device__ __forceinline__ void mbar_init_a(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ uint32_t ld_shared_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void sf_cp_e(uint32_t tmem_col, uint32_t saddr) {
  const uint64_t d = smem_desc(saddr, 0, 128, 0);  // 32 rows x 16 B, 8-row core matrices 128 B apart
  asm volatile(MXQ_ELECT "tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;\n\t}" ::"r"(tmem_col), "l"(d) : "memory");
}
// Start a 16-column TMEM load without waiting (the caller waits once for all).
__device__ __forceinline__ void tmem_ld16_nw(uint32_t taddr, float* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
}

// Pin values produced by tcgen05.ld behind tcgen05.wait::ld: the arithmetic
// below is ordinary (non-volatile) asm/C++ that the compiler could otherwise
// hoist above the wait.
template <int N>
__device__ __forceinline__ void reg_fence(float* v) {
#pragma unroll
  for (int i = 0; i < N; i += 8)
    asm volatile("" : "+f"(v[i]), "+f"(v[i + 1]), "+f"(v[i + 2]), "+f"(v[i + 3]), "+f"(v[i + 4]), "+f"(v[i + 5]),
                 "+f"(v[i + 6]), "+f"(v[i + 7]));
}

// Fused MBS-S quantization of A: A's rows are cut into
// slices of FQ_ROWS rows that the running CTAs CLAIM from a work counter
// (p.ready[1], zeroed before the launch) FQ_CLAIM slices at a time, so all
// SMs stream the activation; each warp takes 32-unit row segments, U in
// flight, through the same sq_unit as the standalone k_stream_quant, so codes
// / scales / mantissas / sigma are bit-identical to mxq_quantize.  A finished
// batch is published with generic stores -> proxy fence -> CTA barrier ->
// release add on the slice counter p.ready[0]; the TMA warp acquires the full
// count before its first load.  Only CTAs that are running claim slices, so
// the wait cannot deadlock when the grid is not fully co-resident (MPS limits,
// green contexts, a concurrent kernel holding SMs): the running CTAs quantize
// every slice themselves.
constexpr int FQ_ROWS = 8, FQ_CLAIM = 2;
#ifndef MXQ_FQ_U
#define MXQ_FQ_U 2
#endif
template <int G, int THREADS>
__device__ __forceinline__ void fused_quant_a(const Params& p, const float* sig_tab, uint32_t* claim_slot) {
  constexpr int NW = THREADS / 32, U = MXQ_FQ_U;
  const int warp = threadIdx.x >> 5;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t nblk = (uint32_t)p.K / 16, segs = (nblk + 31) / 32;
  const uint32_t nslices = (uint32_t)(p.M + FQ_ROWS - 1) / FQ_ROWS;
  const uint32_t per_slice = FQ_ROWS * segs;
  uint32_t bad = 0, ovf = 0;
  for (;;) {
    if (threadIdx.x == 0) *claim_slot = atomicAdd(p.ready + 1, (uint32_t)FQ_CLAIM);
    __syncthreads();
    const uint32_t first = *claim_slot;
    __syncthreads();
    if (first >= nslices) break;
    const uint32_t mine = min((uint32_t)FQ_CLAIM, nslices - first);
    const uint32_t nseg = mine * per_slice;
    for (uint32_t s0 = warp; s0 < nseg; s0 += U * NW) {
      Blk16<DT_BF16> xb[U];
      uint32_t rr[U], kk[U];
      bool live[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t j = s0 + u * NW;
        const uint32_t js = j / per_slice, jr = j - js * per_slice;
        const uint32_t rl = jr / segs;
        rr[u] = (first + js) * FQ_ROWS + rl;
        kk[u] = (jr - rl * segs) * 32 + lane;
        live[u] = j < nseg && rr[u] < (uint32_t)p.M;
        if (live[u] && kk[u] < nblk) ld_blk<DT_BF16>(p.xa, (int64_t)rr[u] * p.xa_ld + kk[u] * 16, xb[u]);
        else zero_blk<DT_BF16>(xb[u]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (live[u])
          sq_unit<DT_BF16, SQ_MBS_S, G>(xb[u], kk[u] < nblk, row_out(p.qa, rr[u]), p.qa.sig_t_ld, kk[u], lane,
                                        sig_tab, bad, ovf);
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p.ready), "r"(mine) : "memory");
    }
  }
  if (bad) atomicOr(p.status, ST_NONFINITE);
  if (ovf) atomicOr(p.status, ST_OVERFLOW);
}

__device__ __forceinline__ void wait_ready(const uint32_t* flag, uint32_t want) {
  uint32_t v;
  for (;;) {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if (v >= want) break;
    __nanosleep(64);
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// TRANS: swap-AB for decode-sized M -- the kernel's A operand is the weight
// matrix (128 weight rows per tile) and its B operand the few activation rows
// (BN >= M), so the output tile is stored transposed into C[token][n].
template <int BN_, int NB_, int EPIW_, bool OUT_BF16, int CL, bool TRANS, bool FUSED, bool GROUPED>
__device__ __forceinline__ void mbs_body(const CUtensorMap* tmA, const CUtensorMap* tmB, const Params& p,
                                         const GroupTable* gt) {
  using C = MbsCfg<BN_, NB_, EPIW_>;
  constexpr int EPIW = C::EPIW, W_TMA = C::W_TMA, W_MMA = C::W_MMA;
  constexpr int BN = C::BN, NB = C::NB, STAGES = C::STAGES, COLS = C::COLS, NRB = C::NRB;
  constexpr int STAGE_B = C::STAGE_B, SFB_BYTES = C::SFB_BYTES, SIG_SLOT = C::SIG_SLOT;
  constexpr int OFF_A = C::OFF_A, OFF_B = C::OFF_B, OFF_SFA = C::OFF_SFA, OFF_SFB = C::OFF_SFB;
  constexpr int OFF_SIG = C::OFF_SIG, OFF_BAR = C::OFF_BAR, COL_SF0 = C::COL_SF0, SF_STRIDE = C::SF_STRIDE;
  extern __shared__ uint8_t smem_raw[];
  // 32-bit shared-window addresses only (a generic 64-bit base gets
  // rematerialised inside the hot loops under register pressure).
  const uint32_t a_smem = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t a_full = a_smem + OFF_BAR, a_empty = a_full + 8 * STAGES;
  const uint32_t a_tfull = a_empty + 8 * STAGES, a_tempty = a_tfull + 8 * NB;
  const uint32_t a_sfull = a_tempty + 8 * NB, a_sempty = a_sfull + 8 * NSIG;
  const uint32_t a_sffree = a_sempty + 8 * NSIG;  // [NSFB] TMEM SF buffer consumed (its stage's MMAs done)
  const uint32_t a_tmem_slot = a_sffree + 8 * NSFB;

  if constexpr (FUSED) {
    // phase 1: quantize this CTA's A row blocks (sigma table in the sigma ring's space)
    float* sig_tab = reinterpret_cast<float*>(smem_raw + (a_smem - smem_u32(smem_raw)) + OFF_SIG);
    for (int i = threadIdx.x; i < 256; i += C::THREADS) sig_tab[i] = 1.0f / mbs_factor((uint32_t)i);
    uint32_t* claim_slot = reinterpret_cast<uint32_t*>(sig_tab + 256);
    __syncthreads();
    if (p.mac_steps == 1) fused_quant_a<4, C::THREADS>(p, sig_tab, claim_slot);
    else if (p.mac_steps == 2) fused_quant_a<8, C::THREADS>(p, sig_tab, claim_slot);
    else fused_quant_a<16, C::THREADS>(p, sig_tab, claim_slot);
    // (the sigma ring is rewritten by bulk copies: order the generic writes first)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
  }

  // warp index through a shuffle so ptxas knows it is warp-uniform
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int tiles_m = (p.M + BM - 1) / BM, tiles_n = (p.N + BN - 1) / BN;
  const int groups_m = (tiles_m + CL - 1) / CL;
  const int ksplit = p.ksplit;
  const int upg = groups_m * tiles_n * ksplit;  // units per group
  const int num_units = GROUPED ? gt->n_groups * upg : upg;
  const int unit0 = blockIdx.x / CL, unit_step = gridDim.x / CL;
  uint32_t crank = 0;
  if constexpr (CL > 1) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  const int n_ksteps = (p.K + KSTEP - 1) / KSTEP;
  const int n_stages = (p.K + KSTAGE - 1) / KSTAGE;
  const int n_chunks = p.n_chunks, mac_steps = p.mac_steps;
  const int cps = mac_steps <= 4 ? 4 / mac_steps : 0;       // chunks per 256-K stage (split-K shapes only)
  const int spl = (n_stages + ksplit - 1) / ksplit;         // stages per K split
  // A work unit: one (128-row group, BN-column tile, K split) of the output;
  // the CTAs of a cluster take consecutive 128-row blocks of it.
  struct Unit { int g, mb, nb, split, s_lo, s_hi, c_lo, c_hi; };
  auto unit_of = [&](int u) {
    Unit r;
    r.g = GROUPED ? u / upg : 0;
    u -= r.g * upg;
    r.split = u % ksplit;
    const int rest = u / ksplit;
    r.mb = (rest % groups_m) * CL + (int)crank;
    r.nb = rest / groups_m;
    r.s_lo = r.split * spl;
    r.s_hi = min(r.s_lo + spl, n_stages);
    // (K splits only when chunks tile the 256-K stages: macro 64 / 128 / 256)
    r.c_lo = ksplit > 1 ? r.s_lo * cps : 0;
    r.c_hi = ksplit > 1 ? min(r.s_hi * cps, n_chunks) : n_chunks;
    return r;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init_a(a_full + 8 * s, 1);
      mbar_init_a(a_empty + 8 * s, CL);
    }
    for (int b = 0; b < NB; ++b) {
      mbar_init_a(a_tfull + 8 * b, 1);
      mbar_init_a(a_tempty + 8 * b, EPIW);
    }
    for (int b = 0; b < NSIG; ++b) {
      mbar_init_a(a_sfull + 8 * b, 1);
      mbar_init_a(a_sempty + 8 * b, EPIW);
    }
    for (int b = 0; b < NSFB; ++b) mbar_init_a(a_sffree + 8 * b, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if constexpr (!GROUPED) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmA)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmB)) : "memory");
    }
  }
  if (warp == W_MMA) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(a_tmem_slot) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CL > 1) cluster_sync();
  tc_fence_after();
  const uint32_t tmem = ld_shared_u32(a_tmem_slot);

  if (warp >= EPIW) {
    if constexpr (C::SETMAXNREG) setmaxnreg_dec<C::CTRL_REGS>();
    if (warp == W_TMA) {
      // ===================== TMA producer =====================
      // (fused: A is complete once every slice is published -- the first wave
      // of tiles covers every row block, so one wait before the loop costs
      // nothing and keeps the 32-register producer loop free of spills)
      if constexpr (FUSED) wait_ready(p.ready, (uint32_t)((p.M + FQ_ROWS - 1) / FQ_ROWS));
      uint32_t st = 0, ph = 0, slot = 0, sph = 0;
      uint32_t tq = 0, tsq = 0;  // (trace only)
      for (int unit = unit0; unit < num_units; unit += unit_step) {
        const Unit U = unit_of(unit);
        const int m0 = U.mb * BM, n0 = U.nb * BN;
        const int rb0 = n0 / 128;
        const int nrb = (rb0 + NRB <= p.sfb_rb) ? NRB : p.sfb_rb - rb0;
        const uint32_t tx = STAGE_A + STAGE_B + SFA_BYTES + nrb * 4 * ATOM;
        const uint8_t* sfa0 = p.sfa;
        const uint8_t* sfb0 = p.sfb;
        const float* sga0 = p.sga;
        const float* sgb0 = p.sgb;
        int64_t sgb_ld = p.sgb_ld;
        if constexpr (GROUPED) {
          const GroupDesc& G = gt->g[U.g];
          sfa0 = G.sfa;
          sfb0 = G.sfb;
          sga0 = G.sga;
          sgb0 = G.sgb;
          sgb_ld = G.sgb_ld;
        }
        const uint8_t* sa = sfa0 + (int64_t)U.mb * p.sfa_kg * ATOM;
        const uint8_t* sb = sfb0 + (int64_t)rb0 * p.sfb_kg * ATOM;
        const float* ga = sga0 + (p.sga_ld ? m0 : 0);
        const float* gb = sgb0 + (sgb_ld ? n0 : 0);
        int sb_bytes = BN * 4;
        if (sgb_ld && sgb_ld - n0 < BN) sb_bytes = (int)(sgb_ld - n0) * 4;
        int chunk = U.c_lo;
        for (int s = U.s_lo; s < U.s_hi; ++s) {
          const uint32_t fb = a_full + st * 8;
          // (grouped: the maps are re-derived per stage from the unit's group
          // index -- param-space addresses -- to keep the producer loop within
          // its 32 registers)
          const CUtensorMap* mA = GROUPED ? &gt->g[U.g].tmA : tmA;
          const CUtensorMap* mB = GROUPED ? &gt->g[U.g].tmB : tmB;
          trace_at(p, tsq, 13);
          mbar_wait_a(a_empty + st * 8, ph ^ 1);
          trace_at(p, tsq++, 14);
          expect_tx_e(fb, tx);
          tma_load_2d_e(a_smem + OFF_A + st * STAGE_A, mA, fb, s * (KSTAGE / 2), m0);
          if constexpr (CL == 1) {
            tma_load_2d_e(a_smem + OFF_B + st * STAGE_B, mB, fb, s * (KSTAGE / 2), n0);
          } else {
            tma_load_2d_mc_e(a_smem + OFF_B + st * STAGE_B + crank * (BN / CL) * (KSTAGE / 2), mB, fb,
                             s * (KSTAGE / 2), n0 + (int)crank * (BN / CL), (uint16_t)((1u << CL) - 1));
          }
          bulk_load_e(a_smem + OFF_SFA + st * SFA_BYTES, sa + (int64_t)s * SFA_BYTES, SFA_BYTES, fb);
          for (int r = 0; r < nrb; ++r)
            bulk_load_e(a_smem + OFF_SFB + st * SFB_BYTES + r * 4 * ATOM,
                        sb + ((int64_t)r * p.sfb_kg + (int64_t)s * 4) * ATOM, 4 * ATOM, fb);
          if (++st == STAGES) { st = 0; ph ^= 1; }
          // sigma slices of the chunks that start in this stage
          while (chunk < U.c_hi && chunk * mac_steps < 4 * (s + 1)) {
            const uint32_t sfb = a_sfull + slot * 8;
            trace_at(p, tq, 11);
            mbar_wait_a(a_sempty + slot * 8, sph ^ 1);
            trace_at(p, tq++, 12);
            expect_tx_e(sfb, BM * 4 + sb_bytes);
            const uint32_t dst = a_smem + OFF_SIG + slot * SIG_SLOT;
            bulk_load_e(dst, ga + (int64_t)chunk * p.sga_ld, BM * 4, sfb);
            bulk_load_e(dst + BM * 4, gb + (int64_t)chunk * sgb_ld, sb_bytes, sfb);
            if (++slot == NSIG) { slot = 0; sph ^= 1; }
            ++chunk;
          }
        }
      }
    } else if (warp == W_MMA) {
      // ===================== MMA issuer =====================
      uint32_t g = 0;             // stages consumed (SF buffer parity)
      uint32_t buf = 0, tph = 0;  // TMEM partial-buffer ring
      uint32_t st = 0;            // smem ring position
      uint32_t q = 0;             // chunks issued (trace only)
      for (int unit = unit0; unit < num_units; unit += unit_step) {
        const Unit U = unit_of(unit);
        const uint32_t sfb_shift = ((U.nb * BN) % 128) ? 2u : 0u;  // odd 192-tiles start 64 rows into the atom
        int ks = U.s_lo * 4;
        uint64_t adesc = 0, bdesc = 0;
        uint32_t sfa_col = 0;
        for (int c = U.c_lo; c < U.c_hi; ++c, ++q) {
          const uint32_t dcol = tmem + buf * BN;
          trace_at(p, q, 0);
          mbar_wait_a(a_tempty + buf * 8, tph ^ 1u);
          trace_at(p, q, 1);
          tc_fence_after();
          int kend = (c + 1) * mac_steps;
          if (kend > n_ksteps) kend = n_ksteps;
          const int kbeg = ks;
          for (; ks < kend; ++ks) {
            const uint32_t j = (uint32_t)ks & 3u;
            if (j == 0) {
              // this stage's SF atoms -> SF buffer g % 2.  Its previous
              // readers are stage g-2's MMAs: tcgen05.cp is NOT ordered after
              // an earlier tcgen05.mma's scale-factor reads (measured: stale
              // scales in a few column groups at the Llama qkv shape when the
              // MMA issue runs a stage ahead), so wait for their commit.
              sfa_col = tmem + COL_SF0 + (g & (NSFB - 1)) * SF_STRIDE;
#ifndef MXQ_NO_SFFREE
              if (g >= NSFB) mbar_wait_a(a_sffree + (g & (NSFB - 1)) * 8, ((g / NSFB) - 1) & 1u);
#endif
              trace_at(p, q, 15);
              mbar_wait_a(a_full + st * 8, (g / STAGES) & 1u);
              trace_at(p, q, 10);
              tc_fence_after();
#pragma unroll
              for (int jj = 0; jj < 4; ++jj) {
                sf_cp_e(sfa_col + 4 * jj, a_smem + OFF_SFA + st * SFA_BYTES + jj * ATOM);
#pragma unroll
                for (int r = 0; r < NRB; ++r)
                  sf_cp_e(sfa_col + 16 + 4 * NRB * jj + 4 * r, a_smem + OFF_SFB + st * SFB_BYTES + r * 4 * ATOM + jj * ATOM);
              }
              adesc = operand_desc(a_smem + OFF_A + st * STAGE_A);
              bdesc = operand_desc(a_smem + OFF_B + st * STAGE_B);
            }
            mma_bs_e<false>(dcol, adesc + (uint64_t)(j * 2), bdesc + (uint64_t)(j * 2), p.idesc, ks > kbeg ? 1u : 0u,
                            sfa_col + 4 * j, sfa_col + 16 + 4 * NRB * j + sfb_shift);
            if (j == 3 || ks + 1 == n_ksteps) {
              if constexpr (CL == 1) tc_commit_e(a_empty + st * 8);
              else tc_commit_mc_e(a_empty + st * 8, (uint16_t)((1u << CL) - 1));
              tc_commit_e(a_sffree + (g & (NSFB - 1)) * 8);
              ++g;
              if (++st == STAGES) st = 0;
            }
          }
          tc_commit_e(a_tfull + buf * 8);
          trace_at(p, q, 2);
          if (++buf == NB) { buf = 0; tph ^= 1; }
        }
      }
    }
  } else {
    // ===================== epilogue (warps 0..EPIW-1) =====================
    if constexpr (C::SETMAXNREG) setmaxnreg_inc<C::EPI_REGS>();
    const int quad = warp & 3, grp = warp >> 2;  // TMEM lane quadrant, column group
    const uint32_t t_ld = tmem + ((uint32_t)(quad * 32) << 16) + grp * COLS;
    const int row_in_tile = quad * 32 + lane;
    const uint32_t sig_a = a_smem + OFF_SIG + row_in_tile * 4;
    const uint32_t sig_b = a_smem + OFF_SIG + (BM + grp * COLS) * 4;
    uint32_t q = 0;  // chunks consumed by this warp (all units)
    // The sigma slot read by the previous chunk is released one chunk late: the
    // SASS scheduler hoists an mbarrier.arrive above the FMULs that consume
    // the slot's LDS results (nothing in PTX ties them), and an LDS still in
    // flight then reads the producer's refill (measured: sigma_B columns 24-47
    // of the slowest warps at the Llama qkv shape).  One chunk later every
    // FMUL of the previous fold has issued -- so every LDS has returned (in-order
    // issue, register scoreboard) -- before the arrive can issue.

    for (int unit = unit0; unit < num_units; unit += unit_step) {
      const Unit U = unit_of(unit);
      const int row = U.mb * BM + row_in_tile;
      const int col0 = U.nb * BN + grp * COLS;
      float acc[COLS];
#pragma unroll
      for (int i = 0; i < COLS; ++i) acc[i] = 0.0f;
      // One chunk.  J >= 0: position J of an NSIG-aligned block of chunks
      // (q % NSIG == J), so the TMEM buffer, its phase and the sigma slot are
      // compile-time constants and only the sigma phase (one bit per block)
      // is a register; J < 0: any position (indices from q).
      auto chunk_step = [&](auto JC) {
        constexpr int J = decltype(JC)::value;
        const uint32_t b = J >= 0 ? (uint32_t)(J & (NB - 1)) : (q & (NB - 1));
        const uint32_t tp = (q / NB) & 1u;  // (q == block start + J in an aligned block)
        const uint32_t sl = J >= 0 ? (uint32_t)J : (q & (NSIG - 1));
        const uint32_t sp = (q / NSIG) & 1u;
        // the chunk's partial: load all of it, then release the TMEM buffer
        if (warp == 0) trace_at(p, q, 3);
        mbar_wait_a(a_tfull + b * 8, tp);
        if (warp == 0) trace_at(p, q, 4);
        if (warp == EPIW - 1) trace_at(p, q, 8);
        tc_fence_after();
        float v[COLS];
#pragma unroll
        for (int h = 0; h < COLS / 16; ++h) tmem_ld16_nw(t_ld + b * BN + h * 16, v + h * 16);
        tmem_wait_ld();
        reg_fence<COLS>(v);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive_a(a_tempty + b * 8);
          // the previous chunk's sigma slot (released one chunk late, see above)
          if (J > 0 || q != 0) mbar_arrive_a(a_sempty + ((sl - 1) & (NSIG - 1)) * 8);
        }
        if (warp == 0) trace_at(p, q, 5);
        // acc += (sigmaA * sigmaB_j) * P_j   (FMUL2 + FFMA2)
        mbar_wait_a(a_sfull + sl * 8, sp);
        if (warp == 0) trace_at(p, q, 6);
        const uint32_t so = sl * SIG_SLOT;
        const float sa = ld_shared_f32(sig_a + so);
#pragma unroll
        for (int i = 0; i < COLS; i += 4) {
          const float4 sb = ld_shared_f32x4(sig_b + so + i * 4);
          float w0, w1, w2, w3;
          mul2(w0, w1, sa, sb.x, sb.y);
          mul2(w2, w3, sa, sb.z, sb.w);
          fma2(acc[i], acc[i + 1], w0, w1, v[i], v[i + 1]);
          fma2(acc[i + 2], acc[i + 3], w2, w3, v[i + 2], v[i + 3]);
        }
        if (warp == 0) trace_at(p, q, 7);
        if (warp == EPIW - 1) trace_at(p, q, 9);
        ++q;
      };
      int c = U.c_lo;
      constexpr bool UNROLL8 = true;
#pragma unroll 1
      while (c < U.c_hi && (!UNROLL8 || (q & (NSIG - 1)))) { chunk_step(std::integral_constant<int, -1>{}); ++c; }
#pragma unroll 1
      for (; c + NSIG <= U.c_hi; c += NSIG) {
        static_assert(NSIG == 8, "the aligned block below is written for eight sigma slots");
        chunk_step(std::integral_constant<int, 0>{});
        chunk_step(std::integral_constant<int, 1>{});
        chunk_step(std::integral_constant<int, 2>{});
        chunk_step(std::integral_constant<int, 3>{});
        chunk_step(std::integral_constant<int, 4>{});
        chunk_step(std::integral_constant<int, 5>{});
        chunk_step(std::integral_constant<int, 6>{});
        chunk_step(std::integral_constant<int, 7>{});
      }
#pragma unroll 1
      for (; c < U.c_hi; ++c) chunk_step(std::integral_constant<int, -1>{});
      // store the tile row (masked to M x N): the output, or this split's f32 partial
      void* const cout = GROUPED ? gt->g[U.g].c : p.c;
      const int n_out = GROUPED ? gt->g[U.g].n : p.N;
      {
        // NVFP4 / UE4M3 pairs: C = s_tA s_tB (sum of the UE4M3-scaled products),
        // the plain NVFP4 kernel's epilogue (src/quantize.py:409-423 applies s_t
        // per element); a side without a tensor scale contributes 1
        const double* ta = GROUPED ? gt->g[U.g].tsa : p.tsa;
        const double* tb = GROUPED ? gt->g[U.g].tsb : p.tsb;
        if (ta || tb) {
          const float ts = (float)((ta ? *ta : 1.0) * (tb ? *tb : 1.0));
#pragma unroll
          for (int i = 0; i < COLS; ++i) acc[i] *= ts;
        }
      }
      if (TRANS && row < p.M) {
        // kernel row = weight row n, kernel column = token: C[token][n] (and the
        // split partials in the same output orientation)
        if (ksplit > 1) {
          float* out = p.ws + ((int64_t)U.split * n_out + col0) * p.ws_ld + row;
#pragma unroll
          for (int i = 0; i < COLS; ++i)
            if (col0 + i < n_out) out[(int64_t)i * p.ws_ld] = acc[i];
        } else if constexpr (OUT_BF16) {
          __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(cout) + (int64_t)col0 * p.ldc + row;
#pragma unroll
          for (int i = 0; i < COLS; ++i)
            if (col0 + i < n_out) out[(int64_t)i * p.ldc] = __float2bfloat16_rn(acc[i]);
        } else {
          float* out = reinterpret_cast<float*>(cout) + (int64_t)col0 * p.ldc + row;
#pragma unroll
          for (int i = 0; i < COLS; ++i)
            if (col0 + i < n_out) out[(int64_t)i * p.ldc] = acc[i];
        }
      } else if (row < (GROUPED ? gt->g[U.g].m : p.M)) {
        if (ksplit > 1) {
          float* out = p.ws + ((int64_t)U.split * p.M + row) * p.ws_ld + col0;
          if (col0 + COLS <= n_out) {
#pragma unroll
            for (int i = 0; i < COLS; i += 4)
              *reinterpret_cast<float4*>(out + i) = make_float4(acc[i], acc[i + 1], acc[i + 2], acc[i + 3]);
          } else {
#pragma unroll
            for (int i = 0; i < COLS; ++i)
              if (col0 + i < n_out) out[i] = acc[i];
          }
        } else if constexpr (OUT_BF16) {
          __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(cout) + (int64_t)row * p.ldc + col0;
          if (col0 + COLS <= n_out && (p.ldc % 8) == 0) {
#pragma unroll
            for (int i = 0; i < COLS; i += 8) {
              uint4 w;
              w.x = pack_bf16x2(acc[i + 0], acc[i + 1]);
              w.y = pack_bf16x2(acc[i + 2], acc[i + 3]);
              w.z = pack_bf16x2(acc[i + 4], acc[i + 5]);
              w.w = pack_bf16x2(acc[i + 6], acc[i + 7]);
              *reinterpret_cast<uint4*>(out + i) = w;
            }
          } else {
#pragma unroll
            for (int i = 0; i < COLS; ++i)
              if (col0 + i < n_out) out[i] = __float2bfloat16_rn(acc[i]);
          }
        } else {
          float* out = reinterpret_cast<float*>(cout) + (int64_t)row * p.ldc + col0;
          if (col0 + COLS <= n_out && (p.ldc % 4) == 0) {
#pragma unroll
            for (int i = 0; i < COLS; i += 4)
              *reinterpret_cast<float4*>(out + i) = make_float4(acc[i], acc[i + 1], acc[i + 2], acc[i + 3]);
          } else {
#pragma unroll
            for (int i = 0; i < COLS; ++i)
              if (col0 + i < n_out) out[i] = acc[i];
          }
        }
      }
    }
    if (q != 0) {  // (the last slot: nothing refills it, released for symmetry)
      __syncwarp();
      arrive_e(a_sempty + ((q - 1) & (NSIG - 1)) * 8);
    }
  }

  tc_fence_before();
  __syncthreads();
  if constexpr (CL > 1) cluster_sync();
  if (warp == W_MMA) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

template <int BN_, int NB_, int EPIW_, bool OUT_BF16, int CL, bool TRANS, bool FUSED = false>
__global__ void __launch_bounds__(MbsCfg<BN_, NB_, EPIW_>::THREADS, 1) __maxnreg__((MbsCfg<BN_, NB_, EPIW_>::MAXNREG))
    k_gemm_mbs(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               const __grid_constant__ Params p) {
  mbs_body<BN_, NB_, EPIW_, OUT_BF16, CL, TRANS, FUSED, false>(&tmA, &tmB, p, nullptr);
}

template <int BN_, int NB_, int EPIW_, bool OUT_BF16, int CL, bool TRANS>
__global__ void __launch_bounds__(MbsCfg<BN_, NB_, EPIW_>::THREADS, 1) __maxnreg__((MbsCfg<BN_, NB_, EPIW_>::MAXNREG))
    k_gemm_mbs_grouped(const __grid_constant__ GroupTable gt) {
  mbs_body<BN_, NB_, EPIW_, OUT_BF16, CL, TRANS, false, true>(nullptr, nullptr, gt.p, &gt);
}

// Split-K partials: C = sum over splits (ascending) of ws[split], as bf16 or f32.
template <bool OUT_BF16>
__global__ void __launch_bounds__(256) k_splitk_reduce(const float* __restrict__ ws, int ksplit, int M, int N,
                                                       int64_t ws_ld, void* __restrict__ c, int64_t ldc) {
  const int64_t total = (int64_t)M * N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / N, col = i - r * N;
    float acc = ws[r * ws_ld + col];
    for (int sp = 1; sp < ksplit; ++sp) acc += ws[((int64_t)sp * M + r) * ws_ld + col];
    if constexpr (OUT_BF16) reinterpret_cast<__nv_bfloat16*>(c)[r * ldc + col] = __float2bfloat16_rn(acc);
    else reinterpret_cast<float*>(c)[r * ldc + col] = acc;
  }
}

template <int BN, int NB, int EPIW, bool OUT_BF16, int CL, bool TRANS, bool FUSED = false>
static int launch(const QDesc& a, const QDesc& b, void* c, int64_t ldc, int ksplit, float* ws, cudaStream_t st,
                  const void* xa = nullptr, int64_t xa_ld = 0, uint32_t* ready = nullptr, uint32_t* status = nullptr) {
  using C = MbsCfg<BN, NB, EPIW>;
  constexpr int SMEM = C::SMEM;
  auto kern = k_gemm_mbs<BN, NB, EPIW, OUT_BF16, CL, TRANS, FUSED>;
  static std::atomic<uint64_t> attr_set{0};
  if (const int rc0 = smem_attr_once(kern, SMEM, attr_set)) return rc0;
  CUtensorMap ta, tb;
  int rc = make_code_map(&ta, a.codes, a.rows, a.cols / 2, a.codes_ld, BM);
  if (rc) return rc;
  rc = make_code_map(&tb, b.codes, b.rows, b.cols / 2, b.codes_ld, BN / CL);
  if (rc) return rc;
  const bool ma = a.variant == MBS_S || a.variant == MBS_D, mbb = b.variant == MBS_S || b.variant == MBS_D;
  const float* ones = ones_buffer();
  if (!ones) return set_error(ERR_INVALID, "could not allocate the sigma ones row");
  Params p{};
  p.sfa = a.scales_mma;
  p.sfb = b.scales_mma;
  p.sfa_kg = a.sf_kpad / 4;
  p.sfb_kg = b.sf_kpad / 4;
  p.sfb_rb = (int)((b.rows + 255) / 256 * 2);
  p.sga = ma ? a.sig_t : ones;
  p.sgb = mbb ? b.sig_t : ones;
  p.sga_ld = ma ? a.sig_t_ld : 0;
  p.sgb_ld = mbb ? b.sig_t_ld : 0;
  p.c = c;
  p.ldc = ldc;
  p.M = (int)a.rows;
  p.N = (int)b.rows;
  p.K = (int)a.cols;
  const int macro = ma ? a.macro_size : b.macro_size;
  p.mac_steps = macro / KSTEP;
  p.n_chunks = (int)((a.cols + macro - 1) / macro);
  p.ksplit = ksplit;
  p.ws = ws;
  p.ws_ld = TRANS ? p.M : p.N;
  p.trace = g_trace;
  p.xa = xa;
  p.xa_ld = xa_ld;
  p.qa = a;
  p.ready = ready;
  p.status = status;
  // E2M1 x E2M1, N = BN, M = 128 (CUTLASS InstrDescriptorBlockScaled layout); scale
  // format UE8M0 (bit 23) unless the pair carries UE4M3 scales
  const bool ue4 = a.variant == NVFP4 || a.sf_format == 1;
  p.idesc = (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((ue4 ? 0u : 1u) << 23) | ((uint32_t)(BM >> 4) << 24);
  p.tsa = a.variant == NVFP4 ? a.tensor_scale : nullptr;
  p.tsb = b.variant == NVFP4 ? b.tensor_scale : nullptr;
  const int units = (((p.M + BM - 1) / BM + CL - 1) / CL) * ((p.N + BN - 1) / BN) * ksplit;
  int clusters = num_sms() / CL;
  if (units < clusters) clusters = units;
  if constexpr (FUSED) {
    // test hook (MXQ_FUSED_OVERSUBSCRIBE=k): k times more CTAs than can be
    // co-resident, to exercise the claim-based quantization phase
    static int over = -1;
    if (over < 0) {
      const char* d = getenv("MXQ_FUSED_OVERSUBSCRIBE");
      over = d ? std::max(1, atoi(d)) : 1;
    }
    clusters *= over;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(clusters * CL);
  cfg.blockDim = dim3(C::THREADS);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ta, tb, p);
  if (e != cudaSuccess) return set_cuda_error(e);
  if (ksplit > 1) {
    const int64_t total = (int64_t)p.M * p.N;
    int g = (int)std::min<int64_t>((total + 255) / 256, (int64_t)num_sms() * 8);
    if (TRANS) k_splitk_reduce<OUT_BF16><<<g, 256, 0, st>>>(ws, ksplit, p.N, p.M, p.ws_ld, c, ldc);
    else k_splitk_reduce<OUT_BF16><<<g, 256, 0, st>>>(ws, ksplit, p.M, p.N, p.ws_ld, c, ldc);
  }
  return check_launch();
}

// Grouped launch.  TRANS (swap-AB, tokens <= 64): kernel A = the weights
// ka[g] (one shared shape), kernel B = the tokens kb[g], C stored [token][n].
// Direct form (tokens <= 128): kernel A = the tokens ka[g] (one 128-row
// block), kernel B = the weights kb[g].  kernel_m / kernel_n: the shared
// kernel extents (the per-group token counts mask the stores).
template <int BN, int NB, int EPIW, bool OUT_BF16, int CL, bool TRANS>
static int launch_grouped(const QDesc* ka, const QDesc* kb, void* const* c, int n, int64_t ldc, int kernel_m,
                          int kernel_n, cudaStream_t st) {
  using C = MbsCfg<BN, NB, EPIW>;
  constexpr int SMEM = C::SMEM;
  auto kern = k_gemm_mbs_grouped<BN, NB, EPIW, OUT_BF16, CL, TRANS>;
  static std::atomic<uint64_t> attr_set{0};
  if (const int rc0 = smem_attr_once(kern, SMEM, attr_set)) return rc0;
  const float* ones = ones_buffer();
  if (!ones) return set_error(ERR_INVALID, "could not allocate the sigma ones row");
  const QDesc& a = ka[0];
  const QDesc& b = kb[0];
  const bool ma = a.variant == MBS_S || a.variant == MBS_D, mbb = b.variant == MBS_S || b.variant == MBS_D;
  std::unique_ptr<GroupTable> t(new GroupTable());
  for (int g0 = 0; g0 < n; g0 += MAXG) {
    const int ng = std::min(MAXG, n - g0);
    memset(t.get(), 0, sizeof(GroupTable));
    Params& p = t->p;
    p.sfa_kg = a.sf_kpad / 4;
    p.sfb_kg = b.sf_kpad / 4;
    p.sfb_rb = (int)((b.rows + 255) / 256 * 2);
    p.sga_ld = ma ? a.sig_t_ld : 0;
    p.ldc = ldc;
    p.M = kernel_m;
    p.N = kernel_n;
    p.K = (int)a.cols;
    const bool nv = a.variant == NVFP4;  // (grouped NVFP4: both sides NVFP4, checked by the caller)
    if (ma || mbb) {
      const int macro = ma ? a.macro_size : b.macro_size;
      p.mac_steps = macro / KSTEP;
      p.n_chunks = (int)((a.cols + macro - 1) / macro);
    } else {
      // no MBS side: one chunk spanning K -- the MMAs accumulate the whole
      // reduction in TMEM and the epilogue folds once (sigma = 1)
      p.mac_steps = (int)((a.cols + KSTEP - 1) / KSTEP);
      p.n_chunks = 1;
    }
    p.ksplit = 1;
    p.trace = g_trace;
    // E2M1 x E2M1, N = BN, M = 128; scale format UE8M0 (bit 23) or UE4M3 (NVFP4)
    p.idesc = (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((nv ? 0u : 1u) << 23) | ((uint32_t)(BM >> 4) << 24);
    t->n_groups = ng;
    for (int j = 0; j < ng; ++j) {
      const QDesc& ag = ka[g0 + j];
      const QDesc& bg = kb[g0 + j];
      GroupDesc& G = t->g[j];
      int rc = make_code_map(&G.tmA, ag.codes, ag.rows, ag.cols / 2, ag.codes_ld, BM);
      if (rc) return rc;
      rc = make_code_map(&G.tmB, bg.codes, bg.rows, bg.cols / 2, bg.codes_ld, BN / CL);
      if (rc) return rc;
      G.sfa = ag.scales_mma;
      G.sfb = bg.scales_mma;
      G.sga = ma ? ag.sig_t : ones;
      G.sgb = mbb ? bg.sig_t : ones;
      G.sgb_ld = mbb ? bg.sig_t_ld : 0;
      G.c = c[g0 + j];
      G.n = TRANS ? (int)bg.rows : kernel_n;
      G.m = TRANS ? kernel_m : (int)ag.rows;
      G.tsa = nv ? ag.tensor_scale : nullptr;
      G.tsb = nv ? bg.tensor_scale : nullptr;
    }
    const int units = ng * (((p.M + BM - 1) / BM + CL - 1) / CL) * ((p.N + BN - 1) / BN);
    const int clusters = std::min(units, num_sms() / CL);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(clusters * CL);
    cfg.blockDim = dim3(C::THREADS);
    cfg.dynamicSmemBytes = SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, *t);
    if (e != cudaSuccess) return set_cuda_error(e);
  }
  return check_launch();
}

}  // namespace mbs

// MBS pair on the tcgen05 path: any macro size that is a multiple of the
// 64-K MMA step (a chunk may straddle 256-K stages; K splits need 64 / 128 /
// 256).  Other macro sizes have no chunk boundary on an MMA step: the exact
// CUDA-core kernel takes them (gemm.py tc_supported).
bool gemm_mbs_supported(const QDesc& a, const QDesc& b) {
  const bool ma = a.variant == MBS_S || a.variant == MBS_D, mb = b.variant == MBS_S || b.variant == MBS_D;
  if (!ma && !mb) return false;
  // one scale format for both operands: UE8M0, or UE4M3 when an NVFP4 side
  // meets an MBS side whose scales were re-expressed (sf_format 1)
  const bool ua = a.variant == NVFP4 || a.sf_format == 1, ub = b.variant == NVFP4 || b.sf_format == 1;
  if (ua != ub) return false;
  const int macro = ma ? a.macro_size : b.macro_size;
  if (ma && mb && a.macro_size != b.macro_size) return false;
  return macro % KSTEP_MBS == 0;
}

// Split count for few-tile shapes: split K at stage boundaries so every SM
// streams weights (decode-like M <= 64 only: at M = 128 the f32 partial
// traffic and the reduce cost more than the parallelism wins, 18 vs 21 us on
// the GPT-OSS gate_up shape, profiles/configs_r01.json).
static int choose_ksplit(int rows_small, int base_clusters, int slots, int n_stages, int macro) {
  if (rows_small > 64 || 2 * base_clusters > slots || n_stages < 4 || 256 % macro) return 1;
  int ks = std::min(slots / base_clusters, n_stages / 2);
  const int spl = (n_stages + ks - 1) / ks;
  return (n_stages + spl - 1) / spl;  // no empty split
}

template <int BN, int NB, int EPIW, bool TRANS>
static int launch_shape(const QDesc& ka, const QDesc& kb, void* c, bool bf, int64_t ldc, int rows_small, cudaStream_t st) {
  const int tiles_m = (int)((ka.rows + mbs::BM - 1) / mbs::BM), tiles_n = (int)((kb.rows + BN - 1) / BN);
  const int n_stages = (int)((ka.cols + mbs::KSTAGE - 1) / mbs::KSTAGE);
  // one 128-row block: no pairing across M, so no cluster (its second CTA would idle)
  const int CL = tiles_m >= 2 ? 2 : 1;
  const int macro = (ka.variant == MBS_S || ka.variant == MBS_D) ? ka.macro_size : kb.macro_size;
  int ksplit = choose_ksplit(rows_small, ((tiles_m + CL - 1) / CL) * tiles_n, num_sms() / CL, n_stages, macro);
  // split-K partials: a stream-ordered allocation per call (pool-cached,
  // graph-capturable, private to this launch -- no workspace shared between
  // streams); without one the launch runs unsplit
  float* ws = nullptr;
  if (ksplit > 1 &&
      cudaMallocAsync(reinterpret_cast<void**>(&ws), (size_t)ksplit * ka.rows * kb.rows * sizeof(float), st) !=
          cudaSuccess) {
    cudaGetLastError();
    ws = nullptr;
    ksplit = 1;
  }
  int rc;
  if (CL == 1)
    rc = bf ? mbs::launch<BN, NB, EPIW, true, 1, TRANS>(ka, kb, c, ldc, ksplit, ws, st)
            : mbs::launch<BN, NB, EPIW, false, 1, TRANS>(ka, kb, c, ldc, ksplit, ws, st);
  else
    rc = bf ? mbs::launch<BN, NB, EPIW, true, 2, TRANS>(ka, kb, c, ldc, ksplit, ws, st)
            : mbs::launch<BN, NB, EPIW, false, 2, TRANS>(ka, kb, c, ldc, ksplit, ws, st);
  if (ws) {
    const cudaError_t e = cudaFreeAsync(ws, st);
    if (!rc && e != cudaSuccess) return set_cuda_error(e);
  }
  return rc;
}

int launch_gemm_mbs(const QDesc& a, const QDesc& b, void* c, int c_dtype, int64_t ldc, cudaStream_t st) {
  const bool bf = c_dtype == MXQ_BF16;
  // Decode-sized A (<= 64 rows) against a wide B: swap-AB -- 128 weight rows
  // per tile on the MMA's M side, the tokens on a narrow N (16-64), four
  // epilogue warps, transposed stores; the kernel streams weights.
  if (a.rows <= 64 && b.rows >= 256) {
    if (a.rows <= 16) return launch_shape<16, 4, 4, true>(b, a, c, bf, ldc, (int)a.rows, st);
    if (a.rows <= 32) return launch_shape<32, 4, 4, true>(b, a, c, bf, ldc, (int)a.rows, st);
    return launch_shape<64, 4, 4, true>(b, a, c, bf, ldc, (int)a.rows, st);
  }
  // prefill shapes: 128 x 192 tiles, two TMEM partial buffers, 16 epilogue warps
  return launch_shape<192, 2, 16, false>(a, b, c, bf, ldc, (int)a.rows, st);
}

// Grouped decode GEMMs (a[g]: tokens, b[g]: weights of one shared shape).
// ERR_UNSUPPORTED when the groups do not fit the grouped kernel (the caller
// then runs them one by one).
int launch_gemm_mbs_grouped(const QDesc* a, const QDesc* b, int n, void* const* c, int c_dtype, int64_t ldc,
                            cudaStream_t st) {
  if (n < 1) return set_error(ERR_INVALID, "no groups");
  int max_tok = 0;
  const bool nv = a[0].variant == NVFP4 && b[0].variant == NVFP4;
  for (int g = 0; g < n; ++g) {
    const QDesc& x = a[g];
    const QDesc& w = b[g];
    const bool pair_ok = nv ? (x.variant == NVFP4 && w.variant == NVFP4 && x.tensor_scale && w.tensor_scale)
                            : gemm_mbs_supported(x, w);
    if (!pair_ok || x.rows < 1 || x.rows > 128 || w.rows < 256 || x.cols != w.cols ||
        w.rows != b[0].rows || w.cols != b[0].cols || w.variant != b[0].variant || x.variant != a[0].variant ||
        w.macro_size != b[0].macro_size || x.macro_size != a[0].macro_size || w.sf_kpad != b[0].sf_kpad ||
        x.sf_kpad != a[0].sf_kpad || w.sig_t_ld != b[0].sig_t_ld || x.sig_t_ld != a[0].sig_t_ld ||
        (x.rows + 255) / 256 != 1)
      return set_error(ERR_UNSUPPORTED, "groups do not share one grouped-kernel shape");
    max_tok = std::max(max_tok, (int)x.rows);
  }
  const bool bf = c_dtype == MXQ_BF16;
  const int wrows = (int)b[0].rows;
  if (max_tok > 64) {  // direct form: one 128-row token block per expert, 128 x 192 tiles over the weights
    return bf ? mbs::launch_grouped<192, 2, 16, true, 1, false>(a, b, c, n, ldc, max_tok, wrows, st)
              : mbs::launch_grouped<192, 2, 16, false, 1, false>(a, b, c, n, ldc, max_tok, wrows, st);
  }
  const bool cl2 = (wrows + mbs::BM - 1) / mbs::BM >= 2;
#define MXQ_GRP(BN_)                                                                                              \
  return cl2 ? (bf ? mbs::launch_grouped<BN_, 4, 4, true, 2, true>(b, a, c, n, ldc, wrows, BN_, st)              \
                   : mbs::launch_grouped<BN_, 4, 4, false, 2, true>(b, a, c, n, ldc, wrows, BN_, st))            \
             : (bf ? mbs::launch_grouped<BN_, 4, 4, true, 1, true>(b, a, c, n, ldc, wrows, BN_, st)              \
                   : mbs::launch_grouped<BN_, 4, 4, false, 1, true>(b, a, c, n, ldc, wrows, BN_, st))
  if (max_tok <= 16) MXQ_GRP(16);
  if (max_tok <= 32) MXQ_GRP(32);
  MXQ_GRP(64);
#undef MXQ_GRP
}

bool gemm_mbs_fusable(const QDesc& a, const QDesc& b, int x_dtype) {
  // (the in-kernel quantizer assigns power-of-two macros to lane groups)
  return x_dtype == DT_BF16 && a.variant == MBS_S && gemm_mbs_supported(a, b) && !(a.rows <= 64 && b.rows >= 256) &&
         (a.macro_size == 64 || a.macro_size == 128 || a.macro_size == 256) && a.scales_mma && a.sig_t;
}

// Fused MBS-S activation quantization + MBS GEMM in one launch (callers check
// gemm_mbs_fusable first; x is bf16 with a 32-byte aligned row pitch).
int launch_gemm_mbs_fused(const void* x, int64_t x_ld, const QDesc& a, const QDesc& b, void* c, int c_dtype,
                          int64_t ldc, uint32_t* status, cudaStream_t st) {
  const bool bf = c_dtype == MXQ_BF16;
  const int tiles_m = (int)((a.rows + mbs::BM - 1) / mbs::BM);
  uint32_t* ready = status + 2;  // the call's own scratch words (published, claimed): nothing shared between launches
  const cudaError_t e = cudaMemsetAsync(ready, 0, 2 * sizeof(uint32_t), st);
  if (e != cudaSuccess) return set_cuda_error(e);
  if (tiles_m >= 2)
    return bf ? mbs::launch<192, 2, 16, true, 2, false, true>(a, b, c, ldc, 1, nullptr, st, x, x_ld, ready, status)
              : mbs::launch<192, 2, 16, false, 2, false, true>(a, b, c, ldc, 1, nullptr, st, x, x_ld, ready, status);
  return bf ? mbs::launch<192, 2, 16, true, 1, false, true>(a, b, c, ldc, 1, nullptr, st, x, x_ld, ready, status)
            : mbs::launch<192, 2, 16, false, 1, false, true>(a, b, c, ldc, 1, nullptr, st, x, x_ld, ready, status);
}

}  // namespace mxq
