// qsnr.cu -- K6: fused dequantise + QSNR / flush-to-zero reduction.
//
// Replaces qsnr_tensor (src/metrics.py:127-153) and flush_to_zero_rate
// (src/metrics.py:165-182).  The reference sums sum(ref^2) and sum(diff^2)
// in f64 with numpy's pairwise algorithm; this kernel reproduces that exact
// summation tree, so the QSNR (and its mse / signal fields) are bit-identical
// to the reference, not merely within 0.01 dB.
//
// Tree: numpy splits a length-n range at n/2 rounded down to a multiple of 8
// until a range is <= 128 (a "leaf", reduced with 8 strided accumulators).
// We embed that tree in a perfect binary tree by treating a leaf at depth l
// as (left = itself, right = empty): x + 0.0 == x exactly, so the sums are
// unchanged.  Each CTA owns one node at depth d (computed by descending from
// the root with the bits of its index), reduces its leaves with warps, and
// folds them in tree order; one final thread folds the top d levels.
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "mxq_arith.cuh"
#include "mxq_internal.h"
#include "mxq_device.cuh"

namespace mxq {

constexpr int QS_THREADS = 256;
constexpr int QS_WARPS = QS_THREADS / 32;
constexpr int QS_MAXLEAF = 320;
constexpr int64_t QS_NODE = 16384;

struct Range { int64_t s, n; };

__host__ __device__ inline int qs_depth(int64_t n) {
  int d = 0;
  while ((n >> d) > QS_NODE) ++d;
  return d;
}

__device__ Range node_at(int64_t n, int depth, int64_t idx) {
  int64_t s = 0, len = n;
  for (int l = depth - 1; l >= 0; --l) {
    const int bit = (int)((idx >> l) & 1);
    if (len <= 128) {
      if (bit) { s += len; len = 0; }
    } else {
      const int64_t n2 = pw_split(len);
      if (bit) { s += n2; len -= n2; } else { len = n2; }
    }
  }
  return {s, len};
}

// Enumerate the leaves of a node in left-to-right order (thread 0; the
// explicit stack lives in shared memory -- no device recursion).
__device__ int enum_leaves(Range r, Range* out, Range* stack) {
  int sp = 0, nl = 0;
  if (r.n > 0) stack[sp++] = r;
  while (sp) {
    Range c = stack[--sp];
    if (c.n <= 128) {
      if (nl < QS_MAXLEAF) out[nl] = c;
      ++nl;
    } else {
      const int64_t n2 = pw_split(c.n);
      stack[sp++] = {c.s + n2, c.n - n2};  // right pushed first -> left popped first
      stack[sp++] = {c.s, n2};
    }
  }
  return nl;
}

struct PairSum { double a, b; };
struct Frame { int64_t n; int state; double la, lb; };

// Post-order fold of a node's subtree over its leaf sums (consumed in
// left-to-right order): sum(node) = sum(left) + sum(right), exactly numpy's
// recursion, evaluated iteratively with a shared-memory frame stack.
__device__ PairSum fold_node(int64_t len, const double* la, const double* lb, Frame* st) {
  int sp = 0, k = 0;
  PairSum res{0.0, 0.0};
  st[sp++] = {len, 0, 0.0, 0.0};
  while (sp) {
    Frame& f = st[sp - 1];
    bool done = false;
    if (f.n == 0) {
      res = {0.0, 0.0};
      done = true;
    } else if (f.n <= 128) {
      res = {la[k], lb[k]};
      ++k;
      done = true;
    } else if (f.state == 0) {
      f.state = 1;
      st[sp++] = {pw_split(f.n), 0, 0.0, 0.0};
    } else if (f.state == 1) {
      f.la = res.a;
      f.lb = res.b;
      f.state = 2;
      const int64_t n2 = pw_split(f.n);
      st[sp++] = {f.n - n2, 0, 0.0, 0.0};
    } else {
      res = {__dadd_rn(f.la, res.a), __dadd_rn(f.lb, res.b)};
      done = true;
    }
    if (done) --sp;
  }
  return res;
}

__device__ __forceinline__ float load_ref(const void* ref, int dtype, int64_t off) {
  if (dtype == DT_BF16)
    return __uint_as_float((uint32_t)reinterpret_cast<const uint16_t*>(ref)[off] << 16);
  return reinterpret_cast<const float*>(ref)[off];
}

__global__ void __launch_bounds__(QS_THREADS, 4) k_qsnr_nodes(const void* __restrict__ ref, int dtype, int64_t ref_ld,
                                                           QDesc q, int has_q, const float* __restrict__ recon,
                                                           int64_t recon_ld, int64_t rows, int64_t cols, int depth,
                                                           double* __restrict__ ws, uint32_t* __restrict__ status) {
  __shared__ Range s_leaf[QS_MAXLEAF];
  __shared__ double s_la[QS_MAXLEAF], s_lb[QS_MAXLEAF];
  __shared__ __align__(16) double s_sq[QS_WARPS][2][2][128];  // [warp][leaf slot][signal/error][element]
  __shared__ int s_nl;
  __shared__ unsigned long long s_cnt[2];
  __shared__ Range s_stack[64];
  __shared__ Frame s_frames[64];
  __shared__ float2 s_uv[256];  // (RN(1/f), RN(1.5/f)) per mantissa byte (see k_dequantize)
  for (int i = threadIdx.x; i < 256; i += QS_THREADS) {
    const float f = mbs_factor((uint32_t)i);
    s_uv[i] = make_float2(__fdiv_rn(1.0f, f), __fdiv_rn(1.5f, f));
  }
  const int64_t n = rows * cols;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Range node = node_at(n, depth, blockIdx.x);
  // A node of 128 * 2^k elements is a perfect tree of consecutive 128-element
  // leaves (numpy's split halves it exactly at every level): its leaves are
  // implicit.  Only irregular nodes are enumerated (serially, by thread 0 --
  // that walk was the CTA's critical path: 22 % barrier stalls).
  const bool implicit = node.n >= 128 && (node.n & 127) == 0 && (((node.n >> 7) & ((node.n >> 7) - 1)) == 0) &&
                        (node.n >> 7) <= QS_MAXLEAF;
  if (threadIdx.x == 0) {
    s_nl = implicit ? (int)(node.n >> 7) : enum_leaves(node, s_leaf, s_stack);
    s_cnt[0] = s_cnt[1] = 0ull;
  }
  __syncthreads();
  const int nl = s_nl;
  if (nl > QS_MAXLEAF) {
    if (threadIdx.x == 0) atomicOr(status, 0x80000000u);
    return;
  }
  const double st = (has_q && q.variant == NVFP4 && q.tensor_scale) ? *q.tensor_scale : 1.0;
  uint32_t bad = 0;
  unsigned long long nz = 0, fl = 0;
  // element -> (row, col) without a 64-bit division per element: one per
  // leaf (warp-uniform), then a 32-bit carry (or division for rows shorter
  // than a leaf); block / macro indices by shift or 32-bit division
  const uint32_t ucols = (uint32_t)cols;
  const int bs_shift = has_q ? (q.block_size == 32 ? 5 : 4) : 4;
  const uint32_t umacro = has_q && q.mant ? (uint32_t)q.macro_size : 1u;
  // Two leaves per warp iteration, eight consecutive elements per lane (lanes
  // 0-15 on leaf li, 16-31 on leaf li + QS_WARPS): a lane's eight elements lie
  // in one row, one 16-block and one macro (leaves start at multiples of 8,
  // rows are multiples of 16 long), so its index math, scale / mantissa loads
  // and dequantisation quotients are done once per eight elements and its
  // reference / code loads are one 16-byte and one 4-byte load.  The two
  // leaves' numpy-order accumulator chains then run side by side.
  const int64_t node_r = node.s / cols;
  const uint32_t node_c = (uint32_t)(node.s - node_r * cols);
  const bool row8 = (ucols % 8u) == 0u;  // (always, with a quantized operand: cols % 16 == 0)
  const bool ref_vec8 = dtype == DT_BF16 && (ref_ld % 8) == 0 && ((uintptr_t)ref % 16) == 0;
  const bool codes_vec = has_q && (q.codes_ld % 4) == 0 && ((uintptr_t)q.codes % 4) == 0;
  const bool mac_pow2 = (umacro & (umacro - 1)) == 0;
  const int mac_shift = __ffs((int)umacro) - 1;
  for (int li = warp; li < nl; li += 2 * QS_WARPS) {
    {
      const int t = lane >> 4, lj = li + t * QS_WARPS;
      const int p0 = 8 * (lane & 15);
      double a8[8], b8[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) a8[j] = b8[j] = 0.0;
      const Range lf = lj < nl ? (implicit ? Range{node.s + 128 * (int64_t)lj, 128} : s_leaf[lj]) : Range{0, 0};
      if (p0 < lf.n) {
        const uint32_t cc = node_c + (uint32_t)(lf.s - node.s) + (uint32_t)p0;
        const uint32_t dr = cc < ucols ? 0u : cc / ucols;
        const int64_t r = node_r + dr;
        const uint32_t c = cc - dr * ucols;
        float xv[8];
        uint32_t codes8 = 0x11111111u;  // (dense recon: no flush statistics)
        if (has_q) {
          const uint8_t* cp = q.codes + r * q.codes_ld + (c >> 1);
          if (codes_vec) {
            codes8 = *reinterpret_cast<const uint32_t*>(cp);
          } else {
            codes8 = 0u;
#pragma unroll
            for (int j = 0; j < 4; ++j) codes8 |= (uint32_t)cp[j] << (8 * j);
          }
          const uint32_t sc = q.scales[r * q.scales_ld + (c >> bs_shift)];
          if (q.variant == NVFP4) {
            bad |= ((sc & 0x7fu) == 0x7fu) ? ST_BAD_E4M3 : 0u;
#pragma unroll
            for (int j = 0; j < 8; ++j) xv[j] = deq_nvfp4((codes8 >> (4 * j)) & 15u, sc, st);
          } else {
            bad |= (sc == 255u) ? ST_BAD_E8M0 : 0u;
            const uint32_t m8 = q.mant ? q.mant[r * q.mant_ld + (mac_pow2 ? (c >> mac_shift) : c / umacro)] : 0u;
            if (sc >= 4u && sc <= 250u) {
              // exact: every magnitude is RN(1/f) or RN(1.5/f) times a power of
              // two (see k_dequantize)
              float u = 1.0f, v = 1.5f;
              if (q.mant) {
                const float2 uv = s_uv[m8];
                u = uv.x;
                v = uv.y;
              }
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const uint32_t code = (codes8 >> (4 * j)) & 15u, idx = code & 7u;
                const float base = ((idx & 1u) && idx > 1u) ? v : u;
                const float mag =
                    idx ? base * __uint_as_float((uint32_t)((int)(idx >> 1) - 1 + (int)sc) << 23) : 0.0f;
                xv[j] = (code & 8u) ? -mag : mag;
              }
            } else {
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const uint32_t code = (codes8 >> (4 * j)) & 15u;
                xv[j] = q.mant ? deq_mbs(code, sc, m8) : deq_pow2(code, sc);
              }
            }
          }
        } else if (row8) {
#pragma unroll
          for (int j = 0; j < 8; ++j) xv[j] = recon[r * recon_ld + c + j];
        }
        float rv8[8];
        if (!row8) {
          // dense reconstruction with rows not a multiple of 8 long: the
          // lane's elements may cross rows, index each one
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint32_t e = cc + (uint32_t)j, dj = e / ucols;
            const int64_t rj = node_r + dj;
            const uint32_t cj = e - dj * ucols;
            xv[j] = recon[rj * recon_ld + cj];
            rv8[j] = load_ref(ref, dtype, rj * ref_ld + cj);
          }
        } else if (ref_vec8) {  // eight bf16 (16 bytes) in one load
          const uint4 w = *reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(ref) + r * ref_ld + c);
          const uint32_t wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            rv8[2 * j] = __uint_as_float(wv[j] << 16);
            rv8[2 * j + 1] = __uint_as_float(wv[j] & 0xFFFF0000u);
          }
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) rv8[j] = load_ref(ref, dtype, r * ref_ld + c + j);
        }
        uint32_t nz8 = 0, fl8 = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float rv = rv8[j];
          const double r64 = (double)rv;
          const double d = __dsub_rn(r64, (double)xv[j]);
          a8[j] = __dmul_rn(r64, r64);
          b8[j] = __dmul_rn(d, d);
          const uint32_t isnz = rv != 0.0f ? 1u : 0u;
          nz8 += isnz;
          fl8 += (((codes8 >> (4 * j)) & 7u) == 0u) ? isnz : 0u;
        }
        nz += nz8;
        fl += fl8;
      }
      double* sa = &s_sq[warp][t][0][p0];
      double* sb = &s_sq[warp][t][1][p0];
#pragma unroll
      for (int j = 0; j < 8; j += 2) {
        *reinterpret_cast<double2*>(sa + j) = make_double2(a8[j], a8[j + 1]);
        *reinterpret_cast<double2*>(sb + j) = make_double2(b8[j], b8[j + 1]);
      }
    }
    __syncwarp();
    // lane = 16 t + 8 w + j: leaf t, w = 0 signal / 1 error, accumulator j
    const int t = lane >> 4, lj = li + t * QS_WARPS;
    double acc = 0.0;
    if (lj < nl) {
      const double* v = s_sq[warp][t][(lane >> 3) & 1];
      const int j = lane & 7, ln = implicit ? 128 : (int)s_leaf[lj].n;
      const double* vj = v + j;
      acc = vj[0];
      if (ln == 128) {  // full leaf: fifteen adds at constant offsets
#pragma unroll 5
        for (int i = 8; i < 128; i += 8) acc = __dadd_rn(acc, vj[i]);
      } else {
        for (int i = 8; i < ln; i += 8) acc = __dadd_rn(acc, vj[i]);
      }
    }
    const int base = lane & 24;
    double r0 = __shfl_sync(0xffffffffu, acc, base | 0), r1 = __shfl_sync(0xffffffffu, acc, base | 1);
    double r2 = __shfl_sync(0xffffffffu, acc, base | 2), r3 = __shfl_sync(0xffffffffu, acc, base | 3);
    double r4 = __shfl_sync(0xffffffffu, acc, base | 4), r5 = __shfl_sync(0xffffffffu, acc, base | 5);
    double r6 = __shfl_sync(0xffffffffu, acc, base | 6), r7 = __shfl_sync(0xffffffffu, acc, base | 7);
    const double res = __dadd_rn(__dadd_rn(__dadd_rn(r0, r1), __dadd_rn(r2, r3)),
                                 __dadd_rn(__dadd_rn(r4, r5), __dadd_rn(r6, r7)));
    if ((lane & 7) == 0 && lj < nl) {
      if (lane & 8) s_lb[lj] = res;
      else s_la[lj] = res;
    }
    __syncwarp();
  }
  for (int o = 16; o > 0; o >>= 1) {
    nz += __shfl_xor_sync(0xffffffffu, nz, o);
    fl += __shfl_xor_sync(0xffffffffu, fl, o);
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  if (lane == 0) {
    atomicAdd(&s_cnt[0], nz);
    atomicAdd(&s_cnt[1], fl);
    if (bad) atomicOr(status, bad);
  }
  __syncthreads();
  // A node of 128 * 2^k elements (every node but the tail ones of an
  // irregular n) is a perfect tree of equal 128-element leaves: fold it level
  // by level with all threads (adjacent pairs, index order -- the same
  // additions as the serial fold).  Otherwise thread 0 walks numpy's split
  // recursion.
  const bool perfect = nl > 0 && nl <= 2 * QS_THREADS && (nl & (nl - 1)) == 0 && node.n == 128LL * nl;
  if (perfect) {
    for (int width = nl; width > 1; width >>= 1) {
      const int half = width >> 1, i = threadIdx.x;
      double va = 0.0, vb = 0.0;
      if (i < half) {
        va = __dadd_rn(s_la[2 * i], s_la[2 * i + 1]);
        vb = __dadd_rn(s_lb[2 * i], s_lb[2 * i + 1]);
      }
      __syncthreads();
      if (i < half) {
        s_la[i] = va;
        s_lb[i] = vb;
      }
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) {
    const PairSum ps = perfect ? PairSum{s_la[0], s_lb[0]} : fold_node(node.n, s_la, s_lb, s_frames);
    const int64_t nodes = (int64_t)1 << depth;
    ws[blockIdx.x] = ps.a;
    ws[nodes + blockIdx.x] = ps.b;
    unsigned long long* cnt = reinterpret_cast<unsigned long long*>(ws + 2 * nodes);
    atomicAdd(cnt, s_cnt[0]);
    atomicAdd(cnt + 1, s_cnt[1]);
  }
}

// Fold of the top `depth` levels.  Every CTA node sits at depth d of a
// perfect binary tree (a numpy leaf above depth d continues as "left = itself,
// right = empty (0.0)"), so the top of the tree is a plain pairwise
// reduction of the 2^d node sums in index order: one CTA, level by level,
// ping-ponging between the node sums and a second buffer in the workspace.
constexpr int QS_TOP_THREADS = 1024;
__global__ void __launch_bounds__(QS_TOP_THREADS) k_qsnr_top(int64_t n, int depth, double* __restrict__ ws,
                                                            double* __restrict__ out4) {
  const int64_t nodes = (int64_t)1 << depth;
  double* sa = ws;
  double* sb = ws + nodes;
  double* ta = ws + 2 * nodes + 2;
  double* tb = ta + nodes;
  for (int64_t width = nodes; width > 1; width >>= 1) {
    const int64_t half = width >> 1;
    for (int64_t i = threadIdx.x; i < half; i += QS_TOP_THREADS) {
      ta[i] = __dadd_rn(sa[2 * i], sa[2 * i + 1]);
      tb[i] = __dadd_rn(sb[2 * i], sb[2 * i + 1]);
    }
    __syncthreads();
    double* t = sa; sa = ta; ta = t;
    t = sb; sb = tb; tb = t;
  }
  if (threadIdx.x == 0) {
    const unsigned long long* cnt = reinterpret_cast<const unsigned long long*>(ws + 2 * nodes);
    out4[0] = sa[0];
    out4[1] = sb[0];
    out4[2] = (double)cnt[0];
    out4[3] = (double)cnt[1];
  }
  (void)n;
}

int64_t qsnr_workspace_bytes(int64_t n) {
  const int d = qs_depth(n);
  return (int64_t)sizeof(double) * (4 * ((int64_t)1 << d) + 2);  // node sums, counts, top-fold ping-pong
}

int launch_qsnr(const void* ref, int dtype, int64_t ref_ld, const QDesc* q, const float* recon, int64_t recon_ld,
                int64_t rows, int64_t cols, void* ws, double* out4, uint32_t* status, cudaStream_t st) {
  const int64_t n = rows * cols;
  const int d = qs_depth(n);
  const int64_t nodes = (int64_t)1 << d;
  double* w = reinterpret_cast<double*>(ws);
  cudaError_t e = cudaMemsetAsync(w + 2 * nodes, 0, 2 * sizeof(double), st);
  if (e != cudaSuccess) return set_cuda_error(e);
  QDesc qd{};
  if (q) qd = *q;
  k_qsnr_nodes<<<(unsigned)nodes, QS_THREADS, 0, st>>>(ref, dtype, ref_ld, qd, q ? 1 : 0, recon, recon_ld, rows,
                                                         cols, d, w, status);
  k_qsnr_top<<<1, QS_TOP_THREADS, 0, st>>>(n, d, w, out4);
  return check_launch();
}

}  // namespace mxq
