// gemm_exact.cu -- reference-exact GEMM on CUDA cores (f64, k ascending).
//
// matmul_reference (src/gemm.py:68-90) accumulates c += outer(a[:,k], b[:,k])
// in f64, k ascending, one rounding to f32; matmul_quantized
// (src/gemm.py:137-172) is bit-identical to it on the dequantised operands.
// Every output element here runs the same sequence: products rounded to f64
// (exact for f32 inputs), added in ascending k with __dadd_rn (no FMA
// contraction).  This is the parity / mixed-scale-type path; throughput
// belongs to the tcgen05 kernels in gemm_tc.cu.
#include <cuda_runtime.h>
#include <stdint.h>

#include "mxq_device.cuh"

namespace mxq {

constexpr int EX_T = 16;   // output tile edge
constexpr int EX_K = 64;   // k chunk staged in shared memory

__global__ void __launch_bounds__(EX_T * EX_T) k_gemm_exact(QDesc a, QDesc b, int quant, const float* __restrict__ fa,
                                                          int64_t lda, const float* __restrict__ fb, int64_t ldb,
                                                          int64_t M, int64_t N, int64_t K, float* __restrict__ c,
                                                          int64_t ldc, uint32_t* __restrict__ status) {
  __shared__ float sa[EX_T][EX_K + 1];
  __shared__ float sb[EX_T][EX_K + 1];
  const int tx = threadIdx.x % EX_T, ty = threadIdx.x / EX_T;
  const int64_t i0 = (int64_t)blockIdx.y * EX_T, j0 = (int64_t)blockIdx.x * EX_T;
  const double sta = (quant && a.variant == NVFP4 && a.tensor_scale) ? *a.tensor_scale : 1.0;
  const double stb = (quant && b.variant == NVFP4 && b.tensor_scale) ? *b.tensor_scale : 1.0;
  uint32_t bad = 0;
  double acc = 0.0;
  for (int64_t k0 = 0; k0 < K; k0 += EX_K) {
    for (int e = threadIdx.x; e < EX_T * EX_K; e += EX_T * EX_T) {
      const int rr = e / EX_K, kk = e % EX_K;
      const int64_t k = k0 + kk;
      float va = 0.0f, vb = 0.0f;
      uint32_t code;
      if (i0 + rr < M && k < K) va = quant ? q_elem(a, sta, i0 + rr, k, code, bad) : fa[(i0 + rr) * lda + k];
      if (j0 + rr < N && k < K) vb = quant ? q_elem(b, stb, j0 + rr, k, code, bad) : fb[(j0 + rr) * ldb + k];
      sa[rr][kk] = va;
      sb[rr][kk] = vb;
    }
    __syncthreads();
    const int kmax = (int)((K - k0) < EX_K ? (K - k0) : EX_K);
    for (int kk = 0; kk < kmax; ++kk)
      acc = __dadd_rn(acc, __dmul_rn((double)sa[ty][kk], (double)sb[tx][kk]));
    __syncthreads();
  }
  if (i0 + ty < M && j0 + tx < N) c[(i0 + ty) * ldc + j0 + tx] = (float)acc;
  if (bad) atomicOr(status, bad);
}

int launch_gemm_exact(const QDesc* a, const QDesc* b, const float* fa, int64_t lda, const float* fb, int64_t ldb,
                      int64_t m, int64_t n, int64_t k, float* c, int64_t ldc, uint32_t* status, cudaStream_t st) {
  QDesc qa{}, qb{};
  const int quant = a != nullptr;
  if (quant) { qa = *a; qb = *b; }
  dim3 grid((unsigned)((n + EX_T - 1) / EX_T), (unsigned)((m + EX_T - 1) / EX_T));
  if (grid.y > 65535u) return set_error(ERR_UNSUPPORTED, "M too large for the exact GEMM grid");
  k_gemm_exact<<<grid, EX_T * EX_T, 0, st>>>(qa, qb, quant, fa, lda, fb, ldb, m, n, k, c, ldc, status);
  return check_launch();
}

}  // namespace mxq
