// layout.cu -- GEMM-side operand layouts built from the reference layout.
//
// The quantizers write the tcgen05 scale-factor atoms directly; these kernels
// exist for QuantizedTensors the user constructs or edits (e.g.
// dataclasses.replace(q, block_scales=...)) and for mixed-block-size pairs
// (an OCP32 operand against a block-16 one: each E8M0 block-32 scale is
// duplicated into two block-16 scales, which is exact).
#include <cuda_runtime.h>
#include <stdint.h>

#include "mxq_arith.cuh"
#include "mxq_internal.h"

namespace mxq {

// One thread per (padded row, padded 16/32-block): padding entries get 0
// (finite in both UE8M0 (2^-127) and UE4M3 (0) and multiplied by zero data).
__global__ void k_build_sf(QDesc q, int sf_block, int64_t rows_pad) {
  const int64_t total = rows_pad * q.sf_kpad;
  const int ratio = q.block_size / sf_block;  // 1 or 2 (32 -> 16)
  const int64_t nb = q.cols / sf_block;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / q.sf_kpad, kb = i - r * q.sf_kpad;
    uint8_t v = 0;
    if (r < q.rows && kb < nb) v = q.scales[r * q.scales_ld + kb / ratio];
    q.scales_mma[sf_mma_offset(r, kb, q.sf_kpad)] = v;
  }
}

__global__ void k_sigma_t(QDesc q, int64_t nmac) {
  const int64_t total = nmac * q.sig_t_ld;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = i / q.sig_t_ld, r = i - m * q.sig_t_ld;
    q.sig_t[i] = r < q.rows ? 1.0f / mbs_factor(q.mant[r * q.mant_ld + m]) : 0.0f;
  }
}

int launch_build_gemm_layout(const QDesc& q, int sf_block, cudaStream_t st) {
  const int64_t rows_pad = (q.rows + 255) / 256 * 256;
  if (q.scales_mma) {
    const int64_t total = rows_pad * q.sf_kpad;
    int64_t g = (total + 255) / 256;
    if (g > 4096) g = 4096;
    k_build_sf<<<(unsigned)g, 256, 0, st>>>(q, sf_block, rows_pad);
  }
  if (q.sig_t && q.mant) {
    const int64_t nmac = (q.cols + q.macro_size - 1) / q.macro_size;
    const int64_t total = nmac * q.sig_t_ld;
    int64_t g = (total + 255) / 256;
    if (g > 4096) g = 4096;
    k_sigma_t<<<(unsigned)g, 256, 0, st>>>(q, nmac);
  }
  return check_launch();
}

}  // namespace mxq
