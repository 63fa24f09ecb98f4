// mxq_device.cuh -- device-side element access shared by the evaluator and
// the reference-exact GEMM.
#pragma once
#include "mxq_arith.cuh"
#include "mxq_internal.h"

namespace mxq {

// Dequantised element of q at (r, c) with the reference formula
// (src/quantize.py:409-423); `code` returns the 4-bit code, `bad` collects
// corrupt-scale status bits (src/quantize.py:228-241).
__device__ __forceinline__ float q_elem(const QDesc& q, double st, int64_t r, int64_t c, uint32_t& code,
                                        uint32_t& bad) {
  const uint8_t byte = q.codes[r * q.codes_ld + (c >> 1)];
  code = (c & 1) ? (byte >> 4) : (byte & 15u);
  const uint32_t s = q.scales[r * q.scales_ld + c / q.block_size];
  if (q.variant == NVFP4) {
    bad |= ((s & 0x7fu) == 0x7fu) ? ST_BAD_E4M3 : 0u;
    return deq_nvfp4(code, s, st);
  }
  bad |= (s == 255u) ? ST_BAD_E8M0 : 0u;
  if (q.mant) return deq_mbs(code, s, q.mant[r * q.mant_ld + c / q.macro_size]);
  return deq_pow2(code, s);
}

}  // namespace mxq
