// TMA delivery rate per SM: one producer thread streams 2-D boxes (ROWS x 128
// B, 128B swizzle) of an L2-resident FP4-code matrix through a STAGES-deep
// shared-memory ring; one consumer thread waits each stage's full barrier and
// frees it.  Every CTA reads its own row band, walking K, like a GEMM's A
// operand.  MODE 0: one box per stage; MODE 1: two boxes per stage (A-like +
// B-like band); MODE 2: cluster of 2, each CTA loads half of the second box
// and multicasts it to both.  Prints bytes per clock per SM.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ void wait_bar(uint32_t bar, uint32_t ph) {
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(bar),
               "r"(ph)
               : "memory");
}

template <int ROWS, int STAGES, int MODE>
__global__ void k(const __grid_constant__ CUtensorMap tm, int kiters, int rows_total, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full[16], empty[16];
  constexpr int NBOX = MODE == 1 ? 2 : 1;
  constexpr int STAGE = ROWS * 128 * NBOX;
  const uint32_t sm = ((uint32_t)__cvta_generic_to_shared(smem_raw) + 1023u) & ~1023u;
  uint32_t rank = 0;
  if (MODE == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&empty[s])),
                   "r"(MODE == 2 ? 2 : 1));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (MODE == 2) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  const int row0 = (blockIdx.x * ROWS) % rows_total;
  const int row1 = ((blockIdx.x / (MODE == 2 ? 2 : 1)) * ROWS + rows_total / 2) % rows_total;
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    uint32_t st = 0, ph = 0;
    for (int it = 0; it < kiters; ++it) {
      const uint32_t fb = (uint32_t)__cvta_generic_to_shared(&full[st]);
      wait_bar((uint32_t)__cvta_generic_to_shared(&empty[st]), ph ^ 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(STAGE) : "memory");
      const int kc = (it % 32) * 128;
      if (MODE != 2)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              sm + st * STAGE),
          "l"(reinterpret_cast<uint64_t>(&tm)), "r"(kc), "r"(row0), "r"(fb)
          : "memory");
      if (MODE == 1)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                sm + st * STAGE + ROWS * 128),
            "l"(reinterpret_cast<uint64_t>(&tm)), "r"(kc), "r"(row1), "r"(fb)
            : "memory");
      if (MODE == 2)  // half of the second box each, multicast to both CTAs
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%2, "
            "%3}], [%4], %5;" ::"r"(sm + st * STAGE + rank * (ROWS / 2) * 128),
            "l"(reinterpret_cast<uint64_t>(&tm) + 128 * 0), "r"(kc), "r"(row1 + (int)rank * (ROWS / 2)), "r"(fb),
            "h"((uint16_t)3)
            : "memory");
      if (++st == STAGES) { st = 0; ph ^= 1; }
    }
  } else if (threadIdx.x == 32) {
    uint32_t st = 0, ph = 0;
    for (int it = 0; it < kiters; ++it) {
      wait_bar((uint32_t)__cvta_generic_to_shared(&full[st]), ph);
      if (MODE == 2) {
        // free the stage in both CTAs (the peer multicasts into it)
        const uint32_t eb = (uint32_t)__cvta_generic_to_shared(&empty[st]);
        for (uint32_t r = 0; r < 2; ++r) {
          uint32_t rem;
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rem) : "r"(eb), "r"(r));
          asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(rem) : "memory");
        }
      } else {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(&empty[st]))
                     : "memory");
      }
      if (++st == STAGES) { st = 0; ph ^= 1; }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (MODE == 2) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
}

template <int ROWS, int STAGES, int MODE>
void run(CUtensorMap* tm, int rows_total) {
  long long* d;
  cudaMalloc(&d, 64);
  constexpr int NBOX = MODE == 1 ? 2 : 1;
  const int smem = ROWS * 128 * NBOX * STAGES + 1024;
  auto kern = k<ROWS, STAGES, MODE>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(64);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = MODE == 2 ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const int kiters = 4096;
  cudaLaunchKernelEx(&cfg, kern, *tm, kiters, rows_total, d);
  cudaDeviceSynchronize();
  cudaLaunchKernelEx(&cfg, kern, *tm, kiters, rows_total, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long c = 0;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  const double bytes = (double)kiters * ROWS * 128 * NBOX;
  printf("rows %3d stages %d mode %d: %6.1f B/clk/SM received (%.0f cyc per stage)  %s\n", ROWS, STAGES, MODE,
         bytes / c, (double)c / kiters, e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  const int rows = 8192, kbytes = 4096;  // 32 MB of codes: L2-resident
  uint8_t* buf;
  cudaMalloc(&buf, (size_t)rows * kbytes);
  cudaMemset(buf, 0x11, (size_t)rows * kbytes);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  PFN_encodeTiled enc = (PFN_encodeTiled)fn;
  CUtensorMap tm128, tm64, tm256;
  cuuint64_t dims[2] = {(cuuint64_t)kbytes, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)kbytes};
  cuuint32_t estr[2] = {1, 1};
  cuuint32_t box128[2] = {128, 128}, box64[2] = {128, 64}, box256[2] = {128, 256};
  enc(&tm128, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dims, strides, box128, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&tm64, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dims, strides, box64, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&tm256, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dims, strides, box256, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  run<128, 4, 0>(&tm128, rows);
  run<128, 8, 0>(&tm128, rows);
  run<128, 4, 1>(&tm128, rows);
  run<64, 8, 1>(&tm64, rows);
  run<256, 3, 0>(&tm256, rows);
  run<128, 4, 2>(&tm64, rows);  // 64-row half per CTA, multicast: 128 rows received
  run<128, 8, 2>(&tm64, rows);
  return 0;
}
