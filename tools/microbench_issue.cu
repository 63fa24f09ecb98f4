// MMA-warp issue ceiling of candidate MBS GEMM schedules (round 2 design).
// One warp per SM issues, per 128-K "chunk": NCP scale-factor atom copies
// (tcgen05.cp 32x128b.warpx4), 2 block-scaled MMAs (mxf4nvf4.block16, N
// columns, K=64 each) into TMEM buffer (chunk % 3), and one commit to that
// buffer's barrier.  Nothing waits on the barriers: this is the issue-side
// cost per chunk that the FP32 epilogue (2*128*N/128 cycles per chunk) must
// hide.  Second test: tcgen05.ld throughput of 8 warps loading 64 columns
// (x64) vs 16 warps loading 32 (x32), bytes per clock per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(layout & 7u) << 61;
  return d;
}

template <int N, int NCP>
__global__ void k_issue(int chunks, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bars[4];
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 98304 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x7f7f7f7f & 0;
  if (threadIdx.x == 0) {
    for (int q = 0; q < 4; ++q)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bars[q])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tbase;
  if (warp == 0) {
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem);
    const uint64_t ad = desc(sb, 16, 1024, 2), bd = desc(sb + 32768, 16, 1024, 2);
    const uint32_t idesc = (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t nbuf_cols = N;
    const uint32_t sf0 = 3 * nbuf_cols <= 448 ? 448 : (2 * nbuf_cols <= 448 ? 448 : 480);
    long long t0 = clock64();
    uint32_t buf = 0;
    for (int c = 0; c < chunks; ++c) {
#pragma unroll
      for (int q = 0; q < NCP; ++q) {
        const uint64_t sd = desc(sb + 65536 + q * 512, 0, 128, 0);
        asm volatile("{\n\t.reg .pred e_;\n\telect.sync _|e_, 0xffffffff;\n\t@e_ tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;\n\t}" ::"r"(
                         tmem + sf0 + (uint32_t)(q * 4) % 32),
                     "l"(sd)
                     : "memory");
      }
      const uint32_t d = tmem + (3 * nbuf_cols <= 448 ? buf : (buf & 1)) * nbuf_cols;
#pragma unroll
      for (int j = 0; j < 2; ++j)
        asm volatile(
            "{\n\t.reg .pred p, e_;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e_, 0xffffffff;\n\t"
            "@e_ tcgen05.mma.cta_group::1.kind::mxf4nvf4.block_scale.block16 [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(d),
            "l"(ad + j * 2), "l"(bd + j * 2), "r"(idesc), "r"(j), "r"(tmem + sf0), "r"(tmem + sf0 + 16)
            : "memory");
      const uint32_t ba = (uint32_t)__cvta_generic_to_shared(&bars[buf]);
      asm volatile("{\n\t.reg .pred e_;\n\telect.sync _|e_, 0xffffffff;\n\t@e_ tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
                       ba)
                   : "memory");
      if (++buf == 3) buf = 0;
    }
    long long t1 = clock64();
    const uint32_t fa = (uint32_t)__cvta_generic_to_shared(&bars[3]);
    asm volatile("{\n\t.reg .pred e_;\n\telect.sync _|e_, 0xffffffff;\n\t@e_ tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
                     fa)
                 : "memory");
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n\t}" ::"r"(fa)
                 : "memory");
    long long t2 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      out[0] = t2 - t0;
      out[1] = t1 - t0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// TMEM load throughput: NW warps, each loading COLS columns of its lane
// quadrant per iteration (x32 or x64 shapes), wait::ld every iteration.
template <int NW, int COLS>
__global__ void k_tmem_ld(int iters, long long* out, float* sink) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tbase;
  const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * COLS);
  float acc = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t r[32];
#pragma unroll
    for (int h = 0; h < COLS; h += 32) {
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%"
          "19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
            "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
            "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
          : "r"(base + h)
          : "memory");
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int i = 0; i < 32; ++i) acc += __uint_as_float(r[i]);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  if (acc == 12345.f) sink[0] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}


// cta_group::2 variant: leader issues per chunk NCP cp.cta_group::2 + 2 MMAs (M=256, N) + commit multicast to both CTAs.
template <int N, int NCP>
__global__ void k_issue2(int chunks, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bars[4];
  const int warp = threadIdx.x / 32;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = threadIdx.x; i < 98304 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    for (int q = 0; q < 4; ++q)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bars[q])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tbase;
  if (warp == 0 && rank == 0) {
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem);
    const uint64_t ad = desc(sb, 16, 1024, 2), bd = desc(sb + 32768, 16, 1024, 2);
    const uint32_t idesc = (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(256 >> 4) << 24);
    const uint32_t sf0 = 448;
    long long t0 = clock64();
    uint32_t buf = 0;
    for (int c = 0; c < chunks; ++c) {
#pragma unroll
      for (int q = 0; q < NCP; ++q) {
        const uint64_t sd = desc(sb + 65536 + q * 512, 0, 128, 0);
        asm volatile("{\n\t.reg .pred e_;\n\telect.sync _|e_, 0xffffffff;\n\t@e_ tcgen05.cp.cta_group::2.32x128b.warpx4 [%0], %1;\n\t}" ::"r"(
                         tmem + sf0 + (uint32_t)(q * 4) % 32),
                     "l"(sd)
                     : "memory");
      }
      const uint32_t d = tmem + (3 * N <= 448 ? buf : (buf & 1)) * N;
#pragma unroll
      for (int j = 0; j < 2; ++j)
        asm volatile(
            "{\n\t.reg .pred p, e_;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e_, 0xffffffff;\n\t"
            "@e_ tcgen05.mma.cta_group::2.kind::mxf4nvf4.block_scale.block16 [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(d),
            "l"(ad + j * 2), "l"(bd + j * 2), "r"(idesc), "r"(j), "r"(tmem + sf0), "r"(tmem + sf0 + 16)
            : "memory");
      const uint32_t ba = (uint32_t)__cvta_generic_to_shared(&bars[buf]);
      asm volatile("{\n\t.reg .pred e_;\n\telect.sync _|e_, 0xffffffff;\n\t@e_ tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
                       ba), "h"((uint16_t)3)
                   : "memory");
      if (++buf == 3) buf = 0;
    }
    long long t1 = clock64();
    const uint32_t fa = (uint32_t)__cvta_generic_to_shared(&bars[3]);
    asm volatile("{\n\t.reg .pred e_;\n\telect.sync _|e_, 0xffffffff;\n\t@e_ tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
                     fa), "h"((uint16_t)3)
                 : "memory");
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n\t}" ::"r"(fa)
                 : "memory");
    long long t2 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      out[0] = t2 - t0;
      out[1] = t1 - t0;
    }
  }
  if (warp == 0 && rank == 1) {
    const uint32_t fa = (uint32_t)__cvta_generic_to_shared(&bars[3]);
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n\t}" ::"r"(fa)
                 : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <int N, int NCP>
void run_issue2(int chunks) {
  long long* d;
  cudaMalloc(&d, 32);
  auto kern = k_issue2<N, NCP>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 98304);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = 98304;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr; cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, chunks, d);
  cudaDeviceSynchronize();
  cudaLaunchKernelEx(&cfg, kern, chunks, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long cc[2] = {0, 0};
  cudaMemcpy(cc, d, 16, cudaMemcpyDeviceToHost);
  printf("pair  N=%3d cp/chunk=%d: %7.1f cyc/chunk (issue loop %7.1f); MMA floor per SM %d  %s\n", N, NCP,
         (double)cc[0] / chunks, (double)cc[1] / chunks, N, e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}

template <int N, int NCP>
void run_issue(int chunks) {
  long long* d;
  cudaMalloc(&d, 32);
  auto kern = k_issue<N, NCP>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 98304);
  kern<<<148, 128, 98304>>>(chunks, d);
  cudaDeviceSynchronize();
  kern<<<148, 128, 98304>>>(chunks, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long cc[2] = {0, 0};
  cudaMemcpy(cc, d, 16, cudaMemcpyDeviceToHost);
  printf("issue N=%3d cp/chunk=%d: %7.1f cyc/chunk (issue loop %7.1f); MMA floor %d, FP32 epilogue %d  %s\n", N, NCP,
         (double)cc[0] / chunks, (double)cc[1] / chunks, N, 2 * N, e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}

template <int NW, int COLS>
void run_ld(int iters) {
  long long* d;
  float* s;
  cudaMalloc(&d, 32);
  cudaMalloc(&s, 32);
  k_tmem_ld<NW, COLS><<<148, NW * 32>>>(iters, d, s);
  cudaDeviceSynchronize();
  k_tmem_ld<NW, COLS><<<148, NW * 32>>>(iters, d, s);
  cudaError_t e = cudaDeviceSynchronize();
  long long cc = 0;
  cudaMemcpy(&cc, d, 8, cudaMemcpyDeviceToHost);
  const double bytes = (double)iters * NW * 32 * COLS * 4;
  printf("tmem ld %2d warps x %3d cols: %6.1f B/clk/SM (%.0f cyc per %d KB)  %s\n", NW, COLS, bytes / cc,
         (double)cc / iters, NW * 32 * COLS * 4 / 1024, e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
  cudaFree(s);
}

int main() {
  run_issue<128, 4>(4096);
  run_issue2<128, 0>(4096);
  run_issue2<128, 4>(4096);
  run_issue2<256, 0>(4096);
  run_issue2<192, 6>(4096);
  return 0;
}
