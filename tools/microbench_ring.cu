// Round-trip latency of the MMA -> epilogue -> MMA partial-buffer ring that
// paces the MBS GEMM.  One MMA warp, 8 epilogue warps, NB TMEM buffers of 128
// columns: the MMA warp waits tempty(b), issues 2 block-scaled N=128 MMAs
// (optional) and commits tfull(b); each epilogue warp waits tfull(b),
// optionally loads its 32 lanes x 64 columns (tcgen05.ld + wait::ld), then
// arrives on tempty(b).  cycles per chunk = ring latency / NB when the ring
// is the bound.
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
__device__ __forceinline__ void wait_bar(uint32_t bar, uint32_t ph) {
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(bar),
               "r"(ph)
               : "memory");
}

template <int NB, bool DO_MMA, bool DO_LD, bool PAIR>
__global__ void k(int chunks, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t tfull[4], tempty[4];
  const int warp = threadIdx.x / 32;
  uint32_t rank = 0;
  if (PAIR) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    for (int q = 0; q < 4; ++q) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&tfull[q])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&tempty[q])), "r"(PAIR ? 16 : 8));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 8) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
          (uint32_t)__cvta_generic_to_shared(&tbase)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
          (uint32_t)__cvta_generic_to_shared(&tbase)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (PAIR) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tbase;
  long long t0 = clock64();
  if (warp == 8 && rank == 0) {
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem);
    const uint64_t ad = desc(sb, 16, 1024, 2), bd = desc(sb + 32768, 16, 1024, 2);
    const uint32_t idesc = (1u << 7) | (1u << 10) | ((uint32_t)(128 >> 3) << 17) | (1u << 23) | ((uint32_t)((PAIR ? 256 : 128) >> 4) << 24);
    uint32_t buf = 0, ph = 0;
    for (int c = 0; c < chunks; ++c) {
      wait_bar((uint32_t)__cvta_generic_to_shared(&tempty[buf]), ph ^ 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (DO_MMA && PAIR) {
#pragma unroll
        for (int j = 0; j < 2; ++j)
          asm volatile(
              "{\n\t.reg .pred p, e_;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e_, 0xffffffff;\n\t"
              "@e_ tcgen05.mma.cta_group::2.kind::mxf4nvf4.block_scale.block16 [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(
                  tmem + buf * 128),
              "l"(ad + j * 2), "l"(bd + j * 2), "r"(idesc), "r"(j), "r"(tmem + 448), "r"(tmem + 464)
              : "memory");
      } else if (DO_MMA) {
#pragma unroll
        for (int j = 0; j < 2; ++j)
          asm volatile(
              "{\n\t.reg .pred p, e_;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e_, 0xffffffff;\n\t"
              "@e_ tcgen05.mma.cta_group::1.kind::mxf4nvf4.block_scale.block16 [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(
                  tmem + buf * 128),
              "l"(ad + j * 2), "l"(bd + j * 2), "r"(idesc), "r"(j), "r"(tmem + 448), "r"(tmem + 464)
              : "memory");
      }
      if (PAIR)
        asm volatile("{\n\t.reg .pred e_;\n\telect.sync _|e_, 0xffffffff;\n\t@e_ tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&tfull[buf])), "h"((uint16_t)3)
                     : "memory");
      else
        asm volatile("{\n\t.reg .pred e_;\n\telect.sync _|e_, 0xffffffff;\n\t@e_ tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&tfull[buf]))
                     : "memory");
      if (++buf == NB) { buf = 0; ph ^= 1; }
    }
  } else if (warp < 8) {
    const uint32_t t_ld = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 64;
    uint32_t buf = 0, ph = 0;
    float sink = 0.f;
    for (int c = 0; c < chunks; ++c) {
      wait_bar((uint32_t)__cvta_generic_to_shared(&tfull[buf]), ph);
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (DO_LD) {
        uint32_t r[32];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%"
              "19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
              : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
              : "r"(t_ld + buf * 128 + h * 32)
              : "memory");
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          sink += __uint_as_float(r[0]) + __uint_as_float(r[31]);
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (PAIR) {
        uint32_t rem;
        asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(rem) : "r"((uint32_t)__cvta_generic_to_shared(&tempty[buf])));
        asm volatile("{\n\t.reg .pred e_;\n\telect.sync _|e_, 0xffffffff;\n\t@e_ mbarrier.arrive.shared::cluster.b64 _, [%0];\n\t}" ::"r"(rem)
                     : "memory");
      } else
        asm volatile("{\n\t.reg .pred e_;\n\telect.sync _|e_, 0xffffffff;\n\t@e_ mbarrier.arrive.shared::cta.b64 _, [%0];\n\t}" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&tempty[buf]))
                     : "memory");
      if (++buf == NB) { buf = 0; ph ^= 1; }
    }
    if (sink == 1234.5f) out[7] = 1;
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (PAIR) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 8) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <int NB, bool DO_MMA, bool DO_LD, bool PAIR = false>
void run(int chunks) {
  long long* d;
  cudaMalloc(&d, 64);
  auto kern = k<NB, DO_MMA, DO_LD, PAIR>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148); cfg.blockDim = dim3(384); cfg.dynamicSmemBytes = 65536 + 1024;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = PAIR ? 2 : 1; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr; cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, chunks, d);
  cudaDeviceSynchronize();
  cudaLaunchKernelEx(&cfg, kern, chunks, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long c = 0;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  printf("%s NB=%d mma=%d ld=%d: %7.1f cyc per chunk -> ring latency ~%7.1f  %s\n", PAIR ? "pair" : "one ", NB, (int)DO_MMA, (int)DO_LD,
         (double)c / chunks, (double)c / chunks * NB, e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<1, true, true>(4096);
  run<3, true, true>(4096);
  run<1, false, false, true>(4096);
  run<1, true, false, true>(4096);
  run<1, true, true, true>(4096);
  run<3, true, true, true>(4096);
  run<3, false, false, true>(4096);
  return 0;
}
