// tcgen05.mma issue-rate ceiling by kind / N / cta_group (one SM or one SM pair).
// One warp issues back-to-back MMAs (elect.sync inside the asm, descriptors
// precomputed, accumulate=1, no commits) on zeroed shared memory, then commits
// once and waits.  Prints cycles per MMA and MACs/clk/SM against the
// 128*N/(256*cg)-cycle floor (bf16 K16, fp8 K32, fp4 K64 all the same cycles).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// KIND: 0 f16(bf16) 1 f8f6f4(e4m3) 2 mxf8f6f4 block32 3 mxf4 block32 4 mxf4nvf4 block16 ue8m0 5 mxf4nvf4 block16 ue4m3
#define MMA_PLAIN(CGV, KS) \
  asm volatile("{\n\t.reg .pred p, e_;\n\tsetp.ne.b32 p, 1, 0;\n\telect.sync _|e_, 0xffffffff;\n\t@e_ tcgen05.mma.cta_group::" CGV ".kind::" KS " [%0], %1, %2, %3, p;\n\t}" \
               :: "r"(d), "l"(a), "l"(b), "r"(idesc) : "memory")
#define MMA_BS(CGV, KS) \
  asm volatile("{\n\t.reg .pred p, e_;\n\tsetp.ne.b32 p, 1, 0;\n\telect.sync _|e_, 0xffffffff;\n\t@e_ tcgen05.mma.cta_group::" CGV ".kind::" KS " [%0], %1, %2, %3, [%4], [%5], p;\n\t}" \
               :: "r"(d), "l"(a), "l"(b), "r"(idesc), "r"(sfa), "r"(sfb) : "memory")
template <int KIND, int CG>
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t sfa, uint32_t sfb) {
  if constexpr (CG == 1) {
    if constexpr (KIND == 0) MMA_PLAIN("1", "f16");
    else if constexpr (KIND == 1) MMA_PLAIN("1", "f8f6f4");
    else if constexpr (KIND == 2) MMA_BS("1", "mxf8f6f4.block_scale.block32");
    else if constexpr (KIND == 3) MMA_BS("1", "mxf4.block_scale.block32");
    else MMA_BS("1", "mxf4nvf4.block_scale.block16");
  } else {
    if constexpr (KIND == 0) MMA_PLAIN("2", "f16");
    else if constexpr (KIND == 1) MMA_PLAIN("2", "f8f6f4");
    else if constexpr (KIND == 2) MMA_BS("2", "mxf8f6f4.block_scale.block32");
    else if constexpr (KIND == 3) MMA_BS("2", "mxf4.block_scale.block32");
    else MMA_BS("2", "mxf4nvf4.block_scale.block16");
  }
}

template <int KIND, int N, int CG>
__global__ void k(int iters, int cmode, long long* out) {
  const int sf_rot = 0;
  const int commit_every = cmode & 0xff;      // commit after every `commit_every` MMAs
  const int do_wait = (cmode >> 8) & 1;       // try_wait on an already-complete barrier after each commit
  const int do_fence = (cmode >> 9) & 1;      // tcgen05.fence::after_thread_sync after each commit
  const int multi_bar = (cmode >> 10) & 1;    // rotate over 4 commit barriers
  const int rot_d = (cmode >> 11) & 1;        // rotate the accumulator over 4 N-column buffers per commit group
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t fin;
  __shared__ __align__(8) uint64_t cb[4];
  __shared__ __align__(8) uint64_t done;
  const int warp = threadIdx.x / 32;
  uint32_t rank = 0;
  if (CG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = threadIdx.x; i < 98304 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"((uint32_t)__cvta_generic_to_shared(&fin)));
    for (int q = 0; q < 4; ++q) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"((uint32_t)__cvta_generic_to_shared(&cb[q])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"((uint32_t)__cvta_generic_to_shared(&done)));
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"((uint32_t)__cvta_generic_to_shared(&done)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    if (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"((uint32_t)__cvta_generic_to_shared(&tbase)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"((uint32_t)__cvta_generic_to_shared(&tbase)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tbase;
  // scale factors: columns 256.. (value 0x7f = 1.0 for UE8M0; 0x38 = 1.0 for UE4M3)
  if (warp < 4) {
    const uint32_t z = KIND == 5 ? 0x38383838u : 0x7f7f7f7fu;
    uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + 256;
    for (int c = 0; c < 256; c += 4)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%1,%1,%1};" :: "r"(taddr + c), "r"(z));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int M = 128 * CG;
  if (warp == 0 && rank == 0) {
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem);
    const uint64_t ad = desc(sb), bd = desc(sb + 32768);
    uint32_t idesc = ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    if (KIND == 0) idesc |= (1u << 4) | (1u << 7) | (1u << 10);  // f32 acc, bf16 x bf16
    if (KIND == 1) idesc |= (1u << 4);                           // f32 acc, e4m3 x e4m3
    if (KIND == 2) idesc |= (1u << 23);                          // e4m3, ue8m0
    if (KIND == 3 || KIND == 4) idesc |= (1u << 7) | (1u << 10) | (1u << 23);  // e2m1, ue8m0
    if (KIND == 5) idesc |= (1u << 7) | (1u << 10);              // e2m1, ue4m3
    const uint32_t fb = (uint32_t)__cvta_generic_to_shared(&fin);
    long long t0 = clock64();
    const uint32_t donea = (uint32_t)__cvta_generic_to_shared(&done);
    int cnt = 0, nc = 0;
    for (int i = 0; i < iters; i += 4) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        mma<KIND, CG>(tmem + (rot_d ? (uint32_t)((nc & 3) * N) : 0u), ad + j * 2, bd + j * 2, idesc, tmem + 256, tmem + 320);
        if (commit_every && ++cnt == commit_every) {
          cnt = 0;
          const uint32_t cba = (uint32_t)__cvta_generic_to_shared(&cb[multi_bar ? (nc & 3) : 0]);
          ++nc;
          asm volatile("{\n\t.reg .pred e_;\n\telect.sync _|e_, 0xffffffff;\n\t@e_ tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" :: "r"(cba) : "memory");
          if (do_wait) asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n\t}" :: "r"(donea) : "memory");
          if (do_fence) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
      }
    }
    long long t1 = clock64();
    if (CG == 1)
      asm volatile("{\n\t.reg .pred e_;\n\telect.sync _|e_, 0xffffffff;\n\t@e_ tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" :: "r"(fb) : "memory");
    else
      asm volatile("{\n\t.reg .pred e_;\n\telect.sync _|e_, 0xffffffff;\n\t@e_ tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" :: "r"(fb), "h"((uint16_t)3) : "memory");
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n\t}" :: "r"(fb) : "memory");
    long long t2 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) { out[0] = t2 - t0; out[1] = t1 - t0; }
  }
  if (CG == 2 && warp == 0 && rank == 1) {
    const uint32_t fb = (uint32_t)__cvta_generic_to_shared(&fin);
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n\t}" :: "r"(fb) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (CG == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tmem));
    else asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" :: "r"(tmem));
  }
}

static const char* kname[] = {"f16(bf16) K16", "f8f6f4(e4m3) K32", "mxf8f6f4.block32 K32", "mxf4.block32 K64",
                              "mxf4nvf4.block16 ue8m0 K64", "mxf4nvf4.block16 ue4m3 K64"};
static const int kK[] = {16, 32, 32, 64, 64, 64};

template <int KIND, int N, int CG>
void run(int iters, int sf_rot = 0) {
  long long* d; cudaMalloc(&d, 32); cudaMemset(d, 0, 32);
  auto kern = k<KIND, N, CG>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 98304);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = 98304;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr; cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, iters, sf_rot, d);
  cudaDeviceSynchronize();
  cudaLaunchKernelEx(&cfg, kern, iters, sf_rot, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long cc[2] = {0, 0}; cudaMemcpy(cc, d, 16, cudaMemcpyDeviceToHost);
  const double per = (double)cc[0] / iters;
  const double floor_c = 128.0 * N / 256.0;  // per SM: each SM does 128 x N x K
  const double macs_sm = 128.0 * N * kK[KIND] / per;
  printf("%-28s cg=%d N=%3d cmode=0x%x: %7.1f cyc/MMA (issue %6.1f), floor %5.1f -> %5.2fx floor, %6.0f MACs/clk/SM %s\n",
         kname[KIND], CG, N, sf_rot, per, (double)cc[1] / iters, floor_c, per / floor_c, macs_sm,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  // decode tiles (16 / 32 / 64 columns): per-chunk commits into rotating buffers
  run<4, 16, 1>(2048, 0);
  run<4, 16, 1>(2048, 2);
  run<4, 16, 1>(2048, 2 | 1024);
  run<4, 16, 1>(2048, 2 | 1024 | 2048);
  run<4, 16, 1>(2048, 4 | 1024 | 2048);
  run<4, 16, 1>(2048, 1 | 1024 | 2048);
  run<5, 16, 1>(2048, 0);
  run<5, 16, 1>(2048, 4);
  run<4, 32, 1>(2048, 0);
  run<4, 32, 1>(2048, 2 | 1024 | 2048);
  run<4, 64, 1>(2048, 0);
  run<4, 64, 1>(2048, 2 | 1024 | 2048);
  run<4, 256, 1>(2048, 0);
  run<4, 256, 1>(2048, 1);
  run<4, 256, 1>(2048, 2);
  run<4, 256, 1>(2048, 4);
  run<4, 256, 1>(2048, 4 | 256);
  run<4, 256, 1>(2048, 4 | 512);
  run<4, 256, 1>(2048, 4 | 1024);
  run<4, 128, 1>(2048, 0);
  run<4, 128, 1>(2048, 2);
  run<4, 128, 1>(2048, 2 | 256 | 512);
  run<4, 128, 1>(2048, 2 | 1024);
  return 0;
}
