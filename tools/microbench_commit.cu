// tcgen05.commit -> mbarrier hand-off latency (warp-converged issue, elect.sync).
// mode 0: MMA x2 -> commit -> same warp waits (round trip per chunk)
// mode 1: ring of NB accumulator buffers: MMA warp issues 2 MMAs per chunk and
//         commits tfull[b]; consumer warp waits tfull[b], arrives tempty[b];
//         MMA waits tempty before reusing b  (the MBS hand-off without math)
// mode 2: as 1 but 4 consumer warps (arrival count 4)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define ELECT "{\n\t.reg .pred e_;\n\telect.sync _|e_, 0xffffffff;\n\t@e_ "

__device__ __forceinline__ uint64_t desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__device__ __forceinline__ void wait(uint32_t bar, uint32_t par) {
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" :: "r"(bar), "r"(par) : "memory");
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc, uint32_t sfa, uint32_t sfb) {
  asm volatile("{\n\t.reg .pred p, e_;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e_, 0xffffffff;\n\t"
               "@e_ tcgen05.mma.cta_group::1.kind::mxf4nvf4.block_scale.block16 [%0], %1, %2, %3, [%5], [%6], p;\n\t}"
               :: "r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(sfa), "r"(sfb) : "memory");
}
__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile(ELECT "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" :: "r"(bar) : "memory");
}

template <int N>
__global__ void k(int mode, int nb, int chunks, int mmas_per_chunk, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t tfull[4], tempty[4];
  const int warp = threadIdx.x / 32;
  const int ncons = mode == 2 ? 4 : 1;
  const int nprod = mode == 4 ? 2 : 1;
  for (int i = threadIdx.x; i < 65536; i += blockDim.x) smem[i] = 0;
  if (threadIdx.x == 0) {
    for (int b = 0; b < 4; ++b) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(&tfull[b])), "r"(nprod));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(&tempty[b])), "r"(ncons));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"((uint32_t)__cvta_generic_to_shared(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tbase;
  if (warp < 4) {
    uint32_t z = 0x7f7f7f7fu;
    uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + 448;
    for (int c = 0; c < 64; c += 4)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%1,%1,%1};" :: "r"(taddr + c), "r"(z));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem);
  const uint64_t ad = desc(sb), bd = desc(sb + 16384);
  const uint32_t idesc = (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (1u << 23) | ((uint32_t)(128 >> 4) << 24);
  long long t0 = clock64();
  if (mode == 3 && (warp == 0 || warp == 1)) {
    // two issuing warps, alternating chunks (warp w issues chunks c = w mod 2)
    uint32_t b = warp, ph = 0;
    for (int c = warp; c < chunks; c += 2) {
      wait((uint32_t)__cvta_generic_to_shared(&tempty[b]), ph ^ 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      for (int j = 0; j < mmas_per_chunk; ++j) mma(tmem + b * N, ad + (j & 3) * 2, bd + (j & 3) * 2, idesc, j > 0, tmem + 448, tmem + 464);
      commit((uint32_t)__cvta_generic_to_shared(&tfull[b]));
      b += 2;
      if (b >= (uint32_t)nb) { b -= nb; ph ^= 1; }
    }
  } else if (mode == 4 && (warp == 0 || warp == 1)) {
    // split N: each warp issues N/2-wide MMAs on its half, both commit every chunk
    const uint32_t idh = (idesc & ~(0x3Fu << 17)) | ((uint32_t)((N / 2) >> 3) << 17);
    uint32_t b = 0, ph = 0;
    for (int c = 0; c < chunks; ++c) {
      wait((uint32_t)__cvta_generic_to_shared(&tempty[b]), ph ^ 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      for (int j = 0; j < mmas_per_chunk; ++j)
        mma(tmem + b * N + warp * (N / 2), ad + (j & 3) * 2, bd + (j & 3) * 2 + warp * ((N / 2) * 128 >> 4), idh, j > 0, tmem + 448, tmem + 464 + warp * 4);
      commit((uint32_t)__cvta_generic_to_shared(&tfull[b]));
      if (++b == (uint32_t)nb) { b = 0; ph ^= 1; }
    }
  } else if (mode != 3 && mode != 4 && warp == 0) {
    uint32_t b = 0, ph = 0;
    for (int c = 0; c < chunks; ++c) {
      if (mode == 0) {
        for (int j = 0; j < mmas_per_chunk; ++j) mma(tmem, ad + (j & 3) * 2, bd + (j & 3) * 2, idesc, j > 0, tmem + 448, tmem + 464);
        const uint32_t fb = (uint32_t)__cvta_generic_to_shared(&tfull[0]);
        commit(fb);
        wait(fb, (uint32_t)(c & 1));
        asm volatile("tcgen05.fence::after_thread_sync;");
      } else {
        wait((uint32_t)__cvta_generic_to_shared(&tempty[b]), ph ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        for (int j = 0; j < mmas_per_chunk; ++j) mma(tmem + b * N, ad + (j & 3) * 2, bd + (j & 3) * 2, idesc, j > 0, tmem + 448, tmem + 464);
        commit((uint32_t)__cvta_generic_to_shared(&tfull[b]));
        if (++b == (uint32_t)nb) { b = 0; ph ^= 1; }
      }
    }
  } else if (mode >= 1 && warp >= 4 && warp < 4 + ncons) {
    uint32_t b = 0, ph = 0;
    for (int c = 0; c < chunks; ++c) {
      wait((uint32_t)__cvta_generic_to_shared(&tfull[b]), ph);
      asm volatile("tcgen05.fence::after_thread_sync;");
      asm volatile("tcgen05.fence::before_thread_sync;");
      if ((threadIdx.x & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"((uint32_t)__cvta_generic_to_shared(&tempty[b])) : "memory");
      if (++b == (uint32_t)nb) { b = 0; ph ^= 1; }
    }
    if (warp == 4 && (threadIdx.x & 31) == 0 && blockIdx.x == 0) out[0] = clock64() - t0;
  }
  if (mode == 0 && threadIdx.x == 0 && blockIdx.x == 0) out[0] = clock64() - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tmem));
  }
}

template <int N>
void run(int mode, int nb, int chunks, int mpc) {
  long long* d; cudaMalloc(&d, 16);
  auto kern = k<N>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  kern<<<148, 256, 65536>>>(mode, nb, chunks, mpc, d);
  cudaDeviceSynchronize();
  kern<<<148, 256, 65536>>>(mode, nb, chunks, mpc, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long c = 0; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  printf("mode %d N=%d nb=%d mmas/chunk=%d: %.1f cyc/chunk (ideal %d) %s\n", mode, N, nb, mpc, (double)c / chunks,
         mpc * N / 2, e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<256>(1, 1, 4000, 4);
  run<256>(4, 1, 4000, 4);
  run<256>(1, 1, 4000, 16);
  run<256>(4, 1, 4000, 16);
  run<128>(3, 3, 4000, 2);
  return 0;
}
