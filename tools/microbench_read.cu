// Pure-read bandwidth on B200 (development aid): sum of a bf16-sized buffer,
// HBM-cold (8 buffers cycled, 8 x 32 MB > L2), per-variant device time.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mbr tools/microbench_read.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

template <int U, int W>  // U loads of W*16 bytes per thread per iteration
__global__ void k_read(const uint4* __restrict__ p, size_t n16, unsigned* out) {
  unsigned acc = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x * U * W;
  for (size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * W; i < n16; i += stride) {
    uint4 v[U][W];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t j = i + (size_t)u * gridDim.x * blockDim.x * W;
#pragma unroll
      for (int w = 0; w < W; ++w) {
        if (j + w < n16) {
          if (W == 2 && w == 0) {
            asm volatile("ld.global.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(v[u][0].x), "=r"(v[u][0].y), "=r"(v[u][0].z), "=r"(v[u][0].w), "=r"(v[u][1].x),
                           "=r"(v[u][1].y), "=r"(v[u][1].z), "=r"(v[u][1].w)
                         : "l"(p + j));
          } else if (W == 1) {
            v[u][w] = p[j + w];
          }
        } else {
          v[u][w] = make_uint4(0, 0, 0, 0);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int w = 0; w < W; ++w) acc ^= v[u][w].x ^ v[u][w].y ^ v[u][w].z ^ v[u][w].w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

template <int U, int W>
float run(const uint4* const* bufs, size_t n16, int grid, int block, unsigned* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 8; ++i) k_read<U, W><<<grid, block>>>(bufs[i], n16, out);
  cudaEventRecord(e0);
  const int reps = 48;
  for (int i = 0; i < reps; ++i) k_read<U, W><<<grid, block>>>(bufs[i % 8], n16, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / reps * 1e3f;
}

int main(int argc, char** argv) {
  const size_t mb = argc > 1 ? atoll(argv[1]) : 32;
  const size_t bytes = mb << 20, n16 = bytes / 16;
  uint4* bufs[8];
  for (int i = 0; i < 8; ++i) {
    cudaMalloc(&bufs[i], bytes);
    cudaMemset(bufs[i], 1, bytes);
  }
  unsigned* out;
  cudaMalloc(&out, 4);
  int sms = 148;
  printf("%zu MB read, HBM-cold (us, GB/s):\n", mb);
#define T(U, W, G, B)                                                                           \
  {                                                                                             \
    float us = run<U, W>(bufs, n16, G, B, out);                                                 \
    printf("U=%d W=%d grid=%5d block=%4d: %7.2f us %6.0f GB/s\n", U, W, G, B, us, bytes / us / 1e3); \
  }
  T(1, 1, (int)(n16 / 256), 256);
  T(4, 1, (int)(n16 / 1024), 256);
  T(4, 1, sms * 8, 256);
  T(8, 1, sms * 4, 256);
  T(2, 2, (int)(n16 / 1024), 256);
  T(4, 2, sms * 4, 256);
  T(4, 2, sms * 8, 256);
  T(1, 2, (int)(n16 / 512), 256);
  T(16, 1, sms * 2, 256);
  T(8, 2, sms * 2, 256);
  // 128 MB reads for the asymptote
  return 0;
}
