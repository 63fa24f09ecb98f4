// FP32 pipe throughput on sm_100a: FFMA vs packed FFMA2 / FMUL2 (the MBS
// epilogue's two ops per output per chunk).  Prints ops/clk/SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float* out, int iters, long long* cyc) {
  float a[16];
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i;
  const float b = 0.999f, c = 1e-7f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      if (MODE == 0) {
        a[i] = fmaf(a[i], b, c);
        a[i + 1] = fmaf(a[i + 1], b, c);
      } else if (MODE == 1) {
        asm volatile("{\n\t.reg .b64 x, y, z;\n\tmov.b64 x, {%0, %1};\n\tmov.b64 y, {%2, %2};\n\tmov.b64 z, {%3, %3};\n\t"
                     "fma.rn.f32x2 x, x, y, z;\n\tmov.b64 {%0, %1}, x;\n\t}"
                     : "+f"(a[i]), "+f"(a[i + 1]) : "f"(b), "f"(c));
      } else {
        asm volatile("{\n\t.reg .b64 x, y;\n\tmov.b64 x, {%0, %1};\n\tmov.b64 y, {%2, %2};\n\t"
                     "mul.rn.f32x2 x, x, y;\n\tmov.b64 {%0, %1}, x;\n\t}"
                     : "+f"(a[i]), "+f"(a[i + 1]) : "f"(b));
      }
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, int sms) {
  float* out; long long* cyc;
  int threads = 1024, iters = 4096;
  cudaMalloc(&out, sms * threads * 4);
  cudaMalloc(&cyc, sms * 8);
  k<MODE><<<sms, threads>>>(out, iters, cyc);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<MODE><<<sms, threads>>>(out, iters, cyc);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  double flops_per_sm = (double)threads * iters * 16;  // scalar FMA-or-MUL ops per SM
  printf("%s: %.1f ops/clk/SM (clock64), %.2f Tops/s chip\n", name, flops_per_sm / c,
         flops_per_sm * sms / (ms * 1e-3) / 1e12);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>("FFMA  ", sms);
  run<1>("FFMA2 ", sms);
  run<2>("FMUL2 ", sms);
  return 0;
}
