// Throughput of the MBS epilogue fold in isolation: NW warps per SM, each
// folding COLS columns per "chunk" (acc += (sA * sB_j) * p_j), sB from shared
// memory (LDS.128 broadcast), p in registers.  FORM 0: FMUL2(sB pair, sA) +
// FFMA2(w, p, acc) [the kernel's form]; FORM 1: FMUL2(p, sB pair) +
// FFMA2(u, sA, acc); FORM 2: scalar FMUL + FFMA; FORM 3: form 0 with sB held
// in registers (no LDS).  Prints cycles per chunk per SM sub-partition against
// the 2*COLS*(NW/4)/32*2-cycle pipe floor.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void mul2(float& o0, float& o1, float a, float b0, float b1) {
  asm("{\n\t.reg .b64 x, y;\n\tmov.b64 x, {%2, %3};\n\tmov.b64 y, {%4, %4};\n\t"
      "mul.rn.f32x2 x, x, y;\n\tmov.b64 {%0, %1}, x;\n\t}"
      : "=f"(o0), "=f"(o1)
      : "f"(b0), "f"(b1), "f"(a));
}
__device__ __forceinline__ void mul2v(float& o0, float& o1, float a0, float a1, float b0, float b1) {
  asm("{\n\t.reg .b64 x, y;\n\tmov.b64 x, {%2, %3};\n\tmov.b64 y, {%4, %5};\n\t"
      "mul.rn.f32x2 x, x, y;\n\tmov.b64 {%0, %1}, x;\n\t}"
      : "=f"(o0), "=f"(o1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
__device__ __forceinline__ void fma2(float& acc0, float& acc1, float w0, float w1, float p0, float p1) {
  asm("{\n\t.reg .b64 w, q, c;\n\tmov.b64 w, {%2, %3};\n\tmov.b64 q, {%4, %5};\n\t"
      "mov.b64 c, {%0, %1};\n\tfma.rn.f32x2 c, w, q, c;\n\tmov.b64 {%0, %1}, c;\n\t}"
      : "+f"(acc0), "+f"(acc1)
      : "f"(w0), "f"(w1), "f"(p0), "f"(p1));
}
__device__ __forceinline__ void fma2s(float& acc0, float& acc1, float u0, float u1, float s) {
  asm("{\n\t.reg .b64 w, q, c;\n\tmov.b64 w, {%2, %3};\n\tmov.b64 q, {%4, %4};\n\t"
      "mov.b64 c, {%0, %1};\n\tfma.rn.f32x2 c, w, q, c;\n\tmov.b64 {%0, %1}, c;\n\t}"
      : "+f"(acc0), "+f"(acc1)
      : "f"(u0), "f"(u1), "f"(s));
}

template <int FORM, int COLS>
__global__ void k(int iters, float* out, long long* cyc) {
  __shared__ __align__(16) float sig[8][256];
  for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) (&sig[0][0])[i] = 1.0f + i * 1e-6f;
  __syncthreads();
  float acc[COLS], p[COLS], sbr[COLS];
#pragma unroll
  for (int i = 0; i < COLS; ++i) {
    acc[i] = 0.f;
    p[i] = threadIdx.x * 1e-3f + i;
    sbr[i] = 1.0f - i * 1e-4f;
  }
  const int warp = threadIdx.x / 32;
  float sa = 0.5f + threadIdx.x * 1e-5f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const float* sb = &sig[it & 7][(warp >> 2) * COLS];
    float sa4[4];
    if (FORM == 4 || FORM == 5) {
      const int q = threadIdx.x & 3;
#pragma unroll
      for (int r = 0; r < 4; ++r) sa4[r] = sig[it & 7][128 + (threadIdx.x & 31) / 4 + 8 * r];
      if (FORM == 4) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float2 v = *reinterpret_cast<const float2*>(sb + 8 * k + 2 * q);
          sbr[2 * k] = v.x;
          sbr[2 * k + 1] = v.y;
        }
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float4 v = *reinterpret_cast<const float4*>(sb + 16 * q + 4 * k);
          sbr[4 * k] = v.x; sbr[4 * k + 1] = v.y; sbr[4 * k + 2] = v.z; sbr[4 * k + 3] = v.w;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < COLS; i += 4) {
      float4 b = make_float4(0.f, 0.f, 0.f, 0.f);
      if (FORM >= 4) {}
      else if (FORM == 3) b = make_float4(sbr[i], sbr[i + 1], sbr[i + 2], sbr[i + 3]);
      else b = *reinterpret_cast<const float4*>(sb + i);
      if (FORM == 0 || FORM == 3) {
        float w0, w1, w2, w3;
        mul2(w0, w1, sa, b.x, b.y);
        mul2(w2, w3, sa, b.z, b.w);
        fma2(acc[i], acc[i + 1], w0, w1, p[i], p[i + 1]);
        fma2(acc[i + 2], acc[i + 3], w2, w3, p[i + 2], p[i + 3]);
      } else if (FORM == 1) {
        float u0, u1, u2, u3;
        mul2v(u0, u1, p[i], p[i + 1], b.x, b.y);
        mul2v(u2, u3, p[i + 2], p[i + 3], b.z, b.w);
        fma2s(acc[i], acc[i + 1], u0, u1, sa);
        fma2s(acc[i + 2], acc[i + 3], u2, u3, sa);
      } else if (FORM == 4 || FORM == 5) {
        // 16x256b layout: element i -> row (i / 16), column pair ((i % 16) / 2); sB for 16 columns per chunk
        float u0, u1, u2, u3;
        const int cp = (i % 16);
        mul2v(u0, u1, p[i], p[i + 1], sbr[cp], sbr[cp + 1]);
        mul2v(u2, u3, p[i + 2], p[i + 3], sbr[cp + 2], sbr[cp + 3]);
        fma2s(acc[i], acc[i + 1], u0, u1, sa4[i / 16]);
        fma2s(acc[i + 2], acc[i + 3], u2, u3, sa4[i / 16]);
      } else {
        acc[i] = fmaf(sa * b.x, p[i], acc[i]);
        acc[i + 1] = fmaf(sa * b.y, p[i + 1], acc[i + 1]);
        acc[i + 2] = fmaf(sa * b.z, p[i + 2], acc[i + 2]);
        acc[i + 3] = fmaf(sa * b.w, p[i + 3], acc[i + 3]);
      }
    }
    sa = sa * 1.0000001f;
#pragma unroll
    for (int i = 0; i < COLS; ++i) asm volatile("" : "+f"(p[i]));
  }
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < COLS; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int FORM, int COLS>
void run(int nw) {
  float* out;
  long long* cyc;
  const int iters = 2048;
  cudaMalloc(&out, 148 * nw * 32 * 4);
  cudaMalloc(&cyc, 148 * 8);
  k<FORM, COLS><<<148, nw * 32>>>(iters, out, cyc);
  cudaDeviceSynchronize();
  k<FORM, COLS><<<148, nw * 32>>>(iters, out, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double per = (double)c / iters;
  const double floor_c = 2.0 * COLS * (nw / 4) * 32 / 32 / 2 * 2;  // FP32 lane-ops per SMSP / 32 lanes
  printf("form %d cols %3d warps/SM %2d: %6.1f cyc per chunk (FP32 floor %5.0f) -> %.2f  %s\n", FORM, COLS, nw, per,
         floor_c, floor_c / per, e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run<0, 64>(8);
  run<1, 64>(8);
  run<2, 64>(8);
  run<3, 64>(8);
  run<0, 32>(16);
  run<1, 32>(16);
  run<4, 64>(8);
  run<5, 64>(8);
  run<4, 64>(16);
  run<4, 64>(4);
  return 0;
}
