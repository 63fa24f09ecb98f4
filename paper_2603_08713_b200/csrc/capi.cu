// capi.cu -- the extern "C" boundary (include/mxq200.h): argument validation,
// error reporting, launch on the caller's stream, and the host-compiled
// scalar helpers built from the same arithmetic header as the kernels.
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <mutex>
#include <string>
#include <vector>

#include "mxq_arith.cuh"
#include "mxq_internal.h"

namespace mxq {

static thread_local std::string g_err;

int set_error(int code, const char* msg) {
  g_err = msg;
  return code;
}

int set_cuda_error(cudaError_t e) {
  g_err = std::string("CUDA error: ") + cudaGetErrorString(e);
  return (int)e;
}

int check_launch() {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_cuda_error(e);
}

int num_sms() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cached[dev]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = n > 0 ? n : 148;
  }
  return cached[dev];
}

static int validate_q(const QDesc* q, bool need_rowmajor) {
  if (!q) return set_error(ERR_INVALID, "null quantized tensor");
  if (q->variant < OCP32 || q->variant > NVFP4) return set_error(ERR_INVALID, "unknown variant");
  const int bs = q->variant == OCP32 ? 32 : 16;
  if (q->block_size != bs) return set_error(ERR_INVALID, "block_size does not match the variant");
  if (q->rows <= 0 || q->cols <= 0) return set_error(ERR_INVALID, "expected a non-empty 2-D tensor");
  if (q->cols % bs) return set_error(ERR_INVALID, "row length is not divisible by block_size");
  if (q->macro_size <= 0 || q->macro_size % bs) return set_error(ERR_INVALID, "macro_size is not a positive multiple of block_size");
  if (!q->codes || q->codes_ld < q->cols / 2) return set_error(ERR_INVALID, "codes buffer missing or too narrow");
  if (need_rowmajor && (!q->scales || q->scales_ld < q->cols / bs))
    return set_error(ERR_INVALID, "row-major scales missing or too narrow");
  if ((q->variant == MBS_S || q->variant == MBS_D) && need_rowmajor && !q->mant)
    return set_error(ERR_INVALID, "MBS tensor without mantissas");
  if (q->variant == NVFP4 && !q->tensor_scale) return set_error(ERR_INVALID, "NVFP4 tensor without tensor_scale");
  if (q->scales_mma) {
    const int64_t kstep = 256 / bs;
    if (q->sf_kpad < q->cols / bs || q->sf_kpad % kstep) return set_error(ERR_INVALID, "sf_kpad must cover cols and be a multiple of 256/block_size");
  }
  return 0;
}

}  // namespace mxq

using namespace mxq;

extern "C" {

int mxq_version(void) { return 100; }

// Development aid: when non-NULL, the next GEMM launches write a clock64()
// trace of CTA 0's MMA / epilogue hand-offs (4 x int64 per chunk) there.
void mxq_debug_set_trace(long long* dev_buf) { set_gemm_trace(dev_buf); }

const char* mxq_last_error(void) { return g_err.c_str(); }

int mxq_device_ok(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return 0;
  }
  int dev = 0, major = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  return major == 10 ? 1 : 0;
}

int mxq_quantize(const void* x, int32_t x_dtype, int64_t x_ld, const mxq_qtensor* q, int32_t mbs_mode,
                 const uint8_t* cand, int32_t n_cand, int32_t augment_static, uint32_t* scratch, void* stream) {
  int rc = validate_q(q, false);
  if (rc) return rc;
  if (!x || !scratch) return set_error(ERR_INVALID, "null input or scratch");
  if (x_dtype != DT_F32 && x_dtype != DT_BF16) return set_error(ERR_INVALID, "x_dtype must be MXQ_F32 or MXQ_BF16");
  if (x_ld < q->cols) return set_error(ERR_INVALID, "x_ld < cols");
  const int esz = x_dtype == DT_BF16 ? 2 : 4, al = x_dtype == DT_BF16 ? 32 : 16;  // (bf16 units are 256-bit loads)
  if (((uintptr_t)x % al) || ((x_ld * esz) % al))
    return set_error(ERR_UNSUPPORTED, "input must be aligned with a row pitch of 32 bytes (bf16) / 16 bytes (f32)");
  if (!q->scales && !q->scales_mma) return set_error(ERR_INVALID, "no scale output buffer");
  {  // the call's status words start at zero (the kernels only OR error bits in)
    const cudaError_t e = cudaMemsetAsync(scratch, 0, 4 * sizeof(uint32_t), (cudaStream_t)stream);
    if (e != cudaSuccess) return set_cuda_error(e);
  }
  const bool mbs = q->variant == MBS_S || q->variant == MBS_D;
  if (mbs && !q->mant && !q->sig_t) return set_error(ERR_INVALID, "MBS quantize needs a mantissa buffer");
  if (q->scales_mma) {  // padding atoms must hold finite scale codes
    const int64_t rows_pad = (q->rows + 255) / 256 * 256;
    if (rows_pad != q->rows || q->sf_kpad != q->cols / q->block_size) {
      cudaError_t e = cudaMemsetAsync(q->scales_mma, 0, (size_t)(rows_pad * q->sf_kpad), (cudaStream_t)stream);
      if (e != cudaSuccess) return set_cuda_error(e);
    }
  }
  if (q->sig_t && q->sig_t_ld > q->rows) {
    const int64_t nmac = (q->cols + q->macro_size - 1) / q->macro_size;
    cudaError_t e = cudaMemsetAsync(q->sig_t, 0, sizeof(float) * (size_t)(nmac * q->sig_t_ld), (cudaStream_t)stream);
    if (e != cudaSuccess) return set_cuda_error(e);
  }
  return launch_quantize(x, x_dtype, x_ld, *q, mbs_mode, cand, n_cand, augment_static, scratch,
                         (cudaStream_t)stream);
}

int mxq_quantize_mbs_lut(const void* x, int32_t x_dtype, int64_t x_ld, const mxq_qtensor* q, const uint8_t* cand,
                         int32_t n_cand, const float* lut_entries, uint32_t* scratch, void* stream) {
  int rc = validate_q(q, false);
  if (rc) return rc;
  if (!x || !scratch || !cand || !lut_entries) return set_error(ERR_INVALID, "null argument");
  if (x_dtype != DT_F32 && x_dtype != DT_BF16) return set_error(ERR_INVALID, "x_dtype must be MXQ_F32 or MXQ_BF16");
  const int esz = x_dtype == DT_BF16 ? 2 : 4;
  if (x_ld < q->cols || ((uintptr_t)x % 16) || ((x_ld * esz) % 16))
    return set_error(ERR_UNSUPPORTED, "input must be 16-byte aligned with a 16-byte row pitch");
  if (!q->mant && !q->sig_t) return set_error(ERR_INVALID, "MBS quantize needs a mantissa buffer");
  {
    const cudaError_t e = cudaMemsetAsync(scratch, 0, 4 * sizeof(uint32_t), (cudaStream_t)stream);
    if (e != cudaSuccess) return set_cuda_error(e);
  }
  if (q->scales_mma) {
    const int64_t rows_pad = (q->rows + 255) / 256 * 256;
    if (rows_pad != q->rows || q->sf_kpad != q->cols / q->block_size) {
      cudaError_t e = cudaMemsetAsync(q->scales_mma, 0, (size_t)(rows_pad * q->sf_kpad), (cudaStream_t)stream);
      if (e != cudaSuccess) return set_cuda_error(e);
    }
  }
  return launch_quantize_lut(x, x_dtype, x_ld, *q, cand, n_cand, lut_entries, scratch, (cudaStream_t)stream);
}

int mxq_dequantize(const mxq_qtensor* q, float* out, int64_t out_ld, uint32_t* scratch, void* stream) {
  int rc = validate_q(q, true);
  if (rc) return rc;
  if (!out || out_ld < q->cols || (out_ld % 4) || ((uintptr_t)out % 16)) return set_error(ERR_INVALID, "bad output buffer");
  return launch_dequantize(*q, out, out_ld, scratch, (cudaStream_t)stream);
}

int64_t mxq_qsnr_workspace_bytes(int64_t n) { return qsnr_workspace_bytes(n); }

int mxq_qsnr(const void* ref, int32_t ref_dtype, int64_t ref_ld, const mxq_qtensor* q, const float* recon,
             int64_t recon_ld, int64_t rows, int64_t cols, void* workspace, double* out4, uint32_t* scratch,
             void* stream) {
  if (!ref || !workspace || !out4 || !scratch) return set_error(ERR_INVALID, "null argument");
  if (rows <= 0 || cols <= 0) return set_error(ERR_INVALID, "expected a non-empty 2-D tensor");
  if (q) {
    int rc = validate_q(q, true);
    if (rc) return rc;
    if (q->rows != rows || q->cols != cols) return set_error(ERR_INVALID, "shape mismatch");
  } else if (!recon) {
    return set_error(ERR_INVALID, "need q or recon");
  }
  if ((rows * cols) % 8) return set_error(ERR_UNSUPPORTED, "element count must be a multiple of 8");
  return launch_qsnr(ref, ref_dtype, ref_ld, q, recon, recon_ld, rows, cols, workspace, out4, scratch,
                     (cudaStream_t)stream);
}

int mxq_gemm(const mxq_qtensor* a, const mxq_qtensor* b, void* c, int32_t c_dtype, int64_t ldc, uint32_t* scratch,
             void* stream) {
  int rc = validate_q(a, false);
  if (rc) return rc;
  rc = validate_q(b, false);
  if (rc) return rc;
  if (a->cols != b->cols) return set_error(ERR_INVALID, "operands disagree on K");
  if (!c || ldc < b->rows) return set_error(ERR_INVALID, "bad output buffer");
  return launch_gemm_tc(*a, *b, c, c_dtype, ldc, scratch, (cudaStream_t)stream);
}

int mxq_quantize_gemm(const void* x, int32_t x_dtype, int64_t x_ld, const mxq_qtensor* a, const mxq_qtensor* b,
                      void* c, int32_t c_dtype, int64_t ldc, uint32_t* scratch, void* stream) {
  int rc = validate_q(a, false);
  if (rc) return rc;
  rc = validate_q(b, false);
  if (rc) return rc;
  if (a->variant != MBS_S) return set_error(ERR_INVALID, "quantize_gemm: the activation side must be MBS_S");
  if (a->cols != b->cols) return set_error(ERR_INVALID, "operands disagree on K");
  if (!c || ldc < b->rows) return set_error(ERR_INVALID, "bad output buffer");
  if (!a->scales_mma || !a->sig_t) return set_error(ERR_INVALID, "quantize_gemm needs A's GEMM layout buffers");
  const bool fuse = gemm_mbs_fusable(*a, *b, x_dtype) && (((uintptr_t)x | (uintptr_t)(x_ld * 2)) % 32) == 0;
  if (!fuse) {  // two launches, same results
    rc = mxq_quantize(x, x_dtype, x_ld, a, 0, nullptr, 0, 0, scratch, stream);
    if (rc) return rc;
    return launch_gemm_tc(*a, *b, c, c_dtype, ldc, scratch, (cudaStream_t)stream);
  }
  if (!x || !scratch) return set_error(ERR_INVALID, "null input or scratch");
  if (x_ld < a->cols) return set_error(ERR_INVALID, "x_ld < cols");
  cudaStream_t st = (cudaStream_t)stream;
  {
    const cudaError_t e = cudaMemsetAsync(scratch, 0, 2 * sizeof(uint32_t), st);  // (words 2-3: launch_gemm_mbs_fused)
    if (e != cudaSuccess) return set_cuda_error(e);
  }
  const int64_t rows_pad = (a->rows + 255) / 256 * 256;
  if (rows_pad != a->rows || a->sf_kpad != a->cols / a->block_size) {  // padding atoms must hold finite codes
    cudaError_t e = cudaMemsetAsync(a->scales_mma, 0, (size_t)(rows_pad * a->sf_kpad), st);
    if (e != cudaSuccess) return set_cuda_error(e);
  }
  if (a->sig_t_ld > a->rows) {
    const int64_t nmac = (a->cols + a->macro_size - 1) / a->macro_size;
    cudaError_t e = cudaMemsetAsync(a->sig_t, 0, sizeof(float) * (size_t)(nmac * a->sig_t_ld), st);
    if (e != cudaSuccess) return set_cuda_error(e);
  }
  return launch_gemm_mbs_fused(x, x_ld, *a, *b, c, c_dtype, ldc, scratch, st);
}

int mxq_gemm_grouped(const mxq_qtensor* a, const mxq_qtensor* b, int32_t n, void* const* c, int32_t c_dtype,
                     int64_t ldc, uint32_t* scratch, void* stream) {
  if (!a || !b || !c || n < 1) return set_error(ERR_INVALID, "bad group arrays");
  for (int g = 0; g < n; ++g) {
    int rc = validate_q(&a[g], false);
    if (rc) return rc;
    rc = validate_q(&b[g], false);
    if (rc) return rc;
    if (a[g].cols != b[g].cols) return set_error(ERR_INVALID, "operands disagree on K");
    if (!c[g] || ldc < b[g].rows) return set_error(ERR_INVALID, "bad output buffer");
  }
  const int rc = launch_gemm_mbs_grouped(a, b, n, c, c_dtype, ldc, (cudaStream_t)stream);
  if (rc != ERR_UNSUPPORTED) return rc;
  for (int g = 0; g < n; ++g) {  // groups the grouped kernel does not take: one launch each
    const int r = launch_gemm_tc(a[g], b[g], c[g], c_dtype, ldc, scratch, (cudaStream_t)stream);
    if (r) return r;
  }
  return 0;
}

int mxq_gemm_exact(const mxq_qtensor* a, const mxq_qtensor* b, float* c, int64_t ldc, uint32_t* scratch,
                   void* stream) {
  int rc = validate_q(a, true);
  if (rc) return rc;
  rc = validate_q(b, true);
  if (rc) return rc;
  if (a->cols != b->cols) return set_error(ERR_INVALID, "operands disagree on K");
  if (!c || ldc < b->rows) return set_error(ERR_INVALID, "bad output buffer");
  return launch_gemm_exact(a, b, nullptr, 0, nullptr, 0, a->rows, b->rows, a->cols, c, ldc, scratch,
                           (cudaStream_t)stream);
}

int mxq_matmul_reference(const float* a, int64_t lda, const float* b, int64_t ldb, int64_t m, int64_t n, int64_t k,
                         float* c, int64_t ldc, void* stream) {
  if (!a || !b || !c || m <= 0 || n <= 0 || k <= 0 || lda < k || ldb < k || ldc < n)
    return set_error(ERR_INVALID, "bad matmul_reference arguments");
  return launch_gemm_exact(nullptr, nullptr, a, lda, b, ldb, m, n, k, c, ldc, nullptr, (cudaStream_t)stream);
}

int mxq_build_gemm_layout(const mxq_qtensor* q, int32_t sf_block, void* stream) {
  int rc = validate_q(q, true);
  if (rc) return rc;
  if (sf_block != 16 && sf_block != 32) return set_error(ERR_INVALID, "sf_block must be 16 or 32");
  if (sf_block > q->block_size) return set_error(ERR_INVALID, "sf_block larger than block_size");
  if (q->scales_mma && (q->sf_kpad < q->cols / sf_block || q->sf_kpad % (256 / sf_block)))
    return set_error(ERR_INVALID, "sf_kpad must cover cols and be a multiple of 256/sf_block");
  if (q->sig_t && q->sig_t_ld < q->rows) return set_error(ERR_INVALID, "sig_t_ld < rows");
  return launch_build_gemm_layout(*q, sf_block, (cudaStream_t)stream);
}

// ---- host scalar helpers ---------------------------------------------------

int mxq_host_encode_e2m1(const double* v, int64_t n, int32_t saturate, uint8_t* out) {
  for (int64_t i = 0; i < n; ++i)
    if (!isfinite(v[i])) return set_error(MXQ_ERR_NONFINITE, "cannot encode non-finite value");
  if (!saturate)
    for (int64_t i = 0; i < n; ++i)
      if (fabs(v[i]) > 6.0) return set_error(MXQ_ERR_RANGE, "magnitude exceeds 6.0 and saturate=False");
  for (int64_t i = 0; i < n; ++i) out[i] = (uint8_t)e2m1_code_f64(v[i]);
  return 0;
}

int mxq_host_encode_e4m3(const double* v, int64_t n, uint8_t* out) {
  for (int64_t i = 0; i < n; ++i)
    if (!isfinite(v[i])) return set_error(MXQ_ERR_NONFINITE, "cannot encode non-finite value");
  for (int64_t i = 0; i < n; ++i) {
    const uint32_t c = e4m3_code_f64(fabs(v[i]));
    out[i] = (uint8_t)((v[i] < 0 && c) ? (c | 0x80u) : c);
  }
  return 0;
}

int mxq_host_e8m0_floor(double x, uint8_t* biased, int32_t* clamped) {
  if (!(isfinite(x) && x > 0)) return set_error(ERR_INVALID, "e8m0_floor requires a positive finite input");
  int e;
  frexp(x, &e);
  int ex = e - 1;
  *clamped = (ex < -127 || ex > 127);
  ex = ex < -127 ? -127 : (ex > 127 ? 127 : ex);
  *biased = (uint8_t)(ex + 127);
  return 0;
}

int mxq_host_extract_mantissa8(double sf, uint8_t* m8) {
  if (!(isfinite(sf) && sf > 0)) return set_error(ERR_INVALID, "extract_mantissa8 requires a positive finite input");
  const float f = (float)sf;
  *m8 = (uint8_t)((f2u(f) & 0x007F8000u) >> 15);
  return 0;
}

int mxq_host_block_scale(const double* block, int64_t n, int32_t kind, uint8_t* biased, int32_t* clamped) {
  const int64_t want = kind == 0 ? 32 : 16;
  if (n != want) return set_error(ERR_INVALID, "wrong block length");
  double a = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    if (!isfinite(block[i])) return set_error(ERR_INVALID, "block contains non-finite elements");
    a = fmax(a, fabs(block[i]));
  }
  int c = 0;
  *biased = (uint8_t)e8m0_block_f64(a, kind, &c);
  *clamped = c;
  return 0;
}

int mxq_host_e8m0_closed_form(const float* alpha, int64_t n, int32_t kind, uint8_t* out) {
  for (int64_t i = 0; i < n; ++i)
    out[i] = kind == 0 ? e8m0_biased_ocp(alpha[i]) : e8m0_biased_16(alpha[i], kind == 2);
  return 0;
}

int mxq_host_static_m8(double alpha, uint8_t* m8) {
  if (alpha == 0.0) { *m8 = 0; return 0; }
  if (!(isfinite(alpha) && alpha > 0)) return set_error(ERR_INVALID, "macro maximum must be positive finite");
  *m8 = static_m8((float)alpha);
  return 0;
}

static double pw_sum_host(const double* a, int64_t n) {
  if (n <= 128) return pw_leaf(a, n);
  const int64_t n2 = pw_split(n);
  return dadd_rn(pw_sum_host(a, n2), pw_sum_host(a + n2, n - n2));
}

// Per-macro MBS-D selection on the host with the kernels' arithmetic
// (exact SSE search when lut == NULL, else the LUT cost).
// Replaces mbs_dynamic_exact / mbs_dynamic_lut (src/quantize.py:464-479, :545-560).
int mxq_host_mbs_choose(const float* x, int64_t n, const uint8_t* cand, int32_t n_cand, int32_t augment,
                        const float* lut, uint8_t* m8_out) {
  if (n <= 0 || n % 16) return set_error(ERR_INVALID, "macro length must be a positive multiple of 16");
  if (n_cand < 1 || n_cand > 256) return set_error(ERR_INVALID, "candidate count out of range");
  if (lut && n_cand != 16) return set_error(ERR_INVALID, "the lookup table holds exactly 16 candidates");
  float amax = 0.0f;
  for (int64_t i = 0; i < n; ++i) {
    if (!isfinite(x[i])) return set_error(ERR_INVALID, "macro contains non-finite elements");
    amax = fmaxf(amax, fabsf(x[i]));
  }
  std::vector<double> sq((size_t)n);
  const int n_trials = n_cand + ((augment && !lut) ? 1 : 0);
  double best = 0.0;
  uint32_t best_m8 = 0;
  for (int t = 0; t < n_trials; ++t) {
    const uint32_t m8 = t < n_cand ? cand[t] : static_m8(amax);
    const float f = mbs_factor(m8);
    for (int64_t b0 = 0; b0 < n; b0 += 16) {
      float y[16], a = 0.0f;
      for (int i = 0; i < 16; ++i) {
        y[i] = mul_rn(x[b0 + i], f);
        a = fmaxf(a, fabsf(y[i]));
      }
      const uint32_t biased = e8m0_biased_16(a, true);
      const double sf = ldexp(1.0, 127 - (int)biased);
      for (int i = 0; i < 16; ++i) {
        const double x64 = (double)x[b0 + i];
        if (lut) {
          const double v = dmul_rn(fabs(x64), sf);
          double tv;
          if (v < 1.0) {
            long long bi = (long long)dmul_rn(v, 64.0);
            bi = bi < 0 ? 0 : (bi > 63 ? 63 : bi);
            tv = (double)lut[(0 * 16 + t) * 64 + bi];
          } else {
            volatile double num = dmul_rn(v - 1.0, 64.0);
            volatile double q = num / 7.0;
            long long bi = (long long)q;
            bi = bi < 0 ? 0 : (bi > 63 ? 63 : bi);
            tv = (double)lut[(1 * 16 + t) * 64 + bi];
          }
          sq[b0 + i] = dmul_rn(dmul_rn(x64, x64), tv);
        } else {
          const uint32_t code = e2m1_code_f64((double)y[i] * sf);
          const double d = (double)deq_mbs(code, biased, m8) - x64;
          sq[b0 + i] = dmul_rn(d, d);
        }
      }
    }
    const double cost = pw_sum_host(sq.data(), n);
    if (t == 0 || cost < best || (cost == best && m8 < best_m8)) {
      best = cost;
      best_m8 = m8;
    }
  }
  *m8_out = (uint8_t)best_m8;
  return 0;
}

float mxq_host_dequant_element(int32_t variant, uint32_t code, uint32_t scale, uint32_t m8, double st) {
  if (variant == NVFP4) return deq_nvfp4(code, scale, st);
  if (variant == MBS_S || variant == MBS_D) return deq_mbs(code, scale, m8);
  return deq_pow2(code, scale);
}

}  // extern "C"
