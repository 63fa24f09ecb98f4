// mxq_internal.h -- shared host/device declarations for the C-ABI library.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "../../include/mxq200.h"

namespace mxq {

using QDesc = mxq_qtensor;

enum { DT_F32 = MXQ_F32, DT_BF16 = MXQ_BF16 };
enum { ERR_INVALID = MXQ_ERR_INVALID, ERR_UNSUPPORTED = MXQ_ERR_UNSUPPORTED };

int set_error(int code, const char* msg);
int set_cuda_error(cudaError_t e);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device):
// `done` is the caller's per-kernel static, one bit per device ordinal.
template <typename K>
inline int smem_attr_once(K kern, int smem, std::atomic<uint64_t>& done) {
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return 0;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return set_cuda_error(e);
  done.fetch_or(bit, std::memory_order_release);
  return 0;
}
int check_launch();
int num_sms();

int launch_quantize(const void* x, int dtype, int64_t x_ld, const QDesc& q, int mbs_mode, const uint8_t* cand,
                    int n_cand, int augment, uint32_t* status, cudaStream_t st);
int launch_quantize_lut(const void* x, int dtype, int64_t x_ld, const QDesc& q, const uint8_t* cand, int n_cand,
                        const float* lut, uint32_t* status, cudaStream_t st);
int launch_dequantize(const QDesc& q, float* out, int64_t out_ld, uint32_t* status, cudaStream_t st);
int64_t qsnr_workspace_bytes(int64_t n);
int launch_qsnr(const void* ref, int dtype, int64_t ref_ld, const QDesc* q, const float* recon, int64_t recon_ld,
                int64_t rows, int64_t cols, void* ws, double* out4, uint32_t* status, cudaStream_t st);
int launch_gemm_exact(const QDesc* a, const QDesc* b, const float* fa, int64_t lda, const float* fb, int64_t ldb,
                      int64_t m, int64_t n, int64_t k, float* c, int64_t ldc, uint32_t* status, cudaStream_t st);
int launch_gemm_tc(const QDesc& a, const QDesc& b, void* c, int c_dtype, int64_t ldc, uint32_t* status,
                   cudaStream_t st);
bool gemm_mbs_supported(const QDesc& a, const QDesc& b);
int launch_gemm_mbs(const QDesc& a, const QDesc& b, void* c, int c_dtype, int64_t ldc, cudaStream_t st);
bool gemm_mbs_fusable(const QDesc& a, const QDesc& b, int x_dtype);
int launch_gemm_mbs_grouped(const QDesc* a, const QDesc* b, int n, void* const* c, int c_dtype, int64_t ldc,
                            cudaStream_t st);
int launch_gemm_mbs_fused(const void* x, int64_t x_ld, const QDesc& a, const QDesc& b, void* c, int c_dtype,
                          int64_t ldc, uint32_t* status, cudaStream_t st);
void set_gemm_trace(long long* p);
int launch_build_gemm_layout(const QDesc& q, int sf_block, cudaStream_t st);

}  // namespace mxq
