/*
 * mxq200.h -- C ABI of the B200-native MXFP4 quantize-and-GEMM path.
 *
 * This is the drop-in boundary for the hot path of arxiv 2603.08713's
 * reference package `mxq` (pure Python + numpy, /root/reference/pkg/src/mxq;
 * written src/... below).  The reference has no FFI of its own: its boundary
 * is the Python module surface re-exported in src/__init__.py:4-66.  Each
 * entry point here replaces the numpy implementation of one of those Python
 * functions; the Python host package `paper_2603_08713_b200` binds them with
 * ctypes (the binding a maintainer would add is shown in INTEGRATION.md).
 *
 * Conventions
 *  - Every function returns int: 0 = ok, < 0 = invalid argument / unsupported
 *    (the wrapper raises ValueError / NotImplementedError), > 0 = a CUDA error
 *    code.  mxq_last_error() returns the message of the last failure on the
 *    calling thread.
 *  - All tensor buffers are caller-allocated DEVICE pointers (PyTorch owns
 *    the memory); launches are stream-ordered on the caller's stream.
 *  - Data-dependent errors (non-finite input, corrupt scale codes) are
 *    reported asynchronously through `scratch[0]` (MXQ_ST_* bits); the caller
 *    synchronises and raises the reference's message.
 *  - No global mutable state other than a per-device TMA-descriptor-free
 *    launch configuration cache and the thread-local error string.
 */
#ifndef MXQ200_H
#define MXQ200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- variants (src/quantize.py:70-76) ------------------------------------ */
#define MXQ_OCP32 0
#define MXQ_MX16 1
#define MXQ_MX16_OAS 2
#define MXQ_MBS_S 3
#define MXQ_MBS_D 4
#define MXQ_NVFP4 5

/* ---- element dtypes of dense inputs / outputs --------------------------- */
#define MXQ_F32 0
#define MXQ_BF16 1

/* ---- return codes -------------------------------------------------------- */
#define MXQ_OK 0
#define MXQ_ERR_INVALID (-1)     /* bad argument: wrapper raises ValueError     */
#define MXQ_ERR_NONFINITE (-2)   /* host scalar helpers: non-finite input       */
#define MXQ_ERR_UNSUPPORTED (-3) /* combination not implemented on this path    */
#define MXQ_ERR_RANGE (-4)       /* host scalar helpers: |v| > 6, no saturate   */

/* ---- device status bits in scratch[0] ------------------------------------ */
#define MXQ_ST_NONFINITE 1u   /* src/quantize.py:581-582 "tensor contains non-finite elements" */
#define MXQ_ST_BAD_E8M0 2u    /* src/quantize.py:239-240 "corrupt block scale: E8M0 code 255"  */
#define MXQ_ST_BAD_E4M3 4u    /* src/quantize.py:235-236 "corrupt block scale: E4M3 NaN code"  */
#define MXQ_ST_OVERFLOW 8u    /* f32 MBS factor multiply overflowed (src/formats.py:197)       */

/*
 * A quantized 2-D tensor (the device image of src/quantize.py:173-193
 * QuantizedTensor).  Field meaning follows the reference: `codes` packs two
 * E2M1 codes per byte, even column in the low nibble; `scales` holds one byte
 * per 1 x block_size block (E8M0 biased exponent of the dequant multiplier D,
 * or the E4M3 byte for NVFP4); `mant` holds the MBS mantissa byte per macro
 * block; `tensor_scale` is the NVFP4 f64 s_t (device scalar).
 *
 * GEMM-side copies (either may be NULL when not needed):
 *  - scales_mma: the tcgen05 scale-factor atom layout, 512-byte atoms of
 *    128 rows x 4 blocks ordered [row/128][block/4], byte
 *    (r%32)*16 + ((r%128)/32)*4 + block%4.  Rows padded to a multiple of 256,
 *    blocks per row padded to `sf_kpad` (a multiple of 256/block_size).
 *  - sig_t: the MBS factor sigma = 1/(1+m8/256) as f32, transposed to
 *    (n_macros, sig_t_ld >= rows) so a GEMM chunk reads it contiguously.
 */
typedef struct mxq_qtensor {
  int32_t variant;     /* MXQ_OCP32 .. MXQ_NVFP4 */
  int32_t block_size;  /* 32 for OCP32, else 16 */
  int32_t macro_size;  /* MBS macro width (multiple of block_size) */
  int32_t sf_format;   /* GEMM only: 0 = the variant's own scale format in scales_mma (UE8M0, or UE4M3 for
                          NVFP4); 1 = scales_mma holds the UE8M0 block scales re-expressed as UE4M3 powers of
                          two (mixed UE8M0 x NVFP4 pairs; the caller folds the power-of-two offset into the
                          NVFP4 side's tensor_scale) */
  int64_t rows, cols;
  uint8_t* codes;       int64_t codes_ld;   /* bytes between rows, >= cols/2   */
  uint8_t* scales;      int64_t scales_ld;  /* bytes between rows, >= cols/bs  */
  uint8_t* scales_mma;  int64_t sf_kpad;    /* padded blocks per row            */
  uint8_t* mant;        int64_t mant_ld;    /* (rows, n_macros) mantissa bytes  */
  float* sig_t;         int64_t sig_t_ld;   /* (n_macros, rows) sigma = 1/(1+m8/256), f32 */
  double* tensor_scale;                     /* NVFP4 s_t (device f64)           */
} mxq_qtensor;

/* ---- library ------------------------------------------------------------- */
int mxq_version(void);
const char* mxq_last_error(void);
/* 1 when a CUDA device of compute capability 10.0 is present. */
int mxq_device_ok(void);
/* Development aid: device buffer (>= 512*4 int64) for a clock64() trace of
 * CTA 0's MMA/epilogue hand-offs in subsequent GEMM launches; NULL disables. */
void mxq_debug_set_trace(long long* dev_buf);

/*
 * Quantize a dense (rows, cols) f32/bf16 device tensor `x` (row stride x_ld
 * elements) into `q` (whose buffers the caller allocated).
 * Replaces: quantize_tensor  src/quantize.py:709-725
 *           _quantize_power_of_two :586-609, _quantize_mbs :612-659,
 *           quantize_nvfp4 :662-706 (two passes: amax, then encode).
 * mbs_mode must be 0 (exact SSE search, src/quantize.py:438-461); the lut
 * mode has its own entry point below.  cand/n_cand: HOST array of candidate bytes
 * (CandidateSet.mantissas); augment_static as SchemeConfig.augment_static.
 * scratch: device u32[4] (scratch[0] status bits, scratch[1] NVFP4 amax); the call
 * zeroes the four words before its kernels run.
 */
int mxq_quantize(const void* x, int32_t x_dtype, int64_t x_ld, const mxq_qtensor* q, int32_t mbs_mode,
                 const uint8_t* cand, int32_t n_cand, int32_t augment_static, uint32_t* scratch, void* stream);

/*
 * MBS-D lookup-table mode: candidate cost sum(x^2 * T[v]) from the 2x16x64
 * table of build_error_lut (HOST f32 copy of the fp16 entries,
 * [regime][candidate][bin]); exactly 16 candidates, no static augmentation.
 * Replaces: _choose_dynamic_lut src/quantize.py:507-542 (+ _quantize_macros).
 */
int mxq_quantize_mbs_lut(const void* x, int32_t x_dtype, int64_t x_ld, const mxq_qtensor* q, const uint8_t* cand,
                         int32_t n_cand, const float* lut_entries, uint32_t* scratch, void* stream);

/*
 * Dequantize to f32 (rows, cols), row stride out_ld.
 * Replaces: dequantize_tensor src/quantize.py:728-746 (_dequantize_values :409-423).
 */
int mxq_dequantize(const mxq_qtensor* q, float* out, int64_t out_ld, uint32_t* scratch, void* stream);

/*
 * QSNR / flush-to-zero evaluator.  Sums sum(ref^2) and sum((ref-x)^2) in f64
 * in numpy's pairwise order (bit-identical to the reference's np.sum), where
 * x is either the dequantization of `q` (fused, q != NULL) or the dense f32
 * tensor `recon`.  out4 (device f64[4]) receives
 *   {signal, error, count(ref != 0), count(ref != 0 && code magnitude == 0)}
 * (the flush counts only when q != NULL).
 * Replaces: qsnr_tensor src/metrics.py:127-153, flush_to_zero_rate :165-182.
 * workspace: device buffer of mxq_qsnr_workspace_bytes(rows*cols) bytes.
 */
int64_t mxq_qsnr_workspace_bytes(int64_t n);
int mxq_qsnr(const void* ref, int32_t ref_dtype, int64_t ref_ld, const mxq_qtensor* q, const float* recon,
             int64_t recon_ld, int64_t rows, int64_t cols, void* workspace, double* out4, uint32_t* scratch,
             void* stream);

/*
 * Block-scaled tcgen05 GEMM  C[M,N] = A[M,K] . B[N,K]^T  on quantized
 * operands (K-major codes, scales_mma, and for MBS operands sig_t).
 * Replaces: matmul_quantized src/gemm.py:137-172 (tolerance parity: the MMA
 * accumulates FP4 products in f32 per 64-K step; the MBS factor
 * sigma = 1/(1+m8/256) of each operand is applied per 128-K macro chunk
 * in the epilogue).
 * Supported pairs: any two of {OCP32, MX16, MX16_OAS, MBS_S, MBS_D}
 * (UE8M0 scales; OCP32 x OCP32 runs kind::mxf4 block32, everything else
 * kind::mxf4nvf4 block16 with UE8M0 after expanding block-32 scales), and
 * NVFP4 x NVFP4 (kind::mxf4nvf4 block16 UE4M3, epilogue x s_tA*s_tB).
 * UE8M0 x UE4M3 pairs return MXQ_ERR_UNSUPPORTED (use mxq_gemm_exact).
 * c_dtype: MXQ_F32 or MXQ_BF16; ldc in elements.
 */
int mxq_gemm(const mxq_qtensor* a, const mxq_qtensor* b, void* c, int32_t c_dtype, int64_t ldc, uint32_t* scratch,
             void* stream);

/*
 * Grouped decode GEMMs (MoE experts; SURVEY section 8 d config 5): the n
 * independent products C_g = A_g . B_g^T (matmul_quantized src/gemm.py:137-172
 * per group), A_g the tokens routed to expert g (<= 128 rows), B_g the
 * expert's weights, every B_g of one shape.  a, b: HOST arrays of n
 * descriptors; c: HOST array of n device output pointers (row stride ldc).
 * When the pairs are MBS / E8M0 pairs of one variant pair and macro size, all
 * groups run in one launch of the MBS kernel per 64 groups (swap-AB up to
 * 64 tokens, direct 128-row tiles up to 128); otherwise
 * one mxq_gemm launch per group.  Same tolerance parity as mxq_gemm.
 */
int mxq_gemm_grouped(const mxq_qtensor* a, const mxq_qtensor* b, int32_t n, void* const* c, int32_t c_dtype,
                     int64_t ldc, uint32_t* scratch, void* stream);

/*
 * Activation quantization fused with the GEMM:
 * quantize the dense activation x (rows a->rows, cols a->cols, MBS-S with
 * a->macro_size; the reference runs quantize_tensor src/quantize.py:709-725
 * then matmul_quantized src/gemm.py:137-172) into `a`, then C = A . B^T.
 * For bf16 x (32-byte aligned rows) against an MBS/E8M0 B with more than 64
 * rows of A, both run in ONE launch of the MBS GEMM: every CTA first
 * quantizes its share of A's 128-row blocks and the GEMM consumes a block as
 * soon as it is published.  Otherwise the call makes the two launches.  `a`
 * and C are bit-identical to mxq_quantize followed by mxq_gemm either way.
 * a must be MBS_S and carry scales_mma and sig_t (scales / mant optional).
 * scratch: device u32[4] as for mxq_quantize; scratch[2] is the launch's
 * published-slice counter (zeroed by the call).
 */
int mxq_quantize_gemm(const void* x, int32_t x_dtype, int64_t x_ld, const mxq_qtensor* a, const mxq_qtensor* b,
                      void* c, int32_t c_dtype, int64_t ldc, uint32_t* scratch, void* stream);

/*
 * Reference-exact GEMM on CUDA cores: every element is the dequantized f32
 * value, products and sums in f64 with k ascending and no FMA, one final
 * rounding -- bit-identical to matmul_reference(dequantize(a), dequantize(b))
 * (src/gemm.py:68-90, :137-172) for every variant pair.
 */
int mxq_gemm_exact(const mxq_qtensor* a, const mxq_qtensor* b, float* c, int64_t ldc, uint32_t* scratch,
                   void* stream);

/* f32 x f32^T with the same exact f64 ascending-k contract.
 * Replaces: matmul_reference src/gemm.py:68-90. */
int mxq_matmul_reference(const float* a, int64_t lda, const float* b, int64_t ldb, int64_t m, int64_t n, int64_t k,
                         float* c, int64_t ldc, void* stream);

/* Build the GEMM-side copies (scales_mma, sig_t) from the row-major fields
 * of a user-constructed QuantizedTensor. */
int mxq_build_gemm_layout(const mxq_qtensor* q, int32_t sf_block, void* stream);

/* ---- host scalar helpers: the same arithmetic header compiled for the CPU --
 * Replace the per-block / scalar API of src/formats.py:154-316 and
 * src/quantize.py:301-479.  No GPU needed. */
int mxq_host_encode_e2m1(const double* v, int64_t n, int32_t saturate, uint8_t* out);  /* src/formats.py:154-200 */
int mxq_host_encode_e4m3(const double* v, int64_t n, uint8_t* out);                    /* src/formats.py:260-292 */
int mxq_host_e8m0_floor(double x, uint8_t* biased, int32_t* clamped);                  /* src/formats.py:210-227 */
int mxq_host_extract_mantissa8(double sf, uint8_t* m8);                                /* src/formats.py:303-316 */
/* kind: 0 = OCP32 (n == 32), 1 = MX16, 2 = MX16 + OAS (n == 16).
 * src/quantize.py:301-334 */
int mxq_host_block_scale(const double* block, int64_t n, int32_t kind, uint8_t* biased, int32_t* clamped);
int mxq_host_static_m8(double alpha, uint8_t* m8);
/* The kernels' integer E8M0 closed form on f32 block maxima,
 * compiled for the host so it can be checked against the reference formula
 * without a GPU.  kind as mxq_host_block_scale. */
int mxq_host_e8m0_closed_form(const float* alpha, int64_t n, int32_t kind, uint8_t* out);                                     /* src/quantize.py:369-380 */
/* MBS-D choice for one macro (n floats, n % 16 == 0): exact SSE search when
 * lut == NULL (src/quantize.py:464-479), else the LUT cost with the
 * [2][16][64] f32 table (src/quantize.py:545-560).  augment_static appends the
 * static mantissa (exact mode only). */
int mxq_host_mbs_choose(const float* x, int64_t n, const uint8_t* cand, int32_t n_cand, int32_t augment_static,
                        const float* lut, uint8_t* m8);
/* Dequantized element f32(g*D/f*s_t) for one code (src/quantize.py:409-423).
 * variant selects the formula; m8 ignored unless MBS; st unless NVFP4. */
float mxq_host_dequant_element(int32_t variant, uint32_t code, uint32_t scale, uint32_t m8, double st);

#ifdef __cplusplus
}
#endif

#endif /* MXQ200_H */
