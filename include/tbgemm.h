/*
 * tbgemm.h — C-ABI of the B200-native GEMM hot path (libtbgemm.so).
 *
 * This is the drop-in boundary for the reference's GEMM operator interface.
 * The reference (tunedblas, pure Python/NumPy) has no FFI of its own; its
 * internal operator call is
 *     run_kernel(family, config, args, ctx, precision)
 *         pkg/src/tunedblas/kernels/compute.py:116-130
 * with GemmIndirectArgs / GemmDirectArgs (compute.py:80-113) carrying padded
 * NumPy workspaces and slice closures, driven from
 *     _gemm_on_arrays   pkg/src/tunedblas/routines/level3.py:48-91
 *     _gemm_batched_core pkg/src/tunedblas/routines/extras.py:188-286
 * Those carry NumPy arrays and closures and cannot cross a C boundary, so the
 * cut sits just below the routine layer's validation (level3.py:94-133,
 * extras.py:188-348): every argument check happens in the Python host layer
 * (identical error types and text), and these entry points receive plain
 * device pointers, element offsets and leading dimensions — the unpadded
 * operands, exactly as the routine's Buffer views describe them.
 *
 * Conventions
 *   - All pointers (a, b, c and the batched arrays) are DEVICE pointers.
 *   - Offsets, leading dimensions and strides are in ELEMENTS.
 *   - Layout/transpose follow the reference enums (core.py:105-117); for the
 *     real precisions CONJUGATE == TRANS (level3.py:135-146).
 *   - Semantics per element: S computes in FP32 with a
 *     sequential-k FMA chain; H reads FP16, accumulates FP32 on the tensor
 *     cores and rounds once (RNE) to FP16.  Epilogue = alpha*acc, or
 *     alpha*acc + beta*C as three separately rounded FP32 ops (compute.py:
 *     408-412).  beta == 0 never reads C; alpha == 0 or k == 0 never reads
 *     A or B (level3.py:125-132).
 *   - Calls are asynchronous on `stream` (a cudaStream_t, NULL = legacy).
 *   - Return value: TB_OK or a TB_ERR_* status; tb_status_str() explains it.
 *     Argument errors are the host layer's job; the library returns
 *     TB_ERR_INVALID only as a last line of defence.
 */
#ifndef TBGEMM_H_
#define TBGEMM_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TBGEMM_ABI_VERSION 2

/* Precision.H / Precision.S   (core.py:43-50) */
enum { TB_PREC_H = 0, TB_PREC_S = 1 };
/* Layout.ROW_MAJOR / COL_MAJOR (core.py:105-107) */
enum { TB_COL_MAJOR = 0, TB_ROW_MAJOR = 1 };
/* Transpose.NO / YES / CONJUGATE (core.py:110-113) */
enum { TB_NO_TRANS = 0, TB_TRANS = 1, TB_CONJ_TRANS = 2 };

/* Status codes. */
enum {
  TB_OK = 0,
  TB_ERR_INVALID = 1,      /* argument rejected by the library */
  TB_ERR_CUDA = 2,         /* CUDA runtime / launch failure */
  TB_ERR_UNSUPPORTED = 3,  /* e.g. TF32 flag on H, or on unsupported operand layout */
  TB_ERR_DRIVER = 4        /* cuTensorMapEncodeTiled unavailable/failed */
};

/* Flags (bitwise OR). */
enum {
  TB_FLAG_NONE = 0,
  TB_FLAG_TF32 = 1,        /* opt-in TF32 tensor-core SGEMM (separate tolerance;
                              16-byte aligned, K-major operands) */
  TB_FLAG_NO_TMA = 2,      /* HGEMM: force the LDG producer (testing)          */
  TB_FLAG_SIMT_GENERAL = 4, /* SGEMM: force the general predicated kernel        */
  TB_FLAG_NO_PACK = 8,       /* HGEMM: no small-instance packing (testing)        */
  TB_FLAG_NO_2SM = 16,       /* HGEMM: no CTA-pair (cta_group::2) kernel (testing) */
  TB_FLAG_NO_SPLITK = 32,    /* HGEMM: no cluster split-K (testing; results then
                                differ from the default route within tolerance) */
  TB_FLAG_WAVE_SYNC = 64     /* HGEMM: CTA-pair kernel's wave barrier on any size
                                (testing; on by default above ~6 TFLOP per call) */
};

/*
 * sm_100a kernel selection: the "gemm_b200" tuning family
 * (paper_1705_05249_b200/kernels/params.py; DESIGN.md §4 "Tuning space").
 * NULL (or every field 0) = the built-in shape routing.  The reference's 14
 * OpenCL parameters (GemmParams, params.py:120-146) describe an OpenCL
 * work-group decomposition; they are validated and recorded by the Python
 * host layer (LaunchRecord.params) and never cross this boundary.
 *   MWG x NWG  CTA tile.  H: 128 x {64,128,256} (cta_group::1), 256 x 256
 *              (cta_group::2 pair), 128 x 128 (split-K).  S: TMA-fed FFMA2
 *              (KWG 32) 128x128 / 64x128 / 128x64 / 64x64 / 64x32 / 32x32;
 *              register-staged (KWG 16) 128x256 / 128x128 / 64x128 / 128x64
 *              / 64x64.  The library maps a tile onto the instantiation for
 *              the operands' major-ness; tb_last_launch names it.
 *   KWG        K depth per pipeline stage (H 64; S 32 TMA / 16 register-staged)
 *   STAGES     shared-memory ring depth (0 = the instantiation's default)
 *   CTA_GROUP  H: 1 or 2 (tcgen05 cta_group::2 CTA pair)
 *   SPLIT_K    H: cluster split-K factor 1, 2, 4, 8 (DSMEM reduction); S: 1
 *   GROUP_M    grouped-raster height in tiles (0 = the kernel's default)
 */
typedef struct tb_gemm_config {
  int32_t MWG, NWG, KWG, STAGES, CTA_GROUP, SPLIT_K, GROUP_M;
} tb_gemm_config;

/*
 * What the last call on this thread launched (engine.py:128-133 records a
 * LaunchRecord; this is its device-side counterpart).
 */
typedef struct tb_launch_record {
  char kernel[64];         /* instantiation name, e.g. "hgemm_tc_tma_128x256" */
  int64_t grid[3];
  int32_t block[3];
  int32_t cluster[3];
  int32_t smem_bytes;
  int32_t launches;        /* kernels launched by the last call (0 = none) */
  int64_t tiles;           /* output tiles (x batch) the launch covers     */
} tb_launch_record;

/* C = alpha*op(A)*op(B) + beta*C   — replaces level3.py:48-91 → compute.py:384-471 */
int tb_gemm(int prec, int layout, int trans_a, int trans_b, int64_t m,
            int64_t n, int64_t k, float alpha, const void* a, int64_t a_off,
            int64_t lda, const void* b, int64_t b_off, int64_t ldb,
            float beta, void* c, int64_t c_off, int64_t ldc,
            const tb_gemm_config* cfg, int flags, void* stream);

/* Instance i uses base offset + i*stride — replaces extras.py:309-348 → 188-286 */
int tb_gemm_strided_batched(int prec, int layout, int trans_a, int trans_b,
                            int64_t m, int64_t n, int64_t k, float alpha,
                            const void* a, int64_t a_off, int64_t lda,
                            int64_t stride_a, const void* b, int64_t b_off,
                            int64_t ldb, int64_t stride_b, float beta, void* c,
                            int64_t c_off, int64_t ldc, int64_t stride_c,
                            int64_t batch, const tb_gemm_config* cfg,
                            int flags, void* stream);

/*
 * Per-instance offsets and scalars — replaces extras.py:289-306 → 188-286.
 * alphas/betas (float32) and a_offs/b_offs/c_offs (int64) are DEVICE arrays
 * of length `batch`.  `offs_aligned` != 0 asserts every offset is a multiple
 * of 8 elements (H) / 4 elements (S) so vector loads may be used.
 */
int tb_gemm_batched(int prec, int layout, int trans_a, int trans_b, int64_t m,
                    int64_t n, int64_t k, const float* alphas, const void* a,
                    const int64_t* a_offs, int64_t lda, const void* b,
                    const int64_t* b_offs, int64_t ldb, const float* betas,
                    void* c, const int64_t* c_offs, int64_t ldc, int64_t batch,
                    int offs_aligned, const tb_gemm_config* cfg, int flags,
                    void* stream);

/*
 * Image patches to columns — replaces extras.py:56-109 (im2col).  `im` holds
 * channels x height x width (row-major planes) from element `im_off`; `col`
 * receives the (channels*kernel_h*kernel_w) x (out_h*out_w) column-major
 * matrix (ld = rows) from element `col_off`, zeros where the window falls in
 * the padding (negative padding crops, as in the reference).  Device
 * pointers; geometry validated by the caller (the
 * Python routine raises the reference's UsageError / RangeError first);
 * returns TB_ERR_INVALID for non-positive output dimensions.
 */
int tb_im2col(int prec, int64_t channels, int64_t height, int64_t width,
              int64_t kernel_h, int64_t kernel_w, int64_t pad_h, int64_t pad_w,
              int64_t stride_h, int64_t stride_w, int64_t dilation_h,
              int64_t dilation_w, const void* im, int64_t im_off, void* col,
              int64_t col_off, void* stream);

/*
 * Implicit GEMM: convolution as im2col + GEMM without materialising the
 * column matrix (the composition the reference's im2col
 * exists for, extras.py:56-109: "a weights-as-rows GEMM against it equals
 * direct cross-correlation").  For each of `batch` images (channel-major,
 * instance b at im + im_off + b*channels*height*width):
 *   result[b][f][q] = sum_r kernel[f][r] * col_b[r][q]
 * with col_b the reference's im2col matrix (r = (ch*kernel_h + ky)*kernel_w +
 * kx, q = oy*out_w + ox), `kernel` num_kernels x (channels*kernel_h*kernel_w)
 * row-major from kernel_off, `result` batch x num_kernels x (out_h*out_w)
 * from result_off (NCHW).  H: FP16 in/out, FP32 accumulation on tcgen05;
 * S: the FP32 sequential-k chain (bitwise im2col + gemm).  Device pointers.
 */
int tb_convgemm(int prec, int64_t channels, int64_t height, int64_t width,
                int64_t kernel_h, int64_t kernel_w, int64_t pad_h, int64_t pad_w,
                int64_t stride_h, int64_t stride_w, int64_t dilation_h,
                int64_t dilation_w, int64_t num_kernels, int64_t batch,
                const void* im, int64_t im_off, const void* kernel,
                int64_t kernel_off, void* result, int64_t result_off, int flags,
                void* stream);

/*
 * Structured level-3 helpers — the reference's transform kinds
 * (kernels/transforms.py:21-147) used by symm/syrk/syr2k/trmm/trsm
 * (routines/level3.py:152-537).  Column-major storage, element offsets.
 *   kind TB_XF_COPY          dst = src                      (rows x cols)
 *   kind TB_XF_SYMMETRIZE    dst = src's `upper` triangle mirrored (square)
 *   kind TB_XF_TRIANGULARIZE dst = src's triangle, zeros elsewhere, unit diag
 *   kind TB_XF_TRI_COPY      dst's triangle = src's triangle, rest untouched
 */
enum { TB_XF_COPY = 0, TB_XF_SYMMETRIZE = 1, TB_XF_TRIANGULARIZE = 2, TB_XF_TRI_COPY = 3 };
int tb_transform(int prec, int kind, int64_t rows, int64_t cols, const void* src,
                 int64_t src_off, int64_t lds, void* dst, int64_t dst_off,
                 int64_t ldd, int upper, int unit, void* stream);
/* FP32 staging (trsm keeps X in FP32, level3.py:474-483):
 * to_f32 (direction 0): dst_f32 = alpha * op(src);  from_f32 (1): dst = RNE(op(src_f32)).
 * op = transpose ? ^T : identity; rows x cols are the DESTINATION's. */
int tb_convert_f32(int prec, int direction, int64_t rows, int64_t cols, float alpha,
                   const void* src, int64_t src_off, int64_t lds, int transpose,
                   void* dst, int64_t dst_off, int64_t ldd, void* stream);
/* Substitution on one nb x nb (nb <= 64) diagonal block of a dense FP32
 * triangular T for ncols right-hand sides X (level2.py:365-387). */
int tb_trsm_block(int64_t nb, int64_t ncols, const float* t, int64_t t_off,
                  int64_t ldt, float* x, int64_t x_off, int64_t ldx, int upper,
                  int unit, void* stream);

/* Allocate the per-device state a launch may need (the CTA-pair kernel's
 * wave-barrier counters) on the current device, outside any stream capture,
 * so later calls allocate nothing.  Idempotent. */
int tb_prepare_device(void);

/* Fill the record of the last launch issued from the calling thread. */
int tb_last_launch(tb_launch_record* out);
/* Human-readable text for a status code (static storage). */
const char* tb_status_str(int status);
/* Text of the last CUDA error seen by the library on this thread. */
const char* tb_last_error(void);
/* TBGEMM_ABI_VERSION of the loaded library. */
int tb_abi_version(void);
/* Number of SMs on the current device (0 if no device). */
int tb_device_sm_count(void);

#ifdef __cplusplus
}
#endif

#endif /* TBGEMM_H_ */
