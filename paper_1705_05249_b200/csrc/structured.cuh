// structured.cuh — helper kernels for the structured level-3 routines
// (SURVEY §8f row 2): symm / syrk / syr2k / trmm / trsm reuse the GPU GEMM,
// exactly as the reference reuses _gemm_on_arrays
// (pkg/src/tunedblas/routines/level3.py:152-537).
//
//  * transform_kernel: the reference's transform kinds on column-major
//    storage (kernels/transforms.py:21-147): plain copy, symmetrize (mirror
//    the stored triangle), triangularize (zero the other triangle, optional
//    unit diagonal) and the triangle-masked copy of the rank-k updates
//    (level3.py:233-246).  Raw 16/32-bit element moves: exact.
//  * f32 staging for trsm (the reference keeps X in the compute dtype, FP32,
//    for every precision and rounds once at the end, level3.py:474-483):
//    to_f32 (alpha * op(src), one rounding) and from_f32 (RNE to FP16).
//  * trsm_block_kernel: substitution of one diagonal block
//    (routines/level2.py:365-387), one thread per right-hand-side column, the
//    block's triangle staged in shared memory.
#pragma once

#include <cuda_fp16.h>

#include <cstdint>

namespace tb {

enum { XF_COPY = 0, XF_SYMMETRIZE = 1, XF_TRIANGULARIZE = 2, XF_TRI_COPY = 3 };

template <typename T>
__global__ void transform_kernel(int kind, int64_t rows, int64_t cols, const T* __restrict__ src, int64_t lds,
                                 T* __restrict__ dst, int64_t ldd, int upper, int unit, T one) {
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = e / rows, i = e - j * rows;
    const bool in_tri = upper ? (i <= j) : (i >= j);
    T* d = dst + i + j * ldd;
    switch (kind) {
      case XF_COPY:
        *d = src[i + j * lds];
        break;
      case XF_SYMMETRIZE:
        *d = in_tri ? src[i + j * lds] : src[j + i * lds];
        break;
      case XF_TRIANGULARIZE:
        *d = !in_tri ? T(0) : ((unit && i == j) ? one : src[i + j * lds]);
        break;
      default:  // XF_TRI_COPY
        if (in_tri) *d = src[i + j * lds];
        break;
    }
  }
}

template <typename T>
__device__ __forceinline__ float elem_to_f32(T v);
template <>
__device__ __forceinline__ float elem_to_f32<__half>(__half v) {
  return __half2float(v);
}
template <>
__device__ __forceinline__ float elem_to_f32<float>(float v) {
  return v;
}
template <typename T>
__device__ __forceinline__ T f32_to_elem(float v);
template <>
__device__ __forceinline__ __half f32_to_elem<__half>(float v) {
  return __float2half_rn(v);
}
template <>
__device__ __forceinline__ float f32_to_elem<float>(float v) {
  return v;
}

// dst (FP32, rows x cols, ld ldd) = alpha * (transpose ? src^T : src)
template <typename T>
__global__ void to_f32_kernel(int64_t rows, int64_t cols, float alpha, const T* __restrict__ src, int64_t lds,
                              int transpose, float* __restrict__ dst, int64_t ldd) {
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = e / rows, i = e - j * rows;
    const float v = elem_to_f32<T>(transpose ? src[j + i * lds] : src[i + j * lds]);
    dst[i + j * ldd] = __fmul_rn(alpha, v);
  }
}

// dst (T, rows x cols, ld ldd) = RNE(transpose ? src^T : src), src FP32
template <typename T>
__global__ void from_f32_kernel(int64_t rows, int64_t cols, const float* __restrict__ src, int64_t lds,
                                int transpose, T* __restrict__ dst, int64_t ldd) {
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = e / rows, i = e - j * rows;
    dst[i + j * ldd] = f32_to_elem<T>(transpose ? src[j + i * lds] : src[i + j * lds]);
  }
}

constexpr int TRSM_MAX_NB = 64;

// Solve T X = X in place for one nb x nb diagonal block T (FP32, column-major,
// ld ldt) and the nb x ncols block X (ld ldx): x_i = (x_i - sum_k t_ik x_k) / t_ii
// in ascending (lower) or descending (upper) i, the sum accumulated in
// ascending k (level2.py:365-387).
__global__ void trsm_block_kernel(int nb, int64_t ncols, const float* __restrict__ t, int64_t ldt,
                                  float* __restrict__ x, int64_t ldx, int upper, int unit) {
  __shared__ float ts[TRSM_MAX_NB * TRSM_MAX_NB];
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    const int j = e / nb, i = e - j * nb;
    ts[i + j * nb] = t[i + j * ldt];
  }
  __syncthreads();
  const int64_t col = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (col >= ncols) return;
  float xv[TRSM_MAX_NB];
  float* xc = x + col * ldx;
#pragma unroll 4
  for (int i = 0; i < nb; ++i) xv[i] = xc[i];
  if (!upper) {
    for (int i = 0; i < nb; ++i) {
      float s = 0.0f;
      for (int k = 0; k < i; ++k) s = __fmaf_rn(ts[i + k * nb], xv[k], s);
      float v = __fsub_rn(xv[i], s);
      if (!unit) v = __fdiv_rn(v, ts[i + i * nb]);
      xv[i] = v;
    }
  } else {
    for (int i = nb - 1; i >= 0; --i) {
      float s = 0.0f;
      for (int k = i + 1; k < nb; ++k) s = __fmaf_rn(ts[i + k * nb], xv[k], s);
      float v = __fsub_rn(xv[i], s);
      if (!unit) v = __fdiv_rn(v, ts[i + i * nb]);
      xv[i] = v;
    }
  }
#pragma unroll 4
  for (int i = 0; i < nb; ++i) xc[i] = xv[i];
}

// Register-resident version for full NB x NB blocks (NB = 16 / 32): both
// loops fully unrolled, x stays in registers; same operation order as
// trsm_block_kernel.
template <int NB>
__global__ void __launch_bounds__(64) trsm_block_reg_kernel(int64_t ncols, const float* __restrict__ t, int64_t ldt,
                                                            float* __restrict__ x, int64_t ldx, int upper, int unit) {
  __shared__ float ts[NB * NB];
  for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
    const int j = e / NB, i = e - j * NB;
    ts[i + j * NB] = t[i + j * ldt];
  }
  __syncthreads();
  const int64_t col = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (col >= ncols) return;
  float xv[NB];
  float* xc = x + col * ldx;
#pragma unroll
  for (int i = 0; i < NB; ++i) xv[i] = xc[i];
  if (!upper) {
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      float s = 0.0f;
#pragma unroll
      for (int k = 0; k < i; ++k) s = __fmaf_rn(ts[i + k * NB], xv[k], s);
      float v = __fsub_rn(xv[i], s);
      if (!unit) v = __fdiv_rn(v, ts[i + i * NB]);
      xv[i] = v;
    }
  } else {
#pragma unroll
    for (int i = NB - 1; i >= 0; --i) {
      float s = 0.0f;
#pragma unroll
      for (int k = i + 1; k < NB; ++k) s = __fmaf_rn(ts[i + k * NB], xv[k], s);
      float v = __fsub_rn(xv[i], s);
      if (!unit) v = __fdiv_rn(v, ts[i + i * NB]);
      xv[i] = v;
    }
  }
#pragma unroll
  for (int i = 0; i < NB; ++i) xc[i] = xv[i];
}

}  // namespace tb
