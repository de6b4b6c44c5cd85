// im2col.cuh — image patches to a column matrix on the GPU.
//
// Replaces the reference's NumPy gather + copy_pad transform
// (pkg/src/tunedblas/routines/extras.py:56-109): the image is channel-major
// with row-major h x w planes; the output is the (C*KH*KW) x (OH*OW) matrix,
// column-major with ld = rows, column q = oy*OW + ox holding the patch at
// output position (oy, ox), row r = (c*KH + ky)*KW + kx, zero where the
// dilated, strided window falls in the padding.  Pure data movement: the
// result is bit-identical to the reference for every precision.
//
// HBM-bound (the output is KH*KW times the image).  A CTA transposes one
// 32 (r) x 64 (q) tile through shared memory so that both global sides are
// coalesced: the gather reads with lanes along q (consecutive output pixels
// -> consecutive image pixels of one row for stride 1), the store writes with
// lanes along r (the column-major output's contiguous dimension).  Index
// arithmetic is per thread and per tile row, not per element.
#pragma once

#include <cstdint>

namespace tb {

struct Im2colGeom {
  int channels, height, width, kh, kw;
  int pad_h, pad_w, stride_h, stride_w, dil_h, dil_w;
  int out_h, out_w;
  int64_t rows, cols;
};

constexpr int IM2COL_TR = 32;  // r per tile (one warp's store width)
constexpr int IM2COL_TQ = 128;  // q per tile (four warp-wide gathers)
constexpr int IM2COL_TY = 8;   // blockDim.y

template <typename T>
__global__ void __launch_bounds__(32 * IM2COL_TY)
    im2col_kernel(const T* __restrict__ im, T* __restrict__ col, Im2colGeom g) {
  __shared__ T tile[IM2COL_TR][IM2COL_TQ + 1];
  __shared__ int r_off[IM2COL_TR], r_dy[IM2COL_TR], r_dx[IM2COL_TR];  // per tile row
  __shared__ int q_y[IM2COL_TQ], q_x[IM2COL_TQ];                      // per tile column
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 32 + tx;
  // 32-bit index math (the host guarantees rows, cols < 2^31).
  const int rows = static_cast<int>(g.rows), cols = static_cast<int>(g.cols);
  const int r0 = static_cast<int>(blockIdx.y) * IM2COL_TR;
  const int q0 = static_cast<int>(blockIdx.x) * IM2COL_TQ;

  // decompose the tile's rows r -> (channel plane, dy, dx) and columns
  // q -> (oy*stride_h, ox*stride_w) once, cooperatively
  if (tid < IM2COL_TR) {
    const int r = min(r0 + tid, rows - 1);
    const int kk = g.kh * g.kw;
    const int c = r / kk, rem = r - c * kk;
    const int ky = rem / g.kw, kx = rem - ky * g.kw;
    r_off[tid] = c * g.height * g.width;
    r_dy[tid] = ky * g.dil_h - g.pad_h;
    r_dx[tid] = kx * g.dil_w - g.pad_w;
  } else if (tid < IM2COL_TR + IM2COL_TQ) {
    const int ql = tid - IM2COL_TR, q = q0 + ql;
    if (q < cols) {
      const int oy = q / g.out_w;
      q_y[ql] = oy * g.stride_h;
      q_x[ql] = (q - oy * g.out_w) * g.stride_w;
    } else {
      q_y[ql] = -(1 << 30);  // out of range: reads as padding
      q_x[ql] = 0;
    }
  }
  __syncthreads();

  // gather: lanes along q (consecutive output pixels -> consecutive image
  // pixels for stride 1), warp-uniform row tables
  constexpr int QH = IM2COL_TQ / 32;
  int qy[QH], qx[QH];
#pragma unroll
  for (int h = 0; h < QH; ++h) {
    qy[h] = q_y[tx + 32 * h];
    qx[h] = q_x[tx + 32 * h];
  }
#pragma unroll
  for (int i = 0; i < IM2COL_TR / IM2COL_TY; ++i) {
    const int rl = ty + IM2COL_TY * i;
    const int off = r_off[rl], dy = r_dy[rl], dx = r_dx[rl];
#pragma unroll
    for (int h = 0; h < QH; ++h) {
      const int y = qy[h] + dy, x = qx[h] + dx;
      const bool ok = static_cast<unsigned>(y) < static_cast<unsigned>(g.height) &&
                      static_cast<unsigned>(x) < static_cast<unsigned>(g.width);
      tile[rl][tx + 32 * h] = ok ? im[off + y * g.width + x] : T(0);
    }
  }
  __syncthreads();

  // store: lanes along r (contiguous in the column-major output)
  const int r = r0 + tx;
  if (r >= rows) return;
  T* out = col + static_cast<int64_t>(q0) * rows + r;
#pragma unroll
  for (int j = 0; j < IM2COL_TQ / IM2COL_TY; ++j) {
    const int ql = ty + IM2COL_TY * j;
    if (q0 + ql < cols) out[static_cast<int64_t>(ql) * rows] = tile[tx][ql];
  }
}

}  // namespace tb
