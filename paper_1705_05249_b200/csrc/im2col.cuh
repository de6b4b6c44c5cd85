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
#include <cstring>
#include <type_traits>

#include "common.cuh"

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

// floor(a / b) for 0 <= a < 2^21 with inv = fl(1/b): exact (the quotient's
// distance to the next integer, >= 1/b, dwarfs the rounding error; checked
// exhaustively for b <= 1024).
__device__ __forceinline__ int im2col_div(int a, float inv) {
  return static_cast<int>((static_cast<float>(a) + 0.5f) * inv);
}

// ---- patch-staged im2col with 16-byte stores ---------------------------------
// The tile kernel above stores 2- or 4-byte values after a shared-memory
// transpose and tests the padding per element: ~1.4 TB/s at the ResNet layer
// even with L2-warm inputs, issue bound.  Here a CTA owns IM2COL_VQ = 128
// consecutive output pixels (a warp per 32) x TR column-matrix rows (TR = one 128-byte
// line per pixel column: 64 rows for H, 32 for S) and
//   1. copies the image patch those rows and pixels touch — the channels of
//      rows [r0, r0 + TR), image rows [y_lo, y_lo + PR), columns
//      [-pad_w, -pad_w + PW) — into shared memory WITH its zero padding, so
//      the gather below has no bounds tests (one coalesced load per patch
//      element, about 1/4 of an output element each);
//   2. per group of VEC rows (one 16-byte vector per pixel), each lane
//      gathers its pixel's VEC values — patch[pixel base + row offset], lanes
//      along consecutive pixels hit consecutive patch columns (no bank
//      conflicts) and the row offsets are broadcast reads of a per-CTA table
//      — packs them, and stores the vector into a warp-private tile at chunk
//      (group ^ (pixel & 7)) (XOR swizzle: conflict-free STS.128);
//   3. writes the tile out with lanes along the rows: 8 lanes per pixel
//      column, one full 128-byte line per pixel per store instruction.
// About 4 instructions per output element (the register-only variants with
// per-element tap stepping and padding tests took ~33 and were issue bound).
// ResNet layer (256 x 56 x 56, 3x3), H: 12.3 us L2-flushed / 7.9 us warm
// against the tile kernel's 14.3-15.2 / 10.3 (8 warps / 256 pixels per CTA:
// 12.45 us; ncu showed SMs idle 42 % of the time with 3-4 CTAs each).  Used for H only: for S (TR =
// 32 rows, patch over-fetch 1.4x) it measured 16.4 / 10.3 against 15.2 /
// 10.3.
// Host conditions (tbgemm.cu tb_im2col): rows a multiple of VEC, a 16-byte
// aligned column matrix, the patch within IM2COL_PATCH_BYTES; otherwise the
// tile kernel runs.  Same values either way.
constexpr int IM2COL_PATCH_BYTES = 15360;
constexpr int IM2COL_VW = 4;                  // warps (32-pixel columns) per CTA
constexpr int IM2COL_VQ = 32 * IM2COL_VW;     // output pixels per CTA

struct Im2colPatch {
  int pw;        // patch columns (the padded x range of an output row)
  int r_chunks;  // TR-row chunks of the column matrix
};

template <typename T>
__global__ void __launch_bounds__(IM2COL_VQ)
    im2col_vec_kernel(const T* __restrict__ im, T* __restrict__ col, Im2colGeom g, Im2colPatch pp) {
  constexpr int VEC = 16 / static_cast<int>(sizeof(T));  // elements per 16-byte vector
  constexpr int TR = 8 * VEC;                              // rows per CTA: 128 bytes per pixel
  __shared__ __align__(16) T patch[IM2COL_PATCH_BYTES / sizeof(T)];
  __shared__ __align__(16) int roff[TR];
  __shared__ __align__(128) uint4 tiles[IM2COL_VW][32 * 8];  // per warp: 32 pixels x 8 vectors
  constexpr int NT = IM2COL_VQ;
  static_assert(NT >= TR, "one thread per row-offset entry");
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rows = static_cast<int>(g.rows), cols = static_cast<int>(g.cols);
  const int q0 = static_cast<int>(blockIdx.x) * IM2COL_VQ, r0 = static_cast<int>(blockIdx.y) * TR;
  const int PW = pp.pw, kk = g.kh * g.kw;
  const int oy_lo = q0 / g.out_w, oy_hi = min(q0 + IM2COL_VQ - 1, cols - 1) / g.out_w;
  const int y_lo = oy_lo * g.stride_h - g.pad_h;
  const int PR = (oy_hi - oy_lo) * g.stride_h + (g.kh - 1) * g.dil_h + 1;
  const int c_lo = r0 / kk, c_hi = (min(r0 + TR, rows) - 1) / kk;
  // 1. patch with zero padding
  const int plane = g.height * g.width;
  const int total = (c_hi - c_lo + 1) * PR * PW;
  const float inv_pw = __frcp_rn(static_cast<float>(PW)), inv_pr = __frcp_rn(static_cast<float>(PR));
  for (int e0 = tid; e0 < total; e0 += 4 * NT) {
    T v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + u * NT;
      const int row = im2col_div(e, inv_pw), x = e - row * PW - g.pad_w;
      const int cl = im2col_div(row, inv_pr), y = y_lo + row - cl * PR;
      const bool ok = e < total && static_cast<unsigned>(y) < static_cast<unsigned>(g.height) &&
                      static_cast<unsigned>(x) < static_cast<unsigned>(g.width);
      const T t = __ldg(im + (ok ? (c_lo + cl) * plane + y * g.width + x : 0));
      v[u] = ok ? t : T(0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (e0 + u * NT < total) patch[e0 + u * NT] = v[u];
  }
  if (tid < TR) {
    const int r = min(r0 + tid, rows - 1);
    const int c = r / kk, rem = r - c * kk;
    const int ky = rem / g.kw, kx = rem - ky * g.kw;
    roff[tid] = ((c - c_lo) * PR + ky * g.dil_h) * PW + kx * g.dil_w;
  }
  __syncthreads();
  // 2. gather into the warp's swizzled tile
  const int qw = q0 + warp * 32;
  if (qw >= cols) return;
  const int qq = min(qw + lane, cols - 1);
  const int oy = qq / g.out_w, ox = qq - oy * g.out_w;
  const int pbase = (oy - oy_lo) * g.stride_h * PW + ox * g.stride_w;
  uint4* tile = tiles[warp];
#pragma unroll
  for (int grp = 0; grp < 8; ++grp) {
    int ro[VEC];
#pragma unroll
    for (int e = 0; e < VEC; e += 4) {
      const int4 r4 = *reinterpret_cast<const int4*>(roff + grp * VEC + e);
      ro[e] = r4.x; ro[e + 1] = r4.y; ro[e + 2] = r4.z; ro[e + 3] = r4.w;
    }
    T v[VEC];
#pragma unroll
    for (int e = 0; e < VEC; ++e) v[e] = patch[pbase + ro[e]];
    uint4 pk;
    memcpy(&pk, v, 16);
    tile[lane * 8 + (grp ^ (lane & 7))] = pk;
  }
  __syncwarp();
  // 3. full-line stores, lanes along the rows
#pragma unroll
  for (int it = 0; it < 8; ++it) {
    const int ql = it * 4 + (lane >> 3), grp = lane & 7;
    const uint4 val = tile[ql * 8 + (grp ^ (ql & 7))];
    const int qo = qw + ql, r = r0 + grp * VEC;
    if (qo < cols && r < rows)  // rows is a multiple of VEC (host)
      *reinterpret_cast<uint4*>(col + static_cast<int64_t>(qo) * rows + r) = val;
  }
}

}  // namespace tb
