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
// HBM-bound in principle (the output is KH*KW times the image); the first
// version was instruction-bound (ncu: 72 % issue slots, ~40 SASS instructions
// per element: per-element address IMADs, a branch around every predicated
// gather, 2-byte stores).  A CTA transposes one TR (r) x 128 (q) tile through
// shared memory stored [q][TR + VEC] (132-byte rows: conflict-free on both
// sides): the gather reads with lanes along q (consecutive output pixels ->
// consecutive image pixels for stride 1) from precomputed row and pixel
// address terms (one IADD per element, branch-free: out-of-window elements
// load element 0 and are zeroed by a select), the store writes 4 bytes per
// lane along r (VEC = 2 halves or 1 float; 128 bytes per warp store).
#pragma once

#include <cstdint>

namespace tb {

struct Im2colGeom {
  int channels, height, width, kh, kw;
  int pad_h, pad_w, stride_h, stride_w, dil_h, dil_w;
  int out_h, out_w;
  int64_t rows, cols;
};

constexpr int IM2COL_TQ = 128;  // q per tile (four warp-wide gathers)
constexpr int IM2COL_TY = 8;    // blockDim.y
template <typename T>
struct Im2colTile {
  static constexpr int VEC = 4 / static_cast<int>(sizeof(T));  // elements per 4-byte store
  static constexpr int TR = 32 * VEC;                            // r per tile
  static constexpr int LD = TR + VEC;                            // 33 words per smem row
};

// VEC4: the output column starts and rows are 4-byte aligned (host-checked),
// so each lane stores VEC consecutive r as one 32-bit word.
template <typename T, bool VEC4>
__global__ void __launch_bounds__(32 * IM2COL_TY)
    im2col_kernel(const T* __restrict__ im, T* __restrict__ col, Im2colGeom g) {
  using Tl = Im2colTile<T>;
  constexpr int TR = Tl::TR, LD = Tl::LD, VEC = Tl::VEC;
  __shared__ __align__(16) T tile[IM2COL_TQ * LD];
  __shared__ int r_base[TR], r_dy[TR], r_dx[TR];  // per tile row: address term, window offsets
  __shared__ int q_y[IM2COL_TQ], q_x[IM2COL_TQ], q_base[IM2COL_TQ];
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 32 + tx;
  // 32-bit index math (the host guarantees rows, cols, C*H*W < 2^31).
  const int rows = static_cast<int>(g.rows), cols = static_cast<int>(g.cols);
  const int r0 = static_cast<int>(blockIdx.y) * TR;
  const int q0 = static_cast<int>(blockIdx.x) * IM2COL_TQ;

  // decompose the tile's rows r -> (channel plane, dy, dx) and columns
  // q -> (oy*stride_h, ox*stride_w) once, cooperatively; the image address
  // of element (r, q) is r_base[r] + q_base[q]
  if (tid < TR) {
    const int r = min(r0 + tid, rows - 1);
    const int kk = g.kh * g.kw;
    const int c = r / kk, rem = r - c * kk;
    const int ky = rem / g.kw, kx = rem - ky * g.kw;
    const int dy = ky * g.dil_h - g.pad_h, dx = kx * g.dil_w - g.pad_w;
    r_base[tid] = c * g.height * g.width + dy * g.width + dx;
    r_dy[tid] = dy;
    r_dx[tid] = dx;
  } else if (tid < TR + IM2COL_TQ) {
    const int ql = tid - TR, q = q0 + ql;
    if (q < cols) {
      const int oy = q / g.out_w;
      const int y = oy * g.stride_h, x = (q - oy * g.out_w) * g.stride_w;
      q_y[ql] = y;
      q_x[ql] = x;
      q_base[ql] = y * g.width + x;
    } else {
      q_y[ql] = -(1 << 29);  // out of range: reads as padding
      q_x[ql] = 0;
      q_base[ql] = 0;
    }
  }
  __syncthreads();

  // gather: lanes along q, warp-uniform row terms
  constexpr int QH = IM2COL_TQ / 32;
  int qy[QH], qx[QH], qb[QH];
#pragma unroll
  for (int h = 0; h < QH; ++h) {
    qy[h] = q_y[tx + 32 * h];
    qx[h] = q_x[tx + 32 * h];
    qb[h] = q_base[tx + 32 * h];
  }
  // all of this thread's gathers are issued before the first shared store,
  // so their latencies overlap (one L2/DRAM round trip per tile, not one per
  // tile row)
  const unsigned H = static_cast<unsigned>(g.height), W = static_cast<unsigned>(g.width);
  constexpr int RI = TR / IM2COL_TY;
  T v[RI][QH];
#pragma unroll
  for (int i = 0; i < RI; ++i) {
    const int rl = ty + IM2COL_TY * i;
    const int base = r_base[rl], dy = r_dy[rl], dx = r_dx[rl];
#pragma unroll
    for (int h = 0; h < QH; ++h) {
      const bool ok = static_cast<unsigned>(qy[h] + dy) < H && static_cast<unsigned>(qx[h] + dx) < W;
      const T x = __ldg(im + (ok ? base + qb[h] : 0));
      v[i][h] = ok ? x : T(0);
    }
  }
#pragma unroll
  for (int i = 0; i < RI; ++i)
#pragma unroll
    for (int h = 0; h < QH; ++h) tile[(tx + 32 * h) * LD + ty + IM2COL_TY * i] = v[i][h];
  __syncthreads();

  // store: lanes along r (contiguous in the column-major output), VEC
  // elements (4 bytes) per lane
  const int r = r0 + tx * VEC;
  if (r >= rows) return;
  T* out = col + static_cast<int64_t>(q0) * rows + r;
  const int64_t step = static_cast<int64_t>(IM2COL_TY) * rows;
  out += static_cast<int64_t>(ty) * rows;
  const bool full_vec = VEC4 && r + VEC <= rows;
#pragma unroll 4
  for (int ql = ty; ql < IM2COL_TQ; ql += IM2COL_TY, out += step) {
    if (q0 + ql >= cols) break;
    const T* src = tile + ql * LD + tx * VEC;
    if (full_vec) {
      *reinterpret_cast<uint32_t*>(out) = *reinterpret_cast<const uint32_t*>(src);
    } else {
#pragma unroll
      for (int e = 0; e < VEC; ++e)
        if (r + e < rows) out[e] = src[e];
    }
  }
}

}  // namespace tb
