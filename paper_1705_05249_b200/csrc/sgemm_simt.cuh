// sgemm_simt.cuh — FP32 GEMM on the FFMA pipe (sm_100a).
//
// Replaces the reference's tiled FP32 arithmetic (_tile_product,
// pkg/src/tunedblas/kernels/compute.py:360-381, driven by gemm_indirect_tasks
// compute.py:384-420 and gemm_direct_tasks compute.py:432-471).
//
// Determinism contract (SURVEY §7 hard part 3): every output element is
//     acc = 0; for kk = 0 .. k-1: acc = fmaf(opA(i,kk), opB(kk,j), acc)
// followed by the reference epilogue (common.cuh Epi).  The chain has
// exactly k FMAs in ascending k for every tile configuration (the K tail is
// iterated with a runtime bound, never padded), so all instantiations below,
// the batched kernels and the C oracle (oracle/sgemm_seqk.c) agree BITWISE.
//
// Structure: BM x BN CTA tile, BK-deep stages double-buffered in shared
// memory, register prefetch of the next stage while the current one is
// consumed, TM x TN register micro-tile built from 4x4 sub-blocks read with
// 128-bit LDS, 128-bit LDG when the operands are 16-byte aligned; the
// outer product issues on FFMA2 (two bitwise-FFMA lanes per instruction).
#pragma once

#include "common.cuh"

namespace tb {

template <int BM, int BN, int BK, int TM, int TN>
struct SimtShape {
  static constexpr int TY = BM / TM;          // threads along M (fastest)
  static constexpr int TX = BN / TN;          // threads along N
  static constexpr int NT = TX * TY;
  static constexpr int QM = TM / 4, QN = TN / 4;
  static constexpr int PAD = 4;
  static constexpr int LDA_S = BM + PAD, LDB_S = BN + PAD;
  static constexpr int A_CHUNKS = BM * BK / 4, B_CHUNKS = BN * BK / 4;
  static constexpr int A_PER_T = A_CHUNKS / NT, B_PER_T = B_CHUNKS / NT;
  static_assert(TM % 4 == 0 && TN % 4 == 0, "micro tile in 4x4 sub-blocks");
  static_assert(A_CHUNKS % NT == 0 && B_CHUNKS % NT == 0, "whole chunks per thread");
  static_assert(BK % 4 == 0, "BK multiple of 4");
};

// Load one BK-deep stage of op(A) (BM x BK) into registers as 4-element
// chunks along the operand's contiguous dimension.
//   AK (K-contiguous):  chunk e -> row i = e / (BK/4), kk = (e % (BK/4))*4
//   !AK (M-contiguous): chunk e -> kk = e / (BM/4),  i = (e % (BM/4))*4
// `rows_left`/`k_left` bound the tile (edge tiles and the K tail).
template <int ROWS, int BK, bool KCONTIG, bool VEC, int PER_T, int NT>
__device__ __forceinline__ void simt_load_stage(float4 (&r)[PER_T], const float* __restrict__ base,
                                                int64_t ld, int rows_left, int k_left) {
#pragma unroll
  for (int j = 0; j < PER_T; ++j) {
    const int e = threadIdx.x + j * NT;
    int row, kk;
    if (KCONTIG) {
      row = e / (BK / 4);
      kk = (e % (BK / 4)) * 4;
    } else {
      kk = e / (ROWS / 4);
      row = (e % (ROWS / 4)) * 4;
    }
    float v[4];
    if (KCONTIG) {
      const float* src = base + static_cast<int64_t>(row) * ld + kk;
      const bool row_ok = row < rows_left;
      if (VEC && row_ok && kk + 3 < k_left) {
        const float4 t = __ldg(reinterpret_cast<const float4*>(src));
        v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] = (row_ok && kk + q < k_left) ? __ldg(src + q) : 0.0f;
      }
    } else {
      const float* src = base + static_cast<int64_t>(kk) * ld + row;
      const bool k_ok = kk < k_left;
      if (VEC && k_ok && row + 3 < rows_left) {
        const float4 t = __ldg(reinterpret_cast<const float4*>(src));
        v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] = (k_ok && row + q < rows_left) ? __ldg(src + q) : 0.0f;
      }
    }
    r[j] = make_float4(v[0], v[1], v[2], v[3]);
  }
}

// Implicit-GEMM variant of simt_load_stage for op(A) (M-contiguous chunk
// layout): chunk e holds positions q = m0 + row .. +3 of K index k0 + kk,
// gathered from the channel-major image `im` (ConvGeom; zero in the padding,
// past m and past k).
template <int ROWS, int BK, int PER_T, int NT>
__device__ __forceinline__ void simt_conv_stage(float4 (&r)[PER_T], const float* __restrict__ im,
                                                const ConvGeom& g, int64_t m, int64_t m0, int64_t k0,
                                                int k_left) {
  // branch-free: every tap loads from a valid address (the plane's first
  // element in the padding) and is masked afterwards, so the loads of the
  // whole stage issue back to back (see hgemm_tc.cuh conv_fill_tile)
  const int khw = g.kh * g.kw;
#pragma unroll
  for (int j = 0; j < PER_T; ++j) {
    const int e = threadIdx.x + j * NT;
    const int kk = e / (ROWS / 4);
    const int row = (e % (ROWS / 4)) * 4;
    const bool k_ok = kk < k_left;
    const int kr = static_cast<int>(k0) + (k_ok ? kk : 0);
    const int ch = kr / khw, rem = kr - ch * khw;
    const int ky = rem / g.kw, kx = rem - ky * g.kw;
    const float* plane = im + static_cast<int64_t>(ch) * g.height * g.width;
    float v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t pos = m0 + row + q;
      const int oy = static_cast<int>(pos / g.out_w), ox = static_cast<int>(pos - static_cast<int64_t>(oy) * g.out_w);
      const int y = oy * g.stride_h + ky * g.dil_h - g.pad_h, x = ox * g.stride_w + kx * g.dil_w - g.pad_w;
      const bool in = k_ok && pos < m && static_cast<unsigned>(y) < static_cast<unsigned>(g.height) &&
                      static_cast<unsigned>(x) < static_cast<unsigned>(g.width);
      const float t = __ldg(plane + (in ? static_cast<int64_t>(y) * g.width + x : 0));
      v[q] = in ? t : 0.0f;
    }
    r[j] = make_float4(v[0], v[1], v[2], v[3]);
  }
}

// Store the register stage into shared memory laid out [BK][ROWS+PAD]
// (contiguous along M or N so the compute loop reads 128-bit fragments).
template <int ROWS, int BK, bool KCONTIG, int PER_T, int NT, int LDS>
__device__ __forceinline__ void simt_store_stage(float* __restrict__ s, const float4 (&r)[PER_T]) {
#pragma unroll
  for (int j = 0; j < PER_T; ++j) {
    const int e = threadIdx.x + j * NT;
    if (KCONTIG) {
      const int row = e / (BK / 4);
      const int kk = (e % (BK / 4)) * 4;
      s[(kk + 0) * LDS + row] = r[j].x;
      s[(kk + 1) * LDS + row] = r[j].y;
      s[(kk + 2) * LDS + row] = r[j].z;
      s[(kk + 3) * LDS + row] = r[j].w;
    } else {
      const int kk = e / (ROWS / 4);
      const int row = (e % (ROWS / 4)) * 4;
      *reinterpret_cast<float4*>(s + kk * LDS + row) = r[j];
    }
  }
}

// Linear CTA index -> (instance, m-tile, n-tile) with grouped rasterisation
// (GROUP_M m-tiles share each B panel while it is hot in L2).
__device__ __forceinline__ void tile_coords(int64_t bid, int tiles_m, int tiles_n, int group_m,
                                            int64_t& z, int& mt, int& nt) {
  const int64_t per_inst = static_cast<int64_t>(tiles_m) * tiles_n;
  if (per_inst == 1) {  // one tile per instance: no division (short-lived CTAs)
    z = bid;
    mt = nt = 0;
    return;
  }
  // 32-bit division when the tile index allows (the usual case)
  z = (bid < 0x7fffffffLL && per_inst < 0x7fffffffLL)
          ? static_cast<int64_t>(static_cast<int>(bid) / static_cast<int>(per_inst))
          : bid / per_inst;
  const int r = static_cast<int>(bid - z * per_inst);
  const int group_size = group_m * tiles_n;
  const int g = r / group_size;
  const int first_m = g * group_m;
  const int gm = min(tiles_m - first_m, group_m);
  const int rr = r - g * group_size;
  mt = first_m + rr % gm;
  nt = rr / gm;
}

// CONV: op(A) gathered from an image (implicit GEMM, ConvGeom; AK false).
template <int BM, int BN, int BK, int TM, int TN, bool AK, bool BNC, bool VEC, int MINB, bool CONV = false>
__global__ void __launch_bounds__(SimtShape<BM, BN, BK, TM, TN>::NT, MINB)
    sgemm_simt_kernel(Problem p, int tiles_m, int tiles_n, int group_m, const ConvGeom conv) {
  using S = SimtShape<BM, BN, BK, TM, TN>;
  static_assert(!CONV || !AK, "the im2col gather fills the M-contiguous layout");
  grid_dep_wait();  // PDL: the previous kernel's writes are visible from here
  __shared__ __align__(16) float As[2][BK * S::LDA_S];
  __shared__ __align__(16) float Bs[2][BK * S::LDB_S];

  int64_t z;
  int mt, nt;
  tile_coords(blockIdx.x, tiles_m, tiles_n, group_m, z, mt, nt);
  const int64_t m0 = static_cast<int64_t>(mt) * BM, n0 = static_cast<int64_t>(nt) * BN;
  const int rows_m = static_cast<int>(min64(BM, p.m - m0));
  const int cols_n = static_cast<int>(min64(BN, p.n - n0));

  Epi epi;
  epi.alpha = inst_alpha(p, z);
  epi.beta = inst_beta(p, z);
  epi.skip_ab = (epi.alpha == 0.0f) || (p.k == 0);

  const int ty = threadIdx.x % S::TY;  // M index (fastest -> coalesced C columns)
  const int tx = threadIdx.x / S::TY;  // N index

  float2 acc2[TM / 2][TN];   // rows (2*i2, 2*i2+1) of column j, see outer_ffma2
#pragma unroll
  for (int i = 0; i < TM / 2; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc2[i][j] = make_float2(0.0f, 0.0f);

  if (!epi.skip_ab) {
    const float* A = static_cast<const float*>(p.a) + inst_off(p.a_off, p.stride_a, p.a_offs, z);
    const float* B = static_cast<const float*>(p.b) + inst_off(p.b_off, p.stride_b, p.b_offs, z);
    // tile origins: op(A) rows m0.., op(B) cols n0..
    const float* a_tile = AK ? A + m0 * p.lda : A + m0;
    const float* b_tile = BNC ? B + n0 : B + n0 * p.ldb;
    const int64_t a_kstep = AK ? BK : BK * p.lda;   // element advance per stage along K
    const int64_t b_kstep = BNC ? BK * p.ldb : BK;

    const int ktiles = static_cast<int>((p.k + BK - 1) / BK);
    float4 ra[S::A_PER_T], rb[S::B_PER_T];
    int k_left = static_cast<int>(min64(p.k, 0x7fffffff));

    int64_t kpos = 0;   // K index of the stage being loaded (CONV)
    if (CONV)
      simt_conv_stage<BM, BK, S::A_PER_T, S::NT>(ra, A, conv, p.m, m0, 0, k_left);
    else
      simt_load_stage<BM, BK, AK, VEC, S::A_PER_T, S::NT>(ra, a_tile, p.lda, rows_m, k_left);
    simt_load_stage<BN, BK, !BNC, VEC, S::B_PER_T, S::NT>(rb, b_tile, p.ldb, cols_n, k_left);
    simt_store_stage<BM, BK, AK, S::A_PER_T, S::NT, S::LDA_S>(As[0], ra);
    simt_store_stage<BN, BK, !BNC, S::B_PER_T, S::NT, S::LDB_S>(Bs[0], rb);
    __syncthreads();

    for (int kt = 0; kt < ktiles; ++kt) {
      const int cur = kt & 1;
      const int kcur = min(k_left, BK);
      if (kt + 1 < ktiles) {
        a_tile += a_kstep;
        b_tile += b_kstep;
        kpos += BK;
        if (CONV)
          simt_conv_stage<BM, BK, S::A_PER_T, S::NT>(ra, A, conv, p.m, m0, kpos, k_left - BK);
        else
          simt_load_stage<BM, BK, AK, VEC, S::A_PER_T, S::NT>(ra, a_tile, p.lda, rows_m, k_left - BK);
        simt_load_stage<BN, BK, !BNC, VEC, S::B_PER_T, S::NT>(rb, b_tile, p.ldb, cols_n, k_left - BK);
      }
      const float* as = As[cur];
      const float* bs = Bs[cur];
      if (kcur == BK) {
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
          float af[TM], bf[TN];
#pragma unroll
          for (int q = 0; q < S::QM; ++q) {
            const float4 t = *reinterpret_cast<const float4*>(as + kk * S::LDA_S + q * (BM / S::QM) + ty * 4);
            af[q * 4 + 0] = t.x; af[q * 4 + 1] = t.y; af[q * 4 + 2] = t.z; af[q * 4 + 3] = t.w;
          }
#pragma unroll
          for (int q = 0; q < S::QN; ++q) {
            const float4 t = *reinterpret_cast<const float4*>(bs + kk * S::LDB_S + q * (BN / S::QN) + tx * 4);
            bf[q * 4 + 0] = t.x; bf[q * 4 + 1] = t.y; bf[q * 4 + 2] = t.z; bf[q * 4 + 3] = t.w;
          }
          outer_ffma2<TM, TN>(acc2, af, bf);
        }
      } else {
        // K tail: exactly kcur more FMAs (no zero padding — keeps the chain
        // identical to every other tile shape and to the C oracle).
#pragma unroll 1
        for (int kk = 0; kk < kcur; ++kk) {
          float af[TM], bf[TN];
#pragma unroll
          for (int q = 0; q < S::QM; ++q) {
            const float4 t = *reinterpret_cast<const float4*>(as + kk * S::LDA_S + q * (BM / S::QM) + ty * 4);
            af[q * 4 + 0] = t.x; af[q * 4 + 1] = t.y; af[q * 4 + 2] = t.z; af[q * 4 + 3] = t.w;
          }
#pragma unroll
          for (int q = 0; q < S::QN; ++q) {
            const float4 t = *reinterpret_cast<const float4*>(bs + kk * S::LDB_S + q * (BN / S::QN) + tx * 4);
            bf[q * 4 + 0] = t.x; bf[q * 4 + 1] = t.y; bf[q * 4 + 2] = t.z; bf[q * 4 + 3] = t.w;
          }
          outer_ffma2<TM, TN>(acc2, af, bf);
        }
      }
      if (kt + 1 < ktiles) {
        simt_store_stage<BM, BK, AK, S::A_PER_T, S::NT, S::LDA_S>(As[cur ^ 1], ra);
        simt_store_stage<BN, BK, !BNC, S::B_PER_T, S::NT, S::LDB_S>(Bs[cur ^ 1], rb);
      }
      k_left -= BK;
      __syncthreads();
    }
  }

  // Epilogue: rows (q*BM/QM + ty*4 + r), cols (q*BN/QN + tx*4 + c).
#define ACC2(i, j) (((i) & 1) ? acc2[(i) >> 1][j].y : acc2[(i) >> 1][j].x)
  float* C = static_cast<float*>(p.c) + inst_off(p.c_off, p.stride_c, p.c_offs, z);
  const int64_t cbase_off = inst_off(p.c_off, p.stride_c, p.c_offs, z);
  const bool cvec = ((cbase_off & 3) == 0) && ((p.ldc & 3) == 0);
#pragma unroll
  for (int qn = 0; qn < S::QN; ++qn) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int col = qn * (BN / S::QN) + tx * 4 + c;
      if (col >= cols_n) continue;
      float* ccol = C + (n0 + col) * p.ldc + m0;
#pragma unroll
      for (int qm = 0; qm < S::QM; ++qm) {
        const int row = qm * (BM / S::QM) + ty * 4;
        if (cvec && row + 3 < rows_m) {
          float4 cv = make_float4(0.f, 0.f, 0.f, 0.f);
          if (epi.reads_c()) cv = *reinterpret_cast<const float4*>(ccol + row);
          float4 o;
          o.x = epi.apply(ACC2(qm * 4 + 0, qn * 4 + c), cv.x);
          o.y = epi.apply(ACC2(qm * 4 + 1, qn * 4 + c), cv.y);
          o.z = epi.apply(ACC2(qm * 4 + 2, qn * 4 + c), cv.z);
          o.w = epi.apply(ACC2(qm * 4 + 3, qn * 4 + c), cv.w);
          *reinterpret_cast<float4*>(ccol + row) = o;
        } else {
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            if (row + r < rows_m) {
              const float cv = epi.reads_c() ? ccol[row + r] : 0.0f;
              ccol[row + r] = epi.apply(ACC2(qm * 4 + r, qn * 4 + c), cv);
            }
          }
        }
      }
    }
  }
#undef ACC2
}

}  // namespace tb
