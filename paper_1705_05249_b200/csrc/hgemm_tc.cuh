// hgemm_tc.cuh — FP16 GEMM on the 5th-gen tensor cores (tcgen05 + TMEM).
//
// Replaces the reference's indirect Xgemm path for Precision.H
// (pkg/src/tunedblas/routines/level3.py:48-91 → compute.py:384-420): the
// pad / transpose / copy pre-kernels (level3.py:71-82, 134-147) disappear —
// TMA tensor maps read the UNPADDED operands in whatever major-ness the
// caller's layout/trans flags imply (OOB boxes zero-fill), and the
// unpad + single FP16 rounding (level3.py:91) is fused into the epilogue.
//
// Persistent, warp-specialised kernel (one CTA per SM):
//   producer  : TMA (one elected thread) or, when operands are not 16-B
//               aligned / offsets are per-instance, 4 warps of predicated
//               LDG + swizzled STS into the identical smem layout;
//   MMA       : one thread issues tcgen05.mma.cta_group::1.kind::f16
//               (M=128, N=BN, K=16) into a double-buffered FP32 TMEM
//               accumulator (2 x BN columns);
//   epilogue  : 4 warps, tcgen05.ld 32x32b → FP32 alpha/beta epilogue
//               (Epi: three separately rounded ops) → RNE to FP16 → global.
// Pipelines: smem full/empty mbarrier ring (STAGES deep), TMEM full/empty
// pair; tiles are visited in grouped raster order (tile_coords).
//
// Both producers fill byte-identical shared memory and the MMA sequence per
// output element (K in 64-deep blocks of 4 x K16 steps, zero-filled tail)
// is the same, so every HGEMM path — TMA or LDG, single or batched — gives
// bitwise-identical results for the same (m, n, k).
#pragma once

#include "common.cuh"
#include "sgemm_simt.cuh"  // tile_coords

namespace tb {

constexpr int HG_BM = 128;
constexpr int HG_BK = 64;  // 64 halves = 128 B = one SW128 row

// ST: ring depth (0 = default: 4 for BN 256, 6 otherwise — the deepest that
// fits next to the epilogue staging; "gemm_b200" STAGES selects the other
// instantiated depth, hgemm.cu).
template <int BN, bool TMA, int ST = 0>
struct HgCfg {
  static constexpr int STAGES = ST > 0 ? ST : ((BN >= 256) ? 4 : 6);
  static constexpr int A_BYTES = HG_BM * HG_BK * 2;            // 16 KB
  static constexpr int B_BYTES = BN * HG_BK * 2;               // 8/16/32 KB
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128
                                  : (2 * BN <= 256) ? 256 : 512;
  // warps 0-7: epilogue (warp w reads TMEM lane quadrant w%4, column half
  // w/4); then the producer warp(s); the last warp allocates TMEM and issues MMAs.
  static constexpr int EPI_WARPS = 8;
  static constexpr int PROD_WARPS = TMA ? 1 : 4;
  static constexpr int PROD_WARP0 = EPI_WARPS;
  static constexpr int MMA_WARP = EPI_WARPS + PROD_WARPS;
  static constexpr int THREADS = (MMA_WARP + 1) * 32;
  static constexpr int BAR_BYTES = 1024;
  static constexpr int EPI_BYTES = EPI_WARPS * 32 * 32 * 4;
  static constexpr int SMEM_BYTES = 1024 /*align slack*/ + STAGES * STAGE_BYTES + BAR_BYTES + EPI_BYTES;
};

// Swizzle-128B placement of 16-byte chunk `c` (0..7) of 128-byte row `r`
// inside a 1024-byte-aligned region (identical to what TMA SWIZZLE_128B writes).
__device__ __forceinline__ uint32_t sw128_off(int r, int c) {
  return static_cast<uint32_t>((r >> 3) * 1024 + (r & 7) * 128 + ((c ^ (r & 7)) << 4));
}

// Load 8 consecutive halves along the operand's contiguous dimension,
// zero-filling past `valid` elements.
template <bool VEC>
__device__ __forceinline__ uint4 ldg_chunk8(const __half* src, int valid) {
  if (VEC && valid >= 8) return __ldg(reinterpret_cast<const uint4*>(src));
  uint16_t h[8];
  const uint16_t* s16 = reinterpret_cast<const uint16_t*>(src);
#pragma unroll
  for (int q = 0; q < 8; ++q) h[q] = (q < valid) ? __ldg(s16 + q) : static_cast<uint16_t>(0);
  uint4 r;
  r.x = h[0] | (static_cast<uint32_t>(h[1]) << 16);
  r.y = h[2] | (static_cast<uint32_t>(h[3]) << 16);
  r.z = h[4] | (static_cast<uint32_t>(h[5]) << 16);
  r.w = h[6] | (static_cast<uint32_t>(h[7]) << 16);
  return r;
}

// LDG producer for one operand tile of ROWS (M or N) x 64 (K):
//   K-major  (!MN): smem = ROWS rows of 128 B (row = M/N index, chunk = K/8)
//   MN-major ( MN): ROWS/64 sub-tiles of 64 K-rows x 128 B (chunk = MN/8)
// `base` points at the operand element (mn0, k0) of this instance; `ld` is
// the stride of the non-contiguous dimension.
template <int ROWS, bool MN, bool VEC>
__device__ __forceinline__ void ldg_fill_tile(uint8_t* smem, const __half* base, int64_t ld,
                                              int mn_left, int k_left, int tid) {
  constexpr int CHUNKS = ROWS * 8;
  constexpr int PER_T = CHUNKS / 128;
  uint4 v[PER_T];
#pragma unroll
  for (int j = 0; j < PER_T; ++j) {
    const int g = tid + j * 128;
    if (!MN) {
      const int r = g >> 3, c = g & 7;       // r: M/N row, c: K chunk
      const int valid = (r < mn_left) ? min(8, k_left - c * 8) : 0;
      v[j] = (valid > 0) ? ldg_chunk8<VEC>(base + static_cast<int64_t>(r) * ld + c * 8, valid)
                         : make_uint4(0, 0, 0, 0);
    } else {
      const int sub = g >> 9, r = (g >> 3) & 63, c = g & 7;  // r: K row, c: MN chunk
      const int mn = sub * 64 + c * 8;
      const int valid = (r < k_left) ? min(8, mn_left - mn) : 0;
      v[j] = (valid > 0) ? ldg_chunk8<VEC>(base + static_cast<int64_t>(r) * ld + mn, valid)
                         : make_uint4(0, 0, 0, 0);
    }
  }
#pragma unroll
  for (int j = 0; j < PER_T; ++j) {
    const int g = tid + j * 128;
    uint32_t off;
    if (!MN) {
      off = sw128_off(g >> 3, g & 7);
    } else {
      off = (g >> 9) * 8192 + sw128_off((g >> 3) & 63, g & 7);
    }
    *reinterpret_cast<uint4*>(smem + off) = v[j];
  }
}


// Implicit-GEMM producer for op(A) (128 positions x 64 K, MN-major layout of
// ldg_fill_tile): every element is gathered from the image (ConvGeom), zero
// in the padding and past m / k.  Each thread owns the same 16 positions of a
// tile (two groups of 8 at c*8 and 64 + c*8, c = tid % 8) and K rows
// tid/8 + 16*i; `yb`/`xb` hold oy*stride - pad / ox*stride - pad per owned
// position (INT_MIN/2 for positions past m), computed once per tile.
__device__ __forceinline__ void conv_tile_coords(const ConvGeom& g, int64_t m, int64_t m0, int tid,
                                                 int (&yb)[16], int (&xb)[16]) {
  const int c = tid & 7;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int64_t q = m0 + (i >> 3) * 64 + c * 8 + (i & 7);
    if (q < m) {
      const int oy = static_cast<int>(q / g.out_w), ox = static_cast<int>(q - static_cast<int64_t>(oy) * g.out_w);
      yb[i] = oy * g.stride_h - g.pad_h;
      xb[i] = ox * g.stride_w - g.pad_w;
    } else {
      yb[i] = -(1 << 30);
      xb[i] = -(1 << 30);
    }
  }
}

__device__ __forceinline__ void conv_fill_tile(uint8_t* smem, const __half* im, const ConvGeom& g,
                                               int64_t k0, int k_left, int tid, const int (&yb)[16],
                                               const int (&xb)[16]) {
  // Branch-free gather: every element is loaded from a valid address (the
  // plane's first element when the tap falls in the padding) and masked
  // afterwards, so the 32 loads of two K rows issue back to back and share
  // one L2 round trip (a predicated load per element compiled to a branch
  // each and serialised them: 5 us per K block at the C3 layer).
  const uint16_t* im16 = reinterpret_cast<const uint16_t*>(im);
  const int khw = g.kh * g.kw;
#pragma unroll
  for (int i0 = 0; i0 < 4; i0 += 2) {
    uint16_t h[2][16];
    uint32_t ok[2];
#pragma unroll
    for (int ii = 0; ii < 2; ++ii) {
      const int r = (tid >> 3) + 16 * (i0 + ii);       // K row of this K block
      const bool row_ok = r < k_left;
      const int kr = static_cast<int>(k0) + (row_ok ? r : 0);
      const int ch = kr / khw, rem = kr - ch * khw;
      const int ky = rem / g.kw, kx = rem - ky * g.kw;
      const int dy = ky * g.dil_h, dx = kx * g.dil_w;
      const uint16_t* plane = im16 + static_cast<int64_t>(ch) * g.height * g.width;
      uint32_t m = 0;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int y = yb[j] + dy, x = xb[j] + dx;
        const bool in = row_ok && static_cast<unsigned>(y) < static_cast<unsigned>(g.height) &&
                        static_cast<unsigned>(x) < static_cast<unsigned>(g.width);
        m |= (in ? 1u : 0u) << j;
        h[ii][j] = __ldg(plane + (in ? y * g.width + x : 0));
      }
      ok[ii] = m;
    }
#pragma unroll
    for (int ii = 0; ii < 2; ++ii) {
      const int r = (tid >> 3) + 16 * (i0 + ii);
#pragma unroll
      for (int sub = 0; sub < 2; ++sub) {
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int j = sub * 8 + 2 * q;
          const uint32_t lo = ((ok[ii] >> j) & 1u) ? h[ii][j] : 0u;
          const uint32_t hi = ((ok[ii] >> (j + 1)) & 1u) ? h[ii][j + 1] : 0u;
          w[q] = lo | (hi << 16);
        }
        *reinterpret_cast<uint4*>(smem + sub * 8192 + sw128_off(r, tid & 7)) = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
  }
}

// K16 MMA steps in K block kb: 4, except in the last block, where steps that
// would multiply only zero padding are not issued.  Every H kernel uses this
// rule, so all H paths issue the same MMA sequence for an output element.
__device__ __forceinline__ int hg_ksteps(int64_t k, int kb) {
  const int64_t left = k - static_cast<int64_t>(kb) * HG_BK;
  return left >= HG_BK ? HG_BK / 16 : static_cast<int>((left + 15) / 16);
}

struct Mma1Sm {
  __device__ __forceinline__ void operator()(uint32_t d, uint64_t a, uint64_t b, uint32_t i, uint32_t acc) const {
    tc_mma_f16(d, a, b, i, acc);
  }
};

// Issue the K16 MMAs of one staged SWIZZLE_128B K block (A 128 rows / B BN
// rows x 64 K).  Call from ALL lanes of the (converged) MMA warp: operands are
// then warp-uniform and live in uniform registers, and one elected lane
// issues.  A K16 step advances the descriptor's 14-bit start-address field by
// 32 B (K-major) or 2048 B (MN-major).  `Mma` is tc_mma_f16 / tc2_mma_f16.
template <bool A_MN, bool B_MN, typename Mma>
__device__ __forceinline__ void hg_issue_kblock(Mma mma, uint32_t d_tmem, uint32_t a_addr, uint32_t b_addr,
                                                uint32_t idesc, int ksteps, bool first_block) {
  const uint64_t a0 = A_MN ? umma_desc_sw128(a_addr, 8192, 1024) : umma_desc_sw128(a_addr, 16, 1024);
  const uint64_t b0 = B_MN ? umma_desc_sw128(b_addr, 8192, 1024) : umma_desc_sw128(b_addr, 16, 1024);
  constexpr uint64_t ASTEP = A_MN ? 128 : 2, BSTEP = B_MN ? 128 : 2;
  if (ksteps == HG_BK / 16) {
#pragma unroll
    for (int kk = 0; kk < HG_BK / 16; ++kk)
      mma(d_tmem, a0 + ASTEP * kk, b0 + BSTEP * kk, idesc, (!first_block || kk != 0) ? 1u : 0u);
  } else {
#pragma unroll 1
    for (int kk = 0; kk < ksteps; ++kk)
      mma(d_tmem, a0 + ASTEP * kk, b0 + BSTEP * kk, idesc, (!first_block || kk != 0) ? 1u : 0u);
  }
}

// Per-warp epilogue staging: 32 rows x 32 FP32 columns (4 KB).  Column c
// holds row r at float index c*32 + (r ^ 4*(c%8)): conflict-free for the
// row-per-lane writes and for the 8-rows-per-lane float4 reads below.
constexpr int EPI_WARP_FLOATS = 32 * 32;
__device__ __forceinline__ int epi_idx(int c, int r) { return c * 32 + (r ^ ((c & 7) << 2)); }

// Store one warp's 32 x 32 accumulator block (lane = row, v[j] = column j)
// to column-major FP16 C through shared memory, so global traffic is 16-byte
// vectors (8 consecutive rows of one column per lane) instead of 2-byte
// scalars.  `cblk` points at C element (row 0, col 0) of the block; rows /
// cols beyond rows_valid / cols_valid are not written.  The reference
// epilogue (Epi) is applied in FP32 and rounded once to FP16.
template <int NCOL>
__device__ __forceinline__ void epi_store_block(float* stage, const uint32_t (&v)[NCOL], __half* cblk,
                                                int64_t ldc, int rows_valid, int cols_valid,
                                                const Epi& epi, int lane) {
  static_assert(NCOL == 16 || NCOL == 32, "16 or 32 columns");
#pragma unroll
  for (int c = 0; c < NCOL; ++c) stage[epi_idx(c, lane)] = __uint_as_float(v[c]);
  __syncwarp();
  const bool vec_ok = ((reinterpret_cast<uintptr_t>(cblk) & 15) == 0) && ((ldc & 7) == 0);
  const bool full = vec_ok && rows_valid >= 32 && cols_valid >= NCOL;
  // 0: alpha == 0 (beta*C or 0), 1: beta == 0 (alpha*acc), 2: general.  One
  // runtime-mode body (measured: per-mode instantiations bloat the kernels
  // and run slower).
  const int mode = epi.skip_ab ? 0 : (epi.beta == 0.0f ? 1 : 2);
  // NCOL columns x 4 groups of 8 rows; quarter-warps cover 8 distinct columns.
#pragma unroll
  for (int it = 0; it < NCOL / 8; ++it) {
    const int item = it * 32 + lane;
    const int c = (NCOL == 32) ? (it * 8 + (lane & 7)) : (item & 15);
    const int rg = (NCOL == 32) ? (lane >> 3) : (item >> 4);
    const float4 x0 = *reinterpret_cast<const float4*>(stage + epi_idx(c, rg * 8));
    const float4 x1 = *reinterpret_cast<const float4*>(stage + epi_idx(c, rg * 8 + 4));
    if (full || (c < cols_valid && rg * 8 < rows_valid)) {
      __half* dst = cblk + static_cast<int64_t>(c) * ldc + rg * 8;
      float x[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
      if (full || (vec_ok && rg * 8 + 8 <= rows_valid)) {
        if (mode == 1) {
#pragma unroll
          for (int i = 0; i < 8; ++i) x[i] = __fmul_rn(epi.alpha, x[i]);
        } else {
          float cv[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
          if (epi.reads_c()) {
            const uint4 raw = *reinterpret_cast<const uint4*>(dst);
            const __half2* h2 = reinterpret_cast<const __half2*>(&raw);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float2 f = __half22float2(h2[i]);
              cv[2 * i] = f.x;
              cv[2 * i + 1] = f.y;
            }
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) x[i] = epi.apply(x[i], cv[i]);
        }
        uint4 out;
        __half2* o2 = reinterpret_cast<__half2*>(&out);
#pragma unroll
        for (int i = 0; i < 4; ++i) o2[i] = __floats2half2_rn(x[2 * i], x[2 * i + 1]);
        *reinterpret_cast<uint4*>(dst) = out;
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (rg * 8 + i < rows_valid) {
            const float cvs = epi.reads_c() ? __half2float(dst[i]) : 0.0f;
            dst[i] = __float2half_rn(epi.apply(x[i], cvs));
          }
        }
      }
    }
  }
  __syncwarp();
}

// CONV: op(A) is gathered from an image (implicit GEMM, ConvGeom; LDG
// producer, A_MN layout); otherwise `conv` is unused.
template <int BN, bool TMA, bool A_MN, bool B_MN, bool VEC, int ST = 0, bool CONV = false>
__global__ void __launch_bounds__(HgCfg<BN, TMA, ST>::THREADS, 1)
    hgemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    Problem p, int tiles_m, int tiles_n, int group_m, int64_t total_tiles,
                    const ConvGeom conv) {
  static_assert(!CONV || (!TMA && A_MN), "the im2col gather runs in the LDG producer, MN-major");
  using C = HgCfg<BN, TMA, ST>;
  constexpr int STAGES = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_align1024(smem_raw);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);
  float* epi_stage = reinterpret_cast<float*>(smem + STAGES * C::STAGE_BYTES + C::BAR_BYTES);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], TMA ? 1 : 128);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 32 * C::EPI_WARPS);
    }
    fence_mbar_init();
  }
  if (TMA && warp == C::PROD_WARP0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == C::MMA_WARP) tmem_alloc(tmem_holder, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  grid_dep_wait();  // prologue above overlapped the previous kernel (PDL)
  grid_dep_launch();

  const int nkb = static_cast<int>((p.k + HG_BK - 1) / HG_BK);

  if (warp >= C::PROD_WARP0 && warp < C::MMA_WARP) {
    // ======================= producer =======================
    int s = 0;
    uint32_t ph = 0;
    if (TMA) {
      // The whole warp runs the loop (uniform coordinates); one elected lane issues.
      for (int64_t t = blockIdx.x; t < total_tiles; t += gridDim.x) {
        int64_t z; int mt, nt;
        tile_coords(t, tiles_m, tiles_n, group_m, z, mt, nt);
        const int m0 = mt * HG_BM, n0 = nt * BN, zz = static_cast<int>(z);
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);
          if (elect_one()) {
            mbar_arrive_expect_tx(&full[s], C::STAGE_BYTES);
            const int k0 = kb * HG_BK;
            uint8_t* a_dst = sA + s * C::A_BYTES;
            uint8_t* b_dst = sB + s * C::B_BYTES;
            if (!A_MN) {
              tma_load_3d(a_dst, &tmA, &full[s], k0, m0, zz);
            } else {
              tma_load_3d(a_dst, &tmA, &full[s], m0, k0, zz);
              tma_load_3d(a_dst + 8192, &tmA, &full[s], m0 + 64, k0, zz);
            }
            if (!B_MN) {
              tma_load_3d(b_dst, &tmB, &full[s], k0, n0, zz);
            } else {
#pragma unroll
              for (int c = 0; c < BN / 64; ++c) tma_load_3d(b_dst + c * 8192, &tmB, &full[s], n0 + c * 64, k0, zz);
            }
          }
          __syncwarp();
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
      }
    } else {
      const int tid = threadIdx.x - C::PROD_WARP0 * 32;  // 0..127
      for (int64_t t = blockIdx.x; t < total_tiles; t += gridDim.x) {
        int64_t z; int mt, nt;
        tile_coords(t, tiles_m, tiles_n, group_m, z, mt, nt);
        const int64_t m0 = static_cast<int64_t>(mt) * HG_BM, n0 = static_cast<int64_t>(nt) * BN;
        const __half* A = static_cast<const __half*>(p.a) + inst_off(p.a_off, p.stride_a, p.a_offs, z);
        const __half* B = static_cast<const __half*>(p.b) + inst_off(p.b_off, p.stride_b, p.b_offs, z);
        const int m_left = static_cast<int>(min64(HG_BM, p.m - m0));
        const int n_left = static_cast<int>(min64(BN, p.n - n0));
        int yb[16], xb[16];
        if (CONV) conv_tile_coords(conv, p.m, m0, tid, yb, xb);
        for (int kb = 0; kb < nkb; ++kb) {
          const int64_t k0 = static_cast<int64_t>(kb) * HG_BK;
          const int k_left = static_cast<int>(min64(HG_BK, p.k - k0));
          mbar_wait(&empty[s], ph ^ 1);
          // A: K-major element (i,kk) at A[i*lda + kk]; MN-major at A[i + kk*lda]
          const __half* a_base = A_MN ? A + k0 * p.lda + m0 : A + m0 * p.lda + k0;
          const __half* b_base = B_MN ? B + k0 * p.ldb + n0 : B + n0 * p.ldb + k0;
          if (CONV)
            conv_fill_tile(sA + s * C::A_BYTES, A, conv, k0, k_left, tid, yb, xb);
          else
            ldg_fill_tile<HG_BM, A_MN, VEC>(sA + s * C::A_BYTES, a_base, p.lda, m_left, k_left, tid);
          ldg_fill_tile<BN, B_MN, VEC>(sB + s * C::B_BYTES, b_base, p.ldb, n_left, k_left, tid);
          fence_proxy_async_smem();
          mbar_arrive(&full[s]);
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == C::MMA_WARP) {
    // ======================= MMA issuer =======================
    // The whole warp runs the loop (uniform operands); one elected lane issues.
    constexpr uint32_t idesc = umma_idesc_f16(HG_BM, BN, A_MN ? 1 : 0, B_MN ? 1 : 0);
    int s = 0;
    uint32_t ph = 0;
    int acc = 0;
    uint32_t aph = 0;
    for (int64_t t = blockIdx.x; t < total_tiles; t += gridDim.x) {
      mbar_wait(&tempty[acc], aph ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint32_t a_addr = smem_u32(sA + s * C::A_BYTES);
        const uint32_t b_addr = smem_u32(sB + s * C::B_BYTES);
        const int ksteps = hg_ksteps(p.k, kb);
        if (elect_one()) {
          hg_issue_kblock<A_MN, B_MN>(Mma1Sm{}, d_tmem, a_addr, b_addr, idesc, ksteps, kb == 0);
          tc_commit(&empty[s]);
        }
        __syncwarp();
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
      if (elect_one()) tc_commit(&tfull[acc]);
      __syncwarp();
      if (++acc == 2) { acc = 0; aph ^= 1; }
    }
  } else if (warp < C::EPI_WARPS) {
    // ======================= epilogue =======================
    const int quad = warp & 3;
    const int half = warp >> 2;
    int acc = 0;
    uint32_t aph = 0;
    for (int64_t t = blockIdx.x; t < total_tiles; t += gridDim.x) {
      int64_t z; int mt, nt;
      tile_coords(t, tiles_m, tiles_n, group_m, z, mt, nt);
      const int64_t m0 = static_cast<int64_t>(mt) * HG_BM, n0 = static_cast<int64_t>(nt) * BN;
      Epi epi;
      epi.alpha = inst_alpha(p, z);
      epi.beta = inst_beta(p, z);
      epi.skip_ab = (epi.alpha == 0.0f);
      const int64_t row0 = m0 + quad * 32;
      const int rows_valid = static_cast<int>(min64(32, p.m - row0));
      __half* Cz = static_cast<__half*>(p.c) + inst_off(p.c_off, p.stride_c, p.c_offs, z);
      const int n_left = static_cast<int>(min64(BN, p.n - n0));
      float* stage = epi_stage + warp * EPI_WARP_FLOATS;  // one buffer per epilogue warp

      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + static_cast<uint32_t>(acc * BN);
#pragma unroll 1
      for (int cb = half * (BN / 64); cb < (half + 1) * (BN / 64); ++cb) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(t_row + cb * 32, v);
        tmem_ld_wait();
        if (rows_valid > 0 && cb * 32 < n_left)
          epi_store_block(stage, v, Cz + (n0 + cb * 32) * p.ldc + row0, p.ldc, rows_valid, n_left - cb * 32, epi, lane);
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; aph ^= 1; }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == C::MMA_WARP) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

// alpha == 0 / k == 0 for H (level3.py:125-132): C = beta == 0 ? 0 : RNE(beta*C)
template <int UNUSED = 0>  // a template: weak linkage across the translation units that include this header
__global__ void hscale_kernel(Problem p) {
  grid_dep_wait();
  const int64_t total = p.m * p.n;
  for (int64_t z = 0; z < p.batch; ++z) {
    const float beta = inst_beta(p, z);
    __half* Cz = static_cast<__half*>(p.c) + inst_off(p.c_off, p.stride_c, p.c_offs, z);
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
      const int64_t i = e % p.m, j = e / p.m;
      __half* cp = Cz + i + j * p.ldc;
      *cp = (beta == 0.0f) ? __float2half_rn(0.0f) : __float2half_rn(__fmul_rn(beta, __half2float(*cp)));
    }
  }
}

}  // namespace tb
