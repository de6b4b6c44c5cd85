// sgemm_ms.cuh — FP32 GEMM on the paired FFMA pipe with a multistage
// cp.async shared-memory ring (sm_100a).
//
// Replaces the reference's tiled FP32 arithmetic (_tile_product,
// pkg/src/tunedblas/kernels/compute.py:360-381, driven by gemm_indirect_tasks
// compute.py:384-420) for the large / mid-size SGEMM shapes.
//
// Same determinism contract as sgemm_simt.cuh: every output element is the
// ascending-k chain acc = fmaf(opA(i,kk), opB(kk,j), acc) of exactly k FMAs
// (K tail iterated with a runtime bound, never zero-padded), then the
// reference epilogue, so it agrees BITWISE with every other S kernel and the
// sequential-k C oracle.
//
// Structure: BM x BN CTA tile; STAGES-deep ring of BK-deep stages in dynamic
// shared memory, both operands stored [kk][row] (M / N contiguous) so the
// compute loop reads 128-bit fragments.  Loads go global -> shared directly
// with cp.async (no register staging): 16-byte chunks along the operand's
// contiguous M/N dimension, 4-byte element copies that transpose a
// K-contiguous operand on the way in.  One __syncthreads per stage; the
// outer product issues as FFMA2 (outer_ffma2, common.cuh).
#pragma once

#include "../paper_1705_05249_b200/csrc/common.cuh"

namespace tb {

template <int BM, int BN, int BK, int TM, int TN, int STAGES, bool BKS = false>
struct MsShape {
  static constexpr int TY = BM / TM;  // threads along M (fastest)
  static constexpr int TX = BN / TN;  // threads along N
  static constexpr int NT = TX * TY;
  static constexpr int QM = TM / 4, QN = TN / 4;
  static constexpr int PAD = 4;
  static constexpr int LDA_S = BM + PAD, LDB_S = BN + PAD;
  // BKS: B kept K-contiguous in shared memory ([n][BK], 16-byte chunks
  // XOR-swizzled by (n/4) so the 4 column groups of a warp hit disjoint banks)
  static constexpr int CPR = BK / 4;  // 16-byte chunks per B row (BKS)
  static constexpr int A_STAGE = BK * LDA_S, B_STAGE = BKS ? BN * BK : BK * LDB_S;  // floats
  static constexpr int SMEM_BYTES = STAGES * (A_STAGE + B_STAGE) * 4;
  static_assert(TM % 4 == 0 && TN % 4 == 0, "micro tile in 4x4 sub-blocks");
  static_assert((BM / 4) * BK % NT == 0 && (BN / 4) * BK % NT == 0, "whole 16-byte chunks per thread");
  static_assert(BM * BK % NT == 0 && BN * BK % NT == 0, "whole elements per thread");
  static_assert(!BKS || ((CPR == 4 || CPR == 8) && (BN / QN / 4) % CPR == 0 && TX >= 4),
                "BKS swizzle: per-thread constant chunk XOR");
};

__device__ __forceinline__ void cp_async_4(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_16_s(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes)
               : "memory");
}

// Issue the cp.async copies of one BK-deep stage of one operand into the
// [kk][row] shared layout (row stride LDS floats).
//   KCONTIG (element (row, kk) at base[row*ld + kk]): 4-byte copies, lanes
//     along kk (coalesced reads), transposed on the way into shared memory.
//   !KCONTIG (element at base[kk*ld + row]): 16-byte chunks of 4 rows when
//     VEC, else 4-byte copies with lanes along rows.
// Elements outside (rows_left, k_left) are zero-filled (src_bytes = 0); the
// compute loop never reads them past k_left, and rows past rows_left are
// never stored.
template <int ROWS, int BK, int NT, int LDS, bool KCONTIG, bool VEC>
__device__ __forceinline__ void ms_load_stage(uint32_t s_base, const float* __restrict__ base,
                                              int64_t ld, int rows_left, int k_left) {
  if (!KCONTIG && VEC) {
    constexpr int PER_T = (ROWS / 4) * BK / NT;
#pragma unroll
    for (int j = 0; j < PER_T; ++j) {
      const int e = threadIdx.x + j * NT;
      const int kk = e / (ROWS / 4);
      const int row = (e % (ROWS / 4)) * 4;
      const int cnt = (kk < k_left) ? max(0, min(4, rows_left - row)) : 0;
      const float* src = cnt ? base + static_cast<int64_t>(kk) * ld + row : base;
      cp_async_16_s(s_base + (kk * LDS + row) * 4, src, cnt * 4);
    }
  } else if (KCONTIG) {
    // a warp covers RP = NT/KL rows x KL kk: KL*4-byte row segments from
    // global, banks (kk*LDS + row) % 32 distinct for LDS % 32 == 4.  One
    // 64-bit pointer walks the rows so no per-element addresses stay live.
    constexpr int KL = BK < 8 ? BK : 8;
    constexpr int RP = NT / KL;
    static_assert(NT % KL == 0 && ROWS % RP == 0 && BK % KL == 0, "K-contiguous copy plan");
    const int kk0 = threadIdx.x % KL, row0 = threadIdx.x / KL;
    const int64_t row_step = static_cast<int64_t>(RP) * ld;
    const float* src = base + static_cast<int64_t>(row0) * ld + kk0;
    const uint32_t dst = s_base + (kk0 * LDS + row0) * 4;
    const bool full = k_left >= BK && rows_left >= ROWS;
#pragma unroll
    for (int rp = 0; rp < ROWS / RP; ++rp) {
#pragma unroll
      for (int kg = 0; kg < BK / KL; ++kg) {
        const bool ok = full || (row0 + rp * RP < rows_left && kk0 + kg * KL < k_left);
        cp_async_4(dst + (kg * KL * LDS + rp * RP) * 4, ok ? src + kg * KL : base, ok ? 4u : 0u);
      }
      src += row_step;
    }
  } else {
    constexpr int PER_T = ROWS * BK / NT;
#pragma unroll
    for (int j = 0; j < PER_T; ++j) {
      const int e = threadIdx.x + j * NT;
      const int kk = e / ROWS;
      const int row = e % ROWS;
      const bool ok = row < rows_left && kk < k_left;
      const float* src = ok ? base + static_cast<int64_t>(kk) * ld + row : base;
      cp_async_4(s_base + (kk * LDS + row) * 4, src, ok ? 4u : 0u);
    }
  }
}

// BKS load: op(B)(kk, n) at base[n*ld + kk] into [n][BK] with 16-byte
// chunks (4 consecutive kk), chunk c of row n stored at chunk c ^ ((n/4) % CPR).
template <int ROWS, int BK, int NT>
__device__ __forceinline__ void ms_load_stage_kc(uint32_t s_base, const float* __restrict__ base,
                                                 int64_t ld, int rows_left, int k_left) {
  constexpr int CPR = BK / 4;
  constexpr int PER_T = ROWS * CPR / NT;
  constexpr int RP = NT / CPR;  // rows per pass
  static_assert(NT % CPR == 0 && ROWS % RP == 0, "BKS copy plan");
  const int ch = threadIdx.x % CPR, row0 = threadIdx.x / CPR;
  const float* src = base + static_cast<int64_t>(row0) * ld + ch * 4;
  const int64_t row_step = static_cast<int64_t>(RP) * ld;
  const int kcnt = max(0, min(4, k_left - ch * 4));
  const bool full = k_left >= BK && rows_left >= ROWS;
#pragma unroll
  for (int j = 0; j < PER_T; ++j) {
    const int row = row0 + j * RP;
    const int cnt = full ? 4 : (row < rows_left ? kcnt : 0);
    const uint32_t dst = s_base + (row * BK + ((ch ^ ((row >> 2) & (CPR - 1))) * 4)) * 4;
    cp_async_16_s(dst, cnt ? src : base, cnt * 4);
    src += row_step;
  }
}

template <int BM, int BN, int BK, int TM, int TN, int STAGES, bool AK, bool BNC, bool VEC, int MINB,
          bool BKS = false>
__global__ void __launch_bounds__(MsShape<BM, BN, BK, TM, TN, STAGES, BKS>::NT, MINB)
    sgemm_ms_kernel(Problem p, int tiles_m, int tiles_n, int group_m) {
  static_assert(!BKS || (!BNC && VEC), "BKS needs a K-contiguous, 16-byte aligned B");
  using S = MsShape<BM, BN, BK, TM, TN, STAGES, BKS>;
  extern __shared__ __align__(16) float ms_smem[];
  float* As = ms_smem;                        // STAGES x [BK][LDA_S]
  float* Bs = ms_smem + STAGES * S::A_STAGE;  // STAGES x [BK][LDB_S]
  const uint32_t as_u32 = smem_u32(As), bs_u32 = smem_u32(Bs);

  // Linear CTA index -> (instance, m-tile, n-tile), grouped rasterisation.
  const int64_t per_inst = static_cast<int64_t>(tiles_m) * tiles_n;
  const int64_t z = blockIdx.x / per_inst;
  int mt, nt;
  {
    const int r = static_cast<int>(blockIdx.x - z * per_inst);
    const int group_size = group_m * tiles_n;
    const int g = r / group_size;
    const int first_m = g * group_m;
    const int gm = min(tiles_m - first_m, group_m);
    const int rr = r - g * group_size;
    mt = first_m + rr % gm;
    nt = rr / gm;
  }
  const int64_t m0 = static_cast<int64_t>(mt) * BM, n0 = static_cast<int64_t>(nt) * BN;
  const int rows_m = static_cast<int>(min64(BM, p.m - m0));
  const int cols_n = static_cast<int>(min64(BN, p.n - n0));

  Epi epi;
  epi.alpha = inst_alpha(p, z);
  epi.beta = inst_beta(p, z);
  epi.skip_ab = (epi.alpha == 0.0f) || (p.k == 0);

  const int ty = threadIdx.x % S::TY;
  const int tx = threadIdx.x / S::TY;

  float2 acc2[TM / 2][TN];  // rows (2*i2, 2*i2+1) of column j
#pragma unroll
  for (int i = 0; i < TM / 2; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc2[i][j] = make_float2(0.0f, 0.0f);

  if (!epi.skip_ab) {
    const float* A = static_cast<const float*>(p.a) + inst_off(p.a_off, p.stride_a, p.a_offs, z);
    const float* B = static_cast<const float*>(p.b) + inst_off(p.b_off, p.stride_b, p.b_offs, z);
    const float* a_tile = AK ? A + m0 * p.lda : A + m0;
    const float* b_tile = BNC ? B + n0 : B + n0 * p.ldb;
    const int64_t a_kstep = AK ? BK : BK * p.lda;
    const int64_t b_kstep = BNC ? BK * p.ldb : BK;
    const int k_total = static_cast<int>(min64(p.k, 0x7fffffff));
    const int ktiles = (k_total + BK - 1) / BK;

    // prologue: stages 0 .. STAGES-2
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
      if (s < ktiles) {
        ms_load_stage<BM, BK, S::NT, S::LDA_S, AK, VEC>(as_u32 + s * S::A_STAGE * 4, a_tile + s * a_kstep,
                                                        p.lda, rows_m, k_total - s * BK);
        if constexpr (BKS)
          ms_load_stage_kc<BN, BK, S::NT>(bs_u32 + s * S::B_STAGE * 4, b_tile + s * b_kstep, p.ldb, cols_n,
                                          k_total - s * BK);
        else
        ms_load_stage<BN, BK, S::NT, S::LDB_S, !BNC, VEC>(bs_u32 + s * S::B_STAGE * 4, b_tile + s * b_kstep,
                                                          p.ldb, cols_n, k_total - s * BK);
      }
      cp_async_commit();
    }

    int rd = 0;               // ring slot being consumed
    int wr = STAGES - 1;      // ring slot being filled
    for (int kt = 0; kt < ktiles; ++kt) {
      cp_async_wait<STAGES - 2>();
      __syncthreads();
      const int nk = kt + STAGES - 1;
      if (nk < ktiles) {
        ms_load_stage<BM, BK, S::NT, S::LDA_S, AK, VEC>(as_u32 + wr * S::A_STAGE * 4, a_tile + nk * a_kstep,
                                                        p.lda, rows_m, k_total - nk * BK);
        if constexpr (BKS)
          ms_load_stage_kc<BN, BK, S::NT>(bs_u32 + wr * S::B_STAGE * 4, b_tile + nk * b_kstep, p.ldb, cols_n,
                                          k_total - nk * BK);
        else
        ms_load_stage<BN, BK, S::NT, S::LDB_S, !BNC, VEC>(bs_u32 + wr * S::B_STAGE * 4, b_tile + nk * b_kstep,
                                                          p.ldb, cols_n, k_total - nk * BK);
      }
      cp_async_commit();
      wr = (wr + 1 == STAGES) ? 0 : wr + 1;

      const float* as = As + rd * S::A_STAGE + ty * 4;
      const float* bs = Bs + rd * S::B_STAGE + (BKS ? tx * 4 * BK : tx * 4);
      rd = (rd + 1 == STAGES) ? 0 : rd + 1;
      const int kcur = min(k_total - kt * BK, BK);
      if constexpr (BKS) {
        // B fragment: for each of the TN columns one 128-bit read covers 4 kk
        // (column n = q*BN/QN + tx*4 + c; chunk XOR (n/4)%CPR == tx%CPR).
        const int swz = tx & (S::CPR - 1);
        if (kcur == BK) {
#pragma unroll
          for (int k4 = 0; k4 < BK / 4; ++k4) {
            float4 bq[TN];
#pragma unroll
            for (int q = 0; q < S::QN; ++q)
#pragma unroll
              for (int c = 0; c < 4; ++c)
                bq[q * 4 + c] = *reinterpret_cast<const float4*>(bs + (q * (BN / S::QN) + c) * BK + ((k4 ^ swz) * 4));
#pragma unroll
            for (int k1 = 0; k1 < 4; ++k1) {
              const int kk = k4 * 4 + k1;
              float af[TM], bf[TN];
#pragma unroll
              for (int q = 0; q < S::QM; ++q) {
                const float4 t = *reinterpret_cast<const float4*>(as + kk * S::LDA_S + q * (BM / S::QM));
                af[q * 4 + 0] = t.x; af[q * 4 + 1] = t.y; af[q * 4 + 2] = t.z; af[q * 4 + 3] = t.w;
              }
#pragma unroll
              for (int j = 0; j < TN; ++j)
                bf[j] = k1 == 0 ? bq[j].x : k1 == 1 ? bq[j].y : k1 == 2 ? bq[j].z : bq[j].w;
              outer_ffma2<TM, TN>(acc2, af, bf);
            }
          }
        } else {
#pragma unroll 1
          for (int kk = 0; kk < kcur; ++kk) {
            float af[TM], bf[TN];
#pragma unroll
            for (int q = 0; q < S::QM; ++q) {
              const float4 t = *reinterpret_cast<const float4*>(as + kk * S::LDA_S + q * (BM / S::QM));
              af[q * 4 + 0] = t.x; af[q * 4 + 1] = t.y; af[q * 4 + 2] = t.z; af[q * 4 + 3] = t.w;
            }
            const int off = (((kk >> 2) ^ swz) * 4) + (kk & 3);
#pragma unroll
            for (int q = 0; q < S::QN; ++q)
#pragma unroll
              for (int c = 0; c < 4; ++c) bf[q * 4 + c] = bs[(q * (BN / S::QN) + c) * BK + off];
            outer_ffma2<TM, TN>(acc2, af, bf);
          }
        }
      } else if (kcur == BK) {
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
          float af[TM], bf[TN];
#pragma unroll
          for (int q = 0; q < S::QM; ++q) {
            const float4 t = *reinterpret_cast<const float4*>(as + kk * S::LDA_S + q * (BM / S::QM));
            af[q * 4 + 0] = t.x; af[q * 4 + 1] = t.y; af[q * 4 + 2] = t.z; af[q * 4 + 3] = t.w;
          }
#pragma unroll
          for (int q = 0; q < S::QN; ++q) {
            const float4 t = *reinterpret_cast<const float4*>(bs + kk * S::LDB_S + q * (BN / S::QN));
            bf[q * 4 + 0] = t.x; bf[q * 4 + 1] = t.y; bf[q * 4 + 2] = t.z; bf[q * 4 + 3] = t.w;
          }
          outer_ffma2<TM, TN>(acc2, af, bf);
        }
      } else {
        // K tail: exactly kcur more FMAs per element (no zero padding).
#pragma unroll 1
        for (int kk = 0; kk < kcur; ++kk) {
          float af[TM], bf[TN];
#pragma unroll
          for (int q = 0; q < S::QM; ++q) {
            const float4 t = *reinterpret_cast<const float4*>(as + kk * S::LDA_S + q * (BM / S::QM));
            af[q * 4 + 0] = t.x; af[q * 4 + 1] = t.y; af[q * 4 + 2] = t.z; af[q * 4 + 3] = t.w;
          }
#pragma unroll
          for (int q = 0; q < S::QN; ++q) {
            const float4 t = *reinterpret_cast<const float4*>(bs + kk * S::LDB_S + q * (BN / S::QN));
            bf[q * 4 + 0] = t.x; bf[q * 4 + 1] = t.y; bf[q * 4 + 2] = t.z; bf[q * 4 + 3] = t.w;
          }
          outer_ffma2<TM, TN>(acc2, af, bf);
        }
      }
    }
    cp_async_wait<0>();
  }

  // Epilogue: rows (q*BM/QM + ty*4 + r), cols (q*BN/QN + tx*4 + c).
#define ACC2(i, j) (((i) & 1) ? acc2[(i) >> 1][j].y : acc2[(i) >> 1][j].x)
  const int64_t cbase_off = inst_off(p.c_off, p.stride_c, p.c_offs, z);
  float* C = static_cast<float*>(p.c) + cbase_off;
  const bool cvec = ((reinterpret_cast<uintptr_t>(C) & 15) == 0) && ((p.ldc & 3) == 0);
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
