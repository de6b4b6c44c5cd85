// sgemm_tma.cuh — FP32 GEMM on the paired FFMA pipe fed by TMA (sm_100a).
//
// Replaces the reference's tiled FP32 arithmetic (_tile_product,
// pkg/src/tunedblas/kernels/compute.py:360-381, driven by gemm_indirect_tasks
// compute.py:384-420) for large SGEMMs with 16-byte aligned operands and
// arithmetic batch offsets.
//
// Determinism contract (as sgemm_simt.cuh / sgemm_ms.cuh): every output
// element is the ascending-k chain acc = fmaf(opA(i,kk), opB(kk,j), acc) of
// exactly k FMAs (the K tail is iterated with a runtime bound, never padded),
// then the reference epilogue — bitwise equal to every other S kernel and the
// sequential-k C oracle.
//
// Why TMA for an FFMA kernel: with FFMA2 (two FP32 FMA lanes per
// instruction) the outer product needs half the issue slots, and what is left
// of the non-FFMA work — per-thread cp.async address arithmetic (IMAD runs on
// the FMA pipe) — was measured to cost 10-25 % of the FMA pipe.  Here one
// thread issues two cp.async.bulk.tensor per BK-deep stage and every other
// instruction in the main loop is an LDS.128 or an FFMA2.
//
// Shared-memory layouts (one stage = A tile + B tile, 1024-byte aligned):
//   M/N-contiguous operand: [BK][ROWS] floats, no swizzle (TMA box {ROWS, BK});
//     fragments are 128-bit reads of 4 consecutive rows at one kk.
//   K-contiguous operand:   [ROWS][BK=32] floats, SWIZZLE_128B (TMA box
//     {32, ROWS}): 16-byte chunk c of row r lives at chunk c ^ (r & 7).  A
//     thread owns rows r = j*T + t (strided) so the 4..8 distinct rows a warp
//     reads at once are consecutive -> distinct chunks -> no bank conflicts;
//     one 128-bit read yields 4 consecutive kk of one row.
// FFMA2 pairs: along M (A fragments come as float4 along M) unless A is
// K-contiguous, then along N (B must be N-contiguous; both-K-contiguous
// operands use the register-staged kernel, sgemm_simt.cuh).
#pragma once

#include <type_traits>

#include "common.cuh"

namespace tb {

template <int BM, int BN, int BK, int TM, int TN, int STAGES, bool A_MN, bool B_MN, bool XP = false>
struct TmaSgemmCfg {
  static constexpr int TY = BM / TM, TX = BN / TN;
  static constexpr int NT = TY * TX;
  static constexpr int NW = NT / 32;
  static constexpr int QM = TM / 4, QN = TN / 4;
  // both operands K-contiguous: A is transposed in shared memory once per
  // stage ([BM][32] -> [32][BM], double-buffered) and then read like an
  // M-contiguous A
  // XP: transpose every K-contiguous operand the same way (B too)
  static constexpr bool A_T = !A_MN && (!B_MN || XP);
  static constexpr bool B_T = !B_MN && XP;
  static constexpr bool PAIR_N = !A_MN && !A_T;
  static constexpr int A_BYTES = BM * BK * 4, B_BYTES = BN * BK * 4;
  // B slot rounded up to 1024 bytes (BN = 60: 7680 B of data in an 8 KB slot)
  static constexpr int B_ALLOC = (B_BYTES + 1023) / 1024 * 1024;
  static constexpr int STAGE_BYTES = A_BYTES + B_ALLOC;
  static constexpr int TX_BYTES = A_BYTES + B_BYTES;  // bytes the two TMA boxes land
  static constexpr int T_BYTES = (A_T ? 2 * A_BYTES : 0) + (B_T ? 2 * B_BYTES : 0);
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + T_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  static_assert(BK == 32, "K-contiguous tiles are 128-byte SWIZZLE_128B rows");
  static_assert(TM % 4 == 0 && TN % 4 == 0 && NT % 32 == 0, "tile shape");
  static_assert(A_BYTES % 1024 == 0, "1024-byte aligned stage tiles");
  static_assert(!A_T || (BM * (BK / 4)) % NT == 0, "A transpose covers the tile");
  static_assert(!B_T || (BN * (BK / 4)) % NT == 0, "B transpose covers the tile");
};

template <int TM, int TN>
__device__ __forceinline__ void outer_ffma2_n(float2 (&acc2)[TM][TN / 2], const float (&af)[TM],
                                              const float (&bf)[TN]) {
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j2 = 0; j2 < TN / 2; ++j2)
      acc2[i][j2] = __ffma2_rn(make_float2(af[i], af[i]), make_float2(bf[2 * j2], bf[2 * j2 + 1]),
                               acc2[i][j2]);
}

// KS > 1: deterministic split-K over a thread-block cluster of KS CTAs
// (launched with cluster dims (KS,1,1)): rank r runs the 32-deep K stages
// [r*kt_per, (r+1)*kt_per) of the tile (kt_per = ceil(ktiles / KS)), i.e.
// the ascending-k FMA chain of its K range from 0; ranks 1.. park their
// accumulators in their own shared memory, and rank 0 reads them through
// DSMEM and adds them in rank order — ((p0 + p1) + p2) + p3, one rounded
// FP32 add each — before the reference epilogue.  The split is chosen from
// (m, n, k) only (sgemm_tma.cu), so single, batched and looped calls of a
// shape agree bitwise; against the sequential-k oracle the result is the
// same chain cut at the rank boundaries (tests: oracle seqk over each K
// range, then the rank-order sum).
template <int BM, int BN, int BK, int TM, int TN, int STAGES, bool A_MN, bool B_MN, int MINB, bool XP = false,
          int KS = 1>
__global__ void __launch_bounds__(TmaSgemmCfg<BM, BN, BK, TM, TN, STAGES, A_MN, B_MN, XP>::NT, MINB)
    sgemm_tma_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                     Problem p, int tiles_m, int tiles_n, int group_m) {
  using Cfg = TmaSgemmCfg<BM, BN, BK, TM, TN, STAGES, A_MN, B_MN, XP>;
  constexpr bool PN = Cfg::PAIR_N;
  extern __shared__ __align__(1024) uint8_t tma_smem_raw[];
  uint8_t* smem = smem_align1024(tma_smem_raw);
  float* a_t = reinterpret_cast<float*>(smem + STAGES * Cfg::STAGE_BYTES);  // A_T buffers
  float* b_t = a_t + (Cfg::A_T ? 2 * BM * BK : 0);                            // B_T buffers
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES + Cfg::T_BYTES);
  uint64_t* empty = full + STAGES;

  const int tid = threadIdx.x;
  const int lane = tid % 32;

  // tile coordinates (grouped rasterisation), one tile per CTA (per
  // cluster of KS CTAs when K is split)
  const int64_t per_inst = static_cast<int64_t>(tiles_m) * tiles_n;
  const int64_t tile_id = blockIdx.x / KS;
  const int krank = KS > 1 ? static_cast<int>(blockIdx.x % KS) : 0;
  // one tile per instance (the batched small shapes): no 64-bit division
  // and no raster arithmetic in the prologue of these short-lived CTAs
  // (ncu: the division and its branches were among the top stall sites)
  // (the host keeps blocks * KS < 2^31, so 32-bit arithmetic is exact)
  const int z = per_inst == 1 ? static_cast<int>(tile_id)
                              : static_cast<int>(tile_id) / static_cast<int>(per_inst);
  int mt = 0, nt = 0;
  if (per_inst != 1) {
    const int r = static_cast<int>(tile_id) - z * static_cast<int>(per_inst);
    const int group_size = group_m * tiles_n;
    const int g = r / group_size;
    const int first_m = g * group_m;
    const int gm = min(tiles_m - first_m, group_m);
    const int rr = r - g * group_size;
    mt = first_m + rr % gm;
    nt = rr / gm;
  }
  const int m0 = mt * BM, n0 = nt * BN;
  const int rows_m = static_cast<int>(min64(BM, p.m - m0));
  const int cols_n = static_cast<int>(min64(BN, p.n - n0));
  const int k_total = static_cast<int>(min64(p.k, 0x7fffffff));
  const int ktiles_all = (k_total + BK - 1) / BK;
  // this CTA's K stages [kt0, kt0 + ktiles)
  const int kt_per = KS > 1 ? (ktiles_all + KS - 1) / KS : ktiles_all;
  const int kt0 = min(ktiles_all, krank * kt_per);
  const int ktiles = min(ktiles_all, kt0 + kt_per) - kt0;

  if (tid == 0) {
    tma_prefetch_desc(&tmap_a);
    tma_prefetch_desc(&tmap_b);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], Cfg::NW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  grid_dep_wait();  // prologue above overlapped the previous kernel (PDL)
  grid_dep_launch();

  auto issue = [&](int t) {  // local stage t -> slot t % STAGES (tid 0 only)
    const int s = t % STAGES;
    const int kg = (kt0 + t) * BK;  // global K coordinate
    uint8_t* sa = smem + s * Cfg::STAGE_BYTES;
    uint8_t* sb = sa + Cfg::A_BYTES;
    mbar_arrive_expect_tx(&full[s], Cfg::TX_BYTES);
    if (A_MN) tma_load_3d(sa, &tmap_a, &full[s], m0, kg, z);
    else      tma_load_3d(sa, &tmap_a, &full[s], kg, m0, z);
    if (B_MN) tma_load_3d(sb, &tmap_b, &full[s], n0, kg, z);
    else      tma_load_3d(sb, &tmap_b, &full[s], kg, n0, z);
  };
  if (tid == 0) {
    for (int t = 0; t < STAGES && t < ktiles; ++t) issue(t);
  }

  const int ty = tid % Cfg::TY;  // M index (fastest)
  const int tx = tid / Cfg::TY;  // N index

  float2 acc2[PN ? TM : TM / 2][PN ? TN / 2 : TN];
#pragma unroll
  for (int i = 0; i < (PN ? TM : TM / 2); ++i)
#pragma unroll
    for (int j = 0; j < (PN ? TN / 2 : TN); ++j) acc2[i][j] = make_float2(0.0f, 0.0f);

  // per-thread fragment offsets (floats) inside a stage tile
  //   MN operand: kk*ROWS + q*(ROWS/Q) + t*4
  //   K  operand: (j*T + t)*BK + ((k4 ^ ((j*T + t) & 7)) * 4)
  const int a_sw = ty & 7;  // (j*TY + ty) & 7 == ty & 7 when TY % 8 == 0
  const int b_sw = tx & 7;
  static_assert(A_MN || Cfg::A_T || Cfg::TY % 8 == 0, "A swizzle phase per thread");
  constexpr bool A_FRAG_MN = A_MN || Cfg::A_T;  // A fragments read from an M-contiguous tile
  static_assert(B_MN || Cfg::B_T || Cfg::TX % 8 == 0, "B swizzle phase per thread");
  constexpr bool B_FRAG_MN = B_MN || Cfg::B_T;

  for (int kt = 0; kt < ktiles; ++kt) {
    const int s = kt % STAGES;
    const uint32_t ph = (kt / STAGES) & 1;
    // refill the slot released one stage ago (tid 0; every warp has already
    // arrived on empty[] for it or arrives shortly)
    if (tid == 0 && kt >= 1 && kt - 1 + STAGES < ktiles) {
      const int t = kt - 1 + STAGES;
      mbar_wait(&empty[(kt - 1) % STAGES], ((kt - 1) / STAGES) & 1);
      issue(t);
    }
    mbar_wait(&full[s], ph);
    const float* sa = reinterpret_cast<const float*>(smem + s * Cfg::STAGE_BYTES);
    const float* sb = reinterpret_cast<const float*>(smem + s * Cfg::STAGE_BYTES + Cfg::A_BYTES);
    if constexpr (Cfg::A_T || Cfg::B_T) {
      // [ROWS][32] SWIZZLE_128B -> [32][ROWS]: lanes take consecutive rows of
      // one 16-byte chunk column (8-row groups cover all banks on the read,
      // the 4 scalar writes per chunk are unit-stride across the warp)
      auto xpose = [&](const float* src, float* dst, auto rows_c) {
        constexpr int ROWS = decltype(rows_c)::value;
#pragma unroll
        for (int j = 0; j < ROWS * (BK / 4) / Cfg::NT; ++j) {
          const int e = tid + j * Cfg::NT;
          const int r = e % ROWS, c = e / ROWS;
          const float4 v = *reinterpret_cast<const float4*>(src + r * BK + ((c ^ (r & 7)) * 4));
          dst[(4 * c + 0) * ROWS + r] = v.x;
          dst[(4 * c + 1) * ROWS + r] = v.y;
          dst[(4 * c + 2) * ROWS + r] = v.z;
          dst[(4 * c + 3) * ROWS + r] = v.w;
        }
      };
      if constexpr (Cfg::A_T) {
        float* dst = a_t + (kt & 1) * (BM * BK);
        xpose(sa, dst, std::integral_constant<int, BM>{});
        sa = dst;
      }
      if constexpr (Cfg::B_T) {
        float* dst = b_t + (kt & 1) * (BN * BK);
        xpose(sb, dst, std::integral_constant<int, BN>{});
        sb = dst;
      }
      __syncthreads();
    }
    const int kcur = min(k_total - (kt0 + kt) * BK, BK);

    auto step = [&](const float (&af)[TM], const float (&bf)[TN]) {
      if constexpr (PN) outer_ffma2_n<TM, TN>(acc2, af, bf);
      else outer_ffma2<TM, TN>(acc2, af, bf);
    };
    auto load_a_mn = [&](int kk, float (&af)[TM]) {
#pragma unroll
      for (int q = 0; q < Cfg::QM; ++q) {
        const float4 t = *reinterpret_cast<const float4*>(sa + kk * BM + q * (BM / Cfg::QM) + ty * 4);
        af[q * 4 + 0] = t.x; af[q * 4 + 1] = t.y; af[q * 4 + 2] = t.z; af[q * 4 + 3] = t.w;
      }
    };
    auto load_b_mn = [&](int kk, float (&bf)[TN]) {
#pragma unroll
      for (int q = 0; q < Cfg::QN; ++q) {
        const float4 t = *reinterpret_cast<const float4*>(sb + kk * BN + q * (BN / Cfg::QN) + tx * 4);
        bf[q * 4 + 0] = t.x; bf[q * 4 + 1] = t.y; bf[q * 4 + 2] = t.z; bf[q * 4 + 3] = t.w;
      }
    };

    if (kcur == BK) {
#pragma unroll
      for (int k4 = 0; k4 < BK / 4; ++k4) {
        float4 aq[A_FRAG_MN ? 1 : TM], bq[B_FRAG_MN ? 1 : TN];
        if constexpr (!A_FRAG_MN) {
#pragma unroll
          for (int i = 0; i < TM; ++i)
            aq[i] = *reinterpret_cast<const float4*>(sa + (i * Cfg::TY + ty) * BK + ((k4 ^ a_sw) * 4));
        }
        if constexpr (!B_FRAG_MN) {
#pragma unroll
          for (int j = 0; j < TN; ++j)
            bq[j] = *reinterpret_cast<const float4*>(sb + (j * Cfg::TX + tx) * BK + ((k4 ^ b_sw) * 4));
        }
#pragma unroll
        for (int k1 = 0; k1 < 4; ++k1) {
          const int kk = k4 * 4 + k1;
          float af[TM], bf[TN];
          if constexpr (A_FRAG_MN) {
            load_a_mn(kk, af);
          } else {
#pragma unroll
            for (int i = 0; i < TM; ++i) af[i] = k1 == 0 ? aq[i].x : k1 == 1 ? aq[i].y : k1 == 2 ? aq[i].z : aq[i].w;
          }
          if constexpr (B_FRAG_MN) {
            load_b_mn(kk, bf);
          } else {
#pragma unroll
            for (int j = 0; j < TN; ++j) bf[j] = k1 == 0 ? bq[j].x : k1 == 1 ? bq[j].y : k1 == 2 ? bq[j].z : bq[j].w;
          }
          step(af, bf);
        }
      }
    } else {
      // K tail: exactly kcur more FMAs per element (TMA zero-filled the rest)
#pragma unroll 1
      for (int kk = 0; kk < kcur; ++kk) {
        float af[TM], bf[TN];
        if constexpr (A_FRAG_MN) {
          load_a_mn(kk, af);
        } else {
#pragma unroll
          for (int i = 0; i < TM; ++i)
            af[i] = sa[(i * Cfg::TY + ty) * BK + (((kk >> 2) ^ a_sw) * 4) + (kk & 3)];
        }
        if constexpr (B_FRAG_MN) {
          load_b_mn(kk, bf);
        } else {
#pragma unroll
          for (int j = 0; j < TN; ++j)
            bf[j] = sb[(j * Cfg::TX + tx) * BK + (((kk >> 2) ^ b_sw) * 4) + (kk & 3)];
        }
        step(af, bf);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  if constexpr (KS > 1) {
    static_assert(BM * BN * 4 <= STAGES * Cfg::STAGE_BYTES + Cfg::T_BYTES, "partials parked in the ring");
    // ---- split-K: ranks 1.. park their partials, rank 0 adds them in order ----
    // Every stage this CTA loaded has been consumed, so the ring is free.
    constexpr int NACC = (PN ? TM : TM / 2) * (PN ? TN / 2 : TN);  // float2 per thread
    float2* park = reinterpret_cast<float2*>(smem) + static_cast<size_t>(tid) * NACC;
    __syncthreads();  // every warp is done reading the ring
    if (krank != 0) {
#pragma unroll
      for (int i = 0; i < (PN ? TM : TM / 2); ++i)
#pragma unroll
        for (int j = 0; j < (PN ? TN / 2 : TN); ++j) park[i * (PN ? TN / 2 : TN) + j] = acc2[i][j];
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (krank == 0) {
      const uint32_t park_s = smem_u32(park);
#pragma unroll
      for (int q = 1; q < KS; ++q) {
        uint32_t remote;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(park_s), "r"(q));
#pragma unroll
        for (int i = 0; i < (PN ? TM : TM / 2); ++i)
#pragma unroll
          for (int j = 0; j < (PN ? TN / 2 : TN); j += 2) {
            float4 v;
            asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];"
                         : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                         : "r"(remote + static_cast<uint32_t>((i * (PN ? TN / 2 : TN) + j) * 8)));
            acc2[i][j].x = __fadd_rn(acc2[i][j].x, v.x);
            acc2[i][j].y = __fadd_rn(acc2[i][j].y, v.y);
            acc2[i][j + 1].x = __fadd_rn(acc2[i][j + 1].x, v.z);
            acc2[i][j + 1].y = __fadd_rn(acc2[i][j + 1].y, v.w);
          }
      }
    }
    // peers keep their shared memory until rank 0 has read it
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (krank != 0) return;
  }

  // ---- epilogue (reference order: alpha*acc, then + beta*C) ----
  Epi epi;
  epi.alpha = inst_alpha(p, z);
  epi.beta = inst_beta(p, z);
  epi.skip_ab = (epi.alpha == 0.0f) || (p.k == 0);
  float* C = static_cast<float*>(p.c) + inst_off(p.c_off, p.stride_c, p.c_offs, z);
  auto acc_at = [&](int i, int j) -> float {
    if constexpr (PN) return (j & 1) ? acc2[i][j >> 1].y : acc2[i][j >> 1].x;
    else return (i & 1) ? acc2[i >> 1][j].y : acc2[i >> 1][j].x;
  };
  auto col_of = [&](int j) -> int {
    if constexpr (B_FRAG_MN) return (j / 4) * (BN / Cfg::QN) + tx * 4 + (j % 4);
    else return j * Cfg::TX + tx;
  };
  if constexpr (A_FRAG_MN) {
    // rows q*(BM/QM) + ty*4 + r: 4 consecutive rows per 128-bit store
    const bool cvec = ((reinterpret_cast<uintptr_t>(C) & 15) == 0) && ((p.ldc & 3) == 0);
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int col = col_of(j);
      if (col >= cols_n) continue;
      float* ccol = C + (static_cast<int64_t>(n0) + col) * p.ldc + m0;
#pragma unroll
      for (int q = 0; q < Cfg::QM; ++q) {
        const int row = q * (BM / Cfg::QM) + ty * 4;
        if (cvec && row + 3 < rows_m) {
          float4 cv = make_float4(0.f, 0.f, 0.f, 0.f);
          if (epi.reads_c()) cv = *reinterpret_cast<const float4*>(ccol + row);
          float4 o;
          o.x = epi.apply(acc_at(q * 4 + 0, j), cv.x);
          o.y = epi.apply(acc_at(q * 4 + 1, j), cv.y);
          o.z = epi.apply(acc_at(q * 4 + 2, j), cv.z);
          o.w = epi.apply(acc_at(q * 4 + 3, j), cv.w);
          *reinterpret_cast<float4*>(ccol + row) = o;
        } else {
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            if (row + r < rows_m) {
              const float cv = epi.reads_c() ? ccol[row + r] : 0.0f;
              ccol[row + r] = epi.apply(acc_at(q * 4 + r, j), cv);
            }
          }
        }
      }
    }
  } else {
    // rows i*TY + ty: a warp's lanes cover consecutive rows of one column
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int col = col_of(j);
      if (col >= cols_n) continue;
      float* ccol = C + (static_cast<int64_t>(n0) + col) * p.ldc + m0;
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        const int row = i * Cfg::TY + ty;
        if (row < rows_m) {
          const float cv = epi.reads_c() ? ccol[row] : 0.0f;
          ccol[row] = epi.apply(acc_at(i, j), cv);
        }
      }
    }
  }
}

}  // namespace tb
