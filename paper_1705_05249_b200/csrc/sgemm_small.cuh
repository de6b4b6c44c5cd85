// sgemm_small.cuh — FP32 GEMM for small instances (m <= MI, n <= NI), the
// batched small-matrix path (BASELINE config C4) on the FFMA pipe.
//
// Persistent CTAs of 256 threads stream "stages" = (group of G instances,
// 32-deep K chunk) through a STAGES-deep cp.async ring in shared memory
// (Ampere-style multistage main loop: wait oldest group, barrier, refill the
// slot just freed, compute).  G = 256*16 / (MI*NI) instances share a stage,
// each computed by MI*NI/16 threads with a 4x4 register micro-tile.
//
// Operands keep their global major-ness in shared memory (cp.async moves
// 16-byte chunks along the contiguous dimension, zero-filling tails); the
// compute loop reads 128-bit fragments along M/N for MN-contiguous operands
// and along K (4 k-steps at a time) for K-contiguous ones.  Each output
// element is the same sequential-k FMA chain as every other SGEMM kernel
// (exactly k FMAs in ascending k; the zero-filled tail is never multiplied),
// so results are bitwise identical to sgemm_simt and the C oracle.
#pragma once

#include "common.cuh"

namespace tb {

template <int MI, int NI, int TM = 4, int TN = 4>
struct SsCfg {
  static constexpr int KC = 32;
  static constexpr int KCP = KC + 4;                    // padded K-contiguous row (floats)
  static constexpr int TY = MI / TM, TX = NI / TN;      // threads per instance = TX*TY
  static constexpr int QM = TM / 4, QN = TN / 4;        // 4x4 sub-blocks, spaced MI/QM, NI/QN
  static constexpr int TPI = TX * TY;
  static constexpr int G = 256 / TPI;                   // instances per stage
  // smem per instance slot: A as [KC][MI] (M-contig) or [MI][KCP]
  // (K-contig, rows padded by 4 floats: 16-byte aligned chunks, and the
  // fragment reads are quarter-warp broadcasts, so the padding costs no
  // conflicts while every read address is base + immediate)
  static constexpr int A_ELEMS_M = KC * MI, A_ELEMS_K = MI * KCP;
  static constexpr int B_ELEMS_N = KC * NI, B_ELEMS_K = NI * KCP;
  static constexpr int A_ELEMS = A_ELEMS_K > A_ELEMS_M ? A_ELEMS_K : A_ELEMS_M;
  static constexpr int B_ELEMS = B_ELEMS_K > B_ELEMS_N ? B_ELEMS_K : B_ELEMS_N;
  static constexpr int STAGE_FLOATS = G * (A_ELEMS + B_ELEMS);
  // 3-4 stages, <= ~100 KB so two CTAs share an SM
  static constexpr int STAGES = (4 * STAGE_FLOATS * 4 <= 110 * 1024) ? 4 : 3;
  static constexpr int SMEM_BYTES = STAGES * STAGE_FLOATS * 4;
  // 8x8 micro-tiles need > 128 registers: one CTA per SM
  static constexpr int MINB = (TM * TN >= 64) ? 1 : 2;
};

template <int MI, int NI, int TM, int TN, bool AK, bool BNC>
__global__ void __launch_bounds__(256, (SsCfg<MI, NI, TM, TN>::MINB))
    sgemm_small_kernel(Problem p, int64_t groups) {
  using C = SsCfg<MI, NI, TM, TN>;
  grid_dep_wait();  // PDL: the previous kernel's writes are visible from here
  constexpr int QM = C::QM, QN = C::QN;
  constexpr int KC = C::KC, G = C::G, STAGES = C::STAGES;
  // K-contiguous slot layout: element (row, kk) of a [rows][KCP] tile
  auto kidx = [](int row, int kk) { return row * C::KCP + kk; };
  extern __shared__ __align__(16) float smem_f[];

  const int tid = threadIdx.x;
  const int slot = tid / C::TPI;
  const int lt = tid % C::TPI;
  const int ty = lt % C::TY, tx = lt / C::TY;
  const int m = static_cast<int>(p.m), n = static_cast<int>(p.n);
  const int kchunks = static_cast<int>((p.k + KC - 1) / KC);
  const float* A = static_cast<const float*>(p.a);
  const float* B = static_cast<const float*>(p.b);

  // Stage sequence of this CTA: (group gi, chunk kc), gi = blockIdx.x + j*gridDim.x
  const int64_t my_groups = (groups - blockIdx.x + gridDim.x - 1) / gridDim.x;
  const int64_t total = my_groups * kchunks;

  auto stage_ptr = [&](int s) { return smem_f + s * C::STAGE_FLOATS; };

  // Issue the cp.async copies of stage index `si` into ring slot `s`.
  // Chunk j of thread t is element chunk e = t + 256 j of the stage; since
  // every per-instance chunk count is a multiple of 256 the instance slot of
  // chunk j is a compile-time constant and its position a per-thread
  // constant, so only the instance pointers are computed per stage.
  constexpr int A_CH = MI * KC / 4, B_CH = NI * KC / 4;
  static_assert(A_CH % 256 == 0 && B_CH % 256 == 0, "whole chunks per thread");
  // Single-chunk K (k <= KC, every C4 case): each thread's chunk offsets and
  // valid counts are stage-invariant — computed once into a compact plan
  // (32-bit offsets + 3-bit counts), so a stage only adds instance bases.
  constexpr int NA = G * A_CH / 256, NB = G * B_CH / 256;
  static_assert(NA + NB <= 21, "plan packs 3-bit counts into one 64-bit word");
  const bool planned = kchunks == 1 && p.lda * (AK ? MI : KC) < (1LL << 31) &&
                       p.ldb * (!BNC ? NI : KC) < (1LL << 31);
  int32_t plan_off[NA + NB];
  uint64_t plan_valid = 0;
  if (planned) {
    const int k_left = static_cast<int>(p.k);
#pragma unroll
    for (int j = 0; j < NA; ++j) {
      const int r = (256 * j) % A_CH + tid;
      int row, kk, valid;
      if (AK) { row = r / (KC / 4); kk = (r % (KC / 4)) * 4; }
      else { kk = r / (MI / 4); row = (r % (MI / 4)) * 4; }
      if (AK) { valid = (row < m) ? max(0, min(4, k_left - kk)) : 0; plan_off[j] = static_cast<int32_t>(row * p.lda + kk); }
      else { valid = (kk < k_left) ? max(0, min(4, m - row)) : 0; plan_off[j] = static_cast<int32_t>(kk * p.lda + row); }
      plan_valid |= static_cast<uint64_t>(valid) << (3 * j);
    }
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      const int r = (256 * j) % B_CH + tid;
      int col, kk, valid;
      if (!BNC) { col = r / (KC / 4); kk = (r % (KC / 4)) * 4; }
      else { kk = r / (NI / 4); col = (r % (NI / 4)) * 4; }
      if (!BNC) { valid = (col < n) ? max(0, min(4, k_left - kk)) : 0; plan_off[NA + j] = static_cast<int32_t>(col * p.ldb + kk); }
      else { valid = (kk < k_left) ? max(0, min(4, n - col)) : 0; plan_off[NA + j] = static_cast<int32_t>(kk * p.ldb + col); }
      plan_valid |= static_cast<uint64_t>(valid) << (3 * (NA + j));
    }
  }

  auto issue = [&](int64_t gi, int kc, int s) {
    const int64_t k0 = static_cast<int64_t>(kc) * KC;
    const int k_left = static_cast<int>(min64(KC, p.k - k0));
    float* st = stage_ptr(s);
    const float* ia[G];
    const float* ib[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int64_t z = gi * G + g;
      ia[g] = z < p.batch ? A + inst_off(p.a_off, p.stride_a, p.a_offs, z) : nullptr;
      ib[g] = z < p.batch ? B + inst_off(p.b_off, p.stride_b, p.b_offs, z) : nullptr;
    }
    if (planned) {
#pragma unroll
      for (int j = 0; j < NA; ++j) {
        const int g = (256 * j) / A_CH;
        const int r = (256 * j) % A_CH + tid;
        const int row = AK ? r / (KC / 4) : (r % (MI / 4)) * 4;
        const int kk = AK ? (r % (KC / 4)) * 4 : r / (MI / 4);
        uint32_t valid = static_cast<uint32_t>(plan_valid >> (3 * j)) & 7u;
        if (ia[g] == nullptr) valid = 0;
        float* dst = st + g * C::A_ELEMS + (AK ? kidx(row, kk) : kk * MI + row);
        cp_async_16(dst, valid ? ia[g] + plan_off[j] : A, valid * 4u);
      }
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        const int g = (256 * j) / B_CH;
        const int r = (256 * j) % B_CH + tid;
        const int col = !BNC ? r / (KC / 4) : (r % (NI / 4)) * 4;
        const int kk = !BNC ? (r % (KC / 4)) * 4 : r / (NI / 4);
        uint32_t valid = static_cast<uint32_t>(plan_valid >> (3 * (NA + j))) & 7u;
        if (ib[g] == nullptr) valid = 0;
        float* dst = st + G * C::A_ELEMS + g * C::B_ELEMS + (!BNC ? kidx(col, kk) : kk * NI + col);
        cp_async_16(dst, valid ? ib[g] + plan_off[NA + j] : B, valid * 4u);
      }
      return;
    }
#pragma unroll
    for (int j = 0; j < G * A_CH / 256; ++j) {
      const int g = (256 * j) / A_CH;
      const int r = (256 * j) % A_CH + tid;
      int row, kk;
      if (AK) { row = r / (KC / 4); kk = (r % (KC / 4)) * 4; }
      else { kk = r / (MI / 4); row = (r % (MI / 4)) * 4; }
      int valid;
      int64_t eoff;
      if (AK) {
        valid = (row < m) ? max(0, min(4, k_left - kk)) : 0;
        eoff = static_cast<int64_t>(row) * p.lda + k0 + kk;
      } else {
        valid = (kk < k_left) ? max(0, min(4, m - row)) : 0;
        eoff = (k0 + kk) * p.lda + row;
      }
      if (ia[g] == nullptr) valid = 0;
      float* dst = st + g * C::A_ELEMS + (AK ? kidx(row, kk) : kk * MI + row);
      cp_async_16(dst, valid > 0 ? ia[g] + eoff : A, static_cast<uint32_t>(valid) * 4u);
    }
#pragma unroll
    for (int j = 0; j < G * B_CH / 256; ++j) {
      const int g = (256 * j) / B_CH;
      const int r = (256 * j) % B_CH + tid;
      int col, kk;
      if (!BNC) { col = r / (KC / 4); kk = (r % (KC / 4)) * 4; }   // K-contiguous
      else { kk = r / (NI / 4); col = (r % (NI / 4)) * 4; }         // N-contiguous
      int valid;
      int64_t eoff;
      if (!BNC) {
        valid = (col < n) ? max(0, min(4, k_left - kk)) : 0;
        eoff = static_cast<int64_t>(col) * p.ldb + k0 + kk;
      } else {
        valid = (kk < k_left) ? max(0, min(4, n - col)) : 0;
        eoff = (k0 + kk) * p.ldb + col;
      }
      if (ib[g] == nullptr) valid = 0;
      float* dst = st + G * C::A_ELEMS + g * C::B_ELEMS + (!BNC ? kidx(col, kk) : kk * NI + col);
      cp_async_16(dst, valid > 0 ? ib[g] + eoff : B, static_cast<uint32_t>(valid) * 4u);
    }
  };

  // Stage coordinates advance incrementally (no 64-bit division per stage):
  // chunk kc of group gi, then chunk 0 of group gi + gridDim.x.
  auto advance = [&](int64_t& gi, int& kc) {
    if (++kc == kchunks) {
      kc = 0;
      gi += gridDim.x;
    }
  };
  int64_t gi_i = blockIdx.x;  // next stage to issue
  int kc_i = 0;

  // prologue: STAGES-1 stages in flight
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < total) {
      issue(gi_i, kc_i, s);
      advance(gi_i, kc_i);
    }
    cp_async_commit();
  }
  int s_i = STAGES - 1, s_c = 0;  // ring slots: next issue / current compute
  int64_t gi = blockIdx.x;        // current compute stage
  int kc = 0;

  // Accumulators as FFMA2 pairs: along M when A fragments arrive as float4
  // along M (!AK), along N when only B's do (AK && BNC); scalar FFMA when both
  // operands are K-contiguous (pairs would need register moves).  Either way
  // each element is the same ascending-k chain of RN fmas.
  constexpr int PAIR = !AK ? 1 : (BNC ? 2 : 0);  // 1: (r, r+1), 2: (c, c+1), 0: scalar
  float2 acc2[TM * TN / 2];
  auto acc_ref = [&](int r, int c) -> float& {
    if (PAIR == 2) return (c & 1) ? acc2[r * (TN / 2) + (c >> 1)].y : acc2[r * (TN / 2) + (c >> 1)].x;
    return (r & 1) ? acc2[(r >> 1) * TN + c].y : acc2[(r >> 1) * TN + c].x;
  };
  auto fma_step = [&](const float (&a)[TM], const float (&b)[TN]) {
    if constexpr (PAIR == 1) {
#pragma unroll
      for (int r2 = 0; r2 < TM / 2; ++r2)
#pragma unroll
        for (int c = 0; c < TN; ++c)
          acc2[r2 * TN + c] = __ffma2_rn(make_float2(b[c], b[c]), make_float2(a[2 * r2], a[2 * r2 + 1]),
                                         acc2[r2 * TN + c]);
    } else if constexpr (PAIR == 2) {
#pragma unroll
      for (int r = 0; r < TM; ++r)
#pragma unroll
        for (int c2 = 0; c2 < TN / 2; ++c2)
          acc2[r * (TN / 2) + c2] = __ffma2_rn(make_float2(a[r], a[r]), make_float2(b[2 * c2], b[2 * c2 + 1]),
                                               acc2[r * (TN / 2) + c2]);
    } else {
#pragma unroll
      for (int r = 0; r < TM; ++r)
#pragma unroll
        for (int c = 0; c < TN; ++c) acc_ref(r, c) = __fmaf_rn(a[r], b[c], acc_ref(r, c));
    }
  };
#pragma unroll
  for (int i = 0; i < TM * TN / 2; ++i) acc2[i] = make_float2(0.0f, 0.0f);

  for (int64_t si = 0; si < total; ++si) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    // refill the slot consumed in the previous iteration
    if (si + STAGES - 1 < total) {
      issue(gi_i, kc_i, s_i);
      advance(gi_i, kc_i);
    }
    cp_async_commit();
    if (++s_i == STAGES) s_i = 0;

    const int s = s_c;
    if (++s_c == STAGES) s_c = 0;
    const int k_left = static_cast<int>(min64(KC, p.k - static_cast<int64_t>(kc) * KC));
    const float* as = stage_ptr(s) + slot * C::A_ELEMS;
    const float* bs = stage_ptr(s) + G * C::A_ELEMS + slot * C::B_ELEMS;
    // micro-tile rows: q*(MI/QM) + ty*4 + {0..3}; cols: q*(NI/QN) + tx*4 + {0..3}
    auto rowof = [&](int r) { return (r >> 2) * (MI / QM) + ty * 4 + (r & 3); };
    auto colof = [&](int c) { return (c >> 2) * (NI / QN) + tx * 4 + (c & 3); };

    // one 4-deep k group: fragments then 4*TM*TN FMAs in ascending k
    auto kgroup = [&](int kk) {
      float a[4][TM], b[4][TN];  // [k][row], [k][col]
      if (AK) {
#pragma unroll
        for (int r = 0; r < TM; ++r) {
          const float4 t = *reinterpret_cast<const float4*>(as + kidx(rowof(r), kk));
          a[0][r] = t.x; a[1][r] = t.y; a[2][r] = t.z; a[3][r] = t.w;
        }
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int h = 0; h < QM; ++h) {
            const float4 t = *reinterpret_cast<const float4*>(as + (kk + q) * MI + rowof(h * 4));
            a[q][h * 4 + 0] = t.x; a[q][h * 4 + 1] = t.y; a[q][h * 4 + 2] = t.z; a[q][h * 4 + 3] = t.w;
          }
      }
      if (!BNC) {
#pragma unroll
        for (int c = 0; c < TN; ++c) {
          const float4 t = *reinterpret_cast<const float4*>(bs + kidx(colof(c), kk));
          b[0][c] = t.x; b[1][c] = t.y; b[2][c] = t.z; b[3][c] = t.w;
        }
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int h = 0; h < QN; ++h) {
            const float4 t = *reinterpret_cast<const float4*>(bs + (kk + q) * NI + colof(h * 4));
            b[q][h * 4 + 0] = t.x; b[q][h * 4 + 1] = t.y; b[q][h * 4 + 2] = t.z; b[q][h * 4 + 3] = t.w;
          }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) fma_step(a[q], b[q]);
    };
    int kk = 0;
    if (k_left == KC) {
#pragma unroll
      for (int g4 = 0; g4 < KC; g4 += 4) kgroup(g4);   // full chunk: offsets are compile-time
      kk = KC;
    } else {
      for (; kk + 4 <= k_left; kk += 4) kgroup(kk);
    }
    for (; kk < k_left; ++kk) {  // K tail: exactly the remaining FMAs
      float a[TM], b[TN];
#pragma unroll
      for (int r = 0; r < TM; ++r) a[r] = AK ? as[kidx(rowof(r), kk)] : as[kk * MI + rowof(r)];
#pragma unroll
      for (int c = 0; c < TN; ++c) b[c] = !BNC ? bs[kidx(colof(c), kk)] : bs[kk * NI + colof(c)];
      fma_step(a, b);
    }

    if (kc == kchunks - 1) {
      // epilogue for this thread's instance, then reset the accumulators
      const int64_t z = gi * G + slot;
      if (z < p.batch) {
        Epi epi;
        epi.alpha = inst_alpha(p, z);
        epi.beta = inst_beta(p, z);
        epi.skip_ab = (epi.alpha == 0.0f) || (p.k == 0);
        const int64_t coff = inst_off(p.c_off, p.stride_c, p.c_offs, z);
        float* Cz = static_cast<float*>(p.c) + coff;
        const bool cal = ((coff & 3) == 0) && ((p.ldc & 3) == 0);
#pragma unroll
        for (int c = 0; c < TN; ++c) {
          const int col = colof(c);
          if (col >= n) continue;
#pragma unroll
          for (int h = 0; h < QM; ++h) {
            const int r0 = rowof(h * 4);
            float* cc = Cz + static_cast<int64_t>(col) * p.ldc + r0;
            if (cal && r0 + 3 < m) {
              float4 cv = make_float4(0.f, 0.f, 0.f, 0.f);
              if (epi.reads_c()) cv = *reinterpret_cast<const float4*>(cc);
              float4 o;
              o.x = epi.apply(acc_ref(h * 4 + 0, c), cv.x);
              o.y = epi.apply(acc_ref(h * 4 + 1, c), cv.y);
              o.z = epi.apply(acc_ref(h * 4 + 2, c), cv.z);
              o.w = epi.apply(acc_ref(h * 4 + 3, c), cv.w);
              *reinterpret_cast<float4*>(cc) = o;
            } else {
#pragma unroll
              for (int r = 0; r < 4; ++r) {
                if (r0 + r < m) {
                  const float cvs = epi.reads_c() ? cc[r] : 0.0f;
                  cc[r] = epi.apply(acc_ref(h * 4 + r, c), cvs);
                }
              }
            }
          }
        }
      }
#pragma unroll
      for (int i = 0; i < TM * TN / 2; ++i) acc2[i] = make_float2(0.0f, 0.0f);
    }
    advance(gi, kc);
  }
  cp_async_wait<0>();
}

}  // namespace tb
