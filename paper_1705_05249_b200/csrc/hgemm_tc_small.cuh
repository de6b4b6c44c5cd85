// hgemm_tc_small.cuh — FP16 GEMM for small instances (m, n <= 64): the
// batched small-matrix path of BASELINE config C4 (16384 x 32^3 / 64^3).
//
// Replaces the reference's per-instance Python loop + one launch over all
// work-groups (pkg/src/tunedblas/routines/extras.py:188-286; gemm_direct_tasks
// compute.py:432-471) for small shapes.
//
// A 128-row UMMA tile is filled with P = 128/MI instances stacked along M
// (rows [z*MI, z*MI+m) hold instance z's A) and the B operands of the same
// P instances side by side along N (columns [z*NI, z*NI+n)): D = A'·B' holds
// instance z's product in the diagonal block (z*MI, z*NI).  The off-diagonal
// blocks are wasted tensor work (the tensor pipe has >100x headroom at these
// arithmetic intensities — the path is HBM-bound), in exchange for P
// instances per MMA / per epilogue / per pipeline stage.  Each output element
// still sees exactly the K sequence of the general kernel (64-deep K blocks of
// 4 x K16 steps, zero-filled tail) and tcgen05 results are independent of the
// tile's N extent and neighbours (tests: test_small_path_bitwise_equals_
// general_path), so small and general paths agree bitwise.
//
// Producer: 4 warps issue 16-byte cp.async (zero-fill for tails / missing
// instances) straight into the SWIZZLE_128B layout the UMMA descriptors
// expect, keeping DEPTH stages in flight per thread; completion is published
// with fence.proxy.async + mbarrier arrive.  Misaligned operands take the
// register path (8 x 2-byte loads per chunk).
#pragma once

#include "hgemm_tc.cuh"

namespace tb {

template <int MI, int NI>
struct HsCfg {
  static constexpr int P = 128 / MI;
  static constexpr int BN = P * NI;
  static_assert(BN % 16 == 0 && BN >= 16 && BN <= 256, "UMMA N");
  static constexpr int A_BYTES = 128 * HG_BK * 2;
  static constexpr int B_BYTES = BN * HG_BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (196608 / STAGE_BYTES) > 8 ? 8 : (196608 / STAGE_BYTES);  // <= 192 KB ring
  static constexpr int DEPTH = STAGES - 1;
  static constexpr int ACC = (BN <= 128) ? 4 : 2;
  // k <= 32: pair two tiles per stage (doubles the bytes in flight per ring slot)
  static constexpr bool PAIR = true;
  static constexpr int TMEM_COLS = (ACC * BN <= 256) ? 256 : 512;
  // warps 0-7 epilogue (TMEM quadrant w%4, warp group w/4 takes alternate tiles), 8-11 producer,
  // 12 TMEM allocation + MMA issue
  static constexpr int EPI_WARPS = 8, PROD_WARP0 = 8, MMA_WARP = 12;
  static constexpr int THREADS = 13 * 32;
  static constexpr int SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + 1024 + EPI_WARPS * EPI_WARP_FLOATS * 4;
};

// Fill one packed operand tile (ROWS = 128 for A', BN for B') of 64 K.
// ROWS are P = ROWS/SLOT instance slots of SLOT rows each; `extent` is the
// instance's m (A) or n (B); `inst[s]` points at instance slot s's operand
// (nullptr when the slot is past the end of the batch).
//   K-major : chunk j of thread t = row (t>>3) + 16j, K chunk t&7;
//   MN-major: chunk j of thread t = sub-tile j/4, K row (t>>3) + 16(j%4),
//             MN chunk t&7.
// K32 (k <= 32: the MMAs read K columns 0..31 only, see hg_ksteps): K-major
// threads cover 4 chunks of a row, row (t>>2) + 32j, K chunk t&3; MN-major
// skips the K rows >= 32.  Either way every chunk's slot and smem offset is a
// compile-time function of j plus a per-thread constant, so the loop body is
// a handful of integer ops and one cp.async, with no divergence.
// inst[idx] for a lane-dependent idx without dynamic indexing (which would
// put the 4 pointers in local memory and add a local load per chunk).
__device__ __forceinline__ const __half* pick4(const __half* const (&inst)[4], int idx) {
  const __half* r = inst[0];
  r = idx == 1 ? inst[1] : r;
  r = idx == 2 ? inst[2] : r;
  r = idx == 3 ? inst[3] : r;
  return r;
}

template <int ROWS, int SLOT, bool MN, bool VEC, bool K32>
__device__ __forceinline__ void small_fill(uint8_t* smem, const __half* const (&inst)[4], const __half* any,
                                           int64_t ld, int extent, int64_t k0, int k_left, int tid) {
  constexpr bool KM32 = K32 && !MN;
  constexpr int PER_T = KM32 ? ROWS / 32 : ROWS * 8 / 128;
  const int q = KM32 ? (tid >> 2) : (tid >> 3);  // 0..31 / 0..15
  const int c = KM32 ? (tid & 3) : (tid & 7);    // 16-byte chunk within a 128-byte row
  const uint32_t off0 = static_cast<uint32_t>((q >> 3) * 1024 + (q & 7) * 128 + ((c ^ (q & 7)) << 4));
#pragma unroll
  for (int j = 0; j < PER_T; ++j) {
    if (K32 && MN && (j & 3) >= 2) continue;  // K rows 32..63: never read
    int slot, idx, valid;
    int64_t eoff;
    uint32_t off;
    if (!MN) {
      constexpr int RSTEP = KM32 ? 32 : 16;
      slot = (RSTEP * j) / SLOT;
      idx = q + (RSTEP * j) % SLOT;
      valid = (idx < extent) ? min(8, k_left - c * 8) : 0;
      eoff = static_cast<int64_t>(idx) * ld + k0 + c * 8;
      off = off0 + j * (RSTEP * 128);
    } else {
      const int sub = j >> 2;
      const int mn = sub * 64 + c * 8;
      slot = mn / SLOT;
      idx = mn % SLOT;
      const int r = q + 16 * (j & 3);
      valid = (r < k_left) ? min(8, extent - idx) : 0;
      eoff = (k0 + r) * ld + idx;
      off = off0 + sub * 8192 + (j & 3) * 2048;
    }
    const __half* base = pick4(inst, slot);
    if (base == nullptr || valid < 0) valid = 0;
    const __half* src = valid > 0 ? base + eoff : any;
    if (VEC) {
      cp_async_16(smem + off, src, static_cast<uint32_t>(valid) * 2u);
    } else {
      const uint4 v = (valid > 0) ? ldg_chunk8<false>(src, valid) : make_uint4(0, 0, 0, 0);
      *reinterpret_cast<uint4*>(smem + off) = v;
    }
  }
}

// Single-K-block fills (k <= 64, every C4 case): each thread's chunk source
// offsets, byte counts and smem offsets do not depend on the tile, only the
// instance base pointers do — precompute them once per thread.
template <int ROWS, int SLOT, bool MN, bool K32>
struct SmallFillPlan {
  static constexpr bool KM32 = K32 && !MN;
  static constexpr int PER_T = KM32 ? ROWS / 32 : ROWS * 8 / 128;
  int64_t eoff[PER_T];
  uint32_t bytes[PER_T];
  uint32_t off[PER_T];
  __device__ __forceinline__ void init(int64_t ld, int extent, int k_left, int tid) {
    const int q = KM32 ? (tid >> 2) : (tid >> 3);
    const int c = KM32 ? (tid & 3) : (tid & 7);
    const uint32_t off0 = static_cast<uint32_t>((q >> 3) * 1024 + (q & 7) * 128 + ((c ^ (q & 7)) << 4));
#pragma unroll
    for (int j = 0; j < PER_T; ++j) {
      int valid;
      if (!MN) {
        constexpr int RSTEP = KM32 ? 32 : 16;
        const int idx = q + (RSTEP * j) % SLOT;
        valid = (idx < extent) ? min(8, k_left - c * 8) : 0;
        eoff[j] = static_cast<int64_t>(idx) * ld + c * 8;
        off[j] = off0 + j * (RSTEP * 128);
      } else {
        const int sub = j >> 2, mn = sub * 64 + c * 8, idx = mn % SLOT, r = q + 16 * (j & 3);
        valid = (r < k_left) ? min(8, extent - idx) : 0;
        eoff[j] = static_cast<int64_t>(r) * ld + idx;
        off[j] = off0 + sub * 8192 + (j & 3) * 2048;
      }
      bytes[j] = valid > 0 ? static_cast<uint32_t>(valid) * 2u : 0u;
    }
  }
  // HI (K32 only): place the chunks in K columns 32..63 of the stage instead
  // (the second tile of a paired stage): chunk c -> c ^ 4 inside the 128-byte
  // K-major row, or the next two 8-row K atoms of an MN-major sub-tile.
  template <bool HI = false>
  __device__ __forceinline__ void issue(uint8_t* smem, const __half* const (&inst)[4], const __half* any) const {
    static_assert(!HI || K32, "hi half is only free when k <= 32");
#pragma unroll
    for (int j = 0; j < PER_T; ++j) {
      if (K32 && MN && (j & 3) >= 2) continue;  // K rows 32..63: never read
      constexpr int RSTEP = KM32 ? 32 : 16;
      const int slot = !MN ? (RSTEP * j) / SLOT : ((j >> 2) * 64 + 0) / SLOT + 0;
      // MN-major: the 8 chunks of a 64-wide sub-tile may straddle two slots
      // when SLOT = 32; the slot is then a per-lane value (c*8 / SLOT).
      const __half* base;
      if (!MN || SLOT >= 64) {
        base = inst[slot];
      } else {
        const int c = threadIdx.x & 7;
        base = pick4(inst, ((j >> 2) * 64 + c * 8) / SLOT);
      }
      uint32_t nb = bytes[j];
      if (base == nullptr) nb = 0;
      const uint32_t o = HI ? (MN ? off[j] + 4096u : (off[j] ^ 64u)) : off[j];
      cp_async_16(smem + o, nb ? base + eoff[j] : any, nb);
    }
  }
};

template <int MI, int NI, bool A_MN, bool B_MN, bool VEC, bool K32>
__global__ void __launch_bounds__(HsCfg<MI, NI>::THREADS, 1)
    hgemm_tc_small_kernel(Problem p, int64_t total_tiles) {
  using C = HsCfg<MI, NI>;
  constexpr int STAGES = C::STAGES, P = C::P, BN = C::BN, ACC = C::ACC;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_align1024(smem_raw);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + ACC;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + ACC);
  float* epi_stage = reinterpret_cast<float*>(smem + STAGES * C::STAGE_BYTES + 1024);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 128);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < ACC; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 32 * 4);  // one warp group per tile
    }
    fence_mbar_init();
  }
  if (warp == C::MMA_WARP) tmem_alloc(tmem_holder, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  grid_dep_wait();  // prologue above overlapped the previous kernel (PDL)
  grid_dep_launch();
  const int nkb = static_cast<int>((p.k + HG_BK - 1) / HG_BK);
  const int m = static_cast<int>(p.m), n = static_cast<int>(p.n);

  if (warp >= C::PROD_WARP0 && warp < C::MMA_WARP) {
    // ===================== producer (cp.async ring) =====================
    const int tid = threadIdx.x - C::PROD_WARP0 * 32;
    const __half* A = static_cast<const __half*>(p.a);
    const __half* B = static_cast<const __half*>(p.b);
    int s = 0;
    uint32_t ph = 0;
    int lag = 0;  // stages committed but not yet published (<= DEPTH - 1)
    int s_pub = 0;
    const bool one_block = VEC && nkb == 1;
    SmallFillPlan<128, MI, A_MN, K32> plan_a;
    SmallFillPlan<BN, NI, B_MN, K32> plan_b;
    if (one_block) {
      const int k_left = static_cast<int>(p.k);
      plan_a.init(p.lda, m, k_left, tid);
      plan_b.init(p.ldb, n, k_left, tid);
    }
    // K32: two tiles per stage (t in K columns 0..31, t + gridDim.x in 32..63)
    constexpr bool PAIR = C::PAIR && K32 && VEC;
    const int64_t tstep = PAIR ? 2 * static_cast<int64_t>(gridDim.x) : gridDim.x;
    for (int64_t t = blockIdx.x; t < total_tiles; t += tstep) {
      const int64_t zbase = t * P;
      const __half* ia[4];
      const __half* ib[4];
      const __half* ja[4];
      const __half* jb[4];
      if constexpr (PAIR) {
        const int64_t z1 = (t + gridDim.x) * P;
#pragma unroll
        for (int sl = 0; sl < 4; ++sl) {
          const int64_t zi = z1 + sl;
          const bool ok = sl < P && zi < p.batch;
          ja[sl] = ok ? A + inst_off(p.a_off, p.stride_a, p.a_offs, zi) : nullptr;
          jb[sl] = ok ? B + inst_off(p.b_off, p.stride_b, p.b_offs, zi) : nullptr;
        }
      }
#pragma unroll
      for (int sl = 0; sl < 4; ++sl) {
        const int64_t zi = zbase + sl;
        const bool ok = sl < P && zi < p.batch;
        ia[sl] = ok ? A + inst_off(p.a_off, p.stride_a, p.a_offs, zi) : nullptr;
        ib[sl] = ok ? B + inst_off(p.b_off, p.stride_b, p.b_offs, zi) : nullptr;
      }
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&empty[s], ph ^ 1);
        const int64_t k0 = static_cast<int64_t>(kb) * HG_BK;
        const int k_left = static_cast<int>(min64(HG_BK, p.k - k0));
        if constexpr (PAIR) {
          plan_a.issue(sA + s * C::A_BYTES, ia, A);
          plan_b.issue(sB + s * C::B_BYTES, ib, B);
          plan_a.template issue<true>(sA + s * C::A_BYTES, ja, A);
          plan_b.template issue<true>(sB + s * C::B_BYTES, jb, B);
        } else if (one_block) {
          plan_a.issue(sA + s * C::A_BYTES, ia, A);
          plan_b.issue(sB + s * C::B_BYTES, ib, B);
        } else {
          small_fill<128, MI, A_MN, VEC, K32>(sA + s * C::A_BYTES, ia, A, p.lda, m, k0, k_left, tid);
          small_fill<BN, NI, B_MN, VEC, K32>(sB + s * C::B_BYTES, ib, B, p.ldb, n, k0, k_left, tid);
        }
        if (VEC) {
          cp_async_commit();
          if (lag == C::DEPTH - 1) {
            cp_async_wait<C::DEPTH - 1>();
            fence_proxy_async_smem();
            mbar_arrive(&full[s_pub]);
            if (++s_pub == STAGES) s_pub = 0;
          } else {
            ++lag;
          }
        } else {
          fence_proxy_async_smem();
          mbar_arrive(&full[s]);
        }
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
    }
    if (VEC) {
      cp_async_wait<0>();
      fence_proxy_async_smem();
      for (; lag > 0; --lag) {
        mbar_arrive(&full[s_pub]);
        if (++s_pub == STAGES) s_pub = 0;
      }
    }
  } else if (warp == C::MMA_WARP) {
    // ===================== MMA issuer =====================
    // The whole warp runs the loop (uniform operands); one elected lane issues.
    constexpr uint32_t idesc = umma_idesc_f16(128, BN, A_MN ? 1 : 0, B_MN ? 1 : 0);
    int s = 0, acc = 0;
    uint32_t ph = 0, aph = 0;
    if constexpr (C::PAIR && K32 && VEC) {
      // one stage = two tiles; the second one's K16 steps start 2 steps in
      // (the descriptors of steps 2, 3 of a full block: same MMA sequence)
      const int ksteps = hg_ksteps(p.k, 0);
      constexpr uint32_t A_HI = A_MN ? 4096u : 64u, B_HI = B_MN ? 4096u : 64u;
      for (int64_t t = blockIdx.x; t < total_tiles; t += 2 * static_cast<int64_t>(gridDim.x)) {
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint32_t a_addr = smem_u32(sA + s * C::A_BYTES);
        const uint32_t b_addr = smem_u32(sB + s * C::B_BYTES);
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
          if (t + h * static_cast<int64_t>(gridDim.x) >= total_tiles) break;
          mbar_wait(&tempty[acc], aph ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
          if (elect_one()) {
            hg_issue_kblock<A_MN, B_MN>(Mma1Sm{}, d_tmem, a_addr + h * A_HI, b_addr + h * B_HI, idesc, ksteps, true);
            tc_commit(&tfull[acc]);
          }
          __syncwarp();
          if (++acc == ACC) { acc = 0; aph ^= 1; }
        }
        if (elect_one()) tc_commit(&empty[s]);
        __syncwarp();
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
    } else
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
      if (++acc == ACC) { acc = 0; aph ^= 1; }
    }
  } else if (warp < C::EPI_WARPS) {
    // ===================== epilogue =====================
    // Warp group g = warp / 4 takes every other tile (tile sequence index
    // i = 2j + g of this CTA), each warp the full NI columns of its TMEM lane
    // quadrant: two tiles drain concurrently (one tile at a time was the
    // per-tile latency floor of the batched small path).
    const int quad = warp & 3;
    const int grp = warp >> 2;
    const int slot = (quad * 32) / MI;
    int64_t seq = grp;
    for (int64_t t = blockIdx.x + static_cast<int64_t>(grp) * gridDim.x; t < total_tiles;
         t += 2 * static_cast<int64_t>(gridDim.x), seq += 2) {
      const int acc = static_cast<int>(seq % ACC);
      const uint32_t aph = static_cast<uint32_t>((seq / ACC) & 1);
      const int64_t zi = t * P + slot;
      const bool inst_ok = zi < p.batch;
      Epi epi;
      epi.alpha = inst_ok ? inst_alpha(p, zi) : 0.0f;
      epi.beta = inst_ok ? inst_beta(p, zi) : 0.0f;
      epi.skip_ab = (epi.alpha == 0.0f);
      __half* Cz = static_cast<__half*>(p.c) + (inst_ok ? inst_off(p.c_off, p.stride_c, p.c_offs, zi) : 0);
      const int row0 = quad * 32 - slot * MI;           // first instance row of this warp
      const int rows_valid = inst_ok ? min(32, m - row0) : 0;
      float* stage = epi_stage + warp * EPI_WARP_FLOATS;  // one buffer per epilogue warp
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) +
                             static_cast<uint32_t>(acc * BN + slot * NI);
#pragma unroll
      for (int h = 0; h < NI / 32; ++h) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(t_row + h * 32, v);
        tmem_ld_wait();
        if (rows_valid > 0 && h * 32 < n)
          epi_store_block<32>(stage, v, Cz + static_cast<int64_t>(h * 32) * p.ldc + row0, p.ldc, rows_valid,
                              n - h * 32, epi, lane);
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == C::MMA_WARP) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

// ---------------------------------------------------------------------------
// TMA-fed variant for the 32 x 32 x (k <= 32) instances of C4 (arithmetic
// batch, 16-byte aligned rows and strides).  One 3-D TMA box {32, 32, 4}
// over (contiguous dim, other dim, batch) per operand per tile lands four
// instances as [instance][row][64 B] with SWIZZLE_64B — exactly the UMMA
// SWIZZLE_64B canonical layouts:
//   K-major  (rows = M or N index, 32 K per 64-byte row): 8-row atoms,
//            SBO = 512 B; a K16 step advances the start by 32 B;
//   MN-major (rows = K index, 32 M/N per 64-byte row): instance s is MN
//            chunk s (LBO = 2048 B), 8-row K groups SBO = 512 B; a K16 step
//            advances 16 rows = 1024 B.
// So four instances stack along M of the 128-row tile and side by side
// along N (BN = 128) as in hgemm_tc_small_kernel, with no per-thread
// address arithmetic: one elected lane issues 2 TMA loads per tile into a
// 12-deep ring of 16 KB stages (vs 32 KB cp.async stages filled by 128
// threads).  Same K16 MMA sequence per element (hg_ksteps), same epilogue:
// bitwise equal to every other H path.
struct Hs32Cfg {
  static constexpr int P = 4, MI = 32, NI = 32, BN = 128;
  static constexpr int A_BYTES = 128 * 32 * 2, B_BYTES = BN * 32 * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;  // 16 KB
  static constexpr int STAGES = 12;
  static constexpr int ACC = 4;
  static constexpr int TMEM_COLS = 512;
  static constexpr int EPI_WARPS = 8, PROD_WARP = 8, MMA_WARP = 9;
  static constexpr int THREADS = 10 * 32;
  static constexpr int SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + 1024 + EPI_WARPS * EPI_WARP_FLOATS * 4;
};

template <bool A_MN, bool B_MN>
__global__ void __launch_bounds__(Hs32Cfg::THREADS, 1)
    hgemm_tc_small32_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                                Problem p, int64_t total_tiles) {
  using C = Hs32Cfg;
  constexpr int STAGES = C::STAGES, P = C::P, BN = C::BN, ACC = C::ACC, MI = C::MI, NI = C::NI;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_align1024(smem_raw);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + ACC;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + ACC);
  float* epi_stage = reinterpret_cast<float*>(smem + STAGES * C::STAGE_BYTES + 1024);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < ACC; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 32 * 4);  // one warp group per tile
    }
    fence_mbar_init();
  }
  if (warp == C::PROD_WARP && lane == 0) {
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
  const int m = static_cast<int>(p.m), n = static_cast<int>(p.n);

  if (warp == C::PROD_WARP) {
    // ===================== producer: 2 TMA boxes per tile =====================
    int s = 0;
    uint32_t ph = 0;
    for (int64_t t = blockIdx.x; t < total_tiles; t += gridDim.x) {
      mbar_wait(&empty[s], ph ^ 1);
      if (elect_one()) {
        mbar_arrive_expect_tx(&full[s], C::STAGE_BYTES);
        const int z0 = static_cast<int>(t * P);
        tma_load_3d(sA + s * C::A_BYTES, &tmA, &full[s], 0, 0, z0);
        tma_load_3d(sB + s * C::B_BYTES, &tmB, &full[s], 0, 0, z0);
      }
      __syncwarp();
      if (++s == STAGES) { s = 0; ph ^= 1; }
    }
  } else if (warp == C::MMA_WARP) {
    // ===================== MMA issuer =====================
    constexpr uint32_t idesc = umma_idesc_f16(128, BN, A_MN ? 1 : 0, B_MN ? 1 : 0);
    const int ksteps = hg_ksteps(p.k, 0);
    int s = 0, acc = 0;
    uint32_t ph = 0, aph = 0;
    for (int64_t t = blockIdx.x; t < total_tiles; t += gridDim.x) {
      mbar_wait(&tempty[acc], aph ^ 1);
      mbar_wait(&full[s], ph);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
      const uint32_t a_addr = smem_u32(sA + s * C::A_BYTES);
      const uint32_t b_addr = smem_u32(sB + s * C::B_BYTES);
      if (elect_one()) {
#pragma unroll 1
        for (int kk = 0; kk < ksteps; ++kk) {
          const uint64_t ad = A_MN ? umma_desc_sw64(a_addr + kk * 1024, 2048, 512)
                                   : umma_desc_sw64(a_addr + kk * 32, 16, 512);
          const uint64_t bd = B_MN ? umma_desc_sw64(b_addr + kk * 1024, 2048, 512)
                                   : umma_desc_sw64(b_addr + kk * 32, 16, 512);
          tc_mma_f16(d_tmem, ad, bd, idesc, kk != 0 ? 1u : 0u);
        }
        tc_commit(&empty[s]);
        tc_commit(&tfull[acc]);
      }
      __syncwarp();
      if (++s == STAGES) { s = 0; ph ^= 1; }
      if (++acc == ACC) { acc = 0; aph ^= 1; }
    }
  } else if (warp < C::EPI_WARPS) {
    // ===================== epilogue (as hgemm_tc_small_kernel) =====================
    const int quad = warp & 3;
    const int grp = warp >> 2;
    const int slot = (quad * 32) / MI;
    int64_t seq = grp;
    for (int64_t t = blockIdx.x + static_cast<int64_t>(grp) * gridDim.x; t < total_tiles;
         t += 2 * static_cast<int64_t>(gridDim.x), seq += 2) {
      const int acc = static_cast<int>(seq % ACC);
      const uint32_t aph = static_cast<uint32_t>((seq / ACC) & 1);
      const int64_t zi = t * P + slot;
      const bool inst_ok = zi < p.batch;
      Epi epi;
      epi.alpha = inst_ok ? inst_alpha(p, zi) : 0.0f;
      epi.beta = inst_ok ? inst_beta(p, zi) : 0.0f;
      epi.skip_ab = (epi.alpha == 0.0f);
      __half* Cz = static_cast<__half*>(p.c) + (inst_ok ? inst_off(p.c_off, p.stride_c, p.c_offs, zi) : 0);
      const int row0 = quad * 32 - slot * MI;
      const int rows_valid = inst_ok ? min(32, m - row0) : 0;
      float* stage = epi_stage + warp * EPI_WARP_FLOATS;
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) +
                             static_cast<uint32_t>(acc * BN + slot * NI);
      uint32_t v[32];
      tmem_ld_32x32b_x32(t_row, v);
      tmem_ld_wait();
      if (rows_valid > 0)
        epi_store_block<32>(stage, v, Cz + row0, p.ldc, rows_valid, n, epi, lane);
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == C::MMA_WARP) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

// ---- 64-wide instances through TMA -----------------------------------------
// m, n, k <= 64 over a strided batch: P = 2 instances per 128 x 128 UMMA tile
// (instance 0 in rows / columns 0-63, instance 1 in 64-127; the product's
// diagonal blocks are the results), each operand ONE 3-D TMA box {64, 64, 2}
// per tile — a 64-element row is exactly one 128-byte SWIZZLE_128B row, so
// the tiles are the ordinary 128-row SW128 layouts (K-major: 8-row atoms,
// MN-major: two 64-element chunks 8 KB apart) and hg_issue_kblock issues
// them.  Replaces 128 producer threads of cp.async (5-7 stages) with one
// elected thread and a 6-stage ring of 32 KB.  Same K16 sequence per element
// as every other H kernel: bitwise equal.
struct Hs64Cfg {
  static constexpr int P = 2, MI = 64, NI = 64, BN = 128;
  static constexpr int A_BYTES = 128 * 64 * 2, B_BYTES = BN * 64 * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;  // 32 KB
  static constexpr int STAGES = 6;
  static constexpr int ACC = 4;
  static constexpr int TMEM_COLS = 512;
  static constexpr int EPI_WARPS = 8, PROD_WARP = 8, MMA_WARP = 9;
  static constexpr int THREADS = 10 * 32;
  static constexpr int SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + 1024 + EPI_WARPS * EPI_WARP_FLOATS * 4;
  static_assert(SMEM_BYTES <= 232448, "fits the 227 KB opt-in shared memory");
};

template <bool A_MN, bool B_MN>
__global__ void __launch_bounds__(Hs64Cfg::THREADS, 1)
    hgemm_tc_small64_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                                Problem p, int64_t total_tiles) {
  using C = Hs64Cfg;
  constexpr int STAGES = C::STAGES, P = C::P, BN = C::BN, ACC = C::ACC, MI = C::MI, NI = C::NI;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_align1024(smem_raw);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + ACC;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + ACC);
  float* epi_stage = reinterpret_cast<float*>(smem + STAGES * C::STAGE_BYTES + 1024);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < ACC; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 32 * C::EPI_WARPS);  // all 8 epilogue warps per tile
    }
    fence_mbar_init();
  }
  if (warp == C::PROD_WARP && lane == 0) {
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
  const int m = static_cast<int>(p.m), n = static_cast<int>(p.n);

  if (warp == C::PROD_WARP) {
    // ===================== producer: 2 TMA boxes per tile =====================
    int s = 0;
    uint32_t ph = 0;
    for (int64_t t = blockIdx.x; t < total_tiles; t += gridDim.x) {
      mbar_wait(&empty[s], ph ^ 1);
      if (elect_one()) {
        mbar_arrive_expect_tx(&full[s], C::STAGE_BYTES);
        const int z0 = static_cast<int>(t * P);
        tma_load_3d(sA + s * C::A_BYTES, &tmA, &full[s], 0, 0, z0);
        tma_load_3d(sB + s * C::B_BYTES, &tmB, &full[s], 0, 0, z0);
      }
      __syncwarp();
      if (++s == STAGES) { s = 0; ph ^= 1; }
    }
  } else if (warp == C::MMA_WARP) {
    // ===================== MMA issuer =====================
    constexpr uint32_t idesc = umma_idesc_f16(128, BN, A_MN ? 1 : 0, B_MN ? 1 : 0);
    const int ksteps = hg_ksteps(p.k, 0);
    int s = 0, acc = 0;
    uint32_t ph = 0, aph = 0;
    for (int64_t t = blockIdx.x; t < total_tiles; t += gridDim.x) {
      mbar_wait(&tempty[acc], aph ^ 1);
      mbar_wait(&full[s], ph);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
      const uint32_t a_addr = smem_u32(sA + s * C::A_BYTES);
      const uint32_t b_addr = smem_u32(sB + s * C::B_BYTES);
      if (elect_one()) {
        hg_issue_kblock<A_MN, B_MN>(Mma1Sm{}, d_tmem, a_addr, b_addr, idesc, ksteps, true);
        tc_commit(&empty[s]);
        tc_commit(&tfull[acc]);
      }
      __syncwarp();
      if (++s == STAGES) { s = 0; ph ^= 1; }
      if (++acc == ACC) { acc = 0; aph ^= 1; }
    }
  } else if (warp < C::EPI_WARPS) {
    // ===== epilogue: warp w -> TMEM lanes of quadrant w%4 (instance (w%4)/2), columns half w/4 =====
    const int quad = warp & 3;
    const int half = warp >> 2;
    const int slot = (quad * 32) / MI;
    int acc = 0;
    uint32_t aph = 0;
    float* stage = epi_stage + warp * EPI_WARP_FLOATS;
    for (int64_t t = blockIdx.x; t < total_tiles; t += gridDim.x) {
      const int64_t zi = t * P + slot;
      const bool inst_ok = zi < p.batch;
      Epi epi;
      epi.alpha = inst_ok ? inst_alpha(p, zi) : 0.0f;
      epi.beta = inst_ok ? inst_beta(p, zi) : 0.0f;
      epi.skip_ab = (epi.alpha == 0.0f);
      __half* Cz = static_cast<__half*>(p.c) + (inst_ok ? inst_off(p.c_off, p.stride_c, p.c_offs, zi) : 0);
      const int row0 = quad * 32 - slot * MI;
      const int rows_valid = inst_ok ? min(32, m - row0) : 0;
      const int cols_valid = n - half * 32;
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) +
                             static_cast<uint32_t>(acc * BN + slot * NI + half * 32);
      uint32_t v[32];
      tmem_ld_32x32b_x32(t_row, v);
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(&tempty[acc]);  // accumulator drained (values in registers)
      if (++acc == ACC) { acc = 0; aph ^= 1; }
      if (rows_valid > 0 && cols_valid > 0)
        epi_store_block<32>(stage, v, Cz + static_cast<int64_t>(half * 32) * p.ldc + row0, p.ldc, rows_valid,
                            cols_valid, epi, lane);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == C::MMA_WARP) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

}  // namespace tb
