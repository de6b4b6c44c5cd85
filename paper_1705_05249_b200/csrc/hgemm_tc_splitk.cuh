// hgemm_tc_splitk.cuh — FP16 GEMM with the K dimension split across the CTAs
// of a thread-block cluster, reduced through distributed shared memory.
//
// For problems with fewer 128x128 output tiles than SMs and a long K (BASELINE
// config C3 (4096, 128, 9216): 32 tiles, 144 K blocks) the single-CTA kernel
// leaves most SMs idle.  Here a cluster of KS CTAs (KS = 2..8 — the built-in
// route stops at 4, convgemm and configurations use 8 — a pure function
// of (m, n, k) and the SM count — never of the batch, so single, batched and
// looped calls of one shape stay bitwise consistent) shares each 128 x 128
// tile: CTA r accumulates K blocks r, r+KS, r+2KS, ... in its own TMEM (same producer / MMA pipeline and
// issue discipline as hgemm_tc_kernel, TMA or LDG producer), drains the FP32
// partial into a column-major shared buffer, and then reduces rows
// [r*128/KS, (r+1)*128/KS) of the tile over all KS buffers — read through
// DSMEM (mapa + ld.shared::cluster) in rank order 0..KS-1, so the sum is
// deterministic — applies the reference epilogue (Epi, one FP16 rounding) and
// stores 16-byte vectors.  No global workspace, no second kernel.
//
// Cluster-scope mbarriers order the exchange: red_full[r] completes when all
// KS x 256 epilogue threads have written their partials (release.cluster
// arrivals, acquire.cluster wait), red_empty[r] when all of them have finished
// reading, so a buffer is rewritten only after every reader is done.
//
// Exchange medium: with a workspace (ws != nullptr; one 64 KB slot per CTA,
// allocated per stream by the host, tbgemm.cu splitk_workspace) the
// partials go through L2 — TMEM -> registers -> st.global.cg, peers read
// with ld.global.cg after the cluster barrier.  DSMEM runs at ~20 B/cycle
// per SM (B300_MICROARCH "DSMEM BW", producer pays the smem port): reading
// 3 peers' 16 KB slices took 3.6 us of a 23 us C3 call (%globaltimer
// timeline, tools/splitk_timeline.py).  Without a workspace (a stream seen
// first under graph capture) the shared-memory buffer below is read
// through DSMEM instead; the sum order is the same, so results are too.
//
// The 64 KB partial buffer ALIASES the first ring stages: a tile's partial is
// written after its last MMA retired (every stage of this tile consumed),
// and the producer starts the loads of a CTA's next tile only after
// red_empty of the previous one (every peer finished reading), so the ring is
// 7 stages deep instead of 5 + a separate buffer — the single-tile CTAs of
// these shapes are load-latency bound, and bytes in flight per SM are what
// they run on.
#pragma once

#include "hgemm_tc.cuh"

namespace tb {

// Optional per-CTA timeline (build with -DTB_SPLITK_TIMING; tools/splitk_timeline.py):
// %globaltimer stamps of the kernel's phases in tb_sk_times[block * 16 + i].
#ifdef TB_SPLITK_TIMING
__device__ unsigned long long tb_sk_times[2048 * 16];
#define SK_STAMP(i)                                                              \
  do {                                                                           \
    unsigned long long _t;                                                       \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));                      \
    tb_sk_times[static_cast<size_t>(blockIdx.x) * 16 + (i)] = _t;                \
  } while (0)
#else
#define SK_STAMP(i) \
  do {              \
  } while (0)
#endif

constexpr int SK_BN = 128;
// Floats per column of the partial buffer.  Unpadded: the row-per-lane
// writes are conflict-free, the float4 reduction reads 2-way; the 4 KB saved
// buys a 5th pipeline stage (single-tile CTAs are load-latency bound).
constexpr int SK_RED_LD = HG_BM;
// Floats of one CTA's partial slot in the global split-K workspace.
constexpr int SK_WS_FLOATS = SK_BN * SK_RED_LD;

template <bool TMA>
struct SkCfg {
  static constexpr int STAGES = 7;
  static constexpr int A_BYTES = HG_BM * HG_BK * 2;   // 16 KB
  static constexpr int B_BYTES = SK_BN * HG_BK * 2;   // 16 KB
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = 2 * SK_BN;         // double-buffered accumulator
  static constexpr int EPI_WARPS = 8;
  static constexpr int PROD_WARPS = TMA ? 1 : 4;
  static constexpr int PROD_WARP0 = EPI_WARPS;
  static constexpr int MMA_WARP = EPI_WARPS + PROD_WARPS;
  static constexpr int THREADS = (MMA_WARP + 1) * 32;
  static constexpr int EPI_THREADS = EPI_WARPS * 32;
  static constexpr int BAR_BYTES = 1024;
  static constexpr int RED_BYTES = SK_BN * SK_RED_LD * 4;  // aliases ring stages (A region)
  static_assert(RED_BYTES <= STAGES * A_BYTES, "partial buffer inside the A ring");
  static constexpr int SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + BAR_BYTES;
  static_assert(SMEM_BYTES <= 232448, "fits the 227 KB opt-in shared memory");
};

__device__ __forceinline__ uint32_t sk_cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t sk_cluster_size() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void sk_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Address of the same shared-memory offset in cluster CTA `rank`.
__device__ __forceinline__ uint32_t sk_mapa(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ void sk_arrive_remote(uint32_t bar_cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster_addr) : "memory");
}
// One cluster-scope fence, then relaxed arrivals on every rank's barrier: a
// release arrive per rank compiled to a full MEMBAR.ALL.GPU each, and after
// the tile's global C stores those waited for the stores to drain (ncu /
// %globaltimer: 5.4 us of the reduction phase at C3).
__device__ __forceinline__ void sk_fence_cluster() { asm volatile("fence.acq_rel.cluster;" ::: "memory"); }
__device__ __forceinline__ void sk_arrive_remote_relaxed(uint32_t bar_cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster_addr) : "memory");
}
__device__ __forceinline__ void sk_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "SKW_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra SKW_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// DSMEM load.  volatile keeps it ordered after the cluster-barrier waits
// (volatile asm with "memory" clobbers); no clobber of its own, so a run of
// these loads issues back to back and their latencies overlap.
__device__ __forceinline__ float4 sk_ld_cluster_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr));
  return v;
}

// CONV: op(A) gathered from an image (implicit GEMM, hgemm_tc.cuh
// conv_fill_tile) in the LDG producer — convgemm's few-tile layers.
template <bool TMA, bool A_MN, bool B_MN, bool VEC, bool CONV = false>
__global__ void __launch_bounds__(SkCfg<TMA>::THREADS, 1)
    hgemm_tc_splitk_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                           Problem p, int tiles_m, int tiles_n, int group_m, int64_t total_tiles,
                           float* __restrict__ ws, const ConvGeom conv) {
  static_assert(!CONV || (!TMA && A_MN), "the im2col gather runs in the LDG producer, MN-major");
  using C = SkCfg<TMA>;
  constexpr int STAGES = C::STAGES, BN = SK_BN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_align1024(smem_raw);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* red_full = tempty + 2;
  uint64_t* red_empty = red_full + 1;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(red_empty + 1);
  float* red = reinterpret_cast<float*>(smem);  // aliases ring stages (see above)

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t ks = sk_cluster_size();
  const uint32_t rank = sk_cluster_rank();
  const int64_t cluster_id = blockIdx.x / ks;
  const int64_t n_clusters = gridDim.x / ks;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], TMA ? 1 : 128);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], C::EPI_THREADS);
    }
    mbar_init(red_full, ks * C::EPI_THREADS);
    mbar_init(red_empty, ks * C::EPI_THREADS);
    fence_mbar_init();
  }
  if (TMA && warp == C::PROD_WARP0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == C::MMA_WARP) tmem_alloc(tmem_holder, C::TMEM_COLS);
  tc_fence_before();
  if (threadIdx.x == 0) SK_STAMP(0);
  sk_cluster_sync();  // barriers of every CTA initialised before any remote arrive
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  grid_dep_wait();  // prologue above overlapped the previous kernel (PDL)
  grid_dep_launch();
  if (threadIdx.x == 0) SK_STAMP(1);

  const int nkb = static_cast<int>((p.k + HG_BK - 1) / HG_BK);
  // K blocks are dealt round-robin (rank r: kb = r, r+KS, ...): the KS CTAs
  // of a cluster then stream adjacent 128-byte segments of the same operand
  // rows at the same time.  (Contiguous K ranges per rank reached 35 % of HBM
  // at C3: every CTA's 128-byte row segments landed on distinct DRAM pages.)

  if (warp >= C::PROD_WARP0 && warp < C::MMA_WARP) {
    // ======================= producer (own K range) =======================
    int s = 0;
    uint32_t ph = 0;
    uint32_t tph = 0;  // parity of red_empty for the previous tile
    if (TMA) {
      for (int64_t t = cluster_id; t < total_tiles; t += n_clusters) {
        if (t != cluster_id) {  // the ring holds the previous tile's partial until every peer read it
          sk_wait_cluster(red_empty, tph);
          tph ^= 1;
        }
        int64_t z; int mt, nt;
        tile_coords(t, tiles_m, tiles_n, group_m, z, mt, nt);
        const int m0 = mt * HG_BM, n0 = nt * BN, zz = static_cast<int>(z);
        for (int kb = static_cast<int>(rank); kb < nkb; kb += static_cast<int>(ks)) {
          mbar_wait(&empty[s], ph ^ 1);
          if (elect_one()) {
            if (kb == static_cast<int>(rank) && t == cluster_id) SK_STAMP(2);
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
              tma_load_3d(b_dst, &tmB, &full[s], n0, k0, zz);
              tma_load_3d(b_dst + 8192, &tmB, &full[s], n0 + 64, k0, zz);
            }
          }
          __syncwarp();
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
      }
    } else {
      const int tid = threadIdx.x - C::PROD_WARP0 * 32;  // 0..127
      for (int64_t t = cluster_id; t < total_tiles; t += n_clusters) {
        if (t != cluster_id) {
          sk_wait_cluster(red_empty, tph);
          tph ^= 1;
        }
        int64_t z; int mt, nt;
        tile_coords(t, tiles_m, tiles_n, group_m, z, mt, nt);
        const int64_t m0 = static_cast<int64_t>(mt) * HG_BM, n0 = static_cast<int64_t>(nt) * BN;
        const __half* A = static_cast<const __half*>(p.a) + inst_off(p.a_off, p.stride_a, p.a_offs, z);
        const __half* B = static_cast<const __half*>(p.b) + inst_off(p.b_off, p.stride_b, p.b_offs, z);
        const int m_left = static_cast<int>(min64(HG_BM, p.m - m0));
        const int n_left = static_cast<int>(min64(BN, p.n - n0));
        int yb[16], xb[16];
        if (CONV) conv_tile_coords(conv, p.m, m0, tid, yb, xb);
        for (int kb = static_cast<int>(rank); kb < nkb; kb += static_cast<int>(ks)) {
          const int64_t k0 = static_cast<int64_t>(kb) * HG_BK;
          const int k_left = static_cast<int>(min64(HG_BK, p.k - k0));
          mbar_wait(&empty[s], ph ^ 1);
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
    // ======================= MMA issuer (own K range) =======================
    constexpr uint32_t idesc = umma_idesc_f16(HG_BM, BN, A_MN ? 1 : 0, B_MN ? 1 : 0);
    int s = 0;
    uint32_t ph = 0;
    int acc = 0;
    uint32_t aph = 0;
    for (int64_t t = cluster_id; t < total_tiles; t += n_clusters) {
      mbar_wait(&tempty[acc], aph ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
      for (int kb = static_cast<int>(rank); kb < nkb; kb += static_cast<int>(ks)) {
        mbar_wait(&full[s], ph);
        tc_fence_after();
        if (lane == 0 && t == cluster_id && kb == static_cast<int>(rank)) SK_STAMP(3);
        if (lane == 0 && t == cluster_id && kb + static_cast<int>(ks) >= nkb) SK_STAMP(4);
        const uint32_t a_addr = smem_u32(sA + s * C::A_BYTES);
        const uint32_t b_addr = smem_u32(sB + s * C::B_BYTES);
        const int ksteps = hg_ksteps(p.k, kb);
        if (elect_one()) {
          hg_issue_kblock<A_MN, B_MN>(Mma1Sm{}, d_tmem, a_addr, b_addr, idesc, ksteps, kb == static_cast<int>(rank));
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
    // ============ epilogue: partial -> shared, cluster reduction ============
    const int quad = warp & 3;
    const int half = warp >> 2;
    const int et = threadIdx.x;  // 0..255
    const int rp = HG_BM / static_cast<int>(ks);  // rows reduced by this CTA
    const int row_base = static_cast<int>(rank) * rp;
    const uint32_t red_s = smem_u32(red);
    const uint32_t rf_local = smem_u32(red_full), re_local = smem_u32(red_empty);
    // global-workspace exchange (ws != nullptr): this CTA's partial slot and
    // rank 0's slot of the cluster (slots are consecutive per cluster)
    float* ws_mine = ws ? ws + static_cast<size_t>(blockIdx.x) * SK_WS_FLOATS : nullptr;
    const float* ws_base = ws ? ws + static_cast<size_t>(blockIdx.x - rank) * SK_WS_FLOATS : nullptr;
    int acc = 0;
    uint32_t aph = 0, rph = 0;
    for (int64_t t = cluster_id; t < total_tiles; t += n_clusters) {
      int64_t z; int mt, nt;
      tile_coords(t, tiles_m, tiles_n, group_m, z, mt, nt);
      const int64_t m0 = static_cast<int64_t>(mt) * HG_BM, n0 = static_cast<int64_t>(nt) * BN;

      // (1) this CTA's partial: TMEM -> red (column-major, [col][row])
      sk_wait_cluster(red_empty, rph ^ 1);  // every reader of the previous tile is done
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      if (et == 0 && t == cluster_id) SK_STAMP(5);
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + static_cast<uint32_t>(acc * BN);
      const int row = quad * 32 + lane;
#pragma unroll 1
      for (int cb = half * 2; cb < half * 2 + 2; ++cb) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(t_row + cb * 32, v);
        tmem_ld_wait();
        if (ws_mine != nullptr) {
#pragma unroll
          for (int j = 0; j < 32; ++j) __stcg(ws_mine + (cb * 32 + j) * SK_RED_LD + row, __uint_as_float(v[j]));
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) red[(cb * 32 + j) * SK_RED_LD + row] = __uint_as_float(v[j]);
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);  // TMEM buffer free for the next tile's MMAs
      if (++acc == 2) { acc = 0; aph ^= 1; }
      sk_fence_cluster();  // the partial is visible cluster-wide before any arrival
      for (uint32_t q = 0; q < ks; ++q) sk_arrive_remote_relaxed(sk_mapa(rf_local, q));

      // (2) reduce rows [row_base, row_base + rp) over all ranks, in rank order
      sk_wait_cluster(red_full, rph);
      if (et == 0 && t == cluster_id) SK_STAMP(6);
      Epi epi;
      epi.alpha = inst_alpha(p, z);
      epi.beta = inst_beta(p, z);
      epi.skip_ab = (epi.alpha == 0.0f);
      __half* Cz = static_cast<__half*>(p.c) + inst_off(p.c_off, p.stride_c, p.c_offs, z);
      const int n_left = static_cast<int>(min64(BN, p.n - n0));
      const bool vec_ok = ((reinterpret_cast<uintptr_t>(Cz) & 15) == 0) && ((p.ldc & 7) == 0);
      const int groups = (rp / 8) * BN;  // (8-row group, column) items: <= 4 per thread (KS >= 2)
      constexpr int MAXIT = 4;
      float xs[MAXIT][8];
      // (2a) every rank's partial values first (up to 16 loads in flight per
      // item), summed in rank order 0..KS-1 (deterministic)
#pragma unroll
      for (int j = 0; j < MAXIT; ++j) {
        const int it = et + j * C::EPI_THREADS;
        if (it >= groups) break;
        const int col = it / (rp / 8);
        const int r0 = row_base + (it % (rp / 8)) * 8;
        const uint32_t off = red_s + static_cast<uint32_t>((col * SK_RED_LD + r0) * 4);
        float4 pv[8][2];
        if (ws_base != nullptr) {
          const float* src = ws_base + (col * SK_RED_LD + r0);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            if (q < static_cast<int>(ks)) {
              pv[q][0] = __ldcg(reinterpret_cast<const float4*>(src + q * SK_WS_FLOATS));
              pv[q][1] = __ldcg(reinterpret_cast<const float4*>(src + q * SK_WS_FLOATS + 4));
            }
          }
        } else {
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            if (q < static_cast<int>(ks)) {
              pv[q][0] = sk_ld_cluster_f4(sk_mapa(off, q));
              pv[q][1] = sk_ld_cluster_f4(sk_mapa(off + 16, q));
            }
          }
        }
        float* x = xs[j];
        x[0] = pv[0][0].x; x[1] = pv[0][0].y; x[2] = pv[0][0].z; x[3] = pv[0][0].w;
        x[4] = pv[0][1].x; x[5] = pv[0][1].y; x[6] = pv[0][1].z; x[7] = pv[0][1].w;
#pragma unroll
        for (int q = 1; q < 8; ++q) {
          if (q < static_cast<int>(ks)) {
            x[0] = __fadd_rn(x[0], pv[q][0].x); x[1] = __fadd_rn(x[1], pv[q][0].y);
            x[2] = __fadd_rn(x[2], pv[q][0].z); x[3] = __fadd_rn(x[3], pv[q][0].w);
            x[4] = __fadd_rn(x[4], pv[q][1].x); x[5] = __fadd_rn(x[5], pv[q][1].y);
            x[6] = __fadd_rn(x[6], pv[q][1].z); x[7] = __fadd_rn(x[7], pv[q][1].w);
          }
        }
      }
      if (et == 0 && t == cluster_id) SK_STAMP(9);
      // (2b) done reading every rank's partial of this tile: release the
      // buffers before the (slow to drain) global stores.  Not after the
      // last tile in workspace mode: nothing waits for it, no peer reads this
      // CTA's shared memory, and the kernel then ends without a cluster
      // barrier (the last remote operation aimed at this CTA, a red_full
      // arrival, has landed once its red_full wait returned).
      if (ws_base == nullptr || t + n_clusters < total_tiles) {
        sk_fence_cluster();
        for (uint32_t q = 0; q < ks; ++q) sk_arrive_remote_relaxed(sk_mapa(re_local, q));
      }
      if (et == 0 && t == cluster_id) SK_STAMP(10);
      // (2c) epilogue and 16-byte stores
#pragma unroll
      for (int j = 0; j < MAXIT; ++j) {
        const int it = et + j * C::EPI_THREADS;
        if (it >= groups) break;
        const int col = it / (rp / 8);
        const int r0 = row_base + (it % (rp / 8)) * 8;
        const float* x = xs[j];
        const int64_t grow = m0 + r0;
        if (col >= n_left || grow >= p.m) continue;
        __half* dst = Cz + (n0 + col) * p.ldc + grow;
        const int rows_valid = static_cast<int>(min64(8, p.m - grow));
        if (vec_ok && rows_valid == 8) {
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
          uint4 out;
          __half2* o2 = reinterpret_cast<__half2*>(&out);
#pragma unroll
          for (int i = 0; i < 4; ++i)
            o2[i] = __floats2half2_rn(epi.apply(x[2 * i], cv[2 * i]), epi.apply(x[2 * i + 1], cv[2 * i + 1]));
          *reinterpret_cast<uint4*>(dst) = out;
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) {  // fully unrolled: x stays in registers
            if (i < rows_valid) {
              const float cvs = epi.reads_c() ? __half2float(dst[i]) : 0.0f;
              dst[i] = __float2half_rn(epi.apply(x[i], cvs));
            }
          }
        }
      }
      if (et == 0 && t == cluster_id) SK_STAMP(7);
      rph ^= 1;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == C::MMA_WARP) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
  // DSMEM mode: no CTA leaves while a peer may still read its partials
  if (ws == nullptr) sk_cluster_sync();
  if (threadIdx.x == 0) SK_STAMP(8);
}

}  // namespace tb
