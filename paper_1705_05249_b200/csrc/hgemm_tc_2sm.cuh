// hgemm_tc_2sm.cuh — FP16 GEMM on CTA pairs: tcgen05.mma.cta_group::2.
//
// Same contract as hgemm_tc_kernel (hgemm_tc.cuh) for large, 16-byte aligned
// problems, re-tiled for the Blackwell 2-SM UMMA: a cluster of two CTAs on
// one TPC computes a 256 x 256 output tile.  CTA r (r = cluster rank) loads
// A rows [m0 + 128 r, +128) and B columns [n0 + 128 r, +128) — half of each
// operand — and the leader's single MMA thread issues
//   tcgen05.mma.cta_group::2.kind::f16  (M = 256, N = 256, K = 16)
// which makes each SM multiply its own A half by BOTH B halves (the pair
// exchanges B internally).  Per FLOP this is 1/3 less shared-memory fill and
// L2 traffic than the 128 x 256 single-CTA tile, which under the 1 kW power
// cap buys clock.
//
// Synchronisation across the pair:
//   * both CTAs' TMA loads complete_tx on the LEADER's full[s] barrier
//     (.cta_group::2 TMA with the peer bit masked off the mbarrier address);
//     the leader's producer posts expect_tx for both halves;
//   * the leader's tcgen05.commit multicasts to empty[s] / tfull[a] in both
//     CTAs (cta mask 0b11);
//   * both CTAs' epilogue threads arrive on the leader's tempty[a]
//     (mapa + mbarrier.arrive.shared::cluster).
// Each CTA's TMEM holds its 128 rows x 256 FP32 columns (double-buffered);
// its 8 epilogue warps store them exactly as the single-CTA kernel does.
#pragma once

#include "hgemm_tc.cuh"

namespace tb {

constexpr int H2_BN = 256;          // pair tile N (per-CTA B half = 128)

// BNP: pair tile N.  256: one UMMA (N = 256) per K16 step, double-buffered
// accumulators (2 x 256 TMEM columns), 6-stage ring.  512: two UMMAs per K16
// step into TMEM columns [0, 256) and [256, 512) (each CTA holds B columns
// n0 + 128 r + {0, 256}, 128 each), one accumulator (the whole TMEM, so the
// epilogue is not overlapped with the next tile's MMAs), 4-stage ring of
// 48 KB: 1/4 less operand traffic per FLOP (L2 -> SM and shared-memory fill).
template <int BNP = 256>
struct H2Cfg {
  static constexpr int STAGES = BNP == 512 ? 4 : 6;
  static constexpr int ACC = BNP == 512 ? 1 : 2;              // accumulator buffers
  static constexpr int A_BYTES = 128 * HG_BK * 2;            // 16 KB: own 128 A rows
  static constexpr int B_BYTES = (BNP / 2) * HG_BK * 2;      // 16 / 32 KB: own B columns
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int EPI_WARPS = 8, PROD_WARP = 8, MMA_WARP = 9;
  static constexpr int THREADS = 10 * 32;
  static constexpr int TMEM_COLS = 512;
  static constexpr int BAR_BYTES = 1024;
  static constexpr int EPI_BYTES = EPI_WARPS * EPI_WARP_FLOATS * 4;
  static constexpr int SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + BAR_BYTES + EPI_BYTES;
  static_assert(SMEM_BYTES <= 232448, "fits the 227 KB opt-in shared memory");
};

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// 2-SM TMA: data lands in this CTA's smem, transaction bytes go to the
// leader CTA's barrier at the same offset.
__device__ __forceinline__ void tma_load_3d_2sm(void* smem_dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1,
                                                int c2) {
  const uint32_t bar_leader = smem_u32(bar) & 0xFEFFFFFFu;
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(bar_leader), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tc2_mma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
struct Mma2Sm {
  __device__ __forceinline__ void operator()(uint32_t d, uint64_t a, uint64_t b, uint32_t i, uint32_t acc) const {
    tc2_mma_f16(d, a, b, i, acc);
  }
};
__device__ __forceinline__ void tc2_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t* bar, uint32_t cta) {
  asm volatile(
      "{\n\t.reg .b32 rem;\n\t"
      "mapa.shared::cluster.u32 rem, %0, %1;\n\t"
      "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [rem];\n\t}" ::"r"(smem_u32(bar)),
      "r"(cta)
      : "memory");
}

// Wave barrier for very long K (wave_ctr != nullptr): the producer of every
// CTA waits before loading its w-th tile until all CTAs have issued the loads
// of their (w-1)-th, and counts each tile it finishes issuing.  Without it the
// persistent clusters drift apart in k over hundreds of tiles, the A/B panel
// slices a wave shares are no longer read close together in time, and at
// K = 32768 (16 MB panels, ~18 panels per wave) L2 reuse collapses (ncu: 329 GB
// DRAM per 32768^3 call; the barrier measured 945 -> 1286 TFLOP/s there).
// The barrier is advisory: the target never exceeds the tiles every CTA will
// finish (ragged last wave), and the first wait that exceeds the launch's
// timeout (%globaltimer; 2 ms above 6 TFLOP, ~2 tiles' time below, set by
// launch_h2) — CTAs not co-resident because other work holds SMs —
// raises an abandon flag (ctr[1]) that turns the barrier off for every CTA
// for the rest of the launch, so a shared GPU costs at most one timeout per
// call, never one per wave.  The launcher also sizes the grid from
// cudaOccupancyMaxActiveClusters.  Both words are zeroed on the launch stream
// before every launch.
__device__ __forceinline__ void wave_wait(unsigned int* ctr, unsigned int target, uint64_t timeout_ns) {
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  unsigned int v, off;
  for (;;) {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    if (v >= target) return;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(off) : "l"(ctr + 1) : "memory");
    if (off != 0u) return;
    uint64_t t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (t1 - t0 > timeout_ns) {
      asm volatile("st.relaxed.gpu.global.u32 [%0], 1;" ::"l"(ctr + 1) : "memory");
      return;
    }
  }
}
__device__ __forceinline__ void wave_arrive(unsigned int* ctr) {
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
}

// 256 x 512 pair tile epilogue, full tile with beta == 0: one warp's 32 rows
// x 256 columns.  Phase 1 drains TMEM — the first 64 columns straight into
// the warp's two 2 KB staging buffers, the other 192 into 96 registers of
// FP16 pairs (half(alpha * acc), the rounding of epi_store_block's mode 1;
// the register file caps at 168 per thread with 10 warps) — and arrives on
// the leader's tempty, so the next tile's MMAs start; phase 2 writes the 32-
// column blocks as 16-byte vectors of 8 consecutive rows of one column.
// Staging: column pair j, row r at word j * 32 + (r ^ 4 (j & 1)), conflict-
// free for the row-per-lane writes and the 8-row reads.
__device__ __forceinline__ void epi_store_early_release(uint32_t t_row, uint64_t* tempty, uint32_t* stage,
                                                        __half* cblk, int64_t ldc, float alpha, int lane) {
  uint32_t h[6][16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {  // 16 columns per tcgen05.ld
    uint32_t v[16];
    tmem_ld_32x32b_x16(t_row + i * 16, v);
    tmem_ld_wait();
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      const __half2 x = __floats2half2_rn(__fmul_rn(alpha, __uint_as_float(v[2 * jj])),
                                          __fmul_rn(alpha, __uint_as_float(v[2 * jj + 1])));
      const uint32_t w = *reinterpret_cast<const uint32_t*>(&x);
      const int chunk = i >> 1, j = (i & 1) * 8 + jj;
      if (chunk < 2)
        stage[chunk * 512 + j * 32 + (lane ^ ((j & 1) << 2))] = w;
      else
        h[chunk - 2][j] = w;
    }
  }
  tc_fence_before();
  mbar_arrive_cluster(tempty, 0);
  // lane's two items per block: column pair j, rows 8 rg .. 8 rg + 7
  const int j0 = lane >> 2, j1 = 8 + (lane >> 2), rg = lane & 3;
  const int r0 = j0 * 32 + ((rg * 8) ^ ((j0 & 1) << 2)), r1 = j1 * 32 + ((rg * 8) ^ ((j1 & 1) << 2));
  __half* d0 = cblk + static_cast<int64_t>(2 * j0) * ldc + rg * 8;
  __half* d1 = cblk + static_cast<int64_t>(2 * j1) * ldc + rg * 8;
  const int64_t step = 32 * ldc;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    uint32_t* buf = stage + (i & 1) * 512;
    if (i >= 2) {
#pragma unroll
      for (int j = 0; j < 16; ++j) buf[j * 32 + (lane ^ ((j & 1) << 2))] = h[i - 2][j];
    }
    __syncwarp();
#pragma unroll
    for (int it = 0; it < 2; ++it) {
      const int r = it ? r1 : r0;
      const uint4 x0 = *reinterpret_cast<const uint4*>(buf + r);
      const uint4 x1 = *reinterpret_cast<const uint4*>(buf + (r ^ 4));
      uint4 lo, hi;  // column 2j / 2j + 1, rows 8 rg .. 8 rg + 7
      lo.x = __byte_perm(x0.x, x0.y, 0x5410); hi.x = __byte_perm(x0.x, x0.y, 0x7632);
      lo.y = __byte_perm(x0.z, x0.w, 0x5410); hi.y = __byte_perm(x0.z, x0.w, 0x7632);
      lo.z = __byte_perm(x1.x, x1.y, 0x5410); hi.z = __byte_perm(x1.x, x1.y, 0x7632);
      lo.w = __byte_perm(x1.z, x1.w, 0x5410); hi.w = __byte_perm(x1.z, x1.w, 0x7632);
      __half* dst = it ? d1 : d0;
      *reinterpret_cast<uint4*>(dst) = lo;
      *reinterpret_cast<uint4*>(dst + ldc) = hi;
    }
    d0 += step;
    d1 += step;
  }
}

template <bool A_MN, bool B_MN, int BNP = 256>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(H2Cfg<BNP>::THREADS, 1)
    hgemm_tc_2sm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, Problem p,
                        int tiles_m, int tiles_n, int group_m, int64_t total_tiles, unsigned int* wave_ctr,
                        unsigned int wave_timeout_us) {
  using C = H2Cfg<BNP>;
  constexpr int STAGES = C::STAGES;
  constexpr int ACC = C::ACC;
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
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int64_t cluster_id = blockIdx.x >> 1;
  const int64_t n_clusters = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < ACC; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * 32 * C::EPI_WARPS);
    }
    fence_mbar_init();
  }
  if (warp == C::PROD_WARP && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == C::MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(C::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  grid_dep_wait();  // prologue above overlapped the previous kernel (PDL)
  grid_dep_launch();
  const int nkb = static_cast<int>((p.k + HG_BK - 1) / HG_BK);

  if (warp == C::PROD_WARP) {
    // =============== producer (both CTAs: own A half + own B half) ===============
    // The whole warp runs the loop (uniform coordinates); one elected lane issues.
    int s = 0;
    uint32_t ph = 0;
    unsigned int wave = 0;
    // waves every cluster completes (the last wave may be ragged)
    const unsigned int full_waves = static_cast<unsigned int>(total_tiles / n_clusters);
    for (int64_t t = cluster_id; t < total_tiles; t += n_clusters, ++wave) {
      if (wave_ctr != nullptr && wave > 0) {
        if (elect_one()) wave_wait(wave_ctr, min(wave, full_waves) * gridDim.x, 1000ull * wave_timeout_us);
        __syncwarp();
      }
      int64_t z; int mt, nt;
      tile_coords(t, tiles_m, tiles_n, group_m, z, mt, nt);
      const int m0 = mt * 256 + static_cast<int>(rank) * 128;
      const int n0 = nt * BNP + static_cast<int>(rank) * 128;
      const int zz = static_cast<int>(z);
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&empty[s], ph ^ 1);
        if (elect_one()) {
          if (leader) mbar_arrive_expect_tx(&full[s], 2 * C::STAGE_BYTES);
          const int k0 = kb * HG_BK;
          uint8_t* a_dst = sA + s * C::A_BYTES;
          uint8_t* b_dst = sB + s * C::B_BYTES;
          if (!A_MN) {
            tma_load_3d_2sm(a_dst, &tmA, &full[s], k0, m0, zz);
          } else {
            tma_load_3d_2sm(a_dst, &tmA, &full[s], m0, k0, zz);
            tma_load_3d_2sm(a_dst + 8192, &tmA, &full[s], m0 + 64, k0, zz);
          }
#pragma unroll
          for (int h = 0; h < BNP / 256; ++h) {  // 128 columns at n0 + 256 h -> b_dst + 16 KB h
            if (!B_MN) {
              tma_load_3d_2sm(b_dst + h * 16384, &tmB, &full[s], k0, n0 + 256 * h, zz);
            } else {
              tma_load_3d_2sm(b_dst + h * 16384, &tmB, &full[s], n0 + 256 * h, k0, zz);
              tma_load_3d_2sm(b_dst + h * 16384 + 8192, &tmB, &full[s], n0 + 256 * h + 64, k0, zz);
            }
          }
        }
        __syncwarp();
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
      if (wave_ctr != nullptr) {
        if (elect_one()) wave_arrive(wave_ctr);
        __syncwarp();
      }
    }
  } else if (warp == C::MMA_WARP) {
    // =============== MMA issuer (leader CTA only) ===============
    // The whole warp runs the loop (uniform operands); one elected lane issues.
    if (leader) {
      constexpr uint32_t idesc = umma_idesc_f16(256, 256, A_MN ? 1 : 0, B_MN ? 1 : 0);
      int s = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t aph = 0;
      for (int64_t t = cluster_id; t < total_tiles; t += n_clusters) {
        mbar_wait(&tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * 256);
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + s * C::A_BYTES);
          const uint32_t b_addr = smem_u32(sB + s * C::B_BYTES);
          const int ksteps = hg_ksteps(p.k, kb);
          if (elect_one()) {
#pragma unroll
            for (int h = 0; h < BNP / 256; ++h)
              hg_issue_kblock<A_MN, B_MN>(Mma2Sm{}, d_tmem + 256 * h, a_addr, b_addr + 16384 * h, idesc, ksteps,
                                          kb == 0);
            tc2_commit_mc(&empty[s], 0x3);
          }
          __syncwarp();
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
        if (elect_one()) tc2_commit_mc(&tfull[acc], 0x3);
        __syncwarp();
        if (++acc == ACC) { acc = 0; aph ^= 1; }
      }
    }
  } else if (warp < C::EPI_WARPS) {
    // =============== epilogue (both CTAs: own 128 rows x 256 columns) ===============
    const int quad = warp & 3;
    const int half = warp >> 2;
    int acc = 0;
    uint32_t aph = 0;
    float* stage = epi_stage + warp * EPI_WARP_FLOATS;
    for (int64_t t = cluster_id; t < total_tiles; t += n_clusters) {
      int64_t z; int mt, nt;
      tile_coords(t, tiles_m, tiles_n, group_m, z, mt, nt);
      const int64_t m0 = static_cast<int64_t>(mt) * 256 + rank * 128, n0 = static_cast<int64_t>(nt) * BNP;
      Epi epi;
      epi.alpha = inst_alpha(p, z);
      epi.beta = inst_beta(p, z);
      epi.skip_ab = (epi.alpha == 0.0f);
      const int64_t row0 = m0 + quad * 32;
      const int rows_valid = static_cast<int>(min64(32, p.m - row0));
      __half* Cz = static_cast<__half*>(p.c) + inst_off(p.c_off, p.stride_c, p.c_offs, z);
      const int n_left = static_cast<int>(min64(BNP, p.n - n0));
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + static_cast<uint32_t>(acc * 256);
      if constexpr (BNP == 512) {
        // One accumulator: the next tile's MMAs wait for this drain.  For
        // full tiles with beta == 0 read all 256 columns out of TMEM first
        // (rounded to FP16 exactly as epi_store_block's mode 1 does), give
        // the accumulator back, then store from registers while the next
        // tile runs.
        __half* cw = Cz + n0 * p.ldc + row0;
        if (!epi.skip_ab && epi.beta == 0.0f && rows_valid >= 32 && n_left >= BNP && (p.ldc & 7) == 0 &&
            (reinterpret_cast<uintptr_t>(cw) & 15) == 0) {
          epi_store_early_release(t_row + half * 256, &tempty[acc], reinterpret_cast<uint32_t*>(stage),
                                  cw + static_cast<int64_t>(half) * 256 * p.ldc, p.ldc, epi.alpha, lane);
          if (++acc == ACC) { acc = 0; aph ^= 1; }
          continue;
        }
      }
#pragma unroll 1
      for (int cb = half * (BNP / 64); cb < (half + 1) * (BNP / 64); ++cb) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(t_row + cb * 32, v);
        tmem_ld_wait();
        if (rows_valid > 0 && cb * 32 < n_left)
          epi_store_block(stage, v, Cz + (n0 + cb * 32) * p.ldc + row0, p.ldc, rows_valid, n_left - cb * 32, epi, lane);
      }
      tc_fence_before();
      mbar_arrive_cluster(&tempty[acc], 0);
      if (++acc == ACC) { acc = 0; aph ^= 1; }
    }
  }

  tc_fence_before();
  cluster_sync_all();
  if (warp == C::MMA_WARP) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(C::TMEM_COLS)
                 : "memory");
  }
}

}  // namespace tb
