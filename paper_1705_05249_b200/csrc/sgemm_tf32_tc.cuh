// sgemm_tf32_tc.cuh — OPT-IN TF32 tensor-core SGEMM (TB_FLAG_TF32).
//
// The north star keeps FP32 GEMM on the FFMA pipe (TF32 inputs exceed the
// reference SGEMM tolerance by 4.5-31x, SURVEY §8a evidence) and allows a
// TF32 tensor-core variant only behind an explicit flag.  This is that
// variant: the same persistent, warp-specialised tcgen05 structure as
// hgemm_tc_kernel, with FP32 operands in shared memory —
//   * a 128-byte SWIZZLE_128B row holds 32 FP32 values, so the K block is 32;
//   * tcgen05.mma.cta_group::1.kind::tf32 consumes K = 8 per instruction
//     (32 bytes of each K-major row, or 8 K-rows of an MN-major tile);
//   * MN-major tiles are 32-element (128-byte) chunks of 32 K-rows (4 KB),
//     loaded with TMA SWIZZLE_128B_ATOM_32B (32-byte granules swizzled in a
//     128-byte row) and described to the MMA as layout type 1
//     (SWIZZLE_128B_BASE32B): LBO 4096 B between 32-element MN chunks, SBO
//     512 B between 4-row K groups, +1024 B per K8 step — the layout the
//     hardware accepted in tools/tf32_mn_probe.cu (every 16-byte-swizzle
//     variant read garbage: FP32 MN-major needs the 32-byte atom);
//   * the epilogue applies the reference FP32 epilogue and stores FP32.
// TMA producer only: operands must be 16-byte aligned (checked by the host).
#pragma once

#include "hgemm_tc.cuh"

namespace tb {

constexpr int TF_BK = 32;  // FP32 elements per 128-byte row

template <int BN>
struct TfCfg {
  static constexpr int STAGES = (BN >= 256) ? 4 : 6;
  static constexpr int A_BYTES = HG_BM * TF_BK * 4;   // 16 KB
  static constexpr int B_BYTES = BN * TF_BK * 4;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = (2 * BN <= 128) ? 128 : (2 * BN <= 256) ? 256 : 512;
  static constexpr int EPI_WARPS = 8, PROD_WARP = 8, MMA_WARP = 9;
  static constexpr int THREADS = 10 * 32;
  static constexpr int BAR_BYTES = 1024;
  static constexpr int EPI_BYTES = EPI_WARPS * EPI_WARP_FLOATS * 4;
  static constexpr int SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + BAR_BYTES + EPI_BYTES;
};

// Instruction descriptor, kind::tf32: TF32 x TF32 -> F32 (a/b format 2).
__host__ __device__ constexpr uint32_t umma_idesc_tf32(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(a_mn) << 15) |
         (static_cast<uint32_t>(b_mn) << 16) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}
__device__ __forceinline__ void tc_mma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// MN-major FP32 operand descriptor (SWIZZLE_128B_BASE32B, layout type 1).
__device__ __forceinline__ uint64_t umma_desc_mn_tf32(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(4096 >> 4) << 16;   // LBO: next 32-element MN chunk
  d |= static_cast<uint64_t>(512 >> 4) << 32;    // SBO: next 4-row K group
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(1) << 61;           // SWIZZLE_128B_BASE32B
  return d;
}

// FP32 variant of epi_store_block: 8 consecutive rows of one column per lane
// become two 16-byte stores.
__device__ __forceinline__ void epi_store_block_f32(float* stage, const uint32_t (&v)[32], float* cblk, int64_t ldc,
                                                    int rows_valid, int cols_valid, const Epi& epi, int lane) {
#pragma unroll
  for (int c = 0; c < 32; ++c) stage[epi_idx(c, lane)] = __uint_as_float(v[c]);
  __syncwarp();
  const int cl = lane & 7, rg = lane >> 3;
  const bool vec_ok = ((reinterpret_cast<uintptr_t>(cblk) & 15) == 0) && ((ldc & 3) == 0);
#pragma unroll
  for (int cgi = 0; cgi < 4; ++cgi) {
    const int c = cgi * 8 + cl;
    const float4 x0 = *reinterpret_cast<const float4*>(stage + epi_idx(c, rg * 8));
    const float4 x1 = *reinterpret_cast<const float4*>(stage + epi_idx(c, rg * 8 + 4));
    if (c < cols_valid && rg * 8 < rows_valid) {
      float* dst = cblk + static_cast<int64_t>(c) * ldc + rg * 8;
      float x[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
      if (vec_ok && rg * 8 + 8 <= rows_valid) {
        float cv[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        if (epi.reads_c()) {
          const float4 c0 = *reinterpret_cast<const float4*>(dst);
          const float4 c1 = *reinterpret_cast<const float4*>(dst + 4);
          cv[0] = c0.x; cv[1] = c0.y; cv[2] = c0.z; cv[3] = c0.w;
          cv[4] = c1.x; cv[5] = c1.y; cv[6] = c1.z; cv[7] = c1.w;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = epi.apply(x[i], cv[i]);
        *reinterpret_cast<float4*>(dst) = make_float4(x[0], x[1], x[2], x[3]);
        *reinterpret_cast<float4*>(dst + 4) = make_float4(x[4], x[5], x[6], x[7]);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (rg * 8 + i < rows_valid) dst[i] = epi.apply(x[i], epi.reads_c() ? dst[i] : 0.0f);
      }
    }
  }
  __syncwarp();
}

template <int BN, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(TfCfg<BN>::THREADS, 1)
    sgemm_tf32_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, Problem p,
                         int tiles_m, int tiles_n, int group_m, int64_t total_tiles) {
  using C = TfCfg<BN>;
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
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 32 * C::EPI_WARPS);
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
  const int nkb = static_cast<int>((p.k + TF_BK - 1) / TF_BK);

  if (warp == C::PROD_WARP) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int64_t t = blockIdx.x; t < total_tiles; t += gridDim.x) {
        int64_t z; int mt, nt;
        tile_coords(t, tiles_m, tiles_n, group_m, z, mt, nt);
        const int m0 = mt * HG_BM, n0 = nt * BN, zz = static_cast<int>(z);
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&full[s], C::STAGE_BYTES);
          const int k0 = kb * TF_BK;
          uint8_t* a_dst = sA + s * C::A_BYTES;
          uint8_t* b_dst = sB + s * C::B_BYTES;
          if (!A_MN) {
            tma_load_3d(a_dst, &tmA, &full[s], k0, m0, zz);
          } else {
#pragma unroll
            for (int c = 0; c < HG_BM / 32; ++c) tma_load_3d(a_dst + c * 4096, &tmA, &full[s], m0 + 32 * c, k0, zz);
          }
          if (!B_MN) {
            tma_load_3d(b_dst, &tmB, &full[s], k0, n0, zz);
          } else {
#pragma unroll
            for (int c = 0; c < BN / 32; ++c) tma_load_3d(b_dst + c * 4096, &tmB, &full[s], n0 + 32 * c, k0, zz);
          }
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == C::MMA_WARP) {
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_tf32(HG_BM, BN, A_MN ? 1 : 0, B_MN ? 1 : 0);
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
#pragma unroll
          for (int kk = 0; kk < TF_BK / 8; ++kk) {
            const uint64_t adesc = A_MN ? umma_desc_mn_tf32(a_addr + kk * 1024)
                                        : umma_desc_sw128(a_addr + kk * 32, 16, 1024);
            const uint64_t bdesc = B_MN ? umma_desc_mn_tf32(b_addr + kk * 1024)
                                        : umma_desc_sw128(b_addr + kk * 32, 16, 1024);
            tc_mma_tf32(d_tmem, adesc, bdesc, idesc, (kb | kk) != 0 ? 1u : 0u);
          }
          tc_commit(&empty[s]);
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
        tc_commit(&tfull[acc]);
        if (++acc == 2) { acc = 0; aph ^= 1; }
      }
    }
  } else if (warp < C::EPI_WARPS) {
    const int quad = warp & 3;
    const int half = warp >> 2;
    int acc = 0;
    uint32_t aph = 0;
    float* stage = epi_stage + warp * EPI_WARP_FLOATS;
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
      float* Cz = static_cast<float*>(p.c) + inst_off(p.c_off, p.stride_c, p.c_offs, z);
      const int n_left = static_cast<int>(min64(BN, p.n - n0));
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + static_cast<uint32_t>(acc * BN);
#pragma unroll 1
      for (int cb = half * (BN / 64); cb < (half + 1) * (BN / 64); ++cb) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(t_row + cb * 32, v);
        tmem_ld_wait();
        if (rows_valid > 0 && cb * 32 < n_left)
          epi_store_block_f32(stage, v, Cz + (n0 + cb * 32) * p.ldc + row0, p.ldc, rows_valid, n_left - cb * 32,
                              epi, lane);
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

}  // namespace tb
