// sgemm.cu — SGEMM dispatch: register-staged FFMA2 kernel (sgemm_simt.cuh),
// cp.async small-instance kernel (sgemm_small.cuh), opt-in TF32 tcgen05
// kernel (sgemm_tf32_tc.cuh); the TMA-fed kernel's routing is in
// sgemm_tma.cu.
#include <cstring>

#include "host.h"
#include "sgemm_simt.cuh"
#include "sgemm_small.cuh"
#include "sgemm_tf32_tc.cuh"

namespace tb {
namespace host {
namespace {

template <int BM, int BN, int BK, int TM, int TN, bool VEC, int MINB, bool CONV = false>
int launch_simt(const Call& c) {
  const Problem& p = c.p;
  const int tiles_m = static_cast<int>((p.m + BM - 1) / BM);
  const int tiles_n = static_cast<int>((p.n + BN - 1) / BN);
  const int64_t blocks = static_cast<int64_t>(tiles_m) * tiles_n * p.batch;
  if (blocks > 0x7fffffffLL) return TB_ERR_INVALID;
  const int group_m = cfg_group_m(c, 8);
  dim3 grid(static_cast<unsigned>(blocks)), block(SimtShape<BM, BN, BK, TM, TN>::NT);
  const int sel = (p.a_kcontig ? 2 : 0) | (p.b_ncontig ? 1 : 0);
  const ConvGeom geom = c.conv ? *c.conv : ConvGeom{};
  int rc;
  if constexpr (CONV) {  // op(A) gathered (M-contiguous layout), filters K-contiguous
    rc = launch_ex("sgemm_conv launch", sgemm_simt_kernel<BM, BN, BK, TM, TN, false, false, VEC, MINB, true>, grid,
                   block, 0, c.stream, 1, p, tiles_m, tiles_n, group_m, geom);
  } else {
    switch (sel) {
      case 0: rc = launch_ex("sgemm_simt launch", sgemm_simt_kernel<BM, BN, BK, TM, TN, false, false, VEC, MINB>, grid, block, 0, c.stream, 1, p, tiles_m, tiles_n, group_m, geom); break;
      case 1: rc = launch_ex("sgemm_simt launch", sgemm_simt_kernel<BM, BN, BK, TM, TN, false, true, VEC, MINB>, grid, block, 0, c.stream, 1, p, tiles_m, tiles_n, group_m, geom); break;
      case 2: rc = launch_ex("sgemm_simt launch", sgemm_simt_kernel<BM, BN, BK, TM, TN, true, false, VEC, MINB>, grid, block, 0, c.stream, 1, p, tiles_m, tiles_n, group_m, geom); break;
      default: rc = launch_ex("sgemm_simt launch", sgemm_simt_kernel<BM, BN, BK, TM, TN, true, true, VEC, MINB>, grid, block, 0, c.stream, 1, p, tiles_m, tiles_n, group_m, geom); break;
    }
  }
  if (rc) return rc;
  char name[64];
  static const char* lay[4] = {"mk", "mn", "kk", "kn"};  // A major x B major
  snprintf(name, sizeof(name), "sgemm_%s_%dx%dx%d_%s_%s", CONV ? "conv" : "simt", BM, BN, BK,
           VEC ? "vec" : "gen", lay[sel]);
  record(name, grid, block, 1, 0, blocks);
  return check_launch("sgemm_simt launch");
}

template <int MI, int NI, int TM, int TN, bool AK, bool BNC>
int launch_ss(const Call& c) {
  using Cfg = SsCfg<MI, NI, TM, TN>;
  const Problem& p = c.p;
  const int64_t groups = (p.batch + Cfg::G - 1) / Cfg::G;
  auto kern = sgemm_small_kernel<MI, NI, TM, TN, AK, BNC>;
  static SmemAttr attr;
  if (int rc = ensure_smem(attr, kern, Cfg::SMEM_BYTES)) return rc;
  static int per_sm = 0;
  if (per_sm == 0) {
    int v = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kern, 256, Cfg::SMEM_BYTES) != cudaSuccess || v < 1) v = 1;
    per_sm = v;
  }
  const int64_t cap = static_cast<int64_t>(sms_or_default()) * per_sm;
  const int64_t g = groups < cap ? groups : cap;
  dim3 grid(static_cast<unsigned>(g)), block(256);
  if (int rc = launch_ex("sgemm_small launch", kern, grid, block, Cfg::SMEM_BYTES, c.stream, 1, p, groups)) return rc;
  char name[64];
  snprintf(name, sizeof(name), "sgemm_small_%dx%d_t%dx%d_g%d_%c%c", MI, NI, TM, TN, Cfg::G, AK ? 'k' : 'm',
           BNC ? 'n' : 'k');
  record(name, grid, block, 1, Cfg::SMEM_BYTES, groups);
  return check_launch("sgemm_small launch");
}

template <int MI, int NI, int TM, int TN>
int launch_ss_layout(const Call& c) {
  const bool ak = c.p.a_kcontig, bnc = c.p.b_ncontig;
  if (!ak && !bnc) return launch_ss<MI, NI, TM, TN, false, false>(c);
  if (!ak && bnc) return launch_ss<MI, NI, TM, TN, false, true>(c);
  if (ak && !bnc) return launch_ss<MI, NI, TM, TN, true, false>(c);
  return launch_ss<MI, NI, TM, TN, true, true>(c);
}

template <int BN, bool AMN, bool BMN>
int launch_tf32(const Call& c, const CUtensorMap& ta, const CUtensorMap& tbm) {
  using Cfg = TfCfg<BN>;
  const Problem& p = c.p;
  const int tiles_m = static_cast<int>((p.m + HG_BM - 1) / HG_BM);
  const int tiles_n = static_cast<int>((p.n + BN - 1) / BN);
  const int64_t total = static_cast<int64_t>(tiles_m) * tiles_n * p.batch;
  auto kern = sgemm_tf32_tc_kernel<BN, AMN, BMN>;
  static SmemAttr attr;  // per instantiation, per device
  if (int rc = ensure_smem(attr, kern, Cfg::SMEM_BYTES)) return rc;
  const int sms = sms_or_default();
  const int64_t g = total < sms ? total : sms;
  dim3 grid(static_cast<unsigned>(g)), block(Cfg::THREADS);
  if (int rc = launch_ex("sgemm_tf32_tc launch", kern, grid, block, Cfg::SMEM_BYTES, c.stream, 1, ta, tbm, p, tiles_m,
                         tiles_n, cfg_group_m(c, 16), total))
    return rc;
  char name[64];
  snprintf(name, sizeof(name), "sgemm_tf32_tc_tma_128x%d_%c%c", BN, AMN ? 'm' : 'k', BMN ? 'n' : 'k');
  record(name, grid, block, 1, Cfg::SMEM_BYTES, total);
  return check_launch("sgemm_tf32_tc launch");
}

template <int BN>
int dispatch_tf32_bn(const Call& c) {
  const Problem& p = c.p;
  const bool amn = !p.a_kcontig, bmn = p.b_ncontig;
  const float* A = static_cast<const float*>(p.a) + p.a_off;
  const float* B = static_cast<const float*>(p.b) + p.b_off;
  CUtensorMap ta, tbm;
  memset(&ta, 0, sizeof(ta));
  memset(&tbm, 0, sizeof(tbm));
  const CUtensorMapDataType F32 = CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  // MN-major FP32 operands: 32-byte swizzle atoms (sgemm_tf32_tc.cuh)
  const CUtensorMapSwizzle MN32 = CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;
  int rc = !amn ? make_map(&ta, A, p.k, p.m, p.batch, p.lda, p.stride_a, 32, 128, F32, 4)
                : make_map(&ta, A, p.m, p.k, p.batch, p.lda, p.stride_a, 32, 32, F32, 4, MN32);
  if (rc != TB_OK) return rc;
  rc = !bmn ? make_map(&tbm, B, p.k, p.n, p.batch, p.ldb, p.stride_b, 32, BN, F32, 4)
            : make_map(&tbm, B, p.n, p.k, p.batch, p.ldb, p.stride_b, 32, 32, F32, 4, MN32);
  if (rc != TB_OK) return rc;
  if (!amn && !bmn) return launch_tf32<BN, false, false>(c, ta, tbm);
  if (!amn && bmn) return launch_tf32<BN, false, true>(c, ta, tbm);
  if (amn && !bmn) return launch_tf32<BN, true, false>(c, ta, tbm);
  return launch_tf32<BN, true, true>(c, ta, tbm);
}

// Opt-in TF32 tensor-core SGEMM (TB_FLAG_TF32): TMA producer only, so the
// operands must be 16-byte aligned with arithmetic batch offsets.
int dispatch_tf32(const Call& c) {
  const Problem& p = c.p;
  bool ok = (p.lda % 4 == 0) && (p.ldb % 4 == 0) && aligned_elems(p.a, p.a_off, 4, 16) &&
            aligned_elems(p.b, p.b_off, 4, 16) && !p.a_offs && !p.b_offs;
  if (p.batch > 1) ok = ok && (p.stride_a % 4 == 0) && (p.stride_b % 4 == 0);
  if (!ok) {
    snprintf(err_buf(), 256,
             "TF32 path needs 16-byte aligned operands (ld and offsets multiples of 4) and strided batches");
    return TB_ERR_UNSUPPORTED;
  }
  const int sms = sms_or_default();
  int bn = 256;
  auto tiles = [&](int b) { return ((p.m + HG_BM - 1) / HG_BM) * ((p.n + b - 1) / b) * p.batch; };
  while (bn > 64 && tiles(bn) < sms) bn /= 2;
  if (bn == 256) return dispatch_tf32_bn<256>(c);
  if (bn == 128) return dispatch_tf32_bn<128>(c);
  return dispatch_tf32_bn<64>(c);
}

// A configured register-staged (KWG 16) tile.
int simt_tile(const Call& c, int mwg, int nwg) {
  if (mwg >= 128 && nwg >= 256) return launch_simt<128, 256, 8, 8, 16, true, 1>(c);
  if (mwg >= 128 && nwg >= 128) return launch_simt<128, 128, 16, 8, 8, true, 1>(c);
  if (mwg >= 128) return launch_simt<128, 64, 16, 8, 4, true, 2>(c);
  if (nwg >= 128) return launch_simt<64, 128, 16, 4, 8, true, 2>(c);
  if (mwg <= 32 && nwg <= 32) return launch_simt<32, 32, 32, 4, 4, true, 8>(c);
  return launch_simt<64, 64, 16, 4, 4, true, 2>(c);
}

}  // namespace

// Implicit GEMM (tb_convgemm) for S: the register-staged FFMA2 kernel with
// op(A) gathered from the image (simt_conv_stage).  The gathered values are
// the im2col entries exactly, so results equal im2col + gemm bitwise (the
// sequential-k chain).  64x64 tiles (4x4 micro-tiles) keep the SMs busy at
// the typical layer shapes (a few thousand positions x tens of filters).
int dispatch_sconv(const Call& c) {
  const Problem& p = c.p;
  const bool vec = (p.ldb % 4 == 0) && aligned_elems(p.b, p.b_off, 4, 16);
  if (vec) return launch_simt<64, 64, 16, 4, 4, true, 2, true>(c);
  return launch_simt<64, 64, 16, 4, 4, false, 2, true>(c);
}

int dispatch_sgemm(const Call& c) {
  const Problem& p = c.p;
  // k == 0 / alpha == 0 need no products: the FFMA kernels' epilogue handles them.
  if ((c.flags & TB_FLAG_TF32) && p.k > 0 && !(p.alphas == nullptr && p.alpha == 0.0f)) return dispatch_tf32(c);
  // 16-byte vector loads need every operand element base and ld to be
  // multiples of 4 floats.
  bool vec = (p.lda % 4 == 0) && (p.ldb % 4 == 0) && aligned_elems(p.a, 0, 4, 16) && aligned_elems(p.b, 0, 4, 16);
  if (p.a_offs || p.b_offs) {
    vec = vec && c.offs_aligned;
  } else {
    vec = vec && (p.a_off % 4 == 0) && (p.b_off % 4 == 0);
    if (p.batch > 1) vec = vec && (p.stride_a % 4 == 0) && (p.stride_b % 4 == 0);
  }
  if (c.flags & TB_FLAG_SIMT_GENERAL) vec = false;
  // Unaligned operands (not the testing flag): repack once into aligned
  // scratch and route the copies (tbgemm.cu repack_operands; 2501^3: 1130
  // us on the general kernel).
  if (!vec && !(c.flags & TB_FLAG_SIMT_GENERAL) && !p.a_offs && !p.b_offs) {
    Call c2 = c;
    int launches = 0;
    if (repack_operands(c, 4, c2, launches) == TB_OK) {
      const int rc = dispatch_sgemm(c2);
      if (rc == TB_OK) note_extra_launches(launches, "+pack");
      return rc;
    }
  }
  // Every SGEMM instantiation computes the same sequential-k FMA chain per
  // element, so tile choice is free to follow speed.
  if (!vec) return launch_simt<64, 64, 16, 4, 4, false, 2>(c);
  const tb_gemm_config* g = c.cfg;
  if (g && g->MWG > 0) {
    // A "gemm_b200" configuration (override / tuning DB): its tile, on the
    // TMA-fed kernel for KWG 32 when the operands allow tensor maps.
    if (g->KWG >= 32) {
      const int rc = dispatch_sgemm_tma(c, -1, g->MWG, g->NWG, g->SPLIT_K);
      if (rc >= 0) return rc;
    }
    return simt_tile(c, g->MWG, g->NWG);
  }
  const bool small_inst = p.k > 0 && p.m <= 64 && p.n <= 64 && (p.batch > 1 || p.k <= 4096);
  if (!small_inst) {
    const int rc = dispatch_sgemm_tma(c, 0, 0, 0);
    if (rc >= 0) return rc;
  }
  // Small instances: persistent cp.async-pipelined kernel (bitwise identical).
  if (small_inst) {
    if (p.m <= 32 && p.n <= 32) {
      // one 32x32 tile per instance on the TMA kernel when the operands allow
      // tensor maps (S32 batched 59.4 -> 48.7 us; a persistent variant of the
      // TMA kernel measured slower: 53.6 us, and 20 % slower at 8192^3)
      const int rc = dispatch_sgemm_tma(c, 3, 0, 0);
      if (rc >= 0) return rc;
      return launch_ss_layout<32, 32, 4, 4>(c);
    }
    // 33..64: one 64x64 tile per instance on the TMA-fed FFMA2 kernel (3-D
    // tensor maps over the batch) when the operands allow tensor maps; else
    // the register-staged tiled kernel with a 4x8 micro-tile (measured faster
    // than the cp.async small kernel for 64^3, tools/sgemm_batched_variants.cu)
    const int rc = dispatch_sgemm_tma(c, 2, 0, 0);
    if (rc >= 0) return rc;
    return launch_simt<64, 64, 16, 4, 8, true, 2>(c);
  }
  // Operands that do not allow tensor maps (per-instance offset arrays, alpha
  // arrays, alpha == 0, k == 0): the register-staged kernel by shape.
  const int sms = sms_or_default();
  const int64_t tiles128 = ((p.m + 127) / 128) * ((p.n + 127) / 128) * p.batch;
  if (p.m <= 32 && p.n <= 32) return launch_simt<32, 32, 32, 4, 4, true, 8>(c);
  // 128x256 (8x16 micro-tile) once there are >= 4 waves of it; else 128x128x16.
  const int64_t tiles256 = ((p.m + 127) / 128) * ((p.n + 255) / 256) * p.batch;
  if (tiles256 >= 4 * sms) return launch_simt<128, 256, 8, 8, 16, true, 1>(c);
  if (tiles128 >= sms) return launch_simt<128, 128, 16, 8, 8, true, 1>(c);
  // < 1 wave of 128x128: 64x128 4x8 (measured 30.7 vs 27.8 TFLOP/s for
  // 64x64 4x4 at 1024^3; tools/sgemm_variants.cu)
  if (p.n >= 128 && tiles128 * 2 * 2 >= sms) return launch_simt<64, 128, 16, 4, 8, true, 2>(c);
  return launch_simt<64, 64, 16, 4, 4, true, 2>(c);
}

}  // namespace host
}  // namespace tb
