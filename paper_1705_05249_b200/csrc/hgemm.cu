// hgemm.cu — HGEMM dispatch over the tcgen05 kernels: single-CTA
// (hgemm_tc.cuh), CTA pair (hgemm_tc_2sm.cuh), cluster split-K
// (hgemm_tc_splitk.cuh); small instances are in hgemm_small.cu.
#include <cstring>

#include "hgemm_tc.cuh"
#include "hgemm_tc_2sm.cuh"
#include "hgemm_tc_splitk.cuh"
#include "host.h"

namespace tb {
namespace host {
namespace {

bool hgemm_aligned(const Call& c) {
  const Problem& p = c.p;
  bool al = (p.lda % 8 == 0) && (p.ldb % 8 == 0) && aligned_elems(p.a, 0, 2, 16) && aligned_elems(p.b, 0, 2, 16);
  if (p.a_offs || p.b_offs) {
    al = al && c.offs_aligned;
  } else {
    al = al && (p.a_off % 8 == 0) && (p.b_off % 8 == 0);
    if (p.batch > 1) al = al && (p.stride_a % 8 == 0) && (p.stride_b % 8 == 0);
  }
  return al;
}

bool tma_ok(const Call& c) {
  const Problem& p = c.p;
  const bool generic = (p.a_offs != nullptr) || (p.b_offs != nullptr);
  const bool fits = p.m < (1LL << 31) && p.n < (1LL << 31) && p.k < (1LL << 31) && p.batch < (1LL << 31);
  return hgemm_aligned(c) && !generic && fits && !(c.flags & TB_FLAG_NO_TMA);
}

template <int BN, bool TMA, bool AMN, bool BMN, bool VEC, int ST = 0, bool CONV = false>
int launch_hg(const Call& c, const CUtensorMap& ta, const CUtensorMap& tbm) {
  using Cfg = HgCfg<BN, TMA, ST>;
  const Problem& p = c.p;
  const int tiles_m = static_cast<int>((p.m + HG_BM - 1) / HG_BM);
  const int tiles_n = static_cast<int>((p.n + BN - 1) / BN);
  const int64_t total = static_cast<int64_t>(tiles_m) * tiles_n * p.batch;
  auto kern = hgemm_tc_kernel<BN, TMA, AMN, BMN, VEC, ST, CONV>;
  static SmemAttr attr;  // per instantiation, per device
  if (int rc = ensure_smem(attr, kern, Cfg::SMEM_BYTES)) return rc;
  const int sms = sms_or_default();
  const int64_t g = total < sms ? total : sms;
  dim3 grid(static_cast<unsigned>(g)), block(Cfg::THREADS);
  const ConvGeom geom = c.conv ? *c.conv : ConvGeom{};
  if (int rc = launch_ex("hgemm_tc launch", kern, grid, block, Cfg::SMEM_BYTES, c.stream, 1, ta, tbm, p, tiles_m,
                         tiles_n, cfg_group_m(c, 16), total, geom))
    return rc;
  char name[64];
  snprintf(name, sizeof(name), "hgemm_tc_%s_128x%d_%c%c%s%s", CONV ? "conv" : (TMA ? "tma" : "ldg"), BN,
           AMN ? 'm' : 'k', BMN ? 'n' : 'k', (!TMA && !VEC) ? "_scalar" : "",
           ST > 0 ? (ST == 3 ? "_st3" : "_st4") : "");
  record(name, grid, block, 1, Cfg::SMEM_BYTES, total);
  return check_launch("hgemm_tc launch");
}

template <int BN, bool TMA, bool VEC, int ST = 0>
int launch_hg_layout(const Call& c, const CUtensorMap& ta, const CUtensorMap& tbm) {
  const bool amn = !c.p.a_kcontig, bmn = c.p.b_ncontig;
  if (!amn && !bmn) return launch_hg<BN, TMA, false, false, VEC, ST>(c, ta, tbm);
  if (!amn && bmn) return launch_hg<BN, TMA, false, true, VEC, ST>(c, ta, tbm);
  if (amn && !bmn) return launch_hg<BN, TMA, true, false, VEC, ST>(c, ta, tbm);
  return launch_hg<BN, TMA, true, true, VEC, ST>(c, ta, tbm);
}

// The shallower ring a "gemm_b200" STAGES asks for (TMA producer only): BN 256
// 4 -> 3, BN 64 / 128 6 -> 4.  Default depth otherwise.
template <int BN>
int launch_hg_tma_stages(const Call& c, const CUtensorMap& ta, const CUtensorMap& tbm) {
  constexpr int SHALLOW = BN >= 256 ? 3 : 4;
  if (c.cfg && c.cfg->STAGES == SHALLOW) return launch_hg_layout<BN, true, true, SHALLOW>(c, ta, tbm);
  // Built-in route, at most 4 K blocks: the shallow ring (the tile's few
  // stages never fill the deep one; tools/route_audit.py: 128^3 x 1024 26.6
  // -> 24.6 us, 8192^2 x 256 75.8 -> 70.6 us)
  if (!(c.cfg && c.cfg->MWG > 0) && c.p.k <= 4 * HG_BK) return launch_hg_layout<BN, true, true, SHALLOW>(c, ta, tbm);
  return launch_hg_layout<BN, true, true>(c, ta, tbm);
}

template <bool AMN, bool BMN, int BNP = 256>
int launch_h2(const Call& c, const CUtensorMap& ta, const CUtensorMap& tbm, bool sync_waves) {
  using Cfg = H2Cfg<BNP>;
  const Problem& p = c.p;
  const int tiles_m = static_cast<int>((p.m + 255) / 256);
  const int tiles_n = static_cast<int>((p.n + BNP - 1) / BNP);
  const int64_t total = static_cast<int64_t>(tiles_m) * tiles_n * p.batch;
  auto kern = hgemm_tc_2sm_kernel<AMN, BMN, BNP>;
  static SmemAttr attr;  // per instantiation, per device
  if (int rc = ensure_smem(attr, kern, Cfg::SMEM_BYTES)) return rc;
  // Persistent clusters: as many pairs as can be co-resident (the wave
  // barrier assumes co-residency; the occupancy query sees only this
  // kernel's limits, hence the barrier's abandon flag).
  static int max_pairs[64] = {0};  // per instantiation, per device
  const int dev = current_device();
  if (max_pairs[dev] == 0) {
    cudaLaunchConfig_t q = {};
    q.gridDim = dim3(2);
    q.blockDim = dim3(Cfg::THREADS);
    q.dynamicSmemBytes = Cfg::SMEM_BYTES;
    int v = 0;
    if (cudaOccupancyMaxActiveClusters(&v, kern, &q) != cudaSuccess || v < 1) {
      cudaGetLastError();
      v = sms_or_default() / 2;
    }
    max_pairs[dev] = v;
  }
  const int64_t clusters = total < max_pairs[dev] ? total : max_pairs[dev];
  dim3 grid(static_cast<unsigned>(2 * clusters)), block(Cfg::THREADS);
  unsigned int* ctr = nullptr;
  if (sync_waves) {
    ctr = wave_counter(c.stream);  // nullptr: run without the (advisory) barrier
    if (ctr && cudaMemsetAsync(ctr, 0, 2 * sizeof(unsigned int), c.stream) != cudaSuccess)
      return check_launch("wave counter");
  }
  // The barrier's one-shot timeout: 2 ms for the > 6 TFLOP calls (tens of
  // ms); below, ~2 pair tiles' time (a 256 x 512 tile at K = 8192 takes
  // ~0.1 ms), at least 200 us — so a call sharing the SMs with other work
  // (CTAs not co-resident) loses at most that, once.
  const double flop = 2.0 * static_cast<double>(p.m) * p.n * p.k * p.batch;
  const int64_t kscaled = p.k * 200 / 8192;
  const unsigned int timeout_us =
      flop > 6e12 ? 2000u : static_cast<unsigned int>(kscaled < 200 ? 200 : (kscaled > 2000 ? 2000 : kscaled));
  // group_m 8: measured best for pair tiles (also with the wave barrier)
  if (int rc = launch_ex("hgemm_tc_2sm launch", kern, grid, block, Cfg::SMEM_BYTES, c.stream, 1, ta, tbm, p,
                         tiles_m, tiles_n, cfg_group_m(c, BNP == 512 ? 16 : 8), total, ctr, timeout_us))
    return rc;
  char name[64];
  snprintf(name, sizeof(name), "hgemm_tc2sm_tma_256x%d_%c%c%s", BNP, AMN ? 'm' : 'k', BMN ? 'n' : 'k',
           ctr ? "_ws" : "");
  record(name, grid, block, 2, Cfg::SMEM_BYTES, total);
  return check_launch("hgemm_tc_2sm launch");
}

// pair: -1 = by shape, 0 = single-CTA kernel, 1 = CTA pair (256 x 256),
// 2 = CTA pair with the 256 x 512 tile.
template <int BN>
int dispatch_hgemm_bn(const Call& c, int pair) {
  const Problem& p = c.p;
  const bool amn = !p.a_kcontig, bmn = p.b_ncontig;
  CUtensorMap ta, tbm;
  memset(&ta, 0, sizeof(ta));
  memset(&tbm, 0, sizeof(tbm));
  if (tma_ok(c)) {
    const __half* A = static_cast<const __half*>(p.a) + p.a_off;
    const __half* B = static_cast<const __half*>(p.b) + p.b_off;
    int rc;
    if (!amn) rc = make_map(&ta, A, p.k, p.m, p.batch, p.lda, p.stride_a, 64, 128);
    else rc = make_map(&ta, A, p.m, p.k, p.batch, p.lda, p.stride_a, 64, 64);
    if (rc != TB_OK) return rc;
    // CTA-pair kernel for large problems (>= one wave of 256x256 pair tiles).
    const int sms = sms_or_default();
    const int64_t pair_tiles = ((p.m + 255) / 256) * ((p.n + 255) / 256) * p.batch;
    const double flop = 2.0 * static_cast<double>(p.m) * p.n * p.k * p.batch;
    // Above ~6 TFLOP per call the pair kernel runs with the wave barrier
    // (hgemm_tc_2sm.cuh): 32768^3 945 -> 1286 TFLOP/s, 16384^3 1256 -> 1398,
    // vs 1150 / 1325 for the single-CTA kernel (tools/hbig_probe.py).  Below
    // that the barrier measured neutral and is left off.
    const bool huge = flop > 6e12;
    // The pair once its CTAs (two per pair tile) fill three quarters of the
    // SMs: 2048^2 x 8192 55.3 us against 61.4 for the single-CTA 128 x 256
    // tiles in the same single wave (tools/route_audit.py).
    // Not for short K: 8192^2 x 256 (4 K blocks) ran 79.9 us on the pair
    // against 70.7 on the single-CTA 128 x 256 tiles.
    const bool two_sm = pair < 0 ? (BN == 256 && !(c.flags & TB_FLAG_NO_2SM) && 8 * pair_tiles >= 3 * sms &&
                                    (p.k + HG_BK - 1) / HG_BK >= 8)
                                 : pair >= 1;
    // The 256 x 512 pair tile (a quarter less L2 traffic, which under the
    // power cap buys clock) above ~6 TFLOP — 32768^3 51.1-51.8 ms against
    // 54.9-55.5 ms, interleaved A/B runs — and for long K wherever its tile
    // waves cost no more than the 256 x 256 ones (ceil(tiles / pairs) x N):
    // idle-start ABBA blocks (tools/pair512_probe.py) 8192^3 686.0 against
    // 700.4 us, 10240^3 1374 / 1424, 12288^3 2416 / 2527; at K <= 6144 the
    // tile's exposed prologue / epilogue ate the gain (6144^3 283.4 / 282.5,
    // 3072^3 49.1 / 47.1).
    const int64_t wide_tiles = ((p.m + 255) / 256) * ((p.n + 511) / 512) * p.batch;
    const int64_t pairs = sms / 2 > 0 ? sms / 2 : 1;
    const bool wide_fits = 2 * ((wide_tiles + pairs - 1) / pairs) <= (pair_tiles + pairs - 1) / pairs;
    const bool wide = two_sm && (pair == 2 || (pair < 0 && (huge || (p.k >= 7168 && wide_fits))));
    // The wave barrier also on the 256 x 512 tile from 4 waves of it: 8192^3
    // 679.9 against 684.0 us (idle-start ABBA blocks, tools/pair512_probe.py
    // PAIR_WS=1).
    const bool sync_waves = two_sm && (huge || (c.flags & TB_FLAG_WAVE_SYNC) ||
                                       (wide && pair < 0 && wide_tiles >= 4 * pairs));
    const uint32_t bbox = two_sm ? 128 : BN;
    if (!bmn) rc = make_map(&tbm, B, p.k, p.n, p.batch, p.ldb, p.stride_b, 64, bbox);
    else rc = make_map(&tbm, B, p.n, p.k, p.batch, p.ldb, p.stride_b, 64, 64);
    if (rc != TB_OK) return rc;
    if (two_sm) {
      if (wide) {
        if (!amn && !bmn) return launch_h2<false, false, 512>(c, ta, tbm, sync_waves);
        if (!amn && bmn) return launch_h2<false, true, 512>(c, ta, tbm, sync_waves);
        if (amn && !bmn) return launch_h2<true, false, 512>(c, ta, tbm, sync_waves);
        return launch_h2<true, true, 512>(c, ta, tbm, sync_waves);
      }
      if (!amn && !bmn) return launch_h2<false, false>(c, ta, tbm, sync_waves);
      if (!amn && bmn) return launch_h2<false, true>(c, ta, tbm, sync_waves);
      if (amn && !bmn) return launch_h2<true, false>(c, ta, tbm, sync_waves);
      return launch_h2<true, true>(c, ta, tbm, sync_waves);
    }
    return launch_hg_tma_stages<BN>(c, ta, tbm);
  }
  // the pair kernel is TMA-only: unaligned operands take the LDG producer
  if (hgemm_aligned(c)) return launch_hg_layout<BN, false, true>(c, ta, tbm);
  return launch_hg_layout<BN, false, false>(c, ta, tbm);
}

// Split-K cluster size for H: a pure function of (m, n, k) and the SM count
// (never of batch or flags, so every H path of one shape issues the same
// per-element MMA / reduction sequence).  Doubles while the 128x128 tiles of
// one instance still leave half the SMs idle and each CTA keeps >= 16 K blocks
// (measured: 1024^3 with 8 K blocks per CTA was slower split than unsplit),
// and KS = 8 only while KS * tiles stays within a quarter of the SMs (512^2 x
// 16384, 16 tiles: KS 4 30.8 us against KS 8 36.8 — eight partials per tile
// cost more than the wider spread saves; 256^2 x 32768, 4 tiles: KS 8 30.8
// against KS 4 45.0).
int hgemm_split_ks(const Problem& p) {
  const int sms = sms_or_default();
  const int64_t t1 = ((p.m + HG_BM - 1) / HG_BM) * ((p.n + SK_BN - 1) / SK_BN);
  const int64_t nkb = (p.k + HG_BK - 1) / HG_BK;
  int ks = 1;
  while (ks < 8 && t1 * ks * 2 <= sms && nkb >= 32 * ks && (ks < 4 || 4 * t1 * ks <= sms)) ks *= 2;
  return ks;
}

template <bool TMA, bool AMN, bool BMN, bool VEC, bool CONV = false>
int launch_hsk(const Call& c, const CUtensorMap& ta, const CUtensorMap& tbm, int ks) {
  using Cfg = SkCfg<TMA>;
  const Problem& p = c.p;
  const int tiles_m = static_cast<int>((p.m + HG_BM - 1) / HG_BM);
  const int tiles_n = static_cast<int>((p.n + SK_BN - 1) / SK_BN);
  const int64_t total = static_cast<int64_t>(tiles_m) * tiles_n * p.batch;
  auto kern = hgemm_tc_splitk_kernel<TMA, AMN, BMN, VEC, CONV>;
  static SmemAttr attr;
  if (int rc = ensure_smem(attr, kern, Cfg::SMEM_BYTES)) return rc;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute la[1];
  la[0].id = cudaLaunchAttributeClusterDimension;
  la[0].val.clusterDim.x = static_cast<unsigned>(ks);
  la[0].val.clusterDim.y = 1;
  la[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(Cfg::THREADS);
  cfg.dynamicSmemBytes = Cfg::SMEM_BYTES;
  cfg.stream = c.stream;
  cfg.attrs = la;
  cfg.numAttrs = 1;
  // Co-resident clusters only (clusters are placed within a GPC): the
  // persistent loop then covers every tile without a second wave.
  static int max_clusters[64][9] = {{0}};
  const int dev = current_device();
  if (max_clusters[dev][ks] == 0) {
    int v = 0;
    cfg.gridDim = dim3(static_cast<unsigned>(ks));
    if (cudaOccupancyMaxActiveClusters(&v, kern, &cfg) != cudaSuccess || v < 1) {
      cudaGetLastError();
      v = sms_or_default() / ks;
    }
    max_clusters[dev][ks] = v;
  }
  const int64_t clusters = total < max_clusters[dev][ks] ? total : max_clusters[dev][ks];
  cfg.gridDim = dim3(static_cast<unsigned>(clusters * ks));
  // partials through L2 when a workspace is available (sized for a grid of
  // up to the SM count, so one allocation per stream serves every shape)
  float* ws = static_cast<float*>(
      splitk_workspace(c.stream, static_cast<size_t>(sms_or_default()) * SK_WS_FLOATS * sizeof(float)));
  if (cfg.gridDim.x > static_cast<unsigned>(sms_or_default())) ws = nullptr;
  const ConvGeom geom = c.conv ? *c.conv : ConvGeom{};
  if (int rc = launch_ex("hgemm_tc_splitk launch", kern, cfg.gridDim, cfg.blockDim, Cfg::SMEM_BYTES, c.stream, ks, ta,
                         tbm, p, tiles_m, tiles_n, cfg_group_m(c, 16), total, ws, geom))
    return rc;
  char name[64];
  snprintf(name, sizeof(name), "hgemm_tc_splitk%d_%s_128x128_%c%c%s%s", ks, CONV ? "conv" : (TMA ? "tma" : "ldg"),
           AMN ? 'm' : 'k',
           BMN ? 'n' : 'k', (!TMA && !VEC) ? "_scalar" : "", ws ? "" : "_dsmem");
  record(name, cfg.gridDim, cfg.blockDim, ks, Cfg::SMEM_BYTES, total);
  return check_launch("hgemm_tc_splitk launch");
}

template <bool TMA, bool VEC>
int launch_hsk_layout(const Call& c, const CUtensorMap& ta, const CUtensorMap& tbm, int ks) {
  const bool amn = !c.p.a_kcontig, bmn = c.p.b_ncontig;
  if (!amn && !bmn) return launch_hsk<TMA, false, false, VEC>(c, ta, tbm, ks);
  if (!amn && bmn) return launch_hsk<TMA, false, true, VEC>(c, ta, tbm, ks);
  if (amn && !bmn) return launch_hsk<TMA, true, false, VEC>(c, ta, tbm, ks);
  return launch_hsk<TMA, true, true, VEC>(c, ta, tbm, ks);
}

int dispatch_hsplit(const Call& c, int ks) {
  const Problem& p = c.p;
  // every CTA of a cluster needs at least one K block of its own
  const int64_t nkb = (p.k + HG_BK - 1) / HG_BK;
  while (ks > 1 && nkb < ks) ks /= 2;
  if (ks < 2) return -1;
  const bool amn = !p.a_kcontig, bmn = p.b_ncontig;
  CUtensorMap ta, tbm;
  memset(&ta, 0, sizeof(ta));
  memset(&tbm, 0, sizeof(tbm));
  if (tma_ok(c)) {
    const __half* A = static_cast<const __half*>(p.a) + p.a_off;
    const __half* B = static_cast<const __half*>(p.b) + p.b_off;
    int rc;
    if (!amn) rc = make_map(&ta, A, p.k, p.m, p.batch, p.lda, p.stride_a, 64, 128);
    else rc = make_map(&ta, A, p.m, p.k, p.batch, p.lda, p.stride_a, 64, 64);
    if (rc != TB_OK) return rc;
    if (!bmn) rc = make_map(&tbm, B, p.k, p.n, p.batch, p.ldb, p.stride_b, 64, SK_BN);
    else rc = make_map(&tbm, B, p.n, p.k, p.batch, p.ldb, p.stride_b, 64, 64);
    if (rc != TB_OK) return rc;
    return launch_hsk_layout<true, true>(c, ta, tbm, ks);
  }
  if (hgemm_aligned(c)) return launch_hsk_layout<false, true>(c, ta, tbm, ks);
  return launch_hsk_layout<false, false>(c, ta, tbm, ks);
}

}  // namespace

// Implicit GEMM (tb_convgemm): op(A) gathered from the image by the LDG
// producer warps (conv_fill_tile), op(B) = the filters (K-contiguous rows),
// UMMA N narrowed while the tiles leave SMs idle, as for a GEMM.
int dispatch_hconv(const Call& c) {
  const Problem& p = c.p;
  CUtensorMap none;
  memset(&none, 0, sizeof(none));
  // Few tiles in the launch (the typical layer, one image: 3136 positions x
  // 64 filters = 25 tiles): split K over a cluster so more SMs gather — the
  // gather is latency-bound per stage.  KS = largest power of two <= 8 with
  // tiles * KS <= SMs and >= 4 K blocks per rank pair, over ALL images of the
  // call (a batch of 32 images has parallelism enough and is not split:
  // measured 465 vs 275 us split / unsplit), so for H the last bits of an
  // image's result can depend on how many images share the call.
  {
    const int sms = sms_or_default();
    const int64_t t1 = ((p.m + HG_BM - 1) / HG_BM) * ((p.n + SK_BN - 1) / SK_BN) * p.batch;
    const int64_t nkb = (p.k + HG_BK - 1) / HG_BK;
    int ks = 1;
    while (ks < 8 && t1 * ks * 2 <= sms && nkb >= 4 * ks) ks *= 2;
    const bool vecb = (p.ldb % 8 == 0) && aligned_elems(p.b, p.b_off, 2, 16);
    if (ks > 1) {
      if (vecb) return launch_hsk<false, true, false, true, true>(c, none, none, ks);
      return launch_hsk<false, true, false, false, true>(c, none, none, ks);
    }
  }
  const bool vec = (p.ldb % 8 == 0) && aligned_elems(p.b, p.b_off, 2, 16);
  auto tiles = [&](int b) { return ((p.m + HG_BM - 1) / HG_BM) * ((p.n + b - 1) / b) * p.batch; };
  const int sms = sms_or_default();
  int bn = 256;
  while (bn > 64 && tiles(bn) < sms) bn /= 2;
  if (vec) {
    if (bn == 256) return launch_hg<256, false, true, false, true, 0, true>(c, none, none);
    if (bn == 128) return launch_hg<128, false, true, false, true, 0, true>(c, none, none);
    return launch_hg<64, false, true, false, true, 0, true>(c, none, none);
  }
  if (bn == 256) return launch_hg<256, false, true, false, false, 0, true>(c, none, none);
  if (bn == 128) return launch_hg<128, false, true, false, false, 0, true>(c, none, none);
  return launch_hg<64, false, true, false, false, 0, true>(c, none, none);
}

// ---- Unaligned operands: repack, then the TMA path ---------------------------
// (tbgemm.cu repack_operands).  2500^3: 1165 us on the LDG producers, 97 us
// repacked.
int hgemm_repacked(const Call& c) {
  if (c.flags & TB_FLAG_NO_TMA) return -1;
  Call c2 = c;
  int launches = 0;
  const int rc = repack_operands(c, 2, c2, launches);
  if (rc != TB_OK) return rc;
  const int rc2 = dispatch_hgemm(c2);
  if (rc2 == TB_OK) note_extra_launches(launches, "+pack");
  return rc2;
}

int dispatch_hgemm(const Call& c) {
  // Small instances (m, n <= 64): packed tcgen05 kernel.  Bitwise identical to
  // the general kernel (same per-element K sequence), so this is a pure
  // function of the shape and single / batched calls stay consistent.
  if (c.p.m <= 64 && c.p.n <= 64 && !(c.flags & TB_FLAG_NO_PACK)) return dispatch_hsmall_any(c);
  if (c.flags & TB_FLAG_TF32) {
    snprintf(err_buf(), 256, "TF32 flag applies to SGEMM only");
    return TB_ERR_UNSUPPORTED;
  }
  const Problem& p = c.p;
  // Unaligned operands: repack once and take the TMA kernels (falls through
  // to the LDG producers when no scratch can be had, e.g. during capture).
  if (!hgemm_aligned(c) && !p.a_offs && !p.b_offs && !(c.flags & TB_FLAG_NO_TMA)) {
    const int rc = hgemm_repacked(c);
    if (rc >= 0) return rc;
  }
  const tb_gemm_config* g = c.cfg;
  if (g && g->MWG > 0) {
    // A "gemm_b200" configuration (override / tuning DB): split-K cluster,
    // CTA pair, or single CTA with UMMA N = NWG.
    if (g->SPLIT_K > 1) {
      const int rc = dispatch_hsplit(c, g->SPLIT_K > 8 ? 8 : g->SPLIT_K);
      if (rc >= 0) return rc;
    }
    if (g->CTA_GROUP == 2 && tma_ok(c)) return dispatch_hgemm_bn<256>(c, g->NWG >= 512 ? 2 : 1);
    if (g->NWG >= 256) return dispatch_hgemm_bn<256>(c, 0);
    if (g->NWG >= 128) return dispatch_hgemm_bn<128>(c, 0);
    return dispatch_hgemm_bn<64>(c, 0);
  }
  // Few output tiles and a long K: split K across a cluster (DSMEM reduction).
  if (const int ks = hgemm_split_ks(p); ks > 1 && !(c.flags & TB_FLAG_NO_SPLITK)) {
    const int rc = dispatch_hsplit(c, ks);
    if (rc >= 0) return rc;
  }
  // Fewer 128 x 256 tiles than SMs: narrow the UMMA N extent when that
  // reduces the tile-waves of work, waves(BN) * BN, ties to the wider tile
  // (results are independent of it — tests/test_gemm_gpu.py).  2048^3: 128
  // tiles of 128 x 256 in one wave, 24.5 us, against 256 tiles of 128 x 128
  // in 1.7 waves, 28.7 us (the earlier "narrow while tiles < SMs" rule);
  // 1536^2 x 4096: 128 x 128 28.7 us against 128 x 64 43.0 us; 1024^3 keeps
  // 128 x 64 (one wave of 128 tiles).  With at least a wave of wide tiles
  // the wide (or CTA-pair) kernel stays: its tiles are the efficient ones.
  const int sms = sms_or_default();
  auto tiles = [&](int b) { return ((p.m + HG_BM - 1) / HG_BM) * ((p.n + b - 1) / b) * p.batch; };
  auto cost = [&](int b) { return ((tiles(b) + sms - 1) / sms) * b; };
  // Batched instances too (their N extent is often narrow: 96^3 x 2048
  // 37.2 us on 128 x 256 against 28.7 on 128 x 128, 384^3 x 64 23.6 -> 20.5);
  // for them only a clear gain (15 %) narrows the tile (200^3 x 256: 22.5 us
  // on 128 x 256, 26.7 on 128 x 128 at a 12.5 % smaller wave count).
  int bn = 256;
  if (tiles(256) < sms)
    for (int b = 128; b >= 64; b /= 2)
      if (cost(b) < cost(bn)) bn = b;
  if (tiles(256) >= sms && p.batch > 1)
    for (int b = 128; b >= 64; b /= 2)
      if (20 * cost(b) < 17 * cost(bn)) bn = b;
  if (bn == 256) return dispatch_hgemm_bn<256>(c, -1);
  if (bn == 128) return dispatch_hgemm_bn<128>(c, -1);
  return dispatch_hgemm_bn<64>(c, -1);
}

int launch_hscale(const Call& c) {
  dim3 block(256);
  const int64_t total = c.p.m * c.p.n;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  if (blocks < 1) blocks = 1;
  dim3 grid(static_cast<unsigned>(blocks));
  if (int rc = launch_ex("hscale launch", hscale_kernel<0>, grid, block, 0, c.stream, 1, c.p)) return rc;
  record("hscale", grid, block, 1, 0, c.p.batch);
  return check_launch("hscale launch");
}

}  // namespace host
}  // namespace tb

#ifdef TB_SPLITK_TIMING
// Debug builds only (tools/splitk_timeline.py): copy the split-K kernel's
// per-CTA %globaltimer stamps to the host.
extern "C" int tb_debug_splitk_times(unsigned long long* host, int count) {
  return cudaMemcpyFromSymbol(host, tb::tb_sk_times, sizeof(unsigned long long) * count) == cudaSuccess ? 0 : 1;
}
#endif
