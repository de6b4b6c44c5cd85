// sgemm_tma.cu — launch + tile routing of the TMA-fed FFMA2 SGEMM
// (sgemm_tma.cuh).  M/N-contiguous operands: box {ROWS, 32} without swizzle;
// K-contiguous: box {32, ROWS} SWIZZLE_128B.
#include <cstring>

#include "host.h"
#include "sgemm_tma.cuh"

namespace tb {
namespace host {
namespace {

template <int BM, int BN, int TM, int TN, int ST, bool AMN, bool BMN, bool XP = false, int MINB = 2, int KS = 1>
int launch_stma(const Call& c) {
  using Cfg = TmaSgemmCfg<BM, BN, 32, TM, TN, ST, AMN, BMN, XP>;
  const Problem& p = c.p;
  const float* A = static_cast<const float*>(p.a) + p.a_off;
  const float* B = static_cast<const float*>(p.b) + p.b_off;
  const CUtensorMapDataType F32 = CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  CUtensorMap ta, tbm;
  memset(&ta, 0, sizeof(ta));
  memset(&tbm, 0, sizeof(tbm));
  int rc = AMN ? make_map(&ta, A, p.m, p.k, p.batch, p.lda, p.stride_a, BM, 32, F32, 4, CU_TENSOR_MAP_SWIZZLE_NONE)
               : make_map(&ta, A, p.k, p.m, p.batch, p.lda, p.stride_a, 32, BM, F32, 4, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc != TB_OK) return rc;
  rc = BMN ? make_map(&tbm, B, p.n, p.k, p.batch, p.ldb, p.stride_b, BN, 32, F32, 4, CU_TENSOR_MAP_SWIZZLE_NONE)
           : make_map(&tbm, B, p.k, p.n, p.batch, p.ldb, p.stride_b, 32, BN, F32, 4, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc != TB_OK) return rc;
  const int tiles_m = static_cast<int>((p.m + BM - 1) / BM);
  const int tiles_n = static_cast<int>((p.n + BN - 1) / BN);
  const int64_t blocks = static_cast<int64_t>(tiles_m) * tiles_n * p.batch;
  if (blocks > 0x7fffffffLL) return TB_ERR_INVALID;
  if (blocks * KS > 0x7fffffffLL) return TB_ERR_INVALID;
  auto kern = sgemm_tma_kernel<BM, BN, 32, TM, TN, ST, AMN, BMN, MINB, XP, KS>;
  static SmemAttr attr;  // per instantiation, per device
  if (int rc2 = ensure_smem(attr, kern, Cfg::SMEM_BYTES)) return rc2;
  dim3 grid(static_cast<unsigned>(blocks * KS)), block(Cfg::NT);
  if (int rc2 = launch_ex("sgemm_tma launch", kern, grid, block, Cfg::SMEM_BYTES, c.stream, KS, ta, tbm, p, tiles_m,
                          tiles_n, cfg_group_m(c, 8)))
    return rc2;
  char name[64];
  snprintf(name, sizeof(name), "sgemm_tma_%dx%dx32_%dx%d_%c%c%s%s", BM, BN, TM, TN, AMN ? 'm' : 'k',
           BMN ? 'n' : 'k', (Cfg::A_T || Cfg::B_T) ? "_xp" : "", KS == 2 ? "_splitk2" : (KS == 4 ? "_splitk4" : ""));
  record(name, grid, block, KS, Cfg::SMEM_BYTES, blocks);
  return check_launch("sgemm_tma launch");
}

// Tile families by operand major-ness (a: A M-contiguous, b: B N-contiguous).
int big_tiles(const Call& c, bool amn, bool bmn) {
  // K-contiguous operands are transposed in shared memory (XP) so every
  // layout runs the M/N-contiguous fragment loop: 8192^3 row-major NN
  // 59.8 -> 63.9, K-contiguous A 58.9 -> 64.5, both 56.7 -> 58.9 TFLOP/s
  // (both K-contiguous on the 128 x 128 / 16 x 8 tile: 18.6 -> 24.4 ms at
  // 8192^3 — two transposed operands per stage; not used)
  if (amn && bmn) return launch_stma<64, 128, 8, 8, 4, true, true>(c);
  if (amn) return launch_stma<128, 128, 16, 8, 2, true, false, true>(c);
  if (bmn) return launch_stma<64, 128, 8, 8, 2, false, true, true>(c);
  return launch_stma<64, 128, 8, 8, 2, false, false, true>(c);
}
// Deterministic split-K for the 128x64 tile (clusters of KS CTAs, DSMEM
// reduction in rank order; sgemm_tma.cuh).  KS is a pure function of the
// per-instance shape (m, n, k) and the SM count — never of the batch — so
// single, batched and looped calls agree bitwise.  Only shapes whose 128x64
// tiles fill at most half the SMs split; among KS in {1, 2, 4} (each rank
// keeping >= 16 K stages: shorter chains are fixed-cost bound — C3b (64,
// 3136, 576), 18 stages, ran 26.5 us split in two against 18.4 us on the
// unsplit 64x32 tiles) the one with the fewest waves of work per SM,
// ceil(tiles * KS / SMs) / KS, wins, ties going to the smaller KS (one CTA
// per SM beats two sharing it).  Measured (tools/route_probe.py, L2 flushed):
// C3 (4096, 128, 9216), 64 tiles: KS 2 215 us / KS 4 223 us / unsplit 265;
// (768, 768, 2048), 72 tiles: KS 2 59.5 / KS 4 90.2; (512, 512, 4096), 32
// tiles: KS 4 63.5 / unsplit 88.0; (300, 520, 4096), 25 tiles: KS 4 63.5 /
// KS 2 102.4 / unsplit 86.1; C1 (1024^3, 128 tiles) ties and stays unsplit
// (split in two measured 59.4 against 55.8 us).
// Returns 1 when K is not split.
int sgemm_split_ks(const Problem& p, int bm = 128, int bn = 64, int per_sm = 1) {
  // per_sm: CTAs of the tile resident per SM (the 64x32 tiles run several)
  const int sms = sms_or_default() * per_sm;
  const int64_t t1 = ((p.m + bm - 1) / bm) * ((p.n + bn - 1) / bn);
  const int64_t ktiles = (p.k + 31) / 32;
  if (2 * t1 > sms) return 1;
  int best = 1;
  int64_t best_waves = (t1 + sms - 1) / sms;  // cost = waves / ks, compared as fractions
  for (int ks = 2; ks <= 4; ks *= 2) {
    if (ktiles < 16 * ks) break;
    const int64_t waves = (t1 * ks + sms - 1) / sms;
    if (waves * best < best_waves * ks) {
      best = ks;
      best_waves = waves;
    }
  }
  return best;
}

template <int KS>
int tiles_128x64_split(const Call& c, bool amn, bool bmn) {
  if (amn && bmn) return launch_stma<128, 64, 4, 8, 4, true, true, false, 2, KS>(c);
  if (amn) return launch_stma<128, 64, 4, 8, 4, true, false, false, 2, KS>(c);
  if (bmn) return launch_stma<128, 64, 4, 8, 4, false, true, false, 2, KS>(c);
  return -1;
}

int tiles_128x64(const Call& c, bool amn, bool bmn) {
  if (amn && bmn) return launch_stma<128, 64, 4, 8, 4, true, true>(c);
  if (amn) return launch_stma<128, 64, 4, 8, 4, true, false>(c);
  if (bmn) return launch_stma<128, 64, 4, 8, 4, false, true>(c);
  return -1;  // both K-contiguous: not instantiated (measured slower)
}
int tiles_64x64(const Call& c, bool amn, bool bmn) {
  if (amn && bmn) return launch_stma<64, 64, 4, 8, 3, true, true>(c);
  if (amn) return launch_stma<64, 64, 4, 8, 3, true, false>(c);
  if (bmn) return launch_stma<64, 64, 8, 4, 4, false, true>(c);
  return launch_stma<64, 64, 4, 8, 3, false, false>(c);
}
int tiles_64x32(const Call& c, bool amn, bool bmn) {
  if (amn && bmn) return launch_stma<64, 32, 4, 4, 3, true, true>(c);
  if (amn) return launch_stma<64, 32, 4, 4, 3, true, false>(c);
  if (bmn) return launch_stma<64, 32, 4, 4, 3, false, true>(c);
  return launch_stma<64, 32, 4, 4, 3, false, false>(c);
}
template <int KS>
int tiles_64x32_split(const Call& c, bool amn, bool bmn) {
  if (amn && bmn) return launch_stma<64, 32, 4, 4, 3, true, true, false, 2, KS>(c);
  if (amn) return launch_stma<64, 32, 4, 4, 3, true, false, false, 2, KS>(c);
  if (bmn) return launch_stma<64, 32, 4, 4, 3, false, true, false, 2, KS>(c);
  return launch_stma<64, 32, 4, 4, 3, false, false, false, 2, KS>(c);
}
int tiles_32x32(const Call& c, bool amn, bool bmn) {
  // k <= 32 is a single K block: one ring slot and a 51-register cap, so 20
  // CTAs per SM fit (2 slots at 92 registers: 10; 49.0 -> 44.3 us at S32;
  // a 42-register cap, 24 CTAs, spills: 47.0 us)
  if (c.p.k <= 32) {
    if (amn && bmn) return launch_stma<32, 32, 4, 4, 1, true, true, false, 20>(c);
    if (amn) return launch_stma<32, 32, 4, 4, 1, true, false, false, 20>(c);
    if (bmn) return launch_stma<32, 32, 4, 4, 1, false, true, true, 20>(c);
    return launch_stma<32, 32, 4, 4, 1, false, false, true, 20>(c);
  }
  if (amn && bmn) return launch_stma<32, 32, 4, 4, 2, true, true>(c);
  if (amn) return launch_stma<32, 32, 4, 4, 2, true, false>(c);
  if (bmn) return launch_stma<32, 32, 4, 4, 2, false, true, true>(c);
  return launch_stma<32, 32, 4, 4, 2, false, false, true>(c);
}

}  // namespace

// Route to the TMA kernel: returns -1 when the problem does not qualify.
// tile: 0 = by shape (built-in routing), 2 = one 64x64 tile per instance
// (batched 33..64), 3 = one 32x32 tile per instance (batched <= 32),
// -1 = the configuration's MWG x NWG.
int dispatch_sgemm_tma(const Call& c, int tile, int mwg, int nwg, int ks) {
  const Problem& p = c.p;
  const bool amn = !p.a_kcontig, bmn = p.b_ncontig;
  if (p.a_offs || p.b_offs || p.alphas || p.betas || p.k <= 0 || p.alpha == 0.0f) return -1;
  if ((p.lda % 4) || (p.ldb % 4) || !aligned_elems(p.a, p.a_off, 4, 16) || !aligned_elems(p.b, p.b_off, 4, 16))
    return -1;
  if (p.batch > 1 && ((p.stride_a % 4) || (p.stride_b % 4))) return -1;
  if (p.m > 0x7fffff00LL || p.n > 0x7fffff00LL || p.k > 0x7fffff00LL || p.batch > 0x7fffffffLL) return -1;
  if (tile == -1) {
    if (ks == 2 || ks == 4) {  // configured deterministic split-K (instantiated tiles only)
      if (mwg == 128 && nwg == 64)
        return ks == 2 ? tiles_128x64_split<2>(c, amn, bmn) : tiles_128x64_split<4>(c, amn, bmn);
      if (mwg == 64 && nwg == 32)
        return ks == 2 ? tiles_64x32_split<2>(c, amn, bmn) : tiles_64x32_split<4>(c, amn, bmn);
    }
    if (mwg >= 128 && nwg >= 128) return big_tiles(c, amn, bmn);
    if (mwg >= 128 && nwg == 64) return tiles_128x64(c, amn, bmn);
    if (mwg == 64 && nwg == 64) return tiles_64x64(c, amn, bmn);
    if (mwg == 64 && nwg == 32) return tiles_64x32(c, amn, bmn);
    if (mwg == 32 && nwg == 32) return tiles_32x32(c, amn, bmn);
    if (mwg == 64 && nwg >= 128) return big_tiles(c, amn, bmn);
    return -1;
  }
  if (tile == 3) return tiles_32x32(c, amn, bmn);
  if (tile == 0 && !(c.flags & TB_FLAG_NO_SPLITK)) {
    // the 128x64 split kernel needs an M- or N-contiguous operand
    const int ks = (amn || bmn) ? sgemm_split_ks(p) : 1;
    // Still fewer than half the SMs busy: the 64x32 tiles (four times as
    // many, every layout) split by the same rule — 128^2 x 65536: 325.6 us
    // against 733.2 on the 128x64 split, 256^2 x 32768: 169.8 against 385.1,
    // both-K-contiguous 512^2 x 16384: 276 against 412 unsplit.
    const int64_t t1 = ((p.m + 127) / 128) * ((p.n + 63) / 64);
    if (2 * t1 * ks < sms_or_default()) {
      const int ks32 = sgemm_split_ks(p, 64, 32, 4);
      const int64_t t32 = ((p.m + 63) / 64) * ((p.n + 31) / 32);
      if (ks32 > 1 && t32 * ks32 > t1 * ks) {  // unsplit: the routing below (it sees the batch)
        if (ks32 == 2) return tiles_64x32_split<2>(c, amn, bmn);
        return tiles_64x32_split<4>(c, amn, bmn);
      }
    }
    if (ks == 2) return tiles_128x64_split<2>(c, amn, bmn);
    if (ks == 4) return tiles_128x64_split<4>(c, amn, bmn);
  }
  const int sms = sms_or_default();
  // Batched instances up to 512 x 512: the tile that pads an instance least,
  // ties to 64x64, then 128x64, then 32x32 (tools/route_audit.py --batched:
  // 96^3 x 2048 on 32x32 94 us, 128^3 x 1024 and 256^3 x 256 on 64x64 100
  // and 180 us, 200^3 x 256 on 32x32 129 us — the big tiles, picked by tile
  // count alone, ran 125-196 us there).
  if (tile == 0 && p.batch > 1 && p.m <= 512 && p.n <= 512 && !(p.m <= 64 && p.n <= 64)) {
    auto padded = [&](int bm, int bn) { return ((p.m + bm - 1) / bm * bm) * ((p.n + bn - 1) / bn * bn); };
    const int64_t w64 = padded(64, 64), w128 = padded(128, 64), w32 = padded(32, 32);
    if (w64 <= w128 && w64 <= w32) return tiles_64x64(c, amn, bmn);
    if ((amn || bmn) && w128 <= w32) return tiles_128x64(c, amn, bmn);
    return tiles_32x32(c, amn, bmn);
  }
  const int64_t tiles128 = ((p.m + 127) / 128) * ((p.n + 127) / 128) * p.batch;
  // Measured on B200 (tools/sgemm_ms_bench.cu): with >= 4 waves of 128x128
  // tiles the big tiles win (64x128 8x8 when both operands are M/N-contiguous:
  // 66 TFLOP/s at 8192^3); below that 64x64 tiles of 4x8 (8x4) micro-tiles
  // keep every SM busy (1024^3 37.6, C3 (4096,128,9216) 34.8 TFLOP/s).
  const bool one_tile = p.m <= 64 && p.n <= 64;  // batched small instances: one 64x64 tile each
  // (3.5 waves and more: 3072^3 1028 us big tiles against 1091 on 64x64)
  if (tile == 0 && 2 * tiles128 >= 7 * sms && !one_tile) return big_tiles(c, amn, bmn);
  // K-contiguous A (its tiles are transposed in shared memory either way):
  // the 64x128 8x8 transposing tiles from one wave of them — 1536^3 NT
  // 149.5 us against 172.9 on 64x64, 4096x512x4096 NT 374.7 against 438.5
  // (tools/route_audit.py --trans=nt)
  const int64_t tiles64x128 = ((p.m + 63) / 64) * ((p.n + 127) / 128) * p.batch;
  if (tile == 0 && !amn && !one_tile && tiles64x128 >= sms) return big_tiles(c, amn, bmn);
  // fewer 64x64 tiles than SMs (e.g. C3 (64, 3136, 576): 49 tiles): 64x32
  // tiles of 4x4 (21 -> 14 us there; tools/sgemm_ms_bench.cu)
  const int64_t tiles64 = ((p.m + 63) / 64) * ((p.n + 63) / 64) * p.batch;
  if (tile == 0 && tiles64 < sms) return tiles_64x32(c, amn, bmn);
  // at most 64 rows: 128-row tiles would be half empty (16384 x 64 x 2048
  // row-major: 64x64 tiles 110.7 us against 195.5 on 128x64)
  if (tile == 0 && p.m <= 64 && !one_tile) return tiles_64x64(c, amn, bmn);
  // 128x64 tiles that fill (nearly) whole waves of one tile per SM: 256
  // threads of 4x8 beat two 64x64 CTAs per SM by 3-7 % (tools/sgemm_ms_bench.cu:
  // 1024^3 56 -> 53 us, 1536^3 148 -> 143 us; both-K-contiguous layouts lose)
  const int64_t tiles128x64 = ((p.m + 127) / 128) * ((p.n + 63) / 64) * p.batch;
  const int64_t waves = (tiles128x64 + sms - 1) / sms;
  if (tile == 0 && !one_tile && (amn || bmn) && waves <= 2 && tiles128x64 * 20 >= waves * sms * 17)
    return tiles_128x64(c, amn, bmn);
  // batched instances of at most 64x64 with k <= 64 (two K blocks): a
  // two-slot ring and a 102-register cap, 5 CTAs per SM instead of 4
  if (one_tile && p.k <= 64) {
    if (amn && bmn) return launch_stma<64, 64, 4, 8, 2, true, true, false, 5>(c);
    if (amn) return launch_stma<64, 64, 4, 8, 2, true, false, false, 5>(c);
    if (bmn) return launch_stma<64, 64, 8, 4, 2, false, true, false, 5>(c);
    return launch_stma<64, 64, 4, 8, 2, false, false, false, 5>(c);
  }
  return tiles_64x64(c, amn, bmn);
}

}  // namespace host
}  // namespace tb
