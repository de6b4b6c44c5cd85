// tbgemm.cu — C-ABI entry points (include/tbgemm.h) and kernel dispatch.
//
// Host-side responsibilities (all argument *validation* happened in the
// Python routine layer, mirroring pkg/src/tunedblas/routines/level3.py:94-133
// and extras.py:188-348):
//   1. canonicalise layout/trans into one column-major problem (row-major C
//      is C^T col-major: swap A<->B and m<->n — common.py:1-7, level3.py:41-45);
//   2. map the 14 reference GemmParams (params.py:120-146) onto the nearest
//      sm_100a instantiation;
//   3. pick the producer (TMA when 16-byte alignment allows, LDG otherwise);
//   4. build TMA tensor maps (cuTensorMapEncodeTiled via the runtime's
//      driver entry point — no link-time libcuda dependency);
//   5. launch on the caller's stream and record a tb_launch_record.
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "hgemm_tc.cuh"
#include "hgemm_tc_small.cuh"
#include "hgemm_tc_2sm.cuh"
#include "hgemm_tc_splitk.cuh"
#include "im2col.cuh"
#include "structured.cuh"
#include "sgemm_tf32_tc.cuh"
#include "sgemm_simt.cuh"
#include "sgemm_small.cuh"
#include "sgemm_tma.cuh"
#include "tbgemm.h"

using namespace tb;

namespace {

thread_local tb_launch_record g_last{};
thread_local char g_last_err[256] = "";

void set_err(const char* what, cudaError_t e) {
  snprintf(g_last_err, sizeof(g_last_err), "%s: %s", what, cudaGetErrorString(e));
}

void record(const char* name, dim3 grid, dim3 block, int cluster, int smem, int64_t tiles) {
  memset(&g_last, 0, sizeof(g_last));
  snprintf(g_last.kernel, sizeof(g_last.kernel), "%s", name);
  g_last.grid[0] = grid.x; g_last.grid[1] = grid.y; g_last.grid[2] = grid.z;
  g_last.block[0] = block.x; g_last.block[1] = block.y; g_last.block[2] = block.z;
  g_last.cluster[0] = cluster; g_last.cluster[1] = 1; g_last.cluster[2] = 1;
  g_last.smem_bytes = smem;
  g_last.launches = 1;
  g_last.tiles = tiles;
}

int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (dev < 0 || dev >= 64) return 0;
  if (cached[dev] == 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
    cached[dev] = v;
  }
  return cached[dev];
}

// The dynamic shared-memory opt-in is a per-device function attribute.
struct SmemAttr {
  std::atomic<uint64_t> devs{0};
};

template <typename K>
int ensure_smem(SmemAttr& st, K kern, int bytes) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
  const uint64_t bit = 1ull << (dev & 63);
  if (st.devs.load(std::memory_order_acquire) & bit) return TB_OK;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) {
    set_err("cudaFuncSetAttribute", e);
    return TB_ERR_CUDA;
  }
  st.devs.fetch_or(bit, std::memory_order_acq_rel);
  return TB_OK;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_err(what, e);
    return TB_ERR_CUDA;
  }
  return TB_OK;
}

// ---------------------------------------------------------------------------
// Driver entry point for tensor maps
// ---------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                  CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                  CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess) {
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
    }
  });
  return fn;
}

// 3-D tensor map (FP16 or FP32): dims {contig, other, batch}, box {box0, box1, 1}, SW128 by default.
int make_map(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t batch, uint64_t ld,
             uint64_t stride, uint32_t box0, uint32_t box1,
             CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_FLOAT16, uint64_t es = 2,
             CUtensorMapSwizzle swizzle = CU_TENSOR_MAP_SWIZZLE_128B) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn) {
    snprintf(g_last_err, sizeof(g_last_err), "cuTensorMapEncodeTiled entry point unavailable");
    return TB_ERR_DRIVER;
  }
  cuuint64_t dims[3] = {d0, d1, batch};
  uint64_t zstride = stride * es;
  if (batch <= 1) zstride = ((ld * d1 * es) + 15) / 16 * 16;
  cuuint64_t strides[2] = {ld * es, zstride};
  cuuint32_t box[3] = {box0, box1, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, dt, 3, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    snprintf(g_last_err, sizeof(g_last_err), "cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
    return TB_ERR_DRIVER;
  }
  return TB_OK;
}

// ---------------------------------------------------------------------------
// Canonicalisation
// ---------------------------------------------------------------------------
struct Call {
  int prec, layout, ta, tbt;
  int64_t m, n, k;
  Problem p;
  int offs_aligned;  // generic batched: host-asserted offset alignment
  const tb_gemm_params* params;
  int flags;
  cudaStream_t stream;
};

void canonicalize(Call& c) {
  Problem& p = c.p;
  int ta = c.ta, tbt = c.tbt;
  if (c.layout == TB_ROW_MAJOR) {
    // C_row (m x n) == C^T col-major (n x m) = op(B)^T op(A)^T
    std::swap(p.a, p.b);
    std::swap(p.lda, p.ldb);
    std::swap(p.a_off, p.b_off);
    std::swap(p.stride_a, p.stride_b);
    std::swap(p.a_offs, p.b_offs);
    std::swap(ta, tbt);
    std::swap(c.m, c.n);
  }
  p.m = c.m;
  p.n = c.n;
  p.k = c.k;
  p.a_kcontig = (ta != TB_NO_TRANS) ? 1 : 0;
  p.b_ncontig = (tbt != TB_NO_TRANS) ? 1 : 0;
}

bool aligned_elems(const void* base, int64_t off, int64_t elem, int64_t vec_bytes) {
  return ((reinterpret_cast<uintptr_t>(base) + off * elem) % vec_bytes) == 0;
}

// ---------------------------------------------------------------------------
// SGEMM dispatch
// ---------------------------------------------------------------------------
template <int BM, int BN, int BK, int TM, int TN, bool VEC, int MINB>
int launch_simt(const Call& c, const char* tag) {
  const Problem& p = c.p;
  const int tiles_m = static_cast<int>((p.m + BM - 1) / BM);
  const int tiles_n = static_cast<int>((p.n + BN - 1) / BN);
  const int64_t blocks = static_cast<int64_t>(tiles_m) * tiles_n * p.batch;
  if (blocks > 0x7fffffffLL) return TB_ERR_INVALID;
  const int group_m = 8;
  dim3 grid(static_cast<unsigned>(blocks)), block(SimtShape<BM, BN, BK, TM, TN>::NT);
  const int sel = (p.a_kcontig ? 2 : 0) | (p.b_ncontig ? 1 : 0);
  switch (sel) {
    case 0: sgemm_simt_kernel<BM, BN, BK, TM, TN, false, false, VEC, MINB><<<grid, block, 0, c.stream>>>(p, tiles_m, tiles_n, group_m); break;
    case 1: sgemm_simt_kernel<BM, BN, BK, TM, TN, false, true, VEC, MINB><<<grid, block, 0, c.stream>>>(p, tiles_m, tiles_n, group_m); break;
    case 2: sgemm_simt_kernel<BM, BN, BK, TM, TN, true, false, VEC, MINB><<<grid, block, 0, c.stream>>>(p, tiles_m, tiles_n, group_m); break;
    default: sgemm_simt_kernel<BM, BN, BK, TM, TN, true, true, VEC, MINB><<<grid, block, 0, c.stream>>>(p, tiles_m, tiles_n, group_m); break;
  }
  char name[64];
  static const char* lay[4] = {"mk", "mn", "kk", "kn"};  // A major x B major
  snprintf(name, sizeof(name), "sgemm_simt_%dx%dx%d_%s_%s", BM, BN, BK, VEC ? "vec" : "gen", lay[sel]);
  (void)tag;
  record(name, grid, block, 1, 0, blocks);
  return check_launch("sgemm_simt launch");
}

// TMA-fed FFMA2 SGEMM (sgemm_tma.cuh).  M/N-contiguous operands: box
// {ROWS, 32} without swizzle; K-contiguous: box {32, ROWS} SWIZZLE_128B.
template <int BM, int BN, int TM, int TN, int ST, bool AMN, bool BMN, bool XP = false, int MINB = 2>
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
  auto kern = sgemm_tma_kernel<BM, BN, 32, TM, TN, ST, AMN, BMN, MINB, XP>;
  static SmemAttr attr;  // per instantiation, per device
  if (int rc2 = ensure_smem(attr, kern, Cfg::SMEM_BYTES)) return rc2;
  dim3 grid(static_cast<unsigned>(blocks)), block(Cfg::NT);
  kern<<<grid, block, Cfg::SMEM_BYTES, c.stream>>>(ta, tbm, p, tiles_m, tiles_n, 8);
  char name[64];
  snprintf(name, sizeof(name), "sgemm_tma_%dx%dx32_%dx%d_%c%c%s", BM, BN, TM, TN, AMN ? 'm' : 'k', BMN ? 'n' : 'k',
           (Cfg::A_T || Cfg::B_T) ? "_xp" : "");
  record(name, grid, block, 1, Cfg::SMEM_BYTES, blocks);
  return check_launch("sgemm_tma launch");
}

// Route to the TMA kernel: returns -1 when the problem does not qualify.
// tile: 0 = by shape (no tuned configuration), 1 = large tiles, 2 = 64x64.
int dispatch_sgemm_tma(const Call& c, int tile) {
  const Problem& p = c.p;
  const bool amn = !p.a_kcontig, bmn = p.b_ncontig;
  if (p.a_offs || p.b_offs || p.alphas || p.betas || p.k <= 0 || p.alpha == 0.0f) return -1;
  if ((p.lda % 4) || (p.ldb % 4) || !aligned_elems(p.a, p.a_off, 4, 16) || !aligned_elems(p.b, p.b_off, 4, 16))
    return -1;
  if (p.batch > 1 && ((p.stride_a % 4) || (p.stride_b % 4))) return -1;
  if (p.m > 0x7fffff00LL || p.n > 0x7fffff00LL || p.k > 0x7fffff00LL || p.batch > 0x7fffffffLL) return -1;
  const int sms = sm_count() > 0 ? sm_count() : 148;
  const int64_t tiles128 = ((p.m + 127) / 128) * ((p.n + 127) / 128) * p.batch;
  // Measured on B200 (tools/sgemm_ms_bench.cu): with >= 4 waves of 128x128
  // tiles the big tiles win (64x128 8x8 when both operands are M/N-contiguous:
  // 66 TFLOP/s at 8192^3); below that 64x64 tiles of 4x8 (8x4) micro-tiles
  // keep every SM busy (1024^3 37.6, C3 (4096,128,9216) 34.8 TFLOP/s).
  if (tile == 3) {
    // batched instances of at most 32x32: one 32x32 tile each, 64 threads of 4x4
    // k <= 32 is a single K block: one ring slot and a 51-register cap, so 20
    // CTAs per SM fit (2 slots at 92 registers: 10; 49.0 -> 44.3 us at S32;
    // a 42-register cap, 24 CTAs, spills: 47.0 us)
    if (p.k <= 32) {
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
  const bool one_tile = p.m <= 64 && p.n <= 64;  // batched small instances: one 64x64 tile each
  const bool big = tile == 0 ? tiles128 >= 4 * sms : tile == 1;
  if (big && !one_tile) {
    // K-contiguous operands are transposed in shared memory (XP) so every
    // layout runs the M/N-contiguous fragment loop: 8192^3 row-major NN
    // 59.8 -> 63.9, K-contiguous A 58.9 -> 64.5, both 56.7 -> 58.9 TFLOP/s
    if (amn && bmn) return launch_stma<64, 128, 8, 8, 4, true, true>(c);
    if (amn) return launch_stma<128, 128, 16, 8, 2, true, false, true>(c);
    if (bmn) return launch_stma<64, 128, 8, 8, 2, false, true, true>(c);
    return launch_stma<64, 128, 8, 8, 2, false, false, true>(c);
  }
  // fewer 64x64 tiles than SMs (e.g. C3 (64, 3136, 576): 49 tiles): 64x32
  // tiles of 4x4 (21 -> 14 us there; tools/sgemm_ms_bench.cu)
  const int64_t tiles64 = ((p.m + 63) / 64) * ((p.n + 63) / 64) * p.batch;
  if (tile == 0 && tiles64 < sms) {
    if (amn && bmn) return launch_stma<64, 32, 4, 4, 3, true, true>(c);
    if (amn) return launch_stma<64, 32, 4, 4, 3, true, false>(c);
    if (bmn) return launch_stma<64, 32, 4, 4, 3, false, true>(c);
    return launch_stma<64, 32, 4, 4, 3, false, false>(c);
  }
  // 128x64 tiles that fill (nearly) whole waves of one tile per SM: 256
  // threads of 4x8 beat two 64x64 CTAs per SM by 3-7 % (tools/sgemm_ms_bench.cu:
  // 1024^3 56 -> 53 us, 1536^3 148 -> 143 us; both-K-contiguous layouts lose)
  const int64_t tiles128x64 = ((p.m + 127) / 128) * ((p.n + 63) / 64) * p.batch;
  const int64_t waves = (tiles128x64 + sms - 1) / sms;
  if (tile == 0 && !one_tile && (amn || bmn) && waves <= 2 && tiles128x64 * 20 >= waves * sms * 17) {
    if (amn && bmn) return launch_stma<128, 64, 4, 8, 4, true, true>(c);
    if (amn) return launch_stma<128, 64, 4, 8, 4, true, false>(c);
    return launch_stma<128, 64, 4, 8, 4, false, true>(c);
  }
  // batched instances of at most 64x64 with k <= 64 (two K blocks): a
  // two-slot ring and a 102-register cap, 5 CTAs per SM instead of 4
  if (one_tile && p.k <= 64) {
    if (amn && bmn) return launch_stma<64, 64, 4, 8, 2, true, true, false, 5>(c);
    if (amn) return launch_stma<64, 64, 4, 8, 2, true, false, false, 5>(c);
    if (bmn) return launch_stma<64, 64, 8, 4, 2, false, true, false, 5>(c);
    return launch_stma<64, 64, 4, 8, 2, false, false, false, 5>(c);
  }
  if (amn && bmn) return launch_stma<64, 64, 4, 8, 3, true, true>(c);
  if (amn) return launch_stma<64, 64, 4, 8, 3, true, false>(c);
  if (bmn) return launch_stma<64, 64, 8, 4, 4, false, true>(c);
  return launch_stma<64, 64, 4, 8, 3, false, false>(c);
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
  const int sms = sm_count() > 0 ? sm_count() : 148;
  const int64_t cap = static_cast<int64_t>(sms) * per_sm;
  const int64_t g = groups < cap ? groups : cap;
  dim3 grid(static_cast<unsigned>(g)), block(256);
  kern<<<grid, block, Cfg::SMEM_BYTES, c.stream>>>(p, groups);
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
  const int sms = sm_count() > 0 ? sm_count() : 148;
  const int64_t g = total < sms ? total : sms;
  dim3 grid(static_cast<unsigned>(g)), block(Cfg::THREADS);
  kern<<<grid, block, Cfg::SMEM_BYTES, c.stream>>>(ta, tbm, p, tiles_m, tiles_n, 16, total);
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
  int rc = !amn ? make_map(&ta, A, p.k, p.m, p.batch, p.lda, p.stride_a, 32, 128, F32, 4)
                : make_map(&ta, A, p.m, p.k, p.batch, p.lda, p.stride_a, 32, 32, F32, 4);
  if (rc != TB_OK) return rc;
  rc = !bmn ? make_map(&tbm, B, p.k, p.n, p.batch, p.ldb, p.stride_b, 32, BN, F32, 4)
            : make_map(&tbm, B, p.n, p.k, p.batch, p.ldb, p.stride_b, 32, 32, F32, 4);
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
    snprintf(g_last_err, sizeof(g_last_err),
             "TF32 path needs 16-byte aligned operands (ld and offsets multiples of 4) and strided batches");
    return TB_ERR_UNSUPPORTED;
  }
  // UMMA reads MN-major 32-bit operands only in the SWIZZLE_128B_BASE32B
  // canonical layout, which this version does not build: K-major operands
  // only (col-major T x N, row-major N x T).
  if (!p.a_kcontig || p.b_ncontig) {
    snprintf(g_last_err, sizeof(g_last_err),
             "TF32 path supports K-major operands only (col-major trans_a=T,trans_b=N / row-major N,T)");
    return TB_ERR_UNSUPPORTED;
  }
  const int sms = sm_count() > 0 ? sm_count() : 148;
  int bn = 256;
  auto tiles = [&](int b) { return ((p.m + HG_BM - 1) / HG_BM) * ((p.n + b - 1) / b) * p.batch; };
  while (bn > 64 && tiles(bn) < sms) bn /= 2;
  if (bn == 256) return dispatch_tf32_bn<256>(c);
  if (bn == 128) return dispatch_tf32_bn<128>(c);
  return dispatch_tf32_bn<64>(c);
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
  // Parameter mapping: VWM = VWN = 1 asks for scalar loads; MWG /
  // NWG choose the CTA tile.  Every instantiation yields bitwise-identical
  // results (sequential-k chain), so the mapping is free to follow speed.
  // A tuned configuration (override / tuning DB; NULL when the built-in
  // default applies) picks the kernel family by KWG — 32: the TMA-fed kernel
  // (32-deep stages), 16: the register-staged kernel — and the tile by MWG x
  // NWG; without one, the shape decides (measured crossovers below).
  int mwg = 128, nwg = 128;
  bool want_tma = true;
  int tma_tile = 0;
  if (c.params) {
    mwg = c.params->MWG;
    nwg = c.params->NWG;
    if (c.params->VWM == 1 && c.params->VWN == 1) vec = false;
    want_tma = c.params->KWG >= 32;
    tma_tile = (mwg >= 128 && nwg >= 128) ? 1 : 2;
  }
  if (!vec) return launch_simt<64, 64, 16, 4, 4, false, 2>(c, "general");
  const bool small_inst = p.k > 0 && p.m <= 64 && p.n <= 64 && (p.batch > 1 || p.k <= 4096);
  if (!small_inst && want_tma) {
    const int rc = dispatch_sgemm_tma(c, tma_tile);
    if (rc >= 0) return rc;
  }
  // Small instances: persistent cp.async-pipelined kernel (bitwise identical).
  if (p.k > 0 && p.m <= 64 && p.n <= 64 && (p.batch > 1 || p.k <= 4096)) {
    if (p.m <= 32 && p.n <= 32) {
      // one 32x32 tile per instance on the TMA kernel when the operands allow
      // tensor maps (S32 batched 59.4 -> 48.7 us; a persistent variant of the
      // TMA kernel measured slower: 53.6 us, and 20 % slower at 8192^3)
      if (want_tma) {
        const int rc = dispatch_sgemm_tma(c, 3);
        if (rc >= 0) return rc;
      }
      return launch_ss_layout<32, 32, 4, 4>(c);
    }
    // 33..64: one 64x64 tile per instance on the TMA-fed FFMA2 kernel (3-D
    // tensor maps over the batch) when the operands allow tensor maps; else
    // the register-staged tiled kernel with a 4x8 micro-tile (measured faster
    // than the cp.async small kernel for 64^3, tools/sgemm_batched_variants.cu)
    if (want_tma) {
      const int rc = dispatch_sgemm_tma(c, 2);
      if (rc >= 0) return rc;
    }
    return launch_simt<64, 64, 16, 4, 8, true, 2>(c, "64x64 4x8");
  }
  const int sms = sm_count() > 0 ? sm_count() : 148;
  const int64_t tiles128 = ((p.m + 127) / 128) * ((p.n + 127) / 128) * p.batch;
  if (p.m <= 32 && p.n <= 32) return launch_simt<32, 32, 32, 4, 4, true, 8>(c, "32");
  if (mwg >= 128 && nwg >= 128) {
    // 128x256 (8x16 micro-tile) once there are >= 4 waves of it; else 128x128x16.
    const int64_t tiles256 = ((p.m + 127) / 128) * ((p.n + 255) / 256) * p.batch;
    if (tiles256 >= 4 * sms) return launch_simt<128, 256, 8, 8, 16, true, 1>(c, "128x256");
    if (tiles128 >= sms) return launch_simt<128, 128, 16, 8, 8, true, 1>(c, "128");
    // < 1 wave of 128x128 (e.g. 1024^3, BASELINE C1): 64x128 4x8 (measured
    // 30.7 vs 27.8 TFLOP/s for 64x64 4x4 at 1024^3; tools/sgemm_variants.cu)
    if (p.n >= 128 && tiles128 * 2 * 2 >= sms) return launch_simt<64, 128, 16, 4, 8, true, 2>(c, "64x128");
  }
  if (mwg >= 128 && nwg < 128 && tiles128 * 2 >= sms) return launch_simt<128, 64, 16, 8, 4, true, 2>(c, "128x64");
  if (mwg < 128 && nwg >= 128 && tiles128 * 2 >= sms) return launch_simt<64, 128, 16, 4, 8, true, 2>(c, "64x128");
  if (mwg <= 32 && nwg <= 32) return launch_simt<32, 32, 32, 4, 4, true, 8>(c, "32");
  return launch_simt<64, 64, 16, 4, 4, true, 2>(c, "64");
}

// ---------------------------------------------------------------------------
// HGEMM dispatch
// ---------------------------------------------------------------------------
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

template <int BN, bool TMA, bool AMN, bool BMN, bool VEC>
int launch_hg(const Call& c, const CUtensorMap& ta, const CUtensorMap& tbm) {
  using Cfg = HgCfg<BN, TMA>;
  const Problem& p = c.p;
  const int tiles_m = static_cast<int>((p.m + HG_BM - 1) / HG_BM);
  const int tiles_n = static_cast<int>((p.n + BN - 1) / BN);
  const int64_t total = static_cast<int64_t>(tiles_m) * tiles_n * p.batch;
  auto kern = hgemm_tc_kernel<BN, TMA, AMN, BMN, VEC>;
  static SmemAttr attr;  // per instantiation, per device
  if (int rc = ensure_smem(attr, kern, Cfg::SMEM_BYTES)) return rc;
  const int sms = sm_count() > 0 ? sm_count() : 148;
  const int64_t g = total < sms ? total : sms;
  dim3 grid(static_cast<unsigned>(g)), block(Cfg::THREADS);
  const int group_m = 16;
  kern<<<grid, block, Cfg::SMEM_BYTES, c.stream>>>(ta, tbm, p, tiles_m, tiles_n, group_m, total);
  char name[64];
  snprintf(name, sizeof(name), "hgemm_tc_%s_128x%d_%c%c%s", TMA ? "tma" : "ldg", BN, AMN ? 'm' : 'k',
           BMN ? 'n' : 'k', (!TMA && !VEC) ? "_scalar" : "");
  record(name, grid, block, 1, Cfg::SMEM_BYTES, total);
  return check_launch("hgemm_tc launch");
}

template <int BN, bool TMA, bool VEC>
int launch_hg_layout(const Call& c, const CUtensorMap& ta, const CUtensorMap& tbm) {
  const bool amn = !c.p.a_kcontig, bmn = c.p.b_ncontig;
  if (!amn && !bmn) return launch_hg<BN, TMA, false, false, VEC>(c, ta, tbm);
  if (!amn && bmn) return launch_hg<BN, TMA, false, true, VEC>(c, ta, tbm);
  if (amn && !bmn) return launch_hg<BN, TMA, true, false, VEC>(c, ta, tbm);
  return launch_hg<BN, TMA, true, true, VEC>(c, ta, tbm);
}

// One zero-initialised wave counter per (device, stream) for the pair kernel's
// wave barrier, allocated on first use and kept (a counter shared between
// streams could be reset under a running launch).
unsigned int* wave_counter(cudaStream_t stream) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<int, cudaStream_t>, unsigned int*>> pool;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  for (auto& e : pool)
    if (e.first.first == dev && e.first.second == stream) return e.second;
  unsigned int* p = nullptr;
  if (cudaMalloc(&p, 256) != cudaSuccess) return nullptr;
  pool.push_back({{dev, stream}, p});
  return p;
}

template <bool AMN, bool BMN>
int launch_h2(const Call& c, const CUtensorMap& ta, const CUtensorMap& tbm, bool sync_waves) {
  const Problem& p = c.p;
  const int tiles_m = static_cast<int>((p.m + 255) / 256);
  const int tiles_n = static_cast<int>((p.n + H2_BN - 1) / H2_BN);
  const int64_t total = static_cast<int64_t>(tiles_m) * tiles_n * p.batch;
  auto kern = hgemm_tc_2sm_kernel<AMN, BMN>;
  static SmemAttr attr;  // per instantiation, per device
  if (int rc = ensure_smem(attr, kern, H2Cfg::SMEM_BYTES)) return rc;
  const int sms = sm_count() > 0 ? sm_count() : 148;
  const int64_t clusters = total < sms / 2 ? total : sms / 2;
  dim3 grid(static_cast<unsigned>(2 * clusters)), block(H2Cfg::THREADS);
  const int group_m = 8;  // measured best for pair tiles (tools/exp7.py; also with the wave barrier)
  unsigned int* ctr = nullptr;
  if (sync_waves) {
    ctr = wave_counter(c.stream);
    if (!ctr) return TB_ERR_CUDA;
    if (cudaMemsetAsync(ctr, 0, sizeof(unsigned int), c.stream) != cudaSuccess) return check_launch("wave counter");
  }
  kern<<<grid, block, H2Cfg::SMEM_BYTES, c.stream>>>(ta, tbm, p, tiles_m, tiles_n, group_m, total, ctr);
  char name[64];
  snprintf(name, sizeof(name), "hgemm_tc2sm_tma_256x256_%c%c", AMN ? 'm' : 'k', BMN ? 'n' : 'k');
  record(name, grid, block, 2, H2Cfg::SMEM_BYTES, total);
  return check_launch("hgemm_tc_2sm launch");
}

template <int BN>
int dispatch_hgemm_bn(const Call& c) {
  const Problem& p = c.p;
  const bool amn = !p.a_kcontig, bmn = p.b_ncontig;
  const bool al = hgemm_aligned(c);
  const bool generic = (p.a_offs != nullptr) || (p.b_offs != nullptr);
  const bool big = p.m < (1LL << 31) && p.n < (1LL << 31) && p.k < (1LL << 31) && p.batch < (1LL << 31);
  CUtensorMap ta, tbm;
  memset(&ta, 0, sizeof(ta));
  memset(&tbm, 0, sizeof(tbm));
  if (al && !generic && big && !(c.flags & TB_FLAG_NO_TMA)) {
    const __half* A = static_cast<const __half*>(p.a) + p.a_off;
    const __half* B = static_cast<const __half*>(p.b) + p.b_off;
    int rc;
    if (!amn) rc = make_map(&ta, A, p.k, p.m, p.batch, p.lda, p.stride_a, 64, 128);
    else rc = make_map(&ta, A, p.m, p.k, p.batch, p.lda, p.stride_a, 64, 64);
    if (rc != TB_OK) return rc;
    // CTA-pair kernel for large problems (>= one wave of 256x256 pair tiles).
    const int sms = sm_count() > 0 ? sm_count() : 148;
    const int64_t pair_tiles = ((p.m + 255) / 256) * ((p.n + 255) / 256) * p.batch;
    // Measured crossover (tools/exp9.py): the pair kernel keeps the tensor pipe
    // ~97% busy vs ~87% up to ~5 TFLOP per call, but for the largest calls
    // (16384^3, 32768^3) its L2 reuse collapses (329 GB DRAM reads at 32768^3
    // vs 69 GB single-CTA), so those stay on the 128x256 single-CTA kernel.
    const double flop = 2.0 * static_cast<double>(p.m) * p.n * p.k * p.batch;
    // Above ~6 TFLOP per call the pair kernel runs with the wave barrier
    // (hgemm_tc_2sm.cuh): 32768^3 945 -> 1286 TFLOP/s, 16384^3 1256 -> 1398,
    // vs 1150 / 1325 for the single-CTA kernel (tools/hbig_probe.py).  Below
    // that the barrier measured neutral and is left off.
    const bool huge = flop > 6e12;
    const bool two_sm = BN == 256 && !(c.flags & TB_FLAG_NO_2SM) && pair_tiles >= sms / 2;
    const bool sync_waves = huge || (c.flags & TB_FLAG_WAVE_SYNC);
    const uint32_t bbox = two_sm ? 128 : BN;
    if (!bmn) rc = make_map(&tbm, B, p.k, p.n, p.batch, p.ldb, p.stride_b, 64, bbox);
    else rc = make_map(&tbm, B, p.n, p.k, p.batch, p.ldb, p.stride_b, 64, 64);
    if (rc != TB_OK) return rc;
    if (two_sm) {
      if (!amn && !bmn) return launch_h2<false, false>(c, ta, tbm, sync_waves);
      if (!amn && bmn) return launch_h2<false, true>(c, ta, tbm, sync_waves);
      if (amn && !bmn) return launch_h2<true, false>(c, ta, tbm, sync_waves);
      return launch_h2<true, true>(c, ta, tbm, sync_waves);
    }
    return launch_hg_layout<BN, true, true>(c, ta, tbm);
  }
  if (al) return launch_hg_layout<BN, false, true>(c, ta, tbm);
  return launch_hg_layout<BN, false, false>(c, ta, tbm);
}

template <int MI, int NI, bool AMN, bool BMN, bool VEC, bool K32>
int launch_hs(const Call& c) {
  using Cfg = HsCfg<MI, NI>;
  const Problem& p = c.p;
  const int64_t total = (p.batch + Cfg::P - 1) / Cfg::P;
  auto kern = hgemm_tc_small_kernel<MI, NI, AMN, BMN, VEC, K32>;
  static SmemAttr attr;  // per instantiation, per device
  if (int rc = ensure_smem(attr, kern, Cfg::SMEM_BYTES)) return rc;
  const int sms = sm_count() > 0 ? sm_count() : 148;
  const int64_t g = total < sms ? total : sms;
  dim3 grid(static_cast<unsigned>(g)), block(Cfg::THREADS);
  kern<<<grid, block, Cfg::SMEM_BYTES, c.stream>>>(p, total);
  char name[64];
  snprintf(name, sizeof(name), "hgemm_tc_small_%dx%d_p%d_%c%c%s%s", MI, NI, Cfg::P, AMN ? 'm' : 'k',
           BMN ? 'n' : 'k', VEC ? "_cpasync" : "_scalar", K32 ? "_k32" : "");
  record(name, grid, block, 1, Cfg::SMEM_BYTES, total);
  return check_launch("hgemm_tc_small launch");
}

template <int MI, int NI, bool VEC, bool K32>
int launch_hs_layout(const Call& c) {
  const bool amn = !c.p.a_kcontig, bmn = c.p.b_ncontig;
  if (!amn && !bmn) return launch_hs<MI, NI, false, false, VEC, K32>(c);
  if (!amn && bmn) return launch_hs<MI, NI, false, true, VEC, K32>(c);
  if (amn && !bmn) return launch_hs<MI, NI, true, false, VEC, K32>(c);
  return launch_hs<MI, NI, true, true, VEC, K32>(c);
}

template <bool VEC, bool K32>
int dispatch_hsmall_k(const Call& c) {
  const Problem& p = c.p;
  if (p.m <= 32) return p.n <= 32 ? launch_hs_layout<32, 32, VEC, K32>(c) : launch_hs_layout<32, 64, VEC, K32>(c);
  return p.n <= 32 ? launch_hs_layout<64, 32, VEC, K32>(c) : launch_hs_layout<64, 64, VEC, K32>(c);
}

// k <= 32 (one partial K block; the MMAs read K columns 0..31 only): the K32
// fill skips the unread half of each staged row.  Same MMA sequence either way.
template <bool VEC>
int dispatch_hsmall(const Call& c) {
  if (VEC && c.p.k <= 32) return dispatch_hsmall_k<VEC, true>(c);
  return dispatch_hsmall_k<VEC, false>(c);
}

// Split-K cluster size for H: a pure function of (m, n, k) and the SM count
// (never of batch or flags, so every H path of one shape issues the same
// per-element MMA / reduction sequence).  Doubles while the 128x128 tiles of
// one instance still leave half the SMs idle and each CTA keeps >= 16 K blocks
// (measured: 1024^3 with 8 K blocks per CTA was slower split than unsplit).
int hgemm_split_ks(const Problem& p) {
  const int sms = sm_count() > 0 ? sm_count() : 148;
  const int64_t t1 = ((p.m + HG_BM - 1) / HG_BM) * ((p.n + SK_BN - 1) / SK_BN);
  const int64_t nkb = (p.k + HG_BK - 1) / HG_BK;
  int ks = 1;
  while (ks < 8 && t1 * ks * 2 <= sms && nkb >= 32 * ks) ks *= 2;
  return ks;
}

template <bool TMA, bool AMN, bool BMN, bool VEC>
int launch_hsk(const Call& c, const CUtensorMap& ta, const CUtensorMap& tbm, int ks) {
  using Cfg = SkCfg<TMA>;
  const Problem& p = c.p;
  const int tiles_m = static_cast<int>((p.m + HG_BM - 1) / HG_BM);
  const int tiles_n = static_cast<int>((p.n + SK_BN - 1) / SK_BN);
  const int64_t total = static_cast<int64_t>(tiles_m) * tiles_n * p.batch;
  auto kern = hgemm_tc_splitk_kernel<TMA, AMN, BMN, VEC>;
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
  static int max_clusters[9] = {0};
  if (max_clusters[ks] == 0) {
    int v = 0;
    cfg.gridDim = dim3(static_cast<unsigned>(ks));
    if (cudaOccupancyMaxActiveClusters(&v, kern, &cfg) != cudaSuccess || v < 1) {
      cudaGetLastError();
      const int sms = sm_count() > 0 ? sm_count() : 148;
      v = sms / ks;
    }
    max_clusters[ks] = v;
  }
  const int64_t clusters = total < max_clusters[ks] ? total : max_clusters[ks];
  cfg.gridDim = dim3(static_cast<unsigned>(clusters * ks));
  const int group_m = 16;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ta, tbm, p, tiles_m, tiles_n, group_m, total);
  if (e != cudaSuccess) {
    set_err("hgemm_tc_splitk launch", e);
    return TB_ERR_CUDA;
  }
  char name[64];
  snprintf(name, sizeof(name), "hgemm_tc_splitk%d_%s_128x128_%c%c%s", ks, TMA ? "tma" : "ldg", AMN ? 'm' : 'k',
           BMN ? 'n' : 'k', (!TMA && !VEC) ? "_scalar" : "");
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
  const bool amn = !p.a_kcontig, bmn = p.b_ncontig;
  const bool al = hgemm_aligned(c);
  const bool generic = (p.a_offs != nullptr) || (p.b_offs != nullptr);
  const bool big = p.m < (1LL << 31) && p.n < (1LL << 31) && p.k < (1LL << 31) && p.batch < (1LL << 31);
  CUtensorMap ta, tbm;
  memset(&ta, 0, sizeof(ta));
  memset(&tbm, 0, sizeof(tbm));
  if (al && !generic && big && !(c.flags & TB_FLAG_NO_TMA)) {
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
  if (al) return launch_hsk_layout<false, true>(c, ta, tbm, ks);
  return launch_hsk_layout<false, false>(c, ta, tbm, ks);
}

int dispatch_hgemm(const Call& c) {
  // Small instances (m, n <= 64): packed tcgen05 kernel.  Bitwise identical to
  // the general kernel (same per-element K sequence), so this is a pure
  // function of the shape and single / batched calls stay consistent.
  if (c.p.m <= 64 && c.p.n <= 64 && !(c.flags & TB_FLAG_NO_PACK)) {
    if (hgemm_aligned(c)) return dispatch_hsmall<true>(c);
    return dispatch_hsmall<false>(c);
  }
  if (c.flags & TB_FLAG_TF32) {
    snprintf(g_last_err, sizeof(g_last_err), "TF32 flag applies to SGEMM only");
    return TB_ERR_UNSUPPORTED;
  }
  // Few output tiles and a long K: split K across a cluster (DSMEM reduction).
  if (const int ks = hgemm_split_ks(c.p); ks > 1 && !(c.flags & TB_FLAG_NO_SPLITK)) return dispatch_hsplit(c, ks);
  // Parameter mapping: NWG picks the UMMA N extent.  Pure function of the
  // parameters (never of batch) so single and batched calls of one shape use
  // the same MMA sequence (bitwise batched == looped).
  int nwg = 128;
  if (c.params) nwg = c.params->NWG;
  int bn = nwg >= 128 ? 256 : (nwg >= 64 ? 128 : 64);
  // Fewer tiles than SMs: narrow the UMMA N extent (results are independent
  // of it — tests/test_gemm_gpu.py) so more CTAs share the work.
  const int sms = sm_count() > 0 ? sm_count() : 148;
  const Problem& p = c.p;
  auto tiles = [&](int b) { return ((p.m + HG_BM - 1) / HG_BM) * ((p.n + b - 1) / b) * p.batch; };
  while (bn > 64 && tiles(bn) < sms) bn /= 2;
  if (bn == 256) return dispatch_hgemm_bn<256>(c);
  if (bn == 128) return dispatch_hgemm_bn<128>(c);
  return dispatch_hgemm_bn<64>(c);
}

int launch_hscale(const Call& c) {
  dim3 block(256);
  const int64_t total = c.p.m * c.p.n;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  if (blocks < 1) blocks = 1;
  dim3 grid(static_cast<unsigned>(blocks));
  hscale_kernel<<<grid, block, 0, c.stream>>>(c.p);
  record("hscale", grid, block, 1, 0, c.p.batch);
  return check_launch("hscale launch");
}

int run(Call& c) {
  memset(&g_last, 0, sizeof(g_last));
  if (c.m < 0 || c.n < 0 || c.k < 0 || c.p.batch < 1) return TB_ERR_INVALID;
  if (c.prec != TB_PREC_H && c.prec != TB_PREC_S) return TB_ERR_INVALID;
  if (c.m == 0 || c.n == 0) return TB_OK;
  canonicalize(c);
  if (c.prec == TB_PREC_S) return dispatch_sgemm(c);
  // H: alpha == 0 everywhere or k == 0 never touches the tensor cores.
  if (c.k == 0 || (c.p.alphas == nullptr && c.p.alpha == 0.0f)) return launch_hscale(c);
  return dispatch_hgemm(c);
}

Call make_call(int prec, int layout, int ta, int tbt, int64_t m, int64_t n, int64_t k, const void* a, int64_t lda,
               const void* b, int64_t ldb, void* cc, int64_t ldc, const tb_gemm_params* params, int flags,
               void* stream) {
  Call c;
  memset(&c, 0, sizeof(c));
  c.prec = prec; c.layout = layout; c.ta = ta; c.tbt = tbt;
  c.m = m; c.n = n; c.k = k;
  c.p.a = a; c.p.lda = lda;
  c.p.b = b; c.p.ldb = ldb;
  c.p.c = cc; c.p.ldc = ldc;
  c.params = params;
  c.flags = flags;
  c.stream = static_cast<cudaStream_t>(stream);
  c.p.batch = 1;
  return c;
}

}  // namespace

extern "C" {

int tb_gemm(int prec, int layout, int trans_a, int trans_b, int64_t m, int64_t n, int64_t k, float alpha,
            const void* a, int64_t a_off, int64_t lda, const void* b, int64_t b_off, int64_t ldb, float beta,
            void* c, int64_t c_off, int64_t ldc, const tb_gemm_params* params, int flags, void* stream) {
  Call call = make_call(prec, layout, trans_a, trans_b, m, n, k, a, lda, b, ldb, c, ldc, params, flags, stream);
  call.p.a_off = a_off; call.p.b_off = b_off; call.p.c_off = c_off;
  call.p.alpha = alpha; call.p.beta = beta;
  return run(call);
}

int tb_gemm_strided_batched(int prec, int layout, int trans_a, int trans_b, int64_t m, int64_t n, int64_t k,
                            float alpha, const void* a, int64_t a_off, int64_t lda, int64_t stride_a, const void* b,
                            int64_t b_off, int64_t ldb, int64_t stride_b, float beta, void* c, int64_t c_off,
                            int64_t ldc, int64_t stride_c, int64_t batch, const tb_gemm_params* params, int flags,
                            void* stream) {
  Call call = make_call(prec, layout, trans_a, trans_b, m, n, k, a, lda, b, ldb, c, ldc, params, flags, stream);
  call.p.a_off = a_off; call.p.b_off = b_off; call.p.c_off = c_off;
  call.p.stride_a = stride_a; call.p.stride_b = stride_b; call.p.stride_c = stride_c;
  call.p.alpha = alpha; call.p.beta = beta;
  call.p.batch = batch;
  return run(call);
}

int tb_gemm_batched(int prec, int layout, int trans_a, int trans_b, int64_t m, int64_t n, int64_t k,
                    const float* alphas, const void* a, const int64_t* a_offs, int64_t lda, const void* b,
                    const int64_t* b_offs, int64_t ldb, const float* betas, void* c, const int64_t* c_offs,
                    int64_t ldc, int64_t batch, int offs_aligned, const tb_gemm_params* params, int flags,
                    void* stream) {
  if (!alphas || !betas || !a_offs || !b_offs || !c_offs) return TB_ERR_INVALID;
  Call call = make_call(prec, layout, trans_a, trans_b, m, n, k, a, lda, b, ldb, c, ldc, params, flags, stream);
  call.p.a_offs = a_offs; call.p.b_offs = b_offs; call.p.c_offs = c_offs;
  call.p.alphas = alphas; call.p.betas = betas;
  call.p.alpha = 1.0f; call.p.beta = 0.0f;
  call.p.batch = batch;
  call.offs_aligned = offs_aligned;
  return run(call);
}

int tb_im2col(int prec, int64_t channels, int64_t height, int64_t width, int64_t kernel_h, int64_t kernel_w,
              int64_t pad_h, int64_t pad_w, int64_t stride_h, int64_t stride_w, int64_t dilation_h,
              int64_t dilation_w, const void* im, int64_t im_off, void* col, int64_t col_off, void* stream) {
  const int64_t lim = (1LL << 31) - 1;
  if (channels < 1 || height < 1 || width < 1 || kernel_h < 1 || kernel_w < 1 || stride_h < 1 || stride_w < 1 ||
      dilation_h < 1 || dilation_w < 1 || !im || !col) {
    snprintf(g_last_err, sizeof(g_last_err), "im2col: invalid geometry");
    return TB_ERR_INVALID;
  }
  const int64_t span_h = dilation_h * (kernel_h - 1) + 1, span_w = dilation_w * (kernel_w - 1) + 1;
  const int64_t out_h = (height + 2 * pad_h - span_h) / stride_h + 1;
  const int64_t out_w = (width + 2 * pad_w - span_w) / stride_w + 1;
  if (height + 2 * pad_h < span_h || width + 2 * pad_w < span_w || out_h <= 0 || out_w <= 0) {
    snprintf(g_last_err, sizeof(g_last_err), "im2col: output dimensions are not positive");
    return TB_ERR_INVALID;
  }
  Im2colGeom g;
  g.rows = channels * kernel_h * kernel_w;
  g.cols = out_h * out_w;
  const int64_t grid_y = (g.rows + IM2COL_TR - 1) / IM2COL_TR;
  if (channels > lim || height > lim || width > lim || kernel_h * kernel_w > lim || height * width > lim ||
      pad_h > lim || pad_w > lim || pad_h < -lim || pad_w < -lim || stride_h > lim || stride_w > lim || dilation_h > lim || dilation_w > lim ||
      out_h > lim || out_w > lim || g.rows > lim || g.cols > lim || channels * height * width > lim ||
      grid_y > 65535) {
    snprintf(g_last_err, sizeof(g_last_err), "im2col: geometry exceeds the 32-bit index range of the kernel");
    return TB_ERR_UNSUPPORTED;
  }
  g.channels = static_cast<int>(channels); g.height = static_cast<int>(height); g.width = static_cast<int>(width);
  g.kh = static_cast<int>(kernel_h); g.kw = static_cast<int>(kernel_w);
  g.pad_h = static_cast<int>(pad_h); g.pad_w = static_cast<int>(pad_w);
  g.stride_h = static_cast<int>(stride_h); g.stride_w = static_cast<int>(stride_w);
  g.dil_h = static_cast<int>(dilation_h); g.dil_w = static_cast<int>(dilation_w);
  g.out_h = static_cast<int>(out_h); g.out_w = static_cast<int>(out_w);
  dim3 grid(static_cast<unsigned>((g.cols + IM2COL_TQ - 1) / IM2COL_TQ), static_cast<unsigned>(grid_y));
  dim3 block(32, IM2COL_TY);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const char* name;
  if (prec == TB_PREC_S) {
    im2col_kernel<uint32_t><<<grid, block, 0, st>>>(static_cast<const uint32_t*>(im) + im_off,
                                                      static_cast<uint32_t*>(col) + col_off, g);
    name = "im2col_b32";
  } else if (prec == TB_PREC_H) {
    im2col_kernel<uint16_t><<<grid, block, 0, st>>>(static_cast<const uint16_t*>(im) + im_off,
                                                      static_cast<uint16_t*>(col) + col_off, g);
    name = "im2col_b16";
  } else {
    snprintf(g_last_err, sizeof(g_last_err), "im2col: precision must be H or S");
    return TB_ERR_UNSUPPORTED;
  }
  record(name, grid, block, 1, 0, g.rows * g.cols);
  return check_launch("im2col launch");
}

static unsigned elementwise_blocks(int64_t total) {
  const int sms = sm_count() > 0 ? sm_count() : 148;
  const int64_t want = (total + 255) / 256, cap = static_cast<int64_t>(sms) * 16;
  return static_cast<unsigned>(want < 1 ? 1 : (want < cap ? want : cap));
}

int tb_transform(int prec, int kind, int64_t rows, int64_t cols, const void* src, int64_t src_off, int64_t lds,
                 void* dst, int64_t dst_off, int64_t ldd, int upper, int unit, void* stream) {
  if (rows < 0 || cols < 0 || kind < TB_XF_COPY || kind > TB_XF_TRI_COPY || !src || !dst ||
      (kind != TB_XF_COPY && rows != cols) || lds < (rows > 0 ? rows : 1) || ldd < (rows > 0 ? rows : 1)) {
    snprintf(g_last_err, sizeof(g_last_err), "transform: invalid arguments");
    return TB_ERR_INVALID;
  }
  if (rows == 0 || cols == 0) return TB_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const dim3 grid(elementwise_blocks(rows * cols)), block(256);
  const char* name;
  if (prec == TB_PREC_S) {
    transform_kernel<uint32_t><<<grid, block, 0, st>>>(kind, rows, cols, static_cast<const uint32_t*>(src) + src_off,
                                                       lds, static_cast<uint32_t*>(dst) + dst_off, ldd, upper, unit,
                                                       0x3F800000u);
    name = "transform_b32";
  } else if (prec == TB_PREC_H) {
    transform_kernel<uint16_t><<<grid, block, 0, st>>>(kind, rows, cols, static_cast<const uint16_t*>(src) + src_off,
                                                       lds, static_cast<uint16_t*>(dst) + dst_off, ldd, upper, unit,
                                                       static_cast<uint16_t>(0x3C00));
    name = "transform_b16";
  } else {
    snprintf(g_last_err, sizeof(g_last_err), "transform: precision must be H or S");
    return TB_ERR_UNSUPPORTED;
  }
  record(name, grid, block, 1, 0, rows * cols);
  return check_launch("transform launch");
}

int tb_convert_f32(int prec, int direction, int64_t rows, int64_t cols, float alpha, const void* src, int64_t src_off,
                   int64_t lds, int transpose, void* dst, int64_t dst_off, int64_t ldd, void* stream) {
  if (rows < 0 || cols < 0 || !src || !dst || (direction != 0 && direction != 1) || ldd < (rows > 0 ? rows : 1) ||
      lds < ((transpose ? cols : rows) > 0 ? (transpose ? cols : rows) : 1)) {
    snprintf(g_last_err, sizeof(g_last_err), "convert_f32: invalid arguments");
    return TB_ERR_INVALID;
  }
  if (rows == 0 || cols == 0) return TB_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const dim3 grid(elementwise_blocks(rows * cols)), block(256);
  if (prec != TB_PREC_S && prec != TB_PREC_H) {
    snprintf(g_last_err, sizeof(g_last_err), "convert_f32: precision must be H or S");
    return TB_ERR_UNSUPPORTED;
  }
  if (direction == 0) {
    float* d = static_cast<float*>(dst) + dst_off;
    if (prec == TB_PREC_S)
      to_f32_kernel<float><<<grid, block, 0, st>>>(rows, cols, alpha, static_cast<const float*>(src) + src_off, lds,
                                                   transpose, d, ldd);
    else
      to_f32_kernel<__half><<<grid, block, 0, st>>>(rows, cols, alpha, static_cast<const __half*>(src) + src_off,
                                                    lds, transpose, d, ldd);
  } else {
    const float* sp = static_cast<const float*>(src) + src_off;
    if (prec == TB_PREC_S)
      from_f32_kernel<float><<<grid, block, 0, st>>>(rows, cols, sp, lds, transpose,
                                                     static_cast<float*>(dst) + dst_off, ldd);
    else
      from_f32_kernel<__half><<<grid, block, 0, st>>>(rows, cols, sp, lds, transpose,
                                                      static_cast<__half*>(dst) + dst_off, ldd);
  }
  record(direction == 0 ? "to_f32" : "from_f32", grid, block, 1, 0, rows * cols);
  return check_launch("convert_f32 launch");
}

int tb_trsm_block(int64_t nb, int64_t ncols, const float* t, int64_t t_off, int64_t ldt, float* x, int64_t x_off,
                  int64_t ldx, int upper, int unit, void* stream) {
  if (nb < 1 || nb > TRSM_MAX_NB || ncols < 0 || !t || !x || ldt < nb || ldx < nb) {
    snprintf(g_last_err, sizeof(g_last_err), "trsm_block: invalid arguments (nb must be 1..%d)", TRSM_MAX_NB);
    return TB_ERR_INVALID;
  }
  if (ncols == 0) return TB_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (nb == 32 || nb == 16) {  // register-resident full blocks, 64-thread CTAs
    const dim3 grid(static_cast<unsigned>((ncols + 63) / 64)), block(64);
    if (nb == 32)
      trsm_block_reg_kernel<32><<<grid, block, 0, st>>>(ncols, t + t_off, ldt, x + x_off, ldx, upper, unit);
    else
      trsm_block_reg_kernel<16><<<grid, block, 0, st>>>(ncols, t + t_off, ldt, x + x_off, ldx, upper, unit);
    record(nb == 32 ? "trsm_block_reg32" : "trsm_block_reg16", grid, block, 1, 0, ncols);
    return check_launch("trsm_block launch");
  }
  const dim3 grid(static_cast<unsigned>((ncols + 63) / 64)), block(64);
  trsm_block_kernel<<<grid, block, 0, st>>>(static_cast<int>(nb), ncols, t + t_off, ldt, x + x_off, ldx, upper, unit);
  record("trsm_block", grid, block, 1, 0, ncols);
  return check_launch("trsm_block launch");
}

int tb_last_launch(tb_launch_record* out) {
  if (!out) return TB_ERR_INVALID;
  *out = g_last;
  return TB_OK;
}

const char* tb_status_str(int status) {
  switch (status) {
    case TB_OK: return "ok";
    case TB_ERR_INVALID: return "invalid argument";
    case TB_ERR_CUDA: return "CUDA error";
    case TB_ERR_UNSUPPORTED: return "unsupported";
    case TB_ERR_DRIVER: return "driver entry point / tensor map error";
    default: return "unknown status";
  }
}

const char* tb_last_error(void) { return g_last_err; }

int tb_abi_version(void) { return TBGEMM_ABI_VERSION; }

int tb_device_sm_count(void) { return sm_count(); }

}  // extern "C"
