// tbgemm.cu — C-ABI entry points (include/tbgemm.h), per-thread launch
// records, tensor-map encoding and the non-GEMM helper kernels.
//
// Host-side responsibilities (all argument *validation* happened in the
// Python routine layer, mirroring pkg/src/tunedblas/routines/level3.py:94-133
// and extras.py:188-348):
//   1. canonicalise layout/trans into one column-major problem (row-major C
//      is C^T col-major: swap A<->B and m<->n — common.py:1-7, level3.py:41-45);
//   2. route to a kernel: by shape (built-in) or by a "gemm_b200"
//      configuration (sgemm.cu, sgemm_tma.cu, hgemm.cu, hgemm_small.cu);
//   3. pick the producer (TMA when 16-byte alignment allows, LDG otherwise);
//   4. build TMA tensor maps (cuTensorMapEncodeTiled via the runtime's
//      driver entry point — no link-time libcuda dependency);
//   5. launch on the caller's stream and record a tb_launch_record.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "host.h"
#include "im2col.cuh"
#include "structured.cuh"

using namespace tb;
using namespace tb::host;

namespace {

thread_local tb_launch_record g_last{};
thread_local char g_last_err[256] = "";

}  // namespace

namespace tb {
namespace host {

char* err_buf() { return g_last_err; }

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

static EncodeTiledFn get_encode_fn() {
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

int make_map(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t batch, uint64_t ld,
             uint64_t stride, uint32_t box0, uint32_t box1, CUtensorMapDataType dt, uint64_t es,
             CUtensorMapSwizzle swizzle, uint32_t box2) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn) {
    snprintf(g_last_err, sizeof(g_last_err), "cuTensorMapEncodeTiled entry point unavailable");
    return TB_ERR_DRIVER;
  }
  cuuint64_t dims[3] = {d0, d1, batch};
  uint64_t zstride = stride * es;
  if (batch <= 1) zstride = ((ld * d1 * es) + 15) / 16 * 16;
  cuuint64_t strides[2] = {ld * es, zstride};
  cuuint32_t box[3] = {box0, box1, box2};
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

// Wave-barrier counters (two words per launch: arrivals and the abandon
// flag): one 256-byte slot per (device, stream), carved from a 64-slot block
// allocated once per device — eagerly by tb_prepare_device(), which the
// Python Context calls, or on first use.  Nothing is allocated while the
// stream is capturing a CUDA graph: without a slot (pool missing during
// capture, or more than 64 streams) the launch simply runs without the
// barrier, which is advisory (same results, only L2 reuse changes).
constexpr int kWaveSlots = 64;
struct WavePool {
  unsigned int* base = nullptr;
  cudaStream_t streams[kWaveSlots] = {};
  int used = 0;
};
static std::mutex g_wave_mu;
static WavePool g_wave[64];

static int wave_pool_alloc(int dev) {
  WavePool& wp = g_wave[dev];
  if (wp.base) return TB_OK;
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, 256 * kWaveSlots);
  if (e != cudaSuccess) {
    set_err("cudaMalloc (wave counters)", e);
    return TB_ERR_CUDA;
  }
  wp.base = static_cast<unsigned int*>(p);
  return TB_OK;
}

unsigned int* wave_counter(cudaStream_t stream) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(g_wave_mu);
  WavePool& wp = g_wave[dev];
  if (!wp.base) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(stream, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
      cudaGetLastError();
      return nullptr;
    }
    if (wave_pool_alloc(dev) != TB_OK) return nullptr;
  }
  for (int i = 0; i < wp.used; ++i)
    if (wp.streams[i] == stream) return wp.base + 64 * i;
  if (wp.used == kWaveSlots) return nullptr;
  wp.streams[wp.used] = stream;
  return wp.base + 64 * wp.used++;
}

// Split-K partial workspace (hgemm_tc_splitk.cuh): one slot of `slot_bytes`
// per CTA of a grid of at most the SM count, per (device, stream), allocated
// on first use outside stream capture.  nullptr: the kernel exchanges
// partials through DSMEM instead (same summation order, same results).
constexpr int kWsSlots = 16;
struct WsPool {
  cudaStream_t streams[kWsSlots] = {};
  void* ptr[kWsSlots] = {};
  int used = 0;
};
static std::mutex g_ws_mu;
static WsPool g_ws[64];

void* splitk_workspace(cudaStream_t stream, size_t bytes) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(g_ws_mu);
  WsPool& wp = g_ws[dev];
  for (int i = 0; i < wp.used; ++i)
    if (wp.streams[i] == stream) return wp.ptr[i];
  if (wp.used == kWsSlots) return nullptr;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(stream, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return nullptr;
  }
  void* p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  wp.streams[wp.used] = stream;
  wp.ptr[wp.used] = p;
  ++wp.used;
  return p;
}

// Repack scratch: one growable buffer per (device, stream), reused in stream
// order (each call's packs and GEMM are queued on that stream).  Growing
// frees the old buffer (cudaFree synchronises, so nothing still reads it).
// Never handed out while the stream is capturing a graph: a captured graph
// would keep the pointer past a later growth.
struct PackPool {
  cudaStream_t streams[kWsSlots] = {};
  void* ptr[kWsSlots] = {};
  size_t bytes[kWsSlots] = {};
  int used = 0;
};
static std::mutex g_pack_mu;
static PackPool g_pack[64];

void* pack_workspace(cudaStream_t stream, size_t bytes) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(stream, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return nullptr;
  }
  std::lock_guard<std::mutex> lock(g_pack_mu);
  PackPool& pp = g_pack[dev];
  int slot = -1;
  for (int i = 0; i < pp.used; ++i)
    if (pp.streams[i] == stream) slot = i;
  if (slot >= 0 && pp.bytes[slot] >= bytes) return pp.ptr[slot];
  if (slot < 0) {
    if (pp.used == kWsSlots) return nullptr;
    slot = pp.used++;
    pp.streams[slot] = stream;
  } else if (pp.ptr[slot] != nullptr) {
    cudaFree(pp.ptr[slot]);
    pp.ptr[slot] = nullptr;
    pp.bytes[slot] = 0;
  }
  void* p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  pp.ptr[slot] = p;
  pp.bytes[slot] = bytes;
  return p;
}

// Unaligned operands: TMA needs 16-byte aligned row pitches and bases; with
// an odd leading dimension the kernels fall back to per-element loads, an
// order of magnitude slower for H (2500^3: 1165 us) and ~2x for S.  Copy each
// offending operand once into the per-stream scratch with its pitch rounded
// up to 16 bytes (the reference pads its operands too, level3.py:71-82) and
// run the aligned kernels on the copies: same values, same bits.
// One thread: one 16-byte vector of a row — element loads from the unaligned
// source, one 16-byte store into the aligned copy (its pitch is a multiple of
// the vector and the tail of the last vector lands in the padding).
template <typename T>
__global__ void __launch_bounds__(256) pack_rows_kernel(const T* __restrict__ src, int64_t src_ld,
                                                        int64_t src_stride, T* __restrict__ dst, int64_t dst_ld,
                                                        int64_t dst_stride, int64_t rows, int64_t cols,
                                                        int64_t batch) {
  constexpr int V = 16 / sizeof(T);
  grid_dep_wait();
  const int64_t c0 = (static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x) * V;
  if (c0 >= cols) return;
  const int nv = cols - c0 < V ? static_cast<int>(cols - c0) : V;
  for (int64_t z = 0; z < batch; ++z)
    for (int64_t r = blockIdx.y; r < rows; r += gridDim.y) {
      const T* s = src + z * src_stride + r * src_ld + c0;
      T v[V];
#pragma unroll
      for (int e = 0; e < V; ++e) v[e] = e < nv ? s[e] : T(0);
      uint4 out;
      memcpy(&out, v, 16);
      *reinterpret_cast<uint4*>(dst + z * dst_stride + r * dst_ld + c0) = out;
    }
}

int repack_operands(const Call& c, int es, Call& c2, int& launches) {
  const Problem& p = c.p;
  if (p.a_offs || p.b_offs) return -1;
  if (p.m <= 0 || p.n <= 0 || p.k <= 0 || p.batch <= 0) return -1;  // nothing to read
  if (p.m >= (1LL << 31) || p.n >= (1LL << 31) || p.k >= (1LL << 31) || p.batch >= (1LL << 31)) return -1;
  const int64_t V = 16 / es;
  // stored (rows, cols) of op(A) / op(B) in the canonical column-major problem
  const int64_t ar = p.a_kcontig ? p.m : p.k, ac = p.a_kcontig ? p.k : p.m;
  const int64_t br = p.b_ncontig ? p.k : p.n, bc = p.b_ncontig ? p.n : p.k;
  const bool pack_a = (p.lda % V) || !aligned_elems(p.a, p.a_off, es, 16) || (p.batch > 1 && (p.stride_a % V));
  const bool pack_b = (p.ldb % V) || !aligned_elems(p.b, p.b_off, es, 16) || (p.batch > 1 && (p.stride_b % V));
  if (!pack_a && !pack_b) return -1;
  const int64_t lda2 = (ac + V - 1) / V * V, ldb2 = (bc + V - 1) / V * V;
  const int64_t sa2 = ar * lda2, sb2 = br * ldb2;
  const int64_t bytes = ((pack_a ? p.batch * sa2 : 0) + (pack_b ? p.batch * sb2 : 0)) * es + 64;
  if (bytes > (int64_t{2} << 30)) return -1;  // at most 2 GB of scratch: otherwise the per-element path
  uint8_t* next = static_cast<uint8_t*>(pack_workspace(c.stream, static_cast<size_t>(bytes)));
  if (next == nullptr) return -1;
  auto pack = [&](const void* base, int64_t off, int64_t ld, int64_t stride, int64_t rows, int64_t cols,
                  int64_t ld2, int64_t stride2) -> const void* {
    dim3 grid(static_cast<unsigned>((cols + 256 * V - 1) / (256 * V)), static_cast<unsigned>(rows < 65535 ? rows : 65535));
    if (es == 4)
      pack_rows_kernel<uint32_t><<<grid, 256, 0, c.stream>>>(static_cast<const uint32_t*>(base) + off, ld, stride,
                                                             reinterpret_cast<uint32_t*>(next), ld2, stride2, rows,
                                                             cols, p.batch);
    else
      pack_rows_kernel<uint16_t><<<grid, 256, 0, c.stream>>>(static_cast<const uint16_t*>(base) + off, ld, stride,
                                                             reinterpret_cast<uint16_t*>(next), ld2, stride2, rows,
                                                             cols, p.batch);
    ++launches;
    const void* out = next;
    next += (p.batch * stride2 * es + 15) / 16 * 16;
    return out;
  };
  c2 = c;
  if (pack_a) {
    c2.p.a = pack(p.a, p.a_off, p.lda, p.stride_a, ar, ac, lda2, sa2);
    c2.p.a_off = 0;
    c2.p.lda = lda2;
    c2.p.stride_a = sa2;
  }
  if (pack_b) {
    c2.p.b = pack(p.b, p.b_off, p.ldb, p.stride_b, br, bc, ldb2, sb2);
    c2.p.b_off = 0;
    c2.p.ldb = ldb2;
    c2.p.stride_b = sb2;
  }
  return check_launch("operand repack");
}

void note_extra_launches(int n, const char* suffix) {
  g_last.launches += n;
  const size_t len = strlen(g_last.kernel);
  snprintf(g_last.kernel + len, sizeof(g_last.kernel) - len, "%s", suffix);
}

}  // namespace host
}  // namespace tb

namespace {

// ---------------------------------------------------------------------------
// Canonicalisation
// ---------------------------------------------------------------------------
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
               const void* b, int64_t ldb, void* cc, int64_t ldc, const tb_gemm_config* cfg, int flags,
               void* stream) {
  Call c;
  memset(&c, 0, sizeof(c));
  c.prec = prec; c.layout = layout; c.ta = ta; c.tbt = tbt;
  c.m = m; c.n = n; c.k = k;
  c.p.a = a; c.p.lda = lda;
  c.p.b = b; c.p.ldb = ldb;
  c.p.c = cc; c.p.ldc = ldc;
  c.cfg = (cfg && cfg->MWG > 0) ? cfg : nullptr;
  c.flags = flags;
  c.stream = static_cast<cudaStream_t>(stream);
  c.p.batch = 1;
  return c;
}

}  // namespace

extern "C" {

int tb_gemm(int prec, int layout, int trans_a, int trans_b, int64_t m, int64_t n, int64_t k, float alpha,
            const void* a, int64_t a_off, int64_t lda, const void* b, int64_t b_off, int64_t ldb, float beta,
            void* c, int64_t c_off, int64_t ldc, const tb_gemm_config* cfg, int flags, void* stream) {
  Call call = make_call(prec, layout, trans_a, trans_b, m, n, k, a, lda, b, ldb, c, ldc, cfg, flags, stream);
  call.p.a_off = a_off; call.p.b_off = b_off; call.p.c_off = c_off;
  call.p.alpha = alpha; call.p.beta = beta;
  return run(call);
}

int tb_gemm_strided_batched(int prec, int layout, int trans_a, int trans_b, int64_t m, int64_t n, int64_t k,
                            float alpha, const void* a, int64_t a_off, int64_t lda, int64_t stride_a, const void* b,
                            int64_t b_off, int64_t ldb, int64_t stride_b, float beta, void* c, int64_t c_off,
                            int64_t ldc, int64_t stride_c, int64_t batch, const tb_gemm_config* cfg, int flags,
                            void* stream) {
  Call call = make_call(prec, layout, trans_a, trans_b, m, n, k, a, lda, b, ldb, c, ldc, cfg, flags, stream);
  call.p.a_off = a_off; call.p.b_off = b_off; call.p.c_off = c_off;
  call.p.stride_a = stride_a; call.p.stride_b = stride_b; call.p.stride_c = stride_c;
  call.p.alpha = alpha; call.p.beta = beta;
  call.p.batch = batch;
  return run(call);
}

int tb_gemm_batched(int prec, int layout, int trans_a, int trans_b, int64_t m, int64_t n, int64_t k,
                    const float* alphas, const void* a, const int64_t* a_offs, int64_t lda, const void* b,
                    const int64_t* b_offs, int64_t ldb, const float* betas, void* c, const int64_t* c_offs,
                    int64_t ldc, int64_t batch, int offs_aligned, const tb_gemm_config* cfg, int flags,
                    void* stream) {
  if (!alphas || !betas || !a_offs || !b_offs || !c_offs) return TB_ERR_INVALID;
  Call call = make_call(prec, layout, trans_a, trans_b, m, n, k, a, lda, b, ldb, c, ldc, cfg, flags, stream);
  call.p.a_offs = a_offs; call.p.b_offs = b_offs; call.p.c_offs = c_offs;
  call.p.alphas = alphas; call.p.betas = betas;
  call.p.alpha = 1.0f; call.p.beta = 0.0f;
  call.p.batch = batch;
  call.offs_aligned = offs_aligned;
  return run(call);
}

int tb_convgemm(int prec, int64_t channels, int64_t height, int64_t width, int64_t kernel_h, int64_t kernel_w,
                int64_t pad_h, int64_t pad_w, int64_t stride_h, int64_t stride_w, int64_t dilation_h,
                int64_t dilation_w, int64_t num_kernels, int64_t batch, const void* im, int64_t im_off,
                const void* kernel, int64_t kernel_off, void* result, int64_t result_off, int flags,
                void* stream) {
  memset(&g_last, 0, sizeof(g_last));
  const int64_t lim = (1LL << 31) - 1;
  if (channels < 1 || height < 1 || width < 1 || kernel_h < 1 || kernel_w < 1 || stride_h < 1 || stride_w < 1 ||
      dilation_h < 1 || dilation_w < 1 || num_kernels < 0 || batch < 1 || !im || !kernel || !result) {
    snprintf(g_last_err, sizeof(g_last_err), "convgemm: invalid geometry");
    return TB_ERR_INVALID;
  }
  const int64_t span_h = dilation_h * (kernel_h - 1) + 1, span_w = dilation_w * (kernel_w - 1) + 1;
  const int64_t out_h = (height + 2 * pad_h - span_h) / stride_h + 1;
  const int64_t out_w = (width + 2 * pad_w - span_w) / stride_w + 1;
  if (height + 2 * pad_h < span_h || width + 2 * pad_w < span_w || out_h <= 0 || out_w <= 0) {
    snprintf(g_last_err, sizeof(g_last_err), "convgemm: output dimensions are not positive");
    return TB_ERR_INVALID;
  }
  const int64_t K = channels * kernel_h * kernel_w, N = out_h * out_w;
  if (channels * height * width > lim || K > lim || N > lim || height > lim || width > lim || pad_h > lim ||
      pad_w > lim || pad_h < -lim || pad_w < -lim || stride_h > lim || stride_w > lim || dilation_h > lim ||
      dilation_w > lim || kernel_h * kernel_w > lim) {
    snprintf(g_last_err, sizeof(g_last_err), "convgemm: geometry exceeds the 32-bit index range of the kernel");
    return TB_ERR_UNSUPPORTED;
  }
  if (num_kernels == 0) return TB_OK;
  ConvGeom g;
  g.channels = static_cast<int>(channels); g.height = static_cast<int>(height); g.width = static_cast<int>(width);
  g.kh = static_cast<int>(kernel_h); g.kw = static_cast<int>(kernel_w);
  g.pad_h = static_cast<int>(pad_h); g.pad_w = static_cast<int>(pad_w);
  g.stride_h = static_cast<int>(stride_h); g.stride_w = static_cast<int>(stride_w);
  g.dil_h = static_cast<int>(dilation_h); g.dil_w = static_cast<int>(dilation_w);
  g.out_h = static_cast<int>(out_h); g.out_w = static_cast<int>(out_w);
  // Canonical column-major problem: C'(q, f) = sum_r col[r][q] * kernel[f][r]
  //   m = N positions, n = num_kernels filters, k = K;
  //   op(A) gathered (MN-major), B' = kernel rows (K-contiguous, ldb = K),
  //   C' = result plane per filter (ldc = N) — the NCHW output.
  Call c;
  memset(&c, 0, sizeof(c));
  c.prec = prec;
  c.m = N; c.n = num_kernels; c.k = K;
  c.p.m = N; c.p.n = num_kernels; c.p.k = K;
  c.p.a = im; c.p.a_off = im_off; c.p.stride_a = channels * height * width; c.p.lda = 1;
  c.p.b = kernel; c.p.b_off = kernel_off; c.p.ldb = K; c.p.stride_b = 0;
  c.p.c = result; c.p.c_off = result_off; c.p.ldc = N; c.p.stride_c = num_kernels * N;
  c.p.alpha = 1.0f; c.p.beta = 0.0f;
  c.p.batch = batch;
  c.p.a_kcontig = 0; c.p.b_ncontig = 0;
  c.conv = &g;
  c.flags = flags;
  c.stream = static_cast<cudaStream_t>(stream);
  if (prec == TB_PREC_H) return dispatch_hconv(c);
  if (prec == TB_PREC_S) return dispatch_sconv(c);
  snprintf(g_last_err, sizeof(g_last_err), "convgemm: precision must be H or S");
  return TB_ERR_UNSUPPORTED;
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
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const char* name;
  // patch-staged kernel (im2col.cuh) when its conditions hold; H only (S:
  // 16.4 us against the tile kernel's 15.2 at the ResNet layer, L2 flushed)
  if (prec == TB_PREC_H) {
    const int es = prec == TB_PREC_S ? 4 : 2, vec = 16 / es, tr = 8 * vec;  // rows per CTA
    const int kk = g.kh * g.kw;
    // worst-case patch of IM2COL_VQ consecutive pixels x tr rows
    const int64_t oy_span = (IM2COL_VQ - 1) / g.out_w + 2;
    const int64_t pr = (oy_span - 1) * g.stride_h + static_cast<int64_t>(g.kh - 1) * g.dil_h + 1;
    const int64_t pw = static_cast<int64_t>(g.out_w - 1) * g.stride_w + static_cast<int64_t>(g.kw - 1) * g.dil_w + 1;
    const int64_t nch = (tr - 1) / kk + 2;
    const int64_t r_chunks = (g.rows + tr - 1) / tr, q_blocks = (g.cols + IM2COL_VQ - 1) / IM2COL_VQ;
    if (g.rows % vec == 0 && aligned_elems(col, col_off, es, 16) && nch * pr * pw * es <= IM2COL_PATCH_BYTES &&
        pw <= 1024 && pr <= 1024 && r_chunks <= 65535 && q_blocks < 0x7fffffff) {
      Im2colPatch pp;
      pp.pw = static_cast<int>(pw);
      pp.r_chunks = static_cast<int>(r_chunks);
      const dim3 grid2(static_cast<unsigned>(q_blocks), static_cast<unsigned>(r_chunks)), block2(IM2COL_VQ);
      im2col_vec_kernel<uint16_t><<<grid2, block2, 0, st>>>(static_cast<const uint16_t*>(im) + im_off,
                                                            static_cast<uint16_t*>(col) + col_off, g, pp);
      name = "im2col_vec_b16";
      record(name, grid2, block2, 1, 0, g.rows * g.cols);
      return check_launch("im2col launch");
    }
  }
  dim3 grid(static_cast<unsigned>((g.cols + IM2COL_TQ - 1) / IM2COL_TQ), static_cast<unsigned>(grid_y));
  dim3 block(32, IM2COL_TY);
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

int tb_prepare_device(void) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) {
    set_err("cudaGetDevice", e);
    return TB_ERR_CUDA;
  }
  if (dev < 0 || dev >= 64) return TB_ERR_UNSUPPORTED;
  std::lock_guard<std::mutex> lock(g_wave_mu);
  return wave_pool_alloc(dev);
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
