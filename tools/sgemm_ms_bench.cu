// Standalone timing harness for the multistage FFMA2 SGEMM (dev tool).
//   ./sgemm_ms_bench N [layout 0..3: bit1 = A K-contig, bit0 = B N-contig]
#include <cstdio>
#include <cstring>
#include <vector>
#include "sgemm_ms.cuh"
#include "../paper_1705_05249_b200/csrc/sgemm_simt.cuh"
#include "../paper_1705_05249_b200/csrc/sgemm_tma.cuh"
#include <cudaTypedefs.h>
using namespace tb;

__global__ void naive(Problem p) {
  int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  if (i >= p.m) return;
  const float* a = (const float*)p.a; const float* b = (const float*)p.b;
  float acc = 0.f;
  for (int kk = 0; kk < p.k; ++kk) {
    float av = p.a_kcontig ? a[(int64_t)i * p.lda + kk] : a[i + (int64_t)kk * p.lda];
    float bv = p.b_ncontig ? b[j + (int64_t)kk * p.ldb] : b[kk + (int64_t)j * p.ldb];
    acc = __fmaf_rn(av, bv, acc);
  }
  ((float*)p.c)[i + (int64_t)j * p.ldc] = __fmul_rn(p.alpha, acc);
}

static float* g_cref;
static int g_reps;
static const char* g_only = nullptr;

static void report(const char* name, float ms, const Problem& p) {
  cudaError_t err = cudaGetLastError();
  std::vector<float> h((size_t)p.m * p.n), r((size_t)p.m * p.n);
  cudaMemcpy(h.data(), p.c, h.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(r.data(), g_cref, r.size() * 4, cudaMemcpyDeviceToHost);
  bool same = memcmp(h.data(), r.data(), h.size() * 4) == 0;
  printf("%-36s %8.3f ms %6.1f TFLOPS bitwise=%d %s\n", name, ms, 2.0 * p.m * p.n * p.k / ms / 1e9, same,
         cudaGetErrorString(err));
  cudaMemset(p.c, 0, h.size() * 4);
}

template <typename F>
static float time_it(F f) {
  f();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < g_reps; ++i) f();
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms / g_reps;
}

template <int BM, int BN, int BK, int TM, int TN, int ST, int MINB, bool AK, bool BNC, bool BKS = false>
void run_ms(Problem p, const char* name) {
  if (g_only && !strstr(name, g_only)) return;
  using S = MsShape<BM, BN, BK, TM, TN, ST, BKS>;
  const int tm = (p.m + BM - 1) / BM, tn = (p.n + BN - 1) / BN;
  auto k = sgemm_ms_kernel<BM, BN, BK, TM, TN, ST, AK, BNC, true, MINB, BKS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, S::SMEM_BYTES);
  float ms = time_it([&] { k<<<tm * tn, S::NT, S::SMEM_BYTES>>>(p, tm, tn, 8); });
  report(name, ms, p);
}

template <int BM, int BN, int BK, int TM, int TN, int MINB, bool AK, bool BNC>
void run_simt(Problem p, const char* name) {
  if (g_only && !strstr(name, g_only)) return;
  const int tm = (p.m + BM - 1) / BM, tn = (p.n + BN - 1) / BN;
  auto k = sgemm_simt_kernel<BM, BN, BK, TM, TN, AK, BNC, true, MINB>;
  float ms = time_it([&] { k<<<tm * tn, SimtShape<BM, BN, BK, TM, TN>::NT>>>(p, tm, tn, 8); });
  report(name, ms, p);
}

static void mk(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t ld, uint32_t b0, uint32_t b1,
               CUtensorMapSwizzle sw) {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&fn, cudaEnableDefault, &q);
  }
  cuuint64_t dims[3] = {d0, d1, 1};
  cuuint64_t str[2] = {ld * 4, ld * d1 * 4};
  cuuint32_t box[3] = {b0, b1, 1}, es[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, str, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r) printf("encode failed %d\n", (int)r);
}

template <int BM, int BN, int TM, int TN, int ST, int MINB, bool AK, bool BNC, bool XP = false>
void run_tma(Problem p, const char* name) {
  if (g_only && !strstr(name, g_only)) return;
  constexpr bool AMN = !AK, BMN = BNC;
  {
    using Cfg = TmaSgemmCfg<BM, BN, 32, TM, TN, ST, AMN, BMN, XP>;
    CUtensorMap ta, tbm;
    if (AMN) mk(&ta, p.a, p.m, p.k, p.lda, BM, 32, CU_TENSOR_MAP_SWIZZLE_NONE);
    else mk(&ta, p.a, p.k, p.m, p.lda, 32, BM, CU_TENSOR_MAP_SWIZZLE_128B);
    if (BMN) mk(&tbm, p.b, p.n, p.k, p.ldb, BN, 32, CU_TENSOR_MAP_SWIZZLE_NONE);
    else mk(&tbm, p.b, p.k, p.n, p.ldb, 32, BN, CU_TENSOR_MAP_SWIZZLE_128B);
    const int tm = (p.m + BM - 1) / BM, tn = (p.n + BN - 1) / BN;
    auto k = sgemm_tma_kernel<BM, BN, 32, TM, TN, ST, AMN, BMN, MINB, XP>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
    float ms = time_it([&] { k<<<tm * tn, Cfg::NT, Cfg::SMEM_BYTES>>>(ta, tbm, p, tm, tn, 8); });
    report(name, ms, p);
  }
}

template <bool AK, bool BNC>
void suite(Problem p) {
  if constexpr (!AK && !BNC) {
    run_tma<64, 64, 4, 8, 3, 2, AK, BNC>(p, "tma 64x64x32 4x8 st3");
    run_tma<64, 64, 4, 8, 2, 2, AK, BNC>(p, "tma 64x64x32 4x8 st2");
    run_tma<64, 32, 4, 4, 3, 2, AK, BNC>(p, "tma 64x32x32 4x4 st3");
    run_tma<32, 64, 4, 8, 3, 2, AK, BNC>(p, "tma 32x64x32 4x8 st3 (64t)");
    run_tma<32, 32, 4, 4, 3, 2, AK, BNC>(p, "tma 32x32x32 4x4 st3 (64t)");
    run_tma<64, 64, 4, 4, 3, 2, AK, BNC>(p, "tma 64x64x32 4x4 st3 (256t)");
    run_tma<128, 32, 4, 4, 3, 2, AK, BNC>(p, "tma 128x32x32 4x4 st3 (256t)");
    // <= 148 tiles at 1024^2: one CTA per SM, larger micro-tiles
    run_tma<128, 64, 8, 8, 3, 1, AK, BNC>(p, "tma 128x64x32 8x8 st3 (128t)");
    run_tma<128, 64, 8, 8, 4, 1, AK, BNC>(p, "tma 128x64x32 8x8 st4 (128t)");
    run_tma<128, 64, 8, 4, 4, 1, AK, BNC>(p, "tma 128x64x32 8x4 st4 (256t)");
    run_tma<128, 64, 4, 8, 4, 1, AK, BNC>(p, "tma 128x64x32 4x8 st4 (256t)");
    run_tma<64, 128, 8, 8, 4, 1, AK, BNC>(p, "tma 64x128x32 8x8 st4 (128t)");
    run_tma<64, 128, 4, 8, 4, 1, AK, BNC>(p, "tma 64x128x32 4x8 st4 (256t)");
    // 144 tiles of 128x60 at 1024^2 (vs 128 of 128x64): measured 78-80 us vs 53 us (5 warps, XP)
    run_tma<128, 60, 4, 12, 4, 1, AK, BNC, true>(p, "tma 128x60x32 4x12 st4 xp (160t)");
    run_tma<128, 60, 4, 12, 5, 1, AK, BNC, true>(p, "tma 128x60x32 4x12 st5 xp (160t)");
    run_tma<128, 64, 4, 8, 4, 1, AK, BNC, true>(p, "tma 128x64x32 4x8 st4 xp (256t)");
    run_tma<64, 64, 4, 4, 4, 2, AK, BNC>(p, "tma 64x64x32 4x4 st4 (256t)");
    run_tma<64, 64, 8, 4, 4, 2, AK, BNC>(p, "tma 64x64x32 8x4 st4");
    run_tma<64, 64, 4, 8, 4, 2, AK, BNC>(p, "tma 64x64x32 4x8 st4");
  } else if constexpr (AK && BNC) {
    // library: 64x64 8x4 st4 (PAIR_N)
    run_tma<64, 64, 8, 4, 4, 2, AK, BNC>(p, "tma 64x64x32 8x4 st4");
    run_tma<128, 64, 8, 4, 4, 1, AK, BNC>(p, "tma 128x64x32 8x4 st4 (256t)");
    run_tma<128, 64, 4, 8, 4, 1, AK, BNC>(p, "tma 128x64x32 4x8 st4 (256t)");
    run_tma<64, 128, 4, 8, 4, 1, AK, BNC>(p, "tma 64x128x32 4x8 st4 (256t)");
  } else if constexpr (!AK && BNC) {
    // library: 64x64 4x8 st3
    run_tma<64, 64, 4, 8, 3, 2, AK, BNC>(p, "tma 64x64x32 4x8 st3");
    run_tma<128, 64, 4, 8, 4, 1, AK, BNC>(p, "tma 128x64x32 4x8 st4 (256t)");
    run_tma<64, 128, 4, 8, 4, 1, AK, BNC>(p, "tma 64x128x32 4x8 st4 (256t)");
  } else {
    // library: 64x64 4x8 st3 (A transposed in shared memory)
    run_tma<64, 64, 4, 8, 3, 2, AK, BNC>(p, "tma 64x64x32 4x8 st3");
    run_tma<128, 64, 4, 8, 4, 1, AK, BNC>(p, "tma 128x64x32 4x8 st4 (256t)");
    run_tma<64, 128, 4, 8, 4, 1, AK, BNC>(p, "tma 64x128x32 4x8 st4 (256t)");
  }
}

int main(int argc, char** argv) {
  int N = argc > 1 ? atoi(argv[1]) : 8192;
  int M_ = N, N_ = N, K_ = N;
  if (argc > 1 && strchr(argv[1], 'x')) { sscanf(argv[1], "%dx%dx%d", &M_, &N_, &K_); N = M_ > N_ ? M_ : N_; N = N > K_ ? N : K_; }
  int lay = argc > 2 ? atoi(argv[2]) : 0;
  if (argc > 3) g_only = argv[3];
  if (argc > 4) g_reps = atoi(argv[4]);
  size_t bytes = (size_t)N * N * 4;
  float *a, *b, *c;
  cudaMalloc(&a, bytes); cudaMalloc(&b, bytes); cudaMalloc(&c, bytes); cudaMalloc(&g_cref, bytes);
  std::vector<float> h((size_t)N * N);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)((i * 2654435761u) % 2001) / 1000.0f - 1.0f;
  cudaMemcpy(a, h.data(), bytes, cudaMemcpyHostToDevice);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)((i * 40503u + 7) % 1999) / 999.0f - 1.0f;
  cudaMemcpy(b, h.data(), bytes, cudaMemcpyHostToDevice);
  Problem p{}; p.m = M_; p.n = N_; p.k = K_; p.a = a; p.b = b; p.c = g_cref; p.ldc = M_;
  p.lda = (lay >> 1) ? K_ : M_; p.ldb = (lay & 1) ? N_ : K_;
  p.alpha = 1.f; p.beta = 0.f; p.batch = 1; p.a_kcontig = lay >> 1; p.b_ncontig = lay & 1;
  if (!g_reps) g_reps = N >= 8192 ? 3 : 20;
  naive<<<dim3((M_ + 255) / 256, N_), 256>>>(p);
  cudaDeviceSynchronize();
  p.c = c;
  printf("%dx%dx%d layout=%d\n", M_, N_, K_, lay);
  switch (lay) {
    case 0: suite<false, false>(p); break;
    case 1: suite<false, true>(p); break;
    case 2: suite<true, false>(p); break;
    default: suite<true, true>(p); break;
  }
  return 0;
}
