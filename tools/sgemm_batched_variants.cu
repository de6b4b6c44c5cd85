// Standalone timing of SIMT tile variants on strided-batched SGEMM (dev tool).
#include <cstdio>
#include <cstring>
#include <vector>
#include "../paper_1705_05249_b200/csrc/sgemm_simt.cuh"
#include "../paper_1705_05249_b200/csrc/sgemm_small.cuh"
using namespace tb;

float* g_ref = nullptr;
template <int BM, int BN, int BK, int TM, int TN, int MINB, bool AK, bool BNC>
void run(Problem p, int reps, const char* name) {
  const int tiles_m = (p.m + BM - 1) / BM, tiles_n = (p.n + BN - 1) / BN;
  dim3 grid(tiles_m * tiles_n * p.batch), block(SimtShape<BM, BN, BK, TM, TN>::NT);
  auto k = sgemm_simt_kernel<BM, BN, BK, TM, TN, AK, BNC, true, MINB>;
  k<<<grid, block>>>(p, tiles_m, tiles_n, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i) k<<<grid, block>>>(p, tiles_m, tiles_n, 8);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
  size_t n = (size_t)p.m * p.n * p.batch;
  std::vector<float> h(n), r(n);
  cudaMemcpy(h.data(), p.c, n * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(r.data(), g_ref, n * 4, cudaMemcpyDeviceToHost);
  printf("%-30s %8.1f us  %7.0f GB/s  %6.1f TFLOPS bitwise=%d %s\n", name, ms * 1e3,
         3.0 * n * 4 / ms / 1e6, 2.0 * p.m * p.n * p.k * p.batch / ms / 1e9, memcmp(h.data(), r.data(), n * 4) == 0,
         cudaGetErrorString(cudaGetLastError()));
}

template <int MI, int NI, int TM, int TN>
void run_small(Problem p, int reps, const char* name) {
  using Cfg = SsCfg<MI, NI, TM, TN>;
  auto k = sgemm_small_kernel<MI, NI, TM, TN, false, false>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 256, Cfg::SMEM_BYTES);
  const int64_t groups = (p.batch + Cfg::G - 1) / Cfg::G;
  int64_t g = 148LL * per_sm; if (g > groups) g = groups;
  k<<<g, 256, Cfg::SMEM_BYTES>>>(p, groups);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i) k<<<g, 256, Cfg::SMEM_BYTES>>>(p, groups);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
  size_t n = (size_t)p.m * p.n * p.batch;
  std::vector<float> h(n), r(n);
  cudaMemcpy(h.data(), p.c, n * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(r.data(), g_ref, n * 4, cudaMemcpyDeviceToHost);
  printf("%-30s %8.1f us  %7.0f GB/s  %6.1f TFLOPS bitwise=%d occ=%d stages=%d %s\n", name, ms * 1e3,
         3.0 * n * 4 / ms / 1e6, 2.0 * p.m * p.n * p.k * p.batch / ms / 1e9, memcmp(h.data(), r.data(), n * 4) == 0,
         per_sm, Cfg::STAGES, cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char** argv) {
  int S = argc > 1 ? atoi(argv[1]) : 64, B = 16384;
  size_t e = (size_t)S * S, bytes = e * B * 4;
  float *a, *b, *c;
  cudaMalloc(&a, bytes); cudaMalloc(&b, bytes); cudaMalloc(&c, bytes); cudaMalloc(&g_ref, bytes);
  std::vector<float> h(e * B);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)((i * 2654435761u) % 2001) / 1000.0f - 1.0f;
  cudaMemcpy(a, h.data(), bytes, cudaMemcpyHostToDevice);
  cudaMemcpy(b, h.data(), bytes, cudaMemcpyHostToDevice);
  // canonical col-major problem of the row-major NN bench: A' M-contig, B' K-contig
  Problem p{}; p.m = p.n = p.k = S; p.a = a; p.lda = S; p.b = b; p.ldb = S; p.c = g_ref; p.ldc = S;
  p.stride_a = p.stride_b = p.stride_c = e; p.alpha = 1.f; p.beta = 0.f; p.batch = B;
  run<64, 64, 16, 4, 4, 2, false, false>(p, 20, "ref 64x64x16 4x4 (256t)");
  p.c = c;
  if (S == 64) {
    run<64, 64, 16, 4, 8, 2, false, false>(p, 20, "simt 64x64x16 4x8 (128t)");
    run_small<64, 64, 8, 4>(p, 20, "small 64 8x4 (128t/inst)");
    run_small<64, 64, 4, 8>(p, 20, "small 64 4x8 (128t/inst)");
    run_small<64, 64, 8, 8>(p, 20, "small 64 8x8 (64t/inst)");
    run_small<64, 64, 4, 4>(p, 20, "small 64 4x4 (256t/inst)");
  } else {
    run_small<32, 32, 4, 4>(p, 20, "small 32 4x4 (64t/inst)");
    run_small<32, 32, 8, 4>(p, 20, "small 32 8x4 (32t/inst)");
    run_small<32, 32, 4, 8>(p, 20, "small 32 4x8 (32t/inst)");
  }
  return 0;
}
