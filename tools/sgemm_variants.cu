// Standalone timing harness for SGEMM SIMT variants (dev tool).
#include <cstdio>
#include <vector>
#include "../paper_1705_05249_b200/csrc/sgemm_simt.cuh"
using namespace tb;

template <int BM, int BN, int BK, int TM, int TN, int MINB>
float run(Problem p, int reps, float* cref, const char* name) {
  const int tiles_m = (p.m + BM - 1) / BM, tiles_n = (p.n + BN - 1) / BN;
  dim3 grid(tiles_m * tiles_n), block(SimtShape<BM, BN, BK, TM, TN>::NT);
  auto k = sgemm_simt_kernel<BM, BN, BK, TM, TN, false, false, true, MINB>;
  k<<<grid, block>>>(p, tiles_m, tiles_n, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < reps; ++i) k<<<grid, block>>>(p, tiles_m, tiles_n, 8);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
  cudaError_t err = cudaGetLastError();
  // compare bitwise with reference output
  std::vector<float> h(p.m * p.n), r(p.m * p.n);
  cudaMemcpy(h.data(), p.c, h.size() * 4, cudaMemcpyDeviceToHost);
  bool same = true;
  if (cref) { cudaMemcpy(r.data(), cref, r.size() * 4, cudaMemcpyDeviceToHost); same = (memcmp(h.data(), r.data(), h.size() * 4) == 0); }
  printf("%-28s %8.3f ms  %6.1f TFLOPS  bitwise=%d %s\n", name, ms, 2.0 * p.m * p.n * p.k / ms / 1e9, same, cudaGetErrorString(err));
  return ms;
}

int main(int argc, char** argv) {
  int N = argc > 1 ? atoi(argv[1]) : 8192;
  size_t bytes = (size_t)N * N * 4;
  float *a, *b, *c, *cref;
  cudaMalloc(&a, bytes); cudaMalloc(&b, bytes); cudaMalloc(&c, bytes); cudaMalloc(&cref, bytes);
  std::vector<float> h((size_t)N * N);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)((i * 2654435761u) % 2001) / 1000.0f - 1.0f;
  cudaMemcpy(a, h.data(), bytes, cudaMemcpyHostToDevice);
  cudaMemcpy(b, h.data(), bytes, cudaMemcpyHostToDevice);
  Problem p{}; p.m = p.n = p.k = N; p.a = a; p.lda = N; p.b = b; p.ldb = N; p.c = cref; p.ldc = N;
  p.alpha = 1.f; p.beta = 0.f; p.batch = 1;
  int reps = N >= 8192 ? 3 : 10;
  run<128, 128, 8, 8, 8, 2>(p, reps, nullptr, "ref 128x128x8 8x8 minb2");
  p.c = c;
  run<128, 256, 8, 8, 16, 1>(p, reps, cref, "128x256x8 8x16 minb1");
  run<128, 128, 16, 8, 8, 1>(p, reps, cref, "128x128x16 8x8 minb1");
  run<64, 64, 16, 4, 4, 2>(p, reps, cref, "64x64x16 4x4 (256t)");
  run<64, 64, 16, 4, 8, 2>(p, reps, cref, "64x64x16 4x8 (128t)");
  run<64, 64, 16, 8, 4, 2>(p, reps, cref, "64x64x16 8x4 (128t)");
  run<64, 64, 16, 8, 8, 2>(p, reps, cref, "64x64x16 8x8 (64t)");
  run<64, 64, 32, 8, 8, 2>(p, reps, cref, "64x64x32 8x8 (64t)");
  run<64, 128, 16, 4, 8, 2>(p, reps, cref, "64x128x16 4x8 (256t)");
  run<128, 64, 16, 8, 4, 2>(p, reps, cref, "128x64x16 8x4 (256t)");
  run<64, 128, 16, 8, 8, 2>(p, reps, cref, "64x128x16 8x8 (128t)");
  run<32, 64, 16, 4, 8, 2>(p, reps, cref, "32x64x16 4x8 (64t)");
  return 0;
}
