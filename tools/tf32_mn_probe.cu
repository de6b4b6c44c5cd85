// tf32_mn_probe.cu — find the shared-memory layout tcgen05.mma.kind::tf32
// accepts for an MN-major FP32 operand (dev tool, not part of the library).
//
// One CTA computes D(128 x 64) = A(128 x 32) * B(32 x 64) with A MN-major
// (m contiguous in global: A[k][m]) and B K-major (B[n][k], the known-good
// layout of sgemm_tf32_tc.cuh).  A lands in shared memory as 4 chunks of
// 32 m x 32 k through TMA with swizzle `swz`; the MMA descriptor of A uses
// layout type `lt`, leading / stride byte offsets `lbo` / `sbo` and a
// per-K8-step start advance `kstep`.  Every variant's max |D - ref| is
// printed (ref on the host in double precision of TF32-rounded inputs).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O2 \
//        -I paper_1705_05249_b200/csrc -I include -o tools/tf32_mn_probe tools/tf32_mn_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "sgemm_tf32_tc.cuh"

using namespace tb;

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t lt) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(lt) << 61;
  return d;
}

__global__ void probe_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                             float* D, uint32_t lt, uint32_t lbo, uint32_t sbo, uint32_t kstep) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_align1024(smem_raw);
  uint8_t* sA = smem;              // 16 KB
  uint8_t* sB = smem + 16384;      // 8 KB
  __shared__ uint64_t bar_load, bar_mma;
  __shared__ uint32_t tmem_holder;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&bar_load, 1);
    mbar_init(&bar_mma, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tmem_holder, 64);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_holder;
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar_load, 16384 + 8192);
    for (int c = 0; c < 4; ++c) tma_load_3d(sA + c * 4096, &tmA, &bar_load, 32 * c, 0, 0);
    tma_load_3d(sB, &tmB, &bar_load, 0, 0, 0);
    mbar_wait(&bar_load, 0);
    tc_fence_after();
    const uint32_t idesc = umma_idesc_tf32(128, 64, 1, 0);
    const uint32_t a_addr = smem_u32(sA), b_addr = smem_u32(sB);
    for (int kk = 0; kk < 4; ++kk) {
      const uint64_t ad = make_desc(a_addr + kk * kstep, lbo, sbo, lt);
      const uint64_t bd = umma_desc_sw128(b_addr + kk * 32, 16, 1024);
      tc_mma_tf32(tmem, ad, bd, idesc, kk != 0 ? 1u : 0u);
    }
    tc_commit(&bar_mma);
  }
  __syncwarp();
  mbar_wait(&bar_mma, 0);
  tc_fence_after();
  for (int cb = 0; cb < 2; ++cb) {
    uint32_t v[32];
    tmem_ld_32x32b_x32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + cb * 32, v);
    tmem_ld_wait();
    for (int j = 0; j < 32; ++j) D[(warp * 32 + lane) * 64 + cb * 32 + j] = __uint_as_float(v[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 64);
  }
}

static float tf32r(float x) {  // round-to-nearest to TF32 (10-bit mantissa); truncation also checked below
  uint32_t u;
  memcpy(&u, &x, 4);
  u = (u + 0x1000u) & ~0x1FFFu;
  float r;
  memcpy(&r, &u, 4);
  return r;
}

int main() {
  const int M = 128, N = 64, K = 32;
  std::vector<float> hA(K * M), hB(N * K);
  uint32_t s = 12345;
  auto rnd = [&] { s = s * 1664525u + 1013904223u; return ((s >> 8) / 16777216.0f) * 2.f - 1.f; };
  for (auto& x : hA) x = rnd();
  for (auto& x : hB) x = rnd();
  std::vector<double> ref(M * N);
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double acc = 0;
      for (int k = 0; k < K; ++k) acc += static_cast<double>(tf32r(hA[k * M + m])) * tf32r(hB[n * K + k]);
      ref[m * N + n] = acc;
    }
  float *dA, *dB, *dD;
  cudaMalloc(&dA, hA.size() * 4);
  cudaMalloc(&dB, hB.size() * 4);
  cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, hA.data(), hA.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), hB.size() * 4, cudaMemcpyHostToDevice);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  EncodeFn enc = reinterpret_cast<EncodeFn>(fp);
  CUtensorMap mB;
  {
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(N), 1};
    cuuint64_t str[2] = {K * 4ull, K * N * 4ull};
    cuuint32_t box[3] = {32, 64, 1}, es[3] = {1, 1, 1};
    enc(&mB, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, dB, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  const CUtensorMapSwizzle swz[2] = {CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B};
  const char* swz_name[2] = {"SW128", "SW128_ATOM32B"};
  const uint32_t lts[2] = {1, 2};
  const uint32_t lbos[4] = {4096, 1024, 4096, 512};
  const uint32_t sbos[4] = {1024, 4096, 512, 4096};
  const uint32_t ksteps[2] = {1024, 512};
  std::vector<float> hD(M * N);
  for (int si = 0; si < 2; ++si) {
    CUtensorMap mA;
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(M), static_cast<cuuint64_t>(K), 1};
    cuuint64_t str[2] = {M * 4ull, M * K * 4ull};
    cuuint32_t box[3] = {32, 32, 1}, es[3] = {1, 1, 1};
    CUresult r = enc(&mA, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, dA, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     swz[si], CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      printf("encode %s failed %d\n", swz_name[si], static_cast<int>(r));
      continue;
    }
    for (uint32_t lt : lts)
      for (int bi = 0; bi < 4; ++bi)
        for (uint32_t ks : ksteps) {
          cudaMemset(dD, 0, M * N * 4);
          probe_kernel<<<1, 128, 32768>>>(mA, mB, dD, lt, lbos[bi], sbos[bi], ks);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) {
            printf("%s lt=%u lbo=%u sbo=%u kstep=%u: %s\n", swz_name[si], lt, lbos[bi], sbos[bi], ks,
                   cudaGetErrorString(e));
            return 1;
          }
          cudaMemcpy(hD.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
          double err = 0;
          for (int i = 0; i < M * N; ++i) err = fmax(err, fabs(hD[i] - ref[i]));
          printf("%-14s lt=%u lbo=%5u sbo=%5u kstep=%4u  max_err=%.3g%s\n", swz_name[si], lt, lbos[bi], sbos[bi], ks,
                 err, err < 0.05 ? "  <== MATCH" : "");
        }
  }
  return 0;
}
