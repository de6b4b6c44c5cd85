// common.cuh — shared device helpers for the sm_100a GEMM kernels.
//
// Thin inline-PTX wrappers for mbarrier, TMA (cp.async.bulk.tensor),
// tcgen05 (alloc / mma / commit / ld) and the canonical problem descriptor
// that every kernel consumes.  Written directly against the PTX ISA for
// sm_100a; no CUTLASS/CuTe.
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace tb {

// ---------------------------------------------------------------------------
// Canonical problem: column-major C (m x n, ldc) = alpha * A' * B' + beta * C
// where (after folding row-major layouts into swapped operands, see
// tbgemm.cu:canonicalize) op(A)(i,kk) lives at
//     a_kcontig ? a[i*lda + kk] : a[i + kk*lda]
// and op(B)(kk,j) at
//     b_ncontig ? b[j + kk*ldb] : b[kk + j*ldb].
// Instance z of a batch adds off(z) = offs ? offs[z] : base + z*stride.
// ---------------------------------------------------------------------------
struct Problem {
  int64_t m, n, k;
  const void* a; int64_t lda; int64_t a_off; int64_t stride_a; const int64_t* a_offs;
  const void* b; int64_t ldb; int64_t b_off; int64_t stride_b; const int64_t* b_offs;
  void* c;       int64_t ldc; int64_t c_off; int64_t stride_c; const int64_t* c_offs;
  float alpha, beta;
  const float* alphas; const float* betas;
  int64_t batch;
  int a_kcontig, b_ncontig;
};

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

// Implicit-GEMM (convgemm) geometry: op(A)(q, r) of the canonical problem is
// the im2col matrix entry col[r][q] (reference extras.py:56-109) gathered
// from the channel-major image of instance z at p.a + off_a(z):
//   r = (ch*kh + ky)*kw + kx,  q = oy*out_w + ox,
//   y = oy*stride_h + ky*dil_h - pad_h,  x = ox*stride_w + kx*dil_w - pad_w,
//   value = image[ch][y][x] inside the image, 0 in the padding.
struct ConvGeom {
  int channels, height, width, kh, kw;
  int pad_h, pad_w, stride_h, stride_w, dil_h, dil_w;
  int out_h, out_w;
};

__device__ __forceinline__ int64_t inst_off(int64_t base, int64_t stride,
                                            const int64_t* offs, int64_t z) {
  return offs ? __ldg(offs + z) : base + z * stride;
}
__device__ __forceinline__ float inst_alpha(const Problem& p, int64_t z) {
  return p.alphas ? __ldg(p.alphas + z) : p.alpha;
}
__device__ __forceinline__ float inst_beta(const Problem& p, int64_t z) {
  return p.betas ? __ldg(p.betas + z) : p.beta;
}

// Programmatic dependent launch: kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization (host.h launch_ex), so a
// CTA may start while the previous kernel on the stream is still finishing.
// Everything before this call (barrier init, TMEM allocation, tensor-map
// prefetch) overlaps that tail; nothing before it touches global memory the
// previous kernel may read or write.  A no-op when launched without PDL.
__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// Let the next kernel on the stream launch now: its CTAs take SMs as ours
// exit and run their prologue, then wait in grid_dep_wait() for this grid's
// completion — so back-to-back GEMMs overlap prologue with tail.
__device__ __forceinline__ void grid_dep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Reference epilogue (compute.py:408-412, 458-463; level3.py:125-132):
//   alpha == 0 or k == 0 : beta == 0 ? 0 : beta*c      (A/B never read)
//   beta == 0            : alpha*acc                    (C never read)
//   otherwise            : (alpha*acc) + (beta*c), each op rounded (no FMA)
struct Epi {
  float alpha, beta;
  bool skip_ab;   // alpha == 0 || k == 0
  __device__ __forceinline__ bool reads_c() const { return beta != 0.0f; }
  __device__ __forceinline__ float apply(float acc, float cval) const {
    if (skip_ab) return beta == 0.0f ? 0.0f : __fmul_rn(beta, cval);
    float v = __fmul_rn(alpha, acc);
    if (beta != 0.0f) v = __fadd_rn(v, __fmul_rn(beta, cval));
    return v;
  }
};

// ---------------------------------------------------------------------------
// Shared-memory / mbarrier / fences
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Round a dynamic shared-memory pointer up to 1024 B (SWIZZLE_128B atoms) by
// pointer arithmetic, so the result keeps the shared address space and the
// compiler emits LDS/STS (a uintptr_t round trip would make it generic).
__device__ __forceinline__ uint8_t* smem_align1024(uint8_t* base) {
  return base + ((1024u - (smem_u32(base) & 1023u)) & 1023u);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// ---------------------------------------------------------------------------
// TMA
// ---------------------------------------------------------------------------
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* smem_dst, const CUtensorMap* m, uint64_t* bar,
                                            int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// ---------------------------------------------------------------------------
// tcgen05 (5th-gen tensor cores, TMEM accumulators)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// D[tmem] (+)= A[smem] * B[smem], kind::f16 (FP16 inputs, FP32 accumulate)
__device__ __forceinline__ void tc_mma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                           uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive on an mbarrier when all previously issued tcgen05.mma complete.
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}
// 32 lanes x 32 columns of 32-bit: lane i of the warp receives row (quadrant
// base + i), registers r[j] = column (col + j).
__device__ __forceinline__ void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_32x32b_x16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// UMMA shared-memory matrix descriptor (sm_100 "version 1"):
//   [0,14) start>>4 | [16,30) LBO>>4 | [32,46) SBO>>4 | [46,48) version=1 |
//   [49,52) base offset | [52] LBO mode | [61,64) layout (2 = SWIZZLE_128B)
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}

// SWIZZLE_64B operand descriptor (layout type 4): 64-byte rows, 8-row atoms.
__device__ __forceinline__ uint64_t umma_desc_sw64(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(4) << 61;
  return d;
}

// Instruction descriptor, kind::f16: F16 x F16 -> F32.
//   [4,6) c_format=1 (F32) | [7,10) a_format=0 (F16) | [10,13) b_format=0 |
//   [15] a_major (1 = MN) | [16] b_major | [17,23) N>>3 | [24,29) M>>4
__host__ __device__ constexpr uint32_t umma_idesc_f16(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (static_cast<uint32_t>(a_mn) << 15) | (static_cast<uint32_t>(b_mn) << 16) |
         (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(M >> 4) << 24);
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

}  // namespace tb

namespace tb {
// ---------------------------------------------------------------------------
// FP32 register-tile outer product on the paired FFMA pipe (FFMA2).
// acc2[i2][j] holds rows (2*i2, 2*i2+1) of column j.  Each lane of
// fma.rn.f32x2 is an ordinary round-to-nearest FP32 fma, so the chain per
// element is bitwise the scalar __fmaf_rn chain; FFMA2 just issues two of
// them per instruction (b[j] is the broadcast scalar operand in SASS).
// ---------------------------------------------------------------------------
template <int TM, int TN>
__device__ __forceinline__ void outer_ffma2(float2 (&acc2)[TM / 2][TN], const float (&af)[TM],
                                            const float (&bf)[TN]) {
#pragma unroll
  for (int i2 = 0; i2 < TM / 2; ++i2)
#pragma unroll
    for (int j = 0; j < TN; ++j)
      acc2[i2][j] = __ffma2_rn(make_float2(bf[j], bf[j]), make_float2(af[2 * i2], af[2 * i2 + 1]),
                               acc2[i2][j]);
}
// ---------------------------------------------------------------------------
// cp.async (LDGSTS): 16-byte global -> shared, zero-filling past src_bytes
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp_async_16(void* smem_dst, const void* gsrc, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem_dst)), "l"(gsrc),
               "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
}  // namespace tb
