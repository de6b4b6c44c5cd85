// hgemm_small.cu — packed small-instance tcgen05 HGEMM (hgemm_tc_small.cuh):
// m, n <= 64 per instance, P = 128/MI instances per UMMA tile.
#include <cstring>

#include "hgemm_tc_small.cuh"
#include "host.h"

namespace tb {
namespace host {
namespace {

template <int MI, int NI, bool AMN, bool BMN, bool VEC, bool K32>
int launch_hs(const Call& c) {
  using Cfg = HsCfg<MI, NI>;
  const Problem& p = c.p;
  const int64_t total = (p.batch + Cfg::P - 1) / Cfg::P;
  auto kern = hgemm_tc_small_kernel<MI, NI, AMN, BMN, VEC, K32>;
  static SmemAttr attr;  // per instantiation, per device
  if (int rc = ensure_smem(attr, kern, Cfg::SMEM_BYTES)) return rc;
  const int sms = sms_or_default();
  const int64_t g = total < sms ? total : sms;
  dim3 grid(static_cast<unsigned>(g)), block(Cfg::THREADS);
  if (int rc = launch_ex("hgemm_tc_small launch", kern, grid, block, Cfg::SMEM_BYTES, c.stream, 1, p, total)) return rc;
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

bool small_aligned(const Call& c) {
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

template <bool AMN, bool BMN>
int launch_hs32_tma(const Call& c, const CUtensorMap& ta, const CUtensorMap& tbm) {
  using Cfg = Hs32Cfg;
  const Problem& p = c.p;
  const int64_t total = (p.batch + Cfg::P - 1) / Cfg::P;
  auto kern = hgemm_tc_small32_tma_kernel<AMN, BMN>;
  static SmemAttr attr;
  if (int rc = ensure_smem(attr, kern, Cfg::SMEM_BYTES)) return rc;
  const int sms = sms_or_default();
  const int64_t g = total < sms ? total : sms;
  dim3 grid(static_cast<unsigned>(g)), block(Cfg::THREADS);
  if (int rc = launch_ex("hgemm_tc_small32_tma launch", kern, grid, block, Cfg::SMEM_BYTES, c.stream, 1, ta, tbm, p,
                         total))
    return rc;
  char name[64];
  snprintf(name, sizeof(name), "hgemm_tc_small_32x32_p4_%c%c_tma", AMN ? 'm' : 'k', BMN ? 'n' : 'k');
  record(name, grid, block, 1, Cfg::SMEM_BYTES, total);
  return check_launch("hgemm_tc_small32_tma launch");
}

// k, m, n <= 32 over an arithmetic batch of >= 4 instances with 16-byte
// aligned rows / strides: one TMA box per operand per tile (Hs32Cfg).
// Returns -1 when the problem does not qualify.
int dispatch_hs32_tma(const Call& c) {
  const Problem& p = c.p;
  if (p.m > 32 || p.n > 32 || p.k > 32 || p.k < 1 || p.batch < 4 || p.a_offs || p.b_offs) return -1;
  if (p.batch > 0x7ffffff0LL || (c.flags & TB_FLAG_NO_TMA)) return -1;
  if ((p.lda % 8) || (p.ldb % 8) || (p.stride_a % 8) || (p.stride_b % 8) || !aligned_elems(p.a, p.a_off, 2, 16) ||
      !aligned_elems(p.b, p.b_off, 2, 16))
    return -1;
  const bool amn = !p.a_kcontig, bmn = p.b_ncontig;
  const __half* A = static_cast<const __half*>(p.a) + p.a_off;
  const __half* B = static_cast<const __half*>(p.b) + p.b_off;
  CUtensorMap ta, tbm;
  memset(&ta, 0, sizeof(ta));
  memset(&tbm, 0, sizeof(tbm));
  const CUtensorMapDataType F16 = CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  const CUtensorMapSwizzle SW64 = CU_TENSOR_MAP_SWIZZLE_64B;
  int rc = amn ? make_map(&ta, A, p.m, p.k, p.batch, p.lda, p.stride_a, 32, 32, F16, 2, SW64, 4)
               : make_map(&ta, A, p.k, p.m, p.batch, p.lda, p.stride_a, 32, 32, F16, 2, SW64, 4);
  if (rc != TB_OK) return rc;
  rc = bmn ? make_map(&tbm, B, p.n, p.k, p.batch, p.ldb, p.stride_b, 32, 32, F16, 2, SW64, 4)
           : make_map(&tbm, B, p.k, p.n, p.batch, p.ldb, p.stride_b, 32, 32, F16, 2, SW64, 4);
  if (rc != TB_OK) return rc;
  if (!amn && !bmn) return launch_hs32_tma<false, false>(c, ta, tbm);
  if (!amn && bmn) return launch_hs32_tma<false, true>(c, ta, tbm);
  if (amn && !bmn) return launch_hs32_tma<true, false>(c, ta, tbm);
  return launch_hs32_tma<true, true>(c, ta, tbm);
}

template <bool AMN, bool BMN>
int launch_hs64_tma(const Call& c, const CUtensorMap& ta, const CUtensorMap& tbm) {
  using Cfg = Hs64Cfg;
  const Problem& p = c.p;
  const int64_t total = (p.batch + Cfg::P - 1) / Cfg::P;
  auto kern = hgemm_tc_small64_tma_kernel<AMN, BMN>;
  static SmemAttr attr;
  if (int rc = ensure_smem(attr, kern, Cfg::SMEM_BYTES)) return rc;
  const int sms = sms_or_default();
  const int64_t g = total < sms ? total : sms;
  dim3 grid(static_cast<unsigned>(g)), block(Cfg::THREADS);
  if (int rc = launch_ex("hgemm_tc_small64_tma launch", kern, grid, block, Cfg::SMEM_BYTES, c.stream, 1, ta, tbm, p,
                         total))
    return rc;
  char name[64];
  snprintf(name, sizeof(name), "hgemm_tc_small_64x64_p2_%c%c_tma", AMN ? 'm' : 'k', BMN ? 'n' : 'k');
  record(name, grid, block, 1, Cfg::SMEM_BYTES, total);
  return check_launch("hgemm_tc_small64_tma launch");
}

// 32 < max(m, n, k) and m, n, k <= 64 over an arithmetic batch of >= 2
// instances with 16-byte aligned rows / strides: one SW128 TMA box per
// operand per tile (Hs64Cfg).  Returns -1 when the problem does not qualify.
int dispatch_hs64_tma(const Call& c) {
  const Problem& p = c.p;
  if (p.m > 64 || p.n > 64 || p.k > 64 || p.k < 1 || p.batch < 2 || p.a_offs || p.b_offs) return -1;
  if (p.m <= 32 && p.n <= 32 && p.k <= 32) return -1;  // the 32-wide kernel's
  if (p.batch > 0x7ffffff0LL || (c.flags & TB_FLAG_NO_TMA)) return -1;
  if ((p.lda % 8) || (p.ldb % 8) || (p.stride_a % 8) || (p.stride_b % 8) || !aligned_elems(p.a, p.a_off, 2, 16) ||
      !aligned_elems(p.b, p.b_off, 2, 16))
    return -1;
  const bool amn = !p.a_kcontig, bmn = p.b_ncontig;
  const __half* A = static_cast<const __half*>(p.a) + p.a_off;
  const __half* B = static_cast<const __half*>(p.b) + p.b_off;
  CUtensorMap ta, tbm;
  memset(&ta, 0, sizeof(ta));
  memset(&tbm, 0, sizeof(tbm));
  const CUtensorMapDataType F16 = CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  const CUtensorMapSwizzle SW128 = CU_TENSOR_MAP_SWIZZLE_128B;
  int rc = amn ? make_map(&ta, A, p.m, p.k, p.batch, p.lda, p.stride_a, 64, 64, F16, 2, SW128, 2)
               : make_map(&ta, A, p.k, p.m, p.batch, p.lda, p.stride_a, 64, 64, F16, 2, SW128, 2);
  if (rc != TB_OK) return rc;
  rc = bmn ? make_map(&tbm, B, p.n, p.k, p.batch, p.ldb, p.stride_b, 64, 64, F16, 2, SW128, 2)
           : make_map(&tbm, B, p.k, p.n, p.batch, p.ldb, p.stride_b, 64, 64, F16, 2, SW128, 2);
  if (rc != TB_OK) return rc;
  if (!amn && !bmn) return launch_hs64_tma<false, false>(c, ta, tbm);
  if (!amn && bmn) return launch_hs64_tma<false, true>(c, ta, tbm);
  if (amn && !bmn) return launch_hs64_tma<true, false>(c, ta, tbm);
  return launch_hs64_tma<true, true>(c, ta, tbm);
}

}  // namespace

int dispatch_hsmall_any(const Call& c) {
  if (const int rc = dispatch_hs32_tma(c); rc >= 0) return rc;
  if (const int rc = dispatch_hs64_tma(c); rc >= 0) return rc;
  if (small_aligned(c)) return dispatch_hsmall<true>(c);
  return dispatch_hsmall<false>(c);
}

}  // namespace host
}  // namespace tb
