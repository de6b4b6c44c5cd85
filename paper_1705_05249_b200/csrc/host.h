// host.h — host-side plumbing shared by the translation units of
// libtbgemm.so (tbgemm.cu: C-ABI + state; sgemm.cu / sgemm_tma.cu: FFMA
// dispatch; hgemm.cu / hgemm_small.cu: tcgen05 dispatch).  Splitting the
// kernels over several TUs lets nvcc build them in parallel.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <utility>

#include "common.cuh"
#include "tbgemm.h"

namespace tb {
namespace host {

// One call, canonicalised to a column-major problem (tbgemm.cu: canonicalize).
struct Call {
  int prec, layout, ta, tbt;
  int64_t m, n, k;
  Problem p;
  int offs_aligned;            // generic batched: host-asserted offset alignment
  const tb_gemm_config* cfg;   // NULL: shape routing (built-in)
  const ConvGeom* conv;        // tb_convgemm: op(A) gathered from an image
  int flags;
  cudaStream_t stream;
};

// Raster group height requested by the configuration (0 = kernel default).
inline int cfg_group_m(const Call& c, int dflt) {
  return (c.cfg && c.cfg->GROUP_M > 0) ? c.cfg->GROUP_M : dflt;
}

// Thread-local state of the last call (tbgemm.cu).
char* err_buf();          // 256 bytes
void set_err(const char* what, cudaError_t e);
void record(const char* name, dim3 grid, dim3 block, int cluster, int smem, int64_t tiles);
int check_launch(const char* what);
int sm_count();
inline int sms_or_default() {
  const int s = sm_count();
  return s > 0 ? s : 148;
}
inline int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  return dev;
}

// Per-device dynamic shared-memory opt-in (a function attribute).
struct SmemAttr {
  std::atomic<uint64_t> devs{0};
};
template <typename K>
int ensure_smem(SmemAttr& st, K kern, int bytes) {
  const uint64_t bit = 1ull << (current_device() & 63);
  if (st.devs.load(std::memory_order_acquire) & bit) return TB_OK;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) {
    set_err("cudaFuncSetAttribute", e);
    return TB_ERR_CUDA;
  }
  st.devs.fetch_or(bit, std::memory_order_acq_rel);
  return TB_OK;
}

// Launch with programmatic dependent launch (PDL; common.cuh grid_dep_wait)
// and, when cluster > 1, a runtime cluster dimension.  TB_NO_PDL=1 in the
// environment turns PDL off (A/B measurement).
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("TB_NO_PDL");
    return !(e && e[0] == '1');
  }();
  return on;
}
template <typename... KArgs, typename... Args>
int launch_ex(const char* what, void (*kern)(KArgs...), dim3 grid, dim3 block, int smem, cudaStream_t stream,
              int cluster, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute la[2];
  int na = 0;
  if (cluster > 1) {
    la[na].id = cudaLaunchAttributeClusterDimension;
    la[na].val.clusterDim.x = static_cast<unsigned>(cluster);
    la[na].val.clusterDim.y = 1;
    la[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl_enabled()) {
    la[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    la[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = static_cast<size_t>(smem);
  cfg.stream = stream;
  cfg.attrs = la;
  cfg.numAttrs = na;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
  if (e != cudaSuccess) {
    set_err(what, e);
    return TB_ERR_CUDA;
  }
  return TB_OK;
}

// 3-D tensor map (FP16 or FP32): dims {contig, other, batch}, box {box0, box1, 1}.
int make_map(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t batch, uint64_t ld,
             uint64_t stride, uint32_t box0, uint32_t box1,
             CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_FLOAT16, uint64_t es = 2,
             CUtensorMapSwizzle swizzle = CU_TENSOR_MAP_SWIZZLE_128B, uint32_t box2 = 1);

inline bool aligned_elems(const void* base, int64_t off, int64_t elem, int64_t vec_bytes) {
  return ((reinterpret_cast<uintptr_t>(base) + off * elem) % vec_bytes) == 0;
}

// Wave-barrier counter slot for (device, stream), or nullptr (tbgemm.cu).
unsigned int* wave_counter(cudaStream_t stream);
// Split-K partial workspace of `bytes` for (device, stream), or nullptr (tbgemm.cu).
void* splitk_workspace(cudaStream_t stream, size_t bytes);
// Per-(device, stream) growable scratch for repacked operands (tbgemm.cu);
// nullptr while the stream is capturing a graph and the slot is too small.
void* pack_workspace(cudaStream_t stream, size_t bytes);
// Fold `n` more launches into the last launch record and tag its name.
void note_extra_launches(int n, const char* suffix);
// Copy the operands whose pitch / base / stride break 16-byte alignment into
// scratch with pitches rounded up to 16 bytes (es: element size); c2 is c
// pointing at the copies.  TB_OK, -1 when not applicable (nothing to copy,
// per-instance offset arrays, no scratch), or a CUDA error.
int repack_operands(const Call& c, int es, Call& c2, int& launches);

// Dispatchers.
int dispatch_sgemm(const Call& c);                                   // sgemm.cu
int dispatch_sgemm_tma(const Call& c, int tile, int mwg, int nwg, int ks = 1);   // sgemm_tma.cu
int dispatch_hgemm(const Call& c);                                   // hgemm.cu
int dispatch_hsmall_any(const Call& c);                              // hgemm_small.cu
int launch_hscale(const Call& c);                                    // hgemm.cu
int dispatch_hconv(const Call& c);                                   // hgemm.cu
int dispatch_sconv(const Call& c);                                   // sgemm.cu

}  // namespace host
}  // namespace tb
