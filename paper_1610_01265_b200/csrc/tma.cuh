// TMA / mbarrier helpers shared by the pipelined stencil kernels (sm_100a).
// Measured constraint (tools/probe/tma_probe2.cu): the innermost box origin of a
// cp.async.bulk.tensor load must be 16 B aligned -- an odd FP64 column origin
// raises an illegal-instruction fault; negative (OOB) origins are fine.
#pragma once

#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>

#include "sts_common.cuh"

namespace sts {
namespace tma {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// Wait for the phase with parity `parity` to complete.  With a suspend-time hint the
// waiting thread is suspended in hardware until the phase completes (or the hint, in ns,
// elapses) instead of re-issuing try_wait: measured on the anisotropic merged PCG pass,
// the producers' spin on their empty barriers was 23 % of all executed instructions
// (ncu source page), issue slots taken from the consumer warps of the same SM.
#ifndef STS_MBAR_HINT
#define STS_MBAR_HINT 0x989680
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#if STS_MBAR_HINT > 0
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "n"(STS_MBAR_HINT)
      : "memory");
#else
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
#endif
}
__device__ __forceinline__ void tma3(double* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
// L2 prefetch of a tensor box (no shared memory, no mbarrier): the producers issue the
// boxes of a plane PF planes ahead, so the bytes in flight from DRAM are no longer bounded
// by the shared-memory ring (the later cp.async.bulk.tensor of that plane hits L2)
__device__ __forceinline__ void tma3_prefetch(const CUtensorMap* map, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];\n" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
// one lane of a converged warp (the isotropic producer warp runs its loop warp-wide and
// issues from the elected lane: the TMA operands then stay in uniform registers -- a
// single-thread producer made the compiler wrap every cp.async.bulk.tensor in an
// ELECT / R2UR.BROADCAST loop, ~20 instructions per box, and the producer's issue
// rate limited the merged isotropic PCG pass; ncu source page, DESIGN.md §5.4.  The
// anisotropic producer, ~60 % busy, measured no gain from it and keeps one thread.)
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "elect.sync _|P, 0xffffffff;\n"
      "selp.u32 %0, 1, 0, P;\n"
      "}\n"
      : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

// ---------------------------------------------------------------- host side
inline PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    STS_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || p == nullptr)
      throw Error{STS_ERR_CUDA, "cuTensorMapEncodeTiled is not available from the driver"};
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

inline void encode(CUtensorMap* m, const double* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides,
                   const cuuint32_t* box) {
  const cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, const_cast<double*>(base), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error{STS_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")"};
}

// plain [nplanes][n2][n3] field (component 0 at base)
inline void map_plain(CUtensorMap* m, const double* base, const Geo& G, int nplanes, int bw, int bh) {
  const cuuint64_t dims[3] = {(cuuint64_t)G.n3, (cuuint64_t)G.n2, (cuuint64_t)nplanes};
  const cuuint64_t str[2] = {(cuuint64_t)G.n3 * 8, (cuuint64_t)G.plane * 8};
  const cuuint32_t box[3] = {(cuuint32_t)bw, (cuuint32_t)bh, 1};
  encode(m, base, 3, dims, str, box);
}

inline bool al16(const void* p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15) == 0; }


}  // namespace tma
}  // namespace sts
