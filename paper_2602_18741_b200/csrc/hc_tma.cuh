// hadacodec-b200: 1-D TMA bulk copies (cp.async.bulk) and mbarrier helpers.
//
// The hot kernels move contiguous pixel runs (G-buffer rows, 324-byte spectral
// rows, code rows) between HBM and shared memory with the bulk-copy engine:
// one elected thread issues the copy, completion is tracked by an mbarrier
// transaction count (loads) or a bulk group (stores).  SASS: UBLKCP.
#pragma once

#include <stdint.h>

namespace hcb {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Programmatic dependent launch: let the next kernel on the stream start its CTAs
// as ours retire, and (in the next kernel) wait until every prior grid has
// completed and flushed before touching global memory.  Both are no-ops when
// the launch carries no programmatic-serialization attribute.
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait_prior_grids() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  const uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(phase)
      : "memory");
}

// global -> shared bulk copy; bytes % 16 == 0, both addresses 16-byte aligned.
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// 2-D tensor TMA load (cp.async.bulk.tensor): box at coordinates (x, y) of the tensor
// map into shared memory (1024-byte aligned for the 128-byte swizzle).  SASS: UTMALDG.
__device__ __forceinline__ void tma_load_2d(void* dst_smem, const void* tmap, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst_smem)),
      "l"(tmap), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// global -> shared bulk copy with an L2 evict-first policy (streamed inputs).
__device__ __forceinline__ void bulk_g2s_evict_first(void* dst_smem, const void* src_gmem,
                                                     uint32_t bytes, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, "
      "[%3], %4;" ::"r"(smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// shared -> global bulk copy (bulk group); bytes % 16 == 0, 16-byte aligned.
__device__ __forceinline__ void bulk_s2g(void* dst_gmem, const void* src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst_gmem),
               "r"(smem_u32(src_smem)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }

// Wait until at most N committed bulk groups are still READING shared memory.
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

// ---- warp-wide issue (`_w`): the whole warp calls, elect.sync inside the asm picks one lane
// (the lowest active, so the same lane every time: bulk groups are per thread).  Issued from
// `if (tid == 0)` with register operands, every UBLKCP / UTMALDG is wrapped by the compiler in a
// per-thread ELECT / BRA.U.ANY loop (tools/mma_probe4.cu measured the same for tcgen05.mma:
// 54 -> 17 cycles per instruction); warp-wide the instruction is straight-line.
#define HC_ELECT_PRED "elect.sync _|e, 0xffffffff;\n"
__device__ __forceinline__ void mbar_arrive_expect_tx_w(uint64_t* bar, uint32_t bytes) {
  asm volatile("{\n.reg .pred e;\n" HC_ELECT_PRED
               "@e mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;\n}\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_w(uint64_t* bar) {
  asm volatile("{\n.reg .pred e;\n" HC_ELECT_PRED "@e mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n}\n" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_g2s_w(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile("{\n.reg .pred e;\n" HC_ELECT_PRED
               "@e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n}\n" ::"r"(
                   smem_u32(dst_smem)),
               "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_g2s_evict_first_w(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                                       uint64_t* bar, uint64_t policy) {
  asm volatile("{\n.reg .pred e;\n" HC_ELECT_PRED
               "@e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, "
               "[%3], %4;\n}\n" ::"r"(smem_u32(dst_smem)),
               "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
               : "memory");
}
__device__ __forceinline__ void tma_load_2d_w(void* dst_smem, const void* tmap, int x, int y, uint64_t* bar) {
  asm volatile("{\n.reg .pred e;\n" HC_ELECT_PRED
               "@e cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
               "%3}], [%4];\n}\n" ::"r"(smem_u32(dst_smem)),
               "l"(tmap), "r"(x), "r"(y), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_s2g_w(void* dst_gmem, const void* src_smem, uint32_t bytes) {
  asm volatile("{\n.reg .pred e;\n" HC_ELECT_PRED "@e cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n}\n" ::"l"(
                   dst_gmem),
               "r"(smem_u32(src_smem)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit_w() {
  asm volatile("{\n.reg .pred e;\n" HC_ELECT_PRED "@e cp.async.bulk.commit_group;\n}\n" ::: "memory");
}

// Make generic-proxy shared-memory writes visible to the async (bulk) proxy.
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

}  // namespace hcb
