// TMA-staged streaming for the elementwise kernels (sm_100a).
//
// Every CTA is persistent and walks tiles t = blockIdx.x + j*gridDim.x of the
// input arrays.  One elected thread issues bulk copies (cp.async.bulk
// global->shared, completion counted on an mbarrier by transaction bytes)
// for up to STAGES tiles ahead; all threads wait on the stage's mbarrier
// phase, pull their elements out of shared memory (LDS.128, conflict-free),
// release the stage with a CTA barrier, and then compute and store
// (st.global.cs: outputs are written once).  Loads therefore stay in flight
// while the FP64 pipe works, without spending registers on prefetch and
// without per-thread 64-bit address arithmetic on the load side.
#pragma once

#include <cstdint>

namespace vem {
namespace tma {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}

// Waits for the stage's phase.  With VEM_MBAR_HINT the waiting thread asks to
// be suspended for up to that many ns per try (it wakes when the phase
// completes) instead of re-issuing try_wait: warps that run ahead of the TMA
// stream then stop consuming issue slots.
#ifndef VEM_MBAR_HINT
#define VEM_MBAR_HINT 0
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t a = smem_addr(bar);
#if VEM_MBAR_HINT
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@P1 bra.uni DONE;\n"
      "bra.uni LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(a),
      "r"(phase), "n"(VEM_MBAR_HINT)
      : "memory");
#else
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra.uni DONE;\n"
      "bra.uni LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(a),
      "r"(phase)
      : "memory");
#endif
}

// Cross-proxy WAR: the generic-proxy LDS reads of a stage (by all threads,
// ordered before this thread by the CTA barrier) must be ordered before the
// async-proxy bulk copy that refills it.  Without this fence a refill can
// land while earlier reads of the stage are still pending (observed: rare
// elements computed from the NEXT tile's inputs).
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// bulk copy global -> shared::cta (via the cluster window of this CTA),
// completion reported to `bar` as transaction bytes; evict-first L2 policy.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
      "%4;" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Per-warp release of a TMA stage (no CTA-wide barrier): after reading its
// part of stage s, every warp's lane 0 adds 1 to the stage's counter
// (acq_rel: the warp's reads, ordered before it by __syncwarp, happen before
// the increment); the warp whose increment completes a set of `nw` learns it
// is last and refills the stage (after fence.proxy.async).  Fast warps run
// ahead of slow ones by up to STAGES - 1 tiles instead of waiting at a
// barrier every tile.  The counter only grows: arrival k of a tile is the
// last one when k % nw == nw - 1.
__device__ __forceinline__ bool stage_release_last(uint32_t* ctr, uint32_t nw) {
  uint32_t old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(smem_addr(ctr)) : "memory");
  return (old % nw) == nw - 1;
}

// Plain shared-memory atomic increment (returns the old value).  Written as
// PTX so the compiler does not wrap it in its warp-aggregation sequence
// (match/popc/shuffle per call): the histogram keys of one warp mostly differ.
__device__ __forceinline__ uint32_t smem_atomic_inc(int* p) {
  uint32_t old;
  asm volatile("atom.shared::cta.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(smem_addr(p)) : "memory");
  return old;
}
__device__ __forceinline__ uint32_t smem_atomic_add(int* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared::cta.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(smem_addr(p)), "r"(v) : "memory");
  return old;
}

// Programmatic dependent launch (the streaming kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization): `wait` blocks until
// the previous grid in the stream has completed and its memory operations
// are visible (a no-op without the attribute), so everything before it may
// only touch kernel-private state (barrier init, constant-table staging);
// `launch_dependents` lets the next grid's CTAs be scheduled as this grid's
// CTAs exit, overlapping its launch and prologue with this grid's tail.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

}  // namespace tma
}  // namespace vem
