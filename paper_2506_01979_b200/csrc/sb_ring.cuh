// sb_ring.cuh — warp-specialised TMA bulk-copy ring (sm_100a).
//
// One producer warp streams row chunks global -> shared with cp.async.bulk (the 1-D
// TMA engine, SASS UBLKCP) completing on per-stage mbarriers; consumer warps wait on
// the "full" barrier, read the chunk with 16-byte LDS and release the stage on the
// "empty" barrier.  Bytes in flight per SM = the whole ring, independent of register
// allocation, so the HBM pipe stays full while consumers do math and per-unit
// epilogues.
#pragma once
#include <stdint.h>

namespace sb {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// One probe of a phase (the warp sleeps in hardware until the phase completes or a
// system-dependent limit expires).  SB_WAIT_HINT=ns builds pass a suspend-time hint: it
// did not shorten k_rows_tma's waits measurably and doubled k_select_tma's time (its
// waits on thread arrivals woke late), so the default passes none.
#ifdef SB_WAIT_HINT
#define SB_TRYWAIT_ASM " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, " SB_STR(SB_WAIT_HINT) ";\n"
#define SB_STR(x) SB_STR2(x)
#define SB_STR2(x) #x
#else
#define SB_TRYWAIT_ASM " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
#endif
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n" SB_TRYWAIT_ASM
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Blocking wait on a phase.  A watchdog traps after ~2^24 expired probes (seconds): a
// protocol bug then surfaces as a launch error instead of a hung GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  for (uint32_t tries = 0;; ++tries) {
    if (mbar_try(bar, parity)) break;
    if (tries > (1u << 24)) __trap();
  }
}
// The consumer warps' waits for a filled stage of the streaming kernels (k_rows_tma,
// k_conf_tma, k_astep): try_wait + branch per probe, no watchdog (two instructions; these
// waits sit on the issue-bound critical path, where the counted loop cost ~2 % of the C4
// verify time).  Only there: in k_select_tma the same tight loop doubled the kernel time
// (0.25 -> 0.45 ms on C4), so every other wait keeps mbar_wait.
__device__ __forceinline__ void mbar_wait_spin(uint64_t* bar, uint32_t parity) {
#ifdef SB_WATCHDOG
  mbar_wait(bar, parity);
#else
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n" SB_TRYWAIT_ASM
      " @!p bra WAIT_%=;\n}\n" ::"r"(0), "r"(smem_u32(bar)), "r"(parity)
      : "memory");
#endif
}
// Waits that last whole units (an epilogue warp waiting for the consumers' partials):
// the same hardware sleep.
__device__ __forceinline__ void mbar_wait_parked(uint64_t* bar, uint32_t parity) { mbar_wait(bar, parity); }
// Per-thread 16-byte asynchronous copies (LDGSTS) for the per-warp rings of the
// warp-per-unit kernels: a lane copies, commits, waits for and reads only its own data.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
// 1-D bulk copy global -> shared, completion (bytes) signalled on bar.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint4 lds128(const void* p) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "r"(smem_u32(p)));
  return r;
}
// named barrier among the consumer warps only (id 1; the producer never joins)
__device__ __forceinline__ void consumer_sync(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

// Ring position bookkeeping shared by producer and consumers.
template <int NS>
struct RingPos {
  int stage = 0;
  uint32_t phase = 0;
  __device__ __forceinline__ void advance() {
    if (++stage == NS) {
      stage = 0;
      phase ^= 1u;
    }
  }
};

}  // namespace sb
