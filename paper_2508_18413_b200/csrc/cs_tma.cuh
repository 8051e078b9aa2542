// Bulk-copy (TMA engine, cp.async.bulk) and mbarrier helpers for sm_100a.
// 1-D bulk copies move a contiguous tile global <-> shared without staging
// through registers; completion is tracked by an mbarrier transaction count.
#pragma once
#include "cs_common.cuh"

namespace cs {

CS_D unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

CS_D void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
CS_D void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
CS_D void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
CS_D void mbar_wait(uint64_t *bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// global -> shared, completes on the mbarrier's transaction count
CS_D void bulk_g2s(void *dst_smem, const void *src, unsigned bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// L2 eviction-priority policies for bulk copies (createpolicy)
CS_D uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
CS_D uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
CS_D void bulk_g2s_hint(void *dst_smem, const void *src, unsigned bytes, uint64_t *bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst_smem)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
CS_D void bulk_s2g_hint(void *dst, const void *src_smem, unsigned bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
               "r"(smem_u32(src_smem)), "r"(bytes), "l"(pol)
               : "memory");
}
// shared -> global, tracked by the bulk async-group of the issuing thread
CS_D void bulk_s2g(void *dst, const void *src_smem, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src_smem)),
               "r"(bytes)
               : "memory");
}
CS_D void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
CS_D void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
CS_D void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

CS_D bool aligned16(const void *p) { return (((uintptr_t)p) & 15u) == 0; }

// p rounded up to an A-byte boundary of the shared window.  Pointer arithmetic
// (not an integer round trip) keeps the compiler's knowledge that the result
// is shared memory, so accesses through it compile to LDS/STS rather than
// generic LD/ST.
template <typename T, unsigned A>
CS_D T *smem_align(void *p) {
  unsigned char *c = (unsigned char *)p;
  return (T *)(c + ((A - (smem_u32(c) & (A - 1))) & (A - 1)));
}

// plain arrive (release at CTA scope): producer/consumer hand-offs inside a CTA
CS_D void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// 16-byte global -> shared copies that bypass L1 (reads are served by L2, so
// data published by other SMs is seen); all of a thread's copies stay in
// flight until cp_async_wait_all
CS_D void cp_async16(void *dst_smem, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst_smem)), "l"(src) : "memory");
}
CS_D void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

}  // namespace cs
