// psa_device.cuh — sm_100a PTX wrappers: mbarrier, TMA (cp.async.bulk.tensor),
// tcgen05 (TMEM alloc, MMA, commit, ld/st, fences) and UMMA descriptors.
#pragma once

#include <cuda.h>
#include <cstdint>

namespace psa {

// Per-block clock64 event traces (tools/trace_report.py) cost instruction-cache space
// on the hot paths: compiled in only with -DPSA_TRACE_EVENTS (PSA_TRACE_EVENTS=1 at build).
#ifdef PSA_TRACE_EVENTS
constexpr bool kTraceEvents = true;
#else
constexpr bool kTraceEvents = false;
#endif
namespace dev {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 2^x on the SFU (one MUFU.EX2; flushes denormals, 2^-inf = +0).
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ---- mbarrier ----------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// Non-blocking: has the phase with the given parity completed?
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Blocks until the phase with the given parity has completed.
#ifdef PSA_BOUNDED_WAIT
// Debug build (build.py with PSA_DEBUG_BUILD=1 -> libpsa_debug.so): a wait that has
// not completed after ~2^31 polls (seconds) records who hung on which barrier in
// psa_hang_info and traps, instead of spinning until the host's timeout.
__device__ int psa_hang_info[8];
__device__ __noinline__ void mbar_hang(uint64_t* bar, uint32_t parity) {
  if (atomicCAS(&psa_hang_info[0], 0, 1) == 0) {
    psa_hang_info[1] = int(blockIdx.x);
    psa_hang_info[2] = int(threadIdx.x);
    psa_hang_info[3] = int(smem_u32(bar));
    psa_hang_info[4] = int(parity);
    __threadfence_system();
    printf("psa: mbarrier wait hung: block %d thread %d barrier smem+0x%x parity %u\n",
           int(blockIdx.x), int(threadIdx.x), smem_u32(bar), parity);
  }
  __trap();
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  for (uint32_t n = 0; n < (1u << 31); ++n) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (ok) return;
  }
  mbar_hang(bar, parity);
}
#else
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
#endif

// ---- TMA -----------------------------------------------------------------------
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0,
                                            int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0,
                                            int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
// L2 prefetch of one tensor-map box (no shared memory, no barrier): warms L2 for a
// TMA load that the ring cannot take yet.
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* m, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---- tcgen05 -------------------------------------------------------------------
template <uint32_t kCols>
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem) {  // whole warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "n"(kCols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
// A CTA of a kernel that contains tcgen05.alloc holds the SM's allocation
// permit until it relinquishes it; a second CTA is not co-scheduled on that SM
// before then. CTAs that will not allocate must give the permit up at once.
__device__ __forceinline__ void tmem_relinquish() {  // whole warp
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <uint32_t kCols>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {  // whole warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols)
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// D[tmem] (+)= A[smem] * B[smem], kind::f16 (bf16/f16 in, fp32 accumulate).
__device__ __forceinline__ void mma_f16_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                           uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem], kind::f16. A (M x 16, K-major) sits in TMEM:
// lane = row, 8 consecutive 32-bit columns = 16 packed 16-bit elements.
__device__ __forceinline__ void mma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                           uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Warp-wide forms: the whole (converged) warp executes them with warp-uniform
// operands and one elected lane issues, so ptxas can keep the descriptors in
// uniform registers instead of a per-instruction R2UR / elect waterfall.
__device__ __forceinline__ void mma_f16_ss_w(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_f16_ts_w(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit_w(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}
// Arrives on `bar` once every previously issued tcgen05.mma of this thread completed.
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

#define PSA_R32(a) \
  "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]), "=r"(a[4]), "=r"(a[5]), "=r"(a[6]), \
  "=r"(a[7]), "=r"(a[8]), "=r"(a[9]), "=r"(a[10]), "=r"(a[11]), "=r"(a[12]), "=r"(a[13]), \
  "=r"(a[14]), "=r"(a[15]), "=r"(a[16]), "=r"(a[17]), "=r"(a[18]), "=r"(a[19]), "=r"(a[20]), \
  "=r"(a[21]), "=r"(a[22]), "=r"(a[23]), "=r"(a[24]), "=r"(a[25]), "=r"(a[26]), "=r"(a[27]), \
  "=r"(a[28]), "=r"(a[29]), "=r"(a[30]), "=r"(a[31])
#define PSA_W32(a) \
  "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]), \
  "r"(a[8]), "r"(a[9]), "r"(a[10]), "r"(a[11]), "r"(a[12]), "r"(a[13]), "r"(a[14]), \
  "r"(a[15]), "r"(a[16]), "r"(a[17]), "r"(a[18]), "r"(a[19]), "r"(a[20]), "r"(a[21]), \
  "r"(a[22]), "r"(a[23]), "r"(a[24]), "r"(a[25]), "r"(a[26]), "r"(a[27]), "r"(a[28]), \
  "r"(a[29]), "r"(a[30]), "r"(a[31])

// 32 consecutive fp32 columns of this thread's TMEM lane (warp w owns lanes 32*(w%4)..).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
      "%28, %29, %30, %31}, [%32];"
      : PSA_R32(r)
      : "r"(taddr));
}

// PSA_MMA_WARP_WIDE (default): the MMA role runs on all 32 lanes of its warp and
// issues through elect.sync (psa_device.cuh *_w forms), so ptxas emits straight-line
// UTCHMMA sequences instead of one elect/R2UR waterfall loop per instruction (the
// lane-0 form spent ~85 cycles issuing each 64-cycle MMA: c3 2985 -> 2801 us, c4
// 612 -> 600 us, c5 15.5 -> 14.6 ms). 0 = lane 0 alone (diagnostics).
#ifndef PSA_MMA_WARP_WIDE
#define PSA_MMA_WARP_WIDE 0
#endif
#if PSA_MMA_WARP_WIDE
#define PSA_MMA_TS ::psa::dev::mma_f16_ts_w
#define PSA_MMA_SS ::psa::dev::mma_f16_ss_w
#define PSA_MMA_COMMIT ::psa::dev::mma_commit_w
#else
#define PSA_MMA_TS ::psa::dev::mma_f16_ts
#define PSA_MMA_SS ::psa::dev::mma_f16_ss
#define PSA_MMA_COMMIT ::psa::dev::mma_commit
#endif

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
      "%28, %29, %30, %31, %32};" ::"r"(taddr),
      PSA_W32(r)
      : "memory");
}
#define PSA_R16(a) \
  "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]), "=r"(a[4]), "=r"(a[5]), "=r"(a[6]), \
  "=r"(a[7]), "=r"(a[8]), "=r"(a[9]), "=r"(a[10]), "=r"(a[11]), "=r"(a[12]), "=r"(a[13]), \
  "=r"(a[14]), "=r"(a[15])
#define PSA_W16(a) \
  "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]), \
  "r"(a[8]), "r"(a[9]), "r"(a[10]), "r"(a[11]), "r"(a[12]), "r"(a[13]), "r"(a[14]), "r"(a[15])
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15}, [%16];"
      : PSA_R16(r)
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      PSA_W16(r)
      : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// ---- UMMA descriptors ------------------------------------------------------------
// Shared-memory matrix descriptor (sm100 "version 1"), 128-byte swizzle.
//   K-major operand:  rows of 128 B, 8-row atoms at SBO = 1024 B (LBO unused).
//   MN-major operand: 128 B (64 elems) per K-row, K-row groups of 8 at SBO,
//                     next 64-element MN chunk at LBO.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t smem_addr, uint32_t lbo_bytes,
                                                    uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= uint64_t((smem_addr & 0x3FFFF) >> 4);
  d |= uint64_t((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;  // version (Blackwell)
  d |= uint64_t(2) << 61;  // SWIZZLE_128B
  return d;
}
// Instruction descriptor, kind::f16: fp32 accumulate; a/b format 0 = f16, 1 = bf16.
__host__ __device__ constexpr uint32_t umma_idesc_f16(uint32_t ab_format, uint32_t M, uint32_t N,
                                                      uint32_t a_mn_major, uint32_t b_mn_major) {
  return (1u << 4)                 // c_format = F32
         | (ab_format << 7)        // a_format
         | (ab_format << 10)       // b_format
         | (a_mn_major << 15)      // a major
         | (b_mn_major << 16)      // b major
         | ((N >> 3) << 17)        // n_dim
         | ((M >> 4) << 24);       // m_dim
}


// gpu-scope acquire/release fence (lighter than the sequentially consistent
// fence.sc.gpu behind __threadfence()); paired with relaxed atomics it forms the
// release / acquire patterns of the PTX memory model.
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
// Warp-wide max of a float (sm_100a CREDUX.MAX.F32; NaN inputs are ignored like fmaxf's).
__device__ __forceinline__ float warp_max_f32(float v) {
  float r;
  asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
  return r;
}
// Coherent-at-L2 load issued where it is written (volatile: not sunk to its use).
__device__ __forceinline__ float ld_cg_f32(const float* p) {
  float v;
  asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ float2 ld_cg_f32x2(const float2* p) {
  float2 v;
  asm volatile("ld.global.cg.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  return v;
}

// ---- CTA-local merge queue ------------------------------------------------------
// Bounded MPMC ring in shared memory: threads that complete work push tasks, merge
// warps pop them (and may push follow-up tasks). Every slot carries a sequence
// number (Vyukov): slot i is free for ticket t when seq[i] == t, holds ticket t's
// task when seq[i] == t + 1, and is released for ticket t + kCap by the reader, so
// a writer never overwrites an unread entry and a reader never sees an unwritten one.
// Termination: `outstanding` counts tasks pushed and not yet finished (a task's
// follow-up pushes happen before it finishes); readers leave once every producer
// closed and nothing is outstanding.
struct MergeQueue {
  static constexpr int kCap = 64;
  int unit[kCap];
  int seq[kCap];
  int resv;         // tickets handed to writers
  int head;         // tickets handed to readers
  int closed;       // producers that will not push again
  int outstanding;  // tasks pushed and not yet finished
};

__device__ __forceinline__ int ld_vol(const int* p) { return *reinterpret_cast<const volatile int*>(p); }
__device__ __forceinline__ void st_vol(int* p, int v) { *reinterpret_cast<volatile int*>(p) = v; }
// The queue's sequence words are its synchronisation flags: a writer publishes an
// entry with a release store of seq, a reader takes it with an acquire load (CTA
// scope, shared memory), so the entry's payload is ordered without a separate fence.
__device__ __forceinline__ int ld_acq_cta(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel_cta(int* p, int v) {
  asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}

// One thread.
__device__ __forceinline__ void mq_init(MergeQueue* q) {
  for (int i = 0; i < MergeQueue::kCap; ++i) q->seq[i] = i;
  q->resv = q->head = q->closed = q->outstanding = 0;
}

// Any thread: hand task u to the merge warps (spins only while kCap tasks are pending).
__device__ __forceinline__ void mq_push(MergeQueue* q, int u) {
  atomicAdd(&q->outstanding, 1);
  const int t = atomicAdd(&q->resv, 1);
  const int i = t & (MergeQueue::kCap - 1);
  while (ld_acq_cta(&q->seq[i]) != t) __nanosleep(32);  // the reader of ticket t - kCap is done
  st_vol(&q->unit[i], u);
  st_rel_cta(&q->seq[i], t + 1);
}

// One producer (thread) is done pushing; its pushes precede this in program order
// (or are ordered before it by a barrier).
__device__ __forceinline__ void mq_close(MergeQueue* q) {
  __threadfence_block();
  atomicAdd(&q->closed, 1);
}

// Tasks pushed and not yet claimed by a reader (negative while readers wait). A
// pusher that sees fewer than kCap / 2 pending can push without blocking as long
// as at most kCap / 4 pushers race (each waiting reader holds at most one slot).
__device__ __forceinline__ int mq_pending(const MergeQueue* q) {
  return ld_vol(&q->resv) - ld_vol(&q->head);
}

// A warp that finished another role and will help drain the queue: sleep until every
// producer closed it, so the helper never competes for issue slots with warps that
// are still computing (only the backlog left at the end is shared out).
__device__ __forceinline__ void mq_wait_closed(const MergeQueue* q, int closers) {
  while (ld_vol(&q->closed) < closers) __nanosleep(2048);
}

// Merge warp: pop tasks until `closers` producers closed the queue and no task is
// outstanding.
template <typename Task>
__device__ __forceinline__ void mq_drain(MergeQueue* q, int closers, Task&& task) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    int u = 0, ok = 0;
    if (lane == 0) {
      const int t = atomicAdd(&q->head, 1);
      const int i = t & (MergeQueue::kCap - 1);
      for (;;) {
        if (ld_acq_cta(&q->seq[i]) == t + 1) {
          u = ld_vol(&q->unit[i]);
          ok = 1;
          st_rel_cta(&q->seq[i], t + MergeQueue::kCap);  // after the payload read
          break;
        }
        if (ld_vol(&q->closed) >= closers) {
          __threadfence_block();
          if (ld_vol(&q->outstanding) == 0) break;
        }
        __nanosleep(64);
      }
    }
    ok = __shfl_sync(0xffffffffu, ok, 0);
    if (!ok) break;
    u = __shfl_sync(0xffffffffu, u, 0);
    fence_acq_rel_gpu();  // acquire: the task's partial rows were published before it was queued
    task(u);
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      atomicSub(&q->outstanding, 1);
    }
  }
}

}  // namespace dev
}  // namespace psa
