// ptx.cuh -- thin inline-PTX wrappers for sm_100a: tcgen05 (MMA / TMEM), mbarrier,
// async-proxy fences, named barriers.  Product code only (no oracle dependency).
#pragma once
#include <cstdint>
#include <cuda_fp16.h>

namespace ntc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------- programmatic dependent launch
// wait until the preceding kernel of the stream has completed and its writes are visible (a
// no-op when this kernel was launched without the programmatic-serialization attribute)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// let the next kernel of the stream (launched with the attribute) start launching its CTAs
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" :::); }

// ---------------------------------------------------------------- barriers
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ void named_bar_arrive(uint32_t id, uint32_t nthreads) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t phase) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    return ok != 0;
}

// try_wait with an explicit suspend-time hint (ns): the warp may sleep until the phase
// completes or the hint expires instead of returning after the default short time limit
__device__ __forceinline__ bool mbar_try_wait_hint(uint64_t* bar, uint32_t phase, uint32_t hint_ns) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase), "r"(hint_ns)
        : "memory");
    return ok != 0;
}

#ifndef NTC_MBAR_HINT
#define NTC_MBAR_HINT 0
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    if constexpr (NTC_MBAR_HINT > 0) {
        while (!mbar_try_wait_hint(bar, phase, NTC_MBAR_HINT)) {
        }
    } else {
        while (!mbar_try_wait(bar, phase)) {
        }
    }
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// arrive on an mbarrier and add `bytes` to its expected transaction count
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

// bulk (non-tensor) TMA copy global -> shared, completing `bytes` transactions on `bar`;
// addresses 16-byte aligned, bytes a multiple of 16
__device__ __forceinline__ void bulk_g2s(uint32_t dst_smem, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     dst_smem),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// bulk (non-tensor) TMA store shared -> global in a bulk group of this thread
__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t src_smem, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src_smem), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// this thread's bulk groups have finished reading their shared-memory source
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// ... and completed
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// generic-proxy smem writes -> visible to the async proxy (tensor core operand reads)
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------- tcgen05 / TMEM
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols)
                 : "memory");
}
__device__ __forceinline__ void tmem_relinquish() {
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// D[tmem] (+)= A[smem] * B[smem]^T, fp16 inputs, fp32 accumulate, cta_group::1
__device__ __forceinline__ void mma_f16_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                           uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// The same MMA issued by a whole converged warp: elect.sync picks lane 0 (the lowest active
// lane, the same one on every call, so tcgen05.commit below tracks all of them).  With
// warp-uniform operands ptxas emits the bare UTCHMMA (no per-instruction ELECT / R2UR /
// BRA.U.ANY waterfall, which a single-thread `lane == 0` guard costs around every MMA).
__device__ __forceinline__ void mma_f16_ss_warp(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                                uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred e, p;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void mma_commit_warp(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
        : "memory");
}

// One whole layer in one asm block (whole converged warp, lane 0 elected): four K = 16 steps
// of D (+)= A B^T with both K-major descriptors advancing 32 bytes (2 units) per step, then
// optionally one more MMA (the ones x bias atom of a hidden layer), then the commit to `bar`.
// A single elect and one conversion of each base operand for the whole group.
#define NTC_MMA4_HEAD                                                                              \
    "{\n\t.reg .pred e, t, f;\n\t.reg .b64 a1, a2, a3, b1, b2, b3;\n\t"                            \
    "elect.sync _|e, 0xffffffff;\n\t"                                                               \
    "setp.eq.u32 t, 0, 0;\n\t"                                                                      \
    "setp.ne.u32 f, 0, 0;\n\t"                                                                      \
    "add.s64 a1, %1, 2;\n\tadd.s64 a2, %1, 4;\n\tadd.s64 a3, %1, 6;\n\t"                            \
    "add.s64 b1, %2, 2;\n\tadd.s64 b2, %2, 4;\n\tadd.s64 b3, %2, 6;\n\t"                            \
    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, f;\n\t"                                 \
    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, t;\n\t"                                 \
    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, t;\n\t"                                 \
    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %3, t;\n\t"
template <bool BIAS>
__device__ __forceinline__ void mma4_commit_warp(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint64_t ones,
                                                 uint64_t bias, uint64_t* bar) {
    if constexpr (BIAS)
        asm volatile(NTC_MMA4_HEAD
                     "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %4, %5, %3, t;\n\t"
                     "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%6];\n\t}" ::"r"(d),
                     "l"(a), "l"(b), "r"(idesc), "l"(ones), "l"(bias), "r"(smem_u32(bar))
                     : "memory");
    else
        asm volatile(NTC_MMA4_HEAD
                     "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%4];\n\t}" ::"r"(d),
                     "l"(a), "l"(b), "r"(idesc), "r"(smem_u32(bar))
                     : "memory");
}

// A chain of N K-steps of D (+)= A B^T in one asm block (whole converged warp, lane 0 elected):
// step i uses descriptors a + i*AST, b + i*BST (16-byte units); the first step accumulates when
// acc0 != 0, the others always; optionally the commit to `bar`.  One elect and one conversion of
// each base operand for the whole chain (the per-MMA form costs ~6 instructions per MMA).
#define NTC_CHAIN4(AS1, BS1, AS2, BS2, AS3, BS3) \
    "{\n\t.reg .pred e, t, p;\n\t.reg .b64 a1, b1, a2, b2, a3, b3;\n\t" \
    "elect.sync _|e, 0xffffffff;\n\t" \
    "setp.eq.u32 t, 0, 0;\n\t" \
    "setp.ne.b32 p, %4, 0;\n\t" \
    "add.s64 a1, %1, " #AS1 ";\n\tadd.s64 b1, %2, " #BS1 ";\n\t" \
    "add.s64 a2, %1, " #AS2 ";\n\tadd.s64 b2, %2, " #BS2 ";\n\t" \
    "add.s64 a3, %1, " #AS3 ";\n\tadd.s64 b3, %2, " #BS3 ";\n\t" \
    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t" \
    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, t;\n\t" \
    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, t;\n\t" \
    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %3, t;\n\t" \
    "}"

#define NTC_CHAIN4_C(AS1, BS1, AS2, BS2, AS3, BS3) \
    "{\n\t.reg .pred e, t, p;\n\t.reg .b64 a1, b1, a2, b2, a3, b3;\n\t" \
    "elect.sync _|e, 0xffffffff;\n\t" \
    "setp.eq.u32 t, 0, 0;\n\t" \
    "setp.ne.b32 p, %4, 0;\n\t" \
    "add.s64 a1, %1, " #AS1 ";\n\tadd.s64 b1, %2, " #BS1 ";\n\t" \
    "add.s64 a2, %1, " #AS2 ";\n\tadd.s64 b2, %2, " #BS2 ";\n\t" \
    "add.s64 a3, %1, " #AS3 ";\n\tadd.s64 b3, %2, " #BS3 ";\n\t" \
    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t" \
    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, t;\n\t" \
    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, t;\n\t" \
    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %3, t;\n\t" \
    "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%5];\n\t" \
    "}"

#define NTC_CHAIN8(AS1, BS1, AS2, BS2, AS3, BS3, AS4, BS4, AS5, BS5, AS6, BS6, AS7, BS7) \
    "{\n\t.reg .pred e, t, p;\n\t.reg .b64 a1, b1, a2, b2, a3, b3, a4, b4, a5, b5, a6, b6, a7, b7;\n\t" \
    "elect.sync _|e, 0xffffffff;\n\t" \
    "setp.eq.u32 t, 0, 0;\n\t" \
    "setp.ne.b32 p, %4, 0;\n\t" \
    "add.s64 a1, %1, " #AS1 ";\n\tadd.s64 b1, %2, " #BS1 ";\n\t" \
    "add.s64 a2, %1, " #AS2 ";\n\tadd.s64 b2, %2, " #BS2 ";\n\t" \
    "add.s64 a3, %1, " #AS3 ";\n\tadd.s64 b3, %2, " #BS3 ";\n\t" \
    "add.s64 a4, %1, " #AS4 ";\n\tadd.s64 b4, %2, " #BS4 ";\n\t" \
    "add.s64 a5, %1, " #AS5 ";\n\tadd.s64 b5, %2, " #BS5 ";\n\t" \
    "add.s64 a6, %1, " #AS6 ";\n\tadd.s64 b6, %2, " #BS6 ";\n\t" \
    "add.s64 a7, %1, " #AS7 ";\n\tadd.s64 b7, %2, " #BS7 ";\n\t" \
    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t" \
    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, t;\n\t" \
    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, t;\n\t" \
    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %3, t;\n\t" \
    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a4, b4, %3, t;\n\t" \
    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a5, b5, %3, t;\n\t" \
    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a6, b6, %3, t;\n\t" \
    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a7, b7, %3, t;\n\t" \
    "}"

#define NTC_CHAIN8_C(AS1, BS1, AS2, BS2, AS3, BS3, AS4, BS4, AS5, BS5, AS6, BS6, AS7, BS7) \
    "{\n\t.reg .pred e, t, p;\n\t.reg .b64 a1, b1, a2, b2, a3, b3, a4, b4, a5, b5, a6, b6, a7, b7;\n\t" \
    "elect.sync _|e, 0xffffffff;\n\t" \
    "setp.eq.u32 t, 0, 0;\n\t" \
    "setp.ne.b32 p, %4, 0;\n\t" \
    "add.s64 a1, %1, " #AS1 ";\n\tadd.s64 b1, %2, " #BS1 ";\n\t" \
    "add.s64 a2, %1, " #AS2 ";\n\tadd.s64 b2, %2, " #BS2 ";\n\t" \
    "add.s64 a3, %1, " #AS3 ";\n\tadd.s64 b3, %2, " #BS3 ";\n\t" \
    "add.s64 a4, %1, " #AS4 ";\n\tadd.s64 b4, %2, " #BS4 ";\n\t" \
    "add.s64 a5, %1, " #AS5 ";\n\tadd.s64 b5, %2, " #BS5 ";\n\t" \
    "add.s64 a6, %1, " #AS6 ";\n\tadd.s64 b6, %2, " #BS6 ";\n\t" \
    "add.s64 a7, %1, " #AS7 ";\n\tadd.s64 b7, %2, " #BS7 ";\n\t" \
    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t" \
    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, t;\n\t" \
    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, t;\n\t" \
    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %3, t;\n\t" \
    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a4, b4, %3, t;\n\t" \
    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a5, b5, %3, t;\n\t" \
    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a6, b6, %3, t;\n\t" \
    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a7, b7, %3, t;\n\t" \
    "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%5];\n\t" \
    "}"

// chains of 4 / 8 K-steps (steps in 16-byte descriptor units), with or without the commit
template <int AS, int BS>
__device__ __forceinline__ void mma_chain4_warp(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc0) {
    asm volatile(NTC_CHAIN4(%5, %6, %7, %8, %9, %10)::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc0), "n"(AS), "n"(BS),
                 "n"(2 * AS), "n"(2 * BS), "n"(3 * AS), "n"(3 * BS)
                 : "memory");
}
template <int AS, int BS>
__device__ __forceinline__ void mma_chain4_commit_warp(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                                       uint32_t acc0, uint64_t* bar) {
    asm volatile(NTC_CHAIN4_C(%6, %7, %8, %9, %10, %11)::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc0),
                 "r"(smem_u32(bar)), "n"(AS), "n"(BS), "n"(2 * AS), "n"(2 * BS), "n"(3 * AS), "n"(3 * BS)
                 : "memory");
}
template <int AS, int BS>
__device__ __forceinline__ void mma_chain8_warp(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc0) {
    asm volatile(NTC_CHAIN8(%5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18)::"r"(d), "l"(a), "l"(b),
                 "r"(idesc), "r"(acc0), "n"(AS), "n"(BS), "n"(2 * AS), "n"(2 * BS), "n"(3 * AS), "n"(3 * BS),
                 "n"(4 * AS), "n"(4 * BS), "n"(5 * AS), "n"(5 * BS), "n"(6 * AS), "n"(6 * BS), "n"(7 * AS), "n"(7 * BS)
                 : "memory");
}
template <int AS, int BS>
__device__ __forceinline__ void mma_chain8_commit_warp(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                                       uint32_t acc0, uint64_t* bar) {
    asm volatile(NTC_CHAIN8_C(%6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19)::"r"(d), "l"(a),
                 "l"(b), "r"(idesc), "r"(acc0), "r"(smem_u32(bar)), "n"(AS), "n"(BS), "n"(2 * AS), "n"(2 * BS),
                 "n"(3 * AS), "n"(3 * BS), "n"(4 * AS), "n"(4 * BS), "n"(5 * AS), "n"(5 * BS), "n"(6 * AS), "n"(6 * BS),
                 "n"(7 * AS), "n"(7 * BS)
                 : "memory");
}
// one MMA (enable-input-d = acc) and the commit to `bar`, whole warp
__device__ __forceinline__ void mma1_commit_warp(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc,
                                                 uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e, p;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%5];\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(smem_u32(bar))
        : "memory");
}

// arrive on an mbarrier when all previously issued tcgen05 ops of this thread complete
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// 32 lanes x 32 bit, 16 consecutive columns -> 16 registers per thread (thread i = lane i)
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
}

// tcgen05.wait::ld that also "defines" r: every later use of r is ordered after the wait
// (a plain wait only orders memory, so the compiler could hoist register uses above it)
__device__ __forceinline__ void tmem_wait_ld_r16(uint32_t (&r)[16]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                   "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                   "+r"(r[15])
                 :
                 : "memory");
}

// fp16 accumulators (one per 32-bit column, low half): 16 / 32 consecutive columns packed
// two per register (.pack::16b: register i = columns 2i | 2i+1 << 16, i.e. one half2)
__device__ __forceinline__ void tmem_ld8_pack(uint32_t taddr, uint32_t (&r)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr)
                 : "memory");
}
__device__ __forceinline__ void tmem_ld16_pack(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.pack::16b.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void tmem_wait_ld_r8(uint32_t (&r)[8]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7])
                 :
                 : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr)
        : "memory");
}

// ---------------------------------------------------------------- UMMA descriptors
// Shared-memory matrix descriptor (sm_100): start>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46),
// version=1 [46,48), base offset [49,52), lbo mode [52], layout type [61,64).
enum : uint32_t { UMMA_SWIZZLE_NONE = 0, UMMA_SWIZZLE_128B = 2, UMMA_SWIZZLE_64B = 4, UMMA_SWIZZLE_32B = 6 };

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes,
                                              uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)(layout & 7u) << 61;
    return d;
}

// K-major operand, 128-byte swizzle: rows of 64 fp16 (128 B), 8-row atoms of 1024 B.
__device__ __forceinline__ uint64_t umma_desc_k_sw128(uint32_t saddr) {
    return umma_desc(saddr, 16, 1024, UMMA_SWIZZLE_128B);
}

// MN-major operand, 128-byte swizzle: each K row holds 64 contiguous MN elements (128 B),
// 8 K-rows form a 1024 B atom; `mn_block_bytes` = stride between 64-wide MN blocks.
__device__ __forceinline__ uint64_t umma_desc_mn_sw128(uint32_t saddr, uint32_t mn_block_bytes) {
    return umma_desc(saddr, mn_block_bytes, 1024, UMMA_SWIZZLE_128B);
}

// Instruction descriptor, kind::f16: D fp32 (bit 4 set) or fp16 (clear: the accumulator is
// rounded to fp16; each value still occupies one 32-bit TMEM column, in its low half), A/B fp16
// (0), K-major unless set, N>>3 at [17,23), M>>4 at [24,29).
__host__ __device__ constexpr uint32_t idesc_f16(uint32_t M, uint32_t N, bool a_mn_major = false,
                                                 bool b_mn_major = false, bool d_f32 = true) {
    return ((d_f32 ? 1u : 0u) << 4) | ((a_mn_major ? 1u : 0u) << 15) | ((b_mn_major ? 1u : 0u) << 16) |
           ((N >> 3) << 17) | ((M >> 4) << 24);
}

// K-major SW32 / SW64 tiles: rows of 32 / 64 B (16 / 32 fp16), 8-row atoms of 256 / 512 B;
// the 16-byte chunk index is XORed with row bit 2 (SW32) or row bits 1-2 (SW64)
__device__ __forceinline__ uint64_t umma_desc_k_sw32(uint32_t saddr) { return umma_desc(saddr, 16, 256, UMMA_SWIZZLE_32B); }
__device__ __forceinline__ uint64_t umma_desc_k_sw64(uint32_t saddr) { return umma_desc(saddr, 16, 512, UMMA_SWIZZLE_64B); }
__host__ __device__ constexpr uint32_t sw32_offset(uint32_t row, uint32_t k) {
    return row * 32u + ((((k >> 3) & 1u) ^ ((row >> 2) & 1u)) << 4) + (k & 7u) * 2u;
}
__host__ __device__ constexpr uint32_t sw64_offset(uint32_t row, uint32_t k) {
    return row * 64u + ((((k >> 3) & 3u) ^ ((row >> 1) & 3u)) << 4) + (k & 7u) * 2u;
}

// byte offset of element (row, k) in a K-major SW128 tile (rows of 128 B, 1024 B aligned)
__host__ __device__ __forceinline__ uint32_t sw128_offset(uint32_t row, uint32_t k) {
    return row * 128u + ((((k >> 3) & 7u) ^ (row & 7u)) << 4) + (k & 7u) * 2u;
}

__device__ __forceinline__ void sts128(uint32_t saddr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(saddr), "r"(a), "r"(b), "r"(c), "r"(d)
                 : "memory");
}

// predicated global stores (no divergent branch structure)
__device__ __forceinline__ void st_global_b32_if(void* p, uint32_t v, bool pred) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.global.b32 [%0], %1;\n\t}" ::"l"(p), "r"(v),
                 "r"((uint32_t)pred)
                 : "memory");
}
__device__ __forceinline__ void st_global_b16_if(void* p, uint16_t v, bool pred) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.global.b16 [%0], %1;\n\t}" ::"l"(p), "h"(v),
                 "r"((uint32_t)pred)
                 : "memory");
}

__device__ __forceinline__ uint32_t pack_half2(float lo, float hi) {
    __half2 h = __floats2half2_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&h);
}

}  // namespace ntc
