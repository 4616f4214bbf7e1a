// sm100.cuh -- thin inline-PTX layer for the sm_100a async machinery used by
// the TCEC kernels: mbarriers, TMA (cp.async.bulk.tensor), tcgen05 (TMEM
// alloc / mma / commit / ld) and the proxy fences that order them.
//
// Everything here is a single PTX instruction (or a try_wait spin) so the
// kernels read like the hardware protocol they implement.  Compile with
// -gencode arch=compute_100a,code=sm_100a.
#pragma once

#include <cstdint>
#include <cuda.h>

namespace tcec {
namespace sm100 {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ------------------------------------------------------- shared-memory I/O --
// Explicit shared-window accesses on 32-bit addresses (never generic LD/ST).
__device__ __forceinline__ float4 lds128(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c,
                                       uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c),
               "r"(d)
               : "memory");
}
__device__ __forceinline__ void sts64(uint32_t addr, uint32_t a, uint32_t b) {
  asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(addr), "r"(a), "r"(b) : "memory");
}

__device__ __forceinline__ void sts128f(uint32_t addr, float a, float b, float c, float d) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a), "f"(b), "f"(c),
               "f"(d)
               : "memory");
}

// ---------------------------------------------------------------- mbarrier --
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

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}

// ------------------------------------------------------------------- fences --
// Generic-proxy smem writes -> visible to the async proxy (tcgen05.mma / TMA).
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// ---------------------------------------------------------------------- TMA --
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* m, uint64_t* bar,
                                            int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* m, const void* src, int32_t c0,
                                             int32_t c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void tma_store_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait0() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ------------------------------------------------------------------ tcgen05 --
template <uint32_t kCols>
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem) {
  // warp-wide (.sync.aligned); writes the TMEM base address to smem
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "n"(kCols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

template <uint32_t kCols>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols)
               : "memory");
}

// D[tmem] (+)= A[smem] * B[smem]^T, both operands K-major, FP32 accumulate.
__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                        uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Arrive (once) on an mbarrier when every tcgen05 op issued so far by this
// thread has completed.  Implies tcgen05.fence::before_thread_sync.
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

// 32 lanes x 16 consecutive 32-bit columns -> 16 registers per thread.
__device__ __forceinline__ void tmem_ld_32x32b_x16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

// 32 lanes x 8 consecutive 32-bit columns -> 8 registers per thread.
__device__ __forceinline__ void tmem_ld_32x32b_x8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// --------------------------------------------------- UMMA descriptor helpers --
// Shared-memory matrix descriptor for a K-major, 128-byte-swizzled operand
// tile whose rows are 128 bytes and whose 8-row atoms are stacked densely
// (stride 1024 B).  Bit layout: start>>4 [0,14), LBO>>4 [16,30), SBO>>4
// [32,46), version=1 [46,48), base_offset [49,52), layout (2 = SW128) [61,64).
__device__ __forceinline__ uint64_t umma_desc_sw128_kmajor(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1u) << 16;            // LBO (unused for swizzled K-major)
  d |= static_cast<uint64_t>(1024u >> 4) << 32;    // SBO: next 8-row group
  d |= static_cast<uint64_t>(1u) << 46;            // descriptor version (sm100)
  d |= static_cast<uint64_t>(2u) << 61;            // SWIZZLE_128B
  return d;
}

// Instruction descriptor (kind::f16 / kind::tf32): D=F32, A/B K-major.
// ab_format: 0 = F16, 2 = TF32.
__host__ __device__ constexpr uint32_t umma_idesc(uint32_t ab_format, uint32_t M, uint32_t N) {
  return (1u << 4)                 // c_format = F32
         | (ab_format << 7)        // a_format
         | (ab_format << 10)       // b_format
         | ((N >> 3) << 17)        // n_dim
         | ((M >> 4) << 24);       // m_dim
}


// ----------------------------------------------------------------- clusters --
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n"
               "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// shared::cta address of this CTA -> shared::cluster address of the same
// offset in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}

// Named barrier over `kThreads` threads (warp multiples) of this CTA; the
// non-.aligned form, so lanes that left a lane-0 branch need not reconverge.
template <uint32_t kId, uint32_t kThreads>
__device__ __forceinline__ void named_barrier_sync() {
  __syncwarp();
  asm volatile("barrier.sync %0, %1;" ::"n"(kId), "n"(kThreads) : "memory");
}

// Arrive on an mbarrier in another CTA of the cluster with the default
// (CTA-scope release) semantics -- no GPU-scope fence.  Used where the arrive
// only has to order this thread's completed TMEM reads, not memory writes.
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

// (a, b) += (c, d) on the f32x2 pipe, round-to-nearest.
__device__ __forceinline__ void fadd2_rn(float& a, float& b, float c, float d) {
  asm("{\n"
      ".reg .b64 x, y;\n"
      "mov.b64 x, {%0, %1};\n"
      "mov.b64 y, {%2, %3};\n"
      "add.rn.f32x2 x, x, y;\n"
      "mov.b64 {%0, %1}, x;\n"
      "}\n"
      : "+f"(a), "+f"(b)
      : "f"(c), "f"(d));
}

// Wait with acquire at cluster scope (for barriers that peer CTAs arrive on).
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAITC_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}

// ---------------------------------------------------------- tcgen05 (pair) --
template <uint32_t kCols>
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "n"(kCols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}

template <uint32_t kCols>
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols)
               : "memory");
}

// CTA-pair MMAs (M = 256 across the pair, issued by the leader CTA), in
// warp-converged form: the whole MMA warp runs the issue loop (warp-uniform
// descriptors, no per-instruction register -> uniform-register hand-off from a
// divergent lane) and elect.sync picks the one lane that issues.
// mma_pair_ts_el: A in tensor memory (each CTA's TMEM holds its 128 rows: lane =
// row, column = 32-bit word of K), B from shared memory.
// mma_pair_split_el: both operands from shared memory, each descriptor given as
// (low, high) 32-bit halves.
template <bool kTF32>
__device__ __forceinline__ void mma_pair_ts_el(uint32_t d_tmem, uint32_t a_tmem, uint32_t b_lo,
                                               uint32_t b_hi, uint32_t idesc, uint32_t accumulate) {
  if constexpr (kTF32) {
    asm volatile(
        "{\n"
        ".reg .pred p, e;\n"
        ".reg .b64 bd;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "mov.b64 bd, {%2, %3};\n"
        "setp.ne.b32 p, %5, 0;\n"
        "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], bd, %4, p;\n"
        "}\n" ::"r"(d_tmem),
        "r"(a_tmem), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(accumulate)
        : "memory");
  } else {
    asm volatile(
        "{\n"
        ".reg .pred p, e;\n"
        ".reg .b64 bd;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "mov.b64 bd, {%2, %3};\n"
        "setp.ne.b32 p, %5, 0;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], bd, %4, p;\n"
        "}\n" ::"r"(d_tmem),
        "r"(a_tmem), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(accumulate)
        : "memory");
  }
}

template <bool kTF32>
__device__ __forceinline__ void mma_pair_split_el(uint32_t d_tmem, uint32_t a_lo, uint32_t a_hi,
                                                  uint32_t b_lo, uint32_t b_hi, uint32_t idesc,
                                                  uint32_t accumulate) {
  if constexpr (kTF32) {
    asm volatile(
        "{\n"
        ".reg .pred p, e;\n"
        ".reg .b64 ad, bd;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "mov.b64 ad, {%1, %2};\n"
        "mov.b64 bd, {%3, %4};\n"
        "setp.ne.b32 p, %6, 0;\n"
        "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], ad, bd, %5, p;\n"
        "}\n" ::"r"(d_tmem),
        "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(accumulate)
        : "memory");
  } else {
    asm volatile(
        "{\n"
        ".reg .pred p, e;\n"
        ".reg .b64 ad, bd;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "mov.b64 ad, {%1, %2};\n"
        "mov.b64 bd, {%3, %4};\n"
        "setp.ne.b32 p, %6, 0;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], ad, bd, %5, p;\n"
        "}\n" ::"r"(d_tmem),
        "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(accumulate)
        : "memory");
  }
}

// 32 lanes x 8 / 16 consecutive 32-bit columns <- registers (one lane per thread).
__device__ __forceinline__ void tmem_st_32x32b_x8(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
      : "memory");
}
__device__ __forceinline__ void tmem_st_32x32b_x16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// Hide a value from the optimiser (stops it hoisting per-stage descriptor
// math for every ring slot into registers).
__device__ __forceinline__ uint32_t opaque(uint32_t x) {
  asm volatile("mov.b32 %0, %0;" : "+r"(x));
  return x;
}

// Arrive on the mbarrier at this offset in every CTA of `cta_mask` once all
// prior tcgen05 ops of the pair have completed.
__device__ __forceinline__ void mma_commit_pair_mc(uint64_t* bar, uint16_t cta_mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(cta_mask)
      : "memory");
}

// Warp-converged form of mma_commit_pair_mc (one elected lane commits).
__device__ __forceinline__ void mma_commit_pair_mc_el(uint64_t* bar, uint16_t cta_mask) {
  asm volatile(
      "{\n"
      ".reg .pred e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "h"(cta_mask)
      : "memory");
}

// Register-count hand-off between warpgroups (all 4 warps of a group execute it).
template <uint32_t kRegs>
__device__ __forceinline__ void regs_dec() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegs));
}
template <uint32_t kRegs>
__device__ __forceinline__ void regs_inc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegs));
}

// Instruction descriptor with an MN-major B operand (bit 16).
__host__ __device__ constexpr uint32_t umma_idesc_bmn(uint32_t ab_format, uint32_t M, uint32_t N) {
  return umma_idesc(ab_format, M, N) | (1u << 16);
}

// ------------------------------------------------------------- packed FP32 --
// (x0 - h0, x1 - h1) on the f32x2 pipe (exact for the split residual).
__device__ __forceinline__ void sub_x2(float x0, float x1, float h0, float h1, float& r0,
                                       float& r1) {
  asm("{\n"
      ".reg .b64 xv, hv, rv;\n"
      "mov.b64 xv, {%2, %3};\n"
      "mov.b64 hv, {%4, %5};\n"
      "sub.rn.f32x2 rv, xv, hv;\n"
      "mov.b64 {%0, %1}, rv;\n"
      "}\n"
      : "=f"(r0), "=f"(r1)
      : "f"(x0), "f"(x1), "f"(h0), "f"(h1));
}

// (x0, x1) * s and fma((h0, h1), t, (y0, y1)) on the sm_100 f32x2 pipe.
__device__ __forceinline__ void residual_x2(float x0, float x1, float h0, float h1, float s,
                                            float& r0, float& r1) {
  // r = (x - h) * s computed as fma(h, -s, x * s): both products are exact
  // (power-of-two s, no overflow while h is finite) and the fma rounds the
  // exact, representable difference once -- bit-identical to (x - h) * s.
  asm("{\n"
      ".reg .b64 xv, hv, sv, nv, rv;\n"
      "mov.b64 xv, {%2, %3};\n"
      "mov.b64 hv, {%4, %5};\n"
      "mov.b64 sv, {%6, %6};\n"
      "mov.b64 nv, {%7, %7};\n"
      "mul.rn.f32x2 xv, xv, sv;\n"
      "fma.rn.f32x2 rv, hv, nv, xv;\n"
      "mov.b64 {%0, %1}, rv;\n"
      "}\n"
      : "=f"(r0), "=f"(r1)
      : "f"(x0), "f"(x1), "f"(h0), "f"(h1), "f"(s), "f"(-s));
}

}  // namespace sm100
}  // namespace tcec
