// tcec_gemm2.cuh -- CTA-pair (cta_group::2) fused error-corrected SGEMM.
//
// Same algorithm as tcec_gemm.cuh (the reference's corrected3 path,
// schemes.py:265-314) on a 256 x 256 output tile shared by a cluster of two
// CTAs on one TPC.  Each CTA stages and splits its own 128 rows of A and its
// own 128 columns of B; the leader CTA issues tcgen05.mma.cta_group::2 with
// M = 256, N = 256, which reads A from each CTA's shared memory and B from both
// halves; each CTA's TMEM receives its 128 rows.  Per SM this halves the
// split work and the tensor-core operand traffic per flop relative to the
// single-CTA 128 x 128 tile.
//
// Warp roles (640 threads, 20 warps, one CTA per SM):
//   warp 0        TMA producer: FP32 A [128 x 32] and B [32 x 128] k-slices
//   warp 1        MMA issuer (leader CTA only)
//   warp 2        TMEM allocator (512 columns: P | dC)
//   warps 4-11    split: FP32 slice -> (hi, lo) operands.  A is stored K-major,
//                 B MN-major (no transpose), both 128-byte swizzled.
//   warps 12-19   drain: C = RN32(C + P) per operand stage (C in registers),
//                 epilogue C = RN32(C + dC * 2^-s) -> TMA store.
#pragma once

#include "tcec_gemm.cuh"

namespace tcec {

template <int V>
struct PairCfg {
  static constexpr int BM = 128;           // rows per CTA (pair M = 256)
  static constexpr int BN = 256;           // pair N = MMA N
  static constexpr int BN_CTA = 128;       // B columns staged / split per CTA
  static constexpr int BK_STG = 32;        // FP32 k per staging slice
  static constexpr int NSTG = 3;
  static constexpr int NOP = 2;
  static constexpr int STG_A_BYTES = BM * BK_STG * 4;      // 16 KB, SW128 rows of 32 k
  static constexpr int STG_B_BOX = BK_STG * 32 * 4;        // 4 KB box: 32 k x 32 n, SW128
  static constexpr int STG_B_BYTES = 4 * STG_B_BOX;        // 16 KB
  static constexpr int STG_BYTES = STG_A_BYTES + STG_B_BYTES;
  static constexpr int OP_A_BYTES = BM * 128;              // K-major, 128-byte k rows
  static constexpr int OP_B_BYTES = BN_CTA * VarCfg<V>::BK_OP * (V == kFP16 ? 2 : 4);  // 16 KB
  static constexpr int OP_BYTES = 2 * OP_A_BYTES + 2 * OP_B_BYTES;
  // MN-major B: atoms of 128-byte n-rows, B_ROWS k-rows each (FP16: SWIZZLE_128B,
  // 64 n x 8 k; TF32: SWIZZLE_128B_BASE32B, 32 n x 4 k); atoms along n, then
  // k-groups.
  static constexpr int B_ATOM_N = V == kFP16 ? 64 : 32;     // n per 128-byte row
  static constexpr int B_ROWS = V == kFP16 ? 8 : 4;         // k rows per atom
  static constexpr int B_LBO = B_ROWS * 128;                // next atom along n
  static constexpr int B_SBO = (BN_CTA / B_ATOM_N) * B_LBO; // next k-group
  static constexpr uint32_t B_LAYOUT = V == kFP16 ? 2u : 1u;
  static constexpr int B_KSTEP_BYTES = (V == kFP16 ? 16 : 8) / B_ROWS * B_SBO;  // per MMA k-step
  static constexpr int OFF_STG = 0;
  static constexpr int OFF_OP = NSTG * STG_BYTES;
  static constexpr int OFF_BAR = OFF_OP + NOP * OP_BYTES;
  static constexpr int NUM_BARS = 2 * NSTG + 2 * NOP + 2;
  static constexpr int SMEM_BYTES = OFF_BAR + NUM_BARS * 8 + 16;
  static constexpr int TMEM_COLS = 512;                    // P [0,256) | dC [256,512)
  static constexpr int NUM_THREADS = 640;
  static constexpr int SPLIT_WARP0 = 4, NUM_SPLIT_WARPS = 8;
  static constexpr int DRAIN_WARP0 = 12, NUM_DRAIN_WARPS = 8;
  static constexpr int EPI_WARP_BYTES = 32 * 128 * 4;      // 32 rows x 128 cols per drain warp
  static_assert(B_KSTEP_BYTES == 4096, "B advance per k-step");
  static_assert(OP_B_BYTES == 16384, "B operand stage size");
  static_assert(NUM_DRAIN_WARPS * EPI_WARP_BYTES <= OFF_BAR, "epilogue staging reuses the rings");
};

// The MMAs of one operand stage (4 MMA k-steps) of the corrected3 schedule,
// issued by the whole (converged) MMA warp through elect.sync.
// corr(ks) issues k-step ks's correction products into dC (schemes.py:294-298);
// mainp(ks, acc) its main product into P.  P is drained every `de` k-steps --
// the main-term block of schemes.py:300-304 with block_k = de x MMA-K: the
// first main product of an interval waits until the drain warps have read the
// previous interval (p_empty) and starts from zero, the last one commits
// p_full.  `pos` counts the k-steps issued into the current interval (0 at a
// unit's start; the unit's last k-step, j0 + ks == nks - 1, closes its last
// interval and resets it), git the intervals committed (running across
// tiles); op_empty is committed once the stage's products are issued.  No
// division on the issue path: the single MMA thread feeds the tensor pipe.
// With stage-aligned intervals the stage's corrections go first, so the drain
// of the previous P overlaps them; otherwise each k-step's corrections precede
// its main product.  The order of products into each accumulator is the same
// either way.
template <typename Corr, typename Main>
__device__ __forceinline__ void c3_stage(int j0, int nks, int de, int& pos, uint32_t& git,
                                         uint64_t* p_empty, uint64_t* p_full, uint64_t* op_empty,
                                         Corr corr, Main mainp) {
  if ((de & 3) == 0) {
    // whole stages per interval: straight-line issue (the tensor pipe is fed by
    // this one thread; a branch between the main products costs throughput)
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) corr(ks);
    const bool first = pos == 0;
    if (first && git > 0) {
      sm100::mbar_wait_cluster(p_empty, (git - 1) & 1);
      sm100::tc_fence_after();
    }
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) mainp(ks, (first && ks == 0) ? 0u : 1u);
    sm100::mma_commit_pair_mc_el(op_empty, 0x3);
    pos += 4;
    if (pos == de || j0 + 4 >= nks) {
      sm100::mma_commit_pair_mc_el(p_full, 0x3);
      ++git;
      pos = 0;
    }
    return;
  }
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    corr(ks);
    if (pos == 0 && git > 0) {
      sm100::mbar_wait_cluster(p_empty, (git - 1) & 1);
      sm100::tc_fence_after();
    }
    mainp(ks, pos == 0 ? 0u : 1u);
    if (++pos == de || j0 + ks == nks - 1) {
      sm100::mma_commit_pair_mc_el(p_full, 0x3);
      ++git;
      pos = 0;
    }
  }
  sm100::mma_commit_pair_mc_el(op_empty, 0x3);
}

// Split one 32-deep FP32 slice of this CTA's A rows and B columns into the
// operand stage (all addresses are 32-bit shared-window addresses).
// Thread t (0..255):
//   A: row r = t & 127, k in [16 (t >> 7), +16)        -> K-major hi / lo
//   B: k = t & 31, n in [16 (t >> 5), +16)             -> MN-major hi / lo
// With kFlags the thread also folds its inputs into the RunFlags accumulator
// (only the CTAs designated to cover each element of A / B exactly once).
// One 16-byte operand chunk of hi and of lo words from consecutive inputs
// (FP16: 8 values -> 4 packed half2 words each; TF32: 4 values -> 4 words,
// the rounded FP32 bit patterns), splitting.py:114-122:
//   hi = round(x), lo = round((x - hi) 2^s), lo = 0 where hi overflowed
// (FP16: a packed mask per half2; TF32: a select per element -- both measured
// cheaper than guarding a rare fix-up with a max over the inputs, which costs
// the 56-register split warps more).
template <int V, int R>
__device__ __forceinline__ void split_chunk(const float* x, float scale, uint32_t (&hw)[4],
                                            uint32_t (&lw)[4]) {
  constexpr bool kFix = R != kRZ;  // RZ saturates: hi never overflows
  if constexpr (V == kFP16) {
#pragma unroll
    for (int j = 0; j < 4; ++j) split_pair16<R>(x[2 * j], x[2 * j + 1], scale, hw[j], lw[j]);
  } else {
#pragma unroll
    for (int j = 0; j < 4; j += 2) {
      hw[j] = tf32_round_bits<R>(__float_as_uint(x[j]));
      hw[j + 1] = tf32_round_bits<R>(__float_as_uint(x[j + 1]));
      float h0 = __uint_as_float(hw[j]), h1 = __uint_as_float(hw[j + 1]);
      float r0, r1;
      sm100::sub_x2(x[j], x[j + 1], h0, h1, r0, r1);
      // lo is read by the tensor core only, which ignores the low 13 bits of a
      // TF32 operand: the carry alone rounds it (tf32_carry_bits).  lo = 0
      // where x - hi is infinite, i.e. where hi overflowed (finite x): one
      // select on the residual (measured +1% TF32 over fixing hi before the
      // subtraction, profiles/r02/ab_fix.log)
      lw[j] = kFix && isinf(r0) ? 0u : tf32_carry_bits<R>(__float_as_uint(r0));
      lw[j + 1] = kFix && isinf(r1) ? 0u : tf32_carry_bits<R>(__float_as_uint(r1));
    }
  }
}

// 16 consecutive values -> hi / lo operand words (FP16: 8 packed half2 each;
// TF32: 16 floats each, stored as their bit patterns).
template <int V, int R>
__device__ __forceinline__ void split16(const float (&x)[16], float scale, uint32_t (&hw)[16],
                                        uint32_t (&lw)[16]) {
  constexpr int EPC = V == kFP16 ? 8 : 4;  // inputs per chunk
#pragma unroll
  for (int q = 0; q < 16 / EPC; ++q) {
    uint32_t h[4], l[4];
    split_chunk<V, R>(x + q * EPC, scale, h, l);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      hw[4 * q + j] = h[j];
      lw[4 * q + j] = l[j];
    }
  }
}

template <int V, int R, bool kFlags, bool kB>
__device__ __forceinline__ void pair_split_part(uint32_t stg, uint32_t op, int sub, int t,
                                                float scale, FlagAcc& fa) {
  using C = PairCfg<V>;
  float x[16];
  uint32_t row, chunk_first;
  if constexpr (!kB) {
    row = t & 127;
    const int half = t >> 7;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float4 v = sm100::lds128(stg + sw128(row, half * 4 + i));
      x[4 * i] = v.x; x[4 * i + 1] = v.y; x[4 * i + 2] = v.z; x[4 * i + 3] = v.w;
    }
    chunk_first = V == kFP16 ? sub * 4 + half * 2 : half * 4;
  } else {
    row = t & 31;  // k within the slice
    const int qn = t >> 5;
    const uint32_t box = stg + C::STG_A_BYTES + (qn >> 1) * C::STG_B_BOX;
    // TF32: lanes 4-7 of every 8-lane phase take their four 16-byte chunks in
    // the order 1,0,3,2 (same data, same registers) so that each STS.128 phase
    // covers both chunk parities of the SW128_BASE32B rows -- conflict-free
    // instead of 2-way (ncu: 1.07e9 excess wavefronts per 16384^3 launch).
    const int h = V == kTF32 ? (t >> 2) & 1 : 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float4 v = sm100::lds128(box + sw128(row, (qn & 1) * 4 + (i ^ h)));
      x[4 * i] = v.x; x[4 * i + 1] = v.y; x[4 * i + 2] = v.z; x[4 * i + 3] = v.w;
    }
    chunk_first = ((qn * 16) % C::B_ATOM_N) * (V == kFP16 ? 2 : 4) / 16;
  }
  if constexpr (kFlags) {
#pragma unroll
    for (int i = 0; i < 16; ++i) fa.add(x[i]);
  }
  const uint32_t hi_base = op + (kB ? 2 * C::OP_A_BYTES : 0);
  const uint32_t lo_base = hi_base + (kB ? C::OP_B_BYTES : C::OP_A_BYTES);
  constexpr int NCH = V == kFP16 ? 2 : 4;  // 16-byte chunks per 16 values
  constexpr int EPC = 16 / NCH;            // inputs per chunk
  // split and store chunk by chunk: few live registers in the 56-register split warps
  if constexpr (!kB) {
#pragma unroll
    for (int q = 0; q < NCH; ++q) {
      uint32_t hw[4], lw[4];
      split_chunk<V, R>(x + q * EPC, scale, hw, lw);
      const uint32_t off = sw128(row, chunk_first + q);
      sm100::sts128(hi_base + off, hw[0], hw[1], hw[2], hw[3]);
      sm100::sts128(lo_base + off, lw[0], lw[1], lw[2], lw[3]);
    }
  } else {
    const int kop = sub * 32 + row;  // k within the operand stage
    const int grp = kop / C::B_ROWS, rr = kop % C::B_ROWS;
    const uint32_t base = grp * C::B_SBO + (((t >> 5) * 16) / C::B_ATOM_N) * C::B_LBO + rr * 128;
    const int h = V == kTF32 ? (t >> 2) & 1 : 0;  // chunk order, see the loads above
#pragma unroll
    for (int q = 0; q < NCH; ++q) {
      uint32_t hw[4], lw[4];
      split_chunk<V, R>(x + q * EPC, scale, hw, lw);  // x chunk q holds source chunk q ^ h
      const int c16 = chunk_first + (q ^ h);
      // FP16 SW128: 16-byte chunk ^ row; TF32 SW128_BASE32B: 32-byte chunk ^ (row & 3)
      const uint32_t off = V == kFP16 ? base + ((c16 ^ rr) << 4)
                                      : base + ((((c16 >> 1) ^ rr) & 3) << 5) + ((c16 & 1) << 4);
      sm100::sts128(hi_base + off, hw[0], hw[1], hw[2], hw[3]);
      sm100::sts128(lo_base + off, lw[0], lw[1], lw[2], lw[3]);
    }
  }
}

template <int V, int R, bool kFlags>
__device__ __forceinline__ void pair_split_loop(uint32_t smem, uint64_t* stg_full,
                                                uint64_t* stg_empty, uint64_t* op_full,
                                                uint64_t* op_empty, int nop, int t, int lane,
                                                float scale, FlagAcc& fa) {
  using C = PairCfg<V>;
  using VC = VarCfg<V>;
  // the leader CTA's MMA thread consumes both CTAs' operand stages
  const uint32_t leader_op_full = sm100::mapa_shared(sm100::smem_u32(op_full), 0);
  for (int kb = 0; kb < nop; ++kb) {
    const int o = kb % C::NOP;
    const uint32_t op = smem + C::OFF_OP + o * C::OP_BYTES;
#pragma unroll
    for (int sub = 0; sub < VC::STG_PER_OP; ++sub) {
      const int st = kb * VC::STG_PER_OP + sub;
      const int s = st % C::NSTG;
      sm100::mbar_wait(&stg_full[s], (st / C::NSTG) & 1);
      if (sub == 0) sm100::mbar_wait(&op_empty[o], ((kb / C::NOP) & 1) ^ 1);
      const uint32_t stg = smem + C::OFF_STG + s * C::STG_BYTES;
      pair_split_part<V, R, kFlags, false>(stg, op, sub, t, scale, fa);
      pair_split_part<V, R, kFlags, true>(stg, op, sub, t, scale, fa);
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&stg_empty[s]);
    }
    // generic-proxy stores -> async proxy (tensor core), then signal the leader
    // (CTA-scope release on the peer barrier, as CUTLASS's 2-SM transform
    // pipelines do)
    sm100::fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) sm100::mbar_arrive_remote(leader_op_full + o * 8);
  }
}

template <int V, int R>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PairCfg<V>::NUM_THREADS, 1)
    tcec_gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA,  // A [m][k], box 32 x 128, SW128
                          const __grid_constant__ CUtensorMap tmB,  // B [k][n], box 32 x 32, SW128
                          const __grid_constant__ CUtensorMap tmC,  // C [m][n], box 32 x 32, SW128
                          const __grid_constant__ CDests cx,        // extra copies of C (all-gather)
                          const GemmShape shp, const float scale, const float inv_scale,
                          const FlagThresholds thr, uint32_t* __restrict__ flags) {
  using C = PairCfg<V>;
  using VC = VarCfg<V>;
  // 1024-byte alignment (SW128 atoms); identical offsets in both CTAs of the pair
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* stg_full = bars;                    // TMA -> split          (local)
  uint64_t* stg_empty = bars + C::NSTG;         // split -> TMA          (local, 8)
  uint64_t* op_full = bars + 2 * C::NSTG;       // split -> MMA          (leader, 16)
  uint64_t* op_empty = op_full + C::NOP;        // MMA commit -> split   (both, multicast)
  uint64_t* p_full = op_empty + C::NOP;         // MMA commit -> drain   (both, multicast)
  uint64_t* p_empty = p_full + 1;               // drain -> MMA          (leader, 16)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::NUM_BARS);
  const uint32_t smem_base = sm100::smem_u32(smem);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = sm100::cluster_ctarank();

  // ---- pair tile (grouped rasterisation along m)
  const int tiles_m = (shp.m + 2 * C::BM - 1) / (2 * C::BM);
  const int tiles_n = (shp.n + C::BN - 1) / C::BN;
  int tile_m, tile_n;
  {
    const int pid = blockIdx.x >> 1;
    const int per_group = shp.group_m * tiles_n;
    const int g = pid / per_group;
    const int first_m = g * shp.group_m;
    const int gsize = min(tiles_m - first_m, shp.group_m);
    const int in_g = pid - g * per_group;
    tile_m = first_m + in_g % gsize;
    tile_n = in_g / gsize;
  }
  const int m_cta = tile_m * 2 * C::BM + rank * C::BM;   // this CTA's A / C rows
  const int n_pair = tile_n * C::BN;                      // C columns of the pair
  const int n_cta = n_pair + rank * C::BN_CTA;            // this CTA's B columns
  const int nop = shp.num_op_stages;
  const int nstg = nop * VC::STG_PER_OP;
  const int de = shp.drain_every;  // MMA k-steps per drain interval
  const int nintervals = (4 * nop + de - 1) / de;

  if (warp == 0 && lane == 0) {
    if (smem_base & 1023u) __trap();  // SW128 operand atoms need 1024-byte alignment
    sm100::tma_prefetch_desc(&tmA);
    sm100::tma_prefetch_desc(&tmB);
    sm100::tma_prefetch_desc(&tmC);
    for (int s = 0; s < C::NSTG; ++s) {
      sm100::mbar_init(&stg_full[s], 1);
      sm100::mbar_init(&stg_empty[s], C::NUM_SPLIT_WARPS);
    }
    for (int o = 0; o < C::NOP; ++o) {
      sm100::mbar_init(&op_full[o], 2 * C::NUM_SPLIT_WARPS);
      sm100::mbar_init(&op_empty[o], 1);
    }
    sm100::mbar_init(p_full, 1);
    sm100::mbar_init(p_empty, 2 * C::NUM_DRAIN_WARPS);
    sm100::fence_mbar_init();
  }
  if (warp == 2) sm100::tmem_alloc_pair<C::TMEM_COLS>(tmem_slot);
  sm100::tc_fence_before();
  sm100::cluster_sync();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t tmem_P = tmem_base;
  const uint32_t tmem_dC = tmem_base + C::BN;

  if (warp < 4) {
    sm100::regs_dec<40>();
    if (warp == 0 && lane == 0) {
      // ===================== TMA producer =====================
      for (int st = 0; st < nstg; ++st) {
        const int s = st % C::NSTG;
        sm100::mbar_wait(&stg_empty[s], ((st / C::NSTG) & 1) ^ 1);
        uint8_t* dst = smem + C::OFF_STG + s * C::STG_BYTES;
        sm100::mbar_arrive_expect_tx(&stg_full[s], C::STG_BYTES);
        sm100::tma_load_2d(dst, &tmA, &stg_full[s], st * C::BK_STG, m_cta);
#pragma unroll
        for (int b = 0; b < 4; ++b)
          sm100::tma_load_2d(dst + C::STG_A_BYTES + b * C::STG_B_BOX, &tmB, &stg_full[s],
                             n_cta + 32 * b, st * C::BK_STG);
      }
    } else if (warp == 1 && rank == 0) {  // the whole warp runs the issue loop; one elected lane issues
      // ===================== MMA issuer (leader CTA) =====================
      constexpr uint32_t idesc = sm100::umma_idesc_bmn(VC::AB_FORMAT, 2 * C::BM, C::BN);
      // descriptor high words: SBO | version 1 | layout (K-major A: SW128; MN-major B)
      constexpr uint32_t a_hi_w = (1024u >> 4) | (1u << 14) | (2u << 29);
      constexpr uint32_t b_hi_w = (uint32_t(C::B_SBO) >> 4) | (1u << 14) | (C::B_LAYOUT << 29);
      constexpr uint32_t b_lbo_w = (uint32_t(C::B_LBO) >> 4) << 16;
      constexpr uint32_t kB = C::B_KSTEP_BYTES >> 4;
      uint32_t git = 0;
      int pos = 0;
      for (int kb = 0; kb < nop; ++kb) {
        const int o = kb % C::NOP;
        sm100::mbar_wait_cluster(&op_full[o], (kb / C::NOP) & 1);
        sm100::tc_fence_after();
        const uint32_t op = sm100::opaque(smem_base + C::OFF_OP + o * C::OP_BYTES) >> 4;
        const uint32_t ahi = op | (1u << 16);                                   // LBO = 16 B
        const uint32_t alo = ahi + (C::OP_A_BYTES >> 4);
        const uint32_t bhi = (op + ((2 * C::OP_A_BYTES) >> 4)) | b_lbo_w;
        const uint32_t blo = bhi + (C::OP_B_BYTES >> 4);
        c3_stage(
            kb * 4, 4 * nop, de, pos, git, p_empty, p_full, &op_empty[o],
            [&](int ks) {  // reference order per k-step: dA*B_hi, then A_hi*dB
              sm100::mma_pair_split_el<V == kTF32>(tmem_dC, alo + 2 * ks, a_hi_w, bhi + kB * ks,
                                                b_hi_w, idesc, (kb | ks) != 0);
              sm100::mma_pair_split_el<V == kTF32>(tmem_dC, ahi + 2 * ks, a_hi_w, blo + kB * ks,
                                                b_hi_w, idesc, 1u);
            },
            [&](int ks, uint32_t acc) {
              sm100::mma_pair_split_el<V == kTF32>(tmem_P, ahi + 2 * ks, a_hi_w, bhi + kB * ks, b_hi_w,
                                                idesc, acc);
            });
      }
    }
  } else if (warp < C::DRAIN_WARP0) {
    sm100::regs_dec<56>();
    // ===================== split warps =====================
    const int t = threadIdx.x - C::SPLIT_WARP0 * 32;
    FlagAcc fa;
    // A flags from the tile_n == 0 column of tiles, B flags from tile_m == 0:
    // every input element is classified exactly once across the grid.
    const bool do_flags = flags != nullptr && (tile_n == 0 || tile_m == 0);
    if (do_flags) {
      pair_split_loop<V, R, true>(smem_base, stg_full, stg_empty, op_full, op_empty, nop, t, lane, scale, fa);
      flag_publish(fa, thr, flags);
    } else {
      pair_split_loop<V, R, false>(smem_base, stg_full, stg_empty, op_full, op_empty, nop, t, lane, scale, fa);
    }
    // the epilogue reuses the staging ring: see the drain warps' barrier below
    sm100::named_barrier_sync<1, 32 * (C::NUM_SPLIT_WARPS + C::NUM_DRAIN_WARPS)>();
  } else {
    // setmaxnreg can only redistribute the launch allocation (96 x 640 registers):
    // 4 x 40 + 8 x 56 + 8 x 160 = 1888 <= 20 x 96 = 1920 per lane slot
    sm100::regs_inc<160>();
    // ===================== drain + epilogue =====================
    const int q = warp & 3;
    const int h = (warp - C::DRAIN_WARP0) >> 2;
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    const uint32_t p_empty_leader = sm100::mapa_shared(sm100::smem_u32(p_empty), 0);
    float acc[128];
#pragma unroll
    for (int j = 0; j < 128; ++j) acc[j] = 0.0f;
    for (int it = 0; it < nintervals; ++it) {
      sm100::mbar_wait(p_full, it & 1);
      sm100::tc_fence_after();
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        // 8 columns at a time: fewer live temporaries next to the 128 accumulators
        uint32_t r[8];
        sm100::tmem_ld_32x32b_x8(tmem_P + lane_off + h * 128 + c * 8, r);
        sm100::tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 8; j += 2)  // schemes.py:300-304: c = RN32(c + partial), f32x2
          sm100::fadd2_rn(acc[c * 8 + j], acc[c * 8 + j + 1], __uint_as_float(r[j]),
                          __uint_as_float(r[j + 1]));
      }
      sm100::tc_fence_before();
      __syncwarp();
      // the TMEM reads above have completed (wait::ld); P may be overwritten
      if (lane == 0) sm100::mbar_arrive_remote(p_empty_leader);
    }
    // every MMA of the pair has completed (the last p_full commit follows them),
    // and so have this CTA's split warps' staging reads; the named barrier says
    // so explicitly (racecheck does not follow mbarrier / tcgen05.commit chains)
    sm100::named_barrier_sync<1, 32 * (C::NUM_SPLIT_WARPS + C::NUM_DRAIN_WARPS)>();
    bool nonfinite = false;
    const uint32_t stage = smem_base + (warp - C::DRAIN_WARP0) * C::EPI_WARP_BYTES;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const uint32_t box = stage + b * 4096;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t r[16];
        sm100::tmem_ld_32x32b_x16(tmem_dC + lane_off + h * 128 + b * 32 + c * 16, r);
        sm100::tmem_ld_wait();
        float o[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          // schemes.py:306-307: one rounding of c + dC * 2^-s
          o[j] = __fmaf_rn(__uint_as_float(r[j]), inv_scale, acc[b * 32 + c * 16 + j]);
          nonfinite |= !isfinite(o[j]);
        }
#pragma unroll
        for (int v = 0; v < 4; ++v)
          sm100::sts128f(box + sw128(lane, c * 4 + v), o[4 * v], o[4 * v + 1], o[4 * v + 2], o[4 * v + 3]);
      }
      sm100::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        sm100::tma_store_2d(&tmC, smem + (box - smem_base), n_pair + h * 128 + b * 32, m_cta + q * 32);
        for (int d = 0; d < cx.count; ++d)  // fused all-gather: the same box to every peer
          sm100::tma_store_2d(&cx.m[d], smem + (box - smem_base), n_pair + h * 128 + b * 32,
                              m_cta + q * 32);
        sm100::tma_store_commit();
      }
    }
    if (lane == 0) sm100::tma_store_wait0();
    if (flags != nullptr && __any_sync(0xFFFFFFFFu, nonfinite) && lane == 0)
      atomicOr(flags, kFlagOverflow);
    sm100::tc_fence_before();
  }

  __syncthreads();
  sm100::cluster_sync();
  if (warp == 2) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc_pair<C::TMEM_COLS>(tmem_base);
  }
}

}  // namespace tcec
