// tcec_gemm6.cuh -- persistent CTA-quad kernel: two CTA pairs share the split of A
// (opts.reserved[1] = 5).
//
// Same algorithm, MMA order, drain and epilogue as the persistent pair kernel
// (tcec_gemm5.cuh), so C is bit-identical.  A cluster of four CTAs holds two
// pairs that compute horizontally adjacent 256 x 256 tiles (tm, 2j) and
// (tm, 2j + 1).  Both pairs need the same 256 rows of A, so each CTA stages
// (TMA, L2 -> shared) and splits only half of its 128 A rows and writes the
// hi / lo operands into its own operand stage and, over distributed shared
// memory, into the same rows of its partner in the other pair (cluster rank
// ^ 2).  Per CTA this removes a quarter of the FP32 tiles moved from L2 and a
// quarter of the split work -- on the power-capped B200 the fused kernel's
// largest energy costs.
//
// Synchronisation on top of the pair kernel:
//   op_full  (pair leader)  32 arrivals: the split warps of all four CTAs (A
//                           halves from both pairs, B from the own pair)
//   op_empty (every CTA)    2 arrivals: the MMA commits of both pairs, so a
//                           stage is rewritten only when neither pair reads it
//   p_full / p_empty / acc_empty as in the pair kernel, within each pair.
// Tile units (tm, j) walk the grouped raster with lock-step waves like the
// persistent pair kernel; a ragged last column pair computes a phantom tile
// (zero-filled B, nothing stored).
//
// Measured slower than the pair kernel (profiles/r01/quad_cluster.log, 8192^3:
// FP16 ~200 vs 440 TF/s, TF32 ~110 vs 290): the distributed-shared-memory
// stores and the cluster-scope release each split warp needs before the other
// pair's MMA may read its rows put a cross-TPC round trip on every operand
// stage, and with both pairs gated by each other's MMA commits the 2-deep ring
// cannot hide it.  Even a measurement build with no remote stores and
// CTA-scope arrives (wrong results) only matched the pair kernel (FP16 437,
// TF32 208-247 on 132 SMs: 33 co-resident clusters of four).  Kept, bit-identical
// and tested, as the measured answer to DESIGN.md 8's split-sharing idea.
#pragma once

#include "tcec_gemm5.cuh"

namespace tcec {

template <int V>
struct QuadCfg {
  using P = PairCfg<V>;
  static constexpr int BM = 128;                            // rows per CTA (pair M = 256)
  static constexpr int BN = 256;                            // pair N
  static constexpr int BN_CTA = 128;
  static constexpr int BK_STG = 32;
  static constexpr int A_ROWS = 64;                         // A rows staged / split per CTA
  static constexpr int NSTG = 4;
  static constexpr int NOP = 2;
  static constexpr int STG_A_BYTES = A_ROWS * BK_STG * 4;   // 8 KB, SW128 rows of 32 k
  static constexpr int STG_B_BOX = P::STG_B_BOX;
  static constexpr int STG_B_BYTES = P::STG_B_BYTES;        // 16 KB
  static constexpr int STG_BYTES = STG_A_BYTES + STG_B_BYTES;
  static constexpr int OP_A_BYTES = P::OP_A_BYTES;
  static constexpr int OP_BYTES = P::OP_BYTES;
  static constexpr int OFF_STG = 0;
  static constexpr int OFF_OP = NSTG * STG_BYTES;
  static constexpr int OFF_BAR = OFF_OP + NOP * OP_BYTES;
  static constexpr int NUM_BARS = 2 * NSTG + 2 * NOP + 2;
  static constexpr int SMEM_BYTES = OFF_BAR + NUM_BARS * 8 + 16;
  static constexpr int TMEM_COLS = 512;                     // P | dC
  static constexpr int NUM_THREADS = 640;
  static constexpr int SPLIT_WARP0 = 4, NUM_SPLIT_WARPS = 8;
  static constexpr int DRAIN_WARP0 = 12, NUM_DRAIN_WARPS = 8;
  static_assert(SMEM_BYTES <= 227 * 1024, "shared memory");
  static_assert(STG_BYTES % 1024 == 0 && OFF_OP % 1024 == 0, "swizzle alignment");
};

// N consecutive values -> hi / lo operand words (split16 for any even N).
template <int V, int R, int N>
__device__ __forceinline__ void split_n(const float (&x)[N], float scale, uint32_t (&hw)[N],
                                        uint32_t (&lw)[N]) {
  if constexpr (V == kFP16) {
#pragma unroll
    for (int j = 0; j < N / 2; ++j) {
      hw[j] = cvt_f16x2<R>(x[2 * j], x[2 * j + 1]);
      float h0, h1, r0, r1;
      unpack_f16x2(hw[j], h0, h1);
      sm100::residual_x2(x[2 * j], x[2 * j + 1], h0, h1, scale, r0, r1);
      lw[j] = cvt_f16x2<R>(r0, r1);
    }
  } else {
#pragma unroll
    for (int j = 0; j < N; j += 2) {
      hw[j] = tf32_round_bits<R>(__float_as_uint(x[j]));
      hw[j + 1] = tf32_round_bits<R>(__float_as_uint(x[j + 1]));
      float r0, r1;
      sm100::sub_x2(x[j], x[j + 1], __uint_as_float(hw[j]), __uint_as_float(hw[j + 1]), r0, r1);
      lw[j] = tf32_round_bits<R>(__float_as_uint(r0));
      lw[j + 1] = tf32_round_bits<R>(__float_as_uint(r1));
    }
  }
}

// This CTA's half of A in one 32-deep slice: thread t takes row t & 63 of the
// staged 64 and k in [8 (t >> 6), +8); the hi / lo words go to operand row
// p * 64 + row of this CTA (op) and of the partner CTA (rop, shared::cluster).
template <int V, int R, bool kFlags>
__device__ __forceinline__ void quad_split_a(uint32_t stg, uint32_t op, uint32_t rop, int sub,
                                             int t, int p, float scale, FlagAcc& fa) {
  using C = QuadCfg<V>;
  const int row = t & 63, qk = t >> 6;
  float x[8];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float4 v = sm100::lds128(stg + sw128(row, qk * 2 + i));
    x[4 * i] = v.x; x[4 * i + 1] = v.y; x[4 * i + 2] = v.z; x[4 * i + 3] = v.w;
  }
  if constexpr (kFlags) {
#pragma unroll
    for (int i = 0; i < 8; ++i) fa.add(x[i]);
  }
  uint32_t hw[8], lw[8];
  split_n<V, R, 8>(x, scale, hw, lw);
  const int orow = p * C::A_ROWS + row;
  constexpr int NCH = V == kFP16 ? 1 : 2;  // 16-byte chunks per 8 values
  const int c0 = V == kFP16 ? sub * 4 + qk : qk * 2;
#pragma unroll
  for (int q = 0; q < NCH; ++q) {
    const uint32_t off = sw128(orow, c0 + q);
    sm100::sts128(op + off, hw[4 * q], hw[4 * q + 1], hw[4 * q + 2], hw[4 * q + 3]);
    sm100::sts128(op + C::OP_A_BYTES + off, lw[4 * q], lw[4 * q + 1], lw[4 * q + 2], lw[4 * q + 3]);
    sm100::sts128_cluster(rop + off, hw[4 * q], hw[4 * q + 1], hw[4 * q + 2], hw[4 * q + 3]);
    sm100::sts128_cluster(rop + C::OP_A_BYTES + off, lw[4 * q], lw[4 * q + 1], lw[4 * q + 2],
                          lw[4 * q + 3]);
  }
}

// Split `nop` operand stages of one tile unit (ring counters continue across units).
template <int V, int R, bool kFlags>
__device__ __forceinline__ void quad_split_tile(uint32_t smem, uint32_t rsmem, uint64_t* stg_full,
                                                uint64_t* stg_empty, uint64_t* op_empty,
                                                uint32_t op_full_l0, uint32_t op_full_l1,
                                                uint32_t g0, int nop, int t, int lane, int p,
                                                float scale, FlagAcc& fa) {
  using C = QuadCfg<V>;
  using VC = VarCfg<V>;
  for (int kb = 0; kb < nop; ++kb) {
    const uint32_t g = g0 + kb;
    const int o = g % C::NOP;
    const uint32_t op = smem + C::OFF_OP + o * C::OP_BYTES;
    const uint32_t rop = rsmem + C::OFF_OP + o * C::OP_BYTES;
#pragma unroll
    for (int sub = 0; sub < VC::STG_PER_OP; ++sub) {
      const uint32_t gst = g * VC::STG_PER_OP + sub;
      const int s = gst % C::NSTG;
      sm100::mbar_wait(&stg_full[s], (gst / C::NSTG) & 1);
      if (sub == 0) sm100::mbar_wait(&op_empty[o], ((g / C::NOP) & 1) ^ 1);
      const uint32_t stg = smem + C::OFF_STG + s * C::STG_BYTES;
      quad_split_a<V, R, kFlags>(stg, op, rop, sub, t, p, scale, fa);
      // B: the pair kernel's split of this CTA's 128 columns; its staging boxes
      // follow the 8 KB A box here instead of the pair kernel's 16 KB one
      pair_split_part<V, R, kFlags, true>(stg + C::STG_A_BYTES - PairCfg<V>::STG_A_BYTES, op, sub,
                                          t, scale, fa);
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&stg_empty[s]);
    }
    sm100::fence_proxy_async_cluster();
    __syncwarp();
    if (lane == 0) {  // release at cluster scope: the partner's rows were written remotely
      sm100::mbar_arrive_cluster(op_full_l0 + o * 8);
      sm100::mbar_arrive_cluster(op_full_l1 + o * 8);
    }
  }
}

template <int V, int R>
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(QuadCfg<V>::NUM_THREADS, 1)
    tcec_gemm_quad_kernel(const __grid_constant__ CUtensorMap tmA,  // A [m][k], box 32 x 64, SW128
                          const __grid_constant__ CUtensorMap tmB,  // B [k][n], box 32 x 32, SW128
                          float* __restrict__ Cout, const int64_t ldc, const GemmShape shp,
                          const float scale, const float inv_scale, const FlagThresholds thr,
                          uint32_t* __restrict__ flags, uint32_t* __restrict__ wave_ctr) {
  using C = QuadCfg<V>;
  using VC = VarCfg<V>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* stg_full = bars;                    // TMA -> split            (local)
  uint64_t* stg_empty = bars + C::NSTG;         // split -> TMA            (local, 8)
  uint64_t* op_full = bars + 2 * C::NSTG;       // split -> MMA            (pair leader, 32)
  uint64_t* op_empty = op_full + C::NOP;        // both pairs' MMA commits -> split (2)
  uint64_t* p_full = op_empty + C::NOP;         // MMA commit -> drain     (pair, multicast)
  uint64_t* p_empty = p_full + 1;               // drain -> MMA            (pair leader, 16)
  uint64_t* acc_empty = bars + C::NUM_BARS;     // epilogue -> next unit's MMA (pair leader, 16)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::NUM_BARS + 1);
  const uint32_t smem_base = sm100::smem_u32(smem);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t crank = sm100::cluster_ctarank();
  const uint32_t rank = crank & 1u;             // rank within the pair (TMEM rows 0-127 / 128-255)
  const int p = static_cast<int>(crank >> 1);   // pair within the quad (tile column 2j + p)
  const uint32_t leader = crank & ~1u;          // this pair's MMA CTA
  const int tiles_m = (shp.m + 2 * C::BM - 1) / (2 * C::BM);
  const int tiles_n = (shp.n + C::BN - 1) / C::BN;
  const int tiles_np = (tiles_n + 1) / 2;
  const int num_units = tiles_m * tiles_np;
  const int nquads = gridDim.x >> 2;
  const int qid = blockIdx.x >> 2;
  const int nop = shp.num_op_stages;
  const int nstg = nop * VC::STG_PER_OP;
  const int de = shp.drain_every;
  const int nintervals = (nop + de - 1) / de;

  if (warp == 0 && lane == 0) {
    if (smem_base & 1023u) __trap();
    sm100::tma_prefetch_desc(&tmA);
    sm100::tma_prefetch_desc(&tmB);
    for (int s = 0; s < C::NSTG; ++s) {
      sm100::mbar_init(&stg_full[s], 1);
      sm100::mbar_init(&stg_empty[s], C::NUM_SPLIT_WARPS);
    }
    for (int o = 0; o < C::NOP; ++o) {
      sm100::mbar_init(&op_full[o], 4 * C::NUM_SPLIT_WARPS);
      sm100::mbar_init(&op_empty[o], 2);
    }
    sm100::mbar_init(p_full, 1);
    sm100::mbar_init(p_empty, 2 * C::NUM_DRAIN_WARPS);
    sm100::mbar_init(acc_empty, 2 * C::NUM_DRAIN_WARPS);
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
      uint32_t gst = 0;
      uint32_t target = 0;
      int wave = 0;
      for (int u = qid; u < num_units; u += nquads, ++wave) {
        if (wave_ctr != nullptr && wave > 0) {  // lock-step waves, bounded wait (tcec_gemm5.cuh)
          target += 4u * static_cast<uint32_t>(min(nquads, num_units - wave * nquads));
          atomicAdd(wave_ctr, 1u);
          uint32_t v;
          for (int spin = 0; spin < 2000; ++spin) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(wave_ctr) : "memory");
            if (v >= target) break;
            __nanosleep(100);
          }
        }
        int tm, tj;
        grouped_tile(u, tiles_m, tiles_np, shp.group_m, tm, tj);
        const int tn = 2 * tj + p;
        const int m_cta = tm * 2 * C::BM + rank * C::BM + p * C::A_ROWS;
        const int n_cta = tn * C::BN + rank * C::BN_CTA;
        for (int st = 0; st < nstg; ++st, ++gst) {
          const int s = gst % C::NSTG;
          sm100::mbar_wait(&stg_empty[s], ((gst / C::NSTG) & 1) ^ 1);
          uint8_t* dst = smem + C::OFF_STG + s * C::STG_BYTES;
          sm100::mbar_arrive_expect_tx(&stg_full[s], C::STG_BYTES);
          sm100::tma_load_2d(dst, &tmA, &stg_full[s], st * C::BK_STG, m_cta);
#pragma unroll
          for (int b = 0; b < 4; ++b)
            sm100::tma_load_2d(dst + C::STG_A_BYTES + b * C::STG_B_BOX, &tmB, &stg_full[s],
                               n_cta + 32 * b, st * C::BK_STG);
        }
      }
    } else if (warp == 1 && lane == 0 && rank == 0) {
      // ===================== MMA issuer (pair leader) =====================
      using PC = PairCfg<V>;
      constexpr uint32_t idesc = sm100::umma_idesc_bmn(VC::AB_FORMAT, 2 * C::BM, C::BN);
      constexpr uint32_t a_hi_w = (1024u >> 4) | (1u << 14) | (2u << 29);
      constexpr uint32_t b_hi_w = (uint32_t(PC::B_SBO) >> 4) | (1u << 14) | (PC::B_LAYOUT << 29);
      constexpr uint32_t b_lbo_w = (uint32_t(PC::B_LBO) >> 4) << 16;
      constexpr uint32_t kB = PC::B_KSTEP_BYTES >> 4;
      const uint16_t pair_mask = static_cast<uint16_t>(0x3u << (2 * p));
      uint32_t g = 0, git = 0, gtile = 0;
      for (int u = qid; u < num_units; u += nquads, ++gtile) {
        for (int kb = 0; kb < nop; ++kb, ++g) {
          const int o = g % C::NOP;
          sm100::mbar_wait_cluster(&op_full[o], (g / C::NOP) & 1);
          sm100::tc_fence_after();
          if (kb == 0 && gtile > 0) {  // the previous unit's epilogue has read dC
            sm100::mbar_wait_cluster(acc_empty, (gtile - 1) & 1);
            sm100::tc_fence_after();
          }
          // descriptor start address: 14 bits of (address >> 4).  The shared
          // address of cluster CTA ranks >= 2 carries the rank above bit 24,
          // which would otherwise spill into the descriptor's LBO field.
          const uint32_t op = (sm100::opaque(smem_base + C::OFF_OP + o * C::OP_BYTES) >> 4) & 0x3FFFu;
          const uint32_t ahi = op | (1u << 16);
          const uint32_t alo = ahi + (C::OP_A_BYTES >> 4);
          const uint32_t bhi = (op + ((2 * C::OP_A_BYTES) >> 4)) | b_lbo_w;
          const uint32_t blo = bhi + (PC::OP_B_BYTES >> 4);
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {  // schemes.py:294-298
            sm100::mma_pair_split<V == kTF32>(tmem_dC, alo + 2 * ks, a_hi_w, bhi + kB * ks, b_hi_w,
                                              idesc, (kb | ks) != 0);
            sm100::mma_pair_split<V == kTF32>(tmem_dC, ahi + 2 * ks, a_hi_w, blo + kB * ks, b_hi_w,
                                              idesc, 1u);
          }
          const bool first_in_interval = (kb % de) == 0;
          if (first_in_interval && git > 0) {
            sm100::mbar_wait_cluster(p_empty, (git - 1) & 1);
            sm100::tc_fence_after();
          }
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)
            sm100::mma_pair_split<V == kTF32>(tmem_P, ahi + 2 * ks, a_hi_w, bhi + kB * ks, b_hi_w,
                                              idesc, !(first_in_interval && ks == 0));
          // the stage's A halves came from both pairs: release it in all four CTAs
          sm100::mma_commit_pair_mc(&op_empty[o], 0xF);
          if ((kb % de) == de - 1 || kb == nop - 1) {
            sm100::mma_commit_pair_mc(p_full, pair_mask);
            ++git;
          }
        }
      }
    }
  } else if (warp < C::DRAIN_WARP0) {
    sm100::regs_dec<56>();
    // ===================== split warps =====================
    const int t = threadIdx.x - C::SPLIT_WARP0 * 32;
    const uint32_t op_full_l0 = sm100::mapa_shared(sm100::smem_u32(op_full), 0);
    const uint32_t op_full_l1 = sm100::mapa_shared(sm100::smem_u32(op_full), 2);
    const uint32_t rsmem = sm100::mapa_shared(smem_base, crank ^ 2u);
    uint32_t g = 0;
    for (int u = qid; u < num_units; u += nquads, g += nop) {
      int tm, tj;
      grouped_tile(u, tiles_m, tiles_np, shp.group_m, tm, tj);
      FlagAcc fa;
      // every A row block is split (half per pair) in the units with tj == 0,
      // every B column block in the units with tm == 0
      if (flags != nullptr && (tj == 0 || tm == 0)) {
        quad_split_tile<V, R, true>(smem_base, rsmem, stg_full, stg_empty, op_empty, op_full_l0,
                                    op_full_l1, g, nop, t, lane, p, scale, fa);
        flag_publish(fa, thr, flags);
      } else {
        quad_split_tile<V, R, false>(smem_base, rsmem, stg_full, stg_empty, op_empty, op_full_l0,
                                     op_full_l1, g, nop, t, lane, p, scale, fa);
      }
    }
  } else {
    // setmaxnreg redistributes the launch allocation: 4 x 40 + 8 x 56 + 8 x 160 <= 20 x 96
    sm100::regs_inc<160>();
    // ===================== drain + epilogue =====================
    const int q = warp & 3;
    const int h = (warp - C::DRAIN_WARP0) >> 2;
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    const uint32_t p_empty_leader = sm100::mapa_shared(sm100::smem_u32(p_empty), leader);
    const uint32_t acc_empty_leader = sm100::mapa_shared(sm100::smem_u32(acc_empty), leader);
    bool nonfinite = false;
    uint32_t git = 0;
    for (int u = qid; u < num_units; u += nquads) {
      int tm, tj;
      grouped_tile(u, tiles_m, tiles_np, shp.group_m, tm, tj);
      const int tn = 2 * tj + p;
      float acc[128];
#pragma unroll
      for (int j = 0; j < 128; ++j) acc[j] = 0.0f;
      for (int it = 0; it < nintervals; ++it, ++git) {
        sm100::mbar_wait(p_full, git & 1);
        sm100::tc_fence_after();
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          uint32_t r[8];
          sm100::tmem_ld_32x32b_x8(tmem_P + lane_off + h * 128 + c * 8, r);
          sm100::tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 8; j += 2)  // schemes.py:300-304: c = RN32(c + partial)
            sm100::fadd2_rn(acc[c * 8 + j], acc[c * 8 + j + 1], __uint_as_float(r[j]),
                            __uint_as_float(r[j + 1]));
        }
        sm100::tc_fence_before();
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive_remote(p_empty_leader);
      }
      const int64_t row = static_cast<int64_t>(tm) * 2 * C::BM + rank * C::BM + q * 32 + lane;
      const int col0 = tn * C::BN + h * 128;
      float* crow = Cout + row * ldc + col0;
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        uint32_t r[8];
        sm100::tmem_ld_32x32b_x8(tmem_dC + lane_off + h * 128 + c * 8, r);
        sm100::tmem_ld_wait();
        float o[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {  // schemes.py:306-307: one rounding of c + dC * 2^-s
          o[j] = __fmaf_rn(__uint_as_float(r[j]), inv_scale, acc[c * 8 + j]);
          nonfinite |= !isfinite(o[j]) && row < shp.m && col0 + c * 8 + j < shp.n;
        }
        if (row < shp.m) {
          const int col = col0 + c * 8;
          if (col + 8 <= shp.n) {
            *reinterpret_cast<float4*>(crow + c * 8) = make_float4(o[0], o[1], o[2], o[3]);
            *reinterpret_cast<float4*>(crow + c * 8 + 4) = make_float4(o[4], o[5], o[6], o[7]);
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (col + j < shp.n) crow[c * 8 + j] = o[j];
          }
        }
      }
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive_remote(acc_empty_leader);
    }
    if (flags != nullptr && __any_sync(0xFFFFFFFFu, nonfinite) && lane == 0)
      atomicOr(flags, kFlagOverflow);
  }

  __syncthreads();
  sm100::cluster_sync();
  if (warp == 2) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc_pair<C::TMEM_COLS>(tmem_base);
  }
}

}  // namespace tcec
