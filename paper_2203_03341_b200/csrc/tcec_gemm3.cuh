// tcec_gemm3.cuh -- CTA-pair TCEC SGEMM with unified split + drain workers.
//
// Same 256 x 256 cta_group::2 tile, operand layouts, barriers and MMA issue
// order as tcec_gemm_pair_kernel (tcec_gemm2.cuh), but the 16 non-control
// warps of each CTA are one pool of "workers" that both split the FP32
// slices into hi / lo operands and drain the main-term partial P:
//
//   for each operand stage kb:
//     split stage kb (8 A + 8 B values per thread per 32-deep slice)
//     signal the leader's op_full
//     drain P of the interval that ended at stage kb - 1 (while the tensor
//     core runs the corrections of stage kb), signal the leader's p_empty
//
// Four workers per scheduler (instead of two splitters and two mostly idle
// drainers) hide the LDS / convert latency of the split, and the drain's
// FADDs use otherwise idle issue slots.  Each worker keeps 64 of the CTA's
// 128 x 256 running C values in registers (lane quadrant w & 3, columns
// 64 (w >> 2) ...).
#pragma once

#include "tcec_gemm2.cuh"

namespace tcec {

struct UniCfg {
  static constexpr int NUM_THREADS = 640;
  static constexpr int WORKER_WARP0 = 4;
  static constexpr int NUM_WORKER_WARPS = 16;
  static constexpr int COLS_PER_WORKER = 64;
  static constexpr int EPI_WORKER_BYTES = 32 * 64 * 4;  // 32 rows x 64 cols
};

// This worker thread's share (8 values of one A row, 8 values of one B k-row)
// of a 32-deep FP32 slice -> operand stage.  t = 0..511:
//   A: row t & 127, k in [8 (t >> 7), +8)
//   B: k t & 31,    n in [8 (t >> 5), +8)
template <int V, int R, bool kFlags, bool kB>
__device__ __forceinline__ void uni_split_part(uint32_t stg, uint32_t op, int sub, int t,
                                               float scale, FlagAcc& fa) {
  using C = PairCfg<V>;
  float x[16];  // only the first 8 are used (split16 works on 16; the tail is ignored)
  uint32_t row;
  int q8;
  if constexpr (!kB) {
    row = t & 127;
    q8 = t >> 7;  // 8-value group within the 32-deep slice
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const float4 v = sm100::lds128(stg + sw128(row, q8 * 2 + i));
      x[4 * i] = v.x; x[4 * i + 1] = v.y; x[4 * i + 2] = v.z; x[4 * i + 3] = v.w;
    }
  } else {
    row = t & 31;
    q8 = t >> 5;  // 8-column group (0..15)
    const uint32_t box = stg + C::STG_A_BYTES + (q8 >> 2) * C::STG_B_BOX;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const float4 v = sm100::lds128(box + sw128(row, (q8 & 3) * 2 + i));
      x[4 * i] = v.x; x[4 * i + 1] = v.y; x[4 * i + 2] = v.z; x[4 * i + 3] = v.w;
    }
  }
#pragma unroll
  for (int i = 8; i < 16; ++i) x[i] = 0.0f;
  if constexpr (kFlags) {
#pragma unroll
    for (int i = 0; i < 8; ++i) fa.add(x[i]);
  }
  const uint32_t hi_base = op + (kB ? 2 * C::OP_A_BYTES : 0);
  const uint32_t lo_base = hi_base + (kB ? C::OP_B_BYTES : C::OP_A_BYTES);
#if TCEC_EXP & 1
  sm100::sts128(hi_base + sw128(t & 127, sub * 4 + ((t >> 7) & 3)), 0x3c003c00u, 0, 0, 0);
  sm100::sts128(lo_base + sw128(t & 127, sub * 4 + ((t >> 7) & 3)), 0x3c003c00u, 0, 0, 0);
  return;
#endif
  uint32_t hw[16], lw[16];
  split16<V, R>(x, scale, hw, lw);
  constexpr int NCH = V == kFP16 ? 1 : 2;  // 16-byte chunks per 8 values
  if constexpr (!kB) {
    const int chunk_first = V == kFP16 ? sub * 4 + q8 : q8 * 2;
#pragma unroll
    for (int q = 0; q < NCH; ++q) {
      const uint32_t off = sw128(row, chunk_first + q);
      sm100::sts128(hi_base + off, hw[4 * q], hw[4 * q + 1], hw[4 * q + 2], hw[4 * q + 3]);
      sm100::sts128(lo_base + off, lw[4 * q], lw[4 * q + 1], lw[4 * q + 2], lw[4 * q + 3]);
    }
  } else {
    const int kop = sub * 32 + row;
    const int grp = kop / C::B_ROWS, rr = kop % C::B_ROWS;
    const int n0 = q8 * 8;
    const uint32_t base = grp * C::B_SBO + (n0 / C::B_ATOM_N) * C::B_LBO + rr * 128;
    const int chunk_first = (n0 % C::B_ATOM_N) * (V == kFP16 ? 2 : 4) / 16;
#pragma unroll
    for (int q = 0; q < NCH; ++q) {
      const int c16 = chunk_first + q;
      const uint32_t off = V == kFP16 ? base + ((c16 ^ rr) << 4)
                                      : base + ((((c16 >> 1) ^ rr) & 3) << 5) + ((c16 & 1) << 4);
      sm100::sts128(hi_base + off, hw[4 * q], hw[4 * q + 1], hw[4 * q + 2], hw[4 * q + 3]);
      sm100::sts128(lo_base + off, lw[4 * q], lw[4 * q + 1], lw[4 * q + 2], lw[4 * q + 3]);
    }
  }
}

// Drain one interval: C += P for this worker's 32 lanes x 64 columns.
__device__ __forceinline__ void uni_drain(float (&acc)[64], uint32_t tmem_P, uint32_t lane_off,
                                          int cb, uint64_t* p_full, int it,
                                          uint32_t p_empty_leader, int lane) {
  sm100::mbar_wait(p_full, it & 1);
  sm100::tc_fence_after();
#if !(TCEC_EXP & 2)
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint32_t r[16];
    sm100::tmem_ld_32x32b_x16(tmem_P + lane_off + cb * 64 + c * 16, r);
    sm100::tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 16; ++j)  // schemes.py:300-304: c = RN32(c + partial)
      acc[c * 16 + j] = __fadd_rn(acc[c * 16 + j], __uint_as_float(r[j]));
  }
#endif
  sm100::tc_fence_before();
  __syncwarp();
  // the TMEM reads above have completed (wait::ld); P may be overwritten
  if (lane == 0) sm100::mbar_arrive_remote(p_empty_leader);
}

template <int V, int R, bool kFlags>
__device__ __forceinline__ void uni_worker_loop(uint32_t smem, uint64_t* stg_full,
                                                uint64_t* stg_empty, uint64_t* op_full,
                                                uint64_t* op_empty, uint64_t* p_full,
                                                uint64_t* p_empty, uint32_t tmem_P, int nop,
                                                int de, int t, int lane, float scale,
                                                FlagAcc& fa, float (&acc)[64]) {
  using C = PairCfg<V>;
  using VC = VarCfg<V>;
  const uint32_t leader_op_full = sm100::mapa_shared(sm100::smem_u32(op_full), 0);
  const uint32_t p_empty_leader = sm100::mapa_shared(sm100::smem_u32(p_empty), 0);
  const int w = t >> 5;
  const uint32_t lane_off = static_cast<uint32_t>((w & 3) * 32) << 16;
  const int cb = w >> 2;
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
      uni_split_part<V, R, kFlags, false>(stg, op, sub, t, scale, fa);
      uni_split_part<V, R, kFlags, true>(stg, op, sub, t, scale, fa);
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&stg_empty[s]);
    }
    sm100::fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) sm100::mbar_arrive_remote(leader_op_full + o * 8);
    // the interval that ended at stage kb - 1 (not the last one) is drained now,
    // while the tensor core runs the corrections of stage kb
    if (kb >= 1 && ((kb - 1) % de) == de - 1)
      uni_drain(acc, tmem_P, lane_off, cb, p_full, (kb - 1) / de, p_empty_leader, lane);
  }
  const int nintervals = (nop + de - 1) / de;
  uni_drain(acc, tmem_P, lane_off, cb, p_full, nintervals - 1, p_empty_leader, lane);
}

template <int V, int R>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(UniCfg::NUM_THREADS, 1)
    tcec_gemm_pair_uni_kernel(const __grid_constant__ CUtensorMap tmA,
                              const __grid_constant__ CUtensorMap tmB,
                              const __grid_constant__ CUtensorMap tmC,
                              const __grid_constant__ CDests cx, const GemmShape shp,
                              const float scale, const float inv_scale, const FlagThresholds thr,
                              uint32_t* __restrict__ flags) {
  using C = PairCfg<V>;
  using VC = VarCfg<V>;
  using U = UniCfg;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* stg_full = bars;                    // TMA -> workers        (local)
  uint64_t* stg_empty = bars + C::NSTG;         // workers -> TMA        (local, 16)
  uint64_t* op_full = bars + 2 * C::NSTG;       // workers -> MMA        (leader, 32)
  uint64_t* op_empty = op_full + C::NOP;        // MMA commit -> workers (both, multicast)
  uint64_t* p_full = op_empty + C::NOP;         // MMA commit -> workers (both, multicast)
  uint64_t* p_empty = p_full + 1;               // workers -> MMA        (leader, 32)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::NUM_BARS);
  const uint32_t smem_base = sm100::smem_u32(smem);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = sm100::cluster_ctarank();

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
  const int m_cta = tile_m * 2 * C::BM + rank * C::BM;
  const int n_pair = tile_n * C::BN;
  const int n_cta = n_pair + rank * C::BN_CTA;
  const int nop = shp.num_op_stages;
  const int nstg = nop * VC::STG_PER_OP;
  const int de = shp.drain_every;

  if (warp == 0 && lane == 0) {
    if (smem_base & 1023u) __trap();
    sm100::tma_prefetch_desc(&tmA);
    sm100::tma_prefetch_desc(&tmB);
    sm100::tma_prefetch_desc(&tmC);
    for (int s = 0; s < C::NSTG; ++s) {
      sm100::mbar_init(&stg_full[s], 1);
      sm100::mbar_init(&stg_empty[s], U::NUM_WORKER_WARPS);
    }
    for (int o = 0; o < C::NOP; ++o) {
      sm100::mbar_init(&op_full[o], 2 * U::NUM_WORKER_WARPS);
      sm100::mbar_init(&op_empty[o], 1);
    }
    sm100::mbar_init(p_full, 1);
    sm100::mbar_init(p_empty, 2 * U::NUM_WORKER_WARPS);
    sm100::fence_mbar_init();
  }
  if (warp == 2) sm100::tmem_alloc_pair<C::TMEM_COLS>(tmem_slot);
  sm100::tc_fence_before();
  sm100::cluster_sync();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t tmem_P = tmem_base;
  const uint32_t tmem_dC = tmem_base + C::BN;

  if (warp < U::WORKER_WARP0) {
    sm100::regs_dec<32>();
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
    } else if (warp == 1 && lane == 0 && rank == 0) {
      // ===================== MMA issuer (leader CTA) =====================
      constexpr uint32_t idesc = sm100::umma_idesc_bmn(VC::AB_FORMAT, 2 * C::BM, C::BN);
      constexpr uint32_t a_hi_w = (1024u >> 4) | (1u << 14) | (2u << 29);
      constexpr uint32_t b_hi_w = (uint32_t(C::B_SBO) >> 4) | (1u << 14) | (C::B_LAYOUT << 29);
      constexpr uint32_t b_lbo_w = (uint32_t(C::B_LBO) >> 4) << 16;
      constexpr uint32_t kB = C::B_KSTEP_BYTES >> 4;
      for (int kb = 0; kb < nop; ++kb) {
        const int o = kb % C::NOP;
        sm100::mbar_wait_cluster(&op_full[o], (kb / C::NOP) & 1);
        sm100::tc_fence_after();
        const uint32_t op = sm100::opaque(smem_base + C::OFF_OP + o * C::OP_BYTES) >> 4;
        const uint32_t ahi = op | (1u << 16);
        const uint32_t alo = ahi + (C::OP_A_BYTES >> 4);
        const uint32_t bhi = (op + ((2 * C::OP_A_BYTES) >> 4)) | b_lbo_w;
        const uint32_t blo = bhi + (C::OP_B_BYTES >> 4);
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          sm100::mma_pair_split<V == kTF32>(tmem_dC, alo + 2 * ks, a_hi_w, bhi + kB * ks, b_hi_w,
                                            idesc, (kb | ks) != 0);
          sm100::mma_pair_split<V == kTF32>(tmem_dC, ahi + 2 * ks, a_hi_w, blo + kB * ks, b_hi_w,
                                            idesc, 1u);
        }
        const bool first_in_interval = (kb % de) == 0;
        if (first_in_interval && kb > 0) {
          sm100::mbar_wait_cluster(p_empty, ((kb / de) - 1) & 1);
          sm100::tc_fence_after();
        }
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          sm100::mma_pair_split<V == kTF32>(tmem_P, ahi + 2 * ks, a_hi_w, bhi + kB * ks, b_hi_w,
                                            idesc, !(first_in_interval && ks == 0));
        sm100::mma_commit_pair_mc(&op_empty[o], 0x3);
        if ((kb % de) == de - 1 || kb == nop - 1) sm100::mma_commit_pair_mc(p_full, 0x3);
      }
    }
  } else {
    sm100::regs_inc<112>();
    // ===================== workers: split + drain + epilogue =====================
    const int t = threadIdx.x - U::WORKER_WARP0 * 32;
    const int w = t >> 5;
    float acc[64];
#pragma unroll
    for (int j = 0; j < 64; ++j) acc[j] = 0.0f;
    FlagAcc fa;
    const bool do_flags = flags != nullptr && (tile_n == 0 || tile_m == 0);
    if (do_flags) {
      uni_worker_loop<V, R, true>(smem_base, stg_full, stg_empty, op_full, op_empty, p_full,
                                  p_empty, tmem_P, nop, de, t, lane, scale, fa, acc);
      flag_publish(fa, thr, flags);
    } else {
      uni_worker_loop<V, R, false>(smem_base, stg_full, stg_empty, op_full, op_empty, p_full,
                                   p_empty, tmem_P, nop, de, t, lane, scale, fa, acc);
    }
    // every MMA of the pair has completed (the last p_full follows them); all
    // workers' staging reads precede the epilogue's staging writes
    sm100::named_barrier_sync<1, 32 * U::NUM_WORKER_WARPS>();
    const int q = w & 3, cb = w >> 2;
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    bool nonfinite = false;
    const uint32_t stage = smem_base + w * U::EPI_WORKER_BYTES;
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const uint32_t box = stage + b * 4096;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t r[16];
        sm100::tmem_ld_32x32b_x16(tmem_dC + lane_off + cb * 64 + b * 32 + c * 16, r);
        sm100::tmem_ld_wait();
        float o[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
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
        sm100::tma_store_2d(&tmC, smem + (box - smem_base), n_pair + cb * 64 + b * 32, m_cta + q * 32);
        for (int d = 0; d < cx.count; ++d)
          sm100::tma_store_2d(&cx.m[d], smem + (box - smem_base), n_pair + cb * 64 + b * 32,
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
