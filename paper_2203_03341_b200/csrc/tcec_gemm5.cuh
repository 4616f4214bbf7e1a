// tcec_gemm5.cuh -- persistent variant of the CTA-pair kernel (opts.reserved[1] = 2).
//
// Same warp roles, rings, MMA order, drain and per-element arithmetic as
// tcec_gemm2.cuh; the difference is the tile loop.  One CTA pair per TPC stays
// resident and walks the grouped-raster tile sequence pid, pid + P, ... (P =
// number of pairs), with every pipeline counter (staging slices, operand
// stages, drain intervals) running on across tiles:
//
//   * the TMA producer and the split warps start the next tile's slices while
//     the drain warps are still in the previous tile's epilogue;
//   * the MMA warp waits for `acc_empty` (both CTAs' drain warps have read dC)
//     before the next tile's first correction MMA, and for `p_empty` as usual
//     before its first main-term MMA;
//   * the epilogue writes C straight from registers (st.global.v4, each thread
//     512 contiguous bytes of its row): the staging ring is busy with the next
//     tile, so there is no shared-memory staging for a TMA store.
//
// C is bit-identical to the non-persistent kernel.
//
// With kSplitK (opts.split_k > 1) the same kernel walks (tile, k part) units
// and stores each part's partial sums for tcec_splitk_reduce_kernel (below),
// which combines them in a fixed part order.
#pragma once

#include "tcec_gemm2.cuh"

namespace tcec {

__device__ __forceinline__ void grouped_tile(int tile, int tiles_m, int tiles_n, int group_m,
                                             int& tile_m, int& tile_n) {
  const int per_group = group_m * tiles_n;
  const int g = tile / per_group;
  const int first_m = g * group_m;
  const int gsize = min(tiles_m - first_m, group_m);
  const int in_g = tile - g * per_group;
  tile_m = first_m + in_g % gsize;
  tile_n = in_g / gsize;
}

// Split `nop` operand stages of one tile; `g0` is the global operand-stage
// counter at the tile's first stage (ring slots and phases continue across tiles).
template <int V, int R, bool kFlags>
__device__ __forceinline__ void pers_split_tile(uint32_t smem, uint64_t* stg_full,
                                                uint64_t* stg_empty, uint64_t* op_empty,
                                                uint32_t leader_op_full, uint32_t g0, int nop,
                                                int t, int lane, float scale, FlagAcc& fa) {
  using C = PairCfg<V>;
  using VC = VarCfg<V>;
  for (int kb = 0; kb < nop; ++kb) {
    const uint32_t g = g0 + kb;
    const int o = g % C::NOP;
    const uint32_t op = smem + C::OFF_OP + o * C::OP_BYTES;
#pragma unroll
    for (int sub = 0; sub < VC::STG_PER_OP; ++sub) {
      const uint32_t gst = g * VC::STG_PER_OP + sub;
      const int s = gst % C::NSTG;
      sm100::mbar_wait(&stg_full[s], (gst / C::NSTG) & 1);
      if (sub == 0) sm100::mbar_wait(&op_empty[o], ((g / C::NOP) & 1) ^ 1);
      const uint32_t stg = smem + C::OFF_STG + s * C::STG_BYTES;
      pair_split_part<V, R, kFlags, false>(stg, op, sub, t, scale, fa);
      pair_split_part<V, R, kFlags, true>(stg, op, sub, t, scale, fa);
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&stg_empty[s]);
    }
    sm100::fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) sm100::mbar_arrive_remote(leader_op_full + o * 8);
  }
}

// kSplitK: the units of work are (tile, k part) pairs -- unit u is tile
// u % T over operand stages [p nop / S, (p + 1) nop / S), p = u / T -- and the
// epilogue stores the part's main-term sum and raw dC to `ws` (planes 2p and
// 2p + 1 of m x n) for tcec_splitk_reduce_kernel instead of combining them.
template <int V, int R, bool kSplitK = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PairCfg<V>::NUM_THREADS, 1)
    tcec_gemm_pers_kernel(const __grid_constant__ CUtensorMap tmA,  // A [m][k], box 32 x 128, SW128
                          const __grid_constant__ CUtensorMap tmB,  // B [k][n], box 32 x 32, SW128
                          float* __restrict__ Cout, const int64_t ldc, const GemmShape shp,
                          const float scale, const float inv_scale, const FlagThresholds thr,
                          uint32_t* __restrict__ flags, uint32_t* __restrict__ wave_ctr,
                          float* __restrict__ ws, const int ksplit) {
  using C = PairCfg<V>;
  using VC = VarCfg<V>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* stg_full = bars;                    // TMA -> split          (local)
  uint64_t* stg_empty = bars + C::NSTG;         // split -> TMA          (local, 8)
  uint64_t* op_full = bars + 2 * C::NSTG;       // split -> MMA          (leader, 16)
  uint64_t* op_empty = op_full + C::NOP;        // MMA commit -> split   (both, multicast)
  uint64_t* p_full = op_empty + C::NOP;         // MMA commit -> drain   (both, multicast)
  uint64_t* p_empty = p_full + 1;               // drain -> MMA          (leader, 16)
  // the 16-byte tail after the barriers: acc_empty (epilogue read dC -> MMA,
  // leader, 16 arrivals) and the TMEM base address
  uint64_t* acc_empty = bars + C::NUM_BARS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::NUM_BARS + 1);
  const uint32_t smem_base = sm100::smem_u32(smem);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = sm100::cluster_ctarank();
  const int tiles_m = (shp.m + 2 * C::BM - 1) / (2 * C::BM);
  const int tiles_n = (shp.n + C::BN - 1) / C::BN;
  const int num_tiles = tiles_m * tiles_n;
  const int npairs = gridDim.x >> 1;
  const int pid = blockIdx.x >> 1;
  const int nop = shp.num_op_stages;
  const int de = shp.drain_every;  // MMA k-steps per drain interval
  const int nparts = kSplitK ? ksplit : 1;
  const int num_units = num_tiles * nparts;
  // unit -> (tile, operand stages [kb0, kb1))
  auto unit_of = [&](int u, int& tile, int& part, int& kb0, int& kb1) {
    if constexpr (kSplitK) {
      tile = u % num_tiles;
      part = u / num_tiles;
      kb0 = static_cast<int>(static_cast<int64_t>(part) * nop / nparts);
      kb1 = static_cast<int>(static_cast<int64_t>(part + 1) * nop / nparts);
    } else {
      tile = u;
      part = 0;
      kb0 = 0;
      kb1 = nop;
    }
  };

  if (warp == 0 && lane == 0) {
    if (smem_base & 1023u) __trap();
    sm100::tma_prefetch_desc(&tmA);
    sm100::tma_prefetch_desc(&tmB);
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
      for (int u = pid; u < num_units; u += npairs, ++wave) {
        int tile, part, kb0, kb1;
        unit_of(u, tile, part, kb0, kb1);
        if (wave_ctr != nullptr && wave > 0) {
          // lock-step waves: the CTAs that have a tile in this wave all finish
          // issuing the previous wave's loads before any starts this one, so the
          // tiles of a wave read the same k-slices while they are in L2.
          // Arrivals for wave w come from the 2 min(P, T - wP) CTAs with a wave-w tile.
          target += 2u * static_cast<uint32_t>(min(npairs, num_units - wave * npairs));
          // The wait is bounded (~0.2 ms): the barrier only shapes L2 reuse, so a
          // CTA that cannot see its peers (e.g. not co-resident because another
          // kernel holds SMs) goes on instead of deadlocking.
          atomicAdd(wave_ctr, 1u);
          uint32_t v;
          for (int spin = 0; spin < 2000; ++spin) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(wave_ctr) : "memory");
            if (v >= target) break;
            __nanosleep(100);
          }
        }
        int tm, tn;
        grouped_tile(tile, tiles_m, tiles_n, shp.group_m, tm, tn);
        const int m_cta = tm * 2 * C::BM + rank * C::BM;
        const int n_cta = tn * C::BN + rank * C::BN_CTA;
        for (int st = kb0 * VC::STG_PER_OP; st < kb1 * VC::STG_PER_OP; ++st, ++gst) {
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
    } else if (warp == 1 && rank == 0) {  // the whole warp runs the issue loop; one elected lane issues
      // ===================== MMA issuer (leader CTA) =====================
      constexpr uint32_t idesc = sm100::umma_idesc_bmn(VC::AB_FORMAT, 2 * C::BM, C::BN);
      constexpr uint32_t a_hi_w = (1024u >> 4) | (1u << 14) | (2u << 29);
      constexpr uint32_t b_hi_w = (uint32_t(C::B_SBO) >> 4) | (1u << 14) | (C::B_LAYOUT << 29);
      constexpr uint32_t b_lbo_w = (uint32_t(C::B_LBO) >> 4) << 16;
      constexpr uint32_t kB = C::B_KSTEP_BYTES >> 4;
      uint32_t g = 0, git = 0, gtile = 0;
      int pos = 0;
      for (int u = pid; u < num_units; u += npairs, ++gtile) {
        int tile, part, kb0, kb1;
        unit_of(u, tile, part, kb0, kb1);
        const int nop_u = kb1 - kb0;
        for (int kb = 0; kb < nop_u; ++kb, ++g) {
          const int o = g % C::NOP;
          sm100::mbar_wait_cluster(&op_full[o], (g / C::NOP) & 1);
          sm100::tc_fence_after();
          if (kb == 0 && gtile > 0) {  // the previous tile's epilogue has read dC
            sm100::mbar_wait_cluster(acc_empty, (gtile - 1) & 1);
            sm100::tc_fence_after();
          }
          const uint32_t op = sm100::opaque(smem_base + C::OFF_OP + o * C::OP_BYTES) >> 4;
          const uint32_t ahi = op | (1u << 16);
          const uint32_t alo = ahi + (C::OP_A_BYTES >> 4);
          const uint32_t bhi = (op + ((2 * C::OP_A_BYTES) >> 4)) | b_lbo_w;
          const uint32_t blo = bhi + (C::OP_B_BYTES >> 4);
          c3_stage(
              kb * 4, 4 * nop_u, de, pos, git, p_empty, p_full, &op_empty[o],
              [&](int ks) {  // schemes.py:294-298: dA*B_hi, then A_hi*dB
                sm100::mma_pair_split_el<V == kTF32>(tmem_dC, alo + 2 * ks, a_hi_w, bhi + kB * ks,
                                                  b_hi_w, idesc, (kb | ks) != 0);
                sm100::mma_pair_split_el<V == kTF32>(tmem_dC, ahi + 2 * ks, a_hi_w, blo + kB * ks,
                                                  b_hi_w, idesc, 1u);
              },
              [&](int ks, uint32_t acc) {
                sm100::mma_pair_split_el<V == kTF32>(tmem_P, ahi + 2 * ks, a_hi_w, bhi + kB * ks,
                                                  b_hi_w, idesc, acc);
              });
        }
      }
    }
  } else if (warp < C::DRAIN_WARP0) {
    sm100::regs_dec<56>();
    // ===================== split warps =====================
    const int t = threadIdx.x - C::SPLIT_WARP0 * 32;
    const uint32_t leader_op_full = sm100::mapa_shared(sm100::smem_u32(op_full), 0);
    uint32_t g = 0;
    for (int u = pid; u < num_units; u += npairs) {
      int tile, part, kb0, kb1;
      unit_of(u, tile, part, kb0, kb1);
      const int nop_u = kb1 - kb0;
      int tm, tn;
      grouped_tile(tile, tiles_m, tiles_n, shp.group_m, tm, tn);
      FlagAcc fa;
      if (flags != nullptr && (tn == 0 || tm == 0)) {
        pers_split_tile<V, R, true>(smem_base, stg_full, stg_empty, op_empty, leader_op_full, g,
                                    nop_u, t, lane, scale, fa);
        flag_publish(fa, thr, flags);
      } else {
        pers_split_tile<V, R, false>(smem_base, stg_full, stg_empty, op_empty, leader_op_full, g,
                                     nop_u, t, lane, scale, fa);
      }
      g += nop_u;
    }
  } else {
    // setmaxnreg redistributes the launch allocation: 4 x 40 + 8 x 56 + 8 x 160 <= 20 x 96
    sm100::regs_inc<160>();
    // ===================== drain + epilogue =====================
    const int q = warp & 3;
    const int h = (warp - C::DRAIN_WARP0) >> 2;
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    const uint32_t p_empty_leader = sm100::mapa_shared(sm100::smem_u32(p_empty), 0);
    const uint32_t acc_empty_leader = sm100::mapa_shared(sm100::smem_u32(acc_empty), 0);
    bool nonfinite = false;
    uint32_t git = 0;
    for (int u = pid; u < num_units; u += npairs) {
      int tile, part, kb0, kb1;
      unit_of(u, tile, part, kb0, kb1);
      const int nintervals = (4 * (kb1 - kb0) + de - 1) / de;
      int tm, tn;
      grouped_tile(tile, tiles_m, tiles_n, shp.group_m, tm, tn);
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
      // epilogue: every MMA of the tile has completed (the last p_full follows them)
      const int64_t row = static_cast<int64_t>(tm) * 2 * C::BM + rank * C::BM + q * 32 + lane;
      const int col0 = tn * C::BN + h * 128;
      float* crow = Cout + row * ldc + col0;
      if constexpr (kSplitK) {
        // this part's main-term sum and raw dC, planes 2p / 2p + 1 (row pitch n8)
        const int64_t n8 = (shp.n + 7) & ~7;
        float* wc = ws + (2 * static_cast<int64_t>(part) * shp.m + row) * n8 + col0;
        float* wd = wc + static_cast<int64_t>(shp.m) * n8;
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          uint32_t r[8];
          sm100::tmem_ld_32x32b_x8(tmem_dC + lane_off + h * 128 + c * 8, r);
          sm100::tmem_ld_wait();
          const int col = col0 + c * 8;
          if (row < shp.m && col < shp.n) {  // n8 pitch: whole 8-column groups fit
            *reinterpret_cast<float4*>(wc + c * 8) =
                make_float4(acc[c * 8], acc[c * 8 + 1], acc[c * 8 + 2], acc[c * 8 + 3]);
            *reinterpret_cast<float4*>(wc + c * 8 + 4) =
                make_float4(acc[c * 8 + 4], acc[c * 8 + 5], acc[c * 8 + 6], acc[c * 8 + 7]);
            *reinterpret_cast<float4*>(wd + c * 8) =
                make_float4(__uint_as_float(r[0]), __uint_as_float(r[1]), __uint_as_float(r[2]),
                            __uint_as_float(r[3]));
            *reinterpret_cast<float4*>(wd + c * 8 + 4) =
                make_float4(__uint_as_float(r[4]), __uint_as_float(r[5]), __uint_as_float(r[6]),
                            __uint_as_float(r[7]));
          }
        }
      } else {
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
      }
      // dC (and the last P) read: the next tile's MMAs may overwrite them
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

// Split-K combine, one thread per 4 outputs, fixed part order (deterministic):
// c = RN(...RN(c_0 + c_1)... + c_{S-1}), d likewise, C = RN(c + d * 2^-s) --
// the single-pass epilogue (schemes.py:306-307) over the parts' partial sums.
__global__ void __launch_bounds__(256)
    tcec_splitk_reduce_kernel(const float* __restrict__ ws, int nparts, int m, int n,
                              float* __restrict__ Cout, int64_t ldc, float inv_scale,
                              uint32_t* __restrict__ flags) {
  const int64_t n8 = (n + 7) & ~7;
  const int64_t plane = static_cast<int64_t>(m) * n8;
  const int64_t quads = static_cast<int64_t>(m) * (n8 / 4);
  bool nonfinite = false;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < quads;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = i / (n8 / 4);
    const int col = static_cast<int>(i - row * (n8 / 4)) * 4;
    if (col >= n) continue;
    const int64_t off = row * n8 + col;
    float4 c = *reinterpret_cast<const float4*>(ws + off);
    float4 d = *reinterpret_cast<const float4*>(ws + plane + off);
    for (int p = 1; p < nparts; ++p) {
      const float4 cp = *reinterpret_cast<const float4*>(ws + 2 * p * plane + off);
      const float4 dp = *reinterpret_cast<const float4*>(ws + (2 * p + 1) * plane + off);
      c.x = __fadd_rn(c.x, cp.x); c.y = __fadd_rn(c.y, cp.y);
      c.z = __fadd_rn(c.z, cp.z); c.w = __fadd_rn(c.w, cp.w);
      d.x = __fadd_rn(d.x, dp.x); d.y = __fadd_rn(d.y, dp.y);
      d.z = __fadd_rn(d.z, dp.z); d.w = __fadd_rn(d.w, dp.w);
    }
    const float o[4] = {__fmaf_rn(d.x, inv_scale, c.x), __fmaf_rn(d.y, inv_scale, c.y),
                        __fmaf_rn(d.z, inv_scale, c.z), __fmaf_rn(d.w, inv_scale, c.w)};
    float* crow = Cout + row * ldc + col;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (col + j < n) {
        crow[j] = o[j];
        nonfinite |= !isfinite(o[j]);
      }
  }
  if (flags != nullptr && __any_sync(0xFFFFFFFFu, nonfinite) && (threadIdx.x & 31) == 0)
    atomicOr(flags, kFlagOverflow);
}

}  // namespace tcec
