// tcec_presplit.cuh -- split-once mode of the error-corrected SGEMM.
//
// The fused kernels (tcec_gemm2.cuh) re-split every A tile once per column
// tile of C and every B tile once per row tile (n / 256 and m / 256 times at
// 16384^3), and on the power-capped B200 the energy of that redundant split
// (FP32 staging through shared memory, split arithmetic, hi/lo stores) is what
// bounds the FP16 variant.  This mode
// splits each input element exactly once in an HBM-bandwidth-bound pass and
// then runs a plain three-product tcgen05 GEMM whose TMA loads the hi / lo
// operands straight into the UMMA layout:
//
//   tcec_presplit_kernel   X (FP32) -> hi, lo in the operand element type (FP16
//                          or TF32 bit patterns), K-major: A as m x k, B
//                          transposed to n x k; RunFlags from the same pass.
//   tcec_gemm_ps_kernel    persistent CTA pair (lock-step waves as in
//                          tcec_gemm5.cuh), 256 x 256 tiles, 3-deep ring of
//                          64 KB operand stages (A_hi, A_lo, B_hi, B_lo;
//                          128-byte swizzled K-major), the same MMA order and
//                          drain as the fused pair kernel, C stored from
//                          registers -- bit-identical C.
//
// Split arithmetic is split.cuh's (splitting.py:114-122), including lo = 0
// where hi overflowed.
#pragma once

#include "tcec_gemm5.cuh"

namespace tcec {

// ---------------------------------------------------------------------------
// Split pass: 64 x 64 tiles, 256 threads.  Output element (r, c) of X goes to
// out[r * ldo + c] (kTrans = false) or out[c * ldo + r] (kTrans = true); ldo is
// a multiple of 16 and every output row is written up to ldo (zeros past the
// matrix edge), so the GEMM's TMA sees a fully initialised, padded operand.
template <int V>
struct PsElem;
template <>
struct PsElem<kFP16> { using T = uint16_t; };
template <>
struct PsElem<kTF32> { using T = uint32_t; };

template <int V, int R, bool kTrans>
__global__ void __launch_bounds__(256)
    tcec_presplit_kernel(const float* __restrict__ X, int32_t rows, int32_t cols, int64_t ldx,
                         void* __restrict__ hi_out, void* __restrict__ lo_out, int64_t ldo,
                         int32_t out_rows, float scale, FlagThresholds thr,
                         uint32_t* __restrict__ flags) {
  using E = typename PsElem<V>::T;
  __shared__ uint32_t sh_hi[64][65];
  __shared__ uint32_t sh_lo[64][65];
  E* hi = static_cast<E*>(hi_out);
  E* lo = static_cast<E*>(lo_out);
  const int t = threadIdx.x;
  const int tiles_c = (cols + 63) / 64;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x / tiles_c) * 64;
  const int64_t c0 = static_cast<int64_t>(blockIdx.x % tiles_c) * 64;
  FlagAcc fa;
  const int cc = (t & 15) * 4;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int rr = (t >> 4) + 16 * i;
    const int64_t r = r0 + rr, c = c0 + cc;
    float x[4] = {0.f, 0.f, 0.f, 0.f};
    if (r < rows) {
      const float* src = X + r * ldx + c;
      if (c + 3 < cols && (reinterpret_cast<uintptr_t>(src) & 15u) == 0) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(src));
        x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (c + j < cols) x[j] = src[j];
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) fa.add(x[j]);
    uint32_t h[4], l[4];
    if constexpr (V == kFP16) {
      uint32_t hp0, lp0, hp1, lp1;
      split_f16_pair<R>(x[0], x[1], scale, hp0, lp0);
      split_f16_pair<R>(x[2], x[3], scale, hp1, lp1);
      h[0] = hp0 & 0xFFFFu; h[1] = hp0 >> 16; h[2] = hp1 & 0xFFFFu; h[3] = hp1 >> 16;
      l[0] = lp0 & 0xFFFFu; l[1] = lp0 >> 16; l[2] = lp1 & 0xFFFFu; l[3] = lp1 >> 16;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float hf, lf;
        split_tf32<R>(x[j], scale, hf, lf);
        h[j] = __float_as_uint(hf);
        l[j] = __float_as_uint(lf);
      }
    }
    if constexpr (!kTrans) {
      if (r < out_rows && c < ldo) {
        if constexpr (V == kFP16) {
          *reinterpret_cast<uint2*>(hi + r * ldo + c) = make_uint2(h[0] | (h[1] << 16), h[2] | (h[3] << 16));
          *reinterpret_cast<uint2*>(lo + r * ldo + c) = make_uint2(l[0] | (l[1] << 16), l[2] | (l[3] << 16));
        } else {
          *reinterpret_cast<uint4*>(hi + r * ldo + c) = make_uint4(h[0], h[1], h[2], h[3]);
          *reinterpret_cast<uint4*>(lo + r * ldo + c) = make_uint4(l[0], l[1], l[2], l[3]);
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        sh_hi[cc + j][rr] = h[j];
        sh_lo[cc + j][rr] = l[j];
      }
    }
  }
  if constexpr (kTrans) {
    __syncthreads();
    // output row c0 + oc (a column of X), elements r0 + orr .. +16
    const int oc = t >> 2, orr = (t & 3) * 16;
    const int64_t orow = c0 + oc, ocol = r0 + orr;
    if (orow < out_rows && ocol < ldo) {
      E* dh = hi + orow * ldo + ocol;
      E* dl = lo + orow * ldo + ocol;
      if constexpr (V == kFP16) {
        uint32_t ph[8], pl[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          ph[j] = sh_hi[oc][orr + 2 * j] | (sh_hi[oc][orr + 2 * j + 1] << 16);
          pl[j] = sh_lo[oc][orr + 2 * j] | (sh_lo[oc][orr + 2 * j + 1] << 16);
        }
        reinterpret_cast<uint4*>(dh)[0] = make_uint4(ph[0], ph[1], ph[2], ph[3]);
        reinterpret_cast<uint4*>(dh)[1] = make_uint4(ph[4], ph[5], ph[6], ph[7]);
        reinterpret_cast<uint4*>(dl)[0] = make_uint4(pl[0], pl[1], pl[2], pl[3]);
        reinterpret_cast<uint4*>(dl)[1] = make_uint4(pl[4], pl[5], pl[6], pl[7]);
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          reinterpret_cast<uint4*>(dh)[q] = make_uint4(sh_hi[oc][orr + 4 * q], sh_hi[oc][orr + 4 * q + 1],
                                                       sh_hi[oc][orr + 4 * q + 2], sh_hi[oc][orr + 4 * q + 3]);
          reinterpret_cast<uint4*>(dl)[q] = make_uint4(sh_lo[oc][orr + 4 * q], sh_lo[oc][orr + 4 * q + 1],
                                                       sh_lo[oc][orr + 4 * q + 2], sh_lo[oc][orr + 4 * q + 3]);
        }
      }
    }
  }
  flag_publish(fa, thr, flags);
}

// ---------------------------------------------------------------------------
// GEMM over pre-split operands.  The product schedule is a template parameter
// so the same pipeline also runs the reference's in-unit comparator schemes on
// the tensor core:
//   kSchC3    corrected3: dC += dA*B_hi, A_hi*dB (one TMEM accumulator over all
//             k), P = A_hi*B_hi drained into an FP32 RN register sum every
//             drain interval, C = RN(C + dC 2^-s)      (schemes.py:265-307)
//   kSchC3DD  corrected3 plus the dA*dB chain in its own accumulator, added
//             last as RN(C + ddC 2^-2s)              (schemes.py:308-313)
//   kSchPlain tc_plain: one product of the converted inputs, accumulated in
//             the unit over all k                    (schemes.py:343-351)
//   kSchIn4   markidis4 / corrected4 (hardware terminal): dA*dB, dA*B, A*dB,
//             A*B per k-step into one accumulator    (schemes.py:352-364)
//   kSchIn4RN corrected4 with the RN terminal (schemes.py:352-364, terminal RN):
//             the same four terms, each in its own TMEM accumulator over one
//             block of `drain_every` MMA k-steps, drained in the reference's
//             term order into an FP32 RN register sum -- c = RN(c + P_t) per
//             block and term (mma.py:84-85), the CUDA-core add standing in for
//             an RN terminal the tensor core does not have
enum Schedule : int { kSchC3 = 0, kSchC3DD = 1, kSchPlain = 2, kSchIn4 = 3, kSchIn4RN = 4 };

template <int V, int S = kSchC3>
struct PsCfg {
  static constexpr int BM = 128;                         // rows per CTA (pair M = 256)
  static constexpr int BN = S == kSchC3DD || S == kSchIn4RN ? 128 : 256;  // 3-4 accumulators: N <= 128
  static constexpr int BN_CTA = BN / 2;                  // B rows (= C columns) loaded per CTA
  static constexpr int A_TILE = 128 * 128;               // 128 rows x 128-byte k chunk
  static constexpr int B_TILE = BN_CTA * 128;
  static constexpr bool kLo = S != kSchPlain;            // lo operands used
  static constexpr int OP_BYTES = (kLo ? 2 : 1) * (A_TILE + B_TILE);  // A_hi [A_lo] B_hi [B_lo]
  static constexpr int OFF_AHI = 0;
  static constexpr int OFF_ALO = A_TILE;
  static constexpr int OFF_BHI = kLo ? 2 * A_TILE : A_TILE;
  static constexpr int OFF_BLO = OFF_BHI + B_TILE;
  static constexpr int NOP = (192 * 1024) / OP_BYTES;    // 3 / 4 / 6 stages
  static constexpr int OFF_OP = 0;
  static constexpr int OFF_BAR = NOP * OP_BYTES;
  static constexpr int NUM_PE = S == kSchIn4RN ? 4 : 1;  // p_empty barriers (one per drained P)
  static constexpr int NUM_BARS = 2 * NOP + 1 + NUM_PE;
  static constexpr int SMEM_BYTES = OFF_BAR + NUM_BARS * 8 + 16;
  static constexpr bool kDrain = S == kSchC3 || S == kSchC3DD;
  static constexpr int NUM_ACC = S == kSchC3 ? 2 : (S == kSchC3DD ? 3 : (S == kSchIn4RN ? 4 : 1));
  static constexpr int TMEM_COLS = NUM_ACC * BN > 256 ? 512 : 256;  // P | dC | ddC
  static constexpr int NUM_THREADS = 384;                // warps 0-3 control, 4-11 drain
  static constexpr int DRAIN_WARP0 = 4, NUM_DRAIN_WARPS = 8;
  static constexpr int DRAIN_COLS = BN / 2;
  static constexpr int EPI_WARP_BYTES = 32 * DRAIN_COLS * 4;
  static_assert(NUM_ACC * BN <= 512, "TMEM budget");
  static_assert(OP_BYTES % 1024 == 0, "stage alignment");
  static_assert(NUM_DRAIN_WARPS * EPI_WARP_BYTES <= OFF_BAR, "epilogue staging reuses the ring");
};

// TMA load that completes on the leader CTA's mbarrier (CTA-pair form).
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* m,
                                                 uint32_t leader_bar, int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(leader_bar), "r"(c0), "r"(c1)
      : "memory");
}

template <int V, int S>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PsCfg<V, S>::NUM_THREADS, 1)
    tcec_gemm_ps_kernel(const __grid_constant__ CUtensorMap tmAh,  // A_hi [m][k] box 128B x 128
                        const __grid_constant__ CUtensorMap tmAl,  // A_lo
                        const __grid_constant__ CUtensorMap tmBh,  // B_hi^T [n][k] box 128B x 128
                        const __grid_constant__ CUtensorMap tmBl,  // B_lo^T
                        float* __restrict__ Cout, const int64_t ldc, const GemmShape shp,
                        const float inv_scale, const float inv_scale2, uint32_t* __restrict__ flags,
                        uint32_t* __restrict__ wave_ctr) {
  // Persistent: one CTA pair per TPC walks the tile sequence (grouped raster),
  // ring / drain counters running across tiles; `acc_empty` orders each tile's
  // epilogue reads of the accumulators before the next tile's first MMA into
  // them; with `wave_ctr` the TMA producers meet once per wave (bounded wait)
  // so each wave's tiles share L2-resident k-slices (as tcec_gemm5.cuh).
  using C = PsCfg<V, S>;
  using VC = VarCfg<V>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* op_full = bars;                 // TMA (both CTAs) -> MMA   (leader, tx)
  uint64_t* op_empty = bars + C::NOP;       // MMA commit -> TMA        (both, multicast)
  uint64_t* p_full = bars + 2 * C::NOP;     // MMA commit -> drain      (both, multicast)
  uint64_t* p_empty = p_full + 1;           // drain -> MMA             (leader, 16; one per P)
  uint64_t* acc_empty = bars + C::NUM_BARS; // epilogue -> next tile's MMA (leader, 16)
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
  const int de = shp.drain_every;
  // drain intervals per tile: blocks of `de` MMA k-steps (4 per op stage) for
  // corrected3 and kSchIn4RN, else one (the epilogue)
  const int nintervals = C::kDrain || S == kSchIn4RN ? (4 * nop + de - 1) / de : 1;

  if (warp == 0 && lane == 0) {
    if (smem_base & 1023u) __trap();
    sm100::tma_prefetch_desc(&tmAh);
    sm100::tma_prefetch_desc(&tmAl);
    sm100::tma_prefetch_desc(&tmBh);
    sm100::tma_prefetch_desc(&tmBl);
    for (int o = 0; o < C::NOP; ++o) {
      sm100::mbar_init(&op_full[o], 1);
      sm100::mbar_init(&op_empty[o], 1);
    }
    sm100::mbar_init(p_full, 1);
    for (int t = 0; t < C::NUM_PE; ++t) sm100::mbar_init(&p_empty[t], 2 * C::NUM_DRAIN_WARPS);
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
  const uint32_t tmem_ddC = tmem_base + 2 * C::BN;

  if (warp < C::DRAIN_WARP0) {
    if (warp == 0 && lane == 0) {
      // ===================== TMA producer (both CTAs) =====================
      const uint32_t leader_full = sm100::mapa_shared(sm100::smem_u32(op_full), 0);
      uint32_t g = 0, target = 0;
      int wave = 0;
      for (int tile = pid; tile < num_tiles; tile += npairs, ++wave) {
        if (wave_ctr != nullptr && wave > 0) {  // lock-step waves, bounded wait
          target += 2u * static_cast<uint32_t>(min(npairs, num_tiles - wave * npairs));
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
        for (int kb = 0; kb < nop; ++kb, ++g) {
          const int o = g % C::NOP;
          sm100::mbar_wait(&op_empty[o], ((g / C::NOP) & 1) ^ 1);
          if (rank == 0) sm100::mbar_arrive_expect_tx(&op_full[o], 2 * C::OP_BYTES);
          const uint32_t dst = smem_base + C::OFF_OP + o * C::OP_BYTES;
          const uint32_t bar = leader_full + o * 8;
          const int kc = kb * VC::BK_OP;
          tma_load_2d_pair(dst + C::OFF_AHI, &tmAh, bar, kc, m_cta);
          tma_load_2d_pair(dst + C::OFF_BHI, &tmBh, bar, kc, n_cta);
          if constexpr (C::kLo) {
            tma_load_2d_pair(dst + C::OFF_ALO, &tmAl, bar, kc, m_cta);
            tma_load_2d_pair(dst + C::OFF_BLO, &tmBl, bar, kc, n_cta);
          }
        }
      }
    } else if (warp == 1 && rank == 0) {  // the whole warp runs the issue loop; one elected lane issues
      // ===================== MMA issuer (leader CTA) =====================
      constexpr uint32_t idesc = sm100::umma_idesc(VC::AB_FORMAT, 2 * C::BM, C::BN);
      constexpr uint32_t hi_w = (1024u >> 4) | (1u << 14) | (2u << 29);  // SBO 1024, v1, SW128
      uint32_t g = 0, git = 0, gtile = 0;
      int pos = 0;  // k-steps into the current drain interval (corrected3)
      for (int tile = pid; tile < num_tiles; tile += npairs, ++gtile) {
        for (int kb = 0; kb < nop; ++kb, ++g) {
          const int o = g % C::NOP;
          sm100::mbar_wait(&op_full[o], (g / C::NOP) & 1);
          sm100::tc_fence_after();
          // the previous tile's epilogue has read the accumulators (kSchIn4RN: its
          // epilogue reads registers only, the P buffers are guarded per block)
          if (S != kSchIn4RN && kb == 0 && gtile > 0) {
            sm100::mbar_wait_cluster(acc_empty, (gtile - 1) & 1);
            sm100::tc_fence_after();
          }
          const uint32_t op = sm100::opaque(smem_base + C::OFF_OP + o * C::OP_BYTES) >> 4;
          const uint32_t ahi = op | (1u << 16);
          const uint32_t alo = ahi + (C::OFF_ALO >> 4);
          const uint32_t bhi = ahi + (C::OFF_BHI >> 4);
          const uint32_t blo = ahi + (C::OFF_BLO >> 4);
          if constexpr (S == kSchPlain) {
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
              sm100::mma_pair_split_el<V == kTF32>(tmem_P, ahi + 2 * ks, hi_w, bhi + 2 * ks, hi_w, idesc,
                                                (kb | ks) != 0);
          } else if constexpr (S == kSchIn4RN) {
            // per MMA k-step, the four terms in the reference's order, each into
            // its own accumulator; a block's first k-step waits for the drain of
            // that accumulator's previous block and starts it from zero
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
              const int kk = kb * 4 + ks;
              const bool first = (kk % de) == 0;
#pragma unroll
              for (int t = 0; t < 4; ++t) {
                if (first && git > 0) {
                  sm100::mbar_wait_cluster(&p_empty[t], (git - 1) & 1);
                  sm100::tc_fence_after();
                }
                sm100::mma_pair_split_el<V == kTF32>(tmem_P + t * C::BN, (t < 2 ? alo : ahi) + 2 * ks,
                                                  hi_w, ((t & 1) ? bhi : blo) + 2 * ks, hi_w, idesc,
                                                  !first);
              }
              if ((kk % de) == de - 1 || (kb == nop - 1 && ks == 3)) {
                sm100::mma_commit_pair_mc_el(p_full, 0x3);
                ++git;
              }
            }
          } else if constexpr (S == kSchIn4) {
            // the reference's four-call order per block: dA*dB, dA*B, A*dB, A*B
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
              sm100::mma_pair_split_el<V == kTF32>(tmem_P, alo + 2 * ks, hi_w, blo + 2 * ks, hi_w, idesc,
                                                (kb | ks) != 0);
              sm100::mma_pair_split_el<V == kTF32>(tmem_P, alo + 2 * ks, hi_w, bhi + 2 * ks, hi_w, idesc, 1u);
              sm100::mma_pair_split_el<V == kTF32>(tmem_P, ahi + 2 * ks, hi_w, blo + 2 * ks, hi_w, idesc, 1u);
              sm100::mma_pair_split_el<V == kTF32>(tmem_P, ahi + 2 * ks, hi_w, bhi + 2 * ks, hi_w, idesc, 1u);
            }
          } else {
            c3_stage(
                kb * 4, 4 * nop, de, pos, git, p_empty, p_full, &op_empty[o],
                [&](int ks) {  // reference order per k-step: dA*B then A*dB (schemes.py:294-298)
                  sm100::mma_pair_split_el<V == kTF32>(tmem_dC, alo + 2 * ks, hi_w, bhi + 2 * ks, hi_w,
                                                    idesc, (kb | ks) != 0);
                  sm100::mma_pair_split_el<V == kTF32>(tmem_dC, ahi + 2 * ks, hi_w, blo + 2 * ks, hi_w,
                                                    idesc, 1u);
                  if constexpr (S == kSchC3DD)  // schemes.py:308-313: the dA*dB chain
                    sm100::mma_pair_split_el<V == kTF32>(tmem_ddC, alo + 2 * ks, hi_w, blo + 2 * ks,
                                                      hi_w, idesc, (kb | ks) != 0);
                },
                [&](int ks, uint32_t acc) {
                  sm100::mma_pair_split_el<V == kTF32>(tmem_P, ahi + 2 * ks, hi_w, bhi + 2 * ks, hi_w,
                                                    idesc, acc);
                });
          }
          if constexpr (!C::kDrain)  // (c3_stage commits op_empty itself)
            sm100::mma_commit_pair_mc_el(&op_empty[o], 0x3);
          if ((S == kSchPlain || S == kSchIn4) && kb == nop - 1) {
            sm100::mma_commit_pair_mc_el(p_full, 0x3);
            ++git;
          }
        }
      }
    }
  } else {
    // ===================== drain + epilogue =====================
    const int q = warp & 3;
    const int h = (warp - C::DRAIN_WARP0) >> 2;
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    const uint32_t p_empty_leader = sm100::mapa_shared(sm100::smem_u32(p_empty), 0);
    const uint32_t acc_empty_leader = sm100::mapa_shared(sm100::smem_u32(acc_empty), 0);
    constexpr int NC = C::DRAIN_COLS;
    bool nonfinite = false;
    uint32_t git = 0;
    for (int tile = pid; tile < num_tiles; tile += npairs) {
      int tm, tn;
      grouped_tile(tile, tiles_m, tiles_n, shp.group_m, tm, tn);
      float acc[NC];
#pragma unroll
      for (int j = 0; j < NC; ++j) acc[j] = 0.0f;
      for (int it = 0; it < nintervals; ++it, ++git) {
        sm100::mbar_wait(p_full, git & 1);
        sm100::tc_fence_after();
        if constexpr (C::kDrain) {
#pragma unroll
          for (int c = 0; c < NC / 8; ++c) {
            uint32_t r[8];
            sm100::tmem_ld_32x32b_x8(tmem_P + lane_off + h * NC + c * 8, r);
            sm100::tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 8; j += 2)  // schemes.py:300-304: c = RN32(c + partial), f32x2
              sm100::fadd2_rn(acc[c * 8 + j], acc[c * 8 + j + 1], __uint_as_float(r[j]),
                              __uint_as_float(r[j + 1]));
          }
          sm100::tc_fence_before();
          __syncwarp();
          if (lane == 0) sm100::mbar_arrive_remote(p_empty_leader);
        } else if constexpr (S == kSchIn4RN) {
          // mma.py:84-85 with an RN terminal, per term in order: c = RN32(c + P_t);
          // each accumulator is released as soon as it has been read
#pragma unroll
          for (int t = 0; t < 4; ++t) {
#pragma unroll
            for (int c = 0; c < NC / 8; ++c) {
              uint32_t r[8];
              sm100::tmem_ld_32x32b_x8(tmem_P + t * C::BN + lane_off + h * NC + c * 8, r);
              sm100::tmem_ld_wait();
#pragma unroll
              for (int j = 0; j < 8; j += 2)
                sm100::fadd2_rn(acc[c * 8 + j], acc[c * 8 + j + 1], __uint_as_float(r[j]),
                                __uint_as_float(r[j + 1]));
            }
            sm100::tc_fence_before();
            __syncwarp();
            if (lane == 0) sm100::mbar_arrive_remote(p_empty_leader + t * 8);
          }
        }
      }
      // epilogue: every MMA of the tile has completed (its last p_full follows them)
      const int64_t row = static_cast<int64_t>(tm) * 2 * C::BM + rank * C::BM + q * 32 + lane;
      const int col0 = tn * C::BN + h * NC;
      float* crow = Cout + row * ldc + col0;
#pragma unroll
      for (int c = 0; c < NC / 8; ++c) {
        uint32_t r[8];
        if constexpr (S != kSchIn4RN) {
          sm100::tmem_ld_32x32b_x8((C::kDrain ? tmem_dC : tmem_P) + lane_off + h * NC + c * 8, r);
          sm100::tmem_ld_wait();
        }
        uint32_t rr[8];
        if constexpr (S == kSchC3DD) {
          sm100::tmem_ld_32x32b_x8(tmem_ddC + lane_off + h * NC + c * 8, rr);
          sm100::tmem_ld_wait();
        }
        float o[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if constexpr (C::kDrain) {
            // schemes.py:306-307: one rounding of c + dC * 2^-s
            o[j] = __fmaf_rn(__uint_as_float(r[j]), inv_scale, acc[c * 8 + j]);
            if constexpr (S == kSchC3DD)  // schemes.py:312-313: then + ddC * 2^-2s
              o[j] = __fmaf_rn(__uint_as_float(rr[j]), inv_scale2, o[j]);
          } else if constexpr (S == kSchIn4RN) {
            o[j] = acc[c * 8 + j];
          } else {
            o[j] = __uint_as_float(r[j]);
          }
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
