// tcec_gemm4.cuh -- CTA-pair fused error-corrected SGEMM with the A operand
// split straight into tensor memory (tcgen05.mma A-from-TMEM, "TS" form).
//
// Same algorithm and per-element arithmetic as tcec_gemm2.cuh (the
// reference's corrected3 path, schemes.py:265-314); what changes is where the
// split A operand lives.  The pair kernel with both operands in shared memory
// is bound by shared-memory traffic (per 64-k FP16 stage and SM,
// 64 KB TMA writes + 64 KB staging reads + 64 KB hi/lo stores + 96 KB
// tensor-core operand reads against 128 B/clk).  Here the split warps write
// A_hi / A_lo with tcgen05.st into a TMEM ring and the MMAs read A from TMEM,
// which removes the A operand stores and the A operand reads from shared
// memory.  TMEM then holds P | dC | A-ring, so the pair tile narrows to
// 256 x 192 (N = 192: P 192 + dC 192 + 2 x 64 A columns = 512).
//
// Warp roles (640 threads, one CTA per SM, cluster of 2 on one TPC):
//   warp 0        TMA producer: FP32 A [128 x 32] + B 3 x [32 x 32] k-slices
//   warp 1        MMA issuer (leader CTA only): tcgen05.mma.cta_group::2 [d], [a_tmem], b_desc
//   warp 2        TMEM allocator (512 columns: P | dC | A ring)
//   warps 4-11    split: A rows (warp % 4 = TMEM lane quarter) -> tcgen05.st;
//                 B columns -> MN-major shared memory (FP16 SW64, TF32 SW128_BASE32B)
//   warps 12-19   drain: C = RN32(C + P) per drain interval (C in registers),
//                 epilogue C = RN32(C + dC * 2^-s) -> TMA store
#pragma once

#include "tcec_gemm2.cuh"

namespace tcec {

template <int V, int BN_ = 192, int NOP_ = 2>
struct TsCfg {
  static constexpr int BM = 128;           // rows per CTA (pair M = 256)
  static constexpr int BN = BN_;           // pair N = MMA N (192, or 128 with a deeper ring)
  static constexpr int BN_CTA = BN / 2;    // B columns staged / split per CTA
  static constexpr int BK_STG = 32;        // FP32 k per staging slice
  static constexpr int NOP = NOP_;         // operand ring (B in smem, A in TMEM)
  static constexpr int STG_A_BYTES = BM * BK_STG * 4;      // 16 KB, SW128 rows of 32 k
  static constexpr int STG_B_BOX = BK_STG * 32 * 4;        // 4 KB box: 32 k x 32 n, SW128
  static constexpr int NUM_B_BOXES = BN_CTA / 32;          // 3
  static constexpr int STG_B_BYTES = NUM_B_BOXES * STG_B_BOX;
  static constexpr int STG_BYTES = STG_A_BYTES + STG_B_BYTES;  // 28 KB
  static constexpr int ESIZE = V == kFP16 ? 2 : 4;
  static constexpr int OP_B_BYTES = BN_CTA * VarCfg<V>::BK_OP * ESIZE;  // 12 KB
  static constexpr int OP_BYTES = 2 * OP_B_BYTES;                      // B_hi | B_lo
  // FP32 staging ring: as deep as shared memory allows, up to 8 slices.  These
  // tiles' MMAs are short, so the TMA latency (~0.9 us under load, measured by
  // a per-stage timeline of the 256 x 64 kernel) must be covered by slices in
  // flight rather than by MMA time.
  static constexpr int NSTG_FIT = (225 * 1024 - NOP * OP_BYTES) / STG_BYTES;
  static constexpr int NSTG = NSTG_FIT < 8 ? NSTG_FIT : 8;
  // MN-major B atoms: 32 n per row (FP16 SWIZZLE_64B: 64-byte rows, 8 k rows;
  // TF32 SWIZZLE_128B_BASE32B: 128-byte rows, 4 k rows); atoms along n (LBO),
  // then k-groups (SBO).
  static constexpr int B_ATOM_N = 32;
  static constexpr int B_ROW_BYTES = 32 * ESIZE;
  static constexpr int B_ROWS = V == kFP16 ? 8 : 4;
  static constexpr int B_LBO = B_ROWS * B_ROW_BYTES;                  // 512
  static constexpr int B_SBO = (BN_CTA / B_ATOM_N) * B_LBO;           // 1536
  static constexpr uint32_t B_LAYOUT = V == kFP16 ? 4u : 1u;          // SW64 / SW128_BASE32B
  static constexpr int MMA_K = V == kFP16 ? 16 : 8;
  static constexpr int B_KSTEP_BYTES = MMA_K / B_ROWS * B_SBO;        // 3072
  static constexpr int OFF_STG = 0;
  static constexpr int OFF_OP = NSTG * STG_BYTES;
  static constexpr int OFF_BAR = OFF_OP + NOP * OP_BYTES;
  // TMEM columns: P [0,BN) | dC [BN,2BN) | A ring [2BN, 2BN + 64 NOP): stage o
  // at 2BN + 64 o, A_hi in its first 32 columns and A_lo in the next 32 (8
  // columns per MMA k-step: 16 FP16 packed in pairs, or 8 TF32) | a second P
  // buffer where the 512 columns leave room (256 x 64 with NOP 4, 256 x 128
  // with NOP 2): the MMAs of drain interval j + 1 then start while the drain
  // warps still read interval j's partial, which removes the per-interval
  // drain round trip from the critical path of the narrow tiles (their MMAs
  // are too short to hide it).
  static constexpr int TMEM_COLS = 512;
  static constexpr int T_DC = BN;
  static constexpr int T_A = 2 * BN;
  static constexpr int T_A_STAGE = 64;
  static constexpr int T_P1 = T_A + NOP * T_A_STAGE;
  static constexpr int NPB = T_P1 + BN <= TMEM_COLS ? 2 : 1;  // P buffers
  static constexpr int NUM_BARS = 2 * NSTG + 2 * NOP + 2 * NPB;
  static constexpr int SMEM_BYTES = OFF_BAR + NUM_BARS * 8 + 16;
  static constexpr int NUM_THREADS = 640;
  static constexpr int SPLIT_WARP0 = 4, NUM_SPLIT_WARPS = 8;
  static constexpr int DRAIN_WARP0 = 12, NUM_DRAIN_WARPS = 8;
  static constexpr int DRAIN_COLS = BN / 2;                            // 96 per drain warp
  static constexpr int EPI_WARP_BYTES = 32 * DRAIN_COLS * 4;          // 32 rows x 96 cols
  static_assert(T_A + NOP * T_A_STAGE <= TMEM_COLS, "TMEM budget");
  static_assert(BN % 64 == 0, "B operand geometry");
  static_assert(STG_BYTES % 1024 == 0 && OP_BYTES % 1024 == 0 && OFF_OP % 1024 == 0, "alignment");
  static_assert(NUM_DRAIN_WARPS * EPI_WARP_BYTES <= OFF_BAR, "epilogue staging reuses the rings");
  static_assert(SMEM_BYTES <= 232448, "shared memory");
};

// One 32-deep staging slice -> this thread's part of the operand stage.
//   A: thread t -> row t & 127 (TMEM lane; warp % 4 is its lane quarter),
//      k in [16 (t >> 7), +16) of the slice -> TMEM columns (tcgen05.st).
//   B: thread t < 192 -> k row t & 31, n in [16 (t >> 5), +16) -> MN-major smem.
template <int V, int R, bool kFlags, int BN, int NOP>
__device__ __forceinline__ void ts_split_slice(uint32_t stg, uint32_t op, uint32_t ta, int sub,
                                               int t, float scale, FlagAcc& fa) {
  using C = TsCfg<V, BN, NOP>;
  // ---- A -> TMEM
  {
    const int row = t & 127, half = t >> 7;
    float x[16];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float4 v = sm100::lds128(stg + sw128(row, half * 4 + i));
      x[4 * i] = v.x; x[4 * i + 1] = v.y; x[4 * i + 2] = v.z; x[4 * i + 3] = v.w;
    }
    if constexpr (kFlags) {
#pragma unroll
      for (int i = 0; i < 16; ++i) fa.add(x[i]);
    }
    uint32_t hw[16], lw[16];
    split16<V, R>(x, scale, hw, lw);
    // lane quarter (row & ~31) in the address's lane field; columns of this k range
    const uint32_t lanes = static_cast<uint32_t>(row & ~31) << 16;
    if constexpr (V == kFP16) {
      const uint32_t col = sub * 16 + half * 8;
      sm100::tmem_st_32x32b_x8(ta + lanes + col, hw);
      sm100::tmem_st_32x32b_x8(ta + lanes + 32 + col, lw);
    } else {
      const uint32_t col = half * 16;
      sm100::tmem_st_32x32b_x16(ta + lanes + col, hw);
      sm100::tmem_st_32x32b_x16(ta + lanes + 32 + col, lw);
    }
  }
  // ---- B -> shared memory (MN-major), spread over all 256 split threads: per
  // 32-column box, each thread splits 4 consecutive n of one k row (so the
  // B work no longer doubles the split time of the first 2 x NUM_B_BOXES
  // warps -- the step that bounded the narrow tiles).  Lane layout per warp:
  // 16 k rows x 8 n, chosen so that the 16-byte LDS phases and the STS phases
  // (FP16: 64-bit stores into SW64 rows; TF32: 128-bit stores into
  // SW128_BASE32B rows) hit distinct banks.
  {
    const int w = t >> 5, l = t & 31;
    const uint32_t hi_base = op, lo_base = op + C::OP_B_BYTES;
#pragma unroll
    for (int bx = 0; bx < C::NUM_B_BOXES; ++bx) {
      int row, c16;  // k within the slice; 16-byte (4 n) chunk within the box
      if constexpr (V == kFP16) {
        row = (w & 1) * 16 + (l >> 4) * 8 + (l & 7);
        c16 = (w >> 1) * 2 + ((l >> 3) & 1);
      } else {
        row = (w & 1) * 16 + (l >> 3) * 4 + (l & 3);
        c16 = (w >> 1) * 2 + ((l >> 2) & 1);
      }
      const uint32_t box = stg + C::STG_A_BYTES + bx * C::STG_B_BOX;
      const float4 v = sm100::lds128(box + sw128(row, c16));
      float x[4] = {v.x, v.y, v.z, v.w};
      if constexpr (kFlags) {
#pragma unroll
        for (int i = 0; i < 4; ++i) fa.add(x[i]);
      }
      const int kop = sub * 32 + row;  // k within the operand stage
      const int grp = kop / C::B_ROWS, rr = kop % C::B_ROWS;
      const uint32_t base = grp * C::B_SBO + bx * C::B_LBO + rr * C::B_ROW_BYTES;
      if constexpr (V == kFP16) {
        uint32_t hw[2], lw[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) split_pair16<R>(x[2 * j], x[2 * j + 1], scale, hw[j], lw[j]);
        // SW64 (Swizzle<2,4,3>): 16-byte chunk (8 n) ^ ((row >> 1) & 3); 4 n = half a chunk
        const int c8 = c16 >> 1;
        const uint32_t off = base + (((c8 ^ (rr >> 1)) & 3) << 4) + ((c16 & 1) << 3);
        sm100::sts64(hi_base + off, hw[0], hw[1]);
        sm100::sts64(lo_base + off, lw[0], lw[1]);
      } else {
        uint32_t hw[4], lw[4];
        split_chunk<V, R>(x, scale, hw, lw);
        // SW128_BASE32B (Swizzle<2,5,2>): 32-byte chunk ^ (row & 3)
        const uint32_t off = base + ((((c16 >> 1) ^ rr) & 3) << 5) + ((c16 & 1) << 4);
        sm100::sts128(hi_base + off, hw[0], hw[1], hw[2], hw[3]);
        sm100::sts128(lo_base + off, lw[0], lw[1], lw[2], lw[3]);
      }
    }
  }
}

template <int V, int R, bool kFlags, int BN, int NOP>
__device__ __forceinline__ void ts_split_loop(uint32_t smem, uint32_t tmem_base, uint64_t* stg_full,
                                              uint64_t* stg_empty, uint64_t* op_full,
                                              uint64_t* op_empty, int nop, int t, int lane,
                                              float scale, FlagAcc& fa) {
  using C = TsCfg<V, BN, NOP>;
  using VC = VarCfg<V>;
  const uint32_t leader_op_full = sm100::mapa_shared(sm100::smem_u32(op_full), 0);
  for (int kb = 0; kb < nop; ++kb) {
    const int o = kb % C::NOP;
    const uint32_t op = smem + C::OFF_OP + o * C::OP_BYTES;
    const uint32_t ta = tmem_base + C::T_A + o * C::T_A_STAGE;
#pragma unroll
    for (int sub = 0; sub < VC::STG_PER_OP; ++sub) {
      const int st = kb * VC::STG_PER_OP + sub;
      const int s = st % C::NSTG;
      sm100::mbar_wait(&stg_full[s], (st / C::NSTG) & 1);
      if (sub == 0) {
        sm100::mbar_wait(&op_empty[o], ((kb / C::NOP) & 1) ^ 1);
        sm100::tc_fence_after();  // the MMAs that read this TMEM stage have completed
      }
      const uint32_t stg = smem + C::OFF_STG + s * C::STG_BYTES;
      ts_split_slice<V, R, kFlags, BN, NOP>(stg, op, ta, sub, t, scale, fa);
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&stg_empty[s]);
    }
    // TMEM stores complete + generic smem stores -> async proxy, then signal the leader
    sm100::tmem_st_wait();
    sm100::fence_proxy_async_smem();
    sm100::tc_fence_before();
    __syncwarp();
    if (lane == 0) sm100::mbar_arrive_remote(leader_op_full + o * 8);
  }
}

template <int V, int R, int BN, int NOP>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(640, 1)
    tcec_gemm_ts_kernel(const __grid_constant__ CUtensorMap tmA,  // A [m][k], box 32 x 128, SW128
                        const __grid_constant__ CUtensorMap tmB,  // B [k][n], box 32 x 32, SW128
                        const __grid_constant__ CUtensorMap tmC,  // C [m][n], box 32 x 32, SW128
                        const GemmShape shp, const float scale, const float inv_scale,
                        const FlagThresholds thr, uint32_t* __restrict__ flags) {
  using C = TsCfg<V, BN, NOP>;
  using VC = VarCfg<V>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* stg_full = bars;                    // TMA -> split          (local)
  uint64_t* stg_empty = bars + C::NSTG;         // split -> TMA          (local, 8)
  uint64_t* op_full = bars + 2 * C::NSTG;       // split -> MMA          (leader, 16)
  uint64_t* op_empty = op_full + C::NOP;        // MMA commit -> split   (both, multicast)
  uint64_t* p_full = op_empty + C::NOP;         // [NPB] MMA commit -> drain (both, multicast)
  uint64_t* p_empty = p_full + C::NPB;          // [NPB] drain -> MMA        (leader, 16)
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
  const int m_cta = tile_m * 2 * C::BM + rank * C::BM;
  const int n_pair = tile_n * C::BN;
  const int n_cta = n_pair + rank * C::BN_CTA;
  const int nop = shp.num_op_stages;
  const int nstg = nop * VC::STG_PER_OP;
  const int de = shp.drain_every / 4;  // operand stages per drain interval (host: a multiple of 4 k-steps)
  const int nintervals = (nop + de - 1) / de;

  if (warp == 0 && lane == 0) {
    if (smem_base & 1023u) __trap();
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
    for (int b = 0; b < C::NPB; ++b) {
      sm100::mbar_init(&p_full[b], 1);
      sm100::mbar_init(&p_empty[b], 2 * C::NUM_DRAIN_WARPS);
    }
    sm100::fence_mbar_init();
  }
  if (warp == 2) sm100::tmem_alloc_pair<C::TMEM_COLS>(tmem_slot);
  sm100::tc_fence_before();
  sm100::cluster_sync();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t tmem_P = tmem_base;
  const uint32_t tmem_dC = tmem_base + C::T_DC;
  // P buffer of drain interval j: j % NPB
  auto p_buf = [&](int j) { return (C::NPB == 2 && (j & 1)) ? tmem_base + C::T_P1 : tmem_P; };

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
        for (int b = 0; b < C::NUM_B_BOXES; ++b)
          sm100::tma_load_2d(dst + C::STG_A_BYTES + b * C::STG_B_BOX, &tmB, &stg_full[s],
                             n_cta + 32 * b, st * C::BK_STG);
      }
    } else if (warp == 1 && rank == 0) {
      // ===================== MMA issuer (leader CTA; the whole warp runs the loop,
      // one elected lane issues) =====================
      constexpr uint32_t idesc = sm100::umma_idesc_bmn(VC::AB_FORMAT, 2 * C::BM, C::BN);
      constexpr uint32_t b_hi_w = (uint32_t(C::B_SBO) >> 4) | (1u << 14) | (C::B_LAYOUT << 29);
      constexpr uint32_t b_lbo_w = (uint32_t(C::B_LBO) >> 4) << 16;
      constexpr uint32_t kB = C::B_KSTEP_BYTES >> 4;
      for (int kb = 0; kb < nop; ++kb) {
        const int o = kb % C::NOP;
        sm100::mbar_wait_cluster(&op_full[o], (kb / C::NOP) & 1);
        sm100::tc_fence_after();
        const uint32_t op = sm100::opaque(smem_base + C::OFF_OP + o * C::OP_BYTES) >> 4;
        const uint32_t bhi = op | b_lbo_w;
        const uint32_t blo = bhi + (C::OP_B_BYTES >> 4);
        const uint32_t ahi = sm100::opaque(tmem_base + C::T_A + o * C::T_A_STAGE);
        const uint32_t alo = ahi + 32;
        // corrections first (reference order per k-step: dA*B then A*dB), so the
        // drain of the previous P overlaps them (schemes.py:294-298)
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          sm100::mma_pair_ts_el<V == kTF32>(tmem_dC, alo + 8 * ks, bhi + kB * ks, b_hi_w, idesc,
                                         (kb | ks) != 0);
          sm100::mma_pair_ts_el<V == kTF32>(tmem_dC, ahi + 8 * ks, blo + kB * ks, b_hi_w, idesc, 1u);
        }
        const bool first_in_interval = (kb % de) == 0;
        const int j = kb / de;  // drain interval
        const int b = j % C::NPB;
        if (first_in_interval && j >= C::NPB) {  // the drain of interval j - NPB has read buffer b
          sm100::mbar_wait_cluster(&p_empty[b], ((j / C::NPB) - 1) & 1);
          sm100::tc_fence_after();
        }
        const uint32_t tP = p_buf(j);
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          sm100::mma_pair_ts_el<V == kTF32>(tP, ahi + 8 * ks, bhi + kB * ks, b_hi_w, idesc,
                                         !(first_in_interval && ks == 0));
        }
        sm100::mma_commit_pair_mc_el(&op_empty[o], 0x3);
        if ((kb % de) == de - 1 || kb == nop - 1) sm100::mma_commit_pair_mc_el(&p_full[b], 0x3);
      }
    }
  } else if (warp < C::DRAIN_WARP0) {
    sm100::regs_dec<56>();
    // ===================== split warps =====================
    const int t = threadIdx.x - C::SPLIT_WARP0 * 32;
    FlagAcc fa;
    const bool do_flags = flags != nullptr && (tile_n == 0 || tile_m == 0);
    if (do_flags) {
      ts_split_loop<V, R, true, BN, NOP>(smem_base, tmem_base, stg_full, stg_empty, op_full, op_empty, nop, t,
                                lane, scale, fa);
      flag_publish(fa, thr, flags);
    } else {
      ts_split_loop<V, R, false, BN, NOP>(smem_base, tmem_base, stg_full, stg_empty, op_full, op_empty, nop, t,
                                 lane, scale, fa);
    }
    // the epilogue reuses the staging ring (see the drain warps' barrier)
    sm100::named_barrier_sync<1, 32 * (C::NUM_SPLIT_WARPS + C::NUM_DRAIN_WARPS)>();
  } else {
    sm100::regs_inc<160>();
    // ===================== drain + epilogue =====================
    const int q = warp & 3;
    const int h = (warp - C::DRAIN_WARP0) >> 2;
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    const uint32_t p_empty_leader = sm100::mapa_shared(sm100::smem_u32(p_empty), 0);
    constexpr int NC = C::DRAIN_COLS;
    float acc[NC];
#pragma unroll
    for (int j = 0; j < NC; ++j) acc[j] = 0.0f;
    for (int it = 0; it < nintervals; ++it) {
      const int b = it % C::NPB;
      sm100::mbar_wait(&p_full[b], (it / C::NPB) & 1);
      sm100::tc_fence_after();
      const uint32_t tP = p_buf(it);
#pragma unroll
      for (int c = 0; c < NC / 16; ++c) {
        uint32_t r[16];
        sm100::tmem_ld_32x32b_x16(tP + lane_off + h * NC + c * 16, r);
        sm100::tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 16; ++j)  // schemes.py:300-304: c = RN32(c + partial)
          acc[c * 16 + j] = __fadd_rn(acc[c * 16 + j], __uint_as_float(r[j]));
      }
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive_remote(p_empty_leader + b * 8);
    }
    bool nonfinite = false;
    // the split warps' staging reads precede the epilogue's staging writes
    sm100::named_barrier_sync<1, 32 * (C::NUM_SPLIT_WARPS + C::NUM_DRAIN_WARPS)>();
    const uint32_t stage = smem_base + (warp - C::DRAIN_WARP0) * C::EPI_WARP_BYTES;
#pragma unroll
    for (int b = 0; b < NC / 32; ++b) {
      const uint32_t box = stage + b * 4096;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t r[16];
        sm100::tmem_ld_32x32b_x16(tmem_dC + lane_off + h * NC + b * 32 + c * 16, r);
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
        sm100::tma_store_2d(&tmC, smem + (box - smem_base), n_pair + h * NC + b * 32, m_cta + q * 32);
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
