// tcec_ring.cuh -- fused error-corrected SGEMM with the split shared through an
// L2-resident ring (kernel_variant 6).
//
// The fused pair kernels (tcec_gemm2.cuh / tcec_gemm5.cuh) split every A tile
// once per column tile of C and every B tile once per row tile: n / 256 and
// m / 256 times (64x at 16384^3).  For FP16 that redundant split -- FP32
// staging through shared memory, the split arithmetic and the hi / lo stores,
// 192 KB of shared-memory traffic per 64-k stage next to the tensor core's own
// 96 KB -- is what holds the kernel below the split-once mode.
//
// Here the persistent CTA pairs walk the tile sequence in waves of `np`
// consecutive tiles (one per pair, grouped raster), and every k-slice of the
// A row-panels and B column-panels a wave reads is split exactly once, by the
// whole grid, into a ring of D slots in global memory that stays in L2:
//
//   split warps (8 per CTA)  units of 16 rows (A) or 16 columns (B) x one
//                            operand stage of k: FP32 loads straight from
//                            A / B into registers, splitting.py:114-122 split
//                            (split_chunk, the fused kernels' arithmetic), hi
//                            and lo stored K-major (B transposed) into ring slot
//                            g mod D as whole 128-byte lines; a release-add on
//                            the panel's ready counter
//   ready watcher (warp 3)   polls this pair's two ready counters per slice and
//                            publishes "slices split" in shared memory
//   TMA producer (warp 0)    waits for that, then loads the four 16 KB hi / lo
//                            tiles of the slice into the operand ring exactly
//                            as the split-once kernel does (tcec_presplit.cuh)
//   MMA issuer, drain        the split-once kernel's corrected3 pipeline; the
//                            non-leader's first drain warp notes which stages
//                            the completed drain intervals cover
//   release (rank 1 warp 1)  adds 1 to freed[g] for each such slice
//   freed watcher (warp 2)   polls freed[] and publishes "slots reusable" in
//                            shared memory for this CTA's split warps
//
// A split warp writing slice g waits until every pair of slice g - D's wave
// has released it (D = 16).  The split never goes to HBM on purpose: a slot
// is rewritten every D slices while it is L2-resident, the FP32 inputs are read
// once per wave (A panels ~7x, B panels 8x over the whole product at 16384^3,
// against 64x each in the fused kernels).  C is bit-identical to the fused and
// split-once kernels (same split, same MMA order, same drain).
//
// Measured (profiles/r02/ring.md): FP16 392 vs 383 TF/s fused at 16384^3 but
// 410 vs 432 at 8192^3; TF32 243 vs 250 -- all below the split-once mode (439
// FP16).  The board is at its power limit either way (ncu: 1.39 GHz, tensor
// pipe 74%), and re-splitting each panel once per wave through L2 (writes plus
// TMA re-reads of the freshly written lines) costs about what the fused
// kernel's shared-memory staging does; one HBM pass (split-once) costs less.
// Hence an option (kernel_variant 6), not the default.
//
// Every CTA of the grid splits, so the grid is the co-resident pair count and
// all waits are bounded (a stall of more than a few seconds traps instead of
// hanging).
#pragma once

#include "tcec_presplit.cuh"

namespace tcec {

// A wave's panels: A row-panels [a_first, a_first + la) (whole raster groups),
// B column-panels b_first, b_first + 1, ... (lb of them, modulo tiles_n).
struct RingWave {
  int a_first, la, b_first, lb;
};

__host__ __device__ inline void ring_tile(int tile, int tiles_m, int tiles_n, int group_m,
                                          int& tm, int& tn) {
  const int per_group = group_m * tiles_n;
  const int g = tile / per_group;
  const int first_m = g * group_m;
  const int gsize = (tiles_m - first_m) < group_m ? (tiles_m - first_m) : group_m;
  const int in_g = tile - g * per_group;
  tm = first_m + in_g % gsize;
  tn = in_g / gsize;
}

__host__ __device__ inline int ring_tile_index(int tm, int tn, int tiles_m, int tiles_n,
                                               int group_m) {
  const int g = tm / group_m;
  const int first_m = g * group_m;
  const int gsize = (tiles_m - first_m) < group_m ? (tiles_m - first_m) : group_m;
  return g * group_m * tiles_n + tn * gsize + (tm - first_m);
}

__host__ __device__ inline RingWave ring_wave(int w, int np, int tiles, int tiles_m, int tiles_n,
                                              int group_m) {
  const int t0 = w * np;
  const int t1 = ((t0 + np) < tiles ? (t0 + np) : tiles) - 1;
  const int per_group = group_m * tiles_n;
  const int g0 = t0 / per_group, g1 = t1 / per_group;
  RingWave r;
  r.a_first = g0 * group_m;
  const int a_end = (g1 + 1) * group_m;
  r.la = (a_end < tiles_m ? a_end : tiles_m) - r.a_first;
  int tm0, tn0, tm1, tn1;
  ring_tile(t0, tiles_m, tiles_n, group_m, tm0, tn0);
  ring_tile(t1, tiles_m, tiles_n, group_m, tm1, tn1);
  if (g0 == g1) {
    r.b_first = tn0;
    r.lb = tn1 - tn0 + 1;
  } else if (g1 == g0 + 1 && tn1 + 1 < tn0) {
    r.b_first = tn0;  // the first group's last columns, then the next group's first
    r.lb = tiles_n - tn0 + tn1 + 1;
  } else {
    r.b_first = 0;
    r.lb = tiles_n;
  }
  return r;
}

struct RingArgs {
  const float* A;  // m x k, row pitch lda (FP32)
  const float* B;  // k x n, row pitch ldb
  int64_t lda, ldb;
  uint8_t* ahi;    // ring: D slots x la_max x 256 rows x 128 bytes (hi), same for lo
  uint8_t* alo;
  uint8_t* bhi;    // D slots x lb_max x 256 rows (= columns of B) x 128 bytes
  uint8_t* blo;
  uint32_t* ready;  // [slices][la_max + lb_max]: units (of 16) split per panel
  uint32_t* freed;  // [slices]: pairs that have consumed the slice
  int32_t depth;    // D
  int32_t la_max, lb_max;
  int32_t np;       // pairs (tiles per wave)
};

constexpr int kRingUnits = 16;  // units per panel (16 rows / columns each)

// shared memory: the split-once kernel's layout plus two watcher words
template <int V>
constexpr int ring_smem_bytes() {
  return PsCfg<V, kSchC3>::SMEM_BYTES + 32;
}

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
// Bounded wait for *p >= target with acquire semantics: relaxed polls (an
// acquire load invalidates L1 each time), one acquire load once it holds;
// ~4 s, then trap (a lost peer must not hang the GPU).
__device__ __forceinline__ void ring_wait_ge(const uint32_t* p, uint32_t target) {
  for (uint32_t spin = 0; ld_relaxed_u32(p) < target; ++spin) {
    __nanosleep(spin < 64 ? 32 : 256);
    if (spin > (1u << 24)) __trap();
  }
  (void)ld_acquire_u32(p);
}

// Plain stores and loads: L2 evict-last stores and evict-first / no-L1 loads
// were measured 6% slower (FP16 369 vs 392 TF/s at 16384^3).
__device__ __forceinline__ void stg128(void* p, const uint32_t (&w)[4]) {
  asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(w[0]), "r"(w[1]),
               "r"(w[2]), "r"(w[3])
               : "memory");
}

// One unit: 16 rows of A (kB = false) or 16 columns of B (kB = true) x the
// operand stage's k-range [k0, k0 + BK); its ring rows are 128 bytes (BK
// operand elements) each.  In pass j (0..3) lane l covers row / column
// 4 j + (l >> 3) and 16-byte operand chunk c = l & 7, i.e. EPC consecutive k,
// so every store instruction writes four whole 128-byte lines.  ring_load_unit
// reads the lane's 4 x EPC FP32 inputs (issued before the wait for the ring
// slot, so their latency overlaps it); ring_store_unit splits each chunk into
// one 16-byte hi and one 16-byte lo chunk.
template <int V>
struct RingUnit {
  static constexpr int EPC = V == kFP16 ? 8 : 4;  // inputs per 16-byte operand chunk
  static constexpr int NX = 4 * EPC;              // inputs per lane
};

template <int V, bool kB>
__device__ __forceinline__ void ring_load_unit(const RingArgs& ra, const GemmShape& shp, int lane,
                                               int k0, int panel, int sub,
                                               float (&x)[RingUnit<V>::NX]) {
  constexpr int EPC = RingUnit<V>::EPC;
  const int kc = k0 + (lane & 7) * EPC;  // first k of the lane's chunk
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int64_t rc = int64_t(panel) * 256 + sub * 16 + 4 * j + (lane >> 3);
    float* xj = x + j * EPC;
    if constexpr (!kB) {
      const float* src = ra.A + rc * ra.lda + kc;
      if (rc < shp.m && kc + EPC <= shp.k) {
#pragma unroll
        for (int i = 0; i < EPC / 4; ++i) {
          const float4 v = __ldg(reinterpret_cast<const float4*>(src) + i);
          xj[4 * i] = v.x; xj[4 * i + 1] = v.y; xj[4 * i + 2] = v.z; xj[4 * i + 3] = v.w;
        }
      } else {
#pragma unroll
        for (int i = 0; i < EPC; ++i) xj[i] = (rc < shp.m && kc + i < shp.k) ? __ldg(src + i) : 0.0f;
      }
    } else {
      const float* src = ra.B + int64_t(kc) * ra.ldb + rc;
      if (rc < shp.n && kc + EPC <= shp.k) {
#pragma unroll
        for (int i = 0; i < EPC; ++i) xj[i] = __ldg(src + int64_t(i) * ra.ldb);
      } else {
#pragma unroll
        for (int i = 0; i < EPC; ++i)
          xj[i] = (rc < shp.n && kc + i < shp.k) ? __ldg(src + int64_t(i) * ra.ldb) : 0.0f;
      }
    }
  }
}

template <int V, int R>
__device__ __forceinline__ void ring_store_unit(int lane, int idx, int sub, uint8_t* hi_row0,
                                                uint8_t* lo_row0, float scale, bool do_flags,
                                                FlagAcc& fa, float (&x)[RingUnit<V>::NX]) {
  constexpr int EPC = RingUnit<V>::EPC;
  if (do_flags) {
#pragma unroll
    for (int i = 0; i < RingUnit<V>::NX; ++i) fa.add(x[i]);
  }
  const int64_t row0 = int64_t(idx) * 256 + sub * 16 + (lane >> 3);
  const int cb = (lane & 7) * 16;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint32_t hw[4], lw[4];
    split_chunk<V, R>(x + j * EPC, scale, hw, lw);
    const int64_t off = (row0 + 4 * j) * 128 + cb;
    stg128(hi_row0 + off, hw);
    stg128(lo_row0 + off, lw);
  }
}

template <int V, int R>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(640, 1)
    tcec_gemm_ring_kernel(const __grid_constant__ CUtensorMap tmAh,  // ring A_hi, box 128 B x 128
                          const __grid_constant__ CUtensorMap tmAl,
                          const __grid_constant__ CUtensorMap tmBh,  // ring B_hi^T
                          const __grid_constant__ CUtensorMap tmBl,
                          float* __restrict__ Cout, const int64_t ldc, const GemmShape shp,
                          const RingArgs ra, const float scale, const float inv_scale,
                          const FlagThresholds thr, uint32_t* __restrict__ flags) {
  using C = PsCfg<V, kSchC3>;
  using VC = VarCfg<V>;
  constexpr int SPLIT_WARP0 = 12, NUM_SPLIT_WARPS = 8;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* op_full = bars;                 // TMA (both CTAs) -> MMA   (leader, tx)
  uint64_t* op_empty = bars + C::NOP;       // MMA commit -> TMA        (both, multicast)
  uint64_t* p_full = bars + 2 * C::NOP;     // MMA commit -> drain      (both, multicast)
  uint64_t* p_empty = p_full + 1;           // drain -> MMA             (leader, 16)
  uint64_t* acc_empty = bars + C::NUM_BARS; // epilogue -> next tile's MMA (leader, 16)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::NUM_BARS + 1);
  // slices [0, *freed_upto) are consumed by every pair of their wave (the
  // CTA's watcher thread publishes it; the split warps read it locally instead
  // of all polling the same global counter)
  uint32_t* freed_upto = tmem_slot + 1;
  uint32_t* ready_upto = tmem_slot + 2;  // this pair's slices [0, *ready_upto) are split
  uint32_t* consumed_upto = tmem_slot + 3;  // this pair's slices [0, ..) are consumed (rank 1)
  const uint32_t smem_base = sm100::smem_u32(smem);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = sm100::cluster_ctarank();
  const int tiles_m = (shp.m + 2 * C::BM - 1) / (2 * C::BM);
  const int tiles_n = (shp.n + C::BN - 1) / C::BN;
  const int num_tiles = tiles_m * tiles_n;
  const int np = ra.np;
  const int pid = blockIdx.x >> 1;
  const int nop = shp.num_op_stages;
  const int de = shp.drain_every;
  const int gm = shp.group_m;
  const int waves = (num_tiles + np - 1) / np;
  const int pmax = ra.la_max + ra.lb_max;
  const int nintervals = (4 * nop + de - 1) / de;

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
    sm100::mbar_init(p_empty, 2 * C::NUM_DRAIN_WARPS);
    sm100::mbar_init(acc_empty, 2 * C::NUM_DRAIN_WARPS);
    *freed_upto = 0u;
    *ready_upto = 0u;
    *consumed_upto = 0u;
    sm100::fence_mbar_init();
  }
  if (warp == 2) sm100::tmem_alloc_pair<C::TMEM_COLS>(tmem_slot);
  sm100::tc_fence_before();
  sm100::cluster_sync();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t tmem_P = tmem_base;
  const uint32_t tmem_dC = tmem_base + C::BN;

  if (warp < C::DRAIN_WARP0) {
    // setmaxnreg only redistributes the launch allocation (96 x 640 registers):
    // 4 x 40 + 8 x 160 + 8 x 56 = 1888 <= 20 x 96 per lane slot
    sm100::regs_dec<40>();
    if (warp == 0 && lane == 0) {
      // ===================== TMA producer (both CTAs) =====================
      const uint32_t leader_full = sm100::mapa_shared(sm100::smem_u32(op_full), 0);
      int g = 0;  // this pair's slices are g = w * nop + kb for its waves w = 0, 1, ...
      for (int w = 0; pid + w * np < num_tiles; ++w) {
        const RingWave rw = ring_wave(w, np, num_tiles, tiles_m, tiles_n, gm);
        int tm, tn;
        ring_tile(pid + w * np, tiles_m, tiles_n, gm, tm, tn);
        const int ia = tm - rw.a_first;
        const int ib = (tn - rw.b_first + tiles_n) % tiles_n;
        for (int kb = 0; kb < nop; ++kb, ++g) {
          const int o = g % C::NOP;
          sm100::mbar_wait(&op_empty[o], ((g / C::NOP) & 1) ^ 1);
          // the ready watcher has seen both panels of this slice split
          {
            for (uint32_t spin = 0;; ++spin) {
              uint32_t v;
              asm volatile("ld.acquire.cta.shared.u32 %0, [%1];"
                           : "=r"(v)
                           : "r"(sm100::smem_u32(ready_upto))
                           : "memory");
              if (v > static_cast<uint32_t>(g)) break;
              if (spin > (1u << 28)) __trap();
            }
          }
          fence_proxy_async_global();
          if (rank == 0) sm100::mbar_arrive_expect_tx(&op_full[o], 2 * C::OP_BYTES);
          const uint32_t dst = smem_base + C::OFF_OP + o * C::OP_BYTES;
          const uint32_t bar = leader_full + o * 8;
          const int s = g % ra.depth;
          const int row_a = (s * ra.la_max + ia) * 256 + rank * C::BM;
          const int row_b = (s * ra.lb_max + ib) * 256 + rank * C::BN_CTA;
          tma_load_2d_pair(dst + C::OFF_AHI, &tmAh, bar, 0, row_a);
          tma_load_2d_pair(dst + C::OFF_BHI, &tmBh, bar, 0, row_b);
          tma_load_2d_pair(dst + C::OFF_ALO, &tmAl, bar, 0, row_a);
          tma_load_2d_pair(dst + C::OFF_BLO, &tmBl, bar, 0, row_b);
        }
      }
    } else if (warp == 3 && lane == 0) {
      // ===================== ready watcher (both CTAs) =====================
      // this pair's slices in order: both panels split -> *ready_upto = g + 1
      int g = 0;
      for (int w = 0; pid + w * np < num_tiles; ++w) {
        const RingWave rw = ring_wave(w, np, num_tiles, tiles_m, tiles_n, gm);
        int tm, tn;
        ring_tile(pid + w * np, tiles_m, tiles_n, gm, tm, tn);
        const uint32_t* pa = ra.ready + (tm - rw.a_first);
        const uint32_t* pb = ra.ready + ra.la_max + (tn - rw.b_first + tiles_n) % tiles_n;
        for (int kb = 0; kb < nop; ++kb, ++g) {
          const int64_t off = int64_t(g) * pmax;
          for (uint32_t spin = 0;; ++spin) {
            const uint32_t va = ld_relaxed_u32(pa + off), vb = ld_relaxed_u32(pb + off);
            if (va >= kRingUnits && vb >= kRingUnits) break;
            __nanosleep(32);
            if (spin > (1u << 26)) __trap();
          }
          (void)ld_acquire_u32(pa + off);
          (void)ld_acquire_u32(pb + off);
          asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"(sm100::smem_u32(ready_upto)),
                       "r"(static_cast<uint32_t>(g + 1))
                       : "memory");
        }
      }
    } else if (warp == 2 && lane == 0) {
      // ===================== freed watcher (both CTAs) =====================
      const int slices = waves * nop;
      for (int g = 0; g + ra.depth < slices; ++g) {
        const int npw = min(np, num_tiles - (g / nop) * np);
        ring_wait_ge(ra.freed + g, static_cast<uint32_t>(npw));
        asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"(sm100::smem_u32(freed_upto)),
                     "r"(static_cast<uint32_t>(g + 1))
                     : "memory");
      }
    } else if (warp == 1 && lane == 0 && rank == 1) {
      // ===================== slice release (non-leader CTA) =====================
      // freed[g] += 1 once this pair's MMAs through slice g have completed
      int tiles_mine = 0;
      for (int t = pid; t < num_tiles; t += np) ++tiles_mine;
      const uint32_t total = static_cast<uint32_t>(tiles_mine * nop);
      uint32_t done = 0;
      for (uint32_t spin = 0; done < total; ++spin) {
        uint32_t v;
        asm volatile("ld.relaxed.cta.shared.u32 %0, [%1];" : "=r"(v)
                     : "r"(sm100::smem_u32(consumed_upto)) : "memory");
        if (v > done) {
          fence_proxy_async_global();
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
          for (; done < v; ++done)
            asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(ra.freed + done) : "memory");
          spin = 0;
        } else {
          __nanosleep(64);
          if (spin > (1u << 26)) __trap();
        }
      }
    } else if (warp == 1 && rank == 0) {  // the whole warp runs the issue loop; one elected lane issues
      // ===================== MMA issuer (leader CTA) =====================
      constexpr uint32_t idesc = sm100::umma_idesc(VC::AB_FORMAT, 2 * C::BM, C::BN);
      constexpr uint32_t hi_w = (1024u >> 4) | (1u << 14) | (2u << 29);  // SBO 1024, v1, SW128
      uint32_t g = 0, git = 0, gtile = 0;
      int pos = 0;
      for (int tile = pid; tile < num_tiles; tile += np, ++gtile) {
        for (int kb = 0; kb < nop; ++kb, ++g) {
          const int o = g % C::NOP;
          sm100::mbar_wait(&op_full[o], (g / C::NOP) & 1);
          sm100::tc_fence_after();
          if (kb == 0 && gtile > 0) {  // the previous tile's epilogue has read dC
            sm100::mbar_wait_cluster(acc_empty, (gtile - 1) & 1);
            sm100::tc_fence_after();
          }
          const uint32_t op = sm100::opaque(smem_base + C::OFF_OP + o * C::OP_BYTES) >> 4;
          const uint32_t ahi = op | (1u << 16);
          const uint32_t alo = ahi + (C::OFF_ALO >> 4);
          const uint32_t bhi = ahi + (C::OFF_BHI >> 4);
          const uint32_t blo = ahi + (C::OFF_BLO >> 4);
          c3_stage(
              kb * 4, 4 * nop, de, pos, git, p_empty, p_full, &op_empty[o],
              [&](int ks) {  // reference order per k-step: dA*B_hi, then A_hi*dB (schemes.py:294-298)
                sm100::mma_pair_split_el<V == kTF32>(tmem_dC, alo + 2 * ks, hi_w, bhi + 2 * ks, hi_w,
                                                  idesc, (kb | ks) != 0);
                sm100::mma_pair_split_el<V == kTF32>(tmem_dC, ahi + 2 * ks, hi_w, blo + 2 * ks, hi_w,
                                                  idesc, 1u);
              },
              [&](int ks, uint32_t acc) {
                sm100::mma_pair_split_el<V == kTF32>(tmem_P, ahi + 2 * ks, hi_w, bhi + 2 * ks, hi_w,
                                                  idesc, acc);
              });
        }
      }
    }
  } else if (warp < SPLIT_WARP0) {
    sm100::regs_inc<160>();
    // ===================== drain + epilogue (the split-once kernel's) =====================
    const int q = warp & 3;
    const int h = (warp - C::DRAIN_WARP0) >> 2;
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    const uint32_t p_empty_leader = sm100::mapa_shared(sm100::smem_u32(p_empty), 0);
    const uint32_t acc_empty_leader = sm100::mapa_shared(sm100::smem_u32(acc_empty), 0);
    constexpr int NC = C::DRAIN_COLS;
    bool nonfinite = false;
    uint32_t git = 0;
    for (int tile = pid; tile < num_tiles; tile += np) {
      int tm, tn;
      ring_tile(tile, tiles_m, tiles_n, gm, tm, tn);
      float acc[NC];
#pragma unroll
      for (int j = 0; j < NC; ++j) acc[j] = 0.0f;
      const int g0 = ((tile - pid) / np) * nop;  // the tile's first slice
      int rel = 0;                               // its stages released so far
      for (int it = 0; it < nintervals; ++it, ++git) {
        sm100::mbar_wait(p_full, git & 1);
        sm100::tc_fence_after();
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
        if (rank == 1 && warp == C::DRAIN_WARP0 && lane == 0) {
          // every MMA through this interval has completed: the operand stages
          // it covers are consumed (the release thread publishes them)
          const int upto = min((it + 1) * de, 4 * nop) / 4;
          if (upto > rel) {
            rel = upto;
            asm volatile("st.relaxed.cta.shared.u32 [%0], %1;" ::"r"(sm100::smem_u32(consumed_upto)),
                         "r"(static_cast<uint32_t>(g0 + rel))
                         : "memory");
          }
        }
      }
      const int64_t row = static_cast<int64_t>(tm) * 2 * C::BM + rank * C::BM + q * 32 + lane;
      const int col0 = tn * C::BN + h * NC;
      float* crow = Cout + row * ldc + col0;
#pragma unroll
      for (int c = 0; c < NC / 8; ++c) {
        uint32_t r[8];
        sm100::tmem_ld_32x32b_x8(tmem_dC + lane_off + h * NC + c * 8, r);
        sm100::tmem_ld_wait();
        float o[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          o[j] = __fmaf_rn(__uint_as_float(r[j]), inv_scale, acc[c * 8 + j]);  // schemes.py:306-307
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
  } else {
    sm100::regs_dec<56>();
    // ===================== split warps (every CTA of the grid) =====================
    const int nw = gridDim.x * NUM_SPLIT_WARPS;
    const int gw = blockIdx.x * NUM_SPLIT_WARPS + (warp - SPLIT_WARP0);
    FlagAcc fa;
    int off = 0;  // (units of all earlier slices) mod nw: unit u of slice g is warp (off + u) mod nw's
    for (int w = 0; w < waves; ++w) {
      const RingWave rw = ring_wave(w, np, num_tiles, tiles_m, tiles_n, gm);
      const int units = kRingUnits * (rw.la + rw.lb);
      for (int kb = 0; kb < nop; ++kb) {
        const int g = w * nop + kb;
        int u = gw - off;
        if (u < 0) u += nw;
        off += units % nw;
        if (off >= nw) off -= nw;
        if (u >= units) continue;
        const int s = g % ra.depth;
        bool waited = g < ra.depth;
        for (; u < units; u += nw) {
          const bool is_b = u >= kRingUnits * rw.la;
          const int uu = is_b ? u - kRingUnits * rw.la : u;
          const int idx = uu / kRingUnits, sub = uu % kRingUnits;
          const int k0 = kb * VC::BK_OP;
          const int panel = is_b ? (rw.b_first + idx) % tiles_n : rw.a_first + idx;
          float x[RingUnit<V>::NX];
          if (is_b)
            ring_load_unit<V, true>(ra, shp, lane, k0, panel, sub, x);
          else
            ring_load_unit<V, false>(ra, shp, lane, k0, panel, sub, x);
          if (!waited) {  // slot s: every pair of slice g - D's wave has consumed it
            const uint32_t need = static_cast<uint32_t>(g - ra.depth + 1);
            const uint32_t fa_addr = sm100::smem_u32(freed_upto);
            for (uint32_t spin = 0;; ++spin) {
              uint32_t v;
              asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"(fa_addr) : "memory");
              if (v >= need) break;
              __nanosleep(64);
              if (spin > (1u << 26)) __trap();
            }
            waited = true;
          }
          // RunFlags: each A row-panel in the wave holding its column-0 tile, each
          // B column-panel in the wave holding its row-0 tile (every element once)
          if (!is_b) {
            const bool fl =
                flags != nullptr && ring_tile_index(panel, 0, tiles_m, tiles_n, gm) / np == w;
            ring_store_unit<V, R>(lane, s * ra.la_max + idx, sub, ra.ahi, ra.alo, scale, fl,
                                         fa, x);
          } else {
            const bool fl =
                flags != nullptr && ring_tile_index(0, panel, tiles_m, tiles_n, gm) / np == w;
            ring_store_unit<V, R>(lane, s * ra.lb_max + idx, sub, ra.bhi, ra.blo, scale, fl,
                                        fa, x);
          }
          __syncwarp();  // (the consumers order their TMA reads after the counter)
          if (lane == 0)
            red_release_add(ra.ready + int64_t(g) * pmax + (is_b ? ra.la_max + idx : idx), 1u);
        }
      }
    }
    flag_publish(fa, thr, flags);
  }

  __syncthreads();
  sm100::cluster_sync();
  if (warp == 2) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc_pair<C::TMEM_COLS>(tmem_base);
  }
}

}  // namespace tcec
