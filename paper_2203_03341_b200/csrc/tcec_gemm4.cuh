// tcec_gemm4.cuh -- CTA-pair TCEC SGEMM, FP32 operands loaded straight into
// registers (no shared-memory staging).
//
// Measurement (scripts/gpu_exp2.sh) showed the staging ring's
// shared-memory traffic -- TMA writing the FP32 k-slices and the split warps
// reading them back -- bounds the pair kernel: without it the same pipeline
// runs 1.5-1.9x faster.  Here the 16 worker warps of each CTA read their FP32
// values with non-allocating global loads (L2 -> registers), split them in
// registers and write only the (hi, lo) operands to shared memory.  With no
// staging ring the operand ring is three stages deep.
//
// Same 256 x 256 cta_group::2 tile, operand layouts, MMA issue order and
// cross-CTA protocol as tcec_gemm_pair_uni_kernel (tcec_gemm3.cuh).  Worker
// thread t (0..511) owns, per 32-deep k-slice, 8 consecutive values of one A
// row (row t & 127, k 8 (t >> 7) ...) and 8 consecutive values of one B k-row
// (k t & 31, n 8 (t >> 5) ...); slices are double-buffered in registers so
// the loads of slice s+1 are in flight while slice s is split.  Warp 0 warms
// L2 with TMA prefetches a few stages ahead, paced by the operand ring.
#pragma once

#include "tcec_gemm3.cuh"

namespace tcec {

template <int V>
struct DirectCfg {
  using P = PairCfg<V>;
  static constexpr int NOP = 3;
  static constexpr int OFF_OP = 0;
  static constexpr int OFF_BAR = NOP * P::OP_BYTES;
  static constexpr int NUM_BARS = 2 * NOP + 2;
  static constexpr int SMEM_BYTES = OFF_BAR + NUM_BARS * 8 + 16;
  static constexpr int NUM_THREADS = 640;
  static constexpr int WORKER_WARP0 = 4;
  static constexpr int NUM_WORKER_WARPS = 16;
  static constexpr int EPI_WORKER_BYTES = 32 * 64 * 4;
  static constexpr int PREFETCH_STAGES = 2;  // L2 warm-up distance beyond the ring
  static_assert(NUM_WORKER_WARPS * EPI_WORKER_BYTES <= OFF_BAR, "epilogue staging fits");
};

__device__ __forceinline__ float4 ldg_stream(const float* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

// 4 consecutive floats p[0..3]; columns [c0, c0+4) checked against `cols`
// (zero beyond), the whole run zeroed when !row_ok.
__device__ __forceinline__ float4 load4(const float* p, bool row_ok, int c0, int cols) {
  if (row_ok && c0 + 4 <= cols) return ldg_stream(p);
  float4 v;
  v.x = (row_ok && c0 + 0 < cols) ? __ldg(p + 0) : 0.0f;
  v.y = (row_ok && c0 + 1 < cols) ? __ldg(p + 1) : 0.0f;
  v.z = (row_ok && c0 + 2 < cols) ? __ldg(p + 2) : 0.0f;
  v.w = (row_ok && c0 + 3 < cols) ? __ldg(p + 3) : 0.0f;
  return v;
}

// One thread's share of a 32-deep k-slice, chosen so that every warp-wide
// load covers whole 128-byte lines (4 rows of A x 128 B, one k-row of B x
// 512 B):
//   a[0..3]: A row (8 w + (lane >> 3)),     k 4 (lane & 7) .. +3
//   a[4..7]: A row (8 w + 4 + (lane >> 3)), same k
//   b[0..3]: B k-row 2 w,     n 4 lane .. +3
//   b[4..7]: B k-row 2 w + 1, same n
struct DirectSlice {
  float4 a0, a1, b0, b1;
};

struct DirectGeom {
  const float* A;
  const float* B;
  int64_t lda, ldb;
  int m, n, k;
  int a_row;   // global row of a0 (a1: + 4)
  int a_k;     // k offset within a slice (multiple of 4)
  int b_k;     // k-row offset within a slice of b0 (b1: + 1)
  int b_col;   // first global column (multiple of 4)
};

__device__ __forceinline__ void direct_load(const DirectGeom& g, int slice, DirectSlice& x) {
  const int ka = slice * 32 + g.a_k;
  const float* pa = g.A + static_cast<int64_t>(g.a_row) * g.lda + ka;
  x.a0 = load4(pa, g.a_row < g.m, ka, g.k);
  x.a1 = load4(pa + 4 * g.lda, g.a_row + 4 < g.m, ka, g.k);
  const int kb = slice * 32 + g.b_k;
  const float* pb = g.B + static_cast<int64_t>(kb) * g.ldb + g.b_col;
  x.b0 = load4(pb, kb < g.k, g.b_col, g.n);
  x.b1 = load4(pb + g.ldb, kb + 1 < g.k, g.b_col, g.n);
}

// 4 consecutive values -> hi / lo words: FP16 2 packed half2 words each
// (8 bytes), TF32 4 words each (16 bytes).
template <int V, int R>
__device__ __forceinline__ void split4(const float4& v, float scale, uint32_t (&hw)[4],
                                       uint32_t (&lw)[4]) {
  if constexpr (V == kFP16) {
    float h0, h1, r0, r1;
    hw[0] = cvt_f16x2<R>(v.x, v.y);
    unpack_f16x2(hw[0], h0, h1);
    sm100::residual_x2(v.x, v.y, h0, h1, scale, r0, r1);
    lw[0] = cvt_f16x2<R>(r0, r1);
    hw[1] = cvt_f16x2<R>(v.z, v.w);
    unpack_f16x2(hw[1], h0, h1);
    sm100::residual_x2(v.z, v.w, h0, h1, scale, r0, r1);
    lw[1] = cvt_f16x2<R>(r0, r1);
  } else {
    const float xs[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 4; j += 2) {
      hw[j] = tf32_round_bits<R>(__float_as_uint(xs[j]));
      hw[j + 1] = tf32_round_bits<R>(__float_as_uint(xs[j + 1]));
      float r0, r1;
      sm100::sub_x2(xs[j], xs[j + 1], __uint_as_float(hw[j]), __uint_as_float(hw[j + 1]), r0, r1);
      lw[j] = tf32_round_bits<R>(__float_as_uint(r0));
      lw[j + 1] = tf32_round_bits<R>(__float_as_uint(r1));
    }
  }
}

__device__ __forceinline__ void sts64(uint32_t addr, uint32_t a, uint32_t b) {
  asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(addr), "r"(a), "r"(b) : "memory");
}

// Store 4 split values: FP16 -> 8-byte half of a 16-byte chunk, TF32 -> the chunk.
template <int V>
__device__ __forceinline__ void store4(uint32_t chunk_addr, uint32_t half_sel,
                                      const uint32_t (&w)[4]) {
  if constexpr (V == kFP16) {
    sts64(chunk_addr + half_sel * 8, w[0], w[1]);
  } else {
    sm100::sts128(chunk_addr, w[0], w[1], w[2], w[3]);
  }
}

// Split one slice held in registers into operand stage `op` (sub = slice index
// within the stage): A -> K-major SW128, B -> MN-major (SW128 FP16 /
// SW128_BASE32B TF32), the layouts of the staged pair kernel.
template <int V, int R, bool kFlags>
__device__ __forceinline__ void direct_split(const DirectSlice& xs, uint32_t op, int sub, int t,
                                             float scale, FlagAcc& fa) {
  using C = PairCfg<V>;
  if constexpr (kFlags) {
    const float4 q[4] = {xs.a0, xs.a1, xs.b0, xs.b1};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      fa.add(q[i].x); fa.add(q[i].y); fa.add(q[i].z); fa.add(q[i].w);
    }
  }
  const int w = t >> 5, lane = t & 31;
  {  // A rows 8w + (lane >> 3) (+4), k = 4 (lane & 7) within the slice
    const int kq = lane & 7;                         // 4-value group
    const int kop = sub * 32 + 4 * kq;               // k within the stage
    const int chunk = V == kFP16 ? kop >> 3 : kop >> 2;
    const uint32_t half_sel = V == kFP16 ? (kq & 1) : 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int row = 8 * w + 4 * h + (lane >> 3);
      uint32_t hw[4], lw[4];
      split4<V, R>(h ? xs.a1 : xs.a0, scale, hw, lw);
      const uint32_t off = sw128(row, chunk);
      store4<V>(op + off, half_sel, hw);
      store4<V>(op + C::OP_A_BYTES + off, half_sel, lw);
    }
  }
  {  // B k-rows 2w (+1), n = 4 lane .. +3 of this CTA's 128 columns
    const int n0 = 4 * lane;
    const int atom = n0 / C::B_ATOM_N;
    const int c16 = (n0 % C::B_ATOM_N) * (V == kFP16 ? 2 : 4) / 16;
    const uint32_t half_sel = V == kFP16 ? (lane & 1) : 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int kop = sub * 32 + 2 * w + h;
      const int grp = kop / C::B_ROWS, rr = kop % C::B_ROWS;
      const uint32_t base = op + 2 * C::OP_A_BYTES + grp * C::B_SBO + atom * C::B_LBO + rr * 128;
      const uint32_t off = V == kFP16 ? ((c16 ^ rr) << 4)
                                      : ((((c16 >> 1) ^ rr) & 3) << 5) + ((c16 & 1) << 4);
      uint32_t hw[4], lw[4];
      split4<V, R>(h ? xs.b1 : xs.b0, scale, hw, lw);
      store4<V>(base + off, half_sel, hw);
      store4<V>(base + C::OP_B_BYTES + off, half_sel, lw);
    }
  }
}

template <int V, int R, bool kFlags>
__device__ __forceinline__ void direct_worker_loop(const DirectGeom& g, uint32_t smem,
                                                   uint64_t* op_full, uint64_t* op_empty,
                                                   uint64_t* p_full, uint64_t* p_empty,
                                                   uint32_t tmem_P, int nop, int de, int t,
                                                   int lane, float scale, FlagAcc& fa,
                                                   float (&acc)[64]) {
  using C = PairCfg<V>;
  using D = DirectCfg<V>;
  constexpr int SPO = VarCfg<V>::STG_PER_OP;  // 32-deep slices per operand stage
  const uint32_t leader_op_full = sm100::mapa_shared(sm100::smem_u32(op_full), 0);
  const uint32_t p_empty_leader = sm100::mapa_shared(sm100::smem_u32(p_empty), 0);
  const int w = t >> 5;
  const uint32_t lane_off = static_cast<uint32_t>((w & 3) * 32) << 16;
  const int cb = w >> 2;
  const int nslices = nop * SPO;

  auto begin_slice = [&](int s) {
    if (s % SPO == 0) {
      const int kb = s / SPO;
      sm100::mbar_wait(&op_empty[kb % D::NOP], ((kb / D::NOP) & 1) ^ 1);
    }
  };
  auto end_slice = [&](int s) {
    if (s % SPO == SPO - 1) {
      const int kb = s / SPO;
      sm100::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive_remote(leader_op_full + (kb % D::NOP) * 8);
      if (kb >= 1 && ((kb - 1) % de) == de - 1)
        uni_drain(acc, tmem_P, lane_off, cb, p_full, (kb - 1) / de, p_empty_leader, lane);
    }
  };
  auto stage_addr = [&](int s) {
    return smem + D::OFF_OP + ((s / SPO) % D::NOP) * C::OP_BYTES;
  };

  DirectSlice bufA, bufB;
  direct_load(g, 0, bufA);
  for (int s = 0; s < nslices; s += 2) {
    if (s + 1 < nslices) direct_load(g, s + 1, bufB);
    begin_slice(s);
    direct_split<V, R, kFlags>(bufA, stage_addr(s), s % SPO, t, scale, fa);
    end_slice(s);
    if (s + 1 >= nslices) break;
    if (s + 2 < nslices) direct_load(g, s + 2, bufA);
    begin_slice(s + 1);
    direct_split<V, R, kFlags>(bufB, stage_addr(s + 1), (s + 1) % SPO, t, scale, fa);
    end_slice(s + 1);
  }
  const int nintervals = (nop + de - 1) / de;
  uni_drain(acc, tmem_P, lane_off, cb, p_full, nintervals - 1, p_empty_leader, lane);
}

template <int V, int R>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(DirectCfg<V>::NUM_THREADS, 1)
    tcec_gemm_direct_kernel(const float* __restrict__ A, int64_t lda,
                            const float* __restrict__ B, int64_t ldb,
                            const __grid_constant__ CUtensorMap tmA,  // L2 prefetch only
                            const __grid_constant__ CUtensorMap tmB,  // L2 prefetch only
                            const __grid_constant__ CUtensorMap tmC,  // C store
                            const GemmShape shp, const float scale, const float inv_scale,
                            const FlagThresholds thr, uint32_t* __restrict__ flags) {
  using C = PairCfg<V>;
  using VC = VarCfg<V>;
  using D = DirectCfg<V>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + D::OFF_BAR);
  uint64_t* op_full = bars;                 // workers -> MMA        (leader, 32)
  uint64_t* op_empty = bars + D::NOP;       // MMA commit -> workers (both, multicast)
  uint64_t* p_full = bars + 2 * D::NOP;     // MMA commit -> workers (both, multicast)
  uint64_t* p_empty = p_full + 1;           // workers -> MMA        (leader, 32)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + D::NUM_BARS);
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
  const int de = shp.drain_every;

  if (warp == 0 && lane == 0) {
    if (smem_base & 1023u) __trap();
    sm100::tma_prefetch_desc(&tmA);
    sm100::tma_prefetch_desc(&tmB);
    sm100::tma_prefetch_desc(&tmC);
    for (int o = 0; o < D::NOP; ++o) {
      sm100::mbar_init(&op_full[o], 2 * D::NUM_WORKER_WARPS);
      sm100::mbar_init(&op_empty[o], 1);
    }
    sm100::mbar_init(p_full, 1);
    sm100::mbar_init(p_empty, 2 * D::NUM_WORKER_WARPS);
    sm100::fence_mbar_init();
  }
  if (warp == 2) sm100::tmem_alloc_pair<C::TMEM_COLS>(tmem_slot);
  sm100::tc_fence_before();
  sm100::cluster_sync();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t tmem_P = tmem_base;
  const uint32_t tmem_dC = tmem_base + C::BN;

  if (warp < D::WORKER_WARP0) {
    sm100::regs_dec<32>();
    if (warp == 0 && lane == 0 && shp.prefetch > 0) {
      // ===================== L2 warm-up, paced by the operand ring =====================
      constexpr int SPO = VC::STG_PER_OP;
      const int ahead = D::NOP + D::PREFETCH_STAGES;
      auto prefetch_stage = [&](int kb) {
        if (kb >= nop) return;
        for (int sub = 0; sub < SPO; ++sub) {
          const int sl = kb * SPO + sub;
          sm100::tma_prefetch_2d(&tmA, sl * 32, m_cta);
#pragma unroll
          for (int b = 0; b < 4; ++b) sm100::tma_prefetch_2d(&tmB, n_cta + 32 * b, sl * 32);
        }
      };
      for (int kb = 0; kb < ahead; ++kb) prefetch_stage(kb);
      for (int kb = 0; kb + ahead < nop; ++kb) {
        sm100::mbar_wait(&op_empty[kb % D::NOP], (kb / D::NOP) & 1);  // stage kb consumed
        prefetch_stage(kb + ahead);
      }
    } else if (warp == 1 && lane == 0 && rank == 0) {
      // ===================== MMA issuer (leader CTA) =====================
      constexpr uint32_t idesc = sm100::umma_idesc_bmn(VC::AB_FORMAT, 2 * C::BM, C::BN);
      constexpr uint32_t a_hi_w = (1024u >> 4) | (1u << 14) | (2u << 29);
      constexpr uint32_t b_hi_w = (uint32_t(C::B_SBO) >> 4) | (1u << 14) | (C::B_LAYOUT << 29);
      constexpr uint32_t b_lbo_w = (uint32_t(C::B_LBO) >> 4) << 16;
      constexpr uint32_t kB = C::B_KSTEP_BYTES >> 4;
      for (int kb = 0; kb < nop; ++kb) {
        const int o = kb % D::NOP;
        sm100::mbar_wait_cluster(&op_full[o], (kb / D::NOP) & 1);
        sm100::tc_fence_after();
        const uint32_t op = sm100::opaque(smem_base + D::OFF_OP + o * C::OP_BYTES) >> 4;
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
    // ===================== workers: load + split + drain + epilogue =====================
    const int t = threadIdx.x - D::WORKER_WARP0 * 32;
    const int w = t >> 5;
    DirectGeom g;
    g.A = A; g.B = B; g.lda = lda; g.ldb = ldb; g.m = shp.m; g.n = shp.n; g.k = shp.k;
    g.a_row = m_cta + 8 * w + ((t & 31) >> 3);
    g.a_k = 4 * (t & 7);
    g.b_k = 2 * w;
    g.b_col = n_cta + 4 * (t & 31);
    float acc[64];
#pragma unroll
    for (int j = 0; j < 64; ++j) acc[j] = 0.0f;
    FlagAcc fa;
    const bool do_flags = flags != nullptr && (tile_n == 0 || tile_m == 0);
    if (do_flags) {
      direct_worker_loop<V, R, true>(g, smem_base, op_full, op_empty, p_full, p_empty, tmem_P,
                                     nop, de, t, lane, scale, fa, acc);
      flag_publish(fa, thr, flags);
    } else {
      direct_worker_loop<V, R, false>(g, smem_base, op_full, op_empty, p_full, p_empty, tmem_P,
                                      nop, de, t, lane, scale, fa, acc);
    }
    const int q = w & 3, cb = w >> 2;
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    bool nonfinite = false;
    const uint32_t stage = smem_base + w * D::EPI_WORKER_BYTES;
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

// ---------------------------------------------------------------------------
// Hybrid: A straight to registers (coalesced non-allocating loads, one slice
// ahead), B through a TMA staging ring (16 KB per 32-deep slice, 6 deep).
// Halves the staging traffic through shared memory with half the register
// footprint of the all-direct kernel.
template <int V>
struct HybridCfg {
  using P = PairCfg<V>;
  static constexpr int NOP = 2;
  static constexpr int NSTG = 6;                       // B staging slices
  static constexpr int STG_BYTES = P::STG_B_BYTES;     // 4 boxes of 32 k x 32 n
  static constexpr int OFF_STG = 0;
  static constexpr int OFF_OP = NSTG * STG_BYTES;
  static constexpr int OFF_BAR = OFF_OP + NOP * P::OP_BYTES;
  static constexpr int NUM_BARS = 2 * NSTG + 2 * NOP + 2;
  static constexpr int SMEM_BYTES = OFF_BAR + NUM_BARS * 8 + 16;
  static constexpr int NUM_THREADS = 640;
  static constexpr int WORKER_WARP0 = 4;
  static constexpr int NUM_WORKER_WARPS = 16;
  static constexpr int EPI_WORKER_BYTES = 32 * 64 * 4;
  static_assert(NUM_WORKER_WARPS * EPI_WORKER_BYTES <= OFF_BAR, "epilogue staging fits");
};

struct HybridA {
  float4 a0, a1;
};

__device__ __forceinline__ void hybrid_load_a(const DirectGeom& g, int slice, HybridA& x) {
  const int ka = slice * 32 + g.a_k;
  const float* pa = g.A + static_cast<int64_t>(g.a_row) * g.lda + ka;
  x.a0 = load4(pa, g.a_row < g.m, ka, g.k);
  x.a1 = load4(pa + 4 * g.lda, g.a_row + 4 < g.m, ka, g.k);
}

template <int V, int R, bool kFlags>
__device__ __forceinline__ void hybrid_split_a(const HybridA& xs, uint32_t op, int sub, int t,
                                               float scale, FlagAcc& fa) {
  using C = PairCfg<V>;
  if constexpr (kFlags) {
    fa.add(xs.a0.x); fa.add(xs.a0.y); fa.add(xs.a0.z); fa.add(xs.a0.w);
    fa.add(xs.a1.x); fa.add(xs.a1.y); fa.add(xs.a1.z); fa.add(xs.a1.w);
  }
  const int w = t >> 5, lane = t & 31;
  const int kq = lane & 7;
  const int kop = sub * 32 + 4 * kq;
  const int chunk = V == kFP16 ? kop >> 3 : kop >> 2;
  const uint32_t half_sel = V == kFP16 ? (kq & 1) : 0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int row = 8 * w + 4 * h + (lane >> 3);
    uint32_t hw[4], lw[4];
    split4<V, R>(h ? xs.a1 : xs.a0, scale, hw, lw);
    const uint32_t off = sw128(row, chunk);
    store4<V>(op + off, half_sel, hw);
    store4<V>(op + C::OP_A_BYTES + off, half_sel, lw);
  }
}

template <int V, int R, bool kFlags>
__device__ __forceinline__ void hybrid_worker_loop(const DirectGeom& g, uint32_t smem,
                                                   uint64_t* stg_full, uint64_t* stg_empty,
                                                   uint64_t* op_full, uint64_t* op_empty,
                                                   uint64_t* p_full, uint64_t* p_empty,
                                                   uint32_t tmem_P, int nop, int de, int t,
                                                   int lane, float scale, FlagAcc& fa,
                                                   float (&acc)[64]) {
  using C = PairCfg<V>;
  using H = HybridCfg<V>;
  constexpr int SPO = VarCfg<V>::STG_PER_OP;
  const uint32_t leader_op_full = sm100::mapa_shared(sm100::smem_u32(op_full), 0);
  const uint32_t p_empty_leader = sm100::mapa_shared(sm100::smem_u32(p_empty), 0);
  const int w = t >> 5;
  const uint32_t lane_off = static_cast<uint32_t>((w & 3) * 32) << 16;
  const int cb = w >> 2;
  const int nslices = nop * SPO;

  auto slice = [&](const HybridA& xa, int s) {
    const int kb = s / SPO, sub = s % SPO;
    const uint32_t op = smem + H::OFF_OP + (kb % H::NOP) * C::OP_BYTES;
    if (sub == 0) sm100::mbar_wait(&op_empty[kb % H::NOP], ((kb / H::NOP) & 1) ^ 1);
    hybrid_split_a<V, R, kFlags>(xa, op, sub, t, scale, fa);
    const int st = s % H::NSTG;
    sm100::mbar_wait(&stg_full[st], (s / H::NSTG) & 1);
    // B part from the staging ring (layout of the staged pair kernel)
    uni_split_part<V, R, kFlags, true>(smem + H::OFF_STG + st * H::STG_BYTES - C::STG_A_BYTES, op,
                                       sub, t, scale, fa);
    __syncwarp();
    if (lane == 0) sm100::mbar_arrive(&stg_empty[st]);
    if (sub == SPO - 1) {
      sm100::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive_remote(leader_op_full + (kb % H::NOP) * 8);
      if (kb >= 1 && ((kb - 1) % de) == de - 1)
        uni_drain(acc, tmem_P, lane_off, cb, p_full, (kb - 1) / de, p_empty_leader, lane);
    }
  };

  HybridA bufA, bufB;
  hybrid_load_a(g, 0, bufA);
  for (int s = 0; s < nslices; s += 2) {
    if (s + 1 < nslices) hybrid_load_a(g, s + 1, bufB);
    slice(bufA, s);
    if (s + 1 >= nslices) break;
    if (s + 2 < nslices) hybrid_load_a(g, s + 2, bufA);
    slice(bufB, s + 1);
  }
  const int nintervals = (nop + de - 1) / de;
  uni_drain(acc, tmem_P, lane_off, cb, p_full, nintervals - 1, p_empty_leader, lane);
}

template <int V, int R>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(HybridCfg<V>::NUM_THREADS, 1)
    tcec_gemm_hybrid_kernel(const float* __restrict__ A, int64_t lda,
                            const __grid_constant__ CUtensorMap tmB,  // B [k][n], box 32 x 32, SW128
                            const __grid_constant__ CUtensorMap tmC,
                            const GemmShape shp, const float scale, const float inv_scale,
                            const FlagThresholds thr, uint32_t* __restrict__ flags) {
  using C = PairCfg<V>;
  using VC = VarCfg<V>;
  using H = HybridCfg<V>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + H::OFF_BAR);
  uint64_t* stg_full = bars;
  uint64_t* stg_empty = bars + H::NSTG;
  uint64_t* op_full = bars + 2 * H::NSTG;
  uint64_t* op_empty = op_full + H::NOP;
  uint64_t* p_full = op_empty + H::NOP;
  uint64_t* p_empty = p_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + H::NUM_BARS);
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
  const int nslices = nop * VC::STG_PER_OP;
  const int de = shp.drain_every;

  if (warp == 0 && lane == 0) {
    if (smem_base & 1023u) __trap();
    sm100::tma_prefetch_desc(&tmB);
    sm100::tma_prefetch_desc(&tmC);
    for (int s = 0; s < H::NSTG; ++s) {
      sm100::mbar_init(&stg_full[s], 1);
      sm100::mbar_init(&stg_empty[s], H::NUM_WORKER_WARPS);
    }
    for (int o = 0; o < H::NOP; ++o) {
      sm100::mbar_init(&op_full[o], 2 * H::NUM_WORKER_WARPS);
      sm100::mbar_init(&op_empty[o], 1);
    }
    sm100::mbar_init(p_full, 1);
    sm100::mbar_init(p_empty, 2 * H::NUM_WORKER_WARPS);
    sm100::fence_mbar_init();
  }
  if (warp == 2) sm100::tmem_alloc_pair<C::TMEM_COLS>(tmem_slot);
  sm100::tc_fence_before();
  sm100::cluster_sync();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t tmem_P = tmem_base;
  const uint32_t tmem_dC = tmem_base + C::BN;

  if (warp < H::WORKER_WARP0) {
    sm100::regs_dec<32>();
    if (warp == 0 && lane == 0) {
      // ===================== TMA producer: B slices only =====================
      for (int st = 0; st < nslices; ++st) {
        const int s = st % H::NSTG;
        sm100::mbar_wait(&stg_empty[s], ((st / H::NSTG) & 1) ^ 1);
        uint8_t* dst = smem + H::OFF_STG + s * H::STG_BYTES;
        sm100::mbar_arrive_expect_tx(&stg_full[s], H::STG_BYTES);
#pragma unroll
        for (int b = 0; b < 4; ++b)
          sm100::tma_load_2d(dst + b * C::STG_B_BOX, &tmB, &stg_full[s], n_cta + 32 * b, st * 32);
      }
    } else if (warp == 1 && lane == 0 && rank == 0) {
      // ===================== MMA issuer (leader CTA) =====================
      constexpr uint32_t idesc = sm100::umma_idesc_bmn(VC::AB_FORMAT, 2 * C::BM, C::BN);
      constexpr uint32_t a_hi_w = (1024u >> 4) | (1u << 14) | (2u << 29);
      constexpr uint32_t b_hi_w = (uint32_t(C::B_SBO) >> 4) | (1u << 14) | (C::B_LAYOUT << 29);
      constexpr uint32_t b_lbo_w = (uint32_t(C::B_LBO) >> 4) << 16;
      constexpr uint32_t kB = C::B_KSTEP_BYTES >> 4;
      for (int kb = 0; kb < nop; ++kb) {
        const int o = kb % H::NOP;
        sm100::mbar_wait_cluster(&op_full[o], (kb / H::NOP) & 1);
        sm100::tc_fence_after();
        const uint32_t op = sm100::opaque(smem_base + H::OFF_OP + o * C::OP_BYTES) >> 4;
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
    const int t = threadIdx.x - H::WORKER_WARP0 * 32;
    const int w = t >> 5;
    DirectGeom g;
    g.A = A; g.B = nullptr; g.lda = lda; g.ldb = 0; g.m = shp.m; g.n = shp.n; g.k = shp.k;
    g.a_row = m_cta + 8 * w + ((t & 31) >> 3);
    g.a_k = 4 * (t & 7);
    g.b_k = 0;
    g.b_col = 0;
    float acc[64];
#pragma unroll
    for (int j = 0; j < 64; ++j) acc[j] = 0.0f;
    FlagAcc fa;
    const bool do_flags = flags != nullptr && (tile_n == 0 || tile_m == 0);
    if (do_flags) {
      hybrid_worker_loop<V, R, true>(g, smem_base, stg_full, stg_empty, op_full, op_empty, p_full,
                                     p_empty, tmem_P, nop, de, t, lane, scale, fa, acc);
      flag_publish(fa, thr, flags);
    } else {
      hybrid_worker_loop<V, R, false>(g, smem_base, stg_full, stg_empty, op_full, op_empty,
                                      p_full, p_empty, tmem_P, nop, de, t, lane, scale, fa, acc);
    }
    const int q = w & 3, cb = w >> 2;
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    bool nonfinite = false;
    const uint32_t stage = smem_base + w * H::EPI_WORKER_BYTES;
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
