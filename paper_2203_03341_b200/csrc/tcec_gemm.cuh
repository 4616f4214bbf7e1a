// tcec_gemm.cuh -- the fused error-corrected SGEMM kernel for sm_100a.
//
// Restates the reference's corrected3 path (schemes.py:265-314, gemm branch
// :365-366) as one warp-specialised kernel per 128 x BN output tile:
//
//   TMA warp     FP32 A/B k-slices (32 deep) -> shared-memory staging ring
//   split warps  staging ring -> (hi, lo) operand ring, UMMA K-major SW128
//                layout (splitting.py:114-122, fused: hi/lo never touch HBM)
//   MMA thread   per operand stage (64 k for FP16, 32 k for TF32):
//                  dC += A_lo*B_hi ; dC += A_hi*B_lo   per MMA k-step (TMEM)
//                  P   = sum A_hi*B_hi                 (TMEM, fresh per drain)
//                corrections are issued first so the drain of the previous
//                P overlaps them; the lo*lo term is dropped (schemes.py:294-298)
//   drain warps  C = RN32(C + P) every drain interval on the CUDA cores
//                (schemes.py:300-304: "avoid RZ"), C held in registers;
//                epilogue C = RN32(C + dC * 2^-s) with one fused rounding
//                (schemes.py:306-307) -> swizzled smem -> TMA store.
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_fp16.h>

#include "sm100.cuh"
#include "split.cuh"

namespace tcec {

struct GemmShape {
  int32_t m, n, k;
  int32_t num_op_stages;   // ceil(k / BK_OP)
  int32_t drain_every;     // MMA k-steps (16 FP16 / 8 TF32 deep) per drain interval (>= 1)
  int32_t group_m;         // tile rasterisation group
};

// Extra destinations of the output tile (fused all-gather: this rank's C slab
// stored into every peer's full C over NVLink by the same TMA-store epilogue).
// Each map covers the same m x n slab (the pointer already offset to it).
constexpr int kMaxExtraC = 7;
struct CDests {
  CUtensorMap m[kMaxExtraC];
  int32_t count;
};

template <int BN_>
struct TileCfg {
  static constexpr int BM = 128;
  static constexpr int BN = BN_;
  static constexpr int BK_STG = 32;          // fp32 elements per staging slice (128 B rows)
  static constexpr int NSTG = 3;             // staging ring depth
  static constexpr int NOP = 2;              // operand ring depth
  static constexpr int STG_A_BYTES = BM * BK_STG * 4;
  static constexpr int STG_B_BYTES = BK_STG * BN * 4;
  static constexpr int STG_BYTES = STG_A_BYTES + STG_B_BYTES;
  static constexpr int OP_A_BYTES = BM * 128;  // one 128-byte K row per M row
  static constexpr int OP_B_BYTES = BN * 128;
  static constexpr int OP_BYTES = 2 * OP_A_BYTES + 2 * OP_B_BYTES;  // hi + lo of A and B
  static constexpr int OFF_STG = 0;
  static constexpr int OFF_OP = NSTG * STG_BYTES;
  static constexpr int OFF_BAR = OFF_OP + NOP * OP_BYTES;
  static constexpr int NUM_BARS = 2 * NSTG + 2 * NOP + 2;
  static constexpr int SMEM_BYTES = OFF_BAR + NUM_BARS * 8 + 16 + 1024;  // + align slack
  static constexpr int TMEM_COLS = (2 * BN <= 256) ? 256 : 512;         // P | dC
  static constexpr int NUM_THREADS = 640;                               // 20 warps
  static constexpr int SPLIT_WARP0 = 4, NUM_SPLIT_WARPS = 8;
  static constexpr int DRAIN_WARP0 = 12, NUM_DRAIN_WARPS = 8;
  static constexpr int EPI_BOX = 32;  // 32 x 32 fp32 TMA store box per drain warp
  static_assert(BN % 64 == 0 && BN <= 256, "BN must be 64..256 in steps of 64");
  static_assert(NUM_DRAIN_WARPS * 32 * 32 * 4 * (BN / 2 / EPI_BOX) <= NSTG * STG_BYTES,
                "epilogue staging must fit in the staging ring");
};

// Operand-stage geometry per variant: 128-byte K rows hold 64 FP16 or 32 TF32.
template <int V>
struct VarCfg;
template <>
struct VarCfg<kFP16> {
  static constexpr int BK_OP = 64;
  static constexpr int STG_PER_OP = 2;
  static constexpr uint32_t AB_FORMAT = 0;  // F16
};
template <>
struct VarCfg<kTF32> {
  static constexpr int BK_OP = 32;
  static constexpr int STG_PER_OP = 1;
  static constexpr uint32_t AB_FORMAT = 2;  // TF32
};

// Byte offset of the 16-byte chunk `chunk` of row `row` in a 128-byte-swizzled
// tile with 128-byte rows (the TMA SWIZZLE_128B / UMMA SW128 K-major layout).
__device__ __forceinline__ uint32_t sw128(uint32_t row, uint32_t chunk) {
  return row * 128u + (((chunk ^ (row & 7u)) & 7u) << 4);
}

// Split one staging slice (32 k of A and B) into the operand stage.
// 256 split threads: thread t owns row / column (t & 127) and k-half (t >> 7).
template <int V, int R, int BN>
__device__ __forceinline__ void split_slice(const uint8_t* stg, uint8_t* op, int sub, int t,
                                            float scale, FlagAcc& fa) {
  using C = TileCfg<BN>;
  const int r = t & 127;
  const int half = t >> 7;
  const uint8_t* stgA = stg;
  const float* stgB = reinterpret_cast<const float*>(stg + C::STG_A_BYTES);
  uint8_t* opAhi = op;
  uint8_t* opAlo = op + C::OP_A_BYTES;
  uint8_t* opBhi = op + 2 * C::OP_A_BYTES;
  uint8_t* opBlo = opBhi + C::OP_B_BYTES;

  // ---- A: row r, k in [16*half, 16*half + 16) of this slice
  float xa[16];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float4 v = *reinterpret_cast<const float4*>(stgA + sw128(r, half * 4 + i));
    xa[4 * i + 0] = v.x;
    xa[4 * i + 1] = v.y;
    xa[4 * i + 2] = v.z;
    xa[4 * i + 3] = v.w;
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) fa.add(xa[i]);

  if constexpr (V == kFP16) {
    uint32_t hp[8], lp[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) split_f16_pair<R>(xa[2 * j], xa[2 * j + 1], scale, hp[j], lp[j]);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const uint32_t off = sw128(r, sub * 4 + half * 2 + q);
      *reinterpret_cast<uint4*>(opAhi + off) = make_uint4(hp[4 * q], hp[4 * q + 1], hp[4 * q + 2], hp[4 * q + 3]);
      *reinterpret_cast<uint4*>(opAlo + off) = make_uint4(lp[4 * q], lp[4 * q + 1], lp[4 * q + 2], lp[4 * q + 3]);
    }
  } else {
    float hf[16], lf[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) split_tf32<R>(xa[j], scale, hf[j], lf[j]);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t off = sw128(r, half * 4 + q);
      *reinterpret_cast<float4*>(opAhi + off) = make_float4(hf[4 * q], hf[4 * q + 1], hf[4 * q + 2], hf[4 * q + 3]);
      *reinterpret_cast<float4*>(opAlo + off) = make_float4(lf[4 * q], lf[4 * q + 1], lf[4 * q + 2], lf[4 * q + 3]);
    }
  }

  // ---- B: column nn (stored K-major as operand row nn), same k-half
#pragma unroll
  for (int nn = r; nn < BN; nn += 128) {
    float xb[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) xb[i] = stgB[(half * 16 + i) * BN + nn];
#pragma unroll
    for (int i = 0; i < 16; ++i) fa.add(xb[i]);
    if constexpr (V == kFP16) {
      uint32_t hp[8], lp[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) split_f16_pair<R>(xb[2 * j], xb[2 * j + 1], scale, hp[j], lp[j]);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const uint32_t off = sw128(nn, sub * 4 + half * 2 + q);
        *reinterpret_cast<uint4*>(opBhi + off) = make_uint4(hp[4 * q], hp[4 * q + 1], hp[4 * q + 2], hp[4 * q + 3]);
        *reinterpret_cast<uint4*>(opBlo + off) = make_uint4(lp[4 * q], lp[4 * q + 1], lp[4 * q + 2], lp[4 * q + 3]);
      }
    } else {
      float hf[16], lf[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) split_tf32<R>(xb[j], scale, hf[j], lf[j]);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t off = sw128(nn, half * 4 + q);
        *reinterpret_cast<float4*>(opBhi + off) = make_float4(hf[4 * q], hf[4 * q + 1], hf[4 * q + 2], hf[4 * q + 3]);
        *reinterpret_cast<float4*>(opBlo + off) = make_float4(lf[4 * q], lf[4 * q + 1], lf[4 * q + 2], lf[4 * q + 3]);
      }
    }
  }
}

template <int V, int R, int BN>
__global__ void __launch_bounds__(TileCfg<BN>::NUM_THREADS, 1)
    tcec_gemm_kernel(const __grid_constant__ CUtensorMap tmA,  // A fp32 [m][k], box 32x128, SW128
                     const __grid_constant__ CUtensorMap tmB,  // B fp32 [k][n], box BNx32, no swizzle
                     const __grid_constant__ CUtensorMap tmC,  // C fp32 [m][n], box 32x32, SW128
                     const GemmShape shp, const float scale, const float inv_scale,
                     const FlagThresholds thr, uint32_t* __restrict__ flags) {
  using C = TileCfg<BN>;
  using VC = VarCfg<V>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* stg_full = bars;
  uint64_t* stg_empty = bars + C::NSTG;
  uint64_t* op_full = bars + 2 * C::NSTG;
  uint64_t* op_empty = op_full + C::NOP;
  uint64_t* p_full = op_empty + C::NOP;
  uint64_t* p_empty = p_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::NUM_BARS);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  // ---- tile coordinates (grouped rasterisation for L2 reuse of A and B)
  const int tiles_m = (shp.m + C::BM - 1) / C::BM;
  const int tiles_n = (shp.n + BN - 1) / BN;
  int tile_m, tile_n;
  {
    const int bid = blockIdx.x;
    const int per_group = shp.group_m * tiles_n;
    const int g = bid / per_group;
    const int first_m = g * shp.group_m;
    const int gsize = min(tiles_m - first_m, shp.group_m);
    const int in_g = bid - g * per_group;
    tile_m = first_m + in_g % gsize;
    tile_n = in_g / gsize;
  }
  const int m0 = tile_m * C::BM;
  const int n0 = tile_n * BN;
  const int nop = shp.num_op_stages;
  const int nstg = nop * VC::STG_PER_OP;
  const int de = shp.drain_every / 4;  // operand stages per drain interval (host: a multiple of 4 k-steps)

  // ---- one-time setup
  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch_desc(&tmA);
    sm100::tma_prefetch_desc(&tmB);
    sm100::tma_prefetch_desc(&tmC);
    for (int s = 0; s < C::NSTG; ++s) {
      sm100::mbar_init(&stg_full[s], 1);
      sm100::mbar_init(&stg_empty[s], C::NUM_SPLIT_WARPS);
    }
    for (int o = 0; o < C::NOP; ++o) {
      sm100::mbar_init(&op_full[o], C::NUM_SPLIT_WARPS);
      sm100::mbar_init(&op_empty[o], 1);
    }
    sm100::mbar_init(p_full, 1);
    sm100::mbar_init(p_empty, C::NUM_DRAIN_WARPS);
    sm100::fence_mbar_init();
  }
  if (warp == 1) sm100::tmem_alloc<C::TMEM_COLS>(tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t tmem_P = tmem_base;        // columns [0, BN)
  const uint32_t tmem_dC = tmem_base + BN;  // columns [BN, 2 BN)

  if (warp == 0) {
    // ===================== TMA producer: FP32 slices of A and B =====================
    if (lane == 0) {
      for (int st = 0; st < nstg; ++st) {
        const int s = st % C::NSTG;
        sm100::mbar_wait(&stg_empty[s], ((st / C::NSTG) & 1) ^ 1);
        uint8_t* dst = smem + C::OFF_STG + s * C::STG_BYTES;
        sm100::mbar_arrive_expect_tx(&stg_full[s], C::STG_BYTES);
        sm100::tma_load_2d(dst, &tmA, &stg_full[s], st * C::BK_STG, m0);
        sm100::tma_load_2d(dst + C::STG_A_BYTES, &tmB, &stg_full[s], n0, st * C::BK_STG);
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (single thread) =====================
    if (lane == 0) {
      constexpr uint32_t idesc = sm100::umma_idesc(VC::AB_FORMAT, C::BM, BN);
      for (int kb = 0; kb < nop; ++kb) {
        const int o = kb % C::NOP;
        sm100::mbar_wait(&op_full[o], (kb / C::NOP) & 1);
        sm100::tc_fence_after();
        const uint32_t op = sm100::smem_u32(smem + C::OFF_OP + o * C::OP_BYTES);
        const uint64_t a_hi = sm100::umma_desc_sw128_kmajor(op);
        const uint64_t a_lo = sm100::umma_desc_sw128_kmajor(op + C::OP_A_BYTES);
        const uint64_t b_hi = sm100::umma_desc_sw128_kmajor(op + 2 * C::OP_A_BYTES);
        const uint64_t b_lo = sm100::umma_desc_sw128_kmajor(op + 2 * C::OP_A_BYTES + C::OP_B_BYTES);
        // correction terms into dC, reference order per k-step: dA*B then A*dB
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint64_t adv = static_cast<uint64_t>(ks * 2);  // 32 bytes >> 4
          const uint32_t acc = (kb | ks) != 0;
          if constexpr (V == kFP16) {
            sm100::mma_f16(tmem_dC, a_lo + adv, b_hi + adv, idesc, acc);
            sm100::mma_f16(tmem_dC, a_hi + adv, b_lo + adv, idesc, 1u);
          } else {
            sm100::mma_tf32(tmem_dC, a_lo + adv, b_hi + adv, idesc, acc);
            sm100::mma_tf32(tmem_dC, a_hi + adv, b_lo + adv, idesc, 1u);
          }
        }
        // main term into P; a fresh P per drain interval must wait for the drain
        const bool first_in_interval = (kb % de) == 0;
        if (first_in_interval && kb > 0) {
          sm100::mbar_wait(p_empty, ((kb / de) - 1) & 1);
          sm100::tc_fence_after();
        }
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint64_t adv = static_cast<uint64_t>(ks * 2);
          const uint32_t acc = !(first_in_interval && ks == 0);
          if constexpr (V == kFP16) {
            sm100::mma_f16(tmem_P, a_hi + adv, b_hi + adv, idesc, acc);
          } else {
            sm100::mma_tf32(tmem_P, a_hi + adv, b_hi + adv, idesc, acc);
          }
        }
        sm100::mma_commit(&op_empty[o]);
        if ((kb % de) == de - 1 || kb == nop - 1) sm100::mma_commit(p_full);
      }
    }
  } else if (warp >= C::SPLIT_WARP0 && warp < C::SPLIT_WARP0 + C::NUM_SPLIT_WARPS) {
    // ===================== split warps: staging -> (hi, lo) operands =====================
    const int t = threadIdx.x - C::SPLIT_WARP0 * 32;
    FlagAcc fa;
    for (int kb = 0; kb < nop; ++kb) {
      const int o = kb % C::NOP;
      sm100::mbar_wait(&op_empty[o], ((kb / C::NOP) & 1) ^ 1);
      uint8_t* op = smem + C::OFF_OP + o * C::OP_BYTES;
#pragma unroll
      for (int sub = 0; sub < VC::STG_PER_OP; ++sub) {
        const int st = kb * VC::STG_PER_OP + sub;
        const int s = st % C::NSTG;
        sm100::mbar_wait(&stg_full[s], (st / C::NSTG) & 1);
        split_slice<V, R, BN>(smem + C::OFF_STG + s * C::STG_BYTES, op, sub, t, scale, fa);
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive(&stg_empty[s]);
      }
      sm100::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&op_full[o]);
    }
    flag_publish(fa, thr, flags);
    // the epilogue reuses the staging ring (see the drain warps' barrier)
    sm100::named_barrier_sync<1, 32 * (C::NUM_SPLIT_WARPS + C::NUM_DRAIN_WARPS)>();
  } else if (warp >= C::DRAIN_WARP0) {
    // ===================== drain + epilogue warps =====================
    constexpr int HALF = BN / 2;
    const int q = warp & 3;                       // TMEM lane quadrant
    const int h = (warp - C::DRAIN_WARP0) >> 2;   // column half
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    float acc[HALF];
#pragma unroll
    for (int j = 0; j < HALF; ++j) acc[j] = 0.0f;
    const int nintervals = (nop + de - 1) / de;
    for (int it = 0; it < nintervals; ++it) {
      sm100::mbar_wait(p_full, it & 1);
      sm100::tc_fence_after();
#pragma unroll
      for (int c = 0; c < HALF / 16; ++c) {
        uint32_t r[16];
        sm100::tmem_ld_32x32b_x16(tmem_P + lane_off + h * HALF + c * 16, r);
        sm100::tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[c * 16 + j] = __fadd_rn(acc[c * 16 + j], __uint_as_float(r[j]));
      }
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(p_empty);
    }
    // Epilogue: every MMA has completed (the last p_full commit follows them), and
    // with it every split warp's staging read; the named barrier states it for
    // tools that do not follow mbarrier / tcgen05.commit ordering (racecheck)
    sm100::named_barrier_sync<1, 32 * (C::NUM_SPLIT_WARPS + C::NUM_DRAIN_WARPS)>();
    bool nonfinite = false;
    uint8_t* stage = smem + C::OFF_STG + (warp - C::DRAIN_WARP0) * (HALF / C::EPI_BOX) * 4096;
#pragma unroll
    for (int b = 0; b < HALF / C::EPI_BOX; ++b) {
      uint8_t* box = stage + b * 4096;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t r[16];
        sm100::tmem_ld_32x32b_x16(tmem_dC + lane_off + h * HALF + b * 32 + c * 16, r);
        sm100::tmem_ld_wait();
        float o[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          // schemes.py:306-307: c = RN32(c + dC * 2^-s), one rounding of the exact sum
          o[j] = __fmaf_rn(__uint_as_float(r[j]), inv_scale, acc[b * 32 + c * 16 + j]);
          nonfinite |= !isfinite(o[j]);
        }
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          *reinterpret_cast<float4*>(box + sw128(lane, c * 4 + v)) =
              make_float4(o[4 * v], o[4 * v + 1], o[4 * v + 2], o[4 * v + 3]);
        }
      }
      sm100::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        sm100::tma_store_2d(&tmC, box, n0 + h * HALF + b * 32, m0 + q * 32);
        sm100::tma_store_commit();
      }
    }
    if (lane == 0) sm100::tma_store_wait0();
    if (flags != nullptr) {
      // schemes.py:369-371: a non-finite output sets saw_overflow
      if (__any_sync(0xFFFFFFFFu, nonfinite) && lane == 0) atomicOr(flags, kFlagOverflow);
    }
    sm100::tc_fence_before();
  }

  __syncthreads();
  if (warp == 1) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc<C::TMEM_COLS>(tmem_base);
  }
}

// Standalone elementwise split (tests, exhaustive parity, diagnostics).
// hi / lo are written as FP32 values (FP16 values widened exactly).
template <int V, int R>
__global__ void tcec_split_kernel(const float* __restrict__ x, int64_t count, float scale,
                                  FlagThresholds thr, float* __restrict__ hi,
                                  float* __restrict__ lo, uint32_t* __restrict__ flags) {
  FlagAcc fa;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x * 2;
  for (int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 2; i < count;
       i += stride) {
    const float x0 = x[i];
    const float x1 = (i + 1 < count) ? x[i + 1] : 0.0f;
    float h0, h1, l0, l1;
    if constexpr (V == kFP16) {
      uint32_t hp, lp;
      split_f16_pair<R>(x0, x1, scale, hp, lp);
      unpack_f16x2(hp, h0, h1);
      unpack_f16x2(lp, l0, l1);
    } else {
      split_tf32<R>(x0, scale, h0, l0);
      split_tf32<R>(x1, scale, h1, l1);
    }
    fa.add(x0);
    hi[i] = h0;
    lo[i] = l0;
    if (i + 1 < count) {
      fa.add(x1);
      hi[i + 1] = h1;
      lo[i + 1] = l1;
    }
  }
  flag_publish(fa, thr, flags);
}

}  // namespace tcec
