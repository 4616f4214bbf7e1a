// split.cuh -- the FP32 -> (hi, lo) split of the error-corrected GEMM, as
// device functions shared by the standalone split kernel and the split warps
// of the fused GEMM (so the exhaustive split parity test covers the exact
// arithmetic the GEMM runs).
//
// Semantics follow the reference split (splitting.py:114-122, _split_arrays):
//   hi = round(x, fmt, mode)
//   lo = round((x - hi) * 2^s, fmt, mode),   lo = 0 where hi overflowed
// with fmt/mode/s from SplitScheme (splitting.py:43-67): scaled_halfhalf =
// FP16, RN, s = 11; tf32tf32 = TF32, RNA, s = 0.  The carrier subtraction
// x - hi is exact in FP32 for every finite FP32 x (both operands lie on the
// FP32 grid and the difference is below hi's half-ulp), and the power-of-two
// scale is exact, so FP32 arithmetic reproduces the reference's float64
// carrier bit for bit.  No FTZ anywhere: build without --use_fast_math.
#pragma once

#include <cstdint>
#include <cstring>
#include <cuda_fp16.h>

#include "sm100.cuh"

namespace tcec {

enum Variant : int { kFP16 = 0, kTF32 = 1 };
enum Rounding : int { kRN = 0, kRNA = 1, kRZ = 2 };

constexpr uint32_t kFlagOverflow = 1u;
constexpr uint32_t kFlagOutOfRange = 2u;
constexpr uint32_t kFlagNonfiniteInput = 4u;

// ------------------------------------------------------------------ FP16 --
// cvt.{rn,rz}.f16x2.f32: IEEE conversion with gradual underflow; RN overflows
// to inf (formats.py:140); RZ saturates to 65504 (formats.py:137-138), which
// needs .satfinite (plain cvt.rz returns inf for inputs near FLT_MAX).
// 0xFFFF in each half of a packed FP16 pair that is not +-inf (NaN included),
// 0 where it is: abs.f16x2 folds into the HSET2 compare.
__device__ __forceinline__ uint32_t f16x2_finite_mask(uint32_t h) {
  uint32_t m;
  asm("{\n"
      ".reg .b32 a, b;\n"
      "abs.f16x2 a, %1;\n"
      "mov.b32 b, 0x7c007c00;\n"
      "set.neu.u32.f16x2 %0, a, b;\n"
      "}"
      : "=r"(m)
      : "r"(h));
  return m;
}

template <int R>
__device__ __forceinline__ uint32_t cvt_f16x2(float lo_elem, float hi_elem) {
  uint32_t d;
  if constexpr (R == kRZ) {
    asm("cvt.rz.satfinite.f16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi_elem), "f"(lo_elem));
  } else {
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi_elem), "f"(lo_elem));
  }
  return d;
}

__device__ __forceinline__ void unpack_f16x2(uint32_t p, float& a, float& b) {
  __half2 h = *reinterpret_cast<__half2*>(&p);
  a = __low2float(h);
  b = __high2float(h);
}

// Two consecutive elements -> packed (hi, lo) half2 words, element 0 in the
// low half (lower address once stored) -- the split warps' arithmetic: the
// residual (x - hi) 2^s as one fma.rn.f32x2 (both products exact, one rounding
// of a representable value), and splitting.py:119-121 (lo = 0 where hi
// overflowed) as one packed compare on |hi| and a mask: the residual there is
// -+inf, so only those halves change; a NaN input keeps its NaN lo.
template <int R>
__device__ __forceinline__ void split_pair16(float x0, float x1, float scale, uint32_t& hw,
                                             uint32_t& lw) {
  constexpr bool kFix = R != kRZ;  // RZ saturates: hi never overflows
  hw = cvt_f16x2<R>(x0, x1);
  float h0, h1, r0, r1;
  unpack_f16x2(hw, h0, h1);
  sm100::residual_x2(x0, x1, h0, h1, scale, r0, r1);
  lw = cvt_f16x2<R>(r0, r1);
  if constexpr (kFix) lw &= f16x2_finite_mask(hw);
}

template <int R>
__device__ __forceinline__ void split_f16_pair(float x0, float x1, float scale, uint32_t& hi,
                                               uint32_t& lo) {
  split_pair16<R>(x0, x1, scale, hi, lo);
}

// ------------------------------------------------------------------ TF32 --
// TF32 keeps FP32's exponent field and 10 fraction bits: rounding is an
// integer operation on the low 13 bits (formats.py:114-142 with man_bits=10,
// min_normal_exp=-126: FP32 subnormals round on the same 2^-136 grid).  A
// carry out of the fraction bumps the exponent; out of 0xFE it yields inf,
// which is the reference's RN/RNA overflow.  RZ cannot exceed max_finite.
template <int R>
__device__ __forceinline__ uint32_t tf32_round_bits(uint32_t u) {
  if constexpr (R == kRNA) {
    return (u + 0x1000u) & 0xFFFFE000u;
  } else if constexpr (R == kRN) {
    return (u + 0x0FFFu + ((u >> 13) & 1u)) & 0xFFFFE000u;
  } else {
    return u & 0xFFFFE000u;
  }
}

// The same rounding without clearing the low 13 bits (value whose top 19 bits
// equal tf32_round_bits); for operands consumed by the tensor core only.
template <int R>
__device__ __forceinline__ uint32_t tf32_carry_bits(uint32_t u) {
  if constexpr (R == kRNA) {
    return u + 0x1000u;
  } else if constexpr (R == kRN) {
    return u + 0x0FFFu + ((u >> 13) & 1u);
  } else {
    return u;
  }
}

// One element, the split warps' arithmetic (split_chunk in tcec_gemm2.cuh runs
// it on pairs with sub.rn.f32x2): lo's rounding carry on the exact residual,
// 0 where x - hi is infinite, i.e. where hi overflowed (splitting.py:119-121);
// the low 13 bits are cleared here (the tensor core ignores them in the GEMM).
// TF32 has no residual scale (tf32tf32: s = 0).
template <int R>
__device__ __forceinline__ void split_tf32(float x, float scale, float& hi, float& lo) {
  (void)scale;
  const uint32_t hb = tf32_round_bits<R>(__float_as_uint(x));
  const float r = __fsub_rn(x, __uint_as_float(hb));
  const uint32_t lb = (R != kRZ && isinf(r)) ? 0u : tf32_carry_bits<R>(__float_as_uint(r));
  hi = __uint_as_float(hb);
  lo = __uint_as_float(lb & 0xFFFFE000u);
}

// ----------------------------------------------------------------- flags --
// RunFlags of the split (schemes.py:237-241 via splitting.py:187-215):
//   out_of_range: some nonzero x with e_v + s <= -24 or e_v > 15   (FP16)
//                 some nonzero x with e_v < -126 (FP32 subnormal)  (TF32)
//   overflow:     some hi = +-inf.
// Tracked per thread as min over (|bits| * 2 - 2) (zero maps to 0xFFFFFFFE,
// so the min is the smallest nonzero magnitude) and max over |x|.  Inf / NaN
// inputs (rejected by the reference, schemes.py:166-167) raise their own bit.
struct FlagAcc {
  uint32_t mn = 0xFFFFFFFFu;
  float mx = 0.0f;
  __device__ __forceinline__ void add(float x) {
    const uint32_t u = __float_as_uint(x);
    mn = min(mn, u + u - 2u);
    // max.NaN propagates NaN so that non-finite inputs are caught too
    asm("max.NaN.f32 %0, %0, %1;" : "+f"(mx) : "f"(fabsf(x)));
  }
};

__host__ __device__ inline float bits_to_float(uint32_t u) {
  float f;
  memcpy(&f, &u, sizeof(f));
  return f;
}

struct FlagThresholds {
  uint32_t tiny2;   // (bits of the smallest in-range magnitude) * 2 - 2
  float big;        // |x| >= big -> out of range (FP16 only; +inf for TF32)
  float ovf;        // |x| >= ovf -> hi overflows (+inf when the mode saturates)
};

__host__ __device__ inline FlagThresholds flag_thresholds(int variant, int rounding,
                                                         int scale_log2) {
  FlagThresholds t;
  const float inf = bits_to_float(0x7F800000u);
  if (variant == kFP16) {
    // e_v + s <= -24  <=>  |x| < 2^(-23 - s)
    const int e = -23 - scale_log2;
    const uint32_t bits = static_cast<uint32_t>(e + 127) << 23;
    t.tiny2 = bits * 2u - 2u;
    t.big = 65536.0f;
    t.ovf = (rounding == kRZ) ? inf : 65520.0f;
  } else {
    t.tiny2 = 0x00800000u * 2u - 2u;
    t.big = inf;
    t.ovf = (rounding == kRZ) ? inf : bits_to_float(0x7F7FF000u);
  }
  return t;
}

// RunFlags of a plain conversion (schemes.py:227-232, _plain_conversion_flags):
// overflow = some converted value is inf; out_of_range = overflow or some
// nonzero x converts to 0.  FP16 RN: x vanishes iff |x| <= 2^-25 (the tie
// rounds to even zero); TF32 RNA: iff |x| < 2^-137 (the tie rounds away).
__host__ __device__ inline FlagThresholds plain_thresholds(int variant, int rounding) {
  FlagThresholds t;
  const float inf = bits_to_float(0x7F800000u);
  if (variant == kFP16) {
    const uint32_t first_kept = ((static_cast<uint32_t>(-25 + 127) << 23) + 1u);  // next above 2^-25
    t.tiny2 = rounding == kRZ ? ((static_cast<uint32_t>(-24 + 127) << 23) * 2u - 2u)
                              : first_kept * 2u - 2u;
    t.ovf = (rounding == kRZ) ? inf : 65520.0f;
  } else {
    const uint32_t first_kept = rounding == kRZ ? 0x2000u : (rounding == kRNA ? 0x1000u : 0x1001u);
    t.tiny2 = first_kept * 2u - 2u;
    t.ovf = (rounding == kRZ) ? inf : bits_to_float(0x7F7FF000u);
  }
  t.big = t.ovf;  // an overflowing conversion is also out of range
  return t;
}

__device__ __forceinline__ uint32_t flag_bits(const FlagAcc& f, const FlagThresholds& t) {
  uint32_t fl = 0;
  if (!(f.mx <= 3.402823466e38f)) return kFlagNonfiniteInput;  // inf or NaN input
  if (f.mn < t.tiny2 || f.mx >= t.big) fl |= kFlagOutOfRange;
  if (f.mx >= t.ovf) fl |= kFlagOverflow;
  return fl;
}

// Warp-reduce the accumulator and publish (one atomic per warp, only when set).
__device__ __forceinline__ void flag_publish(const FlagAcc& f, const FlagThresholds& t,
                                             uint32_t* flags) {
  if (flags == nullptr) return;
  const uint32_t fl = __reduce_or_sync(0xFFFFFFFFu, flag_bits(f, t));
  if (fl != 0 && (threadIdx.x & 31) == 0) atomicOr(flags, fl);
}

}  // namespace tcec
