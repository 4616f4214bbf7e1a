// tcec_census.cuh -- exhaustive split statistics on the GPU.
//
// The reference enumerates every 23-bit FP32 mantissa on the CPU with numpy
// (analysis.py:138-165 exhaustive_length_distribution, 2^23 values) and samples
// the residual-underflow rates by Monte Carlo (analysis.py:106-135
// empirical_underflow).  Here one thread per mantissa does both exhaustively:
//
//   kind 0 (kept length): v = 1 + m 2^-23 (e_v = 0), markidis_halfhalf split
//     (FP16, unscaled) with the given rounding, kept length from the
//     reconstruction error (splitting.py:157-161): 23 when exact, else
//     clamp(-frexp_exp(|v - (hi + lo)|), 0, 23)  -> 24-bin histogram.
//   kind 1 (underflow): v = (1 + m 2^-23) 2^e_v, hi = FP16 RZ (saturating,
//     formats.py:137-138), d = v - hi exactly; position = binade of d (or
//     e_v - 24 when d = 0); counts[0] += position < -24 (underflow), counts[1]
//     += position < -14 (underflow or gradual underflow).
//
// FP16 rounding of these values: cvt.rn / cvt.rz.satfinite for RN / RZ; RNA
// (no conversion instruction) by rounding the FP32 fraction to 10 bits, which is
// exact here because every value is either FP16-normal or a multiple of 2^-23
// below 2^-14 (at most 9 significant bits, representable as an FP16 subnormal).
#pragma once

#include <cstdint>
#include <cuda_fp16.h>

#include "split.cuh"

namespace tcec {

template <int R>
__device__ __forceinline__ float census_round_f16(float x) {
  if constexpr (R == kRNA) {
    return __uint_as_float(tf32_round_bits<kRNA>(__float_as_uint(x)));
  } else {
    const uint32_t p = cvt_f16x2<R>(x, 0.0f);
    float a, b;
    unpack_f16x2(p, a, b);
    return a;
  }
}

template <int KIND, int R>
__global__ void __launch_bounds__(256) tcec_census_kernel(int e_v, unsigned long long* counts) {
  __shared__ unsigned long long hist[24];
  if (threadIdx.x < 24) hist[threadIdx.x] = 0;
  __syncthreads();
  const uint32_t m = blockIdx.x * blockDim.x + threadIdx.x;  // grid covers exactly 2^23
  if constexpr (KIND == 0) {
    const float v = __uint_as_float(0x3F800000u | m);  // 1 + m 2^-23
    const float hi = census_round_f16<R>(v);
    const float lo = census_round_f16<R>(v - hi);    // v - hi exact in FP32
    const double err = fabs(static_cast<double>(v) - (static_cast<double>(hi) + lo));
    int len = 23;
    if (err != 0.0) {
      int e2;
      frexp(err, &e2);
      len = min(23, max(0, -e2));
    }
    atomicAdd(&hist[len], 1ull);
  } else {
    const double v = ldexp(1.0 + ldexp(static_cast<double>(m), -23), e_v);
    const float vf = static_cast<float>(v);  // exact whenever v is an FP32 value
    const double hi = static_cast<double>(census_round_f16<kRZ>(vf));
    const double d = v - hi;
    int pos;
    if (d != 0.0) {
      int e2;
      frexp(fabs(d), &e2);
      pos = e2 - 1;
    } else {
      pos = e_v - 24;
    }
    if (pos < -24) atomicAdd(&hist[0], 1ull);
    if (pos < -14) atomicAdd(&hist[1], 1ull);
  }
  __syncthreads();
  if (threadIdx.x < 24 && hist[threadIdx.x] != 0) atomicAdd(&counts[threadIdx.x], hist[threadIdx.x]);
}

}  // namespace tcec
