/*
 * tcec.h -- C ABI of the B200 (sm_100a) error-corrected single-precision GEMM
 * (Ootomo & Yokota, arXiv 2203.03341: FP16-TCEC and TF32-TCEC).
 *
 * This is the drop-in boundary for the reference's GEMM entry point
 * (reference: /root/reference/pkg/src/tcgemm/schemes.py).  Plain pointers and
 * sizes only; no framework types.  Every entry point is reentrant and
 * stream-ordered, and works on whichever device is current (per-device state:
 * the shared-memory opt-in and occupancy are cached per kernel and device, the
 * workspaces come from that device's stream-ordered pool); results are
 * deterministic (no atomics in any reduction of C).
 *
 * Library: paper_2203_03341_b200/libtcec.so (nvcc, -gencode arch=compute_100a,code=sm_100a).
 */
#ifndef TCEC_H_
#define TCEC_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Variants: the two corrected3 schemes of the reference registry
 * (schemes.py:135-136 "corrected3_halfhalf" / "corrected3_tf32";
 * split recipes splitting.py:70-79 scaled_halfhalf() / tf32tf32()). */
#define TCEC_FP16 0 /* FP16-TCEC: hi/lo in FP16, residual scaled by 2^11 */
#define TCEC_TF32 1 /* TF32-TCEC: hi/lo in TF32, no residual scaling      */

/* Split rounding modes (formats.py:43-55 RoundingMode). */
#define TCEC_ROUND_DEFAULT (-1) /* RN for FP16, RNA for TF32 (splitting.py:50-59) */
#define TCEC_ROUND_RN 0
#define TCEC_ROUND_RNA 1 /* TF32 only */
#define TCEC_ROUND_RZ 2

/* Device flag bits (RunFlags, schemes.py:140-143). */
#define TCEC_FLAG_OVERFLOW 1u     /* some hi overflowed, or some output non-finite */
#define TCEC_FLAG_OUT_OF_RANGE 2u /* some input outside the split's representable band */
#define TCEC_FLAG_NONFINITE_INPUT 4u /* some input is inf or NaN (the reference raises) */

/* Product schedules (tcec_opts.scheme).  CORRECTED3 is the accelerated path;
 * the others run the reference's comparator schemes on the tensor core so the
 * paper's ablations can be reproduced on hardware (they use split-once mode):
 *   CORRECTED3_DD  corrected3 plus the dA*dB chain in a separate accumulator
 *                  (schemes.py:308-313, delta_term_ablation :422-451)
 *   TC_PLAIN       tc_plain_fp16 / tc_plain_tf32: one product of the inputs
 *                  converted RN (FP16) / RNA (TF32) (schemes.py:343-351)
 *   INUNIT4        markidis4 / corrected4 with the hardware's terminal
 *                  rounding: four products in one accumulator, unscaled split
 *                  (schemes.py:99-117, :352-364)
 *   INUNIT4_RN     corrected4_rn: the same four products with an RN terminal,
 *                  emulated: each product accumulates one block of drain_k
 *                  in its own tensor-memory accumulator, and the blocks are
 *                  added in term order into an FP32 round-to-nearest sum on
 *                  the CUDA cores (mma.py:84-85).  drain_k is the reference's
 *                  block_k here: 0 = 16, else a multiple of the MMA k-step
 *                  (16 FP16, 8 TF32).  */
#define TCEC_SCHEME_CORRECTED3 0
#define TCEC_SCHEME_CORRECTED3_DD 1
#define TCEC_SCHEME_TC_PLAIN 2
#define TCEC_SCHEME_INUNIT4 3
#define TCEC_SCHEME_INUNIT4_RN 4

/* Status codes. */
#define TCEC_OK 0
#define TCEC_ERR_ARG (-1)         /* bad shape / leading dimension / option      */
#define TCEC_ERR_ALIGN (-2)       /* pointer or leading dimension not 16-B aligned */
#define TCEC_ERR_UNSUPPORTED (-3) /* variant/rounding/drain combination not built  */
#define TCEC_ERR_CUDA (-4)        /* CUDA runtime / driver error                   */
#define TCEC_ERR_ARCH (-5)        /* current device is not sm_100                  */

typedef struct tcec_opts {
  /* Split rounding (TCEC_ROUND_*); replaces SplitScheme.rounding. */
  int32_t split_rounding;
  /* log2 of the residual scale: -1 = scheme default (11 FP16, 0 TF32);
   * 0 with FP16 is the unscaled markidis_halfhalf split (splitting.py:70-71). */
  int32_t scale_log2;
  /* Drain interval of the main-term partial in k -- the reference's
   * MmaConfig.block_k (mma.py:34, schemes.py:300-304): 0 = default (128 for
   * FP16, 64 for TF32); otherwise a positive multiple of the MMA k-step (16 for
   * FP16, 8 for TF32), e.g. 16 = the reference's default schedule.  The narrow
   * tiles (block_n 128 / 192) need a multiple of 4 k-steps.
   * TCEC_SCHEME_INUNIT4_RN: the block of each drained product (see above). */
  int32_t drain_k;
  /* Output tile width: 0 = automatic (the CTA-pair 256 x 256 tile, or below
   * 8 waves of those the width among 256 / 192 / 128 / 64 with the fewest
   * cost-weighted waves; same results); 192 / 128 / 64 = CTA-pair 256 x 192 /
   * 256 x 128 / 256 x 64 tile with the split A operand in tensor memory (128
   * with kernel_variant = 1: the single-CTA 128 x 128 kernel). */
  int32_t block_n;
  /* Tile rasterisation group along m in 128-row tiles: 0 = default (8). */
  int32_t group_m;
  /* Where the hi/lo split runs: 0 = default, 1 = fused into the GEMM's TMA
   * pipeline (FP32 tiles split in shared memory), 2 = split once per input
   * element in a separate HBM pass, then a three-product GEMM over the
   * pre-split operands (workspace 2(m + n)k operand elements, stream-ordered
   * allocation).  Results are bit-identical. */
  int32_t split_mode;
  /* Product schedule, TCEC_SCHEME_* (0 = corrected3). */
  int32_t scheme;
  /* tcec_sgemm_host only: number of row / column blocks of C that the host
   * buffers are streamed in (0 = automatic, at most 8 each). */
  int32_t host_row_blocks;
  int32_t host_col_blocks;
  /* Split-K parts (corrected3, fused split): 0 / 1 = off.  S > 1 splits k into
   * S contiguous parts computed as separate persistent-kernel units; each part
   * keeps its own main-term sum and dC, and a second kernel combines them in
   * part order, C = RN(sum c_p + (sum dC_p) 2^-s) -- deterministic, but not the
   * single-pass rounding sequence, so results match the reference within the
   * GEMM tolerance instead of bit for bit.  For products with fewer output
   * tiles than SMs (small m x n, long k).  -1 = automatic: S = min(8, idle
   * pairs per tile, k / 1024 (FP16) or k / 512 (TF32)) when the tiles fill at
   * most half of the CTA pairs, else off. */
  int32_t split_k;
  /* Kernel: 0 = automatic (persistent with lock-step waves for products of
   * >= 8 waves of 256 x 256 tiles, else per-tile); 1 = the single-CTA kernel
   * (block_n 128 only); 2 = persistent; 3 = persistent with lock-step waves;
   * 4 = per-tile (for a kernel sharing the GPU with other work); 6 =
   * persistent with the split shared through an L2-resident ring (each wave's
   * A / B k-slices split once by the whole grid; corrected3, block_n 256, fused
   * split; needs every SM -- not for a GPU shared with other kernels; measured
   * slower than the default, so only in libraries built with `make RING=1`,
   * TCEC_ERR_UNSUPPORTED otherwise).
   * Results are bit-identical across kernels. */
  int32_t kernel_variant;
  int32_t reserved[2];
} tcec_opts;

/* Library version (major * 10000 + minor * 100 + patch). */
int tcec_version(void);

/* Human-readable text for a status code. */
const char* tcec_status_str(int status);

/* C = A * B with the corrected3 scheme.  Replaces
 *   tcgemm.gemm(a, b, SCHEMES_BY_NAME["corrected3_halfhalf" | "corrected3_tf32"], cfg)
 * (schemes.py:317-373; core _corrected_core :265-314).
 * A: m x k, row-major, leading dimension lda (>= k) -- device pointer
 * B: k x n, row-major, leading dimension ldb (>= n) -- device pointer
 * C: m x n, row-major, leading dimension ldc (>= n) -- device pointer, written
 * Pointers must be 16-byte aligned and lda/ldb/ldc multiples of 4 (TMA).
 * opts may be NULL (defaults).  d_flags (device uint32, may be NULL) is OR-ed
 * with TCEC_FLAG_* bits (the caller zeroes it).  stream is a cudaStream_t.
 * k == 0 writes zeros; m == 0 or n == 0 is a no-op. */
int tcec_sgemm(int variant, int64_t m, int64_t n, int64_t k, const float* A, int64_t lda,
               const float* B, int64_t ldb, float* C, int64_t ldc, const tcec_opts* opts,
               uint32_t* d_flags, void* stream);

/* Same computation, with C stored to each of the n_c (1..8) destinations C[0..n_c-1]
 * (same ldc) by the same TMA-store epilogue -- the fused all-gather of the
 * row-sharded multi-GPU GEMM: C[d] is this rank's slab inside rank d's full C
 * (peer memory mapped into this GPU's address space, e.g. CUDA IPC / symmetric
 * memory over NVLink), so the gather overlaps the GEMM tile by tile and needs no
 * separate collective.  Default kernel options only (pair kernel, fused split,
 * corrected3); the caller synchronises the ranks before reading the full C. */
int tcec_sgemm_multi(int variant, int64_t m, int64_t n, int64_t k, const float* A, int64_t lda,
                     const float* B, int64_t ldb, float* const* C, int n_c, int64_t ldc,
                     const tcec_opts* opts, uint32_t* d_flags, void* stream);

/* Same computation on HOST buffers (the numpy-facing binding): copies A and B
 * to the device, runs tcec_sgemm, copies C back and synchronises the stream.
 * C is produced in row x column blocks so that the GEMM starts after the first
 * block of A and of B arrive and the download overlaps the uploads.
 * Host buffers may be pageable; pinned buffers copy faster.  h_flags may be
 * NULL.  Row-major, leading dimensions as above (no alignment requirement). */
int tcec_sgemm_host(int variant, int64_t m, int64_t n, int64_t k, const float* A, int64_t lda,
                    const float* B, int64_t ldb, float* C, int64_t ldc, const tcec_opts* opts,
                    uint32_t* h_flags, void* stream);

/* Frees the device copies of A, B and C that tcec_sgemm_host keeps cached on
 * the current device between calls (its streams and events stay). */
int tcec_host_release(void);

/* Elementwise split of count FP32 values (splitting.py:114-122 _split_arrays,
 * split_matrix :139-147): hi and lo are written as FP32 values (FP16 values
 * widened exactly).  d_flags as above (classify_array :187-215).  Device
 * pointers, 4-byte aligned. */
int tcec_split(int variant, int rounding, int scale_log2, const float* X, int64_t count,
               float* hi, float* lo, uint32_t* d_flags, void* stream);

/* Exhaustive split census over all 2^23 FP32 mantissas (one thread each),
 * added into d_counts (device, 24 x uint64, caller-zeroed):
 *   TCEC_CENSUS_KEPT_LENGTH: histogram of the kept mantissa length of the
 *     markidis_halfhalf split at e_v = 0 with `rounding` (RN / RNA / RZ) --
 *     analysis.py:138-165 exhaustive_length_distribution (split-stats);
 *   TCEC_CENSUS_UNDERFLOW: counts[0] = residuals below the FP16 subnormals,
 *     counts[1] = residuals below the FP16 normals, for inputs of exponent e_v
 *     split with FP16 RZ -- the exhaustive form of analysis.py:106-135
 *     empirical_underflow (underflow). */
#define TCEC_CENSUS_KEPT_LENGTH 0
#define TCEC_CENSUS_UNDERFLOW 1
int tcec_split_census(int kind, int rounding, int e_v, unsigned long long* d_counts, void* stream);

/* Number of kernel launches issued by this library since load (diagnostic). */
uint64_t tcec_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* TCEC_H_ */
