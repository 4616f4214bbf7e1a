// tcec_capi.cu -- host side of the C ABI declared in include/tcec.h.
//
// Validation mirrors the reference's gemm() contract (schemes.py:163-171,
// :327-330): shape errors are reported, numerical anomalies only raise flags.
// Tensor maps are encoded per call through the driver entry point obtained
// from the runtime (no link-time libcuda dependency).
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <set>
#include <utility>

#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include "tcec.h"
#include "tcec_gemm.cuh"
#include "tcec_gemm2.cuh"
#include "tcec_gemm4.cuh"
#include "tcec_gemm5.cuh"
#include "tcec_presplit.cuh"
#ifdef TCEC_WITH_RING  // kernel_variant 6, measured slower: built with `make RING=1` only
#include "tcec_ring.cuh"
#endif
#include "tcec_census.cuh"

namespace {

std::atomic<uint64_t> g_launches{0};

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;
int g_encode_status = TCEC_ERR_CUDA;

int get_encoder() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess && fn != nullptr) {
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
      g_encode_status = TCEC_OK;
    }
  });
  return g_encode_status;
}

int check_arch() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return TCEC_ERR_CUDA;
  int major = 0, minor = 0;
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess)
    return TCEC_ERR_CUDA;
  return (major == 10 && minor == 0) ? TCEC_OK : TCEC_ERR_ARCH;
}

// 2-D fp32 tensor map over a row-major [outer][inner] matrix.
int make_tmap(CUtensorMap* tm, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld_elems,
              uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle swz) {
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {ld_elems * sizeof(float)};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = g_encode(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims,
                              strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? TCEC_OK : TCEC_ERR_CUDA;
}

// 2-D tensor map over a row-major [outer][inner] operand workspace (FP16 or
// 32-bit elements), 128-byte swizzled boxes of 128 bytes x box_outer.
int make_tmap_op(CUtensorMap* tm, const void* ptr, CUtensorMapDataType dt, uint32_t esize,
                 uint64_t inner, uint64_t outer, uint64_t ld_elems, uint32_t box_outer) {
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {ld_elems * esize};
  const cuuint32_t box[2] = {128u / esize, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = g_encode(tm, dt, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? TCEC_OK : TCEC_ERR_CUDA;
}

// Keep freed blocks cached in the device's stream-ordered pool between calls
// (workspaces of the host path and of the split-once mode).
void keep_pool(int dev) {
  static std::once_flag pool_once[64];
  if (dev < 0 || dev >= 64) return;
  std::call_once(pool_once[dev], [dev] {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  });
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Extra destinations of C (tcec_sgemm_multi): the pair kernel stores every
// output box to each of them as well.
struct ExtraC {
  float* c[tcec::kMaxExtraC];
  int count;
};

// Dynamic shared-memory opt-in, once per (kernel, device): the attribute
// belongs to the device context, so a process driving several GPUs sets it on
// each of them.
template <typename K>
cudaError_t smem_optin(K kern, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const auto key = std::make_pair(reinterpret_cast<const void*>(kern), dev);
  std::lock_guard<std::mutex> lk(mu);
  if (done.count(key)) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.insert(key);
  return e;
}

template <int V, int R, int BN>
int launch_gemm(int64_t m, int64_t n, int64_t k, const float* A, int64_t lda, const float* B,
                int64_t ldb, float* C, int64_t ldc, int scale_log2, int drain_every, int group_m,
                uint32_t* d_flags, cudaStream_t stream) {
  using Cfg = tcec::TileCfg<BN>;
  using VC = tcec::VarCfg<V>;
  CUtensorMap tmA, tmB, tmC;
  int st;
  if ((st = make_tmap(&tmA, A, k, m, lda, Cfg::BK_STG, Cfg::BM, CU_TENSOR_MAP_SWIZZLE_128B)))
    return st;
  if ((st = make_tmap(&tmB, B, n, k, ldb, BN, Cfg::BK_STG, CU_TENSOR_MAP_SWIZZLE_NONE))) return st;
  if ((st = make_tmap(&tmC, C, n, m, ldc, Cfg::EPI_BOX, Cfg::EPI_BOX, CU_TENSOR_MAP_SWIZZLE_128B)))
    return st;

  auto kern = tcec::tcec_gemm_kernel<V, R, BN>;
  const cudaError_t attr_err = smem_optin(kern, Cfg::SMEM_BYTES);
  if (attr_err != cudaSuccess) return TCEC_ERR_CUDA;

  tcec::GemmShape shp;
  shp.m = static_cast<int32_t>(m);
  shp.n = static_cast<int32_t>(n);
  shp.k = static_cast<int32_t>(k);
  shp.num_op_stages = static_cast<int32_t>((k + VC::BK_OP - 1) / VC::BK_OP);
  shp.drain_every = drain_every;
  shp.group_m = group_m;
  const float scale = ldexpf(1.0f, scale_log2);
  const float inv_scale = ldexpf(1.0f, -scale_log2);
  const tcec::FlagThresholds thr = tcec::flag_thresholds(V, R, scale_log2);
  const int64_t tiles = ((m + Cfg::BM - 1) / Cfg::BM) * ((n + BN - 1) / BN);
  kern<<<static_cast<unsigned>(tiles), Cfg::NUM_THREADS, Cfg::SMEM_BYTES, stream>>>(
      tmA, tmB, tmC, shp, scale, inv_scale, thr, d_flags);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError() == cudaSuccess ? TCEC_OK : TCEC_ERR_CUDA;
}

template <int V, int R>
int launch_gemm_pair(int64_t m, int64_t n, int64_t k, const float* A, int64_t lda, const float* B,
                     int64_t ldb, float* C, int64_t ldc, int scale_log2, int drain_every,
                     int group_m, const ExtraC* ex, uint32_t* d_flags, cudaStream_t stream) {
  using Cfg = tcec::PairCfg<V>;
  using VC = tcec::VarCfg<V>;
  CUtensorMap tmA, tmB, tmC;
  int st;
  if ((st = make_tmap(&tmA, A, k, m, lda, Cfg::BK_STG, Cfg::BM, CU_TENSOR_MAP_SWIZZLE_128B)))
    return st;
  if ((st = make_tmap(&tmB, B, n, k, ldb, 32, Cfg::BK_STG, CU_TENSOR_MAP_SWIZZLE_128B))) return st;
  if ((st = make_tmap(&tmC, C, n, m, ldc, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B))) return st;
  tcec::CDests cx;
  memset(&cx, 0, sizeof(cx));
  cx.count = ex ? ex->count : 0;
  for (int d = 0; d < cx.count; ++d)
    if ((st = make_tmap(&cx.m[d], ex->c[d], n, m, ldc, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B)))
      return st;

  auto kern = tcec::tcec_gemm_pair_kernel<V, R>;
  const cudaError_t attr_err = smem_optin(kern, Cfg::SMEM_BYTES);
  if (attr_err != cudaSuccess) return TCEC_ERR_CUDA;

  tcec::GemmShape shp;
  shp.m = static_cast<int32_t>(m);
  shp.n = static_cast<int32_t>(n);
  shp.k = static_cast<int32_t>(k);
  shp.num_op_stages = static_cast<int32_t>((k + VC::BK_OP - 1) / VC::BK_OP);
  shp.drain_every = drain_every;
  shp.group_m = group_m;
  const float scale = ldexpf(1.0f, scale_log2);
  const float inv_scale = ldexpf(1.0f, -scale_log2);
  const tcec::FlagThresholds thr = tcec::flag_thresholds(V, R, scale_log2);
  const int64_t pairs = ((m + 2 * Cfg::BM - 1) / (2 * Cfg::BM)) * ((n + Cfg::BN - 1) / Cfg::BN);
  kern<<<static_cast<unsigned>(2 * pairs), Cfg::NUM_THREADS, Cfg::SMEM_BYTES, stream>>>(
      tmA, tmB, tmC, cx, shp, scale, inv_scale, thr, d_flags);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError() == cudaSuccess ? TCEC_OK : TCEC_ERR_CUDA;
}

template <int V, int R, int BN, int NOP>
int launch_gemm_ts(int64_t m, int64_t n, int64_t k, const float* A, int64_t lda, const float* B,
                   int64_t ldb, float* C, int64_t ldc, int scale_log2, int drain_every,
                   int group_m, uint32_t* d_flags, cudaStream_t stream) {
  using Cfg = tcec::TsCfg<V, BN, NOP>;
  using VC = tcec::VarCfg<V>;
  CUtensorMap tmA, tmB, tmC;
  int st;
  if ((st = make_tmap(&tmA, A, k, m, lda, Cfg::BK_STG, Cfg::BM, CU_TENSOR_MAP_SWIZZLE_128B)))
    return st;
  if ((st = make_tmap(&tmB, B, n, k, ldb, 32, Cfg::BK_STG, CU_TENSOR_MAP_SWIZZLE_128B))) return st;
  if ((st = make_tmap(&tmC, C, n, m, ldc, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B))) return st;

  auto kern = tcec::tcec_gemm_ts_kernel<V, R, BN, NOP>;
  const cudaError_t attr_err = smem_optin(kern, Cfg::SMEM_BYTES);
  if (attr_err != cudaSuccess) return TCEC_ERR_CUDA;

  tcec::GemmShape shp;
  shp.m = static_cast<int32_t>(m);
  shp.n = static_cast<int32_t>(n);
  shp.k = static_cast<int32_t>(k);
  shp.num_op_stages = static_cast<int32_t>((k + VC::BK_OP - 1) / VC::BK_OP);
  shp.drain_every = drain_every;
  shp.group_m = group_m;
  const float scale = ldexpf(1.0f, scale_log2);
  const float inv_scale = ldexpf(1.0f, -scale_log2);
  const tcec::FlagThresholds thr = tcec::flag_thresholds(V, R, scale_log2);
  const int64_t pairs = ((m + 2 * Cfg::BM - 1) / (2 * Cfg::BM)) * ((n + Cfg::BN - 1) / Cfg::BN);
  kern<<<static_cast<unsigned>(2 * pairs), Cfg::NUM_THREADS, Cfg::SMEM_BYTES, stream>>>(
      tmA, tmB, tmC, shp, scale, inv_scale, thr, d_flags);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError() == cudaSuccess ? TCEC_OK : TCEC_ERR_CUDA;
}

// Split-once mode: one split pass per input (A as m x k, B transposed to
// n x k, both K-major in the operand type), then the three-product GEMM.
template <int V, int R, int S>
int launch_gemm_presplit(int64_t m, int64_t n, int64_t k, const float* A, int64_t lda,
                         const float* B, int64_t ldb, float* C, int64_t ldc, int scale_log2,
                         int drain_every, int group_m, int group_user, bool lockstep_ok,
                         uint32_t* d_flags, cudaStream_t stream) {
  using Cfg = tcec::PsCfg<V, S>;
  using VC = tcec::VarCfg<V>;
  const uint32_t esize = V == tcec::kFP16 ? 2u : 4u;
  const CUtensorMapDataType dt =
      V == tcec::kFP16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  const int64_t ldk = (k + 15) / 16 * 16;
  const size_t a_bytes = size_t(m) * ldk * esize, b_bytes = size_t(n) * ldk * esize;
  uint8_t* ws = nullptr;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return TCEC_ERR_CUDA;
  keep_pool(dev);
  if (cudaMallocAsync(reinterpret_cast<void**>(&ws), 2 * (a_bytes + b_bytes), stream) != cudaSuccess)
    return TCEC_ERR_CUDA;
  void* ah = ws;
  void* al = ws + a_bytes;
  void* bh = ws + 2 * a_bytes;
  void* bl = ws + 2 * a_bytes + b_bytes;
  int st = TCEC_OK;
  CUtensorMap tmAh, tmAl, tmBh, tmBl;
  if (!st) st = make_tmap_op(&tmAh, ah, dt, esize, k, m, ldk, Cfg::BM);
  if (!st) st = make_tmap_op(&tmAl, al, dt, esize, k, m, ldk, Cfg::BM);
  if (!st) st = make_tmap_op(&tmBh, bh, dt, esize, k, n, ldk, Cfg::BN_CTA);
  if (!st) st = make_tmap_op(&tmBl, bl, dt, esize, k, n, ldk, Cfg::BN_CTA);
  auto kern = tcec::tcec_gemm_ps_kernel<V, S>;
  const cudaError_t attr_err = smem_optin(kern, Cfg::SMEM_BYTES);
  if (!st && attr_err != cudaSuccess) st = TCEC_ERR_CUDA;
  // persistent: one pair per TPC; lock-step waves of 8 x 9 tiles from 8 waves on
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tiles = ((m + 2 * Cfg::BM - 1) / (2 * Cfg::BM)) * ((n + Cfg::BN - 1) / Cfg::BN);
  int64_t pairs = sms / 2;
  if (pairs > tiles) pairs = tiles;
  if (pairs < 1) pairs = 1;
  const bool lockstep = lockstep_ok && tiles >= 8 * int64_t(sms / 2);
  uint32_t* wave_ctr = nullptr;
  if (!st && lockstep) {
    if (cudaMallocAsync(reinterpret_cast<void**>(&wave_ctr), sizeof(uint32_t), stream) != cudaSuccess ||
        cudaMemsetAsync(wave_ctr, 0, sizeof(uint32_t), stream) != cudaSuccess)
      st = TCEC_ERR_CUDA;
  }
  if (!st) {
    const float scale = ldexpf(1.0f, scale_log2);
    const float inv_scale = ldexpf(1.0f, -scale_log2);
    const float inv_scale2 = ldexpf(1.0f, -2 * scale_log2);
    const tcec::FlagThresholds thr = S == tcec::kSchPlain ? tcec::plain_thresholds(V, R)
                                                          : tcec::flag_thresholds(V, R, scale_log2);
    const unsigned ga = static_cast<unsigned>(((m + 63) / 64) * ((k + 63) / 64));
    tcec::tcec_presplit_kernel<V, R, false><<<ga, 256, 0, stream>>>(
        A, static_cast<int32_t>(m), static_cast<int32_t>(k), lda, ah, al, ldk,
        static_cast<int32_t>(m), scale, thr, d_flags);
    const unsigned gb = static_cast<unsigned>(((k + 63) / 64) * ((n + 63) / 64));
    tcec::tcec_presplit_kernel<V, R, true><<<gb, 256, 0, stream>>>(
        B, static_cast<int32_t>(k), static_cast<int32_t>(n), ldb, bh, bl, ldk,
        static_cast<int32_t>(n), scale, thr, d_flags);
    tcec::GemmShape shp;
    shp.m = static_cast<int32_t>(m);
    shp.n = static_cast<int32_t>(n);
    shp.k = static_cast<int32_t>(k);
    shp.num_op_stages = static_cast<int32_t>((k + VC::BK_OP - 1) / VC::BK_OP);
    shp.drain_every = drain_every;
    shp.group_m = group_user > 0 ? group_m : (lockstep ? 8 : group_m);
    kern<<<static_cast<unsigned>(2 * pairs), Cfg::NUM_THREADS, Cfg::SMEM_BYTES, stream>>>(
        tmAh, tmAl, tmBh, tmBl, C, ldc, shp, inv_scale, inv_scale2, d_flags, wave_ctr);
    g_launches.fetch_add(3, std::memory_order_relaxed);
    if (cudaGetLastError() != cudaSuccess) st = TCEC_ERR_CUDA;
  }
  if (wave_ctr) cudaFreeAsync(wave_ctr, stream);
  cudaFreeAsync(ws, stream);
  return st;
}

#ifdef TCEC_WITH_RING
// Fused GEMM with the split shared through an L2-resident ring (kernel_variant
// 6, tcec_ring.cuh): every CTA of a co-resident persistent grid splits its
// share of each wave's k-slices once; the pairs TMA the split operands.
template <int V, int R>
int launch_gemm_ring(int64_t m, int64_t n, int64_t k, const float* A, int64_t lda, const float* B,
                     int64_t ldb, float* C, int64_t ldc, int scale_log2, int drain_every,
                     int group_m, uint32_t* d_flags, cudaStream_t stream) {
  using Cfg = tcec::PsCfg<V, tcec::kSchC3>;
  using VC = tcec::VarCfg<V>;
  const uint32_t esize = V == tcec::kFP16 ? 2u : 4u;
  const CUtensorMapDataType dt =
      V == tcec::kFP16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return TCEC_ERR_CUDA;
  auto kern = tcec::tcec_gemm_ring_kernel<V, R>;
  if (smem_optin(kern, tcec::ring_smem_bytes<V>()) != cudaSuccess) return TCEC_ERR_CUDA;
  // every CTA splits: the grid must be co-resident (one pair per TPC)
  static std::mutex occ_mu;
  static int occ_pairs[64] = {0};
  int max_pairs = 0;
  {
    std::lock_guard<std::mutex> lk(occ_mu);
    if (dev >= 0 && dev < 64 && occ_pairs[dev] == 0) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(2, 1, 1);
      cfg.blockDim = dim3(640, 1, 1);
      cfg.dynamicSmemBytes = tcec::ring_smem_bytes<V>();
      if (cudaOccupancyMaxActiveClusters(&occ_pairs[dev], kern, &cfg) != cudaSuccess) {
        cudaGetLastError();
        occ_pairs[dev] = -1;
      }
    }
    if (dev >= 0 && dev < 64) max_pairs = occ_pairs[dev];
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int np = sms / 2;
  if (max_pairs > 0 && max_pairs < np) np = max_pairs;
  const int tiles_m = static_cast<int>((m + 255) / 256), tiles_n = static_cast<int>((n + 255) / 256);
  const int tiles = tiles_m * tiles_n;
  if (np > tiles) np = tiles;
  if (np < 1) return TCEC_ERR_CUDA;
  const int gm = group_m > 0 ? group_m : 8;
  const int waves = (tiles + np - 1) / np;
  const int nop = static_cast<int>((k + VC::BK_OP - 1) / VC::BK_OP);
  int la_max = 1, lb_max = 1;
  for (int w = 0; w < waves; ++w) {
    const tcec::RingWave rw = tcec::ring_wave(w, np, tiles, tiles_m, tiles_n, gm);
    la_max = std::max(la_max, rw.la);
    lb_max = std::max(lb_max, rw.lb);
  }
  // ring depth in slices: 16 covers the split -> release -> TMA chain
  // (8: FP16 331, 12: 361, 16-32: 364-368 TF/s at 16384^3, profiles/r02/ring.md)
  const int depth = 16;
  const size_t slot_rows_a = size_t(la_max) * 256, slot_rows_b = size_t(lb_max) * 256;
  const size_t ring_a = depth * slot_rows_a * 128, ring_b = depth * slot_rows_b * 128;
  const size_t slices = size_t(waves) * nop;
  const size_t ctr_bytes = slices * (la_max + lb_max + 1) * sizeof(uint32_t);
  keep_pool(dev);
  uint8_t* ws = nullptr;
  if (cudaMallocAsync(reinterpret_cast<void**>(&ws), 2 * (ring_a + ring_b) + ctr_bytes, stream) !=
      cudaSuccess)
    return TCEC_ERR_CUDA;
  tcec::RingArgs ra;
  ra.A = A;
  ra.B = B;
  ra.lda = lda;
  ra.ldb = ldb;
  ra.ahi = ws;
  ra.alo = ws + ring_a;
  ra.bhi = ws + 2 * ring_a;
  ra.blo = ws + 2 * ring_a + ring_b;
  ra.ready = reinterpret_cast<uint32_t*>(ws + 2 * (ring_a + ring_b));
  ra.freed = ra.ready + slices * (la_max + lb_max);
  ra.depth = depth;
  ra.la_max = la_max;
  ra.lb_max = lb_max;
  ra.np = np;
  int st = TCEC_OK;
  CUtensorMap tmAh, tmAl, tmBh, tmBl;
  const uint64_t bk = VC::BK_OP;
  if (!st) st = make_tmap_op(&tmAh, ra.ahi, dt, esize, bk, depth * slot_rows_a, bk, Cfg::BM);
  if (!st) st = make_tmap_op(&tmAl, ra.alo, dt, esize, bk, depth * slot_rows_a, bk, Cfg::BM);
  if (!st) st = make_tmap_op(&tmBh, ra.bhi, dt, esize, bk, depth * slot_rows_b, bk, Cfg::BN_CTA);
  if (!st) st = make_tmap_op(&tmBl, ra.blo, dt, esize, bk, depth * slot_rows_b, bk, Cfg::BN_CTA);
  if (!st && cudaMemsetAsync(ra.ready, 0, ctr_bytes, stream) != cudaSuccess) st = TCEC_ERR_CUDA;
  if (!st) {
    tcec::GemmShape shp;
    shp.m = static_cast<int32_t>(m);
    shp.n = static_cast<int32_t>(n);
    shp.k = static_cast<int32_t>(k);
    shp.num_op_stages = nop;
    shp.drain_every = drain_every;
    shp.group_m = gm;
    const float scale = ldexpf(1.0f, scale_log2);
    const float inv_scale = ldexpf(1.0f, -scale_log2);
    const tcec::FlagThresholds thr = tcec::flag_thresholds(V, R, scale_log2);
    kern<<<static_cast<unsigned>(2 * np), 640, tcec::ring_smem_bytes<V>(), stream>>>(
        tmAh, tmAl, tmBh, tmBl, C, ldc, shp, ra, scale, inv_scale, thr, d_flags);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (cudaGetLastError() != cudaSuccess) st = TCEC_ERR_CUDA;
  }
  cudaFreeAsync(ws, stream);
  return st;
}
#endif  // TCEC_WITH_RING

// Persistent CTA-pair kernel (kernel_variant 2): one pair per TPC walks the
// tile sequence with its pipelines running across tiles.
template <int V, int R>
int launch_gemm_pers(int64_t m, int64_t n, int64_t k, const float* A, int64_t lda, const float* B,
                     int64_t ldb, float* C, int64_t ldc, int scale_log2, int drain_every,
                     int group_m, bool lockstep, uint32_t* d_flags, cudaStream_t stream,
                     int ksplit = 1) {
  using Cfg = tcec::PairCfg<V>;
  using VC = tcec::VarCfg<V>;
  CUtensorMap tmA, tmB;
  int st;
  if ((st = make_tmap(&tmA, A, k, m, lda, Cfg::BK_STG, Cfg::BM, CU_TENSOR_MAP_SWIZZLE_128B)))
    return st;
  if ((st = make_tmap(&tmB, B, n, k, ldb, 32, Cfg::BK_STG, CU_TENSOR_MAP_SWIZZLE_128B))) return st;
  auto kern = tcec::tcec_gemm_pers_kernel<V, R>;
  const cudaError_t attr_err = smem_optin(kern, Cfg::SMEM_BYTES);
  if (attr_err != cudaSuccess) return TCEC_ERR_CUDA;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  tcec::GemmShape shp;
  shp.m = static_cast<int32_t>(m);
  shp.n = static_cast<int32_t>(n);
  shp.k = static_cast<int32_t>(k);
  shp.num_op_stages = static_cast<int32_t>((k + VC::BK_OP - 1) / VC::BK_OP);
  shp.drain_every = drain_every;
  shp.group_m = group_m;
  const float scale = ldexpf(1.0f, scale_log2);
  const float inv_scale = ldexpf(1.0f, -scale_log2);
  const tcec::FlagThresholds thr = tcec::flag_thresholds(V, R, scale_log2);
  if (ksplit > shp.num_op_stages) ksplit = shp.num_op_stages;
  const int64_t tiles = ((m + 2 * Cfg::BM - 1) / (2 * Cfg::BM)) * ((n + Cfg::BN - 1) / Cfg::BN) *
                        (ksplit > 1 ? ksplit : 1);
  int64_t pairs = sms / 2;
  if (pairs > tiles) pairs = tiles;
  if (pairs < 1) pairs = 1;
  uint32_t* wave_ctr = nullptr;
  if (lockstep) {  // a zeroed counter per launch, from the stream-ordered pool
    keep_pool(dev);
    if (cudaMallocAsync(reinterpret_cast<void**>(&wave_ctr), sizeof(uint32_t), stream) != cudaSuccess)
      return TCEC_ERR_CUDA;
    if (cudaMemsetAsync(wave_ctr, 0, sizeof(uint32_t), stream) != cudaSuccess) {
      cudaFreeAsync(wave_ctr, stream);
      return TCEC_ERR_CUDA;
    }
  }
  if (ksplit > 1) {
    // split-K: (tile, part) units, partial sums to a stream-ordered workspace,
    // then the fixed-order combine (tcec_splitk_reduce_kernel)
    auto kern_sk = tcec::tcec_gemm_pers_kernel<V, R, true>;
    if (smem_optin(kern_sk, Cfg::SMEM_BYTES) != cudaSuccess) {
      if (wave_ctr) cudaFreeAsync(wave_ctr, stream);
      return TCEC_ERR_CUDA;
    }
    const int64_t n8 = (n + 7) & ~int64_t(7);
    float* ws = nullptr;
    if (cudaMallocAsync(reinterpret_cast<void**>(&ws), sizeof(float) * 2 * ksplit * m * n8,
                        stream) != cudaSuccess) {
      if (wave_ctr) cudaFreeAsync(wave_ctr, stream);
      return TCEC_ERR_CUDA;
    }
    kern_sk<<<static_cast<unsigned>(2 * pairs), Cfg::NUM_THREADS, Cfg::SMEM_BYTES, stream>>>(
        tmA, tmB, C, ldc, shp, scale, inv_scale, thr, d_flags, wave_ctr, ws, ksplit);
    bool ok = cudaGetLastError() == cudaSuccess;
    const int64_t quads = m * (n8 / 4);
    int64_t blocks = (quads + 255) / 256;
    if (blocks > 8 * int64_t(sms)) blocks = 8 * int64_t(sms);
    tcec::tcec_splitk_reduce_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(
        ws, ksplit, static_cast<int>(m), static_cast<int>(n), C, ldc, inv_scale, d_flags);
    ok = ok && cudaGetLastError() == cudaSuccess;
    g_launches.fetch_add(2, std::memory_order_relaxed);
    cudaFreeAsync(ws, stream);
    if (wave_ctr) cudaFreeAsync(wave_ctr, stream);
    return ok ? TCEC_OK : TCEC_ERR_CUDA;
  }
  kern<<<static_cast<unsigned>(2 * pairs), Cfg::NUM_THREADS, Cfg::SMEM_BYTES, stream>>>(
      tmA, tmB, C, ldc, shp, scale, inv_scale, thr, d_flags, wave_ctr, nullptr, 1);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  const bool launched = cudaGetLastError() == cudaSuccess;
  if (wave_ctr) cudaFreeAsync(wave_ctr, stream);
  return launched ? TCEC_OK : TCEC_ERR_CUDA;
}

int device_sms() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

// Resolved options of one call (sgemm_impl -> dispatch).
struct Plan {
  int block_n;        // 256 / 192 / 128
  int kvariant;       // 1 single-CTA (block_n 128), 2 persistent, 3 lock-step, 4 per-tile
  int kv_user;        // as requested (0 = automatic)
  int split_mode;     // 0 / 1 fused, 2 split-once
  int scheme;         // TCEC_SCHEME_*
  int split_k;        // parts (<= 1: off)
  int drain_every;    // MMA k-steps per drain interval (corrected3) / per block (INUNIT4_RN)
  int group_m;        // rasterisation group in 128-row tiles
  int group_user;     // the caller's group_m (0 = default)
  int scale_log2;
};

template <int V, int R>
int dispatch(const Plan& p, int64_t m, int64_t n, int64_t k, const float* A, int64_t lda,
             const float* B, int64_t ldb, float* C, int64_t ldc, const ExtraC* ex, uint32_t* fl,
             cudaStream_t st) {
  const int s = p.scale_log2, de = p.drain_every, kv = p.kvariant, gm = p.group_m;
  const int gpair = gm / 2 > 0 ? gm / 2 : 1;  // group in pair-tile rows
  const bool extra = ex && ex->count > 0;
  if (extra && (p.block_n != 256 || p.split_mode == 2 || p.scheme != TCEC_SCHEME_CORRECTED3 ||
                p.split_k > 1 || kv != 4))
    return TCEC_ERR_UNSUPPORTED;  // extra destinations: the per-tile pair kernel only
  if (p.split_k > 1) {  // split-K: the persistent pair kernel over (tile, part) units
    if (p.split_mode == 2 || p.scheme != TCEC_SCHEME_CORRECTED3 || p.block_n != 256)
      return TCEC_ERR_UNSUPPORTED;
    const int g = p.group_user > 0 ? gpair : 8;
    // lock-step waves unless the caller pinned the per-tile variant (a kernel
    // sharing the GPU with other work, e.g. the host path's concurrent blocks)
    return launch_gemm_pers<V, R>(m, n, k, A, lda, B, ldb, C, ldc, s, de, g, p.kv_user != 4, fl,
                                  st, p.split_k);
  }
  if (p.split_mode == 2 || p.scheme != TCEC_SCHEME_CORRECTED3) {
    if (p.block_n != 256 || (p.kv_user != 0 && p.kv_user != 4)) return TCEC_ERR_UNSUPPORTED;
    const bool ls = p.kv_user != 4;  // lock-step waves once the product spans >= 8 of them
    const int gu = p.group_user;
    switch (p.scheme) {
      case TCEC_SCHEME_CORRECTED3:
        return launch_gemm_presplit<V, R, tcec::kSchC3>(m, n, k, A, lda, B, ldb, C, ldc, s, de, gpair, gu, ls, fl, st);
      case TCEC_SCHEME_CORRECTED3_DD:
        return launch_gemm_presplit<V, R, tcec::kSchC3DD>(m, n, k, A, lda, B, ldb, C, ldc, s, de, gpair, gu, ls, fl, st);
      case TCEC_SCHEME_TC_PLAIN:
        return launch_gemm_presplit<V, R, tcec::kSchPlain>(m, n, k, A, lda, B, ldb, C, ldc, 0, de, gpair, gu, ls, fl, st);
      case TCEC_SCHEME_INUNIT4:
        return launch_gemm_presplit<V, R, tcec::kSchIn4>(m, n, k, A, lda, B, ldb, C, ldc, s, de, gpair, gu, ls, fl, st);
      case TCEC_SCHEME_INUNIT4_RN:  // de = MMA k-steps per drained block
        return launch_gemm_presplit<V, R, tcec::kSchIn4RN>(m, n, k, A, lda, B, ldb, C, ldc, s, de, gpair, gu, ls, fl, st);
      default:
        return TCEC_ERR_UNSUPPORTED;
    }
  }
  if (p.block_n == 256) {
    if (kv == 6) {  // split shared through the L2-resident ring
#ifdef TCEC_WITH_RING
      const int g = p.group_user > 0 ? gpair : 8;
      return launch_gemm_ring<V, R>(m, n, k, A, lda, B, ldb, C, ldc, s, de, g, fl, st);
#else
      return TCEC_ERR_UNSUPPORTED;
#endif
    }
    if (kv == 2 || kv == 3) {  // persistent; 3 = with lock-step waves
      const int g = p.group_user > 0 ? gpair : (kv == 3 ? 8 : 4);
      return launch_gemm_pers<V, R>(m, n, k, A, lda, B, ldb, C, ldc, s, de, g, kv == 3, fl, st);
    }
    if (kv != 4) return TCEC_ERR_UNSUPPORTED;
    return launch_gemm_pair<V, R>(m, n, k, A, lda, B, ldb, C, ldc, s, de, gpair, ex, fl, st);
  }
  // the narrow tiles run whole operand stages per drain interval
  if (de % 4 != 0) return TCEC_ERR_UNSUPPORTED;
  if (p.block_n == 192) {
    if (kv != 4) return TCEC_ERR_UNSUPPORTED;
    return launch_gemm_ts<V, R, 192, 2>(m, n, k, A, lda, B, ldb, C, ldc, s, de, gpair, fl, st);
  }
  if (p.block_n == 128) {
    // kernel_variant 1: the single-CTA 128 x 128 kernel (tcec_gemm.cuh, the
    // first kernel); otherwise the CTA-pair 256 x 128 tile with A in TMEM
    if (kv == 1) return launch_gemm<V, R, 128>(m, n, k, A, lda, B, ldb, C, ldc, s, de, gm, fl, st);
    if (kv != 4) return TCEC_ERR_UNSUPPORTED;
    return launch_gemm_ts<V, R, 128, 2>(m, n, k, A, lda, B, ldb, C, ldc, s, de, gpair, fl, st);
  }
  if (p.block_n == 64) {  // 256 x 64: small products, more CTA pairs busy
    if (kv != 4) return TCEC_ERR_UNSUPPORTED;
    return launch_gemm_ts<V, R, 64, 4>(m, n, k, A, lda, B, ldb, C, ldc, s, de, gpair, fl, st);
  }
  return TCEC_ERR_UNSUPPORTED;
}

// Per-device resources of the host-buffer entry (tcec_sgemm_host), kept
// across calls: four streams, the block events and device copies of A, B, C
// (grown on demand, freed by tcec_host_release).  One call at a time per
// device (the mutex); the call itself is synchronous.
constexpr int kMaxDevices = 64;
struct HostCtx {
  static constexpr int kMaxBlk = 8;
  std::mutex mu;
  bool ready = false;
  cudaStream_t s_in = nullptr, s_out = nullptr, s_c[2] = {nullptr, nullptr};
  cudaEvent_t ev_start = nullptr, ev_a[kMaxBlk] = {}, ev_b[kMaxBlk] = {},
              ev_g[kMaxBlk * kMaxBlk] = {};
  float *dA = nullptr, *dB = nullptr, *dC = nullptr;
  size_t capA = 0, capB = 0, capC = 0;  // floats
  uint32_t* dF = nullptr;

  cudaError_t init() {
    cudaError_t e;
    for (cudaStream_t* x : {&s_in, &s_out, &s_c[0], &s_c[1]})
      if ((e = cudaStreamCreateWithFlags(x, cudaStreamNonBlocking)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming)) != cudaSuccess) return e;
    for (int i = 0; i < kMaxBlk; ++i) {
      if ((e = cudaEventCreateWithFlags(&ev_a[i], cudaEventDisableTiming)) != cudaSuccess) return e;
      if ((e = cudaEventCreateWithFlags(&ev_b[i], cudaEventDisableTiming)) != cudaSuccess) return e;
    }
    for (int i = 0; i < kMaxBlk * kMaxBlk; ++i)
      if ((e = cudaEventCreateWithFlags(&ev_g[i], cudaEventDisableTiming)) != cudaSuccess) return e;
    if ((e = cudaMalloc(reinterpret_cast<void**>(&dF), sizeof(uint32_t))) != cudaSuccess) return e;
    ready = true;
    return cudaSuccess;
  }
  static cudaError_t grow(float*& p, size_t& cap, size_t need) {
    if (need <= cap) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    const cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&p), need * sizeof(float));
    if (e == cudaSuccess) cap = need;
    return e;
  }
  cudaError_t reserve(size_t a, size_t b, size_t c) {
    cudaError_t e;
    if ((e = grow(dA, capA, a)) != cudaSuccess) return e;
    if ((e = grow(dB, capB, b)) != cudaSuccess) return e;
    return grow(dC, capC, c);
  }
  cudaError_t release() {
    cudaError_t e = cudaSuccess;
    for (float** p : {&dA, &dB, &dC})
      if (*p) {
        const cudaError_t f = cudaFree(*p);
        if (e == cudaSuccess) e = f;
        *p = nullptr;
      }
    capA = capB = capC = 0;
    return e;
  }
};
HostCtx g_host[kMaxDevices];

int resolve_rounding(int variant, int rounding) {
  if (rounding == TCEC_ROUND_DEFAULT) return variant == TCEC_FP16 ? TCEC_ROUND_RN : TCEC_ROUND_RNA;
  return rounding;
}

// Built (variant, rounding) pairs: FP16 {RN, RZ} (cvt.rn / cvt.rz), TF32 {RN, RNA, RZ}.
bool rounding_supported(int variant, int rounding) {
  if (variant == TCEC_FP16) return rounding == TCEC_ROUND_RN || rounding == TCEC_ROUND_RZ;
  return rounding == TCEC_ROUND_RN || rounding == TCEC_ROUND_RNA || rounding == TCEC_ROUND_RZ;
}

template <int V, int R>
int launch_split(const float* X, int64_t count, int scale_log2, float* hi, float* lo,
                 uint32_t* d_flags, cudaStream_t stream) {
  const float scale = ldexpf(1.0f, scale_log2);
  const tcec::FlagThresholds thr = tcec::flag_thresholds(V, R, scale_log2);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t pairs = (count + 1) / 2;
  int64_t blocks = (pairs + 255) / 256;
  const int64_t cap = static_cast<int64_t>(sms) * 16;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  tcec::tcec_split_kernel<V, R><<<static_cast<unsigned>(blocks), 256, 0, stream>>>(
      X, count, scale, thr, hi, lo, d_flags);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError() == cudaSuccess ? TCEC_OK : TCEC_ERR_CUDA;
}

}  // namespace

extern "C" {

int tcec_version(void) { return 100; }

uint64_t tcec_launch_count(void) { return g_launches.load(); }

const char* tcec_status_str(int status) {
  switch (status) {
    case TCEC_OK: return "ok";
    case TCEC_ERR_ARG: return "invalid argument (shape, leading dimension or option)";
    case TCEC_ERR_ALIGN: return "pointer or leading dimension not 16-byte aligned";
    case TCEC_ERR_UNSUPPORTED: return "unsupported variant / rounding / drain / tile option";
    case TCEC_ERR_CUDA: return "CUDA error";
    case TCEC_ERR_ARCH: return "current device is not an sm_100 (B200) GPU";
    default: return "unknown status";
  }
}

}  // extern "C"

namespace {

int sgemm_impl(int variant, int64_t m, int64_t n, int64_t k, const float* A, int64_t lda,
               const float* B, int64_t ldb, float* C, int64_t ldc, const tcec_opts* opts,
               const ExtraC* ex, uint32_t* d_flags, void* stream) {
  if (variant != TCEC_FP16 && variant != TCEC_TF32) return TCEC_ERR_ARG;
  if (m < 0 || n < 0 || k < 0) return TCEC_ERR_ARG;
  if (m > INT32_MAX || n > INT32_MAX || k > INT32_MAX) return TCEC_ERR_ARG;
  if (lda < (k > 0 ? k : 1) || ldb < (n > 0 ? n : 1) || ldc < (n > 0 ? n : 1)) return TCEC_ERR_ARG;
  tcec_opts o;
  memset(&o, 0, sizeof(o));
  o.split_rounding = TCEC_ROUND_DEFAULT;
  o.scale_log2 = -1;
  if (opts) o = *opts;
  const int rounding = resolve_rounding(variant, o.split_rounding);
  if (!rounding_supported(variant, rounding)) return TCEC_ERR_UNSUPPORTED;
  const bool in_unit = o.scheme == TCEC_SCHEME_INUNIT4 || o.scheme == TCEC_SCHEME_INUNIT4_RN;
  Plan p;
  p.scale_log2 = o.scale_log2 < 0 ? (variant == TCEC_FP16 && !in_unit &&
                                     o.scheme != TCEC_SCHEME_TC_PLAIN ? 11 : 0)
                                  : o.scale_log2;
  if (variant == TCEC_TF32 && p.scale_log2 != 0) return TCEC_ERR_UNSUPPORTED;
  if (variant == TCEC_FP16 && p.scale_log2 != 0 && p.scale_log2 != 11) return TCEC_ERR_UNSUPPORTED;
  if (o.scheme < TCEC_SCHEME_CORRECTED3 || o.scheme > TCEC_SCHEME_INUNIT4_RN)
    return TCEC_ERR_UNSUPPORTED;
  if (in_unit && o.scale_log2 > 0) return TCEC_ERR_UNSUPPORTED;
  p.scheme = o.scheme;
  // Drain interval in MMA k-steps (16 deep FP16, 8 deep TF32).  corrected3:
  // the main-term block of schemes.py:300-304, default 128 (FP16) / 64 (TF32)
  // -- measured both faster and more accurate against FP64 than draining every
  // operand stage; INUNIT4_RN: the reference's block_k, default 16.
  const int kstep = variant == TCEC_FP16 ? 16 : 8;
  const int drain_k = o.drain_k != 0 ? o.drain_k
                                     : (o.scheme == TCEC_SCHEME_INUNIT4_RN ? 16 : 8 * kstep);
  if (drain_k <= 0 || drain_k % kstep != 0) return TCEC_ERR_UNSUPPORTED;
  p.drain_every = drain_k / kstep;
  if (o.block_n != 0 && o.block_n != 64 && o.block_n != 128 && o.block_n != 192 &&
      o.block_n != 256)
    return TCEC_ERR_UNSUPPORTED;
  // the narrow tiles drain whole operand stages (4 k-steps)
  if ((o.block_n == 64 || o.block_n == 128 || o.block_n == 192) && p.drain_every % 4 != 0)
    return TCEC_ERR_UNSUPPORTED;
  p.group_user = o.group_m;
  p.group_m = o.group_m <= 0 ? 8 : o.group_m;
  // kernel_variant: 0 = automatic, 1 = single-CTA (block_n 128), 2 = persistent,
  // 3 = persistent with lock-step waves, 4 = per-tile, 6 = persistent with the
  // split shared through an L2-resident ring (tcec_ring.cuh)
  p.kvariant = p.kv_user = o.kernel_variant;
  if (p.kvariant < 0 || p.kvariant > 6 || p.kvariant == 5) return TCEC_ERR_UNSUPPORTED;
  if (p.kvariant == 6 && (o.block_n != 0 && o.block_n != 256)) return TCEC_ERR_UNSUPPORTED;
  if (p.kvariant == 1 && o.block_n != 128) return TCEC_ERR_UNSUPPORTED;
  // split_mode: 0 / 1 = split fused into the GEMM, 2 = split once in a separate pass
  p.split_mode = o.split_mode;
  if (p.split_mode < 0 || p.split_mode > 2) return TCEC_ERR_UNSUPPORTED;
  if (o.split_k < -1 || o.split_k > 64) return TCEC_ERR_UNSUPPORTED;
  const bool fused_c3 = p.scheme == TCEC_SCHEME_CORRECTED3 && p.split_mode != 2;
  const int sms = device_sms();
  const int64_t pairs = sms / 2 > 0 ? sms / 2 : 1;
  const int64_t tiles256 = ((m + 255) / 256) * ((n + 255) / 256);
  p.split_k = o.split_k;
  if (p.split_k == -1) {
    // automatic: split only when the 256 x 256 tiles leave most CTA pairs idle
    // and k is long enough that each part keeps >= 16 operand stages; measured
    // 2.2-2.7x at 1024 x 1024 x 16384, a loss on small squares
    const int64_t nop = (k + (variant == TCEC_FP16 ? 63 : 31)) / (variant == TCEC_FP16 ? 64 : 32);
    int64_t parts = tiles256 > 0 ? pairs / tiles256 : 1;
    if (parts > nop / 16) parts = nop / 16;
    if (parts > 8) parts = 8;
    const bool eligible = fused_c3 && ex == nullptr && (o.block_n == 0 || o.block_n == 256) &&
                          p.kvariant != 1;
    p.split_k = (eligible && 2 * tiles256 <= pairs && parts >= 2) ? static_cast<int>(parts) : 0;
  }
  p.block_n = o.block_n;
  if (p.block_n == 0) {
    // automatic tile.  Below 8 waves of 256 x 256 tiles (the persistent
    // kernel's range) the per-tile kernels are wave-quantised: pick the width
    // minimising waves x width x per-flop cost, with the narrow A-from-TMEM
    // tiles' measured costs 1.1 (256 x 192), 1.25 (256 x 128) and 2.0 (256 x
    // 64) -- products that fit one wave of 256 x 64 tiles (1024^2, 768^2,
    // 512 x 1024) take 64, 1536^2 takes 128, 1792^2 and 2560^2 take 192, 2048^2
    // and >= 3072^2 keep 256 (profiles/r01/smallbn.log, midbn.log,
    // profiles/r02/smallbn_r02.jsonl).  Results are bit-identical.
    // The narrow tiles drain per operand stage (multiples of 4 k-steps).
    p.block_n = 256;
    if ((p.kvariant == 0 || p.kvariant == 4) && fused_c3 && ex == nullptr && p.split_k <= 1 &&
        p.drain_every % 4 == 0 && tiles256 < 8 * pairs) {
      const int64_t rows = (m + 255) / 256;
      double best = 0.0;
      const int widths[4] = {256, 192, 128, 64};
      const double eff[4] = {1.0, 1.1, 1.25, 2.0};
      for (int i = 0; i < 4; ++i) {
        const int64_t waves = (rows * ((n + widths[i] - 1) / widths[i]) + pairs - 1) / pairs;
        const double cost = double(waves) * widths[i] * eff[i];
        if (i == 0 || cost < best) {
          best = cost;
          p.block_n = widths[i];
        }
      }
    }
  }
  if (p.kvariant == 0) {
    // automatic kernel: the persistent kernel with lock-step waves of 8 x 9
    // pair tiles once a 256 x 256 product spans >= 8 waves (measured +2-8% at
    // 8192^3 .. 32768 x 16384^2, DRAM reads -21..-52%), else per-tile
    p.kvariant = (p.block_n == 256 && fused_c3 && ex == nullptr && tiles256 >= 8 * pairs) ? 3 : 4;
  }
  if (m == 0 || n == 0) return TCEC_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (k == 0) {
    // schemes.py:210-218 + 300-307 with zero blocks: C = 0 exactly
    return cudaMemset2DAsync(C, ldc * sizeof(float), 0, n * sizeof(float), m, st) == cudaSuccess
               ? TCEC_OK
               : TCEC_ERR_CUDA;
  }
  if (!aligned16(A) || !aligned16(B) || !aligned16(C) || (lda % 4) || (ldb % 4) || (ldc % 4))
    return TCEC_ERR_ALIGN;
  int s;
  if ((s = check_arch())) return s;
  if ((s = get_encoder())) return s;
  using namespace tcec;
  if (variant == TCEC_FP16) {
    if (rounding == TCEC_ROUND_RN)
      return dispatch<kFP16, kRN>(p, m, n, k, A, lda, B, ldb, C, ldc, ex, d_flags, st);
    if (rounding == TCEC_ROUND_RZ)
      return dispatch<kFP16, kRZ>(p, m, n, k, A, lda, B, ldb, C, ldc, ex, d_flags, st);
    return TCEC_ERR_UNSUPPORTED;
  }
  if (rounding == TCEC_ROUND_RNA)
    return dispatch<kTF32, kRNA>(p, m, n, k, A, lda, B, ldb, C, ldc, ex, d_flags, st);
  if (rounding == TCEC_ROUND_RN)
    return dispatch<kTF32, kRN>(p, m, n, k, A, lda, B, ldb, C, ldc, ex, d_flags, st);
  if (rounding == TCEC_ROUND_RZ)
    return dispatch<kTF32, kRZ>(p, m, n, k, A, lda, B, ldb, C, ldc, ex, d_flags, st);
  return TCEC_ERR_UNSUPPORTED;
}

}  // namespace

extern "C" {

int tcec_sgemm(int variant, int64_t m, int64_t n, int64_t k, const float* A, int64_t lda,
               const float* B, int64_t ldb, float* C, int64_t ldc, const tcec_opts* opts,
               uint32_t* d_flags, void* stream) {
  return sgemm_impl(variant, m, n, k, A, lda, B, ldb, C, ldc, opts, nullptr, d_flags, stream);
}

int tcec_sgemm_multi(int variant, int64_t m, int64_t n, int64_t k, const float* A, int64_t lda,
                     const float* B, int64_t ldb, float* const* C, int n_c, int64_t ldc,
                     const tcec_opts* opts, uint32_t* d_flags, void* stream) {
  if (C == nullptr || n_c < 1 || n_c > 1 + tcec::kMaxExtraC) return TCEC_ERR_ARG;
  ExtraC ex;
  ex.count = n_c - 1;
  for (int d = 0; d < ex.count; ++d) {
    if (C[1 + d] == nullptr || !aligned16(C[1 + d])) return TCEC_ERR_ALIGN;
    ex.c[d] = C[1 + d];
  }
  if (k == 0 && ex.count > 0) {  // zeros into every destination
    for (int d = 0; d < n_c; ++d) {
      const int s = sgemm_impl(variant, m, n, 0, A, lda, B, ldb, C[d], ldc, opts, nullptr, d_flags,
                               stream);
      if (s != TCEC_OK) return s;
    }
    return TCEC_OK;
  }
  return sgemm_impl(variant, m, n, k, A, lda, B, ldb, C[0], ldc, opts, &ex, d_flags, stream);
}

int tcec_sgemm_host(int variant, int64_t m, int64_t n, int64_t k, const float* A, int64_t lda,
                    const float* B, int64_t ldb, float* C, int64_t ldc, const tcec_opts* opts,
                    uint32_t* h_flags, void* stream) {
  // Host buffers.  C is computed in R x Cb blocks (rows multiple of the 256-row
  // pair tile, columns of the 256-column tile).  The inputs go up in the order
  // A_0, B_0, A_1, B_1, ... (A row blocks contiguous, B column blocks as 2-D
  // copies, which run at full PCIe rate); block (i, j) launches on one of two
  // compute streams as soon as A_i and B_j are resident, and its C block goes
  // down on the copy-out stream as soon as it is done.  So the GEMM starts after
  // 1/R of A and 1/Cb of B instead of after all of B, and the download overlaps
  // the remaining uploads.  Rows and columns are independent, so the result is
  // bit-identical to one launch over the whole product.  Streams, events and
  // device buffers are cached per device (HostCtx) across calls.
  if (m < 0 || n < 0 || k < 0) return TCEC_ERR_ARG;
  if (lda < (k > 0 ? k : 1) || ldb < (n > 0 ? n : 1) || ldc < (n > 0 ? n : 1)) return TCEC_ERR_ARG;
  if (h_flags) *h_flags = 0;
  if (m == 0 || n == 0) return TCEC_OK;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return TCEC_ERR_CUDA;
  if (dev < 0 || dev >= kMaxDevices) return TCEC_ERR_CUDA;
  HostCtx& H = g_host[dev];
  std::lock_guard<std::mutex> lk(H.mu);
  int status = TCEC_OK;
  auto cu = [&](cudaError_t e) {
    if (e != cudaSuccess && status == TCEC_OK) status = TCEC_ERR_CUDA;
    return e == cudaSuccess;
  };
  if (!H.ready && !cu(H.init())) return status;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t dlda = ((k > 0 ? k : 1) + 3) / 4 * 4;
  const int64_t dldb = (n + 3) / 4 * 4;
  const int64_t dldc = dldb;
  const int64_t kk = k > 0 ? k : 1;
  // blocking (automatic): up to 8 row blocks and 8 (TF32) / 4 (FP16, whose GEMM
  // is shorter than the upload) column blocks of >= 2048; measured at 16384^3
  // (DESIGN.md 5): TF32 e2e 57.2 -> 48.8 ms against row blocks only, FP16 46.3 -> 45.4
  auto blocks = [](int64_t extent, int requested, int cap) {
    int64_t nb = requested > 0 ? requested : (extent + 2047) / 2048;
    if (requested <= 0 && nb > cap) nb = cap;
    if (nb > HostCtx::kMaxBlk) nb = HostCtx::kMaxBlk;
    if (nb < 1) nb = 1;
    int64_t sz = ((extent + nb - 1) / nb + 255) / 256 * 256;
    return sz < 256 ? int64_t(256) : sz;
  };
  // The blocks run on two concurrent streams: keep them on the per-tile kernel
  // (the persistent lock-step kernel assumes it has the GPU to itself).
  tcec_opts bo;
  memset(&bo, 0, sizeof(bo));
  bo.split_rounding = TCEC_ROUND_DEFAULT;
  bo.scale_log2 = -1;
  if (opts) bo = *opts;
  if (bo.kernel_variant == 0) bo.kernel_variant = 4;
  const int64_t rb = blocks(m, opts ? opts->host_row_blocks : 0, 8);
  const int64_t cbk = blocks(n, opts ? opts->host_col_blocks : 0, variant == TCEC_FP16 ? 4 : 8);
  const int R = static_cast<int>((m + rb - 1) / rb);
  const int Cb = static_cast<int>((n + cbk - 1) / cbk);
  bool ok = cu(H.reserve(size_t(m) * dlda, size_t(kk) * dldb, size_t(m) * dldc)) &&
            cu(cudaMemsetAsync(H.dF, 0, sizeof(uint32_t), st)) &&
            cu(cudaEventRecord(H.ev_start, st));
  float* const dA = H.dA;
  float* const dB = H.dB;
  float* const dC = H.dC;
  for (cudaStream_t x : {H.s_in, H.s_out, H.s_c[0], H.s_c[1]})
    if (ok) ok = cu(cudaStreamWaitEvent(x, H.ev_start, 0));  // prior work on `stream`
  // uploads, interleaved A_0 B_0 A_1 B_1 ...
  for (int s = 0; ok && s < (R > Cb ? R : Cb); ++s) {
    if (s < R) {
      const int64_t r0 = s * rb, rows = (r0 + rb <= m) ? rb : m - r0;
      if (k > 0)
        ok = cu(cudaMemcpy2DAsync(dA + r0 * dlda, dlda * sizeof(float), A + r0 * lda,
                                  lda * sizeof(float), k * sizeof(float), rows,
                                  cudaMemcpyHostToDevice, H.s_in));
      ok = ok && cu(cudaEventRecord(H.ev_a[s], H.s_in));
    }
    if (ok && s < Cb) {
      const int64_t c0 = s * cbk, cols = (c0 + cbk <= n) ? cbk : n - c0;
      if (k > 0)
        ok = cu(cudaMemcpy2DAsync(dB + c0, dldb * sizeof(float), B + c0, ldb * sizeof(float),
                                  cols * sizeof(float), k, cudaMemcpyHostToDevice, H.s_in));
      ok = ok && cu(cudaEventRecord(H.ev_b[s], H.s_in));
    }
  }
  // GEMM blocks in arrival order, downloads as they complete
  int launched = 0;
  for (int s = 0; ok && s < (R > Cb ? R : Cb); ++s) {
    for (int pass = 0; ok && pass < 2; ++pass) {
      // pass 0: row s against columns 0..s; pass 1: rows 0..s-1 against column s
      const int count = pass == 0 ? (s < R ? (s + 1 < Cb ? s + 1 : Cb) : 0) : (s < Cb ? (s < R ? s : R) : 0);
      for (int t = 0; ok && t < count; ++t) {
        const int i = pass == 0 ? s : t, j = pass == 0 ? t : s;
        const int64_t r0 = i * rb, rows = (r0 + rb <= m) ? rb : m - r0;
        const int64_t c0 = j * cbk, cols = (c0 + cbk <= n) ? cbk : n - c0;
        cudaStream_t sc = H.s_c[launched & 1];
        ok = cu(cudaStreamWaitEvent(sc, H.ev_a[i], 0)) && cu(cudaStreamWaitEvent(sc, H.ev_b[j], 0));
        if (!ok) break;
        const int s2 = tcec_sgemm(variant, rows, cols, k, dA + r0 * dlda, dlda, dB + c0, dldb,
                                  dC + r0 * dldc + c0, dldc, &bo, H.dF, sc);
        if (s2 != TCEC_OK) {
          status = s2;
          ok = false;
          break;
        }
        cudaEvent_t eg = H.ev_g[launched];
        ok = cu(cudaEventRecord(eg, sc)) && cu(cudaStreamWaitEvent(H.s_out, eg, 0)) &&
             cu(cudaMemcpy2DAsync(C + r0 * ldc + c0, ldc * sizeof(float), dC + r0 * dldc + c0,
                                  dldc * sizeof(float), cols * sizeof(float), rows,
                                  cudaMemcpyDeviceToHost, H.s_out));
        ++launched;
      }
    }
  }
  if (ok && h_flags)  // s_out has waited on every block's GEMM
    cu(cudaMemcpyAsync(h_flags, H.dF, sizeof(uint32_t), cudaMemcpyDeviceToHost, H.s_out));
  for (cudaStream_t x : {H.s_out, H.s_in, H.s_c[0], H.s_c[1]}) cu(cudaStreamSynchronize(x));
  return status;
}

int tcec_host_release(void) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return TCEC_ERR_CUDA;
  if (dev < 0 || dev >= kMaxDevices) return TCEC_ERR_CUDA;
  HostCtx& H = g_host[dev];
  std::lock_guard<std::mutex> lk(H.mu);
  return H.release() == cudaSuccess ? TCEC_OK : TCEC_ERR_CUDA;
}

int tcec_split_census(int kind, int rounding, int e_v, unsigned long long* d_counts,
                      void* stream) {
  if (kind != TCEC_CENSUS_KEPT_LENGTH && kind != TCEC_CENSUS_UNDERFLOW) return TCEC_ERR_ARG;
  if (d_counts == nullptr) return TCEC_ERR_ARG;
  if (rounding == TCEC_ROUND_DEFAULT) rounding = TCEC_ROUND_RN;
  if (rounding != TCEC_ROUND_RN && rounding != TCEC_ROUND_RNA && rounding != TCEC_ROUND_RZ)
    return TCEC_ERR_ARG;
  if (kind == TCEC_CENSUS_KEPT_LENGTH && e_v != 0) return TCEC_ERR_UNSUPPORTED;
  if (e_v < -126 || e_v > 127) return TCEC_ERR_ARG;
  int s;
  if ((s = check_arch())) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const unsigned grid = (1u << 23) / 256u;
  if (kind == TCEC_CENSUS_UNDERFLOW)
    tcec::tcec_census_kernel<1, tcec::kRZ><<<grid, 256, 0, st>>>(e_v, d_counts);
  else if (rounding == TCEC_ROUND_RN)
    tcec::tcec_census_kernel<0, tcec::kRN><<<grid, 256, 0, st>>>(0, d_counts);
  else if (rounding == TCEC_ROUND_RNA)
    tcec::tcec_census_kernel<0, tcec::kRNA><<<grid, 256, 0, st>>>(0, d_counts);
  else
    tcec::tcec_census_kernel<0, tcec::kRZ><<<grid, 256, 0, st>>>(0, d_counts);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError() == cudaSuccess ? TCEC_OK : TCEC_ERR_CUDA;
}

int tcec_split(int variant, int rounding, int scale_log2, const float* X, int64_t count,
               float* hi, float* lo, uint32_t* d_flags, void* stream) {
  if (variant != TCEC_FP16 && variant != TCEC_TF32) return TCEC_ERR_ARG;
  if (count < 0) return TCEC_ERR_ARG;
  if (count == 0) return TCEC_OK;
  rounding = resolve_rounding(variant, rounding);
  if (!rounding_supported(variant, rounding)) return TCEC_ERR_UNSUPPORTED;
  if (scale_log2 < 0) scale_log2 = variant == TCEC_FP16 ? 11 : 0;
  if (variant == TCEC_TF32 && scale_log2 != 0) return TCEC_ERR_UNSUPPORTED;
  if (variant == TCEC_FP16 && scale_log2 != 0 && scale_log2 != 11) return TCEC_ERR_UNSUPPORTED;
  int s;
  if ((s = check_arch())) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (variant == TCEC_FP16) {
    if (rounding == TCEC_ROUND_RN)
      return launch_split<tcec::kFP16, tcec::kRN>(X, count, scale_log2, hi, lo, d_flags, st);
    if (rounding == TCEC_ROUND_RZ)
      return launch_split<tcec::kFP16, tcec::kRZ>(X, count, scale_log2, hi, lo, d_flags, st);
    return TCEC_ERR_UNSUPPORTED;
  }
  if (rounding == TCEC_ROUND_RNA)
    return launch_split<tcec::kTF32, tcec::kRNA>(X, count, 0, hi, lo, d_flags, st);
  if (rounding == TCEC_ROUND_RN)
    return launch_split<tcec::kTF32, tcec::kRN>(X, count, 0, hi, lo, d_flags, st);
  if (rounding == TCEC_ROUND_RZ)
    return launch_split<tcec::kTF32, tcec::kRZ>(X, count, 0, hi, lo, d_flags, st);
  return TCEC_ERR_UNSUPPORTED;
}

}  // extern "C"
