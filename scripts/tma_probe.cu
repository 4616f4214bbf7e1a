// TMA load throughput per SM by box shape and element type (measurement aid).
//
// One CTA per SM; thread 0 keeps NS boxes in flight through a shared-memory
// ring (one mbarrier per slot) and walks the boxes of a row-major matrix; the
// kernel reports bytes / time per SM.  The same 128-byte rows are loaded as
// FP32 (32 elements), FP16 (64) or UINT8 (128) boxes with SWIZZLE_128B, so
// the bytes and the shared-memory layout are identical across element types.
//
// build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a \
//          -I paper_2203_03341_b200/csrc scripts/tma_probe.cu -lcuda -o exp_libs/tma_probe
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace tcec::sm100;

constexpr int kMaxSlots = 12;

__global__ void __launch_bounds__(32, 1)
    probe(const __grid_constant__ CUtensorMap tm, int rows_total, int box_rows, int box_bytes,
          int ns, int iters, unsigned long long* out_ns) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bars[kMaxSlots];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < ns; ++s) mbar_init(&bars[s], 1);
  fence_mbar_init();
  const int boxes_per_col = rows_total / box_rows;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 0; i < iters; ++i) {
    const int s = i % ns;
    if (i >= ns) mbar_wait(&bars[s], ((i / ns) - 1) & 1);
    mbar_arrive_expect_tx(&bars[s], box_bytes);
    // box b of this CTA: spread CTAs over the matrix, walk down the rows
    const int b = (blockIdx.x * 7 + i) % boxes_per_col;
    tma_load_2d(smem + s * box_bytes, &tm, &bars[s], 0, b * box_rows);
  }
  for (int i = iters; i < iters + ns; ++i) {
    const int s = i % ns;
    mbar_wait(&bars[s], ((i / ns) - 1) & 1);
  }
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  out_ns[blockIdx.x] = t1 - t0;
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* m, uint64_t* bar,
                                            int32_t c0, int32_t c1, int32_t c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// One FP32 staging slice of the fused GEMM per iteration: an A box of 128 rows
// x 32 floats and B either as four 32 k x 32 n boxes (mode 0, as the kernels
// do) or one 3-D box 32 n x 4 blocks x 32 k (mode 1).
__global__ void __launch_bounds__(32, 1)
    probe_slice(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB2,
                const __grid_constant__ CUtensorMap tB3, int mode, int ns, int iters,
                int a_blocks, int b_blocks, int kslices, unsigned long long* out_ns) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bars[kMaxSlots];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < ns; ++s) mbar_init(&bars[s], 1);
  fence_mbar_init();
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  const int m0 = (blockIdx.x % a_blocks) * 128, n0 = (blockIdx.x % b_blocks) * 128;
  for (int i = 0; i < iters; ++i) {
    const int s = i % ns;
    if (i >= ns) mbar_wait(&bars[s], ((i / ns) - 1) & 1);
    mbar_arrive_expect_tx(&bars[s], 32768);
    uint8_t* dst = smem + s * 32768;
    const int k0 = (i % kslices) * 32;
    tma_load_2d(dst, &tA, &bars[s], k0, m0);
    if (mode == 0) {
      for (int b = 0; b < 4; ++b) tma_load_2d(dst + 16384 + b * 4096, &tB2, &bars[s], n0 + 32 * b, k0);
    } else {
      tma_load_3d(dst + 16384, &tB3, &bars[s], 0, n0 / 32, k0);
    }
  }
  for (int i = iters; i < iters + ns; ++i) {
    const int s = i % ns;
    mbar_wait(&bars[s], ((i / ns) - 1) & 1);
  }
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  out_ns[blockIdx.x] = t1 - t0;
}

int slice_probe(int sms, unsigned long long* d_ns, int M, int K, int N) {
  // A: M x K FP32, B: K x N FP32 (row strides 4K / 4N bytes)
  float *A = nullptr, *B = nullptr;
  cudaMalloc(&A, size_t(M) * K * 4);
  cudaMalloc(&B, size_t(K) * N * 4);
  cudaMemset(A, 0, size_t(M) * K * 4);
  cudaMemset(B, 0, size_t(K) * N * 4);
  struct Fr { float* p; ~Fr() { cudaFree(p); } } fa{A}, fb{B};
  CUtensorMap tA, tB2, tB3;
  const cuuint32_t e2[2] = {1, 1}, e3[3] = {1, 1, 1};
  { const cuuint64_t d[2] = {cuuint64_t(K), cuuint64_t(M)}; const cuuint64_t st[1] = {cuuint64_t(K) * 4};
    const cuuint32_t bx[2] = {32, 128};
    if (cuTensorMapEncodeTiled(&tA, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, A, d, st, bx, e2, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)) return 1; }
  { const cuuint64_t d[2] = {cuuint64_t(N), cuuint64_t(K)}; const cuuint64_t st[1] = {cuuint64_t(N) * 4};
    const cuuint32_t bx[2] = {32, 32};
    if (cuTensorMapEncodeTiled(&tB2, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, B, d, st, bx, e2, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)) return 2; }
  { const cuuint64_t d[3] = {32, cuuint64_t(N / 32), cuuint64_t(K)};
    const cuuint64_t st[2] = {128, cuuint64_t(N) * 4};
    const cuuint32_t bx[3] = {32, 4, 32};
    if (cuTensorMapEncodeTiled(&tB3, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, B, d, st, bx, e3, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)) return 3; }
  cudaFuncSetAttribute(probe_slice, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int ab : {8})
  for (int mode = 0; mode < 2; ++mode)
    for (int ns : {3, 4, 6}) {
      const int iters = 1024;
      for (int rep = 0; rep < 2; ++rep)
        probe_slice<<<sms, 32, 200 * 1024>>>(tA, tB2, tB3, mode, ns, iters, ab < M / 128 ? ab : M / 128, N / 128 < 32 ? N / 128 : 32, K / 32, d_ns);
      if (cudaDeviceSynchronize() != cudaSuccess) return 4;
      std::vector<unsigned long long> h(sms);
      cudaMemcpy(h.data(), d_ns, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
      double sum = 0; for (auto v : h) sum += v;
      printf("M %5d K %5d N %5d: A row blocks shared by %3d CTAs: slice A 16 KB + B %s, %d slices in flight: %.0f ns per slice per SM (%.1f GB/s per SM)\n",
             M, K, N, sms / ab, mode == 0 ? "4 x 4 KB boxes" : "one 3-D 16 KB box", ns, sum / sms / iters, 32768.0 * iters / (sum / sms));
    }
  return 0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t rows_total = 65536;  // x 128 B = 8 MB: L2-resident after the first pass
  uint8_t* buf = nullptr;
  cudaMalloc(&buf, rows_total * 128 * 2);
  cudaMemset(buf, 1, rows_total * 128 * 2);
  unsigned long long* d_ns = nullptr;
  cudaMalloc(&d_ns, sizeof(unsigned long long) * sms);
  struct Ty { CUtensorMapDataType dt; int esize; const char* name; };
  const Ty types[3] = {{CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, "f32"},
                       {CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, "f16"},
                       {CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, "u8"}};
  for (int sz : {1024, 2048, 4096, 8192, 16384})
    if (int e = slice_probe(sms, d_ns, sz, sz, sz)) { printf("slice probe failed %d\n", e); return 1; }
  return 0;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int pitch_mul : {1}) {  // row pitch 128 B (dense) or 256 B (every other row)
    for (const Ty& ty : types) {
      for (int box_rows : {32, 64, 128, 256}) {
        for (int ns : {4}) {
          const int box_bytes = box_rows * 128;
          if (ns * box_bytes > 200 * 1024) continue;
          CUtensorMap tm;
          const cuuint64_t dims[2] = {cuuint64_t(128 / ty.esize), cuuint64_t(rows_total)};
          const cuuint64_t strides[1] = {cuuint64_t(128 * pitch_mul)};
          const cuuint32_t box[2] = {cuuint32_t(128 / ty.esize), cuuint32_t(box_rows)};
          const cuuint32_t estr[2] = {1, 1};
          CUresult r = cuTensorMapEncodeTiled(&tm, ty.dt, 2, buf, dims, strides, box, estr,
                                              CU_TENSOR_MAP_INTERLEAVE_NONE,
                                              CU_TENSOR_MAP_SWIZZLE_128B,
                                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
          if (r != CUDA_SUCCESS) { printf("encode failed %d\n", int(r)); return 1; }
          const int iters = 4096 * 32 / box_rows;
          for (int rep = 0; rep < 2; ++rep)
            probe<<<sms, 32, 200 * 1024>>>(tm, int(rows_total), box_rows, box_bytes, ns, iters, d_ns);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) { printf("cuda error %s\n", cudaGetErrorString(e)); return 1; }
          std::vector<unsigned long long> h(sms);
          cudaMemcpy(h.data(), d_ns, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
          double mx = 0, sum = 0;
          for (auto v : h) { mx = v > mx ? v : mx; sum += v; }
          const double bytes = double(iters) * box_bytes;
          printf("pitch %3d B  %-3s box %3d rows x 128 B  in-flight %d: per SM %.1f GB/s (mean), total %.2f TB/s\n",
                 128 * pitch_mul, ty.name, box_rows, ns, bytes / (sum / sms), bytes * sms / mx / 1e3);
        }
      }
    }
  }
  return 0;
}
