"""Build a measurement copy of the library whose persistent kernel records
per-operand-stage globaltimer stamps for CTA 0 (split warp, MMA warp, drain
warp) and prints them at exit -- the tool behind profiles/r02/elect/.

usage: pers_timeline_build.py SRC_CSRC_DIR OUT.so
(run scripts/pers_timeline.py with TCEC_LIB=OUT.so on the GPU).  Results of the
instrumented library are correct; only CTA 0 pays for the stamps."""
import os, shutil, subprocess, sys, tempfile

src, out = sys.argv[1], os.path.abspath(sys.argv[2])
tmp = tempfile.mkdtemp()
for f in os.listdir(src):
    if f.endswith((".cu", ".cuh")):
        shutil.copy(os.path.join(src, f), tmp)
p = os.path.join(tmp, "tcec_gemm5.cuh")
s = open(p).read()


def rep(a, b):
    global s
    assert a in s, a[:80]
    s = s.replace(a, b, 1)


rep('#include "tcec_gemm2.cuh"', '#include "tcec_gemm2.cuh"\n#include <cstdio>\n'
    '__device__ __forceinline__ unsigned long long gt_ns() { unsigned long long t; '
    'asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }\n'
    '__device__ unsigned long long g_tl[8][64];')
rep("""      sm100::mbar_wait(&stg_full[s], (gst / C::NSTG) & 1);
      if (sub == 0) sm100::mbar_wait(&op_empty[o], ((g / C::NOP) & 1) ^ 1);""",
    """      const bool dbg = blockIdx.x == 0 && t == 0 && g < 64;
      if (dbg && sub == 0) g_tl[0][g] = gt_ns();
      sm100::mbar_wait(&stg_full[s], (gst / C::NSTG) & 1);
      if (dbg && sub == 0) g_tl[1][g] = gt_ns();
      if (sub == 0) sm100::mbar_wait(&op_empty[o], ((g / C::NOP) & 1) ^ 1);
      if (dbg && sub == 0) g_tl[2][g] = gt_ns();""")
rep("""    sm100::fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) sm100::mbar_arrive_remote(leader_op_full + o * 8);
  }
}""", """    if (blockIdx.x == 0 && t == 0 && g < 64) g_tl[3][g] = gt_ns();
    sm100::fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) sm100::mbar_arrive_remote(leader_op_full + o * 8);
  }
}""")
rep("""          sm100::mbar_wait_cluster(&op_full[o], (g / C::NOP) & 1);
          sm100::tc_fence_after();""", """          if (blockIdx.x == 0 && lane == 0 && g < 64) g_tl[4][g] = gt_ns();
          sm100::mbar_wait_cluster(&op_full[o], (g / C::NOP) & 1);
          sm100::tc_fence_after();
          if (blockIdx.x == 0 && lane == 0 && g < 64) g_tl[5][g] = gt_ns();""")
rep("""  __syncthreads();
  sm100::cluster_sync();
  if (warp == 2) {""", """  __syncthreads();
  sm100::cluster_sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const long long b0 = (long long)g_tl[0][0];
    for (int i = 0; i < 48; ++i)
      printf("stage %2d split: wait_stg %6lld stg_ok %6lld opslot_ok %6lld done %6lld | mma: wait %6lld go %6lld\\n", i,
             (long long)g_tl[0][i] - b0, (long long)g_tl[1][i] - b0, (long long)g_tl[2][i] - b0,
             (long long)g_tl[3][i] - b0, (long long)g_tl[4][i] - b0, (long long)g_tl[5][i] - b0);
  }
  if (warp == 2) {""")
open(p, "w").write(s)
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
subprocess.run(["nvcc", "-O3", "-std=c++17", "-lineinfo", "-gencode", "arch=compute_100a,code=sm_100a",
                "-Xcompiler", "-fPIC", "-I" + os.path.join(root, "include"), "--expt-relaxed-constexpr",
                "-shared", "-o", out, os.path.join(tmp, "tcec_capi.cu"), "-lcudart"], check=True)
print("built", out)
