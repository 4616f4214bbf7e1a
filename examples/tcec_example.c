/* Minimal C caller of the drop-in boundary (include/tcec.h): one TF32-TCEC
 * SGEMM through tcec_sgemm_host (host buffers), checked against a double
 * precision reference on a few rows.  Build (see examples/Makefile):
 *   cc -O2 -I../include tcec_example.c -L../paper_2203_03341_b200 -ltcec -o tcec_example
 * Run: ./tcec_example [n]   (needs an sm_100 GPU) */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "tcec.h"

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 1024;
  float* A = malloc(sizeof(float) * n * n);
  float* B = malloc(sizeof(float) * n * n);
  float* C = malloc(sizeof(float) * n * n);
  if (!A || !B || !C) return 2;
  uint64_t s = 88172645463325252ull;
  for (int64_t i = 0; i < n * n; ++i) {  /* xorshift uniform in [-1, 1) */
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    A[i] = (float)((double)(s >> 11) / 9007199254740992.0 * 2.0 - 1.0);
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    B[i] = (float)((double)(s >> 11) / 9007199254740992.0 * 2.0 - 1.0);
  }
  uint32_t flags = 0;
  const int st = tcec_sgemm_host(TCEC_TF32, n, n, n, A, n, B, n, C, n, NULL, &flags, NULL);
  if (st != TCEC_OK) {
    fprintf(stderr, "tcec_sgemm_host: %s\n", tcec_status_str(st));
    return 1;
  }
  double num = 0.0, den = 0.0;
  for (int64_t i = 0; i < n; i += (n / 16 > 0 ? n / 16 : 1))
    for (int64_t j = 0; j < n; ++j) {
      double ref = 0.0;
      for (int64_t t = 0; t < n; ++t) ref += (double)A[i * n + t] * (double)B[t * n + j];
      num += (ref - C[i * n + j]) * (ref - C[i * n + j]);
      den += ref * ref;
    }
  const double relres = sqrt(num / den);
  printf("tcec %d: TF32-TCEC %lldx%lldx%lld relres vs FP64 %.3e flags %u\n", tcec_version(),
         (long long)n, (long long)n, (long long)n, relres, flags);
  free(A); free(B); free(C);
  return relres < 1e-6 ? 0 : 1;
}
