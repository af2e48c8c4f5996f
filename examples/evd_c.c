/*
 * examples/evd_c.c -- the C ABI (include/jsvd.h) used from plain C, without
 * Python or torch: a batch of complex Hermitian 2x2 EVDs (Alg 2.3 of the
 * paper) on device buffers, then the same batch through the host-buffer entry
 * point, and a check that both give the same bits and satisfy A = U L U^H.
 *
 * build: gcc -O2 -std=c11 examples/evd_c.c -Iinclude -I/usr/local/cuda/include \
 *          -Lpaper_2202_08361_b200 -ljsvd -L/usr/local/cuda/lib64 -lcudart -lm \
 *          -Wl,-rpath,$PWD/paper_2202_08361_b200 -o evd_c
 * run:   ./evd_c [r]
 */
#include <cuda_runtime_api.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "jsvd.h"

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));                  \
      return 1;                                                                 \
    }                                                                           \
  } while (0)
#define JK(x)                                                                   \
  do {                                                                          \
    jsvd_status s_ = (x);                                                       \
    if (s_ != JSVD_OK) {                                                        \
      fprintf(stderr, "%s: %s\n", #x, jsvd_status_string(s_));                 \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

int main(int argc, char **argv)
{
  const int64_t r = argc > 1 ? atoll(argv[1]) : 100003;
  double *h[9], *d[9];
  for (int k = 0; k < 9; ++k) {
    h[k] = (double *)malloc(sizeof(double) * r);
    CK(cudaMalloc((void **)&d[k], sizeof(double) * r));
  }
  int32_t *hz = (int32_t *)malloc(4 * r), *dz;
  CK(cudaMalloc((void **)&dz, 4 * r));
  srand(7);
  for (int64_t l = 0; l < r; ++l)
    for (int k = 0; k < 4; ++k)  /* a11, a22, re a21, im a21 over a wide exponent range */
      h[k][l] = ldexp((double)rand() / RAND_MAX - 0.5, rand() % 400 - 200);
  for (int k = 0; k < 4; ++k) CK(cudaMemcpy(d[k], h[k], sizeof(double) * r, cudaMemcpyHostToDevice));

  /* device buffers: lam1, lam2, cos, sin (re, im), zeta */
  JK(jsvd_evd2_batched(JSVD_C64, r, d[0], d[1], d[2], d[3], d[4], d[5], d[6], d[7], d[8], dz,
                       NULL, 0, NULL));
  CK(cudaDeviceSynchronize());
  for (int k = 4; k < 9; ++k) CK(cudaMemcpy(h[k], d[k], sizeof(double) * r, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hz, dz, 4 * r, cudaMemcpyDeviceToHost));

  /* the same through the host-buffer entry point (chunked, three streams) */
  const int64_t chunk = 1 << 15;
  size_t wb = 0;
  JK(jsvd_evd2_host_workspace(JSVD_C64, chunk, &wb));
  void *work;
  CK(cudaMalloc(&work, wb));
  double *o[5];
  for (int k = 0; k < 5; ++k) o[k] = (double *)malloc(sizeof(double) * r);
  JK(jsvd_evd2_batched_host(JSVD_C64, r, h[0], h[1], h[2], h[3], o[0], o[1], o[2], o[3], o[4],
                            NULL, NULL, 0, chunk, work, wb, NULL));
  CK(cudaDeviceSynchronize());
  for (int k = 0; k < 5; ++k)
    if (memcmp(o[k], h[4 + k], sizeof(double) * r)) {
      fprintf(stderr, "host-buffer result differs from the device entry point (stream %d)\n", k);
      return 1;
    }

  /* residual of A = U diag(l1, l2) U^H, U = [[c, -conj(s)], [s, c]], relative to max|a| */
  double worst = 0.0;
  for (int64_t l = 0; l < r; ++l) {
    const double c = h[6][l], sr = h[7][l], si = h[8][l], l1 = h[4][l], l2 = h[5][l];
    const double a11 = c * c * l1 + (sr * sr + si * si) * l2;
    const double a22 = (sr * sr + si * si) * l1 + c * c * l2;
    const double a21r = sr * c * (l1 - l2), a21i = si * c * (l1 - l2);
    const double m = fmax(fmax(fabs(h[0][l]), fabs(h[1][l])), fmax(fabs(h[2][l]), fabs(h[3][l])));
    if (m == 0.0) continue;
    const double e = fmax(fmax(fabs(a11 - h[0][l]), fabs(a22 - h[1][l])),
                          fmax(fabs(a21r - h[2][l]), fabs(a21i - h[3][l]))) / m;
    if (e > worst) worst = e;
  }
  printf("r = %lld complex EVDs: host-buffer path bit-identical; max |A - U L U^H| / max|A| = %.2e\n",
         (long long)r, worst);
  return worst < 1e-14 ? 0 : 1;
}
