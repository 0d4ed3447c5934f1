/*
 * The C ABI without Python or PyTorch: a 24^3 Cartesian heat-equation problem
 * (configs[0]'s recipe at a smaller size: isotropic constant diffusivity, zero-flux
 * walls) advanced by RKL2 (Fig. 2) and by backward Euler + Jacobi-PCG
 * (Fig. 1) through include/sts_b200.h on device arrays from cudaMalloc.
 * Checks: the volume-weighted total is conserved by both advances (uniform cells:
 * the plain sum) and, at dt = 5 dt_Euler, the two agree to BE's first-order error.
 *
 *   gcc -O2 examples/c_abi_demo.c -Iinclude -I/usr/local/cuda/include \
 *       -Lpaper_1610_01265_b200 -lsts_b200 -L/usr/local/cuda/lib64 -lcudart -lm \
 *       -Wl,-rpath,$PWD/paper_1610_01265_b200 -o c_abi_demo && ./c_abi_demo
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "sts_b200.h"

#define CHECK(call)                                                                 \
  do {                                                                              \
    int rc_ = (call);                                                               \
    if (rc_ != STS_OK) {                                                            \
      fprintf(stderr, "%s failed (%d): %s\n", #call, rc_, sts_last_error());        \
      return 1;                                                                     \
    }                                                                               \
  } while (0)

static double total(const double* d, size_t n) {
  double* h = (double*)malloc(n * sizeof(double));
  cudaMemcpy(h, d, n * sizeof(double), cudaMemcpyDeviceToHost);
  double s = 0.0;
  for (size_t i = 0; i < n; ++i) s += h[i];
  free(h);
  return s;
}

int main(void) {
  enum { N = 24 };
  const size_t n = (size_t)N * N * N;
  double xf[N + 1], xc[N];
  for (int i = 0; i <= N; ++i) xf[i] = i;
  for (int i = 0; i < N; ++i) xc[i] = i + 0.5;
  sts_grid* g = NULL;
  CHECK(sts_grid_create(&g, STS_GEOM_CARTESIAN, N, N, N, xf, xc, xf, xc, xf, xc, 0, 0, N, 1, 0));

  double* h = (double*)malloc(n * sizeof(double));
  double *u, *k1, *k2, *k3, *urk, *ube;
  cudaMalloc((void**)&u, n * sizeof(double));
  cudaMalloc((void**)&k1, n * sizeof(double));
  cudaMalloc((void**)&k2, n * sizeof(double));
  cudaMalloc((void**)&k3, n * sizeof(double));
  cudaMalloc((void**)&urk, n * sizeof(double));
  cudaMalloc((void**)&ube, n * sizeof(double));
  for (size_t e = 0; e < n; ++e) h[e] = 1.0;                 /* constant face diffusivity */
  cudaMemcpy(k1, h, n * sizeof(double), cudaMemcpyHostToDevice);
  cudaMemcpy(k2, h, n * sizeof(double), cudaMemcpyHostToDevice);
  cudaMemcpy(k3, h, n * sizeof(double), cudaMemcpyHostToDevice);
  for (int i = 0; i < N; ++i)                                /* Gaussian bump, sigma = 3 cells */
    for (int j = 0; j < N; ++j)
      for (int k = 0; k < N; ++k) {
        const double r2 = (xc[i] - 12) * (xc[i] - 12) + (xc[j] - 12) * (xc[j] - 12) + (xc[k] - 12) * (xc[k] - 12);
        h[((size_t)i * N + j) * N + k] = exp(-r2 / 18.0);
      }
  cudaMemcpy(u, h, n * sizeof(double), cudaMemcpyHostToDevice);

  double dte = 0.0;
  CHECK(sts_dt_euler(g, STS_MODE_ISO, k1, k2, k3, NULL, NULL, &dte, NULL));
  const double dt = 5.0 * dte;   /* BE is first order: compare the two at a moderate step */
  const int s = rkl2_num_stages(dt, dte, 0);
  int iters = 0;
  CHECK(rkl2_advance(g, STS_MODE_ISO, 1, u, urk, k1, k2, k3, NULL, NULL, dt, s, NULL));
  CHECK(be_pcg_solve(g, STS_MODE_ISO, 1, u, ube, k1, k2, k3, NULL, NULL, dt, 1e-12, 10000, &iters, NULL));
  cudaDeviceSynchronize();

  const double t0 = total(u, n), trk = total(urk, n), tbe = total(ube, n);
  double* a = (double*)malloc(n * sizeof(double));
  double* b = (double*)malloc(n * sizeof(double));
  cudaMemcpy(a, urk, n * sizeof(double), cudaMemcpyDeviceToHost);
  cudaMemcpy(b, ube, n * sizeof(double), cudaMemcpyDeviceToHost);
  double d2 = 0.0, n2 = 0.0;
  for (size_t e = 0; e < n; ++e) {
    d2 += (a[e] - b[e]) * (a[e] - b[e]);
    n2 += a[e] * a[e];
  }
  const double rel = sqrt(d2 / n2);
  printf("dt_euler %.6g  s %d  PCG iterations %d  total %.15g -> RKL2 %.15g, BE %.15g  |RKL2-BE|/|RKL2| %.3g\n",
         dte, s, iters, t0, trk, tbe, rel);
  const int ok = fabs(trk - t0) <= 1e-12 * t0 && fabs(tbe - t0) <= 1e-10 * t0 && rel < 0.05 && iters > 0;
  CHECK(sts_grid_destroy(g));
  printf(ok ? "c_abi_demo ok\n" : "c_abi_demo FAILED\n");
  return ok ? 0 : 1;
}
