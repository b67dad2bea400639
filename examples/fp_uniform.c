/* fp_uniform.c -- a C caller of the cyltomo_b200 C-ABI.
 *
 * Forward-projects a uniform cylinder (mu = 1 everywhere) in one view and
 * checks the identity the projector must satisfy for it: the line integral
 * of a constant 1 is the in-support path length, i.e. out_p == out_w for
 * every pixel (both are the in-support sample count times the step, and the
 * trilinear interpolation of a constant is the constant).  Also checks the
 * error path (a null pointer returns CT_ERR_ARG, no crash).
 *
 *   gcc -Iinclude -I/usr/local/cuda/include examples/fp_uniform.c \
 *       -Lpaper_2005_11976_b200 -lcyltomo_b200 -L/usr/local/cuda/lib64 -lcudart -o fp_uniform
 *   LD_LIBRARY_PATH=paper_2005_11976_b200:/usr/local/cuda/lib64 ./fp_uniform
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "cyltomo_b200.h"

#define CHECK(x)                                                                  \
  do {                                                                            \
    int rc_ = (x);                                                                \
    if (rc_ != CT_OK) {                                                           \
      fprintf(stderr, "%s failed: %d (%s)\n", #x, rc_, ct_last_error());         \
      return 1;                                                                   \
    }                                                                             \
  } while (0)

int main(void) {
  if (ct_abi_version() != CT_ABI_VERSION) {
    fprintf(stderr, "ABI mismatch: library %d, header %d\n", ct_abi_version(), CT_ABI_VERSION);
    return 1;
  }
  /* grid: (n_h, n_theta, n_r) = (16, 64, 16), radius 4 mm, height 8 mm, no pose */
  ct_cyl_grid g;
  memset(&g, 0, sizeof g);
  g.n_h = 16; g.n_theta = 64; g.n_r = 16;
  g.radius = 4.0; g.height = 8.0;
  g.rot[0] = g.rot[4] = g.rot[8] = 1.0;
  /* one view of a 48 x 40 detector, 0.2 mm pixels, SOD 200, SDD 400, stage angle 0:
   * source (0, -SOD, 0), pixel (0,0) centre (-u0 p, SDD - SOD, -v0 p), du = (p,0,0),
   * dv = (0,0,p) (cyltomo/geometry.py:257-273); identity pose, so the grid frame is
   * the world frame */
  const int rows = 40, cols = 48;
  const double p = 0.2, u0 = 23.5, v0 = 19.5, sod = 200.0, sdd = 400.0;
  ct_ray_view v = {{0.0, -sod, 0.0}, {-u0 * p, sdd - sod, -v0 * p}, {p, 0.0, 0.0},
                   {0.0, 0.0, p}};
  ct_sampling s = {0.5 * fmin(g.radius / g.n_r, g.height / g.n_h), 1, 0};
  ct_batch b;
  memset(&b, 0, sizeof b);
  b.n_batch = 1; b.det_rows = rows; b.det_cols = cols;

  const size_t nvox = (size_t)g.n_h * g.n_theta * g.n_r, npix = (size_t)rows * cols;
  float* h_mu = (float*)malloc(nvox * sizeof(float));
  for (size_t i = 0; i < nvox; ++i) h_mu[i] = 1.0f;
  float *d_mu, *d_p, *d_w;
  ct_ray_view* d_v;
  if (cudaMalloc((void**)&d_mu, nvox * 4) || cudaMalloc((void**)&d_p, npix * 4) ||
      cudaMalloc((void**)&d_w, npix * 4) || cudaMalloc((void**)&d_v, sizeof v)) {
    fprintf(stderr, "no CUDA device\n");
    return 2;
  }
  cudaMemcpy(d_mu, h_mu, nvox * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(d_v, &v, sizeof v, cudaMemcpyHostToDevice);

  /* the error channel: a null mu is rejected with a status, not a crash */
  if (ct_fp_cyl(NULL, NULL, &g, d_v, &b, &s, d_p, d_w, NULL) != CT_ERR_ARG) {
    fprintf(stderr, "null mu not rejected\n");
    return 1;
  }
  CHECK(ct_fp_cyl(d_mu, NULL, &g, d_v, &b, &s, d_p, d_w, NULL));
  cudaDeviceSynchronize();
  float* h_p = (float*)malloc(npix * 4);
  float* h_w = (float*)malloc(npix * 4);
  cudaMemcpy(h_p, d_p, npix * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(h_w, d_w, npix * 4, cudaMemcpyDeviceToHost);
  int hit = 0, bad = 0;
  double maxw = 0.0;
  for (size_t i = 0; i < npix; ++i) {
    if (h_w[i] > 0.0f) ++hit;
    if (h_p[i] != h_w[i]) ++bad;
    if (h_w[i] > maxw) maxw = h_w[i];
  }
  /* the longest chord is the diameter, 8 mm (+ one step of sampling slack) */
  const int ok = bad == 0 && hit > 0 && maxw <= 2.0 * g.radius + s.step + 1e-6;
  printf("fp_uniform: %d of %zu rays hit, max path %.4f mm, %d pixels with p != w: %s\n", hit,
         npix, maxw, bad, ok ? "OK" : "FAIL");
  cudaFree(d_mu); cudaFree(d_p); cudaFree(d_w); cudaFree(d_v);
  free(h_mu); free(h_p); free(h_w);
  return ok ? 0 : 1;
}
