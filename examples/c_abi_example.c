/* The C ABI without Python: flat-depth RGB (one level, and the smoothed
 * three-level pyramid of K7), a static press force field and the
 * InvalidQuery status through libtacsl_b200.so, checked against closed-form
 * answers (render/lut.py:52-54: flat depth -> the LUT's background colour at
 * every level; tactile/field.py:61-76: a taxel pressed d = -1 mm into a
 * plane with k_n = 1000 N/m feels |f_n| = 1 N; geometry/sdf.py:324-328:
 * an out-of-grid query -> InvalidQuery).
 *
 *   gcc -O2 -I include -I /usr/local/cuda/include examples/c_abi_example.c \
 *       -L paper_2408_06506_b200 -ltacsl_b200 -L /usr/local/cuda/lib64 -lcudart \
 *       -lm -Wl,-rpath,$PWD/paper_2408_06506_b200 -o /tmp/c_abi_example && /tmp/c_abi_example
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "tacsl_b200.h"

#define CHECK(x)                                                              \
  do {                                                                        \
    int rc_ = (x);                                                            \
    if (rc_) {                                                                \
      fprintf(stderr, "%s failed: %d %s\n", #x, rc_, tacsl_last_error());     \
      return 1;                                                               \
    }                                                                         \
  } while (0)

int main(void) {
  if (!tacsl_device_supported(0)) {
    fprintf(stderr, "no sm_100 device\n");
    return 2;
  }
  /* ---- RGB: 3 flat 60x80 depth maps -> every pixel = background colour */
  const int W = 80, H = 60, N = 3, T = 6;
  double coeffs[3 * 6] = {0};
  const double bg[3] = {0.35, 0.38, 0.45};
  for (int c = 0; c < 3; ++c) {
    coeffs[c * T + 0] = bg[c];
    coeffs[c * T + 1] = 3.5;  /* gradient terms vanish on a flat map */
    coeffs[c * T + 2] = -1.5;
  }
  tacsl_lut_t lut;
  CHECK(tacsl_lut_create(coeffs, 2, W, H, &lut));
  float* h_depth = (float*)malloc(sizeof(float) * N * H * W);
  for (int i = 0; i < N * H * W; ++i) h_depth[i] = 0.022f;
  float* d_depth;
  unsigned char* d_rgb;
  cudaMalloc((void**)&d_depth, sizeof(float) * N * H * W);
  cudaMalloc((void**)&d_rgb, (size_t)N * H * W * 3);
  cudaMemcpy(d_depth, h_depth, sizeof(float) * N * H * W, cudaMemcpyHostToDevice);
  CHECK(tacsl_depth_to_rgb(lut, d_depth, N, H, W, d_rgb, NULL, NULL));
  unsigned char* h_rgb = (unsigned char*)malloc((size_t)N * H * W * 3);
  cudaMemcpy(h_rgb, d_rgb, (size_t)N * H * W * 3, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < N * H * W; ++i)
    for (int c = 0; c < 3; ++c) bad += h_rgb[3 * i + c] != (unsigned char)lrint(bg[c] * 255.0);
  printf("rgb: %d of %d channel values differ from the background colour\n", bad, N * H * W * 3);
  /* wrong resolution -> LUT_RESOLUTION_MISMATCH (lut.py:70-74) */
  if (tacsl_depth_to_rgb(lut, d_depth, N, H + 1, W, d_rgb, NULL, NULL) != TACSL_ERR_LUT_RESOLUTION_MISMATCH) {
    fprintf(stderr, "expected LUT_RESOLUTION_MISMATCH\n");
    return 1;
  }

  /* ---- K7: sigma = 1 smoothing + a 3-level RGB pyramid of the same flat
   * maps: every level is the background colour too */
  tacsl_lut_t luts[3];
  unsigned char* d_lvl[3];
  int bad_pyr = 0;
  for (int l = 0; l < 3; ++l) {
    CHECK(tacsl_lut_create(coeffs, 2, W >> l, H >> l, &luts[l]));
    cudaMalloc((void**)&d_lvl[l], (size_t)N * (H >> l) * (W >> l) * 3);
  }
  const float taps[9] = {0.00013383f, 0.00443305f, 0.05399100f, 0.24197072f, 0.39894353f,
                         0.24197072f, 0.05399100f, 0.00443305f, 0.00013383f};
  if (!tacsl_rgb_pyramid_supported(H, W, 4, 3)) {
    fprintf(stderr, "pyramid shape not supported\n");
    return 1;
  }
  CHECK(tacsl_rgb_pyramid(luts, 3, d_depth, N, H, W, taps, 4, d_lvl, NULL));
  for (int l = 0; l < 3; ++l) {
    const size_t np = (size_t)N * (H >> l) * (W >> l);
    unsigned char* h = (unsigned char*)malloc(np * 3);
    cudaMemcpy(h, d_lvl[l], np * 3, cudaMemcpyDeviceToHost);
    for (size_t i = 0; i < np; ++i)
      for (int c = 0; c < 3; ++c) bad_pyr += h[3 * i + c] != (unsigned char)lrint(bg[c] * 255.0);
    free(h);
    cudaFree(d_lvl[l]);
    tacsl_lut_destroy(luts[l]);
  }
  printf("pyramid: %d channel values differ from the background colour over 3 levels\n", bad_pyr);

  /* ---- force field: a plane z <= 0 as an SDF (d = z, grad = +z), one taxel
   * at the sensor origin, sensor 1 mm below the surface, at rest */
  const int n = 8;
  const int dims[3] = {n, n, n};
  const double spacing = 0.002, origin[3] = {-0.007, -0.007, -0.007};
  double* values = (double*)malloc(sizeof(double) * n * n * n);
  double* grads = (double*)malloc(sizeof(double) * n * n * n * 3);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      for (int k = 0; k < n; ++k) {
        const size_t c = ((size_t)i * n + j) * n + k;
        values[c] = origin[2] + spacing * k; /* z of the cell */
        grads[3 * c] = 0.0;
        grads[3 * c + 1] = 0.0;
        grads[3 * c + 2] = 1.0;
      }
  tacsl_sdf_t sdf;
  CHECK(tacsl_sdf_create(0, values, grads, dims, origin, spacing, &sdf));
  const double taxel[3] = {0.0, 0.0, 0.0};
  /* state = pos[3], quat(w,x,y,z)[4], v[3], w[3] */
  const double obj[13] = {0, 0, 0, 1, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  const double sen[13] = {0, 0, -0.001, 1, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  double *d_tax, *d_obj, *d_sen, *d_fn, *d_ft, *d_w;
  cudaMalloc((void**)&d_tax, sizeof taxel);
  cudaMalloc((void**)&d_obj, sizeof obj);
  cudaMalloc((void**)&d_sen, sizeof sen);
  cudaMalloc((void**)&d_fn, 3 * sizeof(double));
  cudaMalloc((void**)&d_ft, 3 * sizeof(double));
  cudaMalloc((void**)&d_w, 6 * sizeof(double));
  cudaMemcpy(d_tax, taxel, sizeof taxel, cudaMemcpyHostToDevice);
  cudaMemcpy(d_obj, obj, sizeof obj, cudaMemcpyHostToDevice);
  cudaMemcpy(d_sen, sen, sizeof sen, cudaMemcpyHostToDevice);
  const tacsl_penalty_t p = {1000.0, 100.0, 10.0, 2.0};
  CHECK(tacsl_force_field(sdf, d_tax, 1, 1, d_obj, 13, d_sen, 13, 1, 1, p, /*out_fp64=*/1, d_fn, d_ft, d_w, NULL,
                          NULL, NULL, NULL));
  double fn[3], wr[6];
  cudaMemcpy(fn, d_fn, sizeof fn, cudaMemcpyDeviceToHost);
  cudaMemcpy(wr, d_w, sizeof wr, cudaMemcpyDeviceToHost);
  printf("force field: f_n = (%.6f, %.6f, %.6f) N, wrench force z = %.6f N\n", fn[0], fn[1], fn[2], wr[2]);
  /* ---- relative_penetration_rate: one query outside the grid -> InvalidQuery */
  const double nrm[6] = {0, 0, 1, 0, 0, 1}, xd[3] = {0, 0, -0.01};
  const unsigned char valid[2] = {1, 0};
  double *d_n, *d_x, *d_rate;
  unsigned char* d_valid;
  int* d_flag;
  cudaMalloc((void**)&d_n, sizeof nrm);
  cudaMalloc((void**)&d_x, sizeof xd);
  cudaMalloc((void**)&d_rate, 2 * sizeof(double));
  cudaMalloc((void**)&d_valid, 2);
  cudaMalloc((void**)&d_flag, sizeof(int));
  cudaMemcpy(d_n, nrm, sizeof nrm, cudaMemcpyHostToDevice);
  cudaMemcpy(d_x, xd, sizeof xd, cudaMemcpyHostToDevice);
  cudaMemcpy(d_valid, valid, 2, cudaMemcpyHostToDevice);
  const int rc_bad = tacsl_relative_penetration_rate(d_n, d_valid, d_x, 2, 1, d_rate, d_flag, NULL);
  const int rc_ok = tacsl_relative_penetration_rate(d_n, d_valid, d_x, 1, 1, d_rate, d_flag, NULL);
  double rate;
  cudaMemcpy(&rate, d_rate, sizeof rate, cudaMemcpyDeviceToHost);
  printf("penetration rate: status %d for an out-of-grid query (INVALID_QUERY = %d), d_dot = %.3f\n", rc_bad,
         TACSL_ERR_INVALID_QUERY, rate);
  const int ok = bad == 0 && bad_pyr == 0 && fabs(fn[2] - 1.0) < 1e-9 && fabs(wr[2] - 1.0) < 1e-9 &&
                 rc_bad == TACSL_ERR_INVALID_QUERY && rc_ok == TACSL_OK && fabs(rate + 0.01) < 1e-15;
  tacsl_lut_destroy(lut);
  tacsl_sdf_destroy(sdf);
  printf(ok ? "ok\n" : "FAILED\n");
  return ok ? 0 : 1;
}
