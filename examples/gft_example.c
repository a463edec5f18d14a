/* gft_example.c -- using the C ABI of include/gft.h from plain C (no Python, no torch).
 *
 * Builds the fast-GFT plan of an n-node cycle (a reflection symmetry at
 * every level), transforms a batch of signals on the GPU and back, checks the round trip,
 * Parseval's identity and the lowest coefficient of a constant signal, saves and reloads
 * the plan (gft_plan_serialize / _deserialize: bit-identical forward), and prints the plan
 * shape.  Device memory comes from the CUDA runtime; the library itself only needs a
 * current CUDA context (gft_forward runs on the given stream, NULL = legacy default).
 *
 *   build : gcc -O2 -std=c11 -I include examples/gft_example.c \
 *               -L paper_1907_07875_b200/_lib -lgft -L /usr/local/cuda/lib64 -lcudart \
 *               -Wl,-rpath,$PWD/paper_1907_07875_b200/_lib -Wl,-rpath,/usr/local/cuda/lib64 -lm
 *   run   : ./gft_example [n] [batch]        (exit 0 = all checks passed)
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "gft.h"

#define CHECK_GFT(call)                                                                  \
  do {                                                                                   \
    gft_status st_ = (call);                                                             \
    if (st_ != GFT_OK) {                                                                 \
      fprintf(stderr, "%s failed: %s (%s)\n", #call, gft_status_str(st_), gft_last_error()); \
      return 2;                                                                          \
    }                                                                                    \
  } while (0)
#define CHECK_CUDA(call)                                                                 \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess) {                                                             \
      fprintf(stderr, "%s failed: %s\n", #call, cudaGetErrorString(e_));                 \
      return 3;                                                                          \
    }                                                                                    \
  } while (0)

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 64;
  const long long batch = argc > 2 ? atoll(argv[2]) : 100000;
  if (n < 3 || n > 256 || batch < 1) {
    fprintf(stderr, "usage: %s [n in 3..256] [batch >= 1]\n", argv[0]);
    return 1;
  }
  /* the cycle 0-1-...-(n-1)-0 with unit weights */
  int32_t* src = malloc(sizeof(int32_t) * n);
  int32_t* dst = malloc(sizeof(int32_t) * n);
  double* w = malloc(sizeof(double) * n);
  for (int i = 0; i < n; ++i) {
    src[i] = i;
    dst[i] = (i + 1) % n;
    w[i] = 1.0;
  }
  gft_plan_opts opts;
  gft_plan_opts_default(&opts);
  opts.dtypes = 1u << GFT_F32;
  gft_plan plan;
  CHECK_GFT(gft_plan_create(&plan, n, n, src, dst, w, NULL, NULL, &opts));
  gft_plan_info info;
  CHECK_GFT(gft_plan_info_get(plan, &info));
  printf("cycle n=%d: %d butterfly levels, %d Haar units, %d leaves (max %d), adds %lld vs dense %lld\n",
         n, info.depth, info.n_units, info.n_leaves, info.max_leaf, (long long)info.adds,
         (long long)info.dense_adds);

  /* signals: row 0 constant (its GFT is concentrated in coefficient 0, lambda = 0),
   * the rest pseudo-random */
  const size_t count = (size_t)batch * n;
  float* hx = malloc(sizeof(float) * count);
  float* hy = malloc(sizeof(float) * count);
  float* hz = malloc(sizeof(float) * count);
  unsigned int seed = 12345u;
  for (size_t i = 0; i < count; ++i) {
    seed = seed * 1664525u + 1013904223u;
    hx[i] = i < (size_t)n ? 1.0f : (float)((seed >> 8) * (1.0 / 16777216.0) - 0.5);
  }
  float *dx, *dy;
  CHECK_CUDA(cudaMalloc((void**)&dx, sizeof(float) * count));
  CHECK_CUDA(cudaMalloc((void**)&dy, sizeof(float) * count));
  CHECK_CUDA(cudaMemcpy(dx, hx, sizeof(float) * count, cudaMemcpyHostToDevice));
  CHECK_GFT(gft_forward(plan, dx, dy, batch, GFT_F32, NULL));
  CHECK_CUDA(cudaMemcpy(hy, dy, sizeof(float) * count, cudaMemcpyDeviceToHost));
  CHECK_GFT(gft_inverse(plan, dy, dx, batch, GFT_F32, NULL));   /* back into dx */
  CHECK_CUDA(cudaMemcpy(hz, dx, sizeof(float) * count, cudaMemcpyDeviceToHost));

  /* measured tuning of the forward kernel (geometry + request pacing, timed on dx -> dy);
   * the arithmetic is unchanged, so the reloaded plan below must still reproduce hy bit for
   * bit -- and it carries the tuning in its serialised bytes */
  int32_t choice[16];
  CHECK_GFT(gft_plan_tune(plan, GFT_F32, 1u, GFT_TUNE_GEOMETRY, dx, dy, batch, 3, NULL, choice));
  printf("tuned forward kernel: R %d, stages %d, warps %d, pace %d ns\n", choice[0], choice[1], choice[2],
         choice[3]);

  /* plan persistence: serialise (size query first), reload, and the reloaded plan's
   * forward must be bit-identical (same decomposition -> same generated kernel) */
  size_t blob_size = 0;
  CHECK_GFT(gft_plan_serialize(plan, NULL, 0, &blob_size));
  void* blob = malloc(blob_size);
  CHECK_GFT(gft_plan_serialize(plan, blob, blob_size, &blob_size));
  gft_plan plan2;
  CHECK_GFT(gft_plan_deserialize(&plan2, blob, blob_size, &opts));
  free(blob);
  float* hw = malloc(sizeof(float) * count);
  CHECK_CUDA(cudaMemcpy(dy, hx, sizeof(float) * count, cudaMemcpyHostToDevice));
  CHECK_GFT(gft_forward(plan2, dy, dy, batch, GFT_F32, NULL));   /* in place */
  CHECK_CUDA(cudaMemcpy(hw, dy, sizeof(float) * count, cudaMemcpyDeviceToHost));
  size_t mismatches = 0;
  for (size_t i = 0; i < count; ++i) mismatches += memcmp(&hw[i], &hy[i], sizeof(float)) != 0;
  CHECK_GFT(gft_plan_destroy(plan2));
  free(hw);
  printf("plan saved (%zu bytes) and reloaded: %zu mismatching outputs\n", blob_size, mismatches);

  double worst_rt = 0, worst_parseval = 0;
  for (long long b = 0; b < batch; ++b) {
    double nx = 0, ny = 0, nd = 0;
    for (int i = 0; i < n; ++i) {
      const size_t k = (size_t)b * n + i;
      nx += (double)hx[k] * hx[k];
      ny += (double)hy[k] * hy[k];
      nd += ((double)hz[k] - hx[k]) * ((double)hz[k] - hx[k]);
    }
    if (sqrt(nd / nx) > worst_rt) worst_rt = sqrt(nd / nx);
    if (fabs(sqrt(ny / nx) - 1.0) > worst_parseval) worst_parseval = fabs(sqrt(ny / nx) - 1.0);
  }
  /* constant signal: y_0 = sqrt(n) (u_0 = 1/sqrt(n), sign rule: first entry positive) */
  double rest = 0;
  for (int i = 1; i < n; ++i) rest += (double)hy[i] * hy[i];
  const double c0_err = fabs(hy[0] - sqrt((double)n)) + sqrt(rest);
  printf("round trip max rel err %.2e, Parseval max dev %.2e, constant-signal error %.2e\n",
         worst_rt, worst_parseval, c0_err);
  const int ok = worst_rt < 2e-5 && worst_parseval < 1e-5 && c0_err < 1e-4 * sqrt((double)n) && mismatches == 0;

  cudaFree(dx);
  cudaFree(dy);
  free(hx); free(hy); free(hz); free(src); free(dst); free(w);
  CHECK_GFT(gft_plan_destroy(plan));
  printf("%s\n", ok ? "OK" : "FAILED");
  return ok ? 0 : 4;
}
