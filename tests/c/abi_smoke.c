/* C99 client of the C ABI (include/tb_bst.h) with no Python or torch: the
 * binding a C / cgo / JNI host would write.  Reconstructs a constant
 * sinogram through tb_bst (bst_backproject, fourier_bp.py:435-461) and checks
 * the constant-sinogram identity c * coverage (pi c inside the unit circle,
 * 2 c asin(1/r) outside; fourier_bp.py:204-220), then the error path of
 * tb_plan_create (ValueError in BstPlan.__post_init__, fourier_bp.py:88-109).
 * Build: make c_smoke.  Exit status 0 = pass. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime_api.h>

#include <string.h>

#include "tb_bst.h"

#define CHECK(x)                                                             \
  do {                                                                       \
    int rc_ = (x);                                                           \
    if (rc_ != 0) {                                                          \
      fprintf(stderr, "%s:%d %s -> %d (%s)\n", __FILE__, __LINE__, #x, rc_,  \
              tb_last_error());                                              \
      return 1;                                                              \
    }                                                                        \
  } while (0)

int main(void) {
  const int n = 256, V = 256, B = 2;
  const float c = 0.75f;
  if (tb_abi_version() != TB_ABI_VERSION) {
    fprintf(stderr, "ABI version mismatch\n");
    return 1;
  }
  tb_plan_desc d = {n, V, 2, 0, 10.0, 0.1, 1, TB_INTERP_BILINEAR, 0, 0, TB_FILTER_RAMP, 1.0, 0, 0};
  tb_plan* plan = NULL;
  CHECK(tb_plan_create(&d, 0, &plan));
  size_t ws_bytes = 0;
  CHECK(tb_workspace_bytes(plan, B, &ws_bytes));
  const size_t cnt = (size_t)B * V * n;
  float* host = (float*)malloc(cnt * sizeof(float));
  for (size_t i = 0; i < cnt; ++i) host[i] = c;
  float *sino = NULL, *img = NULL;
  void* ws = NULL;
  if (cudaMalloc((void**)&sino, cnt * sizeof(float)) || cudaMalloc((void**)&img, cnt * sizeof(float)) ||
      cudaMalloc(&ws, ws_bytes)) {
    fprintf(stderr, "cudaMalloc failed\n");
    return 1;
  }
  cudaMemcpy(sino, host, cnt * sizeof(float), cudaMemcpyHostToDevice);
  CHECK(tb_reset_status(plan, ws, NULL));
  CHECK(tb_bst(plan, sino, img, B, B, ws, ws_bytes, NULL));
  CHECK(tb_read_status(plan, ws, NULL));
  cudaMemcpy(host, img, cnt * sizeof(float), cudaMemcpyDeviceToHost);
  double worst = 0.0;
  for (int q = 0; q < B; ++q)
    for (int i2 = 0; i2 < n; ++i2)
      for (int i1 = 0; i1 < n; ++i1) {
        const double x1 = -1.0 + (i1 + 0.5) * 2.0 / n, x2 = -1.0 + (i2 + 0.5) * 2.0 / n;
        const double r = sqrt(x1 * x1 + x2 * x2);
        const double expect = r <= 1.0 ? M_PI * c : 2.0 * c * asin(1.0 / r);
        const double e = fabs(host[((size_t)q * n + i2) * n + i1] - expect);
        if (e > worst) worst = e;
      }
  /* the GPU parity test bounds the same identity at 1e-4 of pi c */
  if (!(worst <= 1e-4 * M_PI * c)) {
    fprintf(stderr, "constant-sinogram identity: max abs error %.3e\n", worst);
    return 1;
  }
  /* fused centre / ring stages (tb_pre_params + tb_fbp_pre): beta 0 and the
   * stripes of a constant sinogram (0) leave tb_fbp's result bitwise intact */
  {
    float *shift = NULL, *stripe = NULL, *img2 = NULL;
    double* scratch = NULL;
    if (cudaMalloc((void**)&shift, (size_t)B * 2 * sizeof(float)) ||
        cudaMalloc((void**)&stripe, (size_t)B * n * sizeof(float)) ||
        cudaMalloc((void**)&scratch, (size_t)B * n * sizeof(double)) ||
        cudaMalloc((void**)&img2, cnt * sizeof(float))) {
      fprintf(stderr, "cudaMalloc failed\n");
      return 1;
    }
    CHECK(tb_pre_params(plan, sino, B, NULL, 9, scratch, shift, stripe, NULL));
    CHECK(tb_fbp(plan, sino, img, B, B, ws, ws_bytes, NULL));
    CHECK(tb_fbp_pre(plan, sino, img2, B, B, ws, ws_bytes, shift, stripe, NULL));
    CHECK(tb_read_status(plan, ws, NULL));
    float* h2 = (float*)malloc(cnt * sizeof(float));
    cudaMemcpy(host, img, cnt * sizeof(float), cudaMemcpyDeviceToHost);
    cudaMemcpy(h2, img2, cnt * sizeof(float), cudaMemcpyDeviceToHost);
    if (memcmp(host, h2, cnt * sizeof(float)) != 0) {
      fprintf(stderr, "tb_fbp_pre with zero shift / stripes differs from tb_fbp\n");
      return 1;
    }
    free(h2);
    cudaFree(shift);
    cudaFree(stripe);
    cudaFree(scratch);
    cudaFree(img2);
  }
  tb_plan_desc bad = d;
  bad.n_t = 1;
  tb_plan* p2 = NULL;
  if (tb_plan_create(&bad, 0, &p2) != TB_ERR_INVALID || tb_last_error()[0] == '\0') {
    fprintf(stderr, "n_t = 1 was not rejected\n");
    return 1;
  }
  CHECK(tb_plan_destroy(plan));
  cudaFree(sino);
  cudaFree(img);
  cudaFree(ws);
  free(host);
  printf("c_abi_smoke ok (max abs error %.3e)\n", worst);
  return 0;
}
