/*
 * capi_demo.c -- the C ABI used from plain C (no Python, no torch):
 * build the spectrum cache of a small padded magnetic grid, apply the forward
 * and transpose operators to host vectors, check the adjoint identity
 * <G x, v> = <x, G^T v>, and print both outputs for comparison.
 *
 *   cc -O2 -I include examples/capi_demo.c -L paper_1912_06976_b200 -lbttb_sm100 \
 *      -Wl,-rpath,paper_1912_06976_b200 -lm -o capi_demo
 *   ./capi_demo            # exit status 0 on success
 *
 * Inputs are deterministic (x_k = sin(k), v_k = cos(k)); the magnetic
 * constants are magnetic_constants(33, 47, 45000) of the reference
 * (kernels.py:48-64), passed in on the command line as five numbers when the
 * caller wants other values.  tests/test_capi_demo.py compiles and runs it.
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "bttb_sm100.h"

int main(int argc, char** argv) {
  const double z[3] = {0.0, 1.0, 2.5};
  const bttb_grid g = {6, 5, 2, 1, 2, 2, 0, 1.0, 1.5, z};
  bttb_kernel k = {BTTB_MAGNETIC, 0.0, {0, 0, 0, 0, 0}};
  if (argc != 6) {
    fprintf(stderr, "usage: %s gc0 gc1 gc2 gc3 gc4\n", argv[0]);
    return 2;
  }
  for (int i = 0; i < 5; ++i) k.gc[i] = atof(argv[1 + i]);
  const int64_t nx = g.sx + g.pxl + g.pxr, ny = g.sy + g.pyl + g.pyr;
  const int64_t n = nx * ny * g.nz, m = g.sx * g.sy;
  double* x = malloc(sizeof(double) * n);
  double* xt = malloc(sizeof(double) * n);
  double* v = malloc(sizeof(double) * m);
  double* d = malloc(sizeof(double) * m);
  for (int64_t i = 0; i < n; ++i) x[i] = sin((double)i);
  for (int64_t i = 0; i < m; ++i) v[i] = cos((double)i);
  bttb_plan* p = NULL;
  if (bttb_plan_create(&p, &g, &k, BTTB_F64, 0, 0, g.nz, 0, 0) != BTTB_OK) {
    fprintf(stderr, "plan: %s\n", bttb_last_error());
    return 1;
  }
  if (bttb_apply(p, BTTB_FORWARD, x, d, 1, BTTB_HOST_PTR, NULL) != BTTB_OK ||
      bttb_apply(p, BTTB_TRANSPOSE, v, xt, 1, BTTB_HOST_PTR, NULL) != BTTB_OK) {
    fprintf(stderr, "apply: %s\n", bttb_last_error());
    return 1;
  }
  double a = 0, b = 0, na = 0;
  for (int64_t i = 0; i < m; ++i) a += d[i] * v[i], na += fabs(d[i] * v[i]);
  for (int64_t i = 0; i < n; ++i) b += x[i] * xt[i];
  printf("forward");
  for (int64_t i = 0; i < m; ++i) printf(" %.17g", d[i]);
  printf("\ntranspose");
  for (int64_t i = 0; i < n; ++i) printf(" %.17g", xt[i]);
  printf("\nadjoint %.3e\n", fabs(a - b) / na);
  bttb_plan_destroy(p);
  free(x), free(xt), free(v), free(d);
  return fabs(a - b) <= 1e-12 * na ? 0 : 1;
}
