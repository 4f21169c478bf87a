/* test_c_abi.c -- the boundary from plain C (no C++): the INTEGRATION.md
 * example as a program.  `test_c_abi cpu` exercises the host functions;
 * `test_c_abi all` also integrates a small jittered mesh on device 0 and
 * checks the reference triangle matrix bitwise. */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "fembatch_b200.h"

static int failures = 0;
#define CHECK(c)                                                       \
  do                                                                   \
  {                                                                    \
    if (!(c))                                                          \
    {                                                                  \
      ++failures;                                                      \
      printf("  FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);            \
    }                                                                  \
  } while (0)

int main(int argc, char** argv)
{
  const int gpu = argc > 1 && strcmp(argv[1], "all") == 0;
  fb_error err;
  CHECK(fb_abi_version() == FB_ABI_VERSION);
  CHECK(fb_flop_count(FB_LAPLACIAN, 3, 1) == 288);
  CHECK(fb_element_matrix_index(3, 4, 2, 3, 0, 0) == 27);

  const int64_t klen = fb_k_len(FB_ELASTICITY, 3);
  double* k = malloc(sizeof(double) * klen);
  CHECK(fb_build_analytic_tensor(FB_ELASTICITY, 3, k, klen, &err) == FB_OK);
  fb_kernel_config cfg = {128, 1, 0, 0, FB_F32, FB_STRICT, FB_STORE_AUTO, 0};
  fb_variant* v = fb_specialize(FB_ELASTICITY, 3, k, klen, &cfg, &err);
  CHECK(v != NULL && fb_variant_path(v) == 3);
  CHECK(strcmp(fb_variant_description(v), "bs128_ce1") == 0);
  fb_kernel_config bad = cfg;
  bad.num_concurrent_elements = 8; /* 144 * 8 > 1024 */
  CHECK(fb_specialize(FB_ELASTICITY, 3, k, klen, &bad, &err) == NULL);
  CHECK(err.code == FB_ERR_INVALID_ARGUMENT && strstr(err.message, "work-group bound") != NULL);

  if (gpu)
  {
    /* reference triangle, Laplacian, f64: [[1,-.5,-.5],[-.5,.5,0],[-.5,0,.5]] bitwise */
    double lk[36];
    fb_build_analytic_tensor(FB_LAPLACIAN, 2, lk, 36, &err);
    fb_kernel_config c1 = {1, 1, 0, 0, FB_F64, FB_STRICT, FB_STORE_AUTO, 0};
    fb_variant* lv = fb_specialize(FB_LAPLACIAN, 2, lk, 36, &c1, &err);
    const double vert[6] = {0, 0, 1, 0, 0, 1};
    const int32_t cell[3] = {0, 1, 2};
    fb_mesh_view m = {2, 0, 3, 1, vert, cell};
    double out[9];
    CHECK(fb_integrate_mesh(lv, &m, NULL, out, 9, NULL, 0, &err) == FB_OK);
    const double want[9] = {1, -0.5, -0.5, -0.5, 0.5, 0, -0.5, 0, 0.5}; /* symmetric: j-major == row-major */
    CHECK(memcmp(out, want, sizeof want) == 0);
    /* a degenerate cell is reported by index with the reference text */
    const int32_t inv[3] = {0, 2, 1};
    fb_mesh_view mi = {2, 0, 3, 1, vert, inv};
    CHECK(fb_integrate_mesh(lv, &mi, NULL, out, 9, NULL, 0, &err) == FB_ERR_RUNTIME);
    CHECK(err.cell == 0 && strstr(err.message, "degenerate element: det(J) <= 0 in cell 0") != NULL);
    fb_variant_free(lv);
  }
  fb_variant_free(v);
  free(k);
  printf("%s: %d failures\n", gpu ? "all" : "cpu", failures);
  return failures != 0;
}
