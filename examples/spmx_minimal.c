/* The C ABI from plain C99: the reference's worked example
 *     [[2, 0], [1, 3]] x [[1, 2], [3, 4]] = [[2, 4], [10, 14]]
 * (proj/tests/test_matrix_core.cpp:181-189) through spmx_spmm_host with malloc'ed host arrays,
 * under each division scheme, in both modes. No C++ on the caller's side:
 *     gcc -std=c99 examples/spmx_minimal.c -Lpaper_2312_05639_b200 -lspmx_b200 -o spmx_minimal
 * `spmx_minimal --link-only` stops after the calls that need no GPU (CPU test-suite). */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../include/spmx_b200.h"

int main(int argc, char** argv) {
  printf("abi %d, build %s\n", spmx_abi_version(), spmx_build_info());
  if (argc > 1 && strcmp(argv[1], "--link-only") == 0) return 0;

  spmx_ctx* ctx = NULL;
  if (spmx_ctx_create(0, NULL, &ctx) != SPMX_OK) {
    fprintf(stderr, "spmx_ctx_create: %s\n", spmx_last_error());
    return 1;
  }
  const uint64_t row_ptr[3] = {0, 1, 3};
  const uint32_t col[3] = {0, 0, 1};
  const float vals[3] = {2.0f, 1.0f, 3.0f};
  const float x[4] = {1.0f, 2.0f, 3.0f, 4.0f};
  const float want[4] = {2.0f, 4.0f, 10.0f, 14.0f};
  const int strategies[3] = {SPMX_ROW_SPLIT, SPMX_NNZ_SPLIT, SPMX_MERGE_SPLIT};
  const unsigned modes[2] = {0u, SPMX_EXACT_ORDER};
  int bad = 0;
  for (int s = 0; s < 3; ++s)
    for (int f = 0; f < 2; ++f) {
      float* y = (float*)malloc(4 * sizeof(float));
      memset(y, 0xff, 4 * sizeof(float));
      if (spmx_spmm_host(ctx, 2, 2, 3, row_ptr, col, vals, x, 2, 2, y, strategies[s], 0, 0, 128, modes[f], NULL) !=
          SPMX_OK) {
        fprintf(stderr, "spmx_spmm_host: %s\n", spmx_last_error());
        bad = 1;
      } else if (memcmp(y, want, sizeof(want)) != 0) {
        fprintf(stderr, "strategy %d flags %u: got %g %g %g %g\n", strategies[s], modes[f], y[0], y[1], y[2], y[3]);
        bad = 1;
      }
      free(y);
    }
  /* the reference's error behaviour: A.n != X.rows is an invalid argument with its message */
  {
    float y[4];
    const int rc = spmx_spmm_host(ctx, 2, 2, 3, row_ptr, col, vals, x, 3, 2, y, SPMX_ROW_SPLIT, 0, 0, 128, 0, NULL);
    if (rc != SPMX_EINVAL || strstr(spmx_last_error(), "A.n != X.rows") == NULL) {
      fprintf(stderr, "shape error not reported: rc %d, %s\n", rc, spmx_last_error());
      bad = 1;
    }
  }
  spmx_ctx_destroy(ctx);
  printf(bad ? "FAILED\n" : "worked example ok: 3 strategies x 2 modes through the C ABI\n");
  return bad;
}
