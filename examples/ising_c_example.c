/* Plain-C use of the library (no Python, no PyTorch): the calls the north_star lists, then
 * a measured chain through the asynchronous API (two calls in flight).
 *   ising_c_example L_rows L_cols seed beta sweeps [lattice.bin]
 *     -> line 1: "up E t sum" after `sweeps` sweeps (and the +-1 bytes, row-major, written
 *        to lattice.bin when given)
 *        line 2: "up E" of 2 x 3 samples, one every 2 sweeps, via ising_sweep_measure_async
 *        line 3: a lattice batch of 3 copies of the lattice (seeds seed, seed+1, seed+2; betas
 *        beta, beta/2, 2 beta): "up E" of each after `sweeps` sweeps (ising_batch_*)
 * Built by __graft_entry__.build(); tests/test_gpu_capi.py runs it against the oracle. */
#include <stdio.h>
#include <stdlib.h>

#include "ising.h"

#define CHECK(call)                                                                   \
  do {                                                                                \
    int st_ = (call);                                                                 \
    if (st_ != ISING_OK) {                                                            \
      fprintf(stderr, "%s -> %s: %s\n", #call, ising_strerror(st_), ising_last_error()); \
      return 1;                                                                       \
    }                                                                                 \
  } while (0)

int main(int argc, char** argv) {
  if (argc != 6 && argc != 7) {
    fprintf(stderr, "usage: %s L_rows L_cols seed beta sweeps [lattice.bin]\n", argv[0]);
    return 2;
  }
  const int64_t N = atoll(argv[1]), M = atoll(argv[2]);
  const uint64_t seed = strtoull(argv[3], NULL, 10);
  const double beta = atof(argv[4]);
  const int64_t sweeps = atoll(argv[5]);
  ising_t h = NULL;
  CHECK(ising_create(&h, N, M, seed, 1));
  CHECK(ising_set_beta(h, beta));
  CHECK(ising_init_random(h));
  CHECK(ising_sweep(h, sweeps));
  int64_t up = 0, E = 0;
  CHECK(ising_observables(h, &up, &E));
  int8_t* lat = (int8_t*)malloc((size_t)(N * M));
  CHECK(ising_read_lattice(h, lat, N * M));
  uint64_t t = 0;
  CHECK(ising_get_sweep(h, &t));
  long long sum = 0;
  for (int64_t k = 0; k < N * M; ++k) sum += lat[k];
  printf("%lld %lld %llu %lld\n", (long long)up, (long long)E, (unsigned long long)t, sum);
  if (argc == 7) {
    FILE* f = fopen(argv[6], "wb");
    if (!f || fwrite(lat, 1, (size_t)(N * M), f) != (size_t)(N * M)) {
      fprintf(stderr, "cannot write %s\n", argv[6]);
      return 1;
    }
    fclose(f);
  }
  free(lat);
  /* asynchronous measured chain: enqueue the second chunk before waiting for the first
   * (host memory here is pageable; pinned memory makes the copies truly asynchronous) */
  int64_t ups[2][3], Es[2][3], tk[2];
  CHECK(ising_sweep_measure_async(h, 3, 2, ups[0], Es[0], &tk[0]));
  CHECK(ising_sweep_measure_async(h, 3, 2, ups[1], Es[1], &tk[1]));
  CHECK(ising_measure_wait(h, tk[0]));
  CHECK(ising_measure_wait(h, tk[1]));
  for (int c = 0; c < 2; ++c)
    for (int k = 0; k < 3; ++k) printf("%lld %lld ", (long long)ups[c][k], (long long)Es[c][k]);
  printf("\n");
  CHECK(ising_destroy(h));
  /* three independent lattices of the same shape in one batch (one CTA each) */
  if (N * M <= 409600) {
    ising_batch_t b = NULL;
    const uint64_t seeds[3] = {seed, seed + 1, seed + 2};
    const double betas[3] = {beta, beta / 2, 2 * beta};
    int64_t bu[3], bE[3];
    CHECK(ising_batch_create(&b, N, M, 3, seeds, 0));
    CHECK(ising_batch_set_beta(b, betas, ISING_RULE_METROPOLIS));
    CHECK(ising_batch_init_random(b));
    CHECK(ising_batch_sweep(b, sweeps));
    CHECK(ising_batch_observables(b, bu, bE));
    for (int k = 0; k < 3; ++k) printf("%lld %lld ", (long long)bu[k], (long long)bE[k]);
    printf("\n");
    CHECK(ising_batch_destroy(b));
  }
  return 0;
}
