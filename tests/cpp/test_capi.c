/* Plain-C client of include/labs_b200.h: the INTEGRATION.md example,
 * compiled with a C compiler (no C++ or torch anywhere on the path). */
#include <stdio.h>
#include <string.h>

#include "labs_b200.h"

int main(void) {
  labs_ctx* ctx = NULL;
  if (labs_ctx_create(0, &ctx) != LABS_OK) {
    fprintf(stderr, "ctx: %s\n", labs_last_error());
    return 1;
  }
  labs_memetic_params p;
  memset(&p, 0, sizeof p);
  p.population_size = 100;
  p.p_comb = 0.9;
  p.p_mutate = -1.0;
  p.target_energy = 26;
  p.max_seconds = 30.0;
  p.max_iterations = -1;
  p.tabu.min_tabu_factor = 0.10;
  p.tabu.max_tabu_factor = 0.12;
  p.rng_kind = LABS_RNG_MT19937_64;
  labs_run_result best, per[2];
  int rc = labs_run_replicas(ctx, 20, 2, 42, &p, &best, per, NULL, 0, NULL);
  int fail = rc != LABS_OK || best.best_energy != 26 || !per[1].reached_target ||
             per[1].iterations != 98 || per[1].best[0] != 0xaf793ULL;
  /* errors map to status codes, message on the calling thread */
  p.population_size = 1;
  rc = labs_run_replicas(ctx, 20, 2, 42, &p, &best, NULL, NULL, 0, NULL);
  fail |= rc != LABS_ERR_INVALID_ARGUMENT || strlen(labs_last_error()) == 0;
  int32_t pos = 7;
  int64_t e[1];
  uint64_t w = 0;
  rc = labs_flip_trace(ctx, 8, 1, &w, 1, &pos, e, NULL);
  fail |= rc != LABS_OK;
  pos = 8;
  rc = labs_flip_trace(ctx, 8, 1, &w, 1, &pos, e, NULL);
  fail |= rc != LABS_ERR_OUT_OF_RANGE;
  labs_ctx_destroy(ctx);
  printf("%s\n", fail ? "FAIL" : "ok");
  return fail;
}
