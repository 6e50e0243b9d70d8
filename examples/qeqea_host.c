/*
 * A C host driving the QEQEA generation loop through the C ABI alone (no
 * Python, no torch): the reference's run loop (report.py:127-168) in C.
 *
 *   gcc -O2 -I include examples/qeqea_host.c -L paper_1809_11134_b200 -lisq \
 *       -Wl,-rpath,$PWD/paper_1809_11134_b200 -o qeqea_host
 *   ./qeqea_host [generations]        -> one line per generation on stdout
 */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "isq.h"

int main(int argc, char** argv) {
  const int gens = argc > 1 ? atoi(argv[1]) : 200;
  isq_qeqea_config cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.number_of_wires = 3; /* Toffoli, C1 shape (engine.py:33-43 defaults) */
  cfg.size_of_individual = 16;
  cfg.size_of_population = 5;
  cfg.probability_of_mutation = 0.3;
  cfg.mutation_range = 0.7853981633974483;
  cfg.n_meas = 1;
  cfg.max_generations = gens;
  cfg.target_fitness = 0.999;
  cfg.seed = 1;
  cfg.world = 1;
  cfg.precision = ISQ_PRECISION_FP64;
  double target[2 * 8 * 8];
  memset(target, 0, sizeof(target));
  for (int r = 0; r < 8; ++r) {
    const int c = r == 6 ? 7 : (r == 7 ? 6 : r); /* Toffoli: swap |110>, |111> */
    target[2 * (r * 8 + c)] = 1.0;
  }
  void* h = NULL;
  if (isq_qeqea_create(&cfg, target, 0, gens, &h) != ISQ_OK) {
    fprintf(stderr, "create: %s\n", isq_last_error());
    return 1;
  }
  isq_generation_record* rec = (isq_generation_record*)calloc((size_t)gens, sizeof(*rec));
  int32_t done = 0, stop = 0;
  if (isq_qeqea_step(h, gens, rec, &done, &stop) != ISQ_OK) {
    fprintf(stderr, "step: %s\n", isq_last_error());
    return 1;
  }
  for (int i = 0; i < done; ++i)
    printf("%d %.17g %.17g %.17g\n", i + 1, rec[i].gen_best, rec[i].gen_mean, rec[i].best_fitness);
  uint8_t codes[16];
  double thetas[16], best = 0.0;
  isq_qeqea_best(h, codes, thetas, &best);
  printf("stop %d best %.17g codes", stop, best);
  for (int p = 0; p < 16; ++p) printf(" %d", codes[p]);
  printf("\n");
  isq_qeqea_destroy(h);
  free(rec);
  return 0;
}
