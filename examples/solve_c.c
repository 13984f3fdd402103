/* Minimal C client of libbnbg.so (include/bnbg.h): generate a synthetic
 * instance, certify it on GPU 0, print the certificate as one JSON line.
 *
 *   gcc -std=c99 -O2 -I include examples/solve_c.c \
 *       -L paper_2605_22188_b200 -lbnbg -Wl,-rpath,$PWD/paper_2605_22188_b200 -o solve_c
 *   ./solve_c n p k rho loss seed
 */
#include <stdio.h>
#include <stdlib.h>

#include "bnbg.h"

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 1000, p = argc > 2 ? atoi(argv[2]) : 100;
  const int k = argc > 3 ? atoi(argv[3]) : 5, loss = argc > 5 ? atoi(argv[5]) : BNBG_SQUARED;
  const double rho = argc > 4 ? atof(argv[4]) : 0.5;
  const unsigned long long seed = argc > 6 ? strtoull(argv[6], NULL, 10) : 0;
  double* X = malloc(sizeof(double) * (size_t)n * p);
  double* y = malloc(sizeof(double) * (size_t)n);
  int32_t* truth = malloc(sizeof(int32_t) * (size_t)k);
  int rc = bnbg_generate_synthetic(n, p, k, rho, loss, 5.0, seed, X, y, truth);
  if (rc) {
    fprintf(stderr, "generate: %s\n", bnbg_last_error(NULL));
    return 1;
  }
  bnbg_handle* h = NULL;
  rc = bnbg_create(X, y, n, p, loss, k, 2.0, 1.0, 0.0, 0, &h);
  if (rc) {
    fprintf(stderr, "create: %s\n", bnbg_last_error(NULL));
    return 1;
  }
  bnbg_solver_cfg cfg;
  bnbg_solver_cfg_default(&cfg);
  int32_t* sup = malloc(sizeof(int32_t) * (size_t)k);
  double* coef = malloc(sizeof(double) * (size_t)k);
  bnbg_certificate cert = {0};
  cert.support = sup;
  cert.coefficients = coef;
  rc = bnbg_solve(h, &cfg, &cert, NULL, NULL, NULL);
  if (rc) {
    fprintf(stderr, "solve: %s\n", bnbg_last_error(h));
    bnbg_destroy(h);
    return 1;
  }
  printf("{\"optimal_value\": %.17g, \"nodes\": %lld, \"status\": %d, \"support\": [", cert.optimal_value,
         cert.nodes_processed, cert.status);
  for (int i = 0; i < cert.support_len; ++i) printf("%s%d", i ? ", " : "", sup[i]);
  printf("]}\n");
  bnbg_destroy(h);
  free(X);
  free(y);
  free(truth);
  free(sup);
  free(coef);
  return 0;
}
