/* A plain-C consumer of include/ppa_b200.h: what a maintainer's binding to
 * the hot path looks like without Python.  Builds config 1 (the reference's
 * CPU-runnable case), solves it on the device and prints the eigenvalues and
 * counters as one line of "key=value" pairs; exit status != 0 on any error.
 *   cc -std=c99 -I include tests/c/abi_consumer.c -L paper_1806_08020_b200 \
 *      -lppa_b200 -Wl,-rpath,$PWD/paper_1806_08020_b200 -lm -o abi_consumer */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "ppa_b200.h"

#define CHECK(call)                                                        \
  do {                                                                     \
    int st_ = (call);                                                      \
    if (st_ != PPA_OK) {                                                   \
      fprintf(stderr, "%s -> %d: %s\n", #call, st_, ppa_last_error());     \
      return 1;                                                            \
    }                                                                      \
  } while (0)

int main(int argc, char** argv) {
  const int config = argc > 1 ? atoi(argv[1]) : 1;
  if (ppa_abi_version() < 3) return 2;
  ppa_host_csr* h = NULL;
  CHECK(ppa_gen_config(config, &h));
  int n = 0;
  long long nnz = 0;
  unsigned long long fp = 0;
  CHECK(ppa_host_csr_info(h, &n, &nnz, &fp));
  ppa_op* a = NULL;
  CHECK(ppa_csr_operator(h, &a));

  ppa_solve_config cfg;
  CHECK(ppa_solve_config_default(&cfg)); /* SolveConfig's defaults (delayed CGS2) */
  cfg.m = 30;
  cfg.k = 15;
  cfg.nev = 10;
  cfg.degree = 10;
  cfg.rtol_multiplier = 1e-8;
  cfg.max_cycles = 100;
  cfg.seed = 1;

  double re[10], im[10], res[10], cyc[100];
  double pre[64], pim[64], ire[64], iim[64];
  int conv[10];
  ppa_solve_result r;
  memset(&r, 0, sizeof r);
  r.cap_nev = 10;
  r.cap_roots = 64;
  r.cap_cycles = 100;
  r.eig_re = re;
  r.eig_im = im;
  r.residuals = res;
  r.converged_flags = conv;
  r.poly_re = pre;
  r.poly_im = pim;
  r.inner_re = ire;
  r.inner_im = iim;
  r.cycle_max_residual = cyc;
  CHECK(ppa_solve(a, &cfg, &r));

  printf("n=%d nnz=%lld converged=%d cycles=%d mvps=%lld dots=%lld vops=%lld eig=", n, nnz,
         r.converged, r.cycles, r.cost.mvps, r.cost.dots, r.cost.vops);
  for (int i = 0; i < r.n_eig && i < 10; ++i) printf("%s%.15g", i ? "," : "", re[i]);
  printf("\n");

  /* error path: a bad argument comes back as a status, not an exception */
  ppa_op* bad = NULL;
  if (ppa_csr_operator(NULL, &bad) != PPA_INVALID_ARGUMENT) return 3;

  ppa_op_free(a);
  ppa_host_csr_free(h);
  return r.converged ? 0 : 4;
}
