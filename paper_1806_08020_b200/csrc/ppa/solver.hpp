#pragma once
// PP-Arnoldi driver (reference inc/solver.hpp).  The reference declares
// these entry points but ships no body; the behaviour follows
// SPEC.md "[MODULE] solver" with the frozen choices listed in DESIGN.md
// ("Solver decisions").

#include <complex>
#include <optional>
#include <vector>

#include "ppa/arnoldi.hpp"
#include "ppa/cost.hpp"
#include "ppa/gmres_poly.hpp"
#include "ppa/operators.hpp"

namespace ppa {

enum class RestartVariant { ritz, harmonic };
enum class DampingMode { off, auto_heuristic, forced };
enum class StabilityMode { off, pof_auto };

/// inc/solver.hpp:21-58, field for field, plus allow_nev_above_k (our
/// extension for BASELINE config 5, whose nev = 20 > k = 15 violates
/// SPEC.md's 0 < nev <= k < m).
struct SolveConfig {
  int m = 50;
  int k = 20;
  int nev = 15;
  int degree = 0;
  double rtol_multiplier = 1e-8;
  std::optional<double> rtol_absolute;
  RestartVariant variant = RestartVariant::ritz;
  DampingMode damping = DampingMode::off;
  double damping_alpha = 0.0;
  int damping_power = 1;
  StabilityMode stability = StabilityMode::off;
  int double_d1 = 0;
  int double_d2 = 0;
  int max_cycles = 100;
  unsigned long long seed = 1;
  bool check_mid_cycle = false;
  int mid_cycle_stride = 5;
  bool stagnation_stop = false;
  int stagnation_window = 5;
  double stagnation_rtol = 0.01;
  std::vector<std::complex<double>> reference;
  bool allow_nev_above_k = false;

  void validate() const;
};

struct CycleStats {
  int cycle = 0;
  bool discarded_probe = false;
  int start_dim = 0;
  int end_dim = 0;
  int restart_k = 0;
  int real_checks = 0;
  int pair_checks = 0;
  double max_residual = 0.0;
};

/// Timing breakdown of one solve (device events + host clock), seconds.
struct SolveTiming {
  double total = 0.0;
  double setup = 0.0;      // norm estimate + polynomial construction
  double extend = 0.0;     // pi(A)v + CGS2 inside the cycles
  double check = 0.0;      // Ritz vectors + true residuals
  double restart = 0.0;    // thick restart
};

struct EigResult {
  std::vector<std::complex<double>> eigenvalues;
  std::vector<double> residuals;
  std::vector<bool> converged_flags;
  bool converged = false;
  int cycles = 0;
  CostRecord cost;
  std::optional<PolyPrecond> poly;
  std::optional<PolyPrecond> inner_poly;
  int composite_degree = 0;
  double rtol = 0.0;
  double max_err = 0.0;
  std::vector<CycleStats> history;
  int correct_count = -1;
  double norm_estimate = 0.0;
  SolveTiming timing;

  int count_correct(const std::vector<std::complex<double>>& reference,
                    double rel_tol = 1e-6) const;
};

EigResult solve(const OperatorPtr& a, const SolveConfig& cfg);
EigResult solve_double(const OperatorPtr& a, const SolveConfig& cfg);
double operator_norm_estimate(const LinearOperator& a, unsigned long long seed, CostRecord& rec);
bool check_ideal_order(const std::vector<std::complex<double>>& mu, int nev);
/// PAPER.md section 6.3 heuristic (inc/solver.hpp:101-106).
PolyPrecond damping_heuristic(const OperatorPtr& a, const SolveConfig& cfg, CostRecord& rec);

}  // namespace ppa
