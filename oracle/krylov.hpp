// ORACLE — TEST INFRASTRUCTURE ONLY (see dense.hpp).
// Krylov layer: minres restates proj/src/minres.cpp:11-127 (ApplyFn contract,
// proj/include/ce/minres.hpp:10-50); pcg is the north star's addition with the
// same contract (x0 = 0, stop on recurrence ||r||/||b|| <= tol,
// iterations = number of A*p products, final true residual reported).
#pragma once

#include <functional>
#include <vector>

#include "dense.hpp"

namespace oracle {

using Vec = std::vector<double>;
using ApplyFn = std::function<Vec(const Vec&)>;

struct IterationSample {
  index_t iter = 0;
  double recurrence_resid = 0.0;
  double true_resid = -1.0;
  double seconds = 0.0;
};

struct SolveReport {
  bool converged = false;
  index_t iterations = 0;
  double final_recurrence_residual = 0.0;
  double final_true_residual = 0.0;
  std::vector<IterationSample> trace;
};

struct MinresOptions {
  double tol = 1e-10;
  index_t maxit = 1000;
  bool track_true_residual = true;
};

struct PcgOptions {
  double tol = 1e-10;
  index_t maxit = 1000;
  bool track_true_residual = false;
};

SolveReport minres(const ApplyFn& a, index_t n, const Vec& b, const ApplyFn& precond, const MinresOptions& opts,
                   Vec& x);
SolveReport pcg(const ApplyFn& a, index_t n, const Vec& b, const ApplyFn& precond, const PcgOptions& opts, Vec& x);
double relative_residual(const ApplyFn& a, const Vec& x, const Vec& b);

}  // namespace oracle
