// The reference-side binding of INTEGRATION.md, compiled as a test (tests/test_shim.py).
//
// A stand-in for proj/include/ce/types.hpp declares ce::Vector (a minimal Eigen::VectorXd-like
// type: Vector(n), data(), size()) and ce::BreakdownError with the reference's constructor
// (types.hpp:26-36); the shim is configured to use both, and the call sites below are the
// reference's own shapes: cli.cpp:107 (ce_factorize), cli.cpp:198/225-226 (ApplyFn matvec /
// precond + minres), plus pcg with the same ApplyFn contract; guarded() mirrors the exception
// -> exit code mapping of cli.cpp:82-95.  Exit code = guarded()'s, so a breakdown must return 2.
//
// usage: shim_reference_binding [solve | breakdown]
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>

namespace ce {
using index_t = std::int64_t;
class Vector {  // the slice of Eigen::VectorXd the shim relies on
 public:
  Vector() = default;
  explicit Vector(std::size_t n) : n_(n), p_(new double[n]()) {}
  Vector(const Vector& o) : Vector(o.n_) { std::memcpy(p_.get(), o.p_.get(), n_ * sizeof(double)); }
  Vector& operator=(const Vector& o) {
    if (this != &o) {
      Vector t(o);
      n_ = t.n_;
      p_ = std::move(t.p_);
    }
    return *this;
  }
  double* data() { return p_.get(); }
  const double* data() const { return p_.get(); }
  std::size_t size() const { return n_; }

 private:
  std::size_t n_ = 0;
  std::unique_ptr<double[]> p_;
};
class BreakdownError : public std::runtime_error {
 public:
  BreakdownError(int level, index_t block, const std::string& what)
      : std::runtime_error(what), level_(level), block_(block) {}
  int level() const { return level_; }
  index_t block() const { return block_; }

 private:
  int level_;
  index_t block_;
};
constexpr int kExitOk = 0, kExitUsage = 1, kExitBreakdown = 2, kExitNoConvergence = 3;
}  // namespace ce

#define CE_B200_VECTOR ::ce::Vector
#define CE_B200_BREAKDOWN_ERROR ::ce::BreakdownError
#include "ce_gpu.hpp"

namespace ce {
using ApplyFn = ce_b200::ApplyFn;
using ce_b200::minres;
using ce_b200::MinresOptions;
using ce_b200::pcg;
using ce_b200::PcgOptions;
using ce_b200::SolveReport;

int guarded(const std::function<int()>& body) {  // cli.cpp:82-95
  try {
    return body();
  } catch (const BreakdownError& e) {
    std::printf("error: %s (level %d, block %lld)\n", e.what(), e.level(), static_cast<long long>(e.block()));
    return kExitBreakdown;
  } catch (const std::exception& e) {
    std::printf("error: %s\n", e.what());
    return kExitUsage;
  }
}
}  // namespace ce

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "solve";
  ce_problem* p = nullptr;
  if (ce_problem_create(1, 32, 32, 0, &p)) return 1;
  ce_csb_host h;
  ce_problem_csb(p, &h);
  ce_plan_host pl;
  ce_problem_plan(p, &pl);
  std::unique_ptr<double[]> vals;
  if (mode == "breakdown") {  // negate the first diagonal entry
    const int64_t nv = h.val_ptr[h.row_ptr[h.m]];
    vals.reset(new double[nv]);
    std::memcpy(vals.get(), h.values, nv * sizeof(double));
    vals[h.val_ptr[0]] = -vals[h.val_ptr[0]];
    h.values = vals.get();
  }
  const int rc = ce::guarded([&]() -> int {
    ce_b200::Context ctx(0);
    ce_b200::BlockSparseMatrix a(ctx, h);
    ce_b200::FactorOptions fo;
    fo.dense_threshold = 64;
    auto fact = ce_b200::ce_factorize(ctx, a, pl, ce_b200::CompressionStrategy::adaptive(1e-4), fo);  // cli.cpp:107
    const ce::index_t n = h.n;
    ce::Vector rhs(static_cast<std::size_t>(n));
    std::memcpy(rhs.data(), ce_problem_rhs(p), n * sizeof(double));
    ce::ApplyFn matvec = [&](const ce::Vector& v) { return a.matvec(v); };       // cli.cpp:198
    ce::ApplyFn precond = [&](const ce::Vector& v) { return fact.solve(v); };    // cli.cpp:225
    ce::MinresOptions mo;
    mo.tol = 1e-8;
    ce::Vector x;
    const ce::SolveReport rm = ce::minres(matvec, n, rhs, precond, mo, x);        // cli.cpp:226
    ce::PcgOptions po;
    po.tol = 1e-8;
    ce::Vector xp;
    const ce::SolveReport rp = ce::pcg(matvec, n, rhs, precond, po, xp);
    ce::Vector xd;
    const ce::SolveReport rd = ce_b200::pcg(ctx, a, n, rhs, &fact, po, xd);      // device fast path
    std::printf("binding ok: minres its=%lld true=%.3e pcg its=%lld true=%.3e device pcg its=%lld\n",
                static_cast<long long>(rm.iterations), rm.final_true_residual, static_cast<long long>(rp.iterations),
                rp.final_true_residual, static_cast<long long>(rd.iterations));
    const bool ok = rm.converged && rp.converged && rd.converged && rm.final_true_residual <= 1e-7 &&
                    rp.final_true_residual <= 1e-7 && (rp.iterations - rd.iterations <= 1) &&
                    (rd.iterations - rp.iterations <= 1);
    return ok ? ce::kExitOk : ce::kExitNoConvergence;
  });
  ce_problem_free(p);
  return rc;
}
