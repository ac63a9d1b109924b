// ce_gpu.hpp — header-only C++ shim over the C-ABI (ce_gpu.h) that re-exposes
// the reference's call shapes from proj/include/ce/ so call sites such as
//   proj/src/cli.cpp:107        fact = ce_factorize(lp.matrix, lp.plan, cfg.strategy(), opts);
//   proj/src/cli.cpp:225-226    ApplyFn precond = [&](const Vector& v) { return fact.solve(v); };
// compile against it with std::vector<double> in place of Eigen::VectorXd.
// Errors map back to the reference exception types' meaning:
//   CE_EBREAKDOWN -> ce_b200::BreakdownError{level, block}   (types.hpp:26-36)
//   CE_EUSAGE     -> std::runtime_error
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "ce_gpu.h"

namespace ce_b200 {

using index_t = std::int64_t;
using Vector = std::vector<double>;

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

inline void check(int rc) {
  if (rc != CE_OK) throw std::runtime_error(ce_last_error());
}

// One GPU (ce_ctx).
class Context {
 public:
  explicit Context(int device = 0) { check(ce_ctx_create(device, &ctx_)); }
  ~Context() { ce_ctx_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  ce_ctx* get() const { return ctx_; }

 private:
  ce_ctx* ctx_ = nullptr;
};

// BlockSparseMatrix (block_matrix.hpp:23-63): uploaded once, device-resident.
class BlockSparseMatrix {
 public:
  BlockSparseMatrix(Context& ctx, const ce_csb_host& host) { check(ce_matrix_upload(ctx.get(), &host, &m_)); }
  ~BlockSparseMatrix() { ce_matrix_free(m_); }
  BlockSparseMatrix(const BlockSparseMatrix&) = delete;
  BlockSparseMatrix& operator=(const BlockSparseMatrix&) = delete;
  index_t dim() const { return ce_matrix_dim(m_); }
  // block_matrix.hpp:45
  Vector matvec(const Vector& x) const {
    Vector y(x.size());
    check(ce_matvec(m_, x.data(), y.data(), static_cast<int64_t>(x.size()), 0, nullptr));
    return y;
  }
  const ce_matrix* get() const { return m_; }

 private:
  ce_matrix* m_ = nullptr;
};

struct CompressionStrategy {  // compression.hpp:15-38
  ce_strategy s{0, 1e-6, 0, 0};
  static CompressionStrategy adaptive(double eps, bool absolute = false) {
    CompressionStrategy c;
    c.s = {0, eps, absolute ? 1 : 0, 0};
    return c;
  }
  static CompressionStrategy fixed_rank(index_t rank) {
    CompressionStrategy c;
    c.s = {1, 0.0, 0, rank};
    return c;
  }
};

struct FactorOptions {  // factorization.hpp:74-77
  index_t dense_threshold = 2048;
  index_t max_levels = 64;
};

// CEFactorization (factorization.hpp:81-102): immutable, device-resident.
class CEFactorization {
 public:
  explicit CEFactorization(ce_factor* f) : f_(f, ce_factor_free) {}
  // factorization.hpp:90
  Vector solve(const Vector& b) const {
    Vector x(b.size());
    const int rc = ce_apply_precond(f_.get(), b.data(), x.data(), static_cast<int64_t>(b.size()), 0, nullptr);
    if (rc != CE_OK) throw std::invalid_argument(ce_last_error());
    return x;
  }
  Vector apply_operator(const Vector& x) const { return tool(0, x); }
  Vector apply_q(const Vector& x) const { return tool(1, x); }
  Vector apply_q_transpose(const Vector& y) const { return tool(2, y); }
  const ce_factor* get() const { return f_.get(); }

 private:
  Vector tool(int which, const Vector& x) const {
    Vector y(x.size());
    check(ce_factor_apply_tool(f_.get(), which, x.data(), y.data(), static_cast<int64_t>(x.size())));
    return y;
  }
  std::shared_ptr<ce_factor> f_;
};

// factorization.hpp:121-123
inline CEFactorization ce_factorize(Context& ctx, const BlockSparseMatrix& a, const ce_plan_host& plan,
                                    const CompressionStrategy& s, const FactorOptions& o = {}) {
  ce_factor_opts opts{o.dense_threshold, o.max_levels, 0, nullptr, nullptr};
  ce_status st{};
  ce_factor* f = nullptr;
  const int rc = ce_factorize(ctx.get(), a.get(), &plan, &s.s, &opts, &f, &st);
  if (rc == CE_EBREAKDOWN) throw BreakdownError(st.level, st.block, st.message);
  check(rc);
  return CEFactorization(f);
}

struct PcgOptions {  // the MinresOptions shape (minres.hpp:34-38)
  double tol = 1e-10;
  index_t maxit = 1000;
  bool track_true_residual = false;
};

struct SolveReport {  // minres.hpp:25-31
  bool converged = false;
  index_t iterations = 0;
  double final_recurrence_residual = 0.0;
  double final_true_residual = 0.0;
};

// minres(a, n, b, precond, opts, x) shape (minres.hpp:46-47) with PCG on the device.
inline SolveReport pcg(Context& ctx, const BlockSparseMatrix& a, index_t n, const Vector& b,
                       const CEFactorization* precond, const PcgOptions& o, Vector& x) {
  x.assign(static_cast<size_t>(n), 0.0);
  ce_pcg_opts opts{o.tol, o.maxit, o.track_true_residual ? 1 : 0};
  ce_solve_report rep{};
  const int rc = ce_pcg(ctx.get(), a.get(), precond ? precond->get() : nullptr, b.data(), x.data(), n, 0, &opts, &rep);
  if (rc != CE_OK && rc != CE_ENOCONV) check(rc);
  return SolveReport{rep.converged != 0, rep.iterations, rep.final_recurrence_residual, rep.final_true_residual};
}

struct MinresOptions {  // minres.hpp:34-38
  double tol = 1e-10;
  index_t maxit = 1000;
  bool track_true_residual = true;
};

// minres(a, n, b, precond, opts, x) (minres.hpp:46-47) on the device.
inline SolveReport minres(Context& ctx, const BlockSparseMatrix& a, index_t n, const Vector& b,
                          const CEFactorization* precond, const MinresOptions& o, Vector& x) {
  x.assign(static_cast<size_t>(n), 0.0);
  ce_pcg_opts opts{o.tol, o.maxit, o.track_true_residual ? 1 : 0};
  ce_solve_report rep{};
  const int rc =
      ce_minres(ctx.get(), a.get(), precond ? precond->get() : nullptr, b.data(), x.data(), n, 0, &opts, &rep);
  if (rc != CE_OK && rc != CE_ENOCONV) check(rc);
  return SolveReport{rep.converged != 0, rep.iterations, rep.final_recurrence_residual, rep.final_true_residual};
}

}  // namespace ce_b200
