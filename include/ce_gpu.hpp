// ce_gpu.hpp — header-only C++ shim over the C-ABI (ce_gpu.h) that re-exposes
// the reference's call shapes from proj/include/ce/ so call sites such as
//   proj/src/cli.cpp:107        fact = ce_factorize(lp.matrix, lp.plan, cfg.strategy(), opts);
//   proj/src/cli.cpp:198        ApplyFn matvec = [&](const Vector& v) { return lp.matrix.matvec(v); };
//   proj/src/cli.cpp:225-226    ApplyFn precond = [&](const Vector& v) { return fact.solve(v); };
//                               SolveReport rep = minres(matvec, n, rhs, precond, opts, x);
// compile against it unchanged.
//
// Customisation points (define before including this header):
//   CE_B200_VECTOR           the Vector type (default std::vector<double>); the reference
//                            binding defines it as ::ce::Vector (Eigen::VectorXd,
//                            proj/include/ce/types.hpp:16).  Needs Vector(n), data(), size().
//   CE_B200_BREAKDOWN_ERROR  the exception thrown on CE_EBREAKDOWN, constructed as
//                            (int level, index_t block, std::string what); the reference
//                            binding defines it as ::ce::BreakdownError
//                            (proj/include/ce/types.hpp:26-36) so guarded()
//                            (proj/src/cli.cpp:82-95) maps it to exit code 2 unchanged.
// Other errors: CE_EUSAGE -> std::runtime_error (std::invalid_argument for size mismatches
// of solve, factorization.cpp:141); Krylov non-convergence is reported, not thrown (minres.hpp).
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "ce_gpu.h"

namespace ce_b200 {

using index_t = std::int64_t;

#ifdef CE_B200_VECTOR
using Vector = CE_B200_VECTOR;
#else
using Vector = std::vector<double>;
#endif

#ifdef CE_B200_BREAKDOWN_ERROR
using BreakdownError = CE_B200_BREAKDOWN_ERROR;
#else
class BreakdownError : public std::runtime_error {  // types.hpp:26-36
 public:
  BreakdownError(int level, index_t block, const std::string& what)
      : std::runtime_error(what), level_(level), block_(block) {}
  int level() const { return level_; }
  index_t block() const { return block_; }

 private:
  int level_;
  index_t block_;
};
#endif

using ApplyFn = std::function<Vector(const Vector&)>;  // minres.hpp:10

inline void check(int rc) {
  if (rc != CE_OK) throw std::runtime_error(ce_last_error());
}

namespace detail {
inline Vector make_vector(index_t n) {
  Vector v(static_cast<std::size_t>(n));
  std::fill_n(v.data(), n, 0.0);
  return v;
}
inline index_t size_of(const Vector& v) { return static_cast<index_t>(v.size()); }
inline double dot(const Vector& a, const Vector& b) {
  double s = 0.0;
  for (index_t i = 0; i < size_of(a); ++i) s += a.data()[i] * b.data()[i];
  return s;
}
inline double norm(const Vector& a) { return std::sqrt(dot(a, a)); }
// relative_residual (minres.hpp:49): ||b - A x|| / ||b||
inline double relative_residual(const ApplyFn& a, const Vector& x, const Vector& b) {
  const Vector ax = a(x);
  const double bn = norm(b);
  double s = 0.0;
  for (index_t i = 0; i < size_of(b); ++i) {
    const double d = b.data()[i] - ax.data()[i];
    s += d * d;
  }
  return bn == 0.0 ? std::sqrt(s) : std::sqrt(s) / bn;
}
// checked inner product r' M^-1 r (the reference's preconditioner check, minres.cpp:11-18)
inline double checked_inner(const Vector& r, const Vector& z) {
  const double h = dot(r, z);
  if (!std::isfinite(h)) throw std::runtime_error("preconditioner produced non-finite values");
  if (h < 0.0) throw std::runtime_error("preconditioner is not positive definite: r' M^-1 r < 0");
  return h;
}
}  // namespace detail

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
    if (detail::size_of(x) != dim()) throw std::invalid_argument("matvec dimension mismatch");
    Vector y = detail::make_vector(dim());
    check(ce_matvec(m_, x.data(), y.data(), dim(), 0, nullptr));
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
  std::string describe() const {  // compression.cpp:10-18
    char buf[96];
    ce_strategy_describe(&s, buf, static_cast<int>(sizeof buf));
    return buf;
  }
};

struct FactorOptions {  // factorization.hpp:74-77
  index_t dense_threshold = 2048;
  index_t max_levels = 64;
};

// CEFactorization (factorization.hpp:81-102): immutable, device-resident; solve() is
// thread-safe (concurrent applies are serialised on the device, ce_gpu.h).
class CEFactorization {
 public:
  explicit CEFactorization(ce_factor* f) : f_(f, ce_factor_free) {}
  index_t dim() const { return ce_factor_dim(f_.get()); }
  // factorization.hpp:90
  Vector solve(const Vector& b) const {
    if (detail::size_of(b) != dim()) throw std::invalid_argument("solve dimension mismatch");
    Vector x = detail::make_vector(dim());
    const int rc = ce_apply_precond(f_.get(), b.data(), x.data(), dim(), 0, nullptr);
    if (rc != CE_OK) throw std::invalid_argument(ce_last_error());
    return x;
  }
  Vector apply_operator(const Vector& x) const { return tool(0, x); }
  Vector apply_q(const Vector& x) const { return tool(1, x); }
  Vector apply_q_transpose(const Vector& y) const { return tool(2, y); }
  const ce_factor* get() const { return f_.get(); }
  // FactorStats / LevelStats (factorization.hpp:38-72) as the C structs of ce_gpu.h
  ce_factor_stats stats() const {
    ce_factor_stats st{};
    check(ce_factor_get_stats(f_.get(), &st));
    return st;
  }
  ce_level_stats level_stats(index_t level) const {
    ce_level_stats ls{};
    check(ce_factor_get_level_stats(f_.get(), level, &ls));
    return ls;
  }

 private:
  Vector tool(int which, const Vector& x) const {
    Vector y = detail::make_vector(detail::size_of(x));
    check(ce_factor_apply_tool(f_.get(), which, x.data(), y.data(), detail::size_of(x)));
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

struct MinresOptions {  // minres.hpp:34-38
  double tol = 1e-10;
  index_t maxit = 1000;
  bool track_true_residual = true;
};

struct IterationSample {  // minres.hpp:12-20
  index_t iter = 0;
  double recurrence_resid = 0.0;
  double true_resid = -1.0;
  double seconds = 0.0;
};

struct IterationTrace {
  std::vector<IterationSample> samples;
};

struct SolveReport {  // minres.hpp:25-31
  bool converged = false;
  index_t iterations = 0;
  double final_recurrence_residual = 0.0;
  double final_true_residual = 0.0;
  IterationTrace trace;
};

// ---------------------------------------------------------------- ApplyFn Krylov
// The reference's callback contract: a and precond are ApplyFn (an empty precond means
// unpreconditioned), x is zero-initialised inside, non-convergence is reported, a negative /
// non-finite r' M^-1 r throws std::runtime_error.  Each ApplyFn here is typically a GPU call
// (BlockSparseMatrix::matvec, CEFactorization::solve) on host vectors; the device-resident
// loops below (pcg/minres taking the objects) avoid the per-iteration copies.

// PCG, minres(a, n, b, precond, opts, x) shape (minres.hpp:46-47): stop when the recurrence
// ||r_k|| / ||b|| <= tol; iterations = number of A*p products.
inline SolveReport pcg(const ApplyFn& a, index_t n, const Vector& b, const ApplyFn& precond, const PcgOptions& o,
                       Vector& x) {
  using namespace detail;
  const auto t0 = std::chrono::steady_clock::now();
  auto elapsed = [&] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };
  if (size_of(b) != n) throw std::invalid_argument("pcg dimension mismatch");
  SolveReport rep;
  x = make_vector(n);
  const double bnorm = norm(b);
  if (bnorm == 0.0) {
    rep.converged = true;
    rep.trace.samples.push_back({0, 0.0, 0.0, elapsed()});
    return rep;
  }
  rep.trace.samples.push_back({0, 1.0, o.track_true_residual ? 1.0 : -1.0, elapsed()});
  Vector r = b;
  Vector z = precond ? precond(r) : r;
  double rz = checked_inner(r, z);
  Vector p = z;
  double rel = 1.0;
  for (index_t itn = 1; itn <= o.maxit; ++itn) {
    const Vector q = a(p);
    const double pq = dot(p, q);
    if (!std::isfinite(pq) || pq <= 0.0) throw std::runtime_error("operator is not positive definite: p' A p <= 0");
    const double alpha = rz / pq;
    for (index_t i = 0; i < n; ++i) {
      x.data()[i] += alpha * p.data()[i];
      r.data()[i] -= alpha * q.data()[i];
    }
    rel = norm(r) / bnorm;
    rep.iterations = itn;
    IterationSample smp{itn, rel, o.track_true_residual ? relative_residual(a, x, b) : -1.0, elapsed()};
    rep.trace.samples.push_back(smp);
    if (rel <= o.tol) {
      rep.converged = true;
      break;
    }
    z = precond ? precond(r) : r;
    const double rzn = checked_inner(r, z);
    const double beta = rzn / rz;
    rz = rzn;
    for (index_t i = 0; i < n; ++i) p.data()[i] = z.data()[i] + beta * p.data()[i];
  }
  rep.final_recurrence_residual = rel;
  rep.final_true_residual = relative_residual(a, x, b);
  if (!rep.trace.samples.empty() && !o.track_true_residual) rep.trace.samples.back().true_resid = rep.final_true_residual;
  return rep;
}

// MINRES, the reference's own entry point (minres.hpp:46-47, the Paige-Saunders recurrence of
// minres.cpp:22-115): stop when the recurrence estimate of the preconditioned residual <= tol
// relative to its start, or on a Lanczos beta < 1e-30 beta1 (exact solution).
inline SolveReport minres(const ApplyFn& a, index_t n, const Vector& b, const ApplyFn& precond,
                          const MinresOptions& o, Vector& x) {
  using namespace detail;
  const auto t0 = std::chrono::steady_clock::now();
  auto elapsed = [&] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };
  if (size_of(b) != n) throw std::invalid_argument("minres dimension mismatch");
  SolveReport rep;
  x = make_vector(n);
  const double bnorm = norm(b);
  if (bnorm == 0.0) {
    rep.converged = true;
    rep.trace.samples.push_back({0, 0.0, 0.0, elapsed()});  // minres.cpp:32-36
    return rep;
  }
  Vector r1 = b;
  Vector y = precond ? precond(b) : b;
  double beta1 = checked_inner(r1, y);
  if (beta1 == 0.0) {
    rep.converged = true;
    rep.trace.samples.push_back({0, 0.0, 1.0, elapsed()});  // minres.cpp:43-47
    return rep;
  }
  beta1 = std::sqrt(beta1);
  rep.trace.samples.push_back({0, 1.0, o.track_true_residual ? 1.0 : -1.0, elapsed()});  // minres.cpp:55
  double oldb = 0.0, beta = beta1, dbar = 0.0, epsln = 0.0, phibar = beta1, cs = -1.0, sn = 0.0;
  Vector r2 = r1, w = make_vector(n), w1 = make_vector(n), w2 = make_vector(n), v = make_vector(n);
  for (index_t itn = 1; itn <= o.maxit; ++itn) {
    for (index_t i = 0; i < n; ++i) v.data()[i] = y.data()[i] / beta;
    y = a(v);
    if (itn >= 2)
      for (index_t i = 0; i < n; ++i) y.data()[i] -= (beta / oldb) * r1.data()[i];
    const double alfa = dot(v, y);
    for (index_t i = 0; i < n; ++i) y.data()[i] -= (alfa / beta) * r2.data()[i];
    r1 = r2;
    r2 = y;
    y = precond ? precond(r2) : r2;
    oldb = beta;
    beta = std::sqrt(checked_inner(r2, y));
    const double oldeps = epsln;
    const double delta = cs * dbar + sn * alfa;
    const double gbar = sn * dbar - cs * alfa;
    epsln = sn * beta;
    dbar = -cs * beta;
    const double gamma = std::max(std::sqrt(gbar * gbar + beta * beta), 1e-290);
    cs = gbar / gamma;
    sn = beta / gamma;
    const double phi = cs * phibar;
    phibar = sn * phibar;
    std::swap(w1, w2);
    std::swap(w2, w);
    for (index_t i = 0; i < n; ++i) {
      w.data()[i] = (v.data()[i] - oldeps * w1.data()[i] - delta * w2.data()[i]) / gamma;
      x.data()[i] += phi * w.data()[i];
    }
    const double rec = phibar / beta1;
    rep.iterations = itn;
    rep.trace.samples.push_back({itn, rec, o.track_true_residual ? relative_residual(a, x, b) : -1.0, elapsed()});
    if (rec <= o.tol || beta / beta1 < 1e-30) {
      rep.converged = true;
      break;
    }
  }
  rep.final_recurrence_residual = phibar / beta1;
  rep.final_true_residual = relative_residual(a, x, b);
  if (!rep.trace.samples.empty() && !o.track_true_residual) rep.trace.samples.back().true_resid = rep.final_true_residual;
  return rep;
}

namespace detail {
inline SolveReport device_report(Context& ctx, const ce_solve_report& rep) {
  SolveReport out;
  out.converged = rep.converged != 0;
  out.iterations = rep.iterations;
  out.final_recurrence_residual = rep.final_recurrence_residual;
  out.final_true_residual = rep.final_true_residual;
  const int64_t k = ce_ctx_last_trace(ctx.get(), nullptr, nullptr, nullptr, nullptr, 0);
  if (k > 0) {
    std::vector<int64_t> it(static_cast<size_t>(k));
    std::vector<double> rec(it.size()), tru(it.size()), sec(it.size());
    ce_ctx_last_trace(ctx.get(), it.data(), rec.data(), tru.data(), sec.data(), k);
    for (size_t j = 0; j < it.size(); ++j) out.trace.samples.push_back({it[j], rec[j], tru[j], sec[j]});
  }
  return out;
}
}  // namespace detail

// ---------------------------------------------------------------- device-resident fast path
// Same contract with the operator and the factor as objects: the whole loop stays on the GPU
// (one 32-byte read per iteration for the stopping test); x is returned on the host.
inline SolveReport pcg(Context& ctx, const BlockSparseMatrix& a, index_t n, const Vector& b,
                       const CEFactorization* precond, const PcgOptions& o, Vector& x) {
  x = detail::make_vector(n);
  ce_pcg_opts opts{o.tol, o.maxit, o.track_true_residual ? 1 : 0};
  ce_solve_report rep{};
  const int rc =
      ce_pcg(ctx.get(), a.get(), precond ? precond->get() : nullptr, b.data(), x.data(), n, 0, &opts, &rep, nullptr);
  if (rc != CE_OK && rc != CE_ENOCONV) check(rc);
  return detail::device_report(ctx, rep);
}

inline SolveReport minres(Context& ctx, const BlockSparseMatrix& a, index_t n, const Vector& b,
                          const CEFactorization* precond, const MinresOptions& o, Vector& x) {
  x = detail::make_vector(n);
  ce_pcg_opts opts{o.tol, o.maxit, o.track_true_residual ? 1 : 0};
  ce_solve_report rep{};
  const int rc = ce_minres(ctx.get(), a.get(), precond ? precond->get() : nullptr, b.data(), x.data(), n, 0, &opts,
                           &rep, nullptr);
  if (rc != CE_OK && rc != CE_ENOCONV) check(rc);
  return detail::device_report(ctx, rep);
}

// ---------------------------------------------------------------- CSV reports (csv.hpp, cli.cpp)
// CsvTable with the reference's semantics (csv.hpp:11-24: no quoting; parse followed by to_string
// reproduces the input bytes) and the report tables of the reference CLI, built by the library's
// text builders so that every binding formats numbers identically (fmt_double: std::to_chars).
struct CsvTable {
  std::vector<std::string> header;
  std::vector<std::vector<std::string>> rows;

  std::string to_string() const {
    std::string out;
    auto put = [&](const std::vector<std::string>& row) {
      for (size_t k = 0; k < row.size(); ++k) {
        if (k) out.push_back(',');
        out += row[k];
      }
      out.push_back('\n');
    };
    put(header);
    for (const auto& r : rows) put(r);
    return out;
  }
  static CsvTable parse(const std::string& text) {
    if (text.empty()) throw std::invalid_argument("csv text has no header row");
    CsvTable t;
    bool first = true;
    for (size_t start = 0; start < text.size();) {
      size_t nl = text.find('\n', start);
      if (nl == std::string::npos) nl = text.size();
      std::vector<std::string> cells;
      for (size_t c0 = start;;) {
        const size_t comma = text.find(',', c0);
        if (comma == std::string::npos || comma >= nl) {
          cells.push_back(text.substr(c0, nl - c0));
          break;
        }
        cells.push_back(text.substr(c0, comma - c0));
        c0 = comma + 1;
      }
      if (first) t.header = std::move(cells);
      else t.rows.push_back(std::move(cells));
      first = false;
      start = nl + 1;
    }
    return t;
  }
  void write(const std::string& path) const {
    std::FILE* fp = std::fopen(path.c_str(), "wb");
    if (!fp) throw std::runtime_error("cannot open " + path + " for writing");
    const std::string text = to_string();
    const bool ok = std::fwrite(text.data(), 1, text.size(), fp) == text.size();
    if (std::fclose(fp) != 0 || !ok) throw std::runtime_error("write failed for " + path);
  }
  static CsvTable load(const std::string& path) {
    std::FILE* fp = std::fopen(path.c_str(), "rb");
    if (!fp) throw std::runtime_error("cannot open " + path);
    std::string text;
    char buf[4096];
    for (size_t k; (k = std::fread(buf, 1, sizeof buf, fp)) > 0;) text.append(buf, k);
    std::fclose(fp);
    return parse(text);
  }
};

namespace detail {
template <class F>
inline std::string text_of(F&& call) {  // C text builder (buf, cap) -> length: size, then fill
  const int64_t n = call(nullptr, 0);
  if (n < 0) throw std::invalid_argument(ce_last_error());
  std::string t(static_cast<size_t>(n) + 1, '\0');
  call(&t[0], n + 1);
  t.resize(static_cast<size_t>(n));
  return t;
}
}  // namespace detail

inline std::string fmt_double(double v) {  // csv.cpp:84-88
  return detail::text_of([&](char* b, int64_t c) { return int64_t(ce_fmt_double(v, b, static_cast<int>(c))); });
}
inline std::string fmt_index(index_t v) { return std::to_string(v); }  // csv.cpp:90-94

// cli.cpp:60-71
inline CsvTable factor_stats_table(const CEFactorization& f) {
  return CsvTable::parse(detail::text_of([&](char* b, int64_t c) { return ce_factor_stats_csv(f.get(), b, c); }));
}
// cli.cpp:167-182 (recon_error: fmt_double of the relative reconstruction error, or "" above n = 4096)
inline CsvTable factor_summary_table(const CEFactorization& f, index_t block, const CompressionStrategy& s,
                                     double seconds, const std::string& recon_error = "") {
  return CsvTable::parse(detail::text_of(
      [&](char* b, int64_t c) { return ce_factor_summary_csv(f.get(), block, &s.s, seconds, recon_error.c_str(), b, c); }));
}
// cli.cpp:73-80
inline CsvTable trace_table(const IterationTrace& trace) {
  std::vector<int64_t> it;
  std::vector<double> rec, tru, sec;
  for (const auto& smp : trace.samples) {
    it.push_back(smp.iter);
    rec.push_back(smp.recurrence_resid);
    tru.push_back(smp.true_resid);
    sec.push_back(smp.seconds);
  }
  return CsvTable::parse(detail::text_of([&](char* b, int64_t c) {
    return ce_trace_csv(static_cast<int64_t>(it.size()), it.data(), rec.data(), tru.data(), sec.data(), b, c);
  }));
}
// cli.cpp:233-247; strategy == nullptr prints "none" (no factorization was made)
inline CsvTable solve_report_table(index_t n, const std::string& mode, const CompressionStrategy* strategy,
                                   bool preconditioned, const SolveReport& rep, double factor_seconds,
                                   double solve_seconds) {
  ce_solve_report r{rep.converged ? 1 : 0, rep.iterations, rep.final_recurrence_residual, rep.final_true_residual, 0.0};
  return CsvTable::parse(detail::text_of([&](char* b, int64_t c) {
    return ce_solve_report_csv(n, mode.c_str(), strategy ? &strategy->s : nullptr, preconditioned ? 1 : 0, &r,
                               factor_seconds, solve_seconds, b, c);
  }));
}

}  // namespace ce_b200
