// ORACLE — TEST INFRASTRUCTURE ONLY.
// extern "C" surface over the REFERENCE's own code (/root/reference/proj/src, compiled
// unmodified by oracle/ref/Makefile against the Eigen stand-in in oracle/ref/eigen_subset),
// so the tests can pin the oracle restatement (oracle/*.cpp) against the reference itself and
// bench.py's reference arm can time it.  Everything below is glue: it builds the reference's
// public types (BlockSparseMatrix::from_triplets, CoarseningPlan) from plain arrays and calls
// its public API (ce_factorize, CEFactorization::solve / apply_*, BlockSparseMatrix::matvec,
// minres); `ceref_pcg` adds the PCG loop the reference lacks on top of its ApplyFn contract.
#include <chrono>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "ce/cli.hpp"
#include "ce/csv.hpp"
#include "ce/factorization.hpp"
#include "ce/minres.hpp"
#include "ce/problems.hpp"

namespace {
thread_local std::string g_err;

struct RefProblem {
  ce::BlockSparseMatrix matrix;
  ce::CoarseningPlan plan;
};
struct RefFactor {
  ce::CEFactorization f;
};

int fail(const std::exception& e, int code = 1) {
  g_err = e.what();
  return code;
}

ce::Vector vec(const double* p, long long n) {
  ce::Vector v(static_cast<Eigen::Index>(n));
  std::memcpy(v.data(), p, static_cast<size_t>(n) * sizeof(double));
  return v;
}
void out(const ce::Vector& v, double* p) { std::memcpy(p, v.data(), static_cast<size_t>(v.size()) * sizeof(double)); }
}  // namespace

extern "C" {

const char* ceref_last_error() { return g_err.c_str(); }

// CSB (both triangles, row-major blocks) + plan (per level block -> group, members ascending as
// geometric_block_ordering lists them, problems.cpp:237-246) -> the reference's types.
int ceref_problem(long long n, long long m, const long long* offsets, const long long* row_ptr,
                  const long long* col_idx, const long long* val_ptr, const double* values, long long join,
                  long long n_levels, const long long* level_blocks, const long long* assign, void** h) {
  try {
    std::vector<ce::index_t> offs(offsets, offsets + m + 1);
    std::vector<ce::Triplet> t;
    t.reserve(static_cast<size_t>(val_ptr[row_ptr[m]]));
    for (long long i = 0; i < m; ++i)
      for (long long k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
        const long long j = col_idx[k], bi = offs[i + 1] - offs[i], bj = offs[j + 1] - offs[j];
        for (long long r = 0; r < bi; ++r)
          for (long long c = 0; c < bj; ++c) t.push_back({offs[i] + r, offs[j] + c, values[val_ptr[k] + r * bj + c]});
      }
    auto* p = new RefProblem;
    p->matrix = ce::BlockSparseMatrix::from_triplets(t, ce::BlockPartition::from_offsets(offs));
    p->plan.partition = ce::BlockPartition::from_offsets(offs);
    p->plan.join = join;
    p->plan.initial_permutation.resize(static_cast<size_t>(n));
    for (long long i = 0; i < n; ++i) p->plan.initial_permutation[static_cast<size_t>(i)] = i;
    long long at = 0;
    for (long long l = 0; l < n_levels; ++l) {
      long long ng = 0;
      for (long long b = 0; b < level_blocks[l]; ++b) ng = std::max(ng, assign[at + b] + 1);
      std::vector<std::vector<ce::index_t>> groups(static_cast<size_t>(ng));
      for (long long b = 0; b < level_blocks[l]; ++b) groups[static_cast<size_t>(assign[at + b])].push_back(b);
      at += level_blocks[l];
      p->plan.levels.push_back(std::move(groups));
    }
    *h = p;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}
void ceref_problem_free(void* h) { delete static_cast<RefProblem*>(h); }

int ceref_matvec(void* h, const double* x, double* y) {
  try {
    auto* p = static_cast<RefProblem*>(h);
    out(p->matrix.matvec(vec(x, p->matrix.dim())), y);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// mode 0 = AdaptiveEps (eps, absolute), 1 = FixedRank (rank).  Returns 2 on BreakdownError.
int ceref_factorize(void* h, int mode, double eps, int absolute, long long rank, long long dense_threshold,
                    void** fout, long long* err_level, long long* err_block, double* seconds) {
  try {
    auto* p = static_cast<RefProblem*>(h);
    ce::CompressionStrategy s;
    if (mode == 1) {
      s.mode = ce::CompressionStrategy::Mode::FixedRank;
      s.rank = rank;
    } else {
      s.mode = ce::CompressionStrategy::Mode::AdaptiveEps;
      s.eps = eps;
      s.absolute = absolute != 0;
    }
    ce::FactorOptions o;
    o.dense_threshold = dense_threshold;
    const auto t0 = std::chrono::steady_clock::now();
    auto* f = new RefFactor{ce::ce_factorize(p->matrix, p->plan, s, o)};
    if (seconds) *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *fout = f;
    return 0;
  } catch (const ce::BreakdownError& e) {
    if (err_level) *err_level = e.level();
    if (err_block) *err_block = e.block();
    return fail(e, 2);
  } catch (const std::exception& e) {
    return fail(e);
  }
}
void ceref_factor_free(void* f) { delete static_cast<RefFactor*>(f); }

// which: 0 solve, 1 apply_operator, 2 apply_q, 3 apply_q_transpose
int ceref_apply(void* hf, int which, const double* in, double* o) {
  try {
    const auto& f = static_cast<RefFactor*>(hf)->f;
    const ce::Vector v = vec(in, f.n);
    out(which == 0 ? f.solve(v) : which == 1 ? f.apply_operator(v) : which == 2 ? f.apply_q(v) : f.apply_q_transpose(v), o);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

long long ceref_levels(void* hf) { return static_cast<long long>(static_cast<RefFactor*>(hf)->f.levels.size()); }
long long ceref_tail_dim(void* hf) { return static_cast<RefFactor*>(hf)->f.tail_dim; }
long long ceref_level_m(void* hf, long long l) {
  return static_cast<RefFactor*>(hf)->f.levels[static_cast<size_t>(l)].partition.block_count();
}
// sizes, retained ranks, basis flags, widths of level l; groups flattened (group sizes + members)
void ceref_level_structure(void* hf, long long l, long long* sizes, long long* retained, long long* has_basis,
                           long long* width) {
  const auto& fl = static_cast<RefFactor*>(hf)->f.levels[static_cast<size_t>(l)];
  for (ce::index_t b = 0; b < fl.partition.block_count(); ++b) {
    sizes[b] = fl.partition.block_size(b);
    retained[b] = fl.retained[static_cast<size_t>(b)];
    has_basis[b] = fl.basis[static_cast<size_t>(b)].size() != 0;
    width[b] = fl.rows[static_cast<size_t>(b)].width;
  }
}
// LevelStats row: block_count, pattern_blocks, factor_blocks, eliminated, retained, max_rank,
// mean_rank, seconds, l_bytes, q_bytes, shift_retries
void ceref_level_stats(void* hf, long long l, double* o) {
  const auto& s = static_cast<RefFactor*>(hf)->f.stats.levels[static_cast<size_t>(l)];
  const double v[11] = {double(s.block_count), double(s.pattern_blocks), double(s.factor_blocks), double(s.eliminated),
                        double(s.retained), double(s.max_rank), s.mean_rank, s.seconds, double(s.l_bytes),
                        double(s.q_bytes), double(s.shift_retries)};
  std::memcpy(o, v, sizeof v);
}
// FactorStats: factor_blocks, predicted_factor_blocks, l_scalar_nnz, l_payload_bytes, q_payload_bytes,
// tail_bytes, total_seconds
void ceref_factor_summary(void* hf, double* o) {
  const auto& s = static_cast<RefFactor*>(hf)->f.stats;
  const double v[7] = {s.factor_blocks, s.predicted_factor_blocks, double(s.l_scalar_nnz), double(s.l_payload_bytes),
                       double(s.q_payload_bytes), double(s.tail_bytes), s.total_seconds};
  std::memcpy(o, v, sizeof v);
}

// method 0 = PCG (added here over the reference's ApplyFn contract, minres.hpp:46-47; the
// reference has no PCG), 1 = the reference's minres.  hf may be null (unpreconditioned).
int ceref_krylov(void* hp, void* hf, int method, const double* b, double* x, double tol, long long maxit,
                 int track_true, long long* iters, double* rec, double* true_resid, int* converged, double* seconds) {
  try {
    auto* p = static_cast<RefProblem*>(hp);
    const ce::index_t n = p->matrix.dim();
    ce::ApplyFn a = [&](const ce::Vector& v) { return p->matrix.matvec(v); };
    ce::ApplyFn m;
    if (hf) m = [&](const ce::Vector& v) { return static_cast<RefFactor*>(hf)->f.solve(v); };
    const ce::Vector bv = vec(b, n);
    const auto t0 = std::chrono::steady_clock::now();
    ce::Vector xv;
    ce::SolveReport rep;
    if (method == 1) {
      ce::MinresOptions o;
      o.tol = tol;
      o.maxit = maxit;
      o.track_true_residual = track_true != 0;
      rep = ce::minres(a, n, bv, m, o, xv);
    } else {  // x0 = 0, stop on ||r_k|| / ||b|| <= tol, iterations = A*p products
      xv = ce::Vector::Zero(n);
      const double bn = bv.norm();
      rep.converged = bn == 0.0;
      if (!rep.converged) {
        ce::Vector r = bv, z = m ? m(r) : r, pv = z;
        double rz = r.dot(z);
        for (ce::index_t it = 1; it <= maxit; ++it) {
          const ce::Vector q = a(pv);
          const double alpha = rz / pv.dot(q);
          xv += alpha * pv;
          r -= alpha * q;
          rep.iterations = it;
          rep.final_recurrence_residual = r.norm() / bn;
          if (rep.final_recurrence_residual <= tol) {
            rep.converged = true;
            break;
          }
          z = m ? m(r) : r;
          const double rzn = r.dot(z);
          pv = z + (rzn / rz) * pv;
          rz = rzn;
        }
      }
      rep.final_true_residual = ce::relative_residual(a, xv, bv);
    }
    if (seconds) *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    out(xv, x);
    *iters = rep.iterations;
    *rec = rep.final_recurrence_residual;
    *true_resid = rep.final_true_residual;
    *converged = rep.converged ? 1 : 0;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// ---- the reference CLI's `file` flow and CSV reports (cli.cpp:114-133,153-247; csv.cpp) ----
static ce::BenchConfig file_config(const char* matrix, const char* rhs, const char* plan, long long block,
                                   int use_rank, long long rank, double eps, int absolute,
                                   long long dense_threshold, const char* out_dir) {
  ce::BenchConfig cfg;
  cfg.problem = "file";
  cfg.matrix_path = matrix ? matrix : "";
  cfg.rhs_path = rhs ? rhs : "";
  cfg.plan_path = plan ? plan : "";
  cfg.block = block;
  cfg.use_rank = use_rank != 0;
  cfg.rank = rank;
  cfg.eps = eps;
  cfg.eps_absolute = absolute != 0;
  cfg.dense_threshold = dense_threshold;
  cfg.out_dir = out_dir;
  return cfg;
}

// run_factor on a `file` problem: writes factor_stats.csv and factor_summary.csv into out_dir;
// returns the CLI exit code.
int ceref_run_factor(const char* matrix, const char* rhs, const char* plan, long long block, int use_rank,
                     long long rank, double eps, int absolute, long long dense_threshold, const char* out_dir) {
  return ce::run_factor(file_config(matrix, rhs, plan, block, use_rank, rank, eps, absolute, dense_threshold, out_dir));
}

// run_solve on a `file` problem: x.txt, trace.csv, solve_report.csv into out_dir.
int ceref_run_solve(const char* matrix, const char* rhs, const char* plan, long long block, int use_rank,
                    long long rank, double eps, int absolute, long long dense_threshold, double tol,
                    long long maxit, int direct, int no_precond, const char* out_dir) {
  ce::BenchConfig cfg = file_config(matrix, rhs, plan, block, use_rank, rank, eps, absolute, dense_threshold, out_dir);
  cfg.tol = tol;
  cfg.maxit = maxit;
  cfg.direct = direct != 0;
  cfg.no_precond = no_precond != 0;
  return ce::run_solve(cfg);
}

int ceref_fmt_double(double v, char* buf, int cap) {
  const std::string t = ce::fmt_double(v);
  if (static_cast<int>(t.size()) < cap) std::memcpy(buf, t.c_str(), t.size() + 1);
  return static_cast<int>(t.size());
}

// CsvTable::parse followed by to_string (csv.hpp: reproduces the input bytes); returns the length
// written (< 0: parse threw).
long long ceref_csv_roundtrip(const char* text, char* buf, long long cap) {
  try {
    const std::string t = ce::CsvTable::parse(text).to_string();
    if (static_cast<long long>(t.size()) < cap) std::memcpy(buf, t.c_str(), t.size() + 1);
    return static_cast<long long>(t.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int ceref_describe(int use_rank, long long rank, double eps, int absolute, char* buf, int cap) {
  const std::string t = (use_rank ? ce::CompressionStrategy::fixed_rank(rank)
                                  : ce::CompressionStrategy::adaptive(eps, absolute != 0)).describe();
  if (static_cast<int>(t.size()) < cap) std::memcpy(buf, t.c_str(), t.size() + 1);
  return static_cast<int>(t.size());
}

}  // extern "C"
