// ORACLE — TEST INFRASTRUCTURE ONLY (see dense.hpp).
// extern "C" surface of the oracle for the Python test-suite (ctypes) and for
// bench.py's cpu_baseline leg.  Never linked into the product library.
#include <cstring>
#include <exception>
#include <memory>
#include <string>

#include "factor.hpp"
#include "krylov.hpp"

using namespace oracle;

namespace {
thread_local std::string g_err;
int fail(const std::exception& e, int code = 1) {
  g_err = e.what();
  return code;
}

struct OProblem {
  BlockSparseMatrix matrix;
  std::vector<double> rhs;
  CoarseningPlan plan;
};

struct OFactor {
  CEFactorization f;
};

CompressionStrategy make_strategy(int mode, double eps, int absolute, index_t rank) {
  return mode == 1 ? CompressionStrategy::fixed_rank(rank) : CompressionStrategy::adaptive(eps, absolute != 0);
}
}  // namespace

extern "C" {

const char* oracle_last_error() { return g_err.c_str(); }

// Problem from a BASELINE config (id 1..5) with optional grid override (0 = keep).
int oracle_problem_config_plan(int id, long long nx, long long ny, long long nz, int plan_kind, void** out);
int oracle_problem_config(int id, long long nx, long long ny, long long nz, void** out) {
  return oracle_problem_config_plan(id, nx, ny, nz, 0, out);
}

// Same with the plan family (0 = reference geometric_block_ordering, 1 = all axes merge per level,
// 2 = all-axis merges with mod-3 colour-major cells).
int oracle_problem_config_plan(int id, long long nx, long long ny, long long nz, int plan_kind, void** out) {
  try {
    ProblemConfig c = baseline_config(id);
    c.plan_kind = plan_kind;
    if (nx > 0) c.nx = nx;
    if (ny > 0) c.ny = ny;
    if (nz > 0 && c.dims == 3) c.nz = nz;
    LoadedProblem lp = load_config(c);
    auto* p = new OProblem{std::move(lp.matrix), std::move(lp.rhs), std::move(lp.plan)};
    *out = p;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Generic problem: reference 3-D diffusion (kind 0) or 2-D 9-point Laplacian (kind 1).
int oracle_problem_reference(int kind, long long nx, long long ny, long long nz, long long block, void** out) {
  try {
    AssembledSystem sys;
    CoarseningPlan plan;
    if (kind == 0) {
      Grid3D g{nx, ny, nz};
      sys = assemble_diffusion_3d(g);
      plan = geometric_block_ordering(g, block, 2);
    } else {
      sys = assemble_laplace_2d_9pt(nx);
      plan = geometric_block_ordering(Grid3D{nx, nx, 1}, block, 2);
    }
    auto* p = new OProblem;
    p->matrix = BlockSparseMatrix::from_triplets(apply_permutation(sys.entries, plan.initial_permutation),
                                                 plan.partition);
    p->rhs = permute_vector(sys.rhs, plan.initial_permutation);
    p->plan = std::move(plan);
    *out = p;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Problem from scalar triplets with an explicit block partition and trivial plan.
int oracle_problem_triplets(long long n, long long nnz, const long long* rows, const long long* cols,
                            const double* vals, long long m, const long long* offsets, int mirror_lower,
                            void** out) {
  try {
    std::vector<Triplet> t(static_cast<size_t>(nnz));
    for (long long k = 0; k < nnz; ++k) t[static_cast<size_t>(k)] = {rows[k], cols[k], vals[k]};
    std::vector<index_t> offs(offsets, offsets + m + 1);
    auto* p = new OProblem;
    p->plan.partition = BlockPartition::from_offsets(offs);
    p->plan.initial_permutation.resize(static_cast<size_t>(n));
    for (long long i = 0; i < n; ++i) p->plan.initial_permutation[static_cast<size_t>(i)] = i;
    p->matrix = BlockSparseMatrix::from_triplets(t, p->plan.partition,
                                                 mirror_lower ? MirrorMode::Lower : MirrorMode::None);
    p->rhs.assign(static_cast<size_t>(n), 1.0);
    *out = p;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

void oracle_problem_free(void* p) { delete static_cast<OProblem*>(p); }

// Conditioning probe: multiply every off-diagonal-symmetric pair of stored values by
// (1 + rel * z), z a deterministic N(0,1) draw; the matrix stays exactly symmetric.
void oracle_problem_perturb(void* h, double rel, unsigned long long seed) {
  auto* p = static_cast<OProblem*>(h);
  auto& a = p->matrix;
  const index_t m = a.partition().block_count();
  for (index_t i = 0; i < m; ++i)
    for (index_t j : a.pattern().row(i)) {
      if (j > i) continue;
      Mat& bij = a.block(i, j);
      Mat& bji = a.block(j, i);
      for (index_t r = 0; r < bij.r; ++r)
        for (index_t c = 0; c < bij.c; ++c) {
          if (i == j && c > r) continue;
          const std::uint64_t key = static_cast<std::uint64_t>(((i * 1000003 + j) * 64 + r) * 64 + c);
          const double f = 1.0 + rel * normal_sample(seed, 7, key);
          bij(r, c) *= f;
          if (i == j) {
            if (c != r) bij(c, r) = bij(r, c);
          } else {
            bji(c, r) = bij(r, c);
          }
        }
    }
}

long long oracle_problem_n(void* p) { return static_cast<OProblem*>(p)->matrix.dim(); }
long long oracle_problem_m(void* p) { return static_cast<OProblem*>(p)->matrix.partition().block_count(); }
long long oracle_problem_nnzb(void* p) { return static_cast<OProblem*>(p)->matrix.pattern().stored_blocks(); }
long long oracle_problem_values(void* p) {
  return static_cast<OProblem*>(p)->matrix.payload_bytes() / static_cast<long long>(sizeof(double));
}

// CSB export (reference layout: both triangles).  val_ptr has nnzb + 1 entries.
void oracle_problem_csb(void* h, long long* offsets, long long* row_ptr, long long* col_idx, long long* val_ptr,
                        double* values) {
  auto* p = static_cast<OProblem*>(h);
  const auto& a = p->matrix;
  const index_t m = a.partition().block_count();
  for (index_t i = 0; i <= m; ++i) offsets[i] = a.partition().offsets()[static_cast<size_t>(i)];
  long long at = 0, vat = 0;
  row_ptr[0] = 0;
  for (index_t i = 0; i < m; ++i) {
    const auto& cols = a.pattern().row(i);
    for (size_t k = 0; k < cols.size(); ++k) {
      col_idx[at] = cols[k];
      val_ptr[at] = vat;
      const Mat& b = a.slot_block(i, k);
      std::memcpy(values + vat, b.a.data(), b.a.size() * sizeof(double));
      vat += b.size();
      ++at;
    }
    row_ptr[i + 1] = at;
  }
  val_ptr[at] = vat;
}

void oracle_problem_rhs(void* h, double* out) {
  auto* p = static_cast<OProblem*>(h);
  std::memcpy(out, p->rhs.data(), p->rhs.size() * sizeof(double));
}

void oracle_problem_perm(void* h, long long* out) {
  auto* p = static_cast<OProblem*>(h);
  for (size_t i = 0; i < p->plan.initial_permutation.size(); ++i) out[i] = p->plan.initial_permutation[i];
}

long long oracle_plan_levels(void* h) { return static_cast<long long>(static_cast<OProblem*>(h)->plan.levels.size()); }
long long oracle_plan_join(void* h) { return static_cast<OProblem*>(h)->plan.join; }
// Blocks at plan level l (the size of its assignment array).
long long oracle_plan_level_blocks(void* h, long long l) {
  long long n = 0;
  for (const auto& g : static_cast<OProblem*>(h)->plan.levels[static_cast<size_t>(l)]) n += static_cast<long long>(g.size());
  return n;
}
void oracle_plan_level_assign(void* h, long long l, long long* assign) {
  const auto& lev = static_cast<OProblem*>(h)->plan.levels[static_cast<size_t>(l)];
  for (size_t g = 0; g < lev.size(); ++g)
    for (index_t b : lev[g]) assign[b] = static_cast<long long>(g);
}

int oracle_matvec(void* h, const double* x, double* y) {
  try {
    auto* p = static_cast<OProblem*>(h);
    std::vector<double> xv(x, x + p->matrix.dim());
    auto yv = p->matrix.matvec(xv);
    std::memcpy(y, yv.data(), yv.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

void oracle_problem_dense(void* h, double* out) {
  auto d = static_cast<OProblem*>(h)->matrix.to_dense();
  std::memcpy(out, d.data(), d.size() * sizeof(double));
}

// forced: optional flat array (-1 = free) over levels, forced_counts[l] rows each.
int oracle_factorize(void* h, int mode, double eps, int absolute, long long rank, long long dense_threshold,
                     long long n_forced_levels, const long long* forced_counts, const long long* forced,
                     void** out, long long* err_level, long long* err_block) {
  try {
    auto* p = static_cast<OProblem*>(h);
    FactorOptions o;
    o.dense_threshold = dense_threshold;
    long long at = 0;
    for (long long l = 0; l < n_forced_levels; ++l) {
      std::vector<index_t> fr(forced + at, forced + at + forced_counts[l]);
      at += forced_counts[l];
      o.forced_ranks.push_back(std::move(fr));
    }
    auto* f = new OFactor{ce_factorize(p->matrix, p->plan, make_strategy(mode, eps, absolute, rank), o)};
    *out = f;
    return 0;
  } catch (const BreakdownError& e) {
    if (err_level) *err_level = e.level();
    if (err_block) *err_block = e.block();
    return fail(e, 2);
  } catch (const std::exception& e) {
    return fail(e);
  }
}

void oracle_factor_free(void* f) { delete static_cast<OFactor*>(f); }

int oracle_factor_solve(void* h, const double* b, double* x) {
  try {
    auto* f = static_cast<OFactor*>(h);
    auto xv = f->f.solve(std::vector<double>(b, b + f->f.n));
    std::memcpy(x, xv.data(), xv.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int oracle_factor_apply(void* h, int which, const double* in, double* out) {
  try {
    auto* f = static_cast<OFactor*>(h);
    std::vector<double> v(in, in + f->f.n), r;
    if (which == 0) r = f->f.apply_operator(v);
    else if (which == 1) r = f->f.apply_q(v);
    else r = f->f.apply_q_transpose(v);
    std::memcpy(out, r.data(), r.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int oracle_factor_reconstruct(void* h, double* out) {
  try {
    auto d = static_cast<OFactor*>(h)->f.reconstruct_dense();
    std::memcpy(out, d.data(), d.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int oracle_factor_dump(void* h, const char* path) {
  try {
    write_factor_dump(static_cast<OFactor*>(h)->f, path);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

long long oracle_factor_levels(void* h) { return static_cast<long long>(static_cast<OFactor*>(h)->f.levels.size()); }
long long oracle_factor_tail_dim(void* h) { return static_cast<OFactor*>(h)->f.tail_dim; }

// Per-level structure for the full-size fixtures (scripts/make_fullsize_fixture.py):
// block sizes, retained ranks and far widths of level l (M entries each).
long long oracle_factor_level_m(void* h, long long l) {
  return static_cast<OFactor*>(h)->f.levels[static_cast<size_t>(l)].partition.block_count();
}
void oracle_factor_level_structure(void* h, long long l, long long* sizes, long long* retained, long long* fcols) {
  const auto& fl = static_cast<OFactor*>(h)->f.levels[static_cast<size_t>(l)];
  for (index_t b = 0; b < fl.partition.block_count(); ++b) {
    sizes[b] = fl.partition.block_size(b);
    retained[b] = fl.retained[static_cast<size_t>(b)];
    fcols[b] = fl.fcols[static_cast<size_t>(b)];
  }
}
// Singular values of row b's far concatenation at level l; returns their count (<= cap written).
long long oracle_factor_row_sigma(void* h, long long l, long long b, double* out, long long cap) {
  const auto& s = static_cast<OFactor*>(h)->f.levels[static_cast<size_t>(l)].sigma[static_cast<size_t>(b)];
  for (size_t k = 0; k < s.size() && static_cast<long long>(k) < cap; ++k) out[k] = s[k];
  return static_cast<long long>(s.size());
}

// Summary stats: [factor_blocks, predicted_factor_blocks, l_scalar_nnz, l_payload_bytes,
// q_payload_bytes, tail_bytes, total_seconds, tail_seconds]
void oracle_factor_summary(void* h, double* out) {
  const auto& s = static_cast<OFactor*>(h)->f.stats;
  out[0] = s.factor_blocks;
  out[1] = s.predicted_factor_blocks;
  out[2] = static_cast<double>(s.l_scalar_nnz);
  out[3] = static_cast<double>(s.l_payload_bytes);
  out[4] = static_cast<double>(s.q_payload_bytes);
  out[5] = static_cast<double>(s.tail_bytes);
  out[6] = s.total_seconds;
  out[7] = s.tail_seconds;
}

// Per-level stats row: [block_count, pattern_blocks, factor_blocks, eliminated, retained, max_rank,
// mean_rank, seconds, l_bytes, q_bytes, shift_retries, predicted_edge]
void oracle_factor_level_stats(void* h, long long l, double* out) {
  const auto& s = static_cast<OFactor*>(h)->f.stats;
  const auto& ls = s.levels[static_cast<size_t>(l)];
  out[0] = static_cast<double>(ls.block_count);
  out[1] = static_cast<double>(ls.pattern_blocks);
  out[2] = static_cast<double>(ls.factor_blocks);
  out[3] = static_cast<double>(ls.eliminated);
  out[4] = static_cast<double>(ls.retained);
  out[5] = static_cast<double>(ls.max_rank);
  out[6] = ls.mean_rank;
  out[7] = ls.seconds;
  out[8] = static_cast<double>(ls.l_bytes);
  out[9] = static_cast<double>(ls.q_bytes);
  out[10] = static_cast<double>(ls.shift_retries);
  out[11] = static_cast<size_t>(l) < s.predicted_level_edges.size()
                ? static_cast<double>(s.predicted_level_edges[static_cast<size_t>(l)])
                : -1.0;
}

// Krylov on a problem with an optional factor preconditioner.  method 0 = pcg, 1 = minres.
int oracle_krylov(void* hp, void* hf, int method, const double* b, double* x, double tol, long long maxit,
                  int track_true, long long* iters, double* rec_resid, double* true_resid, int* converged,
                  double* seconds) {
  try {
    auto* p = static_cast<OProblem*>(hp);
    auto* f = static_cast<OFactor*>(hf);
    const index_t n = p->matrix.dim();
    ApplyFn a = [&](const Vec& v) { return p->matrix.matvec(v); };
    ApplyFn m;
    if (f) m = [&](const Vec& v) { return f->f.solve(v); };
    Vec bv(b, b + n), xv;
    SolveReport rep;
    if (method == 0) {
      PcgOptions o;
      o.tol = tol;
      o.maxit = maxit;
      o.track_true_residual = track_true != 0;
      rep = pcg(a, n, bv, m, o, xv);
    } else {
      MinresOptions o;
      o.tol = tol;
      o.maxit = maxit;
      o.track_true_residual = track_true != 0;
      rep = minres(a, n, bv, m, o, xv);
    }
    std::memcpy(x, xv.data(), xv.size() * sizeof(double));
    *iters = rep.iterations;
    *rec_resid = rep.final_recurrence_residual;
    *true_resid = rep.final_true_residual;
    *converged = rep.converged ? 1 : 0;
    *seconds = rep.trace.empty() ? 0.0 : rep.trace.back().seconds;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Compression KAT hook: F is b x f row-major; U (b x b) written when a basis exists.
int oracle_compress(long long b, long long f, const double* F, int mode, double eps, int absolute, long long rank,
                    long long* retained, int* has_basis, double* U, double* sigma, long long* nsigma) {
  try {
    Mat m(b, f);
    std::memcpy(m.a.data(), F, static_cast<size_t>(b * f) * sizeof(double));
    RowCompression c = compress_far_concat(m, b, make_strategy(mode, eps, absolute, rank));
    *retained = c.retained;
    *has_basis = c.basis.empty() ? 0 : 1;
    if (!c.basis.empty()) std::memcpy(U, c.basis.a.data(), c.basis.a.size() * sizeof(double));
    *nsigma = static_cast<long long>(c.sigma.size());
    for (size_t k = 0; k < c.sigma.size(); ++k) sigma[k] = c.sigma[k];
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Pattern algebra KAT hooks over CSR patterns.  op 0 = square, 1 = far, 2 = coarsen (groups
// given as assign[m] -> group id, ng groups).  Output capacity `cap`; returns nnz or -1.
long long oracle_pattern_op(int op, long long m, const long long* row_ptr, const long long* cols, long long ng,
                            const long long* assign, long long* out_row_ptr, long long* out_cols, long long cap) {
  try {
    BlockSparsityPattern p(m);
    for (long long i = 0; i < m; ++i)
      for (long long k = row_ptr[i]; k < row_ptr[i + 1]; ++k) p.insert(i, cols[k]);
    BlockSparsityPattern q;
    if (op == 0) q = pattern_square(p);
    else if (op == 1) q = far_pattern(p);
    else {
      std::vector<std::vector<index_t>> groups(static_cast<size_t>(ng));
      for (long long b = 0; b < m; ++b) groups[static_cast<size_t>(assign[b])].push_back(b);
      q = coarsen_pattern(p, groups);
    }
    long long at = 0;
    out_row_ptr[0] = 0;
    for (index_t i = 0; i < q.block_rows(); ++i) {
      for (index_t j : q.row(i)) {
        if (at >= cap) return -1;
        out_cols[at++] = j;
      }
      out_row_ptr[i + 1] = at;
    }
    return at;
  } catch (const std::exception& e) {
    fail(e);
    return -1;
  }
}

}  // extern "C"
