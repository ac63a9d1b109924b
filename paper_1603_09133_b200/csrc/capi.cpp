// C-ABI of the library (include/ce_gpu.h).  No exceptions cross this layer;
// return codes follow the reference CLI exit codes (proj/include/ce/cli.hpp:16-19,
// exception mapping of proj/src/cli.cpp:82-95).
#include <algorithm>
#include <charconv>
#include <cstring>
#include <sstream>
#include <exception>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/ce_gpu.h"
#include "assemble.hpp"
#include "pattern.hpp"
#include "driver.hpp"
#include "kernels.hpp"

struct ce_ctx {
  ceg::Context ctx;
  ceg::SolveOut last_solve;  // the last ce_pcg / ce_minres of this context (ce_ctx_last_trace)
};
struct ce_matrix {
  ceg::Matrix m;
};
struct ce_problem {
  ceg::Problem p;
};
struct ce_factor {
  std::unique_ptr<ceg::Factor> f;
  // symbolic inputs kept for the lazily computed predicted_nnz (factorization.cpp:463-485)
  std::vector<int64_t> a_ptr;
  std::vector<int> a_col;
  std::vector<int64_t> plan_blocks, plan_assign;
  int64_t join = 2, rank_hint = 1, bmax = 1;
  double predicted = -1.0;
  // host-buffer path of ce_apply_precond: staging buffers, one call at a time
  mutable std::mutex stage_mu;
  mutable ceg::DevArray<double> stage_in, stage_out;
};

namespace {
thread_local std::string g_err;

int fail(const std::exception& e, int code = CE_EUSAGE) {
  g_err = e.what();
  return code;
}

template <class F>
int guarded(F&& body, ce_status* st = nullptr) {
  try {
    body();
    if (st) st->code = CE_OK;
    return CE_OK;
  } catch (const ceg::Breakdown& e) {
    if (st) {
      st->code = CE_EBREAKDOWN;
      st->level = e.level;
      st->block = e.block;
      std::strncpy(st->message, e.what(), sizeof st->message - 1);
    }
    return fail(e, CE_EBREAKDOWN);
  } catch (const std::exception& e) {
    if (st) {
      st->code = CE_EUSAGE;
      std::strncpy(st->message, e.what(), sizeof st->message - 1);
    }
    return fail(e);
  }
}

// Boolean square + coarsening iteration of predicted_nnz.
double predicted_nnz(const ce_factor& h, int64_t k_levels, std::vector<int64_t>* edges_out) {
  std::vector<int64_t> ptr = h.a_ptr;
  std::vector<int> col = h.a_col;
  int64_t last_blocks = static_cast<int64_t>(ptr.size()) - 1;
  std::vector<int64_t> edges;
  int64_t at = 0;
  for (int64_t l = 0; l < k_levels; ++l) {
    const int64_t m = static_cast<int64_t>(ptr.size()) - 1;
    int64_t lower = 0;
    for (int64_t i = 0; i < m; ++i)
      for (int64_t k = ptr[static_cast<size_t>(i)]; k < ptr[static_cast<size_t>(i + 1)]; ++k)
        if (col[static_cast<size_t>(k)] <= i) ++lower;
    edges.push_back(lower);
    last_blocks = m;
    std::vector<int64_t> group_of(static_cast<size_t>(m));
    int64_t ng = 0;
    if (l < static_cast<int64_t>(h.plan_blocks.size())) {
      for (int64_t b = 0; b < m; ++b) {
        group_of[static_cast<size_t>(b)] = h.plan_assign[static_cast<size_t>(at + b)];
        ng = std::max(ng, group_of[static_cast<size_t>(b)] + 1);
      }
      at += h.plan_blocks[static_cast<size_t>(l)];
    } else {
      for (int64_t b = 0; b < m; ++b) group_of[static_cast<size_t>(b)] = b / h.join;
      ng = (m + h.join - 1) / h.join;
    }
    // coarsen(square(p))
    std::vector<int64_t> mark(static_cast<size_t>(m), -1), gmark(static_cast<size_t>(ng), -1);
    std::vector<std::vector<int>> rows(static_cast<size_t>(ng));
    for (int64_t i = 0; i < m; ++i) {
      const int64_t gi = group_of[static_cast<size_t>(i)];
      for (int64_t k = ptr[static_cast<size_t>(i)]; k < ptr[static_cast<size_t>(i + 1)]; ++k) {
        const int kk = col[static_cast<size_t>(k)];
        for (int64_t e = ptr[static_cast<size_t>(kk)]; e < ptr[static_cast<size_t>(kk + 1)]; ++e) {
          const int64_t gj = group_of[static_cast<size_t>(col[static_cast<size_t>(e)])];
          if (gmark[static_cast<size_t>(gj)] == gi) continue;
          gmark[static_cast<size_t>(gj)] = gi;
          rows[static_cast<size_t>(gi)].push_back(static_cast<int>(gj));
        }
      }
      // groups may be non-contiguous: reset marks per block so dedup happens after sorting
      for (int64_t k = ptr[static_cast<size_t>(i)]; k < ptr[static_cast<size_t>(i + 1)]; ++k) {
        const int kk = col[static_cast<size_t>(k)];
        for (int64_t e = ptr[static_cast<size_t>(kk)]; e < ptr[static_cast<size_t>(kk + 1)]; ++e)
          gmark[static_cast<size_t>(group_of[static_cast<size_t>(col[static_cast<size_t>(e)])])] = -1;
      }
    }
    std::vector<int64_t> nptr(static_cast<size_t>(ng + 1), 0);
    std::vector<int> ncol;
    for (int64_t g = 0; g < ng; ++g) {
      auto& r = rows[static_cast<size_t>(g)];
      std::sort(r.begin(), r.end());
      r.erase(std::unique(r.begin(), r.end()), r.end());
      ncol.insert(ncol.end(), r.begin(), r.end());
      nptr[static_cast<size_t>(g + 1)] = static_cast<int64_t>(ncol.size());
    }
    ptr = std::move(nptr);
    col = std::move(ncol);
    (void)mark;
  }
  const double tail_rows = k_levels == 0 ? static_cast<double>(last_blocks) * static_cast<double>(h.bmax)
                                         : static_cast<double>(last_blocks) * static_cast<double>(h.rank_hint);
  double total = 0.5 * tail_rows * tail_rows;
  for (int64_t e : edges) total += 2.0 * static_cast<double>(e);
  if (edges_out) *edges_out = edges;
  return total;
}

// live contexts per device: the allocator cache of a device is trimmed when its last context goes
std::mutex g_ctx_mu;
std::map<int, int> g_live_ctx;
}  // namespace

extern "C" {

const char* ce_last_error(void) { return g_err.c_str(); }

int ce_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  int k = 0;
  for (int d = 0; d < n; ++d) {
    cudaDeviceProp p{};
    if (cudaGetDeviceProperties(&p, d) == cudaSuccess && p.major == 10) ++k;
  }
  return k;
}

int ce_ctx_create(int device, ce_ctx** out) {
  return guarded([&] {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
      cudaGetLastError();
      throw std::runtime_error("no CUDA device visible: the CE hot path requires an sm_100a GPU (no CPU fallback)");
    }
    if (device < 0 || device >= n) throw std::invalid_argument("device index out of range");
    cudaDeviceProp p{};
    CE_CUDA(cudaGetDeviceProperties(&p, device));
    if (p.major != 10) throw std::runtime_error("device is not sm_100 (Blackwell B200 required)");
    CE_CUDA(cudaSetDevice(device));
    auto c = std::make_unique<ce_ctx>();
    c->ctx.device = device;
    c->ctx.sm_count = p.multiProcessorCount;
    CE_CUDA(cudaStreamCreateWithFlags(&c->ctx.stream, cudaStreamNonBlocking));
    {
      std::lock_guard<std::mutex> lk(g_ctx_mu);
      ++g_live_ctx[device];
    }
    *out = c.release();
  });
}

int ce_ctx_stream(const ce_ctx* ctx, void** stream) {
  if (!ctx || !stream) return CE_EUSAGE;
  *stream = ctx->ctx.stream;
  return CE_OK;
}

int64_t ce_launch_count(void) { return ceg::launch_count(); }

void ce_ctx_destroy(ce_ctx* ctx) {
  if (!ctx) return;
  if (ctx->ctx.stream) {
    cudaStreamSynchronize(ctx->ctx.stream);
    cudaStreamDestroy(ctx->ctx.stream);
  }
  const int dev = ctx->ctx.device;
  delete ctx;
  bool last = false;
  {
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    last = --g_live_ctx[dev] <= 0;
    if (last) g_live_ctx.erase(dev);
  }
  if (last) ceg::pool_trim(dev);  // the device's cached blocks go back with its last context
}

int ce_matrix_upload(ce_ctx* ctx, const ce_csb_host* a, ce_matrix** out) {
  return guarded([&] {
    if (!ctx || !a) throw std::invalid_argument("null argument");
    CE_CUDA(cudaSetDevice(ctx->ctx.device));
    auto h = std::make_unique<ce_matrix>();
    ceg::Matrix& M = h->m;
    M.ctx = &ctx->ctx;
    M.n = a->n;
    M.m = a->m;
    M.offsets.assign(a->offsets, a->offsets + a->m + 1);
    M.row_ptr.assign(a->row_ptr, a->row_ptr + a->m + 1);
    M.nnzb = M.row_ptr.back();
    M.col_idx.assign(a->col_idx, a->col_idx + M.nnzb);
    M.val_ptr.assign(a->val_ptr, a->val_ptr + M.nnzb + 1);
    if (M.offsets.front() != 0 || M.offsets.back() != M.n) throw std::invalid_argument("partition offsets must span [0, n)");
    for (int64_t i = 0; i < M.m; ++i) {
      if (M.offsets[static_cast<size_t>(i + 1)] <= M.offsets[static_cast<size_t>(i)])
        throw std::invalid_argument("partition offsets must be strictly increasing");
      bool diag = false;
      for (int64_t k = M.row_ptr[static_cast<size_t>(i)]; k < M.row_ptr[static_cast<size_t>(i + 1)]; ++k) {
        const int64_t j = M.col_idx[static_cast<size_t>(k)];
        if (j < 0 || j >= M.m) throw std::invalid_argument("pattern position outside block grid");
        if (k > M.row_ptr[static_cast<size_t>(i)] && j <= M.col_idx[static_cast<size_t>(k - 1)])
          throw std::invalid_argument("pattern rows must be sorted and unique");
        if (j == i) diag = true;
        const int64_t need = (M.offsets[static_cast<size_t>(i + 1)] - M.offsets[static_cast<size_t>(i)]) *
                             (M.offsets[static_cast<size_t>(j + 1)] - M.offsets[static_cast<size_t>(j)]);
        if (M.val_ptr[static_cast<size_t>(k + 1)] - M.val_ptr[static_cast<size_t>(k)] != need)
          throw std::invalid_argument("block value extent does not match the partition");
      }
      if (!diag) throw std::invalid_argument("pattern must contain all diagonal positions");
    }
    cudaStream_t s = ctx->ctx.stream;
    M.d_offsets.upload(M.offsets, s);
    M.d_row_ptr.upload(M.row_ptr, s);
    M.d_val_ptr.upload(M.val_ptr, s);
    std::vector<int> col(M.col_idx.begin(), M.col_idx.end()), bsz(static_cast<size_t>(M.m));
    for (int64_t i = 0; i < M.m; ++i) bsz[static_cast<size_t>(i)] = static_cast<int>(M.offsets[static_cast<size_t>(i + 1)] - M.offsets[static_cast<size_t>(i)]);
    M.d_col_idx.upload(col, s);
    M.d_bsz.upload(bsz, s);
    std::vector<int64_t> row_of(static_cast<size_t>(M.n));
    for (int64_t i = 0; i < M.m; ++i)
      for (int64_t p = M.offsets[static_cast<size_t>(i)]; p < M.offsets[static_cast<size_t>(i + 1)]; ++p) row_of[static_cast<size_t>(p)] = i;
    M.d_row_of.upload(row_of, s);
    M.d_values.alloc(static_cast<size_t>(M.val_ptr.back()));
    CE_CUDA(cudaMemcpyAsync(M.d_values.p, a->values, static_cast<size_t>(M.val_ptr.back()) * sizeof(double),
                            cudaMemcpyHostToDevice, s));
    CE_CUDA(cudaStreamSynchronize(s));
    *out = h.release();
  });
}

int ce_matrix_from_triplets(ce_ctx* ctx, int64_t n, int64_t nnz, const int64_t* rows, const int64_t* cols,
                            const double* vals, int64_t m, const int64_t* offsets, int mirror_lower, int on_device,
                            ce_matrix** out) {
  return guarded([&] {
    if (!ctx || !out || !offsets || (nnz > 0 && (!rows || !cols || !vals))) throw std::invalid_argument("null argument");
    if (m < 1 || n < 1) throw std::invalid_argument("empty partition");
    std::vector<int64_t> offs(offsets, offsets + m + 1);  // BlockPartition::from_offsets (partition.cpp)
    if (offs.front() != 0 || offs.back() != n) throw std::invalid_argument("partition offsets must span [0, n)");
    for (int64_t i = 0; i < m; ++i)
      if (offs[static_cast<size_t>(i + 1)] <= offs[static_cast<size_t>(i)])
        throw std::invalid_argument("partition offsets must be strictly increasing");
    CE_CUDA(cudaSetDevice(ctx->ctx.device));
    cudaStream_t s = ctx->ctx.stream;
    ceg::DevArray<int64_t> d_r, d_c, d_off;
    ceg::DevArray<double> d_v;
    const int64_t *pr = rows, *pc = cols;
    const double* pv = vals;
    if (!on_device && nnz > 0) {
      d_r.alloc(static_cast<size_t>(nnz));
      d_c.alloc(static_cast<size_t>(nnz));
      d_v.alloc(static_cast<size_t>(nnz));
      CE_CUDA(cudaMemcpyAsync(d_r.p, rows, static_cast<size_t>(nnz) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
      CE_CUDA(cudaMemcpyAsync(d_c.p, cols, static_cast<size_t>(nnz) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
      CE_CUDA(cudaMemcpyAsync(d_v.p, vals, static_cast<size_t>(nnz) * sizeof(double), cudaMemcpyHostToDevice, s));
      pr = d_r.p;
      pc = d_c.p;
      pv = d_v.p;
    }
    d_off.upload(offs, s);
    ceg::AssembleResult R = ceg::assemble_from_triplets(n, nnz, pr, pc, pv, m, d_off.p, mirror_lower != 0, s);
    if (!R.error.empty()) throw std::invalid_argument(R.error);
    auto h = std::make_unique<ce_matrix>();
    ceg::Matrix& M = h->m;
    M.ctx = &ctx->ctx;
    M.n = n;
    M.m = m;
    M.offsets = std::move(offs);
    M.row_ptr = std::move(R.row_ptr);
    M.nnzb = M.row_ptr.back();
    M.col_idx = std::move(R.col_idx);
    M.val_ptr = std::move(R.val_ptr);
    M.d_offsets = std::move(d_off);
    M.d_row_ptr.upload(M.row_ptr, s);
    M.d_val_ptr.upload(M.val_ptr, s);
    std::vector<int> col(M.col_idx.begin(), M.col_idx.end()), bsz(static_cast<size_t>(m));
    for (int64_t i = 0; i < m; ++i)
      bsz[static_cast<size_t>(i)] = static_cast<int>(M.offsets[static_cast<size_t>(i + 1)] - M.offsets[static_cast<size_t>(i)]);
    M.d_col_idx.upload(col, s);
    M.d_bsz.upload(bsz, s);
    std::vector<int64_t> row_of(static_cast<size_t>(n));
    for (int64_t i = 0; i < m; ++i)
      for (int64_t p = M.offsets[static_cast<size_t>(i)]; p < M.offsets[static_cast<size_t>(i + 1)]; ++p) row_of[static_cast<size_t>(p)] = i;
    M.d_row_of.upload(row_of, s);
    M.d_values = std::move(R.values);
    CE_CUDA(cudaStreamSynchronize(s));
    *out = h.release();
  });
}

namespace {
int pattern_out(const std::vector<int64_t>& ptr, const std::vector<int>& col, int64_t rows, int64_t* out_ptr,
                int64_t* out_col, int64_t cap, int64_t* nnz) {
  *nnz = ptr[static_cast<size_t>(rows)];
  if (*nnz > cap) throw std::invalid_argument("output capacity too small");
  for (int64_t i = 0; i <= rows; ++i) out_ptr[i] = ptr[static_cast<size_t>(i)];
  for (int64_t k = 0; k < *nnz; ++k) out_col[k] = col[static_cast<size_t>(k)];
  return CE_OK;
}
}  // namespace

int ce_pattern_square(ce_ctx* ctx, int64_t m, const int64_t* row_ptr, const int64_t* cols, int64_t* out_row_ptr,
                      int64_t* out_cols, int64_t cap, int64_t* nnz) {
  return guarded([&] {
    if (!ctx || !row_ptr || !out_row_ptr || !nnz || m < 1) throw std::invalid_argument("null argument");
    CE_CUDA(cudaSetDevice(ctx->ctx.device));
    std::vector<int64_t> ptr(row_ptr, row_ptr + m + 1);
    std::vector<int> col(cols, cols + ptr.back());
    std::vector<int64_t> sp;
    std::vector<int> sc;
    ceg::device_square(m, ptr, col, ctx->ctx.stream, sp, sc);
    pattern_out(sp, sc, m, out_row_ptr, out_cols, cap, nnz);
  });
}

int ce_pattern_coarsen(ce_ctx* ctx, int64_t m, const int64_t* row_ptr, const int64_t* cols, int64_t ng,
                       const int64_t* group_of, int64_t* out_row_ptr, int64_t* out_cols, int64_t cap, int64_t* nnz) {
  return guarded([&] {
    if (!ctx || !row_ptr || !group_of || !out_row_ptr || !nnz || m < 1 || ng < 1) throw std::invalid_argument("null argument");
    CE_CUDA(cudaSetDevice(ctx->ctx.device));
    std::vector<int64_t> ptr(row_ptr, row_ptr + m + 1), gof(group_of, group_of + m);
    std::vector<int> col(cols, cols + ptr.back());
    for (int64_t g : gof)
      if (g < -1 || g >= ng) throw std::invalid_argument("group index out of range");
    std::vector<int64_t> cp;
    std::vector<int> cc;
    ceg::device_coarsen(m, ptr, col, ng, gof, ctx->ctx.stream, cp, cc);
    pattern_out(cp, cc, ng, out_row_ptr, out_cols, cap, nnz);
  });
}

int ce_matrix_csb(const ce_matrix* a, ce_csb_host* view, double* values) {
  return guarded([&] {
    if (!a || !view) throw std::invalid_argument("null argument");
    const ceg::Matrix& M = a->m;
    view->n = M.n;
    view->m = M.m;
    view->offsets = M.offsets.data();
    view->row_ptr = M.row_ptr.data();
    view->col_idx = M.col_idx.data();
    view->val_ptr = M.val_ptr.data();
    view->values = nullptr;
    if (values && M.val_ptr.back() > 0) {
      CE_CUDA(cudaSetDevice(M.ctx->device));
      CE_CUDA(cudaMemcpy(values, M.d_values.p, static_cast<size_t>(M.val_ptr.back()) * sizeof(double),
                         cudaMemcpyDeviceToHost));
    }
  });
}

void ce_matrix_free(ce_matrix* a) { delete a; }
int64_t ce_matrix_dim(const ce_matrix* a) { return a ? a->m.n : 0; }

int ce_matvec(const ce_matrix* a, const double* x, double* y, int64_t n, int on_device, void* stream) {
  return guarded([&] {
    if (!a || n != a->m.n) throw std::invalid_argument("matvec dimension mismatch");
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : a->m.ctx->stream;
    if (on_device) {
      ceg::matvec_device(a->m, x, y, s);
      CE_CUDA(cudaGetLastError());
      return;
    }
    ceg::DevArray<double> dx(static_cast<size_t>(n)), dy(static_cast<size_t>(n));
    CE_CUDA(cudaMemcpyAsync(dx.p, x, static_cast<size_t>(n) * sizeof(double), cudaMemcpyHostToDevice, s));
    ceg::matvec_device(a->m, dx.p, dy.p, s);
    CE_CUDA(cudaMemcpyAsync(y, dy.p, static_cast<size_t>(n) * sizeof(double), cudaMemcpyDeviceToHost, s));
    CE_CUDA(cudaStreamSynchronize(s));
  });
}

namespace {
int factorize_impl(ce_ctx* ctx, const ce_matrix* a, const ce_plan_host* plan, const ce_strategy* s,
                   const ce_factor_opts* opts, const ce_shard* shard, ce_factor** out, ce_status* st) {
  if (st) std::memset(st, 0, sizeof *st);
  return guarded(
      [&] {
        if (!ctx || !a || !out) throw std::invalid_argument("null argument");
        if (s && s->mode == 1 && s->rank < 0) throw std::invalid_argument("fixed rank must be nonnegative");
        CE_CUDA(cudaSetDevice(ctx->ctx.device));
        int64_t shifts = 0;
        auto h = std::make_unique<ce_factor>();
        ceg::ShardSpec spec;
        if (shard) {
          if (!shard->box_of_block || !shard->bcast) throw std::invalid_argument("sharded factorization: null labels / bcast");
          spec.rank = shard->rank;
          spec.n_ranks = shard->n_ranks;
          spec.n_boxes = shard->n_boxes;
          spec.box_l1.assign(shard->box_of_block, shard->box_of_block + a->m.m);
          spec.bcast = shard->bcast;
          spec.user = shard->user;
        }
        h->f.reset(ceg::factorize(&ctx->ctx, &a->m, plan, s, opts, &shifts, shard ? &spec : nullptr));
        h->a_ptr = a->m.row_ptr;
        h->a_col.assign(a->m.col_idx.begin(), a->m.col_idx.end());
        if (plan) {
          h->plan_blocks.assign(plan->level_blocks, plan->level_blocks + plan->n_levels);
          int64_t tot = 0;
          for (int64_t v : h->plan_blocks) tot += v;
          h->plan_assign.assign(plan->assign, plan->assign + tot);
          h->join = plan->join;
        }
        int64_t bmax = 1;
        for (int64_t i = 0; i < a->m.m; ++i) bmax = std::max(bmax, a->m.offsets[static_cast<size_t>(i + 1)] - a->m.offsets[static_cast<size_t>(i)]);
        h->bmax = bmax;
        h->rank_hint = (s && s->mode == 1) ? s->rank : std::max<int64_t>(1, bmax / 2);
        if (st) st->shift_retries = shifts;
        *out = h.release();
      },
      st);
}
}  // namespace

int ce_factorize(ce_ctx* ctx, const ce_matrix* a, const ce_plan_host* plan, const ce_strategy* s,
                 const ce_factor_opts* opts, ce_factor** out, ce_status* st) {
  return factorize_impl(ctx, a, plan, s, opts, nullptr, out, st);
}

int ce_factorize_sharded(ce_ctx* ctx, const ce_matrix* a, const ce_plan_host* plan, const ce_strategy* s,
                         const ce_factor_opts* opts, const ce_shard* shard, ce_factor** out, ce_status* st) {
  if (!shard) {
    g_err = "ce_factorize_sharded: null shard";
    return CE_EUSAGE;
  }
  return factorize_impl(ctx, a, plan, s, opts, shard, out, st);
}

int ce_shard_plan_summary(const ce_problem* p, int n_ranks, int64_t max_levels, int64_t* out, int64_t* n_levels) {
  return guarded([&] {
    if (!p || !out || !n_levels || n_ranks < 1) throw std::invalid_argument("null argument / n_ranks < 1");
    if (p->p.box_of_block.empty()) throw std::invalid_argument("not a CE_PLAN_SHARDED problem");
    ceg::ShardSpec spec;
    spec.n_ranks = n_ranks;
    spec.n_boxes = ceg::kShardBoxes;
    spec.box_l1 = p->p.box_of_block;
    *n_levels = ceg::shard_symbolic_summary(p->p, spec, max_levels, out);
  });
}

void ce_factor_free(ce_factor* f) { delete f; }
int64_t ce_factor_dim(const ce_factor* f) { return f ? f->f->n : 0; }

int ce_apply_precond(const ce_factor* f, const double* b, double* x, int64_t n, int on_device, void* stream) {
  return guarded([&] {
    if (!f || n != f->f->n) throw std::invalid_argument("solve dimension mismatch");
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : f->f->ctx->stream;
    if (on_device) {
      ceg::apply_device(*f->f, b, x, s);
      return;
    }
    std::lock_guard<std::mutex> lk(f->stage_mu);
    if (f->stage_in.n != static_cast<size_t>(n)) {
      f->stage_in.alloc(static_cast<size_t>(n));
      f->stage_out.alloc(static_cast<size_t>(n));
    }
    CE_CUDA(cudaMemcpyAsync(f->stage_in.p, b, static_cast<size_t>(n) * sizeof(double), cudaMemcpyHostToDevice, s));
    ceg::apply_device(*f->f, f->stage_in.p, f->stage_out.p, s);
    CE_CUDA(cudaMemcpyAsync(x, f->stage_out.p, static_cast<size_t>(n) * sizeof(double), cudaMemcpyDeviceToHost, s));
    CE_CUDA(cudaStreamSynchronize(s));
  });
}

int ce_factor_apply_tool(const ce_factor* f, int which, const double* x, double* y, int64_t n) {
  return guarded([&] {
    if (!f || n != f->f->n) throw std::invalid_argument("apply dimension mismatch");
    if (which < 0 || which > 2) throw std::invalid_argument("which must be 0, 1 or 2");
    cudaStream_t s = f->f->ctx->stream;
    ceg::DevArray<double> dx(static_cast<size_t>(n)), dy(static_cast<size_t>(n));
    CE_CUDA(cudaMemcpyAsync(dx.p, x, static_cast<size_t>(n) * sizeof(double), cudaMemcpyHostToDevice, s));
    CE_CUDA(cudaMemsetAsync(dy.p, 0, static_cast<size_t>(n) * sizeof(double), s));
    ceg::apply_tool_device(*f->f, which, dx.p, dy.p, s);
    CE_CUDA(cudaMemcpyAsync(y, dy.p, static_cast<size_t>(n) * sizeof(double), cudaMemcpyDeviceToHost, s));
    CE_CUDA(cudaStreamSynchronize(s));
  });
}

int ce_factor_get_stats(const ce_factor* fh, ce_factor_stats* out) {
  return guarded([&] {
    if (!fh || !out) throw std::invalid_argument("null argument");
    auto* h = const_cast<ce_factor*>(fh);
    const ceg::Factor& f = *h->f;
    if (h->predicted < 0) h->predicted = predicted_nnz(*h, static_cast<int64_t>(f.levels.size()), nullptr);
    std::memset(out, 0, sizeof *out);
    out->n_levels = static_cast<int64_t>(f.levels.size());
    out->tail_dim = f.tail_dim;
    out->factor_blocks = f.factor_blocks;
    out->predicted_factor_blocks = h->predicted;
    out->l_scalar_nnz = f.l_scalar_nnz;
    out->l_payload_bytes = f.l_payload_bytes;
    out->q_payload_bytes = f.q_payload_bytes;
    out->tail_bytes = f.tail_bytes;
    out->shift_retries = f.shift_retries;
    out->total_seconds = f.total_seconds;
    out->device_seconds = f.device_seconds;
    out->sweep_kernel_seconds = f.sweep_seconds;
    double by = 0.0, fl = 0.0;
    for (const auto& L : f.levels) {
      by += L.alg_bytes;
      fl += L.alg_flops;
    }
    const double t = static_cast<double>(f.tail_dim);
    by += 16.0 * t * t;
    fl += t * t * t / 3.0;
    out->algorithmic_bytes = by;
    out->algorithmic_flops = fl;
    out->validate_seconds = f.validate_seconds;
    out->max_orth_error = f.max_orth_error;
    // SURVEY.md §8d apply bytes: nonzero factor payload read by the forward and the backward
    // sweep (t > i neighbours full b_t x w, t < i only their r_t retained rows), the bases,
    // the tail's triangle, plus ~10 n-vector passes
    double pay = 0.0;
    for (const auto& L : f.levels)
      for (int64_t b = 0; b < L.M; ++b) {
        const double w = L.width[static_cast<size_t>(b)], r = L.rank[static_cast<size_t>(b)];
        if (L.has_basis[static_cast<size_t>(b)]) pay += static_cast<double>(L.bsz[static_cast<size_t>(b)]) * L.bsz[static_cast<size_t>(b)];
        if (w == 0) continue;
        pay += w * (w + 1) / 2 + r * w;
        for (int64_t e = L.cptr[static_cast<size_t>(b)]; e < L.cptr[static_cast<size_t>(b + 1)]; ++e) {
          const int t = L.ccol[static_cast<size_t>(e)];
          pay += (t > b ? L.bsz[static_cast<size_t>(t)] : L.rank[static_cast<size_t>(t)]) * w;
        }
      }
    pay += t * (t + 1) / 2;
    out->apply_algorithmic_bytes = 2.0 * 8.0 * pay + 8.0 * static_cast<double>(f.n) * 10.0;
    out->shard_phase1_rows = f.shard.phase1_rows;
    out->shard_own_rows = f.shard.own_rows;
    out->shard_phase3_rows = f.shard.phase3_rows;
    out->shard_exchange_bytes = f.shard.exchange_bytes;
    out->shard_exchange_seconds = f.shard.exchange_seconds;
  });
}

int ce_factor_get_level_stats(const ce_factor* fh, int64_t level, ce_level_stats* out) {
  return guarded([&] {
    if (!fh || !out) throw std::invalid_argument("null argument");
    const ceg::Factor& f = *fh->f;
    if (level < 0 || level >= static_cast<int64_t>(f.levels.size())) throw std::out_of_range("level index");
    const ceg::LevelFactor& L = f.levels[static_cast<size_t>(level)];
    std::memset(out, 0, sizeof *out);
    out->block_count = L.M;
    out->pattern_blocks = L.pattern_blocks;
    out->factor_blocks = 2 * L.pattern_blocks;
    out->eliminated = L.n_elim;
    out->retained = L.n_kept;
    double rs = 0.0;
    for (int64_t b = 0; b < L.M; ++b) {
      out->max_rank = std::max<int64_t>(out->max_rank, L.rank[static_cast<size_t>(b)]);
      rs += L.rank[static_cast<size_t>(b)];
      out->max_block = std::max<int64_t>(out->max_block, L.bsz[static_cast<size_t>(b)]);
      const int64_t w = L.width[static_cast<size_t>(b)], r = L.rank[static_cast<size_t>(b)];
      if (w > 0) {
        int64_t cs = 0;
        for (int64_t e = L.cptr[static_cast<size_t>(b)]; e < L.cptr[static_cast<size_t>(b + 1)]; ++e) cs += L.bsz[static_cast<size_t>(L.ccol[static_cast<size_t>(e)])];
        out->l_bytes += (w * w + r * w + cs * w) * 8;
      }
      if (L.has_basis[static_cast<size_t>(b)]) out->q_bytes += static_cast<int64_t>(L.bsz[static_cast<size_t>(b)]) * L.bsz[static_cast<size_t>(b)] * 8;
    }
    out->mean_rank = L.M ? rs / static_cast<double>(L.M) : 0.0;
    out->seconds = L.seconds;
    out->sweep_seconds = L.sweep_seconds;
    out->shift_retries = L.shift_retries;
    out->max_far_cols = L.max_far;
    out->max_close = L.max_close;
    out->algorithmic_bytes = L.alg_bytes;
    out->algorithmic_flops = L.alg_flops;
    out->n_waves = L.n_waves;
    out->n_items = L.n_items;
  });
}

int ce_factor_level_rows(const ce_factor* fh, int64_t level, int64_t* sizes, int64_t* retained, int64_t* fcols,
                         int64_t* nsigma) {
  return guarded([&] {
    if (!fh) throw std::invalid_argument("null argument");
    const ceg::Factor& f = *fh->f;
    if (level < 0 || level >= static_cast<int64_t>(f.levels.size())) throw std::out_of_range("level index");
    const ceg::LevelFactor& L = f.levels[static_cast<size_t>(level)];
    for (int64_t b = 0; b < L.M; ++b) {
      if (sizes) sizes[b] = L.bsz[static_cast<size_t>(b)];
      if (retained) retained[b] = L.rank[static_cast<size_t>(b)];
      if (fcols) fcols[b] = L.fcols[static_cast<size_t>(b)];
      if (nsigma) nsigma[b] = L.nsig[static_cast<size_t>(b)];
    }
  });
}

int64_t ce_factor_row_sigma(const ce_factor* fh, int64_t level, int64_t row, double* out, int64_t cap) {
  int64_t count = -1;
  const int rc = guarded([&] {
    if (!fh || (!out && cap > 0)) throw std::invalid_argument("null argument");
    const ceg::Factor& f = *fh->f;
    if (level < 0 || level >= static_cast<int64_t>(f.levels.size())) throw std::out_of_range("level index");
    const ceg::LevelFactor& L = f.levels[static_cast<size_t>(level)];
    if (row < 0 || row >= L.M) throw std::out_of_range("row index");
    count = L.nsig[static_cast<size_t>(row)];
    const int64_t k = std::min(count, cap);
    if (k > 0) {
      CE_CUDA(cudaSetDevice(f.ctx->device));
      CE_CUDA(cudaMemcpy(out, L.d_sigma.p + L.sigma_off[static_cast<size_t>(row)], static_cast<size_t>(k) * sizeof(double),
                         cudaMemcpyDeviceToHost));
    }
  });
  return rc == CE_OK ? count : -1;
}

int ce_factor_dump(const ce_factor* f, const char* path) {
  return guarded([&] {
    if (!f || !path) throw std::invalid_argument("null argument");
    ceg::dump_factor(*f->f, path);
  });
}

namespace {
// shared body of the two Krylov entry points (minres.hpp:46-47 contract)
int krylov(bool use_minres, ce_ctx* ctx, const ce_matrix* a, const ce_factor* precond, const double* b, double* x,
           int64_t n, int on_device, const ce_pcg_opts* opts, ce_solve_report* rep, void* stream) {
  if (rep) std::memset(rep, 0, sizeof *rep);
  ceg::SolveOut so;
  const char* what = use_minres ? "minres" : "pcg";
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : (ctx ? ctx->ctx.stream : nullptr);
  auto run = [&](const ce_matrix* am, const ceg::Factor* m, const double* db, double* dx, double tol, int64_t maxit,
                 bool track) {
    return use_minres ? ceg::minres_device(am->m, m, db, dx, tol, maxit, track, s)
                      : ceg::pcg_device(am->m, m, db, dx, tol, maxit, track, s);
  };
  const int rc = guarded([&] {
    if (!ctx || !a || n != a->m.n) throw std::invalid_argument(std::string(what) + " dimension mismatch");
    if (precond && precond->f->n != n) throw std::invalid_argument("preconditioner dimension mismatch");
    const double tol = opts ? opts->tol : 1e-10;
    const int64_t maxit = opts ? opts->maxit : 1000;
    const bool track = opts && opts->track_true_residual;
    CE_CUDA(cudaSetDevice(ctx->ctx.device));
    if (on_device) {
      so = run(a, precond ? precond->f.get() : nullptr, b, x, tol, maxit, track);
    } else {
      ceg::DevArray<double> db(static_cast<size_t>(n)), dx(static_cast<size_t>(n));
      CE_CUDA(cudaMemcpyAsync(db.p, b, static_cast<size_t>(n) * sizeof(double), cudaMemcpyHostToDevice, s));
      so = run(a, precond ? precond->f.get() : nullptr, db.p, dx.p, tol, maxit, track);
      CE_CUDA(cudaMemcpyAsync(x, dx.p, static_cast<size_t>(n) * sizeof(double), cudaMemcpyDeviceToHost, s));
      CE_CUDA(cudaStreamSynchronize(s));
    }
  });
  if (rc != CE_OK) return rc;
  ctx->last_solve = so;
  if (rep) {
    rep->converged = so.converged ? 1 : 0;
    rep->iterations = so.iterations;
    rep->final_recurrence_residual = so.final_rec;
    rep->final_true_residual = so.final_true;
    rep->seconds = so.seconds;
  }
  if (!so.converged) {
    g_err = std::string(what) + " did not converge";
    return CE_ENOCONV;
  }
  return CE_OK;
}
}  // namespace

int ce_pcg(ce_ctx* ctx, const ce_matrix* a, const ce_factor* precond, const double* b, double* x, int64_t n,
           int on_device, const ce_pcg_opts* opts, ce_solve_report* rep, void* stream) {
  return krylov(false, ctx, a, precond, b, x, n, on_device, opts, rep, stream);
}

int ce_minres(ce_ctx* ctx, const ce_matrix* a, const ce_factor* precond, const double* b, double* x, int64_t n,
              int on_device, const ce_pcg_opts* opts, ce_solve_report* rep, void* stream) {
  return krylov(true, ctx, a, precond, b, x, n, on_device, opts, rep, stream);
}

int64_t ce_ctx_last_trace(const ce_ctx* ctx, int64_t* iter, double* recurrence, double* true_resid, double* seconds,
                          int64_t cap) {
  if (!ctx) return -1;
  const ceg::SolveOut& so = ctx->last_solve;
  const int64_t k = static_cast<int64_t>(so.trace_rec.size());
  for (int64_t j = 0; j < k && j < cap; ++j) {
    const size_t u = static_cast<size_t>(j);
    if (iter) iter[j] = so.trace_iter[u];
    if (recurrence) recurrence[j] = so.trace_rec[u];
    if (true_resid) true_resid[j] = so.trace_true[u];
    if (seconds) seconds[j] = so.trace_sec[u];
  }
  return k;
}

// ---- CSV reports (csv.cpp:84-96; cli.cpp:60-80,153-183,233-247) ----
namespace {
std::string fmt_double(double v) {  // shortest text that round-trips (csv.cpp:84-88)
  char buf[64];
  const auto res = std::to_chars(buf, buf + sizeof buf, v);
  return std::string(buf, res.ptr);
}
std::string fmt_index(int64_t v) { return std::to_string(v); }
std::string describe(const ce_strategy* s) {  // CompressionStrategy::describe (compression.cpp:10-18)
  if (!s) return "none";
  std::ostringstream os;
  if (s->mode == 1) os << "rank=" << s->rank;
  else os << (s->absolute ? "abseps=" : "eps=") << s->eps;
  return os.str();
}
std::string csv_row(const std::vector<std::string>& cells) {
  std::string out;
  for (size_t k = 0; k < cells.size(); ++k) {
    if (k) out.push_back(',');
    out += cells[k];
  }
  out.push_back('\n');
  return out;
}
int64_t emit(const std::string& t, char* buf, int64_t cap) {
  if (buf && static_cast<int64_t>(t.size()) < cap) std::memcpy(buf, t.c_str(), t.size() + 1);
  return static_cast<int64_t>(t.size());
}
}  // namespace

int ce_fmt_double(double v, char* buf, int cap) { return static_cast<int>(emit(fmt_double(v), buf, cap)); }

int ce_strategy_describe(const ce_strategy* s, char* buf, int cap) {
  return static_cast<int>(emit(describe(s), buf, cap));
}

int64_t ce_factor_stats_csv(const ce_factor* f, char* buf, int64_t cap) {
  std::string t;
  const int rc = guarded([&] {
    if (!f) throw std::invalid_argument("null argument");
    t = csv_row({"level", "blocks_eliminated", "l_blocks", "max_rank", "mean_rank", "seconds", "bytes"});
    const int64_t nl = static_cast<int64_t>(f->f->levels.size());
    for (int64_t l = 0; l < nl; ++l) {
      ce_level_stats ls;
      if (ce_factor_get_level_stats(f, l, &ls) != CE_OK) throw std::runtime_error(g_err);
      t += csv_row({fmt_index(l + 1), fmt_index(ls.eliminated), fmt_index(ls.factor_blocks), fmt_index(ls.max_rank),
                    fmt_double(ls.mean_rank), fmt_double(ls.seconds), fmt_index(ls.l_bytes + ls.q_bytes)});
    }
  });
  return rc == CE_OK ? emit(t, buf, cap) : -1;
}

int64_t ce_factor_summary_csv(const ce_factor* f, int64_t block, const ce_strategy* s, double seconds,
                              const char* recon_error, char* buf, int64_t cap) {
  std::string t;
  const int rc = guarded([&] {
    if (!f || !s) throw std::invalid_argument("null argument");
    ce_factor_stats st;
    if (ce_factor_get_stats(f, &st) != CE_OK) throw std::runtime_error(g_err);
    t = csv_row({"n", "block", "strategy", "levels", "tail_dim", "l_blocks", "predicted_l_blocks", "block_ratio",
                 "l_scalar_nnz", "l_bytes", "q_bytes", "tail_bytes", "total_bytes", "seconds", "recon_error"});
    const double ratio = st.predicted_factor_blocks > 0 ? st.factor_blocks / st.predicted_factor_blocks : 0.0;
    t += csv_row({fmt_index(f->f->n), fmt_index(block), describe(s), fmt_index(st.n_levels), fmt_index(st.tail_dim),
                  fmt_double(st.factor_blocks), fmt_double(st.predicted_factor_blocks), fmt_double(ratio),
                  fmt_index(st.l_scalar_nnz), fmt_index(st.l_payload_bytes), fmt_index(st.q_payload_bytes),
                  fmt_index(st.tail_bytes), fmt_index(st.l_payload_bytes + st.q_payload_bytes + st.tail_bytes),
                  fmt_double(seconds), recon_error ? recon_error : ""});
  });
  return rc == CE_OK ? emit(t, buf, cap) : -1;
}

int64_t ce_solve_report_csv(int64_t n, const char* mode, const ce_strategy* s, int preconditioned,
                            const ce_solve_report* rep, double factor_seconds, double solve_seconds, char* buf,
                            int64_t cap) {
  if (!rep || !mode) return -1;
  std::string t = csv_row({"n", "mode", "strategy", "preconditioned", "converged", "iterations", "recurrence_resid",
                           "true_resid", "factor_seconds", "solve_seconds"});
  t += csv_row({fmt_index(n), mode, describe(s), preconditioned ? "1" : "0", rep->converged ? "1" : "0",
                fmt_index(rep->iterations), fmt_double(rep->final_recurrence_residual),
                fmt_double(rep->final_true_residual), fmt_double(factor_seconds), fmt_double(solve_seconds)});
  return emit(t, buf, cap);
}

int64_t ce_trace_csv(int64_t count, const int64_t* iter, const double* recurrence, const double* true_resid,
                     const double* seconds, char* buf, int64_t cap) {
  std::string t = csv_row({"iter", "recurrence_resid", "true_resid", "seconds"});
  for (int64_t j = 0; j < count; ++j)
    t += csv_row({fmt_index(iter ? iter[j] : j + 1), fmt_double(recurrence[j]), fmt_double(true_resid[j]),
                  fmt_double(seconds[j])});
  return emit(t, buf, cap);
}

int ce_problem_create(int cfg, int64_t nx, int64_t ny, int64_t nz, ce_problem** out) {
  return ce_problem_create_plan(cfg, nx, ny, nz, CE_PLAN_REFERENCE, out);
}

int ce_problem_create_plan(int cfg, int64_t nx, int64_t ny, int64_t nz, int plan_kind, ce_problem** out) {
  return guarded([&] {
    if (!out) throw std::invalid_argument("null argument");
    if (plan_kind < CE_PLAN_REFERENCE || plan_kind > CE_PLAN_SHARDED)
      throw std::invalid_argument(
          "plan_kind must be one of CE_PLAN_REFERENCE / _MERGE_ALL_AXES / _MERGE_ALL_COLORED / _SHARDED");
    auto p = std::make_unique<ce_problem>();
    p->p.build(cfg, nx, ny, nz, plan_kind);
    *out = p.release();
  });
}

int ce_problem_load(const char* matrix_path, const char* plan_path, const char* rhs_path, int64_t block,
                    ce_problem** out) {
  return guarded([&] {
    if (!out) throw std::invalid_argument("null argument");
    auto p = std::make_unique<ce_problem>();
    p->p.load(matrix_path, plan_path, rhs_path, block);
    *out = p.release();
  });
}

int ce_problem_save(const ce_problem* p, const char* matrix_path, const char* plan_path, const char* rhs_path) {
  return guarded([&] {
    if (!p) throw std::invalid_argument("null argument");
    p->p.save(matrix_path, plan_path, rhs_path);
  });
}

void ce_problem_free(ce_problem* p) { delete p; }

int ce_problem_csb(const ce_problem* p, ce_csb_host* out) {
  if (!p || !out) return CE_EUSAGE;
  out->n = p->p.n;
  out->m = p->p.m;
  out->offsets = p->p.offsets.data();
  out->row_ptr = p->p.row_ptr.data();
  out->col_idx = p->p.col_idx.data();
  out->val_ptr = p->p.val_ptr.data();
  out->values = p->p.values.data();
  return CE_OK;
}

int ce_problem_plan(const ce_problem* p, ce_plan_host* out) {
  if (!p || !out) return CE_EUSAGE;
  out->join = p->p.join;
  out->n_levels = static_cast<int64_t>(p->p.plan_level_blocks.size());
  out->level_blocks = p->p.plan_level_blocks.data();
  out->assign = p->p.plan_assign.data();
  return CE_OK;
}

int ce_problem_boxes(const ce_problem* p, const int64_t** box_of_block, int64_t* n_boxes) {
  if (!p || !box_of_block || !n_boxes) return CE_EUSAGE;
  *box_of_block = p->p.box_of_block.empty() ? nullptr : p->p.box_of_block.data();
  *n_boxes = p->p.box_of_block.empty() ? 0 : ceg::kShardBoxes;
  return CE_OK;
}

const double* ce_problem_rhs(const ce_problem* p) { return p ? p->p.rhs.data() : nullptr; }
const int64_t* ce_problem_perm(const ce_problem* p) { return p ? p->p.perm.data() : nullptr; }

int ce_problem_params(const ce_problem* p, double* eps, double* tol, int64_t* block) {
  if (!p) return CE_EUSAGE;
  if (eps) *eps = p->p.eps;
  if (tol) *tol = p->p.tol;
  if (block) *block = p->p.block;
  return CE_OK;
}

}  // extern "C"
