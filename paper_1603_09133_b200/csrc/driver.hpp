// Host driver entry points (internal).
#pragma once

#include <string>
#include <vector>

#include "../../include/ce_gpu.h"
#include "host_api.hpp"

namespace ceg {

LevelPlan plan_level(std::vector<int> bsz, std::vector<int64_t> bptr, std::vector<int> bcol, cudaStream_t dev = nullptr);

// shard != nullptr: this rank's part of a subdomain-sharded factorization; the
// returned factor is complete and identical on every rank.
Factor* factorize(Context* ctx, const Matrix* A, const ce_plan_host* plan, const ce_strategy* st,
                  const ce_factor_opts* opts, int64_t* shift_total, const ShardSpec* shard = nullptr);

// Symbolic phase split of a sharded plan (every group alive), for ce_shard_plan_summary.
int64_t shard_symbolic_summary(const Problem& p, const ShardSpec& spec, int64_t max_levels, int64_t* out);

void apply_device(const Factor& f, const double* d_b, double* d_x, cudaStream_t s);
void apply_tool_device(const Factor& f, int which, const double* d_x, double* d_y, cudaStream_t s);
void matvec_device(const Matrix& A, const double* d_x, double* d_y, cudaStream_t s);

struct SolveOut {
  bool converged = false;
  int64_t iterations = 0;
  double final_rec = 0.0, final_true = 0.0, seconds = 0.0;
  // IterationTrace (minres.hpp:12-23): sample 0 before the loop, then one per iteration; true = -1 untracked
  std::vector<int64_t> trace_iter;
  std::vector<double> trace_rec, trace_true, trace_sec;
};
// Both Krylov loops run on stream `s` (the caller's, so its producers of b / consumers of x
// are ordered against the solve).
SolveOut pcg_device(const Matrix& A, const Factor* M, const double* d_b, double* d_x, double tol, int64_t maxit,
                    bool track_true, cudaStream_t s);

// MINRES with an SPD preconditioner (minres.cpp:22-115, the paper's solver) on the device.
SolveOut minres_device(const Matrix& A, const Factor* M, const double* d_b, double* d_x, double tol, int64_t maxit,
                       bool track_true, cudaStream_t s);

void dump_factor(const Factor& f, const std::string& path);

}  // namespace ceg
