// ORACLE — TEST INFRASTRUCTURE ONLY (see dense.hpp).
// Restates the CE factorization path of the reference:
//   CompressionStrategy / compress_far_concat  proj/include/ce/compression.hpp:15-50, proj/src/compression.cpp:20-61
//   LevelMatrix (compress_row, eliminate_subrow, extract_remainder)
//                                              proj/include/ce/level_matrix.hpp:24-98, proj/src/level_matrix.cpp:10-248
//   FactorLevel / level_sweep / ce_factorize / solve / apply_q / apply_operator / validate / predicted_nnz
//                                              proj/include/ce/factorization.hpp:19-137, proj/src/factorization.cpp:18-485
// Additions for parity: per-row singular values and far widths
// are recorded, and ranks can be forced per (level, row).
#pragma once

#include <string>
#include <utility>
#include <vector>

#include "csb.hpp"
#include "problems.hpp"

namespace oracle {

struct CompressionStrategy {
  enum class Mode { AdaptiveEps, FixedRank };
  Mode mode = Mode::AdaptiveEps;
  double eps = 1e-6;
  bool absolute = false;
  index_t rank = 0;
  static CompressionStrategy adaptive(double eps, bool absolute = false) {
    CompressionStrategy s;
    s.eps = eps;
    s.absolute = absolute;
    return s;
  }
  static CompressionStrategy fixed_rank(index_t rank) {
    CompressionStrategy s;
    s.mode = Mode::FixedRank;
    s.rank = rank;
    return s;
  }
};

struct RowCompression {
  Mat basis;  // empty = identity
  index_t retained = 0;
  std::vector<double> sigma;  // singular values of F (empty when not computed)
  index_t fcols = 0;
};

// forced_rank >= 0 replaces the eps rule's rank (parity re-synchronisation).
RowCompression compress_far_concat(const Mat& f, index_t block_size, const CompressionStrategy& s,
                                   index_t forced_rank = -1);

struct RowFactor {
  index_t block = -1;
  index_t width = 0;
  Mat chol;      // width x width lower
  Mat coupling;  // retained x width
  std::vector<std::pair<index_t, Mat>> neighbors;  // (t, b_t x width), ascending t
};

class LevelMatrix {
 public:
  LevelMatrix(const BlockSparseMatrix& a, int level_index);
  const BlockPartition& partition() const { return work_.partition(); }
  const BlockSparsityPattern& base_pattern() const { return base_pattern_; }
  BlockSparseMatrix& work() { return work_; }
  const std::vector<index_t>& far_row(index_t i) const { return far_rows_[static_cast<size_t>(i)]; }
  const std::vector<index_t>& close_row(index_t i) const { return close_rows_[static_cast<size_t>(i)]; }
  const RowCompression& compress_row(index_t i, const CompressionStrategy& s, index_t forced_rank = -1);
  void eliminate_subrow(index_t i, index_t retained);
  index_t retained_of(index_t i) const { return retained_[static_cast<size_t>(i)]; }
  index_t shift_retries() const { return shift_retries_; }

  struct Remainder {
    BlockSparseMatrix matrix;
    BlockSparsityPattern full_pattern;
    std::vector<index_t> alive;
  };
  Remainder extract_remainder(const std::vector<std::vector<index_t>>& groups) const;
  std::vector<RowFactor> take_row_factors() { return std::move(factors_); }
  std::vector<RowCompression> take_compressions() { return std::move(compressions_); }

 private:
  int level_index_;
  BlockSparsityPattern base_pattern_;
  BlockSparseMatrix work_;
  std::vector<std::vector<index_t>> far_rows_, close_rows_;
  std::vector<RowCompression> compressions_;
  std::vector<char> compressed_;
  std::vector<index_t> retained_;
  std::vector<RowFactor> factors_;
  std::vector<std::vector<std::pair<index_t, index_t>>> pending_;
  index_t cursor_ = 0;
  index_t shift_retries_ = 0;
};

struct FactorLevel {
  BlockPartition partition;
  std::vector<Mat> basis;
  std::vector<index_t> retained;
  std::vector<RowFactor> rows;
  std::vector<std::vector<index_t>> groups;
  std::vector<index_t> elim_gather, kept_gather, elim_offset;
  // parity extras
  std::vector<std::vector<double>> sigma;
  std::vector<index_t> fcols;
  index_t dim() const { return partition.dim(); }
  index_t eliminated() const { return static_cast<index_t>(elim_gather.size()); }
  index_t kept() const { return static_cast<index_t>(kept_gather.size()); }
  void apply_basis_transpose(std::vector<double>& v) const;
  void apply_basis(std::vector<double>& v) const;
};

struct LevelStats {
  int level = 0;
  index_t block_count = 0, pattern_blocks = 0, factor_blocks = 0;
  index_t eliminated = 0, retained = 0, max_rank = 0;
  double mean_rank = 0.0, seconds = 0.0;
  index_t l_bytes = 0, q_bytes = 0, shift_retries = 0;
  std::vector<index_t> rank_histogram;
};

struct FactorStats {
  std::vector<LevelStats> levels;
  index_t tail_dim = 0;
  double tail_seconds = 0.0;
  index_t tail_bytes = 0;
  double factor_blocks = 0.0, predicted_factor_blocks = 0.0;
  std::vector<index_t> predicted_level_edges;
  index_t l_scalar_nnz = 0, l_payload_bytes = 0, q_payload_bytes = 0;
  double total_seconds = 0.0;
};

struct FactorOptions {
  index_t dense_threshold = 2048;
  index_t max_levels = 64;
  // forced_ranks[level][row] >= 0 overrides the rank decision (empty = none).
  std::vector<std::vector<index_t>> forced_ranks;
};

struct CEFactorization {
  index_t n = 0;
  std::vector<FactorLevel> levels;
  index_t tail_dim = 0;
  Mat tail_chol;
  FactorStats stats;
  std::vector<double> solve(const std::vector<double>& b) const;
  std::vector<double> apply_q(const std::vector<double>& x) const;
  std::vector<double> apply_q_transpose(const std::vector<double>& y) const;
  std::vector<double> apply_operator(const std::vector<double>& x) const;
  std::vector<double> reconstruct_dense() const;
  void validate() const;
};

struct SweepResult {
  FactorLevel level;
  BlockSparseMatrix remainder;
  BlockSparsityPattern full_coarse_pattern;
  std::vector<index_t> alive;
  index_t shift_retries = 0;
};

SweepResult level_sweep(const BlockSparseMatrix& a, const CompressionStrategy& s,
                        const std::vector<std::vector<index_t>>& groups, int level_index,
                        const std::vector<index_t>* forced = nullptr);

CEFactorization ce_factorize(const BlockSparseMatrix& a, const CoarseningPlan& plan,
                             const CompressionStrategy& s, const FactorOptions& opts = {});

struct NnzPrediction {
  std::vector<index_t> level_edges;
  double tail_term = 0.0, total = 0.0;
};
NnzPrediction predicted_nnz(const BlockSparsityPattern& p, const CoarseningPlan& plan, index_t k_levels,
                            index_t rank, index_t block);

// Binary factor dump shared with the GPU library's ce_factor_dump.
void write_factor_dump(const CEFactorization& f, const std::string& path);

}  // namespace oracle
