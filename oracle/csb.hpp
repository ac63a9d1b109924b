// ORACLE — TEST INFRASTRUCTURE ONLY (see dense.hpp).
// Restates the reference's block layout layer:
//   BlockPartition        proj/include/ce/partition.hpp:11-40, proj/src/partition.cpp:8-47
//   BlockSparsityPattern  proj/include/ce/pattern.hpp:12-61,  proj/src/pattern.cpp:8-126
//   BlockSparseMatrix     proj/include/ce/block_matrix.hpp:23-63, proj/src/block_matrix.cpp:11-146
#pragma once

#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "dense.hpp"

namespace oracle {

struct Triplet {
  index_t row = 0, col = 0;
  double value = 0.0;
};

// Reference BreakdownError (proj/include/ce/types.hpp:26-36).
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

class BlockPartition {
 public:
  BlockPartition() : offsets_{0} {}
  static BlockPartition from_offsets(std::vector<index_t> offsets);
  static BlockPartition uniform(index_t n, index_t block);
  static BlockPartition from_sizes(const std::vector<index_t>& sizes);
  index_t block_count() const { return static_cast<index_t>(offsets_.size()) - 1; }
  index_t dim() const { return offsets_.back(); }
  index_t offset(index_t b) const { return offsets_[static_cast<size_t>(b)]; }
  index_t block_size(index_t b) const {
    return offsets_[static_cast<size_t>(b) + 1] - offsets_[static_cast<size_t>(b)];
  }
  index_t max_block_size() const;
  index_t block_of(index_t i) const;
  const std::vector<index_t>& offsets() const { return offsets_; }
  bool operator==(const BlockPartition& o) const { return offsets_ == o.offsets_; }

 private:
  std::vector<index_t> offsets_;
};

class BlockSparsityPattern {
 public:
  BlockSparsityPattern() = default;
  explicit BlockSparsityPattern(index_t m) : rows_(static_cast<size_t>(m)) {}
  index_t block_rows() const { return static_cast<index_t>(rows_.size()); }
  void insert(index_t i, index_t j);
  void insert_symmetric(index_t i, index_t j);
  void add_full_diagonal();
  bool contains(index_t i, index_t j) const;
  const std::vector<index_t>& row(index_t i) const { return rows_[static_cast<size_t>(i)]; }
  std::vector<index_t>& row_mut(index_t i) { return rows_[static_cast<size_t>(i)]; }
  index_t stored_blocks() const;
  index_t lower_blocks() const;
  index_t max_row_degree() const;
  bool is_structurally_symmetric() const;
  bool has_full_diagonal() const;
  bool operator==(const BlockSparsityPattern& o) const { return rows_ == o.rows_; }

 private:
  std::vector<std::vector<index_t>> rows_;
};

BlockSparsityPattern pattern_square(const BlockSparsityPattern& p);
BlockSparsityPattern far_pattern(const BlockSparsityPattern& p);
BlockSparsityPattern coarsen_pattern(const BlockSparsityPattern& p,
                                     const std::vector<std::vector<index_t>>& groups);
bool pattern_is_subset(const BlockSparsityPattern& sub, const BlockSparsityPattern& sup);

enum class MirrorMode { None, Lower };

// Both triangles stored, one dense block per pattern slot (reference layout).
class BlockSparseMatrix {
 public:
  BlockSparseMatrix() = default;
  BlockSparseMatrix(BlockPartition partition, BlockSparsityPattern pattern);
  static BlockSparseMatrix from_triplets(const std::vector<Triplet>& entries,
                                         BlockPartition partition,
                                         MirrorMode mirror = MirrorMode::None);
  const BlockPartition& partition() const { return partition_; }
  const BlockSparsityPattern& pattern() const { return pattern_; }
  index_t dim() const { return partition_.dim(); }
  bool has_block(index_t i, index_t j) const { return pattern_.contains(i, j); }
  const Mat& block(index_t i, index_t j) const;
  Mat& block(index_t i, index_t j);
  // blocks_[i][k] pairs with pattern().row(i)[k]
  const Mat& slot_block(index_t i, size_t k) const { return blocks_[static_cast<size_t>(i)][k]; }
  std::vector<double> matvec(const std::vector<double>& x) const;
  index_t scalar_nnz() const;
  index_t payload_bytes() const;
  double symmetry_error() const;
  std::vector<double> to_dense() const;  // row-major n x n

 private:
  index_t slot(index_t i, index_t j) const;
  BlockPartition partition_;
  BlockSparsityPattern pattern_;
  std::vector<std::vector<Mat>> blocks_;
};

}  // namespace oracle
