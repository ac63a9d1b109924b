// ORACLE — TEST INFRASTRUCTURE ONLY (see dense.hpp).
#include "csb.hpp"

#include <algorithm>
#include <cmath>
#include <sstream>

namespace oracle {

// partition.cpp:8-18
BlockPartition BlockPartition::from_offsets(std::vector<index_t> offsets) {
  if (offsets.empty() || offsets.front() != 0)
    throw std::invalid_argument("partition offsets must start at 0");
  for (size_t k = 1; k < offsets.size(); ++k)
    if (offsets[k] <= offsets[k - 1])
      throw std::invalid_argument("partition offsets must be strictly increasing");
  BlockPartition p;
  p.offsets_ = std::move(offsets);
  return p;
}

// partition.cpp:20-28
BlockPartition BlockPartition::uniform(index_t n, index_t block) {
  if (n <= 0 || block <= 0) throw std::invalid_argument("uniform partition needs n > 0 and block > 0");
  std::vector<index_t> offs;
  for (index_t o = 0; o < n; o += block) offs.push_back(o);
  offs.push_back(n);
  return from_offsets(std::move(offs));
}

// partition.cpp:30-36
BlockPartition BlockPartition::from_sizes(const std::vector<index_t>& sizes) {
  std::vector<index_t> offs{0};
  for (index_t s : sizes) offs.push_back(offs.back() + s);
  return from_offsets(std::move(offs));
}

index_t BlockPartition::max_block_size() const {
  index_t m = 0;
  for (index_t b = 0; b < block_count(); ++b) m = std::max(m, block_size(b));
  return m;
}

// partition.cpp:42-46
index_t BlockPartition::block_of(index_t i) const {
  if (i < 0 || i >= dim()) throw std::out_of_range("scalar index outside partition");
  auto it = std::upper_bound(offsets_.begin(), offsets_.end(), i);
  return static_cast<index_t>(it - offsets_.begin()) - 1;
}

// pattern.cpp:8-14
void BlockSparsityPattern::insert(index_t i, index_t j) {
  if (i < 0 || i >= block_rows() || j < 0 || j >= block_rows())
    throw std::out_of_range("pattern position outside block grid");
  auto& r = rows_[static_cast<size_t>(i)];
  auto it = std::lower_bound(r.begin(), r.end(), j);
  if (it == r.end() || *it != j) r.insert(it, j);
}

void BlockSparsityPattern::insert_symmetric(index_t i, index_t j) {
  insert(i, j);
  if (i != j) insert(j, i);
}

void BlockSparsityPattern::add_full_diagonal() {
  for (index_t i = 0; i < block_rows(); ++i) insert(i, i);
}

bool BlockSparsityPattern::contains(index_t i, index_t j) const {
  if (i < 0 || i >= block_rows() || j < 0 || j >= block_rows()) return false;
  const auto& r = rows_[static_cast<size_t>(i)];
  return std::binary_search(r.begin(), r.end(), j);
}

index_t BlockSparsityPattern::stored_blocks() const {
  index_t n = 0;
  for (const auto& r : rows_) n += static_cast<index_t>(r.size());
  return n;
}

// pattern.cpp:37-43 (diagonal included)
index_t BlockSparsityPattern::lower_blocks() const {
  index_t n = 0;
  for (index_t i = 0; i < block_rows(); ++i)
    for (index_t j : rows_[static_cast<size_t>(i)])
      if (j <= i) ++n;
  return n;
}

index_t BlockSparsityPattern::max_row_degree() const {
  index_t d = 0;
  for (const auto& r : rows_) d = std::max(d, static_cast<index_t>(r.size()));
  return d;
}

bool BlockSparsityPattern::is_structurally_symmetric() const {
  for (index_t i = 0; i < block_rows(); ++i)
    for (index_t j : rows_[static_cast<size_t>(i)])
      if (!contains(j, i)) return false;
  return true;
}

bool BlockSparsityPattern::has_full_diagonal() const {
  for (index_t i = 0; i < block_rows(); ++i)
    if (!contains(i, i)) return false;
  return true;
}

// pattern.cpp:64-86 (mark-array boolean product)
BlockSparsityPattern pattern_square(const BlockSparsityPattern& p) {
  const index_t m = p.block_rows();
  BlockSparsityPattern sq(m);
  std::vector<char> mark(static_cast<size_t>(m), 0);
  std::vector<index_t> touched;
  for (index_t i = 0; i < m; ++i) {
    touched.clear();
    for (index_t k : p.row(i))
      for (index_t j : p.row(k))
        if (!mark[static_cast<size_t>(j)]) {
          mark[static_cast<size_t>(j)] = 1;
          touched.push_back(j);
        }
    std::sort(touched.begin(), touched.end());
    sq.row_mut(i) = touched;
    for (index_t j : touched) mark[static_cast<size_t>(j)] = 0;
  }
  return sq;
}

// pattern.cpp:88-95
BlockSparsityPattern far_pattern(const BlockSparsityPattern& p) {
  BlockSparsityPattern sq = pattern_square(p);
  BlockSparsityPattern far(p.block_rows());
  for (index_t i = 0; i < p.block_rows(); ++i)
    for (index_t j : sq.row(i))
      if (j != i && !p.contains(i, j)) far.row_mut(i).push_back(j);
  return far;
}

// pattern.cpp:97-118
BlockSparsityPattern coarsen_pattern(const BlockSparsityPattern& p,
                                     const std::vector<std::vector<index_t>>& groups) {
  const index_t m = p.block_rows();
  std::vector<index_t> group_of(static_cast<size_t>(m), -1);
  for (size_t g = 0; g < groups.size(); ++g)
    for (index_t b : groups[g]) {
      if (b < 0 || b >= m || group_of[static_cast<size_t>(b)] != -1)
        throw std::invalid_argument("groups must partition the block index range");
      group_of[static_cast<size_t>(b)] = static_cast<index_t>(g);
    }
  for (index_t b = 0; b < m; ++b)
    if (group_of[static_cast<size_t>(b)] == -1) throw std::invalid_argument("groups must cover every block");
  const index_t ng = static_cast<index_t>(groups.size());
  BlockSparsityPattern c(ng);
  std::vector<char> mark(static_cast<size_t>(ng), 0);
  for (size_t g = 0; g < groups.size(); ++g) {
    std::vector<index_t>& row = c.row_mut(static_cast<index_t>(g));
    for (index_t i : groups[g])
      for (index_t j : p.row(i)) {
        const index_t gj = group_of[static_cast<size_t>(j)];
        if (!mark[static_cast<size_t>(gj)]) {
          mark[static_cast<size_t>(gj)] = 1;
          row.push_back(gj);
        }
      }
    std::sort(row.begin(), row.end());
    for (index_t gj : row) mark[static_cast<size_t>(gj)] = 0;
  }
  return c;
}

bool pattern_is_subset(const BlockSparsityPattern& sub, const BlockSparsityPattern& sup) {
  if (sub.block_rows() != sup.block_rows()) return false;
  for (index_t i = 0; i < sub.block_rows(); ++i)
    for (index_t j : sub.row(i))
      if (!sup.contains(i, j)) return false;
  return true;
}

// block_matrix.cpp:11-27
BlockSparseMatrix::BlockSparseMatrix(BlockPartition partition, BlockSparsityPattern pattern)
    : partition_(std::move(partition)), pattern_(std::move(pattern)) {
  if (pattern_.block_rows() != partition_.block_count())
    throw std::invalid_argument("pattern size does not match partition");
  if (!pattern_.is_structurally_symmetric())
    throw std::invalid_argument("pattern must be structurally symmetric");
  if (!pattern_.has_full_diagonal())
    throw std::invalid_argument("pattern must contain all diagonal positions");
  blocks_.resize(static_cast<size_t>(pattern_.block_rows()));
  for (index_t i = 0; i < pattern_.block_rows(); ++i) {
    auto& row = blocks_[static_cast<size_t>(i)];
    row.reserve(pattern_.row(i).size());
    for (index_t j : pattern_.row(i)) row.emplace_back(partition_.block_size(i), partition_.block_size(j));
  }
}

index_t BlockSparseMatrix::slot(index_t i, index_t j) const {
  const auto& r = pattern_.row(i);
  auto it = std::lower_bound(r.begin(), r.end(), j);
  if (it == r.end() || *it != j) return -1;
  return static_cast<index_t>(it - r.begin());
}

const Mat& BlockSparseMatrix::block(index_t i, index_t j) const {
  const index_t s = slot(i, j);
  if (s < 0) throw std::out_of_range("block position not in pattern");
  return blocks_[static_cast<size_t>(i)][static_cast<size_t>(s)];
}

Mat& BlockSparseMatrix::block(index_t i, index_t j) {
  const index_t s = slot(i, j);
  if (s < 0) throw std::out_of_range("block position not in pattern");
  return blocks_[static_cast<size_t>(i)][static_cast<size_t>(s)];
}

// block_matrix.cpp:48-90
BlockSparseMatrix BlockSparseMatrix::from_triplets(const std::vector<Triplet>& entries,
                                                   BlockPartition partition, MirrorMode mirror) {
  const index_t n = partition.dim();
  std::map<std::pair<index_t, index_t>, double> coo;
  double max_abs = 0.0;
  for (const Triplet& t : entries) {
    if (t.row < 0 || t.row >= n || t.col < 0 || t.col >= n)
      throw std::invalid_argument("triplet index outside matrix dimension");
    coo[{t.row, t.col}] += t.value;
    if (mirror == MirrorMode::Lower && t.row != t.col) coo[{t.col, t.row}] += t.value;
    max_abs = std::max(max_abs, std::abs(t.value));
  }
  if (mirror == MirrorMode::None) {
    const double tol = 1e-12 * std::max(max_abs, 1e-300);
    for (const auto& [pos, v] : coo) {
      auto it = coo.find({pos.second, pos.first});
      const double vt = it == coo.end() ? 0.0 : it->second;
      if (std::abs(v - vt) > tol) {
        std::ostringstream os;
        os << "asymmetric input: |a(" << pos.first << "," << pos.second << ") - a(" << pos.second
           << "," << pos.first << ")| = " << std::abs(v - vt);
        throw std::invalid_argument(os.str());
      }
    }
  }
  BlockSparsityPattern pat(partition.block_count());
  for (const auto& kv : coo)
    pat.insert_symmetric(partition.block_of(kv.first.first), partition.block_of(kv.first.second));
  pat.add_full_diagonal();
  BlockSparseMatrix a(std::move(partition), std::move(pat));
  for (const auto& [pos, v] : coo) {
    const index_t bi = a.partition_.block_of(pos.first);
    const index_t bj = a.partition_.block_of(pos.second);
    a.block(bi, bj)(pos.first - a.partition_.offset(bi), pos.second - a.partition_.offset(bj)) = v;
  }
  return a;
}

// block_matrix.cpp:92-105
std::vector<double> BlockSparseMatrix::matvec(const std::vector<double>& x) const {
  if (static_cast<index_t>(x.size()) != dim()) throw std::invalid_argument("matvec dimension mismatch");
  std::vector<double> y(static_cast<size_t>(dim()), 0.0);
  for (index_t i = 0; i < partition_.block_count(); ++i) {
    const index_t oi = partition_.offset(i), bi = partition_.block_size(i);
    const auto& cols = pattern_.row(i);
    for (size_t k = 0; k < cols.size(); ++k) {
      const index_t j = cols[k];
      const index_t oj = partition_.offset(j), bj = partition_.block_size(j);
      const Mat& blk = blocks_[static_cast<size_t>(i)][k];
      for (index_t a = 0; a < bi; ++a) {
        double s = 0.0;
        for (index_t c = 0; c < bj; ++c) s += blk(a, c) * x[static_cast<size_t>(oj + c)];
        y[static_cast<size_t>(oi + a)] += s;
      }
    }
  }
  return y;
}

index_t BlockSparseMatrix::scalar_nnz() const {
  index_t n = 0;
  for (const auto& row : blocks_)
    for (const auto& b : row)
      for (double v : b.a) n += v != 0.0;
  return n;
}

index_t BlockSparseMatrix::payload_bytes() const {
  index_t n = 0;
  for (const auto& row : blocks_)
    for (const auto& b : row) n += b.size() * static_cast<index_t>(sizeof(double));
  return n;
}

double BlockSparseMatrix::symmetry_error() const {
  double e = 0.0;
  for (index_t i = 0; i < partition_.block_count(); ++i) {
    const auto& cols = pattern_.row(i);
    for (size_t k = 0; k < cols.size(); ++k) {
      const index_t j = cols[k];
      if (j < i) continue;
      const Mat& aij = blocks_[static_cast<size_t>(i)][k];
      const Mat& aji = block(j, i);
      for (index_t a = 0; a < aij.r; ++a)
        for (index_t c = 0; c < aij.c; ++c) e = std::max(e, std::abs(aij(a, c) - aji(c, a)));
    }
  }
  return e;
}

std::vector<double> BlockSparseMatrix::to_dense() const {
  const index_t n = dim();
  std::vector<double> d(static_cast<size_t>(n * n), 0.0);
  for (index_t i = 0; i < partition_.block_count(); ++i) {
    const auto& cols = pattern_.row(i);
    for (size_t k = 0; k < cols.size(); ++k) {
      const index_t j = cols[k];
      const Mat& blk = blocks_[static_cast<size_t>(i)][k];
      for (index_t a = 0; a < blk.r; ++a)
        for (index_t c = 0; c < blk.c; ++c)
          d[static_cast<size_t>((partition_.offset(i) + a) * n + partition_.offset(j) + c)] = blk(a, c);
    }
  }
  return d;
}

}  // namespace oracle
