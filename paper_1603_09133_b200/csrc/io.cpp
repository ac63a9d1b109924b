// File-based problems for the product library (host setup, untimed): the reference's
// `file` problem flow (proj/src/cli.cpp:114-133 load_problem, :136-150 run_gen) restated
// for the C-ABI, so a user of the reference CLI's matrix.mtx / plan.txt / rhs.txt files
// feeds them to the device factorization unchanged.
//   read_matrix_market  proj/src/matrix_market.cpp:21-59   (coordinate real general|symmetric)
//   write_matrix_market proj/src/matrix_market.cpp:61-93   (lower triangle, (col,row) order, %.17g)
//   read/write_vector   proj/src/matrix_market.cpp:95-115
//   CoarseningPlan::load / save / validate / trivial   proj/src/problems.cpp:84-182
//   apply_permutation / permute_vector / unpermute_vector  proj/src/problems.cpp:260-290
//   BlockSparseMatrix::from_triplets (MirrorMode::None)    proj/src/block_matrix.cpp:48-90
// The block store is built without the reference's std::map: triplets are sorted by
// (row, col), duplicates summed, then scattered into block rows.
#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <numeric>
#include <sstream>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "host_api.hpp"

namespace ceg {

namespace {

struct Trip {
  int64_t row, col;
  double value;
};

std::string lower(std::string s) {
  std::transform(s.begin(), s.end(), s.begin(), [](unsigned char c) { return static_cast<char>(std::tolower(c)); });
  return s;
}

// matrix_market.cpp:21-59
std::vector<Trip> read_matrix_market(const std::string& path, int64_t& rows) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open " + path);
  std::string line;
  if (!std::getline(in, line)) throw std::runtime_error(path + ": empty file");
  std::istringstream banner(line);
  std::string tag, object, format, field, symmetry;
  banner >> tag >> object >> format >> field >> symmetry;
  if (tag != "%%MatrixMarket" || lower(object) != "matrix" || lower(format) != "coordinate" || lower(field) != "real")
    throw std::runtime_error(path + ": expected a coordinate real MatrixMarket banner");
  const std::string sym = lower(symmetry);
  if (sym != "general" && sym != "symmetric") throw std::runtime_error(path + ": unsupported symmetry '" + symmetry + "'");
  while (std::getline(in, line))
    if (!line.empty() && line[0] != '%') break;
  std::istringstream sizes(line);
  int64_t r = 0, c = 0, nnz = 0;
  if (!(sizes >> r >> c >> nnz)) throw std::runtime_error(path + ": bad size line");
  if (r != c) throw std::runtime_error(path + ": matrix must be square");
  std::vector<Trip> out;
  out.reserve(static_cast<size_t>(sym == "symmetric" ? 2 * nnz : nnz));
  for (int64_t k = 0; k < nnz; ++k) {
    int64_t i = 0, j = 0;
    double v = 0.0;
    if (!(in >> i >> j >> v)) throw std::runtime_error(path + ": truncated entry list");
    if (i < 1 || i > r || j < 1 || j > c) throw std::runtime_error(path + ": entry index out of range");
    out.push_back({i - 1, j - 1, v});
    if (sym == "symmetric" && i != j) out.push_back({j - 1, i - 1, v});
  }
  rows = r;
  return out;
}

// matrix_market.cpp:95-102
std::vector<double> read_vector(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open " + path);
  std::vector<double> v;
  double x;
  while (in >> x) v.push_back(x);
  return v;
}

void write_vector(const std::vector<double>& v, const std::string& path) {
  std::FILE* fp = std::fopen(path.c_str(), "w");
  if (!fp) throw std::runtime_error("cannot open " + path + " for writing");
  for (double x : v) std::fprintf(fp, "%.17g\n", x);
  if (std::fclose(fp) != 0) throw std::runtime_error("write failed for " + path);
}

}  // namespace

void Problem::load(const char* matrix_path, const char* plan_path, const char* rhs_path, int64_t blk) {
  if (!matrix_path) throw std::invalid_argument("matrix path is required");
  int64_t rows = 0;
  std::vector<Trip> entries = read_matrix_market(matrix_path, rows);
  // plan: CoarseningPlan::load (problems.cpp:140-174) or ::trivial (:175-182)
  std::vector<int64_t> offs, pm, lv_blocks, assign;
  int64_t jn = 2;
  if (plan_path && plan_path[0]) {
    std::ifstream in(plan_path);
    if (!in) throw std::runtime_error(std::string("cannot open ") + plan_path);
    int64_t pn = 0, pmb = 0, k = 0;
    if (!(in >> pn >> pmb >> k >> jn)) throw std::runtime_error(std::string(plan_path) + ": bad plan header");
    if (pn < 0 || pmb < 0 || k < 0) throw std::runtime_error(std::string(plan_path) + ": bad plan header");
    pm.resize(static_cast<size_t>(pn));
    for (auto& p : pm)
      if (!(in >> p)) throw std::runtime_error(std::string(plan_path) + ": truncated permutation");
    offs.resize(static_cast<size_t>(pmb) + 1);
    for (auto& o : offs)
      if (!(in >> o)) throw std::runtime_error(std::string(plan_path) + ": truncated offsets");
    int64_t blocks = pmb;
    for (int64_t l = 0; l < k; ++l) {
      int64_t groups = 0;
      const size_t a0 = assign.size();
      for (int64_t b = 0; b < blocks; ++b) {
        int64_t a = 0;
        if (!(in >> a)) throw std::runtime_error(std::string(plan_path) + ": truncated level assignments");
        if (a < 0) throw std::runtime_error(std::string(plan_path) + ": negative group id");
        groups = std::max(groups, a + 1);
        assign.push_back(a);
      }
      // validate (problems.cpp:84-112): every group of the level non-empty
      std::vector<char> used(static_cast<size_t>(groups), 0);
      for (size_t q = a0; q < assign.size(); ++q) used[static_cast<size_t>(assign[q])] = 1;
      if (std::find(used.begin(), used.end(), 0) != used.end())
        throw std::invalid_argument("empty group in coarsening level");
      lv_blocks.push_back(blocks);
      blocks = groups;
    }
  } else {
    if (rows <= 0 || blk <= 0) throw std::invalid_argument("uniform partition needs n > 0 and block > 0");
    for (int64_t o = 0; o < rows; o += blk) offs.push_back(o);
    offs.push_back(rows);
    pm.resize(static_cast<size_t>(rows));
    std::iota(pm.begin(), pm.end(), int64_t{0});
  }
  // BlockPartition::from_offsets (partition.cpp:8-17) + validate's permutation check
  if (offs.empty() || offs.front() != 0) throw std::invalid_argument("partition offsets must start at 0");
  for (size_t q = 1; q < offs.size(); ++q)
    if (offs[q] <= offs[q - 1]) throw std::invalid_argument("partition offsets must be strictly increasing");
  const int64_t N = offs.back();
  if (static_cast<int64_t>(pm.size()) != N) throw std::invalid_argument("permutation length does not match partition");
  {
    std::vector<char> seen(static_cast<size_t>(N), 0);
    for (int64_t p : pm) {
      if (p < 0 || p >= N || seen[static_cast<size_t>(p)]) throw std::invalid_argument("initial permutation is not a bijection");
      seen[static_cast<size_t>(p)] = 1;
    }
  }
  if (N != rows) throw std::invalid_argument("plan dimension does not match the matrix");  // cli.cpp:120-121
  std::vector<double> r0;
  if (rhs_path && rhs_path[0]) {
    r0 = read_vector(rhs_path);
    if (static_cast<int64_t>(r0.size()) != rows) throw std::invalid_argument("rhs length does not match the matrix");
  } else {
    r0.assign(static_cast<size_t>(rows), 1.0);
  }
  // finish_load (cli.cpp:49-58): permuted triplets and rhs
  std::vector<int64_t> inv(static_cast<size_t>(N));
  for (int64_t p = 0; p < N; ++p) inv[static_cast<size_t>(pm[static_cast<size_t>(p)])] = p;
  for (Trip& t : entries) {
    if (t.row < 0 || t.row >= N || t.col < 0 || t.col >= N)
      throw std::invalid_argument("triplet index outside matrix dimension");
    t.row = inv[static_cast<size_t>(t.row)];
    t.col = inv[static_cast<size_t>(t.col)];
  }
  // from_triplets: duplicates sum (in input order, as the reference's map accumulates), symmetry to
  // 1e-12 max|a|, pattern = symmetric closure of the touched blocks + full diagonal
  double max_abs = 0.0;
  for (const Trip& t : entries) max_abs = std::max(max_abs, std::fabs(t.value));
  std::stable_sort(entries.begin(), entries.end(),
                   [](const Trip& a, const Trip& b) { return std::tie(a.row, a.col) < std::tie(b.row, b.col); });
  std::vector<Trip> coo;
  coo.reserve(entries.size());
  for (const Trip& t : entries) {
    if (!coo.empty() && coo.back().row == t.row && coo.back().col == t.col) coo.back().value += t.value;
    else coo.push_back(t);
  }
  {
    const double tol = 1e-12 * std::max(max_abs, 1e-300);
    auto find = [&](int64_t r, int64_t c) -> double {
      auto it = std::lower_bound(coo.begin(), coo.end(), Trip{r, c, 0.0},
                                 [](const Trip& a, const Trip& b) { return std::tie(a.row, a.col) < std::tie(b.row, b.col); });
      return (it != coo.end() && it->row == r && it->col == c) ? it->value : 0.0;
    };
    for (const Trip& t : coo) {
      const double vt = find(t.col, t.row);
      if (std::fabs(t.value - vt) > tol) {
        std::ostringstream os;
        os << "asymmetric input: |a(" << t.row << "," << t.col << ") - a(" << t.col << "," << t.row
           << ")| = " << std::fabs(t.value - vt);
        throw std::invalid_argument(os.str());
      }
    }
  }
  const int64_t M = static_cast<int64_t>(offs.size()) - 1;
  std::vector<int64_t> blk_of(static_cast<size_t>(N));
  for (int64_t b = 0; b < M; ++b)
    for (int64_t p = offs[static_cast<size_t>(b)]; p < offs[static_cast<size_t>(b + 1)]; ++p) blk_of[static_cast<size_t>(p)] = b;
  std::vector<std::vector<int64_t>> bcols(static_cast<size_t>(M));
  for (int64_t b = 0; b < M; ++b) bcols[static_cast<size_t>(b)].push_back(b);
  for (const Trip& t : coo) {
    const int64_t bi = blk_of[static_cast<size_t>(t.row)], bj = blk_of[static_cast<size_t>(t.col)];
    bcols[static_cast<size_t>(bi)].push_back(bj);
    bcols[static_cast<size_t>(bj)].push_back(bi);
  }
  for (auto& c : bcols) {
    std::sort(c.begin(), c.end());
    c.erase(std::unique(c.begin(), c.end()), c.end());
  }
  cfg = 0;
  n = N;
  m = M;
  block = blk;
  join = jn;
  offsets = offs;
  perm = pm;
  plan_level_blocks = lv_blocks;
  plan_assign = assign;
  row_ptr.assign(static_cast<size_t>(M + 1), 0);
  for (int64_t b = 0; b < M; ++b) row_ptr[static_cast<size_t>(b + 1)] = row_ptr[static_cast<size_t>(b)] + static_cast<int64_t>(bcols[static_cast<size_t>(b)].size());
  col_idx.resize(static_cast<size_t>(row_ptr.back()));
  val_ptr.assign(static_cast<size_t>(row_ptr.back() + 1), 0);
  for (int64_t b = 0; b < M; ++b) {
    const int64_t bi = offs[static_cast<size_t>(b + 1)] - offs[static_cast<size_t>(b)];
    for (size_t k = 0; k < bcols[static_cast<size_t>(b)].size(); ++k) {
      const int64_t s = row_ptr[static_cast<size_t>(b)] + static_cast<int64_t>(k);
      const int64_t j = bcols[static_cast<size_t>(b)][k];
      col_idx[static_cast<size_t>(s)] = j;
      val_ptr[static_cast<size_t>(s + 1)] = val_ptr[static_cast<size_t>(s)] + bi * (offs[static_cast<size_t>(j + 1)] - offs[static_cast<size_t>(j)]);
    }
  }
  values.assign(static_cast<size_t>(val_ptr.back()), 0.0);
  for (const Trip& t : coo) {
    const int64_t bi = blk_of[static_cast<size_t>(t.row)], bj = blk_of[static_cast<size_t>(t.col)];
    const auto& c = bcols[static_cast<size_t>(bi)];
    const int64_t s = row_ptr[static_cast<size_t>(bi)] + (std::lower_bound(c.begin(), c.end(), bj) - c.begin());
    const int64_t wj = offs[static_cast<size_t>(bj + 1)] - offs[static_cast<size_t>(bj)];
    values[static_cast<size_t>(val_ptr[static_cast<size_t>(s)] + (t.row - offs[static_cast<size_t>(bi)]) * wj +
                               (t.col - offs[static_cast<size_t>(bj)]))] = t.value;
  }
  rhs.resize(static_cast<size_t>(N));
  for (int64_t p = 0; p < N; ++p) rhs[static_cast<size_t>(p)] = r0[static_cast<size_t>(pm[static_cast<size_t>(p)])];
}

// run_gen (cli.cpp:136-150): the matrix and rhs in natural (unpermuted) order, the plan with its
// permutation, so that load() of the three files reproduces this problem.
void Problem::save(const char* matrix_path, const char* plan_path, const char* rhs_path) const {
  if (matrix_path && matrix_path[0]) {
    std::vector<Trip> low;
    for (int64_t b = 0; b < m; ++b) {
      const int64_t bi = offsets[static_cast<size_t>(b + 1)] - offsets[static_cast<size_t>(b)];
      for (int64_t s = row_ptr[static_cast<size_t>(b)]; s < row_ptr[static_cast<size_t>(b + 1)]; ++s) {
        const int64_t j = col_idx[static_cast<size_t>(s)];
        const int64_t wj = offsets[static_cast<size_t>(j + 1)] - offsets[static_cast<size_t>(j)];
        for (int64_t a = 0; a < bi; ++a)
          for (int64_t c = 0; c < wj; ++c) {
            const double v = values[static_cast<size_t>(val_ptr[static_cast<size_t>(s)] + a * wj + c)];
            const int64_t gi = perm[static_cast<size_t>(offsets[static_cast<size_t>(b)] + a)];
            const int64_t gj = perm[static_cast<size_t>(offsets[static_cast<size_t>(j)] + c)];
            if (gj > gi || v == 0.0) continue;
            low.push_back({gi, gj, v});
          }
      }
    }
    std::sort(low.begin(), low.end(),
              [](const Trip& x, const Trip& y) { return std::tie(x.col, x.row) < std::tie(y.col, y.row); });
    std::FILE* fp = std::fopen(matrix_path, "w");
    if (!fp) throw std::runtime_error(std::string("cannot open ") + matrix_path + " for writing");
    std::fprintf(fp, "%%%%MatrixMarket matrix coordinate real symmetric\n%lld %lld %lld\n", static_cast<long long>(n),
                 static_cast<long long>(n), static_cast<long long>(low.size()));
    for (const Trip& t : low)
      std::fprintf(fp, "%lld %lld %.17g\n", static_cast<long long>(t.row + 1), static_cast<long long>(t.col + 1), t.value);
    if (std::fclose(fp) != 0) throw std::runtime_error(std::string("write failed for ") + matrix_path);
  }
  if (rhs_path && rhs_path[0]) {
    std::vector<double> nat(static_cast<size_t>(n));
    for (int64_t p = 0; p < n; ++p) nat[static_cast<size_t>(perm[static_cast<size_t>(p)])] = rhs[static_cast<size_t>(p)];
    write_vector(nat, rhs_path);
  }
  if (plan_path && plan_path[0]) {  // CoarseningPlan::save (problems.cpp:114-138)
    std::FILE* fp = std::fopen(plan_path, "w");
    if (!fp) throw std::runtime_error(std::string("cannot open ") + plan_path + " for writing");
    std::fprintf(fp, "%lld %lld %lld %lld\n", static_cast<long long>(n), static_cast<long long>(m),
                 static_cast<long long>(plan_level_blocks.size()), static_cast<long long>(join));
    for (int64_t i = 0; i < n; ++i)
      std::fprintf(fp, "%lld%c", static_cast<long long>(perm[static_cast<size_t>(i)]), i + 1 == n ? '\n' : ' ');
    for (int64_t i = 0; i <= m; ++i)
      std::fprintf(fp, "%lld%c", static_cast<long long>(offsets[static_cast<size_t>(i)]), i == m ? '\n' : ' ');
    size_t at = 0;
    for (int64_t blocks : plan_level_blocks) {
      for (int64_t b = 0; b < blocks; ++b)
        std::fprintf(fp, "%lld%c", static_cast<long long>(plan_assign[at++]), b + 1 == blocks ? '\n' : ' ');
    }
    if (std::fclose(fp) != 0) throw std::runtime_error(std::string("write failed for ") + plan_path);
  }
}

}  // namespace ceg
