// BASELINE problem generation for the product library (setup, untimed).
//
// Builds the permuted CSB matrix, coarsening plan and right-hand side of the
// five BASELINE.json configurations directly in block form (no COO map):
//   stencil  : finite-volume -div(k grad u), 5-point (2-D) / 7-point (3-D),
//              per-cell k, harmonic faces, Dirichlet ghost k_f = k_cell,
//              rows scaled by hmin^2 (reference scaling, proj/src/problems.cpp:22-23,44)
//   ordering : reference geometric_block_ordering semantics (problems.cpp:195-258),
//              3-D cell_shape (problems.cpp:184-191) or the 2-D analogue
//   RNG      : counter-based splitmix64 + Box-Muller, stream 0 = g, stream 1 = b
// The oracle (oracle/problems.cpp) restates the same conventions independently;
// tests/test_library_cpu.py (test_generator_matches_oracle_bitwise, test_merge_all_axes_plan_matches_oracle) and
// tests/test_shard_cpu.py check the two CSBs and plans agree bit for bit.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "host_api.hpp"

namespace ceg {

namespace {

inline std::uint64_t mix64(std::uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

double normal01(std::uint64_t seed, std::uint64_t stream, std::uint64_t i) {
  const std::uint64_t key = mix64(seed * 0x9E3779B97F4A7C15ULL + 0x632BE59BD9B4E019ULL) ^
                            mix64((stream + 1) * 0xD1B54A32D192ED03ULL);
  const std::uint64_t a = mix64(key + (2 * i + 1) * 0x9E3779B97F4A7C15ULL);
  const std::uint64_t b = mix64(key + (2 * i + 2) * 0x9E3779B97F4A7C15ULL);
  const double u1 = (static_cast<double>(a >> 11) + 0.5) * 0x1.0p-53;
  const double u2 = static_cast<double>(b >> 11) * 0x1.0p-53;
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
}

}  // namespace

// CE_PLAN_SHARDED boxes: 8 spatial subdomains, 4 x 2 (2-D) or 2 x 2 x 2 (3-D), of any level's
// cell grid g; box k along an axis holds the cells x with floor(x * B / g) = k.  A cell is a box
// interior cell when it is >= 2 cells away from every box face shared with another box: with
// all-axis merges a row's squared pattern stays within Chebyshev distance 2 in cells at every
// level, so an interior row's whole squared-pattern row is inside its box.
// Identical in oracle/problems.cpp (shard_box).
int64_t shard_box(const int64_t* g, int64_t q, int dims, bool* interior) {
  const int64_t B[3] = {dims == 2 ? 4 : 2, 2, dims == 2 ? 1 : 2};
  const int64_t x[3] = {q % g[0], (q / g[0]) % g[1], q / (g[0] * g[1])};
  int64_t box = 0, stride = 1;
  bool inner = true;
  for (int a = 0; a < 3; ++a) {
    const int64_t k = x[a] * B[a] / g[a];
    const int64_t lo = (k * g[a] + B[a] - 1) / B[a], hi = ((k + 1) * g[a] + B[a] - 1) / B[a] - 1;
    if (!(lo == 0 || x[a] - lo >= 2) || !(hi == g[a] - 1 || hi - x[a] >= 2)) inner = false;
    box += k * stride;
    stride *= B[a];
  }
  if (interior) *interior = inner;
  return box;
}

namespace {

int ilog2_exact(int64_t block) {
  int b = 0;
  while ((int64_t{1} << (b + 1)) <= block) ++b;
  if ((int64_t{1} << b) != block) throw std::invalid_argument("block size must be a power of two");
  return b;
}

}  // namespace

void Problem::build(int cfg_id, int64_t onx, int64_t ony, int64_t onz, int plan_kind) {
  cfg = cfg_id;
  int dims = 2;
  double ksig = 0.0;
  bool random_k = false;
  std::uint64_t seed = 0;
  switch (cfg_id) {
    case 1: dims = 2; nx = ny = 128; block = 8; eps = 1e-4; tol = 1e-8; seed = 0; break;
    case 2: dims = 2; nx = ny = 1024; block = 16; eps = 1e-6; tol = 1e-10; seed = 1; break;
    case 3: dims = 2; nx = ny = 2048; block = 16; eps = 1e-6; tol = 1e-8; seed = 2; random_k = true; ksig = 1.0; break;
    case 4: dims = 3; nx = ny = nz = 128; block = 32; eps = 1e-5; tol = 1e-8; seed = 3; break;
    case 5: dims = 3; nx = ny = nz = 256; block = 32; eps = 1e-4; tol = 1e-6; seed = 4; random_k = true; ksig = 1.5; break;
    default: throw std::invalid_argument("config id must be 1..5");
  }
  if (onx > 0) nx = onx;
  if (ony > 0) ny = ony;
  if (onz > 0 && dims == 3) nz = onz;
  if (dims == 2) nz = 1;
  const int64_t N = nx * ny * nz;
  n = N;

  // per-cell coefficient and natural-order rhs
  std::vector<double> kcell(static_cast<size_t>(N), 1.0);
  if (random_k)
    for (int64_t i = 0; i < N; ++i) kcell[static_cast<size_t>(i)] = std::exp(ksig * normal01(seed, 0, static_cast<std::uint64_t>(i)));

  // cell shape and ordering (perm[new] = old)
  const int lb = ilog2_exact(block);
  std::array<int64_t, 3> shape;
  if (dims == 2) shape = {int64_t{1} << ((lb + 1) / 2), int64_t{1} << (lb / 2), 1};
  else shape = {int64_t{1} << ((lb + 2) / 3), int64_t{1} << ((lb + 1) / 3), int64_t{1} << (lb / 3)};
  const int64_t nc[3] = {(nx + shape[0] - 1) / shape[0], (ny + shape[1] - 1) / shape[1], (nz + shape[2] - 1) / shape[2]};
  // position -> lexicographic cell id on a cells grid; colour-major (mod-3 colouring) for
  // CE_PLAN_MERGE_ALL_COLORED, so that one colour's rows share no squared-pattern entry;
  // CE_PLAN_SHARDED: box-interior cells first, box by box (each colour-major), then every
  // interface cell (colour-major) -- DESIGN.md §7, shard_box()
  const bool merge_all_axes = plan_kind >= 1, colored = plan_kind >= 2, sharded = plan_kind == 3;
  auto order = [&](const int64_t* g) {
    std::vector<int64_t> ord(static_cast<size_t>(g[0] * g[1] * g[2]));
    for (size_t q = 0; q < ord.size(); ++q) ord[q] = static_cast<int64_t>(q);
    if (colored) {
      auto key = [&](int64_t q) {
        const int64_t x = q % g[0], y = (q / g[0]) % g[1], z = q / (g[0] * g[1]);
        const int64_t color = x % 3 + 3 * (y % 3) + 9 * (z % 3);
        int64_t section = 0;
        if (sharded) {
          bool interior = false;
          const int64_t box = shard_box(g, q, dims, &interior);
          section = interior ? box : kShardBoxes;
        }
        return section * 27 + color;
      };
      std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) { return key(a) < key(b); });
    }
    return ord;
  };
  std::vector<int64_t> ord = order(nc);
  box_of_block.clear();
  if (sharded)
    for (const int64_t q : ord) box_of_block.push_back(shard_box(nc, q, dims, nullptr));
  perm.clear();
  perm.reserve(static_cast<size_t>(N));
  std::vector<int64_t> sizes;
  for (const int64_t q : ord) {
    const int64_t cx = q % nc[0], cy = (q / nc[0]) % nc[1], cz = q / (nc[0] * nc[1]);
    const int64_t x0 = cx * shape[0], y0 = cy * shape[1], z0 = cz * shape[2];
    const int64_t x1 = std::min(x0 + shape[0], nx), y1 = std::min(y0 + shape[1], ny), z1 = std::min(z0 + shape[2], nz);
    for (int64_t k = z0; k < z1; ++k)
      for (int64_t j = y0; j < y1; ++j)
        for (int64_t i = x0; i < x1; ++i) perm.push_back(i + nx * (j + ny * k));
    sizes.push_back((x1 - x0) * (y1 - y0) * (z1 - z0));
  }
  m = static_cast<int64_t>(sizes.size());
  offsets.assign(static_cast<size_t>(m + 1), 0);
  for (int64_t b = 0; b < m; ++b) offsets[static_cast<size_t>(b + 1)] = offsets[static_cast<size_t>(b)] + sizes[static_cast<size_t>(b)];
  std::vector<int64_t> inv(static_cast<size_t>(N)), blk_of(static_cast<size_t>(N));
  for (int64_t p = 0; p < N; ++p) inv[static_cast<size_t>(perm[static_cast<size_t>(p)])] = p;
  for (int64_t b = 0; b < m; ++b)
    for (int64_t p = offsets[static_cast<size_t>(b)]; p < offsets[static_cast<size_t>(b + 1)]; ++p) blk_of[static_cast<size_t>(p)] = b;

  // plan levels: pairwise merges along cyclically alternating non-exhausted axes (the
  // reference's geometric_block_ordering), or along all of them at once (merge_all_axes)
  join = 2;
  plan_level_blocks.clear();
  plan_assign.clear();
  {
    int64_t cur[3] = {nc[0], nc[1], nc[2]};
    int axis = 0;
    while (cur[0] * cur[1] * cur[2] > 1) {
      int tries = 0;
      while (cur[axis] == 1 && tries < 3) {
        axis = (axis + 1) % 3;
        ++tries;
      }
      bool merged[3];
      for (int a = 0; a < 3; ++a) merged[a] = merge_all_axes ? cur[a] > 1 : a == axis;
      int64_t next[3] = {cur[0], cur[1], cur[2]};
      for (int a = 0; a < 3; ++a)
        if (merged[a]) next[a] = (cur[a] + join - 1) / join;
      const std::vector<int64_t> nord = order(next);
      std::vector<int64_t> ninv(nord.size());
      for (size_t p = 0; p < nord.size(); ++p) ninv[static_cast<size_t>(nord[p])] = static_cast<int64_t>(p);
      plan_level_blocks.push_back(cur[0] * cur[1] * cur[2]);
      for (const int64_t q : ord) {
        int64_t gc[3] = {q % cur[0], (q / cur[0]) % cur[1], q / (cur[0] * cur[1])};
        for (int a = 0; a < 3; ++a)
          if (merged[a]) gc[a] /= join;
        plan_assign.push_back(ninv[static_cast<size_t>(gc[0] + next[0] * (gc[1] + next[1] * gc[2]))]);
      }
      ord = nord;
      cur[0] = next[0];
      cur[1] = next[1];
      cur[2] = next[2];
      axis = (axis + 1) % 3;
    }
  }

  // stencil rows in permuted order, straight into block rows
  const double h[3] = {1.0 / static_cast<double>(nx + 1), 1.0 / static_cast<double>(ny + 1), 1.0 / static_cast<double>(nz + 1)};
  double hmin = std::min(h[0], h[1]);
  if (dims == 3) hmin = std::min(hmin, h[2]);
  const double scale = hmin * hmin;
  const int64_t nn[3] = {nx, ny, nz};
  struct Ent { int64_t col; double v; };
  std::vector<std::vector<Ent>> rows(static_cast<size_t>(N));
  for (int64_t kk = 0; kk < nz; ++kk)
    for (int64_t jj = 0; jj < ny; ++jj)
      for (int64_t ii = 0; ii < nx; ++ii) {
        const int64_t q = ii + nx * (jj + ny * kk);
        const double kp = kcell[static_cast<size_t>(q)];
        const int64_t idx[3] = {ii, jj, kk};
        double diag = 0.0;
        auto& row = rows[static_cast<size_t>(inv[static_cast<size_t>(q)])];
        for (int a = 0; a < dims; ++a) {
          const double w = scale / (h[a] * h[a]);
          for (int side = 0; side < 2; ++side) {
            const bool inside = side == 0 ? idx[a] > 0 : idx[a] + 1 < nn[a];
            if (!inside) {
              diag += w * kp;
              continue;
            }
            int64_t nb[3] = {ii, jj, kk};
            nb[a] = side == 0 ? idx[a] - 1 : idx[a] + 1;
            const int64_t qq = nb[0] + nx * (nb[1] + ny * nb[2]);
            const double kq = kcell[static_cast<size_t>(qq)];
            const double kf = 2.0 * (kp * kq) / (kp + kq);
            diag += w * kf;
            row.push_back({inv[static_cast<size_t>(qq)], -w * kf});
          }
        }
        row.push_back({inv[static_cast<size_t>(q)], diag});
      }

  // block pattern per block row (sorted, with diagonal)
  row_ptr.assign(static_cast<size_t>(m + 1), 0);
  col_idx.clear();
  std::vector<int64_t> mark(static_cast<size_t>(m), -1);
  std::vector<std::vector<int64_t>> bcols(static_cast<size_t>(m));
  for (int64_t b = 0; b < m; ++b) {
    auto& cols = bcols[static_cast<size_t>(b)];
    cols.push_back(b);
    mark[static_cast<size_t>(b)] = b;
    for (int64_t p = offsets[static_cast<size_t>(b)]; p < offsets[static_cast<size_t>(b + 1)]; ++p)
      for (const Ent& e : rows[static_cast<size_t>(p)]) {
        const int64_t bj = blk_of[static_cast<size_t>(e.col)];
        if (mark[static_cast<size_t>(bj)] != b) {
          mark[static_cast<size_t>(bj)] = b;
          cols.push_back(bj);
        }
      }
    std::sort(cols.begin(), cols.end());
  }
  for (int64_t b = 0; b < m; ++b) row_ptr[static_cast<size_t>(b + 1)] = row_ptr[static_cast<size_t>(b)] + static_cast<int64_t>(bcols[static_cast<size_t>(b)].size());
  col_idx.resize(static_cast<size_t>(row_ptr.back()));
  val_ptr.assign(static_cast<size_t>(row_ptr.back() + 1), 0);
  for (int64_t b = 0; b < m; ++b) {
    const int64_t bi = sizes[static_cast<size_t>(b)];
    for (size_t k = 0; k < bcols[static_cast<size_t>(b)].size(); ++k) {
      const int64_t s = row_ptr[static_cast<size_t>(b)] + static_cast<int64_t>(k);
      const int64_t j = bcols[static_cast<size_t>(b)][k];
      col_idx[static_cast<size_t>(s)] = j;
      val_ptr[static_cast<size_t>(s + 1)] = val_ptr[static_cast<size_t>(s)] + bi * sizes[static_cast<size_t>(j)];
    }
  }
  values.assign(static_cast<size_t>(val_ptr.back()), 0.0);
  for (int64_t b = 0; b < m; ++b) {
    const auto& cols = bcols[static_cast<size_t>(b)];
    for (int64_t p = offsets[static_cast<size_t>(b)]; p < offsets[static_cast<size_t>(b + 1)]; ++p)
      for (const Ent& e : rows[static_cast<size_t>(p)]) {
        const int64_t bj = blk_of[static_cast<size_t>(e.col)];
        const size_t k = static_cast<size_t>(std::lower_bound(cols.begin(), cols.end(), bj) - cols.begin());
        const int64_t s = row_ptr[static_cast<size_t>(b)] + static_cast<int64_t>(k);
        const int64_t a = p - offsets[static_cast<size_t>(b)];
        const int64_t c = e.col - offsets[static_cast<size_t>(bj)];
        values[static_cast<size_t>(val_ptr[static_cast<size_t>(s)] + a * sizes[static_cast<size_t>(bj)] + c)] = e.v;
      }
  }

  rhs.resize(static_cast<size_t>(N));
  for (int64_t p = 0; p < N; ++p) rhs[static_cast<size_t>(p)] = normal01(seed, 1, static_cast<std::uint64_t>(perm[static_cast<size_t>(p)]));
}

}  // namespace ceg
