// ORACLE — TEST INFRASTRUCTURE ONLY (see dense.hpp).
// Problem generators and geometric ordering:
//   assemble_diffusion_3d      proj/src/problems.cpp:18-61
//   assemble_laplace_2d_9pt    proj/src/problems.cpp:63-83
//   CoarseningPlan (+save/load) proj/include/ce/problems.hpp:51-65, problems.cpp:85-179
//   geometric_block_ordering   proj/src/problems.cpp:184-258
//   apply_permutation/permute  proj/src/problems.cpp:260-283
// plus the BASELINE inputs the reference lacks (SURVEY.md §8d conventions):
//   5/7-point finite-volume diffusion with per-cell k and harmonic faces,
//   counter-based splitmix64 + Box-Muller normals, 2-D cell shapes.
#pragma once

#include <array>
#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include "csb.hpp"

namespace oracle {

struct Grid3D {
  index_t nx = 0, ny = 0, nz = 0;
  index_t dim() const { return nx * ny * nz; }
  double hx() const { return 1.0 / static_cast<double>(nx + 1); }
  double hy() const { return 1.0 / static_cast<double>(ny + 1); }
  double hz() const { return 1.0 / static_cast<double>(nz + 1); }
  index_t point(index_t i, index_t j, index_t k) const { return i + nx * (j + ny * k); }
};

using DiffusionCoeff = std::function<std::array<double, 3>(double, double, double)>;
DiffusionCoeff default_diffusion_coefficient();

struct AssembledSystem {
  index_t dim = 0;
  std::vector<Triplet> entries;
  std::vector<double> rhs;
};

AssembledSystem assemble_diffusion_3d(const Grid3D& grid,
                                      const DiffusionCoeff& coeff = default_diffusion_coefficient());
AssembledSystem assemble_laplace_2d_9pt(index_t n);

// Counter-based standard normal z(seed, stream, i) (SURVEY.md §8d RNG).
double normal_sample(std::uint64_t seed, std::uint64_t stream, std::uint64_t i);

// Finite-volume -div(k grad u) on the grid (nz == 1 gives the 5-point 2-D
// stencil), per-cell k, harmonic-mean faces 2 ka kb / (ka + kb), Dirichlet
// boundary faces with k_f = k_cell, rows scaled by hmin^2 (problems.cpp:22-23,44).
// The rhs is left empty (BASELINE rhs comes from normal_sample, stream 1).
AssembledSystem assemble_fv(const Grid3D& grid, const std::vector<double>& kcell);

struct CoarseningPlan {
  std::vector<index_t> initial_permutation;  // perm[new] = old
  BlockPartition partition;
  index_t join = 2;
  std::vector<std::vector<std::vector<index_t>>> levels;
  void validate() const;
  void save(const std::string& path) const;
  static CoarseningPlan load(const std::string& path);
  static CoarseningPlan trivial(index_t n, index_t block);
};

// Reference ordering with its 3-D near-cubic cell shape (problems.cpp:184-191).
CoarseningPlan geometric_block_ordering(const Grid3D& grid, index_t block, index_t join = 2);
// Same ordering with an explicit cell shape (2-D: 2^bx x 2^by x 1, bx >= by).
CoarseningPlan geometric_block_ordering_shape(const Grid3D& grid, std::array<index_t, 3> shape,
                                              index_t join = 2, int plan_kind = 0);
std::array<index_t, 3> cell_shape_3d(index_t block);
std::array<index_t, 3> cell_shape_2d(index_t block);

std::vector<Triplet> apply_permutation(const std::vector<Triplet>& entries,
                                       const std::vector<index_t>& perm);
std::vector<double> permute_vector(const std::vector<double>& v, const std::vector<index_t>& perm);
std::vector<double> unpermute_vector(const std::vector<double>& v, const std::vector<index_t>& perm);

// One BASELINE.json configuration, optionally on a
// smaller grid with the same stencil family / block / eps.
constexpr index_t kShardBoxes = 8;
index_t shard_box(const index_t* g, index_t q, int dims, bool* interior);

struct ProblemConfig {
  int id = 0;
  int dims = 2;
  index_t nx = 0, ny = 0, nz = 1;
  index_t block = 8;
  double eps = 1e-4;
  double tol = 1e-8;
  bool random_k = false;
  double k_sigma = 0.0;
  std::uint64_t seed = 0;
  // Plan family.  false: the reference's geometric_block_ordering (join 2 along one
  // cyclically alternating axis per level).  true: every non-exhausted axis merges by 2
  // at each level (2x2 / 2x2x2 groups, J = 2^d), a plan the reference's ce_factorize
  // accepts through its plan-file interface (problems.cpp:114-171); its pattern reach
  // stays bounded, which is what lets the 3-D configs fit in memory at full size.
  // 2: as true, with every level's cells ordered colour-major (mod-3 colouring; see
  // geometric_block_ordering_shape)
  int plan_kind = 0;
};
ProblemConfig baseline_config(int id);

struct LoadedProblem {
  BlockSparseMatrix matrix;   // permuted into plan order
  std::vector<double> rhs;    // permuted
  CoarseningPlan plan;
  ProblemConfig cfg;
};
LoadedProblem load_config(const ProblemConfig& cfg);

}  // namespace oracle
