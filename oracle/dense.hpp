// ORACLE — TEST INFRASTRUCTURE ONLY.
// CPU restatement of the reference's dense arithmetic (the reference calls
// Eigen3, which is absent from /root/reference and from this image; Eigen
// >= 3.3 unpinned, proj/CMakeLists.txt:12).  Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference legs may link or run this.
//
// Eigen call sites restated here:
//   JacobiSVD(f, ComputeFullU)        proj/src/compression.cpp:38,48
//   LLT                               proj/src/level_matrix.cpp:110-115, factorization.cpp:423-427
//   triangularView<Lower>::solveInPlace  level_matrix.cpp:128,135, factorization.cpp:105,127,153
//   dense operator* / noalias         level_matrix.cpp:53-68,141-158
//
// Parity note: Eigen's JacobiSVD returns U in an arbitrary gauge (column signs,
// rotations in degenerate clusters, any basis of the discarded complement).
// The oracle and the GPU both emit the CANONICAL GAUGE defined in svd_left()
// below, so factor blocks are comparable entrywise.
#pragma once

#include <cstdint>
#include <vector>

namespace oracle {

using index_t = std::int64_t;

// Row-major dense matrix (reference DenseBlock, proj/include/ce/types.hpp:12-13).
struct Mat {
  index_t r = 0, c = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(index_t rows, index_t cols) : r(rows), c(cols), a(static_cast<size_t>(rows * cols), 0.0) {}
  double& operator()(index_t i, index_t j) { return a[static_cast<size_t>(i * c + j)]; }
  double operator()(index_t i, index_t j) const { return a[static_cast<size_t>(i * c + j)]; }
  index_t size() const { return r * c; }
  bool empty() const { return r * c == 0; }
  static Mat identity(index_t n) {
    Mat m(n, n);
    for (index_t i = 0; i < n; ++i) m(i, i) = 1.0;
    return m;
  }
  Mat transpose() const;
  double max_abs() const;
};

// C = A * B
Mat matmul(const Mat& A, const Mat& B);
// C = A^T * B
Mat matmul_tn(const Mat& A, const Mat& B);
// C = A * B^T
Mat matmul_nt(const Mat& A, const Mat& B);

// In-place lower Cholesky of the lower triangle of P (upper triangle ignored,
// zeroed on return).  Returns false on a non-positive pivot like Eigen's
// LLT::info() != Success.
bool llt_lower(Mat& P);

// Y <- L^{-1} Y  (L lower triangular, forward substitution).
void trsm_lower_left(const Mat& L, Mat& Y);
// y <- L^{-1} y
void trsv_lower(const Mat& L, double* y);
// y <- L^{-T} y
void trsv_lower_t(const Mat& L, double* y);

// Generic weights c_k used by the canonical gauge's sign rules (singletons, complement QR).
double gauge_weight(index_t k);
// Cluster gauge weights G_c(k, j): zero-mean hash values in [-1, 1), independent across j, so
// U_c^T G_c stays well conditioned for clusters of any size (the earlier 1 + frac((k+1) c_j)
// columns were nearly affine in j and lost orthogonality at cluster sizes >= ~4).
double gauge_weight2(index_t k, index_t j);
// Singular values closer than kClusterTol * sigma_1 share one canonical basis.
constexpr double kClusterTol = 1e-9;
// Jacobi skips pairs of columns whose squared norms are both <= kNoise2 * ||R||_F^2.
constexpr double kNoise2 = 1e-28;

struct SvdLeft {
  std::vector<double> sigma;  // min(rows, cols) singular values, descending
  Mat V;                      // rows x rows left singular vectors (column k <-> sigma_k)
  int sweeps = 0;
};

// Left singular vectors and singular values of F (b x f): Householder QR of
// F^T, then one-sided (Hestenes) Jacobi on the b-column R, V accumulated.
SvdLeft svd_left(const Mat& F);

// Canonical gauge: U = [U1 | U2] with U1 = first r columns of V, each sign-fixed
// so sum_k c_k u_k >= 0 -- or, for a cluster of singular values within
// kClusterTol * sigma_1 of each other, the orthonormalised projection
// orth(U_c U_c^T G_c) of fixed generic vectors -- and U2 = trailing columns of the Householder QR Q of U1
// (reflector signs chosen by the same generic functional, Parlett's formula
// when that choice cancels).
Mat canonical_basis(const Mat& V, const std::vector<double>& sigma, index_t r);

}  // namespace oracle
