// ORACLE — TEST INFRASTRUCTURE ONLY (see dense.hpp).
#include "dense.hpp"

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <numeric>
#include <stdexcept>

namespace oracle {

Mat Mat::transpose() const {
  Mat t(c, r);
  for (index_t i = 0; i < r; ++i)
    for (index_t j = 0; j < c; ++j) t(j, i) = (*this)(i, j);
  return t;
}

double Mat::max_abs() const {
  double m = 0.0;
  for (double v : a) m = std::max(m, std::abs(v));
  return m;
}

Mat matmul(const Mat& A, const Mat& B) {
  if (A.c != B.r) throw std::invalid_argument("matmul shape");
  Mat C(A.r, B.c);
  for (index_t i = 0; i < A.r; ++i)
    for (index_t k = 0; k < A.c; ++k) {
      const double aik = A(i, k);
      if (aik == 0.0) continue;
      for (index_t j = 0; j < B.c; ++j) C(i, j) += aik * B(k, j);
    }
  return C;
}

Mat matmul_tn(const Mat& A, const Mat& B) {
  if (A.r != B.r) throw std::invalid_argument("matmul_tn shape");
  Mat C(A.c, B.c);
  for (index_t k = 0; k < A.r; ++k)
    for (index_t i = 0; i < A.c; ++i) {
      const double aki = A(k, i);
      if (aki == 0.0) continue;
      for (index_t j = 0; j < B.c; ++j) C(i, j) += aki * B(k, j);
    }
  return C;
}

Mat matmul_nt(const Mat& A, const Mat& B) {
  if (A.c != B.c) throw std::invalid_argument("matmul_nt shape");
  Mat C(A.r, B.r);
  for (index_t i = 0; i < A.r; ++i)
    for (index_t j = 0; j < B.r; ++j) {
      double s = 0.0;
      for (index_t k = 0; k < A.c; ++k) s += A(i, k) * B(j, k);
      C(i, j) = s;
    }
  return C;
}

// Unblocked left-looking Cholesky over the lower triangle, failing on a
// non-positive pivot (Eigen llt_inplace::unblocked semantics).
bool llt_lower(Mat& P) {
  const index_t n = P.r;
  for (index_t j = 0; j < n; ++j) {
    double d = P(j, j);
    for (index_t k = 0; k < j; ++k) d -= P(j, k) * P(j, k);
    if (!(d > 0.0)) return false;
    d = std::sqrt(d);
    P(j, j) = d;
    for (index_t i = j + 1; i < n; ++i) {
      double s = P(i, j);
      for (index_t k = 0; k < j; ++k) s -= P(i, k) * P(j, k);
      P(i, j) = s / d;
    }
  }
  for (index_t i = 0; i < n; ++i)
    for (index_t j = i + 1; j < n; ++j) P(i, j) = 0.0;
  return true;
}

void trsm_lower_left(const Mat& L, Mat& Y) {
  const index_t n = L.r;
  for (index_t i = 0; i < n; ++i) {
    for (index_t k = 0; k < i; ++k) {
      const double lik = L(i, k);
      if (lik == 0.0) continue;
      for (index_t j = 0; j < Y.c; ++j) Y(i, j) -= lik * Y(k, j);
    }
    const double d = L(i, i);
    for (index_t j = 0; j < Y.c; ++j) Y(i, j) /= d;
  }
}

void trsv_lower(const Mat& L, double* y) {
  const index_t n = L.r;
  for (index_t i = 0; i < n; ++i) {
    double s = y[i];
    for (index_t k = 0; k < i; ++k) s -= L(i, k) * y[k];
    y[i] = s / L(i, i);
  }
}

void trsv_lower_t(const Mat& L, double* y) {
  const index_t n = L.r;
  for (index_t i = n - 1; i >= 0; --i) {
    double s = y[i];
    for (index_t k = i + 1; k < n; ++k) s -= L(k, i) * y[k];
    y[i] = s / L(i, i);
  }
}

double gauge_weight(index_t k) {
  // 1 + 0.5 * frac((k+1) * c), c = (sqrt(5)-1)/2: positive, irregular, deterministic.
  const double x = static_cast<double>(k + 1) * 0.6180339887498949;
  return 1.0 + 0.5 * (x - std::floor(x));
}

double gauge_weight2(index_t k, index_t j) {
  // splitmix64 finaliser of (k, j) -> 53-bit uniform in [0, 1) -> [-1, 1); the GPU computes the
  // same integers (sweep.cu gauge_weight2).
  unsigned long long z = static_cast<unsigned long long>(k) * 0x9E3779B97F4A7C15ull +
                         static_cast<unsigned long long>(j) * 0xD1B54A32D192ED03ull + 0x632BE59BD9B4E019ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return static_cast<double>(z >> 11) * 0x1.0p-52 - 1.0;
}

namespace {

// Householder QR of A (m x n, row-major, in place), LAPACK sign convention.
// On return the upper trapezoid of A holds R (min(m,n) x n); below is junk.
void householder_r(Mat& A) {
  const index_t m = A.r, n = A.c;
  const index_t kmax = std::min(m, n);
  std::vector<double> v(static_cast<size_t>(m));
  for (index_t k = 0; k < kmax; ++k) {
    // Scaled reflector (Eigen makeHouseholder / LAPACK dlarfg): v = [1; x_tail / (x_k - beta)],
    // tau = (beta - x_k) / beta.  No reflection when the tail's squared norm is <= DBL_MIN, so
    // roundoff-level columns (norms ~1e-155) cannot overflow tau (the unscaled 2 / v^T v did,
    // and turned a whole F into NaN singular values).
    double s2 = 0.0;
    for (index_t i = k + 1; i < m; ++i) s2 += A(i, k) * A(i, k);
    if (s2 <= DBL_MIN) continue;
    const double xk = A(k, k);
    const double nrm = std::sqrt(xk * xk + s2);
    const double beta = xk >= 0.0 ? -nrm : nrm;
    const double tau = (beta - xk) / beta;
    const double scale = 1.0 / (xk - beta);
    v[static_cast<size_t>(k)] = 1.0;
    for (index_t i = k + 1; i < m; ++i) v[static_cast<size_t>(i)] = A(i, k) * scale;
    A(k, k) = beta;
    for (index_t i = k + 1; i < m; ++i) A(i, k) = 0.0;
    for (index_t j = k + 1; j < n; ++j) {
      double s = 0.0;
      for (index_t i = k; i < m; ++i) s += v[static_cast<size_t>(i)] * A(i, j);
      s *= tau;
      for (index_t i = k; i < m; ++i) A(i, j) -= s * v[static_cast<size_t>(i)];
    }
  }
}

}  // namespace

SvdLeft svd_left(const Mat& F) {
  const index_t b = F.r, f = F.c;
  SvdLeft out;
  const index_t m = std::min(b, f);
  // R = triu(qr(F^T)), m x b.
  Mat T = F.transpose();  // f x b
  householder_r(T);
  Mat R(m, b);
  for (index_t i = 0; i < m; ++i)
    for (index_t j = i; j < b; ++j) R(i, j) = T(i, j);

  // QR preconditioning (Drmac-Veselic): R^T = Q2 R2, so R = [R2^T 0] Q2^T and the
  // right singular vectors of R are Q2 times those of X = [R2^T 0] (m x b).
  // One-sided Jacobi on X converges in a few sweeps; V accumulates its rotations.
  Mat Rt = R.transpose();  // b x m
  std::vector<std::vector<double>> hv(static_cast<size_t>(m));
  std::vector<double> htau(static_cast<size_t>(m), 0.0);
  for (index_t k = 0; k < m; ++k) {
    double s2 = 0.0;
    for (index_t i = k + 1; i < b; ++i) s2 += Rt(i, k) * Rt(i, k);
    std::vector<double>& v = hv[static_cast<size_t>(k)];
    v.assign(static_cast<size_t>(b), 0.0);
    if (s2 <= DBL_MIN) continue;  // dlarfg / Eigen makeHouseholder: tau = 0
    const double x0 = Rt(k, k);
    const double nrm = std::sqrt(x0 * x0 + s2);
    const double beta = x0 >= 0.0 ? -nrm : nrm;
    const double tau = (beta - x0) / beta;
    const double scale = 1.0 / (x0 - beta);
    v[static_cast<size_t>(k)] = 1.0;
    for (index_t i = k + 1; i < b; ++i) v[static_cast<size_t>(i)] = Rt(i, k) * scale;
    htau[static_cast<size_t>(k)] = tau;
    Rt(k, k) = beta;
    for (index_t i = k + 1; i < b; ++i) Rt(i, k) = 0.0;
    for (index_t j = k + 1; j < m; ++j) {
      double d = Rt(k, j);
      for (index_t i = k + 1; i < b; ++i) d += v[static_cast<size_t>(i)] * Rt(i, j);
      d *= tau;
      Rt(k, j) -= d;
      for (index_t i = k + 1; i < b; ++i) Rt(i, j) -= d * v[static_cast<size_t>(i)];
    }
  }
  for (index_t i = 0; i < m; ++i)
    for (index_t j = 0; j < b; ++j) R(i, j) = (j < m && j <= i) ? Rt(j, i) : 0.0;  // X = [R2^T 0]

  Mat V = Mat::identity(b);
  const double tol = std::sqrt(static_cast<double>(std::max<index_t>(m, 1))) * DBL_EPSILON;
  int sweep = 0;
  for (; sweep < 100; ++sweep) {
    bool rotated = false;
    for (index_t p = 0; p < b - 1; ++p) {
      for (index_t q = p + 1; q < b; ++q) {
        double alpha = 0.0, beta = 0.0, gamma = 0.0;
        for (index_t i = 0; i < m; ++i) {
          alpha += R(i, p) * R(i, p);
          beta += R(i, q) * R(i, q);
          gamma += R(i, p) * R(i, q);
        }
        if (alpha == 0.0 || beta == 0.0) continue;
        if (!(std::abs(gamma) > tol * std::sqrt(alpha) * std::sqrt(beta))) continue;
        rotated = true;
        const double zeta = (beta - alpha) / (2.0 * gamma);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / std::sqrt(1.0 + t * t);
        const double sn = cs * t;
        for (index_t i = 0; i < m; ++i) {
          const double ap = R(i, p), aq = R(i, q);
          R(i, p) = cs * ap - sn * aq;
          R(i, q) = sn * ap + cs * aq;
        }
        for (index_t i = 0; i < b; ++i) {
          const double vp = V(i, p), vq = V(i, q);
          V(i, p) = cs * vp - sn * vq;
          V(i, q) = sn * vp + cs * vq;
        }
      }
    }
    if (!rotated) break;
  }
  out.sweeps = sweep + 1;
  // V <- Q2 V = H_0 ... H_{m-1} V
  for (index_t k = m - 1; k >= 0; --k) {
    const double tau = htau[static_cast<size_t>(k)];
    if (tau == 0.0) continue;
    const std::vector<double>& v = hv[static_cast<size_t>(k)];
    for (index_t j = 0; j < b; ++j) {
      double d = 0.0;
      for (index_t i = k; i < b; ++i) d += v[static_cast<size_t>(i)] * V(i, j);
      d *= tau;
      for (index_t i = k; i < b; ++i) V(i, j) -= d * v[static_cast<size_t>(i)];
    }
  }

  std::vector<double> norms(static_cast<size_t>(b));
  for (index_t j = 0; j < b; ++j) {
    double s = 0.0;
    for (index_t i = 0; i < m; ++i) s += R(i, j) * R(i, j);
    norms[static_cast<size_t>(j)] = std::sqrt(s);
  }
  std::vector<index_t> order(static_cast<size_t>(b));
  std::iota(order.begin(), order.end(), index_t{0});
  std::stable_sort(order.begin(), order.end(), [&](index_t x, index_t y) {
    return norms[static_cast<size_t>(x)] > norms[static_cast<size_t>(y)];
  });
  out.V = Mat(b, b);
  for (index_t k = 0; k < b; ++k)
    for (index_t i = 0; i < b; ++i) out.V(i, k) = V(i, order[static_cast<size_t>(k)]);
  out.sigma.resize(static_cast<size_t>(m));
  for (index_t k = 0; k < m; ++k) out.sigma[static_cast<size_t>(k)] = norms[static_cast<size_t>(order[static_cast<size_t>(k)])];
  return out;
}

Mat canonical_basis(const Mat& V, const std::vector<double>& sigma, index_t r) {
  const index_t b = V.r;
  Mat U(b, b);
  // U1: leading singular vectors; clusters of (numerically) equal singular values
  // get the basis orth(P_c G_c) of their span, singletons a sign fix.
  Mat A(b, r);
  const index_t ns = static_cast<index_t>(sigma.size());
  index_t k0 = 0;
  while (k0 < r) {
    index_t k1 = k0 + 1;
    while (k1 < r && k1 < ns && sigma[static_cast<size_t>(k1 - 1)] - sigma[static_cast<size_t>(k1)] <= kClusterTol * sigma[0]) ++k1;
    const index_t c = k1 - k0;
    if (c == 1) {
      double g = 0.0;
      for (index_t i = 0; i < b; ++i) g += gauge_weight(i) * V(i, k0);
      const double s = g >= 0.0 ? 1.0 : -1.0;
      for (index_t i = 0; i < b; ++i) A(i, k0) = s * V(i, k0);
    } else {
      // Z = U_c (U_c^T G_c)
      for (index_t j = 0; j < c; ++j) {
        for (index_t i = 0; i < b; ++i) A(i, k0 + j) = 0.0;
        for (index_t q = 0; q < c; ++q) {
          double m = 0.0;
          for (index_t i = 0; i < b; ++i) m += V(i, k0 + q) * gauge_weight2(i, j);
          for (index_t i = 0; i < b; ++i) A(i, k0 + j) += V(i, k0 + q) * m;
        }
      }
      // Modified Gram-Schmidt (two passes), then project onto span(U_c) once more and
      // orthonormalise again: the first orthonormalisation amplifies Z's rounding outside
      // span(U_c) by cond(U_c^T G_c); the re-projection removes it (U1 stays orthogonal to 1e-15).
      for (int round = 0; round < 2; ++round) {
        if (round == 1)
          for (index_t j = 0; j < c; ++j) {
            std::vector<double> m(static_cast<size_t>(c));
            for (index_t q = 0; q < c; ++q) {
              double d = 0.0;
              for (index_t i = 0; i < b; ++i) d += V(i, k0 + q) * A(i, k0 + j);
              m[static_cast<size_t>(q)] = d;
            }
            for (index_t i = 0; i < b; ++i) {
              double z = 0.0;
              for (index_t q = 0; q < c; ++q) z += V(i, k0 + q) * m[static_cast<size_t>(q)];
              A(i, k0 + j) = z;
            }
          }
        for (index_t j = 0; j < c; ++j) {
          for (int pass = 0; pass < 2; ++pass)
            for (index_t q = 0; q < j; ++q) {
              double d = 0.0;
              for (index_t i = 0; i < b; ++i) d += A(i, k0 + q) * A(i, k0 + j);
              for (index_t i = 0; i < b; ++i) A(i, k0 + j) -= d * A(i, k0 + q);
            }
          double nrm = 0.0;
          for (index_t i = 0; i < b; ++i) nrm += A(i, k0 + j) * A(i, k0 + j);
          nrm = std::sqrt(nrm);
          for (index_t i = 0; i < b; ++i) A(i, k0 + j) /= nrm;
        }
      }
    }
    k0 = k1;
  }
  for (index_t k = 0; k < r; ++k)
    for (index_t i = 0; i < b; ++i) U(i, k) = A(i, k);
  // Householder QR of U1 with generic sign rule; Q = H_0 ... H_{r-1}.
  std::vector<std::vector<double>> vs(static_cast<size_t>(r));
  std::vector<double> taus(static_cast<size_t>(r), 0.0);
  for (index_t k = 0; k < r; ++k) {
    double nrm2 = 0.0, rest2 = 0.0, g = 0.0;
    for (index_t i = k; i < b; ++i) {
      nrm2 += A(i, k) * A(i, k);
      if (i > k) rest2 += A(i, k) * A(i, k);
      g += gauge_weight(i) * A(i, k);
    }
    const double nrm = std::sqrt(nrm2);
    std::vector<double>& v = vs[static_cast<size_t>(k)];
    v.assign(static_cast<size_t>(b), 0.0);
    if (nrm == 0.0) continue;
    const double s = g >= 0.0 ? 1.0 : -1.0;
    const double xk = A(k, k);
    const double beta = -s * nrm;
    double vk;
    if (xk == 0.0 || (xk > 0.0) == (s > 0.0)) {
      vk = xk - beta;  // same signs: no cancellation
    } else {
      vk = -rest2 / (xk + beta);  // Parlett: x_k - beta = (x_k^2 - nrm^2)/(x_k + beta)
    }
    v[static_cast<size_t>(k)] = vk;
    double vtv = vk * vk;
    for (index_t i = k + 1; i < b; ++i) {
      v[static_cast<size_t>(i)] = A(i, k);
      vtv += A(i, k) * A(i, k);
    }
    const double tau = vtv > 0.0 ? 2.0 / vtv : 0.0;
    taus[static_cast<size_t>(k)] = tau;
    for (index_t j = k; j < r; ++j) {
      double d = 0.0;
      for (index_t i = k; i < b; ++i) d += v[static_cast<size_t>(i)] * A(i, j);
      d *= tau;
      for (index_t i = k; i < b; ++i) A(i, j) -= d * v[static_cast<size_t>(i)];
    }
  }
  // Q[:, r:] = H_0 ... H_{r-1} E_{r:}
  Mat Q(b, b - r);
  for (index_t j = 0; j < b - r; ++j) Q(r + j, j) = 1.0;
  for (index_t k = r - 1; k >= 0; --k) {
    const std::vector<double>& v = vs[static_cast<size_t>(k)];
    const double tau = taus[static_cast<size_t>(k)];
    if (tau == 0.0) continue;
    for (index_t j = 0; j < b - r; ++j) {
      double d = 0.0;
      for (index_t i = k; i < b; ++i) d += v[static_cast<size_t>(i)] * Q(i, j);
      d *= tau;
      for (index_t i = k; i < b; ++i) Q(i, j) -= d * v[static_cast<size_t>(i)];
    }
  }
  for (index_t i = 0; i < b; ++i)
    for (index_t j = 0; j < b - r; ++j) U(i, r + j) = Q(i, j);
  return U;
}

}  // namespace oracle
