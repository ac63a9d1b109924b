// Level sweep kernels (sm_100a): batched compression + subrow elimination.
//
// Reference semantics (one row at a time, ascending):
//   LevelMatrix::compress_row      proj/src/level_matrix.cpp:33-82
//   compress_far_concat (JacobiSVD) proj/src/compression.cpp:20-61
//   LevelMatrix::eliminate_subrow  proj/src/level_matrix.cpp:84-178
//   level_sweep hot loop           proj/src/factorization.cpp:56-59
//
// B200 design: one persistent kernel per level walks a task graph.  Rows are
// issued in wave (topological) order of the squared-pattern DAG; row j's first
// task waits until every row i < j of sq(j) has finished all its tasks (rows at
// block-graph distance >= 3 commute), so every block receives
// its updates in the reference order without atomics on data.  A row is
//   [A1 x nA1]  far-block gather + Householder TSQR leaves (fat rows only)
//   [A2]        TSQR combine, one-sided Jacobi SVD, rank rule, canonical U,
//               rotated diagonal, pivot Cholesky (+ shift retry), coupling
//   [A3 x nA3]  rotation / truncation / TRSM / retained Schur / zeroing of the
//               row's strip blocks (fat rows only; thin rows do it in A2)
//   [B  x nB ]  Schur panel-pair updates X_st -= g_s g_t^T from smem tiles
// Thin rows (level 1) are a single task done by one CTA.
#include <cfloat>
#include <cstdio>

#include "kernels.hpp"

namespace ceg {
namespace {

constexpr int T = kSweepThreads;
constexpr int NW = T / 32;
constexpr double kClusterTol = 1e-9;  // oracle/dense.hpp
constexpr int kPanelNb = 32;          // close neighbours per Schur panel (host planner matches)
constexpr int kPanelRows = 260;       // g rows per Schur panel (<= 256 + padding)

__device__ __forceinline__ double ldg(const double* p) { return __ldcg(p); }

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double gauge_weight2(int k, int j) {
  const double cj = __dadd_rn(0.6180339887498949, __dmul_rn(0.2071067811865475, static_cast<double>(j)));
  const double x = __dmul_rn(static_cast<double>(k + 1), cj);
  return 1.0 + 0.5 * (x - floor(x));
}
__device__ __forceinline__ double gauge_weight(int k) { return gauge_weight2(k, 0); }

__device__ __forceinline__ int rr_player(int k, int round, int nb) {
  return k == 0 ? 0 : 1 + (k - 1 + round) % (nb - 1);
}

__device__ int64_t find_slot(const int64_t* sq_ptr, const int* sq_col, const int64_t* sq_slot, int row, int col) {
  int64_t lo = sq_ptr[row], hi = sq_ptr[row + 1];
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    const int c = sq_col[mid];
    if (c == col) return sq_slot[mid];
    if (c < col) lo = mid + 1;
    else hi = mid;
  }
  return -1;
}

// index of neighbour t in row i's close list (or -1)
__device__ int64_t close_index(const SweepArgs& A, int i, int t) {
  int64_t lo = A.cl_ptr[i], hi = A.cl_ptr[i + 1];
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    const int c = A.cl_col[mid];
    if (c == t) return mid;
    if (c < t) lo = mid + 1;
    else hi = mid;
  }
  return -1;
}

struct Buf {
  double *R, *V, *U, *D, *C, *sig, *tau, *nrm;
  int* perm;
};

__device__ Buf carve(double* base, int bmax, int kcap) {
  Buf s;
  const int64_t bb = static_cast<int64_t>(bmax) * bmax;
  s.R = base;
  s.V = s.R + bb;
  s.U = s.V + bb;
  s.D = s.U + bb;
  s.C = s.D + bb;
  s.sig = s.C + static_cast<int64_t>(kcap) * bmax;
  s.tau = s.sig + bmax;
  s.nrm = s.tau + bmax;
  s.perm = reinterpret_cast<int*>(s.nrm + bmax);
  return s;
}

__device__ __forceinline__ void prof_add(const SweepArgs& A, int k, long long v) {
  if (A.prof && threadIdx.x == 0) atomicAdd(A.prof + k, static_cast<unsigned long long>(v));
}

__device__ void set_error(int* err, int code, int level, int64_t row) {
  if (atomicCAS(err, 0, code) == 0) {
    err[1] = level;
    err[2] = static_cast<int>(row & 0x7fffffff);
    err[3] = static_cast<int>(row >> 31);
  }
}

// Element (a, c) of X_ij (b_i x b_j) in the half-symmetric store.
__device__ __forceinline__ int64_t xidx(int a, int c, int bi, int bj, bool trans) {
  return trans ? static_cast<int64_t>(c) * bi + a : static_cast<int64_t>(a) * bj + c;
}

// Structured Householder QR update [R; C] -> [R'; 0].  R: b x b column-major
// (R[k][j] at R[j*b+k]); C: K x b column-major with leading dimension ldc
// (element (m, j) at C[j*ldc+m]: column walks are bank-conflict free).
// LAPACK dlarfg conventions.
__device__ void tsqr_update(double* R, double* C, int K, int b, int ldc, double* shr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k = 0; k < b; ++k) {
    double* Ck = C + static_cast<int64_t>(k) * ldc;
    if (warp == 0) {
      double s2 = 0.0;
      for (int m = lane; m < K; m += 32) {
        const double c = Ck[m];
        s2 += c * c;
      }
      s2 = warp_sum(s2);
      double tau = 0.0, scale = 0.0, beta = 0.0;
      if (s2 > 0.0) {
        const double x0 = R[k * b + k];
        const double nrm = sqrt(x0 * x0 + s2);
        beta = x0 >= 0.0 ? -nrm : nrm;
        tau = (beta - x0) / beta;
        scale = 1.0 / (x0 - beta);
      }
      __syncwarp();
      if (tau != 0.0) {
        if (lane == 0) R[k * b + k] = beta;
        for (int m = lane; m < K; m += 32) Ck[m] *= scale;
      }
      if (lane == 0) shr[0] = tau;
    }
    __syncthreads();
    const double tau = shr[0];
    if (tau != 0.0) {
      for (int j = k + 1 + warp; j < b; j += NW) {
        double* Cj = C + static_cast<int64_t>(j) * ldc;
        double s = 0.0;
        for (int m = lane; m < K; m += 32) s += Ck[m] * Cj[m];
        s = warp_sum(s);
        const double tw = tau * (R[j * b + k] + s);
        __syncwarp();
        if (lane == 0) R[j * b + k] -= tw;
        for (int m = lane; m < K; m += 32) Cj[m] -= tw * Ck[m];
      }
    }
    __syncthreads();
  }
}

// One-sided Jacobi on the columns of R (b x b, column-major); V accumulates.
__device__ void jacobi(double* R, double* V, int b, int meff, int* any) {
  // a group of G lanes handles one column pair per round (short reductions, many pairs in flight)
  const int G = b <= 64 ? 8 : (b <= 128 ? 16 : 32);
  const int gpw = 32 / G;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane / G, gl = lane % G;
  const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (grp * G));
  for (int idx = threadIdx.x; idx < b * b; idx += T) V[idx] = (idx / b == idx % b) ? 1.0 : 0.0;
  const double tol = sqrt(static_cast<double>(meff > 1 ? meff : 1)) * DBL_EPSILON;
  const int nb = b + (b & 1);
  for (int sweep = 0; sweep < 100; ++sweep) {
    if (threadIdx.x == 0) *any = 0;
    __syncthreads();
    for (int round = 0; round < nb - 1; ++round) {
      for (int pi = warp * gpw + grp; pi < nb / 2; pi += NW * gpw) {
        int p = rr_player(pi, round, nb), q = rr_player(nb - 1 - pi, round, nb);
        if (p > q) {
          const int t = p;
          p = q;
          q = t;
        }
        if (q >= b) continue;
        double* cp = R + p * b;
        double* cq = R + q * b;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int k = gl; k < b; k += G) {
          const double x = cp[k], y = cq[k];
          al += x * x;
          be += y * y;
          ga += x * y;
        }
        for (int o = G >> 1; o > 0; o >>= 1) {
          al += __shfl_xor_sync(gmask, al, o);
          be += __shfl_xor_sync(gmask, be, o);
          ga += __shfl_xor_sync(gmask, ga, o);
        }
        if (al == 0.0 || be == 0.0) continue;
        if (!(fabs(ga) > tol * sqrt(al) * sqrt(be))) continue;
        const double zeta = (be - al) / (2.0 * ga);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / sqrt(1.0 + t * t);
        const double sn = cs * t;
        __syncwarp(gmask);
        for (int k = gl; k < b; k += G) {
          const double x = cp[k], y = cq[k];
          cp[k] = cs * x - sn * y;
          cq[k] = sn * x + cs * y;
        }
        double* vp = V + p * b;
        double* vq = V + q * b;
        for (int k = gl; k < b; k += G) {
          const double x = vp[k], y = vq[k];
          vp[k] = cs * x - sn * y;
          vq[k] = sn * x + cs * y;
        }
        if (gl == 0) *any = 1;
      }
      __syncthreads();
    }
    const int a = *any;
    __syncthreads();
    if (!a) break;
  }
}

// QR preconditioning of the Jacobi SVD (Drmac-Veselic; oracle/dense.cpp svd_left):
// R^T = Q2 R2 by Householder on s.C (reflectors kept below the diagonal, tau in
// s.tau), then s.R <- X = R2^T (column-major, lower triangular).
__device__ void precondition_qr(const Buf& s, int b, double* shr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* Aq = s.C;  // b x b column-major, ld b
  for (int idx = threadIdx.x; idx < b * b; idx += T) {
    const int j = idx / b, i = idx % b;  // Aq(i, j) = R^T(i, j) = R(j, i)
    Aq[idx] = s.R[i * b + j];
  }
  __syncthreads();
  for (int k = 0; k < b; ++k) {
    double* Ak = Aq + k * b;
    if (warp == 0) {
      double s2 = 0.0;
      for (int i = k + 1 + lane; i < b; i += 32) s2 += Ak[i] * Ak[i];
      s2 = warp_sum(s2);
      double tau = 0.0, scale = 0.0, beta = 0.0;
      if (s2 > 0.0) {
        const double x0 = Ak[k];
        const double nrm = sqrt(x0 * x0 + s2);
        beta = x0 >= 0.0 ? -nrm : nrm;
        tau = (beta - x0) / beta;
        scale = 1.0 / (x0 - beta);
      }
      __syncwarp();
      if (tau != 0.0) {
        if (lane == 0) Ak[k] = beta;
        for (int i = k + 1 + lane; i < b; i += 32) Ak[i] *= scale;
      }
      if (lane == 0) s.tau[k] = tau;
    }
    __syncthreads();
    const double tau = s.tau[k];
    if (tau != 0.0) {
      for (int j = k + 1 + warp; j < b; j += NW) {
        double* Aj = Aq + j * b;
        double d = 0.0;
        for (int i = k + 1 + lane; i < b; i += 32) d += Ak[i] * Aj[i];
        d = warp_sum(d);
        d = tau * (Aj[k] + d);
        __syncwarp();
        if (lane == 0) Aj[k] -= d;
        for (int i = k + 1 + lane; i < b; i += 32) Aj[i] -= d * Ak[i];
      }
    }
    __syncthreads();
  }
  for (int idx = threadIdx.x; idx < b * b; idx += T) {
    const int j = idx / b, i = idx % b;  // X(i, j) = R2(j, i) for i >= j
    s.R[idx] = i >= j ? Aq[i * b + j] : 0.0;
  }
  __syncthreads();
  (void)shr;
}

// V <- Q2 V with Q2 = H_0 ... H_{b-1} from precondition_qr (V column-major).
__device__ void apply_q2(const Buf& s, int b) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* Aq = s.C;
  for (int k = b - 1; k >= 0; --k) {
    const double tau = s.tau[k];
    if (tau == 0.0) continue;
    const double* v = Aq + k * b;  // v_k = 1, v_i (i > k) below the diagonal
    for (int j = warp; j < b; j += NW) {
      double* Vj = s.V + j * b;
      double d = 0.0;
      for (int i = k + 1 + lane; i < b; i += 32) d += v[i] * Vj[i];
      d = warp_sum(d);
      d = tau * (Vj[k] + d);
      __syncwarp();
      if (lane == 0) Vj[k] -= d;
      for (int i = k + 1 + lane; i < b; i += 32) Vj[i] -= d * v[i];
    }
    __syncthreads();
  }
}

// Canonical gauge (oracle/dense.cpp canonical_basis): U1 = leading singular
// vectors (clusters of equal singular values -> orth(U_c U_c^T G_c), singletons
// sign-fixed), U2 = trailing columns of the Householder QR of U1.
// V: column-major right singular vectors of R (unsorted), perm: sorted order.
// Writes U row-major into s.U.  Uses s.C (A, then Q) and s.R (reflectors).
__device__ void canonical_basis(const Buf& s, int b, int r, int nsig) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* A = s.C;   // b x r column-major
  double* Vh = s.R;  // reflectors, column-major
  __shared__ int cstart[512];
  if (threadIdx.x == 0) {
    int k0 = 0;
    while (k0 < r) {
      int k1 = k0 + 1;
      while (k1 < r && k1 < nsig && s.sig[k1 - 1] - s.sig[k1] <= kClusterTol * s.sig[0]) ++k1;
      for (int k = k0; k < k1; ++k) cstart[k] = k0;
      k0 = k1;
    }
  }
  __syncthreads();
  int nclus = 0;
  for (int k0 = 0; k0 < r; ++k0) {
    if (cstart[k0] != k0) continue;
    int k1 = k0 + 1;
    while (k1 < r && cstart[k1] == k0) ++k1;
    const int c = k1 - k0;
    if ((nclus++ % NW) != warp) continue;
    if (c == 1) {
      const double* v = s.V + static_cast<int64_t>(s.perm[k0]) * b;
      double g = 0.0;
      for (int a = lane; a < b; a += 32) g += gauge_weight(a) * v[a];
      g = warp_sum(g);
      const double sg = g >= 0.0 ? 1.0 : -1.0;
      for (int a = lane; a < b; a += 32) A[k0 * b + a] = sg * v[a];
    } else {
      for (int j = 0; j < c; ++j) {
        double* z = A + (k0 + j) * b;
        for (int a = lane; a < b; a += 32) z[a] = 0.0;
        for (int q = 0; q < c; ++q) {
          const double* v = s.V + static_cast<int64_t>(s.perm[k0 + q]) * b;
          double m = 0.0;
          for (int a = lane; a < b; a += 32) m += v[a] * gauge_weight2(a, j);
          m = warp_sum(m);
          for (int a = lane; a < b; a += 32) z[a] += v[a] * m;
        }
      }
      __syncwarp();
      for (int j = 0; j < c; ++j) {
        double* z = A + (k0 + j) * b;
        for (int pass = 0; pass < 2; ++pass)
          for (int q = 0; q < j; ++q) {
            const double* y = A + (k0 + q) * b;
            double d = 0.0;
            for (int a = lane; a < b; a += 32) d += y[a] * z[a];
            d = warp_sum(d);
            for (int a = lane; a < b; a += 32) z[a] -= d * y[a];
            __syncwarp();
          }
        double n2 = 0.0;
        for (int a = lane; a < b; a += 32) n2 += z[a] * z[a];
        const double nrm = sqrt(warp_sum(n2));
        for (int a = lane; a < b; a += 32) z[a] /= nrm;
        __syncwarp();
      }
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < b * r; idx += T) {
    const int k = idx / b, a = idx % b;
    s.U[a * b + k] = A[idx];
  }
  __syncthreads();
  for (int k = 0; k < r; ++k) {
    if (warp == 0) {
      double n2 = 0.0, rest = 0.0, g = 0.0;
      for (int a = k + lane; a < b; a += 32) {
        const double x = A[k * b + a];
        n2 += x * x;
        if (a > k) rest += x * x;
        g += gauge_weight(a) * x;
      }
      n2 = warp_sum(n2);
      rest = warp_sum(rest);
      g = warp_sum(g);
      const double nrm = sqrt(n2);
      double tau = 0.0;
      if (nrm != 0.0) {
        const double sg = g >= 0.0 ? 1.0 : -1.0;
        const double xk = A[k * b + k];
        const double beta = -sg * nrm;
        double vk;
        if (xk == 0.0 || (xk > 0.0) == (sg > 0.0)) vk = xk - beta;
        else vk = -rest / (xk + beta);
        const double vtv = vk * vk + rest;
        tau = vtv > 0.0 ? 2.0 / vtv : 0.0;
        for (int a = k + lane; a < b; a += 32) Vh[k * b + a] = (a == k) ? vk : A[k * b + a];
      }
      if (lane == 0) s.tau[k] = tau;
    }
    __syncthreads();
    const double tau = s.tau[k];
    if (tau != 0.0) {
      for (int j = k + 1 + warp; j < r; j += NW) {
        double d = 0.0;
        for (int a = k + lane; a < b; a += 32) d += Vh[k * b + a] * A[j * b + a];
        d = warp_sum(d) * tau;
        __syncwarp();
        for (int a = k + lane; a < b; a += 32) A[j * b + a] -= d * Vh[k * b + a];
      }
    }
    __syncthreads();
  }
  double* Q = s.C;
  const int nq = b - r;
  for (int idx = threadIdx.x; idx < nq * b; idx += T) {
    const int jj = idx / b, a = idx % b;
    Q[idx] = (a == r + jj) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int k = r - 1; k >= 0; --k) {
    const double tau = s.tau[k];
    if (tau != 0.0) {
      for (int jj = warp; jj < nq; jj += NW) {
        double d = 0.0;
        for (int a = k + lane; a < b; a += 32) d += Vh[k * b + a] * Q[jj * b + a];
        d = warp_sum(d) * tau;
        __syncwarp();
        for (int a = k + lane; a < b; a += 32) Q[jj * b + a] -= d * Vh[k * b + a];
      }
    }
    __syncthreads();
  }
  for (int idx = threadIdx.x; idx < nq * b; idx += T) {
    const int jj = idx / b, a = idx % b;
    s.U[a * b + r + jj] = Q[idx];
  }
  __syncthreads();
}

// Gather the far blocks with far-ordinal in [fb, fe) of row i into F^T chunks
// and fold them into the TSQR triangle s.R.  Returns far columns seen.
__device__ int gather_tsqr(const SweepArgs& A, int i, int b, const Buf& s, int fb, int fe, int* nzflag,
                           double* shr) {
  const int tid = threadIdx.x;
  int fcols = 0, kfill = 0, ord = 0;
  for (int64_t e = A.sq_ptr[i]; e < A.sq_ptr[i + 1]; ++e) {
    if (A.sq_kind[e] != 2) continue;
    const int o = ord++;
    if (o < fb) continue;
    if (o >= fe) break;
    const int j = A.sq_col[e];
    const int bj = A.bsz[j];
    const bool tr = j > i;
    const double* X = A.store + A.slot_off[A.sq_slot[e]];
    if (kfill + bj > A.kcap) {
      tsqr_update(s.R, s.C, kfill, b, A.kcap, shr);
      kfill = 0;
    }
    for (int idx = tid; idx < bj * b; idx += T) {
      int a, c;
      if (tr) {
        c = idx / b;
        a = idx % b;
      } else {
        a = idx / bj;
        c = idx % bj;
      }
      const double v = ldg(X + xidx(a, c, b, bj, tr));
      s.C[static_cast<int64_t>(a) * A.kcap + kfill + c] = v;  // F^T chunk, column-major
      if (v != 0.0) *nzflag = 1;
    }
    __syncthreads();
    kfill += bj;
    fcols += bj;
  }
  if (kfill > 0) tsqr_update(s.R, s.C, kfill, b, A.kcap, shr);
  __syncthreads();
  return fcols;
}

// Strip block e of row i: rotate by U (basis) or keep, truncate far rows >= r,
// then for close blocks g_t = (L^{-1} X[r:, :])^T and X[:r, :] -= C g_t^T, and
// finally zero rows >= r (level_matrix.cpp:51-65, 125-171).
// s.U = U (row-major), s.R = L (w x w), s.V = C (r x w); s.C, s.D scratch.
__device__ void strip_block(const SweepArgs& A, int i, int b, int r, int w, bool basis, int64_t e, const Buf& s) {
  const int tid = threadIdx.x;
  const int j = A.sq_col[e];
  const int bj = A.bsz[j];
  const bool tr = j > i;
  const int kind = A.sq_kind[e];
  double* X = A.store + A.slot_off[A.sq_slot[e]];
  const int n = b * bj;
  if (basis) {
    for (int idx = tid; idx < n; idx += T) {
      int a, c;
      if (tr) {
        c = idx / b;
        a = idx % b;
      } else {
        a = idx / bj;
        c = idx % bj;
      }
      s.C[a * bj + c] = ldg(X + xidx(a, c, b, bj, tr));
    }
    __syncthreads();
    for (int idx = tid; idx < n; idx += T) {
      const int a = idx / bj, c = idx % bj;
      double acc = 0.0;
      if (!(kind == 2 && a >= r))
        for (int k = 0; k < b; ++k) acc += s.U[k * b + a] * s.C[k * bj + c];
      s.D[idx] = acc;
    }
  } else {
    for (int idx = tid; idx < n; idx += T) {
      int a, c;
      if (tr) {
        c = idx / b;
        a = idx % b;
      } else {
        a = idx / bj;
        c = idx % bj;
      }
      s.D[a * bj + c] = (kind == 2 && a >= r) ? 0.0 : ldg(X + xidx(a, c, b, bj, tr));
    }
  }
  __syncthreads();
  if (kind == 1 && w > 0) {
    const int64_t ci = close_index(A, i, j);
    const int roff = A.cl_roff[ci];
    double* G = A.fac + A.g_off[i];
    for (int c = tid; c < bj; c += T) {
      double* gc = G + static_cast<int64_t>(r + roff + c) * w;
      for (int q = 0; q < w; ++q) {
        double acc = s.D[(r + q) * bj + c];
        for (int p = 0; p < q; ++p) acc -= s.R[q * w + p] * s.D[(r + p) * bj + c];
        acc /= s.R[q * w + q];
        s.D[(r + q) * bj + c] = acc;
        gc[q] = acc;
      }
    }
    __syncthreads();
    for (int idx = tid; idx < r * bj; idx += T) {
      const int a = idx / bj, c = idx % bj;
      double acc = 0.0;
      for (int q = 0; q < w; ++q) acc += s.V[a * w + q] * s.D[(r + q) * bj + c];
      s.D[idx] -= acc;
    }
    __syncthreads();
  }
  for (int idx = tid; idx < n; idx += T) {
    int a, c;
    if (tr) {
      c = idx / b;
      a = idx % b;
    } else {
      a = idx / bj;
      c = idx % bj;
    }
    X[xidx(a, c, b, bj, tr)] = (w > 0 && a >= r) ? 0.0 : s.D[a * bj + c];
  }
  __syncthreads();
}

// Schur update of one panel pair (P, Q), P <= Q, of row i's close list:
// X_ts -= g_t g_s^T for s in panel P, t in panel Q, s <= t (level_matrix.cpp:148-162).
// g rows of both panels are staged in shared memory.
__device__ void panel_update(const SweepArgs& A, int i, int r, int w, int P, int Q, double* sm) {
  __shared__ long long slot_tab[kPanelNb * kPanelNb];  // value offset of stored (t, s), -1: not updated
  __shared__ int tab_bs[kPanelNb];
  __shared__ unsigned char xblk[kPanelRows], yblk[kPanelRows];
  __shared__ unsigned short xloc[kPanelRows], yloc[kPanelRows];
  const int tid = threadIdx.x;
  const int64_t c0 = A.cl_ptr[i];
  const int* ps = A.pan_start + A.pan_ptr[i];
  const int s0 = ps[P], s1 = ps[P + 1], t0 = ps[Q], t1 = ps[Q + 1];
  const int ns = s1 - s0, nt = t1 - t0;
  const int rs0 = A.cl_roff[c0 + s0];
  const int rsn = A.cl_roff[c0 + s1 - 1] + A.bsz[A.cl_col[c0 + s1 - 1]] - rs0;
  const int rt0 = A.cl_roff[c0 + t0];
  const int rtn = A.cl_roff[c0 + t1 - 1] + A.bsz[A.cl_col[c0 + t1 - 1]] - rt0;
  const int lds = (rsn + 3) & ~3, ldt = (rtn + 3) & ~3;
  // g rows transposed into shared memory: GsT[q][y], GtT[q][x]
  const double* G = A.fac + A.g_off[i];
  double* GsT = sm;
  double* GtT = P == Q ? sm : sm + static_cast<int64_t>(lds) * w;
  for (int idx = tid; idx < lds * w; idx += T) {
    const int y = idx / w, q = idx % w;
    GsT[q * lds + y] = y < rsn ? ldg(G + static_cast<int64_t>(r + rs0 + y) * w + q) : 0.0;
  }
  if (P != Q)
    for (int idx = tid; idx < ldt * w; idx += T) {
      const int x = idx / w, q = idx % w;
      GtT[q * ldt + x] = x < rtn ? ldg(G + static_cast<int64_t>(r + rt0 + x) * w + q) : 0.0;
    }
  for (int idx = tid; idx < nt * ns; idx += T) {
    const int kt = idx / ns, ks = idx % ns;
    long long off = -1;
    if (!(P == Q && ks > kt)) {
      const int t = A.cl_col[c0 + t0 + kt], s = A.cl_col[c0 + s0 + ks];
      const int64_t slot = find_slot(A.sq_ptr, A.sq_col, A.sq_slot, t, s);
      if (slot < 0) set_error(A.err, kErrPattern, A.level, i);
      else off = A.slot_off[slot];
    }
    slot_tab[idx] = off;
  }
  for (int ks = tid; ks < ns; ks += T) {
    const int e = static_cast<int>(c0) + s0 + ks;
    const int bs_ = A.bsz[A.cl_col[e]];
    tab_bs[ks] = bs_;
    const int y0 = A.cl_roff[e] - rs0;
    for (int y = 0; y < bs_; ++y) {
      yblk[y0 + y] = static_cast<unsigned char>(ks);
      yloc[y0 + y] = static_cast<unsigned short>(y);
    }
  }
  for (int kt = tid; kt < nt; kt += T) {
    const int e = static_cast<int>(c0) + t0 + kt;
    const int bt = A.bsz[A.cl_col[e]];
    const int x0 = A.cl_roff[e] - rt0;
    for (int x = 0; x < bt; ++x) {
      xblk[x0 + x] = static_cast<unsigned char>(kt);
      xloc[x0 + x] = static_cast<unsigned short>(x);
    }
  }
  __syncthreads();
  // rtn x rsn outer product in 4x4 register tiles; epilogue scatters into the (t, s) blocks
  const int mx = ldt / 4, my = lds / 4;
  for (int mt = tid; mt < mx * my; mt += T) {
    const int x0 = (mt / my) * 4, y0 = (mt % my) * 4;
    double acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[a][c] = 0.0;
    for (int q = 0; q < w; ++q) {
      const double2 ta = *reinterpret_cast<const double2*>(GtT + q * ldt + x0);
      const double2 tb = *reinterpret_cast<const double2*>(GtT + q * ldt + x0 + 2);
      const double2 sa = *reinterpret_cast<const double2*>(GsT + q * lds + y0);
      const double2 sb = *reinterpret_cast<const double2*>(GsT + q * lds + y0 + 2);
      const double av[4] = {ta.x, ta.y, tb.x, tb.y}, cv[4] = {sa.x, sa.y, sb.x, sb.y};
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[a][c] += av[a] * cv[c];
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int x = x0 + a;
      if (x >= rtn) break;
      const int kt = xblk[x], xl = xloc[x];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int y = y0 + c;
        if (y >= rsn) break;
        const int ks = yblk[y];
        const long long off = slot_tab[kt * ns + ks];
        if (off < 0) continue;
        double* X = A.store + off + static_cast<int64_t>(xl) * tab_bs[ks] + yloc[y];
        *X = ldg(X) - acc[a][c];
      }
    }
  }
  __syncthreads();
}

__device__ void all_panels(const SweepArgs& A, int i, int r, int w, double* sm) {
  const int np = static_cast<int>(A.pan_ptr[i + 1] - A.pan_ptr[i]) - 1;
  for (int P = 0; P < np; ++P)
    for (int Q = P; Q < np; ++Q) panel_update(A, i, r, w, P, Q, sm);
}

// A2: compression decision + basis + pivot factorisation; with nA3 == 0 also the strip,
// with nB == 0 also the Schur panels.
__device__ void task_a2(const SweepArgs& A, int i, const Buf& s, int nA1, int nA3, int nB) {
  __shared__ double shr[4];
  __shared__ int sflag[4];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long t_a2 = clock64();
  const int b = A.bsz[i];
  const int64_t p0 = A.sq_ptr[i], p1 = A.sq_ptr[i + 1];
  int64_t dslot = -1;
  for (int64_t e = p0; e < p1; ++e)
    if (A.sq_col[e] == i) {
      dslot = A.sq_slot[e];
      break;
    }
  double* Dg = A.store + A.slot_off[dslot];
  for (int idx = tid; idx < b * b; idx += T) {
    s.D[idx] = ldg(Dg + idx);
    s.R[idx] = 0.0;
  }
  if (tid == 0) sflag[0] = 0;
  __syncthreads();

  // ---- far-block triangle (compression.cpp:38-48) ----
  int fcols;
  if (nA1 == 0) {
    fcols = gather_tsqr(A, i, b, s, 0, 1 << 30, &sflag[0], shr);
  } else {
    fcols = static_cast<int>(A.fsum[i]);
    // fold the leaf triangles, as many per chunk as fit (chunk rows <= kcap)
    const int per = A.kcap / b > 0 ? A.kcap / b : 1;
    for (int k0 = 0; k0 < nA1; k0 += per) {
      const int nk = nA1 - k0 < per ? nA1 - k0 : per;
      const int K = nk * b;
      for (int idx = tid; idx < K * b; idx += T) {
        const int j = idx / K, m = idx % K;  // chunk element (m, j) = R_{k0 + m/b}[m%b][j]
        const double* Rk = A.rscratch + A.rs_off[i] + static_cast<int64_t>(k0 + m / b) * b * b;
        s.C[static_cast<int64_t>(j) * A.kcap + m] = ldg(Rk + j * b + m % b);
      }
      __syncthreads();
      tsqr_update(s.R, s.C, K, b, A.kcap, shr);
    }
    if (tid == 0) sflag[0] = ld_acquire(A.nzflag + i);
    __syncthreads();
  }
  const bool nonzero = sflag[0] != 0;
  const int meff = fcols < b ? fcols : b;
  long long tp = clock64();
  prof_add(A, kProfA2Tsqr, tp - t_a2);

  // ---- rank decision + basis (compression.cpp:20-61) ----
  int r = 0, nsig = 0;
  bool basis = false;
  if (fcols > 0) {
    bool need_svd;
    if (A.mode == 1) {
      r = A.fixed_rank < b ? A.fixed_rank : b;
      need_svd = nonzero && r < b;
    } else {
      need_svd = nonzero;
    }
    if (need_svd) {
      precondition_qr(s, b, shr);
      jacobi(s.R, s.V, b, meff, &sflag[1]);
      apply_q2(s, b);
      for (int j = warp; j < b; j += NW) {
        double acc = 0.0;
        for (int k = lane; k < b; k += 32) acc += s.R[j * b + k] * s.R[j * b + k];
        acc = warp_sum(acc);
        if (lane == 0) s.nrm[j] = sqrt(acc);
      }
      __syncthreads();
      for (int j = tid; j < b; j += T) {
        const double sj = s.nrm[j];
        int rank = 0;
        for (int k = 0; k < b; ++k) {
          const double sk = s.nrm[k];
          if (sk > sj || (sk == sj && k < j)) ++rank;
        }
        s.perm[rank] = j;
        s.sig[rank] = sj;
      }
      __syncthreads();
      nsig = meff;
      for (int k = tid; k < nsig; k += T) A.sigma[A.sigma_off[i] + k] = s.sig[k];
      if (A.mode == 0) {
        const double thr = A.absolute ? A.eps : A.eps * s.sig[0];
        r = nsig;
        for (int k = 0; k < nsig; ++k)
          if (s.sig[k] <= thr) {
            r = k;
            break;
          }
        if (A.forced && A.forced[i] >= 0) r = A.forced[i];
        if (r > b) r = b;
      }
      basis = r < b;
    } else if (A.mode == 0) {
      r = 0;
    }
  }
  const int w = b - r;
  {
    const long long t = clock64();
    prof_add(A, kProfA2Svd, t - tp);
    tp = t;
  }

  // ---- basis and rotated diagonal (level_matrix.cpp:51-54) ----
  if (basis) {
    canonical_basis(s, b, r, nsig);
    double* Ug = A.basis + A.basis_off[i];
    for (int idx = tid; idx < b * b; idx += T) Ug[idx] = s.U[idx];
    for (int idx = tid; idx < b * b; idx += T) {
      const int a = idx / b, c = idx % b;
      double acc = 0.0;
      for (int k = 0; k < b; ++k) acc += s.D[a * b + k] * s.U[k * b + c];
      s.C[idx] = acc;
    }
    __syncthreads();
    for (int idx = tid; idx < b * b; idx += T) {
      const int a = idx / b, c = idx % b;
      double acc = 0.0;
      for (int k = 0; k < b; ++k) acc += s.U[k * b + a] * s.C[k * b + c];
      s.R[idx] = acc;
    }
    __syncthreads();
    for (int idx = tid; idx < b * b; idx += T) {
      const int a = idx / b, c = idx % b;
      s.D[idx] = 0.5 * (s.R[a * b + c] + s.R[c * b + a]);
    }
    __syncthreads();
  }

  {
    const long long t = clock64();
    prof_add(A, kProfA2Basis, t - tp);
    tp = t;
  }
  // ---- pivot factorisation (level_matrix.cpp:104-138) ----
  if (w > 0) {
    double* P = s.R;     // w x w
    double* Pbak = s.V;  // shift-retry backup, then the coupling C (r x w)
    for (int idx = tid; idx < w * w; idx += T) {
      const int q = idx / w, p = idx % w;
      P[idx] = s.D[(r + q) * b + r + p];
      Pbak[idx] = P[idx];
    }
    __syncthreads();
    for (int attempt = 0; attempt < 2; ++attempt) {
      if (attempt == 1) {
        if (tid == 0) {
          double tr = 0.0;
          for (int q = 0; q < w; ++q) tr += Pbak[q * w + q];
          shr[1] = 1e-12 * tr / static_cast<double>(w);
        }
        __syncthreads();
        for (int idx = tid; idx < w * w; idx += T) {
          const int q = idx / w, p = idx % w;
          P[idx] = Pbak[idx] + (q == p ? shr[1] : 0.0);
        }
        __syncthreads();
      }
      if (tid == 0) sflag[2] = 0;
      __syncthreads();
      for (int k = 0; k < w; ++k) {
        if (tid == 0) {
          const double d = P[k * w + k];
          if (!(d > 0.0)) sflag[2] = 1;
          else P[k * w + k] = sqrt(d);
        }
        __syncthreads();
        if (sflag[2]) break;
        const double dk = P[k * w + k];
        for (int q = k + 1 + tid; q < w; q += T) P[q * w + k] /= dk;
        __syncthreads();
        const int m = w - k - 1;
        for (int idx = tid; idx < m * m; idx += T) {
          const int q = k + 1 + idx / m, p = k + 1 + idx % m;
          if (p <= q) P[q * w + p] -= P[q * w + k] * P[p * w + k];
        }
        __syncthreads();
      }
      if (!sflag[2]) {
        if (attempt == 1 && tid == 0) atomicAdd(A.shifts, 1);
        break;
      }
      if (attempt == 1) {
        if (tid == 0) set_error(A.err, kErrBreakdown, A.level, i);
        return;
      }
    }
    double* L = A.fac + A.chol_off[i];
    for (int idx = tid; idx < w * w; idx += T) {
      const int q = idx / w, p = idx % w;
      const double v = p <= q ? P[idx] : 0.0;
      P[idx] = v;
      L[idx] = v;
    }
    __syncthreads();
    // coupling C = (L^{-1} D[r:, :r])^T -> G rows [0, r) and s.V
    double* G = A.fac + A.g_off[i];
    for (int rho = tid; rho < r; rho += T) {
      double* y = s.V + rho * w;
      for (int q = 0; q < w; ++q) {
        double acc = s.D[(r + q) * b + rho];
        for (int p = 0; p < q; ++p) acc -= P[q * w + p] * y[p];
        y[q] = acc / P[q * w + q];
      }
      for (int q = 0; q < w; ++q) G[static_cast<int64_t>(rho) * w + q] = y[q];
    }
    __syncthreads();
    // D[:r, :r] -= C C^T; eliminated rows/cols of D leave the level
    for (int idx = tid; idx < b * b; idx += T) {
      const int a = idx / b, c = idx % b;
      if (a >= r || c >= r) {
        s.D[idx] = 0.0;
      } else {
        double acc = 0.0;
        for (int q = 0; q < w; ++q) acc += s.V[a * w + q] * s.V[c * w + q];
        s.D[idx] -= acc;
      }
    }
    __syncthreads();
  }
  for (int idx = tid; idx < b * b; idx += T) Dg[idx] = s.D[idx];
  if (tid == 0) {
    A.rank[i] = r;
    A.width[i] = w;
    A.has_basis[i] = basis ? 1 : 0;
    A.fcols[i] = fcols;
    A.nsig[i] = nsig;
  }
  __syncthreads();
  {
    const long long t = clock64();
    prof_add(A, kProfA2Pivot, t - tp);
    tp = t;
  }

  // ---- strip (thin rows) ----
  if (nA3 == 0 && (basis || w > 0)) {
    for (int64_t e = p0; e < p1; ++e)
      if (A.sq_kind[e] != 0) strip_block(A, i, b, r, w, basis, e, s);
    {
      const long long t = clock64();
      prof_add(A, kProfA2Strip, t - tp);
      tp = t;
    }
    if (nB == 0 && w > 0) all_panels(A, i, r, w, s.R);
    prof_add(A, kProfA2Panels, clock64() - tp);
  }
}

// A3 tile k: strip entries with strip-ordinal in [k*ns/nA3, (k+1)*ns/nA3).
__device__ void task_a3(const SweepArgs& A, int i, const Buf& s, int k, int nA3, int nB) {
  const int tid = threadIdx.x;
  const int b = A.bsz[i];
  const int r = __ldcg(A.rank + i), w = __ldcg(A.width + i);
  const bool basis = __ldcg(reinterpret_cast<const unsigned char*>(A.has_basis) + i) != 0;
  if (!basis && w == 0) return;
  if (basis)
    for (int idx = tid; idx < b * b; idx += T) s.U[idx] = ldg(A.basis + A.basis_off[i] + idx);
  if (w > 0) {
    for (int idx = tid; idx < w * w; idx += T) s.R[idx] = ldg(A.fac + A.chol_off[i] + idx);
    for (int idx = tid; idx < r * w; idx += T) s.V[idx] = ldg(A.fac + A.g_off[i] + idx);
  }
  __syncthreads();
  const int64_t p0 = A.sq_ptr[i], p1 = A.sq_ptr[i + 1];
  const int ns = static_cast<int>(p1 - p0) - 1;
  const int ob = static_cast<int>(static_cast<int64_t>(ns) * k / nA3);
  const int oe = static_cast<int>(static_cast<int64_t>(ns) * (k + 1) / nA3);
  int ord = 0;
  for (int64_t e = p0; e < p1; ++e) {
    if (A.sq_kind[e] == 0) continue;
    const int o = ord++;
    if (o < ob) continue;
    if (o >= oe) break;
    strip_block(A, i, b, r, w, basis, e, s);
  }
  (void)nB;
}

__global__ void __launch_bounds__(T) sweep_kernel(SweepArgs A) {
  extern __shared__ double smem_dyn[];
  double* base = A.use_global_scratch ? A.scratch + static_cast<int64_t>(blockIdx.x) * A.scratch_per_cta : smem_dyn;
  const Buf s = carve(base, A.bmax, A.kcap);
  __shared__ long long s_item;
  __shared__ int s_stop;
  __shared__ double shr[4];
  __shared__ int nz;
  for (;;) {
    if (threadIdx.x == 0) {
      s_stop = *reinterpret_cast<volatile int*>(A.err) != 0;
      s_item = s_stop ? 0 : static_cast<long long>(atomicAdd(A.ticket, 1ULL));
    }
    __syncthreads();
    if (s_stop) break;
    const long long item = s_item;
    if (item >= A.n_items) break;
    const int i = A.item_row[item];
    const int part = A.item_part[item];
    const int nA1 = A.nA1[i], nA3 = A.nA3[i], nB = A.nB[i];
    // stage of the item and the number of this row's items it must wait for
    int stage, k = 0, need = 0;
    if (part < nA1) {
      stage = 1;
      k = part;
    } else if (part == nA1) {
      stage = 2;
      need = nA1;
    } else if (part <= nA1 + nA3) {
      stage = 3;
      k = part - nA1 - 1;
      need = nA1 + 1;
    } else {
      stage = 4;
      k = part - nA1 - 1 - nA3;
      need = nA1 + 1 + nA3;
    }
    const bool first = (stage == 1) || (stage == 2 && nA1 == 0);
    const long long t_wait = clock64();
    if (threadIdx.x == 0) {
      if (first) {
        for (int64_t e = A.sq_ptr[i]; e < A.sq_ptr[i + 1]; ++e) {
          const int j = A.sq_col[e];
          if (j >= i) break;
          const int target = 1 + A.nA1[j] + A.nA3[j] + A.nB[j];
          while (ld_acquire(A.done + j) < target) {
            if (*reinterpret_cast<volatile int*>(A.err) != 0) {
              s_stop = 1;
              break;
            }
            __nanosleep(64);
          }
          if (s_stop) break;
        }
      } else {
        while (ld_acquire(A.done + i) < need) {
          if (*reinterpret_cast<volatile int*>(A.err) != 0) {
            s_stop = 1;
            break;
          }
          __nanosleep(64);
        }
      }
      __threadfence();
      nz = 0;
    }
    __syncthreads();
    if (s_stop) break;
    const long long t_run = clock64();
    prof_add(A, kProfWait, t_run - t_wait);
    if (stage == 1) {
      const int b = A.bsz[i];
      for (int idx = threadIdx.x; idx < b * b; idx += T) s.R[idx] = 0.0;
      __syncthreads();
      // far-ordinal range of this leaf
      int nf = 0;
      for (int64_t e = A.sq_ptr[i]; e < A.sq_ptr[i + 1]; ++e) nf += A.sq_kind[e] == 2;
      const int fb = static_cast<int>(static_cast<int64_t>(nf) * k / nA1);
      const int fe = static_cast<int>(static_cast<int64_t>(nf) * (k + 1) / nA1);
      gather_tsqr(A, i, b, s, fb, fe, &nz, shr);
      double* Rk = A.rscratch + A.rs_off[i] + static_cast<int64_t>(k) * b * b;
      for (int idx = threadIdx.x; idx < b * b; idx += T) Rk[idx] = s.R[idx];
      if (threadIdx.x == 0 && nz) atomicOr(A.nzflag + i, 1);
    } else if (stage == 2) {
      task_a2(A, i, s, nA1, nA3, nB);
    } else if (stage == 3) {
      task_a3(A, i, s, k, nA3, nB);
    } else {
      const int w = __ldcg(A.width + i);
      if (w > 0) {
        const int r = __ldcg(A.rank + i);
        const int np = static_cast<int>(A.pan_ptr[i + 1] - A.pan_ptr[i]) - 1;
        if (nB == 1) {
          all_panels(A, i, r, w, s.R);
        } else {
          // tile k -> panel pair (P, Q), P <= Q
          int P = 0, kk = k;
          while (kk >= np - P) {
            kk -= np - P;
            ++P;
          }
          panel_update(A, i, r, w, P, P + kk, s.R);
        }
      }
    }
    __syncthreads();
    {
      const int slot = stage == 1 ? kProfA1 : stage == 2 ? kProfA2 : stage == 3 ? kProfA3 : kProfB;
      prof_add(A, slot, clock64() - t_run);
      prof_add(A, stage == 1 ? kProfNA1 : stage == 2 ? kProfNA2 : stage == 3 ? kProfNA3 : kProfNB, 1);
    }
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(A.done + i, 1);
    }
  }
}

// g_t <- U_t^T g_t for every pending (row i, neighbor t > i) pair.
__global__ void __launch_bounds__(T) pending_kernel(SweepArgs A) {
  extern __shared__ double tmp[];
  const int i = blockIdx.x;
  const int w = A.width[i];
  if (w == 0) return;
  const int r = A.rank[i];
  const int64_t c0 = A.cl_ptr[i], c1 = A.cl_ptr[i + 1];
  double* G = A.fac + A.g_off[i];
  for (int64_t e = c0; e < c1; ++e) {
    const int t = A.cl_col[e];
    if (t <= i || !A.has_basis[t]) continue;
    const int bt = A.bsz[t];
    const double* U = A.basis + A.basis_off[t];
    double* g = G + static_cast<int64_t>(r + A.cl_roff[e]) * w;
    for (int idx = threadIdx.x; idx < bt * w; idx += T) tmp[idx] = g[idx];
    __syncthreads();
    for (int idx = threadIdx.x; idx < bt * w; idx += T) {
      const int a = idx / w, q = idx % w;
      double acc = 0.0;
      for (int c = 0; c < bt; ++c) acc += U[c * bt + a] * tmp[c * w + q];
      g[idx] = acc;
    }
    __syncthreads();
  }
}

__global__ void init_store_kernel(int64_t M, const int* bsz, const int64_t* a_row_ptr, const int* a_col,
                                  const int64_t* a_val_ptr, const double* a_values, const int64_t* sq_ptr,
                                  const int* sq_col, const int64_t* sq_slot, const int64_t* slot_off, double* store) {
  for (int64_t i = blockIdx.x; i < M; i += gridDim.x) {
    const int bi = bsz[i];
    for (int64_t k = a_row_ptr[i]; k < a_row_ptr[i + 1]; ++k) {
      const int j = a_col[k];
      if (j > i) break;
      const int64_t slot = find_slot(sq_ptr, sq_col, sq_slot, static_cast<int>(i), j);
      const int n = bi * bsz[j];
      const double* src = a_values + a_val_ptr[k];
      double* dst = store + slot_off[slot];
      for (int e = threadIdx.x; e < n; e += blockDim.x) dst[e] = src[e];
    }
  }
}

__global__ void remainder_kernel(RemainderArgs A) {
  for (int64_t s = blockIdx.x; s < A.M; s += gridDim.x) {
    const int rs = A.rank[s];
    if (rs == 0) continue;
    const int ga = A.next_block[s], ls = A.next_loc[s];
    for (int64_t e = A.sq_ptr[s]; e < A.sq_ptr[s + 1]; ++e) {
      const int t = A.sq_col[e];
      if (t > s) break;
      const int rt = A.rank[t];
      if (rt == 0) continue;
      const int bt = A.bsz[t];
      const int gb = A.next_block[t], lt = A.next_loc[t];
      const double* X = A.store + A.slot_off[A.sq_slot[e]];  // stored (s, t): bs x bt
      const int hi = ga > gb ? ga : gb, lo = ga > gb ? gb : ga;
      const int64_t slot = find_slot(A.nsq_ptr, A.nsq_col, A.nsq_slot, hi, lo);
      if (slot < 0) {
        if (threadIdx.x == 0) atomicCAS(A.err, 0, kErrPattern);
        continue;
      }
      double* Y = A.nstore + A.nslot_off[slot];
      const int Bh = A.nbsz[hi], Bl = A.nbsz[lo];
      for (int idx = threadIdx.x; idx < rs * rt; idx += blockDim.x) {
        const int a = idx / rt, c = idx % rt;
        const double v = X[static_cast<int64_t>(a) * bt + c];
        if (ga > gb) {
          Y[static_cast<int64_t>(ls + a) * Bl + lt + c] = v;
        } else if (ga < gb) {
          Y[static_cast<int64_t>(lt + c) * Bl + ls + a] = v;
        } else {
          Y[static_cast<int64_t>(ls + a) * Bh + lt + c] = v;
          if (s != t) Y[static_cast<int64_t>(lt + c) * Bh + ls + a] = v;
        }
      }
    }
  }
}

}  // namespace

int64_t sweep_smem_doubles(int bmax, int kcap) {
  return 4LL * bmax * bmax + static_cast<int64_t>(kcap) * bmax + 3LL * bmax + (bmax + 1) / 2 + 4;
}

int sweep_max_ctas_per_sm(size_t smem_bytes) {
  int n = 0;
  cudaError_t e = cudaFuncSetAttribute(sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem_bytes));
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, sweep_kernel, T, smem_bytes);
  if (e != cudaSuccess) {
    std::fprintf(stderr, "[ce] sweep occupancy query failed: %s\n", cudaGetErrorString(e));
    cudaGetLastError();
    return 0;
  }
  return n;
}

void launch_sweep(const SweepArgs& a, int grid, size_t smem_bytes, cudaStream_t s) {
  cudaFuncSetAttribute(sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_bytes));
  note_launch();
  sweep_kernel<<<grid, T, smem_bytes, s>>>(a);
}

void launch_pending_rotation(const SweepArgs& a, cudaStream_t s) {
  if (a.M <= 0) return;
  const size_t smem = static_cast<size_t>(a.bmax) * a.bmax * sizeof(double);
  cudaFuncSetAttribute(pending_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  note_launch();
  pending_kernel<<<static_cast<unsigned>(a.M), T, smem, s>>>(a);
}

void launch_init_store_from_matrix(int64_t M, const int* bsz, const int64_t* a_row_ptr, const int* a_col,
                                   const int64_t* a_val_ptr, const double* a_values, const int64_t* sq_ptr,
                                   const int* sq_col, const int64_t* sq_slot, const int64_t* slot_off,
                                   double* store, cudaStream_t s) {
  if (M <= 0) return;
  const unsigned grid = static_cast<unsigned>(M < 65535 * 8 ? M : 65535 * 8);
  note_launch();
  init_store_kernel<<<grid, 128, 0, s>>>(M, bsz, a_row_ptr, a_col, a_val_ptr, a_values, sq_ptr, sq_col, sq_slot,
                                         slot_off, store);
}

void launch_remainder(const RemainderArgs& a, cudaStream_t s) {
  if (a.M <= 0) return;
  const unsigned grid = static_cast<unsigned>(a.M < 65535 * 8 ? a.M : 65535 * 8);
  note_launch();
  remainder_kernel<<<grid, 128, 0, s>>>(a);
}

}  // namespace ceg
