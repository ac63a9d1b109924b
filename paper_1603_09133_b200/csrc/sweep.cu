// Level sweep kernels (sm_100a): batched compression + subrow elimination.
//
// Reference semantics (one row at a time, ascending):
//   LevelMatrix::compress_row      proj/src/level_matrix.cpp:33-82
//   compress_far_concat (JacobiSVD) proj/src/compression.cpp:20-61
//   LevelMatrix::eliminate_subrow  proj/src/level_matrix.cpp:84-178
//   level_sweep hot loop           proj/src/factorization.cpp:56-59
//
// B200 design: one persistent kernel per level.  Work items are taken from a
// global ticket in plan order; item 0 of row i compresses and eliminates the
// row (phase A, one CTA), items 1..T_i apply its Schur pair updates
// X_st -= g_s g_t^T in tiles spread over other CTAs (phase B, fat rows only).
// Row j's phase A waits until every row i < j of sq(j) has finished all its
// items (rows at block-graph distance >= 3 commute), so every
// block receives its updates in the reference order and no atomics touch data.
// The far-block concatenation F_i is never materialised: its transpose is
// streamed through shared memory in chunks into a Householder TSQR, the b x b
// triangle is diagonalised by parallel one-sided Jacobi (round-robin pairs, one
// warp per pair), and U is emitted in the canonical gauge (oracle/dense.hpp).
#include <cfloat>
#include <cstdio>

#include "kernels.hpp"

namespace ceg {
namespace {

constexpr int T = kSweepThreads;
constexpr int NW = T / 32;

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

__device__ __forceinline__ double gauge_weight(int k) {
  const double x = __dmul_rn(static_cast<double>(k + 1), 0.6180339887498949);
  return 1.0 + 0.5 * (x - floor(x));
}

// Deterministic block-wide sum; every thread receives the same value.
__device__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < NW; ++k) s += red[k];
  return s;
}

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

__device__ void set_error(int* err, int code, int level, int64_t row) {
  if (atomicCAS(err, 0, code) == 0) {
    err[1] = level;
    err[2] = static_cast<int>(row & 0x7fffffff);
    err[3] = static_cast<int>(row >> 31);
  }
}

// Structured Householder QR update [R; C] -> [R'; 0].  R: b x b column-major
// (R[k][j] at R[j*b+k]); C: K x b row-major.  LAPACK dlarfg conventions.
__device__ void tsqr_update(double* R, double* C, int K, int b, double* shr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k = 0; k < b; ++k) {
    if (warp == 0) {
      double s2 = 0.0;
      for (int m = lane; m < K; m += 32) {
        const double c = C[m * b + k];
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
        for (int m = lane; m < K; m += 32) C[m * b + k] *= scale;
      }
      if (lane == 0) shr[0] = tau;
    }
    __syncthreads();
    const double tau = shr[0];
    if (tau != 0.0) {
      for (int j = k + 1 + warp; j < b; j += NW) {
        double s = 0.0;
        for (int m = lane; m < K; m += 32) s += C[m * b + k] * C[m * b + j];
        s = warp_sum(s);
        const double tw = tau * (R[j * b + k] + s);
        __syncwarp();
        if (lane == 0) R[j * b + k] -= tw;
        for (int m = lane; m < K; m += 32) C[m * b + j] -= tw * C[m * b + k];
      }
    }
    __syncthreads();
  }
}

// One-sided Jacobi on the columns of R (b x b, column-major); V accumulates.
__device__ void jacobi(double* R, double* V, int b, int meff, int* any) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int idx = threadIdx.x; idx < b * b; idx += T) V[idx] = (idx / b == idx % b) ? 1.0 : 0.0;
  const double tol = sqrt(static_cast<double>(meff > 1 ? meff : 1)) * DBL_EPSILON;
  const int nb = b + (b & 1);
  for (int sweep = 0; sweep < 100; ++sweep) {
    if (threadIdx.x == 0) *any = 0;
    __syncthreads();
    for (int round = 0; round < nb - 1; ++round) {
      for (int pi = warp; pi < nb / 2; pi += NW) {
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
        for (int k = lane; k < b; k += 32) {
          const double x = cp[k], y = cq[k];
          al += x * x;
          be += y * y;
          ga += x * y;
        }
        al = warp_sum(al);
        be = warp_sum(be);
        ga = warp_sum(ga);
        if (al == 0.0 || be == 0.0) continue;
        if (!(fabs(ga) > tol * sqrt(al) * sqrt(be))) continue;
        const double zeta = (be - al) / (2.0 * ga);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / sqrt(1.0 + t * t);
        const double sn = cs * t;
        __syncwarp();
        for (int k = lane; k < b; k += 32) {
          const double x = cp[k], y = cq[k];
          cp[k] = cs * x - sn * y;
          cq[k] = sn * x + cs * y;
        }
        double* vp = V + p * b;
        double* vq = V + q * b;
        for (int k = lane; k < b; k += 32) {
          const double x = vp[k], y = vq[k];
          vp[k] = cs * x - sn * y;
          vq[k] = sn * x + cs * y;
        }
        if (lane == 0) *any = 1;
      }
      __syncthreads();
    }
    const int a = *any;
    __syncthreads();
    if (!a) break;
  }
}

// Canonical gauge (oracle/dense.cpp canonical_basis): U1 = sign-fixed leading
// singular vectors, U2 = trailing columns of the Householder QR of U1.
// V: column-major right singular vectors of R (unsorted), perm: sorted order.
// Writes U row-major into s.U.  Uses s.C (A, then Q) and s.R (reflectors).
__device__ __forceinline__ double gauge_weight2(int k, int j) {
  const double cj = __dadd_rn(0.6180339887498949, __dmul_rn(0.2071067811865475, static_cast<double>(j)));
  const double x = __dmul_rn(static_cast<double>(k + 1), cj);
  return 1.0 + 0.5 * (x - floor(x));
}

constexpr double kClusterTol = 1e-9;  // oracle/dense.hpp

__device__ void canonical_basis(const Buf& s, int b, int r, int nsig, double* shr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* A = s.C;   // b x r column-major
  double* Vh = s.R;  // reflectors, column-major
  __shared__ int cstart[512];  // cstart[k] = first index of k's cluster
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
  // one warp per cluster: singletons get the sign fix, clusters orth(U_c U_c^T G_c)
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
  // Q[:, r:] = H_0 ... H_{r-1} E_{r:} (column-major in C)
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
  (void)shr;
}

// Element (a, c) of X_ij (b_i x b_j) in the half-symmetric store.
__device__ __forceinline__ int64_t xidx(int a, int c, int bi, int bj, bool trans) {
  return trans ? static_cast<int64_t>(c) * bi + a : static_cast<int64_t>(a) * bj + c;
}

// Schur pair updates of row i for pairs [p_begin, p_end) of close(i) x close(i), ks <= kt.
__device__ void pair_updates(const SweepArgs& A, int i, int r, int w, int64_t p_begin, int64_t p_end) {
  const int64_t c0 = A.cl_ptr[i];
  const int nc = static_cast<int>(A.cl_ptr[i + 1] - c0);
  const double* G = A.fac + A.g_off[i];
  int ks = 0;
  int64_t idx = p_begin;
  while (ks < nc && idx >= nc - ks) {
    idx -= nc - ks;
    ++ks;
  }
  int kt = ks + static_cast<int>(idx);
  for (int64_t p = p_begin; p < p_end; ++p) {
    const int s = A.cl_col[c0 + ks], t = A.cl_col[c0 + kt];  // s <= t
    const int bs_ = A.bsz[s], bt = A.bsz[t];
    const int64_t slot = find_slot(A.sq_ptr, A.sq_col, A.sq_slot, t, s);
    if (slot < 0) {
      if (threadIdx.x == 0) set_error(A.err, kErrPattern, A.level, i);
      return;
    }
    double* X = A.store + A.slot_off[slot];  // stored (t, s): bt x bs
    const double* gs = G + static_cast<int64_t>(r + A.cl_roff[c0 + ks]) * w;
    const double* gt = G + static_cast<int64_t>(r + A.cl_roff[c0 + kt]) * w;
    for (int e = threadIdx.x; e < bt * bs_; e += T) {
      const int x = e / bs_, y = e % bs_;
      double acc = 0.0;
      for (int q = 0; q < w; ++q) acc += ldg(gt + static_cast<int64_t>(x) * w + q) * ldg(gs + static_cast<int64_t>(y) * w + q);
      X[e] = ldg(X + e) - acc;
    }
    if (++kt == nc) {
      ++ks;
      kt = ks;
    }
  }
}

// Phase A: compress_row(i) + eliminate_subrow(i) (+ inline pairs when the row has no tiles).
__device__ void phase_a(const SweepArgs& A, int i, const Buf& s, int ntiles) {
  __shared__ double shr[4];
  __shared__ double red[NW];
  __shared__ int sflag[4];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
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

  // ---- gather F^T chunk by chunk into the TSQR (compression.cpp:38-48) ----
  int fcols = 0, kfill = 0;
  for (int64_t e = p0; e < p1; ++e) {
    if (A.sq_kind[e] != 2) continue;
    const int j = A.sq_col[e];
    const int bj = A.bsz[j];
    const bool tr = j > i;
    const double* X = A.store + A.slot_off[A.sq_slot[e]];
    if (kfill + bj > A.kcap) {
      tsqr_update(s.R, s.C, kfill, b, shr);
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
      s.C[(kfill + c) * b + a] = v;
      if (v != 0.0) sflag[0] = 1;
    }
    __syncthreads();
    kfill += bj;
    fcols += bj;
  }
  if (kfill > 0) tsqr_update(s.R, s.C, kfill, b, shr);
  __syncthreads();
  const bool nonzero = sflag[0] != 0;
  const int meff = fcols < b ? fcols : b;

  // ---- rank decision + basis (compression.cpp:20-61) ----
  int r = 0;
  bool basis = false;
  int nsig = 0;
  if (fcols > 0) {
    bool need_svd;
    if (A.mode == 1) {
      r = A.fixed_rank < b ? A.fixed_rank : b;
      need_svd = nonzero && r < b;
    } else {
      need_svd = nonzero;
    }
    if (need_svd) {
      jacobi(s.R, s.V, b, meff, &sflag[1]);
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
      r = 0;  // all-zero fill (compression.cpp:44-47)
    }
  }
  // (fcols == 0: r = 0, identity basis, compression.cpp:26-30)

  // ---- rotate the row (level_matrix.cpp:51-76) ----
  if (basis) {
    canonical_basis(s, b, r, nsig, shr);
    double* Ug = A.basis + A.basis_off[i];
    for (int idx = tid; idx < b * b; idx += T) Ug[idx] = s.U[idx];
    // D <- sym(U^T (D U))
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
    for (int64_t e = p0; e < p1; ++e) {
      const int kind = A.sq_kind[e];
      if (kind == 0) continue;
      const int j = A.sq_col[e];
      const int bj = A.bsz[j];
      const bool tr = j > i;
      double* X = A.store + A.slot_off[A.sq_slot[e]];
      for (int idx = tid; idx < b * bj; idx += T) {
        const int a = idx / bj, c = idx % bj;
        s.C[idx] = ldg(X + xidx(a, c, b, bj, tr));
      }
      __syncthreads();
      for (int idx = tid; idx < b * bj; idx += T) {
        int a, c;
        if (tr) {
          c = idx / b;
          a = idx % b;
        } else {
          a = idx / bj;
          c = idx % bj;
        }
        double acc = 0.0;
        if (!(kind == 2 && a >= r))
          for (int k = 0; k < b; ++k) acc += s.U[k * b + a] * s.C[k * bj + c];
        X[xidx(a, c, b, bj, tr)] = acc;
      }
      __syncthreads();
    }
  } else if (r < b) {
    for (int64_t e = p0; e < p1; ++e) {
      if (A.sq_kind[e] != 2) continue;
      const int j = A.sq_col[e];
      const int bj = A.bsz[j];
      const bool tr = j > i;
      double* X = A.store + A.slot_off[A.sq_slot[e]];
      for (int idx = tid; idx < (b - r) * bj; idx += T) {
        const int a = r + idx / bj, c = idx % bj;
        X[xidx(a, c, b, bj, tr)] = 0.0;
      }
    }
    __syncthreads();
  }

  // ---- eliminate_subrow (level_matrix.cpp:84-178) ----
  const int w = b - r;
  if (w > 0) {
    double* P = s.R;      // w x w row-major
    double* Pbak = s.V;   // backup for the shift retry
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
    // TRSM: coupling and neighbor blocks, one right-hand side column per thread
    const int64_t c0 = A.cl_ptr[i];
    const int nc = static_cast<int>(A.cl_ptr[i + 1] - c0);
    const int csum = nc > 0 ? A.cl_roff[c0 + nc - 1] + A.bsz[A.cl_col[c0 + nc - 1]] : 0;
    double* G = A.fac + A.g_off[i];
    for (int rho = tid; rho < r + csum; rho += T) {
      double* y = G + static_cast<int64_t>(rho) * w;
      if (rho < r) {
        for (int q = 0; q < w; ++q) {
          double acc = s.D[(r + q) * b + rho];
          for (int p = 0; p < q; ++p) acc -= P[q * w + p] * y[p];
          y[q] = acc / P[q * w + q];
        }
      } else {
        const int off = rho - r;
        int lo = 0, hi = nc - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (A.cl_roff[c0 + mid] <= off) lo = mid;
          else hi = mid - 1;
        }
        const int t = A.cl_col[c0 + lo];
        const int bt = A.bsz[t];
        const int c = off - A.cl_roff[c0 + lo];
        const bool tr = t > i;
        const double* X = A.store + A.slot_off[A.cl_slot[c0 + lo]];
        for (int q = 0; q < w; ++q) {
          double acc = ldg(X + xidx(r + q, c, b, bt, tr));
          for (int p = 0; p < q; ++p) acc -= P[q * w + p] * y[p];
          y[q] = acc / P[q * w + q];
        }
      }
    }
    __syncthreads();
    // Schur update of the retained part (level_matrix.cpp:140-147)
    if (r > 0) {
      for (int idx = tid; idx < r * r; idx += T) {
        const int a = idx / r, c = idx % r;
        double acc = 0.0;
        for (int q = 0; q < w; ++q) acc += ldg(G + a * w + q) * ldg(G + c * w + q);
        s.D[a * b + c] -= acc;
      }
      for (int64_t idx = tid; idx < static_cast<int64_t>(r) * csum; idx += T) {
        const int a = static_cast<int>(idx / csum);
        const int off = static_cast<int>(idx % csum);
        int lo = 0, hi = nc - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (A.cl_roff[c0 + mid] <= off) lo = mid;
          else hi = mid - 1;
        }
        const int t = A.cl_col[c0 + lo];
        const int bt = A.bsz[t];
        const int c = off - A.cl_roff[c0 + lo];
        const bool tr = t > i;
        double* X = A.store + A.slot_off[A.cl_slot[c0 + lo]];
        const double* ga = G + static_cast<int64_t>(a) * w;
        const double* gt = G + static_cast<int64_t>(r + off) * w;
        double acc = 0.0;
        for (int q = 0; q < w; ++q) acc += ldg(ga + q) * ldg(gt + q);
        const int64_t xi = xidx(a, c, b, bt, tr);
        X[xi] = ldg(X + xi) - acc;
      }
    }
    __syncthreads();
    if (ntiles == 0) {
      pair_updates(A, i, r, w, 0, static_cast<int64_t>(nc) * (nc + 1) / 2);
      __syncthreads();
    }
    // eliminated rows/cols leave the level (level_matrix.cpp:165-171)
    for (int idx = tid; idx < b * b; idx += T) {
      const int a = idx / b, c = idx % b;
      if (a >= r || c >= r) s.D[idx] = 0.0;
    }
    for (int64_t e = p0; e < p1; ++e) {
      if (A.sq_kind[e] == 0) continue;
      const int j = A.sq_col[e];
      const int bj = A.bsz[j];
      const bool tr = j > i;
      double* X = A.store + A.slot_off[A.sq_slot[e]];
      for (int idx = tid; idx < w * bj; idx += T) {
        int a, c;
        if (tr) {
          c = idx / w;
          a = r + idx % w;
        } else {
          a = r + idx / bj;
          c = idx % bj;
        }
        X[xidx(a, c, b, bj, tr)] = 0.0;
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
}

__global__ void __launch_bounds__(T) sweep_kernel(SweepArgs A) {
  extern __shared__ double smem_dyn[];
  double* base = A.use_global_scratch ? A.scratch + static_cast<int64_t>(blockIdx.x) * A.scratch_per_cta : smem_dyn;
  const Buf s = carve(base, A.bmax, A.kcap);
  __shared__ long long s_item;
  __shared__ int s_stop;
  for (;;) {
    if (threadIdx.x == 0) {
      s_stop = *reinterpret_cast<volatile int*>(A.err) != 0;
      s_item = s_stop ? 0 : static_cast<long long>(atomicAdd(A.ticket, 1ULL));
    }
    __syncthreads();
    if (s_stop) break;
    const long long item = s_item;
    if (item >= A.n_items) break;
    // row owning the item: largest i with item_start[i] <= item
    int64_t lo = 0, hi = A.M - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (A.item_start[mid] <= item) lo = mid;
      else hi = mid - 1;
    }
    const int i = static_cast<int>(lo);
    const int part = static_cast<int>(item - A.item_start[i]);
    const int ntiles = static_cast<int>(A.item_start[i + 1] - A.item_start[i]) - 1;
    if (threadIdx.x == 0) {
      if (part == 0) {
        for (int64_t e = A.sq_ptr[i]; e < A.sq_ptr[i + 1]; ++e) {
          const int j = A.sq_col[e];
          if (j >= i) break;
          const int target = static_cast<int>(A.item_start[j + 1] - A.item_start[j]);
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
        while (ld_acquire(A.done + i) < 1) {
          if (*reinterpret_cast<volatile int*>(A.err) != 0) {
            s_stop = 1;
            break;
          }
          __nanosleep(64);
        }
      }
      __threadfence();
    }
    __syncthreads();
    if (s_stop) break;
    if (part == 0) {
      phase_a(A, i, s, ntiles);
    } else {
      const int r = __ldcg(A.rank + i), w = __ldcg(A.width + i);
      if (w > 0) {
        const int nc = static_cast<int>(A.cl_ptr[i + 1] - A.cl_ptr[i]);
        const int64_t P = static_cast<int64_t>(nc) * (nc + 1) / 2;
        const int64_t pb = P * (part - 1) / ntiles, pe = P * part / ntiles;
        pair_updates(A, i, r, w, pb, pe);
      }
    }
    __syncthreads();
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
    const int bs_ = A.bsz[s];
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
  cudaFuncSetAttribute(sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_bytes));
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, sweep_kernel, T, smem_bytes);
  return n;
}

void launch_sweep(const SweepArgs& a, int grid, size_t smem_bytes, cudaStream_t s) {
  cudaFuncSetAttribute(sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_bytes));
  note_launch();
  sweep_kernel<<<grid, T, smem_bytes, s>>>(a);
}

void launch_pending_rotation(const SweepArgs& a, cudaStream_t s) {
  const size_t smem = static_cast<size_t>(a.bmax) * a.bmax * sizeof(double);
  cudaFuncSetAttribute(pending_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (a.M > 0) {
    note_launch();
    pending_kernel<<<static_cast<unsigned>(a.M), T, smem, s>>>(a);
  }
}

void launch_init_store_from_matrix(int64_t M, const int* bsz, const int64_t* a_row_ptr, const int* a_col,
                                   const int64_t* a_val_ptr, const double* a_values, const int64_t* sq_ptr,
                                   const int* sq_col, const int64_t* sq_slot, const int64_t* slot_off,
                                   double* store, cudaStream_t s) {
  const unsigned grid = static_cast<unsigned>(M < 65535 * 8 ? M : 65535 * 8);
  if (M > 0)
    note_launch();
    init_store_kernel<<<grid, 128, 0, s>>>(M, bsz, a_row_ptr, a_col, a_val_ptr, a_values, sq_ptr, sq_col, sq_slot,
                                           slot_off, store);
}

void launch_remainder(const RemainderArgs& a, cudaStream_t s) {
  const unsigned grid = static_cast<unsigned>(a.M < 65535 * 8 ? a.M : 65535 * 8);
  if (a.M > 0) {
    note_launch();
    remainder_kernel<<<grid, 128, 0, s>>>(a);
  }
}

}  // namespace ceg
