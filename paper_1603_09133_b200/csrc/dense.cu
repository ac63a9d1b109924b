// Dense tail of the factorization (proj/src/factorization.cpp:419-436):
// densify the final remainder, blocked right-looking Cholesky (diagonal block
// in shared memory, panel TRSM and trailing SYRK across the grid), one shift
// retry decided by the host, then L^{-1} for the apply's two GEMVs.
#include "kernels.hpp"

namespace ceg {
namespace {

constexpr int NB = 64;

__device__ int64_t find_slot_d(const int64_t* sq_ptr, const int* sq_col, const int64_t* sq_slot, int row, int col) {
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

__global__ void densify_kernel(int64_t M, const int* bsz, const int64_t* offsets, const int64_t* sq_ptr,
                               const int* sq_col, const int64_t* sq_slot, const int64_t* slot_off,
                               const double* store, double* dense, int64_t n) {
  for (int64_t s = blockIdx.x; s < M; s += gridDim.x) {
    const int bs = bsz[s];
    for (int64_t e = sq_ptr[s]; e < sq_ptr[s + 1]; ++e) {
      const int t = sq_col[e];
      if (t > s) break;
      const int bt = bsz[t];
      const double* X = store + slot_off[sq_slot[e]];
      const int64_t os = offsets[s], ot = offsets[t];
      for (int idx = threadIdx.x; idx < bs * bt; idx += blockDim.x) {
        const int a = idx / bt, c = idx % bt;
        dense[(os + a) * n + ot + c] = X[idx];
        if (s != t) dense[(ot + c) * n + os + a] = X[idx];
      }
    }
  }
  (void)find_slot_d;
}

// Unblocked Cholesky of the nb x nb diagonal block at k0 (lower), in shared memory.
__global__ void potrf_diag_kernel(double* a, int64_t n, int64_t k0, int nb, int* fail) {
  __shared__ double P[NB * NB];
  __shared__ int bad;
  for (int idx = threadIdx.x; idx < nb * nb; idx += blockDim.x) P[idx] = a[(k0 + idx / nb) * n + k0 + idx % nb];
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int k = 0; k < nb; ++k) {
    if (threadIdx.x == 0) {
      const double d = P[k * nb + k];
      if (!(d > 0.0)) bad = 1;
      else P[k * nb + k] = sqrt(d);
    }
    __syncthreads();
    if (bad) break;
    const double dk = P[k * nb + k];
    for (int q = k + 1 + threadIdx.x; q < nb; q += blockDim.x) P[q * nb + k] /= dk;
    __syncthreads();
    const int m = nb - k - 1;
    for (int idx = threadIdx.x; idx < m * m; idx += blockDim.x) {
      const int q = k + 1 + idx / m, p = k + 1 + idx % m;
      if (p <= q) P[q * nb + p] -= P[q * nb + k] * P[p * nb + k];
    }
    __syncthreads();
  }
  if (bad) {
    if (threadIdx.x == 0) *fail = 1;
    return;
  }
  for (int idx = threadIdx.x; idx < nb * nb; idx += blockDim.x) {
    const int q = idx / nb, p = idx % nb;
    a[(k0 + q) * n + k0 + p] = p <= q ? P[idx] : 0.0;
  }
}

// Rows below the diagonal block: A[i, k0:k0+nb] <- A[i, k0:k0+nb] L_kk^{-T}; 64 rows per CTA.
__global__ void trsm_panel_kernel(double* a, int64_t n, int64_t k0, int nb) {
  __shared__ double L[NB * NB];
  for (int idx = threadIdx.x; idx < nb * nb; idx += blockDim.x) L[idx] = a[(k0 + idx / nb) * n + k0 + idx % nb];
  __syncthreads();
  const int64_t row = k0 + nb + static_cast<int64_t>(blockIdx.x) * 64 + threadIdx.x;
  if (threadIdx.x >= 64 || row >= n) return;
  double* x = a + row * n + k0;
  double y[NB];
  for (int q = 0; q < nb; ++q) {
    double acc = x[q];
    for (int p = 0; p < q; ++p) acc -= L[q * nb + p] * y[p];
    y[q] = acc / L[q * nb + q];
  }
  for (int q = 0; q < nb; ++q) x[q] = y[q];
}

// Trailing update A[i, j] -= sum_p A[i, k0+p] A[j, k0+p] for k0+nb <= j <= i; 32x32 tiles.
__global__ void syrk_kernel(double* a, int64_t n, int64_t k0, int nb) {
  const int64_t base = k0 + nb;
  const int64_t ti = base + static_cast<int64_t>(blockIdx.y) * 32, tj = base + static_cast<int64_t>(blockIdx.x) * 32;
  if (tj > ti) return;
  __shared__ double Ai[32][NB + 1];
  __shared__ double Aj[32][NB + 1];
  for (int idx = threadIdx.x; idx < 32 * nb; idx += blockDim.x) {
    const int rr = idx / nb, p = idx % nb;
    Ai[rr][p] = ti + rr < n ? a[(ti + rr) * n + k0 + p] : 0.0;
    Aj[rr][p] = tj + rr < n ? a[(tj + rr) * n + k0 + p] : 0.0;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < 32 * 32; idx += blockDim.x) {
    const int rr = idx / 32, cc = idx % 32;
    const int64_t gi = ti + rr, gj = tj + cc;
    if (gi >= n || gj >= n || gj > gi) continue;
    double acc = 0.0;
    for (int p = 0; p < nb; ++p) acc += Ai[rr][p] * Aj[cc][p];
    a[gi * n + gj] -= acc;
  }
}

__global__ void zero_upper_kernel(double* a, int64_t n) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n * n; k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = k / n, j = k % n;
    if (j > i) a[k] = 0.0;
  }
}

__global__ void add_shift_kernel(double* a, int64_t n, double shift) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n; k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    a[k * n + k] += shift;
}

__global__ void trace_kernel(const double* a, int64_t n, double* out) {
  __shared__ double red[256];
  double s = 0.0;
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x) s += a[k * n + k];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

// Linv = L^{-1}: CTA per 32-column block, row tiles of 32 solved in order.
__global__ void tri_inverse_kernel(const double* L, double* X, int64_t n) {
  const int64_t j0 = static_cast<int64_t>(blockIdx.x) * 32;
  __shared__ double acc[32][33];
  __shared__ double Lt[32][33];
  __shared__ double Xt[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 256 threads: ty 0..7
  for (int64_t q0 = j0; q0 < n; q0 += 32) {
    // acc = I_QJ - sum_{p in [j0, q0)} L[Q][p] X[p][J]
    for (int rr = ty; rr < 32; rr += 8) acc[rr][tx] = (q0 + rr == j0 + tx) ? 1.0 : 0.0;
    for (int64_t p0 = j0; p0 < q0; p0 += 32) {
      __syncthreads();
      for (int rr = ty; rr < 32; rr += 8) {
        Lt[rr][tx] = (q0 + rr < n) ? L[(q0 + rr) * n + p0 + tx] : 0.0;
        Xt[rr][tx] = (p0 + rr < n && j0 + tx < n) ? X[(p0 + rr) * n + j0 + tx] : 0.0;
      }
      __syncthreads();
      for (int rr = ty; rr < 32; rr += 8) {
        double s = 0.0;
        for (int k = 0; k < 32; ++k) s += Lt[rr][k] * Xt[k][tx];
        acc[rr][tx] -= s;
      }
    }
    __syncthreads();
    for (int rr = ty; rr < 32; rr += 8) Lt[rr][tx] = (q0 + rr < n && q0 + tx < n) ? L[(q0 + rr) * n + q0 + tx] : (rr == tx ? 1.0 : 0.0);
    __syncthreads();
    if (ty == 0) {
      // forward substitution within the diagonal tile, one column per lane
      for (int rr = 0; rr < 32; ++rr) {
        double s = acc[rr][tx];
        for (int k = 0; k < rr; ++k) s -= Lt[rr][k] * acc[k][tx];
        acc[rr][tx] = s / Lt[rr][rr];
      }
    }
    __syncthreads();
    for (int rr = ty; rr < 32; rr += 8)
      if (q0 + rr < n && j0 + tx < n) X[(q0 + rr) * n + j0 + tx] = acc[rr][tx];
  }
  // zero the strictly upper part of this column block
  for (int64_t rr = ty; rr < j0 + 32 && rr < n; rr += 8)
    if (j0 + tx < n && j0 + tx > rr) X[rr * n + j0 + tx] = 0.0;
}

}  // namespace

void launch_densify(int64_t M, const int* bsz, const int64_t* offsets, const int64_t* sq_ptr, const int* sq_col,
                    const int64_t* sq_slot, const int64_t* slot_off, const double* store, double* dense, int64_t n,
                    cudaStream_t s) {
  if (M <= 0) return;
  note_launch();
    densify_kernel<<<static_cast<unsigned>(M < 65535 ? M : 65535), 128, 0, s>>>(M, bsz, offsets, sq_ptr, sq_col, sq_slot,
                                                                              slot_off, store, dense, n);
}

void dense_cholesky(double* a, int64_t n, int* d_fail, cudaStream_t s) {
  for (int64_t k0 = 0; k0 < n; k0 += NB) {
    const int nb = static_cast<int>(n - k0 < NB ? n - k0 : NB);
    note_launch();
    potrf_diag_kernel<<<1, 256, 0, s>>>(a, n, k0, nb, d_fail);
    const int64_t rest = n - k0 - nb;
    if (rest > 0) {
      note_launch();
      trsm_panel_kernel<<<static_cast<unsigned>((rest + 63) / 64), 64, 0, s>>>(a, n, k0, nb);
      const unsigned t = static_cast<unsigned>((rest + 31) / 32);
      note_launch();
      syrk_kernel<<<dim3(t, t), 256, 0, s>>>(a, n, k0, nb);
    }
  }
  note_launch();
  zero_upper_kernel<<<1024, 256, 0, s>>>(a, n);
}

void dense_add_shift(double* a, int64_t n, double shift, cudaStream_t s) {
  note_launch();
  add_shift_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(a, n, shift);
}

void dense_trace(const double* a, int64_t n, double* d_out, cudaStream_t s) { trace_kernel<<<1, 256, 0, s>>>(a, n, d_out); }

void dense_tri_inverse(const double* L, double* Linv, int64_t n, cudaStream_t s) {
  if (n > 0) {
    note_launch();
    tri_inverse_kernel<<<static_cast<unsigned>((n + 31) / 32), 256, 0, s>>>(L, Linv, n);
  }
}

}  // namespace ceg
