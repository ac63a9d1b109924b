// Device half of CEFactorization::validate (proj/src/factorization.cpp:272-334), run inside
// ce_factorize like the reference (factorization.cpp:459): per level, every stored basis U must
// satisfy max|U^T U - I| <= 1e-12 (:294-303) and every pivot factor must be lower triangular
// (:307-310).  The structural invariants (telescoping dimensions, gather lists partitioning the
// level, width + retained = block size, ascending neighbour lists) are checked on the host by
// the driver from its own plan arrays.
#include "kernels.hpp"

namespace ceg {
namespace {

constexpr int kValThreads = 128;

// One CTA per block row.  out[0] = max orthogonality error (non-negative double as its bit
// pattern, so integer atomicMax orders it), out[1] = nonzero entries above the pivot
// diagonal, out[2] = smallest block index that violates either rule (tol).
__global__ void __launch_bounds__(kValThreads) validate_level_kernel(
    int64_t M, const int* __restrict__ bsz, const unsigned char* __restrict__ has_basis,
    const double* __restrict__ basis, const int64_t* __restrict__ basis_off, const int* __restrict__ width,
    const double* __restrict__ fac, const int64_t* __restrict__ chol_off, double tol, unsigned long long* out) {
  __shared__ double red[kValThreads];
  __shared__ unsigned long long nup[kValThreads];
  const int64_t blk = blockIdx.x;
  if (blk >= M) return;
  const int b = bsz[blk];
  double err = 0.0;
  if (has_basis[blk]) {
    const double* U = basis + basis_off[blk];  // b x b row-major
    // (p, q) over the upper triangle of U^T U, one pair per thread step
    const int pairs = b * (b + 1) / 2;
    for (int k = threadIdx.x; k < pairs; k += blockDim.x) {
      int p = 0, rem = k;
      while (rem >= b - p) {
        rem -= b - p;
        ++p;
      }
      const int q = p + rem;
      double s = 0.0;
      for (int r = 0; r < b; ++r) s = fma(U[r * b + p], U[r * b + q], s);
      err = fmax(err, fabs(s - (p == q ? 1.0 : 0.0)));
    }
  }
  unsigned long long up = 0;
  const int w = width[blk];
  if (w > 1) {
    const double* Lc = fac + chol_off[blk];  // w x w row-major
    for (int k = threadIdx.x; k < w * w; k += blockDim.x)
      if (k % w > k / w && Lc[k] != 0.0) ++up;
  }
  red[threadIdx.x] = err;
  nup[threadIdx.x] = up;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + o]);
      nup[threadIdx.x] += nup[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double e = red[0];
    atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(e)));
    if (nup[0]) atomicAdd(out + 1, nup[0]);
    if (!(e <= tol) || nup[0]) atomicMin(out + 2, static_cast<unsigned long long>(blk));
  }
}

}  // namespace

void launch_validate_level(int64_t M, const int* bsz, const unsigned char* has_basis, const double* basis,
                           const int64_t* basis_off, const int* width, const double* fac, const int64_t* chol_off,
                           double tol, unsigned long long* d_out, cudaStream_t s) {
  if (M <= 0) return;
  validate_level_kernel<<<static_cast<unsigned>(M), kValThreads, 0, s>>>(M, bsz, has_basis, basis, basis_off, width, fac,
                                                                        chol_off, tol, d_out);
  note_launch();
}

}  // namespace ceg
