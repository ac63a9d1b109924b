// Krylov building blocks on the device: block-sparse matvec (replaces
// BlockSparseMatrix::matvec, proj/src/block_matrix.cpp:92-105), deterministic
// two-stage dot products, and the fused PCG vector updates.
#include <atomic>

#include "kernels.hpp"

namespace ceg {
namespace {

constexpr int kDotBlocks = 592;  // 4 x 148 SMs
constexpr int kDotThreads = 256;

// One thread per scalar row; the row's block row is streamed block by block.
__global__ void bsr_matvec_kernel(int64_t n, const int64_t* row_of, const int64_t* offsets, const int* bsz,
                                  const int64_t* row_ptr, const int* col_idx, const int64_t* val_ptr,
                                  const double* values, const double* x, double* y) {
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < n;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = row_of[p];
    const int64_t a = p - offsets[i];
    double acc = 0.0;
    for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
      const int j = col_idx[k];
      const int bj = bsz[j];
      const double* blk = values + val_ptr[k] + a * bj;
      const double* xj = x + offsets[j];
      for (int c = 0; c < bj; ++c) acc += blk[c] * xj[c];
    }
    y[p] = acc;
  }
}

__global__ void dot_kernel(const double* x, const double* y, int64_t n, double* partial) {
  __shared__ double red[kDotThreads / 32];
  double s = 0.0;
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    s += x[k] * y[k];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < kDotThreads / 32; ++k) t += red[k];
    partial[blockIdx.x] = t;
  }
}

__global__ void sum_kernel(const double* partial, int np, double* out) {
  __shared__ double red[1024];
  double s = 0.0;
  for (int k = threadIdx.x; k < np; k += blockDim.x) s += partial[k];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

// y += sign * (num / den) * x
__global__ void axpy_kernel(double* y, const double* x, const double* num, const double* den, double sign, int64_t n) {
  const double alpha = sign * (*num / *den);
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    y[k] += alpha * x[k];
}

// p = z + (rz_new / rz_old) p
__global__ void update_p_kernel(double* p, const double* z, const double* rz_new, const double* rz_old, int64_t n) {
  const double beta = *rz_new / *rz_old;
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    p[k] = z[k] + beta * p[k];
}

__global__ void copy_kernel(double* dst, const double* src, int64_t n) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[k] = src[k];
}

// MINRES vector step (minres.cpp:57-89), IEEE operations in the reference's order (no
// contraction): out = (x - a y - c z) / g, with y / z optional (null = term absent).
__global__ void lincomb_kernel(double* out, const double* x, const double* y, double a, const double* z, double c,
                               double g, int64_t n) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double v = x[k];
    if (y) v = __dsub_rn(v, __dmul_rn(a, y[k]));
    if (z) v = __dsub_rn(v, __dmul_rn(c, z[k]));
    out[k] = g == 1.0 ? v : __ddiv_rn(v, g);
  }
}

// out = s x  /  out += s x (accumulate), single-rounded products as in the reference
__global__ void scale_kernel(double* out, double s, const double* x, int accumulate, int64_t n) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[k] = accumulate ? __dadd_rn(out[k], __dmul_rn(s, x[k])) : __dmul_rn(s, x[k]);
}

unsigned vec_grid(int64_t n) {
  const int64_t g = (n + 255) / 256;
  return static_cast<unsigned>(g < 148 * 16 ? (g > 0 ? g : 1) : 148 * 16);
}

std::atomic<int64_t> g_launches{0};

}  // namespace

void note_launch(int64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
int64_t launch_count() { return g_launches.load(); }

void launch_bsr_matvec(int64_t n, const int64_t* row_of, const int64_t* offsets, const int* bsz,
                       const int64_t* row_ptr, const int* col_idx, const int64_t* val_ptr, const double* values,
                       const double* x, double* y, cudaStream_t s) {
  note_launch();
  bsr_matvec_kernel<<<vec_grid(n), 256, 0, s>>>(n, row_of, offsets, bsz, row_ptr, col_idx, val_ptr, values, x, y);
}

int dot_partials_capacity() { return kDotBlocks; }

int launch_dot(const double* x, const double* y, int64_t n, double* d_partial, cudaStream_t s) {
  int64_t g = (n + kDotThreads - 1) / kDotThreads;
  if (g > kDotBlocks) g = kDotBlocks;
  if (g < 1) g = 1;
  note_launch();
  dot_kernel<<<static_cast<unsigned>(g), kDotThreads, 0, s>>>(x, y, n, d_partial);
  return static_cast<int>(g);
}

void launch_sum_partials(const double* partial, int np, double* out, cudaStream_t s) {
  note_launch();
  sum_kernel<<<1, 1024, 0, s>>>(partial, np, out);
}

void launch_axpy(double* y, const double* x, const double* num, const double* den, double sign, int64_t n,
                 cudaStream_t s) {
  note_launch();
  axpy_kernel<<<vec_grid(n), 256, 0, s>>>(y, x, num, den, sign, n);
}

void launch_pcg_update_p(double* p, const double* z, const double* rz_new, const double* rz_old, int64_t n,
                         cudaStream_t s) {
  note_launch();
  update_p_kernel<<<vec_grid(n), 256, 0, s>>>(p, z, rz_new, rz_old, n);
}

void launch_lincomb(double* out, const double* x, const double* y, double a, const double* z, double c, double g,
                    int64_t n, cudaStream_t s) {
  note_launch();
  lincomb_kernel<<<vec_grid(n), 256, 0, s>>>(out, x, y, a, z, c, g, n);
}

void launch_scale(double* out, double sc, const double* x, bool accumulate, int64_t n, cudaStream_t s) {
  note_launch();
  scale_kernel<<<vec_grid(n), 256, 0, s>>>(out, sc, x, accumulate ? 1 : 0, n);
}

void launch_copy(double* dst, const double* src, int64_t n, cudaStream_t s) {
  note_launch();
  copy_kernel<<<vec_grid(n), 256, 0, s>>>(dst, src, n);
}

}  // namespace ceg
