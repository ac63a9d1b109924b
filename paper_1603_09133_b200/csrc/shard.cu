// Device side of the subdomain-sharded factorization: the
// exchange buffers between ranks are packed / unpacked here, and the rows another rank swept
// are marked complete so this rank's interface phase does not wait for them.
#include <algorithm>

#include "kernels.hpp"

namespace ceg {
namespace {

constexpr int kShardThreads = 256;

// Segment k = rows x cols doubles at src + off[k] with leading dimension ld[k] (row-major);
// its packed image is contiguous at buf + boff[k].  to_buf: gather (pack), else scatter.
__global__ void __launch_bounds__(kShardThreads) segments_kernel(double* base, double* buf, const int64_t* off,
                                                                const int* rows, const int* cols, const int* ld,
                                                                const int64_t* boff, int64_t nseg, int to_buf) {
  for (int64_t k = blockIdx.x; k < nseg; k += gridDim.x) {
    const int r = rows[k], c = cols[k], l = ld[k];
    double* a = base + off[k];
    double* b = buf + boff[k];
    for (int idx = threadIdx.x; idx < r * c; idx += blockDim.x) {
      const int i = idx / c, j = idx - i * c;
      if (to_buf) b[idx] = a[static_cast<int64_t>(i) * l + j];
      else a[static_cast<int64_t>(i) * l + j] = b[idx];
    }
  }
}

// Per-row integers of a level (rank, width, has_basis, fcols, nsig) <-> 5 doubles per row.
__global__ void row_ints_kernel(const int* rows, int64_t n, int* rank, int* width, unsigned char* has_basis,
                                int* fcols, int* nsig, double* buf, int to_buf) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int i = rows[k];
    double* b = buf + 5 * k;
    if (to_buf) {
      b[0] = rank[i];
      b[1] = width[i];
      b[2] = has_basis[i];
      b[3] = fcols[i];
      b[4] = nsig[i];
    } else {
      rank[i] = static_cast<int>(b[0]);
      width[i] = static_cast<int>(b[1]);
      has_basis[i] = static_cast<unsigned char>(b[2]);
      fcols[i] = static_cast<int>(b[3]);
      nsig[i] = static_cast<int>(b[4]);
    }
  }
}

// Rows swept by another rank count as finished: their completion counters take the values
// the sweep's waits test for (sweep_body.cuh: done >= target, panel counters >= panels).
__global__ void precomplete_kernel(const int* rows, int64_t n, const int* target, const int64_t* pan_ptr, int* done,
                                   int* pdone, int* bready) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int i = rows[k];
    done[i] = target[i];
    bready[i] = 1;
    const int np = static_cast<int>(pan_ptr[i + 1] - pan_ptr[i]) - 1;
    for (int64_t p = pan_ptr[i]; p < pan_ptr[i + 1]; ++p) pdone[p] = np;
  }
}

}  // namespace

void launch_segments(double* base, double* buf, const int64_t* off, const int* rows, const int* cols, const int* ld,
                     const int64_t* boff, int64_t nseg, bool to_buf, cudaStream_t s) {
  if (nseg <= 0) return;
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>(nseg, 148 * 16));
  segments_kernel<<<grid, kShardThreads, 0, s>>>(base, buf, off, rows, cols, ld, boff, nseg, to_buf ? 1 : 0);
  note_launch();
}

void launch_row_ints(const int* rows, int64_t n, int* rank, int* width, unsigned char* has_basis, int* fcols, int* nsig,
                     double* buf, bool to_buf, cudaStream_t s) {
  if (n <= 0) return;
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 148 * 8));
  row_ints_kernel<<<grid, 256, 0, s>>>(rows, n, rank, width, has_basis, fcols, nsig, buf, to_buf ? 1 : 0);
  note_launch();
}

void launch_precomplete(const int* rows, int64_t n, const int* target, const int64_t* pan_ptr, int* done, int* pdone,
                        int* bready, cudaStream_t s) {
  if (n <= 0) return;
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 148 * 8));
  precomplete_kernel<<<grid, 256, 0, s>>>(rows, n, target, pan_ptr, done, pdone, bready);
  note_launch();
}

}  // namespace ceg
