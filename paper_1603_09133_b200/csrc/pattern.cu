// Symbolic pattern algebra on the device (SURVEY.md §8f-1 "device symbolic planner"):
//   pattern_square  (proj/src/pattern.cpp:64-86): row i of P^2 = union of the rows k in P(i);
//   coarsen_pattern (pattern.cpp:97-118): row g = the groups of every column of every member row.
// Both are "emit candidate (row, col) pairs, keep the distinct ones": every candidate becomes a
// 64-bit key row * ncols + col, a CUB radix sort orders them (row-major = sorted rows), a head
// flag per run of equal keys marks the distinct entries, and a scan / compaction produces the
// CSR.  The driver uses them where the planning is on the critical path with the device idle:
// the first level's plan (before any sweep) and the re-plan after a level whose groups died.
// The speculative plans that overlap a sweep stay on the host threads (the persistent sweep
// kernel owns every SM).  Dense deep levels (candidates > ~64M) use the host's bitset square.
#include <cub/cub.cuh>

#include <algorithm>

#include "kernels.hpp"
#include "pattern.hpp"

namespace ceg {
namespace {

constexpr int kPT = 256;
inline unsigned pblocks(int64_t n) { return static_cast<unsigned>(std::min<int64_t>((n + kPT - 1) / kPT, 148 * 64)); }

// candidates of row i: sum over k in row i of deg(k)   (square)
__global__ void sq_count_kernel(int64_t m, const int64_t* ptr, const int* col, int64_t* cnt) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < m; i += stride) {
    int64_t c = 0;
    for (int64_t e = ptr[i]; e < ptr[i + 1]; ++e) {
      const int k = col[e];
      c += ptr[k + 1] - ptr[k];
    }
    cnt[i] = c;
  }
}

__global__ void sq_emit_kernel(int64_t m, const int64_t* ptr, const int* col, const int64_t* at,
                               unsigned long long* keys) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < m; i += stride) {
    int64_t o = at[i];
    for (int64_t e = ptr[i]; e < ptr[i + 1]; ++e) {
      const int k = col[e];
      for (int64_t f = ptr[k]; f < ptr[k + 1]; ++f)
        keys[o++] = static_cast<unsigned long long>(i) * static_cast<unsigned long long>(m) + col[f];
    }
  }
}

// coarsen: every entry (b, j) -> (group(b), group(j)); group -1 (a dead group) drops the entry
__global__ void coarsen_emit_kernel(int64_t m, int64_t ng, const int64_t* ptr, const int* col, const int64_t* gof,
                                    unsigned long long* keys) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; b < m; b += stride) {
    const int64_t gb = gof[b];
    for (int64_t e = ptr[b]; e < ptr[b + 1]; ++e) {
      const int64_t gj = gof[col[e]];
      keys[e] = (gb < 0 || gj < 0) ? ~0ull
                                   : static_cast<unsigned long long>(gb) * static_cast<unsigned long long>(ng) +
                                         static_cast<unsigned long long>(gj);
    }
  }
}

__global__ void head_kernel(int64_t n, const unsigned long long* k, int* h) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride)
    h[i] = k[i] != ~0ull && (i == 0 || k[i] != k[i - 1]) ? 1 : 0;  // ~0: dropped entry
}

// distinct keys -> columns, and per-row counts
__global__ void compact_kernel(int64_t n, int64_t ncols, const unsigned long long* k, const int* h, const int* pos,
                               int* out_col, int* row_cnt) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride)
    if (h[i]) {
      out_col[pos[i]] = static_cast<int>(k[i] % static_cast<unsigned long long>(ncols));
      atomicAdd(row_cnt + k[i] / static_cast<unsigned long long>(ncols), 1);
    }
}

template <class T>
void excl_scan(const T* in, T* out, int64_t n, cudaStream_t s) {
  size_t tmp = 0;
  CE_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, static_cast<int>(n), s));
  DevArray<unsigned char> t(std::max<size_t>(tmp, 1));
  CE_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tmp, in, out, static_cast<int>(n), s));
}

// sort the candidate keys, keep the distinct ones -> CSR with `rows` rows over `ncols` columns
void keys_to_csr(DevArray<unsigned long long>& keys, int64_t n, int64_t rows, int64_t ncols, cudaStream_t s,
                 std::vector<int64_t>& out_ptr, std::vector<int>& out_col, bool has_dropped = false) {
  out_ptr.assign(static_cast<size_t>(rows + 1), 0);
  out_col.clear();
  if (n == 0) return;
  DevArray<unsigned long long> sorted(static_cast<size_t>(n));
  size_t tmp = 0;
  int bits = 1;
  while (bits < 64 && (static_cast<unsigned long long>(rows) * static_cast<unsigned long long>(ncols) >> bits) != 0) ++bits;
  if (has_dropped) bits = 64;  // the ~0 markers must sort last
  CE_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, keys.p, sorted.p, static_cast<int>(n), 0, bits, s));
  {
    DevArray<unsigned char> t(std::max<size_t>(tmp, 1));
    CE_CUDA(cub::DeviceRadixSort::SortKeys(t.p, tmp, keys.p, sorted.p, static_cast<int>(n), 0, bits, s));
  }
  DevArray<int> h(static_cast<size_t>(n)), pos(static_cast<size_t>(n));
  head_kernel<<<pblocks(n), kPT, 0, s>>>(n, sorted.p, h.p);
  note_launch();
  excl_scan(h.p, pos.p, n, s);
  int last_pos = 0, last_h = 0;
  CE_CUDA(cudaMemcpyAsync(&last_pos, pos.p + n - 1, sizeof(int), cudaMemcpyDeviceToHost, s));
  CE_CUDA(cudaMemcpyAsync(&last_h, h.p + n - 1, sizeof(int), cudaMemcpyDeviceToHost, s));
  CE_CUDA(cudaStreamSynchronize(s));
  const int64_t u = static_cast<int64_t>(last_pos) + last_h;
  DevArray<int> d_col(static_cast<size_t>(u)), cnt(static_cast<size_t>(rows));
  cnt.zero(s);
  compact_kernel<<<pblocks(n), kPT, 0, s>>>(n, ncols, sorted.p, h.p, pos.p, d_col.p, cnt.p);
  note_launch();
  std::vector<int> hc(static_cast<size_t>(rows));
  out_col.resize(static_cast<size_t>(u));
  CE_CUDA(cudaMemcpyAsync(out_col.data(), d_col.p, static_cast<size_t>(u) * sizeof(int), cudaMemcpyDeviceToHost, s));
  CE_CUDA(cudaMemcpyAsync(hc.data(), cnt.p, static_cast<size_t>(rows) * sizeof(int), cudaMemcpyDeviceToHost, s));
  CE_CUDA(cudaStreamSynchronize(s));
  for (int64_t i = 0; i < rows; ++i) out_ptr[static_cast<size_t>(i + 1)] = out_ptr[static_cast<size_t>(i)] + hc[static_cast<size_t>(i)];
}

}  // namespace

int64_t square_candidates(int64_t m, const std::vector<int64_t>& ptr, const std::vector<int>& col) {
  int64_t c = 0;
  for (int64_t i = 0; i < m; ++i)
    for (int64_t e = ptr[static_cast<size_t>(i)]; e < ptr[static_cast<size_t>(i + 1)]; ++e) {
      const int k = col[static_cast<size_t>(e)];
      c += ptr[static_cast<size_t>(k) + 1] - ptr[static_cast<size_t>(k)];
    }
  return c;
}

void device_square(int64_t m, const std::vector<int64_t>& ptr, const std::vector<int>& col, cudaStream_t s,
                   std::vector<int64_t>& sptr, std::vector<int>& scol) {
  DevArray<int64_t> d_ptr, cnt(static_cast<size_t>(std::max<int64_t>(m, 1))), at(static_cast<size_t>(std::max<int64_t>(m, 1)));
  DevArray<int> d_col;
  d_ptr.upload(ptr, s);
  d_col.upload(col, s);
  sq_count_kernel<<<pblocks(m), kPT, 0, s>>>(m, d_ptr.p, d_col.p, cnt.p);
  note_launch();
  excl_scan(cnt.p, at.p, m, s);
  int64_t last_at = 0, last_cnt = 0;
  CE_CUDA(cudaMemcpyAsync(&last_at, at.p + m - 1, sizeof last_at, cudaMemcpyDeviceToHost, s));
  CE_CUDA(cudaMemcpyAsync(&last_cnt, cnt.p + m - 1, sizeof last_cnt, cudaMemcpyDeviceToHost, s));
  CE_CUDA(cudaStreamSynchronize(s));
  const int64_t n = last_at + last_cnt;
  DevArray<unsigned long long> keys(static_cast<size_t>(std::max<int64_t>(n, 1)));
  sq_emit_kernel<<<pblocks(m), kPT, 0, s>>>(m, d_ptr.p, d_col.p, at.p, keys.p);
  note_launch();
  keys_to_csr(keys, n, m, m, s, sptr, scol);
}

void device_coarsen(int64_t m, const std::vector<int64_t>& ptr, const std::vector<int>& col, int64_t ng,
                    const std::vector<int64_t>& group_of, cudaStream_t s, std::vector<int64_t>& cptr,
                    std::vector<int>& ccol) {
  DevArray<int64_t> d_ptr, d_gof;
  DevArray<int> d_col;
  d_ptr.upload(ptr, s);
  d_col.upload(col, s);
  d_gof.upload(group_of, s);
  const int64_t n = ptr[static_cast<size_t>(m)];
  DevArray<unsigned long long> keys(static_cast<size_t>(std::max<int64_t>(n, 1)));
  coarsen_emit_kernel<<<pblocks(m), kPT, 0, s>>>(m, ng, d_ptr.p, d_col.p, d_gof.p, keys.p);
  note_launch();
  keys_to_csr(keys, n, ng, ng, s, cptr, ccol, true);
}

}  // namespace ceg
