// BlockSparseMatrix::from_triplets on the device (proj/src/block_matrix.cpp:48-90; SURVEY.md
// §8f-2 "device problem assembly / CSB construction").  The reference accumulates the triplets
// in a std::map keyed by scalar position (duplicates summed in input order), optionally mirrors
// the lower triangle, checks symmetry to 1e-12 max|a|, inserts every touched block
// symmetrically plus the full diagonal, and writes each entry into its dense row-major block.
// Here:
//   expand    every triplet (and, for MirrorMode::Lower, its mirror) -> 64-bit key r*n + c,
//             entry 2k / 2k+1 = triplet k / its mirror, so a stable sort keeps input order;
//   sort      cub::DeviceRadixSort (stable) on the keys, values carried along;
//   reduce    one thread per run of equal keys sums it left to right from 0.0 -- the map's
//             `+=` order, so the result is bit-identical to the reference's;
//   check     symmetry (binary search of the transposed key), index range;
//   pattern   block keys of every entry and its transpose + the diagonal -> sort -> unique;
//   scatter   every entry into its block (val_ptr prefix of b_i b_j).
// The host receives only the block structure (for the planner) and error reports.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>

#include "assemble.hpp"
#include "kernels.hpp"

namespace ceg {
namespace {

constexpr int kAsmThreads = 256;
inline unsigned blocks_for(int64_t n) { return static_cast<unsigned>(std::min<int64_t>((n + kAsmThreads - 1) / kAsmThreads, 148 * 64)); }

__global__ void expand_kernel(int64_t nnz, int64_t n, const int64_t* rows, const int64_t* cols, const double* vals,
                              int mirror, unsigned long long* keys, double* v, unsigned long long* bad) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < nnz; k += stride) {
    const int64_t r = rows[k], c = cols[k];
    const double x = vals[k];
    const bool ok = r >= 0 && r < n && c >= 0 && c < n;
    if (!ok) atomicMin(bad, static_cast<unsigned long long>(k));
    const unsigned long long none = ~0ull;
    const int64_t e = mirror ? 2 * k : k;
    keys[e] = ok ? static_cast<unsigned long long>(r) * n + c : none;
    v[e] = x;
    if (mirror) {
      keys[e + 1] = (ok && r != c) ? static_cast<unsigned long long>(c) * n + r : none;
      v[e + 1] = x;
    }
  }
}

__global__ void absmax_kernel(int64_t nnz, const double* vals, unsigned long long* out) {
  double m = 0.0;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < nnz; k += stride)
    m = fmax(m, fabs(vals[k]));
  atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(m)));
}

// heads[i] = 1 where a run of equal keys starts (and the key is a real entry)
__global__ void heads_kernel(int64_t e, const unsigned long long* keys, int* heads) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < e; i += stride)
    heads[i] = keys[i] != ~0ull && (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

// run u starts at start[u] (exclusive scan position of its head): sum left to right from 0.0
__global__ void run_sum_kernel(int64_t e, const unsigned long long* keys, const double* v, const int* heads,
                               const int* pos, unsigned long long* ukeys, double* usum) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < e; i += stride) {
    if (!heads[i]) continue;
    const unsigned long long key = keys[i];
    double s = 0.0;
    for (int64_t j = i; j < e && keys[j] == key; ++j) s += v[j];
    ukeys[pos[i]] = key;
    usum[pos[i]] = s;
  }
}

__device__ int64_t find_key(const unsigned long long* k, int64_t n, unsigned long long x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) / 2;
    if (k[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo < n && k[lo] == x ? lo : -1;
}

__device__ int64_t block_of(const int64_t* offsets, int64_t m, int64_t i) {
  int64_t lo = 0, hi = m;  // largest b with offsets[b] <= i
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) / 2;
    if (offsets[mid] <= i) lo = mid;
    else hi = mid;
  }
  return lo;
}

// symmetry (MirrorMode::None): |a(r,c) - a(c,r)| > tol -> smallest offending position
__global__ void symmetry_kernel(int64_t u, int64_t n, const unsigned long long* ukeys, const double* usum, double tol,
                                unsigned long long* bad) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < u; i += stride) {
    const unsigned long long key = ukeys[i];
    const unsigned long long r = key / n, c = key % n;
    const int64_t t = find_key(ukeys, u, c * n + r);
    const double vt = t >= 0 ? usum[t] : 0.0;
    if (fabs(usum[i] - vt) > tol) atomicMin(bad, static_cast<unsigned long long>(i));
  }
}

// block keys: every entry's block and its transpose, then the diagonal blocks
__global__ void block_keys_kernel(int64_t u, int64_t n, int64_t m, const unsigned long long* ukeys,
                                  const int64_t* offsets, unsigned long long* bkeys) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < u + m; i += stride) {
    if (i >= u) {
      const unsigned long long d = static_cast<unsigned long long>(i - u);
      bkeys[2 * u + (i - u)] = d * m + d;
      continue;
    }
    const unsigned long long key = ukeys[i];
    const int64_t br = block_of(offsets, m, static_cast<int64_t>(key / n));
    const int64_t bc = block_of(offsets, m, static_cast<int64_t>(key % n));
    bkeys[2 * i] = static_cast<unsigned long long>(br) * m + bc;
    bkeys[2 * i + 1] = static_cast<unsigned long long>(bc) * m + br;
  }
}

__global__ void block_heads_kernel(int64_t e, const unsigned long long* k, int* heads) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < e; i += stride)
    heads[i] = (i == 0 || k[i] != k[i - 1]) ? 1 : 0;
}

__global__ void block_compact_kernel(int64_t e, const unsigned long long* k, const int* heads, const int* pos,
                                     unsigned long long* ub) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < e; i += stride)
    if (heads[i]) ub[pos[i]] = k[i];
}

// per block (slot): column, size b_i * b_j; row counts
__global__ void block_meta_kernel(int64_t nb, int64_t m, const unsigned long long* ub, const int64_t* offsets,
                                  int* col, int64_t* bytes, int* row_cnt) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; s < nb; s += stride) {
    const int64_t br = static_cast<int64_t>(ub[s] / m), bc = static_cast<int64_t>(ub[s] % m);
    col[s] = static_cast<int>(bc);
    bytes[s] = (offsets[br + 1] - offsets[br]) * (offsets[bc + 1] - offsets[bc]);
    atomicAdd(row_cnt + br, 1);
  }
}

__global__ void scatter_kernel(int64_t u, int64_t n, int64_t m, const unsigned long long* ukeys, const double* usum,
                               const int64_t* offsets, const unsigned long long* ub, int64_t nb, const int64_t* val_ptr,
                               double* values) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < u; i += stride) {
    const int64_t r = static_cast<int64_t>(ukeys[i] / n), c = static_cast<int64_t>(ukeys[i] % n);
    const int64_t br = block_of(offsets, m, r), bc = block_of(offsets, m, c);
    const int64_t slot = find_key(ub, nb, static_cast<unsigned long long>(br) * m + bc);
    const int64_t bcs = offsets[bc + 1] - offsets[bc];
    values[val_ptr[slot] + (r - offsets[br]) * bcs + (c - offsets[bc])] = usum[i];
  }
}

template <class T>
void exclusive_scan(const T* in, T* out, int64_t n, cudaStream_t s) {
  size_t tmp = 0;
  CE_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, static_cast<int>(n), s));
  DevArray<unsigned char> t(std::max<size_t>(tmp, 1));
  CE_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tmp, in, out, static_cast<int>(n), s));
}

void radix_sort(DevArray<unsigned long long>& keys, DevArray<double>* vals, int64_t n, cudaStream_t s) {
  DevArray<unsigned long long> k2(static_cast<size_t>(std::max<int64_t>(n, 1)));
  DevArray<double> v2;
  if (vals) v2.alloc(static_cast<size_t>(std::max<int64_t>(n, 1)));
  size_t tmp = 0;
  if (vals)
    CE_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, keys.p, k2.p, vals->p, v2.p, static_cast<int>(n), 0, 64, s));
  else
    CE_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, keys.p, k2.p, static_cast<int>(n), 0, 64, s));
  DevArray<unsigned char> t(std::max<size_t>(tmp, 1));
  if (vals)
    CE_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tmp, keys.p, k2.p, vals->p, v2.p, static_cast<int>(n), 0, 64, s));
  else
    CE_CUDA(cub::DeviceRadixSort::SortKeys(t.p, tmp, keys.p, k2.p, static_cast<int>(n), 0, 64, s));
  keys = std::move(k2);
  if (vals) *vals = std::move(v2);
}

int64_t read_int_at(const int* p, int64_t i, cudaStream_t s) {
  int v = 0;
  CE_CUDA(cudaMemcpyAsync(&v, p + i, sizeof v, cudaMemcpyDeviceToHost, s));
  CE_CUDA(cudaStreamSynchronize(s));
  return v;
}

}  // namespace

AssembleResult assemble_from_triplets(int64_t n, int64_t nnz, const int64_t* d_rows, const int64_t* d_cols,
                                      const double* d_vals, int64_t m, const int64_t* d_offsets, bool mirror,
                                      cudaStream_t s) {
  AssembleResult R;
  const int64_t e = mirror ? 2 * nnz : nnz;
  DevArray<unsigned long long> keys(static_cast<size_t>(std::max<int64_t>(e, 1)));
  DevArray<double> v(static_cast<size_t>(std::max<int64_t>(e, 1)));
  DevArray<unsigned long long> flags(2);  // [0] first bad triplet, [1] max |a| bits
  const unsigned long long init[2] = {~0ull, 0ull};
  CE_CUDA(cudaMemcpyAsync(flags.p, init, sizeof init, cudaMemcpyHostToDevice, s));
  if (nnz > 0) {
    expand_kernel<<<blocks_for(nnz), kAsmThreads, 0, s>>>(nnz, n, d_rows, d_cols, d_vals, mirror ? 1 : 0, keys.p, v.p,
                                                          flags.p);
    absmax_kernel<<<blocks_for(nnz), kAsmThreads, 0, s>>>(nnz, d_vals, flags.p + 1);
    note_launch(2);
  }
  unsigned long long hf[2];
  CE_CUDA(cudaMemcpyAsync(hf, flags.p, sizeof hf, cudaMemcpyDeviceToHost, s));
  CE_CUDA(cudaStreamSynchronize(s));
  if (hf[0] != ~0ull) {
    R.error = "triplet index outside matrix dimension";
    return R;
  }
  double maxabs = 0.0;
  std::memcpy(&maxabs, &hf[1], sizeof maxabs);
  if (e > 0) radix_sort(keys, &v, e, s);
  // runs of equal keys -> unique entries, summed in input order
  DevArray<int> heads(static_cast<size_t>(std::max<int64_t>(e, 1))), pos(static_cast<size_t>(std::max<int64_t>(e, 1)));
  int64_t u = 0;
  if (e > 0) {
    heads_kernel<<<blocks_for(e), kAsmThreads, 0, s>>>(e, keys.p, heads.p);
    note_launch();
    exclusive_scan(heads.p, pos.p, e, s);
    u = read_int_at(pos.p, e - 1, s) + read_int_at(heads.p, e - 1, s);
  }
  DevArray<unsigned long long> ukeys(static_cast<size_t>(std::max<int64_t>(u, 1)));
  DevArray<double> usum(static_cast<size_t>(std::max<int64_t>(u, 1)));
  if (e > 0) {
    run_sum_kernel<<<blocks_for(e), kAsmThreads, 0, s>>>(e, keys.p, v.p, heads.p, pos.p, ukeys.p, usum.p);
    note_launch();
  }
  if (!mirror && u > 0) {  // block_matrix.cpp:62-73
    const double tol = 1e-12 * std::max(maxabs, 1e-300);
    CE_CUDA(cudaMemcpyAsync(flags.p, init, sizeof(unsigned long long), cudaMemcpyHostToDevice, s));
    symmetry_kernel<<<blocks_for(u), kAsmThreads, 0, s>>>(u, n, ukeys.p, usum.p, tol, flags.p);
    note_launch();
    unsigned long long bad = 0;
    CE_CUDA(cudaMemcpyAsync(&bad, flags.p, sizeof bad, cudaMemcpyDeviceToHost, s));
    CE_CUDA(cudaStreamSynchronize(s));
    if (bad != ~0ull) {
      unsigned long long key = 0;
      double x = 0.0;
      CE_CUDA(cudaMemcpy(&key, ukeys.p + bad, sizeof key, cudaMemcpyDeviceToHost));
      CE_CUDA(cudaMemcpy(&x, usum.p + bad, sizeof x, cudaMemcpyDeviceToHost));
      // the transposed value, as the reference reports |v - vt|
      std::vector<unsigned long long> hk(static_cast<size_t>(u));
      CE_CUDA(cudaMemcpy(hk.data(), ukeys.p, static_cast<size_t>(u) * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
      const unsigned long long r = key / n, c = key % n, tk = c * n + r;
      const auto it = std::lower_bound(hk.begin(), hk.end(), tk);
      double xt = 0.0;
      if (it != hk.end() && *it == tk)
        CE_CUDA(cudaMemcpy(&xt, usum.p + (it - hk.begin()), sizeof xt, cudaMemcpyDeviceToHost));
      char buf[160];
      std::snprintf(buf, sizeof buf, "asymmetric input: |a(%llu,%llu) - a(%llu,%llu)| = %g", r, c, c, r, std::fabs(x - xt));
      R.error = buf;
      return R;
    }
  }
  // block pattern: insert_symmetric of every entry's block + add_full_diagonal
  const int64_t eb = 2 * u + m;
  DevArray<unsigned long long> bkeys(static_cast<size_t>(std::max<int64_t>(eb, 1)));
  block_keys_kernel<<<blocks_for(u + m), kAsmThreads, 0, s>>>(u, n, m, ukeys.p, d_offsets, bkeys.p);
  note_launch();
  radix_sort(bkeys, nullptr, eb, s);
  DevArray<int> bheads(static_cast<size_t>(eb)), bpos(static_cast<size_t>(eb));
  block_heads_kernel<<<blocks_for(eb), kAsmThreads, 0, s>>>(eb, bkeys.p, bheads.p);
  note_launch();
  exclusive_scan(bheads.p, bpos.p, eb, s);
  const int64_t nb = read_int_at(bpos.p, eb - 1, s) + read_int_at(bheads.p, eb - 1, s);
  DevArray<unsigned long long> ub(static_cast<size_t>(nb));
  block_compact_kernel<<<blocks_for(eb), kAsmThreads, 0, s>>>(eb, bkeys.p, bheads.p, bpos.p, ub.p);
  DevArray<int> col(static_cast<size_t>(nb)), row_cnt(static_cast<size_t>(m));
  DevArray<int64_t> sizes(static_cast<size_t>(nb)), vptr(static_cast<size_t>(nb) + 1);
  row_cnt.zero(s);
  block_meta_kernel<<<blocks_for(nb), kAsmThreads, 0, s>>>(nb, m, ub.p, d_offsets, col.p, sizes.p, row_cnt.p);
  note_launch(2);
  exclusive_scan(sizes.p, vptr.p, nb, s);
  std::vector<int64_t> hsz(static_cast<size_t>(nb));
  R.val_ptr.resize(static_cast<size_t>(nb) + 1);
  CE_CUDA(cudaMemcpyAsync(R.val_ptr.data(), vptr.p, static_cast<size_t>(nb) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CE_CUDA(cudaMemcpyAsync(hsz.data(), sizes.p, static_cast<size_t>(nb) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  std::vector<int> hcol(static_cast<size_t>(nb)), hcnt(static_cast<size_t>(m));
  CE_CUDA(cudaMemcpyAsync(hcol.data(), col.p, static_cast<size_t>(nb) * sizeof(int), cudaMemcpyDeviceToHost, s));
  CE_CUDA(cudaMemcpyAsync(hcnt.data(), row_cnt.p, static_cast<size_t>(m) * sizeof(int), cudaMemcpyDeviceToHost, s));
  CE_CUDA(cudaStreamSynchronize(s));
  R.val_ptr[static_cast<size_t>(nb)] = R.val_ptr[static_cast<size_t>(nb) - 1] + hsz[static_cast<size_t>(nb) - 1];
  R.row_ptr.assign(static_cast<size_t>(m) + 1, 0);
  for (int64_t i = 0; i < m; ++i) R.row_ptr[static_cast<size_t>(i) + 1] = R.row_ptr[static_cast<size_t>(i)] + hcnt[static_cast<size_t>(i)];
  R.col_idx.assign(hcol.begin(), hcol.end());
  R.values.alloc(static_cast<size_t>(std::max<int64_t>(R.val_ptr.back(), 1)));
  R.values.zero(s);
  DevArray<int64_t> d_vptr;
  d_vptr.upload(R.val_ptr, s);
  if (u > 0) {
    scatter_kernel<<<blocks_for(u), kAsmThreads, 0, s>>>(u, n, m, ukeys.p, usum.p, d_offsets, ub.p, nb, d_vptr.p,
                                                         R.values.p);
    note_launch();
  }
  CE_CUDA(cudaGetLastError());
  CE_CUDA(cudaStreamSynchronize(s));
  R.unique_entries = u;
  return R;
}

}  // namespace ceg
