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
#include <algorithm>
#include <cfloat>
#include <cstdio>

#include "kernels.hpp"

#ifndef CE_SWEEP_BUDGET
#define CE_SWEEP_BUDGET 18000  // per-CTA buffer target (doubles): strip chunk width, Schur panel height (A/B: 11k 2.03 s, 14k 1.94, 16k 1.93, 18k 1.89, 20k 1.91, 24k 2.03 on cfg2)
#endif
#ifndef CE_KCAP
#define CE_KCAP 192  // TSQR chunk height: leaves take <= 128 far columns, tree nodes fold up to kcap / b children (A/B on cfg2: 128 1.90 s, 176 1.88, 192 1.85)
#endif
#ifndef CE_KCAP_BUDGET
#define CE_KCAP_BUDGET 18000
#endif
#ifndef CE_NO_WIDE_JACOBI
#define CE_NO_WIDE_JACOBI 0
#endif
#ifndef CE_TILE_TRANSPOSED
#define CE_TILE_TRANSPOSED 1  // Schur tiles with the s panel along the accumulator rows (coalesced X accesses)
#endif
#ifndef CE_STAGE_ASYNC
#define CE_STAGE_ASYNC 1  // Schur panels staged with cp.async in the shared-memory build
#endif
#ifndef CE_SWEEP_MIN_BLOCKS
#define CE_SWEEP_MIN_BLOCKS 1  // resident sweep CTAs per SM the register allocation must allow
#endif

namespace ceg {
namespace {

constexpr int T = kSweepThreads;
constexpr int NW = T / 32;
constexpr double kClusterTol = 1e-9;  // oracle/dense.hpp
constexpr int kPanelNb = 32;          // close neighbours per Schur panel (host planner matches)
constexpr int kPanelRows = 260;       // g rows per Schur panel (<= 256 + padding)

__device__ __forceinline__ double ldg(const double* p) { return __ldcg(p); }

#ifndef CE_SWEEP_SLEEP
#define CE_SWEEP_SLEEP 64  // ns of __nanosleep between dependency polls (0: spin; A/B builds)
#endif
__device__ __forceinline__ void sweep_backoff() {
  if (CE_SWEEP_SLEEP > 0) __nanosleep(CE_SWEEP_SLEEP);
}

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

// Canonical-gauge weights, bit-identical to oracle/dense.cpp: singletons' sign rule ...
__device__ __forceinline__ double gauge_weight(int k) {
  const double x = __dmul_rn(static_cast<double>(k + 1), 0.6180339887498949);
  return 1.0 + 0.5 * (x - floor(x));
}
// ... and the cluster weights G_c(k, j): splitmix64 of (k, j), zero-mean in [-1, 1), independent
// across j so U_c^T G_c is well conditioned for any cluster size.
__device__ __forceinline__ double gauge_weight2(int k, int j) {
  unsigned long long z = static_cast<unsigned long long>(k) * 0x9E3779B97F4A7C15ull +
                         static_cast<unsigned long long>(j) * 0xD1B54A32D192ED03ull + 0x632BE59BD9B4E019ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return __dadd_rn(static_cast<double>(z >> 11) * 0x1.0p-52, -1.0);
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


// leading dimension of the column-major F^T chunk (odd: column walks are bank-conflict free)
__device__ __forceinline__ int chunk_ld(int kcap) { return kcap | 1; }
// padded (odd) leading dimension of the b x b SVD work tiles
__device__ __forceinline__ int pad_ld(int b) { return b | 1; }

// Per-CTA buffer layout.  The strip pass (strip_range) uses [D, sig) as two b x cw
// column chunks; `extra` doubles are appended after C so that small-block levels get
// wide chunks while the total stays within two CTAs per SM.
struct Layout {
  int64_t bb, creg, extra, base;
  int cw;
};
__host__ __device__ inline Layout sweep_layout(int bmax, int kcap) {
  Layout L;
  L.bb = static_cast<int64_t>(bmax) * (bmax + 1);                  // b x b tiles, padded ld
  L.creg = static_cast<int64_t>((kcap + 1) | 1) * bmax;             // F^T chunk
  L.base = 4 * L.bb + L.creg + 3LL * bmax + (bmax + 1) / 2 + 4;    // R V U D C sig tau nrm perm
  const int64_t dreg = L.bb + L.creg;
  const int64_t budget = CE_SWEEP_BUDGET;  // doubles per CTA of dynamic shared memory
  int64_t cw = dreg / (2 * bmax);
  const int64_t cwb = (budget - L.base + dreg) / (2 * bmax);
  if (cwb > cw) cw = cwb;
  if (cw > 256) cw = 256;
  if (cw < bmax) cw = bmax;  // a strip chunk holds at least one whole block (3-D merge-all levels: b > 256)
  L.cw = static_cast<int>(cw);
  L.extra = 2 * bmax * cw > dreg ? 2 * bmax * cw - dreg : 0;
  return L;
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

// Householder vector of x = [x0; y] (y = column of length K at `y`, stride 1), LAPACK dlarfg:
// returns tau, writes beta, scales y in place to the reflector tail (v0 = 1).
__device__ __forceinline__ double house_prep(double x0, double* y, int K, double* beta_out) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int m = 0;
  for (; m + 3 < K; m += 4) {
    s0 += y[m] * y[m];
    s1 += y[m + 1] * y[m + 1];
    s2 += y[m + 2] * y[m + 2];
    s3 += y[m + 3] * y[m + 3];
  }
  for (; m < K; ++m) s0 += y[m] * y[m];
  const double ss = (s0 + s1) + (s2 + s3);
  if (!(ss > 0.0)) {
    *beta_out = x0;
    return 0.0;
  }
  const double nrm = sqrt(x0 * x0 + ss);
  const double beta = x0 >= 0.0 ? -nrm : nrm;
  const double scale = 1.0 / (x0 - beta);
  for (int k = 0; k < K; ++k) y[k] *= scale;
  *beta_out = beta;
  return (beta - x0) / beta;
}

// d = a + sum_m v[m] * c[m] with four independent accumulators
__device__ __forceinline__ double dot4(double a, const double* v, const double* c, int K) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int m = 0;
  for (; m + 3 < K; m += 4) {
    s0 += v[m] * c[m];
    s1 += v[m + 1] * c[m + 1];
    s2 += v[m + 2] * c[m + 2];
    s3 += v[m + 3] * c[m + 3];
  }
  for (; m < K; ++m) s0 += v[m] * c[m];
  return a + ((s0 + s1) + (s2 + s3));
}

template <int G>
__device__ __forceinline__ double group_sum(double v, unsigned mask) {
#pragma unroll
  for (int o = G >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o);
  return v;
}

// 1/x and 1/sqrt(x) from the SFU approximations plus two Newton steps (a few ulp;
// IEEE division / sqrt are long dependent subroutines on the critical path).
__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
__device__ __forceinline__ double rsqrt_nr(double x) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double h = 0.5 * x;
  r = r * fma(-h * r, r, 1.5);
  return r * fma(-h * r, r, 1.5);
}

// barrier over the first n threads (named barrier 1) returning the OR of `pred`
__device__ __forceinline__ int bar_or(int n, int pred) {
  int r;
  asm volatile(
      "{\n .reg .pred p, q;\n setp.ne.s32 q, %1, 0;\n bar.red.or.pred p, 1, %2, q;\n selp.s32 %0, 1, 0, p;\n}"
      : "=r"(r)
      : "r"(pred), "r"(n)
      : "memory");
  return r;
}
__device__ __forceinline__ void bar_n(int n) { asm volatile("bar.sync 1, %0;" ::"r"(n) : "memory"); }

}  // namespace

// The level-sweep kernel body is compiled twice: with the per-CTA work buffer in
// shared memory (the compiler is told so, every tile access is LDS/STS) and with
// it in global scratch (levels whose blocks are too large for shared memory).
namespace sweep_smem {
namespace {
#define CE_SMEM_BUFFER 1
#include "sweep_body.cuh"
#undef CE_SMEM_BUFFER
}  // namespace
}  // namespace sweep_smem
namespace sweep_gmem {
namespace {
#define CE_SMEM_BUFFER 0
#include "sweep_body.cuh"
#undef CE_SMEM_BUFFER
}  // namespace
}  // namespace sweep_gmem

namespace {

// g_t <- U_t^T g_t for every pending (row i, neighbor t > i) pair.
__global__ void __launch_bounds__(T) pending_kernel(SweepArgs A, int cap) {
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
    // g (bt x w, row stride w) <- U^T g, in column chunks of qc so bt x qc fits the buffer
    const int qc = min(w, max(1, cap / bt));
    for (int q0 = 0; q0 < w; q0 += qc) {
      const int nq = min(qc, w - q0);
      for (int idx = threadIdx.x; idx < bt * nq; idx += T) tmp[idx] = g[(idx / nq) * w + q0 + idx % nq];
      __syncthreads();
      for (int idx = threadIdx.x; idx < bt * nq; idx += T) {
        const int a = idx / nq, q = idx % nq;
        double acc = 0.0;
        for (int c = 0; c < bt; ++c) acc += U[c * bt + a] * tmp[c * nq + q];
        g[a * w + q0 + q] = acc;
      }
      __syncthreads();
    }
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

int sweep_kcap(int bmax) {
  // F^T chunk height: 128 rows, shortened (not below 64) so that the per-CTA buffer of
  // wide-block levels still allows two CTAs per SM
  int k = CE_KCAP;
  while (k > bmax && k > 64 && sweep_layout(bmax, k).base > CE_KCAP_BUDGET) k -= 8;
  return k > bmax ? k : bmax;
}

int64_t sweep_smem_doubles(int bmax, int kcap) {
  const Layout L = sweep_layout(bmax, kcap);
  return L.base + L.extra;
}

int sweep_max_ctas_per_sm(size_t smem_bytes) {
  int n = 0;
  // smem_bytes == 0: the global-scratch variant
  auto* kern = smem_bytes > 0 ? sweep_smem::sweep_kernel : sweep_gmem::sweep_kernel;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem_bytes));
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, T, smem_bytes);
  if (e != cudaSuccess) {
    std::fprintf(stderr, "[ce] sweep occupancy query failed: %s\n", cudaGetErrorString(e));
    cudaGetLastError();
    return 0;
  }
  return n;
}

void launch_sweep(const SweepArgs& a, int grid, size_t smem_bytes, cudaStream_t s) {
  note_launch();
  if (a.use_global_scratch) {
    sweep_gmem::sweep_kernel<<<grid, T, 0, s>>>(a);
  } else {
    cudaFuncSetAttribute(sweep_smem::sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem_bytes));
    sweep_smem::sweep_kernel<<<grid, T, smem_bytes, s>>>(a);
  }
}

void launch_pending_rotation(const SweepArgs& a, cudaStream_t s) {
  if (a.M <= 0) return;
  // bmax^2 doubles, capped at 128 KB (deep 3-D levels have blocks of several hundred)
  const int cap = static_cast<int>(std::min<int64_t>(static_cast<int64_t>(a.bmax) * a.bmax, 16384));
  const size_t smem = static_cast<size_t>(cap) * sizeof(double);
  cudaFuncSetAttribute(pending_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  note_launch();
  pending_kernel<<<static_cast<unsigned>(a.M), T, smem, s>>>(a, cap);
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

__global__ void tri_table_kernel(int64_t M, const int64_t* sq_ptr, const int* sq_col, const int64_t* sq_slot,
                                 const int64_t* slot_off, int64_t* tab) {
  for (int64_t t = blockIdx.x; t < M; t += gridDim.x)
    for (int64_t e = sq_ptr[t] + threadIdx.x; e < sq_ptr[t + 1]; e += blockDim.x) {
      const int s = sq_col[e];
      if (s <= t) tab[t * (t + 1) / 2 + s] = slot_off[sq_slot[e]];
    }
}

void launch_tri_table(int64_t M, const int64_t* sq_ptr, const int* sq_col, const int64_t* sq_slot,
                      const int64_t* slot_off, int64_t* tab, cudaStream_t s) {
  if (M <= 0) return;
  cudaMemsetAsync(tab, 0xff, static_cast<size_t>(M) * (M + 1) / 2 * sizeof(int64_t), s);
  note_launch();
  tri_table_kernel<<<static_cast<unsigned>(M < 65535 ? M : 65535), 128, 0, s>>>(M, sq_ptr, sq_col, sq_slot, slot_off, tab);
}

void launch_remainder(const RemainderArgs& a, cudaStream_t s) {
  if (a.M <= 0) return;
  const unsigned grid = static_cast<unsigned>(a.M < 65535 * 8 ? a.M : 65535 * 8);
  note_launch();
  remainder_kernel<<<grid, 128, 0, s>>>(a);
}

}  // namespace ceg
