// Preconditioner apply on the device: x = Q^T L^-T L^-1 Q b
// (CEFactorization::solve, proj/src/factorization.cpp:140-168).
//
// Per level: blockdiag U^T (factorization.cpp:34-41), the forward block
// triangular sweep (level_forward :98-111), gathers, the dense tail, then the
// backward sweep (level_backward :115-130) and blockdiag U (:43-50).
// The triangular sweeps are persistent sync-free kernels in PULL form: row j
// waits on flags of its close neighbours that precede it in the sweep order,
// gathers their contributions g_{i->j} u_i itself (no atomics, deterministic),
// and publishes u_j.  Retained coordinates, which only receive contributions,
// are reduced afterwards by an embarrassingly parallel kernel.
#include "kernels.hpp"

namespace ceg {
namespace {

constexpr int T = kApplyThreads;
constexpr int kApplyWarps = T / 32;
constexpr int kWmax = 256;  // max eliminated width per block handled by the apply sweeps
// dynamic shared memory of the sweeps: z/s (kWmax) + per-warp partial sums and u staging
constexpr size_t kSweepSmem = (kWmax + 2 * kWmax * kApplyWarps) * sizeof(double);

__device__ __forceinline__ double ldg(const double* p) { return __ldcg(p); }

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Row offset of neighbour `j` inside row i's close list, or -1.
__device__ int close_roff(const ApplyLevelArgs& A, int i, int j) {
  int64_t lo = A.cl_ptr[i], hi = A.cl_ptr[i + 1];
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    const int c = A.cl_col[mid];
    if (c == j) return A.cl_roff[mid];
    if (c < j) lo = mid + 1;
    else hi = mid;
  }
  return -1;
}

__global__ void basis_kernel(ApplyLevelArgs A, int transpose) {
  extern __shared__ double seg[];
  for (int64_t b = blockIdx.x; b < A.M; b += gridDim.x) {
    if (!A.has_basis[b]) continue;
    const int n = A.bsz[b];
    double* v = A.v + A.offsets[b];
    const double* U = A.basis + A.basis_off[b];
    for (int k = threadIdx.x; k < n; k += T) seg[k] = v[k];
    __syncthreads();
    for (int a = threadIdx.x; a < n; a += T) {
      double acc = 0.0;
      if (transpose)
        for (int c = 0; c < n; ++c) acc += U[c * n + a] * seg[c];
      else
        for (int c = 0; c < n; ++c) acc += U[a * n + c] * seg[c];
      v[a] = acc;
    }
    __syncthreads();
  }
}

// Forward sweep, rows in ascending order.
__global__ void __launch_bounds__(T) forward_kernel(ApplyLevelArgs A) {
  extern __shared__ double z[];
  __shared__ long long s_row;
  for (;;) {
    if (threadIdx.x == 0) s_row = static_cast<long long>(atomicAdd(A.ticket, 1ULL));
    __syncthreads();
    const long long jl = s_row;
    if (jl >= A.M) break;
    const int j = A.order[jl];
    const int64_t c0 = A.cl_ptr[j], c1 = A.cl_ptr[j + 1];
    if (threadIdx.x == 0) {
      for (int64_t e = c0; e < c1; ++e) {
        const int i = A.cl_col[e];
        if (i >= j) break;
        while (ld_acquire(A.flags + i) == 0) __nanosleep(32);
      }
      __threadfence();
    }
    __syncthreads();
    const int w = A.width[j];
    if (w > 0) {
      const int r = A.rank[j];
      double* vj = A.v + A.offsets[j];
      // warps pull incoming neighbours i < j: z[q] -= g_{i->j}[r_j + q, :] u_i (lane <-> q)
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      double* part = z + kWmax + warp * 2 * kWmax;
      double* ub = part + kWmax;
      for (int q = lane; q < w; q += 32) part[q] = 0.0;
      int nb = 0;
      for (int64_t e = c0; e < c1; ++e) {
        const int i = A.cl_col[e];
        if (i >= j) break;
        const int wi = A.width[i];
        if (wi == 0) continue;
        if ((nb++ % kApplyWarps) != warp) continue;
        const int ri = A.rank[i];
        const int ro = close_roff(A, i, j);
        const double* ui = A.v + A.offsets[i] + ri;
        for (int p = lane; p < wi; p += 32) ub[p] = ldg(ui + p);
        __syncwarp();
        const double* g = A.fac + A.g_off[i] + static_cast<int64_t>(ri + ro + r) * wi;
        for (int q = lane; q < w; q += 32) {
          const double* gq = g + static_cast<int64_t>(q) * wi;
          double acc = 0.0;
          for (int p = 0; p < wi; ++p) acc += gq[p] * ub[p];
          part[q] += acc;
        }
        __syncwarp();
      }
      __syncthreads();
      for (int q = threadIdx.x; q < w; q += T) {
        double acc = ldg(vj + r + q);
        for (int k = 0; k < kApplyWarps; ++k) acc -= z[kWmax + k * 2 * kWmax + q];
        z[q] = acc;
      }
      __syncthreads();
      if (threadIdx.x < 32) {
        const double* L = A.fac + A.chol_off[j];
        for (int p = 0; p < w; ++p) {
          const double up = z[p] / L[p * w + p];
          __syncwarp();
          for (int q = p + 1 + threadIdx.x; q < w; q += 32) z[q] -= L[q * w + p] * up;
          if (threadIdx.x == 0) z[p] = up;
          __syncwarp();
        }
      }
      __syncthreads();
      for (int q = threadIdx.x; q < w; q += T) vj[r + q] = z[q];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicExch(A.flags + j, 1);
    }
  }
}

// Retained coordinates: v_j[:r_j] -= C_j u_j + sum_{i in close(j)} g_{i->j}[:r_j] u_i.
__global__ void __launch_bounds__(T) retained_kernel(ApplyLevelArgs A) {
  extern __shared__ double rsm[];
  for (int64_t jl = blockIdx.x; jl < A.M; jl += gridDim.x) {
    const int j = static_cast<int>(jl);
    const int r = A.rank[j];
    if (r == 0) continue;
    const int w = A.width[j];
    double* vj = A.v + A.offsets[j];
    const int64_t c0 = A.cl_ptr[j], c1 = A.cl_ptr[j + 1];
    // segment 0: own coupling C_j u_j; segment k: g_{i->j}[:r_j] u_i for the k-th close neighbour i
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* part = rsm + warp * 2 * kWmax;
    double* ub = part + kWmax;
    for (int a = lane; a < r; a += 32) part[a] = 0.0;
    __syncwarp();
    const int nseg = static_cast<int>(c1 - c0) + 1;
    for (int sgi = warp; sgi < nseg; sgi += kApplyWarps) {
      const double* g;
      int wi, ri;
      const double* ui;
      if (sgi == 0) {
        wi = w;
        if (wi == 0) continue;
        g = A.fac + A.g_off[j];
        ui = vj + r;
      } else {
        const int i = A.cl_col[c0 + sgi - 1];
        wi = A.width[i];
        if (wi == 0) continue;
        ri = A.rank[i];
        g = A.fac + A.g_off[i] + static_cast<int64_t>(ri + close_roff(A, i, j)) * wi;
        ui = A.v + A.offsets[i] + ri;
      }
      for (int p = lane; p < wi; p += 32) ub[p] = ui[p];
      __syncwarp();
      for (int a = lane; a < r; a += 32) {
        const double* ga = g + static_cast<int64_t>(a) * wi;
        double acc = 0.0;
        for (int p = 0; p < wi; ++p) acc += ga[p] * ub[p];
        part[a] += acc;
      }
      __syncwarp();
    }
    __syncthreads();
    for (int a = threadIdx.x; a < r; a += T) {
      double acc = 0.0;
      for (int k = 0; k < kApplyWarps; ++k) acc += rsm[k * 2 * kWmax + a];
      vj[a] -= acc;
    }
    __syncthreads();
  }
}

// Backward sweep, rows in descending order.
__global__ void __launch_bounds__(T) backward_kernel(ApplyLevelArgs A) {
  extern __shared__ double sb[];
  __shared__ long long s_t;
  for (;;) {
    if (threadIdx.x == 0) s_t = static_cast<long long>(atomicAdd(A.ticket, 1ULL));
    __syncthreads();
    const long long tk = s_t;
    if (tk >= A.M) break;
    const int j = A.order[tk];
    const int64_t c0 = A.cl_ptr[j], c1 = A.cl_ptr[j + 1];
    if (threadIdx.x == 0) {
      for (int64_t e = c1 - 1; e >= c0; --e) {
        const int t = A.cl_col[e];
        if (t <= j) break;
        while (ld_acquire(A.flags + t) == 0) __nanosleep(32);
      }
      __threadfence();
    }
    __syncthreads();
    const int w = A.width[j];
    if (w > 0) {
      const int r = A.rank[j];
      double* vj = A.v + A.offsets[j];
      const double* G = A.fac + A.g_off[j];
      // s[q] = v_j[r+q] - sum_rows G[a][q] * v(a): warps over segments (coupling, then each neighbour),
      // lanes over q so every G row is read coalesced
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      double* part = sb + kWmax + warp * kWmax;
      for (int q = lane; q < w; q += 32) part[q] = 0.0;
      __syncwarp();
      const int nseg = static_cast<int>(c1 - c0) + 1;
      for (int sgi = warp; sgi < nseg; sgi += kApplyWarps) {
        const double* rows;
        const double* vt;
        int nt;
        if (sgi == 0) {
          rows = G;
          vt = vj;
          nt = r;
        } else {
          const int64_t e = c0 + sgi - 1;
          const int t = A.cl_col[e];
          nt = t > j ? A.bsz[t] : A.rank[t];
          rows = G + static_cast<int64_t>(r + A.cl_roff[e]) * w;
          vt = A.v + A.offsets[t];
        }
        for (int a = 0; a < nt; ++a) {
          const double va = ldg(vt + a);
          const double* ga = rows + static_cast<int64_t>(a) * w;
          for (int q = lane; q < w; q += 32) part[q] += ga[q] * va;
        }
      }
      __syncthreads();
      for (int q = threadIdx.x; q < w; q += T) {
        double acc = ldg(vj + r + q);
        for (int k = 0; k < kApplyWarps; ++k) acc -= sb[kWmax + k * kWmax + q];
        sb[q] = acc;
      }
      __syncthreads();
      if (threadIdx.x < 32) {
        const double* L = A.fac + A.chol_off[j];
        for (int q = w - 1; q >= 0; --q) {
          const double uq = sb[q] / L[q * w + q];
          __syncwarp();
          for (int p = threadIdx.x; p < q; p += 32) sb[p] -= L[q * w + p] * uq;
          if (threadIdx.x == 0) sb[q] = uq;
          __syncwarp();
        }
      }
      __syncthreads();
      for (int q = threadIdx.x; q < w; q += T) vj[r + q] = sb[q];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicExch(A.flags + j, 1);
    }
  }
}

// apply_operator forward (factorization.cpp:219-235): c_i = L^T v[r:] + C^T v[:r] + sum g^T v_t.
__global__ void op_forward_kernel(ApplyLevelArgs A, const int64_t* elim_off, double* c) {
  for (int64_t il = blockIdx.x; il < A.M; il += gridDim.x) {
    const int i = static_cast<int>(il);
    const int w = A.width[i];
    if (w == 0) continue;
    const int r = A.rank[i];
    const double* vi = A.v + A.offsets[i];
    const double* L = A.fac + A.chol_off[i];
    const double* G = A.fac + A.g_off[i];
    for (int q = threadIdx.x; q < w; q += T) {
      double acc = 0.0;
      for (int p = q; p < w; ++p) acc += L[p * w + q] * vi[r + p];
      for (int a = 0; a < r; ++a) acc += G[static_cast<int64_t>(a) * w + q] * vi[a];
      for (int64_t e = A.cl_ptr[i]; e < A.cl_ptr[i + 1]; ++e) {
        const int t = A.cl_col[e];
        const double* gt = G + static_cast<int64_t>(r + A.cl_roff[e]) * w;
        const double* vt = A.v + A.offsets[t];
        for (int a = 0; a < A.bsz[t]; ++a) acc += gt[static_cast<int64_t>(a) * w + q] * vt[a];
      }
      c[elim_off[i] + q] = acc;
    }
  }
}

// apply_operator backward (factorization.cpp:241-256), push with atomics (validation tool only).
__global__ void op_backward_kernel(ApplyLevelArgs A, const int64_t* elim_off, const double* c) {
  for (int64_t il = blockIdx.x; il < A.M; il += gridDim.x) {
    const int i = static_cast<int>(il);
    const int w = A.width[i];
    if (w == 0) continue;
    const int r = A.rank[i];
    double* vi = A.v + A.offsets[i];
    const double* L = A.fac + A.chol_off[i];
    const double* G = A.fac + A.g_off[i];
    const double* ci = c + elim_off[i];
    for (int p = threadIdx.x; p < w; p += T) {
      double acc = 0.0;
      for (int q = 0; q <= p; ++q) acc += L[p * w + q] * ci[q];
      atomicAdd(vi + r + p, acc);
    }
    for (int a = threadIdx.x; a < r; a += T) {
      double acc = 0.0;
      for (int q = 0; q < w; ++q) acc += G[static_cast<int64_t>(a) * w + q] * ci[q];
      atomicAdd(vi + a, acc);
    }
    for (int64_t e = A.cl_ptr[i]; e < A.cl_ptr[i + 1]; ++e) {
      const int t = A.cl_col[e];
      const double* gt = G + static_cast<int64_t>(r + A.cl_roff[e]) * w;
      double* vt = A.v + A.offsets[t];
      for (int a = threadIdx.x; a < A.bsz[t]; a += T) {
        double acc = 0.0;
        for (int q = 0; q < w; ++q) acc += gt[static_cast<int64_t>(a) * w + q] * ci[q];
        atomicAdd(vt + a, acc);
      }
    }
  }
}

__global__ void gather_kernel(const double* src, const int64_t* idx, double* dst, int64_t n) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n; k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[k] = src[idx[k]];
}

__global__ void scatter_kernel(const double* src, const int64_t* idx, double* dst, int64_t n) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n; k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[idx[k]] = src[k];
}

// y = L x (trans 0) or y = L^T x (trans 1) for a dense lower-triangular row-major L; one warp per output.
__global__ void trmv_kernel(const double* L, const double* x, double* y, int64_t n, int trans) {
  const int64_t warp = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= n) return;
  double acc = 0.0;
  if (!trans) {
    for (int64_t c = lane; c <= warp; c += 32) acc += L[warp * n + c] * x[c];
  } else {
    for (int64_t rr = warp + lane; rr < n; rr += 32) acc += L[rr * n + warp] * x[rr];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) y[warp] = acc;
}

unsigned grid_for(int64_t M) { return static_cast<unsigned>(M < 65535 * 8 ? (M > 0 ? M : 1) : 65535 * 8); }

}  // namespace

void launch_basis_apply(const ApplyLevelArgs& a, int transpose, cudaStream_t s) {
  if (a.M == 0) return;
  int bmax = 0;
  (void)bmax;
  note_launch();
  basis_kernel<<<grid_for(a.M), T, 1024 * sizeof(double), s>>>(a, transpose);
}

void launch_forward_sweep(const ApplyLevelArgs& a, int grid, cudaStream_t s) {
  if (a.M == 0) return;
  note_launch();
  forward_kernel<<<grid, T, kSweepSmem, s>>>(a);
}

void launch_forward_retained(const ApplyLevelArgs& a, cudaStream_t s) {
  if (a.M == 0) return;
  note_launch();
  retained_kernel<<<grid_for(a.M), T, 2 * kWmax * kApplyWarps * sizeof(double), s>>>(a);
}

void launch_backward_sweep(const ApplyLevelArgs& a, int grid, cudaStream_t s) {
  if (a.M == 0) return;
  note_launch();
  backward_kernel<<<grid, T, kSweepSmem, s>>>(a);
}

void launch_operator_forward(const ApplyLevelArgs& a, const int64_t* elim_off, double* c, cudaStream_t s) {
  if (a.M) {
    note_launch();
    op_forward_kernel<<<grid_for(a.M), T, 0, s>>>(a, elim_off, c);
  }
}

void launch_operator_backward(const ApplyLevelArgs& a, const int64_t* elim_off, const double* c, cudaStream_t s) {
  if (a.M) {
    note_launch();
    op_backward_kernel<<<grid_for(a.M), T, 0, s>>>(a, elim_off, c);
  }
}

void launch_gather(const double* src, const int64_t* idx, double* dst, int64_t n, cudaStream_t s) {
  if (n > 0) {
    note_launch();
    gather_kernel<<<static_cast<unsigned>((n + 255) / 256 < 65535 * 4 ? (n + 255) / 256 : 65535 * 4), 256, 0, s>>>(src, idx, dst, n);
  }
}

void launch_scatter(const double* src, const int64_t* idx, double* dst, int64_t n, cudaStream_t s) {
  if (n > 0) {
    note_launch();
    scatter_kernel<<<static_cast<unsigned>((n + 255) / 256 < 65535 * 4 ? (n + 255) / 256 : 65535 * 4), 256, 0, s>>>(src, idx, dst, n);
  }
}

void launch_dense_trmv(const double* L, const double* x, double* y, int64_t n, int trans, cudaStream_t s) {
  if (n > 0) {
    note_launch();
    trmv_kernel<<<static_cast<unsigned>((n * 32 + 255) / 256), 256, 0, s>>>(L, x, y, n, trans);
  }
}

}  // namespace ceg
