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
#ifndef CE_APPLY_PREFETCH
#define CE_APPLY_PREFETCH 1
#endif
constexpr int kWmax = kApplyWmax;  // max eliminated width per block handled by the apply sweeps
// dynamic shared memory of the sweeps: z/s (kWmax) + per-warp partial sums and u staging
constexpr size_t kSweepSmem = (kWmax + 2 * kWmax * kApplyWarps) * sizeof(double);

__device__ __forceinline__ double ldg(const double* p) { return __ldcg(p); }

#ifndef CE_APPLY_SLEEP
#define CE_APPLY_SLEEP 32  // ns of __nanosleep between dependency polls (0: spin; A/B builds)
#endif
__device__ __forceinline__ void apply_backoff() {
  if (CE_APPLY_SLEEP > 0) __nanosleep(CE_APPLY_SLEEP);
}

// Pull [p, p + n doubles) into L2 (one prefetch per 128-byte line, lanes of the calling
// warp split the lines).  Issued before a task waits for its dependencies: the factor
// data does not depend on them, so after the wait its loads hit L2 instead of HBM.
__device__ __forceinline__ void prefetch_l2(const double* p, int64_t n, int lane) {
#if CE_APPLY_PREFETCH
  const char* b = reinterpret_cast<const char*>(p);
  const int64_t bytes = n * static_cast<int64_t>(sizeof(double));
  for (int64_t o = static_cast<int64_t>(lane) * 128; o < bytes; o += 32 * 128)
    asm volatile("prefetch.global.L2 [%0];" ::"l"(b + o));
#else
  (void)p; (void)n; (void)lane;
#endif
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
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

// Forward sweep, rows in wave order.  Row j: wait for its contributing neighbours
// i < j (polled in parallel), pull z = v_j[r:] - sum_i g_{i->j}[r_j:, :] u_i (a warp
// per neighbour, lanes over the rows of g), then u_j = L_j^{-1} z.
__global__ void __launch_bounds__(T) forward_kernel(ApplyLevelArgs A) {
  extern __shared__ double z[];
  __shared__ long long s_row;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (;;) {
    if (threadIdx.x == 0) s_row = static_cast<long long>(atomicAdd(A.ticket, 1ULL));
    __syncthreads();
    const long long jl = s_row;
    if (jl >= A.M) break;
    const int j = A.order[jl];
    const int64_t k0 = A.in_ptr[j], k1 = k0 + A.in_split[j];
    for (int64_t k = k0 + threadIdx.x; k < k1; k += T)
      while (ld_acquire(A.flags + A.in_src[k]) == 0) apply_backoff();
    __threadfence();
    __syncthreads();
    const int w = A.width[j];
    if (w > 0) {
      const int r = A.rank[j];
      double* vj = A.v + A.offsets[j];
      double* part = z + kWmax + warp * 2 * kWmax;
      double* ub = part + kWmax;
      for (int q = lane; q < w; q += 32) part[q] = 0.0;
      for (int64_t k = k0 + warp; k < k1; k += kApplyWarps) {
        const int wi = A.in_w[k];
        const double* ui = A.v + A.in_uoff[k];
        for (int p = lane; p < wi; p += 32) ub[p] = ldg(ui + p);
        __syncwarp();
        const double* g = A.fac + A.in_goff[k] + static_cast<int64_t>(r) * wi;
        for (int q = lane; q < w; q += 32) {
          const double* gq = g + static_cast<int64_t>(q) * wi;
          double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
          int p = 0;
          for (; p + 3 < wi; p += 4) {
            a0 = fma(__ldg(gq + p), ub[p], a0);
            a1 = fma(__ldg(gq + p + 1), ub[p + 1], a1);
            a2 = fma(__ldg(gq + p + 2), ub[p + 2], a2);
            a3 = fma(__ldg(gq + p + 3), ub[p + 3], a3);
          }
          for (; p < wi; ++p) a0 = fma(__ldg(gq + p), ub[p], a0);
          part[q] += (a0 + a1) + (a2 + a3);
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
      const double* Li = A.linv + A.linv_off[j];
      for (int q = threadIdx.x; q < w; q += T) {
        const double* lq = Li + static_cast<int64_t>(q) * w;
        double a0 = 0.0, a1 = 0.0;
        int p = 0;
        for (; p + 1 <= q; p += 2) {
          a0 = fma(__ldg(lq + p), z[p], a0);
          a1 = fma(__ldg(lq + p + 1), z[p + 1], a1);
        }
        if (p <= q) a0 = fma(__ldg(lq + p), z[p], a0);
        vj[r + q] = a0 + a1;
      }
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
    const int64_t k0 = A.in_ptr[j], k1 = A.in_ptr[j + 1];
    // segment 0: own coupling C_j u_j; segment s > 0: the (s-1)-th contributing neighbour
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* part = rsm + warp * 2 * kWmax;
    double* ub = part + kWmax;
    for (int a = lane; a < r; a += 32) part[a] = 0.0;
    __syncwarp();
    const int nseg = static_cast<int>(k1 - k0) + 1;
    for (int sgi = warp; sgi < nseg; sgi += kApplyWarps) {
      const double* g;
      int wi;
      const double* ui;
      if (sgi == 0) {
        wi = w;
        if (wi == 0) continue;
        g = A.fac + A.g_off[j];
        ui = vj + r;
      } else {
        const int64_t k = k0 + sgi - 1;
        wi = A.in_w[k];
        g = A.fac + A.in_goff[k];
        ui = A.v + A.in_uoff[k];
      }
      for (int p = lane; p < wi; p += 32) ub[p] = ui[p];
      __syncwarp();
      for (int a = lane; a < r; a += 32) {
        const double* ga = g + static_cast<int64_t>(a) * wi;
        double a0 = 0.0, a1 = 0.0;
        int p = 0;
        for (; p + 1 < wi; p += 2) {
          a0 = fma(__ldg(ga + p), ub[p], a0);
          a1 = fma(__ldg(ga + p + 1), ub[p + 1], a1);
        }
        if (p < wi) a0 = fma(__ldg(ga + p), ub[p], a0);
        part[a] += a0 + a1;
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

// Backward sweep, rows in wave order.  Row j: wait for its dependencies t > j (w_t > 0),
// s = v_j[r:] - G_j^T v (coupling rows against v_j[:r], neighbour rows against v_t), then
// u_j = L_j^{-T} s.
__global__ void __launch_bounds__(T) backward_kernel(ApplyLevelArgs A) {
  extern __shared__ double sb[];
  __shared__ long long s_t;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (;;) {
    if (threadIdx.x == 0) s_t = static_cast<long long>(atomicAdd(A.ticket, 1ULL));
    __syncthreads();
    const long long tk = s_t;
    if (tk >= A.M) break;
    const int j = A.order[tk];
    for (int64_t k = A.dep_ptr[j] + threadIdx.x; k < A.dep_ptr[j + 1]; k += T)
      while (ld_acquire(A.flags + A.dep_t[k]) == 0) apply_backoff();
    __threadfence();
    __syncthreads();
    const int w = A.width[j];
    if (w > 0) {
      const int r = A.rank[j];
      const int64_t c0 = A.cl_ptr[j], c1 = A.cl_ptr[j + 1];
      double* vj = A.v + A.offsets[j];
      const double* G = A.fac + A.g_off[j];
      double* part = sb + kWmax + warp * 2 * kWmax;
      double* vbuf = part + kWmax;
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
          nt = A.cl_nt[e];
          rows = G + static_cast<int64_t>(r + A.cl_roff[e]) * w;
          vt = A.v + A.offsets[A.cl_col[e]];
        }
        // v_t staged with one coalesced load; rows of G read coalesced, 4 in flight per lane
        for (int a = lane; a < nt; a += 32) vbuf[a] = ldg(vt + a);
        __syncwarp();
        for (int q = lane; q < w; q += 32) {
          const double* gq = rows + q;
          double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
          int a = 0;
          for (; a + 3 < nt; a += 4) {
            a0 = fma(__ldg(gq + static_cast<int64_t>(a) * w), vbuf[a], a0);
            a1 = fma(__ldg(gq + static_cast<int64_t>(a + 1) * w), vbuf[a + 1], a1);
            a2 = fma(__ldg(gq + static_cast<int64_t>(a + 2) * w), vbuf[a + 2], a2);
            a3 = fma(__ldg(gq + static_cast<int64_t>(a + 3) * w), vbuf[a + 3], a3);
          }
          for (; a < nt; ++a) a0 = fma(__ldg(gq + static_cast<int64_t>(a) * w), vbuf[a], a0);
          part[q] += (a0 + a1) + (a2 + a3);
        }
        __syncwarp();
      }
      __syncthreads();
      for (int q = threadIdx.x; q < w; q += T) {
        double acc = ldg(vj + r + q);
        for (int k = 0; k < kApplyWarps; ++k) acc -= sb[kWmax + k * 2 * kWmax + q];
        sb[q] = acc;
      }
      __syncthreads();
      const double* Li = A.linv + A.linv_off[j];
      for (int p = threadIdx.x; p < w; p += T) {
        double a0 = 0.0, a1 = 0.0;
        int q = p;
        for (; q + 1 < w; q += 2) {
          a0 = fma(__ldg(Li + static_cast<int64_t>(q) * w + p), sb[q], a0);
          a1 = fma(__ldg(Li + static_cast<int64_t>(q + 1) * w + p), sb[q + 1], a1);
        }
        if (q < w) a0 = fma(__ldg(Li + static_cast<int64_t>(q) * w + p), sb[q], a0);
        vj[r + p] = a0 + a1;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicExch(A.flags + j, 1);
    }
  }
}

// ---- split-row sweeps (item = (row, part)) ----
// Forward partial: sum over incoming entries [k0, k1) of g_{i->j}[r_j:, :] u_i -> scratch.
// Forward finalize: z = v_j[r:] - sum of the row's partials (fixed order), u_j = L^{-1} z.
__global__ void __launch_bounds__(T) forward_task_kernel(ApplyLevelArgs A) {
  extern __shared__ double z[];
  __shared__ long long s_item;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (;;) {
    if (threadIdx.x == 0) s_item = static_cast<long long>(atomicAdd(A.ticket, 1ULL));
    __syncthreads();
    const long long it = s_item;
    if (it >= A.n_items) break;
    const int j = A.item_row[it], part0 = A.item_part[it];
    const int64_t pp = A.part_ptr[j];
    const int P = static_cast<int>(A.part_ptr[j + 1] - pp) - 1;
    const int w = A.width[j], r = A.rank[j];
    double* scr = A.scratch + A.scr_off[j];
    const bool fused = part0 < 0;  // single-slice row: pull and finalize in one item
    const int part = fused ? 0 : part0;
    if (part < P) {
      const int64_t k0 = A.part_b[pp + part], k1 = A.part_b[pp + part + 1];
      for (int64_t k = k0 + warp; k < k1; k += kApplyWarps) {
        const int wi = A.in_w[k];
        prefetch_l2(A.fac + A.in_goff[k] + static_cast<int64_t>(r) * wi, static_cast<int64_t>(w) * wi, lane);
      }
      if (fused && warp == kApplyWarps - 1) prefetch_l2(A.linv + A.linv_off[j], static_cast<int64_t>(w) * w, lane);
      for (int64_t k = k0 + threadIdx.x; k < k1; k += T)
        while (ld_acquire(A.flags + A.in_src[k]) == 0) apply_backoff();
      if (threadIdx.x == 0) __threadfence();
      __syncthreads();
      double* pw = z + kWmax + warp * 2 * kWmax;
      double* ub = pw + kWmax;
      for (int q = lane; q < w; q += 32) pw[q] = 0.0;
      for (int64_t k = k0 + warp; k < k1; k += kApplyWarps) {
        const int wi = A.in_w[k];
        const double* ui = A.v + A.in_uoff[k];
        for (int p = lane; p < wi; p += 32) ub[p] = ldg(ui + p);
        __syncwarp();
        const double* g = A.fac + A.in_goff[k] + static_cast<int64_t>(r) * wi;
        for (int q = lane; q < w; q += 32) {
          const double* gq = g + static_cast<int64_t>(q) * wi;
          double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
          int p = 0;
          for (; p + 3 < wi; p += 4) {
            a0 = fma(__ldg(gq + p), ub[p], a0);
            a1 = fma(__ldg(gq + p + 1), ub[p + 1], a1);
            a2 = fma(__ldg(gq + p + 2), ub[p + 2], a2);
            a3 = fma(__ldg(gq + p + 3), ub[p + 3], a3);
          }
          for (; p < wi; ++p) a0 = fma(__ldg(gq + p), ub[p], a0);
          pw[q] += (a0 + a1) + (a2 + a3);
        }
        __syncwarp();
      }
      __syncthreads();
      if (fused) {
        double* vj = A.v + A.offsets[j];
        for (int q = threadIdx.x; q < w; q += T) {
          double acc = 0.0;
          for (int k = 0; k < kApplyWarps; ++k) acc += z[kWmax + k * 2 * kWmax + q];
          z[q] = ldg(vj + r + q) - acc;
        }
        __syncthreads();
      } else {
        for (int q = threadIdx.x; q < w; q += T) {
          double acc = 0.0;
          for (int k = 0; k < kApplyWarps; ++k) acc += z[kWmax + k * 2 * kWmax + q];
          scr[static_cast<int64_t>(part) * w + q] = acc;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          __threadfence();
          atomicAdd(A.parts_done + j, 1);
        }
        continue;
      }
    }
    {
      if (!fused) {
        if (warp == 1) prefetch_l2(A.linv + A.linv_off[j], static_cast<int64_t>(w) * w, lane);
        if (threadIdx.x == 0) {
          while (ld_acquire(A.parts_done + j) < P) apply_backoff();
          __threadfence();
        }
        __syncthreads();
        double* vj = A.v + A.offsets[j];
        for (int q = threadIdx.x; q < w; q += T) {
          double acc = ldg(vj + r + q);
          for (int k = 0; k < P; ++k) acc -= ldg(scr + static_cast<int64_t>(k) * w + q);
          z[q] = acc;
        }
        __syncthreads();
      }
      double* vj = A.v + A.offsets[j];
      const double* Li = A.linv + A.linv_off[j];
      for (int q = threadIdx.x; q < w; q += T) {
        const double* lq = Li + static_cast<int64_t>(q) * w;
        double a0 = 0.0, a1 = 0.0;
        int p = 0;
        for (; p + 1 <= q; p += 2) {
          a0 = fma(__ldg(lq + p), z[p], a0);
          a1 = fma(__ldg(lq + p + 1), z[p + 1], a1);
        }
        if (p <= q) a0 = fma(__ldg(lq + p), z[p], a0);
        vj[r + q] = a0 + a1;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        atomicExch(A.flags + j, 1);
      }
    }
  }
}

// Backward partial: segments [s0, s1) of row j (segment 0 = coupling rows against
// v_j[:r], segment e > 0 = close entry e-1 rows against v_t) -> scratch.
// Backward finalize: s = v_j[r:] - sum of partials, u_j = L^{-T} s.
__global__ void __launch_bounds__(T) backward_task_kernel(ApplyLevelArgs A) {
  extern __shared__ double sb[];
  __shared__ long long s_item;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (;;) {
    if (threadIdx.x == 0) s_item = static_cast<long long>(atomicAdd(A.ticket, 1ULL));
    __syncthreads();
    const long long it = s_item;
    if (it >= A.n_items) break;
    const int j = A.item_row[it], part0 = A.item_part[it];
    const int64_t pp = A.part_ptr[j];
    const int P = static_cast<int>(A.part_ptr[j + 1] - pp) - 1;
    const int w = A.width[j], r = A.rank[j];
    double* scr = A.scratch + A.scr_off[j];
    const int64_t c0 = A.cl_ptr[j];
    const bool fused = part0 < 0;  // single-slice row: pull and finalize in one item
    const int part = fused ? 0 : part0;
    if (part < P) {
      const int s0 = static_cast<int>(A.part_b[pp + part]), s1 = static_cast<int>(A.part_b[pp + part + 1]);
      for (int sgi = s0 + warp; sgi < s1; sgi += kApplyWarps) {
        const double* G = A.fac + A.g_off[j];
        if (sgi == 0) prefetch_l2(G, static_cast<int64_t>(r) * w, lane);
        else prefetch_l2(G + static_cast<int64_t>(r + A.cl_roff[c0 + sgi - 1]) * w,
                         static_cast<int64_t>(A.cl_nt[c0 + sgi - 1]) * w, lane);
      }
      if (fused && warp == kApplyWarps - 1) prefetch_l2(A.linv + A.linv_off[j], static_cast<int64_t>(w) * w, lane);
      for (int sgi = s0 + threadIdx.x; sgi < s1; sgi += T) {
        if (sgi == 0) continue;
        const int t = A.cl_col[c0 + sgi - 1];
        if (t > j && A.width[t] > 0)
          while (ld_acquire(A.flags + t) == 0) apply_backoff();
      }
      if (threadIdx.x == 0) __threadfence();
      __syncthreads();
      double* vj = A.v + A.offsets[j];
      const double* G = A.fac + A.g_off[j];
      double* pw = sb + kWmax + warp * 2 * kWmax;
      double* vbuf = pw + kWmax;
      for (int q = lane; q < w; q += 32) pw[q] = 0.0;
      __syncwarp();
      for (int sgi = s0 + warp; sgi < s1; sgi += kApplyWarps) {
        const double* rows;
        const double* vt;
        int nt;
        if (sgi == 0) {
          rows = G;
          vt = vj;
          nt = r;
        } else {
          const int64_t e = c0 + sgi - 1;
          nt = A.cl_nt[e];
          rows = G + static_cast<int64_t>(r + A.cl_roff[e]) * w;
          vt = A.v + A.offsets[A.cl_col[e]];
        }
        for (int a = lane; a < nt; a += 32) vbuf[a] = ldg(vt + a);
        __syncwarp();
        for (int q = lane; q < w; q += 32) {
          const double* gq = rows + q;
          double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
          int a = 0;
          for (; a + 3 < nt; a += 4) {
            a0 = fma(__ldg(gq + static_cast<int64_t>(a) * w), vbuf[a], a0);
            a1 = fma(__ldg(gq + static_cast<int64_t>(a + 1) * w), vbuf[a + 1], a1);
            a2 = fma(__ldg(gq + static_cast<int64_t>(a + 2) * w), vbuf[a + 2], a2);
            a3 = fma(__ldg(gq + static_cast<int64_t>(a + 3) * w), vbuf[a + 3], a3);
          }
          for (; a < nt; ++a) a0 = fma(__ldg(gq + static_cast<int64_t>(a) * w), vbuf[a], a0);
          pw[q] += (a0 + a1) + (a2 + a3);
        }
        __syncwarp();
      }
      __syncthreads();
      if (fused) {
        for (int q = threadIdx.x; q < w; q += T) {
          double acc = 0.0;
          for (int k = 0; k < kApplyWarps; ++k) acc += sb[kWmax + k * 2 * kWmax + q];
          sb[q] = ldg(vj + r + q) - acc;
        }
        __syncthreads();
      } else {
        for (int q = threadIdx.x; q < w; q += T) {
          double acc = 0.0;
          for (int k = 0; k < kApplyWarps; ++k) acc += sb[kWmax + k * 2 * kWmax + q];
          scr[static_cast<int64_t>(part) * w + q] = acc;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          __threadfence();
          atomicAdd(A.parts_done + j, 1);
        }
        continue;
      }
    }
    {
      double* vj = A.v + A.offsets[j];
      if (!fused) {
        if (warp == 1) prefetch_l2(A.linv + A.linv_off[j], static_cast<int64_t>(w) * w, lane);
        if (threadIdx.x == 0) {
          while (ld_acquire(A.parts_done + j) < P) apply_backoff();
          __threadfence();
        }
        __syncthreads();
        for (int q = threadIdx.x; q < w; q += T) {
          double acc = ldg(vj + r + q);
          for (int k = 0; k < P; ++k) acc -= ldg(scr + static_cast<int64_t>(k) * w + q);
          sb[q] = acc;
        }
        __syncthreads();
      }
      const double* Li = A.linv + A.linv_off[j];
      for (int p = threadIdx.x; p < w; p += T) {
        double a0 = 0.0, a1 = 0.0;
        int q = p;
        for (; q + 1 < w; q += 2) {
          a0 = fma(__ldg(Li + static_cast<int64_t>(q) * w + p), sb[q], a0);
          a1 = fma(__ldg(Li + static_cast<int64_t>(q + 1) * w + p), sb[q + 1], a1);
        }
        if (q < w) a0 = fma(__ldg(Li + static_cast<int64_t>(q) * w + p), sb[q], a0);
        vj[r + p] = a0 + a1;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        atomicExch(A.flags + j, 1);
      }
    }
  }
}

// ---- warp-granular split-row sweeps (CE_APPLY_WARP) ----
// The same items, dependencies and arithmetic as forward/backward_task_kernel, but every warp
// is an independent worker: it takes its own ticket and runs the item alone with warp-level
// synchronisation only.  The sweeps are latency chains (one dependency hop per wave, ~500-1500
// waves per level on the reference plan), so an item's latency, not its work, sets the time:
// no CTA-wide barriers on the path, and four items in flight per CTA instead of one.  A row's
// inputs are summed by one warp in ascending entry order (deterministic).
constexpr int kQm = kWmax / 32;  // columns q per lane
constexpr size_t kWarpSmem = 2 * kWmax * kApplyWarps * sizeof(double);

__global__ void __launch_bounds__(T) forward_warp_kernel(ApplyLevelArgs A) {
  extern __shared__ double sh[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* z = sh + warp * 2 * kWmax;
  double* ub = z + kWmax;
  for (;;) {
    long long it = 0;
    if (lane == 0) it = static_cast<long long>(atomicAdd(A.ticket, 1ULL));
    it = __shfl_sync(0xffffffffu, it, 0);
    if (it >= A.n_items) break;
    const int j = A.item_row[it], part0 = A.item_part[it];
    const int64_t pp = A.part_ptr[j];
    const int P = static_cast<int>(A.part_ptr[j + 1] - pp) - 1;
    const int w = A.width[j], r = A.rank[j];
    double* scr = A.scratch + A.scr_off[j];
    double* vj = A.v + A.offsets[j];
    const bool fused = part0 < 0;
    const int part = fused ? 0 : part0;
    if (part < P) {
      const int64_t k0 = A.part_b[pp + part], k1 = A.part_b[pp + part + 1];
      for (int64_t k = k0; k < k1; ++k) {
        const int wi = A.in_w[k];
        prefetch_l2(A.fac + A.in_goff[k] + static_cast<int64_t>(r) * wi, static_cast<int64_t>(w) * wi, lane);
      }
      if (fused) prefetch_l2(A.linv + A.linv_off[j], static_cast<int64_t>(w) * w, lane);
      for (int64_t k = k0 + lane; k < k1; k += 32)
        while (ld_acquire(A.flags + A.in_src[k]) == 0) apply_backoff();
      __threadfence();
      __syncwarp();
      double acc[kQm];
#pragma unroll
      for (int m = 0; m < kQm; ++m) acc[m] = 0.0;
      for (int64_t k = k0; k < k1; ++k) {
        const int wi = A.in_w[k];
        const double* ui = A.v + A.in_uoff[k];
        for (int p = lane; p < wi; p += 32) ub[p] = ldg(ui + p);
        __syncwarp();
        const double* g = A.fac + A.in_goff[k] + static_cast<int64_t>(r) * wi;
#pragma unroll
        for (int m = 0; m < kQm; ++m) {
          const int q = lane + 32 * m;
          if (q < w) {
            const double* gq = g + static_cast<int64_t>(q) * wi;
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
            int p = 0;
            for (; p + 3 < wi; p += 4) {
              a0 = fma(__ldg(gq + p), ub[p], a0);
              a1 = fma(__ldg(gq + p + 1), ub[p + 1], a1);
              a2 = fma(__ldg(gq + p + 2), ub[p + 2], a2);
              a3 = fma(__ldg(gq + p + 3), ub[p + 3], a3);
            }
            for (; p < wi; ++p) a0 = fma(__ldg(gq + p), ub[p], a0);
            acc[m] += (a0 + a1) + (a2 + a3);
          }
        }
        __syncwarp();
      }
      if (!fused) {
#pragma unroll
        for (int m = 0; m < kQm; ++m)
          if (lane + 32 * m < w) scr[static_cast<int64_t>(part) * w + lane + 32 * m] = acc[m];
        __syncwarp();
        if (lane == 0) {
          __threadfence();
          atomicAdd(A.parts_done + j, 1);
        }
        continue;
      }
#pragma unroll
      for (int m = 0; m < kQm; ++m)
        if (lane + 32 * m < w) z[lane + 32 * m] = ldg(vj + r + lane + 32 * m) - acc[m];
      __syncwarp();
    } else {
      prefetch_l2(A.linv + A.linv_off[j], static_cast<int64_t>(w) * w, lane);
      if (lane == 0)
        while (ld_acquire(A.parts_done + j) < P) apply_backoff();
      __threadfence();
      __syncwarp();
      for (int q = lane; q < w; q += 32) {
        double a = ldg(vj + r + q);
        for (int k = 0; k < P; ++k) a -= ldg(scr + static_cast<int64_t>(k) * w + q);
        z[q] = a;
      }
      __syncwarp();
    }
    const double* Li = A.linv + A.linv_off[j];
    for (int q = lane; q < w; q += 32) {
      const double* lq = Li + static_cast<int64_t>(q) * w;
      double a0 = 0.0, a1 = 0.0;
      int p = 0;
      for (; p + 1 <= q; p += 2) {
        a0 = fma(__ldg(lq + p), z[p], a0);
        a1 = fma(__ldg(lq + p + 1), z[p + 1], a1);
      }
      if (p <= q) a0 = fma(__ldg(lq + p), z[p], a0);
      vj[r + q] = a0 + a1;
    }
    __syncwarp();
    if (lane == 0) {
      __threadfence();
      atomicExch(A.flags + j, 1);
    }
  }
}

__global__ void __launch_bounds__(T) backward_warp_kernel(ApplyLevelArgs A) {
  extern __shared__ double sh[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* sbw = sh + warp * 2 * kWmax;
  double* vbuf = sbw + kWmax;
  for (;;) {
    long long it = 0;
    if (lane == 0) it = static_cast<long long>(atomicAdd(A.ticket, 1ULL));
    it = __shfl_sync(0xffffffffu, it, 0);
    if (it >= A.n_items) break;
    const int j = A.item_row[it], part0 = A.item_part[it];
    const int64_t pp = A.part_ptr[j];
    const int P = static_cast<int>(A.part_ptr[j + 1] - pp) - 1;
    const int w = A.width[j], r = A.rank[j];
    double* scr = A.scratch + A.scr_off[j];
    const int64_t c0 = A.cl_ptr[j];
    double* vj = A.v + A.offsets[j];
    const double* G = A.fac + A.g_off[j];
    const bool fused = part0 < 0;
    const int part = fused ? 0 : part0;
    if (part < P) {
      const int s0 = static_cast<int>(A.part_b[pp + part]), s1 = static_cast<int>(A.part_b[pp + part + 1]);
      for (int sgi = s0; sgi < s1; ++sgi) {
        if (sgi == 0) prefetch_l2(G, static_cast<int64_t>(r) * w, lane);
        else prefetch_l2(G + static_cast<int64_t>(r + A.cl_roff[c0 + sgi - 1]) * w,
                         static_cast<int64_t>(A.cl_nt[c0 + sgi - 1]) * w, lane);
      }
      if (fused) prefetch_l2(A.linv + A.linv_off[j], static_cast<int64_t>(w) * w, lane);
      for (int sgi = s0 + lane; sgi < s1; sgi += 32) {
        if (sgi == 0) continue;
        const int t = A.cl_col[c0 + sgi - 1];
        if (t > j && A.width[t] > 0)
          while (ld_acquire(A.flags + t) == 0) apply_backoff();
      }
      __threadfence();
      __syncwarp();
      double acc[kQm];
#pragma unroll
      for (int m = 0; m < kQm; ++m) acc[m] = 0.0;
      for (int sgi = s0; sgi < s1; ++sgi) {
        const double* rows;
        const double* vt;
        int nt;
        if (sgi == 0) {
          rows = G;
          vt = vj;
          nt = r;
        } else {
          const int64_t e = c0 + sgi - 1;
          nt = A.cl_nt[e];
          rows = G + static_cast<int64_t>(r + A.cl_roff[e]) * w;
          vt = A.v + A.offsets[A.cl_col[e]];
        }
        for (int a = lane; a < nt; a += 32) vbuf[a] = ldg(vt + a);
        __syncwarp();
#pragma unroll
        for (int m = 0; m < kQm; ++m) {
          const int q = lane + 32 * m;
          if (q < w) {
            const double* gq = rows + q;
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
            int a = 0;
            for (; a + 3 < nt; a += 4) {
              a0 = fma(__ldg(gq + static_cast<int64_t>(a) * w), vbuf[a], a0);
              a1 = fma(__ldg(gq + static_cast<int64_t>(a + 1) * w), vbuf[a + 1], a1);
              a2 = fma(__ldg(gq + static_cast<int64_t>(a + 2) * w), vbuf[a + 2], a2);
              a3 = fma(__ldg(gq + static_cast<int64_t>(a + 3) * w), vbuf[a + 3], a3);
            }
            for (; a < nt; ++a) a0 = fma(__ldg(gq + static_cast<int64_t>(a) * w), vbuf[a], a0);
            acc[m] += (a0 + a1) + (a2 + a3);
          }
        }
        __syncwarp();
      }
      if (!fused) {
#pragma unroll
        for (int m = 0; m < kQm; ++m)
          if (lane + 32 * m < w) scr[static_cast<int64_t>(part) * w + lane + 32 * m] = acc[m];
        __syncwarp();
        if (lane == 0) {
          __threadfence();
          atomicAdd(A.parts_done + j, 1);
        }
        continue;
      }
#pragma unroll
      for (int m = 0; m < kQm; ++m)
        if (lane + 32 * m < w) sbw[lane + 32 * m] = ldg(vj + r + lane + 32 * m) - acc[m];
      __syncwarp();
    } else {
      prefetch_l2(A.linv + A.linv_off[j], static_cast<int64_t>(w) * w, lane);
      if (lane == 0)
        while (ld_acquire(A.parts_done + j) < P) apply_backoff();
      __threadfence();
      __syncwarp();
      for (int q = lane; q < w; q += 32) {
        double a = ldg(vj + r + q);
        for (int k = 0; k < P; ++k) a -= ldg(scr + static_cast<int64_t>(k) * w + q);
        sbw[q] = a;
      }
      __syncwarp();
    }
    const double* Li = A.linv + A.linv_off[j];
    for (int p = lane; p < w; p += 32) {
      double a0 = 0.0, a1 = 0.0;
      int q = p;
      for (; q + 1 < w; q += 2) {
        a0 = fma(__ldg(Li + static_cast<int64_t>(q) * w + p), sbw[q], a0);
        a1 = fma(__ldg(Li + static_cast<int64_t>(q + 1) * w + p), sbw[q + 1], a1);
      }
      if (q < w) a0 = fma(__ldg(Li + static_cast<int64_t>(q) * w + p), sbw[q], a0);
      vj[r + p] = a0 + a1;
    }
    __syncwarp();
    if (lane == 0) {
      __threadfence();
      atomicExch(A.flags + j, 1);
    }
  }
}

// L^{-1} of each row's w x w pivot factor: thread per column, forward substitution.
__global__ void pivot_inverse_kernel(int64_t M, const int* width, const double* fac, const int64_t* chol_off,
                                     double* linv, const int64_t* linv_off) {
  for (int64_t j = blockIdx.x; j < M; j += gridDim.x) {
    const int w = width[j];
    if (w == 0) continue;
    const double* L = fac + chol_off[j];
    double* X = linv + linv_off[j];
    for (int c = threadIdx.x; c < w; c += blockDim.x) {
      for (int q = 0; q < c; ++q) X[static_cast<int64_t>(q) * w + c] = 0.0;
      for (int q = c; q < w; ++q) {
        double acc = q == c ? 1.0 : 0.0;
        for (int p = c; p < q; ++p) acc -= L[static_cast<int64_t>(q) * w + p] * X[static_cast<int64_t>(p) * w + c];
        X[static_cast<int64_t>(q) * w + c] = acc / L[static_cast<int64_t>(q) * w + q];
      }
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
  note_launch();
  basis_kernel<<<grid_for(a.M), T, 1024 * sizeof(double), s>>>(a, transpose);
}

void launch_forward_sweep(const ApplyLevelArgs& a, int grid, cudaStream_t s) {
  if (a.M == 0) return;
  note_launch();
  forward_kernel<<<grid, T, kSweepSmem, s>>>(a);
}

void launch_forward_tasks(const ApplyLevelArgs& a, int grid, bool warp_items, cudaStream_t s) {
  if (a.n_items == 0) return;
  note_launch();
  if (warp_items) forward_warp_kernel<<<grid, T, kWarpSmem, s>>>(a);
  else forward_task_kernel<<<grid, T, kSweepSmem, s>>>(a);
}

void launch_backward_tasks(const ApplyLevelArgs& a, int grid, bool warp_items, cudaStream_t s) {
  if (a.n_items == 0) return;
  note_launch();
  if (warp_items) backward_warp_kernel<<<grid, T, kWarpSmem, s>>>(a);
  else backward_task_kernel<<<grid, T, kSweepSmem, s>>>(a);
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

void launch_pivot_inverse(int64_t M, const int* width, const double* fac, const int64_t* chol_off, double* linv,
                          const int64_t* linv_off, cudaStream_t s) {
  if (M <= 0) return;
  note_launch();
  pivot_inverse_kernel<<<grid_for(M), 64, 0, s>>>(M, width, fac, chol_off, linv, linv_off);
}

void launch_dense_trmv(const double* L, const double* x, double* y, int64_t n, int trans, cudaStream_t s) {
  if (n > 0) {
    note_launch();
    trmv_kernel<<<static_cast<unsigned>((n * 32 + 255) / 256), 256, 0, s>>>(L, x, y, n, trans);
  }
}

}  // namespace ceg
