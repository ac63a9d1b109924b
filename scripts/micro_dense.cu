// Micro-benchmark of the sweep kernel's small dense routines (TSQR update, Jacobi SVD)
// in isolation: 2 CTAs per SM, each running the routine on seeded random tiles, SM
// cycles per call averaged over CTAs.  Development tool, not part of the library.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_1603_09133_b200/csrc \
//        scripts/micro_dense.cu -o scripts/build/micro_dense
#include "../paper_1603_09133_b200/csrc/sweep.cu"

#include <vector>
#include <cstdlib>

namespace ceg {
void note_launch(int64_t) {}
}  // namespace ceg

namespace ceg {
namespace {
using namespace ceg::sweep_smem;

// previous CTA-wide variant (one warp per column, warp reductions, two barriers per step)
__device__ void tsqr_warps(double* R, double* C, int K, int b, int ldc, double* shr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k = 0; k < b; ++k) {
    double* Ck = C + static_cast<int64_t>(k) * ldc;
    if (warp == 0) {
      double s2 = 0.0;
      for (int m = lane; m < K; m += 32) s2 += Ck[m] * Ck[m];
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
        for (int m = lane; m < K; m += 32) Ck[m] *= scale;
      }
      if (lane == 0) shr[0] = tau;
    }
    __syncthreads();
    const double tau = shr[0];
    if (tau != 0.0) {
      for (int j = k + 1 + warp; j < b; j += NW) {
        double* Cj = C + static_cast<int64_t>(j) * ldc;
        double s = 0.0;
        for (int m = lane; m < K; m += 32) s += Ck[m] * Cj[m];
        s = warp_sum(s);
        const double tw = tau * (R[j * b + k] + s);
        __syncwarp();
        if (lane == 0) R[j * b + k] -= tw;
        for (int m = lane; m < K; m += 32) Cj[m] -= tw * Ck[m];
      }
    }
    __syncthreads();
  }
}

// instrumented copy of tsqr_group_t: MODE 0 full, 1 no prep (fixed tau), 2 no update, 3 fast division
template <int G, int MODE>
__device__ void tsqr_probe(double* R, double* C, int K, int b, int ldc, double* shr) {
  constexpr int NG = T / G;
  const int tid = threadIdx.x, grp = tid / G, gl = tid % G;
  const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << ((tid & 31) / G * G));
  auto prep = [&](int j) {
    if (MODE == 1) {
      if (gl == 0) shr[j & 1] = 1e-3;
      return;
    }
    double* Cj = C + static_cast<int64_t>(j) * ldc;
    double s0 = 0.0, s1 = 0.0;
    int m = gl;
    for (; m + G < K; m += 2 * G) {
      s0 += Cj[m] * Cj[m];
      s1 += Cj[m + G] * Cj[m + G];
    }
    if (m < K) s0 += Cj[m] * Cj[m];
    const double ss = group_sum<G>(s0 + s1, gmask);
    const double x0 = R[j * b + j];
    double tau = 0.0;
    if (ss > 0.0) {
      const double nrm = sqrt(x0 * x0 + ss);
      const double beta = x0 >= 0.0 ? -nrm : nrm;
      double scale;
      if (MODE == 3) {
        const double den = x0 - beta;
        double r = static_cast<double>(__frcp_rn(static_cast<float>(den)));
        r = r * (2.0 - den * r);
        r = r * (2.0 - den * r);
        scale = r * (2.0 - den * r);
        tau = -den * __drcp_rn(beta);
      } else {
        scale = 1.0 / (x0 - beta);
        tau = (beta - x0) / beta;
      }
      for (int q = gl; q < K; q += G) Cj[q] *= scale;
      __syncwarp(gmask);
      if (gl == 0) R[j * b + j] = beta;
    }
    if (gl == 0) shr[j & 1] = tau;
  };
  if (grp == 0 && b > 0) prep(0);
  __syncthreads();
  for (int k = 0; k + 1 < b; ++k) {
    const double tau = shr[k & 1];
    const double* Ck = C + static_cast<int64_t>(k) * ldc;
    for (int j = k + 1 + grp; j < b; j += NG) {
      double* Cj = C + static_cast<int64_t>(j) * ldc;
      if (MODE != 2 && tau != 0.0) {
        const double rkj = R[j * b + k];
        double s0 = 0.0, s1 = 0.0;
        int m = gl;
        for (; m + G < K; m += 2 * G) {
          s0 += Ck[m] * Cj[m];
          s1 += Ck[m + G] * Cj[m + G];
        }
        if (m < K) s0 += Ck[m] * Cj[m];
        const double d = tau * (rkj + group_sum<G>(s0 + s1, gmask));
        for (int q = gl; q < K; q += G) Cj[q] -= d * Ck[q];
        if (gl == 0) R[j * b + k] = rkj - d;
      }
      if (j == k + 1) {
        __syncwarp(gmask);
        prep(j);
      }
    }
    __syncthreads();
  }
}

__device__ long long g_stage[16];
// stage-stamped update loop (no prep) for one thread
template <int G>
__device__ void tsqr_stamp(double* R, double* C, int K, int b, int ldc, double* shr) {
  constexpr int NG = T / G;
  const int tid = threadIdx.x, grp = tid / G, gl = tid % G;
  long long st[5] = {0, 0, 0, 0, 0};
  for (int k = 0; k + 1 < b; ++k) {
    long long c0 = clock64();
    const double tau = shr[k & 1] + 1e-3;
    const double* Ck = C + static_cast<int64_t>(k) * ldc;
    long long c1 = c0, c2 = c0, c3 = c0, c4 = c0;
    for (int j = k + 1 + grp; j < b; j += NG) {
      double* Cj = C + static_cast<int64_t>(j) * ldc;
      const double rkj = R[j * b + k];
      double s0 = 0.0, s1 = 0.0;
      int m = gl;
      for (; m + G < K; m += 2 * G) {
        s0 += Ck[m] * Cj[m];
        s1 += Ck[m + G] * Cj[m + G];
      }
      if (m < K) s0 += Ck[m] * Cj[m];
      double sum = s0 + s1;
      c1 = clock64();
      sum = group_sum<G>(sum, G == 32 ? 0xffffffffu : (((1u << G) - 1u) << ((tid & 31) / G * G)));
      const double d = tau * (rkj + sum);
      c2 = clock64();
      for (int q = gl; q < K; q += G) Cj[q] -= d * Ck[q];
      if (gl == 0) R[j * b + k] = rkj - d;
      c3 = clock64();
    }
    __syncthreads();
    c4 = clock64();
    st[0] += c1 - c0; st[1] += c2 - c1; st[2] += c3 - c2; st[3] += c4 - c3;
  }
  if (tid == 0 && blockIdx.x == 0) for (int q = 0; q < 4; ++q) g_stage[q] = st[q] / (b - 1);
}

template <int G, int E, int NC>
__device__ void tsqr_stamp_t(double* R, double* C, int K, int b, int ldc, double* shr) {
  __builtin_assume(__isShared(R));
  __builtin_assume(__isShared(C));
  constexpr int NG = T / G;
  const int tid = threadIdx.x, grp = tid / G, gl = tid % G;
  const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << ((tid & 31) / G * G));
  double x[NC][E];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int j = grp + c * NG;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int m = gl + e * G;
      x[c][e] = (j < b && m < K) ? C[static_cast<int64_t>(j) * ldc + m] : 0.0;
    }
  }
  // reflector of column j (= grp + c * NG): scale the registers, publish v and tau
  auto prep = [&](double* xc, int j) {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int e = 0; e < E; e += 2) {
      s0 = fma(xc[e], xc[e], s0);
      if (e + 1 < E) s1 = fma(xc[e + 1], xc[e + 1], s1);
    }
    const double x0 = R[j * b + j];  // read before the group shuffle (lane 0 overwrites it)
    const double ss = group_sum<G>(s0 + s1, gmask);
    double tau = 0.0;
    if (ss > 0.0) {
      const double n2 = fma(x0, x0, ss);
      const bool fast = n2 > 1e-290 && n2 < 1e290;  // SFU + Newton only away from under/overflow
      const double nrm = fast ? n2 * rsqrt_nr(n2) : sqrt(n2);
      const double beta = x0 >= 0.0 ? -nrm : nrm;
      const double den = x0 - beta;
      const double scale = fast ? rcp_nr(den) : 1.0 / den;
      tau = fast ? -den * rcp_nr(beta) : (beta - x0) / beta;
      double* Cj = C + static_cast<int64_t>(j) * ldc;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int m = gl + e * G;
        xc[e] *= scale;
        if (m < K) Cj[m] = xc[e];
      }
      if (gl == 0) R[j * b + j] = beta;
    }
    if (gl == 0) shr[j & 1] = tau;
  };
  if (grp == 0 && b > 0) prep(x[0], 0);
  __syncthreads();
  long long st[6] = {0, 0, 0, 0, 0, 0};
  const long long tloop0 = clock64();
  for (int k = 0; k + 1 < b; ++k) {
    long long c0 = clock64();
    const double tau = shr[k & 1];
    if (tau != 0.0) {
      const double* Ck = C + static_cast<int64_t>(k) * ldc;
      // partial dots of every owned column against v_k (v read once), then the update
      // (v re-read: keeping it in registers as well would spill for NC > 1)
      double sd[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) sd[c] = 0.0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int m = gl + e * G;
        const double ve = m < K ? Ck[m] : 0.0;
#pragma unroll
        for (int c = 0; c < NC; ++c) sd[c] = fma(ve, x[c][e], sd[c]);
      }
      st[0] += clock64() - c0;
      c0 = clock64();
      double dd[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int j = grp + c * NG;
        dd[c] = 0.0;
        if (j > k && j < b) {
          const double rkj = R[j * b + k];
          dd[c] = tau * (rkj + group_sum<G>(sd[c], gmask));
          if (gl == 0) R[j * b + k] = rkj - dd[c];
        }
      }
      st[1] += clock64() - c0;
      c0 = clock64();
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int m = gl + e * G;
        const double ve = m < K ? Ck[m] : 0.0;
#pragma unroll
        for (int c = 0; c < NC; ++c) x[c][e] = fma(-dd[c], ve, x[c][e]);
      }
      st[2] += clock64() - c0;
    }
    c0 = clock64();
#pragma unroll
    for (int c = 0; c < NC; ++c)
      if (grp + c * NG == k + 1) prep(x[c], k + 1);
    st[3] += clock64() - c0;
    c0 = clock64();
    __syncthreads();
    st[4] += clock64() - c0;
  }
  st[5] = clock64() - tloop0;
  if (blockIdx.x == 0 && (threadIdx.x == 0 || threadIdx.x == G))
    for (int q = 0; q < 6; ++q) g_stage[q + (threadIdx.x == 0 ? 0 : 6)] = st[q] / (b - 1);
}


template <int G, int E, int NC, int MODE>
__device__ __noinline__ void tsqr_abl_t(double* R, double* C, int K, int b, int ldc, double* shr) {
  __builtin_assume(__isShared(R));
  __builtin_assume(__isShared(C));
  constexpr int NG = T / G;
  constexpr unsigned kFull = 0xffffffffu;
  // control flow is warp-uniform around every shuffle (full-mask shuffles: partial masks
  // make the compiler emit MATCH/REDUX convergence checks on the critical path)
  const int tid = threadIdx.x, grp = tid / G, gl = tid % G, warp = tid >> 5;
  const int wmax = ((warp + 1) * 32) / G - 1 + (NC - 1) * NG;  // largest column owned in this warp
  double x[NC][E];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int j = grp + c * NG;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int m = gl + e * G;
      x[c][e] = (j < b && m < K) ? C[static_cast<int64_t>(j) * ldc + m] : 0.0;
    }
  }
  // reflector of column j: every lane of the owner's warp runs it (full-mask shuffles),
  // only the owner group (own) scales its registers and publishes v, beta and tau
  auto prep = [&](double (&xc)[E], int j, bool own) {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int e = 0; e < E; e += 2) {
      s0 = fma(xc[e], xc[e], s0);
      if (e + 1 < E) s1 = fma(xc[e + 1], xc[e + 1], s1);
    }
    const double x0 = R[j * b + j];  // read before the shuffle (lane 0 overwrites it)
    const double ss = group_sum<G>(s0 + s1, kFull);
    if (!own) return;
    if (MODE & 1) {
      if (gl == 0) shr[j & 1] = 1e-3 + 1e-30 * ss;
      return;
    }
    double tau = 0.0;
    if (ss > 0.0) {
      const double n2 = fma(x0, x0, ss);
      const bool fast = n2 > 1e-290 && n2 < 1e290;  // SFU + Newton only away from under/overflow
      const double nrm = fast ? n2 * rsqrt_nr(n2) : sqrt(n2);
      const double beta = x0 >= 0.0 ? -nrm : nrm;
      const double den = x0 - beta;
      const double scale = fast ? rcp_nr(den) : 1.0 / den;
      tau = fast ? -den * rcp_nr(beta) : (beta - x0) / beta;
      double* Cj = C + static_cast<int64_t>(j) * ldc;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int m = gl + e * G;
        xc[e] *= scale;
        if (m < K) Cj[m] = xc[e];
      }
      if (gl == 0) R[j * b + j] = beta;
    }
    if (gl == 0) shr[j & 1] = tau;
  };
  if (warp == 0 && b > 0) prep(x[0], 0, grp == 0);
  __syncthreads();
  for (int k = 0; k + 1 < b; ++k) {
    const double tau = shr[k & 1];
    if (!(MODE & 2) && tau != 0.0 && wmax > k) {
      const double* Ck = C + static_cast<int64_t>(k) * ldc;
      double sd[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) sd[c] = 0.0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int m = gl + e * G;
        const double ve = m < K ? Ck[m] : 0.0;
#pragma unroll
        for (int c = 0; c < NC; ++c) sd[c] = fma(ve, x[c][e], sd[c]);
      }
      double dd[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int j = grp + c * NG;
        const bool valid = j > k && j < b;
        const double rkj = valid ? R[j * b + k] : 0.0;
        const double tot = group_sum<G>(sd[c], kFull);
        dd[c] = valid ? tau * (rkj + tot) : 0.0;
        if (valid && gl == 0) R[j * b + k] = rkj - dd[c];
      }
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int m = gl + e * G;
        const double ve = m < K ? Ck[m] : 0.0;
#pragma unroll
        for (int c = 0; c < NC; ++c) x[c][e] = fma(-dd[c], ve, x[c][e]);
      }
    }
    const int jn = k + 1, og = jn % NG, oc = jn / NG;
    if ((og * G) >> 5 == warp) {
#pragma unroll
      for (int c = 0; c < NC; ++c)
        if (c == oc) prep(x[c], jn, grp == og);
    }
    __syncthreads();
  }
}


// barrier-loop floor: per step LDS of a flag written by one thread + barrier
__device__ __noinline__ void barrier_loop(double* R, double* C, int b, double* shr) {
  double acc = 0.0;
  for (int k = 0; k + 1 < b; ++k) {
    const double t = shr[k & 1];
    if (t != 0.0) acc += t * C[threadIdx.x];
    if (threadIdx.x == (k & 255)) shr[(k + 1) & 1] = acc + 1.0;
    __syncthreads();
  }
  if (acc == 12345.0) R[0] = acc;
}
__device__ __noinline__ void barrier_only(int b) {
  for (int k = 0; k + 1 < b; ++k) __syncthreads();
}

__device__ __forceinline__ double hrand(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  x ^= x >> 31;
  return static_cast<double>(x >> 11) * (1.0 / 9007199254740992.0) - 0.5;
}

__global__ void __launch_bounds__(T) micro_kernel(int which, int b, int K, int reps, unsigned long long* cyc,
                                                  double* out, int* sweeps) {
  extern __shared__ double sm[];
  __shared__ double shr[4];
  const int ldc = K | 1;
  const int ld = pad_ld(b);
  double* R = sm;                 // b x b (tsqr) / X (jacobi, ld)
  double* V = R + b * ld;         // jacobi V
  double* C = V + b * ld;         // K x b chunk
  unsigned long long acc = 0;
  int nsw_tot = 0;
  for (int rep = 0; rep < reps; ++rep) {
    const uint64_t seed = (static_cast<uint64_t>(blockIdx.x) * 1000003ull + rep) * 7919ull;
    if (which != 3 && which != 13 && (which < 30 || which >= 40)) {
      if (which == 50 && threadIdx.x == 0) { shr[0] = 1.0; shr[1] = 1.0; }
      for (int idx = threadIdx.x; idx < b * b; idx += T) R[idx] = 0.0;
      for (int idx = threadIdx.x; idx < K * b; idx += T) C[(idx / K) * ldc + idx % K] = hrand(seed + idx);
    } else {
      for (int idx = threadIdx.x; idx < b * b; idx += T) {
        const int j = idx / b, i = idx % b;
        R[j * ld + i] = i >= j ? hrand(seed + idx) : 0.0;
      }
    }
    __syncthreads();
    const long long t0 = clock64();
    if (which == 0) tsqr_warps(R, C, K, b, ldc, shr);
    else if (which == 1) tsqr_update(R, C, K, b, ldc, shr);
    else if (which == 2) tsqr_group(R, C, K, b, ldc, shr);
    else if (which == 3) nsw_tot += jacobi(R, V, b, ld, b);
    else if (which == 4) tsqr_group_t<4>(R, C, K, b, ldc, shr);
    else if (which == 5) tsqr_group_t<16>(R, C, K, b, ldc, shr);
    else if (which == 6) tsqr_group_t<32>(R, C, K, b, ldc, shr);
    else if (which == 7) tsqr_probe<16, 1>(R, C, K, b, ldc, shr);
    else if (which == 8) tsqr_probe<16, 2>(R, C, K, b, ldc, shr);
    else if (which == 9) tsqr_probe<16, 3>(R, C, K, b, ldc, shr);
    else if (which == 10) tsqr_probe<16, 0>(R, C, K, b, ldc, shr);
    else if (which == 11) tsqr_stamp<16>(R, C, K, b, ldc, shr);
    else if (which == 12) tsqr_fast(R, C, K, b, ldc, shr);
    else if (which == 13) nsw_tot += jacobi_fast(R, V, b, ld, b);
    else if (which == 14) tsqr_reg_t<16, 8, 3>(R, C, K, b, ldc, shr);
    else if (which == 15) tsqr_reg_t<8, 16, 2>(R, C, K, b, ldc, shr);
    else if (which == 16) tsqr_reg_t<4, 32, 1>(R, C, K, b, ldc, shr);
    else if (which == 17) tsqr_reg_t<16, 8, 4>(R, C, K, b, ldc, shr);
    else if (which == 18) tsqr_reg_t<32, 4, 6>(R, C, K, b, ldc, shr);
    else if (which == 19) tsqr_reg_t<8, 16, 1>(R, C, K, b, ldc, shr);
    else if (which == 20) tsqr_reg_t<16, 8, 1>(R, C, K, b, ldc, shr);
    else if (which == 21) tsqr_stamp_t<16, 8, 1>(R, C, K, b, ldc, shr);
    else if (which == 23) tsqr_abl_t<16, 8, 1, 0>(R, C, K, b, ldc, shr);
    else if (which == 40) tsqr_blk_t<16, 8, 1, 8>(R, C, K, b, ldc, shr);
    else if (which == 41) tsqr_blk_t<8, 16, 1, 8>(R, C, K, b, ldc, shr);
    else if (which == 42) tsqr_blk_t<8, 16, 2, 4>(R, C, K, b, ldc, shr);
    else if (which == 43) tsqr_blk_t<8, 16, 2, 8>(R, C, K, b, ldc, shr);
    else if (which == 44) tsqr_blk_t<16, 8, 3, 8>(R, C, K, b, ldc, shr);
    else if (which == 50) barrier_loop(R, C, b, shr);
    else if (which == 51) barrier_only(b);
    else if (which == 30) nsw_tot += jacobi_t<1, 16>(R, V, b, ld, b);
    else if (which == 31) nsw_tot += jacobi_t<2, 8>(R, V, b, ld, b);
    else if (which == 32) nsw_tot += jacobi_t<4, 4>(R, V, b, ld, b);
    else if (which == 33) nsw_tot += jacobi_t<8, 2>(R, V, b, ld, b);
    else if (which == 34) nsw_tot += jacobi_t<16, 1>(R, V, b, ld, b);
    else if (which == 35) nsw_tot += jacobi_t<1, 40>(R, V, b, ld, b);
    else if (which == 36) nsw_tot += jacobi_t<2, 20>(R, V, b, ld, b);
    else if (which == 37) nsw_tot += jacobi_t<4, 10>(R, V, b, ld, b);
    else if (which == 38) nsw_tot += jacobi_t<8, 5>(R, V, b, ld, b);
    else if (which == 24) tsqr_abl_t<16, 8, 1, 1>(R, C, K, b, ldc, shr);
    else if (which == 25) tsqr_abl_t<16, 8, 1, 2>(R, C, K, b, ldc, shr);
    else if (which == 26) tsqr_abl_t<16, 8, 1, 3>(R, C, K, b, ldc, shr);
    else if (which == 22) tsqr_stamp_t<16, 8, 3>(R, C, K, b, ldc, shr);
    __syncthreads();
    const long long t1 = clock64();
    acc += static_cast<unsigned long long>(t1 - t0);
  }
  if (threadIdx.x == 0) {
    cyc[blockIdx.x] = acc / reps;
    sweeps[blockIdx.x] = nsw_tot;
    if (blockIdx.x == 0)
      for (int k = 0; k < b; ++k) out[k] = (which != 3 && which != 13 && (which < 30 || which >= 40)) ? fabs(R[k * b + k]) : R[k * ld + k];
  }
}

__global__ void lat_kernel(double* out, long long* cyc, double seed) {
  __shared__ int chase[1024];
  __shared__ double dchase[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
    chase[i] = (i * 37 + 11) & 1023;
    dchase[i] = 1.0 + 1e-9 * i;
  }
  __syncthreads();
  double x = seed + threadIdx.x * 1e-3, y = 0.999999;
  long long t0 = clock64();
  for (int i = 0; i < 1024; ++i) x = fma(x, y, 1e-7);
  long long t1 = clock64();
  int p = threadIdx.x & 1023;
  for (int i = 0; i < 1024; ++i) p = chase[p];
  long long t2 = clock64();
  for (int i = 0; i < 1024; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1e-9;
  long long t3 = clock64();
  for (int i = 0; i < 128; ++i) x = 1.0 / (x + 1.5);
  long long t4 = clock64();
  for (int i = 0; i < 128; ++i) x = sqrt(x + 1.5);
  long long t5 = clock64();
  for (int i = 0; i < 128; ++i) x = rsqrt(x + 1.5);
  long long t6 = clock64();
  double z = 0.0;
  for (int i = 0; i < 1024; ++i) z = dchase[(p + i + static_cast<int>(z)) & 1023] - 1.0;
  long long t7 = clock64();
  for (int i = 0; i < 128; ++i) x = (x + 0.5) / (x + 1.5);
  long long t8 = clock64();
  __syncthreads();
  long long t9 = clock64();
  for (int i = 0; i < 1024; ++i) __syncthreads();
  long long t10 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = (t1 - t0) / 1024; cyc[1] = (t2 - t1) / 1024; cyc[2] = (t3 - t2) / 1024; cyc[3] = (t4 - t3) / 128;
    cyc[4] = (t5 - t4) / 128; cyc[5] = (t6 - t5) / 128; cyc[6] = (t7 - t6) / 1024; cyc[7] = (t8 - t7) / 128;
    cyc[8] = (t10 - t9) / 1024;
  }
  out[threadIdx.x] = x + p + z;
}

__global__ void thr_kernel(double* out, long long* cyc, int mode) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double y = 0.999999;
  __syncthreads();
  long long t0 = clock64();
  if (mode == 0) {
    for (int i = 0; i < 256; ++i) {
      a0 = fma(a0, y, 1e-7); a1 = fma(a1, y, 1e-7); a2 = fma(a2, y, 1e-7); a3 = fma(a3, y, 1e-7);
      a4 = fma(a4, y, 1e-7); a5 = fma(a5, y, 1e-7); a6 = fma(a6, y, 1e-7); a7 = fma(a7, y, 1e-7);
    }
  } else if (mode == 1) {
    for (int i = 0; i < 256; ++i) {
      a0 += __shfl_xor_sync(0xffffffffu, a1, 1); a1 += __shfl_xor_sync(0xffffffffu, a2, 2);
      a2 += __shfl_xor_sync(0xffffffffu, a3, 4); a3 += __shfl_xor_sync(0xffffffffu, a0, 8);
    }
  } else {
    float f0 = a0, f1 = a1, f2 = a2, f3 = a3, f4 = a4, f5 = a5, f6 = a6, f7 = a7;
    const float yf = 0.999f;
    for (int i = 0; i < 256; ++i) {
      f0 = fmaf(f0, yf, 1e-7f); f1 = fmaf(f1, yf, 1e-7f); f2 = fmaf(f2, yf, 1e-7f); f3 = fmaf(f3, yf, 1e-7f);
      f4 = fmaf(f4, yf, 1e-7f); f5 = fmaf(f5, yf, 1e-7f); f6 = fmaf(f6, yf, 1e-7f); f7 = fmaf(f7, yf, 1e-7f);
    }
    a0 = f0 + f1 + f2 + f3 + f4 + f5 + f6 + f7;
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

}  // namespace
}  // namespace ceg

int main() {
  using namespace ceg;
  setvbuf(stdout, nullptr, _IONBF, 0);
  int dev = 0;
  cudaSetDevice(dev);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (getenv("MICRO_CPS") ? atoi(getenv("MICRO_CPS")) : 2) * nsm;
  unsigned long long* d_cyc;
  double* d_out;
  int* d_sw;
  cudaMalloc(&d_cyc, grid * sizeof(unsigned long long));
  cudaMalloc(&d_out, 1024 * sizeof(double));
  cudaMalloc(&d_sw, grid * sizeof(int));
  cudaFuncSetAttribute(micro_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  {
    long long* d_l;
    double* d_o;
    cudaMalloc(&d_l, 16 * sizeof(long long));
    cudaMalloc(&d_o, 1024 * sizeof(double));
    for (int mode = 0; mode < 0; ++mode)
      for (int nt : {32, 128, 256, 512, 1024}) {
        thr_kernel<<<1, nt>>>(d_o, d_l, mode);
        cudaDeviceSynchronize();
        long long l;
        cudaMemcpy(&l, d_l, sizeof(l), cudaMemcpyDeviceToHost);
        const double ops = (mode == 1 ? 4.0 : 8.0) * 256 * nt / 32;  // warp-instructions
        std::printf("throughput mode %d (%s) threads %4d: %lld cycles, %.3f warp-instr/cycle/SM\n", mode,
                    mode == 0 ? "dfma" : (mode == 1 ? "shfl64" : "ffma"), nt, l, ops / l);
      }
  }
  if (!getenv("MICRO_CASE")) {
    long long* d_l;
    cudaMalloc(&d_l, 16 * sizeof(long long));
    for (int nt : {32}) {
      lat_kernel<<<1, nt>>>(d_out, d_l, 0.5);
      cudaDeviceSynchronize();
      long long l[16];
      cudaMemcpy(l, d_l, sizeof(l), cudaMemcpyDeviceToHost);
      std::printf("latency (threads %d): dfma %lld lds %lld shfl64+dadd %lld 1/x %lld sqrt %lld rsqrt %lld lds64+cvt %lld div %lld bar %lld\n",
                  nt, l[0], l[1], l[2], l[3], l[4], l[5], l[6], l[7], l[8]);
    }
  }
  struct Case { int which, b, K; };
  const Case cases[] = {{50, 64, 64}, {51, 64, 64}, {12, 16, 128}};
  const char* names[] = {"tsqr_warps", "tsqr_update", "tsqr_group", "jacobi", "tsqr_g4", "tsqr_g16", "tsqr_g32", "noprep", "noupdate", "fastdiv", "probe_full", "stamp", "tsqr_fast", "jacobi_fast", "reg16x8x3", "reg8x16x2", "reg4x32x1", "reg16x8x4", "reg32x4x6", "reg8x16x1", "reg16x8x1", "stamp16", "stamp40", "abl_full", "abl_noprep", "abl_noupd", "abl_none", "", "", "", "j1x16", "j2x8", "j4x4", "j8x2", "j16x1", "j1x40", "j2x20", "j4x10", "j8x5", "", "blk16", "blk32", "blk40nb4", "blk40nb8", "blk40g16", "", "", "", "", "", "barrier_loop", "barrier_only"};
  const int only = getenv("MICRO_CASE") ? atoi(getenv("MICRO_CASE")) : -1;
  for (const Case& c : cases) {
    if (only >= 0 && c.which != only) continue;
    const int ld = c.b | 1;
    const size_t smem = (2 * c.b * ld + (c.K | 1) * c.b + 64) * sizeof(double);
    const int reps = 20;
    micro_kernel<<<grid, T, smem>>>(c.which, c.b, c.K, reps, d_cyc, d_out, d_sw);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      std::printf("error %s\n", cudaGetErrorString(e));
      return 1;
    }
    std::vector<unsigned long long> cyc(grid);
    std::vector<int> sw(grid);
    std::vector<double> out(c.b);
    cudaMemcpy(cyc.data(), d_cyc, grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    cudaMemcpy(sw.data(), d_sw, grid * sizeof(int), cudaMemcpyDeviceToHost);
    cudaMemcpy(out.data(), d_out, c.b * sizeof(double), cudaMemcpyDeviceToHost);
    double mean = 0, sws = 0;
    for (int g = 0; g < grid; ++g) {
      mean += static_cast<double>(cyc[g]) / grid;
      sws += static_cast<double>(sw[g]) / grid / reps;
    }
    std::printf("%-12s b=%3d K=%3d  cycles/call %9.0f  (%.1f us @1.9GHz)", names[c.which], c.b, c.K, mean,
                mean / 1900.0);
    if (c.which == 3 || c.which == 13 || (c.which >= 30 && c.which < 40)) std::printf("  sweeps %.2f  cycles/round %.0f", sws, mean / (sws * ((c.b + (c.b & 1)) - 1)));
    std::printf("  out[0..2] %.6f %.6f %.6f\n", out[0], out[1], out[2]);
    if (c.which == 21 || c.which == 22) {
      long long st[16];
      cudaMemcpyFromSymbol(st, g_stage, sizeof(st));
      std::printf("   thread0: v+dot %lld  reduce %lld  update %lld  prep %lld  barrier %lld  loop/step %lld\n", st[0], st[1], st[2], st[3], st[4], st[5]);
      std::printf("   thread G: v+dot %lld  reduce %lld  update %lld  prep %lld  barrier %lld  loop/step %lld\n", st[6], st[7], st[8], st[9], st[10], st[11]);
    }
    if (c.which == 11) {
      long long st[8];
      cudaMemcpyFromSymbol(st, g_stage, sizeof(st));
      std::printf("   stage cycles/step: dot %lld  reduce %lld  update %lld  barrier %lld\n", st[0], st[1], st[2], st[3]);
    }
  }
  return 0;
}
