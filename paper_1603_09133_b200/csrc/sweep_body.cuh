// Level-sweep kernel body (included twice by sweep.cu, see there): task graph
// walker, TSQR / Jacobi SVD / canonical basis / pivot Cholesky / strip / Schur
// panels.  CE_SMEM_BUFFER selects where the per-CTA work buffer lives.
#if CE_SMEM_BUFFER
#define CE_SHARED(p) __builtin_assume(__isShared(p))
#else
#define CE_SHARED(p) ((void)0)
#endif
// all tiles of a (local copy of a) Buf
#define CE_SHARED_BUF(s)                                                                             \
  do {                                                                                               \
    CE_SHARED(s.R); CE_SHARED(s.V); CE_SHARED(s.U); CE_SHARED(s.D); CE_SHARED(s.C);               \
    CE_SHARED(s.sig); CE_SHARED(s.tau); CE_SHARED(s.nrm); CE_SHARED(s.perm);                       \
  } while (0)

struct Buf {
  double *R, *V, *U, *D, *C, *sig, *tau, *nrm;
  int* perm;
};

__device__ Buf carve(double* base, int bmax, int kcap) {
  Buf s;
  const Layout L = sweep_layout(bmax, kcap);
  s.R = base;
  s.V = s.R + L.bb;
  s.U = s.V + L.bb;
  s.D = s.U + L.bb;
  s.C = s.D + L.bb;
  s.sig = s.C + L.creg + L.extra;
  s.tau = s.sig + bmax;
  s.nrm = s.tau + bmax;
  s.perm = reinterpret_cast<int*>(s.nrm + bmax);
  return s;
}

// Structured Householder QR update [R; C] -> [R'; 0].  R: b x b column-major
// (R[k][j] at R[j*b+k]); C: K x b column-major with odd leading dimension ldc
// (element (m, j) at C[j*ldc+m]).  One thread per column: step k applies reflector
// k to every column j > k, and the owner of column k+1 prepares reflector k+1 right
// after its own update, so each step costs a single barrier.  LAPACK dlarfg conventions.
__device__ void tsqr_update(double* R, double* C, int K, int b, int ldc, double* shr) {
  if (threadIdx.x == 0 && b > 0) {
    double beta;
    const double tau = house_prep(R[0], C, K, &beta);
    if (tau != 0.0) R[0] = beta;
    shr[0] = tau;
  }
  __syncthreads();
  for (int k = 0; k + 1 < b; ++k) {
    const double tau = shr[k & 1];
    for (int j = k + 1 + threadIdx.x; j < b; j += T) {
      double* Cj = C + static_cast<int64_t>(j) * ldc;
      if (tau != 0.0) {
        const double* Ck = C + static_cast<int64_t>(k) * ldc;
        const double d = tau * dot4(R[j * b + k], Ck, Cj, K);
        R[j * b + k] -= d;
        for (int m = 0; m < K; ++m) Cj[m] -= d * Ck[m];
      }
      if (j == k + 1) {
        double beta;
        const double t1 = house_prep(R[j * b + j], Cj, K, &beta);
        if (t1 != 0.0) R[j * b + j] = beta;
        shr[(k + 1) & 1] = t1;
      }
    }
    __syncthreads();
  }
}

// Group variant of tsqr_update: G lanes per column (partial dots combined with xor
// shuffles inside the group), T / G columns per pass, one barrier per step; the group
// owning column k + 1 prepares reflector k + 1 after its update.
template <int G>
__device__ void tsqr_group_t(double* R, double* C, int K, int b, int ldc, double* shr) {
  constexpr int NG = T / G;
  const int tid = threadIdx.x, grp = tid / G, gl = tid % G;
  const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << ((tid & 31) / G * G));
  auto prep = [&](int j) {
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
      const double scale = 1.0 / (x0 - beta);
      for (int q = gl; q < K; q += G) Cj[q] *= scale;
      tau = (beta - x0) / beta;
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
      if (tau != 0.0) {
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

__device__ void tsqr_group(double* R, double* C, int K, int b, int ldc, double* shr) {
  if (b <= 16) tsqr_group_t<16>(R, C, K, b, ldc, shr);
  else if (b <= 32) tsqr_group_t<8>(R, C, K, b, ldc, shr);
  else tsqr_group_t<8>(R, C, K, b, ldc, shr);
}

// Register-resident Householder QR update [R; C] -> [R'; 0] (same contract as
// tsqr_update).  A group of G lanes keeps NC columns of the chunk in registers
// (E = K / G elements per lane, K <= G * E); per step only the reflector is read
// from shared memory (the owner writes it back into its chunk column), so shared
// traffic per step is one K-vector per warp instead of five per column.
template <int G, int E, int NC>
__device__ __noinline__ void tsqr_reg_t(double* R, double* C, int K, int b, int ldc, double* shr) {
  CE_SHARED(R);
  CE_SHARED(C);
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
    if (tau != 0.0 && wmax > k) {
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

// Blocked TSQR update (same contract as tsqr_update): panels of NB columns are factored
// by warp 0 alone (rows spread over lanes, columns in registers: no CTA barrier inside
// the panel), then every group applies the panel's NB reflectors to the columns it keeps
// in registers (reflectors read-only in shared memory: no barriers between them).  Two
// barriers per panel instead of one per column.
template <int G, int E, int NC, int NB>
__device__ __noinline__ void tsqr_blk_t(double* R, double* C, int K, int b, int ldc, double* shr) {
  CE_SHARED(R);
  CE_SHARED(C);
  constexpr int NG = T / G;
  constexpr int EP = 4;  // panel rows per lane (K <= 128)
  constexpr unsigned kFull = 0xffffffffu;
  __shared__ double ptau[NB];
  const int tid = threadIdx.x, grp = tid / G, gl = tid % G, warp = tid >> 5, lane = tid & 31;
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
  for (int p0 = 0; p0 < b; p0 += NB) {
    const int nb = b - p0 < NB ? b - p0 : NB;
    if (p0 > 0) {  // owners publish the (updated) panel columns
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int j = grp + c * NG;
        if (j >= p0 && j < p0 + nb)
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int m = gl + e * G;
            if (m < K) C[static_cast<int64_t>(j) * ldc + m] = x[c][e];
          }
      }
    }
    __syncthreads();
    if (warp == 0) {
      double pc[NB][EP];
#pragma unroll
      for (int jj = 0; jj < NB; ++jj)
#pragma unroll
        for (int e = 0; e < EP; ++e) {
          const int m = lane + 32 * e;
          pc[jj][e] = (jj < nb && m < K) ? C[static_cast<int64_t>(p0 + jj) * ldc + m] : 0.0;
        }
#pragma unroll
      for (int kk = 0; kk < NB; ++kk) {
        if (kk >= nb) break;
        const int k = p0 + kk;
        double ss = 0.0;
#pragma unroll
        for (int e = 0; e < EP; ++e) ss = fma(pc[kk][e], pc[kk][e], ss);
        const double x0 = R[k * b + k];
        ss = warp_sum(ss);
        double t = 0.0;
        if (ss > 0.0) {
          const double n2 = fma(x0, x0, ss);
          const bool fast = n2 > 1e-290 && n2 < 1e290;
          const double nrm = fast ? n2 * rsqrt_nr(n2) : sqrt(n2);
          const double beta = x0 >= 0.0 ? -nrm : nrm;
          const double den = x0 - beta;
          const double scale = fast ? rcp_nr(den) : 1.0 / den;
          t = fast ? -den * rcp_nr(beta) : (beta - x0) / beta;
#pragma unroll
          for (int e = 0; e < EP; ++e) pc[kk][e] *= scale;
          __syncwarp();
          if (lane == 0) R[k * b + k] = beta;
        }
        if (lane == 0) ptau[kk] = t;
        if (t != 0.0) {
          double dsum[NB];
#pragma unroll
          for (int jj = 0; jj < NB; ++jj) {
            dsum[jj] = 0.0;
            if (jj > kk)
#pragma unroll
              for (int e = 0; e < EP; ++e) dsum[jj] = fma(pc[kk][e], pc[jj][e], dsum[jj]);
          }
#pragma unroll
          for (int jj = 0; jj < NB; ++jj)
            if (jj > kk) dsum[jj] = warp_sum(dsum[jj]);
#pragma unroll
          for (int jj = 0; jj < NB; ++jj) {
            if (jj <= kk || jj >= nb) continue;
            const double rkj = R[(p0 + jj) * b + k];
            const double d = t * (rkj + dsum[jj]);
#pragma unroll
            for (int e = 0; e < EP; ++e) pc[jj][e] = fma(-d, pc[kk][e], pc[jj][e]);
            __syncwarp();
            if (lane == 0) R[(p0 + jj) * b + k] = rkj - d;
          }
        }
      }
      // reflector tails back to the panel columns of C
#pragma unroll
      for (int jj = 0; jj < NB; ++jj)
#pragma unroll
        for (int e = 0; e < EP; ++e) {
          const int m = lane + 32 * e;
          if (jj < nb && m < K) C[static_cast<int64_t>(p0 + jj) * ldc + m] = pc[jj][e];
        }
    }
    __syncthreads();
    // trailing columns: apply the panel's reflectors (read-only) without barriers
    for (int kk = 0; kk < nb; ++kk) {
      const double t = ptau[kk];
      if (t == 0.0) continue;
      const int k = p0 + kk;
      const double* Ck = C + static_cast<int64_t>(k) * ldc;
      double v[E];
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int m = gl + e * G;
        v[e] = m < K ? Ck[m] : 0.0;
      }
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int j = grp + c * NG;
        double sd = 0.0;
#pragma unroll
        for (int e = 0; e < E; ++e) sd = fma(v[e], x[c][e], sd);
        sd = group_sum<G>(sd, kFull);
        if (j >= p0 + nb && j < b) {
          const double rkj = R[j * b + k];
          const double d = t * (rkj + sd);
#pragma unroll
          for (int e = 0; e < E; ++e) x[c][e] = fma(-d, v[e], x[c][e]);
          if (gl == 0) R[j * b + k] = rkj - d;
        }
      }
    }
  }
  __syncthreads();
  (void)shr;
}

// Dispatch: register-resident variants for b <= 64 and K <= 128, else the generic one.
__device__ void tsqr_fast(double* R, double* C, int K, int b, int ldc, double* shr) {
  if (K <= 128 && b <= 16) tsqr_reg_t<16, 8, 1>(R, C, K, b, ldc, shr);
  else if (K <= 128 && b <= 32) tsqr_reg_t<8, 16, 1>(R, C, K, b, ldc, shr);
  else if (K <= 128 && b <= 64) tsqr_reg_t<8, 16, 2>(R, C, K, b, ldc, shr);
#if CE_KCAP > 128
  // taller combine chunks (more children per TSQR tree node)
  else if (K <= 192 && b <= 16) tsqr_reg_t<16, 12, 1>(R, C, K, b, ldc, shr);
  else if (K <= 192 && b <= 32) tsqr_reg_t<8, 24, 1>(R, C, K, b, ldc, shr);
  else if (K <= 192 && b <= 64) tsqr_reg_t<8, 24, 2>(R, C, K, b, ldc, shr);
#endif
  else tsqr_group(R, C, K, b, ldc, shr);
}

// One-sided Jacobi (Hestenes) on the columns of X (b x b, column-major, odd leading
// dimension ld); V (same layout) accumulates the rotations.  Round-robin rounds of
// disjoint column pairs; a group of G lanes owns one pair, partial dots are combined
// with xor shuffles inside the group.  Small blocks (all pairs fit one warp) run on
// warp 0 with no CTA barrier; larger ones use the whole CTA with one barrier per round.
// Rotation test |gamma| > tol sqrt(alpha beta), tol = sqrt(m) eps (oracle/dense.cpp svd_left).
__device__ int jacobi(double* X, double* V, int b, int ld, int meff) {
  const int tid = threadIdx.x;
  for (int idx = tid; idx < b * ld; idx += T) V[idx] = (idx / ld == idx % ld) ? 1.0 : 0.0;
  __syncthreads();
  const double tol = sqrt(static_cast<double>(meff > 1 ? meff : 1)) * DBL_EPSILON;
  const double tol2 = tol * tol;
  const int nb = b + (b & 1);
  const int np = nb / 2;
  int G = 1;
  while (G < 16 && np * G * 2 <= T) G *= 2;
  const bool one_warp = np * 4 <= 32;
  if (one_warp) G = 32 / np >= 8 ? 8 : (32 / np >= 4 ? 4 : 2);
  const int pi = tid / G, gl = tid % G;
  __shared__ int s_sweeps;
  if (one_warp && tid >= 32) {
    __syncthreads();
    return s_sweeps;
  }
  int nsw = 100;
  for (int sweep = 0; sweep < 100; ++sweep) {
    int rotated = 0;
    for (int round = 0; round < nb - 1; ++round) {
      for (int base = 0; base < np; base += T / G) {
        int p = 0, q = b;
        if (base + pi < np) {
          p = rr_player(base + pi, round, nb);
          q = rr_player(nb - 1 - base - pi, round, nb);
          if (p > q) {
            const int t = p;
            p = q;
            q = t;
          }
        }
        const bool valid = q < b;
        double al = 0.0, be = 0.0, ga = 0.0;
        double* cp = X + p * ld;
        double* cq = X + q * ld;
        if (valid) {
          for (int k = gl; k < b; k += G) {
            const double x = cp[k], y = cq[k];
            al += x * x;
            be += y * y;
            ga += x * y;
          }
        }
        for (int o = G >> 1; o > 0; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          ga += __shfl_xor_sync(0xffffffffu, ga, o);
        }
        if (valid && al != 0.0 && be != 0.0 && ga * ga > tol2 * al * be) {
          const double zeta = (be - al) / (2.0 * ga);
          const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double cs = rsqrt(1.0 + t * t);
          const double sn = cs * t;
          for (int k = gl; k < b; k += G) {
            const double x = cp[k], y = cq[k];
            cp[k] = cs * x - sn * y;
            cq[k] = sn * x + cs * y;
          }
          double* vp = V + p * ld;
          double* vq = V + q * ld;
          for (int k = gl; k < b; k += G) {
            const double x = vp[k], y = vq[k];
            vp[k] = cs * x - sn * y;
            vq[k] = sn * x + cs * y;
          }
          rotated = 1;
        }
      }
      if (one_warp) __syncwarp();
      else if (round < nb - 2) __syncthreads();
    }
    const int any = one_warp ? __any_sync(0xffffffffu, rotated) : __syncthreads_or(rotated);
    if (!any) {
      nsw = sweep + 1;
      break;
    }
  }
  if (one_warp) {
    if (tid == 0) s_sweeps = nsw;
    __syncthreads();
  }
  return nsw;
}

// Unrolled one-sided Jacobi for b <= G * E: G lanes per column pair, the pair's two
// columns held in registers for the round (E elements per lane); only the first
// roundup(np * G, 32) threads take part (warp-synchronous when that is one warp).
// Angle: t = sign(d) 2g / (|d| + sqrt(d^2 + 4g^2)) with d = beta - alpha, the same
// root as oracle/dense.cpp (zeta = d / 2g), from SFU approximations + Newton steps.
template <int G, int E>
__device__ __noinline__ int jacobi_t(double* X, double* V, int b, int ld, int meff) {
  CE_SHARED(X);
  CE_SHARED(V);
  const int tid = threadIdx.x;
  for (int idx = tid; idx < b * ld; idx += T) V[idx] = (idx / ld == idx % ld) ? 1.0 : 0.0;
  const int nb = b + (b & 1), np = nb / 2, nr = nb - 1;
  const int nact = (np * G + 31) & ~31;
  __shared__ int s_sweeps;
  __syncthreads();
  if (tid >= nact) {
    __syncthreads();
    return s_sweeps;
  }
  const double tol = sqrt(static_cast<double>(meff > 1 ? meff : 1)) * DBL_EPSILON;
  const double tol2 = tol * tol;
  const int pi = tid / G, gl = tid % G;
  int nsw = 100;
  for (int sweep = 0; sweep < 100; ++sweep) {
    int rotated = 0;
    for (int round = 0; round < nr; ++round) {
      // round-robin players of pair pi: 0 and nb-1-pi rotate through 1..nb-1
      int p = 0, q = b;
      if (pi < np) {
        int a = pi - 1 + round;
        a = pi == 0 ? -1 : (a >= nr ? a - nr : a);
        int c = nb - 2 - pi + round;
        c = c >= nr ? c - nr : c;
        p = a + 1;
        q = c + 1;
        if (p > q) {
          const int t = p;
          p = q;
          q = t;
        }
      }
      const bool valid = q < b;
      double* cp = X + p * ld;
      double* cq = X + (valid ? q : p) * ld;
      double x[E], y[E];
      double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int k = gl + e * G;
        const bool in = valid && k < b;
        x[e] = in ? cp[k] : 0.0;
        y[e] = in ? cq[k] : 0.0;
        al = fma(x[e], x[e], al);
        be = fma(y[e], y[e], be);
        ga = fma(x[e], y[e], ga);
      }
#pragma unroll
      for (int o = G >> 1; o > 0; o >>= 1) {
        al += __shfl_xor_sync(0xffffffffu, al, o);
        be += __shfl_xor_sync(0xffffffffu, be, o);
        ga += __shfl_xor_sync(0xffffffffu, ga, o);
      }
      // rotation test |gamma| > tol sqrt(alpha) sqrt(beta), squared unless alpha beta underflows
      const double ab = al * be;
      const bool rot = valid && al != 0.0 && be != 0.0 &&
                       (ab > 1e-290 ? ga * ga > tol2 * ab : fabs(ga) > tol * sqrt(al) * sqrt(be));
      if (rot) {
        const double d = be - al;
        const double g2 = ga + ga;
        const double hh = fma(d, d, g2 * g2);
        double t;
        if (hh > 1e-290 && hh < 1e290) {
          const double h = hh * rsqrt_nr(hh);
          t = (d >= 0.0 ? g2 : -g2) * rcp_nr(fabs(d) + h);
        } else {  // extreme magnitudes: the oracle's IEEE formula
          const double zeta = d / g2;
          t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        }
        const double cs = rsqrt_nr(fma(t, t, 1.0));
        const double sn = cs * t;
        double* vp = V + p * ld;
        double* vq = V + q * ld;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int k = gl + e * G;
          if (k < b) {
            cp[k] = cs * x[e] - sn * y[e];
            cq[k] = sn * x[e] + cs * y[e];
            const double u = vp[k], w = vq[k];
            vp[k] = cs * u - sn * w;
            vq[k] = sn * u + cs * w;
          }
        }
        rotated = 1;
      }
      if (nact == 32) __syncwarp();
      else if (round + 1 < nr) bar_n(nact);
    }
    const int any = nact == 32 ? __any_sync(0xffffffffu, rotated) : bar_or(nact, rotated);
    if (!any) {
      nsw = sweep + 1;
      break;
    }
  }
  if (tid == 0) s_sweeps = nsw;
  __syncthreads();
  return nsw;
}

// Wide blocks (64 < b <= 256, typically 3-D deep levels whose tiles live in global scratch):
// a whole warp per column pair, both columns and both V columns held in registers for the
// step (all loads of a pair in flight together instead of a dependent loop over the rows),
// warp-shuffle dot products.  Same rotation arithmetic and stopping rule as `jacobi`.
__device__ __noinline__ int jacobi_wide(double* X, double* V, int b, int ld, int meff) {
  constexpr int E = 8;  // b <= 32 E
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int idx = tid; idx < b * ld; idx += T) V[idx] = (idx / ld == idx % ld) ? 1.0 : 0.0;
  __syncthreads();
  const double tol = sqrt(static_cast<double>(meff > 1 ? meff : 1)) * DBL_EPSILON;
  const double tol2 = tol * tol;
  const int nb = b + (b & 1);
  const int np = nb / 2;
  int nsw = 100;
  for (int sweep = 0; sweep < 100; ++sweep) {
    int rotated = 0;
    for (int round = 0; round < nb - 1; ++round) {
      for (int pi = warp; pi < np; pi += NW) {
        int p = rr_player(pi, round, nb), q = rr_player(nb - 1 - pi, round, nb);
        if (p > q) {
          const int t = p;
          p = q;
          q = t;
        }
        if (q >= b) continue;  // warp-uniform
        double* cp = X + p * ld;
        double* cq = X + q * ld;
        double x[E], y[E];
        double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int k = lane + 32 * e;
          x[e] = k < b ? cp[k] : 0.0;
          y[e] = k < b ? cq[k] : 0.0;
        }
#pragma unroll
        for (int e = 0; e < E; ++e) {
          al += x[e] * x[e];
          be += y[e] * y[e];
          ga += x[e] * y[e];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          ga += __shfl_xor_sync(0xffffffffu, ga, o);
        }
        if (al != 0.0 && be != 0.0 && ga * ga > tol2 * al * be) {
          const double zeta = (be - al) / (2.0 * ga);
          const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double cs = rsqrt(1.0 + t * t);
          const double sn = cs * t;
          double* vp = V + p * ld;
          double* vq = V + q * ld;
          double u[E], v[E];
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int k = lane + 32 * e;
            u[e] = k < b ? vp[k] : 0.0;
            v[e] = k < b ? vq[k] : 0.0;
          }
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int k = lane + 32 * e;
            if (k < b) {
              cp[k] = cs * x[e] - sn * y[e];
              cq[k] = sn * x[e] + cs * y[e];
              vp[k] = cs * u[e] - sn * v[e];
              vq[k] = sn * u[e] + cs * v[e];
            }
          }
          rotated = 1;
        }
      }
      if (round < nb - 2) __syncthreads();
    }
    if (!__syncthreads_or(rotated)) {
      nsw = sweep + 1;
      break;
    }
  }
  return nsw;
}

__device__ int jacobi_fast(double* X, double* V, int b, int ld, int meff) {
  // more lanes per pair beats shorter shuffle trees (micro_dense: b=16 897 vs 1174 cycles/round)
  if (b <= 16) return jacobi_t<16, 1>(X, V, b, ld, meff);
  if (b <= 32) return jacobi_t<16, 2>(X, V, b, ld, meff);
  if (b <= 64) return jacobi_t<8, 8>(X, V, b, ld, meff);
  if (b <= 256 && !(CE_NO_WIDE_JACOBI)) return jacobi_wide(X, V, b, ld, meff);
  return jacobi(X, V, b, ld, meff);
}

// Register-resident Householder QR of a b x b column-major matrix A (leading dimension
// ld) in place: R in the upper triangle, reflector tails below the diagonal, tau[k]
// (LAPACK dlarfg conventions, same results layout as the thread-per-column loop).  Groups
// of G lanes own NC columns (E rows per lane); the owner of column k+1 prepares reflector
// k+1 right after its update and publishes it in a double buffer (vb0 / vb1, b doubles
// each); one barrier per step.
template <int G, int E, int NC>
__device__ __noinline__ void hqr_reg_t(double* A, int b, int ld, double* tau, double* vb0, double* vb1) {
  CE_SHARED(A);
  CE_SHARED(tau);
  CE_SHARED(vb0);
  CE_SHARED(vb1);
  constexpr int NG = T / G;
  constexpr unsigned kFull = 0xffffffffu;
  const int tid = threadIdx.x, grp = tid / G, gl = tid % G, warp = tid >> 5;
  const int wmax = ((warp + 1) * 32) / G - 1 + (NC - 1) * NG;
  double x[NC][E];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int j = grp + c * NG;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int m = gl + e * G;
      x[c][e] = (j < b && m < b) ? A[j * ld + m] : 0.0;
    }
  }
  auto prep = [&](double (&xc)[E], int j, bool own) {
    double ss = 0.0, x0 = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int m = gl + e * G;
      if (m > j && m < b) ss = fma(xc[e], xc[e], ss);
      if (m == j) x0 = xc[e];
    }
    ss = group_sum<G>(ss, kFull);
    x0 = group_sum<G>(x0, kFull);
    if (!own) return;
    double* vb = (j & 1) ? vb1 : vb0;
    double t = 0.0;
    if (ss > 0.0) {
      const double n2 = fma(x0, x0, ss);
      const bool fast = n2 > 1e-290 && n2 < 1e290;
      const double nrm = fast ? n2 * rsqrt_nr(n2) : sqrt(n2);
      const double beta = x0 >= 0.0 ? -nrm : nrm;
      const double den = x0 - beta;
      const double scale = fast ? rcp_nr(den) : 1.0 / den;
      t = fast ? -den * rcp_nr(beta) : (beta - x0) / beta;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int m = gl + e * G;
        if (m >= b) continue;
        if (m > j) {
          xc[e] *= scale;
          vb[m] = xc[e];
        } else if (m == j) {
          xc[e] = beta;
          vb[m] = 1.0;
        } else {
          vb[m] = 0.0;
        }
      }
    }
    if (gl == 0) tau[j] = t;
  };
  if (warp == 0 && b > 0) prep(x[0], 0, grp == 0);
  __syncthreads();
  for (int k = 0; k + 1 < b; ++k) {
    const double t = tau[k];
    if (t != 0.0 && wmax > k) {
      const double* vb = (k & 1) ? vb1 : vb0;
      double v[E];
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int m = gl + e * G;
        v[e] = m < b ? vb[m] : 0.0;
      }
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int j = grp + c * NG;
        double sd = 0.0;
#pragma unroll
        for (int e = 0; e < E; ++e) sd = fma(v[e], x[c][e], sd);
        sd = group_sum<G>(sd, kFull);
        const double d = (j > k && j < b) ? t * sd : 0.0;
#pragma unroll
        for (int e = 0; e < E; ++e) x[c][e] = fma(-d, v[e], x[c][e]);
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
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int j = grp + c * NG;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int m = gl + e * G;
      if (j < b && m < b) A[j * ld + m] = x[c][e];
    }
  }
  __syncthreads();
}

// Householder QR with column pivoting (largest remaining column norm first) of a b x b
// column-major A, register-resident as hqr_reg_t.  Step k: every warp finds the pivot p
// from the published trailing norms (double buffered), the group owning p prepares
// reflector k from rows >= k of column p and records perm[k] = p; after the barrier the
// other groups apply it and downdate their trailing norms (selection only: the reflector
// itself always uses an exact norm).  Result layout: column perm[k] holds R(0..k, k) and
// the tail of reflector k below row k; tau[k].  Rank-revealing R makes the one-sided
// Jacobi on X = R^T converge in fewer sweeps (Drmac-Veselic preconditioning).
constexpr int kQrcpMin = 17;  // block size from which the preconditioning QR pivots (thin level-1 rows converge fast anyway)

template <int G, int E, int NC>
__device__ __noinline__ void hqrcp_reg_t(double* A, int b, int ld, double* tau, double* vb0, double* vb1, int* perm,
                                         double* cn0, double* cn1) {
  CE_SHARED(A);
  CE_SHARED(tau);
  CE_SHARED(vb0);
  CE_SHARED(vb1);
  CE_SHARED(perm);
  CE_SHARED(cn0);
  CE_SHARED(cn1);
  constexpr int NG = T / G;
  constexpr unsigned kFull = 0xffffffffu;
  const int tid = threadIdx.x, grp = tid / G, gl = tid % G, warp = tid >> 5, lane = tid & 31;
  double x[NC][E], n2[NC];
  bool chosen[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int j = grp + c * NG;
    double ss = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int m = gl + e * G;
      x[c][e] = (j < b && m < b) ? A[j * ld + m] : 0.0;
      ss = fma(x[c][e], x[c][e], ss);
    }
    n2[c] = group_sum<G>(ss, kFull);
    chosen[c] = false;
    if (j < b && gl == 0) cn0[j] = n2[c];
  }
  __syncthreads();
  for (int k = 0; k < b; ++k) {
    const double* cn = (k & 1) ? cn1 : cn0;
    double* cnn = (k & 1) ? cn0 : cn1;
    // pivot: largest published norm, ties to the smaller index (every warp, same answer)
    double bv = -2.0;
    int bi = b;
    for (int jj = lane; jj < b; jj += 32) {
      const double v = cn[jj];
      if (v > bv) {
        bv = v;
        bi = jj;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(kFull, bv, o);
      const int oi = __shfl_xor_sync(kFull, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    const int p = bi, pg = p % NG, pc = p / NG;
    if ((pg * G) >> 5 == warp) {
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        if (c != pc) continue;
        const bool own = grp == pg;
        double ss = 0.0, x0 = 0.0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int m = gl + e * G;
          if (m > k && m < b) ss = fma(x[c][e], x[c][e], ss);
          if (m == k) x0 = x[c][e];
        }
        ss = group_sum<G>(ss, kFull);
        x0 = group_sum<G>(x0, kFull);
        if (own) {
          double* vb = (k & 1) ? vb1 : vb0;
          double t = 0.0;
          if (ss > 0.0) {
            const double nn = fma(x0, x0, ss);
            const bool fast = nn > 1e-290 && nn < 1e290;
            const double nrm = fast ? nn * rsqrt_nr(nn) : sqrt(nn);
            const double beta = x0 >= 0.0 ? -nrm : nrm;
            const double den = x0 - beta;
            const double scale = fast ? rcp_nr(den) : 1.0 / den;
            t = fast ? -den * rcp_nr(beta) : (beta - x0) / beta;
#pragma unroll
            for (int e = 0; e < E; ++e) {
              const int m = gl + e * G;
              if (m >= b) continue;
              if (m > k) {
                x[c][e] *= scale;
                vb[m] = x[c][e];
              } else if (m == k) {
                x[c][e] = beta;
                vb[m] = 1.0;
              } else {
                vb[m] = 0.0;
              }
            }
          }
          chosen[c] = true;
          if (gl == 0) {
            tau[k] = t;
            perm[k] = p;
          }
        }
      }
    }
    __syncthreads();
    const double t = tau[k];
    const double* vb = (k & 1) ? vb1 : vb0;
    double v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int m = gl + e * G;
      v[e] = (t != 0.0 && m < b) ? vb[m] : 0.0;
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int j = grp + c * NG;
      const bool live = j < b && !chosen[c];
      double sd = 0.0;
#pragma unroll
      for (int e = 0; e < E; ++e) sd = fma(v[e], x[c][e], sd);
      sd = group_sum<G>(sd, kFull);
      const double d = (live && t != 0.0) ? t * sd : 0.0;
      double xk = 0.0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        x[c][e] = fma(-d, v[e], x[c][e]);
        if (gl + e * G == k) xk = x[c][e];
      }
      xk = group_sum<G>(xk, kFull);  // the row-k entry leaves the trailing part
      n2[c] = fmax(n2[c] - xk * xk, 0.0);
      if (j < b && gl == 0) cnn[j] = live ? n2[c] : -1.0;
    }
    __syncthreads();
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int j = grp + c * NG;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int m = gl + e * G;
      if (j < b && m < b) A[j * ld + m] = x[c][e];
    }
  }
  __syncthreads();
}

// V <- Q2 V, Q2 = H_0 ... H_{b-2} from the reflectors below the diagonal of A: every group
// applies all reflectors to the V columns it keeps in registers; the reflectors are
// read-only, so no barriers are needed between steps.
template <int G, int E, int NC>
__device__ __noinline__ void apply_refl_reg_t(const double* A, const double* tau, double* V, int b, int ld,
                                              const int* perm = nullptr) {
  CE_SHARED(A);
  CE_SHARED(tau);
  CE_SHARED(V);
  constexpr int NG = T / G;
  constexpr unsigned kFull = 0xffffffffu;
  const int tid = threadIdx.x, grp = tid / G, gl = tid % G;
  double x[NC][E];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int j = grp + c * NG;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int m = gl + e * G;
      x[c][e] = (j < b && m < b) ? V[j * ld + m] : 0.0;
    }
  }
  for (int k = b - (perm ? 1 : 2); k >= 0; --k) {
    const double t = tau[k];
    if (t == 0.0) continue;
    double v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int m = gl + e * G;
      v[e] = m == k ? 1.0 : ((m > k && m < b) ? A[(perm ? perm[k] : k) * ld + m] : 0.0);
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      double sd = 0.0;
#pragma unroll
      for (int e = 0; e < E; ++e) sd = fma(v[e], x[c][e], sd);
      const double d = t * group_sum<G>(sd, kFull);
#pragma unroll
      for (int e = 0; e < E; ++e) x[c][e] = fma(-d, v[e], x[c][e]);
    }
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int j = grp + c * NG;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int m = gl + e * G;
      if (j < b && m < b) V[j * ld + m] = x[c][e];
    }
  }
  __syncthreads();
}

// QR preconditioning of the Jacobi SVD (Drmac-Veselic; oracle/dense.cpp svd_left):
// R^T = Q2 R2 by Householder on s.C (b x b column-major, leading dimension pad_ld(b);
// reflectors kept below the diagonal, tau in s.tau), then s.R <- X = R2^T
// (column-major, leading dimension pad_ld(b), lower triangular).  One thread per column,
// the owner of column k + 1 prepares reflector k + 1 right after its own update.
__device__ __noinline__ void precondition_qr(const Buf& s_, int b) {
  const Buf s = s_;
  CE_SHARED_BUF(s);
  const int ld = pad_ld(b);
  double* Aq = s.C;
  for (int idx = threadIdx.x; idx < b * b; idx += T) {
    const int j = idx / b, i = idx % b;  // Aq(i, j) = R^T(i, j) = R(j, i)
    Aq[j * ld + i] = s.R[i * b + j];
  }
  __syncthreads();
  if (b <= 64) {
    if (b >= kQrcpMin) {
      // column-pivoted (pays off beyond the thin level-1 blocks: fewer Jacobi sweeps than the pivot search
      // costs); trailing norms double-buffered in the (still unused) U tile
      if (b <= 32) hqrcp_reg_t<8, 4, 1>(Aq, b, ld, s.tau, s.nrm, s.sig, s.perm, s.U, s.U + b);
      else hqrcp_reg_t<8, 8, 2>(Aq, b, ld, s.tau, s.nrm, s.sig, s.perm, s.U, s.U + b);
      for (int idx = threadIdx.x; idx < b * b; idx += T) {
        const int j = idx / b, i = idx % b;  // X(i, j) = R(j, i) = row j of the step-i pivot column
        s.R[j * ld + i] = i >= j ? Aq[s.perm[i] * ld + j] : 0.0;
      }
    } else {
      if (b <= 16) hqr_reg_t<16, 1, 1>(Aq, b, ld, s.tau, s.nrm, s.sig);
      else if (b <= 32) hqr_reg_t<8, 4, 1>(Aq, b, ld, s.tau, s.nrm, s.sig);
      else hqr_reg_t<8, 8, 2>(Aq, b, ld, s.tau, s.nrm, s.sig);
      for (int idx = threadIdx.x; idx < b * b; idx += T) {
        const int j = idx / b, i = idx % b;
        s.R[j * ld + i] = i >= j ? Aq[i * ld + j] : 0.0;
      }
    }
    __syncthreads();
    return;
  }
  if (threadIdx.x == 0 && b > 0) {
    double beta;
    const double tau = house_prep(Aq[0], Aq + 1, b - 1, &beta);
    if (tau != 0.0) Aq[0] = beta;
    s.tau[0] = tau;
  }
  __syncthreads();
  for (int k = 0; k + 1 < b; ++k) {
    const double tau = s.tau[k];
    const double* Ak = Aq + k * ld;
    for (int j = k + 1 + threadIdx.x; j < b; j += T) {
      double* Aj = Aq + j * ld;
      if (tau != 0.0) {
        const double d = tau * dot4(Aj[k], Ak + k + 1, Aj + k + 1, b - k - 1);
        Aj[k] -= d;
        for (int i = k + 1; i < b; ++i) Aj[i] -= d * Ak[i];
      }
      if (j == k + 1) {
        double beta;
        const double t1 = house_prep(Aj[j], Aj + j + 1, b - j - 1, &beta);
        if (t1 != 0.0) Aj[j] = beta;
        s.tau[j] = t1;
      }
    }
    __syncthreads();
  }
  for (int idx = threadIdx.x; idx < b * b; idx += T) {
    const int j = idx / b, i = idx % b;  // X(i, j) = R2(j, i) for i >= j
    s.R[j * ld + i] = i >= j ? Aq[i * ld + j] : 0.0;
  }
  __syncthreads();
}

// V <- Q2 V with Q2 = H_0 ... H_{b-1} from precondition_qr (V column-major, ld pad_ld(b)).
// One thread per column of V, one barrier per reflector.
__device__ __noinline__ void apply_q2(const Buf& s_, int b) {
  const Buf s = s_;
  CE_SHARED_BUF(s);
  const int ld = pad_ld(b);
  const double* Aq = s.C;
  if (b <= 64) {
    const int* pv = b >= kQrcpMin ? s.perm : nullptr;
    if (b <= 16) apply_refl_reg_t<16, 1, 1>(Aq, s.tau, s.V, b, ld, pv);
    else if (b <= 32) apply_refl_reg_t<8, 4, 1>(Aq, s.tau, s.V, b, ld, pv);
    else apply_refl_reg_t<8, 8, 2>(Aq, s.tau, s.V, b, ld, pv);
    return;
  }
  for (int k = b - 2; k >= 0; --k) {
    const double tau = s.tau[k];
    if (tau == 0.0) continue;
    const double* v = Aq + k * ld;  // v_k = 1, v_i (i > k) below the diagonal
    for (int j = threadIdx.x; j < b; j += T) {
      double* Vj = s.V + j * ld;
      const double d = tau * dot4(Vj[k], v + k + 1, Vj + k + 1, b - k - 1);
      Vj[k] -= d;
      for (int i = k + 1; i < b; ++i) Vj[i] -= d * v[i];
    }
    __syncthreads();
  }
}

// Canonical gauge (oracle/dense.cpp canonical_basis): U1 = leading singular
// vectors (clusters of equal singular values -> orth(U_c U_c^T G_c), singletons
// sign-fixed), U2 = trailing columns of the Householder QR of U1.
// V: column-major right singular vectors of R (unsorted), perm: sorted order.
// Writes U row-major into s.U.  Uses s.C (A, then Q) and s.R (reflectors).
__device__ __noinline__ void canonical_basis(const Buf& s_, int b, int r, int nsig) {
  const Buf s = s_;
  CE_SHARED_BUF(s);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* A = s.C;   // b x r column-major
  double* Vh = s.R;  // reflectors, column-major
  __shared__ int cstart[kSweepBlockMax];
  if (threadIdx.x == 0) {
    int k0 = 0;
    while (k0 < r) {
      int k1 = k0 + 1;
      while (k1 < r && k1 < nsig && s.sig[k1 - 1] - s.sig[k1] <= kClusterTol * s.sig[0]) ++k1;
      for (int k = k0; k < k1; ++k) cstart[k] = k0;
      k0 = k1;
    }
  }
  __syncthreads();
  int nclus = 0;
  for (int k0 = 0; k0 < r; ++k0) {
    if (cstart[k0] != k0) continue;
    int k1 = k0 + 1;
    while (k1 < r && cstart[k1] == k0) ++k1;
    const int c = k1 - k0;
    if ((nclus++ % NW) != warp) continue;
    if (c == 1) {
      const double* v = s.V + static_cast<int64_t>(s.perm[k0]) * pad_ld(b);
      double g = 0.0;
      for (int a = lane; a < b; a += 32) g += gauge_weight(a) * v[a];
      g = warp_sum(g);
      const double sg = g >= 0.0 ? 1.0 : -1.0;
      for (int a = lane; a < b; a += 32) A[k0 * b + a] = sg * v[a];
    } else {
      for (int j = 0; j < c; ++j) {
        double* z = A + (k0 + j) * b;
        for (int a = lane; a < b; a += 32) z[a] = 0.0;
        for (int q = 0; q < c; ++q) {
          const double* v = s.V + static_cast<int64_t>(s.perm[k0 + q]) * pad_ld(b);
          double m = 0.0;
          for (int a = lane; a < b; a += 32) m += v[a] * gauge_weight2(a, j);
          m = warp_sum(m);
          for (int a = lane; a < b; a += 32) z[a] += v[a] * m;
        }
      }
      __syncwarp();
      // MGS (two passes), re-projection onto span(U_c), MGS again (oracle/dense.cpp): the
      // re-projection removes rounding outside the span that the first orthonormalisation
      // amplified by cond(U_c^T G_c).  s.tau[k0 .. k1) is this cluster's private scratch.
      for (int round = 0; round < 2; ++round) {
        if (round == 1)
          for (int j = 0; j < c; ++j) {
            double* z = A + (k0 + j) * b;
            for (int q = 0; q < c; ++q) {
              const double* v = s.V + static_cast<int64_t>(s.perm[k0 + q]) * pad_ld(b);
              double d = 0.0;
              for (int a = lane; a < b; a += 32) d += v[a] * z[a];
              d = warp_sum(d);
              if (lane == 0) s.tau[k0 + q] = d;
            }
            __syncwarp();
            for (int a = lane; a < b; a += 32) {
              double acc = 0.0;
              for (int q = 0; q < c; ++q)
                acc += s.V[static_cast<int64_t>(s.perm[k0 + q]) * pad_ld(b) + a] * s.tau[k0 + q];
              z[a] = acc;
            }
            __syncwarp();
          }
        for (int j = 0; j < c; ++j) {
          double* z = A + (k0 + j) * b;
          for (int pass = 0; pass < 2; ++pass)
            for (int q = 0; q < j; ++q) {
              const double* y = A + (k0 + q) * b;
              double d = 0.0;
              for (int a = lane; a < b; a += 32) d += y[a] * z[a];
              d = warp_sum(d);
              for (int a = lane; a < b; a += 32) z[a] -= d * y[a];
              __syncwarp();
            }
          double n2 = 0.0;
          for (int a = lane; a < b; a += 32) n2 += z[a] * z[a];
          const double nrm = sqrt(warp_sum(n2));
          for (int a = lane; a < b; a += 32) z[a] /= nrm;
          __syncwarp();
        }
      }
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < b * r; idx += T) {
    const int k = idx / b, a = idx % b;
    s.U[a * b + k] = A[idx];
  }
  __syncthreads();
  for (int k = 0; k < r; ++k) {
    if (warp == 0) {
      double n2 = 0.0, rest = 0.0, g = 0.0;
      for (int a = k + lane; a < b; a += 32) {
        const double x = A[k * b + a];
        n2 += x * x;
        if (a > k) rest += x * x;
        g += gauge_weight(a) * x;
      }
      n2 = warp_sum(n2);
      rest = warp_sum(rest);
      g = warp_sum(g);
      const double nrm = sqrt(n2);
      double tau = 0.0;
      if (nrm != 0.0) {
        const double sg = g >= 0.0 ? 1.0 : -1.0;
        const double xk = A[k * b + k];
        const double beta = -sg * nrm;
        double vk;
        if (xk == 0.0 || (xk > 0.0) == (sg > 0.0)) vk = xk - beta;
        else vk = -rest / (xk + beta);
        const double vtv = vk * vk + rest;
        tau = vtv > 0.0 ? 2.0 / vtv : 0.0;
        for (int a = k + lane; a < b; a += 32) Vh[k * b + a] = (a == k) ? vk : A[k * b + a];
      }
      if (lane == 0) s.tau[k] = tau;
    }
    __syncthreads();
    const double tau = s.tau[k];
    if (tau != 0.0) {
      for (int j = k + 1 + warp; j < r; j += NW) {
        double d = 0.0;
        for (int a = k + lane; a < b; a += 32) d += Vh[k * b + a] * A[j * b + a];
        d = warp_sum(d) * tau;
        __syncwarp();
        for (int a = k + lane; a < b; a += 32) A[j * b + a] -= d * Vh[k * b + a];
      }
    }
    __syncthreads();
  }
  double* Q = s.C;
  const int nq = b - r;
  for (int idx = threadIdx.x; idx < nq * b; idx += T) {
    const int jj = idx / b, a = idx % b;
    Q[idx] = (a == r + jj) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int k = r - 1; k >= 0; --k) {
    const double tau = s.tau[k];
    if (tau != 0.0) {
      for (int jj = warp; jj < nq; jj += NW) {
        double d = 0.0;
        for (int a = k + lane; a < b; a += 32) d += Vh[k * b + a] * Q[jj * b + a];
        d = warp_sum(d) * tau;
        __syncwarp();
        for (int a = k + lane; a < b; a += 32) Q[jj * b + a] -= d * Vh[k * b + a];
      }
    }
    __syncthreads();
  }
  for (int idx = threadIdx.x; idx < nq * b; idx += T) {
    const int jj = idx / b, a = idx % b;
    s.U[a * b + r + jj] = Q[idx];
  }
  __syncthreads();
}

__device__ void tsqr_sel(const SweepArgs& A, double* R, double* C, int K, int b, int ldc, double* shr) {
  if (A.dbg & 1) tsqr_group(R, C, K, b, ldc, shr);
  else tsqr_fast(R, C, K, b, ldc, shr);
}

// Window of a row's squared-pattern entries staged in shared memory (one coalesced
// pass over the host-built per-entry tables) plus the column map of the current chunk.
constexpr int kEW = 256;
constexpr int kChunkMax = kSweepBlockMax;  // chunk widths are >= bmax (sweep_kcap, sweep_layout)
struct EntWin {
  long long off[kEW];
  int col[kEW];
  int roff[kEW];
  unsigned short bsz[kEW];
  unsigned char kind[kEW];
  unsigned short cblk[kChunkMax];  // chunk column -> window entry
  unsigned short ccol[kChunkMax];  // chunk column -> column inside its block
};

__device__ int load_window(const SweepArgs& A, int64_t e0, int64_t e1, EntWin& W) {
  const int n = static_cast<int>(e1 - e0 < kEW ? e1 - e0 : kEW);
  for (int t = threadIdx.x; t < n; t += T) {
    const int64_t e = e0 + t;
    W.off[t] = A.sq_boff[e];
    W.col[t] = A.sq_col[e];
    W.roff[t] = A.sq_roff[e];
    W.bsz[t] = static_cast<unsigned short>(A.sq_bsz[e]);
    W.kind[t] = A.sq_kind[e];
  }
  __syncthreads();
  return n;
}

// Gather the far blocks among entries [eb, ee) of row i into F^T chunks (chunk row =
// far column, column = row of the block row) and fold them into the TSQR triangle
// s.R.  Returns far columns seen.
__device__ int gather_tsqr(const SweepArgs& A, int i, int b, const Buf& s_, int64_t eb, int64_t ee, int* nzflag,
                           double* shr, EntWin& W) {
  const Buf s = s_;
  CE_SHARED_BUF(s);
  __shared__ int g_add, g_next, g_full;
  const int tid = threadIdx.x;
  const int ldc = chunk_ld(A.kcap);
  int fcols = 0, kfill = 0, nzl = 0;
  for (int64_t w0 = eb; w0 < ee; w0 += kEW) {
    const int n = load_window(A, w0, ee, W);
    int k = 0;
    while (k < n) {
      if (tid == 0) {
        int kk = k, add = 0, full = 0;
        for (; kk < n; ++kk) {
          if (W.kind[kk] != 2) continue;
          const int bj = W.bsz[kk];
          if (kfill + add + bj > A.kcap) {
            full = 1;
            break;
          }
          for (int c = 0; c < bj; ++c) {
            W.cblk[add + c] = static_cast<unsigned short>(kk);
            W.ccol[add + c] = static_cast<unsigned short>(c);
          }
          add += bj;
        }
        if (full && add == 0 && kfill == 0) {  // a block wider than the chunk: impossible by kcap >= bmax
          set_error(A.err, kErrChunk, A.level, i);
          kk = n;
          full = 0;
        }
        g_add = add;
        g_next = kk;
        g_full = full;
      }
      __syncthreads();
      const int add = g_add, full = g_full;
      k = g_next;
      const int tot = add * b;
      for (int base = tid; base < tot; base += 4 * T) {
        double v[4];
        int dst[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int idx = base + u * T;
          dst[u] = -1;
          v[u] = 0.0;
          if (idx < tot) {
            const int m = idx % add, a = idx / add;
            const int blk = W.cblk[m];
            const int bj = W.bsz[blk];
            v[u] = ldg(A.store + W.off[blk] + xidx(a, W.ccol[m], b, bj, W.col[blk] > i));
            dst[u] = a * ldc + kfill + m;
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (dst[u] >= 0) {
            s.C[dst[u]] = v[u];
            nzl |= v[u] != 0.0;
          }
      }
      kfill += add;
      fcols += add;
      __syncthreads();
      if (full) {
        tsqr_sel(A, s.R, s.C, kfill, b, ldc, shr);
        kfill = 0;
      }
    }
  }
  if (kfill > 0) tsqr_sel(A, s.R, s.C, kfill, b, ldc, shr);
  if (nzl) *nzflag = 1;
  __syncthreads();
  return fcols;
}

// Strip entries [eb, ee) of row i (kind != 0), in column chunks of up to cw columns
// (the blocks' columns side by side, one thread per column):
//   rotate by U (basis rows) or keep; far blocks keep rows < r only;
//   close blocks: g_t = (L^{-1} X[r:, :])^T -> G rows, X[:r, :] -= C g_t^T;
//   rows >= r are zeroed on write-back (level_matrix.cpp:51-65, 125-171).
// s.U = U (row-major), s.R = L (w x w), s.V = C (r x w); [s.D, s.sig) holds the chunks.
__device__ __noinline__ void strip_range(const SweepArgs& A, int i, int b, int r, int w, bool basis, int64_t eb,
                                         int64_t ee, const Buf& s_, EntWin& W) {
  const Buf s = s_;
  CE_SHARED_BUF(s);
  __shared__ int c_n, c_next;
  const int tid = threadIdx.x;
  const int cw = sweep_layout(A.bmax, A.kcap).cw;
  double* IN = s.D;
  double* OUT = basis ? s.D + static_cast<int64_t>(b) * cw : s.D;
  for (int q = tid; q < w; q += T) s.tau[q] = 1.0 / s.R[q * w + q];
  for (int64_t w0 = eb; w0 < ee; w0 += kEW) {
    const int n = load_window(A, w0, ee, W);
    int k = 0;
    while (k < n) {
      if (tid == 0) {
        int kk = k, cols = 0;
        for (; kk < n; ++kk) {
          if (W.kind[kk] == 0 || W.kind[kk] == 3) continue;  // diagonal / far block still exactly zero
          const int bj = W.bsz[kk];
          if (cols + bj > cw) break;
          for (int c = 0; c < bj; ++c) {
            W.cblk[cols + c] = static_cast<unsigned short>(kk);
            W.ccol[cols + c] = static_cast<unsigned short>(c);
          }
          cols += bj;
        }
        if (cols == 0 && kk < n) {  // a block wider than the chunk: impossible by cw >= bmax
          set_error(A.err, kErrStrip, A.level, i);
          kk = n;
        }
        c_n = cols;
        c_next = kk;
      }
      __syncthreads();
      const int ncol = c_n;
      k = c_next;
      if (ncol == 0) continue;
      const int tot = ncol * b;
      for (int base = tid; base < tot; base += 4 * T) {
        double v[4];
        int dst[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int idx = base + u * T;
          dst[u] = -1;
          v[u] = 0.0;
          if (idx < tot) {
            const int m = idx % ncol, a = idx / ncol;
            const int blk = W.cblk[m];
            const bool far = W.roff[blk] < 0;
            if (!(!basis && far && a >= r))
              v[u] = ldg(A.store + W.off[blk] + xidx(a, W.ccol[m], b, W.bsz[blk], W.col[blk] > i));
            dst[u] = a * cw + m;
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (dst[u] >= 0) IN[dst[u]] = v[u];
      }
      __syncthreads();
      for (int c = tid; c < ncol; c += T) {
        const int blk = W.cblk[c];
        const int roff = W.roff[blk];
        const bool far = roff < 0;
        if (basis) {
          const int na = far ? r : b;
          for (int a0 = 0; a0 < na; a0 += 8) {
            double acc[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) acc[u] = 0.0;
            for (int kk = 0; kk < b; ++kk) {
              const double x = IN[kk * cw + c];
              const double* Ur = s.U + kk * b + a0;
#pragma unroll
              for (int u = 0; u < 8; ++u) acc[u] = fma(Ur[u], x, acc[u]);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u)
              if (a0 + u < na) OUT[(a0 + u) * cw + c] = acc[u];
          }
        }
        if (!far && w > 0) {
          double* G = A.fac + A.g_off[i] + static_cast<int64_t>(r + roff + W.ccol[c]) * w;
          double* y = OUT + static_cast<int64_t>(r) * cw + c;
          for (int q = 0; q < w; ++q) {
            const double* Lq = s.R + q * w;
            double a0 = y[q * cw], a1 = 0.0;
            int p = 0;
            for (; p + 1 < q; p += 2) {
              a0 = fma(-Lq[p], y[p * cw], a0);
              a1 = fma(-Lq[p + 1], y[(p + 1) * cw], a1);
            }
            if (p < q) a0 = fma(-Lq[p], y[p * cw], a0);
            const double v = (a0 + a1) * s.tau[q];
            y[q * cw] = v;
            G[q] = v;
          }
          int a = 0;
          for (; a + 3 < r; a += 4) {
            double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
            for (int q = 0; q < w; ++q) {
              const double yq = y[q * cw];
              c0 = fma(s.V[a * w + q], yq, c0);
              c1 = fma(s.V[(a + 1) * w + q], yq, c1);
              c2 = fma(s.V[(a + 2) * w + q], yq, c2);
              c3 = fma(s.V[(a + 3) * w + q], yq, c3);
            }
            OUT[a * cw + c] -= c0;
            OUT[(a + 1) * cw + c] -= c1;
            OUT[(a + 2) * cw + c] -= c2;
            OUT[(a + 3) * cw + c] -= c3;
          }
          for (; a < r; ++a) {
            double c0 = 0.0;
            for (int q = 0; q < w; ++q) c0 = fma(s.V[a * w + q], y[q * cw], c0);
            OUT[a * cw + c] -= c0;
          }
        }
      }
      __syncthreads();
      for (int idx = tid; idx < tot; idx += T) {
        const int m = idx % ncol, a = idx / ncol;
        const int blk = W.cblk[m];
        double* X = A.store + W.off[blk] + xidx(a, W.ccol[m], b, W.bsz[blk], W.col[blk] > i);
        *X = (w > 0 && a >= r) ? 0.0 : OUT[a * cw + m];
      }
      __syncthreads();
    }
  }
}

// Schur update of one panel pair (P, Q), P <= Q, of row i's close list:
// X_ts -= g_t g_s^T for s in panel P, t in panel Q, s <= t (level_matrix.cpp:148-162).
// g rows of both panels are staged in shared memory.  The task is a short chain of
// dependent global loads (close columns -> slot offsets -> g rows / X tile), so the
// first X tile of every warp is loaded before the panels are staged and both sets of
// loads are in flight together.
__device__ __noinline__ void panel_update(const SweepArgs& A, int i, int r, int w, int P, int Q, double* sm,
                                          bool reuse_s) {
  CE_SHARED(sm);
  const long long tb0 = clock64();
  __shared__ long long slot_tab[kPanelNb * kPanelNb];  // value offset of stored (t, s), -1: not updated
  __shared__ int tab_bs[kPanelNb];
  __shared__ int roff_s[kPanelNb], roff_t[kPanelNb];
  __shared__ int col_s[kPanelNb], col_t[kPanelNb];
  __shared__ int n_live[2];
  __shared__ unsigned char xblk[kPanelRows], yblk[kPanelRows];
  __shared__ unsigned short xloc[kPanelRows], yloc[kPanelRows];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t c0 = A.cl_ptr[i];
  const int* ps = A.pan_start + A.pan_ptr[i];
  const int s0 = ps[P], s1 = ps[P + 1], t0 = ps[Q], t1 = ps[Q + 1];
  const int ns = s1 - s0, nt = t1 - t0;
  // Live rows of each neighbour's g block: a neighbour u < i was eliminated earlier in
  // this level, its block row is zero below its rank, so g_u (= columns of X_iu) is zero
  // in rows >= rank(u) and X_st only changes in the retained rows / columns.  The panel
  // is compacted to live rows (bit-identical result: the skipped terms are exact zeros).
  // reuse_s: panel P's tables and staged rows are still in shared memory from the previous
  // pair of this task (same P, P != Q now), only panel Q is rebuilt
  if (warp < 2 && !(reuse_s && warp == 0)) {
    const int n = warp == 0 ? ns : nt, base = warp == 0 ? s0 : t0;
    int live = 0, roff = 0, bu = 0, u = 0;
    if (lane < n) {
      const int64_t e = c0 + base + lane;
      u = A.cl_col[e];
      bu = A.bsz[u];
      roff = A.cl_roff[e];
      live = u < i ? __ldcg(A.rank + u) : bu;
    }
    int incl = live;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int y0 = incl - live;
    if (lane < n) {
      if (warp == 0) {
        tab_bs[lane] = bu;
        roff_s[lane] = roff;
        col_s[lane] = u;
        for (int y = 0; y < live; ++y) {
          yblk[y0 + y] = static_cast<unsigned char>(lane);
          yloc[y0 + y] = static_cast<unsigned short>(y);
        }
      } else {
        roff_t[lane] = roff;
        col_t[lane] = u;
        for (int x = 0; x < live; ++x) {
          xblk[y0 + x] = static_cast<unsigned char>(lane);
          xloc[y0 + x] = static_cast<unsigned short>(x);
        }
      }
    }
    if (lane == 31) n_live[warp] = incl;
  }
  // value offsets of the stored (t, s) blocks: every thread reads its pair's columns from the
  // close list itself, so this chain of dependent loads runs beside the table warps' chain
  // instead of behind it (one barrier and one load latency less per pair)
  for (int idx = tid; idx < nt * ns; idx += T) {
    const int kt = idx / ns, ks = idx % ns;
    long long off = -1;
    if (!(P == Q && ks > kt)) {
      const int t = A.cl_col[c0 + t0 + kt], s = A.cl_col[c0 + s0 + ks];
      if (A.tri_off) {  // dense triangular table (levels with M <= 8192): one load
        off = __ldg(A.tri_off + static_cast<int64_t>(t) * (t + 1) / 2 + s);
        if (off < 0) set_error(A.err, kErrPattern, A.level, i);
      } else {  // binary search of the squared pattern
        const int64_t slot = find_slot(A.sq_ptr, A.sq_col, A.sq_slot, t, s);
        if (slot < 0) set_error(A.err, kErrPattern, A.level, i);
        else off = A.slot_off[slot];
      }
    }
    slot_tab[idx] = off;
  }
  __syncthreads();
  const long long tb1 = clock64();
  prof_add(A, kProfBSetup, tb1 - tb0);
  const int rsn = n_live[0], rtn = n_live[1];
  // row strides = 8 (mod 16) doubles: the four k-rows of an m8n8k4 fragment load hit
  // disjoint bank halves (two wavefronts, the minimum for 32 doubles)
  const int lds = ((rsn + 7) & ~15) + 8, ldt = ((rtn + 7) & ~15) + 8;
  // rtn x rsn product on the FP64 tensor cores (mma.m8n8k4): a warp owns a 16 x 32 tile
  // (2 x 4 fragments), the k loop runs over the w g-columns in steps of 4 (masked tail);
  // the epilogue scatters into the (t, s) blocks.
  const int g = lane >> 2, t4 = lane & 3;
  const int ntx = (rtn + 15) / 16, nty = (rsn + 31) / 32;
#if CE_TILE_TRANSPOSED
  // Transposed fragments: the warp's 16 x 32 tile (16 compacted t-rows x, 32 compacted s-rows y)
  // is computed as (G_s G_t^T)^T, i.e. the accumulator fragments have y along their rows.  Lane
  // (g, t4) then owns y = yb + 8 fy + g and x = xb + 8 fx + 2 t4 + e: one load instruction reads,
  // for each of 4 X rows, 8 CONTIGUOUS doubles across the lanes g (every 32-byte sector of an X
  // row is requested from L2 once per tile; with x along the fragment rows a lane's two adjacent
  // columns came from two instructions and every sector was requested twice).  Same products
  // summed in the same order: bit-identical results.
  double* px[4][4];  // element addresses of the lane's 16 X entries (nullptr: outside the live tile)
  double xv[4][4];   // [2 fx + e][fy]
  auto load_tile = [&](int wt) {
    int ktv[4], xlv[4], ksv[4], ylv[4], bsv[4];
    const int xb = (wt / nty) * 16, yb = (wt % nty) * 32;
#pragma unroll
    for (int xi = 0; xi < 4; ++xi) {
      const int x = xb + 8 * (xi >> 1) + 2 * t4 + (xi & 1);
      ktv[xi] = x < rtn ? xblk[x] : -1;
      xlv[xi] = x < rtn ? xloc[x] : 0;
    }
#pragma unroll
    for (int fy = 0; fy < 4; ++fy) {
      const int y = yb + 8 * fy + g;
      ksv[fy] = y < rsn ? yblk[y] : -1;
      ylv[fy] = y < rsn ? yloc[y] : 0;
      bsv[fy] = ksv[fy] >= 0 ? tab_bs[ksv[fy]] : 0;
    }
#pragma unroll
    for (int xi = 0; xi < 4; ++xi)
#pragma unroll
      for (int fy = 0; fy < 4; ++fy) {
        xv[xi][fy] = 0.0;
        px[xi][fy] = nullptr;
        if (ktv[xi] >= 0 && ksv[fy] >= 0) {
          const long long off = slot_tab[ktv[xi] * ns + ksv[fy]];
          if (off >= 0) {
            px[xi][fy] = A.store + off + static_cast<int64_t>(xlv[xi]) * bsv[fy] + ylv[fy];
            xv[xi][fy] = ldg(px[xi][fy]);
          }
        }
      }
  };
#else
  int ktv[2], xlv[2], ksv[8], ylv[8], bsv[8];
  double xv[2][8];
  auto load_tile = [&](int wt) {
    const int xb = (wt / nty) * 16, yb = (wt % nty) * 32;
#pragma unroll
    for (int i2 = 0; i2 < 2; ++i2) {
      const int x = xb + 8 * i2 + g;
      ktv[i2] = x < rtn ? xblk[x] : -1;
      xlv[i2] = x < rtn ? xloc[x] : 0;
    }
#pragma unroll
    for (int j2 = 0; j2 < 8; ++j2) {
      const int y = yb + 8 * (j2 >> 1) + 2 * t4 + (j2 & 1);
      ksv[j2] = y < rsn ? yblk[y] : -1;
      ylv[j2] = y < rsn ? yloc[y] : 0;
      bsv[j2] = ksv[j2] >= 0 ? tab_bs[ksv[j2]] : 0;
    }
#pragma unroll
    for (int i2 = 0; i2 < 2; ++i2)
#pragma unroll
      for (int j2 = 0; j2 < 8; ++j2) {
        xv[i2][j2] = 0.0;
        if (ktv[i2] >= 0 && ksv[j2] >= 0) {
          const long long off = slot_tab[ktv[i2] * ns + ksv[j2]];
          if (off >= 0) xv[i2][j2] = ldg(A.store + off + static_cast<int64_t>(xlv[i2]) * bsv[j2] + ylv[j2]);
        }
      }
  };
#endif
  // first tile's X in flight while the panels are staged
  if (warp < ntx * nty) load_tile(warp);
  // g rows transposed into shared memory: GsT[q][y], GtT[q][x] (live rows only)
  const double* G = A.fac + A.g_off[i];
  double* GsT = sm;
  double* GtT = P == Q ? sm : sm + static_cast<int64_t>(lds) * w;
  // staged with 8 independent loads in flight per thread (the rows are short, latency dominates)
  auto stage = [&](double* dst, int ld, int n, const int* roff, const unsigned char* blk, const unsigned short* loc) {
    const int tot = ld * w;
    for (int base = tid; base < tot; base += 8 * T) {
      double v[8];
      int di[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int idx = base + u * T;
        di[u] = -1;
        v[u] = 0.0;
        if (idx < tot) {
          const int y = idx / w, q = idx % w;
          di[u] = q * ld + y;
          if (y < n) v[u] = ldg(G + static_cast<int64_t>(r + roff[blk[y]] + loc[y]) * w + q);
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (di[u] >= 0) dst[di[u]] = v[u];
    }
  };
#if CE_SMEM_BUFFER && CE_STAGE_ASYNC
  // shared-memory build: every element is an 8-byte cp.async (LDGSTS), so a thread's whole share
  // of the panel is in flight at once with no register staging -- one global-memory latency per
  // panel instead of one per batch of 8 loads; padding rows are plain zero stores
  auto stage_async = [&](double* dst, int ld, int n, const int* roff, const unsigned char* blk,
                         const unsigned short* loc) {
    // 8 lanes along a g row (64 contiguous bytes), 32 rows per pass: the row's source address
    // is looked up once and reused for its w / 8 elements (no division by w, no per-element
    // table lookups)
    const int ql = tid & 7;
    for (int y = tid >> 3; y < ld; y += T / 8) {
      double* d = dst + y;
      if (y < n) {
        const double* src = G + static_cast<int64_t>(r + roff[blk[y]] + loc[y]) * w;
        const unsigned da = static_cast<unsigned>(__cvta_generic_to_shared(d));
        for (int q = ql; q < w; q += 8)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(da + static_cast<unsigned>(q * ld) * 8u), "l"(src + q)
                       : "memory");
      } else {
        for (int q = ql; q < w; q += 8) d[q * ld] = 0.0;
      }
    }
  };
  if (!reuse_s) stage_async(GsT, lds, rsn, roff_s, yblk, yloc);
  if (P != Q) stage_async(GtT, ldt, rtn, roff_t, xblk, xloc);
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
#else
  if (!reuse_s) stage(GsT, lds, rsn, roff_s, yblk, yloc);
  if (P != Q) stage(GtT, ldt, rtn, roff_t, xblk, xloc);
  __syncthreads();
#endif
  const long long tb2 = clock64();
  prof_add(A, kProfBStage, tb2 - tb1);
#if CE_TILE_TRANSPOSED
  for (int wt = warp; wt < ntx * nty; wt += T / 32) {
    if (wt != warp) load_tile(wt);
    const int xb = (wt / nty) * 16, yb = (wt % nty) * 32;
    double acc[4][2][2];  // [fy][fx][e]
#pragma unroll
    for (int fy = 0; fy < 4; ++fy)
#pragma unroll
      for (int fx = 0; fx < 2; ++fx) acc[fy][fx][0] = acc[fy][fx][1] = 0.0;
    for (int q0 = 0; q0 < w; q0 += 4) {
      const int q = q0 + t4;
      double af[4], bf[2];
#pragma unroll
      for (int fy = 0; fy < 4; ++fy) {
        const int y = yb + 8 * fy + g;
        af[fy] = (q < w && y < lds) ? GsT[q * lds + y] : 0.0;
      }
#pragma unroll
      for (int fx = 0; fx < 2; ++fx) {
        const int x = xb + 8 * fx + g;
        bf[fx] = (q < w && x < ldt) ? GtT[q * ldt + x] : 0.0;
      }
#pragma unroll
      for (int fy = 0; fy < 4; ++fy)
#pragma unroll
        for (int fx = 0; fx < 2; ++fx)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                       : "+d"(acc[fy][fx][0]), "+d"(acc[fy][fx][1])
                       : "d"(af[fy]), "d"(bf[fx]));
    }
#pragma unroll
    for (int xi = 0; xi < 4; ++xi)
#pragma unroll
      for (int fy = 0; fy < 4; ++fy)
        if (px[xi][fy]) *px[xi][fy] = xv[xi][fy] - acc[fy][xi >> 1][xi & 1];
  }
#else
  for (int wt = warp; wt < ntx * nty; wt += T / 32) {
    if (wt != warp) load_tile(wt);
    const int xb = (wt / nty) * 16, yb = (wt % nty) * 32;
    double acc[2][8];
#pragma unroll
    for (int i2 = 0; i2 < 2; ++i2)
#pragma unroll
      for (int j2 = 0; j2 < 8; ++j2) acc[i2][j2] = 0.0;
    for (int q0 = 0; q0 < w; q0 += 4) {
      const int q = q0 + t4;
      double af[2], bf[4];
#pragma unroll
      for (int i2 = 0; i2 < 2; ++i2) {
        const int x = xb + 8 * i2 + g;
        af[i2] = (q < w && x < ldt) ? GtT[q * ldt + x] : 0.0;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int y = yb + 8 * j + g;
        bf[j] = (q < w && y < lds) ? GsT[q * lds + y] : 0.0;
      }
#pragma unroll
      for (int i2 = 0; i2 < 2; ++i2)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                       : "+d"(acc[i2][2 * j]), "+d"(acc[i2][2 * j + 1])
                       : "d"(af[i2]), "d"(bf[j]));
    }
#pragma unroll
    for (int i2 = 0; i2 < 2; ++i2)
#pragma unroll
      for (int j2 = 0; j2 < 8; ++j2)
        if (ktv[i2] >= 0 && ksv[j2] >= 0) {
          const long long off = slot_tab[ktv[i2] * ns + ksv[j2]];
          if (off >= 0)
            A.store[off + static_cast<int64_t>(xlv[i2]) * bsv[j2] + ylv[j2]] = xv[i2][j2] - acc[i2][j2];
        }
  }
#endif
  __syncthreads();
  prof_add(A, kProfBTiles, clock64() - tb2);
}

__device__ void all_panels(const SweepArgs& A, int i, int r, int w, double* sm) {
  const int np = static_cast<int>(A.pan_ptr[i + 1] - A.pan_ptr[i]) - 1;
  for (int P = 0; P < np; ++P)
    for (int Q = P; Q < np; ++Q) panel_update(A, i, r, w, P, Q, sm, Q > P);
}

// A2: compression decision + basis + pivot factorisation; with nA3 == 0 also the strip,
// with nB == 0 also the Schur panels.
__device__ __noinline__ void task_a2(const SweepArgs& A, int i, const Buf& s_, int nA1, int nA3, int nB, EntWin& W) {
  const Buf s = s_;
  CE_SHARED_BUF(s);
  __shared__ double shr[4];
  __shared__ int sflag[4];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long t_a2 = clock64();
  const int b = A.bsz[i];
  const int64_t p0 = A.sq_ptr[i], p1 = A.sq_ptr[i + 1];
  double* Dg = A.store + A.sq_boff[A.sq_diag[i]];
  for (int idx = tid; idx < b * b; idx += T) {
    s.D[idx] = ldg(Dg + idx);
    s.R[idx] = 0.0;
  }
  if (tid == 0) sflag[0] = 0;
  __syncthreads();

  // ---- far-block triangle (compression.cpp:38-48) ----
  int fcols;
  if (nA1 == 0) {
    gather_tsqr(A, i, b, s, p0, p1, &sflag[0], shr, W);
    fcols = static_cast<int>(A.fsum[i]);  // every far column, also the still-zero ones it skipped
  } else {
    fcols = static_cast<int>(A.fsum[i]);
    // the TSQR tree's root triangle (its last node)
    const double* Rr = A.rscratch + A.rs_off[i] + static_cast<int64_t>(nA1 - 1) * b * b;
    for (int idx = tid; idx < b * b; idx += T) s.R[idx] = ldg(Rr + idx);
    if (tid == 0) sflag[0] = ld_acquire(A.nzflag + i);
    __syncthreads();
  }
  const bool nonzero = sflag[0] != 0;
  const int meff = fcols < b ? fcols : b;
  long long tp = clock64();
  prof_add(A, kProfA2Tsqr, tp - t_a2);

  // ---- rank decision + basis (compression.cpp:20-61) ----
  int r = 0, nsig = 0;
  bool basis = false;
  if (fcols > 0) {
    bool need_svd;
    if (A.mode == 1) {
      r = A.fixed_rank < b ? A.fixed_rank : b;
      need_svd = nonzero && r < b;
    } else {
      need_svd = nonzero;
    }
    if (need_svd) {
      long long t0 = clock64();
      precondition_qr(s, b);
      long long t1 = clock64();
      const int nsw = (A.dbg & 2) ? jacobi(s.R, s.V, b, pad_ld(b), meff) : jacobi_fast(s.R, s.V, b, pad_ld(b), meff);
      long long t2 = clock64();
      apply_q2(s, b);
      prof_add(A, kProfSvdPre, t1 - t0);
      prof_add(A, kProfSvdJac, t2 - t1);
      prof_add(A, kProfSvdPost, clock64() - t2);
      prof_add(A, kProfSweeps, nsw);
      prof_add(A, kProfSvds, 1);
      for (int j = warp; j < b; j += NW) {
        double acc = 0.0;
        for (int k = lane; k < b; k += 32) acc += s.R[j * pad_ld(b) + k] * s.R[j * pad_ld(b) + k];
        acc = warp_sum(acc);
        if (lane == 0) s.nrm[j] = sqrt(acc);
      }
      __syncthreads();
      for (int j = tid; j < b; j += T) {
        const double sj = s.nrm[j];
        if (!isfinite(sj)) set_error(A.err, kErrNaN, A.level, i);  // never rank a NaN
        int rank = 0;
        for (int k = 0; k < b; ++k) {
          const double sk = s.nrm[k];
          if (sk > sj || (sk == sj && k < j)) ++rank;
        }
        s.perm[rank] = j;
        s.sig[rank] = sj;
      }
      __syncthreads();
      nsig = meff;
      for (int k = tid; k < nsig; k += T) A.sigma[A.sigma_off[i] + k] = s.sig[k];
      if (A.mode == 0) {
        const double thr = A.absolute ? A.eps : A.eps * s.sig[0];
        r = nsig;
        for (int k = 0; k < nsig; ++k)
          if (s.sig[k] <= thr) {
            r = k;
            break;
          }
        if (A.forced && A.forced[i] >= 0) r = A.forced[i];
        if (r > b) r = b;
      }
      basis = r < b;
    } else if (A.mode == 0) {
      r = 0;
    }
  }
  const int w = b - r;
  {
    const long long t = clock64();
    prof_add(A, kProfA2Svd, t - tp);
    tp = t;
  }

  // ---- basis and rotated diagonal (level_matrix.cpp:51-54) ----
  if (basis) {
    canonical_basis(s, b, r, nsig);
    double* Ug = A.basis + A.basis_off[i];
    for (int idx = tid; idx < b * b; idx += T) Ug[idx] = s.U[idx];
    for (int idx = tid; idx < b * b; idx += T) {
      const int a = idx / b, c = idx % b;
      double acc = 0.0;
      for (int k = 0; k < b; ++k) acc += s.D[a * b + k] * s.U[k * b + c];
      s.C[idx] = acc;
    }
    __syncthreads();
    for (int idx = tid; idx < b * b; idx += T) {
      const int a = idx / b, c = idx % b;
      double acc = 0.0;
      for (int k = 0; k < b; ++k) acc += s.U[k * b + a] * s.C[k * b + c];
      s.R[idx] = acc;
    }
    __syncthreads();
    for (int idx = tid; idx < b * b; idx += T) {
      const int a = idx / b, c = idx % b;
      s.D[idx] = 0.5 * (s.R[a * b + c] + s.R[c * b + a]);
    }
    __syncthreads();
  }

  {
    const long long t = clock64();
    prof_add(A, kProfA2Basis, t - tp);
    tp = t;
  }
  // ---- pivot factorisation (level_matrix.cpp:104-138) ----
  if (w > 0) {
    double* P = s.R;     // w x w
    double* Pbak = s.V;  // shift-retry backup, then the coupling C (r x w)
    for (int idx = tid; idx < w * w; idx += T) {
      const int q = idx / w, p = idx % w;
      P[idx] = s.D[(r + q) * b + r + p];
      Pbak[idx] = P[idx];
    }
    __syncthreads();
    for (int attempt = 0; attempt < 2; ++attempt) {
      if (attempt == 1) {
        if (tid == 0) {
          double tr = 0.0;
          for (int q = 0; q < w; ++q) tr += Pbak[q * w + q];
          shr[1] = 1e-12 * tr / static_cast<double>(w);
        }
        __syncthreads();
        for (int idx = tid; idx < w * w; idx += T) {
          const int q = idx / w, p = idx % w;
          P[idx] = Pbak[idx] + (q == p ? shr[1] : 0.0);
        }
        __syncthreads();
      }
      if (tid == 0) sflag[2] = 0;
      __syncthreads();
      for (int k = 0; k < w; ++k) {
        if (tid == 0) {
          const double d = P[k * w + k];
          if (!(d > 0.0)) sflag[2] = 1;
          else P[k * w + k] = sqrt(d);
        }
        __syncthreads();
        if (sflag[2]) break;
        const double dk = P[k * w + k];
        for (int q = k + 1 + tid; q < w; q += T) P[q * w + k] /= dk;
        __syncthreads();
        const int m = w - k - 1;
        for (int idx = tid; idx < m * m; idx += T) {
          const int q = k + 1 + idx / m, p = k + 1 + idx % m;
          if (p <= q) P[q * w + p] -= P[q * w + k] * P[p * w + k];
        }
        __syncthreads();
      }
      if (!sflag[2]) {
        if (attempt == 1 && tid == 0) atomicAdd(A.shifts, 1);
        break;
      }
      if (attempt == 1) {
        if (tid == 0) set_error(A.err, kErrBreakdown, A.level, i);
        return;
      }
    }
    double* L = A.fac + A.chol_off[i];
    for (int idx = tid; idx < w * w; idx += T) {
      const int q = idx / w, p = idx % w;
      const double v = p <= q ? P[idx] : 0.0;
      P[idx] = v;
      L[idx] = v;
    }
    __syncthreads();
    // coupling C = (L^{-1} D[r:, :r])^T -> G rows [0, r) and s.V
    double* G = A.fac + A.g_off[i];
    for (int rho = tid; rho < r; rho += T) {
      double* y = s.V + rho * w;
      for (int q = 0; q < w; ++q) {
        double acc = s.D[(r + q) * b + rho];
        for (int p = 0; p < q; ++p) acc -= P[q * w + p] * y[p];
        y[q] = acc / P[q * w + q];
      }
      for (int q = 0; q < w; ++q) G[static_cast<int64_t>(rho) * w + q] = y[q];
    }
    __syncthreads();
    // D[:r, :r] -= C C^T; eliminated rows/cols of D leave the level
    for (int idx = tid; idx < b * b; idx += T) {
      const int a = idx / b, c = idx % b;
      if (a >= r || c >= r) {
        s.D[idx] = 0.0;
      } else {
        double acc = 0.0;
        for (int q = 0; q < w; ++q) acc += s.V[a * w + q] * s.V[c * w + q];
        s.D[idx] -= acc;
      }
    }
    __syncthreads();
  }
  for (int idx = tid; idx < b * b; idx += T) Dg[idx] = s.D[idx];
  if (tid == 0) {
    A.rank[i] = r;
    A.width[i] = w;
    A.has_basis[i] = basis ? 1 : 0;
    A.fcols[i] = fcols;
    A.nsig[i] = nsig;
  }
  __syncthreads();
  {
    const long long t = clock64();
    prof_add(A, kProfA2Pivot, t - tp);
    tp = t;
  }

  // ---- strip (thin rows) ----
  if (nA3 == 0 && (basis || w > 0)) {
    strip_range(A, i, b, r, w, basis, p0, p1, s, W);
    {
      const long long t = clock64();
      prof_add(A, kProfA2Strip, t - tp);
      tp = t;
    }
    if (nB == 0 && w > 0) all_panels(A, i, r, w, s.R);
    prof_add(A, kProfA2Panels, clock64() - tp);
  }
}

// A3 tile k: strip entries with strip-ordinal in [k*ns/nA3, (k+1)*ns/nA3).
__device__ __noinline__ void task_a3(const SweepArgs& A, int i, const Buf& s_, int k, int nA3, int nB, EntWin& W) {
  const Buf s = s_;
  CE_SHARED_BUF(s);
  const int tid = threadIdx.x;
  const int b = A.bsz[i];
  const int r = __ldcg(A.rank + i), w = __ldcg(A.width + i);
  const bool basis = __ldcg(reinterpret_cast<const unsigned char*>(A.has_basis) + i) != 0;
  if (!basis && w == 0) return;
  if (basis)
    for (int idx = tid; idx < b * b; idx += T) s.U[idx] = ldg(A.basis + A.basis_off[i] + idx);
  if (w > 0) {
    for (int idx = tid; idx < w * w; idx += T) s.R[idx] = ldg(A.fac + A.chol_off[i] + idx);
    for (int idx = tid; idx < r * w; idx += T) s.V[idx] = ldg(A.fac + A.g_off[i] + idx);
  }
  __syncthreads();
  const int64_t* se = A.strip_e + A.strip_ptr[i] + k;
  strip_range(A, i, b, r, w, basis, se[0], se[1], s, W);
  (void)nA3;
  (void)nB;
}

// A1: TSQR tree node `part` of row i (leaf k at level 0, else combine k at level tlev).
__device__ __noinline__ void task_a1(const SweepArgs& A, int i, const Buf& s_, int part, int k, int tlev, int tprev,
                                     int tprevn, int* nzp, double* shr, EntWin& W) {
  const Buf s = s_;
  CE_SHARED_BUF(s);
  int& nz = *nzp;
  const int b = A.bsz[i];
  for (int idx = threadIdx.x; idx < b * b; idx += T) s.R[idx] = 0.0;
  __syncthreads();
  if (tlev == 0) {
    // leaf: far-entry range of this leaf
    const int64_t* le = A.leaf_e + A.leaf_ptr[i] + k;
    gather_tsqr(A, i, b, s, le[0], le[1], &nz, shr, W);
  } else {
    // combine the F child triangles (tree nodes tprev + F k ...): the first becomes R,
    // the others are folded in as stacked chunks of <= kcap rows
    const int F = A.kcap / b > 2 ? A.kcap / b : 2;
    const int per = A.kcap / b > 1 ? A.kcap / b : 1;
    const int c0 = F * k, nc = tprevn - c0 < F ? tprevn - c0 : F;
    const int ldc = chunk_ld(A.kcap);
    const double* R0 = A.rscratch + A.rs_off[i] + static_cast<int64_t>(tprev + c0) * b * b;
    for (int idx = threadIdx.x; idx < b * b; idx += T) s.R[idx] = ldg(R0 + idx);
    __syncthreads();
    for (int f0 = 1; f0 < nc; f0 += per) {
      const int nk = nc - f0 < per ? nc - f0 : per;
      const int K = nk * b;
      const double* Rf = R0 + static_cast<int64_t>(f0) * b * b;
      for (int idx = threadIdx.x; idx < K * b; idx += T) {
        const int j = idx / K, m = idx % K;  // chunk element (m, j) = R_child(m / b)[m % b][j]
        s.C[static_cast<int64_t>(j) * ldc + m] = ldg(Rf + static_cast<int64_t>(m / b) * b * b + j * b + m % b);
      }
      __syncthreads();
      tsqr_sel(A, s.R, s.C, K, b, ldc, shr);
    }
  }
  double* Rk = A.rscratch + A.rs_off[i] + static_cast<int64_t>(part) * b * b;
  for (int idx = threadIdx.x; idx < b * b; idx += T) Rk[idx] = s.R[idx];
  if (threadIdx.x == 0 && nz) atomicOr(A.nzflag + i, 1);
}

__global__ void __launch_bounds__(T, CE_SWEEP_MIN_BLOCKS) sweep_kernel(SweepArgs A) {
  extern __shared__ double smem_dyn[];
#if CE_SMEM_BUFFER
  double* base = smem_dyn;
#else
  double* base = A.scratch + static_cast<int64_t>(blockIdx.x) * A.scratch_per_cta;
#endif
  const Buf s = carve(base, A.bmax, A.kcap);
  CE_SHARED_BUF(s);
  __shared__ long long s_item;
  __shared__ int s_stop;
  __shared__ EntWin W;
  __shared__ double shr[4];
  __shared__ int nz;
  __shared__ int s_bready;
  for (;;) {
    if (threadIdx.x == 0) {
      s_stop = *reinterpret_cast<volatile int*>(A.err) != 0;
      s_item = s_stop ? 0 : static_cast<long long>(atomicAdd(A.ticket, 1ULL));
    }
    __syncthreads();
    if (s_stop) break;
    const long long item = s_item;
    if (item >= A.n_items) break;
    if (A.trace && threadIdx.x == 0) {
      unsigned long long g;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
      A.trace[4 * item] = g;
    }
    const int i = A.item_row[item];
    const int part = A.item_part[item];
    const int nA1 = A.nA1[i], nA3 = A.nA3[i], nB = A.nB[i];
    // stage of the item and the number of this row's items it must wait for
    int stage, k = 0, need = 0;
    int tlev = 0, tprev = 0, tprevn = 0;  // TSQR tree: level, first node / size of the level below
    if (part < nA1) {
      stage = 1;
      // node `part` of the TSQR tree: leaves first, then levels of F-way combines
      const int F = A.kcap / A.bsz[i] > 2 ? A.kcap / A.bsz[i] : 2;
      int n = A.nleaf[i], start = 0, p = part;
      while (p >= n) {
        p -= n;
        tprev = start;
        tprevn = n;
        start += n;
        n = (n + F - 1) / F;
        ++tlev;
      }
      k = p;
      need = start;  // combines wait for every node of the levels below
    } else if (part == nA1) {
      stage = 2;
      need = nA1;
    } else if (part <= nA1 + nA3) {
      stage = 3;
      k = part - nA1 - 1;
      need = nA1 + 1;
    } else {
      stage = 4;
      k = part - nA1 - 1 - nA3;
      need = nA1 + 1 + nA3;
    }
    const bool first = (stage == 1 && tlev == 0) || (stage == 2 && nA1 == 0);
    const long long t_wait = clock64();
    if (first) {
      // every predecessor j < i of sq(i) far enough along (one poller per entry, in parallel):
      // a far predecessor's A stages (its Schur pairs never touch row i), a close one's A stages
      // and the Schur pairs touching row i's panel (sq_pan), else all of its tasks
      const int64_t pb = A.sq_ptr[i], pe = A.sq_diag[i];
      for (int64_t e = pb + threadIdx.x; e < pe; e += T) {
        const int j = A.sq_col[e];
        const int pan = A.sq_pan[e];
        const bool far = A.sq_kind[e] >= 2;
        const int tgt = (far || pan >= 0) ? A.nA1[j] + 1 + A.nA3[j] : A.target[j];
        const int* pd = nullptr;
        int ptgt = 0;
        if (!far && pan >= 0) {
          pd = A.pdone + A.pan_ptr[j] + pan;
          ptgt = static_cast<int>(A.pan_ptr[j + 1] - A.pan_ptr[j]) - 1;
        }
        while (ld_acquire(A.done + j) < tgt || (pd && ld_acquire(pd) < ptgt)) {
          if (*reinterpret_cast<volatile int*>(A.err) != 0) {
            s_stop = 1;
            break;
          }
          sweep_backoff();
        }
        if (s_stop) break;
      }
    }
    if (stage == 4) {
      // Schur pairs write blocks shared with every predecessor's pairs: all of them first
      if (threadIdx.x == 0) s_bready = ld_acquire(A.bready + i);
      __syncthreads();
      if (!s_bready) {
        const int64_t pb = A.sq_ptr[i], pe = A.sq_diag[i];
        for (int64_t e = pb + threadIdx.x; e < pe; e += T) {
          const int j = A.sq_col[e];
          const int tgt = A.target[j];
          while (ld_acquire(A.done + j) < tgt) {
            if (*reinterpret_cast<volatile int*>(A.err) != 0) {
              s_stop = 1;
              break;
            }
            sweep_backoff();
          }
          if (s_stop) break;
        }
      }
      __syncthreads();
      if (threadIdx.x == 0 && !s_bready) {
        __threadfence();
        atomicExch(A.bready + i, 1);
      }
    }
    if (threadIdx.x == 0) {
      if (!first) {
        while (ld_acquire(A.done + i) < need) {
          if (*reinterpret_cast<volatile int*>(A.err) != 0) {
            s_stop = 1;
            break;
          }
          sweep_backoff();
        }
      }
      __threadfence();
      nz = 0;
    }
    __syncthreads();
    if (s_stop) break;
    const long long t_run = clock64();
    prof_add(A, kProfWait, t_run - t_wait);
    if (A.trace && threadIdx.x == 0) {
      unsigned long long g;
      unsigned sm;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      A.trace[4 * item + 1] = g;
      A.trace[4 * item + 3] = sm;
    }
    if (stage == 1) {
      task_a1(A, i, s, part, k, tlev, tprev, tprevn, &nz, shr, W);
    } else if (stage == 2) {
      task_a2(A, i, s, nA1, nA3, nB, W);
    } else if (stage == 3) {
      task_a3(A, i, s, k, nA3, nB, W);
    } else {
      const int w = __ldcg(A.width + i);
      const int np = static_cast<int>(A.pan_ptr[i + 1] - A.pan_ptr[i]) - 1;
      if (nB == 1) {
        if (w > 0) all_panels(A, i, __ldcg(A.rank + i), w, s.R);
      } else {
        // task k -> panel P and pairs (P, Q0 .. Q0 + g - 1), Q0 >= P (driver.cpp pair_tasks)
        // Panel P has ceil((np - P) / g) tasks, so the last m panels have
        // T(m) = g q (q + 1) / 2 + (q + 1) r tasks (m = q g + r): closed-form inverse instead of a
        // walk over the panels (hundreds of panels per row at the deep levels, every thread)
        const int g = row_pair_group(A.pair_group, np);
        const int qn = np / g, rn = np - qn * g;
        const int ntask = g * qn * (qn + 1) / 2 + (qn + 1) * rn;
        const int need = ntask - k;  // tasks from this one to the row's last: smallest m with T(m) >= need
        int q = static_cast<int>((sqrt(1.0 + 8.0 * static_cast<double>(need) / g) - 1.0) * 0.5);
        while (q > 0 && g * q * (q + 1) / 2 >= need) --q;
        while (g * (q + 1) * (q + 2) / 2 < need) ++q;
        const int rem = need - g * q * (q + 1) / 2;  // 1 .. g (q + 1)
        const int m = q * g + (rem + q) / (q + 1);
        const int tm = g * q * (q + 1) / 2 + (q + 1) * (m - q * g);
        const int P = np - m, kk = k - (ntask - tm);
        const int q0 = P + kk * g, q1 = min(np, q0 + g);
        for (int Q = q0; Q < q1; ++Q)
          if (w > 0) panel_update(A, i, __ldcg(A.rank + i), w, P, Q, s.R, Q > q0);
        __syncthreads();
        if (threadIdx.x == 0) {  // panel-pair completion for the lookahead waits (above)
          __threadfence();
          for (int Q = q0; Q < q1; ++Q) {
            atomicAdd(A.pdone + A.pan_ptr[i] + P, 1);
            if (Q != P) atomicAdd(A.pdone + A.pan_ptr[i] + Q, 1);
          }
        }
      }
    }
    __syncthreads();
    {
      const int slot = stage == 1 ? kProfA1 : stage == 2 ? kProfA2 : stage == 3 ? kProfA3 : kProfB;
      prof_add(A, slot, clock64() - t_run);
      prof_add(A, stage == 1 ? kProfNA1 : stage == 2 ? kProfNA2 : stage == 3 ? kProfNA3 : kProfNB, 1);
    }
    if (threadIdx.x == 0) {
      if (A.trace) {
        unsigned long long g;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
        A.trace[4 * item + 2] = g;
      }
      __threadfence();
      atomicAdd(A.done + i, 1);
    }
  }
}


#undef CE_SHARED_BUF
#undef CE_SHARED
