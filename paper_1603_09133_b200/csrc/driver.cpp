// Host driver of the B200 CE factorization: per-level symbolic planning,
// the multilevel loop (ce_factorize, proj/src/factorization.cpp:336-461),
// the device preconditioner apply (:140-168), device PCG, stats and dumps.
#include "driver.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <future>
#include <map>
#include <mutex>
#include <thread>
#include <memory>
#include <numeric>
#include <sstream>

#include "kernels.hpp"
#include "pattern.hpp"

namespace ceg {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    std::ostringstream os;
    os << "CUDA error " << cudaGetErrorString(e) << " in " << what;
    throw CudaError(os.str());
  }
}

namespace {

// Task-splitting thresholds of the sweep task graph.  CE_FORCE_TASKS=1 (tests) drops them so
// that small problems exercise the multi-task path of fat rows.
struct Thresholds {
  int64_t pair_inline = int64_t{1} << 19;  // FMA below which a row's Schur pairs stay in A2
  int64_t leaf_work = int64_t{1} << 15;    // far gather f*b^2 above which TSQR leaves are split off
  int64_t leaf_cols = 192;                 // far columns per TSQR leaf (0: min(kcap, 128), the round-1 value)
  int64_t strip_work = int64_t{1} << 15;   // strip rotation S*b^2 above which the strip is split off
  int64_t strip_cols = 192;                // strip columns per task (64 until the chain tickets moved: with the
                                           // chain overlapped, fewer and larger strip / leaf tasks win -- per-level
                                           // A/B in profiles/r2_summary.md: cfg3 sweep 5101 -> 4660 ms)
  bool small_panels = false;               // one close neighbour per Schur panel
  bool no_tri_table = false;               // CE_NO_TRI=1: binary-search slot lookups at every level
  int64_t panel_cap = 0;                   // Schur panel height limit in rows (0: buffer-derived)
  double chain_frac = 0.4;                 // share of rest(w-1) over which wave w's chain tickets are spread
                                           // (build_tickets; 1: the chain follows rest(w-1), the round-1 order;
                                           // A/B on cfg3: 1.0 7250 ms, 0.6 6250, 0.4 6080, 0.25 6180)
  double strip_frac = 1.0;                 // share of rest(w-1) emitted before wave w's strips (>= chain_frac)
  int64_t pre_leaf = -1;                   // rest(w-1) tickets emitted before wave w's TSQR leaves (-1: per-wave rule)
  int64_t pair_group = 0;                  // Schur panel pairs (P, Q..Q+g-1) per task, panel P staged once;
                                           // 0: per row, kernels.hpp row_pair_group(np)
                                           // (A/B on cfg2: g=1 1.82 s, 2 1.89, 3 1.97, 5 2.19: per-wave parallelism wins)
  Thresholds() {
    no_tri_table = std::getenv("CE_NO_TRI") && std::getenv("CE_NO_TRI")[0] == '1';
    const char* f = std::getenv("CE_FORCE_TASKS");  // bitmask: 1 leaves, 2 strip tasks, 4 Schur panels
    const int m = f ? std::atoi(f) : 0;
    if (m & 1) {
      leaf_work = 0;
      leaf_cols = 16;
    }
    if (m & 2) {
      strip_work = 0;
      strip_cols = 16;
    }
    if (m & 4) {
      pair_inline = 0;
      small_panels = true;
    }
    // development overrides
    auto env = [](const char* k, int64_t& v) {
      if (const char* e = std::getenv(k)) v = std::atoll(e);
    };
    env("CE_LEAF_WORK", leaf_work);
    env("CE_LEAF_COLS", leaf_cols);
    env("CE_STRIP_WORK", strip_work);
    env("CE_STRIP_COLS", strip_cols);
    env("CE_PAIR_INLINE", pair_inline);
    env("CE_PAIR_GROUP", pair_group);
    env("CE_PANEL_CAP", panel_cap);
    if (pair_group < 0) pair_group = 0;
    if (const char* e = std::getenv("CE_CHAIN_FRAC")) chain_frac = std::atof(e);
    if (!(chain_frac >= 0.0 && chain_frac <= 1.0)) chain_frac = 0.4;
    if (const char* e = std::getenv("CE_STRIP_FRAC")) strip_frac = std::atof(e);
    if (!(strip_frac >= 0.0 && strip_frac <= 1.0)) strip_frac = 1.0;
    env("CE_PRE_LEAF", pre_leaf);
  }
};
const Thresholds& thresholds() {
  static const Thresholds t;
  return t;
}

}  // namespace

// ---- caching device allocator (host_api.hpp) ----
namespace {
struct Pool {
  std::mutex mu;
  std::multimap<size_t, std::pair<int, void*>> free_blocks;  // rounded bytes -> (device, ptr)
};
Pool& pool() {
  static Pool* p = new Pool();  // intentionally leaked: blocks may be released during static destruction
  return *p;
}
size_t pool_round(size_t bytes) {
  if (bytes <= 4096) return 4096;
  size_t g = size_t{1} << (63 - __builtin_clzll(bytes));  // power of two <= bytes
  g = std::max<size_t>(g / 8, 4096);                       // 12.5% granularity
  return (bytes + g - 1) / g * g;
}
}  // namespace

void* pool_alloc(size_t bytes) {
  const size_t rb = pool_round(bytes);
  int dev = 0;
  cudaGetDevice(&dev);
  {
    Pool& P = pool();
    std::lock_guard<std::mutex> lk(P.mu);
    for (auto it = P.free_blocks.lower_bound(rb); it != P.free_blocks.end() && it->first <= rb + rb / 4; ++it)
      if (it->second.first == dev) {
        void* p = it->second.second;
        P.free_blocks.erase(it);
        return p;
      }
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, rb);
  if (e == cudaErrorMemoryAllocation) {  // drop the cache and retry once
    cudaGetLastError();
    pool_trim();
    e = cudaMalloc(&p, rb);
  }
  CE_CUDA(e);
  return p;
}

void pool_free(void* p, size_t bytes) {
  if (!p) return;
  int dev = 0;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) == cudaSuccess) dev = at.device;
  else cudaGetLastError();
  Pool& P = pool();
  std::lock_guard<std::mutex> lk(P.mu);
  P.free_blocks.emplace(pool_round(bytes), std::make_pair(dev, p));
}

void pool_trim(int device) {
  Pool& P = pool();
  std::lock_guard<std::mutex> lk(P.mu);
  int cur = 0;
  cudaGetDevice(&cur);
  for (auto it = P.free_blocks.begin(); it != P.free_blocks.end();) {
    if (device >= 0 && it->second.first != device) {
      ++it;
      continue;
    }
    cudaSetDevice(it->second.first);
    cudaFree(it->second.second);
    it = P.free_blocks.erase(it);
  }
  cudaSetDevice(cur);
}

namespace {

// Run f(r0, r1) over row chunks on up to 16 host threads (small ranges run inline).
template <class F>
void parallel_rows(int64_t M, F&& f) {
  // CE_HOST_THREADS: host planning threads of this process (one process per GPU: the ranks of a
  // node share its cores, bench.py divides them)
  static const int64_t nt = [] {
    const int64_t hw = std::max<int64_t>(1, static_cast<int64_t>(std::thread::hardware_concurrency()));
    int64_t n = std::min<int64_t>(16, hw);
    if (const char* e = std::getenv("CE_HOST_THREADS")) n = std::max<int64_t>(1, std::min<int64_t>(64, std::atoll(e)));
    return n;
  }();
  if (M < 64 || nt <= 1) {
    f(int64_t{0}, M);
    return;
  }
  std::vector<std::thread> th;
  const int64_t chunk = (M + nt - 1) / nt;
  for (int64_t t = 1; t < nt; ++t) {
    const int64_t a = t * chunk, b = std::min(M, a + chunk);
    if (a < b) th.emplace_back([&f, a, b]() { f(a, b); });
  }
  f(int64_t{0}, std::min(M, chunk));
  for (auto& x : th) x.join();
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

struct Events {
  cudaEvent_t a = nullptr, b = nullptr;
  Events() {
    CE_CUDA(cudaEventCreate(&a));
    CE_CUDA(cudaEventCreate(&b));
  }
  ~Events() {
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
  double seconds() {
    float ms = 0.f;
    CE_CUDA(cudaEventElapsedTime(&ms, a, b));
    return ms * 1e-3;
  }
};

// pattern_square (proj/src/pattern.cpp:64-86), CSR in / CSR out.
template <class F>
void parallel_rows(int64_t M, F&& f);

// sq(P) = pattern of P^2 (sorted rows), two parallel passes: count, then fill + sort.
void square_pattern(int64_t m, const std::vector<int64_t>& ptr, const std::vector<int>& col, std::vector<int64_t>& sptr,
                    std::vector<int>& scol) {
  sptr.assign(static_cast<size_t>(m + 1), 0);
  // Dense deep levels (base degree d > m / 32): row i's square is the OR of the neighbours'
  // rows as bitsets, m d m/64 word operations instead of m d^2 marks (level 7 of cfg3:
  // m = 2048, d ~ 300, 9x fewer operations); sparse levels keep the mark arrays.
  const int64_t nnz = ptr[static_cast<size_t>(m)];
  if (m > 0 && m <= 32768 && nnz * 32 > m * m) {
    const int64_t words = (m + 63) / 64;
    std::vector<uint64_t> nb(static_cast<size_t>(m * words), 0);  // base rows as bitsets
    parallel_rows(m, [&](int64_t r0, int64_t r1) {
      for (int64_t i = r0; i < r1; ++i)
        for (int64_t k = ptr[static_cast<size_t>(i)]; k < ptr[static_cast<size_t>(i + 1)]; ++k) {
          const int j = col[static_cast<size_t>(k)];
          nb[static_cast<size_t>(i * words + j / 64)] |= uint64_t{1} << (j % 64);
        }
    });
    std::vector<std::vector<int>> rows(static_cast<size_t>(m));
    parallel_rows(m, [&](int64_t r0, int64_t r1) {
      std::vector<uint64_t> acc(static_cast<size_t>(words));
      for (int64_t i = r0; i < r1; ++i) {
        std::fill(acc.begin(), acc.end(), 0);
        for (int64_t k = ptr[static_cast<size_t>(i)]; k < ptr[static_cast<size_t>(i + 1)]; ++k) {
          const uint64_t* src = nb.data() + static_cast<int64_t>(col[static_cast<size_t>(k)]) * words;
          for (int64_t w = 0; w < words; ++w) acc[static_cast<size_t>(w)] |= src[w];
        }
        auto& r = rows[static_cast<size_t>(i)];
        for (int64_t w = 0; w < words; ++w)
          for (uint64_t x = acc[static_cast<size_t>(w)]; x; x &= x - 1)
            r.push_back(static_cast<int>(w * 64 + __builtin_ctzll(x)));
      }
    });
    for (int64_t i = 0; i < m; ++i)
      sptr[static_cast<size_t>(i + 1)] = sptr[static_cast<size_t>(i)] + static_cast<int64_t>(rows[static_cast<size_t>(i)].size());
    scol.resize(static_cast<size_t>(sptr[static_cast<size_t>(m)]));
    parallel_rows(m, [&](int64_t r0, int64_t r1) {
      for (int64_t i = r0; i < r1; ++i)
        std::copy(rows[static_cast<size_t>(i)].begin(), rows[static_cast<size_t>(i)].end(),
                  scol.begin() + sptr[static_cast<size_t>(i)]);
    });
    return;
  }
  std::vector<int64_t> cnt(static_cast<size_t>(m), 0);
  parallel_rows(m, [&](int64_t r0, int64_t r1) {
    std::vector<int64_t> mark(static_cast<size_t>(m), -1);
    for (int64_t i = r0; i < r1; ++i) {
      int64_t c = 0;
      for (int64_t k = ptr[static_cast<size_t>(i)]; k < ptr[static_cast<size_t>(i + 1)]; ++k) {
        const int kk = col[static_cast<size_t>(k)];
        for (int64_t e = ptr[static_cast<size_t>(kk)]; e < ptr[static_cast<size_t>(kk + 1)]; ++e) {
          const int j = col[static_cast<size_t>(e)];
          if (mark[static_cast<size_t>(j)] != i) {
            mark[static_cast<size_t>(j)] = i;
            ++c;
          }
        }
      }
      cnt[static_cast<size_t>(i)] = c;
    }
  });
  for (int64_t i = 0; i < m; ++i) sptr[static_cast<size_t>(i + 1)] = sptr[static_cast<size_t>(i)] + cnt[static_cast<size_t>(i)];
  scol.assign(static_cast<size_t>(sptr[static_cast<size_t>(m)]), 0);
  parallel_rows(m, [&](int64_t r0, int64_t r1) {
    std::vector<int64_t> mark(static_cast<size_t>(m), -1);
    for (int64_t i = r0; i < r1; ++i) {
      int64_t at = sptr[static_cast<size_t>(i)];
      for (int64_t k = ptr[static_cast<size_t>(i)]; k < ptr[static_cast<size_t>(i + 1)]; ++k) {
        const int kk = col[static_cast<size_t>(k)];
        for (int64_t e = ptr[static_cast<size_t>(kk)]; e < ptr[static_cast<size_t>(kk + 1)]; ++e) {
          const int j = col[static_cast<size_t>(e)];
          if (mark[static_cast<size_t>(j)] != i) {
            mark[static_cast<size_t>(j)] = i;
            scol[static_cast<size_t>(at++)] = j;
          }
        }
      }
      std::sort(scol.begin() + sptr[static_cast<size_t>(i)], scol.begin() + sptr[static_cast<size_t>(i + 1)]);
    }
  });
}

bool csr_contains(const std::vector<int64_t>& ptr, const std::vector<int>& col, int64_t i, int j) {
  auto b = col.begin() + ptr[static_cast<size_t>(i)], e = col.begin() + ptr[static_cast<size_t>(i + 1)];
  return std::binary_search(b, e, j);
}

int64_t csr_find(const std::vector<int64_t>& ptr, const std::vector<int>& col, int64_t i, int j) {
  auto b = col.begin() + ptr[static_cast<size_t>(i)], e = col.begin() + ptr[static_cast<size_t>(i + 1)];
  auto it = std::lower_bound(b, e, j);
  if (it == e || *it != j) return -1;
  return it - col.begin();
}

}  // namespace

// ---------------------------------------------------------------- planner
// Symbolic part of a level plan (block sizes not needed): squared pattern, entry kinds,
// stored-slot numbering, close lists and the wave order of the row DAG.  Runs on a host
// thread for level l+1 while level l sweeps on the device (speculating that every group
// of level l keeps a nonzero rank).
// dev != nullptr: the caller's device is idle (first level, re-plan after dead groups), so the
// square runs on the GPU (pattern.cu) when the level is large and not dense.
LevelPlan plan_symbolic(int64_t M, std::vector<int64_t> bptr, std::vector<int> bcol, cudaStream_t dev = nullptr) {
  LevelPlan P;
  P.M = M;
  P.bptr = std::move(bptr);
  P.bcol = std::move(bcol);
  for (int64_t i = 0; i < M; ++i)
    for (int64_t k = P.bptr[static_cast<size_t>(i)]; k < P.bptr[static_cast<size_t>(i + 1)]; ++k)
      if (P.bcol[static_cast<size_t>(k)] <= i) ++P.lower_blocks;

  const bool prof = std::getenv("CE_PROFILE") && std::getenv("CE_PROFILE")[0] == '1';
  const double t0 = now_s();
  if (dev && M >= 16384 && square_candidates(M, P.bptr, P.bcol) <= (int64_t{1} << 26))
    device_square(M, P.bptr, P.bcol, dev, P.sptr, P.scol);
  else
    square_pattern(M, P.bptr, P.bcol, P.sptr, P.scol);
  const double t1 = now_s();
  const int64_t nnz = static_cast<int64_t>(P.scol.size());
  P.skind.resize(static_cast<size_t>(nnz));
  P.sslot.assign(static_cast<size_t>(nnz), -1);
  parallel_rows(M, [&](int64_t r0, int64_t r1) {
    for (int64_t i = r0; i < r1; ++i)
      for (int64_t e = P.sptr[static_cast<size_t>(i)]; e < P.sptr[static_cast<size_t>(i + 1)]; ++e) {
        const int j = P.scol[static_cast<size_t>(e)];
        P.skind[static_cast<size_t>(e)] = j == i ? 0 : (csr_contains(P.bptr, P.bcol, i, j) ? 1 : 2);
      }
  });
  // stored (lower) slots numbered row by row: per-row counts, prefix, parallel fill
  std::vector<int64_t> lower_at(static_cast<size_t>(M) + 1, 0);
  parallel_rows(M, [&](int64_t r0, int64_t r1) {
    for (int64_t i = r0; i < r1; ++i) {
      int64_t c = 0;
      for (int64_t e = P.sptr[static_cast<size_t>(i)]; e < P.sptr[static_cast<size_t>(i + 1)]; ++e) {
        if (P.scol[static_cast<size_t>(e)] > i) break;
        ++c;
      }
      lower_at[static_cast<size_t>(i) + 1] = c;
    }
  });
  for (int64_t i = 0; i < M; ++i) lower_at[static_cast<size_t>(i) + 1] += lower_at[static_cast<size_t>(i)];
  parallel_rows(M, [&](int64_t r0, int64_t r1) {
    for (int64_t i = r0; i < r1; ++i) {
      int64_t slot = lower_at[static_cast<size_t>(i)];
      for (int64_t e = P.sptr[static_cast<size_t>(i)]; e < P.sptr[static_cast<size_t>(i + 1)]; ++e) {
        if (P.scol[static_cast<size_t>(e)] > i) break;
        P.sslot[static_cast<size_t>(e)] = slot++;
      }
    }
  });
  P.nslots = lower_at[static_cast<size_t>(M)];
  parallel_rows(M, [&](int64_t r0, int64_t r1) {
    for (int64_t i = r0; i < r1; ++i)
      for (int64_t e = P.sptr[static_cast<size_t>(i)]; e < P.sptr[static_cast<size_t>(i + 1)]; ++e) {
        const int j = P.scol[static_cast<size_t>(e)];
        if (j <= i) continue;
        P.sslot[static_cast<size_t>(e)] = P.sslot[static_cast<size_t>(csr_find(P.sptr, P.scol, j, static_cast<int>(i)))];
      }
  });

  P.cptr.assign(static_cast<size_t>(M + 1), 0);
  for (int64_t i = 0; i < M; ++i) {
    for (int64_t k = P.bptr[static_cast<size_t>(i)]; k < P.bptr[static_cast<size_t>(i + 1)]; ++k) {
      const int t = P.bcol[static_cast<size_t>(k)];
      if (t == i) continue;
      P.ccol.push_back(t);
    }
    P.cptr[static_cast<size_t>(i + 1)] = static_cast<int64_t>(P.ccol.size());
    P.cmax = std::max<int64_t>(P.cmax, static_cast<int64_t>(P.cptr[static_cast<size_t>(i + 1)] - P.cptr[static_cast<size_t>(i)]));
  }
  P.sdiag.resize(static_cast<size_t>(M));
  for (int64_t i = 0; i < M; ++i) P.sdiag[static_cast<size_t>(i)] = csr_find(P.sptr, P.scol, i, static_cast<int>(i));
  // Far blocks still exactly zero when their row is compressed (kind 3): a far block (i, j)
  // starts at zero (not in the level's base pattern) and only the Schur update of an earlier
  // row k with i, j in close(k) writes it (level_matrix.cpp:148-162).  Without such a k < i
  // it contributes zero columns to F_i, and the compression gather / strip skip it; sizes,
  // nsig and the F-empty test keep counting it (kind 2 or 3 = far).
  if (!(std::getenv("CE_NO_DEAD_FAR") && std::getenv("CE_NO_DEAD_FAR")[0] == '1'))
    parallel_rows(M, [&](int64_t r0, int64_t r1) {
      std::vector<int64_t> mark(static_cast<size_t>(M), -1);
      for (int64_t i = r0; i < r1; ++i) {
        for (int64_t k = P.cptr[static_cast<size_t>(i)]; k < P.cptr[static_cast<size_t>(i + 1)]; ++k) {
          const int t = P.ccol[static_cast<size_t>(k)];
          if (t < i) mark[static_cast<size_t>(t)] = i;
        }
        for (int64_t e = P.sptr[static_cast<size_t>(i)]; e < P.sptr[static_cast<size_t>(i + 1)]; ++e) {
          if (P.skind[static_cast<size_t>(e)] != 2) continue;
          const int j = P.scol[static_cast<size_t>(e)];
          bool live = false;
          for (int64_t k = P.cptr[static_cast<size_t>(j)]; k < P.cptr[static_cast<size_t>(j + 1)] && !live; ++k) {
            const int t = P.ccol[static_cast<size_t>(k)];
            live = t < i && mark[static_cast<size_t>(t)] == i;
          }
          if (!live) P.skind[static_cast<size_t>(e)] = 3;
        }
      }
    });
  // Wave (topological) order of the dependency DAG: row j depends on every i < j in sq(j)
  // (SURVEY.md A.2).  Items are issued in this order, so the ticket window always holds
  // the current wavefront instead of a run of consecutive (mutually dependent) rows.
  P.wave.assign(static_cast<size_t>(M), 0);
  for (int64_t j = 0; j < M; ++j) {
    int64_t w = 0;
    for (int64_t e = P.sptr[static_cast<size_t>(j)]; e < P.sptr[static_cast<size_t>(j + 1)]; ++e) {
      const int i = P.scol[static_cast<size_t>(e)];
      if (i >= j) break;
      w = std::max(w, P.wave[static_cast<size_t>(i)] + 1);
    }
    P.wave[static_cast<size_t>(j)] = w;
    P.n_waves = std::max(P.n_waves, w + 1);
  }
  P.order.resize(static_cast<size_t>(M));
  std::iota(P.order.begin(), P.order.end(), 0);
  std::stable_sort(P.order.begin(), P.order.end(),
                   [&](int x, int y) { return P.wave[static_cast<size_t>(x)] < P.wave[static_cast<size_t>(y)]; });
  if (prof)
    std::fprintf(stderr, "[ce-profile] plan_symbolic M=%lld nnz=%zu: square %.1f ms, rest %.1f ms\n", static_cast<long long>(M),
                 P.scol.size(), 1e3 * (t1 - t0), 1e3 * (now_s() - t1));
  return P;
}

// Schur tasks of a row with np panels: for each P, the pairs (P, Q >= P) in groups of g.
int64_t pair_tasks(int64_t np, int64_t g) {
  int64_t t = 0;
  for (int64_t p = 0; p < np; ++p) t += (np - p + g - 1) / g;
  return t;
}

// Ticket order of the row tasks (wave order from the symbolic plan; plan_numeric's comment):
// wave by wave, stage by stage across the wave's rows, with the lookahead split of every
// row's Schur pairs into urgent (urg_of) / rest (rest_of).  `mask` (optional) restricts the
// tickets to a subset of rows -- the sharded sweep's phases; the relative order
// of the kept tickets is unchanged, so every wait is still on an earlier ticket.
void build_tickets(const LevelPlan& P, const std::vector<char>* mask, std::vector<int>& item_row,
                   std::vector<int>& item_part) {
  const int64_t M = P.M;
  const std::vector<int64_t>& wave = P.wave;
  // Segments of a wave w: leaves(w), rest(w-1), the TSQR combines of w by tree level (kLv
  // segments; deeper levels share the last one, row-major, so a node still follows its
  // children), A2(w), strips(w), urgent(w).  The emitted order is
  //   [leaves(w)] [rest(w-1) with w's chain stages -- combine levels, then A2 -- interleaved]
  //   [strips(w)] [urgent(w)],
  // rows in `order` within each segment.  The chain of a wave is a handful of short serial
  // tasks (one CTA each) while rest(w-1) is hundreds of independent Schur tasks: with the chain
  // after rest(w-1) its tickets are only taken once every rest ticket is out, so the chain
  // runs when the grid has nothing else left and every wave pays it in idle CTAs.  Chain stage
  // s of S is instead placed after the first chain_frac (s+1)/S of rest(w-1): it is taken
  // about when it becomes ready, a too-early pick parks one CTA, and rest(w-1) keeps the other
  // CTAs busy meanwhile.  (The strips stay behind rest(w-1): there are hundreds per row, and
  // parked strip tickets would hold the whole grid.)  Every row's share of each segment is
  // known up front, so segment starts come from prefix sums over the rows and the rows fill
  // their slots in parallel (the tickets of one level are millions of items).
  constexpr int kLv = 8;
  constexpr int kSeg = 5 + kLv;  // 0 leaves, 1 rest, 2..2+kLv-1 combine levels, then A2, strips, urgent
  constexpr int sA2 = 2 + kLv, sStrip = 3 + kLv, sUrg = 4 + kLv;
  constexpr int kStage = kLv + 3;  // stages inserted into rest(w-1): leaves, combine levels, A2, strips
  auto stage_seg = [](int st) { return st == 0 ? 0 : (st == kStage - 1 ? sStrip : 1 + st); };
  const double frac = thresholds().chain_frac;
  const double sfrac = std::max(thresholds().strip_frac, frac);
  const int64_t kcap = sweep_kcap(std::max(P.bmax, 1));
  std::vector<int64_t> wstart;
  for (int64_t k = 0; k < M;) {
    wstart.push_back(k);
    const int64_t wv = wave[static_cast<size_t>(P.order[static_cast<size_t>(k)])];
    while (k < M && wave[static_cast<size_t>(P.order[static_cast<size_t>(k)])] == wv) ++k;
  }
  wstart.push_back(M);
  const int64_t nw = static_cast<int64_t>(wstart.size()) - 1;
  // rest(w-1) tickets emitted before leaves(w).  The leaves wait for urgent(w-1); when that
  // segment has fewer tickets than the grid has CTAs, the other CTAs would park on the leaves for
  // about one Schur task, and a round of rest tickets fills the gap -- if rest(w-1) is large
  // enough that the chain placed in it is not delayed (cfg3 levels 7 / 8: -3% / -6%).  A fixed
  // count everywhere loses on the other levels (+1-5%: cfg3 levels 5, 6, 9, cfg2 levels 7, 8), so
  // the rule is per wave; CE_PRE_LEAF >= 0 forces a count.
  const int64_t pre_force = thresholds().pre_leaf;
  constexpr int64_t kGrid = 148;  // CTAs of the persistent sweep on a B200 (a scheduling hint only)
  // combine nodes of `row` per tree level (sweep_body.cuh sweep_kernel: leaves first, then
  // levels of F-way combines down to one triangle)
  auto comb_levels = [&](size_t r, int64_t* lv) {
    for (int l = 0; l < kLv; ++l) lv[l] = 0;
    if (P.nA1[r] <= P.nleaf[r]) return;
    const int64_t F = std::max<int64_t>(2, kcap / std::max<int64_t>(P.bsz[r], 1));
    int l = 0;
    for (int64_t n = (P.nleaf[r] + F - 1) / F;; n = (n + F - 1) / F) {
      lv[std::min(l, kLv - 1)] += n;
      ++l;
      if (n == 1) break;
    }
  };
  auto counts = [&](int row, int64_t* c) {
    const size_t r = static_cast<size_t>(row);
    for (int s = 0; s < kSeg; ++s) c[s] = 0;
    if (mask && !(*mask)[r]) return;
    c[0] = P.nleaf[r];
    c[1] = static_cast<int64_t>(P.rest_of[r].size());
    comb_levels(r, c + 2);
    c[sA2] = 1;
    c[sStrip] = P.nA3[r];
    c[sUrg] = static_cast<int64_t>(P.urg_of[r].size());
  };
  // start[k * kSeg + seg]: first ticket of the row at order position k inside segment seg
  std::vector<int64_t> start(static_cast<size_t>(M) * kSeg, 0), segsum(static_cast<size_t>(nw) * kSeg, 0);
  parallel_rows(nw, [&](int64_t w0, int64_t w1) {
    int64_t c[kSeg], t[kSeg];
    for (int64_t w = w0; w < w1; ++w) {
      for (int s = 0; s < kSeg; ++s) t[s] = 0;
      for (int64_t k = wstart[static_cast<size_t>(w)]; k < wstart[static_cast<size_t>(w + 1)]; ++k) {
        counts(P.order[static_cast<size_t>(k)], c);
        for (int s = 0; s < kSeg; ++s) {
          start[static_cast<size_t>(k) * kSeg + static_cast<size_t>(s)] = t[s];
          t[s] += c[s];
        }
      }
      for (int s = 0; s < kSeg; ++s) segsum[static_cast<size_t>(w) * kSeg + static_cast<size_t>(s)] = t[s];
    }
  });
  // segment bases in emission order.  Section w holds rest(w-1) with the stages of wave w
  // inserted at cut[w][st] (rest items emitted before stage st), then urgent(w); a rest item g of
  // wave w-1 lands at base + g + (items of the stages cut at or before g).  Stages: leaves,
  // combine levels, A2, strips.  urgent(w) follows all of rest(w-1): a row's Schur tasks wait
  // for every task of its predecessors, rest(w-1) included.
  std::vector<int64_t> base(static_cast<size_t>(nw + 1) * kSeg, 0);
  std::vector<int64_t> cut(static_cast<size_t>(nw + 1) * kStage, 0);
  int64_t at = 0;
  auto seg_n = [&](int64_t w, int s) { return segsum[static_cast<size_t>(w) * kSeg + static_cast<size_t>(s)]; };
  for (int64_t w = 0; w <= nw; ++w) {
    const int64_t R = w > 0 ? seg_n(w - 1, 1) : 0;
    if (w > 0) base[static_cast<size_t>(w - 1) * kSeg + 1] = at;  // rest(w-1): position of its item 0
    int64_t done = 0;  // rest items already emitted
    if (w < nw) {
      // chain stages (combine levels, A2) present in this wave
      int S = 0, si = 0;
      for (int s = 0; s <= kLv; ++s)
        if (seg_n(w, 2 + s) > 0) ++S;
      const int64_t U = w > 0 ? seg_n(w - 1, sUrg) : 0;
      int64_t pre = 0;
      if (pre_force >= 0) pre = pre_force;
      else if (U > 0 && U < kGrid && R > 4 * kGrid) pre = std::min<int64_t>(R / 4, 2 * kGrid);
      pre = std::min<int64_t>(R, pre);
      for (int st = 0; st < kStage; ++st) {
        const int seg = stage_seg(st);
        const int64_t n = seg_n(w, seg);
        int64_t c = done;  // an empty stage cuts nothing
        if (n > 0) {
          if (st == 0) {
            c = pre;
          } else if (st == kStage - 1) {
            c = sfrac >= 1.0 ? R : pre + static_cast<int64_t>(sfrac * static_cast<double>(R - pre));
          } else {
            ++si;
            c = frac >= 1.0 ? R : pre + static_cast<int64_t>(frac * static_cast<double>(R - pre) * si / S);
          }
          c = std::max(std::min(c, R), done);
        }
        cut[static_cast<size_t>(w) * kStage + static_cast<size_t>(st)] = c;
        at += c - done;
        done = c;
        base[static_cast<size_t>(w) * kSeg + static_cast<size_t>(seg)] = at;
        at += n;
      }
    }
    at += R - done;
    if (w == nw) break;
    base[static_cast<size_t>(w) * kSeg + sUrg] = at;
    at += seg_n(w, sUrg);
  }
  item_row.assign(static_cast<size_t>(at), 0);
  item_part.assign(static_cast<size_t>(at), 0);
  parallel_rows(nw, [&](int64_t w0, int64_t w1) {
    int64_t lv[kLv];
    for (int64_t w = w0; w < w1; ++w)
      for (int64_t k = wstart[static_cast<size_t>(w)]; k < wstart[static_cast<size_t>(w + 1)]; ++k) {
        const int row = P.order[static_cast<size_t>(k)];
        const size_t r = static_cast<size_t>(row);
        if (mask && !(*mask)[r]) continue;
        auto put = [&](int seg, int64_t j, int part) {
          int64_t idx = base[static_cast<size_t>(w) * kSeg + static_cast<size_t>(seg)] +
                        start[static_cast<size_t>(k) * kSeg + static_cast<size_t>(seg)] + j;
          if (seg == 1 && w + 1 < nw) {
            // rest item g of wave w: shifted by the chain stages of wave w+1 cut at or before g
            const int64_t g = start[static_cast<size_t>(k) * kSeg + 1] + j;
            for (int st = 0; st < kStage; ++st)
              if (cut[static_cast<size_t>(w + 1) * kStage + static_cast<size_t>(st)] <= g)
                idx += seg_n(w + 1, stage_seg(st));
          }
          item_row[static_cast<size_t>(idx)] = row;
          item_part[static_cast<size_t>(idx)] = part;
        };
        for (int p = 0; p < P.nleaf[r]; ++p) put(0, p, p);
        for (size_t j = 0; j < P.rest_of[r].size(); ++j) put(1, static_cast<int64_t>(j), P.rest_of[r][j]);
        if (P.nA1[r] > P.nleaf[r]) {
          comb_levels(r, lv);
          // tree levels in part order; levels >= kLv - 1 share the last segment
          const int64_t F = std::max<int64_t>(2, kcap / std::max<int64_t>(P.bsz[r], 1));
          int p = P.nleaf[r], l = 0;
          int64_t in_last = 0;
          for (int64_t n = (P.nleaf[r] + F - 1) / F;; n = (n + F - 1) / F, ++l) {
            const int seg = std::min(l, kLv - 1);
            for (int64_t q = 0; q < n; ++q, ++p) put(2 + seg, (seg == kLv - 1 ? in_last : 0) + q, p);
            if (seg == kLv - 1) in_last += n;
            if (n == 1) break;
          }
        }
        put(sA2, 0, P.nA1[r]);
        for (int p = 0; p < P.nA3[r]; ++p) put(sStrip, p, P.nA1[r] + 1 + p);
        for (size_t j = 0; j < P.urg_of[r].size(); ++j) put(sUrg, static_cast<int64_t>(j), P.urg_of[r][j]);
      }
  });
}

// Numeric part: everything that depends on the block sizes.
void plan_numeric(LevelPlan& P, std::vector<int> bsz) {
  const int64_t M = P.M;
  const double tn0 = now_s();
  P.bsz = std::move(bsz);
  P.offsets.assign(static_cast<size_t>(M + 1), 0);
  for (int64_t i = 0; i < M; ++i) P.offsets[static_cast<size_t>(i + 1)] = P.offsets[static_cast<size_t>(i)] + P.bsz[static_cast<size_t>(i)];
  P.dim = P.offsets.back();
  P.bmax = 0;
  for (int b : P.bsz) P.bmax = std::max(P.bmax, b);
  P.slot_off.assign(static_cast<size_t>(P.nslots), 0);
  // stored lower blocks in row order: per-row sizes, prefix, then every row's offsets (parallel)
  std::vector<int64_t> row_doubles(static_cast<size_t>(M) + 1, 0);
  parallel_rows(M, [&](int64_t r0, int64_t r1) {
    for (int64_t i = r0; i < r1; ++i) {
      int64_t t = 0;
      for (int64_t e = P.sptr[static_cast<size_t>(i)]; e < P.sptr[static_cast<size_t>(i + 1)]; ++e) {
        const int j = P.scol[static_cast<size_t>(e)];
        if (j > i) break;
        t += static_cast<int64_t>(P.bsz[static_cast<size_t>(i)]) * P.bsz[static_cast<size_t>(j)];
      }
      row_doubles[static_cast<size_t>(i) + 1] = t;
    }
  });
  for (int64_t i = 0; i < M; ++i) row_doubles[static_cast<size_t>(i) + 1] += row_doubles[static_cast<size_t>(i)];
  P.csum.assign(static_cast<size_t>(M), 0);
  P.fsum.assign(static_cast<size_t>(M), 0);
  P.croff.assign(P.ccol.size(), 0);
  parallel_rows(M, [&](int64_t r0, int64_t r1) {
    for (int64_t i = r0; i < r1; ++i) {
      int64_t off = row_doubles[static_cast<size_t>(i)];
      for (int64_t e = P.sptr[static_cast<size_t>(i)]; e < P.sptr[static_cast<size_t>(i + 1)]; ++e) {
        const int j = P.scol[static_cast<size_t>(e)];
        if (j > i) break;
        P.slot_off[static_cast<size_t>(P.sslot[static_cast<size_t>(e)])] = off;
        off += static_cast<int64_t>(P.bsz[static_cast<size_t>(i)]) * P.bsz[static_cast<size_t>(j)];
      }
      int64_t c = 0;
      for (int64_t k = P.cptr[static_cast<size_t>(i)]; k < P.cptr[static_cast<size_t>(i + 1)]; ++k) {
        P.croff[static_cast<size_t>(k)] = static_cast<int>(c);
        c += P.bsz[static_cast<size_t>(P.ccol[static_cast<size_t>(k)])];
      }
      P.csum[static_cast<size_t>(i)] = c;
      int64_t f = 0;
      for (int64_t e = P.sptr[static_cast<size_t>(i)]; e < P.sptr[static_cast<size_t>(i + 1)]; ++e)
        if (P.skind[static_cast<size_t>(e)] >= 2) f += P.bsz[static_cast<size_t>(P.scol[static_cast<size_t>(e)])];
      P.fsum[static_cast<size_t>(i)] = f;
    }
  });
  P.store_doubles = row_doubles[static_cast<size_t>(M)];
  P.fmax = 0;
  for (int64_t i = 0; i < M; ++i) P.fmax = std::max(P.fmax, P.fsum[static_cast<size_t>(i)]);
  P.chol_off.resize(static_cast<size_t>(M));
  P.g_off.resize(static_cast<size_t>(M));
  P.basis_off.resize(static_cast<size_t>(M));
  P.sigma_off.resize(static_cast<size_t>(M));
  P.item_start.assign(static_cast<size_t>(M + 1), 0);
  P.nA1.assign(static_cast<size_t>(M), 0);
  P.nA3.assign(static_cast<size_t>(M), 0);
  P.nB.assign(static_cast<size_t>(M), 0);
  P.rs_off.assign(static_cast<size_t>(M), 0);
  P.pan_ptr.assign(static_cast<size_t>(M + 1), 0);
  // Schur panel height: both panels' g rows (<= cap x w doubles each) must fit the CTA buffer.
  const int64_t bmax = std::max(P.bmax, 1);
  const int64_t buf = sweep_smem_doubles(static_cast<int>(bmax), sweep_kcap(static_cast<int>(bmax)));
  // (sweep.cu kPanelRows / kPanelNb bound the panel height / neighbour count)
  // (rows + 16 bounds the padded row strides of both staged panels, sweep_body.cuh panel_update)
  int64_t cap = thresholds().small_panels ? bmax : std::max<int64_t>(bmax, std::min<int64_t>(256, buf / (2 * bmax) - 16));
  if (thresholds().panel_cap > 0) cap = std::max<int64_t>(bmax, std::min(cap, thresholds().panel_cap));
  constexpr int64_t kPanelNb = 32;
  const double tp1 = now_s();
  // per-row task counts (parallel over rows), then prefix offsets
  const Thresholds& th = thresholds();
  const int64_t kcap = sweep_kcap(static_cast<int>(bmax));
  // far columns per TSQR leaf (<= 128: the register-resident leaf QR)
  const int64_t lcols = th.leaf_cols > 0 ? th.leaf_cols : std::min<int64_t>(kcap, 128);
  P.nleaf.assign(static_cast<size_t>(M), 0);
  std::vector<int> np_row(static_cast<size_t>(M), 0);
  parallel_rows(M, [&](int64_t r0, int64_t r1) {
    for (int64_t i = r0; i < r1; ++i) {
      const size_t iu = static_cast<size_t>(i);
      const int64_t b = P.bsz[iu];
      // A1: TSQR leaves when the far gather is large (work ~ f b^2)
      int64_t nfar = 0, nstrip = 0, strip_cols = 0, flive = 0;
      for (int64_t e = P.sptr[iu]; e < P.sptr[iu + 1]; ++e) {
        const unsigned char kind = P.skind[static_cast<size_t>(e)];
        if (kind == 2) {
          ++nfar;
          flive += P.bsz[static_cast<size_t>(P.scol[static_cast<size_t>(e)])];
        }
        if (kind == 1 || kind == 2) {
          ++nstrip;
          strip_cols += P.bsz[static_cast<size_t>(P.scol[static_cast<size_t>(e)])];
        }
      }
      if (flive * b * b > th.leaf_work && flive > lcols) {
        // TSQR tree: leaves of <= lcols far columns (greedy over the far blocks), then
        // levels combining F = max(2, kcap / b) triangles each, down to one triangle
        int64_t n0 = 0, cols = 0;
        for (int64_t e = P.sptr[iu]; e < P.sptr[iu + 1]; ++e) {
          if (P.skind[static_cast<size_t>(e)] != 2) continue;
          const int64_t bj = P.bsz[static_cast<size_t>(P.scol[static_cast<size_t>(e)])];
          if (n0 == 0 || cols + bj > lcols) {
            ++n0;
            cols = 0;
          }
          cols += bj;
        }
        if (n0 >= 2) {
          const int64_t F = std::max<int64_t>(2, kcap / std::max<int64_t>(b, 1));
          int64_t items = 0;
          for (int64_t n = n0;; n = (n + F - 1) / F) {
            items += n;
            if (n == 1) break;
          }
          P.nleaf[iu] = static_cast<int>(n0);
          P.nA1[iu] = static_cast<int>(items);
        }
      }
      // A3: strip tasks when rotating the strip is large (work ~ S b^2)
      if (strip_cols * b * b > th.strip_work) {
        const int64_t tasks = std::min<int64_t>(nstrip, (strip_cols + th.strip_cols - 1) / th.strip_cols);
        if (tasks >= 2) P.nA3[iu] = static_cast<int>(tasks);
      }
      // B: Schur panels of the close list (greedy, <= cap rows each)
      int64_t np = 0, rows = 0, nbs = 0, sq2 = 0;
      for (int64_t k = P.cptr[iu]; k < P.cptr[iu + 1]; ++k) {
        const int64_t bt = P.bsz[static_cast<size_t>(P.ccol[static_cast<size_t>(k)])];
        if (np == 0 || rows + bt > cap || nbs == kPanelNb) {
          ++np;
          rows = 0;
          nbs = 0;
        }
        rows += bt;
        ++nbs;
        sq2 += bt * bt;
      }
      np_row[iu] = static_cast<int>(np);
      // Schur pair work: sum_{s<=t in close} b_s b_t * w, with w <= b
      const int64_t cs = P.csum[iu];
      const int64_t work = (cs * cs + sq2) / 2 * b;
      if (work > th.pair_inline && np * (np + 1) / 2 > 1) P.nB[iu] = static_cast<int>(pair_tasks(np, row_pair_group(static_cast<int>(th.pair_group), static_cast<int>(np))));
      // with strip tasks the Schur update must follow all of them: one task runs every panel pair
      if (P.nA3[iu] > 0 && P.nB[iu] == 0 && np > 0) P.nB[iu] = 1;
    }
  });
  int64_t fo = 0, bo = 0, so = 0, ro = 0;
  for (int64_t i = 0; i < M; ++i) {
    const size_t iu = static_cast<size_t>(i);
    const int64_t b = P.bsz[iu];
    P.chol_off[iu] = fo;
    fo += b * b;
    P.g_off[iu] = fo;
    fo += (b + P.csum[iu]) * b;
    P.basis_off[iu] = bo;
    bo += b * b;
    P.sigma_off[iu] = so;
    so += std::min<int64_t>(b, P.fsum[iu]);
    if (P.nA1[iu] > 0) {
      P.rs_off[iu] = ro;
      ro += static_cast<int64_t>(P.nA1[iu]) * b * b;
    }
    P.pan_ptr[iu + 1] = P.pan_ptr[iu] + np_row[iu] + 1;
  }
  P.rscratch_doubles = ro;
  const double tp2 = now_s();
  P.pan_start.assign(static_cast<size_t>(P.pan_ptr[static_cast<size_t>(M)]), 0);
  parallel_rows(M, [&](int64_t r0, int64_t r1) {
    for (int64_t i = r0; i < r1; ++i) {
      const size_t iu = static_cast<size_t>(i);
      int64_t at = P.pan_ptr[iu], np = 0, rows = 0, nbs = 0;
      for (int64_t k = P.cptr[iu]; k < P.cptr[iu + 1]; ++k) {
        const int64_t bt = P.bsz[static_cast<size_t>(P.ccol[static_cast<size_t>(k)])];
        if (np == 0 || rows + bt > cap || nbs == kPanelNb) {
          P.pan_start[static_cast<size_t>(at++)] = static_cast<int>(k - P.cptr[iu]);
          ++np;
          rows = 0;
          nbs = 0;
        }
        rows += bt;
        ++nbs;
      }
      P.pan_start[static_cast<size_t>(at)] = static_cast<int>(P.cptr[iu + 1] - P.cptr[iu]);
    }
  });
  const double tp3 = now_s();
  // Per-entry metadata the sweep tasks load in one coalesced pass (no dependent chains
  // sq_col -> bsz, sq_slot -> slot_off, close-list search on the device), the diagonal
  // entry and completion target of every row, and the entry ranges of the A1 / A3 tasks
  // (same far-ordinal / strip-ordinal partitions as before).
  {
    const size_t nnz = P.scol.size();
    P.sboff.resize(nnz);
    P.sbsz.resize(nnz);
    P.sroff.assign(nnz, -1);
    P.target.resize(static_cast<size_t>(M));
    P.leaf_ptr.assign(static_cast<size_t>(M + 1), 0);
    P.strip_ptr.assign(static_cast<size_t>(M + 1), 0);
    for (int64_t i = 0; i < M; ++i) {
      const size_t iu = static_cast<size_t>(i);
      P.target[iu] = 1 + P.nA1[iu] + P.nA3[iu] + P.nB[iu];
      P.leaf_ptr[iu + 1] = P.leaf_ptr[iu] + P.nleaf[iu] + 1;
      P.strip_ptr[iu + 1] = P.strip_ptr[iu] + P.nA3[iu] + 1;
    }
    P.leaf_e.assign(static_cast<size_t>(P.leaf_ptr[static_cast<size_t>(M)]), 0);
    P.strip_e.assign(static_cast<size_t>(P.strip_ptr[static_cast<size_t>(M)]), 0);
    parallel_rows(M, [&](int64_t r0, int64_t r1) {
      for (int64_t i = r0; i < r1; ++i) {
        const size_t iu = static_cast<size_t>(i);
        int64_t nf = 0, ns = 0;
        int64_t kc = P.cptr[iu];  // close(i) is the ascending sub-list of sq(i) with kind 1: walk both
        for (int64_t e = P.sptr[iu]; e < P.sptr[iu + 1]; ++e) {
          const size_t eu = static_cast<size_t>(e);
          const int j = P.scol[eu];
          P.sboff[eu] = P.slot_off[static_cast<size_t>(P.sslot[eu])];
          P.sbsz[eu] = P.bsz[static_cast<size_t>(j)];
          if (P.skind[eu] == 1) {
            while (kc < P.cptr[iu + 1] && P.ccol[static_cast<size_t>(kc)] < j) ++kc;
            if (kc == P.cptr[iu + 1] || P.ccol[static_cast<size_t>(kc)] != j) throw std::logic_error("close entry missing from the close list");
            P.sroff[eu] = P.croff[static_cast<size_t>(kc)];
          }
          nf += P.skind[eu] == 2;
          ns += P.skind[eu] == 1 || P.skind[eu] == 2;
        }
        // leaf boundaries: greedy packing of the far blocks into <= lcols columns (as counted);
        // strip task k starts at the strip entry with ordinal ns k / nA3 (row end if none)
        const int64_t pend = P.sptr[iu + 1];
        const int nl = P.nleaf[iu], na3 = P.nA3[iu];
        int kl = 0, ks = 0;
        int64_t os = 0, cols = 0;
        auto next_o = [](int64_t n, int k, int parts) { return parts > 0 ? n * k / parts : 0; };
        for (int64_t e = P.sptr[iu]; e < pend; ++e) {
          const unsigned char kind = P.skind[static_cast<size_t>(e)];
          if (kind == 2 && nl > 0) {
            const int64_t bj = P.sbsz[static_cast<size_t>(e)];
            if (kl == 0 || cols + bj > lcols) {
              P.leaf_e[static_cast<size_t>(P.leaf_ptr[iu] + kl++)] = e;
              cols = 0;
            }
            cols += bj;
          }
          if (kind == 1 || kind == 2) {
            while (ks <= na3 && next_o(ns, ks, na3) == os && os < ns) P.strip_e[static_cast<size_t>(P.strip_ptr[iu] + ks++)] = e;
            ++os;
          }
        }
        while (kl <= nl) P.leaf_e[static_cast<size_t>(P.leaf_ptr[iu] + kl++)] = pend;
        while (ks <= na3) P.strip_e[static_cast<size_t>(P.strip_ptr[iu] + ks++)] = pend;
        (void)nf;
      }
    });
  }
  const double tp4 = now_s();
  double tp5 = tp4;
  // ticket order of the row tasks (wave order from the symbolic plan)
  {
    const std::vector<int64_t>& wave = P.wave;
    int64_t it = 0;
    for (int64_t k = 0; k < M; ++k) {
      P.item_start[static_cast<size_t>(k)] = it;
      const size_t r = static_cast<size_t>(P.order[static_cast<size_t>(k)]);
      it += 1 + P.nA1[r] + P.nA3[r] + P.nB[r];
    }
    P.item_start[static_cast<size_t>(M)] = it;
    P.n_items = it;
    // Ticket order: wave by wave, and inside a wave stage by stage across its (independent)
    // rows, so the rows of one wave advance through their stages together.  Lookahead: the
    // Schur panel pairs of wave k that touch a row of wave k+1 ("urgent", U) are issued right
    // after wave k's A stages; wave k+1's TSQR leaves follow, then wave k's remaining pairs
    // (R), then wave k+1's tree combines, A2 and strips.  R(k) thus fills the CTAs while wave
    // k+1's compression chain runs (the A stages of one row leave most CTAs idle).  A row's A
    // stages wait only for the pairs of its close predecessors that touch its own panel
    // (sq_pan), its Schur pairs for every task of every predecessor; every wait is on an
    // earlier ticket (no deadlock).  Rows whose Schur update is 0 or 1 task keep the full wait.
    P.rest_of.assign(static_cast<size_t>(M), {});
    P.urg_of.assign(static_cast<size_t>(M), {});
    auto& rest_of = P.rest_of;
    auto& urg_of = P.urg_of;
    const bool lookahead = !(std::getenv("CE_NO_LOOKAHEAD") && std::getenv("CE_NO_LOOKAHEAD")[0] == '1');
    parallel_rows(M, [&](int64_t r0, int64_t r1) {
      std::vector<char> hot;
      for (int64_t i = r0; i < r1; ++i) {
        const size_t iu = static_cast<size_t>(i);
        const int nb = P.nB[iu];
        if (nb == 0) continue;
        const int np = static_cast<int>(P.pan_ptr[iu + 1] - P.pan_ptr[iu]) - 1;
        const int b0 = P.nA1[iu] + 1 + P.nA3[iu];
        if (nb == 1 || !lookahead) {
          for (int k = 0; k < nb; ++k) urg_of[iu].push_back(b0 + k);
          continue;
        }
        hot.assign(static_cast<size_t>(np), 0);
        const int64_t wnext = wave[iu] + 1;
        for (int p = 0; p < np; ++p)
          for (int q = P.pan_start[static_cast<size_t>(P.pan_ptr[iu] + p)];
               q < P.pan_start[static_cast<size_t>(P.pan_ptr[iu] + p + 1)]; ++q) {
            const int t = P.ccol[static_cast<size_t>(P.cptr[iu] + q)];
            if (t > i && wave[static_cast<size_t>(t)] == wnext) hot[static_cast<size_t>(p)] = 1;
          }
        const int g = row_pair_group(static_cast<int>(thresholds().pair_group), np);
        int k = 0;
        for (int pp = 0; pp < np; ++pp)
          for (int q0 = pp; q0 < np; q0 += g, ++k) {
            bool h = hot[static_cast<size_t>(pp)];
            for (int qq = q0; qq < std::min(np, q0 + g); ++qq) h = h || hot[static_cast<size_t>(qq)];
            (h ? urg_of[iu] : rest_of[iu]).push_back(b0 + k);
          }
      }
    });
    build_tickets(P, nullptr, P.item_row, P.item_part);
    if (static_cast<int64_t>(P.item_row.size()) != it) throw std::logic_error("ticket order lost items");
    if (std::getenv("CE_CHECK_TICKETS") && std::getenv("CE_CHECK_TICKETS")[0] == '1') {
      // development check: every (row, part) exactly once, and inside a row the A stages in
      // dependency order (tree nodes after every node of the level below, then A2, then the
      // strips; Schur tasks after the strips)
      std::vector<int64_t> pos(static_cast<size_t>(it), -1), row_item0(static_cast<size_t>(M), 0);
      for (int64_t k = 0; k < M; ++k) row_item0[static_cast<size_t>(P.order[static_cast<size_t>(k)])] = P.item_start[static_cast<size_t>(k)];
      for (int64_t t = 0; t < it; ++t) {
        const size_t r = static_cast<size_t>(P.item_row[static_cast<size_t>(t)]);
        const int part = P.item_part[static_cast<size_t>(t)];
        const int64_t n = 1 + P.nA1[r] + P.nA3[r] + P.nB[r];
        if (part < 0 || part >= n) throw std::logic_error("ticket check: part out of range");
        int64_t& slot = pos[static_cast<size_t>(row_item0[r] + part)];
        if (slot >= 0) throw std::logic_error("ticket check: duplicate item");
        slot = t;
      }
      const int64_t kc = sweep_kcap(std::max(P.bmax, 1));
      for (int64_t i = 0; i < M; ++i) {
        const size_t r = static_cast<size_t>(i);
        const int64_t* q = pos.data() + row_item0[r];
        const int nA1 = P.nA1[r], nA3 = P.nA3[r], nB = P.nB[r];
        int64_t lo_prev = -1;  // latest ticket of the tree level below
        if (nA1 > 0) {
          const int64_t F = std::max<int64_t>(2, kc / std::max<int64_t>(P.bsz[r], 1));
          int p = 0;
          for (int64_t n = P.nleaf[r];; n = (n + F - 1) / F) {
            int64_t hi = -1;
            for (int64_t c = 0; c < n; ++c, ++p) {
              if (q[p] <= lo_prev) throw std::logic_error("ticket check: tree node before its children's level");
              hi = std::max(hi, q[p]);
            }
            lo_prev = hi;
            if (n == 1) break;
          }
          if (p != nA1) throw std::logic_error("ticket check: tree size");
        }
        if (q[nA1] <= lo_prev) throw std::logic_error("ticket check: A2 before the tree root");
        int64_t last = q[nA1];
        for (int p = 0; p < nA3; ++p) {
          if (q[nA1 + 1 + p] <= q[nA1]) throw std::logic_error("ticket check: strip before A2");
          last = std::max(last, q[nA1 + 1 + p]);
        }
        for (int p = 0; p < nB; ++p)
          if (q[nA1 + 1 + nA3 + p] <= last) throw std::logic_error("ticket check: Schur task before the strips");
      }
    }
    tp5 = now_s();
    // sq_pan: panel of j inside close(i) for each close predecessor entry (j, i), i < j
    P.sq_pan.assign(P.scol.size(), -1);
    if (lookahead)
      parallel_rows(M, [&](int64_t r0, int64_t r1) {
        for (int64_t j = r0; j < r1; ++j) {
          for (int64_t e = P.sptr[static_cast<size_t>(j)]; e < P.sdiag[static_cast<size_t>(j)]; ++e) {
            if (P.skind[static_cast<size_t>(e)] != 1) continue;
            const int i = P.scol[static_cast<size_t>(e)];
            const size_t iu = static_cast<size_t>(i);
            if (P.nB[iu] <= 1) continue;
            const int64_t q = csr_find(P.cptr, P.ccol, i, static_cast<int>(j)) - P.cptr[iu];
            const int np = static_cast<int>(P.pan_ptr[iu + 1] - P.pan_ptr[iu]) - 1;
            // panel p with pan_start[p] <= q < pan_start[p + 1]
            const int* ps = P.pan_start.data() + P.pan_ptr[iu];
            const int p = static_cast<int>(std::upper_bound(ps, ps + np, static_cast<int>(q)) - ps) - 1;
            P.sq_pan[static_cast<size_t>(e)] = p;
          }
        }
      });
  }
  P.fac_doubles = fo;
  P.basis_doubles = bo;
  P.sigma_doubles = so;
  if (std::getenv("CE_PROFILE") && std::getenv("CE_PROFILE")[0] == '1')
    std::fprintf(stderr, "[ce-profile] plan_numeric M=%lld: %.1f ms (offsets %.1f, counts %.1f, panels %.1f, entries %.1f, tickets %.1f, sq_pan %.1f)\n",
                 static_cast<long long>(M), 1e3 * (now_s() - tn0), 1e3 * (tp1 - tn0), 1e3 * (tp2 - tp1), 1e3 * (tp3 - tp2),
                 1e3 * (tp4 - tp3), 1e3 * (tp5 - tp4), 1e3 * (now_s() - tp5));
}

LevelPlan plan_level(std::vector<int> bsz, std::vector<int64_t> bptr, std::vector<int> bcol, cudaStream_t dev) {
  LevelPlan P = plan_symbolic(static_cast<int64_t>(bsz.size()), std::move(bptr), std::move(bcol), dev);
  plan_numeric(P, std::move(bsz));
  return P;
}

// Apply pull lists, task graphs and pivot inverses of one completed level (host loops +
// uploads on the context stream).  Runs on a host thread while the next level sweeps.
void build_apply_lists(LevelFactor& LF, size_t li, cudaStream_t main_stream) {
  // own non-blocking stream: pageable uploads on the main stream would wait behind the
  // next level's sweep kernel
  (void)main_stream;
  cudaStream_t s = nullptr;
  CE_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  } guard{s};
  {
    // Apply pull lists: for row j every close neighbour i with w_i > 0 (ascending), the fac
    // offset of g_{i->j} and of u_i in v; backward dependencies t > j with w_t > 0; rows of
    // v_t read by the backward pull; pivot inverses.  Wave orders of both sweeps follow the
    // same (refined) dependencies.
    const int64_t M = LF.M;
    std::vector<int64_t> in_ptr(static_cast<size_t>(M + 1), 0), in_goff, in_uoff, dep_ptr(static_cast<size_t>(M + 1), 0),
        linv_off(static_cast<size_t>(M), 0);
    std::vector<int> in_split(static_cast<size_t>(M), 0), in_src, in_w, dep_t, cl_nt(LF.ccol.size());
    int64_t lo = 0;
    for (int64_t j = 0; j < M; ++j) {
      const size_t ju = static_cast<size_t>(j);
      linv_off[ju] = lo;
      lo += static_cast<int64_t>(LF.width[ju]) * LF.width[ju];
      for (int64_t e = LF.cptr[ju]; e < LF.cptr[ju + 1]; ++e) {
        const int t = LF.ccol[static_cast<size_t>(e)];
        const size_t tu = static_cast<size_t>(t);
        cl_nt[static_cast<size_t>(e)] = t > j ? LF.bsz[tu] : LF.rank[tu];
        if (LF.width[tu] == 0) continue;
        const int64_t k = csr_find(LF.cptr, LF.ccol, t, static_cast<int>(j));
        in_src.push_back(t);
        in_goff.push_back(LF.g_off[tu] + static_cast<int64_t>(LF.rank[tu] + LF.croff[static_cast<size_t>(k)]) * LF.width[tu]);
        in_w.push_back(LF.width[tu]);
        in_uoff.push_back(LF.offsets[tu] + LF.rank[tu]);
        if (t < j) ++in_split[ju];
        if (t > j) dep_t.push_back(t);
      }
      in_ptr[ju + 1] = static_cast<int64_t>(in_src.size());
      dep_ptr[ju + 1] = static_cast<int64_t>(dep_t.size());
    }
    std::vector<int64_t> wf(static_cast<size_t>(M), 0), wb(static_cast<size_t>(M), 0);
    for (int64_t j = 0; j < M; ++j)
      for (int64_t k = in_ptr[static_cast<size_t>(j)]; k < in_ptr[static_cast<size_t>(j)] + in_split[static_cast<size_t>(j)]; ++k) {
        const int i = in_src[static_cast<size_t>(k)];
        wf[static_cast<size_t>(j)] = std::max(wf[static_cast<size_t>(j)], wf[static_cast<size_t>(i)] + 1);
      }
    for (int64_t j = M - 1; j >= 0; --j)
      for (int64_t k = dep_ptr[static_cast<size_t>(j)]; k < dep_ptr[static_cast<size_t>(j + 1)]; ++k) {
        const int t = dep_t[static_cast<size_t>(k)];
        wb[static_cast<size_t>(j)] = std::max(wb[static_cast<size_t>(j)], wb[static_cast<size_t>(t)] + 1);
      }
    std::vector<int> of(static_cast<size_t>(M)), ob(static_cast<size_t>(M));
    std::iota(of.begin(), of.end(), 0);
    std::iota(ob.begin(), ob.end(), 0);
    std::stable_sort(of.begin(), of.end(), [&](int x, int y) { return wf[static_cast<size_t>(x)] < wf[static_cast<size_t>(y)]; });
    std::stable_sort(ob.begin(), ob.end(), [&](int x, int y) {
      return wb[static_cast<size_t>(x)] < wb[static_cast<size_t>(y)] || (wb[static_cast<size_t>(x)] == wb[static_cast<size_t>(y)] && x > y);
    });
    LF.d_fwd_order.upload(of, s);
    LF.d_bwd_order.upload(ob, s);
    LF.d_in_ptr.upload(in_ptr, s);
    LF.d_in_split.upload(in_split, s);
    LF.d_in_src.upload(in_src, s);
    LF.d_in_goff.upload(in_goff, s);
    LF.d_in_w.upload(in_w, s);
    LF.d_in_uoff.upload(in_uoff, s);
    LF.d_dep_ptr.upload(dep_ptr, s);
    LF.d_dep_t.upload(dep_t, s);
    LF.d_cl_nt.upload(cl_nt, s);
    LF.d_linv_off.upload(linv_off, s);
    // split-row task graphs: slices of ~kSlice doubles of factor data per partial task
    {
      static const int64_t kSlice = std::getenv("CE_APPLY_SLICE") ? std::atoll(std::getenv("CE_APPLY_SLICE")) : 256;
      auto build = [&](bool fwd, const std::vector<int64_t>& wave, DevArray<int64_t>& d_ptr, DevArray<int64_t>& d_b,
                       DevArray<int64_t>& d_scr, DevArray<int>& d_irow, DevArray<int>& d_ipart, int64_t& n_items) {
        std::vector<int64_t> ptr(static_cast<size_t>(M + 1), 0), bnd, scr(static_cast<size_t>(M), 0);
        std::vector<int> P(static_cast<size_t>(M), 0);
        int64_t so = 0;
        for (int64_t j = 0; j < M; ++j) {
          const size_t ju = static_cast<size_t>(j);
          const int64_t w = LF.width[ju];
          scr[ju] = so;
          if (fwd) {
            const int64_t k0 = in_ptr[ju], k1 = k0 + in_split[ju];
            bnd.push_back(k0);
            int64_t acc = 0;
            for (int64_t k = k0; k < k1; ++k) {
              acc += w * in_w[static_cast<size_t>(k)];
              if (acc >= kSlice && k + 1 < k1) {
                bnd.push_back(k + 1);
                acc = 0;
              }
            }
            if (k1 > k0) bnd.push_back(k1);
          } else {
            const int64_t nseg = 1 + LF.cptr[ju + 1] - LF.cptr[ju];
            bnd.push_back(0);
            int64_t acc = 0;
            for (int64_t sg = 0; sg < nseg; ++sg) {
              const int64_t rows = sg == 0 ? LF.rank[ju] : cl_nt[static_cast<size_t>(LF.cptr[ju] + sg - 1)];
              acc += w * rows;
              if (acc >= kSlice && sg + 1 < nseg) {
                bnd.push_back(sg + 1);
                acc = 0;
              }
            }
            bnd.push_back(nseg);
          }
          ptr[ju + 1] = static_cast<int64_t>(bnd.size());
          P[ju] = static_cast<int>(ptr[ju + 1] - ptr[ju]) - 1;
          so += static_cast<int64_t>(P[ju]) * w;
        }
        // items in wave order: the wave's partial tasks, then its finalizes
        std::vector<int> ord(static_cast<size_t>(M));
        std::iota(ord.begin(), ord.end(), 0);
        std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return wave[static_cast<size_t>(x)] < wave[static_cast<size_t>(y)]; });
        std::vector<int> irow, ipart;
        for (int64_t a0 = 0; a0 < M;) {
          int64_t a1 = a0 + 1;
          const int64_t wv = wave[static_cast<size_t>(ord[static_cast<size_t>(a0)])];
          while (a1 < M && wave[static_cast<size_t>(ord[static_cast<size_t>(a1)])] == wv) ++a1;
          // rows with a single slice are one fused item (part -1)
          for (int pass = 0; pass < 2; ++pass)
            for (int64_t a = a0; a < a1; ++a) {
              const int j = ord[static_cast<size_t>(a)];
              if (LF.width[static_cast<size_t>(j)] == 0) continue;
              const bool fused = P[static_cast<size_t>(j)] == 1;
              if (pass == 0) {
                if (fused) continue;
                for (int t = 0; t < P[static_cast<size_t>(j)]; ++t) {
                  irow.push_back(j);
                  ipart.push_back(t);
                }
              } else {
                irow.push_back(j);
                ipart.push_back(fused ? -1 : P[static_cast<size_t>(j)]);
              }
            }
          a0 = a1;
        }
        d_ptr.upload(ptr, s);
        d_b.upload(bnd, s);
        d_scr.upload(scr, s);
        d_irow.upload(irow, s);
        d_ipart.upload(ipart, s);
        n_items = static_cast<int64_t>(irow.size());
        LF.scratch_doubles = std::max(LF.scratch_doubles, so);
      };
      if (std::getenv("CE_PROFILE") && std::getenv("CE_PROFILE")[0] == '1') {
        const int64_t nwf = M ? *std::max_element(wf.begin(), wf.end()) + 1 : 0;
        const int64_t nwb = M ? *std::max_element(wb.begin(), wb.end()) + 1 : 0;
        std::fprintf(stderr, "[ce-profile] level %zu apply waves: forward %lld backward %lld\n", li + 1,
                     static_cast<long long>(nwf), static_cast<long long>(nwb));
      }
      build(true, wf, LF.d_fpart_ptr, LF.d_fpart_b, LF.d_fscr_off, LF.d_fitem_row, LF.d_fitem_part, LF.n_fitems);
      build(false, wb, LF.d_bpart_ptr, LF.d_bpart_b, LF.d_bscr_off, LF.d_bitem_row, LF.d_bitem_part, LF.n_bitems);
    }
    LF.d_linv.alloc(static_cast<size_t>(std::max<int64_t>(lo, 1)));
    launch_pivot_inverse(M, LF.d_width.p, LF.d_fac.p, LF.d_chol_off.p, LF.d_linv.p, LF.d_linv_off.p, s);
    CE_CUDA(cudaGetLastError());
  }
}

namespace {

// Device copy of a plan's symbolic arrays (freed after the level).
struct DevPlan {
  DevArray<int> bsz, scol, ccol, croff, order, nA1, nA3, nB, pan_start, item_row, item_part, sbsz, sroff, target, nleaf,
      sq_pan;
  DevArray<int64_t> sptr, sslot, slot_off, cptr, chol_off, g_off, basis_off, sigma_off, item_start, offsets, cl_slot,
      fsum, rs_off, pan_ptr, sboff, sdiag, leaf_ptr, leaf_e, strip_ptr, strip_e;  // (cl_slot unused)
  DevArray<unsigned char> skind;
  DevArray<char> arena;  // backing store of every array above (views)
  // All plan arrays go through one pinned staging buffer (grow-only, per host thread): the
  // host copies them in and the DMAs run asynchronously (pageable copies would stage
  // synchronously).  The buffer is reused by the next level's upload, which happens
  // after the stream has been synchronised.
  void upload(const LevelPlan& P, cudaStream_t s) {
    struct Stage {
      char* p = nullptr;
      size_t cap = 0;
      ~Stage() {
        if (p) cudaFreeHost(p);
      }
    };
    thread_local Stage st;
    const double tu_start = now_s();
    size_t total = 0;
    auto add = [&](size_t bytes) { total += (bytes + 255) / 256 * 256; };
    auto sz = [](const auto& v) { return v.size() * sizeof(v[0]); };
    add(sz(P.order)); add(sz(P.item_row)); add(sz(P.item_part)); add(sz(P.nA1)); add(sz(P.nleaf)); add(sz(P.nA3));
    add(sz(P.nB)); add(sz(P.pan_start)); add(sz(P.fsum)); add(sz(P.rs_off)); add(sz(P.pan_ptr)); add(sz(P.bsz));
    add(sz(P.scol)); add(sz(P.ccol)); add(sz(P.croff)); add(sz(P.sptr)); add(sz(P.sslot)); add(sz(P.slot_off));
    add(sz(P.cptr)); add(sz(P.chol_off)); add(sz(P.g_off)); add(sz(P.basis_off)); add(sz(P.sigma_off));
    add(sz(P.item_start)); add(sz(P.offsets)); add(sz(P.skind)); add(sz(P.sboff)); add(sz(P.sbsz)); add(sz(P.sroff));
    add(sz(P.sdiag)); add(sz(P.target)); add(sz(P.leaf_ptr)); add(sz(P.leaf_e)); add(sz(P.strip_ptr)); add(sz(P.strip_e));
    add(sz(P.sq_pan));
    if (total > st.cap) {
      if (st.p) cudaFreeHost(st.p);
      st.p = nullptr;
      st.cap = total + total / 4;
      CE_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&st.p), st.cap, cudaHostAllocDefault));
    }
    const double tu0 = now_s();
    // one device arena for all plan arrays, laid out like the staging buffer: one allocation
    // (every level asks for the high-water size, so the cached block of the previous level or
    // factorization always fits; 36 separate arrays used to miss the allocator cache whenever
    // a level's sizes moved by more than its rounding, a cudaMalloc of up to 100 ms between
    // two sweeps) and one DMA
    static std::atomic<size_t> arena_hwm{0};
    size_t want = arena_hwm.load();
    while (want < total && !arena_hwm.compare_exchange_weak(want, total)) {
    }
    want = std::max(want, total);
    if (arena.n < total) arena.alloc(want);
    size_t off = 0;
    // the staging copies run in parallel on the host threads (one 200 MB level plan was a
    // 30-60 ms single-thread memcpy on the critical path between two sweeps), then every
    // array's DMA is queued on the stream
    struct Job {
      void* dst;
      const void* src;
      size_t bytes, at;
    };
    std::vector<Job> jobs;
    std::vector<size_t> owned;  // jobs whose array outlives the plan (moved into the level factor)
    auto put = [&](auto& d, const auto& h, bool keep = false) {
      const size_t bytes = h.size() * sizeof(h[0]);
      if (keep) {
        d.alloc(h.size());
        if (bytes) owned.push_back(jobs.size());
      } else {
        d.set_view(arena.p + off, h.size());
      }
      if (bytes) jobs.push_back({d.p, h.data(), bytes, off});
      off += (bytes + 255) / 256 * 256;
    };
    put(order, P.order); put(item_row, P.item_row); put(item_part, P.item_part); put(nA1, P.nA1); put(nleaf, P.nleaf);
    put(nA3, P.nA3); put(nB, P.nB); put(pan_start, P.pan_start); put(fsum, P.fsum); put(rs_off, P.rs_off);
    put(pan_ptr, P.pan_ptr); put(bsz, P.bsz, true); put(scol, P.scol); put(ccol, P.ccol, true); put(croff, P.croff, true);
    put(sptr, P.sptr); put(sslot, P.sslot); put(slot_off, P.slot_off); put(cptr, P.cptr, true); put(chol_off, P.chol_off, true);
    put(g_off, P.g_off, true); put(basis_off, P.basis_off, true); put(sigma_off, P.sigma_off, true); put(item_start, P.item_start);
    put(offsets, P.offsets, true); put(skind, P.skind); put(sboff, P.sboff); put(sbsz, P.sbsz); put(sroff, P.sroff);
    put(sdiag, P.sdiag); put(target, P.target); put(leaf_ptr, P.leaf_ptr); put(leaf_e, P.leaf_e);
    put(strip_ptr, P.strip_ptr); put(strip_e, P.strip_e); put(sq_pan, P.sq_pan);
    const double tu1 = now_s();
    constexpr size_t kChunk = size_t{1} << 20;
    std::vector<std::pair<size_t, size_t>> pieces;  // (job, first byte) of 1 MB pieces
    for (size_t j = 0; j < jobs.size(); ++j)
      for (size_t b = 0; b < jobs[j].bytes; b += kChunk) pieces.emplace_back(j, b);
    char* const stage = st.p;  // `st` is thread_local: the worker threads must not name it
    parallel_rows(static_cast<int64_t>(pieces.size()), [&](int64_t r0, int64_t r1) {
      for (int64_t k = r0; k < r1; ++k) {
        const Job& jb = jobs[pieces[static_cast<size_t>(k)].first];
        const size_t b = pieces[static_cast<size_t>(k)].second, n = std::min(kChunk, jb.bytes - b);
        std::memcpy(stage + jb.at + b, static_cast<const char*>(jb.src) + b, n);
      }
    });
    const double tu2 = now_s();
    if (total) CE_CUDA(cudaMemcpyAsync(arena.p, stage, total, cudaMemcpyHostToDevice, s));
    for (size_t j : owned) CE_CUDA(cudaMemcpyAsync(jobs[j].dst, stage + jobs[j].at, jobs[j].bytes, cudaMemcpyHostToDevice, s));
    if (std::getenv("CE_PROFILE") && std::getenv("CE_PROFILE")[0] == '1')
      std::fprintf(stderr, "[ce-profile] plan upload %.1f MB: stage buffer %.1f ms, device arrays %.1f ms, staging copy %.1f ms, enqueue %.1f ms\n",
                   total / 1e6, 1e3 * (tu0 - tu_start), 1e3 * (tu1 - tu0), 1e3 * (tu2 - tu1), 1e3 * (now_s() - tu2));
  }
};

std::vector<std::vector<int64_t>> pair_groups(int64_t blocks, int64_t join) {
  std::vector<std::vector<int64_t>> g;
  for (int64_t b = 0; b < blocks; b += join) {
    std::vector<int64_t> m;
    for (int64_t k = b; k < std::min(b + join, blocks); ++k) m.push_back(k);
    g.push_back(std::move(m));
  }
  return g;
}

std::vector<std::vector<std::vector<int64_t>>> plan_levels_from(const ce_plan_host* plan) {
  std::vector<std::vector<std::vector<int64_t>>> levels;
  if (!plan) return levels;
  int64_t at = 0;
  for (int64_t l = 0; l < plan->n_levels; ++l) {
    const int64_t nb = plan->level_blocks[l];
    int64_t ng = 0;
    for (int64_t b = 0; b < nb; ++b) ng = std::max(ng, plan->assign[at + b] + 1);
    std::vector<std::vector<int64_t>> groups(static_cast<size_t>(ng));
    for (int64_t b = 0; b < nb; ++b) {
      const int64_t g = plan->assign[at + b];
      if (g < 0 || g >= ng) throw std::invalid_argument("plan: negative group id");
      groups[static_cast<size_t>(g)].push_back(b);
    }
    for (const auto& g : groups)
      if (g.empty()) throw std::invalid_argument("empty group in coarsening level");
    levels.push_back(std::move(groups));
    at += nb;
  }
  return levels;
}

// Algorithmic bytes / flops of one row (SURVEY.md §8d contract).
void row_counts(double b, double c, double f, double r, double w, double p, double P, bool U, bool svd, double& bytes,
                double& flops) {
  double words = 0.0, fl = 0.0;
  if (f > 0) words += b * f;
  if (svd) fl += 2 * b * b * f + 12 * b * b * b;
  if (U) {
    words += 2 * (b * b + b * c + b * f) + 2 * b * p + b * b;
    fl += 4 * b * b * b + 2 * b * b * (c + f) + 2 * b * p;
  }
  if (w > 0) {
    words += b * c + 2 * P + (w * (w + 1) / 2 + r * w + c * w);
    fl += w * w * w / 3 + w * w * (r + c) + 2 * r * r * w + 2 * r * w * c + 2 * w * P;
  }
  bytes += 8 * words;
  flops += fl;
}

}  // namespace

// ---------------------------------------------------------------- sharding
// A level of a CE_PLAN_SHARDED plan starts with the box-interior rows (row i interior: every
// row of sq(i) carries i's box label), box by box, then every other ("interface") row.  An
// interior row's reads and writes stay inside its box, so each rank sweeps the
// interior rows of the boxes it owns (phase 1) with no communication; then
//   E1  the owners broadcast the per-row integers of their phase-1 rows and every within-box
//       block the interface rows will touch (their squared-pattern rows and Schur pairs);
//   phase 3  every rank sweeps all interface rows (replicated, bit-identical inputs);
//   E2  owners broadcast their phase-1 rows' factor slices (chol, coupling, g_t), bases, sigma;
//   E3  owners broadcast the retained corners of the other within-box blocks phase 1 wrote,
// so every rank ends the level with the whole level factor and a consistent store: the next
// level, the tail and the apply run on complete data, and the factor is bit-identical to the
// single-GPU factorization of the same plan (tests/test_gpu_shard.py).
namespace {

struct Seg {
  int64_t off;
  int rows, cols, ld;
  int owner;
};

void shard_sync_bcast(const ShardSpec& sh, void* p, int64_t bytes, int root) {
  if (bytes <= 0) return;
  if (sh.bcast(sh.user, p, bytes, root) != 0) throw std::runtime_error("sharded factorization: broadcast failed");
}

// Owners pack their segments of `base` into a buffer, broadcast them in rank order, the
// other ranks unpack.  Every rank passes the same segment list.
void shard_exchange(const ShardSpec& sh, cudaStream_t s, double* base, std::vector<Seg> segs, ShardStats& st) {
  if (segs.empty()) return;
  const double t0 = now_s();
  std::stable_sort(segs.begin(), segs.end(), [](const Seg& a, const Seg& b) { return a.owner < b.owner; });
  const size_t n = segs.size();
  std::vector<int64_t> off(n), boff(n), lo(static_cast<size_t>(sh.n_ranks) + 1, 0);
  std::vector<int> rows(n), cols(n), ld(n);
  std::vector<size_t> first(static_cast<size_t>(sh.n_ranks) + 1, n);
  int64_t at = 0;
  for (size_t k = 0; k < n; ++k) {
    off[k] = segs[k].off;
    rows[k] = segs[k].rows;
    cols[k] = segs[k].cols;
    ld[k] = segs[k].ld;
    boff[k] = at;
    at += static_cast<int64_t>(segs[k].rows) * segs[k].cols;
  }
  for (int r = sh.n_ranks; r >= 0; --r) {
    size_t k = 0;
    while (k < n && segs[k].owner < r) ++k;
    first[static_cast<size_t>(r)] = k;
    lo[static_cast<size_t>(r)] = k < n ? boff[k] : at;
  }
  DevArray<double> buf(static_cast<size_t>(std::max<int64_t>(at, 1)));
  DevArray<int64_t> d_off, d_boff;
  DevArray<int> d_rows, d_cols, d_ld;
  d_off.upload(off, s);
  d_boff.upload(boff, s);
  d_rows.upload(rows, s);
  d_cols.upload(cols, s);
  d_ld.upload(ld, s);
  const size_t s0 = first[static_cast<size_t>(sh.rank)], s1 = first[static_cast<size_t>(sh.rank) + 1];
  launch_segments(base, buf.p, d_off.p + s0, d_rows.p + s0, d_cols.p + s0, d_ld.p + s0, d_boff.p + s0,
                  static_cast<int64_t>(s1 - s0), true, s);
  CE_CUDA(cudaStreamSynchronize(s));
  for (int r = 0; r < sh.n_ranks; ++r)
    shard_sync_bcast(sh, buf.p + lo[static_cast<size_t>(r)],
                     (lo[static_cast<size_t>(r) + 1] - lo[static_cast<size_t>(r)]) * static_cast<int64_t>(sizeof(double)), r);
  launch_segments(base, buf.p, d_off.p, d_rows.p, d_cols.p, d_ld.p, d_boff.p, static_cast<int64_t>(s0), false, s);
  launch_segments(base, buf.p, d_off.p + s1, d_rows.p + s1, d_cols.p + s1, d_ld.p + s1, d_boff.p + s1,
                  static_cast<int64_t>(n - s1), false, s);
  CE_CUDA(cudaStreamSynchronize(s));
  st.exchange_bytes += static_cast<double>(at) * sizeof(double);
  st.exchange_seconds += now_s() - t0;
}

// Phase split of one level.
struct ShardLevel {
  int64_t prefix = 0;                     // rows [0, prefix): interior (phase 1)
  std::vector<char> own1, phase3;         // masks: this rank's phase-1 rows, interface rows
  std::vector<int> foreign1;              // phase-1 rows of the other ranks
  std::vector<std::vector<int>> by_owner; // phase-1 rows per owner rank
};

ShardLevel shard_level(const ShardSpec& sh, const LevelPlan& P, const std::vector<int64_t>& label) {
  ShardLevel L;
  const int64_t M = P.M;
  L.prefix = M;
  for (int64_t i = 0; i < M && L.prefix == M; ++i) {
    bool interior = label[static_cast<size_t>(i)] >= 0;
    for (int64_t e = P.sptr[static_cast<size_t>(i)]; e < P.sptr[static_cast<size_t>(i + 1)] && interior; ++e)
      interior = label[static_cast<size_t>(P.scol[static_cast<size_t>(e)])] == label[static_cast<size_t>(i)];
    if (!interior) L.prefix = i;
  }
  L.own1.assign(static_cast<size_t>(M), 0);
  L.phase3.assign(static_cast<size_t>(M), 0);
  L.by_owner.assign(static_cast<size_t>(sh.n_ranks), {});
  for (int64_t i = 0; i < M; ++i) {
    if (i >= L.prefix) {
      L.phase3[static_cast<size_t>(i)] = 1;
      continue;
    }
    const int o = sh.owner(label[static_cast<size_t>(i)]);
    L.by_owner[static_cast<size_t>(o)].push_back(static_cast<int>(i));
    if (o == sh.rank) L.own1[static_cast<size_t>(i)] = 1;
    else L.foreign1.push_back(static_cast<int>(i));
  }
  return L;
}

// Per-row integers of the phase-1 rows (rank, width, has_basis, fcols, nsig), owners first.
void shard_exchange_ints(const ShardSpec& sh, cudaStream_t s, const ShardLevel& L, LevelFactor& LF, ShardStats& st) {
  const double t0 = now_s();
  std::vector<int> rows;
  std::vector<int64_t> lo(static_cast<size_t>(sh.n_ranks) + 1, 0);
  for (int r = 0; r < sh.n_ranks; ++r) {
    lo[static_cast<size_t>(r)] = static_cast<int64_t>(rows.size());
    rows.insert(rows.end(), L.by_owner[static_cast<size_t>(r)].begin(), L.by_owner[static_cast<size_t>(r)].end());
  }
  lo[static_cast<size_t>(sh.n_ranks)] = static_cast<int64_t>(rows.size());
  if (rows.empty()) return;
  DevArray<int> d_rows;
  d_rows.upload(rows, s);
  DevArray<double> buf(5 * rows.size());
  const int64_t a0 = lo[static_cast<size_t>(sh.rank)], a1 = lo[static_cast<size_t>(sh.rank) + 1];
  launch_row_ints(d_rows.p + a0, a1 - a0, LF.d_rank.p, LF.d_width.p, LF.d_has_basis.p, LF.d_fcols.p, LF.d_nsig.p,
                  buf.p + 5 * a0, true, s);
  CE_CUDA(cudaStreamSynchronize(s));
  for (int r = 0; r < sh.n_ranks; ++r)
    shard_sync_bcast(sh, buf.p + 5 * lo[static_cast<size_t>(r)],
                     5 * (lo[static_cast<size_t>(r) + 1] - lo[static_cast<size_t>(r)]) * static_cast<int64_t>(sizeof(double)), r);
  launch_row_ints(d_rows.p, a0, LF.d_rank.p, LF.d_width.p, LF.d_has_basis.p, LF.d_fcols.p, LF.d_nsig.p, buf.p, false, s);
  launch_row_ints(d_rows.p + a1, static_cast<int64_t>(rows.size()) - a1, LF.d_rank.p, LF.d_width.p, LF.d_has_basis.p,
                  LF.d_fcols.p, LF.d_nsig.p, buf.p + 5 * a1, false, s);
  CE_CUDA(cudaStreamSynchronize(s));
  st.exchange_bytes += 40.0 * static_cast<double>(rows.size());
  st.exchange_seconds += now_s() - t0;
}

// Every rank's sweep status after a phase: a breakdown / error anywhere stops every rank.
void shard_check_status(const ShardSpec& sh, cudaStream_t s, int* d_err) {
  DevArray<double> st(4 * static_cast<size_t>(sh.n_ranks));
  st.zero(s);
  std::vector<int> h(4, 0);
  CE_CUDA(cudaMemcpyAsync(h.data(), d_err, 4 * sizeof(int), cudaMemcpyDeviceToHost, s));
  CE_CUDA(cudaStreamSynchronize(s));
  const double mine[4] = {static_cast<double>(h[0]), static_cast<double>(h[1]), static_cast<double>(h[2]),
                          static_cast<double>(h[3])};
  CE_CUDA(cudaMemcpy(st.p + 4 * sh.rank, mine, sizeof mine, cudaMemcpyHostToDevice));
  for (int r = 0; r < sh.n_ranks; ++r) shard_sync_bcast(sh, st.p + 4 * r, 4 * sizeof(double), r);
  std::vector<double> all;
  st.download(all, s);
  CE_CUDA(cudaStreamSynchronize(s));
  for (int r = 0; r < sh.n_ranks; ++r)
    if (all[static_cast<size_t>(4 * r)] != 0.0 && r != sh.rank) {
      // adopt the first failing rank's status so every rank raises the same error
      const int v[4] = {static_cast<int>(all[static_cast<size_t>(4 * r)]), static_cast<int>(all[static_cast<size_t>(4 * r + 1)]),
                        static_cast<int>(all[static_cast<size_t>(4 * r + 2)]), static_cast<int>(all[static_cast<size_t>(4 * r + 3)])};
      if (h[0] == 0) CE_CUDA(cudaMemcpy(d_err, v, sizeof v, cudaMemcpyHostToDevice));
      break;
    }
}

// Stored slot of (s, t) in the squared pattern (both triangles map to the lower slot).
int64_t sq_slot_of(const LevelPlan& P, int64_t s, int64_t t) {
  const int64_t e = csr_find(P.sptr, P.scol, s, static_cast<int>(t));
  return e < 0 ? -1 : P.sslot[static_cast<size_t>(e)];
}

}  // namespace

int64_t shard_symbolic_summary(const Problem& p, const ShardSpec& spec, int64_t max_levels, int64_t* out) {
  std::vector<int64_t> labels = spec.box_l1;
  std::vector<int64_t> bptr = p.row_ptr;
  std::vector<int> bcol(p.col_idx.begin(), p.col_idx.end());
  int64_t M = p.m, at = 0, lv = 0;
  const int64_t stride = 2 + spec.n_ranks;
  for (; lv < max_levels && lv < static_cast<int64_t>(p.plan_level_blocks.size()) && M > 1; ++lv) {
    LevelPlan P = plan_symbolic(M, bptr, bcol);
    ShardLevel L = shard_level(spec, P, labels);
    out[lv * stride] = M;
    out[lv * stride + 1] = L.prefix;
    for (int r = 0; r < spec.n_ranks; ++r)
      out[lv * stride + 2 + r] = static_cast<int64_t>(L.by_owner[static_cast<size_t>(r)].size());
    // next level: coarsen(sq) over the plan's groups, labels by common membership
    int64_t ng = 0;
    for (int64_t b = 0; b < M; ++b) ng = std::max(ng, p.plan_assign[static_cast<size_t>(at + b)] + 1);
    std::vector<int64_t> gof(static_cast<size_t>(M)), nl(static_cast<size_t>(ng), -2);
    for (int64_t b = 0; b < M; ++b) {
      const int64_t g = p.plan_assign[static_cast<size_t>(at + b)];
      gof[static_cast<size_t>(b)] = g;
      int64_t& v = nl[static_cast<size_t>(g)];
      v = v == -2 ? labels[static_cast<size_t>(b)] : (v == labels[static_cast<size_t>(b)] ? v : -1);
    }
    at += M;
    std::vector<std::vector<int>> rows(static_cast<size_t>(ng));
    for (int64_t i = 0; i < M; ++i)
      for (int64_t e = P.sptr[static_cast<size_t>(i)]; e < P.sptr[static_cast<size_t>(i + 1)]; ++e)
        rows[static_cast<size_t>(gof[static_cast<size_t>(i)])].push_back(static_cast<int>(gof[static_cast<size_t>(P.scol[static_cast<size_t>(e)])]));
    bptr.assign(static_cast<size_t>(ng + 1), 0);
    bcol.clear();
    for (int64_t g = 0; g < ng; ++g) {
      auto& r = rows[static_cast<size_t>(g)];
      std::sort(r.begin(), r.end());
      r.erase(std::unique(r.begin(), r.end()), r.end());
      bcol.insert(bcol.end(), r.begin(), r.end());
      bptr[static_cast<size_t>(g + 1)] = static_cast<int64_t>(bcol.size());
    }
    labels = std::move(nl);
    M = ng;
  }
  return lv;
}

// CEFactorization::validate (proj/src/factorization.cpp:272-334), run at the end of every
// ce_factorize like the reference's (:459): structure on the host from the driver's arrays,
// basis orthogonality (<= 1e-12) and lower-triangular pivots on the device (validate.cu), one
// 24-byte read.  Violations throw std::logic_error (exit code 1, as in the reference).
void validate_factor(Factor& F, cudaStream_t s) {
  const double t0 = now_s();
  int64_t expect = F.n, accounted = 0;
  for (size_t l = 0; l < F.levels.size(); ++l) {
    const LevelFactor& L = F.levels[l];
    if (L.dim != expect) throw std::logic_error("level dimensions do not telescope");
    if (L.n_elim + L.n_kept != L.dim) throw std::logic_error("eliminated plus kept must cover the level");
    for (int64_t b = 0; b < L.M; ++b) {
      if (L.width[static_cast<size_t>(b)] + L.rank[static_cast<size_t>(b)] != L.bsz[static_cast<size_t>(b)])
        throw std::logic_error("width plus retained must equal the block size");
      if (L.width[static_cast<size_t>(b)] == 0) continue;
      int64_t prev = -1;
      for (int64_t e = L.cptr[static_cast<size_t>(b)]; e < L.cptr[static_cast<size_t>(b + 1)]; ++e) {
        const int64_t t = L.ccol[static_cast<size_t>(e)];
        if (t <= prev || t == b) throw std::logic_error("neighbor list must be ascending and off-diagonal");
        prev = t;
      }
    }
    accounted += L.n_elim;
    expect = L.n_kept;
  }
  if (!F.levels.empty() && expect != F.tail_dim) throw std::logic_error("tail dimension does not match the last level");
  if (accounted + F.tail_dim != F.n) throw std::logic_error("eliminated plus tail must cover the matrix");
  DevArray<unsigned long long> d_out(3 * std::max<size_t>(F.levels.size(), 1));
  std::vector<unsigned long long> init(d_out.n);
  for (size_t k = 0; k < init.size(); k += 3) {
    init[k] = 0;
    init[k + 1] = 0;
    init[k + 2] = ~0ull;
  }
  CE_CUDA(cudaMemcpyAsync(d_out.p, init.data(), init.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice, s));
  for (size_t l = 0; l < F.levels.size(); ++l) {
    const LevelFactor& L = F.levels[l];
    launch_validate_level(L.M, L.d_bsz.p, L.d_has_basis.p, L.d_basis.p, L.d_basis_off.p, L.d_width.p, L.d_fac.p,
                          L.d_chol_off.p, 1e-12, d_out.p + 3 * l, s);
  }
  CE_CUDA(cudaGetLastError());
  std::vector<unsigned long long> res(d_out.n);
  CE_CUDA(cudaMemcpyAsync(res.data(), d_out.p, res.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  CE_CUDA(cudaStreamSynchronize(s));
  for (size_t l = 0; l < F.levels.size(); ++l) {
    double err = 0.0;
    std::memcpy(&err, &res[3 * l], sizeof err);
    F.max_orth_error = std::max(F.max_orth_error, err);
    if (res[3 * l + 2] != ~0ull) {
      std::ostringstream os;
      if (res[3 * l + 1]) os << "pivot factor must be lower triangular (level " << l + 1 << ", block " << res[3 * l + 2] << ")";
      else os << "basis orthogonality violated at level " << l + 1 << ", block " << res[3 * l + 2] << ": " << err;
      throw std::logic_error(os.str());
    }
  }
  F.validate_seconds = now_s() - t0;
}

Factor* factorize(Context* ctx, const Matrix* A, const ce_plan_host* plan_host, const ce_strategy* st,
                  const ce_factor_opts* op, int64_t* shift_total, const ShardSpec* shard) {
  const double t_start = now_s();
  if (shard && (shard->n_ranks < 1 || shard->rank < 0 || shard->rank >= shard->n_ranks || shard->n_boxes < 1 ||
                !shard->bcast || static_cast<int64_t>(shard->box_l1.size()) != A->m))
    throw std::invalid_argument("sharded factorization: invalid shard spec (ranks, boxes, labels, broadcast)");
  std::vector<int64_t> labels;  // box label of every block of the current level (-1: mixed)
  if (shard) {
    labels = shard->box_l1;
    for (int64_t v : labels)
      if (v < -1 || v >= shard->n_boxes) throw std::invalid_argument("sharded factorization: box label out of range");
  }
  cudaStream_t s = ctx->stream;
  const int64_t dense_threshold = op ? op->dense_threshold : 2048;
  const int64_t max_levels = op ? op->max_levels : 64;
  std::vector<std::vector<int64_t>> forced;
  if (op && op->n_forced_levels > 0) {
    int64_t at = 0;
    for (int64_t l = 0; l < op->n_forced_levels; ++l) {
      forced.emplace_back(op->forced + at, op->forced + at + op->forced_counts[l]);
      at += op->forced_counts[l];
    }
  }
  const auto plan_levels = plan_levels_from(plan_host);
  const int64_t join = plan_host ? plan_host->join : 2;
  if (join < 1) throw std::invalid_argument("join must be positive");
  if (!plan_levels.empty() && static_cast<int64_t>(plan_levels[0].size()) > 0) {
    int64_t nb = 0;
    for (const auto& g : plan_levels[0]) nb += static_cast<int64_t>(g.size());
    if (nb != A->m) throw std::invalid_argument("plan partition does not match the matrix");
  }

  auto F = std::make_unique<Factor>();
  F->levels.reserve(static_cast<size_t>(std::max<int64_t>(max_levels, 1)) + 1);  // stable addresses for apply_jobs
  std::vector<std::future<void>> apply_jobs;
  F->ctx = ctx;
  F->n = A->n;

  // level-1 plan from A's block structure
  std::vector<int> bsz(static_cast<size_t>(A->m));
  for (int64_t i = 0; i < A->m; ++i) bsz[static_cast<size_t>(i)] = static_cast<int>(A->offsets[static_cast<size_t>(i + 1)] - A->offsets[static_cast<size_t>(i)]);
  std::vector<int> bcol(A->col_idx.begin(), A->col_idx.end());
  LevelPlan cur = plan_level(bsz, A->row_ptr, bcol, s);  // device idle: squares on the GPU
  DevPlan dcur, dprev;
  dcur.upload(cur, s);
  DevArray<double> store(static_cast<size_t>(cur.store_doubles));
  store.zero(s);
  DevArray<double> nstore;  // next level's store; the two buffers are swapped and reused (grow-only)
  Events ev_all;
  CE_CUDA(cudaEventRecord(ev_all.a, s));
  launch_init_store_from_matrix(cur.M, dcur.bsz.p, A->d_row_ptr.p, A->d_col_idx.p, A->d_val_ptr.p, A->d_values.p,
                                dcur.sptr.p, dcur.scol.p, dcur.sslot.p, dcur.slot_off.p, store.p, s);
  CE_CUDA(cudaGetLastError());

  std::vector<int64_t> alive_map(static_cast<size_t>(A->m));
  std::iota(alive_map.begin(), alive_map.end(), int64_t{0});
  DevArray<int> d_err(4), d_shifts(1);
  DevArray<unsigned long long> d_ticket(1);
  int64_t shifts = 0;
  int64_t elim_total = 0;

  const double t_loop0 = now_s();
  double t_loop1 = t_loop0;
  while (cur.dim > dense_threshold && static_cast<int64_t>(F->levels.size()) < max_levels) {
    const size_t li = F->levels.size();
    const double h_t0 = now_s();
    const auto plan_groups = li < plan_levels.size() ? plan_levels[li] : pair_groups(static_cast<int64_t>(alive_map.size()), join);
    std::vector<std::vector<int64_t>> cur_groups;
    std::vector<int64_t> slot_of_group(plan_groups.size(), -1);
    for (size_t g = 0; g < plan_groups.size(); ++g) {
      std::vector<int64_t> mem;
      for (int64_t b : plan_groups[g]) {
        if (b < 0 || b >= static_cast<int64_t>(alive_map.size())) throw std::invalid_argument("groups must partition the level's blocks");
        if (alive_map[static_cast<size_t>(b)] >= 0) mem.push_back(alive_map[static_cast<size_t>(b)]);
      }
      if (!mem.empty()) {
        slot_of_group[g] = static_cast<int64_t>(cur_groups.size());
        cur_groups.push_back(std::move(mem));
      }
    }
    {
      std::vector<char> seen(static_cast<size_t>(cur.M), 0);
      int64_t cov = 0;
      for (const auto& g : cur_groups)
        for (int64_t b : g) {
          if (b < 0 || b >= cur.M || seen[static_cast<size_t>(b)]) throw std::invalid_argument("groups must partition the block index range");
          seen[static_cast<size_t>(b)] = 1;
          ++cov;
        }
      if (cov != cur.M) throw std::invalid_argument("groups must cover every block");
    }

    LevelFactor LF;
    std::function<void()> shard_post;  // sharded level: exchanges after the pending rotation
    LF.M = cur.M;
    LF.dim = cur.dim;
    LF.pattern_blocks = cur.lower_blocks;
    LF.max_far = cur.fmax;
    LF.max_close = cur.cmax;
    LF.n_waves = cur.n_waves;
    LF.n_items = cur.n_items;
    LF.d_rank.alloc(static_cast<size_t>(cur.M));
    LF.d_width.alloc(static_cast<size_t>(cur.M));
    LF.d_has_basis.alloc(static_cast<size_t>(cur.M));
    LF.d_fcols.alloc(static_cast<size_t>(cur.M));
    LF.d_nsig.alloc(static_cast<size_t>(cur.M));
    LF.d_basis.alloc(static_cast<size_t>(cur.basis_doubles));
    LF.d_sigma.alloc(static_cast<size_t>(std::max<int64_t>(cur.sigma_doubles, 1)));
    LF.d_fac.alloc(static_cast<size_t>(cur.fac_doubles));
    DevArray<int> d_done(static_cast<size_t>(cur.M));
    d_done.zero(s);
    d_err.zero(s);
    d_shifts.zero(s);
    d_ticket.zero(s);
    DevArray<int> d_forced;
    if (li < forced.size() && !forced[li].empty()) {
      std::vector<int> fr(static_cast<size_t>(cur.M), -1);
      for (size_t k = 0; k < forced[li].size() && k < fr.size(); ++k) fr[k] = static_cast<int>(forced[li][k]);
      d_forced.upload(fr, s);
    }

    // speculative symbolic plan of the next level on a host thread while this level sweeps.  It
    // assumes every group keeps a nonzero rank except the groups that are dead by structure:
    // with an eps strategy a row whose far blocks are all absent or still structurally zero
    // (kind 3) gets rank 0 (compression.cpp:20-36: an empty / zero far concat retains nothing), so a
    // group of such rows vanishes from the next level.  The assumed alive set is checked after
    // the sweep and the plan recomputed if it was wrong.
    const bool predict_dead = !st || st->mode != 1;
    std::future<std::pair<LevelPlan, std::vector<char>>> spec =
        std::async(std::launch::async, [&cur, &cur_groups, predict_dead]() {
          const int64_t ng = static_cast<int64_t>(cur_groups.size());
          std::vector<int64_t> gof(static_cast<size_t>(cur.M), 0), amap(static_cast<size_t>(ng), -1);
          std::vector<char> alive(static_cast<size_t>(ng), 1);
          int64_t nA = 0;
          for (int64_t g = 0; g < ng; ++g) {
            bool any = !predict_dead;
            for (int64_t b : cur_groups[static_cast<size_t>(g)]) {
              gof[static_cast<size_t>(b)] = g;
              for (int64_t e = cur.sptr[static_cast<size_t>(b)]; !any && e < cur.sptr[static_cast<size_t>(b + 1)]; ++e)
                any = cur.skind[static_cast<size_t>(e)] == 2;
            }
            alive[static_cast<size_t>(g)] = any ? 1 : 0;
            if (any) amap[static_cast<size_t>(g)] = nA++;
          }
          std::vector<int64_t> nptr(static_cast<size_t>(nA + 1), 0), mark(static_cast<size_t>(ng), -1);
          std::vector<int> ncol, row;
          for (int64_t g = 0; g < ng; ++g) {
            if (!alive[static_cast<size_t>(g)]) continue;
            row.clear();
            for (int64_t b : cur_groups[static_cast<size_t>(g)])
              for (int64_t e = cur.sptr[static_cast<size_t>(b)]; e < cur.sptr[static_cast<size_t>(b + 1)]; ++e) {
                const int64_t h = gof[static_cast<size_t>(cur.scol[static_cast<size_t>(e)])];
                if (!alive[static_cast<size_t>(h)] || mark[static_cast<size_t>(h)] == g) continue;
                mark[static_cast<size_t>(h)] = g;
                row.push_back(static_cast<int>(amap[static_cast<size_t>(h)]));
              }
            std::sort(row.begin(), row.end());
            ncol.insert(ncol.end(), row.begin(), row.end());
            nptr[static_cast<size_t>(amap[static_cast<size_t>(g)] + 1)] = static_cast<int64_t>(ncol.size());
          }
          return std::make_pair(plan_symbolic(nA, std::move(nptr), std::move(ncol)), std::move(alive));
        });

    SweepArgs a{};
    a.dbg = std::getenv("CE_DBG") ? std::atoi(std::getenv("CE_DBG")) : 0;
    a.M = cur.M;
    a.level = static_cast<int>(li) + 1;
    a.bsz = dcur.bsz.p;
    a.sq_ptr = dcur.sptr.p;
    a.sq_col = dcur.scol.p;
    a.sq_slot = dcur.sslot.p;
    a.sq_kind = dcur.skind.p;
    a.slot_off = dcur.slot_off.p;
    // Schur panels look up stored (t, s) blocks; with M <= 8192 a dense triangular table
    // (<= 268 MB) replaces the per-pair binary search of the squared pattern
    DevArray<int64_t> d_tri;
    if (cur.M <= 8192 && !thresholds().no_tri_table) {
      d_tri.alloc(static_cast<size_t>(cur.M) * static_cast<size_t>(cur.M + 1) / 2);
      launch_tri_table(cur.M, dcur.sptr.p, dcur.scol.p, dcur.sslot.p, dcur.slot_off.p, d_tri.p, s);
      a.tri_off = d_tri.p;
    }
    a.store = store.p;
    a.cl_ptr = dcur.cptr.p;
    a.cl_col = dcur.ccol.p;
    a.cl_roff = dcur.croff.p;
    a.cl_slot = dcur.cl_slot.p;
    a.rank = LF.d_rank.p;
    a.width = LF.d_width.p;
    a.has_basis = LF.d_has_basis.p;
    a.fcols = LF.d_fcols.p;
    a.nsig = LF.d_nsig.p;
    a.basis = LF.d_basis.p;
    a.basis_off = dcur.basis_off.p;
    a.sigma = LF.d_sigma.p;
    a.sigma_off = dcur.sigma_off.p;
    a.fac = LF.d_fac.p;
    a.chol_off = dcur.chol_off.p;
    a.g_off = dcur.g_off.p;
    a.item_start = dcur.item_start.p;
    a.order = dcur.order.p;
    a.item_row = dcur.item_row.p;
    a.item_part = dcur.item_part.p;
    a.nA1 = dcur.nA1.p;
    a.nleaf = dcur.nleaf.p;
    a.nA3 = dcur.nA3.p;
    a.nB = dcur.nB.p;
    a.fsum = dcur.fsum.p;
    a.rs_off = dcur.rs_off.p;
    a.pan_ptr = dcur.pan_ptr.p;
    a.pan_start = dcur.pan_start.p;
    a.sq_boff = dcur.sboff.p;
    a.sq_bsz = dcur.sbsz.p;
    a.sq_roff = dcur.sroff.p;
    a.sq_diag = dcur.sdiag.p;
    a.target = dcur.target.p;
    a.leaf_ptr = dcur.leaf_ptr.p;
    a.leaf_e = dcur.leaf_e.p;
    a.strip_ptr = dcur.strip_ptr.p;
    a.strip_e = dcur.strip_e.p;
    DevArray<double> d_rscratch(static_cast<size_t>(std::max<int64_t>(cur.rscratch_doubles, 1)));
    DevArray<int> d_nz(static_cast<size_t>(cur.M));
    d_nz.zero(s);
    DevArray<int> d_pdone(static_cast<size_t>(std::max<int64_t>(cur.pan_ptr[static_cast<size_t>(cur.M)], 1)));
    d_pdone.zero(s);
    DevArray<int> d_bready(static_cast<size_t>(cur.M));
    d_bready.zero(s);
    a.sq_pan = dcur.sq_pan.p;
    a.pair_group = static_cast<int>(thresholds().pair_group);
    a.pdone = d_pdone.p;
    a.bready = d_bready.p;
    a.rscratch = d_rscratch.p;
    a.nzflag = d_nz.p;
    a.done = d_done.p;
    a.ticket = d_ticket.p;
    a.n_items = cur.n_items;
    a.forced = d_forced.p;
    a.mode = st ? st->mode : 0;
    a.absolute = st ? st->absolute : 0;
    a.eps = st ? st->eps : 1e-6;
    a.fixed_rank = st ? static_cast<int>(st->rank) : 0;
    a.err = d_err.p;
    a.shifts = d_shifts.p;
    a.bmax = std::max(cur.bmax, 1);
    if (a.bmax > kSweepBlockMax) {
      std::ostringstream os;
      os << "level " << li + 1 << ": block size " << a.bmax << " exceeds the sweep kernel's limit " << kSweepBlockMax;
      throw std::invalid_argument(os.str());
    }
    a.kcap = sweep_kcap(a.bmax);
    // per-CTA buffer, rounded to 256 B so every CTA's (global-scratch) base keeps double2 alignment
    int64_t need = (sweep_smem_doubles(a.bmax, a.kcap) + 31) / 32 * 32;
    size_t smem = static_cast<size_t>(need) * sizeof(double);
    DevArray<double> scratch;
    int per_sm = 0;
    if (smem <= 200 * 1024) {
      per_sm = sweep_max_ctas_per_sm(smem);
    }
    if (per_sm < 1) {
      std::fprintf(stderr, "[ce] level %zu: sweep buffer %lld doubles -> global scratch\n", li + 1,
                   static_cast<long long>(need));
      a.use_global_scratch = 1;
      smem = 0;
      per_sm = std::max(1, sweep_max_ctas_per_sm(0));
      per_sm = std::min(per_sm, 4);
    }
    if (const char* cps = std::getenv("CE_CTAS_PER_SM")) per_sm = std::max(1, std::min(per_sm, std::atoi(cps)));
    int grid = ctx->sm_count * per_sm;
    if (grid > cur.n_items) grid = static_cast<int>(std::max<int64_t>(cur.n_items, 1));
    if (a.use_global_scratch) {
      scratch.alloc(static_cast<size_t>(need) * static_cast<size_t>(grid));
      a.scratch = scratch.p;
      a.scratch_per_cta = need;
    }
    static const bool profile = std::getenv("CE_PROFILE") && std::getenv("CE_PROFILE")[0] == '1';
    DevArray<unsigned long long> d_prof;
    if (profile) {
      d_prof.alloc(kProfCount);
      d_prof.zero(s);
      a.prof = d_prof.p;
    }
    DevArray<unsigned long long> d_trace;
    static const int trace_level = std::getenv("CE_TRACE") ? std::atoi(std::getenv("CE_TRACE")) : 0;
    if (trace_level == static_cast<int>(li) + 1) {
      d_trace.alloc(static_cast<size_t>(4 * cur.n_items));
      d_trace.zero(s);
      a.trace = d_trace.p;
    }
    // sharded level: phase split, per-phase tickets
    ShardLevel SL;
    const bool sharded_level = shard && shard->n_ranks >= 1 && [&] {
      SL = shard_level(*shard, cur, labels);
      return SL.prefix > 0;
    }();
    DevArray<int> d_it1r, d_it1p, d_it3r, d_it3p, d_foreign;
    int64_t n_it1 = 0, n_it3 = 0;
    if (sharded_level) {
      std::vector<int> r1, p1, r3, p3;
      build_tickets(cur, &SL.own1, r1, p1);
      build_tickets(cur, &SL.phase3, r3, p3);
      n_it1 = static_cast<int64_t>(r1.size());
      n_it3 = static_cast<int64_t>(r3.size());
      d_it1r.upload(r1, s);
      d_it1p.upload(p1, s);
      d_it3r.upload(r3, s);
      d_it3p.upload(p3, s);
      d_foreign.upload(SL.foreign1, s);
      F->shard.phase1_rows += SL.prefix;
      F->shard.phase3_rows += cur.M - SL.prefix;
      F->shard.own_rows += static_cast<int64_t>(SL.by_owner[static_cast<size_t>(shard->rank)].size());
    }
    Events ev_lvl, ev_sw;
    const double h_t1 = now_s();
    CE_CUDA(cudaEventRecord(ev_lvl.a, s));
    CE_CUDA(cudaEventRecord(ev_sw.a, s));
    if (!sharded_level) {
      launch_sweep(a, grid, smem, s);
    } else {
      // phase 1: this rank's box-interior rows, no communication
      a.item_row = d_it1r.p;
      a.item_part = d_it1p.p;
      a.n_items = n_it1;
      if (n_it1 > 0) launch_sweep(a, static_cast<int>(std::min<int64_t>(grid, n_it1)), smem, s);
      CE_CUDA(cudaGetLastError());
      shard_check_status(*shard, s, d_err.p);
      int h0 = 0;
      CE_CUDA(cudaMemcpy(&h0, d_err.p, sizeof h0, cudaMemcpyDeviceToHost));
      if (h0 == 0) {
        // E1: phase-1 rows' integers, then every within-box block the interface rows touch
        shard_exchange_ints(*shard, s, SL, LF, F->shard);
        std::vector<char> mark(static_cast<size_t>(cur.nslots), 0);
        std::vector<Seg> segs;
        auto add_block = [&](int64_t x, int64_t y, std::vector<char>& mk, std::vector<Seg>& out, bool corner) {
          const int64_t lx = labels[static_cast<size_t>(x)], ly = labels[static_cast<size_t>(y)];
          if (lx < 0 || lx != ly) return;
          const int64_t hi = std::max(x, y), lo2 = std::min(x, y);
          const int64_t sl = sq_slot_of(cur, hi, lo2);
          if (sl < 0 || mk[static_cast<size_t>(sl)]) return;
          mk[static_cast<size_t>(sl)] = 1;
          const int bh = cur.bsz[static_cast<size_t>(hi)], bl = cur.bsz[static_cast<size_t>(lo2)];
          const int rr = corner ? LF.rank[static_cast<size_t>(hi)] : bh, cc = corner ? LF.rank[static_cast<size_t>(lo2)] : bl;
          if (rr > 0 && cc > 0) out.push_back({cur.slot_off[static_cast<size_t>(sl)], rr, cc, bl, shard->owner(lx)});
        };
        auto footprint = [&](int64_t i, auto&& add) {  // blocks row i reads / writes in its sweep
          for (int64_t e = cur.sptr[static_cast<size_t>(i)]; e < cur.sptr[static_cast<size_t>(i + 1)]; ++e)
            add(i, cur.scol[static_cast<size_t>(e)]);
          const int64_t c0 = cur.cptr[static_cast<size_t>(i)], c1 = cur.cptr[static_cast<size_t>(i + 1)];
          for (int64_t x = c0; x < c1; ++x)
            for (int64_t y = x; y < c1; ++y) add(cur.ccol[static_cast<size_t>(x)], cur.ccol[static_cast<size_t>(y)]);
        };
        for (int64_t i = SL.prefix; i < cur.M; ++i)
          footprint(i, [&](int64_t x, int64_t y) { add_block(x, y, mark, segs, false); });
        shard_exchange(*shard, s, store.p, std::move(segs), F->shard);
        // phase 3: every interface row on every rank; the other ranks' phase-1 rows are done
        launch_precomplete(d_foreign.p, static_cast<int64_t>(SL.foreign1.size()), dcur.target.p, dcur.pan_ptr.p,
                           d_done.p, d_pdone.p, d_bready.p, s);
        d_ticket.zero(s);
        a.item_row = d_it3r.p;
        a.item_part = d_it3p.p;
        a.n_items = n_it3;
        if (n_it3 > 0) launch_sweep(a, static_cast<int>(std::min<int64_t>(grid, n_it3)), smem, s);
        CE_CUDA(cudaGetLastError());
        shard_check_status(*shard, s, d_err.p);
        // after the pending rotation below: E2 (factor rows) and E3 (retained corners)
        shard_post = [&, mark]() mutable {
          std::vector<Seg> fsegs, bsegs, ssegs, csegs;
          for (int r = 0; r < shard->n_ranks; ++r)
            for (int i : SL.by_owner[static_cast<size_t>(r)]) {
              const size_t iu = static_cast<size_t>(i);
              const int64_t b = cur.bsz[iu];
              fsegs.push_back({cur.chol_off[iu], 1, static_cast<int>(b * b + (b + cur.csum[iu]) * b), 0, r});
              bsegs.push_back({cur.basis_off[iu], 1, static_cast<int>(b * b), 0, r});
              const int64_t ns = std::min<int64_t>(b, cur.fsum[iu]);
              if (ns > 0) ssegs.push_back({cur.sigma_off[iu], 1, static_cast<int>(ns), 0, r});
            }
          for (auto* v : {&fsegs, &bsegs, &ssegs})
            for (Seg& g : *v) g.ld = g.cols;
          shard_exchange(*shard, s, LF.d_fac.p, std::move(fsegs), F->shard);
          shard_exchange(*shard, s, LF.d_basis.p, std::move(bsegs), F->shard);
          shard_exchange(*shard, s, LF.d_sigma.p, std::move(ssegs), F->shard);
          // E3: retained corners of the other within-box blocks the phase-1 rows wrote
          LF.d_rank.download(LF.rank, s);
          CE_CUDA(cudaStreamSynchronize(s));
          for (int64_t i = 0; i < SL.prefix; ++i)
            footprint(i, [&](int64_t x, int64_t y) { add_block(x, y, mark, csegs, true); });
          shard_exchange(*shard, s, store.p, std::move(csegs), F->shard);
        };
      }
    }
    CE_CUDA(cudaGetLastError());
    CE_CUDA(cudaEventRecord(ev_sw.b, s));
    int herr[4] = {0, 0, 0, 0};
    int hsh = 0;
    CE_CUDA(cudaMemcpyAsync(herr, d_err.p, sizeof herr, cudaMemcpyDeviceToHost, s));
    CE_CUDA(cudaMemcpyAsync(&hsh, d_shifts.p, sizeof hsh, cudaMemcpyDeviceToHost, s));
    CE_CUDA(cudaStreamSynchronize(s));
    if (herr[0] == kErrBreakdown) {
      const int64_t row = static_cast<int64_t>(herr[2]) | (static_cast<int64_t>(herr[3]) << 31);
      std::ostringstream os;
      os << "elimination breakdown at level " << herr[1] << ", block " << row
         << ": trailing pivot not positive definite after shift";
      throw Breakdown(herr[1], row, os.str());
    }
    if (profile) {
      std::vector<unsigned long long> hp;
      d_prof.download(hp, s);
      CE_CUDA(cudaStreamSynchronize(s));
      const char* names[] = {"wait", "A1", "A2", "A2.tsqr", "A2.svd", "A2.basis", "A2.pivot", "A2.strip", "A2.panels",
                             "A3", "B", "nA1", "nA2", "nA3", "nB", "svd.pre", "svd.jac", "svd.post", "sweeps", "svds", "B.setup", "B.stage", "B.tiles"};
      std::fprintf(stderr, "[ce-profile] level %zu M=%lld grid=%d waves=%lld items=%lld sweep=%.3f ms |", li + 1,
                   static_cast<long long>(cur.M), grid, static_cast<long long>(cur.n_waves),
                   static_cast<long long>(cur.n_items), 1e3 * ev_sw.seconds());
      for (int k = 0; k < kProfCount; ++k)
        std::fprintf(stderr, " %s=%.3g", names[k], (k < kProfNA1 || (k >= kProfSvdPre && k <= kProfSvdPost)) ? static_cast<double>(hp[static_cast<size_t>(k)]) / 1.9e9 : static_cast<double>(hp[static_cast<size_t>(k)]));
      std::fprintf(stderr, "  (cycle sums in SM-seconds @1.9GHz)\n");
    }
    if (herr[0] == kErrPattern) throw std::logic_error("update outside the squared pattern");
    if (herr[0] != 0) {
      const int64_t row = static_cast<int64_t>(herr[2]) | (static_cast<int64_t>(herr[3]) << 31);
      const char* what = herr[0] == kErrChunk ? "far-gather chunk narrower than a block"
                         : herr[0] == kErrStrip ? "strip chunk narrower than a block"
                         : herr[0] == kErrNaN ? "non-finite column norm" : "internal";
      std::ostringstream os;
      os << "internal sweep error (" << what << ") at level " << herr[1] << " row " << row;
      throw std::logic_error(os.str());
    }
    if (a.trace) {  // development trace: items (row, part) + timestamps -> CE_TRACE_FILE
      std::vector<unsigned long long> tr;
      d_trace.download(tr, s);
      CE_CUDA(cudaStreamSynchronize(s));
      const char* path = std::getenv("CE_TRACE_FILE") ? std::getenv("CE_TRACE_FILE") : "/tmp/ce_trace.bin";
      if (FILE* fp = std::fopen(path, "wb")) {
        const int64_t n = cur.n_items, m = cur.M;
        std::fwrite(&n, sizeof n, 1, fp);
        std::fwrite(&m, sizeof m, 1, fp);
        std::fwrite(cur.item_row.data(), sizeof(int), static_cast<size_t>(n), fp);
        std::fwrite(cur.item_part.data(), sizeof(int), static_cast<size_t>(n), fp);
        std::fwrite(cur.nA1.data(), sizeof(int), static_cast<size_t>(cur.M), fp);
        std::fwrite(cur.nA3.data(), sizeof(int), static_cast<size_t>(cur.M), fp);
        std::fwrite(cur.wave.data(), sizeof(int64_t), static_cast<size_t>(cur.M), fp);
        std::fwrite(tr.data(), sizeof(unsigned long long), tr.size(), fp);
        std::fclose(fp);
      }
    }
    Events ev_pend;
    if (profile) CE_CUDA(cudaEventRecord(ev_pend.a, s));
    launch_pending_rotation(a, s);
    CE_CUDA(cudaGetLastError());
    if (profile) {
      CE_CUDA(cudaEventRecord(ev_pend.b, s));
      CE_CUDA(cudaStreamSynchronize(s));
      std::fprintf(stderr, "[ce-profile] level %zu pending-rotation kernel %.2f ms\n", li + 1, 1e3 * ev_pend.seconds());
    }
    if (shard_post) {
      shard_post();
      shard_post = nullptr;
    }
    LF.d_rank.download(LF.rank, s);
    LF.d_width.download(LF.width, s);
    LF.d_has_basis.download(LF.has_basis, s);
    LF.d_fcols.download(LF.fcols, s);
    LF.d_nsig.download(LF.nsig, s);
    CE_CUDA(cudaStreamSynchronize(s));
    const double h_ts = now_s();
    int64_t eliminated = 0;
    for (int w : LF.width) {
      eliminated += w;
      if (w > kApplyWmax)
        throw std::runtime_error("eliminated block width " + std::to_string(w) + " exceeds the apply limit " +
                                 std::to_string(kApplyWmax));
    }
    if (eliminated == 0) break;  // factorization.cpp:374 (store untouched: every r_i = b_i)
    shifts += hsh;
    LF.shift_retries = hsh;

    // ---- remainder (level_matrix.cpp:185-248) + next level plan ----
    const int64_t ng = static_cast<int64_t>(cur_groups.size());
    std::vector<int64_t> group_of(static_cast<size_t>(cur.M));
    for (int64_t g = 0; g < ng; ++g)
      for (int64_t b : cur_groups[static_cast<size_t>(g)]) group_of[static_cast<size_t>(b)] = g;
    std::vector<int64_t> gsize(static_cast<size_t>(ng), 0), alive(static_cast<size_t>(ng), -1);
    for (int64_t g = 0; g < ng; ++g)
      for (int64_t b : cur_groups[static_cast<size_t>(g)]) gsize[static_cast<size_t>(g)] += LF.rank[static_cast<size_t>(b)];
    std::vector<int> nbsz;
    for (int64_t g = 0; g < ng; ++g)
      if (gsize[static_cast<size_t>(g)] > 0) {
        alive[static_cast<size_t>(g)] = static_cast<int64_t>(nbsz.size());
        nbsz.push_back(static_cast<int>(gsize[static_cast<size_t>(g)]));
      }
    // coarse pattern of sq over groups restricted to alive groups
    const int64_t nM = static_cast<int64_t>(nbsz.size());
    std::vector<int64_t> nptr(static_cast<size_t>(nM + 1), 0);
    std::vector<int> ncol;
    // the speculative plan applies when it assumed exactly this alive set
    std::pair<LevelPlan, std::vector<char>> sp = spec.get();
    bool spec_ok = true;
    for (int64_t g = 0; g < ng && spec_ok; ++g) spec_ok = (alive[static_cast<size_t>(g)] >= 0) == (sp.second[static_cast<size_t>(g)] != 0);
    if (!spec_ok) {  // a group died (or survived) against the structural prediction: plan again
      // coarse rows of the alive groups, in parallel (one mark array per host thread)
      std::vector<std::vector<int>> rows(static_cast<size_t>(ng));
      parallel_rows(ng, [&](int64_t g0, int64_t g1) {
        std::vector<int64_t> mark(static_cast<size_t>(ng), -1);
        for (int64_t g = g0; g < g1; ++g) {
          if (alive[static_cast<size_t>(g)] < 0) continue;
          auto& row = rows[static_cast<size_t>(g)];
          for (int64_t b : cur_groups[static_cast<size_t>(g)])
            for (int64_t e = cur.sptr[static_cast<size_t>(b)]; e < cur.sptr[static_cast<size_t>(b + 1)]; ++e) {
              const int64_t h = group_of[static_cast<size_t>(cur.scol[static_cast<size_t>(e)])];
              if (alive[static_cast<size_t>(h)] < 0 || mark[static_cast<size_t>(h)] == g) continue;
              mark[static_cast<size_t>(h)] = g;
              row.push_back(static_cast<int>(alive[static_cast<size_t>(h)]));
            }
          std::sort(row.begin(), row.end());
        }
      });
      for (int64_t g = 0; g < ng; ++g) {
        if (alive[static_cast<size_t>(g)] < 0) continue;
        ncol.insert(ncol.end(), rows[static_cast<size_t>(g)].begin(), rows[static_cast<size_t>(g)].end());
        nptr[static_cast<size_t>(alive[static_cast<size_t>(g)] + 1)] = static_cast<int64_t>(ncol.size());
      }
    }
    std::vector<int> next_block(static_cast<size_t>(cur.M), -1), next_loc(static_cast<size_t>(cur.M), 0);
    for (int64_t g = 0; g < ng; ++g) {
      int at = 0;
      for (int64_t b : cur_groups[static_cast<size_t>(g)]) {
        next_loc[static_cast<size_t>(b)] = at;
        next_block[static_cast<size_t>(b)] = static_cast<int>(alive[static_cast<size_t>(g)]);
        at += LF.rank[static_cast<size_t>(b)];
      }
    }
    // next level's numeric plan on a host thread (it is on the critical path to the next sweep);
    // the gathers, their checks and uploads below run meanwhile
    LevelPlan next;
    std::future<void> next_fut;
    if (nM > 0)
      next_fut = std::async(std::launch::async, [&]() {
        if (spec_ok) {
          next = std::move(sp.first);
          plan_numeric(next, nbsz);
        } else {
          next = plan_level(nbsz, nptr, ncol, s);  // after the sweep: the device is idle
        }
      });
    // gathers (factorization.cpp:76-85)
    std::vector<int64_t> elim, kept;
    for (int64_t b = 0; b < cur.M; ++b)
      for (int64_t rr = LF.rank[static_cast<size_t>(b)]; rr < cur.bsz[static_cast<size_t>(b)]; ++rr) elim.push_back(cur.offsets[static_cast<size_t>(b)] + rr);
    for (const auto& g : cur_groups)
      for (int64_t b : g)
        for (int64_t rr = 0; rr < LF.rank[static_cast<size_t>(b)]; ++rr) kept.push_back(cur.offsets[static_cast<size_t>(b)] + rr);
    LF.n_elim = static_cast<int64_t>(elim.size());
    LF.n_kept = static_cast<int64_t>(kept.size());
    {  // validate (factorization.cpp:283-288): the gather lists partition the level space
      std::vector<int> seen(static_cast<size_t>(cur.M), 0);
      for (const auto& g : cur_groups)
        for (int64_t b : g) ++seen[static_cast<size_t>(b)];
      for (int64_t b = 0; b < cur.M; ++b)
        if (LF.rank[static_cast<size_t>(b)] > 0 && seen[static_cast<size_t>(b)] != 1)
          throw std::logic_error("gather lists must partition the level space");
      if (LF.n_elim + LF.n_kept != cur.dim) throw std::logic_error("eliminated plus kept must cover the level");
    }
    LF.d_elim_gather.upload(elim, s);
    LF.d_kept_gather.upload(kept, s);

    DevPlan dnext;
    const double h_t2 = now_s();
    double h_t3 = h_t2;
    if (nM > 0) {
      next_fut.get();
      h_t3 = now_s();
      dnext.upload(next, s);
      const double h_up = now_s();
      if (nstore.n < static_cast<size_t>(next.store_doubles)) nstore.alloc(static_cast<size_t>(next.store_doubles));
      if (next.store_doubles > 0)
        CE_CUDA(cudaMemsetAsync(nstore.p, 0, static_cast<size_t>(next.store_doubles) * sizeof(double), s));
      const double h_al = now_s();
      Events ev_rem;
      if (profile) {
        CE_CUDA(cudaStreamSynchronize(s));
        std::fprintf(stderr, "[ce-profile] level %zu next plan: upload(host) %.1f ms, alloc+memset %.1f ms, drained %.1f ms\n",
                     li + 1, 1e3 * (h_up - h_t3), 1e3 * (h_al - h_up), 1e3 * (now_s() - h_al));
        CE_CUDA(cudaEventRecord(ev_rem.a, s));
      }
      DevArray<int> d_nb, d_nl;
      d_nb.upload(next_block, s);
      d_nl.upload(next_loc, s);
      RemainderArgs ra{};
      ra.M = cur.M;
      ra.bsz = dcur.bsz.p;
      ra.rank = LF.d_rank.p;
      ra.sq_ptr = dcur.sptr.p;
      ra.sq_col = dcur.scol.p;
      ra.sq_slot = dcur.sslot.p;
      ra.slot_off = dcur.slot_off.p;
      ra.store = store.p;
      ra.next_block = d_nb.p;
      ra.next_loc = d_nl.p;
      ra.nbsz = dnext.bsz.p;
      ra.nsq_ptr = dnext.sptr.p;
      ra.nsq_col = dnext.scol.p;
      ra.nsq_slot = dnext.sslot.p;
      ra.nslot_off = dnext.slot_off.p;
      ra.nstore = nstore.p;
      ra.err = d_err.p;
      launch_remainder(ra, s);
      CE_CUDA(cudaGetLastError());
      if (profile) {
        CE_CUDA(cudaEventRecord(ev_rem.b, s));
        CE_CUDA(cudaStreamSynchronize(s));
        std::fprintf(stderr, "[ce-profile] level %zu remainder kernel %.2f ms\n", li + 1, 1e3 * ev_rem.seconds());
      }
      CE_CUDA(cudaEventRecord(ev_lvl.b, s));
      CE_CUDA(cudaMemcpyAsync(herr, d_err.p, sizeof herr, cudaMemcpyDeviceToHost, s));
      CE_CUDA(cudaStreamSynchronize(s));
      if (herr[0] != 0) throw std::logic_error("remainder block outside the coarse squared pattern");
    } else {
      CE_CUDA(cudaEventRecord(ev_lvl.b, s));
      CE_CUDA(cudaStreamSynchronize(s));
    }
    LF.seconds = ev_lvl.seconds();
    LF.sweep_seconds = ev_sw.seconds();
    if (profile)
      std::fprintf(stderr, "[ce-profile] level %zu host: setup %.1f ms, sweep+downloads %.1f ms, coarse pattern %.1f ms, plan %.1f ms, upload+remainder %.1f ms\n",
                   li + 1, 1e3 * (h_t1 - h_t0), 1e3 * (h_ts - h_t1), 1e3 * (h_t2 - h_ts), 1e3 * (h_t3 - h_t2), 1e3 * (now_s() - h_t3));
    F->sweep_seconds += LF.sweep_seconds;

    // host copies needed by apply / dump / stats
    LF.bsz = cur.bsz;
    LF.offsets = cur.offsets;
    LF.cptr = cur.cptr;
    LF.ccol = cur.ccol;
    LF.croff = cur.croff;
    LF.chol_off = cur.chol_off;
    LF.g_off = cur.g_off;
    LF.basis_off = cur.basis_off;
    LF.sigma_off = cur.sigma_off;
    LF.groups = cur_groups;
    LF.d_bsz = std::move(dcur.bsz);
    LF.d_offsets = std::move(dcur.offsets);
    LF.d_cptr = std::move(dcur.cptr);
    LF.d_ccol = std::move(dcur.ccol);
    LF.d_croff = std::move(dcur.croff);
    LF.d_chol_off = std::move(dcur.chol_off);
    LF.d_g_off = std::move(dcur.g_off);
    LF.d_basis_off = std::move(dcur.basis_off);
    LF.d_sigma_off = std::move(dcur.sigma_off);
    const double h_ta = now_s();
    const double h_tb = now_s();
    // stats (factorization.cpp:376-405) + §8d algorithmic counts
    {
      std::vector<int64_t> pend(static_cast<size_t>(cur.M), 0);
      for (int64_t k = 0; k < cur.M; ++k)
        for (int64_t e = cur.cptr[static_cast<size_t>(k)]; e < cur.cptr[static_cast<size_t>(k + 1)]; ++e) {
          const int t = cur.ccol[static_cast<size_t>(e)];
          if (t > k) pend[static_cast<size_t>(t)] += LF.width[static_cast<size_t>(k)];
        }
      double by = 0.0, fl = 0.0;
      for (int64_t i = 0; i < cur.M; ++i) {
        const double b = cur.bsz[static_cast<size_t>(i)], c = static_cast<double>(cur.csum[static_cast<size_t>(i)]);
        const double r = LF.rank[static_cast<size_t>(i)], w = LF.width[static_cast<size_t>(i)];
        double sq2 = 0.0;
        for (int64_t e = cur.cptr[static_cast<size_t>(i)]; e < cur.cptr[static_cast<size_t>(i + 1)]; ++e) {
          const double bt = cur.bsz[static_cast<size_t>(cur.ccol[static_cast<size_t>(e)])];
          sq2 += bt * bt;
        }
        const double Pp = (c * c + sq2) / 2;
        row_counts(b, c, static_cast<double>(LF.fcols[static_cast<size_t>(i)]), r, w,
                   LF.has_basis[static_cast<size_t>(i)] ? static_cast<double>(pend[static_cast<size_t>(i)]) : 0.0, Pp,
                   LF.has_basis[static_cast<size_t>(i)] != 0, LF.nsig[static_cast<size_t>(i)] > 0, by, fl);
        const int64_t wi = LF.width[static_cast<size_t>(i)], ri = LF.rank[static_cast<size_t>(i)];
        if (wi > 0) {
          const int64_t cs = cur.csum[static_cast<size_t>(i)];
          F->l_payload_bytes += (wi * wi + ri * wi + cs * wi) * 8;
          F->l_scalar_nnz += wi * (wi + 1) / 2 + ri * wi + cs * wi;
        }
        if (LF.has_basis[static_cast<size_t>(i)]) F->q_payload_bytes += static_cast<int64_t>(b * b) * 8;
      }
      // remainder extraction traffic
      double rem = 0.0;
      for (int64_t sI = 0; sI < cur.M; ++sI)
        for (int64_t e = cur.sptr[static_cast<size_t>(sI)]; e < cur.sptr[static_cast<size_t>(sI + 1)]; ++e) {
          const int t = cur.scol[static_cast<size_t>(e)];
          if (t > sI) break;
          rem += static_cast<double>(LF.rank[static_cast<size_t>(sI)]) * LF.rank[static_cast<size_t>(t)];
        }
      by += 2 * 8 * rem;
      LF.alg_bytes = by;
      LF.alg_flops = fl;
      F->factor_blocks += 2.0 * static_cast<double>(cur.lower_blocks);
    }
    elim_total += LF.n_elim;

    if (shard) {  // next level's box labels: a group's common label, -1 when its members differ
      std::vector<int64_t> nl(static_cast<size_t>(nM), -1);
      for (int64_t g = 0; g < ng; ++g) {
        if (alive[static_cast<size_t>(g)] < 0) continue;
        const auto& mem = cur_groups[static_cast<size_t>(g)];
        int64_t v = labels[static_cast<size_t>(mem[0])];
        for (int64_t b : mem)
          if (labels[static_cast<size_t>(b)] != v) v = -1;
        nl[static_cast<size_t>(alive[static_cast<size_t>(g)])] = v;
      }
      labels = std::move(nl);
    }
    std::vector<int64_t> next_alive(plan_groups.size(), -1);
    for (size_t g = 0; g < plan_groups.size(); ++g)
      if (slot_of_group[g] >= 0) next_alive[g] = alive[static_cast<size_t>(slot_of_group[g])];
    alive_map = std::move(next_alive);
    F->levels.push_back(std::move(LF));
    apply_jobs.push_back(std::async(std::launch::async, build_apply_lists, std::ref(F->levels.back()), li, s));
    if (std::getenv("CE_PROFILE") && std::getenv("CE_PROFILE")[0] == '1')
      std::fprintf(stderr, "[ce-profile] level %zu host: apply lists %.1f ms, stats+rest %.1f ms, iteration %.1f ms\n", li + 1,
                   1e3 * (h_tb - h_ta), 1e3 * (now_s() - h_tb), 1e3 * (now_s() - h_t0));

    if (spec.valid()) spec.wait();  // the speculative planner reads `cur` (early exits above)
    cur = std::move(next);
    // the remainder kernel queued above still reads this level's device plan: keep it (and
    // its arena, out of the allocator cache that other host threads draw from) until the
    // next level's sweep has completed
    dprev = std::move(dcur);
    dcur = std::move(dnext);
    std::swap(store, nstore);
    if (nM == 0) break;
  }

  t_loop1 = now_s();
  // ---- dense tail (factorization.cpp:419-436) ----
  F->tail_dim = cur.M > 0 ? cur.dim : 0;
  if (F->tail_dim > 0) {
    const int64_t n = F->tail_dim;
    F->d_tail_L.alloc(static_cast<size_t>(n * n));
    F->d_tail_Linv.alloc(static_cast<size_t>(n * n));
    F->d_tail_L.zero(s);
    launch_densify(cur.M, dcur.bsz.p, dcur.offsets.p, dcur.sptr.p, dcur.scol.p, dcur.sslot.p, dcur.slot_off.p,
                   store.p, F->d_tail_L.p, n, s);
    CE_CUDA(cudaGetLastError());
    DevArray<double> backup(static_cast<size_t>(n * n)), d_tr(1);
    CE_CUDA(cudaMemcpyAsync(backup.p, F->d_tail_L.p, static_cast<size_t>(n * n) * sizeof(double), cudaMemcpyDeviceToDevice, s));
    dense_trace(backup.p, n, d_tr.p, s);
    DevArray<int> d_fail(1);
    d_fail.zero(s);
    dense_cholesky(F->d_tail_L.p, n, d_fail.p, s);
    int hf = 0;
    CE_CUDA(cudaMemcpyAsync(&hf, d_fail.p, sizeof hf, cudaMemcpyDeviceToHost, s));
    CE_CUDA(cudaStreamSynchronize(s));
    if (hf) {
      double tr = 0.0;
      CE_CUDA(cudaMemcpy(&tr, d_tr.p, sizeof tr, cudaMemcpyDeviceToHost));
      const double shift = 1e-12 * tr / static_cast<double>(n);
      CE_CUDA(cudaMemcpyAsync(F->d_tail_L.p, backup.p, static_cast<size_t>(n * n) * sizeof(double), cudaMemcpyDeviceToDevice, s));
      dense_add_shift(F->d_tail_L.p, n, shift, s);
      d_fail.zero(s);
      dense_cholesky(F->d_tail_L.p, n, d_fail.p, s);
      CE_CUDA(cudaMemcpyAsync(&hf, d_fail.p, sizeof hf, cudaMemcpyDeviceToHost, s));
      CE_CUDA(cudaStreamSynchronize(s));
      if (hf) {
        std::ostringstream os;
        os << "dense tail not positive definite after shift " << shift;
        throw Breakdown(static_cast<int>(F->levels.size()) + 1, -1, os.str());
      }
    }
    dense_tri_inverse(F->d_tail_L.p, F->d_tail_Linv.p, n, s);
    CE_CUDA(cudaGetLastError());
  }
  validate_factor(*F, s);
  CE_CUDA(cudaEventRecord(ev_all.b, s));
  CE_CUDA(cudaStreamSynchronize(s));
  F->device_seconds = ev_all.seconds();
  F->tail_bytes = F->tail_dim * F->tail_dim * 8;
  F->l_scalar_nnz += F->tail_dim * (F->tail_dim + 1) / 2;
  F->factor_blocks += 0.5 * static_cast<double>(F->tail_dim) * static_cast<double>(F->tail_dim);
  F->shift_retries = shifts;
  if (shift_total) *shift_total = shifts;

  for (auto& j : apply_jobs) j.get();  // rethrows a failed list build
  // apply workspaces
  F->w_v.alloc(static_cast<size_t>(std::max<int64_t>(F->n, 1)));
  F->w_active.alloc(static_cast<size_t>(std::max<int64_t>(F->n, 1)));
  F->w_elim.alloc(static_cast<size_t>(std::max<int64_t>(elim_total, 1)));
  int64_t mmax = 1;
  F->elim_base.clear();
  int64_t eb = 0;
  for (const auto& L : F->levels) {
    mmax = std::max(mmax, L.M);
    F->elim_base.push_back(eb);
    eb += L.n_elim;
  }
  F->w_flags.alloc(static_cast<size_t>(mmax));
  F->w_parts.alloc(static_cast<size_t>(mmax));
  F->w_ticket.alloc(1);
  int64_t scr = 1;
  for (const auto& L : F->levels) scr = std::max(scr, L.scratch_doubles);
  F->w_scratch.alloc(static_cast<size_t>(scr));
  F->total_seconds = now_s() - t_start;
  if (std::getenv("CE_PROFILE") && std::getenv("CE_PROFILE")[0] == '1')
    std::fprintf(stderr, "[ce-profile] factorize host: before level loop %.1f ms, level loop %.1f ms, after %.1f ms, total %.1f ms\n",
                 1e3 * (t_loop0 - t_start), 1e3 * (t_loop1 - t_loop0), 1e3 * (now_s() - t_start - (t_loop1 - t_start)),
                 1e3 * F->total_seconds);
  return F.release();
}

// ---------------------------------------------------------------- apply
namespace {
ApplyLevelArgs level_args(const Factor& f, const LevelFactor& L, double* v) {
  ApplyLevelArgs a{};
  a.M = L.M;
  a.bsz = L.d_bsz.p;
  a.offsets = L.d_offsets.p;
  a.rank = L.d_rank.p;
  a.width = L.d_width.p;
  a.has_basis = L.d_has_basis.p;
  a.basis = L.d_basis.p;
  a.basis_off = L.d_basis_off.p;
  a.fac = L.d_fac.p;
  a.chol_off = L.d_chol_off.p;
  a.g_off = L.d_g_off.p;
  a.cl_ptr = L.d_cptr.p;
  a.cl_col = L.d_ccol.p;
  a.cl_roff = L.d_croff.p;
  a.v = v;
  a.flags = f.w_flags.p;
  a.ticket = f.w_ticket.p;
  a.in_ptr = L.d_in_ptr.p;
  a.in_split = L.d_in_split.p;
  a.in_src = L.d_in_src.p;
  a.in_goff = L.d_in_goff.p;
  a.in_w = L.d_in_w.p;
  a.in_uoff = L.d_in_uoff.p;
  a.dep_ptr = L.d_dep_ptr.p;
  a.dep_t = L.d_dep_t.p;
  a.cl_nt = L.d_cl_nt.p;
  a.linv = L.d_linv.p;
  a.linv_off = L.d_linv_off.p;
  a.scratch = f.w_scratch.p;
  a.parts_done = f.w_parts.p;
  return a;
}
}  // namespace

namespace {
// Serialises the applies of one factor (they share its workspaces, host_api.hpp): the
// enqueue happens under the factor's mutex and waits for the previous apply's event.
struct ApplyGuard {
  const Factor& f;
  cudaStream_t s;
  std::lock_guard<std::mutex> lk;
  ApplyGuard(const Factor& fa, cudaStream_t st) : f(fa), s(st), lk(fa.apply_mu) {
    if (!f.apply_done) CE_CUDA(cudaEventCreateWithFlags(&f.apply_done, cudaEventDisableTiming));
    else CE_CUDA(cudaStreamWaitEvent(s, f.apply_done, 0));
  }
  ~ApplyGuard() { cudaEventRecord(f.apply_done, s); }
};
}  // namespace

void apply_device(const Factor& f, const double* d_b, double* d_x, cudaStream_t s) {
  ApplyGuard guard(f, s);
  const int grid = f.ctx->sm_count * 8;
  static const bool aprof = std::getenv("CE_PROFILE") && std::getenv("CE_PROFILE")[0] == '1';
  std::vector<Events> evs(aprof ? 2 * f.levels.size() : 0);
  double* active = f.w_active.p;
  double* v = f.w_v.p;
  CE_CUDA(cudaMemcpyAsync(active, d_b, static_cast<size_t>(f.n) * sizeof(double), cudaMemcpyDeviceToDevice, s));
  for (size_t l = 0; l < f.levels.size(); ++l) {
    const LevelFactor& L = f.levels[l];
    CE_CUDA(cudaMemcpyAsync(v, active, static_cast<size_t>(L.dim) * sizeof(double), cudaMemcpyDeviceToDevice, s));
    ApplyLevelArgs a = level_args(f, L, v);
    launch_basis_apply(a, 1, s);
    CE_CUDA(cudaMemsetAsync(f.w_flags.p, 0, static_cast<size_t>(L.M) * sizeof(int), s));
    CE_CUDA(cudaMemsetAsync(f.w_ticket.p, 0, sizeof(unsigned long long), s));
    CE_CUDA(cudaMemsetAsync(f.w_parts.p, 0, static_cast<size_t>(L.M) * sizeof(int), s));
    a.item_row = L.d_fitem_row.p;
    a.item_part = L.d_fitem_part.p;
    a.n_items = L.n_fitems;
    a.part_ptr = L.d_fpart_ptr.p;
    a.part_b = L.d_fpart_b.p;
    a.scr_off = L.d_fscr_off.p;
    if (aprof) CE_CUDA(cudaEventRecord(evs[2 * l].a, s));
    // warp-granular items where the level is throughput-bound (many independent rows per wave:
    // colour-major / sharded plans, A/B -33% apply time); CTA items where it is a latency chain
    // (the reference plan's ~500-1500 waves: the 4-warp split of a row's inputs is shorter)
    const bool warp_items = L.max_close <= CE_APPLY_WARP_MAX_CLOSE && L.M >= CE_APPLY_WARP_ROWS_PER_WAVE * std::max<int64_t>(L.n_waves, 1);
    launch_forward_tasks(a, static_cast<int>(std::min<int64_t>(grid, std::max<int64_t>(L.n_fitems, 1))), warp_items, s);
    if (aprof) CE_CUDA(cudaEventRecord(evs[2 * l].b, s));
    launch_forward_retained(a, s);
    launch_gather(v, L.d_elim_gather.p, f.w_elim.p + f.elim_base[l], L.n_elim, s);
    launch_gather(v, L.d_kept_gather.p, active, L.n_kept, s);
  }
  if (f.tail_dim > 0) {
    launch_dense_trmv(f.d_tail_Linv.p, active, v, f.tail_dim, 0, s);
    launch_dense_trmv(f.d_tail_Linv.p, v, active, f.tail_dim, 1, s);
  }
  for (size_t l = f.levels.size(); l-- > 0;) {
    const LevelFactor& L = f.levels[l];
    CE_CUDA(cudaMemsetAsync(v, 0, static_cast<size_t>(L.dim) * sizeof(double), s));
    launch_scatter(active, L.d_kept_gather.p, v, L.n_kept, s);
    launch_scatter(f.w_elim.p + f.elim_base[l], L.d_elim_gather.p, v, L.n_elim, s);
    ApplyLevelArgs a = level_args(f, L, v);
    CE_CUDA(cudaMemsetAsync(f.w_flags.p, 0, static_cast<size_t>(L.M) * sizeof(int), s));
    CE_CUDA(cudaMemsetAsync(f.w_ticket.p, 0, sizeof(unsigned long long), s));
    CE_CUDA(cudaMemsetAsync(f.w_parts.p, 0, static_cast<size_t>(L.M) * sizeof(int), s));
    a.item_row = L.d_bitem_row.p;
    a.item_part = L.d_bitem_part.p;
    a.n_items = L.n_bitems;
    a.part_ptr = L.d_bpart_ptr.p;
    a.part_b = L.d_bpart_b.p;
    a.scr_off = L.d_bscr_off.p;
    if (aprof) CE_CUDA(cudaEventRecord(evs[2 * l + 1].a, s));
    launch_backward_tasks(a, static_cast<int>(std::min<int64_t>(grid, std::max<int64_t>(L.n_bitems, 1))),
                          L.max_close <= CE_APPLY_WARP_MAX_CLOSE &&
                              L.M >= CE_APPLY_WARP_ROWS_PER_WAVE * std::max<int64_t>(L.n_waves, 1),
                          s);
    if (aprof) CE_CUDA(cudaEventRecord(evs[2 * l + 1].b, s));
    launch_basis_apply(a, 0, s);
    CE_CUDA(cudaMemcpyAsync(active, v, static_cast<size_t>(L.dim) * sizeof(double), cudaMemcpyDeviceToDevice, s));
  }
  CE_CUDA(cudaMemcpyAsync(d_x, active, static_cast<size_t>(f.n) * sizeof(double), cudaMemcpyDeviceToDevice, s));
  CE_CUDA(cudaGetLastError());
  if (aprof) {
    CE_CUDA(cudaStreamSynchronize(s));
    for (size_t l = 0; l < f.levels.size(); ++l)
      std::fprintf(stderr, "[ce-profile] apply level %zu: forward %.3f ms, backward %.3f ms (M=%lld)\n", l + 1,
                   1e3 * evs[2 * l].seconds(), 1e3 * evs[2 * l + 1].seconds(), static_cast<long long>(f.levels[l].M));
  }
}

// Validation tools (factorization.cpp:170-257) on the device.
void apply_tool_device(const Factor& f, int which, const double* d_x, double* d_y, cudaStream_t s) {
  ApplyGuard guard(f, s);
  double* active = f.w_active.p;
  double* v = f.w_v.p;
  CE_CUDA(cudaMemcpyAsync(active, d_x, static_cast<size_t>(f.n) * sizeof(double), cudaMemcpyDeviceToDevice, s));
  if (which == 2) {  // apply_q_transpose: y = [elim_1 | ... | tail]
    int64_t at = 0;
    for (const auto& L : f.levels) at += L.n_elim;
    CE_CUDA(cudaMemcpyAsync(v, d_x + at, static_cast<size_t>(f.n - at) * sizeof(double), cudaMemcpyDeviceToDevice, s));
    CE_CUDA(cudaMemcpyAsync(active, v, static_cast<size_t>(f.n - at) * sizeof(double), cudaMemcpyDeviceToDevice, s));
    for (size_t l = f.levels.size(); l-- > 0;) {
      const LevelFactor& L = f.levels[l];
      CE_CUDA(cudaMemsetAsync(v, 0, static_cast<size_t>(L.dim) * sizeof(double), s));
      launch_scatter(active, L.d_kept_gather.p, v, L.n_kept, s);
      launch_scatter(d_x + f.elim_base[l], L.d_elim_gather.p, v, L.n_elim, s);
      ApplyLevelArgs a = level_args(f, L, v);
      launch_basis_apply(a, 0, s);
      CE_CUDA(cudaMemcpyAsync(active, v, static_cast<size_t>(L.dim) * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
    CE_CUDA(cudaMemcpyAsync(d_y, active, static_cast<size_t>(f.n) * sizeof(double), cudaMemcpyDeviceToDevice, s));
    return;
  }
  std::vector<DevArray<int64_t>> eoffs;
  std::vector<DevArray<double>> cvals;
  for (size_t l = 0; l < f.levels.size(); ++l) {
    const LevelFactor& L = f.levels[l];
    CE_CUDA(cudaMemcpyAsync(v, active, static_cast<size_t>(L.dim) * sizeof(double), cudaMemcpyDeviceToDevice, s));
    ApplyLevelArgs a = level_args(f, L, v);
    launch_basis_apply(a, 1, s);
    if (which == 1) {
      launch_gather(v, L.d_elim_gather.p, d_y + f.elim_base[l], L.n_elim, s);
    } else {
      std::vector<int64_t> eo(static_cast<size_t>(L.M));
      int64_t at = 0;
      for (int64_t b = 0; b < L.M; ++b) {
        eo[static_cast<size_t>(b)] = at;
        at += L.width[static_cast<size_t>(b)];
      }
      eoffs.emplace_back();
      eoffs.back().upload(eo, s);
      cvals.emplace_back(static_cast<size_t>(std::max<int64_t>(at, 1)));
      launch_operator_forward(a, eoffs.back().p, cvals.back().p, s);
    }
    launch_gather(v, L.d_kept_gather.p, active, L.n_kept, s);
  }
  if (which == 1) {
    int64_t at = 0;
    for (const auto& L : f.levels) at += L.n_elim;
    CE_CUDA(cudaMemcpyAsync(d_y + at, active, static_cast<size_t>(f.n - at) * sizeof(double), cudaMemcpyDeviceToDevice, s));
    return;
  }
  if (f.tail_dim > 0) {
    launch_dense_trmv(f.d_tail_L.p, active, v, f.tail_dim, 1, s);
    launch_dense_trmv(f.d_tail_L.p, v, active, f.tail_dim, 0, s);
  }
  for (size_t l = f.levels.size(); l-- > 0;) {
    const LevelFactor& L = f.levels[l];
    CE_CUDA(cudaMemsetAsync(v, 0, static_cast<size_t>(L.dim) * sizeof(double), s));
    launch_scatter(active, L.d_kept_gather.p, v, L.n_kept, s);
    ApplyLevelArgs a = level_args(f, L, v);
    launch_operator_backward(a, eoffs[l].p, cvals[l].p, s);
    launch_basis_apply(a, 0, s);
    CE_CUDA(cudaMemcpyAsync(active, v, static_cast<size_t>(L.dim) * sizeof(double), cudaMemcpyDeviceToDevice, s));
  }
  CE_CUDA(cudaMemcpyAsync(d_y, active, static_cast<size_t>(f.n) * sizeof(double), cudaMemcpyDeviceToDevice, s));
  CE_CUDA(cudaStreamSynchronize(s));
}

void matvec_device(const Matrix& A, const double* d_x, double* d_y, cudaStream_t s) {
  launch_bsr_matvec(A.n, A.d_row_of.p, A.d_offsets.p, A.d_bsz.p, A.d_row_ptr.p, A.d_col_idx.p, A.d_val_ptr.p,
                    A.d_values.p, d_x, d_y, s);
}

// ---------------------------------------------------------------- PCG
SolveOut pcg_device(const Matrix& A, const Factor* M, const double* d_b, double* d_x, double tol, int64_t maxit,
                    bool track_true, cudaStream_t s) {
  const int64_t n = A.n;
  SolveOut out;
  const double t0 = now_s();
  DevArray<double> r(static_cast<size_t>(n)), z(static_cast<size_t>(n)), p(static_cast<size_t>(n)), q(static_cast<size_t>(n));
  DevArray<double> part(static_cast<size_t>(dot_partials_capacity())), sc(8);
  auto dot = [&](const double* x, const double* y, int slot) {
    const int np = launch_dot(x, y, n, part.p, s);
    launch_sum_partials(part.p, np, sc.p + slot, s);
  };
  auto fetch = [&](double* h, int slot, int cnt) {
    CE_CUDA(cudaMemcpyAsync(h, sc.p + slot, static_cast<size_t>(cnt) * sizeof(double), cudaMemcpyDeviceToHost, s));
    CE_CUDA(cudaStreamSynchronize(s));
  };
  auto precond = [&](const double* in, double* o) {
    if (M) apply_device(*M, in, o, s);
    else launch_copy(o, in, n, s);
  };
  const double one = 1.0;
  CE_CUDA(cudaMemcpyAsync(sc.p + 7, &one, sizeof(double), cudaMemcpyHostToDevice, s));
  auto true_resid = [&](double bnorm) {
    matvec_device(A, d_x, q.p, s);
    launch_copy(z.p, d_b, n, s);
    launch_axpy(z.p, q.p, sc.p + 7, sc.p + 7, -1.0, n, s);  // z = b - A x
    dot(z.p, z.p, 5);
    double h = 0.0;
    fetch(&h, 5, 1);
    return std::sqrt(h) / bnorm;
  };
  CE_CUDA(cudaMemsetAsync(d_x, 0, static_cast<size_t>(n) * sizeof(double), s));
  dot(d_b, d_b, 4);
  double hb = 0.0;
  fetch(&hb, 4, 1);
  const double bnorm = std::sqrt(hb);
  auto sample = [&](int64_t it, double rec, double tru) {  // IterationSample (minres.hpp:12-20)
    out.trace_iter.push_back(it);
    out.trace_rec.push_back(rec);
    out.trace_true.push_back(tru);
    out.trace_sec.push_back(now_s() - t0);
  };
  if (bnorm == 0.0) {
    out.converged = true;
    sample(0, 0.0, 0.0);
    out.seconds = now_s() - t0;
    return out;
  }
  sample(0, 1.0, track_true ? 1.0 : -1.0);
  launch_copy(r.p, d_b, n, s);
  precond(r.p, z.p);
  dot(r.p, z.p, 0);
  double h[4];
  fetch(h, 0, 1);
  if (!std::isfinite(h[0])) throw std::runtime_error("preconditioner produced non-finite values");
  if (h[0] < 0.0) throw std::runtime_error("preconditioner is not positive definite: r' M^-1 r < 0");
  launch_copy(p.p, z.p, n, s);
  double rel = 1.0;
  for (int64_t itn = 1; itn <= maxit; ++itn) {
    matvec_device(A, p.p, q.p, s);
    dot(p.p, q.p, 2);
    launch_axpy(d_x, p.p, sc.p + 0, sc.p + 2, 1.0, n, s);
    launch_axpy(r.p, q.p, sc.p + 0, sc.p + 2, -1.0, n, s);
    dot(r.p, r.p, 3);
    fetch(h, 0, 4);
    if (!std::isfinite(h[2]) || h[2] <= 0.0) throw std::runtime_error("operator is not positive definite: p' A p <= 0");
    rel = std::sqrt(h[3]) / bnorm;
    out.iterations = itn;
    sample(itn, rel, track_true ? true_resid(bnorm) : -1.0);
    if (rel <= tol) {
      out.converged = true;
      break;
    }
    precond(r.p, z.p);
    dot(r.p, z.p, 1);
    launch_pcg_update_p(p.p, z.p, sc.p + 1, sc.p + 0, n, s);
    CE_CUDA(cudaMemcpyAsync(sc.p + 0, sc.p + 1, sizeof(double), cudaMemcpyDeviceToDevice, s));
    double rzn = 0.0;
    fetch(&rzn, 1, 1);
    if (!std::isfinite(rzn)) throw std::runtime_error("preconditioner produced non-finite values");
    if (rzn < 0.0) throw std::runtime_error("preconditioner is not positive definite: r' M^-1 r < 0");
  }
  out.final_rec = rel;
  out.final_true = true_resid(bnorm);
  if (!out.trace_true.empty() && !track_true) out.trace_true.back() = out.final_true;
  CE_CUDA(cudaGetLastError());
  out.seconds = now_s() - t0;
  return out;
}

// MINRES (minres.cpp:22-115): Lanczos on the preconditioned operator with Givens QR of the
// tridiagonal; the vectors live on the device, the scalar recurrence runs on the host with
// the two inner products of each iteration fetched (one 8-byte read each).  Same stopping
// rules as the reference: recurrence <= tol, or a Lanczos beta below 1e-30 beta1 (exact
// solution); a negative / non-finite r' M^-1 r is an error (minres.cpp:11-18).
SolveOut minres_device(const Matrix& A, const Factor* M, const double* d_b, double* d_x, double tol, int64_t maxit,
                       bool track_true, cudaStream_t s) {
  const int64_t n = A.n;
  SolveOut out;
  const double t0 = now_s();
  DevArray<double> v(static_cast<size_t>(n)), ya(static_cast<size_t>(n)), r1a(static_cast<size_t>(n)),
      r2a(static_cast<size_t>(n)), wa(static_cast<size_t>(n)), w1a(static_cast<size_t>(n)), w2a(static_cast<size_t>(n)),
      tmp(static_cast<size_t>(n));
  DevArray<double> part(static_cast<size_t>(dot_partials_capacity())), sc(2);
  double *y = ya.p, *r1 = r1a.p, *r2 = r2a.p, *w = wa.p, *w1 = w1a.p, *w2 = w2a.p;
  auto dot = [&](const double* a, const double* b) {
    const int np = launch_dot(a, b, n, part.p, s);
    launch_sum_partials(part.p, np, sc.p, s);
    double h = 0.0;
    CE_CUDA(cudaMemcpyAsync(&h, sc.p, sizeof(double), cudaMemcpyDeviceToHost, s));
    CE_CUDA(cudaStreamSynchronize(s));
    return h;
  };
  auto checked_inner = [&](const double* r, const double* z) {  // minres.cpp:11-18
    const double h = dot(r, z);
    if (!std::isfinite(h)) throw std::runtime_error("preconditioner produced non-finite values");
    if (h < 0.0) throw std::runtime_error("preconditioner is not positive definite: r' M^-1 r < 0");
    return h;
  };
  auto precond = [&](const double* in, double* o) {
    if (M) apply_device(*M, in, o, s);
    else launch_copy(o, in, n, s);
  };
  auto true_resid = [&](double bnorm) {  // relative_residual (minres.cpp:117-122)
    matvec_device(A, d_x, tmp.p, s);
    launch_lincomb(tmp.p, d_b, tmp.p, 1.0, nullptr, 0.0, 1.0, n, s);  // b - A x
    return std::sqrt(dot(tmp.p, tmp.p)) / bnorm;
  };
  CE_CUDA(cudaMemsetAsync(d_x, 0, static_cast<size_t>(n) * sizeof(double), s));
  const double bnorm = std::sqrt(dot(d_b, d_b));
  auto sample = [&](int64_t it, double rec, double tru) {  // IterationSample (minres.hpp:12-20)
    out.trace_iter.push_back(it);
    out.trace_rec.push_back(rec);
    out.trace_true.push_back(tru);
    out.trace_sec.push_back(now_s() - t0);
  };
  if (bnorm == 0.0) {
    out.converged = true;
    sample(0, 0.0, 0.0);  // minres.cpp:32-36
    out.seconds = now_s() - t0;
    return out;
  }
  launch_copy(r1, d_b, n, s);
  precond(d_b, y);
  double beta1 = checked_inner(r1, y);
  if (beta1 == 0.0) {  // minres.cpp:43-47: report left at its defaults
    out.converged = true;
    sample(0, 0.0, 1.0);
    out.seconds = now_s() - t0;
    return out;
  }
  beta1 = std::sqrt(beta1);
  sample(0, 1.0, track_true ? 1.0 : -1.0);  // minres.cpp:55
  double oldb = 0.0, beta = beta1, dbar = 0.0, epsln = 0.0, qrnorm = beta1, phibar = beta1, cs = -1.0, sn = 0.0;
  launch_copy(r2, r1, n, s);
  CE_CUDA(cudaMemsetAsync(w, 0, static_cast<size_t>(n) * sizeof(double), s));
  CE_CUDA(cudaMemsetAsync(w2, 0, static_cast<size_t>(n) * sizeof(double), s));
  const double tiny = 1e-290;
  for (int64_t itn = 1; itn <= maxit; ++itn) {
    launch_scale(v.p, 1.0 / beta, y, false, n, s);                              // v = y / beta
    matvec_device(A, v.p, y, s);                                                 // y = A v
    if (itn >= 2) launch_lincomb(y, y, r1, beta / oldb, nullptr, 0.0, 1.0, n, s);  // y -= (beta/oldb) r1
    const double alfa = dot(v.p, y);
    launch_lincomb(y, y, r2, alfa / beta, nullptr, 0.0, 1.0, n, s);             // y -= (alfa/beta) r2
    std::swap(r1, r2);  // r1 = r2
    std::swap(r2, y);   // r2 = y (the old r1 buffer becomes the next y)
    precond(r2, y);
    oldb = beta;
    beta = std::sqrt(checked_inner(r2, y));
    const double oldeps = epsln;
    const double delta = cs * dbar + sn * alfa;
    const double gbar = sn * dbar - cs * alfa;
    epsln = sn * beta;
    dbar = -cs * beta;
    double gamma = std::sqrt(gbar * gbar + beta * beta);
    gamma = std::max(gamma, tiny);
    cs = gbar / gamma;
    sn = beta / gamma;
    const double phi = cs * phibar;
    phibar = sn * phibar;
    // w1 = w2, w2 = w, w = (v - oldeps w1 - delta w2) / gamma; x += phi w
    std::swap(w1, w2);  // w1 = old w2
    std::swap(w2, w);   // w2 = old w; w = old w1 buffer (overwritten)
    launch_lincomb(w, v.p, w1, oldeps, w2, delta, gamma, n, s);
    launch_scale(d_x, phi, w, true, n, s);
    qrnorm = phibar;
    const double rec = qrnorm / beta1;
    out.iterations = itn;
    sample(itn, rec, track_true ? true_resid(bnorm) : -1.0);
    if (rec <= tol || beta / beta1 < 1e-30) {
      out.converged = true;
      break;
    }
  }
  out.final_rec = qrnorm / beta1;
  out.final_true = true_resid(bnorm);
  if (!out.trace_true.empty() && !track_true) out.trace_true.back() = out.final_true;
  CE_CUDA(cudaGetLastError());
  out.seconds = now_s() - t0;
  return out;
}

// ---------------------------------------------------------------- dump
void dump_factor(const Factor& f, const std::string& path) {
  std::FILE* fp = std::fopen(path.c_str(), "wb");
  if (!fp) throw std::runtime_error("cannot open " + path);
  auto i64 = [&](int64_t v) { std::fwrite(&v, sizeof v, 1, fp); };
  auto f64 = [&](const double* p, size_t k) {
    if (k) std::fwrite(p, sizeof(double), k, fp);
  };
  cudaStream_t s = f.ctx->stream;
  std::fwrite("CEFD", 1, 4, fp);
  i64(1);
  i64(f.n);
  i64(static_cast<int64_t>(f.levels.size()));
  i64(f.tail_dim);
  for (const LevelFactor& L : f.levels) {
    std::vector<double> basis, sigma, fac;
    L.d_basis.download(basis, s);
    L.d_sigma.download(sigma, s);
    L.d_fac.download(fac, s);
    CE_CUDA(cudaStreamSynchronize(s));
    i64(L.M);
    for (int64_t v : L.offsets) i64(v);
    for (int v : L.rank) i64(v);
    for (unsigned char v : L.has_basis) i64(v);
    for (int64_t b = 0; b < L.M; ++b)
      if (L.has_basis[static_cast<size_t>(b)]) {
        const int64_t bs = L.bsz[static_cast<size_t>(b)];
        f64(basis.data() + L.basis_off[static_cast<size_t>(b)], static_cast<size_t>(bs * bs));
      }
    for (int v : L.fcols) i64(v);
    for (int v : L.nsig) i64(v);
    for (int64_t b = 0; b < L.M; ++b) f64(sigma.data() + L.sigma_off[static_cast<size_t>(b)], static_cast<size_t>(L.nsig[static_cast<size_t>(b)]));
    for (int64_t b = 0; b < L.M; ++b) {
      const int64_t w = L.width[static_cast<size_t>(b)], r = L.rank[static_cast<size_t>(b)];
      i64(w);
      if (w == 0) continue;
      f64(fac.data() + L.chol_off[static_cast<size_t>(b)], static_cast<size_t>(w * w));
      const double* G = fac.data() + L.g_off[static_cast<size_t>(b)];
      f64(G, static_cast<size_t>(r * w));
      const int64_t c0 = L.cptr[static_cast<size_t>(b)], c1 = L.cptr[static_cast<size_t>(b + 1)];
      i64(c1 - c0);
      for (int64_t e = c0; e < c1; ++e) {
        const int t = L.ccol[static_cast<size_t>(e)];
        i64(t);
        f64(G + (r + L.croff[static_cast<size_t>(e)]) * w, static_cast<size_t>(L.bsz[static_cast<size_t>(t)] * w));
      }
    }
    i64(static_cast<int64_t>(L.groups.size()));
    for (const auto& g : L.groups) {
      i64(static_cast<int64_t>(g.size()));
      for (int64_t b : g) i64(b);
    }
  }
  if (f.tail_dim > 0) {
    std::vector<double> t;
    f.d_tail_L.download(t, s);
    CE_CUDA(cudaStreamSynchronize(s));
    f64(t.data(), t.size());
  }
  std::fclose(fp);
}

}  // namespace ceg
