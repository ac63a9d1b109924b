// Internal host-side structures of the CE B200 library (not part of the C ABI).
#pragma once

#include <cstdint>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>

namespace ceg {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// BreakdownError{level, block} of the reference (proj/include/ce/types.hpp:26-36).
struct Breakdown : std::runtime_error {
  Breakdown(int lvl, int64_t blk, const std::string& w) : std::runtime_error(w), level(lvl), block(blk) {}
  int level;
  int64_t block;
};

void cuda_check(cudaError_t e, const char* what);
#define CE_CUDA(x) ::ceg::cuda_check((x), #x)

// Caching device allocator: blocks are kept per device on release and reused by later
// allocations of a similar size (a factorization allocates the same large arrays every
// time; cudaMalloc/cudaFree would otherwise add host stalls and implicit device syncs
// between levels).  Releases happen only after the owning stream has drained.
void* pool_alloc(size_t bytes);
void pool_free(void* p, size_t bytes);
void pool_trim(int device = -1);  // return the cached blocks of `device` (-1: all) to the driver

// Owning device array.
template <class T>
struct DevArray {
  T* p = nullptr;
  size_t n = 0;
  bool view = false;  // p points into another allocation (set_view): never freed here
  DevArray() = default;
  explicit DevArray(size_t count) { alloc(count); }
  DevArray(const DevArray&) = delete;
  DevArray& operator=(const DevArray&) = delete;
  DevArray(DevArray&& o) noexcept : p(o.p), n(o.n), view(o.view) { o.p = nullptr; o.n = 0; o.view = false; }
  DevArray& operator=(DevArray&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      n = o.n;
      view = o.view;
      o.p = nullptr;
      o.n = 0;
      o.view = false;
    }
    return *this;
  }
  ~DevArray() { release(); }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) p = static_cast<T*>(pool_alloc(count * sizeof(T)));
  }
  void release() {
    if (p && !view) pool_free(p, n * sizeof(T));
    p = nullptr;
    n = 0;
    view = false;
  }
  // non-owning window into a larger device allocation (the level plan's arena)
  void set_view(void* ptr, size_t count) {
    release();
    p = count ? static_cast<T*>(ptr) : nullptr;
    n = count;
    view = count != 0;
  }
  void upload(const std::vector<T>& h, cudaStream_t s) {
    alloc(h.size());
    if (!h.empty()) CE_CUDA(cudaMemcpyAsync(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  void download(std::vector<T>& h, cudaStream_t s) const {
    h.resize(n);
    if (n) CE_CUDA(cudaMemcpyAsync(h.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost, s));
  }
  void zero(cudaStream_t s) {
    if (n) CE_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
};

// BASELINE problem (host CSB, plan, rhs).
struct Problem {
  int cfg = 0;
  int64_t nx = 0, ny = 0, nz = 1, block = 8;
  double eps = 1e-6, tol = 1e-8;
  int64_t n = 0, m = 0;
  std::vector<int64_t> offsets, row_ptr, col_idx, val_ptr, perm;
  std::vector<double> values, rhs;
  int64_t join = 2;
  std::vector<int64_t> plan_level_blocks, plan_assign;
  std::vector<int64_t> box_of_block;  // CE_PLAN_SHARDED: subdomain (box) of every level-1 block
  void build(int cfg_id, int64_t nx, int64_t ny, int64_t nz, int plan_kind = 0);  // CE_PLAN_*
  // reference `file` problems (io.cpp): matrix.mtx + optional plan.txt / rhs.txt
  void load(const char* matrix_path, const char* plan_path, const char* rhs_path, int64_t block);
  void save(const char* matrix_path, const char* plan_path, const char* rhs_path) const;
};

// CE_PLAN_SHARDED geometry (problem.cpp): 8 boxes; box of cell q of grid g, interior flag.
constexpr int64_t kShardBoxes = 8;
int64_t shard_box(const int64_t* g, int64_t q, int dims, bool* interior);

// Subdomain-sharded factorization (ce_factorize_sharded): this rank's index, the
// rank count, the box label of every level-1 block (box -> owner rank box * n_ranks / n_boxes)
// and the in-place device broadcast every rank calls in the same order.
struct ShardSpec {
  int rank = 0, n_ranks = 1;
  int64_t n_boxes = 0;
  std::vector<int64_t> box_l1;
  int (*bcast)(void* user, void* dev_ptr, int64_t bytes, int root) = nullptr;
  void* user = nullptr;
  int owner(int64_t box) const { return static_cast<int>(box * n_ranks / n_boxes); }
};

// Per-factorization sharding statistics (LevelStats-like, host-side).
struct ShardStats {
  int64_t phase1_rows = 0, phase3_rows = 0, own_rows = 0;
  double exchange_bytes = 0.0, exchange_seconds = 0.0;
};

struct Context {
  int device = 0;
  int sm_count = 0;
  cudaStream_t stream = nullptr;
};

// Device-resident operator A (both triangles, BSR) + host copy of its structure.
struct Matrix {
  Context* ctx = nullptr;
  int64_t n = 0, m = 0, nnzb = 0;
  std::vector<int64_t> offsets, row_ptr, col_idx, val_ptr;
  DevArray<int64_t> d_offsets, d_row_ptr, d_val_ptr;
  DevArray<int> d_col_idx, d_bsz;
  DevArray<double> d_values;
  DevArray<int64_t> d_row_of;  // scalar row -> block row
};

// Symbolic plan of one level (host) — SURVEY.md §8a a3/a7: squared pattern,
// half-symmetric slot layout, close/far split, factor layout, schedule.
struct LevelPlan {
  int64_t M = 0, dim = 0;
  std::vector<int> bsz;
  std::vector<int64_t> offsets;
  std::vector<int64_t> bptr;  // base pattern CSR (both triangles, sorted, with diagonal)
  std::vector<int> bcol;
  std::vector<int64_t> sptr;  // squared pattern CSR
  std::vector<int> scol;
  std::vector<unsigned char> skind;  // 0 diag, 1 close, 2 far
  std::vector<int64_t> sslot;        // stored (lower) slot of (i, j)
  int64_t nslots = 0;
  std::vector<int64_t> slot_off;     // value offset (doubles) of each stored slot
  int64_t store_doubles = 0;
  std::vector<int64_t> cptr;         // close lists (base minus diagonal)
  std::vector<int> ccol, croff;
  std::vector<int64_t> csum;         // sum of close block sizes per row
  std::vector<int64_t> fsum;         // far columns per row
  std::vector<int64_t> chol_off, g_off, basis_off, sigma_off;
  int64_t fac_doubles = 0, basis_doubles = 0, sigma_doubles = 0;
  std::vector<int64_t> item_start;   // by position in `order`
  std::vector<int> order;            // rows in wave (topological) order of the sq-DAG
  std::vector<int64_t> wave;         // wave index of every row
  std::vector<int> item_row, item_part;  // ticket -> (row, task index within the row)
  std::vector<std::vector<int>> rest_of, urg_of;  // per row: Schur pair tasks after / with the next wave
  std::vector<int> nA1, nA3, nB;     // per-row task counts (sweep.cu header)
  std::vector<int> nleaf;            // per-row TSQR tree leaves (nA1 = all tree nodes)
  std::vector<int64_t> pan_ptr, rs_off;
  std::vector<int> pan_start;
  int64_t rscratch_doubles = 0;
  std::vector<int64_t> sboff;        // per sq entry: value offset of its stored block
  std::vector<int> sbsz, sroff;      // per sq entry: block size, close-list row offset (-1: not close)
  std::vector<int64_t> sdiag;        // per row: sq entry of the diagonal
  std::vector<int> target;           // per row: items of the row (completion count)
  std::vector<int> sq_pan;           // per sq entry (j, i), i < j close: panel of j in close(i)
                                     // (-1: far, or i's Schur runs in <= 1 task -> wait for all of i)
  std::vector<int64_t> leaf_ptr, leaf_e, strip_ptr, strip_e;  // A1 / A3 task entry ranges
  int64_t n_items = 0, n_waves = 0;
  int bmax = 0;
  int64_t fmax = 0, cmax = 0;
  int64_t lower_blocks = 0;          // of the base pattern (LevelStats.pattern_blocks)
};

// Persistent device data of one completed level (FactorLevel, factorization.hpp:19-36).
struct LevelFactor {
  int64_t M = 0, dim = 0, n_elim = 0, n_kept = 0;
  std::vector<int> bsz, rank, width;
  std::vector<int64_t> offsets;
  std::vector<unsigned char> has_basis;
  std::vector<int64_t> cptr, chol_off, g_off, basis_off, sigma_off;
  std::vector<int> ccol, croff, fcols, nsig;
  std::vector<std::vector<int64_t>> groups;
  DevArray<int> d_bsz, d_rank, d_width, d_ccol, d_croff, d_nsig, d_fcols;
  DevArray<int64_t> d_offsets, d_cptr, d_chol_off, d_g_off, d_basis_off, d_sigma_off;
  DevArray<unsigned char> d_has_basis;
  DevArray<double> d_fac, d_basis, d_sigma;
  DevArray<int64_t> d_elim_gather, d_kept_gather;
  DevArray<int> d_fwd_order, d_bwd_order;
  // apply pull lists (apply.cu) and pivot inverses
  DevArray<int64_t> d_in_ptr, d_in_goff, d_in_uoff, d_dep_ptr, d_linv_off;
  DevArray<int> d_in_split, d_in_src, d_in_w, d_dep_t, d_cl_nt;
  DevArray<double> d_linv;
  // split-row task graphs of the apply sweeps (forward f / backward b)
  DevArray<int64_t> d_fpart_ptr, d_fpart_b, d_fscr_off, d_bpart_ptr, d_bpart_b, d_bscr_off;
  DevArray<int> d_fitem_row, d_fitem_part, d_bitem_row, d_bitem_part;
  int64_t n_fitems = 0, n_bitems = 0, scratch_doubles = 0;
  // stats
  int64_t pattern_blocks = 0, shift_retries = 0, max_far = 0, max_close = 0, n_waves = 0, n_items = 0;
  double seconds = 0.0, sweep_seconds = 0.0, alg_bytes = 0.0, alg_flops = 0.0;
};

struct Factor {
  Context* ctx = nullptr;
  int64_t n = 0;
  std::vector<LevelFactor> levels;
  int64_t tail_dim = 0;
  DevArray<double> d_tail_L, d_tail_Linv;
  int64_t shift_retries = 0;
  double total_seconds = 0.0, device_seconds = 0.0, sweep_seconds = 0.0;
  double validate_seconds = 0.0, max_orth_error = 0.0;  // validate(), factorization.cpp:272-334
  ShardStats shard;                                       // zero unless ce_factorize_sharded
  double apply_alg_bytes = 0.0;  // SURVEY.md §8d apply byte count (forward + backward + vector passes)
  double factor_blocks = 0.0, predicted_factor_blocks = 0.0;
  int64_t l_scalar_nnz = 0, l_payload_bytes = 0, q_payload_bytes = 0, tail_bytes = 0;
  // apply workspaces (sized to the level dims)
  mutable DevArray<double> w_v, w_active, w_elim;
  mutable std::vector<int64_t> elim_base;
  mutable DevArray<int> w_flags;
  mutable DevArray<unsigned long long> w_ticket;
  mutable DevArray<double> w_scratch;  // apply partial sums
  mutable DevArray<int> w_parts;       // apply per-row finished partial tasks
  mutable DevArray<double> w_host_stage;
  // The apply workspaces above are shared by every apply on this factor.  Applies are
  // serialised: `apply_mu` orders their enqueue on the host and each apply's stream waits
  // for `apply_done`, recorded by the previous apply (any stream), before touching them.
  mutable std::mutex apply_mu;
  mutable cudaEvent_t apply_done = nullptr;
  Factor() = default;
  Factor(const Factor&) = delete;
  Factor& operator=(const Factor&) = delete;
  ~Factor() {
    if (apply_done) cudaEventDestroy(apply_done);
  }
};

}  // namespace ceg
