// Kernel argument blocks and launchers shared by the .cu files and the host driver.
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

namespace ceg {

#ifndef CE_SWEEP_THREADS
#define CE_SWEEP_THREADS 256  // threads per sweep CTA (A/B builds: scripts/build_variant.sh -DCE_SWEEP_THREADS=...)
#endif
constexpr int kSweepThreads = CE_SWEEP_THREADS;
constexpr int kApplyThreads = 128;
constexpr int kApplyWmax = 256;
#ifndef CE_APPLY_WARP_MAX_CLOSE
#define CE_APPLY_WARP_MAX_CLOSE 16  // warp apply items only for levels of short rows (<= this many neighbours)
#endif
#ifndef CE_APPLY_WARP_ROWS_PER_WAVE
#define CE_APPLY_WARP_ROWS_PER_WAVE 512  // ... that are throughput-bound (>= this many rows per sweep wave)
#endif
// Schur pairs per B task of a row with np panels (forced > 0, else adaptive): one pair per task
// while the row has few panels (the wave needs the parallelism: A/B on cfg2, g = 2 / 3 / 5 lose
// 4 / 8 / 20%), more once a row has hundreds of panels (3-D deep levels, each panel is staged
// once per pair otherwise).
#ifndef CE_PAIR_DIV
#define CE_PAIR_DIV 16  // panels per extra pair in a Schur task (A/B builds: -DCE_PAIR_DIV=...)
#endif
__host__ __device__ inline int row_pair_group(int forced, int np) {
  if (forced > 0) return forced;
  const int g = np / CE_PAIR_DIV;
  return g < 1 ? 1 : (g > 8 ? 8 : g);
}  // largest eliminated width per block the apply sweeps stage in shared memory

enum : int { kErrNone = 0, kErrBreakdown = 2, kErrPattern = 5, kErrInternal = 6, kErrChunk = 7, kErrStrip = 8, kErrNaN = 9 };

// validate (factorization.cpp:272-334), device half: basis orthogonality and lower-triangular
// pivots of one level; d_out = {max |U^T U - I| as double bits, upper nonzeros, first bad block}.
void launch_validate_level(int64_t M, const int* bsz, const unsigned char* has_basis, const double* basis,
                           const int64_t* basis_off, const int* width, const double* fac, const int64_t* chol_off,
                           double tol, unsigned long long* d_out, cudaStream_t s);

// Sharded factorization exchange (shard.cu): 2-D segments <-> a contiguous buffer, per-row
// integers <-> 5 doubles per row, and completion of the rows another rank swept.
void launch_segments(double* base, double* buf, const int64_t* off, const int* rows, const int* cols, const int* ld,
                     const int64_t* boff, int64_t nseg, bool to_buf, cudaStream_t s);
void launch_row_ints(const int* rows, int64_t n, int* rank, int* width, unsigned char* has_basis, int* fcols, int* nsig,
                     double* buf, bool to_buf, cudaStream_t s);
void launch_precomplete(const int* rows, int64_t n, const int* target, const int64_t* pan_ptr, int* done, int* pdone,
                        int* bready, cudaStream_t s);

// Launch accounting (every launcher calls note_launch once per kernel launch).
void note_launch(int64_t n = 1);
int64_t launch_count();

// One level sweep: rows are compressed and
// eliminated by a persistent kernel that walks the plan's ascending order as
// a dependency DAG (row j waits for every i < j in sq(j), A.2).
struct SweepArgs {
  int64_t M;
  int level;
  const int* bsz;
  const int64_t* sq_ptr;
  const int* sq_col;
  const int64_t* sq_slot;
  const unsigned char* sq_kind;
  const int64_t* slot_off;
  const int64_t* tri_off;  // dense lower-triangular (t, s) -> value offset table (-1: not stored), or null
  double* store;
  const int64_t* cl_ptr;
  const int* cl_col;
  const int* cl_roff;
  const int64_t* cl_slot;  // stored slot of (i, t) per close entry
  int* rank;
  int* width;
  unsigned char* has_basis;
  int* fcols;
  int* nsig;
  double* basis;
  const int64_t* basis_off;
  double* sigma;
  const int64_t* sigma_off;
  double* fac;
  const int64_t* chol_off;
  const int64_t* g_off;
  const int64_t* item_start;  // first item of the row at each position of `order`
  const int* order;           // rows in wave order
  const int* item_row;        // ticket -> row
  const int* item_part;       // ticket -> task index within the row
  const int* nA1;             // TSQR tree tasks per row (0 = gather inside A2): leaves, then combine levels
  const int* nleaf;           // TSQR tree leaves per row
  const int* nA3;             // strip tasks per row (0 = strip inside A2)
  const int* nB;              // Schur panel-pair tasks per row (0 = inline)
  const int64_t* fsum;        // far columns per row
  const int64_t* rs_off;      // per-row offset of the TSQR leaf triangles in rscratch
  double* rscratch;
  int* nzflag;                // per-row "far fill nonzero" flag from the leaves
  const int64_t* pan_ptr;     // per-row offset into pan_start (np + 1 entries per row)
  const int* pan_start;       // close-list index where each Schur panel starts
  const int64_t* sq_boff;     // per sq entry: value offset of the stored block
  const int* sq_bsz;          // per sq entry: block size of the column block
  const int* sq_roff;         // per sq entry: row offset in the close list (-1: not close)
  const int64_t* sq_diag;     // per row: sq entry of the diagonal block
  const int* target;          // per row: number of items (done[] value when the row is finished)
  const int* sq_pan;          // per sq entry (j, i < j) close: panel of j in close(i), -1: wait for all of i
  int* pdone;                 // per (row, panel) (pan_ptr index): finished Schur pairs touching the panel
  int* bready;                // per row: every predecessor finished (set by the row's first Schur task)
  const int64_t* leaf_ptr;    // per row: range into leaf_e (nA1 + 1 entries)
  const int64_t* leaf_e;      // first sq entry of each TSQR leaf (last = row end)
  const int64_t* strip_ptr;   // per row: range into strip_e (nA3 + 1 entries)
  const int64_t* strip_e;     // first sq entry of each strip task (last = row end)
  int* done;
  unsigned long long* ticket;
  int64_t n_items;
  const int* forced;  // nullptr or M entries (-1 = free)
  int mode;           // 0 eps, 1 fixed rank
  int absolute;
  double eps;
  int fixed_rank;
  int pair_group;             // Schur pairs (P, Q..Q+pair_group-1) per B task
  int* err;           // [0] code, [1] level, [2] row (low), [3] row (high)
  int* shifts;
  int bmax;
  int kcap;
  double* scratch;    // per-CTA global scratch when the tiles do not fit shared memory
  int64_t scratch_per_cta;
  int use_global_scratch;
  int dbg;  // CE_DBG bitmask (development): 1 generic TSQR, 2 generic Jacobi
  unsigned long long* prof;  // CE_PROFILE=1: per-stage SM-cycle counters (kProf*), else nullptr
  unsigned long long* trace; // CE_TRACE=<level>: per item {claim, run, end (globaltimer ns), smid}, else nullptr
};

// Cycle counters of the sweep kernel (CE_PROFILE=1).
enum : int {
  kProfWait = 0, kProfA1, kProfA2, kProfA2Tsqr, kProfA2Svd, kProfA2Basis, kProfA2Pivot, kProfA2Strip,
  kProfA2Panels, kProfA3, kProfB, kProfNA1, kProfNA2, kProfNA3, kProfNB, kProfSvdPre, kProfSvdJac, kProfSvdPost,
  kProfSweeps, kProfSvds, kProfBSetup, kProfBStage, kProfBTiles, kProfCount
};

// smem doubles needed by one sweep CTA for a level
int64_t sweep_smem_doubles(int bmax, int kcap);
// Largest block the level sweep accepts: the Schur panels hold whole neighbours in kPanelRows
// (260) compacted rows (sweep.cu), the chunk maps / cluster table are static shared arrays of this
// size, and the apply sweeps stage kApplyWmax = 256 eliminated columns.  The driver rejects larger
// levels with an error instead of overrunning them.  (Round 1 accepted 512 here, which the panel
// tables did not cover: a neighbour with more than 260 live rows overran them.)
#ifndef CE_SWEEP_BLOCK_MAX
#define CE_SWEEP_BLOCK_MAX 256
#endif
static_assert(CE_SWEEP_BLOCK_MAX <= 256, "Schur panel tables (kPanelRows) hold at most 256 + 4 rows per neighbour");
constexpr int kSweepBlockMax = CE_SWEEP_BLOCK_MAX;
int sweep_kcap(int bmax);  // F^T chunk height for a level
void launch_sweep(const SweepArgs& a, int grid, size_t smem_bytes, cudaStream_t s);
int sweep_max_ctas_per_sm(size_t smem_bytes);

// Deferred pending-factor rotations g <- U_t^T g (level_matrix.cpp:66-69 deferred, A.2).
void launch_pending_rotation(const SweepArgs& a, cudaStream_t s);

// Level-1 store initialisation: scatter the lower blocks of A into the squared-pattern store.
void launch_init_store_from_matrix(int64_t M, const int* bsz, const int64_t* a_row_ptr, const int* a_col,
                                   const int64_t* a_val_ptr, const double* a_values, const int64_t* sq_ptr,
                                   const int* sq_col, const int64_t* sq_slot, const int64_t* slot_off,
                                   double* store, cudaStream_t s);

// Remainder extraction straight into the next level's store (level_matrix.cpp:185-248).
struct RemainderArgs {
  int64_t M;
  const int* bsz;
  const int* rank;
  const int64_t* sq_ptr;
  const int* sq_col;
  const int64_t* sq_slot;
  const int64_t* slot_off;
  const double* store;
  const int* next_block;  // current block -> next block (-1 if dead)
  const int* next_loc;    // local offset inside the super block
  const int* nbsz;        // next block sizes
  const int64_t* nsq_ptr;
  const int* nsq_col;
  const int64_t* nsq_slot;
  const int64_t* nslot_off;
  double* nstore;
  int* err;
};
void launch_remainder(const RemainderArgs& a, cudaStream_t s);
// dense lower-triangular (t, s) -> value offset table of the squared pattern (for small M)
void launch_tri_table(int64_t M, const int64_t* sq_ptr, const int* sq_col, const int64_t* sq_slot,
                      const int64_t* slot_off, int64_t* tab, cudaStream_t s);

// Dense tail (factorization.cpp:419-436): densify the last store, Cholesky, inverse.
void launch_densify(int64_t M, const int* bsz, const int64_t* offsets, const int64_t* sq_ptr, const int* sq_col,
                    const int64_t* sq_slot, const int64_t* slot_off, const double* store, double* dense, int64_t n,
                    cudaStream_t s);
// In-place blocked lower Cholesky of the n x n row-major matrix; *fail set to 1 on a non-positive pivot.
void dense_cholesky(double* a, int64_t n, int* d_fail, cudaStream_t s);
void dense_add_shift(double* a, int64_t n, double shift, cudaStream_t s);
void dense_trace(const double* a, int64_t n, double* d_out, cudaStream_t s);
// Linv = L^{-1} (lower), row-major n x n.
void dense_tri_inverse(const double* L, double* Linv, int64_t n, cudaStream_t s);

// ---- apply (CEFactorization::solve, factorization.cpp:140-168) ----
struct ApplyLevelArgs {
  int64_t M;
  const int* bsz;
  const int64_t* offsets;
  const int* rank;
  const int* width;
  const unsigned char* has_basis;
  const double* basis;
  const int64_t* basis_off;
  const double* fac;
  const int64_t* chol_off;
  const int64_t* g_off;
  const int64_t* cl_ptr;
  const int* cl_col;
  const int* cl_roff;
  double* v;
  int* flags;
  const int* order;  // sweep order (wave order of the forward / backward DAG)
  unsigned long long* ticket;
  // host-built pull lists (no close-list searches on the device)
  const int64_t* in_ptr;    // per row j: range of its contributing close neighbours i (w_i > 0), ascending i
  const int* in_split;      // per row j: number of those with i < j (the forward sweep's dependencies)
  const int* in_src;        // i
  const int64_t* in_goff;   // fac offset of g_{i->j} (b_j rows x w_i)
  const int* in_w;          // w_i
  const int64_t* in_uoff;   // v offset of u_i (offsets[i] + r_i)
  const int64_t* dep_ptr;   // per row j: backward-sweep dependencies t > j (w_t > 0)
  const int* dep_t;
  const int* cl_nt;         // per close entry (j, t): rows of v_t read by the backward pull
  const double* linv;       // per row: L^{-1} (w x w, row-major, lower)
  const int64_t* linv_off;
  // split-row task graph of the sweeps: items (row, part) in wave order; part < P_j is a
  // partial pull over a slice of the row's inputs, part == P_j the row's finalize
  const int* item_row;
  const int* item_part;
  int64_t n_items;
  const int64_t* part_ptr;  // per row: range into part_b (P_j + 1 boundaries)
  const int64_t* part_b;    // slice boundaries (forward: in_* entries; backward: segments)
  const int64_t* scr_off;   // per row: offset of its P_j x w partial sums in scratch
  double* scratch;
  int* parts_done;          // per row: finished partial tasks
};
// L^{-1} of every row's pivot factor (apply sweeps multiply instead of substituting).
void launch_pivot_inverse(int64_t M, const int* width, const double* fac, const int64_t* chol_off, double* linv,
                          const int64_t* linv_off, cudaStream_t s);
void launch_basis_apply(const ApplyLevelArgs& a, int transpose, cudaStream_t s);
void launch_forward_sweep(const ApplyLevelArgs& a, int grid, cudaStream_t s);
// warp_items: every warp an independent worker (levels of short rows: the sweep is a latency
// chain and CTA barriers sit on it); else one 4-warp CTA per item (levels of long rows).
void launch_forward_tasks(const ApplyLevelArgs& a, int grid, bool warp_items, cudaStream_t s);
void launch_backward_tasks(const ApplyLevelArgs& a, int grid, bool warp_items, cudaStream_t s);
void launch_forward_retained(const ApplyLevelArgs& a, cudaStream_t s);
void launch_backward_sweep(const ApplyLevelArgs& a, int grid, cudaStream_t s);
// operator tool (apply_operator) pieces
void launch_operator_forward(const ApplyLevelArgs& a, const int64_t* elim_off, double* c, cudaStream_t s);
void launch_operator_backward(const ApplyLevelArgs& a, const int64_t* elim_off, const double* c, cudaStream_t s);
void launch_gather(const double* src, const int64_t* idx, double* dst, int64_t n, cudaStream_t s);
void launch_scatter(const double* src, const int64_t* idx, double* dst, int64_t n, cudaStream_t s);
// y = op(L) x with the dense lower matrix: trans 0 -> y = L x, 1 -> y = L^T x
void launch_dense_trmv(const double* L, const double* x, double* y, int64_t n, int trans, cudaStream_t s);

// ---- Krylov helpers ----
void launch_bsr_matvec(int64_t n, const int64_t* row_of, const int64_t* offsets, const int* bsz,
                       const int64_t* row_ptr, const int* col_idx, const int64_t* val_ptr, const double* values,
                       const double* x, double* y, cudaStream_t s);
// partial dot products -> d_partial[nblocks]; returns nblocks used
int launch_dot(const double* x, const double* y, int64_t n, double* d_partial, cudaStream_t s);
int dot_partials_capacity();
void launch_sum_partials(const double* partial, int np, double* out, cudaStream_t s);
void launch_axpy(double* y, const double* x, const double* alpha_num, const double* alpha_den, double sign,
                 int64_t n, cudaStream_t s);
void launch_pcg_update_p(double* p, const double* z, const double* rz_new, const double* rz_old, int64_t n,
                         cudaStream_t s);
void launch_copy(double* dst, const double* src, int64_t n, cudaStream_t s);
// MINRES vector steps with host scalars: out = (x - a y - c z) / g (y, z may be null); out (+)= sc x
void launch_lincomb(double* out, const double* x, const double* y, double a, const double* z, double c, double g,
                    int64_t n, cudaStream_t s);
void launch_scale(double* out, double sc, const double* x, bool accumulate, int64_t n, cudaStream_t s);

}  // namespace ceg
