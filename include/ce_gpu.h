/* ce_gpu.h — C-ABI of the B200-native compress-and-eliminate (CE) hot path.
 *
 * Drop-in boundary for the reference's public header set proj/include/ce/
 * (SURVEY.md §8b).  Every entry point names the reference interface it
 * replaces.  Plain pointers and sizes only; no exceptions cross the ABI.
 * Return codes equal the reference CLI exit codes (proj/include/ce/cli.hpp:16-19):
 *   CE_OK 0, CE_EUSAGE 1 (usage / IO / invalid argument / CUDA failure),
 *   CE_EBREAKDOWN 2 (BreakdownError, proj/include/ce/types.hpp:26-36),
 *   CE_ENOCONV 3 (Krylov non-convergence).
 * The factor is device-resident and opaque.  There is no CPU fallback: every
 * compute entry point fails with CE_EUSAGE when no sm_100 device is present.
 */
#ifndef CE_GPU_H
#define CE_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CE_OK 0
#define CE_EUSAGE 1
#define CE_EBREAKDOWN 2
#define CE_ENOCONV 3

typedef struct ce_ctx ce_ctx;
typedef struct ce_matrix ce_matrix;
typedef struct ce_factor ce_factor;
typedef struct ce_problem ce_problem;

/* Host CSB matrix: the reference BlockSparseMatrix (proj/include/ce/block_matrix.hpp:23-63):
 * a BlockPartition (m+1 offsets), a structurally symmetric BlockSparsityPattern with full
 * diagonal (CSR over block rows, both triangles, sorted columns) and one dense row-major
 * block per pattern slot (values[val_ptr[k] ...], b_i x b_j). */
typedef struct {
  int64_t n;                /* scalar dimension */
  int64_t m;                /* block count */
  const int64_t* offsets;   /* m + 1 */
  const int64_t* row_ptr;   /* m + 1 */
  const int64_t* col_idx;   /* nnzb */
  const int64_t* val_ptr;   /* nnzb + 1 */
  const double* values;
} ce_csb_host;

/* Host CoarseningPlan (proj/include/ce/problems.hpp:51-65): per plan level, the block -> group
 * assignment (the reference's plan text format, problems.cpp:114-136).  The initial permutation
 * is applied by the caller before assembling the CSB (cli.cpp:49-58), so it is not needed here. */
typedef struct {
  int64_t join;               /* J used once the plan levels are exhausted (factorization.cpp:18-26) */
  int64_t n_levels;
  const int64_t* level_blocks;  /* n_levels: blocks at each plan level */
  const int64_t* assign;        /* concatenated assignments, sum(level_blocks) entries */
} ce_plan_host;

/* CompressionStrategy (proj/include/ce/compression.hpp:15-38). mode 0 = AdaptiveEps, 1 = FixedRank. */
typedef struct {
  int mode;
  double eps;
  int absolute;
  int64_t rank;
} ce_strategy;

/* FactorOptions (proj/include/ce/factorization.hpp:74-77) + parity hook: forced ranks per
 * (level, row), -1 = free (SURVEY.md §8c "--force-ranks"). */
typedef struct {
  int64_t dense_threshold;    /* default 2048 */
  int64_t max_levels;         /* default 64 */
  int64_t n_forced_levels;
  const int64_t* forced_counts;
  const int64_t* forced;      /* concatenated */
} ce_factor_opts;

/* Error context: BreakdownError{level, block} (types.hpp:26-36), block = -1 for the dense tail. */
typedef struct {
  int code;
  int level;
  int64_t block;
  int64_t shift_retries;
  char message[256];
} ce_status;

/* MinresOptions-shaped PCG options (proj/include/ce/minres.hpp:34-38). */
typedef struct {
  double tol;
  int64_t maxit;
  int track_true_residual;
} ce_pcg_opts;

/* SolveReport (proj/include/ce/minres.hpp:25-31). */
typedef struct {
  int converged;
  int64_t iterations;
  double final_recurrence_residual;
  double final_true_residual;
  double seconds;
} ce_solve_report;

/* FactorStats summary (proj/include/ce/factorization.hpp:56-72). */
typedef struct {
  int64_t n_levels;
  int64_t tail_dim;
  double factor_blocks;
  double predicted_factor_blocks;
  int64_t l_scalar_nnz;
  int64_t l_payload_bytes;
  int64_t q_payload_bytes;
  int64_t tail_bytes;
  int64_t shift_retries;
  double total_seconds;         /* host wall time of ce_factorize */
  double device_seconds;        /* CUDA-event time of the device work */
  double sweep_kernel_seconds;  /* CUDA-event time of the level sweep kernels */
  double algorithmic_bytes;     /* SURVEY.md §8d per-row byte contract, summed */
  double algorithmic_flops;     /* SURVEY.md §8d per-row flop contract, summed */
  double validate_seconds;      /* validate() inside ce_factorize (factorization.cpp:272-334,459) */
  double max_orth_error;        /* max |U^T U - I| over every stored basis (validate bound 1e-12) */
  double apply_algorithmic_bytes;  /* SURVEY.md §8d bytes of one preconditioner apply (ce_apply_precond) */
  int64_t shard_phase1_rows;    /* sharded factorizations: box-interior rows over all levels */
  int64_t shard_own_rows;       /* ... of which this rank swept */
  int64_t shard_phase3_rows;    /* interface rows (swept by every rank) */
  double shard_exchange_bytes;  /* bytes this rank packed / received in the exchanges */
  double shard_exchange_seconds;
} ce_factor_stats;

/* LevelStats (factorization.hpp:38-54) for level l (0-based). */
typedef struct {
  int64_t block_count, pattern_blocks, factor_blocks, eliminated, retained, max_rank;
  double mean_rank;
  double seconds;              /* CUDA-event time of the level's device work */
  int64_t l_bytes, q_bytes, shift_retries;
  int64_t max_block, max_far_cols, max_close;
  double sweep_seconds;        /* CUDA-event time of the sweep kernel alone */
  double algorithmic_bytes, algorithmic_flops;
  int64_t n_waves;             /* depth of the row dependency DAG */
  int64_t n_items;             /* work items of the persistent sweep (rows + Schur tiles) */
} ce_level_stats;

/* ---- context / device ---- */
int ce_ctx_create(int device, ce_ctx** out);
void ce_ctx_destroy(ce_ctx* ctx);
const char* ce_last_error(void);
/* Number of sm_100 devices visible (0 when none). */
int ce_device_count(void);
/* The context's CUDA stream (cudaStream_t), for event timing by the caller. */
int ce_ctx_stream(const ce_ctx* ctx, void** stream);
/* Kernels launched by this library since it was loaded (launch accounting for benchmarks). */
int64_t ce_launch_count(void);

/* ---- operator: BlockSparseMatrix on the device ---- */
/* Upload a host CSB (replaces BlockSparseMatrix construction, block_matrix.cpp:11-27). */
int ce_matrix_upload(ce_ctx* ctx, const ce_csb_host* a, ce_matrix** out);
/* BlockSparseMatrix::from_triplets (block_matrix.cpp:48-90) on the device: scalar COO triplets
 * (duplicates summed in input order, bit-identical to the reference's std::map accumulation),
 * mirror_lower != 0 = MirrorMode::Lower (the transposed entries are generated), else the input must
 * be symmetric to 1e-12 max|a|; every touched block is inserted symmetrically, plus the full
 * diagonal.  The values never leave the device; the block structure is kept on the host for the
 * planner.  on_device != 0: rows / cols / vals are device pointers.  Errors: CE_EUSAGE with the
 * reference's message ("triplet index outside matrix dimension", "asymmetric input: ..."). */
int ce_matrix_from_triplets(ce_ctx* ctx, int64_t n, int64_t nnz, const int64_t* rows, const int64_t* cols,
                            const double* vals, int64_t m, const int64_t* offsets, int mirror_lower, int on_device,
                            ce_matrix** out);
/* Symbolic planner pieces on the device, CSR patterns with sorted rows:
 * pattern_square (proj/src/pattern.cpp:64-86) and coarsen_pattern (pattern.cpp:97-118; group_of[b]
 * = -1 drops block b, as a dead group).  Outputs: rows + 1 row pointers and up to cap columns,
 * *nnz = the result's entry count (CE_EUSAGE if it exceeds cap).  ce_factorize uses them for the
 * plans it makes while the device is idle. */
int ce_pattern_square(ce_ctx* ctx, int64_t m, const int64_t* row_ptr, const int64_t* cols, int64_t* out_row_ptr,
                      int64_t* out_cols, int64_t cap, int64_t* nnz);
int ce_pattern_coarsen(ce_ctx* ctx, int64_t m, const int64_t* row_ptr, const int64_t* cols, int64_t ng,
                       const int64_t* group_of, int64_t* out_row_ptr, int64_t* out_cols, int64_t cap, int64_t* nnz);
/* The matrix's CSB: structure views (valid while the matrix lives; out->values = NULL) and, when
 * values != NULL, a copy of the block values (val_ptr[nnzb] doubles) into it. */
int ce_matrix_csb(const ce_matrix* a, ce_csb_host* out, double* values);
void ce_matrix_free(ce_matrix* a);
int64_t ce_matrix_dim(const ce_matrix* a);
/* y = A x (replaces BlockSparseMatrix::matvec, block_matrix.cpp:92-105; ApplyFn at cli.cpp:198).
 * on_device != 0: x, y are device pointers used on `stream`; else host arrays (copies included). */
int ce_matvec(const ce_matrix* a, const double* x, double* y, int64_t n, int on_device, void* stream);

/* ---- factorization ---- */
/* Replaces ce_factorize(const BlockSparseMatrix&, const CoarseningPlan&, const CompressionStrategy&,
 * const FactorOptions&) (factorization.hpp:121-123, factorization.cpp:336-461). */
int ce_factorize(ce_ctx* ctx, const ce_matrix* a, const ce_plan_host* plan, const ce_strategy* s,
                 const ce_factor_opts* opts, ce_factor** out, ce_status* st);
void ce_factor_free(ce_factor* f);
int64_t ce_factor_dim(const ce_factor* f);
/* ---- subdomain-sharded factorization ----
 * One process per GPU, each with its own ce_ctx on its device; every rank calls
 * ce_factorize_sharded with the same matrix, plan and strategy.  The plan must put each
 * level's box-interior rows first (CE_PLAN_SHARDED does); box b belongs to rank
 * b * n_ranks / n_boxes.  Each rank sweeps the interior rows of its boxes, the interface rows
 * are swept by every rank, and the ranks exchange blocks through `bcast` -- an in-place
 * broadcast of `bytes` device bytes at `dev_ptr` from rank `root` to all ranks (NCCL over
 * NVLink in the Python binding; it returns 0 on success, must complete before returning, and
 * every rank issues the same calls in the same order).  The resulting factor is complete on
 * every rank and bit-identical to ce_factorize of the same plan on one GPU. */
typedef int (*ce_bcast_fn)(void* user, void* dev_ptr, int64_t bytes, int root);
typedef struct {
  int rank;
  int n_ranks;
  int64_t n_boxes;
  const int64_t* box_of_block; /* level-1 block -> box, m entries (ce_problem_boxes) */
  ce_bcast_fn bcast;
  void* user;
} ce_shard;
int ce_factorize_sharded(ce_ctx* ctx, const ce_matrix* a, const ce_plan_host* plan, const ce_strategy* s,
                         const ce_factor_opts* opts, const ce_shard* shard, ce_factor** out, ce_status* st);
/* Host-side symbolic split of a CE_PLAN_SHARDED problem over n_ranks (every group assumed
 * alive): per level l < *n_levels (<= max_levels), out[l * (2 + n_ranks) + {0, 1, 2 + r}] =
 * {block count, interior (phase-1) rows, rows rank r sweeps alone}.  No GPU needed. */
int ce_shard_plan_summary(const ce_problem* p, int n_ranks, int64_t max_levels, int64_t* out, int64_t* n_levels);

/* Preconditioner apply x = Q^T L^-T L^-1 Q b (replaces CEFactorization::solve,
 * factorization.cpp:140-168; used as ApplyFn at cli.cpp:225).  Thread-safe: concurrent calls
 * on one factor (any threads, any streams) are serialised on the device, because they share
 * the factor's apply workspaces (each waits for the previous apply's completion event). */
int ce_apply_precond(const ce_factor* f, const double* b, double* x, int64_t n, int on_device, void* stream);
/* Validation tools (factorization.cpp:170-257): which 0 = apply_operator (Q^T L L^T Q x),
 * 1 = apply_q, 2 = apply_q_transpose.  Host arrays. */
int ce_factor_apply_tool(const ce_factor* f, int which, const double* x, double* y, int64_t n);
int ce_factor_get_stats(const ce_factor* f, ce_factor_stats* out);
int ce_factor_get_level_stats(const ce_factor* f, int64_t level, ce_level_stats* out);
/* Per-row structure of level `level` (0-based), M entries each (any pointer may be NULL): block
 * sizes, retained ranks (FactorLevel::retained, factorization.hpp:19-36), far-concatenation
 * widths and singular-value counts -- the parity structure without a full dump. */
int ce_factor_level_rows(const ce_factor* f, int64_t level, int64_t* sizes, int64_t* retained, int64_t* fcols,
                         int64_t* nsigma);
/* Singular values of the far concatenation of (level, row) (compress_far_concat,
 * compression.cpp:48-49), descending; writes min(count, cap), returns the count (< 0 on error). */
int64_t ce_factor_row_sigma(const ce_factor* f, int64_t level, int64_t row, double* out, int64_t cap);
/* Binary factor dump in the oracle's format, for parity checks. */
int ce_factor_dump(const ce_factor* f, const char* path);

/* ---- CSV reports of the reference CLI (proj/src/csv.cpp, proj/src/cli.cpp) ----
 * Text builders: each writes a NUL-terminated table (header row + rows, '\n' line ends, no
 * quoting: CsvTable::to_string, csv.cpp:37-42) into buf when it fits in cap and returns the text
 * length (call with cap = 0 to size the buffer; < 0 on error).  Numbers are formatted like
 * fmt_double / fmt_index (csv.cpp:84-96): the shortest text that round-trips. */
int ce_fmt_double(double v, char* buf, int cap);
/* CompressionStrategy::describe (compression.cpp:10-18): "eps=1e-06", "abseps=...", "rank=8"; NULL -> "none". */
int ce_strategy_describe(const ce_strategy* s, char* buf, int cap);
/* factor_stats.csv (factor_stats_table, cli.cpp:60-71): level, blocks_eliminated, l_blocks, max_rank,
 * mean_rank, seconds, bytes -- one row per level. */
int64_t ce_factor_stats_csv(const ce_factor* f, char* buf, int64_t cap);
/* factor_summary.csv (run_factor, cli.cpp:167-182); recon_error may be NULL / "" (n > 4096). */
int64_t ce_factor_summary_csv(const ce_factor* f, int64_t block, const ce_strategy* s, double seconds,
                              const char* recon_error, char* buf, int64_t cap);
/* solve_report.csv (run_solve, cli.cpp:233-247); mode "minres" | "pcg" | "direct", s NULL = "none". */
int64_t ce_solve_report_csv(int64_t n, const char* mode, const ce_strategy* s, int preconditioned,
                            const ce_solve_report* rep, double factor_seconds, double solve_seconds, char* buf,
                            int64_t cap);
/* trace.csv (trace_table, cli.cpp:73-80) from IterationSample arrays. */
int64_t ce_trace_csv(int64_t count, const int64_t* iter, const double* recurrence, const double* true_resid,
                     const double* seconds, char* buf, int64_t cap);
/* IterationTrace (minres.hpp:12-23) of the context's last ce_pcg / ce_minres: one sample per
 * iteration preceded by the iteration-0 sample (minres.cpp:55); true_resid = -1 where it was not
 * tracked (the last sample always carries the final true residual, minres.cpp:112-113).  Returns
 * the sample count (writes min(count, cap)). */
int64_t ce_ctx_last_trace(const ce_ctx* ctx, int64_t* iter, double* recurrence, double* true_resid, double* seconds,
                          int64_t cap);

/* ---- Krylov ---- */
/* PCG with the minres contract (minres.hpp:46-47): x0 = 0, stop when the
 * recurrence ||r||/||b|| <= tol, iterations = number of A*p products.  precond may be NULL
 * (unpreconditioned).  on_device != 0: b, x are device pointers, read and written in order on
 * `stream` (NULL = the context's stream), like ce_apply_precond / ce_matvec; with host
 * arrays the call is synchronous. */
int ce_pcg(ce_ctx* ctx, const ce_matrix* a, const ce_factor* precond, const double* b, double* x, int64_t n,
           int on_device, const ce_pcg_opts* opts, ce_solve_report* rep, void* stream);
/* MINRES (replaces ce::minres, proj/include/ce/minres.hpp:46-47 / proj/src/minres.cpp:22-115, the
 * paper's solver; ApplyFn pair at proj/src/cli.cpp:198,225-226): x0 = 0, stop when the recurrence
 * estimate of the preconditioned residual <= tol relative to its start, or on a Lanczos beta
 * < 1e-30 beta1; iterations = number of A*v products.  Same options, report, error codes and
 * memory conventions as ce_pcg (opts->track_true_residual = the MinresOptions field). */
int ce_minres(ce_ctx* ctx, const ce_matrix* a, const ce_factor* precond, const double* b, double* x, int64_t n,
              int on_device, const ce_pcg_opts* opts, ce_solve_report* rep, void* stream);

/* ---- BASELINE problem generation (setup, untimed; SURVEY.md §8d conventions) ----
 * cfg 1..5, optional grid override (0 = keep).  Builds the permuted CSB, plan and rhs on the host
 * (replaces assemble_diffusion_3d + geometric_block_ordering + finish_load, problems.cpp:18-258,
 * cli.cpp:33-58, extended with the 2-D/FV/random-k/RNG inputs BASELINE.json names). */
int ce_problem_create(int cfg, int64_t nx, int64_t ny, int64_t nz, ce_problem** out);
/* Same, choosing the plan family: CE_PLAN_REFERENCE = geometric_block_ordering(grid, block, 2)
 * (problems.cpp:195-258: join 2 along one cyclically alternating axis per level);
 * CE_PLAN_MERGE_ALL_AXES = every non-exhausted axis merges by 2 at each level (2x2 / 2x2x2
 * groups, J = 2^d).  The latter is an ordinary CoarseningPlan (problems.hpp:51-65) that the
 * reference's ce_factorize takes through its plan file (problems.cpp:114-171); its block
 * pattern reach stays bounded, so the 3-D configs fit in HBM at full size. */
#define CE_PLAN_REFERENCE 0
#define CE_PLAN_MERGE_ALL_AXES 1
/* CE_PLAN_MERGE_ALL_COLORED = CE_PLAN_MERGE_ALL_AXES with every level's cells ordered
 * colour-major, colour = (cx mod 3, cy mod 3, cz mod 3): with all-axis merges a row's squared
 * pattern stays within Chebyshev distance 2 (in cells), so rows of one colour are independent
 * and each level's sweep has at most 9 (2-D) / 27 (3-D) waves. */
#define CE_PLAN_MERGE_ALL_COLORED 2
/* CE_PLAN_SHARDED = CE_PLAN_MERGE_ALL_COLORED with 8 spatial boxes (4 x 2 in 2-D, 2 x 2 x 2 in
 * 3-D): at every level the cells >= 2 cells inside their box come first, box by box (each
 * colour-major), then every other ("interface") cell, colour-major.  An interior row's
 * squared-pattern row never leaves its box, so the boxes' interiors factor independently:
 * the plan ce_factorize_sharded distributes over GPUs.  Box labels of the
 * level-1 blocks: ce_problem_boxes. */
#define CE_PLAN_SHARDED 3
int ce_problem_create_plan(int cfg, int64_t nx, int64_t ny, int64_t nz, int plan_kind, ce_problem** out);
void ce_problem_free(ce_problem* p);
/* The reference CLI's `file` problem (proj/src/cli.cpp:114-133 load_problem + finish_load :49-58):
 * Matrix Market "coordinate real general|symmetric" (matrix_market.cpp:21-59), a CoarseningPlan
 * file (problems.cpp:140-174; NULL = CoarseningPlan::trivial(n, block), problems.cpp:175-182) and
 * an rhs vector file (NULL = ones); the plan's initial permutation is applied and the CSB built
 * with BlockSparseMatrix::from_triplets semantics (block_matrix.cpp:48-90: duplicates summed,
 * symmetry checked to 1e-12 max|a|, full diagonal).  Errors (IO, asymmetric input, invalid plan)
 * return CE_EUSAGE with the reference's message in ce_last_error(). */
int ce_problem_load(const char* matrix_path, const char* plan_path, const char* rhs_path, int64_t block,
                    ce_problem** out);
/* run_gen's writer (cli.cpp:136-150): natural-order matrix (write_matrix_market, lower triangle,
 * 17 digits), rhs (write_vector) and plan (CoarseningPlan::save); any path may be NULL (skipped). */
int ce_problem_save(const ce_problem* p, const char* matrix_path, const char* plan_path, const char* rhs_path);
/* CE_PLAN_SHARDED problems: the box (subdomain) label of every level-1 block and the box count
 * (*n_boxes = 0, *box_of_block = NULL for the other plan families). */
int ce_problem_boxes(const ce_problem* p, const int64_t** box_of_block, int64_t* n_boxes);
/* Views into the problem (valid until ce_problem_free). */
int ce_problem_csb(const ce_problem* p, ce_csb_host* out);
int ce_problem_plan(const ce_problem* p, ce_plan_host* out);
const double* ce_problem_rhs(const ce_problem* p);
const int64_t* ce_problem_perm(const ce_problem* p);
/* eps, tol, block of the config. */
int ce_problem_params(const ce_problem* p, double* eps, double* tol, int64_t* block);

#ifdef __cplusplus
}
#endif

#endif /* CE_GPU_H */
