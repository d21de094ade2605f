/*
 * batchlp_cuda.h — C-ABI of the B200-native batched PDHG LP solver.
 *
 * This is the drop-in boundary for the reference's hot path
 * `batchlp::solve_batch` (reference: proj/include/batchlp/batch_solver.hpp:78-82)
 * and the helpers its callers and tests use. Plain pointers and sizes only:
 * no C++ types, no torch types, no exceptions cross this boundary. Every entry
 * returns an int status code that maps 1:1 onto the exception the reference
 * throws at the same point; the message is read with bl_last_error().
 *
 * Ownership: a bl_ctx owns one CUDA stream on one device and the device
 * workspace of its last solve (grow-only, like BatchWorkspace,
 * batch_solver.hpp:59-67). A bl_problem is an immutable device-resident copy
 * of an LpProblem (problem.hpp:32-40) — A in CSR, its explicit transpose, the
 * objective and both bound vectors — and may be shared by solves on the same
 * context. One context per (host thread, device).
 *
 * Dense host buffers are column-major with one contiguous column per LP, the
 * reference's DenseColumnBlock layout (sparse.hpp:46-88). On the device the
 * solver keeps its own column-block-tiled layout.
 */
#ifndef BATCHLP_CUDA_H_
#define BATCHLP_CUDA_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BL_ABI_VERSION 1

/* Return codes; each maps onto one reference exception type. */
enum bl_code {
  BL_OK = 0,
  BL_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument */
  BL_ERR_OUT_OF_RANGE = 2,     /* std::out_of_range */
  BL_ERR_DOMAIN = 3,           /* std::domain_error (broken step size, solver.hpp:257-259) */
  BL_ERR_LOGIC = 4,            /* std::logic_error (batch_solver.hpp:350-351) */
  BL_ERR_CUDA = 5              /* device / driver failure (std::runtime_error) */
};

/* SolveStatus, solver.hpp:105-110 (same order). */
enum bl_status {
  BL_OPTIMAL = 0,
  BL_PRIMAL_INFEASIBLE = 1,
  BL_DUAL_INFEASIBLE = 2,
  BL_ITERATION_LIMIT = 3
};

/* OverrideKind, problem.hpp:124 (same order). */
enum bl_override_kind {
  BL_OVERRIDE_OBJECTIVE = 0,
  BL_OVERRIDE_LOWER = 1,
  BL_OVERRIDE_UPPER = 2
};

/* ObjectiveMode, problem.hpp:134-137 (same order). */
enum bl_objective_mode { BL_SHARED_OBJECTIVE = 0, BL_SIGNED_UNIT_COLUMNS = 1 };

/* RestartReason, solver.hpp:112 (same order). */
enum bl_restart_reason {
  BL_RESTART_SUFFICIENT = 0,
  BL_RESTART_NECESSARY = 1,
  BL_RESTART_ARTIFICIAL = 2
};

/* What a solve keeps for copy-back (extension: the reference always returns
 * x/y/reduced costs by value; FSB and OBBT only need the scalars). */
enum bl_vectors {
  BL_VECTORS_NONE = 0,        /* scalars only (status, objective, residuals) */
  BL_VECTORS_SOLUTION = 1,    /* + x, y, reduced costs per LP */
  BL_VECTORS_CERTIFICATE = 2  /* + infeasibility certificate vectors */
};

typedef struct bl_ctx bl_ctx;
typedef struct bl_problem bl_problem;

/* SolverConfig, solver.hpp:66-103 (field for field), plus two extensions. */
typedef struct bl_config {
  double eps_opt;
  double eps_infeas;
  double eps_dual; /* < 0: use eps_opt (solver.hpp:88) */
  double theta;
  double beta_sufficient;
  double beta_necessary;
  double beta_artificial;
  int64_t max_iterations;
  int64_t termination_check_period;
  double w_init;
  int32_t robust_bound_contribution;
  int32_t average_over_all_columns;
  int32_t trace_iterates;
  int32_t vectors; /* enum bl_vectors; extension */
  double eta;      /* > 0: use this step size instead of 0.998/||A||_2; extension */
} bl_config;

/* Per-LP variation, ColumnOverride problem.hpp:127-132. */
typedef struct bl_override {
  int32_t column;
  int32_t kind; /* enum bl_override_kind */
  int32_t variable;
  int32_t reserved;
  double value;
} bl_override;

/* Scalar part of SolveResult (solver.hpp:134-145) for one LP. */
typedef struct bl_column_result {
  int32_t status; /* enum bl_status */
  int32_t restarts;
  int64_t iterations;
  double objective;
  double gap, primal, dual, fixed_point; /* Residuals, solver.hpp:127-132 */
  /* OptimalityReport::bound_support / row_support of the returned triple
   * (solver.hpp:340-354); lets callers such as OBBT's margin
   * (obbt.hpp:121-137) skip copying vectors back. */
  double bound_support, row_support;
  /* Support of the returned reduced costs over the BASE variable bounds,
   * exactly the sup_r of obbt_margin (obbt.hpp:123-126). */
  double base_bound_support;
  int32_t has_solution;    /* bl_fetch_solution will return x/y/reduced */
  int32_t has_certificate; /* bl_fetch_certificate will return vectors */
  int32_t certificate_kind;/* 0 none, 1 primal (dx,dy,dr), 2 dual (dx only) */
  /* 1 when the reference would return non-empty x/y/reduced costs for this
   * LP (false only for an iteration-limited LP that never had a candidate),
   * independent of what this solve kept for copy-back. */
  int32_t vectors_exist;
} bl_column_result;

/* RestartEvent, solver.hpp:114-119. */
typedef struct bl_restart_event {
  int64_t at_iteration;
  int32_t reason; /* enum bl_restart_reason */
  int32_t reserved;
  double residual;
  double anchor_residual;
} bl_restart_event;

/* BatchSolveSummary scalars, batch_solver.hpp:50-57. */
typedef struct bl_summary {
  int64_t iterations;
  int32_t restarts;
  int32_t restart_log_size; /* events recorded (== restarts unless truncated) */
  int64_t sparse_products;
  uint64_t trajectory_hash;
  double eta;      /* step size used */
  double device_ms;/* device time of the solve (CUDA events), setup included */
  int64_t kernel_launches; /* kernels the solve launched on the device */
  int64_t loop_passes;     /* operator applications (iterations + restarts) */
} bl_summary;

/* In-situ timing of one kernel kind over the last solve: device
 * %globaltimer span of each launch (first CTA entry to last CTA exit) and
 * the algorithmic bytes credited to it. */
typedef struct bl_kernel_stat {
  char name[16];
  double launches;
  double total_ns;
  double alg_bytes;
} bl_kernel_stat;

/* ---- context ------------------------------------------------------------ */
void bl_config_default(bl_config* cfg);
int bl_abi_version(void);
int bl_ctx_create(int device, bl_ctx** out);
void bl_ctx_destroy(bl_ctx* ctx);
/* Last error message of this context (or of creation when ctx is NULL). */
const char* bl_last_error(const bl_ctx* ctx);

/* ---- problem upload (LpProblem + SparseMatrix, problem.hpp:32-40,
 *      sparse.hpp:93-171) ---------------------------------------------------
 * rowptr/col/val: CSR of A (m rows); t_rowptr/t_col/t_val: the explicit
 * transpose (n rows), as SparseMatrix::view()/transpose_view() expose them.
 * The five vectors are objective (n), var_lower/var_upper (n) and
 * row_lower/row_upper (m). Infinite bounds are +-INFINITY. */
int bl_problem_upload(bl_ctx* ctx, int32_t m, int32_t n, int64_t nnz,
                      const int32_t* rowptr, const int32_t* col,
                      const double* val, const int32_t* t_rowptr,
                      const int32_t* t_col, const double* t_val,
                      const double* objective, const double* var_lower,
                      const double* var_upper, const double* row_lower,
                      const double* row_upper, bl_problem** out);
void bl_problem_free(bl_problem* p);
/* Re-fills an uploaded problem with new arrays (same meaning as
 * bl_problem_upload). Device buffers only grow, so re-uploading a problem
 * of the same size keeps every device address and the solver's captured
 * CUDA graphs are reused; the cached spectral norm is invalidated. */
int bl_problem_assign(bl_ctx* ctx, bl_problem* p, int32_t m, int32_t n, int64_t nnz,
                      const int32_t* rowptr, const int32_t* col, const double* val,
                      const int32_t* t_rowptr, const int32_t* t_col,
                      const double* t_val, const double* objective,
                      const double* var_lower, const double* var_upper,
                      const double* row_lower, const double* row_upper);

/* ---- sparse helpers (sparse.hpp) -----------------------------------------
 * spectral_norm (sparse.hpp:297-319): ||A||_2 estimate x 1.01, computed by
 * the device power iteration. BL_ERR_INVALID_ARGUMENT on a zero matrix. */
int bl_spectral_norm(bl_ctx* ctx, bl_problem* p, double* out);
/* spmm (sparse.hpp:213-238): out[:, j] = op(A) x[:, j] for j < active;
 * columns j >= active of `out` are left untouched. x and out are host
 * column-major blocks with `width` columns. Per-row accumulation follows the
 * stored CSR order without FMA contraction, so every entry is bit-identical
 * to the reference csr_apply (sparse.hpp:176-183). */
int bl_spmm(bl_ctx* ctx, const bl_problem* p, int transpose, int32_t width,
            int32_t active, const double* x, double* out);
/* csr_apply (sparse.hpp:176-183) on a bare CSR view (CsrView, sparse.hpp:28-
 * 36) that is not an uploaded problem: out = M x for the rows x cols matrix
 * (rowptr, col, val), computed by the same SpMM kernel (bit-identical to the
 * reference's stored-order sum). The view is uploaded into grow-only
 * context scratch on every call. BL_ERR_INVALID_ARGUMENT for malformed
 * offsets, BL_ERR_OUT_OF_RANGE for a column index outside [0, cols). */
int bl_csr_apply(bl_ctx* ctx, int32_t rows, int32_t cols, int64_t nnz, const int32_t* rowptr,
                 const int32_t* col, const double* val, const double* x, double* out);
/* measure_spmm (tuner.hpp:72-108) on the device: `repetitions` products
 * A X and `repetitions` products A'Y of `width` columns (seeded blocks, two
 * untimed warm-up rounds), timed with CUDA events on the context's stream;
 * the cost of an empty event interval is subtracted and a clamp to zero is
 * reported through *clamped. Seconds. BL_ERR_INVALID_ARGUMENT for width < 1
 * or repetitions < 3, as the reference. */
int bl_measure_spmm(bl_ctx* ctx, const bl_problem* p, int32_t width, int32_t repetitions,
                    double* total_s, double* per_column_s, int32_t* clamped);

/* ---- the hot path: solve_batch (batch_solver.hpp:78-355) -----------------
 * width LPs share A, the row bounds and (mode SHARED) the objective; each
 * column differs through `overrides` (any order; later entries win within a
 * column, as in ColumnView, problem.hpp:209-236) or, in SIGNED_UNIT mode
 * (width == 2n), by the objective +e_j / -e_{j-n}.
 * preset_columns: columns frozen before iterating (PresetColumn,
 * batch_solver.hpp:45-48); their results are the caller's and are left
 * untouched in `results`.
 * initial_weights: NULL or width primal weights (batch_solver.hpp:115-120).
 * warm_x / warm_y: NULL or column-major start points (width x n, width x m);
 * x is projected onto each column's box (WarmStart, solver.hpp:590-597).
 * results: width entries, original column order. */
int bl_solve_batch(bl_ctx* ctx, bl_problem* p, int32_t width, int32_t mode,
                   const bl_override* overrides, int32_t n_overrides,
                   const bl_config* cfg, const int32_t* preset_columns,
                   int32_t n_presets, const double* initial_weights,
                   const double* warm_x, const double* warm_y,
                   bl_summary* summary, bl_column_result* results);

/* ---- multi-GPU: the batch sharded across devices ----------
 * One (context, problem) pair per shard -- normally one per GPU, each with
 * its own replica of A uploaded by bl_problem_upload on that context. The
 * width LPs are split into n_shards contiguous near-equal column slices
 * (shard s: [s*width/G ...), the first width % G slices one longer); each
 * shard runs bl_solve_batch on its slice on its own host thread, with no
 * communication while iterating (restarts synchronise on the SLICE's
 * averaged residual, i.e. this is exactly n_shards reference solve_batch
 * runs on the slices, the parity definition of SURVEY §8(e)). Overrides,
 * presets and initial weights are given for the whole batch (original
 * column indices) and routed to their shard; signed-unit batches stay
 * signed-unit per slice. Every shard copies its per-LP records straight
 * into its slice of `results` (original column order): the gather is one
 * device-to-host copy per GPU, nothing crosses between devices.
 * summaries: NULL or n_shards entries (per-shard iterations, restarts, eta,
 * device time). Vectors of shard s are fetched from ctxs[s] with the
 * column index local to its slice. Errors: the whole-batch checks come
 * first (codes as bl_solve_batch); a shard's failure is reported as
 * "shard s: ..." with that shard's code on ctxs[0]. */
int bl_solve_batch_sharded(bl_ctx* const* ctxs, bl_problem* const* probs, int32_t n_shards,
                           int32_t width, int32_t mode, const bl_override* overrides,
                           int32_t n_overrides, const bl_config* cfg,
                           const int32_t* preset_columns, int32_t n_presets,
                           const double* initial_weights, bl_summary* summaries,
                           bl_column_result* results);

/* Vectors of the last solve on this context (lazy copy-back). */
int bl_fetch_solution(bl_ctx* ctx, int32_t column, double* x, double* y,
                      double* reduced);
int bl_fetch_certificate(bl_ctx* ctx, int32_t column, double* delta_x,
                         double* delta_y, double* delta_r);
/* Per-kernel timing of the last solve (up to cap kinds). */
int bl_fetch_profile(bl_ctx* ctx, bl_kernel_stat* out, int32_t cap, int32_t* n_out);
/* Copies min(cap, restart_log_size) events; returns the count in *n_out. */
int bl_fetch_restart_log(bl_ctx* ctx, bl_restart_event* out, int32_t cap,
                         int32_t* n_out);

/* ---- instance generators (tools; not on the hot path) --------------------
 * Deterministic synthetic instances used by the benchmarks. Output arrays
 * are malloc'ed by the library and released with bl_free. */
typedef struct bl_instance {
  int32_t m, n;
  int64_t nnz;
  int32_t *rowptr, *col;
  double* val;
  int32_t *t_rowptr, *t_col;
  double* t_val;
  double *objective, *var_lower, *var_upper, *row_lower, *row_upper;
} bl_instance;
/* generate_set_cover (reference generators.hpp:76-109), same draws. */
int bl_gen_set_cover(int32_t rows, int32_t cols, double density, uint64_t seed,
                     bl_instance* out);
/* O(nnz) set-cover-like family of SURVEY §8(d) C3-C5: each column picks d
 * distinct rows, uncovered rows get one random column. */
int bl_gen_sparse_cover(int32_t rows, int32_t cols, int32_t per_col,
                        uint64_t seed, bl_instance* out);
/* Scaled random_feasible_lp family of SURVEY §8(d) C2 (OBBT). */
int bl_gen_boxed_feasible(int32_t rows, int32_t cols, int32_t per_col,
                          uint64_t seed, bl_instance* out);
void bl_instance_free(bl_instance* inst);

#ifdef __cplusplus
}
#endif

#endif /* BATCHLP_CUDA_H_ */
