/*
 * lsamgdd_b200.h — C ABI of the B200-native least-squares AMG-DD hot path.
 *
 * This is the drop-in boundary for the reference's header API in
 * /root/reference/proj/include/lsamgdd/ (there is no plugin registry in the
 * reference; callers include lsamgdd/lsamgdd.hpp, lsamgdd.hpp:16-26). Each
 * entry point below names the reference interface it replaces (file:line).
 * The C++ shim in include/lsamgdd_b200/lsamgdd.hpp re-exports these under
 * the reference's own names and types; INTEGRATION.md shows the ctypes and
 * C++ bindings.
 *
 * Conventions
 *  - Plain pointers and sizes only; no torch or CUDA types cross the ABI.
 *  - CSR matrices use int64 row offsets and column indices and FP64 values
 *    (the reference's SparseMatrix holds size_t/double, sparse.hpp:28-72).
 *  - Every function returns an lsamgdd_status. A non-zero status maps 1:1 to
 *    the reference exception class of the same name (errors.hpp:11-69); the
 *    message is written to err (NUL-terminated, truncated to errlen).
 *  - A hierarchy handle is immutable after lsamgdd_setup and may be shared by
 *    concurrent vcycle/pcg/schwarz calls (hierarchy.hpp:56-57): each call uses
 *    its own stream and workspace.
 *  - Device-memory arguments (lsamgdd_memory == LSAMGDD_DEVICE): the library
 *    runs on its own non-blocking CUDA streams. Before it first reads such an
 *    argument a call waits for the caller's pending device work: for the
 *    stream registered with lsamgdd_set_caller_stream (per host thread), or,
 *    when none is registered, for the whole device (cudaDeviceSynchronize).
 *    Every call returns with its outputs complete (the library's stream is
 *    synchronised), so the caller may read them from any stream.
 *  - There is no CPU fallback: on a machine without a usable sm_100 device,
 *    every compute entry point fails with LSAMGDD_ERR_CUDA.
 */
#ifndef LSAMGDD_B200_H
#define LSAMGDD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LSAMGDD_B200_ABI_VERSION 1

/* Status codes. 1..10 mirror lsamgdd::Error and its subclasses
 * (errors.hpp:14-69) in declaration order. */
typedef enum lsamgdd_status {
  LSAMGDD_OK = 0,
  LSAMGDD_ERR_ERROR = 1,            /* lsamgdd::Error           errors.hpp:14 */
  LSAMGDD_ERR_INDEX = 2,            /* IndexError               errors.hpp:20 */
  LSAMGDD_ERR_DIM = 3,              /* DimError                 errors.hpp:26 */
  LSAMGDD_ERR_INPUT = 4,            /* InputError               errors.hpp:32 */
  LSAMGDD_ERR_FORMAT = 5,           /* FormatError              errors.hpp:38 */
  LSAMGDD_ERR_SPLITTING = 6,        /* SplittingError           errors.hpp:44 */
  LSAMGDD_ERR_EIG = 7,              /* EigError                 errors.hpp:50 */
  LSAMGDD_ERR_SETUP = 8,            /* SetupError               errors.hpp:56 */
  LSAMGDD_ERR_INDEFINITE = 9,       /* IndefiniteError          errors.hpp:62 */
  LSAMGDD_ERR_SIZE = 10,            /* SizeError                errors.hpp:68 */
  LSAMGDD_ERR_CUDA = 64,            /* device/runtime failure (no reference twin) */
  LSAMGDD_ERR_OOM = 65              /* device allocation failed */
} lsamgdd_status;

/* Where the arrays of an lsamgdd_csr / vector argument live. */
typedef enum lsamgdd_memory { LSAMGDD_HOST = 0, LSAMGDD_DEVICE = 1 } lsamgdd_memory;

/* CSR view, caller-owned (replaces SparseMatrix, sparse.hpp:28-72).
 * Column indices strictly increasing within a row, values finite. */
typedef struct lsamgdd_csr {
  int64_t n_rows;
  int64_t n_cols;
  int64_t nnz;
  const int64_t* row_offsets; /* n_rows + 1 */
  const int64_t* col_indices; /* nnz */
  const double* values;       /* nnz */
  int32_t memory;             /* lsamgdd_memory */
  int32_t reserved;
} lsamgdd_csr;

/* LevelParams (hierarchy.hpp:19-30) plus opt-in extensions. With the
 * extension fields at their defaults, setup follows the reference exactly. */
typedef struct lsamgdd_params {
  uint64_t max_levels;         /* 25 */
  uint64_t coarse_size;        /* 400 */
  uint64_t aggregation_passes; /* 1 */
  double kappa;                /* 50 */
  double must_keep;            /* 5 */
  uint64_t n_ratios;           /* 2 */
  uint64_t coarsening_ratios[8]; /* {2,3}; the last entry repeats */
  uint64_t pre_sweeps;         /* 1 */
  uint64_t post_sweeps;        /* 1 */
  int32_t gevp_variant;        /* 0 SchurReduced, 1 WeightedLhs (splitting.hpp:45) */
  int32_t keep_spectra;        /* 1: keep per-aggregate eigenvalues (spectra_csv, hierarchy.hpp:121-127) */
  /* ---- extensions ---- */
  const int64_t* level0_partition; /* NULL: multi_pass_aggregation at level 0 */
  int64_t level0_n_aggregates;
  int32_t level0_overlap;      /* 0/1: reference Γ (one layer); 2: two layers of A_0 */
  int32_t device;              /* CUDA ordinal, default 0 */
  double thresh_override;      /* <= 0: eigen_threshold (splitting.hpp:170); > 0: direct threshold on every level */
  uint64_t level0_max_modes;   /* 0: reference (cap = |omega| at level 0, hierarchy.hpp:156-157) */
  uint64_t probe_levels;       /* 0: full setup. k > 0 (stage-wise parity and timing of the fine levels at full
                                  size): build k levels with interpolation and the operators of level k, then stop
                                  without factoring the coarsest level. Such a handle serves exports, level_spmv and
                                  schwarz_apply on levels < k; vcycle and pcg fail with InputError. */
  uint64_t level_offset;       /* 0: the factor is level 0. k > 0 (distributed setup): the factor is level k of a
                                  hierarchy whose finer levels were built elsewhere — ratios, caps and max_levels
                                  count from level k, the level-0 hooks do not apply */
  uint64_t reserved[2];
} lsamgdd_params;

/* LevelSummary (hierarchy.hpp:32-41). */
typedef struct lsamgdd_level_summary {
  uint64_t level;
  uint64_t dim;
  uint64_t nnz;
  uint64_t n_aggregates;
  uint64_t k_c;
  uint64_t n_mult;
  double thresh;
  uint64_t modes_kept;
} lsamgdd_level_summary;

/* SolveReport (krylov.hpp:24-33). residual_history is caller-owned; at most
 * history_capacity entries are written, history_len reports the full count. */
typedef struct lsamgdd_report {
  uint64_t iterations;
  int32_t converged;
  int32_t reserved;
  double avg_conv_factor;
  double iters_to_tenth;
  double operator_complexity;
  double setup_seconds;
  double solve_seconds;
  double* residual_history;
  uint64_t history_capacity;
  uint64_t history_len;
} lsamgdd_report;

/* SchwarzMode (smoother.hpp:21). */
typedef enum lsamgdd_schwarz_mode { LSAMGDD_RAS = 0, LSAMGDD_RAST = 1, LSAMGDD_ASM = 2 } lsamgdd_schwarz_mode;

/* What lsamgdd_level_export returns (host mirrors of Level, hierarchy.hpp:46-51). */
typedef enum lsamgdd_export_what {
  LSAMGDD_EXPORT_A = 0,         /* CSR: sizes {rows, cols, nnz}; idx0 offsets, idx1 cols, vals */
  LSAMGDD_EXPORT_G = 1,         /* CSR */
  LSAMGDD_EXPORT_P = 2,         /* CSR (only levels with interpolation) */
  LSAMGDD_EXPORT_PARTITION = 3, /* sizes {n_nodes, n_aggregates, 0}; idx0 assignment */
  LSAMGDD_EXPORT_GAMMA = 4,     /* sizes {n_aggregates, total, 0}; idx0 offsets, idx1 nodes */
  LSAMGDD_EXPORT_COLORS = 5,    /* sizes {n_aggregates, n_colors, 0}; idx0 colors */
  LSAMGDD_EXPORT_SPECTRA = 6,   /* sizes {n_aggregates, total, 0}; idx0 offsets, vals eigenvalues */
  LSAMGDD_EXPORT_MULTIPLICITY = 7 /* sizes {rows of G, n_mult, 0}; idx0 multiplicity */
} lsamgdd_export_what;

void lsamgdd_params_default(lsamgdd_params* p);
int32_t lsamgdd_abi_version(void);
/* 1 if a usable sm_100 device is visible, else 0 (no error). */
int32_t lsamgdd_device_available(void);

/* Registers (enable != 0) or clears the CUDA stream (a cudaStream_t) on which
 * the calling host thread produces device-memory arguments; see Conventions. */
int lsamgdd_set_caller_stream(void* stream, int32_t enable);

/* setup(g0, params)                                    hierarchy.hpp:106 */
int lsamgdd_setup(const lsamgdd_csr* g0, const lsamgdd_params* params, void** out_handle,
                  char* err, size_t errlen);
int lsamgdd_destroy(void* handle);

int lsamgdd_num_levels(const void* handle, int64_t* out);
int lsamgdd_get_level_summary(const void* handle, int64_t level, lsamgdd_level_summary* out);
/* operator_complexity(h)                               hierarchy.hpp:257 */
int lsamgdd_operator_complexity(const void* handle, double* out);

/* vcycle(h, level, r)                                  hierarchy.hpp:205, :229 */
int lsamgdd_vcycle(const void* handle, int64_t level, const double* r, double* e, int32_t memory,
                   char* err, size_t errlen);
/* apply(smoother_l, r, mode)                           smoother.hpp:65 */
int lsamgdd_schwarz_apply(const void* handle, int64_t level, int32_t mode, const double* r,
                          double* e, int32_t memory, char* err, size_t errlen);
/* pcg(Gᵀ(G·), vcycle(h,·), b, tol, maxit)               krylov.hpp:42-92 with the
 * factored operator of lsamgdd_cli.cpp:137-142. g == NULL uses the setup factor. */
int lsamgdd_pcg(const void* handle, const lsamgdd_csr* g, const double* b, double tol,
                uint64_t maxit, double* x, int32_t memory, lsamgdd_report* report, char* err,
                size_t errlen);
/* spmv(A_l or G_l or P_l, x) and spmv_transpose       sparse.hpp:110, :125 */
int lsamgdd_level_spmv(const void* handle, int64_t level, int32_t what, int32_t transpose,
                       const double* x, double* y, int32_t memory, char* err, size_t errlen);

/* ---- the sparse kernels on caller matrices (no hierarchy needed) ---- */
/* spmv(a, x) (transpose == 0, sparse.hpp:110) or spmv_transpose(a, x)
 * (sparse.hpp:125): row sums in CSR order, bit-identical to the reference. */
int lsamgdd_spmv(const lsamgdd_csr* a, int32_t transpose, const double* x, double* y,
                 int32_t memory, char* err, size_t errlen);
/* spgemm(a, b, SpgemmMode::Symbolic) (sparse.hpp:167-204): the structural
 * pattern with exact zeros kept, accumulated over k in the reference's order.
 * The product stays on the device behind *out_matrix. */
int lsamgdd_spgemm(const lsamgdd_csr* a, const lsamgdd_csr* b, void** out_matrix, char* err,
                   size_t errlen);
/* transpose(a) (sparse.hpp:139-153), stable in the source row order. */
int lsamgdd_transpose(const lsamgdd_csr* a, void** out_matrix, char* err, size_t errlen);
/* build_smoother(a, topo) (smoother.hpp:38-58) on a caller operator and
 * topology: omega/gamma are the aggregates' interior and boundary node lists
 * (AggregateTopology, aggregation.hpp:33-40; the interiors partition the
 * nodes), colors a proper colouring of the subdomain-intersection graph
 * (aggregation.hpp:213-229). Concurrent applies on one smoother are not
 * supported (it owns a single stream). */
int lsamgdd_build_smoother(const lsamgdd_csr* a, int64_t n_aggregates, const int64_t* omega_offsets,
                           const int64_t* omega, const int64_t* gamma_offsets, const int64_t* gamma,
                           const int64_t* colors, void** out_smoother, char* err, size_t errlen);
/* apply(smoother, r, mode) (smoother.hpp:65-83); mode LSAMGDD_RAS or LSAMGDD_RAST. */
int lsamgdd_smoother_apply(const void* smoother, int32_t mode, const double* r, double* e,
                           int32_t memory, char* err, size_t errlen);
int lsamgdd_smoother_destroy(void* smoother);
/* A caller matrix kept on the device for repeated products (the distributed
 * solve's strip operators): y = m x or y = mᵀ x (the transposed operator is
 * built on first use), same kernels and summation order as lsamgdd_spmv. */
int lsamgdd_matrix_create(const lsamgdd_csr* a, void** out_matrix, char* err, size_t errlen);
int lsamgdd_matrix_spmv(void* matrix, int32_t transpose, const double* x, double* y, int32_t memory,
                        char* err, size_t errlen);
/* Host copy of a device matrix: sizes {rows, cols, nnz}; NULL arrays to query. */
int lsamgdd_matrix_export(const void* matrix, int64_t sizes[3], int64_t* offsets, int64_t* cols,
                          double* vals);
int lsamgdd_matrix_destroy(void* matrix);

/* Host mirrors (two-call protocol: pass NULL arrays to query sizes). */
int lsamgdd_level_export(const void* handle, int64_t level, int32_t what, int64_t sizes[3],
                         int64_t* idx0, int64_t* idx1, double* vals);

/* Per-stage device timings of the last setup (ms): fills up to n entries of
 * names (static strings) and ms; returns the count in *count. */
int lsamgdd_setup_timings(const void* handle, const char** names, double* ms, int64_t n,
                          int64_t* count);

/* Measured kernel statistics of the last timed call on this handle. */
typedef struct lsamgdd_kernel_stats {
  double schwarz_ms;      /* summed device time of Schwarz sweeps */
  double schwarz_bytes;   /* algorithmic bytes of those sweeps */
  int64_t schwarz_launches;
  double spmv_ms;
  double spmv_bytes;
  int64_t spmv_launches;
  int64_t total_launches; /* all kernels this library launched */
} lsamgdd_kernel_stats;
int lsamgdd_profile_pcg(const void* handle, const double* b, double tol, uint64_t maxit,
                        double* x, int32_t memory, lsamgdd_report* report,
                        lsamgdd_kernel_stats* stats, char* err, size_t errlen);

/* sym_eig (eigen.hpp:35-118) of one dense n×n row-major matrix through a
 * device path of the batched eigensolver: 0 warp team, 1 CTA team, 2 CTA
 * producer/consumer pipeline (cp.async-prefetched rows), 3 CTA pipeline with
 * one barrier per rotation, 4 thread-block-cluster wavefront (tiles staged by
 * 1-D bulk/TMA copies, rotation-log replay on helper CTAs; 2 <= n <= 608).
 * Values ascending, vectors column k. Used by the parity tests to pin each
 * path bit-for-bit against the reference. */
int lsamgdd_dense_sym_eig(int64_t n, const double* a, double* values, double* vectors, int32_t path, char* err,
                          size_t errlen);

/* Kernels this library has launched from the calling thread so far (graph
 * replays counted per captured kernel). The bench's gpu_launches claim. */
int64_t lsamgdd_launch_count(void);

/* Device memory: every buffer of the library comes from a memory pool it owns
 * (one per device, stream-ordered). Freed blocks stay mapped between calls, so
 * a second setup does not pay for mapping its workspaces again; the host
 * application's default pool and its release threshold are not touched. This
 * call synchronises the device and returns the cached, unused memory to the
 * driver (live hierarchies keep theirs). */
int lsamgdd_trim_memory(int32_t device);

/* ---- synthetic inputs (BASELINE.json configs) ---- */
/* mt19937_64(seed) + uniform_real_distribution(lo,hi), the CLI recipe of
 * lsamgdd_cli.cpp:103-107; host only. */
void lsamgdd_uniform(uint64_t seed, double lo, double hi, int64_t n, double* out);

/* On-device generator of a constant-coefficient grid factor (
 * the constructions of BASELINE configs 2, 3 and 5 — SURVEY.md Appendix A.1 —
 * and, with two rows per node, build_rotated_aniso of problems.hpp:106-132
 * with its gradient rows of problems.hpp:84-104). The factor is written
 * straight into device memory, so only the right-hand side crosses PCIe.
 *   grid[3]      extents (nx, ny, nz), x fastest; node = (z*ny + y)*nx + x
 *   offsets      [rows_per_node][max_entries][3] neighbour offsets (dx, dy, dz)
 *   coefs        [rows_per_node][max_entries]; an exact 0.0 is no entry
 * Row rows_per_node*node + k holds coefs[k][e] at column node + offset e for
 * every neighbour inside the grid (homogeneous Dirichlet closure), columns
 * ascending. rows_per_node, max_entries <= 8. *out_csr views device arrays
 * (memory = LSAMGDD_DEVICE) owned by *out_owner; pass it to lsamgdd_setup /
 * lsamgdd_pcg and release it with lsamgdd_generated_destroy afterwards. */
int lsamgdd_generate_stencil_rows(const int64_t grid[3], int32_t rows_per_node, int32_t max_entries,
                                  const int32_t* offsets, const double* coefs, int32_t device,
                                  void** out_owner, lsamgdd_csr* out_csr, char* err, size_t errlen);
/* Host copy of a generated factor (offsets n_rows+1, cols/values nnz; NULL skips an array). */
int lsamgdd_generated_export(const void* owner, int64_t* offsets, int64_t* cols, double* values, char* err,
                             size_t errlen);
int lsamgdd_generated_destroy(void* owner);

#ifdef __cplusplus
}
#endif

#endif /* LSAMGDD_B200_H */
