/*
 * aapdhg_cuda.h — C-ABI of the B200 (sm_100a) AA-PDHG / FAA-PDHG hot path.
 *
 * Plain C: pointers, sizes and POD structs only, no torch or C++ types.
 * Every entry point names the reference interface it replaces
 * (paths relative to the reference checkout, `proj/...`).
 *
 * Conventions
 *   - Host arrays passed in are borrowed for the duration of the call and
 *     copied to the device; output arrays are caller-allocated.
 *   - Iterates are stacked u = (x[n], y[m]) exactly as concat_iterate
 *     (proj/src/pdhg_core.cpp:94-98); y = (inequality rows m1, equality m2).
 *   - Return value is an aapdhg_status code; on error a NUL-terminated
 *     message is written to err (if err != NULL and errlen > 0).
 *     Codes map 1:1 onto the reference exception taxonomy
 *     (proj/include/aapdhg/errors.hpp:8-30).
 *   - A handle owns all device memory of one problem. It may be reused for
 *     many calls (sweeps) but must not be used from two threads at once;
 *     distinct handles are independent (re-entrant, no global mutable state).
 *   - No CPU fallback exists: every compute entry point runs CUDA kernels
 *     and fails with AAPDHG_ERR_CUDA when no sm_100 device is usable.
 */
#ifndef AAPDHG_CUDA_H_
#define AAPDHG_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AAPDHG_ABI_VERSION 3

/* Error codes (errors.hpp:8-30). */
typedef enum aapdhg_status {
  AAPDHG_OK = 0,
  AAPDHG_ERR_INPUT = 1,       /* InputError       */
  AAPDHG_ERR_DIMENSION = 2,   /* DimensionError   */
  AAPDHG_ERR_UNSUPPORTED = 3, /* UnsupportedError */
  AAPDHG_ERR_SINGULAR = 4,    /* SingularError    */
  AAPDHG_ERR_CUDA = 5,        /* runtime: CUDA / device */
  AAPDHG_ERR_INTERNAL = 6     /* runtime: anything else */
} aapdhg_status;

/* Method (solver.hpp:15). */
enum { AAPDHG_METHOD_PDHG = 0, AAPDHG_METHOD_AA = 1, AAPDHG_METHOD_FAA = 2 };

/* SolveStatus (solver.hpp:17-23), same order. */
enum {
  AAPDHG_SOLVE_RESIDUAL_TOL = 0,
  AAPDHG_SOLVE_KKT_TOL = 1,
  AAPDHG_SOLVE_MAX_ITERS = 2,
  AAPDHG_SOLVE_TIMEOUT = 3,
  AAPDHG_SOLVE_FIXED_POINT_START = 4
};

/* Reduction order of the norms / dot products on the device.
 *   SERIAL: every reduction summed in index order by one thread, exactly as
 *           vec.hpp:16-29 — with the CSR-ordered SpMV rows this reproduces the
 *           CPU reference bit for bit (iteration counts identical).
 *   TREE:   fixed-shape blocked tree reductions; deterministic run to run but
 *           rounding differs from the CPU in the last bits.
 *   AUTO:   SERIAL when n+m <= 65536, else TREE. */
enum { AAPDHG_REDUCE_AUTO = 0, AAPDHG_REDUCE_SERIAL = 1, AAPDHG_REDUCE_TREE = 2 };

/* CSR matrix, int32 row_ptr/col_idx + fp64 vals (sparse_linalg.hpp:18-28).
 * Column indices strictly increasing within a row. */
typedef struct aapdhg_csr_view {
  int32_t nrows;
  int32_t ncols;
  int64_t nnz;
  const int32_t* row_ptr; /* nrows + 1 */
  const int32_t* col_idx; /* nnz */
  const double* vals;     /* nnz */
} aapdhg_csr_view;

/* Four-block LP  min c'x  s.t. Gx >= h, Ax = b, l <= x <= u
 * given through K = [G; A] and q = [h; b] (lp_model.hpp:32-53). */
/* One (row, col, value) entry — the layout of the reference's Triplet
 * (proj/include/aapdhg/sparse_linalg.hpp:12-16). */
typedef struct aapdhg_triplet {
  int32_t row;
  int32_t col;
  double val;
} aapdhg_triplet;

typedef struct aapdhg_problem_view {
  aapdhg_csr_view k; /* (m1 + m2) x n */
  int32_t m1;        /* leading inequality rows of K */
  const double* c;   /* n */
  const double* q;   /* m1 + m2 */
  const double* l;   /* n, may hold -inf */
  const double* u;   /* n, may hold +inf */
} aapdhg_problem_view;

/* SolverConfig (solver.hpp:25-39) + AAParams (anderson.hpp:21-25)
 * + FilterParams (filtering.hpp:14-17), flattened. */
typedef struct aapdhg_solve_params {
  int32_t method;        /* AAPDHG_METHOD_* */
  int32_t reduction;     /* AAPDHG_REDUCE_* */
  uint64_t m;            /* memory capacity */
  double safeguard_d;    /* D */
  double safeguard_eps;  /* eps */
  double beta;
  const double* d_hat;   /* NULL = identity, else n + m entries > 0 */
  double eta;
  double c_s;
  double kappa_bar;
  double toll;
  double kkt_eps;
  int32_t kkt_terminate;
  int32_t pad0;
  uint64_t max_iters;
  double max_wall_seconds;
  double tau;            /* <= 0 (both) selects by power iteration */
  double sigma;
} aapdhg_solve_params;

/* TrajectoryRecord (solver.hpp:49-58). */
typedef struct aapdhg_record {
  uint64_t k;
  double g_norm;
  int32_t aa_step;
  int32_t pad0;
  uint64_t i;
  uint64_t j;
  double r_gap;
  double r_primal;
  double r_dual;
  double objective;
  double elapsed_s;
} aapdhg_record;

/* SolveResult (solver.hpp:60-73) minus the vectors (returned separately). */
typedef struct aapdhg_solve_result {
  int32_t status; /* AAPDHG_SOLVE_* */
  int32_t pad0;
  uint64_t iterations;
  uint64_t i;
  uint64_t j;
  uint64_t aa_failures;
  double g_norm;
  double r_gap;
  double r_primal;
  double r_dual;
  double objective;
  double tau;
  double sigma;
  double wall_seconds;
} aapdhg_solve_result;

/* Receives trajectory records in order, in chunks, during/after a solve. */
typedef void (*aapdhg_record_sink)(const aapdhg_record* recs, uint64_t count,
                                   void* ctx);

typedef struct aapdhg_handle aapdhg_handle;

/* Sharded (multi-GPU) solve, SURVEY.md §8(e) / DESIGN.md §8: the LP's rows
 * and columns are split into `world` contiguous nnz-balanced blocks; shard r
 * owns row block R_r (y, q, K x) and column block C_r (x, c, l, u).
 *   NCCL:     one shard per process (rank, world), one GPU each; all shards
 *             pass the same whole LP and the same 128-byte NCCL id (made by
 *             aapdhg_cuda_nccl_id on rank 0 and broadcast by the caller).
 *   LOOPBACK: all `world` shards in this process on `device`, exchanging by
 *             device copies (tests the partitioned path on one GPU).
 *   P2P:      as NCCL (same id, NCCL for setup and the non-iteration
 *             exchanges), but inside the iteration every producing kernel
 *             stores its chunk straight into every shard's buffer over
 *             peer memory (CUDA IPC, NVLink / NVSwitch) and each exchange is
 *             a flag barrier: no collective call on the iteration path.
 *             world <= 8.
 *   LOOPBACK_P2P: all shards in this process with the P2P exchanges (the
 *             peers are the in-process shards' buffers).
 * No reference counterpart: the reference solve() is single-threaded
 * (proj/src/solver.cpp:125-253); results match it within the TREE-mode
 * tolerance (scalar sums meet in rank order). */
enum {
  AAPDHG_DIST_NCCL = 0,
  AAPDHG_DIST_LOOPBACK = 1,
  AAPDHG_DIST_P2P = 2,          /* one shard per process; peer-memory exchanges */
  AAPDHG_DIST_LOOPBACK_P2P = 3  /* all shards in this process; peer-memory exchanges */
};
#define AAPDHG_NCCL_ID_BYTES 128
typedef struct aapdhg_dist_view {
  int32_t rank;       /* this process's shard (NCCL); ignored by LOOPBACK */
  int32_t world;      /* number of shards, 1 <= world <= min(n, m) */
  int32_t transport;  /* AAPDHG_DIST_* */
  int32_t pad0;
  const uint8_t* nccl_id; /* AAPDHG_NCCL_ID_BYTES bytes (NCCL only) */
} aapdhg_dist_view;

/* ---- library ------------------------------------------------------------ */

int aapdhg_cuda_abi_version(void);
/* Fills `out` with "<device name>, sm_XY, <SMs> SMs"; returns AAPDHG_ERR_CUDA
 * when no usable device is present. */
int aapdhg_cuda_device_info(char* out, size_t outlen);

/* ---- problem lifetime --------------------------------------------------- */

/* Uploads K, builds K' (CSR of the transpose, entries per column in ascending
 * row order so K'y matches matvec_transpose's row-ordered scatter,
 * proj/src/sparse_linalg.cpp:77-87) and the row-block schedules.
 * Replaces: constructing ProblemData for solve() (lp_model.hpp:34-53). */
int aapdhg_cuda_problem_create(const aapdhg_problem_view* prob, int device,
                               aapdhg_handle** out, char* err, size_t errlen);
int aapdhg_cuda_problem_destroy(aapdhg_handle* h);
/* Sizes of the uploaded problem: n, m1, m2, nnz. */
int aapdhg_cuda_problem_dims(const aapdhg_handle* h, int32_t* n, int32_t* m1,
                             int32_t* m2, int64_t* nnz);

/* ---- the solver --------------------------------------------------------- */

/* Replaces: SolveOutput solve(const ProblemData&, const SolverConfig&,
 *           const Iterate& u0)            proj/include/aapdhg/solver.hpp:93-96
 *           and solve(p, cfg) (u0 = 0)    proj/include/aapdhg/solver.hpp:98-99
 * x0/y0 may be NULL (zero start). x_out[n], y_out[m], lambda_out[n] may be
 * NULL. Records are streamed to `sink` (may be NULL). */
int aapdhg_cuda_solve(aapdhg_handle* h, const aapdhg_solve_params* prm,
                      const double* x0, const double* y0,
                      aapdhg_solve_result* res, double* x_out, double* y_out,
                      double* lambda_out, aapdhg_record_sink sink, void* ctx,
                      char* err, size_t errlen);

/* Replaces: StepSizes select_step_sizes(const ProblemData&, const SolverConfig&)
 *           proj/include/aapdhg/solver.hpp:89-91 (proj/src/solver.cpp:112-123) */
int aapdhg_cuda_select_step_sizes(aapdhg_handle* h,
                                  const aapdhg_solve_params* prm, double* tau,
                                  double* sigma, char* err, size_t errlen);

/* Replaces: double power_iteration_norm(const SparseMatrix&, int max_iters,
 *           double rel_tol, std::uint64_t seed)
 *           proj/include/aapdhg/sparse_linalg.hpp:44-47 (sparse_linalg.cpp:95-123)
 * The seeded start vector is drawn on the host (mt19937_64 +
 * uniform_real_distribution(-1, 1)) exactly as the reference does. */
int aapdhg_cuda_power_norm(aapdhg_handle* h, int32_t max_iters, double rel_tol,
                           uint64_t seed, int32_t reduction, double* out,
                           int32_t* rounds, char* err, size_t errlen);

/* ---- single-op entry points (per-kernel parity tests) ------------------- */

/* Replaces: matvec (sparse_linalg.hpp:34-35, sparse_linalg.cpp:60-69). */
int aapdhg_cuda_matvec(aapdhg_handle* h, const double* x, double* out,
                       char* err, size_t errlen);
/* Replaces: matvec_transpose (sparse_linalg.hpp:38-39, sparse_linalg.cpp:77-87). */
int aapdhg_cuda_matvec_transpose(aapdhg_handle* h, const double* y,
                                 double* out, char* err, size_t errlen);

/* Replaces: Iterate pdhg_step(const Iterate&, const ProblemData&,
 *           const StepSizes&)  proj/include/aapdhg/pdhg_core.hpp:33
 *           (proj/src/pdhg_core.cpp:45-63) */
int aapdhg_cuda_pdhg_step(aapdhg_handle* h, double tau, double sigma,
                          const double* x, const double* y, double* xn,
                          double* yn, char* err, size_t errlen);

/* Replaces: kkt_metrics(const Iterate&, const ProblemData&, const LambdaSpec&)
 *           proj/include/aapdhg/solver.hpp:85-87 (proj/src/solver.cpp:64-110)
 * kkt[0..2] = r_gap, r_primal, r_dual; kkt[3] = c'x. lambda may be NULL. */
int aapdhg_cuda_kkt_metrics(aapdhg_handle* h, int32_t reduction,
                            const double* x, const double* y, double* kkt,
                            double* lambda, char* err, size_t errlen);

/* Replaces: Vec aa_apply(const AAMemory&, const AAParams&, const Vec& u,
 *           const Vec& g)  proj/include/aapdhg/anderson.hpp:38-39
 *           (proj/src/anderson.cpp:106-135)
 * du_cols / dg_cols: p columns of length n+m, column-major, oldest first.
 * Returns AAPDHG_ERR_SINGULAR when the regularised Gram is not PD. */
int aapdhg_cuda_aa_apply(aapdhg_handle* h, int32_t reduction, int32_t p,
                         const double* du_cols, const double* dg_cols,
                         double beta, const double* d_hat, double eta,
                         const double* u, const double* g, double* out,
                         char* err, size_t errlen);

/* Replaces: build_filtered_memory (filtering.hpp:52-53, filtering.cpp:140-157)
 *           followed by filtered_aa_apply (filtering.hpp:57-58,
 *           filtering.cpp:159-181).
 * kept[p] receives 1 for columns that survive the angle + length filters.
 * Returns AAPDHG_ERR_SINGULAR as the reference throws SingularError. */
int aapdhg_cuda_filtered_aa_apply(aapdhg_handle* h, int32_t reduction,
                                  int32_t p, const double* e_cols,
                                  const double* f_cols, double c_s,
                                  double kappa_bar, double beta,
                                  const double* d_hat, const double* u,
                                  const double* g, double* out, int32_t* kept,
                                  char* err, size_t errlen);

/* Replaces: SparseMatrix::from_triplets (sparse_linalg.hpp:22-23,
 * sparse_linalg.cpp:11-42), and with row_map / row_neg the split of
 * to_standard_form (lp_model.cpp:232-291): CSR of `count` triplets built on
 * `device` — entries sorted by (row_map[row], col), duplicates summed left
 * to right in input order, exact cancellations kept as structural zeros.
 * row_map (nrows_in entries, may be null = identity) sends input rows to
 * output rows < nrows_out; row_neg (nrows_in, may be null) negates a row's
 * values. Outputs: row_ptr[nrows_out + 1], col_idx / vals with room for
 * `count` entries; *nnz receives the entry count. AAPDHG_ERR_DIMENSION for
 * an entry outside nrows_in x ncols. */
int aapdhg_cuda_csr_from_triplets(int32_t device, int32_t nrows_in, int32_t nrows_out,
                                  int32_t ncols, int64_t count, const aapdhg_triplet* triplets,
                                  const int32_t* row_map, const uint8_t* row_neg,
                                  int32_t* row_ptr, int32_t* col_idx, double* vals, int64_t* nnz,
                                  char* err, size_t errlen);

/* A handle for the per-op AA / FAA entries on vectors of length n (no LP:
 * the C++ drop-in's aa_apply / angle_filter / economy_qr ... of
 * anderson.hpp, filtering.hpp and sparse_linalg.hpp work on bare columns).
 * Destroy with aapdhg_cuda_problem_destroy. */
int aapdhg_cuda_workspace_create(int32_t device, int64_t n, aapdhg_handle** out, char* err,
                                 size_t errlen);

/* FAA steps of build_filtered_memory + filtered_aa_apply (filtering.hpp:
 * 20-59) on p columns (oldest first), with stages skipped by `skip`
 * (1: the angle filter, 2: the length filter). kept[p] receives the kept
 * set; when out is non-null the candidate u + beta Dhat g - sum w_j (e_j +
 * beta Dhat f_j) is formed (w from the double-double least squares of the
 * kept f). Replaces angle_filter / length_filter / build_filtered_memory's
 * selection and filtered_aa_apply (filtering.cpp:61-181). e_cols may be
 * null when only the kept set is wanted. */
int aapdhg_cuda_faa_op(aapdhg_handle* h, int32_t reduction, int32_t p, const double* e_cols,
                       const double* f_cols, double c_s, double kappa_bar, double beta,
                       const double* d_hat, int32_t skip, const double* u, const double* g,
                       double* out, int32_t* kept, char* err, size_t errlen);

/* Replaces: QRFactors economy_qr(const DenseMatrix& f)
 * (proj/include/aapdhg/sparse_linalg.hpp:67-69, sparse_linalg.cpp:131-192).
 * f_cols: p columns of length n (the handle's n). R (p x p, column-major,
 * upper, diag >= 0) from the Cholesky of the double-double Gram F'F; Q
 * (n x p, column-major) = F R^{-1}. AAPDHG_ERR_SINGULAR for rank-deficient
 * columns (the reference's Householder QR returns a zero r_ii there). */
int aapdhg_cuda_economy_qr(aapdhg_handle* h, int32_t reduction, int32_t p, const double* f_cols,
                           double* q_out, double* r_out, char* err, size_t errlen);

/* ---- streams & instrumentation (bench / profiling) ---------------------- */

/* Makes the handle enqueue all its work on `stream` (a cudaStream_t owned by
 * the caller, must not be the legacy default stream; NULL restores the
 * handle's own stream). Lets a caller bracket a solve with its own CUDA
 * events or order it after its own kernels. */
int aapdhg_cuda_set_stream(aapdhg_handle* h, void* stream);

/* Per-kernel device time accounting, measured with CUDA events recorded on
 * the handle's own stream around each launch. Enabling it switches the
 * solve loop from CUDA-graph replay to eager launches for that call. */
int aapdhg_cuda_set_profiling(aapdhg_handle* h, int32_t enable);
/* names: '\n'-separated kernel names; ms[k]/launches[k] accumulated totals
 * over the launches that did work (a launch under 30% of the kernel's longest
 * is taken for a device-predicated no-op and left out).
 * Returns the number of kernels in *count. */
int aapdhg_cuda_kernel_times(aapdhg_handle* h, char* names, size_t names_len,
                             double* ms, uint64_t* launches, int32_t cap,
                             int32_t* count);
/* Number of kernel launches issued by the last solve's iteration loop (graph
 * nodes counted individually) and the iterations it ran. */
int aapdhg_cuda_last_launch_count(aapdhg_handle* h, uint64_t* launches,
                                  uint64_t* loop_iterations);
/* The persistent plain-step kernel (k_plain_loop) in the last solve: the
 * iterations it completed, its device time (globaltimer from each launch's
 * start to its stop, summed) and its launches; zeros when the solve ran on
 * the per-kernel graph. Not for sharded handles. */
int aapdhg_cuda_last_plain_loop(aapdhg_handle* h, uint64_t* iterations, double* seconds,
                                uint64_t* launches);

/* ---- sharded solve ------------------------------------------------------ */

/* Fills out[0..AAPDHG_NCCL_ID_BYTES) with a fresh NCCL unique id.
 * AAPDHG_ERR_UNSUPPORTED when libnccl.so.2 cannot be loaded. */
int aapdhg_cuda_nccl_id(uint8_t* out, size_t len, char* err, size_t errlen);
/* k_plain_loop's calibrated partition (host only, no GPU needed; engine.cu
 * rebalance_partition): from the current slice starts per worker CTA
 * cur_starts[workers + 1], each worker's mean phase time phase_ns[workers], its
 * SM sm[workers] and the work of each slice slice_work[nslices], the new
 * starts (each SM's share in proportion to the rate it showed, <= 8 slices per
 * worker) in new_starts[workers + 1]. */
int aapdhg_cuda_balance_partition(int32_t workers, int32_t nslices, const int32_t* cur_starts,
                                  const double* phase_ns, const int32_t* sm,
                                  const int32_t* slice_work, int32_t* new_starts);
/* The row / column blocks a world-way sharded solve uses (host only, no GPU
 * needed): row_bounds[world + 1], col_bounds[world + 1]. */
int aapdhg_cuda_partition(const aapdhg_csr_view* k, int32_t world, int32_t* row_bounds,
                          int32_t* col_bounds);
/* Like aapdhg_cuda_problem_create, for one process's part of a sharded
 * solve. aapdhg_cuda_solve / aapdhg_cuda_select_step_sizes on the handle are
 * collective (every rank calls them with the same arguments) and return the
 * whole x, y, lambda and the same records on every rank. The single-op
 * entry points return AAPDHG_ERR_UNSUPPORTED on such a handle. */
int aapdhg_cuda_problem_create_dist(const aapdhg_problem_view* prob, int device,
                                    const aapdhg_dist_view* dist, aapdhg_handle** out,
                                    char* err, size_t errlen);

#ifdef __cplusplus
}
#endif

#endif /* AAPDHG_CUDA_H_ */
