/*
 * mpg.h — C ABI of the B200-native shifted-solve engine (libmpg.so).
 *
 * Drop-in boundary for the reference `morprec` solve path
 * (/root/reference/proj/include/morprec). Every entry point below names the
 * reference interface it replaces. Plain pointers and sizes only; no torch or
 * Eigen types. Vector arguments documented as "any memory" may point to host
 * (pageable or pinned) or device memory of the handle's device: the library
 * resolves them through unified addressing and copies as needed.
 *
 * Threading: handles are immutable after creation (as SparseMatrix and
 * PrecondChain are, proj/include/morprec/sparse.hpp:29-32, chain.hpp:50-54)
 * and may be shared between host threads; each call is synchronous with
 * respect to the host and runs on the library's stream for the handle's
 * device (mpg_stream()).
 *
 * Errors: every int-returning call returns MPG_OK or one of the codes below;
 * mpg_last_error() gives the thread's last message. The reference raises
 * std::invalid_argument / ConfigError / SolverError
 * (proj/include/morprec/errors.hpp:12-28); GMRES non-convergence and
 * breakdown are report flags, not errors (proj/include/morprec/gmres.hpp:41-48).
 */
#ifndef MPG_H_
#define MPG_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPG_OK 0
#define MPG_ERR_INVALID 1 /* std::invalid_argument */
#define MPG_ERR_CONFIG 2  /* morprec::ConfigError  (CLI exit 2) */
#define MPG_ERR_SOLVER 3  /* morprec::SolverError  (CLI exit 3) */
#define MPG_ERR_LOGIC 4   /* std::logic_error, other */
#define MPG_ERR_CUDA 5    /* CUDA runtime failure / no device */
#define MPG_ERR_NOMEM 6   /* device allocation failed */
#define MPG_ERR_IO 7      /* morprec::IoError      (CLI exit 4) */

/* PrecondMode (proj/include/morprec/chain.hpp:21) + one extension. */
#define MPG_PRECOND_NONE 0
#define MPG_PRECOND_FRESH 1
#define MPG_PRECOND_REUSE_CHAIN 2
#define MPG_PRECOND_REUSE_FROZEN 3 /* build once at the first shift, apply unchanged afterwards */

/* PrecondKind (proj/include/morprec/report.hpp:14-20). */
#define MPG_KIND_NONE 0
#define MPG_KIND_FRESH 1
#define MPG_KIND_HORIZONTAL 2
#define MPG_KIND_VERTICAL 3
#define MPG_KIND_REUSED_SAME_MATRIX 4

typedef struct mpg_csr mpg_csr;     /* device CSR matrix (int32 indices, fp64 values) */
typedef struct mpg_op mpg_op;       /* shifted operator family sigma*E - A on one device */
typedef struct mpg_chain mpg_chain; /* immutable preconditioner chain P, Q_1..Q_L */

/* SpaiConfig (proj/include/morprec/spai.hpp:25-33); pattern_kind 0 = Diagonal,
 * 1 = PatternOfA (default). */
typedef struct {
  int pattern_kind, power;
  double fill_tol;
  int max_fill_per_col, max_pattern_sweeps, threads;
} mpg_spai_cfg;

/* GmresConfig (proj/include/morprec/gmres.hpp:20-24). */
typedef struct {
  double rel_tol;
  int max_iter, record_history;
} mpg_gmres_cfg;

/* GmresReport (proj/include/morprec/gmres.hpp:26-34); the residual history,
 * when recorded, is returned through a separate array. */
typedef struct {
  int iterations, converged, breakdown, history_len;
  double rhs_norm, final_residual, solve_seconds;
  int reorth_passes; /* iterations that needed the measured second Gram-Schmidt pass */
} mpg_gmres_report;

/* BirkaConfig (proj/include/morprec/birka.hpp:49-61) for N = 0; decoupled = 1
 * solves one GMRES per shift unit (the GPU path always does). */
typedef struct {
  int r;
  double tol;
  int max_sweeps;
  int decoupled;
  unsigned long long seed;
  mpg_gmres_cfg gmres;
  mpg_spai_cfg spai;
  int max_chain_len;
  long long explicit_nnz_cap, standard_residual_max_dim;
  int mirror_unstable; /* extension: reflect Re(lambda) > 0 into the left half plane before solving */
} mpg_irka_cfg;

/* ReportRow (proj/include/morprec/report.hpp:28-40). */
typedef struct {
  int sweep, point, kind, solves;
  long long iterations;
  double build_seconds, gmres_seconds, min_residual, matrix_change, standard_residual;
} mpg_report_row;

/* Per-solve record of the multi-shift batch (one row per solve). */
typedef struct {
  double sigma_re, sigma_im;
  int transpose, chain_length;
  mpg_gmres_report report;
} mpg_solve_record;

/* ---- errors, devices, streams ------------------------------------------- */
const char* mpg_last_error(void);
int mpg_device_count(int* count);
/* The library stream used for `device` (a cudaStream_t), for event timing. */
int mpg_stream(int device, void** stream);
int mpg_synchronize(int device);
/* Kernels launched by this library since load (for gpu_launches accounting). */
long long mpg_launch_count(void);
/* cudaMemcpy with unified addressing (host or device pointers). */
int mpg_copy(void* dst, const void* src, int64_t bytes);
/* Kernel-class profile of the GMRES engine: when enabled (and reset), GMRES
 * launches each iteration's kernels directly, bracketed by CUDA events on the
 * library stream, and accumulates per class the launch count, device time and
 * algorithmic bytes. Profiled solves are slower; the bench
 * runs one profiled step after the timed region. */
void mpg_profile_enable(int on);
int mpg_profile_count(void);
int mpg_profile_read(int kind, const char** name, long long* launches, double* ms, double* bytes);

/* ---- matrices: SparseMatrix (proj/include/morprec/sparse.hpp:33-101) -----
 * from_csr validates like SparseMatrix::from_csr (sparse.cpp:48-74):
 * nondecreasing offsets, in-range and strictly increasing columns. */
int mpg_csr_create(int device, int64_t nrows, int64_t ncols, const int64_t* rowptr, const int64_t* colind,
                   const double* values, mpg_csr** out);
void mpg_csr_destroy(mpg_csr* m);
int mpg_csr_info(const mpg_csr* m, int64_t* nrows, int64_t* ncols, int64_t* nnz);
/* Copies the CSR arrays back to host buffers (rowptr: nrows+1, colind/values: nnz). */
int mpg_csr_download(const mpg_csr* m, int64_t* rowptr, int64_t* colind, double* values);
/* y = A x / y = A^T x (SparseMatrix::multiply / multiply_transpose, sparse.cpp:236-269);
 * x, y any memory. */
int mpg_csr_multiply(const mpg_csr* m, const double* x, double* y);
int mpg_csr_multiply_transpose(const mpg_csr* m, const double* x, double* y);
/* SparseMatrix::transpose (sparse.cpp:289-299), built on the device. */
int mpg_csr_transpose(const mpg_csr* m, mpg_csr** out);
double mpg_csr_frobenius_norm(const mpg_csr* m);

/* ---- shifted operator: replaces linear_combination(sigma*D, -K)
 * (proj/src/qbihomm.cpp:164-171, sparse.cpp:156-202) and the N = 0
 * KroneckerOperator::apply (proj/src/kron.cpp:34-64) — sigma*E - A is formed
 * on the fly, never materialised. E == NULL means the identity (the
 * reference's BIRKA case); diagonal E and E sharing A's pattern get fused
 * fast paths. */
int mpg_op_create(const mpg_csr* a, const mpg_csr* e, mpg_op** out);
void mpg_op_destroy(mpg_op* op);
int64_t mpg_op_dim(const mpg_op* op);
/* Real shift (sigma_im == 0): y = (sigma E - A) x on n-vectors. Complex pair
 * (sigma_im != 0): the real 2x2-block form of the reference's Kronecker
 * operator on [x1; x2] (2n-vectors):
 *   [ sigma_re E - A   sigma_im E      ] [x1]
 *   [ -sigma_im E      sigma_re E - A  ] [x2]
 * with sigma = -lambda for the block [[a, b], [-b, a]] (proj/src/birka.cpp:117).
 * transpose != 0 uses A^T and E^T in the same form (the reference's test side,
 * birka.cpp:198). x, y any memory. */
int mpg_op_apply(const mpg_op* op, double sigma_re, double sigma_im, int transpose, const double* x, double* y);
/* Explicit unit matrix of the operator above (input of the SPAI builds), the
 * N = 0 block of assemble_explicit (proj/src/kron.cpp:72-131). */
int mpg_op_explicit(const mpg_op* op, double sigma_re, double sigma_im, int transpose, mpg_csr** out);

/* ---- preconditioner builds ------------------------------------------------
 * spai_build (proj/src/spai.cpp:175-238): warp-per-column adaptive SPAI.
 * column_residuals (nrows doubles, host) may be NULL. */
int mpg_spai_build(const mpg_csr* a, const mpg_spai_cfg* cfg, mpg_csr** p, double* column_residuals,
                   int64_t* fallback_count, double* build_seconds);
/* spai_column_solve (proj/src/spai.cpp:158-173): fixed-pattern column solve. */
int mpg_spai_column_solve(const mpg_csr* a, int64_t col, int64_t npattern, const int64_t* pattern, double* values,
                          double* residual, int* rank_deficient);
/* update_build (proj/src/chain.cpp:16-98): Q = argmin ||A_prev - A_new Q||_F. */
int mpg_update_build(const mpg_csr* a_prev, const mpg_csr* a_new, const mpg_spai_cfg* cfg, mpg_csr** q,
                     double* min_residual, double* matrix_change, int64_t* fallback_count, double* build_seconds);

/* ---- chains: PrecondChain (proj/include/morprec/chain.hpp:55-77) ----------
 * Immutable and reference counted; extend shares the prefix factors. */
int mpg_chain_create(const mpg_csr* base, mpg_chain** out);
int mpg_chain_extend(const mpg_chain* chain, const mpg_csr* q, mpg_chain** out);
void mpg_chain_destroy(mpg_chain* chain);
int mpg_chain_length(const mpg_chain* chain);
/* Identity of factor i (0 = base): the same pointer for shared prefixes. */
const void* mpg_chain_factor_id(const mpg_chain* chain, int i);
/* out = Q_L(...Q_1(P in)) (chain.cpp:117-126); x, y any memory. */
int mpg_chain_apply(const mpg_chain* chain, const double* x, double* y);
/* ||I - A P||_F / sqrt(n) (chain.cpp:140-157), probing n columns. */
int mpg_standard_residual(const mpg_csr* a, const mpg_chain* chain, double* out);

/* ---- GMRES: gmres_right_preconditioned (proj/src/gmres.cpp:40-186) --------
 * Full right-preconditioned GMRES, x0 = 0, with the reference's control flow
 * (Gram-Schmidt + measured second pass at 1e-10, invariance at 1e-14, true
 * residual recheck with the 0.25 back-off). chain == NULL is the identity.
 * history (max_iter+1 doubles, host) may be NULL. b, x any memory. */
int mpg_gmres_csr(const mpg_csr* m, const mpg_chain* chain, const double* b, double* x, const mpg_gmres_cfg* cfg,
                  mpg_gmres_report* report, double* history);
int mpg_gmres_shifted(const mpg_op* op, double sigma_re, double sigma_im, int transpose, const mpg_chain* chain,
                      const double* b, double* x, const mpg_gmres_cfg* cfg, mpg_gmres_report* report,
                      double* history);
/* Multi-shift batch: nsolves independent solves advanced in lockstep on one
 * device (shared launches, per-solve state). chains[i] may be NULL. */
int mpg_gmres_batch(const mpg_op* op, int nsolves, const double* sigma_re, const double* sigma_im,
                    const int* transpose, const mpg_chain* const* chains, const double* const* b, double* const* x,
                    const mpg_gmres_cfg* cfg, mpg_gmres_report* reports);

/* ---- IRKA: birka_reduce with N = 0 (proj/src/birka.cpp:139-310),
 * generalised to E (E_r = W^T E V, A_r = W^T A V, K_r = E_r^{-1} A_r);
 * one GMRES per shift unit, V/W by CholQR2 on the device.
 * Inputs b (n x m) and c (n x q) column-major, any memory. init_shifts
 * (r doubles) sets K_r = diag(-init_shifts) with fr/cr from the default-seed
 * stream (birka.cpp:41-89); NULL uses the default seed entirely.
 * Outputs (host, any may be NULL): kr, er, ar (r x r), fr (r x m), cr (r x q),
 * lambda (r), v, w (n x r). */
int mpg_irka_reduce(const mpg_op* op, const double* b, int m, const double* c, int q, const mpg_irka_cfg* cfg,
                    int mode, const double* init_shifts, double* kr, double* fr, double* cr, double* er, double* ar,
                    double* lam_re, double* lam_im, double* v, double* w, int* sweeps, int* converged,
                    mpg_report_row* rows, int max_rows, int* nrows);

/* The same from a caller-supplied initial reduced state: birka_reduce's
 * `const BirkaState* init` argument (proj/include/morprec/birka.hpp:78-80,
 * proj/src/birka.cpp:145). init_kr (r x r), init_fr (r x m), init_cr (r x q)
 * column-major on the host; a NULL part keeps the default seed's
 * (birka.cpp:41-89). A K_r with complex-conjugate eigenvalue pairs starts
 * the iteration at complex shifts. */
int mpg_irka_reduce_from(const mpg_op* op, const double* b, int m, const double* c, int q, const mpg_irka_cfg* cfg,
                         int mode, const double* init_kr, const double* init_fr, const double* init_cr, double* kr,
                         double* fr, double* cr, double* er, double* ar, double* lam_re, double* lam_im, int* sweeps,
                         int* converged, mpg_report_row* rows, int max_rows, int* nrows);

/* BIRKA with couplings N_1..N_m (birka_reduce, proj/src/birka.cpp:139-310;
 * the coupled path is the reference's joint solve): per sweep and side one
 * GMRES of order n r on the explicitly assembled Kronecker operator
 * -(Lambda (x) I) - (I (x) K) - sum_j (S_j^T (x) N_j) (kron.cpp:72-131),
 * preconditioned per `mode` with a vertical chain per side; a side whose
 * assembly would exceed cfg->explicit_nnz_cap continues unpreconditioned
 * with a warning (birka.cpp:214-236). n_ops: m CSR handles (n x n) on k's
 * device. Outputs as mpg_irka_reduce plus nr (m blocks of r x r,
 * column-major); warnings: malloc'ed text (mpg_buffer_free), may be NULL. */
int mpg_birka_reduce(const mpg_csr* k, const mpg_csr* const* n_ops, const double* b, int m, const double* c, int q,
                     const mpg_irka_cfg* cfg, int mode, double* kr, double* nr, double* fr, double* cr,
                     double* lam_re, double* lam_im, double* v, double* w, int* sweeps, int* converged,
                     mpg_report_row* rows, int max_rows, int* nrows, char** warnings);

/* IRKA projection (birka.cpp:283-291, generalised to E): E_r = W^T E V and
 * A_r = W^T A V (r x r, column-major, host) for V, W (n x r, column-major, any
 * memory); r <= 32. With E = I, E_r = W^T V as in the reference. */
int mpg_project(const mpg_op* op, const double* v, const double* w, int r, double* er, double* ar);

/* Multi-GPU IRKA: this process (rank of world) solves its shard of the
 * (unit, side) solves; `allgather` (provided by the caller, e.g. NCCL through
 * torch.distributed) concatenates per-rank byte buffers; buffers are device
 * pointers of this rank's device. */
typedef int (*mpg_allgather_fn)(void* ctx, const void* send, void* recv, int64_t bytes_per_rank);
int mpg_irka_reduce_sharded(const mpg_op* op, const double* b, int m, const double* c, int q,
                            const mpg_irka_cfg* cfg, int mode, const double* init_shifts, int rank, int world,
                            mpg_allgather_fn allgather, void* ctx, double* kr, double* fr, double* cr,
                            double* lam_re, double* lam_im, int* sweeps, int* converged, mpg_report_row* rows,
                            int max_rows, int* nrows);

/* Owner map used by mpg_irka_reduce_sharded (identical on every rank): units
 * (cost[i], or fixed[i] >= 0 to pin a unit to a rank) placed longest-first on
 * the least-loaded rank. cost of a unit = width * K * (K + 40) from its
 * slot's previous-sweep iterations K (mpg_shard_cost; K < 0: unknown). */
double mpg_shard_cost(int width, int last_iterations);
int mpg_shard_plan(int nunits, const double* cost, const int* fixed, int world, int* owner);

/* Native exchange: an NCCL communicator owned by the library (NCCL bound at
 * run time, libnccl.so.2). Rank 0 makes the id with mpg_comm_unique_id, the
 * caller's rendezvous hands it to every rank, each rank calls
 * mpg_comm_create on its device. mpg_comm_allgather is an mpg_allgather_fn:
 * pass (mpg_comm_allgather, comm) to mpg_irka_reduce_sharded and the V/W
 * columns move device to device on the library stream (ncclAllGather). */
typedef struct mpg_comm mpg_comm;
#define MPG_COMM_ID_BYTES 128
int mpg_comm_unique_id(char* id, int len);
int mpg_comm_create(int device, int rank, int world, const char* id, mpg_comm** out);
int mpg_comm_destroy(mpg_comm* comm);
int mpg_comm_allgather(void* comm, const void* send, void* recv, int64_t bytes_per_rank);
int mpg_comm_stats(const mpg_comm* comm, long long* calls, double* bytes);
int mpg_nccl_version(int* version);

/* ---- shift sweep: run_spai_bench (proj/src/bench.cpp:159-249) for
 * sigma_i E - A with a horizontal chain (fresh at i == 0 or when the chain
 * would exceed max_chain_len). Non-convergence is recorded, not raised.
 * x_out (n x npoints, any memory) may be NULL. */
int mpg_spai_bench(const mpg_op* op, const double* b, int npoints, const double* points, const mpg_spai_cfg* spai,
                   const mpg_gmres_cfg* gmres, int mode, int max_chain_len, double* x_out, mpg_report_row* rows,
                   int max_rows, int* nrows, int* failed);

/* ---- QB-IHOMM: qbihomm_reduce (proj/src/qbihomm.cpp:144-208) -------------
 * QbConfig (proj/include/morprec/qbihomm.hpp:35-43). */
typedef struct {
  int p_moments, q_moments;
  mpg_gmres_cfg gmres;
  mpg_spai_cfg spai;
  int max_chain_len;
  long long standard_residual_max_dim;
} mpg_qb_cfg;

/* D x' = K x + H (x (x) x) + N x u + F u, y = C^T x (SISO). `op` is the
 * shifted family built by mpg_op_create(K, D) (A = K, E = D; D may be NULL =
 * identity); n_op = N; H (n x n^2) as host triplets (row a, column b n + c,
 * value; duplicates summed). f, c: n-vectors, any memory. Trial side solves
 * (sigma_i D - K) x = F and p + q further moments against D x_prev; test side
 * (2 sigma_i D - K)^T y = C and q moments against D^T y_prev; the union basis
 * U (two-pass MGS with deflation, orth.cpp:16-40) gives the reduced model
 * U^T D U, U^T K U, U^T N U, U^T H (U (x) U) (r x r^2), U^T F, U^T C.
 * Outputs for order r <= max_order (host; basis n x r any memory; any may be
 * NULL). Non-convergence raises MPG_ERR_SOLVER (qbihomm.cpp:120-129). */
int mpg_qbihomm_reduce(const mpg_op* op, const mpg_csr* n_op, int64_t h_nnz, const int64_t* h_row,
                       const int64_t* h_col, const double* h_val, const double* f, const double* c, int npoints,
                       const double* sigmas, const mpg_qb_cfg* cfg, int mode, int max_order, int* order,
                       double* basis, double* red_d, double* red_k, double* red_n, double* red_h, double* red_f,
                       double* red_c, mpg_report_row* rows, int max_rows, int* nrows);

/* ---- host CSR / system structs (Matrix Market IO, triplet ingestion) -------- */
typedef struct {
  int64_t nrows, ncols, nnz;
  int64_t* rowptr;
  int64_t* colind;
  double* val;
} mpg_host_csr;

typedef struct {
  int64_t n;
  mpg_host_csr* a; /* A (n x n) */
  mpg_host_csr* e; /* E as CSR, or NULL */
  double* e_diag;  /* diagonal E, or NULL (both NULL: identity) */
  int m, q, r;
  double* b; /* n x m column-major */
  double* c; /* n x q column-major */
  double* shifts; /* r initial shifts */
} mpg_host_system;

void mpg_host_csr_free(mpg_host_csr* m);
/* SparseMatrix::from_triplets (proj/src/sparse.cpp:80-115): sorted row-major,
 * duplicates summed, exact-zero sums kept; out-of-range indices are
 * MPG_ERR_INVALID. The result is freed with mpg_host_csr_free. */
int mpg_host_csr_from_triplets(int64_t nr, int64_t nc, int64_t nnz, const int64_t* ri, const int64_t* ci,
                               const double* v, mpg_host_csr** out);

/* ---- transfer_function_error (proj/src/airga.cpp:386-447) ---------------------
 * Relative error ||H(s) - H_r(s)||_F / ||H(s)||_F on a grid for the
 * second-order model M x'' + D x' + K x = F u, y = C^T x, against a reduced
 * model (host, column-major: r x r m, d, k; r x n_in f; r x n_out c). The
 * full-order H(s) = C^T (s^2 M + s D + K)^{-1} F runs through the GPU solver
 * stack with one preconditioner per mode (none, fresh, horizontal chain along
 * the grid); errors[g] is NaN for s <= 0, failed solves, a singular reduced
 * pencil or H(s) = 0. f (n x n_in), c (n x n_out) column-major, any memory. */
int mpg_transfer_function_error(const mpg_csr* m, const mpg_csr* d, const mpg_csr* k, const double* f, int n_in,
                                const double* c, int n_out, const double* red_m, const double* red_d,
                                const double* red_k, const double* red_f, const double* red_c, int r,
                                const double* grid, int ngrid, const mpg_gmres_cfg* gmres, const mpg_spai_cfg* spai,
                                int mode, int max_chain_len, double* errors, long long* total_iterations);

/* ---- AIRGA: airga_reduce (proj/src/airga.cpp:136-317) -----------------------
 * AirgaConfig (proj/include/morprec/airga.hpp:43-62). */
typedef struct {
  int r_max;
  double outer_tol, inner_tol;
  int max_outer;
  mpg_gmres_cfg gmres;
  mpg_spai_cfg spai;
  int max_chain_len;
  long long standard_residual_max_dim;
} mpg_airga_cfg;

/* Moment-matching reduction of M x'' + D x' + K x = F u, y = C^T x over
 * adaptively refreshed expansion points; alpha, beta are the stored damping
 * coefficients (a warning is recorded when D deviates from alpha M + beta K).
 * The full-order solves run on the device (s^2 M + s D + K formed on the
 * fly from the merged pattern); the r x r reduced model, the H2 gaps and the
 * expansion-point update on the host. Outputs (host, column-major, order r <=
 * max_order = cfg->r_max): red_m/d/k (r x r), red_f (r x n_in), red_c
 * (r x n_out), basis (n x r, any memory, may be NULL), final_points (npoints);
 * warnings: '\n'-separated text in a malloc'ed buffer (mpg_buffer_free). */
int mpg_airga_reduce(const mpg_csr* m, const mpg_csr* d, const mpg_csr* k, const double* f, int n_in, const double* c,
                     int n_out, double alpha, double beta, const double* points, int npoints,
                     const mpg_airga_cfg* cfg, int mode, int* order, double* red_m, double* red_d, double* red_k,
                     double* red_f, double* red_c, double* basis, double* final_points, int* sweeps, int* converged,
                     mpg_report_row* rows, int max_rows, int* nrows, char** warnings);

/* update_expansion_points (airga.cpp:319-384) on a reduced pencil (host, r x r). */
int mpg_update_expansion_points(const double* m, const double* d, const double* k, int r, const double* current,
                                int ncurrent, double* next);
/* h2_norm (proj/src/h2.cpp:28-60) of x' = A x + B u, y = C x (host, column-major). */
int mpg_h2_norm(const double* a, const double* b, const double* c, int ns, int m, int q, double* out);

/* ---- Matrix Market IO (proj/src/matrix_market.cpp) and the report CSV
 * (proj/src/report.cpp:46-63); host-side, no device needed. --------------------
 * read_matrix_market / _file: coordinate real general|symmetric, symmetric
 * expanded, duplicates summed; malformed input fails with MPG_ERR_IO and
 * "origin:line: what". threads <= 0: all host threads (parsing and CSR
 * assembly run in parallel; results are independent of the thread count).
 * write_matrix_market: general, row-major, shortest round-trip values; dense
 * blocks store every entry. Text buffers are malloc'ed; free with mpg_buffer_free. */
int mpg_mm_read_file(const char* path, int threads, mpg_host_csr** out);
int mpg_mm_read_buffer(const char* data, int64_t len, const char* origin, int threads, mpg_host_csr** out);
int mpg_mm_write_file(const char* path, const mpg_host_csr* a, int threads);
int mpg_mm_write_buffer(const mpg_host_csr* a, int threads, char** out, int64_t* len);
int mpg_mm_write_dense_buffer(int64_t rows, int64_t cols, const double* colmajor, char** out, int64_t* len);
int mpg_report_csv(const mpg_report_row* rows, int nrows, char** out, int64_t* len);
void mpg_buffer_free(char* p);

#ifdef __cplusplus
}
#endif

#endif /* MPG_H_ */
