/* gaplra_cuda — C ABI of the B200 (sm_100a) shift-and-invert hot path.
 *
 * Drop-in boundary for the reference `gaplra` library (arXiv 1607.02925,
 * /root/reference/proj/core).  Every entry point is extern "C", takes plain
 * pointers and sizes, never throws, and returns a gaplra_status; the message
 * of the last failure is gaplra_last_error(ctx).  Host d x p blocks are
 * ROW-MAJOR with leading dimension p, exactly the reference's DenseMatrix
 * (proj/core/include/gaplra/dense_matrix.hpp:22-23).  X is uploaded once and
 * stays resident in HBM (dense column-major, or CSC + a CSR copy).
 *
 * Entry point                          replaces (reference file:line)
 * -----------------------------------  -----------------------------------------------
 * gaplra_matrix_dense / _csc           SparseColumnsMatrix ctor + from_dense
 *                                      (sparse_matrix.hpp:23-25, sparse_matrix.cpp:10-49)
 * gaplra_gram_apply                    GramOperator::apply (linear_operator.hpp:56,
 *                                      linear_operator.cpp:23-29) = gram_apply
 *                                      (sparse_matrix.cpp:93-99)
 * gaplra_gram_block(_device)           p x GramOperator::apply in one X·(XᵀW) pass
 * gaplra_index_stream                  Rng(seed).uniform_index(n) x m (rng.cpp:61-69)
 * gaplra_gaussian_init                 gaussian_init (orthonormalize.hpp:12)
 * gaplra_qr_orthonormalize             qr_orthonormalize (orthonormalize.hpp:18)
 * gaplra_orthonormality_defect         orthonormality_defect (orthonormalize.hpp:25)
 * gaplra_jacobi_eigh                   jacobi_eigh (jacobi.hpp:19)
 * gaplra_svrg_epoch / gaplra_svrg_solve  solve_svrg (unshipped)
 * gaplra_estimate_top                  estimate_eigenvalues, k = 1
 * gaplra_tune_shift                    tune_shift
 * gaplra_restricted_projection         restricted_projection
 * gaplra_shift_invert                  Alg. 7 ShiftedInverse branch on I = {1..k}
 *                                      (SPEC.md:505-516,546-549 / PAPER.md:341-351)
 * gaplra_detect_*_gap                  Alg. 4 / Alg. 5
 * gaplra_estimate_eigenvalues          estimate_eigenvalues, any k
 * gaplra_approximate                   approximate = Alg. 7
 * gaplra_accsvrg_solve                 solve_accelerated_svrg
 * gaplra_cg_solve                      solve_cg / inverse_operator(cg)
 * gaplra_error_report                  error_report
 * gaplra_principal_angles              principal_angles
 */
#ifndef GAPLRA_CUDA_H
#define GAPLRA_CUDA_H

#include <stdint.h>

#if defined(__GNUC__)
#define GAPLRA_API __attribute__((visibility("default")))
#else
#define GAPLRA_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  GAPLRA_OK = 0,
  GAPLRA_CONTRACT_VIOLATION = 1,       /* gaplra::ContractViolation  (errors.hpp:17) */
  GAPLRA_RANK_DEFICIENT = 2,           /* gaplra::RankDeficient      (errors.hpp:23) */
  GAPLRA_INDEFINITE_SHIFT = 3,         /* gaplra::IndefiniteShift    (errors.hpp:40) */
  GAPLRA_SOLVER_STALLED = 4,           /* gaplra::SolverStalled      (errors.hpp:46) */
  GAPLRA_SHIFT_OUT_OF_RANGE = 5,       /* gaplra::ShiftOutOfRange    (errors.hpp:60) */
  GAPLRA_SHIFT_TUNING_STALLED = 6,     /* gaplra::ShiftTuningStalled (errors.hpp:73) */
  GAPLRA_NO_PRECONDITIONING_NEEDED = 7,/* SPEC.md:425 signal */
  GAPLRA_DEVICE_ERROR = 8,
  GAPLRA_OUT_OF_MEMORY = 9,
  GAPLRA_NO_USABLE_GAP = 10,           /* find_gap_budget */
  GAPLRA_DEGENERATE_PROGRESS = 11      /* gaplra::DegenerateProgress (errors.hpp:95-98) */
} gaplra_status;

typedef struct gaplra_ctx gaplra_ctx;
typedef struct gaplra_matrix gaplra_matrix;

/* SVRG parameters; layout identical to oracle/oracle.h. */
typedef struct {
  double eta;            /* <= 0: 1/(4(lambda + n max_j |x_j|^2)) */
  int64_t m;             /* <= 0: 2n steps per epoch */
  double tol;            /* stop when max_c |M_c| / |B_c| <= tol */
  int epoch_cap;         /* <= 0: ceil(200 ln(1/tol)) */
  double monotone_slack; /* > 0: stall if residual > slack * best so far */
  uint64_t root_seed;    /* stream = derive_seed(root, 0x73767267 ^ (solve_id << 20) ^ epoch) */
  double lambda1_hint;   /* > 0: upper estimate of lambda_1 for step sizing:
                            eta = min(eta, (lambda - hint) / (|X|_F^2 hint)) */
} gaplra_svrg_params;

/* CostLedger (linear_operator.hpp:16-30) plus epoch/outer counters. */
typedef struct {
  uint64_t gram_applies;
  uint64_t operator_applies;
  uint64_t qr_factorizations;
  uint64_t linear_solves;
  uint64_t solver_column_samples;
  uint64_t epochs;
  uint64_t outer_iterations;
} gaplra_ledger;

typedef struct {
  int k, p;
  double eps, mu;
  double delta;
  double lambda; /* > 0: explicit shift, skips tune_shift */
  uint64_t seed;
  double tol_solve, tol_tune, conv_tol, rq_tol;
  int max_outer;
  int force;
  int epoch_cap;
  double monotone_slack;
  double lambda1_hint; /* with an explicit lambda: upper estimate of lambda_1 (0: none) */
  int backend;         /* inverse_operator backend: 0 svrg, 1 cg, 2 accsvrg */
} gaplra_si_config;

typedef struct {
  double lambda;
  double lambda1_hat;
  double lambda1_hint;
  int tune_steps;
  double tune_lambda[64];
  double tune_inv[64];
  int outer_iterations;
  int outer_cap;
  gaplra_ledger ledger;
  /* device time per phase (CUDA events on the context stream), ms */
  double ms_tune, ms_subspace, ms_rayleigh_ritz, ms_total;
} gaplra_si_report;

/* Executed partition plan of gaplra_approximate (Alg. 7):
 * per interval {s..q}: strategy 0 PlainPower / 1 ShiftedInverse, block width,
 * subspace iterations, shift (0 for PlainPower). */
typedef struct {
  int n_intervals;
  int s[64], q[64], strategy[64], width[64], iterations[64];
  double shift[64];
  gaplra_ledger ledger;
  double ms_total;
  double delta; /* the gap budget used (supplied, or find_gap_budget's) */
} gaplra_ap_report;

/* Live per-kernel-class device time (CUDA events on the context stream) and
 * the algorithmic bytes / flops of those launches.
 * Classes: 0 gram pass X(XᵀW) (p > 1), 1 SVRG epoch chain (p > 1), 2 H = XᵀC
 * pass, 3 index stream, 4 QR (MGS2), 5 anchor epilogue, 6 per-block Gram/T
 * precompute (TT, M; run beside the previous epoch's chain), 7 gram pass
 * (p = 1), 8 SVRG epoch chain (p = 1), 9 per-block U coefficients. */
#define GAPLRA_PROF_CLASSES 12
typedef struct {
  double ms[GAPLRA_PROF_CLASSES];
  uint64_t count[GAPLRA_PROF_CLASSES];
  double bytes[GAPLRA_PROF_CLASSES];
  double flops[GAPLRA_PROF_CLASSES];
} gaplra_profile;

/* ---- context ---- */
GAPLRA_API int gaplra_ctx_create(int device, gaplra_ctx** out);
GAPLRA_API int gaplra_ctx_destroy(gaplra_ctx* ctx);
GAPLRA_API const char* gaplra_last_error(const gaplra_ctx* ctx);
GAPLRA_API int gaplra_ctx_set_stream(gaplra_ctx* ctx, void* cuda_stream); /* NULL = context's own stream */
GAPLRA_API int gaplra_ctx_synchronize(gaplra_ctx* ctx);
GAPLRA_API int gaplra_ledger_get(const gaplra_ctx* ctx, gaplra_ledger* out);
GAPLRA_API int gaplra_ledger_reset(gaplra_ctx* ctx);
GAPLRA_API int gaplra_version(void);
/* number of kernels this library has launched (process-wide; kernels replayed by
 * the device-resident epoch loop's CUDA graph are counted per execution) */
GAPLRA_API unsigned long long gaplra_launch_count(void);
/* times the host has waited on the context's stream (device-resident control:
 * a dense SVRG solve waits ~3 times, not once per epoch) */
GAPLRA_API unsigned long long gaplra_host_syncs(const gaplra_ctx* ctx);
GAPLRA_API int gaplra_profile_enable(gaplra_ctx* ctx, int on);
GAPLRA_API int gaplra_profile_get(gaplra_ctx* ctx, gaplra_profile* out);
GAPLRA_API int gaplra_profile_reset(gaplra_ctx* ctx);

/* ---- X (resident in HBM) ----
 * dense: column-major, ldx >= d.  on_device = 0: host pointer, copied in.
 *        on_device = 1: device pointer, BORROWED (caller keeps it alive, as
 *        GramOperator borrows X, linear_operator.hpp:53-60); requires
 *        ldx == round_up(d, 4) and rows [d, ldx) zero.
 *        Either way X is read once on the device at creation: a non-finite
 *        entry (sparse_matrix.cpp:29) or a non-zero pad row is a
 *        GAPLRA_CONTRACT_VIOLATION.
 * csc:   colptr[n+1], rowidx (strictly increasing per column), val. */
GAPLRA_API int gaplra_matrix_dense(gaplra_ctx* ctx, int d, int n, const double* x, int64_t ldx, int on_device,
                        gaplra_matrix** out);
GAPLRA_API int gaplra_matrix_csc(gaplra_ctx* ctx, int d, int n, const int64_t* colptr, const int32_t* rowidx,
                      const double* val, int on_device, gaplra_matrix** out);
GAPLRA_API int gaplra_matrix_destroy(gaplra_matrix* x);
GAPLRA_API int gaplra_matrix_info(const gaplra_matrix* x, int* d, int* n, int64_t* nnz, int64_t* ld);

/* ---- hot-path units (host buffers, row-major) ---- */
GAPLRA_API int gaplra_gram_apply(gaplra_ctx* ctx, const gaplra_matrix* x, const double* v, double* out);
GAPLRA_API int gaplra_gram_block(gaplra_ctx* ctx, const gaplra_matrix* x, int p, const double* w, double* z,
                      double* y /* nullable: X^T W, n x p */);
/* Device-resident variant: row-major device blocks with leading dimension ld*
 * (ldw, ldz even when p > 1), d_pad = round_up(d, 4) rows, zero pad rows. */
GAPLRA_API int gaplra_gram_block_device(gaplra_ctx* ctx, const gaplra_matrix* x, int p, const double* w, int64_t ldw,
                             double* z, int64_t ldz, double* y, int64_t ldy);
GAPLRA_API int gaplra_index_stream(gaplra_ctx* ctx, uint64_t seed, uint64_t n, int64_t m, int32_t* out);
GAPLRA_API int gaplra_gaussian_init(int d, int p, uint64_t seed, double* out);
GAPLRA_API int gaplra_qr_orthonormalize(gaplra_ctx* ctx, int d, int p, const double* y, double* q, int* bad_col);
GAPLRA_API int gaplra_orthonormality_defect(gaplra_ctx* ctx, int d, int p, const double* q, double* defect);
GAPLRA_API int gaplra_jacobi_eigh(gaplra_ctx* ctx, int n, const double* h, double* vals, double* vecs);
GAPLRA_API int gaplra_svrg_epoch(gaplra_ctx* ctx, const gaplra_matrix* x, int p, double* w, const double* y,
                      const double* c, double eta, double lambda, uint64_t stream_seed, int64_t m);
GAPLRA_API int gaplra_svrg_solve(gaplra_ctx* ctx, const gaplra_matrix* x, double lambda, int p, const double* b,
                      double* w, const gaplra_svrg_params* prm, int64_t solve_id, int* epochs,
                      double* history, int hist_cap, int* hist_len);
GAPLRA_API int gaplra_estimate_top(gaplra_ctx* ctx, const gaplra_matrix* x, int inverse, double lambda,
                        double eps_prime, uint64_t seed, double rq_tol, const gaplra_svrg_params* prm,
                        int64_t* solve_counter, double* value, int* iterations);
GAPLRA_API int gaplra_tune_shift(gaplra_ctx* ctx, const gaplra_matrix* x, double delta, const gaplra_si_config* cfg,
                      int64_t* solve_counter, gaplra_si_report* rep);
GAPLRA_API int gaplra_restricted_projection(gaplra_ctx* ctx, const gaplra_matrix* x, int p, const double* s, int k,
                                 double* w, double* ritz);
/* solve_cg: block CG on (lambda I - X Xᵀ) W = B from W = 0,
 * per-column recurrences, stop when max_c |r_c|/|b_c| <= tol; max_iter <= 0:
 * d + 10.  IndefiniteShift on nonpositive curvature. */
/* solve_accelerated_svrg: Catalyst outer loop around block
 * SVRG (kappa = sqrt(h (lambda - h)), h = prm->lambda1_hint required). */
GAPLRA_API int gaplra_accsvrg_solve(gaplra_ctx* ctx, const gaplra_matrix* x, double lambda, int p, const double* b,
                                    double* w, const gaplra_svrg_params* prm, int64_t solve_id, int* epochs,
                                    double* history, int hist_cap, int* hist_len);
GAPLRA_API int gaplra_cg_solve(gaplra_ctx* ctx, const gaplra_matrix* x, double lambda, int p, const double* b,
                               double* w, double tol, int max_iter, int* iterations, double* history, int hist_cap,
                               int* hist_len);
/* error_report: |X - W Wᵀ X|_F exactly (|X|_F^2 - |WᵀX|_F^2)
 * and the spectral norm by `iters` power iterations (seeded start). */
GAPLRA_API int gaplra_error_report(gaplra_ctx* ctx, const gaplra_matrix* x, int k, const double* w, int iters,
                                   uint64_t seed, double* frob, double* spec);
/* principal_angles: cosines (descending) between span(U),
 * U d x k orthonormal, and span(S), S d x p full column rank. */
GAPLRA_API int gaplra_principal_angles(gaplra_ctx* ctx, int d, int k, const double* u, int p, const double* s,
                                       double* cosines);
/* Alg. 4 detect_multiplicative_gap: est[i] = lambda_hat_{s+i};
 * *q = smallest global q with est_{q+1} <= est_q (1 - p^-2), or -1. */
GAPLRA_API int gaplra_detect_multiplicative_gap(const double* est, int count, int s, int p, int* q);
/* Alg. 5 detect_additive_gap: inv[i] = lambda~_{s+i}^-1;
 * GAPLRA_SHIFT_OUT_OF_RANGE unless inv[0] in [delta/27, delta/5]. */
GAPLRA_API int gaplra_detect_additive_gap(gaplra_ctx* ctx, const double* inv, int count, int s, int k, double delta,
                                          int* q);
/* estimate_eigenvalues (Alg. 3) for k <= 64 on A = X Xᵀ or D⁻¹. */
GAPLRA_API int gaplra_estimate_eigenvalues(gaplra_ctx* ctx, const gaplra_matrix* x, int inverse, double lambda, int k,
                                           double eps_prime, uint64_t seed, double rq_tol,
                                           const gaplra_svrg_params* prm, double* values, int* iterations);
/* approximate (Alg. 7) with the caller's gap budget cfg->delta:
 * W (d x k row-major), top-k Ritz values, the executed partition plan. */
/* find_gap_budget: delta from Alg. 3 estimates of lambda_k and
 * lambda_{p+1} at eps' = 1/100; GAPLRA_NO_USABLE_GAP without a gap. */
GAPLRA_API int gaplra_find_gap_budget(gaplra_ctx* ctx, const gaplra_matrix* x, int k, int p, uint64_t seed,
                                      double rq_tol, double* delta);
/* cfg->delta <= 0: the gap budget comes from gaplra_find_gap_budget. */
GAPLRA_API int gaplra_approximate(gaplra_ctx* ctx, const gaplra_matrix* x, const gaplra_si_config* cfg, double* w,
                                  double* ritz, gaplra_ap_report* rep);
GAPLRA_API int gaplra_shift_invert(gaplra_ctx* ctx, const gaplra_matrix* x, const gaplra_si_config* cfg, double* w,
                        double* ritz, double* s, gaplra_si_report* rep);

#ifdef __cplusplus
}
#endif

#endif /* GAPLRA_CUDA_H */
