/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the shift-and-invert hot path.
 *
 * A plain C ABI over oracle/oracle.cpp, a from-scratch CPU restatement of the
 * reference's algorithm for the north-star path (arXiv 1607.02925, `gaplra`):
 *   - shipped primitives, restated bit-for-bit (same loop and rounding order,
 *     no FMA contraction): xoshiro256++/splitmix64 Rng and uniform_index
 *     (proj/core/src/rng.cpp:9-76), gaussian_init (orthonormalize.cpp:12-21),
 *     two-pass MGS qr_orthonormalize (orthonormalize.cpp:25-79), cyclic
 *     jacobi_eigh (jacobi.cpp:13-109), gram_apply = spmv(spmv_transpose(v))
 *     (sparse_matrix.cpp:66-99), gram_with / multiply (dense_matrix.cpp:65-93);
 *   - spec-only pieces (SPEC.md has them, proj/ does not ship them), restated
 *     with every unpinned choice pinned here and in DESIGN.md §2: solve_svrg
 *     (SPEC.md:327-335,362-365), inverse_operator (:345-353), subspace_iterate
 *     (:234-242), estimate_eigenvalues (:254-262), restricted_projection
 *     (:244-252), tune_shift (:423-431), solve_cg (:317-325),
 *     error_report (:528-536), principal_angles (:181-189), Alg. 4/5 gap
 *     detection (:403-421), approximate = Alg. 7 (:505-551).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load this library, and only as the checker or the timed CPU
 * baseline — never as the product path.
 */
#ifndef GAPLRA_ORACLE_H
#define GAPLRA_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes — identical numbering to include/gaplra_cuda.h. */
enum {
  ORC_OK = 0,
  ORC_CONTRACT_VIOLATION = 1,
  ORC_RANK_DEFICIENT = 2,
  ORC_INDEFINITE_SHIFT = 3,
  ORC_SOLVER_STALLED = 4,
  ORC_SHIFT_OUT_OF_RANGE = 5,
  ORC_SHIFT_TUNING_STALLED = 6,
  ORC_NO_PRECONDITIONING_NEEDED = 7,
  ORC_NO_USABLE_GAP = 10, /* find_gap_budget */
  ORC_DEGENERATE_PROGRESS = 11 /* errors.hpp:95-98 */
};

/* X in R^{d x n}: kind 0 = dense column-major (ld = d), kind 1 = CSC
 * (colptr[n+1] int64, rowidx int32 strictly increasing per column, val). */
typedef struct {
  int kind;
  int d, n;
  const double* x;
  const int64_t* colptr;
  const int32_t* rowidx;
  const double* val;
} orc_mat;

typedef struct {
  double eta;            /* <= 0: 1/(4(lambda + n max_j |x_j|^2)) */
  int64_t m;             /* <= 0: 2n steps per epoch */
  double tol;            /* stop when max_c |M_c|/|B_c| <= tol          */
  int epoch_cap;         /* <= 0: ceil(200 ln(1/tol)) */
  double monotone_slack; /* > 0: stall if res_e > slack * min_{e'<e} res */
  uint64_t root_seed;    /* stream seed = derive_seed(root, TAG_SVRG ^ (solve_id<<20) ^ epoch) */
  double lambda1_hint;   /* > 0: upper estimate of lambda_1 used for step sizing:
                            eta = min(eta_spec, (lambda - hint) / (|X|_F^2 hint)) */
} orc_svrg_params;

typedef struct {
  uint64_t gram_applies;      /* per vector, as GramOperator::apply counts */
  uint64_t operator_applies;
  uint64_t qr_factorizations;
  uint64_t linear_solves;     /* per block solve */
  uint64_t solver_column_samples;
  uint64_t epochs;
  uint64_t outer_iterations;
} orc_ledger;

typedef struct {
  int k, p;
  double eps, mu;
  double delta;       /* gap budget for tune_shift (used when lambda <= 0) */
  double lambda;      /* explicit shift (> 0 skips tune_shift)            */
  uint64_t seed;
  double tol_solve;   /* inner SVRG tolerance of the main iteration        */
  double tol_tune;    /* inner SVRG tolerance inside tune_shift            */
  double conv_tol;    /* subspace early stop on |SS^T - S'S'^T|_F          */
  double rq_tol;      /* Alg. 3 early stop on relative Rayleigh change     */
  int max_outer;      /* <= 0: ceil(4 k ln(k d / eps_int))                 */
  int force;          /* ignore NoPreconditioningNeeded                    */
  int epoch_cap;      /* 0: spec cap                                       */
  double monotone_slack;
  double lambda1_hint; /* with an explicit lambda: upper estimate of lambda_1 (0: none) */
  int backend;         /* inverse_operator backend: 0 svrg, 1 cg, 2 accsvrg */
} orc_si_config;

typedef struct {
  double lambda;
  double lambda1_hat;
  double lambda1_hint; /* lambda_1 upper estimate handed to the main solves */
  int tune_steps;
  double tune_lambda[64];
  double tune_inv[64];
  int outer_iterations;
  int outer_cap;
  orc_ledger ledger;
} orc_si_report;

/* Executed partition plan of approximate (Alg. 7): per interval {s..q}, the
 * branch (0 PlainPower, 1 ShiftedInverse), block width, iterations, shift. */
typedef struct {
  int n_intervals;
  int s[64], q[64], strategy[64], width[64], iterations[64];
  double shift[64];
  orc_ledger ledger;
  double delta; /* the gap budget used (supplied, or find_gap_budget's) */
} orc_ap_report;

/* ---- primitives (bit-exact restatements) ---- */
uint64_t orc_derive_seed(uint64_t root, uint64_t tag);
void orc_next_u64(uint64_t seed, int64_t count, uint64_t* out);
void orc_uniform_index(uint64_t seed, uint64_t n, int64_t count, uint64_t* out);
void orc_normal(uint64_t seed, int64_t count, double* out);
int orc_gaussian_init(int d, int p, uint64_t seed, double* out_rowmajor);
int orc_qr(int d, int p, const double* in_rowmajor, double* out_rowmajor, int* bad_col);
int orc_jacobi(int n, const double* in_rowmajor, double* vals, double* vecs_rowmajor);
double orc_max_col_norm2(const orc_mat* x);

/* Z = X (X^T W) for a d x p row-major block, one gram_apply per column.
 * Optionally Y = X^T W (n x p row-major). */
int orc_gram_block(const orc_mat* x, int p, const double* w_rowmajor, double* z_rowmajor,
                   double* y_rowmajor, int nthreads);

/* One stochastic epoch (m steps) in lockstep form; W in/out row-major d x p,
 * Y row-major n x p, C row-major d x p.  idx_out (m entries) optional. */
int orc_svrg_epoch(const orc_mat* x, int p, double* w_rowmajor, const double* y_rowmajor,
                   const double* c_rowmajor, double eta, double lambda, uint64_t stream_seed,
                   int64_t m, uint64_t* idx_out, int nthreads);

/* Block SVRG solve of (lambda I - X X^T) W = B.  B, W row-major d x p.
 * history (capacity hist_cap) receives the residual per anchor. */
int orc_svrg_solve(const orc_mat* x, double lambda, int p, const double* b_rowmajor,
                   double* w_rowmajor, const orc_svrg_params* prm, int64_t solve_id,
                   int* epochs, double* history, int hist_cap, int* hist_len, int nthreads);

/* Alg. 3 with k = 1 on either A = X X^T (inverse = 0) or D^-1 (inverse = 1). */
int orc_estimate_top(const orc_mat* x, int inverse, double lambda, double eps_prime,
                     uint64_t seed, double rq_tol, const orc_svrg_params* prm,
                     int64_t* solve_counter, double* value, int* iterations,
                     orc_ledger* ledger, int nthreads);

int orc_tune_shift(const orc_mat* x, double delta, const orc_si_config* cfg,
                   int64_t* solve_counter, orc_si_report* rep, int nthreads);

/* S (d x p row-major, orthonormal) -> W = S U_k (d x k row-major), ritz[k]. */
int orc_restricted_projection(const orc_mat* x, int p, const double* s_rowmajor, int k,
                              double* w_rowmajor, double* ritz, int nthreads);

/* Full shift-and-invert pipeline on I = {1..k}: tune (or given lambda) ->
 * subspace_iterate(D^-1, p) -> restricted_projection(XX^T, S, k). */
int orc_shift_invert(const orc_mat* x, const orc_si_config* cfg, double* w_rowmajor,
                     double* ritz, double* s_rowmajor, orc_si_report* rep, int nthreads);

/* sin of the largest principal angle between range(U) (d x k, orthonormal)
 * and range(Q) (d x q, orthonormal), computed as |(I - QQ^T)U|_2. */
int orc_detect_multiplicative_gap(const double* est, int count, int s, int p);
int orc_detect_additive_gap(const double* inv, int count, int s, int k, double delta, int* q);
int orc_estimate_eigenvalues(const orc_mat* x, int inverse, double lambda, int k, double eps_prime, uint64_t seed,
                             double rq_tol, const orc_svrg_params* prm, double* values, int* iterations,
                             int nthreads);
int orc_find_gap_budget(const orc_mat* x, int k, int p, uint64_t seed, double rq_tol, double* delta, int nthreads);
int orc_approximate(const orc_mat* x, const orc_si_config* cfg, double* w_rowmajor, double* ritz,
                    orc_ap_report* rep, int nthreads);
int orc_accsvrg_solve(const orc_mat* x, double lambda, int p, const double* b_rowmajor, double* w_rowmajor,
                      const orc_svrg_params* prm, int64_t solve_id, int* epochs, double* history, int hist_cap,
                      int* hist_len, int nthreads);
int orc_cg_solve(const orc_mat* x, double lambda, int p, const double* b_rowmajor, double* w_rowmajor,
                 double tol, int max_iter, int* iterations, double* history, int hist_cap, int* hist_len,
                 int nthreads);
int orc_error_report(const orc_mat* x, int k, const double* w_rowmajor, int iters, uint64_t seed, double* frob,
                     double* spec);
int orc_principal_angles(int d, int k, const double* u_rowmajor, int p, const double* s_rowmajor,
                         double* cosines);
double orc_sin_theta(int d, int k, const double* u_rowmajor, int q, const double* q_rowmajor);

#ifdef __cplusplus
}
#endif

#endif
