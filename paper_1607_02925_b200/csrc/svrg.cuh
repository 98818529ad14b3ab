// SVRG epoch + anchor kernels (see svrg.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace gaplra_cuda {

struct EpochArgs {
  const double* X;  // dense column-major
  int64_t ldx;
  int d_pad, n;
  const int32_t* idx;  // m sampled columns
  int64_t m;
  double* W;  // row-major d_pad x ldw (in: anchor W̃, out: W after m steps)
  const double* C;
  int64_t ldw;
  const double* Y;  // n x ldy: Y_i = x_iᵀ W̃
  const double* H;  // n x ldy: H_i = x_iᵀ C
  int64_t ldy;
  const double* zcol;  // d_pad zeros (masked Gram columns)
  double* slab;     // per s-step block: [TT | M | (M2) | U(groups)] (launch_block_prep)
  int64_t slab_len;
  int slab_head;    // doubles before U: 2 B² (TT | M), 3 B² with the two-block lookahead (| M2)
  int p;
  double rho, eta_n;
  int rows_per_cta, stages, pc, groups;
  long long* dbg;  // optional per-CTA phase cycle counters (8 per CTA)
  int skip;        // debug ablation mask: 1 coef, 2 dots, 4 update (results invalid)
  int prefetch;    // chain producers: L2-prefetch the slices this many blocks ahead (0: off)
  // XG chains (cfg.xg): the group's all-reduce goes through L2 instead of DSMEM
  double* xg_slot;   // [kXgSlots][groups][cluster][NV] partials
  unsigned* xg_count;  // [groups][kXgSlots] arrivals, zeroed before each launch
  int fast_reducer;  // p = 1 DSMEM chain: TT / M columns preloaded in registers before the all-reduce wait
  int push_async;    // p = 1 DSMEM chain: partials pushed with st.async from registers (0: staged bulk copies)
  int ncl;           // clusters the rows are split over (2: paired clusters, k_svrg_chain_v3 at p = 1)
  int xg_ll;         // p = 1 XG chains: partials as 16-byte flag-in-data cells (xg_slot zeroed before each launch)
};

struct SparseEpochArgs {
  int d, n, p;
  const int64_t* colptr;
  const int32_t* rowidx;
  const double* val;
  const int32_t* idx;
  int64_t m;
  double* W;
  const double* C;
  int64_t ldw;
  const double* Y;
  int64_t ldy;
  double rho, eta_n;
};

struct EpochConfig {
  int cluster, pc, b, rows_per_cta, groups, stages;
  size_t smem;
  int xg = 0;  // 1: the `cluster` CTAs of a group are plain CTAs exchanging through L2 (no cluster launch)
  int nclusters = 1;  // p = 1: 2 = two paired clusters (pairwise L2 swap of the cluster sums; needs xg_slot)
  int la = 1;  // chain lookahead in s-step blocks (2: the p = 1 chain k_chain_p1_la2)
};
int slab_head(const EpochConfig& cfg);
// XG exchange buffers of an epoch layout (doubles / counters); 0 when !cfg.xg
size_t xg_slot_elems(const EpochConfig& cfg);
size_t xg_count_elems(const EpochConfig& cfg);

EpochConfig choose_epoch_config(int d_pad, int p);
// doubles of the per-block slabs of an m-step epoch
size_t epoch_slab_elems(int64_t m, const EpochConfig& cfg);
// Per-block coefficients that depend only on the index stream and X: TT and M
// (needs X, ldx, d_pad, idx, m, rho, eta_n, zcol, slab)
void launch_block_prep(const EpochArgs& a, const EpochConfig& cfg, cudaStream_t st);
// The epoch-dependent part U (needs idx, m, rho, p, Y, H, ldy and the slab's TT)
void launch_block_u(const EpochArgs& a, const EpochConfig& cfg, cudaStream_t st);
void launch_svrg_epoch_dense(const EpochArgs& a, const EpochConfig& cfg, cudaStream_t st);
void launch_svrg_epoch_sparse(const SparseEpochArgs& a, cudaStream_t st);
void read_chain_hops(long long* out);  // GAPLRA_EPOCH_TIMING: hop stamps of blocks 1000..1007 (p = 1 chain v3)
// Block-parallel sparse epoch (sparse_epoch.cu): steps per block, scratch ints
// (zeroed by the caller), and the launch (cooperative, one CTA per SM).
bool sparse_blocked_supported(int p);
int sparse_block_steps(int d, double col_nnz, int p);
size_t sparse_scratch_ints(int d, int bs, int max_col_nnz);
void launch_svrg_epoch_sparse_blocked(const SparseEpochArgs& a, int bs, int max_col_nnz, double* dbuf, int* ibuf,
                                      cudaStream_t st);

// Level-scheduled sparse epoch (sparse_levels.cu): the per-epoch symbolic plan
// (entries by row, coupled pairs by target step, dependency levels) is built by
// one kernel for all blocks, then a cooperative kernel runs b / solve / scatter
// per block.  `bytes` of scratch; the plan depends on (d, m, nnz per column).
struct SparseLevelPlan {
  int bs, ecap, rcap, pcap, scap, sym_ctas, d;
  int64_t nblk;
  size_t bytes;
  size_t off_meta, off_rows, off_rptr, off_ej, off_ev, off_pptr, off_pl, off_pv, off_lrec, off_lptr, off_cnt,
      off_off, off_pkey, off_b, off_u, off_dcb, off_yb, off_rho;
};
bool sparse_levels_supported(int p);
SparseLevelPlan sparse_levels_plan(int d, int64_t m, double col_nnz, int max_col_nnz);
void launch_svrg_epoch_sparse_levels(const SparseEpochArgs& a, const SparseLevelPlan& plan, void* scratch,
                                     cudaStream_t st);

// Device-resident control of a solve's epoch loop (a CUDA-graph WHILE node):
// after each anchor, k_epoch_control applies the host loop's tests to the
// residual (non-finite / <= tol / > slack x best / epoch cap), appends it to
// the history, derives the next epoch's index-stream seed and sets the loop
// condition.  status: 0 running, 1 converged, 2 non-finite, 3 stalled, 4 cap.
struct EpochCtl {
  double best;
  int e;       // index of the last anchor evaluated
  int status;
  unsigned long long next_seed;  // stream seed of epoch e + 1 (its k_block_prep runs in the next iteration)
};
void launch_epoch_control(const double* res, EpochCtl* ctl, double* hist, int hist_cap, double tol, double slack,
                          int cap, uint64_t root, int64_t solve_id, unsigned long long cond, cudaStream_t st);

// C = η(Z + B), per-column |λW − Z − B|; out_max = max_c |M_c| / bnorm_c
// (NaN if any is non-finite).  part needs anchor_parts(d) * 64 doubles.
int anchor_parts(int d);
void launch_anchor(const double* W, const double* Z, const double* Bm, int64_t ld, int d, int p, double lambda,
                   double eta, double* C, double* part, const double* bnorm, double* colnorm, double* out_max,
                   cudaStream_t st);

}  // namespace gaplra_cuda
