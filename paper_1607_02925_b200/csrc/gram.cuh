// X·(XᵀW) pass kernels (dense column-major fp64 and CSC/CSR sparse).
//
// Replaces the reference's per-vector GramOperator::apply
// (proj/core/src/linear_operator.cpp:23-29) = SparseColumnsMatrix::gram_apply
// = spmv(spmv_transpose(v)) (proj/core/src/sparse_matrix.cpp:66-99), applied
// p times for a d x p block, by two block kernels that read X once each:
//   xtw:  Y = Xᵀ W          (n x p, row-major, ldy)  — spmv_transpose for all p
//   xy :  Z = X Y           (d x p, column-major)    — spmv for all p
// Both are FP64-FMA bound for p >= 8 (arithmetic intensity p/2 FLOP/B).
// All reductions use a fixed order, so results are bitwise run-to-run stable.
#pragma once

#include "common.cuh"

namespace gaplra_cuda {

struct DenseX {
  const double* x;  // column-major, ld % 4 == 0, rows [d, ld) are zero
  int64_t ld;
  int d, n;
};

struct SparseX {
  int d, n;
  int64_t nnz;
  const int64_t* colptr;  // CSC (column access, as the reference stores X)
  const int32_t* rowidx;
  const double* val;
  const int64_t* rowptr;  // CSR copy (row access) for the gather-form Z = X Y
  const int32_t* colidx;
  const double* rval;
};

// Workspace for split reductions (grown by the caller).
struct GramWork {
  double* part = nullptr;
  size_t part_elems = 0;
};

// Workspace (doubles) the split reductions of a p-column pass need.
size_t gram_work_elems(const DenseX& X, int p);

// Y[j, c] (row-major, ldy) = sum_r X[r, j] W[r, c], c < p; W row-major (ldw
// even when p > 1), X.ld rows with zero pad rows.
void launch_xtw(const DenseX& X, const double* W, int64_t ldw, int p, double* Y, int64_t ldy,
                GramWork& work, cudaStream_t st);

// Z (row-major, ldz; X.ld rows) = X Y, Y row-major (ldy), p columns.
void launch_xy(const DenseX& X, const double* Y, int64_t ldy, int p, double* Z, int64_t ldz,
               GramWork& work, cudaStream_t st);

// Single-pass Z = X (Xᵀ W) and Y = Xᵀ W (X read once; cluster row split, W and
// Z resident on chip).  Fits when X.ld <= 16 * 256 and is the default where it
// measured faster (d <= 1024); gram_fused_applies says.
bool gram_fused_applies(const DenseX& X, int p);
void launch_gram_fused(const DenseX& X, const double* W, int64_t ldw, int p, double* Y, int64_t ldy, double* Z,
                       int64_t ldz, GramWork& work, cudaStream_t st);

// Single-pass p = 1 pass (X read once; 512-thread CTA per SM, a column pair in
// registers while its dots are reduced; w in shared memory and single columns
// above 4096 rows), X.ld <= 8192; gram_p1_applies says.
// Z == nullptr: Y = Xᵀ W only.
bool gram_p1_applies(const DenseX& X);
void launch_gram_p1(const DenseX& X, const double* W, int64_t ldw, double* Y, int64_t ldy, double* Z, int64_t ldz,
                    GramWork& work, cudaStream_t st);

void launch_xtw_sparse(const SparseX& X, const double* W, int64_t ldw, int p, double* Y,
                       int64_t ldy, cudaStream_t st);
void launch_xy_sparse(const SparseX& X, const double* Y, int64_t ldy, int p, double* Z,
                      int64_t ldz, cudaStream_t st);

// Per-column |x_j|^2 into out[n]; reduce_sum_max: out2 = {sum, max} (SVRG step size).
void col_norm2_dense(const DenseX& X, double* out, cudaStream_t st);
void col_norm2_sparse(const SparseX& X, double* out, cudaStream_t st);
// flags[0] = 1 (non-finite entry) | 2 (non-zero pad row d..ld-1); one read of X.
void check_dense(const DenseX& X, int* flags, cudaStream_t st);
void reduce_sum_max(const double* v, int n, double* out2, cudaStream_t st);

}  // namespace gaplra_cuda
