// TEST INFRASTRUCTURE ONLY — never linked into the product path.
//
// A thin extern "C" shim over the *reference's own* shipped sources
// (/root/reference/proj/core/src/*.cpp), compiled with -Dgaplra=gaplra_ref by
// oracle/Makefile into oracle/_ref/libgaplra_ref.so.  It lets the Python test
// suite pin oracle/oracle.cpp (our CPU restatement) against the reference's
// real arithmetic: RNG bit streams, gaussian_init, two-pass MGS, cyclic Jacobi,
// gram_apply, and an SVRG epoch built *only* from the reference's primitives
// (Rng::uniform_index + SparseColumnsMatrix::column_dot/column_axpy), which is
// how SPEC.md:362 prescribes the (unshipped) solver.
//
// Nothing here is copied from the reference: it only calls its public API
// (declared in proj/core/include/gaplra/*.hpp).

#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "gaplra/dense_matrix.hpp"
#include "gaplra/errors.hpp"
#include "gaplra/jacobi.hpp"
#include "gaplra/linear_operator.hpp"
#include "gaplra/orthonormalize.hpp"
#include "gaplra/rng.hpp"
#include "gaplra/sparse_matrix.hpp"

using namespace gaplra;  // expands to gaplra_ref under -Dgaplra=gaplra_ref

namespace {

SparseColumnsMatrix make_dense(int d, int n, const double* x_colmajor) {
  // from_dense() drops exact zeros (sparse_matrix.cpp:39-49); build the
  // row-major DenseMatrix it expects from our column-major buffer.
  DenseMatrix m(d, n);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < d; ++i) m(i, j) = x_colmajor[static_cast<size_t>(j) * d + i];
  return SparseColumnsMatrix::from_dense(m);
}

SparseColumnsMatrix make_csc(int d, int n, const int64_t* colptr, const int32_t* rowidx,
                             const double* val) {
  std::vector<std::vector<SparseEntry>> cols(n);
  for (int j = 0; j < n; ++j)
    for (int64_t e = colptr[j]; e < colptr[j + 1]; ++e) cols[j].push_back({rowidx[e], val[e]});
  return SparseColumnsMatrix(d, n, std::move(cols));
}

}  // namespace

extern "C" {

uint64_t ref_derive_seed(uint64_t root, uint64_t tag) { return derive_seed(root, tag); }

void ref_next_u64(uint64_t seed, int64_t count, uint64_t* out) {
  Rng r(seed);
  for (int64_t i = 0; i < count; ++i) out[i] = r.next_u64();
}

void ref_uniform_index(uint64_t seed, uint64_t n, int64_t count, uint64_t* out) {
  Rng r(seed);
  for (int64_t i = 0; i < count; ++i) out[i] = r.uniform_index(n);
}

void ref_normal(uint64_t seed, int64_t count, double* out) {
  Rng r(seed);
  for (int64_t i = 0; i < count; ++i) out[i] = r.normal();
}

int ref_gaussian_init(int d, int p, uint64_t seed, double* out_rowmajor) {
  try {
    DenseMatrix m = gaussian_init(d, p, seed);
    std::memcpy(out_rowmajor, m.entries().data(), sizeof(double) * d * p);
    return 0;
  } catch (const Error&) {
    return 1;
  }
}

// Returns 0 on success, 2 on RankDeficient (column in *bad_col), 1 on contract.
int ref_qr(int d, int p, const double* in_rowmajor, double* out_rowmajor, int* bad_col) {
  try {
    DenseMatrix y(d, p, std::vector<double>(in_rowmajor, in_rowmajor + static_cast<size_t>(d) * p));
    DenseMatrix q = qr_orthonormalize(y);
    std::memcpy(out_rowmajor, q.entries().data(), sizeof(double) * d * p);
    return 0;
  } catch (const RankDeficient& e) {
    if (bad_col) *bad_col = e.column();
    return 2;
  } catch (const Error&) {
    return 1;
  }
}

int ref_jacobi(int n, const double* in_rowmajor, double* vals, double* vecs_rowmajor) {
  try {
    DenseMatrix h(n, n, std::vector<double>(in_rowmajor, in_rowmajor + static_cast<size_t>(n) * n));
    SymmetricEigen e = jacobi_eigh(h);
    std::memcpy(vals, e.values.data(), sizeof(double) * n);
    std::memcpy(vecs_rowmajor, e.vectors.entries().data(), sizeof(double) * n * n);
    return 0;
  } catch (const Error&) {
    return 1;
  }
}

// out = X (X^T v), via GramOperator::apply on the dense-as-sparse X.
int ref_gram_apply_dense(int d, int n, const double* x_colmajor, const double* v, double* out) {
  try {
    SparseColumnsMatrix x = make_dense(d, n, x_colmajor);
    GramOperator op(x);
    std::vector<double> in(v, v + d), o;
    op.apply(in, o);
    std::memcpy(out, o.data(), sizeof(double) * d);
    return 0;
  } catch (const Error&) {
    return 1;
  }
}

int ref_gram_apply_csc(int d, int n, const int64_t* colptr, const int32_t* rowidx,
                       const double* val, const double* v, double* out) {
  try {
    SparseColumnsMatrix x = make_csc(d, n, colptr, rowidx, val);
    GramOperator op(x);
    std::vector<double> in(v, v + d), o;
    op.apply(in, o);
    std::memcpy(out, o.data(), sizeof(double) * d);
    return 0;
  } catch (const Error&) {
    return 1;
  }
}

// One SVRG epoch (direct form) for a d x p block sharing one index
// stream, built only from reference primitives.  Inputs are row-major d x p:
// W (in/out, the iterate which starts at the anchor), Y (n x p, = X^T anchor),
// C (d x p, = eta (X X^T anchor + B)).  Steps: i = uniform_index(n);
// r = eta*n*(x_i^T w_c - Y[i,c]); w_c = rho*w_c + C_c; w_c += r x_i.
int ref_svrg_epoch_dense(int d, int n, const double* x_colmajor, int p, double* w_rowmajor,
                         const double* y_rowmajor, const double* c_rowmajor, double eta,
                         double lambda, uint64_t stream_seed, int64_t m, uint64_t* idx_out) {
  try {
    SparseColumnsMatrix x = make_dense(d, n, x_colmajor);
    const double rho = 1.0 - eta * lambda;
    const double eta_n = eta * static_cast<double>(n);
    std::vector<std::vector<double>> w(p, std::vector<double>(d));
    for (int c = 0; c < p; ++c)
      for (int i = 0; i < d; ++i) w[c][i] = w_rowmajor[static_cast<size_t>(i) * p + c];
    Rng rng(stream_seed);
    for (int64_t s = 0; s < m; ++s) {
      const int j = static_cast<int>(rng.uniform_index(static_cast<uint64_t>(n)));
      if (idx_out) idx_out[s] = static_cast<uint64_t>(j);
      for (int c = 0; c < p; ++c) {
        const double t = x.column_dot(j, w[c]);
        const double r = eta_n * (t - y_rowmajor[static_cast<size_t>(j) * p + c]);
        std::vector<double>& wc = w[c];
        for (int i = 0; i < d; ++i) wc[i] = rho * wc[i] + c_rowmajor[static_cast<size_t>(i) * p + c];
        x.column_axpy(j, r, wc);
      }
    }
    for (int c = 0; c < p; ++c)
      for (int i = 0; i < d; ++i) w_rowmajor[static_cast<size_t>(i) * p + c] = w[c][i];
    return 0;
  } catch (const Error&) {
    return 1;
  }
}

}  // extern "C"
