// Device MGS2 QR, bit-exact Jacobi and skinny products (see linalg.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace gaplra_cuda {

constexpr int kJacobiMax = 64;

// In place on row-major Y (d x ldy, p columns); scratch >= p * round4(d)
// doubles; status[0] = code, status[1] = bad column.
void launch_qr_mgs2(double* Y, int64_t ldy, int d, int p, double* colmajor_scratch, int* status,
                    cudaStream_t st);
// H row-major n x n (n <= 64) -> vals (descending), vecs row-major.
void launch_jacobi(const double* H, int n, double* vals, double* vecs, cudaStream_t st);
// out (pa x pb row-major) = Aᵀ B over d rows; part needs small_gram_parts(d) * pa * pb doubles.
int small_gram_parts(int d);
void launch_small_gram(const double* A, int64_t lda, int pa, const double* B, int64_t ldb, int pb, int d,
                       double* part, double* out, cudaStream_t st);
// C = alpha C + beta A U  (A: d x pa, U: pa x pb row-major with ldu, pa, pb <= 64)
void launch_small_mul(const double* A, int64_t lda, int pa, const double* U, int64_t ldu, int pb, int d,
                      double alpha, double beta, double* C, int64_t ldc, cudaStream_t st);
// out[0] = |A|_F^2 over d rows x p columns (deterministic); part: small_gram_parts(d) doubles.
void launch_frob2(const double* A, int64_t lda, int d, int p, double* part, double* out, cudaStream_t st);

// out[c] = sum_r A[r][c] B[r][c] (p <= 64; deterministic); part: small_gram_parts(d) * p doubles.
void launch_col_dots(const double* A, int64_t lda, const double* B, int64_t ldb, int d, int p, double* part,
                     double* out, cudaStream_t st);
// Block CG pieces on row-major d x p blocks with leading dimension ld:
//   Q = lambda P - Zg;  alpha = rr / pq (status[0] = 1 on pq <= 0 with rr > 0);
//   W += alpha P, R -= alpha Q;  P = R + (rr_new / rr) P.
void launch_cg_dq(const double* P, const double* Zg, double lambda, double* Q, int64_t ld, int d, int p,
                  cudaStream_t st);
void launch_cg_alpha(const double* rr, const double* pq, int p, double* alpha, int* status, cudaStream_t st);
void launch_cg_xr(const double* alpha, const double* P, const double* Q, double* W, double* R, int64_t ld, int d,
                  int p, cudaStream_t st);
void launch_cg_dir(const double* rr, const double* rr_new, const double* R, double* P, int64_t ld, int d, int p,
                   cudaStream_t st);
// H = (H + Hᵀ) / 2 (k x k row-major, in place; no-op for k = 1)
void launch_symmetrize(double* H, int k, cudaStream_t st);
// out = alpha A + beta B (d x p row-major, ld; out may alias A or B)
void launch_axpby(double alpha, const double* A, double beta, const double* B, double* out, int64_t ld, int d, int p,
                  cudaStream_t st);
// device-to-device copy by the SMs (cudaMemcpyAsync fallback when unaligned)
void launch_copy(const void* src, void* dst, size_t bytes, cudaStream_t st);
// v *= 1 / sqrt(*s2) when *s2 > 0 (device scalar)
void launch_scale_inv_sqrt(double* v, int64_t ld, int d, int p, const double* s2, cudaStream_t st);

}  // namespace gaplra_cuda
