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

}  // namespace gaplra_cuda
