// Block orthonormalisation (two-pass MGS), p x p cyclic Jacobi, and the
// skinny products of the subspace engine, as device kernels.
//
//  * qr_mgs2 follows qr_orthonormalize / mgs_columns
//    (proj/core/src/orthonormalize.cpp:25-79): scale = largest column norm,
//    for each column two MGS passes against all earlier columns, rank test
//    !(nrm > 1e-13 * scale) -> RankDeficient(j), then multiply by 1/nrm.
//    Dots are deterministic block reductions (tolerance parity, not bitwise:
//    the reference sums rows sequentially).
//  * jacobi follows jacobi_eigh (proj/core/src/jacobi.cpp:13-109) operation by
//    operation with explicitly rounded intrinsics (no FMA contraction), so it
//    is BIT-EXACT with the reference for the same input matrix.
#include <algorithm>

#include "common.cuh"
#include "linalg.cuh"

namespace gaplra_cuda {

namespace {

constexpr int kQrThreads = 1024;

// Column-major working copy: Q[j * ldq + i].  E = elements per thread held in
// registers (d <= E * 1024); E == 0 streams the column through global memory.
template <int E>
__global__ void __launch_bounds__(kQrThreads) k_qr_mgs2(double* __restrict__ Q, int64_t ldq, int d, int p,
                                                        int* __restrict__ status) {
  __shared__ double red[32];
  const int tid = threadIdx.x;
  // scale = max_j |y_j|
  double scale = 0.0;
  for (int j = 0; j < p; ++j) {
    const double* q = Q + j * ldq;
    double s = 0.0;
    for (int i = tid; i < d; i += kQrThreads) s = fma(q[i], q[i], s);
    s = block_sum(s, red);
    scale = fmax(scale, sqrt(s));
  }
  if (scale == 0.0) {
    if (tid == 0) {
      status[0] = kRankDeficient;
      status[1] = 0;
    }
    return;
  }
  for (int j = 0; j < p; ++j) {
    double* qj = Q + j * ldq;
    double col[E > 0 ? E : 1];
    if constexpr (E > 0) {
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int i = tid + e * kQrThreads;
        col[e] = i < d ? qj[i] : 0.0;
      }
    }
    for (int pass = 0; pass < 2; ++pass) {
      for (int prev = 0; prev < j; ++prev) {
        const double* qp = Q + prev * ldq;
        double s = 0.0;
        if constexpr (E > 0) {
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int i = tid + e * kQrThreads;
            if (i < d) s = fma(qp[i], col[e], s);
          }
        } else {
          for (int i = tid; i < d; i += kQrThreads) s = fma(qp[i], qj[i], s);
        }
        const double proj = block_sum(s, red);
        if constexpr (E > 0) {
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int i = tid + e * kQrThreads;
            if (i < d) col[e] = fma(-proj, qp[i], col[e]);
          }
        } else {
          for (int i = tid; i < d; i += kQrThreads) qj[i] = fma(-proj, qp[i], qj[i]);
          __syncthreads();
        }
      }
    }
    double s = 0.0;
    if constexpr (E > 0) {
#pragma unroll
      for (int e = 0; e < E; ++e) s = fma(col[e], col[e], s);
    } else {
      for (int i = tid; i < d; i += kQrThreads) s = fma(qj[i], qj[i], s);
    }
    const double nrm = sqrt(block_sum(s, red));
    if (!(nrm > 1e-13 * scale)) {
      if (tid == 0) {
        status[0] = kRankDeficient;
        status[1] = j;
      }
      return;
    }
    const double inv = 1.0 / nrm;
    if constexpr (E > 0) {
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int i = tid + e * kQrThreads;
        if (i < d) qj[i] = col[e] * inv;
      }
    } else {
      for (int i = tid; i < d; i += kQrThreads) qj[i] = qj[i] * inv;
    }
    __syncthreads();
  }
  if (tid == 0) status[0] = kOk;
}

// row-major (rows x ld_in) <-> column-major (cols x ld_out) transposes
__global__ void k_transpose(const double* __restrict__ in, int64_t ldi, int rows, int cols,
                            double* __restrict__ out, int64_t ldo) {
  __shared__ double tile[32][33];
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int r = r0 + k, c = c0 + threadIdx.x;
    tile[k][threadIdx.x] = (r < rows && c < cols) ? in[static_cast<int64_t>(r) * ldi + c] : 0.0;
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int c = c0 + k, r = r0 + threadIdx.x;
    if (r < rows && c < cols) out[static_cast<int64_t>(c) * ldo + r] = tile[threadIdx.x][k];
  }
}

// ---------------------------------------------------------------------------
// Jacobi (one warp; lanes own matrix rows/cols i and i+32).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

__global__ void k_jacobi(const double* __restrict__ H, int n, double* __restrict__ vals,
                         double* __restrict__ vecs) {
  extern __shared__ double jsm[];
  double(*A)[kJacobiMax + 1] = reinterpret_cast<double(*)[kJacobiMax + 1]>(jsm);
  double(*V)[kJacobiMax + 1] = reinterpret_cast<double(*)[kJacobiMax + 1]>(jsm + kJacobiMax * (kJacobiMax + 1));
  int* order = reinterpret_cast<int*>(jsm + 2 * kJacobiMax * (kJacobiMax + 1));
  const int lane = threadIdx.x;
  for (int i = lane; i < n; i += 32)
    for (int j = 0; j < n; ++j) {
      A[i][j] = H[i * n + j];
      V[i][j] = (i == j) ? 1.0 : 0.0;
    }
  __syncwarp();
  if (lane == 0) {  // symmetrize (jacobi.cpp:41-48)
    for (int i = 0; i < n; ++i)
      for (int j = i + 1; j < n; ++j) {
        const double m = mul(0.5, add(A[i][j], A[j][i]));
        A[i][j] = m;
        A[j][i] = m;
      }
  }
  __syncwarp();
  const double tol2 = mul(1e-14, 1e-14);
  for (int sweep = 0; sweep < 60; ++sweep) {
    int done = 0;
    if (lane == 0) {  // convergence test, sequential order (jacobi.cpp:52-58)
      double off = 0.0, diag = 0.0;
      for (int i = 0; i < n; ++i) {
        diag = add(diag, mul(A[i][i], A[i][i]));
        for (int j = i + 1; j < n; ++j) off = add(off, mul(mul(2.0, A[i][j]), A[i][j]));
      }
      done = off <= mul(tol2, fmax(diag, 1e-300));
    }
    done = __shfl_sync(0xffffffffu, done, 0);
    if (done) break;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = A[p][q];
        if (apq == 0.0) continue;
        const double app = A[p][p], aqq = A[q][q];
        const double tau = __ddiv_rn(sub(aqq, app), mul(2.0, apq));
        const double root = __dsqrt_rn(add(1.0, mul(tau, tau)));
        const double t = (tau >= 0.0) ? __ddiv_rn(1.0, add(tau, root)) : __ddiv_rn(1.0, sub(tau, root));
        const double c = __ddiv_rn(1.0, __dsqrt_rn(add(1.0, mul(t, t))));
        const double s = mul(t, c);
        for (int i = lane; i < n; i += 32) {
          const double aip = A[i][p], aiq = A[i][q];
          A[i][p] = sub(mul(c, aip), mul(s, aiq));
          A[i][q] = add(mul(s, aip), mul(c, aiq));
        }
        __syncwarp();
        for (int i = lane; i < n; i += 32) {
          const double api = A[p][i], aqi = A[q][i];
          A[p][i] = sub(mul(c, api), mul(s, aqi));
          A[q][i] = add(mul(s, api), mul(c, aqi));
        }
        for (int i = lane; i < n; i += 32) {
          const double vip = V[i][p], viq = V[i][q];
          V[i][p] = sub(mul(c, vip), mul(s, viq));
          V[i][q] = add(mul(s, vip), mul(c, viq));
        }
        __syncwarp();
      }
  }
  if (lane == 0) {  // stable descending sort (jacobi.cpp:95-98)
    for (int i = 0; i < n; ++i) order[i] = i;
    for (int i = 1; i < n; ++i) {
      const int key = order[i];
      int j = i - 1;
      while (j >= 0 && A[key][key] > A[order[j]][order[j]]) {
        order[j + 1] = order[j];
        --j;
      }
      order[j + 1] = key;
    }
  }
  __syncwarp();
  for (int j = lane; j < n; j += 32) {
    vals[j] = A[order[j]][order[j]];
    int arg = 0;
    double best = 0.0;
    for (int i = 0; i < n; ++i) {
      const double a = fabs(V[i][order[j]]);
      if (a > best) {
        best = a;
        arg = i;
      }
    }
    const bool flip = V[arg][order[j]] < 0.0;
    for (int i = 0; i < n; ++i) {
      const double v = V[i][order[j]];
      vecs[i * n + j] = flip ? -v : v;
    }
  }
}

// ---------------------------------------------------------------------------
// G[a][b] = sum_i A[i][a] B[i][b]  (row-major blocks, pa, pb <= 64), two-level
// deterministic reduction: per-CTA partials over row chunks, then a fixed-order
// sum.
// ---------------------------------------------------------------------------
constexpr int kGramThreads = 256;

__global__ void k_small_gram_part(const double* __restrict__ A, int64_t lda, int pa, const double* __restrict__ B,
                                  int64_t ldb, int pb, int d, int rows_per_cta, double* __restrict__ part) {
  const int r0 = blockIdx.x * rows_per_cta;
  const int r1 = min(r0 + rows_per_cta, d);
  const int npair = pa * pb;
  double* out = part + static_cast<int64_t>(blockIdx.x) * npair;
  for (int e = threadIdx.x; e < npair; e += blockDim.x) {
    const int a = e / pb, b = e - (e / pb) * pb;
    double s = 0.0;
    for (int r = r0; r < r1; ++r)
      s = fma(A[static_cast<int64_t>(r) * lda + a], B[static_cast<int64_t>(r) * ldb + b], s);
    out[e] = s;
  }
}

__global__ void k_sum_parts(const double* __restrict__ part, int nparts, int len, double* __restrict__ out) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < len; e += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < nparts; ++k) s += part[static_cast<int64_t>(k) * len + e];
    out[e] = s;
  }
}

// C[i][b] = alpha * C[i][b] + beta * sum_a A[i][a] U[a][b]   (U: pa x pb, ldu; <= 64 x 64)
__global__ void k_small_mul(const double* __restrict__ A, int64_t lda, int pa, const double* __restrict__ U,
                            int64_t ldu, int pb, int d, double alpha, double beta, double* __restrict__ C,
                            int64_t ldc) {
  __shared__ double Us[kJacobiMax * kJacobiMax];
  for (int e = threadIdx.x; e < pa * pb; e += blockDim.x) Us[e] = U[(e / pb) * ldu + (e % pb)];
  __syncthreads();
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < static_cast<int64_t>(d) * pb;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = e / pb;
    const int b = static_cast<int>(e - i * pb);
    double s = 0.0;
    for (int a = 0; a < pa; ++a) s = fma(A[i * lda + a], Us[a * pb + b], s);
    double* c = C + i * ldc + b;
    *c = alpha == 0.0 ? beta * s : fma(alpha, *c, beta * s);
  }
}

// part[blk] = sum over the block's rows of sum_c A[r][c]^2 ; out = sum_blk part
__global__ void k_frob2_part(const double* __restrict__ A, int64_t lda, int d, int p, int rows_per,
                             double* __restrict__ part) {
  __shared__ double red[32];
  const int r0 = blockIdx.x * rows_per, r1 = min(r0 + rows_per, d);
  double s = 0.0;
  for (int64_t e = threadIdx.x; e < static_cast<int64_t>(r1 - r0) * p; e += blockDim.x) {
    const int64_t r = r0 + e / p;
    const double v = A[r * lda + e % p];
    s = fma(v, v, s);
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// part[blk][c] = sum over the block's rows of A[r][c] B[r][c]: thread (c, sub)
// strides the rows by nsub, then a fixed-order shared-memory sum over sub.
__global__ void k_col_dots_part(const double* __restrict__ A, int64_t lda, const double* __restrict__ B, int64_t ldb,
                                int d, int p, int rows_per, double* __restrict__ part) {
  __shared__ double red[256];
  const int nsub = blockDim.x / p;
  const int c = threadIdx.x % p, sub = threadIdx.x / p;
  const int r0 = blockIdx.x * rows_per, r1 = min(r0 + rows_per, d);
  double s = 0.0;
  if (sub < nsub)
    for (int r = r0 + sub; r < r1; r += nsub) s = fma(A[static_cast<int64_t>(r) * lda + c], B[static_cast<int64_t>(r) * ldb + c], s);
  red[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x < p) {
    double t = 0.0;
    for (int q = 0; q < nsub; ++q) t += red[q * p + threadIdx.x];
    part[static_cast<int64_t>(blockIdx.x) * p + threadIdx.x] = t;
  }
}

// CG pieces (runtime.cu cg_solve_dev; oracle.cpp cg_solve)
__global__ void k_cg_dq(const double* __restrict__ P, const double* __restrict__ Zg, double lambda,
                        double* __restrict__ Q, int64_t ld, int d, int p) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < static_cast<int64_t>(d) * p;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = e / p, o = i * ld + (e - i * p);
    Q[o] = lambda * P[o] - Zg[o];
  }
}
// alpha = rr / pq (0 for a frozen column), status[0] = 1 on nonpositive curvature
__global__ void k_cg_alpha(const double* __restrict__ rr, const double* __restrict__ pq, int p,
                           double* __restrict__ alpha, int* __restrict__ status) {
  const int c = threadIdx.x;
  if (c >= p) return;
  const bool live = rr[c] > 0.0;
  if (live && !(pq[c] > 0.0)) status[0] = 1;
  alpha[c] = live ? rr[c] / pq[c] : 0.0;
}
__global__ void k_cg_xr(const double* __restrict__ alpha, const double* __restrict__ P, const double* __restrict__ Q,
                        double* __restrict__ W, double* __restrict__ R, int64_t ld, int d, int p) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < static_cast<int64_t>(d) * p;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = e / p;
    const int c = static_cast<int>(e - i * p);
    const int64_t o = i * ld + c;
    W[o] += alpha[c] * P[o];
    R[o] -= alpha[c] * Q[o];
  }
}
// beta = rr_new / rr (0 for a frozen column); P = R + beta P
__global__ void k_cg_dir(const double* __restrict__ rr, const double* __restrict__ rr_new, const double* __restrict__ R,
                         double* __restrict__ P, int64_t ld, int d, int p) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < static_cast<int64_t>(d) * p;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = e / p;
    const int c = static_cast<int>(e - i * p);
    const double beta = rr[c] > 0.0 ? rr_new[c] / rr[c] : 0.0;
    const int64_t o = i * ld + c;
    P[o] = R[o] + beta * P[o];
  }
}
// v *= 1 / sqrt(*s2) when *s2 > 0
__global__ void k_scale_inv_sqrt(double* __restrict__ v, int64_t ld, int d, int p, const double* __restrict__ s2) {
  const double s = *s2;
  if (!(s > 0.0)) return;
  const double inv = 1.0 / sqrt(s);
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < static_cast<int64_t>(d) * p;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = e / p;
    v[i * ld + (e - i * p)] *= inv;
  }
}

// H = (H + Hᵀ) / 2 in place (k x k row-major), the oracle's expression 0.5 * (h_ab + h_ba)
__global__ void k_symmetrize(double* __restrict__ H, int k) {
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
    const int a = e / k, b = e - (e / k) * k;
    if (b <= a) continue;
    const double m = 0.5 * (H[a * k + b] + H[b * k + a]);
    H[a * k + b] = m;
    H[b * k + a] = m;
  }
}

// out = alpha A + beta B (d x p row-major blocks, leading dimension ld; out may alias A or B)
__global__ void k_axpby(double alpha, const double* A, double beta, const double* Bm, double* out, int64_t ld, int d,
                        int p) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < static_cast<int64_t>(d) * p;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = e / p, o = i * ld + (e - i * p);
    out[o] = alpha * A[o] + beta * Bm[o];
  }
}

}  // namespace

void launch_qr_mgs2(double* Y, int64_t ldy, int d, int p, double* colmajor_scratch, int* status,
                    cudaStream_t st) {
  // Row-major Y -> column-major scratch -> MGS2 -> back.
  const int64_t ldq = ceil_div(d, 4) * 4;
  dim3 tb(32, 8);
  k_transpose<<<dim3(ceil_div(p, 32), ceil_div(d, 32)), tb, 0, st>>>(Y, ldy, d, p, colmajor_scratch, ldq);
  GAPLRA_LAUNCH_CHECK();
  if (d <= kQrThreads)
    k_qr_mgs2<1><<<1, kQrThreads, 0, st>>>(colmajor_scratch, ldq, d, p, status);
  else if (d <= 2 * kQrThreads)
    k_qr_mgs2<2><<<1, kQrThreads, 0, st>>>(colmajor_scratch, ldq, d, p, status);
  else if (d <= 4 * kQrThreads)
    k_qr_mgs2<4><<<1, kQrThreads, 0, st>>>(colmajor_scratch, ldq, d, p, status);
  else if (d <= 8 * kQrThreads)
    k_qr_mgs2<8><<<1, kQrThreads, 0, st>>>(colmajor_scratch, ldq, d, p, status);
  else
    k_qr_mgs2<0><<<1, kQrThreads, 0, st>>>(colmajor_scratch, ldq, d, p, status);
  GAPLRA_LAUNCH_CHECK();
  k_transpose<<<dim3(ceil_div(d, 32), ceil_div(p, 32)), tb, 0, st>>>(colmajor_scratch, ldq, p, d, Y, ldy);
  GAPLRA_LAUNCH_CHECK();
}

void launch_jacobi(const double* H, int n, double* vals, double* vecs, cudaStream_t st) {
  if (n < 1 || n > kJacobiMax) throw Error(kContractViolation, "jacobi: n out of range");
  const size_t smem = (2 * kJacobiMax * (kJacobiMax + 1) + kJacobiMax) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    GAPLRA_CUDA_CHECK(cudaFuncSetAttribute(k_jacobi, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    attr = true;
  }
  k_jacobi<<<1, 32, smem, st>>>(H, n, vals, vecs);
  GAPLRA_LAUNCH_CHECK();
}

int small_gram_parts(int d) { return static_cast<int>(std::min<int64_t>(ceil_div(d, 64), 296)); }

void launch_small_gram(const double* A, int64_t lda, int pa, const double* B, int64_t ldb, int pb, int d,
                       double* part, double* out, cudaStream_t st) {
  const int parts = small_gram_parts(d);
  const int rows_per = static_cast<int>(ceil_div(d, parts));
  k_small_gram_part<<<parts, kGramThreads, 0, st>>>(A, lda, pa, B, ldb, pb, d, rows_per, part);
  GAPLRA_LAUNCH_CHECK();
  k_sum_parts<<<ceil_div(pa * pb, 256), 256, 0, st>>>(part, parts, pa * pb, out);
  GAPLRA_LAUNCH_CHECK();
}

void launch_small_mul(const double* A, int64_t lda, int pa, const double* U, int64_t ldu, int pb, int d,
                      double alpha, double beta, double* C, int64_t ldc, cudaStream_t st) {
  if (pa > kJacobiMax || pb > kJacobiMax) throw Error(kContractViolation, "small_mul: width > 64");
  k_small_mul<<<std::min<int64_t>(ceil_div(static_cast<int64_t>(d) * pb, 256), 1184), 256, 0, st>>>(
      A, lda, pa, U, ldu, pb, d, alpha, beta, C, ldc);
  GAPLRA_LAUNCH_CHECK();
}

void launch_frob2(const double* A, int64_t lda, int d, int p, double* part, double* out, cudaStream_t st) {
  const int parts = small_gram_parts(d);
  const int rows_per = static_cast<int>(ceil_div(d, parts));
  k_frob2_part<<<parts, 256, 0, st>>>(A, lda, d, p, rows_per, part);
  GAPLRA_LAUNCH_CHECK();
  k_sum_parts<<<1, 32, 0, st>>>(part, parts, 1, out);
  GAPLRA_LAUNCH_CHECK();
}

void launch_col_dots(const double* A, int64_t lda, const double* B, int64_t ldb, int d, int p, double* part,
                     double* out, cudaStream_t st) {
  const int parts = small_gram_parts(d);
  const int rows_per = static_cast<int>(ceil_div(d, parts));
  k_col_dots_part<<<parts, 256, 0, st>>>(A, lda, B, ldb, d, p, rows_per, part);
  GAPLRA_LAUNCH_CHECK();
  k_sum_parts<<<1, 64, 0, st>>>(part, parts, p, out);
  GAPLRA_LAUNCH_CHECK();
}

static int ew_grid(int64_t n) { return static_cast<int>(std::min<int64_t>(ceil_div(n, 256), 148 * 8)); }

void launch_cg_dq(const double* P, const double* Zg, double lambda, double* Q, int64_t ld, int d, int p,
                  cudaStream_t st) {
  k_cg_dq<<<ew_grid(static_cast<int64_t>(d) * p), 256, 0, st>>>(P, Zg, lambda, Q, ld, d, p);
  GAPLRA_LAUNCH_CHECK();
}
void launch_cg_alpha(const double* rr, const double* pq, int p, double* alpha, int* status, cudaStream_t st) {
  k_cg_alpha<<<1, 64, 0, st>>>(rr, pq, p, alpha, status);
  GAPLRA_LAUNCH_CHECK();
}
void launch_cg_xr(const double* alpha, const double* P, const double* Q, double* W, double* R, int64_t ld, int d,
                  int p, cudaStream_t st) {
  k_cg_xr<<<ew_grid(static_cast<int64_t>(d) * p), 256, 0, st>>>(alpha, P, Q, W, R, ld, d, p);
  GAPLRA_LAUNCH_CHECK();
}
void launch_cg_dir(const double* rr, const double* rr_new, const double* R, double* P, int64_t ld, int d, int p,
                   cudaStream_t st) {
  k_cg_dir<<<ew_grid(static_cast<int64_t>(d) * p), 256, 0, st>>>(rr, rr_new, R, P, ld, d, p);
  GAPLRA_LAUNCH_CHECK();
}
void launch_scale_inv_sqrt(double* v, int64_t ld, int d, int p, const double* s2, cudaStream_t st) {
  k_scale_inv_sqrt<<<ew_grid(static_cast<int64_t>(d) * p), 256, 0, st>>>(v, ld, d, p, s2);
  GAPLRA_LAUNCH_CHECK();
}

void launch_symmetrize(double* H, int k, cudaStream_t st) {
  if (k < 2) return;
  k_symmetrize<<<1, 256, 0, st>>>(H, k);
  GAPLRA_LAUNCH_CHECK();
}

// dst = src for `bytes` (multiple of 16, 16-byte aligned): an SM copy (a graph
// memcpy node of the 1.5 GB C5 slab ran on a copy engine at ~12 ms per epoch)
__global__ void k_copy16(const double2* __restrict__ src, double2* __restrict__ dst, size_t n16) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n16; i += stride) dst[i] = src[i];
}

void launch_copy(const void* src, void* dst, size_t bytes, cudaStream_t st) {
  if (bytes % 16 != 0 || reinterpret_cast<uintptr_t>(src) % 16 || reinterpret_cast<uintptr_t>(dst) % 16) {
    GAPLRA_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, st));
    return;
  }
  int sms = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  k_copy16<<<std::max(1, sms) * 4, 512, 0, st>>>(static_cast<const double2*>(src), static_cast<double2*>(dst),
                                                   bytes / 16);
  GAPLRA_LAUNCH_CHECK();
}

void launch_axpby(double alpha, const double* A, double beta, const double* B, double* out, int64_t ld, int d, int p,
                  cudaStream_t st) {
  k_axpby<<<ew_grid(static_cast<int64_t>(d) * p), 256, 0, st>>>(alpha, A, beta, B, out, ld, d, p);
  GAPLRA_LAUNCH_CHECK();
}

}  // namespace gaplra_cuda
