// X·(XᵀW) pass kernels — see gram.cuh for the contract.
//
// Layouts: X dense column-major (ld % 4 == 0, zero pad rows); d x p blocks are
// ROW-MAJOR (d_pad x ldp), the reference's DenseMatrix layout
// (proj/core/include/gaplra/dense_matrix.hpp:22-23), so host and device blocks
// share one layout and no transposes happen at the boundary.
#include "gram.cuh"

#include <algorithm>

namespace gaplra_cuda {

namespace {

constexpr int kXtwThreads = 128;
constexpr int kXyThreads = 128;

__device__ __forceinline__ void ld4(const double* p, double (&v)[4]) {
  asm("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
      : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
      : "l"(p));
}

// W row r, columns [0, NC) with c < pc, as a register array (broadcast loads,
// L1-cached: every warp of the SM walks the same rows).
template <int NC>
__device__ __forceinline__ void load_row(const double* __restrict__ w, int pc, double (&out)[NC]) {
  if constexpr (NC % 2 == 0) {
#pragma unroll
    for (int c = 0; c < NC; c += 2) {
      if (c + 1 < pc) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(w + c));
        out[c] = v.x;
        out[c + 1] = v.y;
      } else {
        out[c] = c < pc ? __ldg(w + c) : 0.0;
        out[c + 1] = 0.0;
      }
    }
  } else {
#pragma unroll
    for (int c = 0; c < NC; ++c) out[c] = c < pc ? __ldg(w + c) : 0.0;
  }
}

// ---------------------------------------------------------------------------
// Y = Xᵀ W.  Thread owns TJ columns (j = j0 + tid + 128 t); each iteration
// streams 4 rows of each column with one 256-bit load and reuses them across
// all NC right-hand sides.  Grid: (column tiles, row splits).  Row split s
// writes part[s] (or Y directly when there is one split).
// ---------------------------------------------------------------------------
template <int NC, int TJ>
__global__ void __launch_bounds__(kXtwThreads) k_xtw(const double* __restrict__ X, int64_t ldx, int n,
                                                     int rows_per_split, int rows_total,
                                                     const double* __restrict__ W, int64_t ldw, int pc,
                                                     double* __restrict__ out, int64_t ldo,
                                                     size_t split_stride) {
  const int j0 = blockIdx.x * (kXtwThreads * TJ) + threadIdx.x;
  const int r0 = blockIdx.y * rows_per_split;
  const int r1 = min(r0 + rows_per_split, rows_total);
  double acc[TJ][NC];
#pragma unroll
  for (int t = 0; t < TJ; ++t)
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[t][c] = 0.0;

  const double* xc[TJ];
  bool live[TJ];
#pragma unroll
  for (int t = 0; t < TJ; ++t) {
    const int j = j0 + t * kXtwThreads;
    live[t] = j < n;
    xc[t] = X + static_cast<int64_t>(live[t] ? j : 0) * ldx;
  }
  double cur[TJ][4], nxt[TJ][4];
  if (r0 < r1) {
#pragma unroll
    for (int t = 0; t < TJ; ++t) ld4(xc[t] + r0, cur[t]);
  }
  for (int r = r0; r < r1; r += 4) {
    if (r + 4 < r1) {
#pragma unroll
      for (int t = 0; t < TJ; ++t) ld4(xc[t] + r + 4, nxt[t]);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      double wr[NC];
      load_row<NC>(W + static_cast<int64_t>(r + q) * ldw, pc, wr);
#pragma unroll
      for (int t = 0; t < TJ; ++t)
#pragma unroll
        for (int c = 0; c < NC; ++c) acc[t][c] = fma(cur[t][q], wr[c], acc[t][c]);
    }
#pragma unroll
    for (int t = 0; t < TJ; ++t)
#pragma unroll
      for (int q = 0; q < 4; ++q) cur[t][q] = nxt[t][q];
  }
  double* o = out + blockIdx.y * split_stride;
#pragma unroll
  for (int t = 0; t < TJ; ++t) {
    if (!live[t]) continue;
    double* row = o + static_cast<int64_t>(j0 + t * kXtwThreads) * ldo;
#pragma unroll
    for (int c = 0; c < NC; ++c)
      if (c < pc) row[c] = acc[t][c];
  }
}

// out[r, c] = sum_s part[s][r, c]  (fixed order => deterministic)
__global__ void k_sum_splits(const double* __restrict__ part, int nsplit, size_t split_stride, int rows,
                             int pc, int64_t ldp, double* __restrict__ out, int64_t ldo) {
  const int64_t total = static_cast<int64_t>(rows) * pc;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = e / pc;
    const int c = static_cast<int>(e - r * pc);
    double s = 0.0;
    for (int k = 0; k < nsplit; ++k) s += part[k * split_stride + r * ldp + c];
    out[r * ldo + c] = s;
  }
}

// ---------------------------------------------------------------------------
// Z = X Y.  Thread owns 2 consecutive rows (one 128-bit load per column j)
// and all NC columns of Z; Y rows are broadcast.  Grid: (row blocks of 256,
// column splits).  Split s writes part[s] (d_pad x pc row-major).
// ---------------------------------------------------------------------------
template <int NC>
__global__ void __launch_bounds__(kXyThreads) k_xy(const double* __restrict__ X, int64_t ldx, int rows_total,
                                                   int cols_per_split, int n, const double* __restrict__ Y,
                                                   int64_t ldy, int pc, double* __restrict__ out, int64_t ldo,
                                                   size_t split_stride) {
  const int r = (blockIdx.x * kXyThreads + threadIdx.x) * 2;
  const int j0 = blockIdx.y * cols_per_split;
  const int j1 = min(j0 + cols_per_split, n);
  const bool live = r < rows_total;
  const double* xr = X + (live ? r : 0);
  double a0[NC], a1[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) a0[c] = a1[c] = 0.0;
  constexpr int U = 4;
  int j = j0;
  for (; j + U <= j1; j += U) {
    double2 xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) xv[u] = ldg2(xr + static_cast<int64_t>(j + u) * ldx);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      double yr[NC];
      load_row<NC>(Y + static_cast<int64_t>(j + u) * ldy, pc, yr);
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        a0[c] = fma(xv[u].x, yr[c], a0[c]);
        a1[c] = fma(xv[u].y, yr[c], a1[c]);
      }
    }
  }
  for (; j < j1; ++j) {
    const double2 xv = ldg2(xr + static_cast<int64_t>(j) * ldx);
    double yr[NC];
    load_row<NC>(Y + static_cast<int64_t>(j) * ldy, pc, yr);
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      a0[c] = fma(xv.x, yr[c], a0[c]);
      a1[c] = fma(xv.y, yr[c], a1[c]);
    }
  }
  if (!live) return;
  double* o = out + blockIdx.y * split_stride + static_cast<int64_t>(r) * ldo;
#pragma unroll
  for (int c = 0; c < NC; ++c)
    if (c < pc) {
      o[c] = a0[c];
      o[ldo + c] = a1[c];
    }
}

int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

// The register-resident column chunk: NC in {1,2,4,8,12,16,20,24,32}.
int pick_nc(int pc) {
  static const int opts[] = {1, 2, 4, 8, 12, 16, 20, 24, 32};
  for (int o : opts)
    if (pc <= o) return o;
  return 32;
}

struct XtwPlan {
  int col_tiles, rs, rows_per_split;
};

XtwPlan xtw_plan(const DenseX& X, int nc) {
  const int tj = nc <= 12 ? 2 : 1;
  XtwPlan pl;
  const int rows_total = static_cast<int>(X.ld);
  pl.col_tiles = static_cast<int>(ceil_div(X.n, kXtwThreads * tj));
  const int slots = sm_count() * 4;
  int rs = static_cast<int>(std::min<int64_t>(ceil_div(2 * slots, pl.col_tiles), rows_total / 256));
  rs = std::max(rs, 1);
  pl.rows_per_split = static_cast<int>(ceil_div(ceil_div(rows_total, rs), 4) * 4);
  pl.rs = static_cast<int>(ceil_div(rows_total, pl.rows_per_split));
  return pl;
}

struct XyPlan {
  int row_blocks, s, cols_per_split;
};

XyPlan xy_plan(const DenseX& X) {
  XyPlan pl;
  const int rows_total = static_cast<int>(X.ld);
  pl.row_blocks = static_cast<int>(ceil_div(rows_total, 2 * kXyThreads));
  const int slots = sm_count() * 4;
  int s = static_cast<int>(std::min<int64_t>(ceil_div(2 * slots, pl.row_blocks), ceil_div(X.n, 64)));
  s = std::max(s, 1);
  pl.cols_per_split = static_cast<int>(ceil_div(X.n, s));
  pl.s = static_cast<int>(ceil_div(X.n, pl.cols_per_split));
  return pl;
}

template <int NC>
void xtw_chunk(const DenseX& X, const double* W, int64_t ldw, int pc, double* Y, int64_t ldy,
               GramWork& work, cudaStream_t st) {
  constexpr int TJ = NC <= 12 ? 2 : 1;
  const int rows_total = static_cast<int>(X.ld);
  const XtwPlan pl = xtw_plan(X, NC);
  dim3 grid(pl.col_tiles, pl.rs);
  if (pl.rs == 1) {
    k_xtw<NC, TJ><<<grid, kXtwThreads, 0, st>>>(X.x, X.ld, X.n, pl.rows_per_split, rows_total, W, ldw, pc, Y,
                                                ldy, 0);
    GAPLRA_LAUNCH_CHECK();
    return;
  }
  const size_t stride = static_cast<size_t>(X.n) * pc;
  if (work.part_elems < stride * pl.rs) throw Error(kContractViolation, "xtw: workspace too small");
  k_xtw<NC, TJ><<<grid, kXtwThreads, 0, st>>>(X.x, X.ld, X.n, pl.rows_per_split, rows_total, W, ldw, pc,
                                              work.part, pc, stride);
  GAPLRA_LAUNCH_CHECK();
  k_sum_splits<<<sm_count() * 4, 256, 0, st>>>(work.part, pl.rs, stride, X.n, pc, pc, Y, ldy);
  GAPLRA_LAUNCH_CHECK();
}

template <int NC>
void xy_chunk(const DenseX& X, const double* Y, int64_t ldy, int pc, double* Z, int64_t ldz, GramWork& work,
              cudaStream_t st) {
  const int rows_total = static_cast<int>(X.ld);
  const XyPlan pl = xy_plan(X);
  dim3 grid(pl.row_blocks, pl.s);
  const size_t stride = static_cast<size_t>(rows_total) * pc;
  if (pl.s == 1) {
    k_xy<NC><<<grid, kXyThreads, 0, st>>>(X.x, X.ld, rows_total, pl.cols_per_split, X.n, Y, ldy, pc, Z, ldz, 0);
    GAPLRA_LAUNCH_CHECK();
    return;
  }
  if (work.part_elems < stride * pl.s) throw Error(kContractViolation, "xy: workspace too small");
  k_xy<NC><<<grid, kXyThreads, 0, st>>>(X.x, X.ld, rows_total, pl.cols_per_split, X.n, Y, ldy, pc, work.part,
                                        pc, stride);
  GAPLRA_LAUNCH_CHECK();
  k_sum_splits<<<sm_count() * 4, 256, 0, st>>>(work.part, pl.s, stride, rows_total, pc, pc, Z, ldz);
  GAPLRA_LAUNCH_CHECK();
}

template <template <int> class F, class... A>
void dispatch_nc(int nc, A&&... a) {
  switch (nc) {
    case 1: F<1>::run(a...); break;
    case 2: F<2>::run(a...); break;
    case 4: F<4>::run(a...); break;
    case 8: F<8>::run(a...); break;
    case 12: F<12>::run(a...); break;
    case 16: F<16>::run(a...); break;
    case 20: F<20>::run(a...); break;
    case 24: F<24>::run(a...); break;
    default: F<32>::run(a...); break;
  }
}

template <int NC>
struct XtwRun {
  template <class... A>
  static void run(A&&... a) {
    xtw_chunk<NC>(a...);
  }
};
template <int NC>
struct XyRun {
  template <class... A>
  static void run(A&&... a) {
    xy_chunk<NC>(a...);
  }
};

// ---------------------------------------------------------------------------
// Sparse (CSC for Xᵀ W, CSR for X Y): one thread per output row of Y / Z.
// ---------------------------------------------------------------------------
template <int NC>
__global__ void k_xtw_sparse(int n, const int64_t* __restrict__ colptr, const int32_t* __restrict__ rowidx,
                             const double* __restrict__ val, const double* __restrict__ W, int64_t ldw, int pc,
                             double* __restrict__ Y, int64_t ldy) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double acc[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) acc[c] = 0.0;
  for (int64_t e = colptr[j]; e < colptr[j + 1]; ++e) {
    const double v = val[e];
    double wr[NC];
    load_row<NC>(W + static_cast<int64_t>(rowidx[e]) * ldw, pc, wr);
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[c] = fma(v, wr[c], acc[c]);
  }
#pragma unroll
  for (int c = 0; c < NC; ++c)
    if (c < pc) Y[static_cast<int64_t>(j) * ldy + c] = acc[c];
}

template <int NC>
__global__ void k_xy_sparse(int d, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ colidx,
                            const double* __restrict__ rval, const double* __restrict__ Y, int64_t ldy, int pc,
                            double* __restrict__ Z, int64_t ldz) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= d) return;
  double acc[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) acc[c] = 0.0;
  for (int64_t e = rowptr[r]; e < rowptr[r + 1]; ++e) {
    const double v = rval[e];
    double yr[NC];
    load_row<NC>(Y + static_cast<int64_t>(colidx[e]) * ldy, pc, yr);
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[c] = fma(v, yr[c], acc[c]);
  }
#pragma unroll
  for (int c = 0; c < NC; ++c)
    if (c < pc) Z[static_cast<int64_t>(r) * ldz + c] = acc[c];
}

template <int NC>
struct XtwSparseRun {
  static void run(const SparseX& X, const double* W, int64_t ldw, int pc, double* Y, int64_t ldy,
                  cudaStream_t st) {
    k_xtw_sparse<NC><<<ceil_div(X.n, 128), 128, 0, st>>>(X.n, X.colptr, X.rowidx, X.val, W, ldw, pc, Y, ldy);
    GAPLRA_LAUNCH_CHECK();
  }
};
template <int NC>
struct XySparseRun {
  static void run(const SparseX& X, const double* Y, int64_t ldy, int pc, double* Z, int64_t ldz,
                  cudaStream_t st) {
    k_xy_sparse<NC><<<ceil_div(X.d, 128), 128, 0, st>>>(X.d, X.rowptr, X.colidx, X.rval, Y, ldy, pc, Z, ldz);
    GAPLRA_LAUNCH_CHECK();
  }
};

__global__ void k_colnorm2_dense(const double* __restrict__ X, int64_t ldx, int d, int n, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int j = warp; j < n; j += nwarps) {
    const double* col = X + static_cast<int64_t>(j) * ldx;
    double s = 0.0;
    for (int i = lane; i < d; i += 32) s = fma(col[i], col[i], s);
    s = warp_sum(s);
    if (lane == 0) out[j] = s;
  }
}

__global__ void k_colnorm2_sparse(int n, const int64_t* __restrict__ colptr, const double* __restrict__ val,
                                  double* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double s = 0.0;
  for (int64_t e = colptr[j]; e < colptr[j + 1]; ++e) s = fma(val[e], val[e], s);
  out[j] = s;
}

// out[0] = sum, out[1] = max of v[0..n) — one CTA, fixed order (deterministic)
__global__ void k_sum_max(const double* __restrict__ v, int n, double* __restrict__ out) {
  __shared__ double red[32];
  double s = 0.0, m = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    s += v[i];
    m = fmax(m, v[i]);
  }
  s = block_sum(s, red);
  m = block_max(m, red);
  if (threadIdx.x == 0) {
    out[0] = s;
    out[1] = m;
  }
}

}  // namespace

size_t gram_work_elems(const DenseX& X, int p) {
  size_t need = 0;
  for (int c0 = 0; c0 < p; c0 += 32) {
    const int pc = std::min(32, p - c0);
    const XtwPlan a = xtw_plan(X, pick_nc(pc));
    if (a.rs > 1) need = std::max(need, static_cast<size_t>(a.rs) * X.n * pc);
    const XyPlan b = xy_plan(X);
    if (b.s > 1) need = std::max(need, static_cast<size_t>(b.s) * X.ld * pc);
  }
  return need;
}

void launch_xtw(const DenseX& X, const double* W, int64_t ldw, int p, double* Y, int64_t ldy, GramWork& work,
                cudaStream_t st) {
  for (int c0 = 0; c0 < p; c0 += 32) {
    const int pc = std::min(32, p - c0);
    dispatch_nc<XtwRun>(pick_nc(pc), X, W + c0, ldw, pc, Y + c0, ldy, work, st);
  }
}

void launch_xy(const DenseX& X, const double* Y, int64_t ldy, int p, double* Z, int64_t ldz, GramWork& work,
               cudaStream_t st) {
  for (int c0 = 0; c0 < p; c0 += 32) {
    const int pc = std::min(32, p - c0);
    dispatch_nc<XyRun>(pick_nc(pc), X, Y + c0, ldy, pc, Z + c0, ldz, work, st);
  }
}

void launch_xtw_sparse(const SparseX& X, const double* W, int64_t ldw, int p, double* Y, int64_t ldy,
                       cudaStream_t st) {
  for (int c0 = 0; c0 < p; c0 += 32) {
    const int pc = std::min(32, p - c0);
    dispatch_nc<XtwSparseRun>(pick_nc(pc), X, W + c0, ldw, pc, Y + c0, ldy, st);
  }
}

void launch_xy_sparse(const SparseX& X, const double* Y, int64_t ldy, int p, double* Z, int64_t ldz,
                      cudaStream_t st) {
  for (int c0 = 0; c0 < p; c0 += 32) {
    const int pc = std::min(32, p - c0);
    dispatch_nc<XySparseRun>(pick_nc(pc), X, Y + c0, ldy, pc, Z + c0, ldz, st);
  }
}

void col_norm2_dense(const DenseX& X, double* out, cudaStream_t st) {
  k_colnorm2_dense<<<sm_count() * 8, 256, 0, st>>>(X.x, X.ld, X.d, X.n, out);
  GAPLRA_LAUNCH_CHECK();
}

void col_norm2_sparse(const SparseX& X, double* out, cudaStream_t st) {
  k_colnorm2_sparse<<<ceil_div(X.n, 256), 256, 0, st>>>(X.n, X.colptr, X.val, out);
  GAPLRA_LAUNCH_CHECK();
}

void reduce_sum_max(const double* v, int n, double* out2, cudaStream_t st) {
  k_sum_max<<<1, 1024, 0, st>>>(v, n, out2);
  GAPLRA_LAUNCH_CHECK();
}

}  // namespace gaplra_cuda
