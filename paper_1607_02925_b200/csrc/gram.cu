// X·(XᵀW) pass kernels — see gram.cuh for the contract.
//
// Layouts: X dense column-major (ld % 4 == 0, zero pad rows); d x p blocks are
// ROW-MAJOR (d_pad x ldp), the reference's DenseMatrix layout
// (proj/core/include/gaplra/dense_matrix.hpp:22-23), so host and device blocks
// share one layout and no transposes happen at the boundary.
#include "gram.cuh"

#include <algorithm>
#include <cstdlib>

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

__device__ __forceinline__ void mma884(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// 8-byte global -> shared copy without register staging (LDGSTS); src_bytes = 0
// writes zeros.  Committed per stage, waited before the stage is read.
__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
               "l"(src), "r"(valid ? 8 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// smem pitch (doubles) for a KC x (8*NT) B-operand tile: ≡ 8 (mod 16) keeps the
// 4 rows x 8 columns of an m8n8k4 B fragment on distinct bank pairs.
template <int NT>
__host__ __device__ constexpr int b_pitch() {
  return (8 * NT) % 16 == 8 ? 8 * NT : 8 * NT + 8;
}

// ---------------------------------------------------------------------------
// Y = Xᵀ W on the FP64 tensor path (DMMA m8n8k4).  M = columns of X (a warp owns
// MW m-tiles of 8 columns), N = right-hand sides (NT n-tiles of 8, zero padded),
// K = rows of X.  The CTA stages each KC-row chunk of W in shared memory (double
// buffered, shared by its 8 warps).  A fragments come straight from X with one
// 256-bit load per lane per 4 k-steps: lane (g, q) loads rows 16kb+4q..+3 of its
// column, so k-step (kb, u) contracts rows {16kb + 4q' + u}; the B fragment uses
// the same permutation.
// ---------------------------------------------------------------------------
constexpr int kMmaThreads = 256;
constexpr int kKC = 64;  // rows of W per smem chunk (4 groups of 16)

template <int NT, int MW>
__global__ void __launch_bounds__(kMmaThreads) k_xtw_mma(const double* __restrict__ X, int64_t ldx, int n,
                                                         int rows_per_split, int rows_total,
                                                         const double* __restrict__ W, int64_t ldw, int pc,
                                                         double* __restrict__ out, int64_t ldo,
                                                         size_t split_stride) {
  constexpr int BP = b_pitch<NT>();
  __shared__ __align__(16) double Ws[2][kKC * BP];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int col0 = (blockIdx.x * (kMmaThreads / 32) + warp) * (8 * MW);
  const int r0 = blockIdx.y * rows_per_split;
  const int r1 = min(r0 + rows_per_split, rows_total);
  double acc[MW][NT][2];
#pragma unroll
  for (int mt = 0; mt < MW; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
  const double* xc[MW];
  bool live[MW];
#pragma unroll
  for (int mt = 0; mt < MW; ++mt) {
    const int col = col0 + mt * 8 + gq;
    live[mt] = col < n;
    xc[mt] = X + static_cast<int64_t>(live[mt] ? col : 0) * ldx + 4 * tq;
  }
  auto stage_w = [&](int buf, int rbase) {  // asynchronous: no register round trip
    for (int e = threadIdx.x; e < kKC * 8 * NT; e += kMmaThreads) {
      const int rr = e / (8 * NT), c = e - rr * (8 * NT);
      const int r = rbase + rr;
      const bool ok = c < pc && r < r1;
      cp_async8(&Ws[buf][rr * BP + c], W + (ok ? static_cast<int64_t>(r) * ldw + c : 0), ok);
    }
    cp_async_commit();
  };
  int buf = 0;
  if (r0 < r1) stage_w(0, r0);
  cp_async_wait_all();
  __syncthreads();
  for (int rb = r0; rb < r1; rb += kKC) {
    if (rb + kKC < r1) stage_w(buf ^ 1, rb + kKC);
    const double* ws = Ws[buf];
    const int nkb = (min(kKC, r1 - rb) + 15) / 16;
    double av[4][MW][4];
#pragma unroll
    for (int kb = 0; kb < 4; ++kb)
#pragma unroll
      for (int mt = 0; mt < MW; ++mt) {
        if (kb < nkb && rb + 16 * kb + 4 * tq < r1) {  // 4-row groups never straddle r1 (multiples of 4)
          asm("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
              : "=d"(av[kb][mt][0]), "=d"(av[kb][mt][1]), "=d"(av[kb][mt][2]), "=d"(av[kb][mt][3])
              : "l"(xc[mt] + rb + 16 * kb));
        } else {
          av[kb][mt][0] = av[kb][mt][1] = av[kb][mt][2] = av[kb][mt][3] = 0.0;
        }
      }
#pragma unroll
    for (int kb = 0; kb < 4; ++kb) {
      if (kb >= nkb) break;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double* wr = ws + (16 * kb + 4 * tq + u) * BP + gq;
        double bfr[NT];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) bfr[nt] = wr[nt * 8];
#pragma unroll
        for (int mt = 0; mt < MW; ++mt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) mma884(acc[mt][nt][0], acc[mt][nt][1], av[kb][mt][u], bfr[nt]);
      }
    }
    cp_async_wait_all();
    __syncthreads();
    buf ^= 1;
  }
  double* o = out + blockIdx.y * split_stride;
#pragma unroll
  for (int mt = 0; mt < MW; ++mt) {
    const int col = col0 + mt * 8 + gq;
    if (col >= n) continue;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int c = nt * 8 + 2 * tq;
      double* dst = o + static_cast<int64_t>(col) * ldo + c;
      if (c + 1 < pc) {
        dst[0] = acc[mt][nt][0];
        dst[1] = acc[mt][nt][1];
      } else if (c < pc) {
        dst[0] = acc[mt][nt][0];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Z = X Y on the FP64 tensor path.  M = rows of X (a warp owns MW = 4 m-tiles:
// 32 rows, loaded 2 consecutive rows per lane with a 128-bit load, so tile
// pairs hold the even / odd rows of 16), N = NT n-tiles, K = columns of X in
// KC-column chunks whose Y rows are staged in shared memory.  Column splits
// write partials (fixed-order sum afterwards).
// ---------------------------------------------------------------------------
template <int NT>
__global__ void __launch_bounds__(kMmaThreads) k_xy_mma(const double* __restrict__ X, int64_t ldx, int rows_total,
                                                        int cols_per_split, int n, const double* __restrict__ Y,
                                                        int64_t ldy, int pc, double* __restrict__ out, int64_t ldo,
                                                        size_t split_stride) {
  constexpr int BP = b_pitch<NT>();
  constexpr int MW = 4;
  __shared__ __align__(16) double Ys[2][kKC * BP];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int rbase = blockIdx.x * (kMmaThreads / 32) * 32 + warp * 32;  // 32 rows per warp
  const int j0 = blockIdx.y * cols_per_split;
  const int j1 = min(j0 + cols_per_split, n);
  double acc[MW][NT][2];
#pragma unroll
  for (int mt = 0; mt < MW; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
  // lane's two row pairs: rows rbase + 16h + 2g + {0, 1}, h = 0, 1
  const bool live0 = rbase + 2 * gq + 1 < rows_total, live1 = rbase + 16 + 2 * gq + 1 < rows_total;
  const double* xr0 = X + (live0 ? rbase + 2 * gq : 0);
  const double* xr1 = X + (live1 ? rbase + 16 + 2 * gq : 0);
  auto stage_y = [&](int buf, int jb) {  // asynchronous: no register round trip
    for (int e = threadIdx.x; e < kKC * 8 * NT; e += kMmaThreads) {
      const int jj = e / (8 * NT), c = e - jj * (8 * NT);
      const int j = jb + jj;
      const bool ok = c < pc && j < j1;
      cp_async8(&Ys[buf][jj * BP + c], Y + (ok ? static_cast<int64_t>(j) * ldy + c : 0), ok);
    }
    cp_async_commit();
  };
  int buf = 0;
  if (j0 < j1) stage_y(0, j0);
  cp_async_wait_all();
  __syncthreads();
  for (int jb = j0; jb < j1; jb += kKC) {
    if (jb + kKC < j1) stage_y(buf ^ 1, jb + kKC);
    const double* ys = Ys[buf];
    const int nk = min(kKC, j1 - jb);
    for (int k0 = 0; k0 < nk; k0 += 16) {
      double2 a0[4], a1[4];
#pragma unroll
      for (int s4 = 0; s4 < 4; ++s4) {
        const int j = jb + k0 + 4 * s4 + tq;
        const bool ok = k0 + 4 * s4 + tq < nk;
        a0[s4] = ok ? ldg2(xr0 + static_cast<int64_t>(j) * ldx) : make_double2(0.0, 0.0);
        a1[s4] = ok ? ldg2(xr1 + static_cast<int64_t>(j) * ldx) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int s4 = 0; s4 < 4; ++s4) {
        const double* yr = ys + (k0 + 4 * s4 + tq) * BP + gq;
        double bfr[NT];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) bfr[nt] = yr[nt * 8];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          mma884(acc[0][nt][0], acc[0][nt][1], a0[s4].x, bfr[nt]);  // even rows of 0..15
          mma884(acc[1][nt][0], acc[1][nt][1], a0[s4].y, bfr[nt]);  // odd rows of 0..15
          mma884(acc[2][nt][0], acc[2][nt][1], a1[s4].x, bfr[nt]);  // even rows of 16..31
          mma884(acc[3][nt][0], acc[3][nt][1], a1[s4].y, bfr[nt]);  // odd rows of 16..31
        }
      }
    }
    cp_async_wait_all();
    __syncthreads();
    buf ^= 1;
  }
  double* o = out + blockIdx.y * split_stride;
#pragma unroll
  for (int mt = 0; mt < MW; ++mt) {
    // C fragment row index gq of tile mt -> physical row
    const int row = rbase + 16 * (mt >> 1) + 2 * gq + (mt & 1);
    if (row >= rows_total) continue;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int c = nt * 8 + 2 * tq;
      double* dst = o + static_cast<int64_t>(row) * ldo + c;
      if (c + 1 < pc) {
        dst[0] = acc[mt][nt][0];
        dst[1] = acc[mt][nt][1];
      } else if (c < pc) {
        dst[0] = acc[mt][nt][0];
      }
    }
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

// ---- tensor-path launchers (pc >= 3) ----------------------------------------
template <int NT>
void xtw_mma_chunk(const DenseX& X, const double* W, int64_t ldw, int pc, double* Y, int64_t ldy, GramWork& work,
                   cudaStream_t st, int rs, int rows_per_split) {
  constexpr int MW = 2;
  const int rows_total = static_cast<int>(X.ld);
  const int col_tiles = static_cast<int>(ceil_div(X.n, (kMmaThreads / 32) * 8 * MW));
  dim3 grid(col_tiles, rs);
  if (rs == 1) {
    k_xtw_mma<NT, MW><<<grid, kMmaThreads, 0, st>>>(X.x, X.ld, X.n, rows_per_split, rows_total, W, ldw, pc, Y, ldy, 0);
    GAPLRA_LAUNCH_CHECK();
    return;
  }
  const size_t stride = static_cast<size_t>(X.n) * pc;
  if (work.part_elems < stride * rs) throw Error(kContractViolation, "xtw_mma: workspace too small");
  k_xtw_mma<NT, MW><<<grid, kMmaThreads, 0, st>>>(X.x, X.ld, X.n, rows_per_split, rows_total, W, ldw, pc, work.part,
                                                  pc, stride);
  GAPLRA_LAUNCH_CHECK();
  k_sum_splits<<<sm_count() * 4, 256, 0, st>>>(work.part, rs, stride, X.n, pc, pc, Y, ldy);
  GAPLRA_LAUNCH_CHECK();
}

struct MmaPlan {
  int rs, rows_per_split;   // xtw
  int s, cols_per_split;    // xy
};

MmaPlan mma_plan(const DenseX& X) {
  MmaPlan pl;
  const int rows_total = static_cast<int>(X.ld);
  const int col_tiles = static_cast<int>(ceil_div(X.n, (kMmaThreads / 32) * 16));
  const int slots = sm_count() * 2;
  int rs = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(3 * slots, col_tiles), rows_total / 512)));
  pl.rows_per_split = static_cast<int>(ceil_div(ceil_div(rows_total, rs), kKC) * kKC);
  pl.rs = static_cast<int>(ceil_div(rows_total, pl.rows_per_split));
  const int row_blocks = static_cast<int>(ceil_div(rows_total, 256));
  int s = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(3 * slots, row_blocks), ceil_div(X.n, 256))));
  pl.cols_per_split = static_cast<int>(ceil_div(ceil_div(X.n, s), kKC) * kKC);
  pl.s = static_cast<int>(ceil_div(X.n, pl.cols_per_split));
  return pl;
}

template <int NT>
void xy_mma_chunk(const DenseX& X, const double* Y, int64_t ldy, int pc, double* Z, int64_t ldz, GramWork& work,
                  cudaStream_t st, int s, int cols_per_split) {
  const int rows_total = static_cast<int>(X.ld);
  dim3 grid(static_cast<unsigned>(ceil_div(rows_total, 256)), s);
  const size_t stride = static_cast<size_t>(rows_total) * pc;
  if (s == 1) {
    k_xy_mma<NT><<<grid, kMmaThreads, 0, st>>>(X.x, X.ld, rows_total, cols_per_split, X.n, Y, ldy, pc, Z, ldz, 0);
    GAPLRA_LAUNCH_CHECK();
    return;
  }
  if (work.part_elems < stride * s) throw Error(kContractViolation, "xy_mma: workspace too small");
  k_xy_mma<NT><<<grid, kMmaThreads, 0, st>>>(X.x, X.ld, rows_total, cols_per_split, X.n, Y, ldy, pc, work.part, pc,
                                             stride);
  GAPLRA_LAUNCH_CHECK();
  k_sum_splits<<<sm_count() * 4, 256, 0, st>>>(work.part, s, stride, rows_total, pc, pc, Z, ldz);
  GAPLRA_LAUNCH_CHECK();
}

bool use_mma(int pc) {
  static const int mode = getenv("GAPLRA_GRAM_MMA") ? atoi(getenv("GAPLRA_GRAM_MMA")) : 1;
  return mode != 0 && pc >= 3;
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
    if (use_mma(pc)) {
      const MmaPlan m = mma_plan(X);
      if (m.rs > 1) need = std::max(need, static_cast<size_t>(m.rs) * X.n * pc);
      if (m.s > 1) need = std::max(need, static_cast<size_t>(m.s) * X.ld * pc);
      continue;
    }
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
    if (use_mma(pc)) {
      const MmaPlan m = mma_plan(X);
      switch ((pc + 7) / 8) {
        case 1: xtw_mma_chunk<1>(X, W + c0, ldw, pc, Y + c0, ldy, work, st, m.rs, m.rows_per_split); break;
        case 2: xtw_mma_chunk<2>(X, W + c0, ldw, pc, Y + c0, ldy, work, st, m.rs, m.rows_per_split); break;
        case 3: xtw_mma_chunk<3>(X, W + c0, ldw, pc, Y + c0, ldy, work, st, m.rs, m.rows_per_split); break;
        default: xtw_mma_chunk<4>(X, W + c0, ldw, pc, Y + c0, ldy, work, st, m.rs, m.rows_per_split); break;
      }
      continue;
    }
    dispatch_nc<XtwRun>(pick_nc(pc), X, W + c0, ldw, pc, Y + c0, ldy, work, st);
  }
}

void launch_xy(const DenseX& X, const double* Y, int64_t ldy, int p, double* Z, int64_t ldz, GramWork& work,
               cudaStream_t st) {
  for (int c0 = 0; c0 < p; c0 += 32) {
    const int pc = std::min(32, p - c0);
    if (use_mma(pc)) {
      const MmaPlan m = mma_plan(X);
      switch ((pc + 7) / 8) {
        case 1: xy_mma_chunk<1>(X, Y + c0, ldy, pc, Z + c0, ldz, work, st, m.s, m.cols_per_split); break;
        case 2: xy_mma_chunk<2>(X, Y + c0, ldy, pc, Z + c0, ldz, work, st, m.s, m.cols_per_split); break;
        case 3: xy_mma_chunk<3>(X, Y + c0, ldy, pc, Z + c0, ldz, work, st, m.s, m.cols_per_split); break;
        default: xy_mma_chunk<4>(X, Y + c0, ldy, pc, Z + c0, ldz, work, st, m.s, m.cols_per_split); break;
      }
      continue;
    }
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
