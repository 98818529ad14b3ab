// X·(XᵀW) pass kernels — see gram.cuh for the contract.
//
// Layouts: X dense column-major (ld % 4 == 0, zero pad rows); d x p blocks are
// ROW-MAJOR (d_pad x ldp), the reference's DenseMatrix layout
// (proj/core/include/gaplra/dense_matrix.hpp:22-23), so host and device blocks
// share one layout and no transposes happen at the boundary.
#include "gram.cuh"

#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <vector>

namespace gaplra_cuda {

namespace cg = cooperative_groups;

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
  extern __shared__ __align__(16) double xtw_ws[];  // [2][kKC * BP]: 74 KB at NT = 8 (dynamic)
  auto Ws = [&](int b) { return xtw_ws + b * (kKC * BP); };
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
      cp_async8(Ws(buf) + rr * BP + c, W + (ok ? static_cast<int64_t>(r) * ldw + c : 0), ok);
    }
    cp_async_commit();
  };
  int buf = 0;
  if (r0 < r1) stage_w(0, r0);
  cp_async_wait_all();
  __syncthreads();
  for (int rb = r0; rb < r1; rb += kKC) {
    if (rb + kKC < r1) stage_w(buf ^ 1, rb + kKC);
    const double* ws = Ws(buf);
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
  constexpr int MW = 2;  // (MW = 1 at NT = 8, two CTAs per SM: 101 vs 81 ms at C5, slower still)
  constexpr size_t smem = 2 * kKC * b_pitch<NT>() * sizeof(double);
  static bool attr = false;
  if (!attr && smem > 48 * 1024) {
    GAPLRA_CUDA_CHECK(cudaFuncSetAttribute(k_xtw_mma<NT, MW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem)));
    attr = true;
  }
  const int rows_total = static_cast<int>(X.ld);
  const int col_tiles = static_cast<int>(ceil_div(X.n, (kMmaThreads / 32) * 8 * MW));
  dim3 grid(col_tiles, rs);
  if (rs == 1) {
    k_xtw_mma<NT, MW><<<grid, kMmaThreads, smem, st>>>(X.x, X.ld, X.n, rows_per_split, rows_total, W, ldw, pc, Y, ldy,
                                                       0);
    GAPLRA_LAUNCH_CHECK();
    return;
  }
  const size_t stride = static_cast<size_t>(X.n) * pc;
  if (work.part_elems < stride * rs) throw Error(kContractViolation, "xtw_mma: workspace too small");
  k_xtw_mma<NT, MW><<<grid, kMmaThreads, smem, st>>>(X.x, X.ld, X.n, rows_per_split, rows_total, W, ldw, pc,
                                                     work.part, pc, stride);
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
// Single-pass Z = X (Xᵀ W) (and Y = Xᵀ W), X read from HBM once (north star
// item 2).
//
// One thread-block cluster of G CTAs splits the d rows (R = 256 or 128 rows per
// CTA); W's row slice stays in shared memory and Z's row slice in registers for
// the whole pass, so only X streams.  The clusters take 16-column tiles of X
// round-robin.  Warp roles per CTA:
//   producer  one cp.async.bulk per column slice into a 2-4 stage ring
//   8 compute A  Ŷ_g = X_tile[rows g]ᵀ W[rows g]  (DMMA m8n8k4; warp = m-tile x
//                K quarter), partials to a double-buffered shared slab
//             B  Z[rows g] += X_tile[rows g] · Y_tile  (DMMA, accumulators in
//                registers; the tile's X fragments are re-read from L2 one
//                iteration ahead, so the stage is freed right after A)
//   2 exchange RS: fixed-order sum of the K quarters, entry chunk q st.async'd
//                to CTA q (complete_tx on q's mbarrier); AG: q sums the G
//                chunks in rank order, writes them to Y and st.async's them to
//                every CTA
// Compute iteration t runs A(t+2) | B(t) while the exchange warps run RS(t+2)
// and AG(t+1), so each DSMEM exchange has a whole iteration to land.  Every
// reduction has a fixed order, so the pass is bitwise run-to-run stable.  The
// cluster partials of Z are summed in cluster order by k_sum_splits.
// Shared-memory pitches (doubles): X slices XP = R + 4 (XP/2 ≡ 2 mod 8), W rows
// BP = 8NT + 2 (≡ 2 mod 8), Y_tile rows YP = 8NT + 4; with the column
// permutation perm(gq) in phase A the fragment loads are bank-conflict free.
// Measured (GAPLRA_GRAM_TIMING, tools/gram_probe.py): at d = 4096 only seven
// 16-CTA clusters are resident (112 of 148 SMs) and a tile costs ~5300 cycles at
// p = 20 (DMMA issue 57 % of peak on the active SMs) — slower than the two-pass
// kernels there, faster at d <= 1024, where it is the default (plan()).
// ---------------------------------------------------------------------------
namespace fused {

constexpr int kNB = 16;  // columns of X per tile
constexpr int kWarps = 8;  // compute (DMMA) warps
constexpr int kXch = 2;    // exchange warps: reduce-scatter / all-gather over DSMEM
constexpr int kThreads = 32 * (kWarps + kXch + 1);  // + one producer warp

__host__ __device__ constexpr int bp(int nt) { return 8 * nt + 2; }
__host__ __device__ constexpr int yp(int nt) { return 8 * nt + 4; }  // ≡ 4 or 12 (mod 16)
constexpr int kSlots = 3;     // exchange slots: tiles t, t+1, t+2 in flight
constexpr int kRedParts = 4;  // phase A: warp = (m-tile, K quarter)

struct Layout {
  int xp, stage, off_w, off_red, off_rs, off_yt, off_ys, off_bar, ch;
  size_t bytes;
};
__host__ __device__ inline Layout layout(int nt, int r, int g, int stages) {
  Layout L;
  L.xp = r + 4;
  L.stage = kNB * L.xp;
  L.ch = kNB * 8 * nt / g;
  L.off_w = stages * L.stage;
  L.off_red = L.off_w + r * bp(nt);
  L.off_rs = L.off_red + 2 * kRedParts * kNB * 8 * nt;
  L.off_yt = L.off_rs + kSlots * g * L.ch;
  L.off_ys = L.off_yt + kSlots * kNB * yp(nt);
  L.off_bar = L.off_ys + L.ch;
  L.bytes = static_cast<size_t>(L.off_bar + 24) * sizeof(double);
  return L;
}

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(count));
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n\t}" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
// producer-side wait: back off instead of spinning (the producers run ahead)
__device__ __forceinline__ void bar_wait_backoff(uint64_t* b, uint32_t parity) {
  for (;;) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(su32(b)), "r"(parity)
        : "memory");
    if (done) return;
    __nanosleep(64);
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(b))
               : "memory");
}
__device__ __forceinline__ uint32_t peer_addr(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
// 16-byte remote store completing 16 transaction bytes on the peer's mbarrier
__device__ __forceinline__ void st_async2(uint32_t raddr, double2 v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];" ::"r"(raddr),
               "l"(__double_as_longlong(v.x)), "l"(__double_as_longlong(v.y)), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void compute_sync() { asm volatile("bar.sync 1, %0;" ::"n"(32 * kWarps) : "memory"); }

struct Args {
  const double* X;
  int64_t ldx;
  int n, rows_total;
  const double* W;
  int64_t ldw;
  int pc;
  double* Y;
  int64_t ldy;
  double* Z;  // Z (one cluster) or part + cluster * zstride (ld = pc)
  int64_t ldz;
  size_t zstride;
  int stages;
  long long* dbg;  // GAPLRA_GRAM_TIMING: per-CTA cycle counters (thread 0), else null
};

template <int NT, int R>
__global__ void __launch_bounds__(kThreads, 1) k_gram_fused(Args a) {
  constexpr int RW = R / kWarps;  // rows per compute warp
  constexpr int NC8 = 8 * NT, BP = bp(NT), YP = yp(NT);
  constexpr int NP = kNB * NC8 / 2;              // entry pairs of a tile's Ŷ
  constexpr int PER = (NP + 32 * kXch - 1) / (32 * kXch);  // pairs per exchange thread
  static_assert(RW % 16 == 0, "phase B takes 16-row groups");
  extern __shared__ __align__(128) double sm[];
  cg::cluster_group cluster = cg::this_cluster();
  const int G = static_cast<int>(cluster.num_blocks());
  const int g = static_cast<int>(cluster.block_rank());
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int S = a.stages;
  const Layout L = layout(NT, R, G, S);
  const int XP = L.xp, CH = L.ch;
  double* Ws = sm + L.off_w;
  double* red = sm + L.off_red;  // [2][kRedParts][kNB][NC8]
  double* rs = sm + L.off_rs;    // [kSlots][G][CH]
  double* yt = sm + L.off_yt;    // [kSlots][kNB][YP]
  double* ysum = sm + L.off_ys;  // [CH]
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + L.off_bar);
  uint64_t* empty = full + 4;
  uint64_t* rsb = full + 8;        // [kSlots]
  uint64_t* agb = full + 11;       // [kSlots]
  uint64_t* red_full = full + 14;  // [2]
  uint64_t* red_empty = full + 16; // [2]
  const int r0 = g * R;
  const int rc = max(0, min(R, a.rows_total - r0));
  const int ncl = gridDim.y, ci = blockIdx.y;
  const int T = static_cast<int>((a.n + kNB - 1) / kNB);
  const int Tl = ci < T ? (T - 1 - ci) / ncl + 1 : 0;
  auto tile_col0 = [&](int lt) { return (ci + lt * ncl) * kNB; };
  // GAPLRA_GRAM_TIMING: wait cycles of lane 0 of the first warp of each role
  long long tw[4] = {0, 0, 0, 0};
  const bool rec = a.dbg && lane == 0 && (warp == 0 || warp == kWarps || warp == kWarps + kXch);
  auto timed_wait = [&](int k, uint64_t* b, uint32_t par) {
    const long long t = rec ? clock64() : 0;
    bar_wait(b, par);
    if (rec) tw[k] += clock64() - t;
  };

  for (int e = tid; e < L.off_bar; e += blockDim.x) sm[e] = 0.0;
  __syncthreads();
  for (int e = tid; e < rc * a.pc; e += blockDim.x) {
    const int r = e / a.pc, c = e - (e / a.pc) * a.pc;
    Ws[r * BP + c] = a.W[static_cast<int64_t>(r0 + r) * a.ldw + c];
  }
  if (tid == 0) {
    for (int s = 0; s < 4; ++s) {
      bar_init(&full[s], 1);
      bar_init(&empty[s], kWarps);
    }
    for (int s = 0; s < kSlots; ++s) {
      bar_init(&rsb[s], 1);
      bar_init(&agb[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      bar_init(&red_full[s], 32 * kWarps);
      bar_init(&red_empty[s], 32 * kXch);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < kSlots && s < Tl; ++s) {
      bar_expect(&rsb[s], static_cast<uint32_t>(G * CH * 8));
      bar_expect(&agb[s], static_cast<uint32_t>(kNB * NC8 * 8));
    }
  }
  cluster.sync();

  if (warp >= kWarps + kXch) {  // ----------------------------------------- producer
    if (lane == 0) {
      for (int lt = 0; lt < Tl; ++lt) {
        const int s = lt % S;
        const long long tb = rec ? clock64() : 0;
        if (lt >= S) bar_wait_backoff(&empty[s], static_cast<uint32_t>(((lt / S) & 1) ^ 1));
        if (rec) tw[0] += clock64() - tb;
        const int j0 = tile_col0(lt);
        const int nv = min(kNB, a.n - j0);
        bar_expect(&full[s], static_cast<uint32_t>(nv * rc * 8));
        double* dst = sm + s * L.stage;
        for (int c = 0; c < nv; ++c)
          bulk_g2s(dst + c * XP, a.X + static_cast<int64_t>(j0 + c) * a.ldx + r0, static_cast<uint32_t>(rc * 8),
                   &full[s]);
      }
    }
  } else if (warp >= kWarps) {  // ------------------------------------------ exchange
    const int xt = tid - 32 * kWarps;
    // fixed per-thread targets: RS pair i -> CTA q = 2i / CH; AG send k -> (pair k % (CH/2), CTA k / (CH/2))
    uint32_t rs_addr[PER], rs_bar[PER], ag_addr[PER], ag_bar[PER];
    int ag_pair[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int i = min(xt + 32 * kXch * j, NP - 1);
      const int e = 2 * i, q = e / CH, off = e - q * CH;
      rs_addr[j] = peer_addr(su32(rs) + (g * CH + off) * 8u, q);
      rs_bar[j] = peer_addr(su32(&rsb[0]), q);
      const int half = CH / 2;
      const int pr = i % half, qa = i / half;
      const int ea = g * CH + 2 * pr, col = ea / NC8, rhs = ea - col * NC8;
      ag_pair[j] = pr;
      ag_addr[j] = peer_addr(su32(yt) + (col * YP + rhs) * 8u, qa);
      ag_bar[j] = peer_addr(su32(&agb[0]), qa);
    }
    auto xch_sync = []() { asm volatile("bar.sync 2, %0;" ::"n"(32 * kXch) : "memory"); };
    auto rs_step = [&](int t) {  // fixed-order sum of the K quarters, reduce-scatter
      const int b = t & 1;
      timed_wait(0, &red_full[b], static_cast<uint32_t>((t >> 1) & 1));
      const double* rb = red + b * kRedParts * kNB * NC8;
      const int slot = t % kSlots;
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        const int i = xt + 32 * kXch * j;
        if (i < NP) {
          double2 v = *reinterpret_cast<const double2*>(rb + 2 * i);
#pragma unroll
          for (int w = 1; w < kRedParts; ++w) {
            const double2 u = *reinterpret_cast<const double2*>(rb + w * kNB * NC8 + 2 * i);
            v.x += u.x;
            v.y += u.y;
          }
          st_async2(rs_addr[j] + slot * G * CH * 8u, v, rs_bar[j] + slot * 8u);
        }
      }
      bar_arrive(&red_empty[b]);
    };
    auto ag_step = [&](int t) {  // owner sum in rank order, all-gather, Y to HBM
      const int slot = t % kSlots;
      timed_wait(1, &rsb[slot], static_cast<uint32_t>((t / kSlots) & 1));
      if (xt == 0 && t + kSlots < Tl) bar_expect(&rsb[slot], static_cast<uint32_t>(G * CH * 8));
      const double* rsl = rs + slot * G * CH;
      xch_sync();  // the previous step's ysum reads are done
      const int j0 = tile_col0(t);
      for (int pr = xt; pr < CH / 2; pr += 32 * kXch) {
        double2 v = *reinterpret_cast<const double2*>(rsl + 2 * pr);
#pragma unroll
        for (int s2 = 1; s2 < 16; ++s2) {
          if (s2 < G) {
            const double2 u = *reinterpret_cast<const double2*>(rsl + s2 * CH + 2 * pr);
            v.x += u.x;
            v.y += u.y;
          }
        }
        *reinterpret_cast<double2*>(ysum + 2 * pr) = v;
        const int e = g * CH + 2 * pr, col = e / NC8, rhs = e - col * NC8;
        if (j0 + col < a.n) {
          double* yo = a.Y + static_cast<int64_t>(j0 + col) * a.ldy + rhs;
          if (rhs + 1 < a.pc) {
            yo[0] = v.x;
            yo[1] = v.y;
          } else if (rhs < a.pc) {
            yo[0] = v.x;
          }
        }
      }
      xch_sync();
#pragma unroll
      for (int j = 0; j < PER; ++j)
        if (xt + 32 * kXch * j < NP)
          st_async2(ag_addr[j] + slot * kNB * YP * 8u, *reinterpret_cast<const double2*>(ysum + 2 * ag_pair[j]),
                    ag_bar[j] + slot * 8u);
    };
#pragma unroll 1
    for (int t = 0; t <= Tl; ++t) {
      if (t < Tl) rs_step(t);
      if (t >= 1) ag_step(t - 1);
    }
  } else {  // ---------------------------------------------------------------- compute
    const int perm = ((gq & 1) << 1) | ((gq >> 1) & 1) | (gq & 4);  // 0 2 1 3 4 6 5 7
    double accz[RW / 16][2][NT][2];
#pragma unroll
    for (int h = 0; h < RW / 16; ++h)
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) accz[h][e][nt][0] = accz[h][e][nt][1] = 0.0;

    // phase A: warp w takes m-tile w / 4 (8 of the 16 columns) and the K
    // quarter w % 4 of the CTA's rows; the exchange warps sum the quarters
    auto phase_a = [&](int lt) {
      constexpr int RQ = R / kRedParts;
      const int mt = warp / kRedParts, kq = warp % kRedParts;
      const int s = lt % S;
      timed_wait(0, &full[s], static_cast<uint32_t>((lt / S) & 1));
      const double* xs = sm + s * L.stage + (mt * 8 + perm) * XP + kq * RQ + 2 * tq;
      const double* wsb = Ws + (kq * RQ + 2 * tq) * BP + gq;
      // NACC independent accumulator sets (summed in order at the end): the
      // DMMA latency (~120 cycles) would otherwise serialise the K loop
      constexpr int NACC = NT == 1 ? 4 : 2;
      double acc[NACC][NT][2];
#pragma unroll
      for (int q = 0; q < NACC; ++q)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) acc[q][nt][0] = acc[q][nt][1] = 0.0;
#pragma unroll
      for (int kb = 0; kb < RQ / 8; ++kb) {
        const double2 av = *reinterpret_cast<const double2*>(xs + 8 * kb);
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int q = (2 * kb + u) % NACC;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
            mma884(acc[q][nt][0], acc[q][nt][1], u ? av.y : av.x, wsb[(8 * kb + u) * BP + nt * 8]);
        }
      }
#pragma unroll
      for (int q = 1; q < NACC; ++q)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          acc[0][nt][0] += acc[q][nt][0];
          acc[0][nt][1] += acc[q][nt][1];
        }
      __syncwarp();
      if (lane == 0) bar_arrive(&empty[s]);  // phase B re-reads the tile from L2, not from the stage
      const int b = lt & 1;
      if (lt >= 2) timed_wait(1, &red_empty[b], static_cast<uint32_t>(((lt >> 1) & 1) ^ 1));
      double* rb = red + b * kRedParts * kNB * NC8;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
        *reinterpret_cast<double2*>(rb + (kq * kNB + mt * 8 + perm) * NC8 + nt * 8 + 2 * tq) =
            make_double2(acc[0][nt][0], acc[0][nt][1]);
      bar_arrive(&red_full[b]);
    };

    // phase B operands: the tile's X fragments, re-read from L2 (the tile left
    // HBM two iterations earlier) into registers one iteration ahead of use,
    // so the shared-memory stage is free as soon as phase A has read it
    const int rbase = warp * RW + 2 * gq;
    auto load_b = [&](int lt, double2 (&xb)[RW / 16][kNB / 4]) {
      const int j0 = tile_col0(lt);
#pragma unroll
      for (int ks = 0; ks < kNB / 4; ++ks) {
        const int j = j0 + 4 * ks + tq;
#pragma unroll
        for (int h = 0; h < RW / 16; ++h) {
          const int row = rbase + 16 * h;
          xb[h][ks] = (j < a.n && row < rc) ? ldg2(a.X + static_cast<int64_t>(j) * a.ldx + r0 + row)
                                            : make_double2(0.0, 0.0);
        }
      }
    };
    auto phase_b = [&](int lt, const double2 (&xb)[RW / 16][kNB / 4]) {
      const int slot = lt % kSlots;
      timed_wait(2, &agb[slot], static_cast<uint32_t>((lt / kSlots) & 1));
      if (tid == 0 && lt + kSlots < Tl) bar_expect(&agb[slot], static_cast<uint32_t>(kNB * NC8 * 8));
      const double* ys = yt + slot * kNB * YP;
      const int nv = min(kNB, a.n - tile_col0(lt));
#pragma unroll
      for (int ks = 0; ks < kNB / 4; ++ks) {
        const int k = 4 * ks + tq;
        double bv[NT];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) bv[nt] = k < nv ? ys[k * YP + nt * 8 + gq] : 0.0;
#pragma unroll
        for (int h = 0; h < RW / 16; ++h) {
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            mma884(accz[h][0][nt][0], accz[h][0][nt][1], xb[h][ks].x, bv[nt]);
            mma884(accz[h][1][nt][0], accz[h][1][nt][1], xb[h][ks].y, bv[nt]);
          }
        }
      }
    };

    // software pipeline: compute iteration t runs A(t+2) then B(t); the
    // exchange warps run RS(t+2) and AG(t+1) meanwhile, so each exchange has
    // a whole iteration to land.  Slot reuse is safe with 3 slots: a peer
    // sends RS(t+3) / AG(t+3) only after this CTA's RS(t+3), which follows
    // the B(t) of every compute warp.
    long long t0 = clock64();
    if (Tl > 0) phase_a(0);
    if (Tl > 1) phase_a(1);
    if constexpr (NT <= 2) {
      // light DMMA work per tile: prefetch phase B's operands two tiles ahead
      double2 xa[RW / 16][kNB / 4], xc[RW / 16][kNB / 4];
      if (Tl > 0) load_b(0, xa);
      if (Tl > 1) load_b(1, xc);
#pragma unroll 1
      for (int lt = 0; lt < Tl; lt += 2) {
        if (lt + 2 < Tl) phase_a(lt + 2);
        phase_b(lt, xa);
        if (lt + 2 < Tl) load_b(lt + 2, xa);
        if (lt + 1 < Tl) {
          if (lt + 3 < Tl) phase_a(lt + 3);
          phase_b(lt + 1, xc);
          if (lt + 3 < Tl) load_b(lt + 3, xc);
        }
      }
    } else {
      double2 xb[RW / 16][kNB / 4];
#pragma unroll 1
      for (int lt = 0; lt < Tl; ++lt) {
        load_b(lt, xb);
        if (lt + 2 < Tl) phase_a(lt + 2);
        phase_b(lt, xb);
      }
    }
    if (a.dbg && tid == 0) {
      const int cta = blockIdx.y * gridDim.x + blockIdx.x;
      a.dbg[cta * 12 + 0] = clock64() - t0;
      a.dbg[cta * 12 + 10] = Tl;
    }
#pragma unroll
    for (int h = 0; h < RW / 16; ++h)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int row = warp * RW + 16 * h + 2 * gq + e;
        if (row >= rc) continue;
        double* zo = a.Z + ci * a.zstride + static_cast<int64_t>(r0 + row) * a.ldz;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int c = nt * 8 + 2 * tq;
          if (c + 1 < a.pc) {
            zo[c] = accz[h][e][nt][0];
            zo[c + 1] = accz[h][e][nt][1];
          } else if (c < a.pc) {
            zo[c] = accz[h][e][nt][0];
          }
        }
      }
  }
  if (rec) {
    const int cta = blockIdx.y * gridDim.x + blockIdx.x;
    const int base = warp == 0 ? 1 : (warp == kWarps ? 4 : 7);
    for (int k = 0; k < 3; ++k) a.dbg[cta * 12 + base + k] = tw[k];
  }
  cluster.sync();  // no CTA leaves while a peer may still st.async into it
}

struct Plan {
  int r = 0, g = 0, stages = 0, ncl = 0;
  size_t smem = 0;
};

template <int NT, int R>
int max_clusters(int G, size_t smem) {
  auto kern = k_gram_fused<NT, R>;
  GAPLRA_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  GAPLRA_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(G, 64, 1);
  lc.blockDim = dim3(kThreads, 1, 1);
  lc.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = G;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &lc) != cudaSuccess || n < 1) {
    (void)cudaGetLastError();
    n = std::max(1, sm_count() / G);
  }
  return n;
}

template <int NT, int R>
int max_clusters_cached(int G, size_t smem) {
  static std::map<std::pair<int, size_t>, int> cache;
  int& c = cache[{G, smem}];
  if (!c) c = max_clusters<NT, R>(G, smem);
  return c;
}

constexpr size_t kSmemCap = 227 * 1024;

// Layout for one <= 32-column chunk; g = 0 when the fused pass does not apply.
Plan plan(const DenseX& X, int pc) {
  Plan pl;
  // GAPLRA_GRAM_FUSED: 0 never, 2 wherever the layout fits, 1 (default) where
  // it measured faster than the two-pass kernels: d <= 1024 (C1: p = 10 0.042
  // vs 0.072 ms, p = 1 0.032 vs 0.062 ms).  At d = 4096 only seven 16-CTA
  // clusters fit (112 SMs) and the per-tile exchange costs more than the
  // second read of X saves (C2 p = 20: 2.4 vs 1.8 ms; p = 1: 1.2 vs 1.13 ms).
  static const int mode = getenv("GAPLRA_GRAM_FUSED") ? atoi(getenv("GAPLRA_GRAM_FUSED")) : 1;
  if (!mode || (mode == 1 && X.ld > 1024)) return pl;
  const int nt = (pc + 7) / 8;
  const int64_t ld = X.ld;
  // prefer 256 rows per CTA (fewer exchange bytes per X byte), then 128, and
  // four X stages (A(t+2) and B(t) hold two, one prefetches) over three
  int r = 0, gp = 0, stages = 0;
  for (int want = 4; want >= 2 && !r; --want)  // the ring holds only the tile phase A reads
    for (int rr : {256, 128}) {
      if (rr == 256 && ld <= 1024) continue;  // small d: keep clusters small
      int g = 1;
      while (g < ceil_div(ld, rr)) g <<= 1;
      if (g > 16 || layout(nt, rr, g, want).bytes > kSmemCap) continue;
      r = rr;
      gp = g;
      stages = want;
      break;
    }
  if (!r) return pl;
  pl.r = r;
  pl.g = gp;
  pl.stages = stages;
  pl.smem = layout(nt, r, gp, stages).bytes;
  return pl;
}

template <int NT, int R>
void launch_chunk(const DenseX& X, const double* W, int64_t ldw, int pc, double* Y, int64_t ldy, double* Z,
                  int64_t ldz, GramWork& work, cudaStream_t st, const Plan& pl) {
  const int T = static_cast<int>(ceil_div(X.n, kNB));
  const int ncl = std::max(1, std::min(max_clusters_cached<NT, R>(pl.g, pl.smem), T));
  Args args;
  args.X = X.x;
  args.ldx = X.ld;
  args.n = X.n;
  args.rows_total = static_cast<int>(X.ld);
  args.W = W;
  args.ldw = ldw;
  args.pc = pc;
  args.Y = Y;
  args.ldy = ldy;
  args.stages = pl.stages;
  args.dbg = nullptr;
  static const bool timing = getenv("GAPLRA_GRAM_TIMING") != nullptr;
  static long long* dbg_buf = nullptr;
  const int nctas = pl.g * ncl;
  if (timing) {
    if (!dbg_buf) GAPLRA_CUDA_CHECK(cudaMalloc(&dbg_buf, 12 * sizeof(long long) * 16 * 64));
    args.dbg = dbg_buf;
  }
  const size_t stride = static_cast<size_t>(X.ld) * pc;
  if (ncl == 1) {
    args.Z = Z;
    args.ldz = ldz;
    args.zstride = 0;
  } else {
    if (work.part_elems < stride * ncl) throw Error(kContractViolation, "gram_fused: workspace too small");
    args.Z = work.part;
    args.ldz = pc;
    args.zstride = stride;
  }
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(pl.g, ncl, 1);
  lc.blockDim = dim3(kThreads, 1, 1);
  lc.dynamicSmemBytes = pl.smem;
  lc.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = pl.g;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  auto kern = k_gram_fused<NT, R>;
  GAPLRA_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(pl.smem)));
  GAPLRA_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  static const bool dbg = getenv("GAPLRA_GRAM_DEBUG") != nullptr;
  if (dbg)
    fprintf(stderr, "gram_fused: ld %lld n %d pc %d -> R %d G %d stages %d smem %zu clusters %d\n",
            static_cast<long long>(X.ld), X.n, pc, pl.r, pl.g, pl.stages, pl.smem, ncl);
  GAPLRA_CUDA_CHECK(cudaLaunchKernelEx(&lc, kern, args));
  GAPLRA_LAUNCH_CHECK();
  if (timing) {  // cycles per tile, averaged over CTAs: wait X, wait RS, wait AG, compute_sync, rest
    std::vector<long long> h(static_cast<size_t>(nctas) * 12);
    GAPLRA_CUDA_CHECK(cudaMemcpyAsync(h.data(), dbg_buf, h.size() * sizeof(long long), cudaMemcpyDeviceToHost, st));
    GAPLRA_CUDA_CHECK(cudaStreamSynchronize(st));
    double v[10] = {}, tiles = 0;
    for (int c = 0; c < nctas; ++c) {
      for (int k = 0; k < 10; ++k) v[k] += h[c * 12 + k];
      tiles += h[c * 12 + 10];
    }
    for (double& x : v) x /= tiles;
    fprintf(stderr,
            "gram_fused timing (cycles/tile): total %.0f | compute wait X %.0f red_empty %.0f AG %.0f | exchange "
            "wait red_full %.0f RS %.0f | producer wait empty %.0f\n",
            v[0], v[1], v[2], v[3], v[4], v[5], v[7]);
  }
  if (ncl > 1) {
    k_sum_splits<<<sm_count() * 4, 256, 0, st>>>(work.part, ncl, stride, static_cast<int>(X.ld), pc, pc, Z, ldz);
    GAPLRA_LAUNCH_CHECK();
  }
}

int clusters_for(const DenseX& X, int pc, const Plan& pl) {
  const int T = static_cast<int>(ceil_div(X.n, kNB));
  int c = 0;
  switch ((pc + 7) / 8 * 1000 + pl.r) {
    case 1128: c = max_clusters_cached<1, 128>(pl.g, pl.smem); break;
    case 1256: c = max_clusters_cached<1, 256>(pl.g, pl.smem); break;
    case 2128: c = max_clusters_cached<2, 128>(pl.g, pl.smem); break;
    case 2256: c = max_clusters_cached<2, 256>(pl.g, pl.smem); break;
    case 3128: c = max_clusters_cached<3, 128>(pl.g, pl.smem); break;
    case 3256: c = max_clusters_cached<3, 256>(pl.g, pl.smem); break;
    case 4128: c = max_clusters_cached<4, 128>(pl.g, pl.smem); break;
    default: c = max_clusters_cached<4, 256>(pl.g, pl.smem); break;
  }
  return std::max(1, std::min(c, T));
}

}  // namespace fused

// ---------------------------------------------------------------------------
// Single-pass p = 1 gram pass (Alg. 3's power steps, tune_shift's estimates,
// every p = 1 SVRG epoch's anchor): z = X (Xᵀ w), y = Xᵀ w with X read once.
// The two-pass kernels read X twice (~1.15 ms at C2, 5.7 TB/s of traffic).
// One 512-thread CTA per SM owns a contiguous column range; a thread owns rows
// {2·tid, 2·tid + 1} + 1024·k of every column (16-byte loads), so a pair of
// columns sits in registers while the CTA reduces their dots (warp shuffles,
// then the 16 warp partials summed in fixed order by every thread) and then
// folds x_j y_j into the thread's z rows.  The next pair's loads are issued
// before the current pair's reduction.  Per-CTA z partials are summed in CTA
// order by k_p1_sum (deterministic).
// ---------------------------------------------------------------------------
namespace p1 {
constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;

// KR: double2 row pairs per thread (ld <= 1024 * KR); WZ = false: y = Xᵀ w only
// (the p = 1 epoch's H = Xᵀ C)
template <int KR, bool WZ>
__global__ void __launch_bounds__(kThreads, 1)
    k_gram_p1(const double* __restrict__ X, int64_t ldx, int n, const double* __restrict__ W, int64_t ldw,
              double* __restrict__ Y, int64_t ldy, double* __restrict__ part, int64_t cols_per_cta) {
  __shared__ double red[2][kWarps][2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t j0 = static_cast<int64_t>(blockIdx.x) * cols_per_cta;
  const int64_t j1 = min(static_cast<int64_t>(n), j0 + cols_per_cta);
  double2 w[KR], z[KR];
#pragma unroll
  for (int k = 0; k < KR; ++k) {
    const int64_t r = 2 * tid + 1024 * k;
    w[k].x = r < ldx ? W[r * ldw] : 0.0;
    w[k].y = r + 1 < ldx ? W[(r + 1) * ldw] : 0.0;
    z[k] = make_double2(0.0, 0.0);
  }
  auto load = [&](int64_t j, double2 (&xx)[2][KR]) {
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int k = 0; k < KR; ++k) {
        const int64_t r = 2 * tid + 1024 * k;
        xx[c][k] = j + c < j1 && r < ldx ? __ldcs(reinterpret_cast<const double2*>(X + (j + c) * ldx + r))
                                          : make_double2(0.0, 0.0);
      }
  };
  auto consume = [&](int64_t j, const double2 (&xx)[2][KR], int par) {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      s0 = fma(xx[0][k].x, w[k].x, fma(xx[0][k].y, w[k].y, s0));
      s1 = fma(xx[1][k].x, w[k].x, fma(xx[1][k].y, w[k].y, s1));
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, o);
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    }
    if (lane == 0) {
      red[par][warp][0] = s0;
      red[par][warp][1] = s1;
    }
    __syncthreads();  // (two parities: a thread writes red[par] again only after the next barrier)
    double y0 = 0.0, y1 = 0.0;
#pragma unroll
    for (int q = 0; q < kWarps; ++q) {
      y0 += red[par][q][0];
      y1 += red[par][q][1];
    }
    if (tid == 0) {
      if (j < j1) Y[j * ldy] = y0;
      if (j + 1 < j1) Y[(j + 1) * ldy] = y1;
    }
    if constexpr (WZ) {
#pragma unroll
      for (int k = 0; k < KR; ++k) {
        z[k].x = fma(xx[1][k].x, y1, fma(xx[0][k].x, y0, z[k].x));
        z[k].y = fma(xx[1][k].y, y1, fma(xx[0][k].y, y0, z[k].y));
      }
    }
  };
  double2 xa[2][KR], xb[2][KR];
  int64_t j = j0;
  if (j < j1) load(j, xa);
#pragma unroll 1
  for (; j < j1; j += 4) {
    load(j + 2, xb);
    consume(j, xa, 0);
    if (j + 2 >= j1) break;
    load(j + 4, xa);
    consume(j + 2, xb, 1);
  }
  if constexpr (WZ) {
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      const int64_t r = 2 * tid + 1024 * k;
      if (r < ldx) *reinterpret_cast<double2*>(part + blockIdx.x * ldx + r) = z[k];
    }
  }
}

// 4096 < ld <= 8192 (C5): a pair of 8192-row columns would not fit in the
// registers beside w and z, so w moves to shared memory and the columns go one
// at a time (still double-buffered: column j + 1's loads before column j's
// reduction)
template <bool WZ>
__global__ void __launch_bounds__(kThreads, 1)
    k_gram_p1_wide(const double* __restrict__ X, int64_t ldx, int n, const double* __restrict__ W, int64_t ldw,
                   double* __restrict__ Y, int64_t ldy, double* __restrict__ part, int64_t cols_per_cta) {
  constexpr int KR = 8;
  extern __shared__ __align__(16) double ws[];  // w, ldx doubles
  __shared__ double red[2][kWarps];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t j0 = static_cast<int64_t>(blockIdx.x) * cols_per_cta;
  const int64_t j1 = min(static_cast<int64_t>(n), j0 + cols_per_cta);
  for (int64_t r = tid; r < ldx; r += kThreads) ws[r] = W[r * ldw];
  __syncthreads();
  double2 z[KR];
#pragma unroll
  for (int k = 0; k < KR; ++k) z[k] = make_double2(0.0, 0.0);
  auto load = [&](int64_t j, double2 (&xx)[KR]) {
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      const int64_t r = 2 * tid + 1024 * k;
      xx[k] = j < j1 && r < ldx ? __ldcs(reinterpret_cast<const double2*>(X + j * ldx + r)) : make_double2(0.0, 0.0);
    }
  };
  auto consume = [&](int64_t j, const double2 (&xx)[KR], int par) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      const int r = 2 * tid + 1024 * k;
      if (r < ldx) {
        const double2 w2 = *reinterpret_cast<const double2*>(ws + r);
        s = fma(xx[k].x, w2.x, fma(xx[k].y, w2.y, s));
      }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) red[par][warp] = s;
    __syncthreads();
    double y = 0.0;
#pragma unroll
    for (int q = 0; q < kWarps; ++q) y += red[par][q];
    if (tid == 0 && j < j1) Y[j * ldy] = y;
    if constexpr (WZ) {
#pragma unroll
      for (int k = 0; k < KR; ++k) {
        z[k].x = fma(xx[k].x, y, z[k].x);
        z[k].y = fma(xx[k].y, y, z[k].y);
      }
    }
  };
  double2 xa[KR], xb[KR];
  int64_t j = j0;
  if (j < j1) load(j, xa);
#pragma unroll 1
  for (; j < j1; j += 2) {
    load(j + 1, xb);
    consume(j, xa, 0);
    if (j + 1 >= j1) break;
    load(j + 2, xa);
    consume(j + 1, xb, 1);
  }
  if constexpr (WZ) {
#pragma unroll
    for (int k = 0; k < KR; ++k) {
      const int64_t r = 2 * tid + 1024 * k;
      if (r < ldx) *reinterpret_cast<double2*>(part + blockIdx.x * ldx + r) = z[k];
    }
  }
}

__global__ void k_p1_sum(const double* __restrict__ part, int nblk, int64_t ldx, double* __restrict__ Z, int64_t ldz) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= ldx) return;
  double s = 0.0;
  for (int b = 0; b < nblk; ++b) s += part[b * ldx + r];
  Z[r * ldz] = s;
}

inline int ctas(const DenseX& X) { return std::max(1, std::min(sm_count(), static_cast<int>(ceil_div(X.n, 2)))); }

// GAPLRA_GRAM_P1=0 keeps the two-pass kernels at p = 1
bool applies(const DenseX& X) {
  static const int env = getenv("GAPLRA_GRAM_P1") ? atoi(getenv("GAPLRA_GRAM_P1")) : 1;
  return env && X.ld <= 8192 && X.ld % 2 == 0;
}
}  // namespace p1

// ---------------------------------------------------------------------------
// Z = X Y with X streamed through shared memory by a TMA producer warp
// (cp.async.bulk column slices into a 3-6 stage ring, the 16 Y rows of the
// tile in the same stage) and 8 DMMA warps — the single-pass kernel's phase B
// without the cluster exchange.  CTA = 256 rows x a column range; the Z row
// slice accumulates in registers; column splits write partials summed in
// order by k_sum_splits.  Replaces k_xy_mma (X loaded straight into registers:
// DRAM latency exposed at every 64-column chunk, long_scoreboard the top stall).
// ---------------------------------------------------------------------------
namespace xyt {

constexpr int kNB = 16, kWarps = 8, kThreads = 32 * (kWarps + 1), kR = 256, kXP = kR + 4;

struct Args {
  const double* X;
  int64_t ldx;
  int n, rows_total;
  const double* Y;
  int64_t ldy;
  int pc;
  double* Z;
  int64_t ldz;
  size_t zstride;
  int cols_per_split, stages;
};

// Y tile pitch ≡ 4 (mod 16) doubles: the B-fragment loads (k = 4 ks + tq, c = 8 nt + gq)
// are then conflict-free (a pitch ≡ 0, e.g. ldy = 64 at C5, was 4-way conflicted)
__host__ __device__ inline int64_t y_pitch(int64_t ldy) { return ldy + ((4 - ldy % 16) + 16) % 16; }
__host__ __device__ inline int stage_len(int64_t ldy) { return kNB * kXP + static_cast<int>(kNB * y_pitch(ldy)); }
__host__ __device__ inline size_t smem_bytes(int64_t ldy, int stages) {
  return (static_cast<size_t>(stage_len(ldy)) * stages + 16) * sizeof(double);
}

template <int NT>
__global__ void __launch_bounds__(kThreads, 1) k_xy_tma(Args a) {
  using namespace fused;
  extern __shared__ __align__(128) double sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int S = a.stages, SL = stage_len(a.ldy);
  const int YP = static_cast<int>(y_pitch(a.ldy));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + static_cast<size_t>(SL) * S);
  uint64_t* empty = full + 8;
  const int r0 = blockIdx.x * kR;
  const int rc = max(0, min(kR, a.rows_total - r0));
  const int j0 = blockIdx.y * a.cols_per_split;
  const int j1 = min(j0 + a.cols_per_split, a.n);
  const int T = j1 > j0 ? (j1 - j0 + kNB - 1) / kNB : 0;
  for (size_t e = tid; e < static_cast<size_t>(SL) * S; e += blockDim.x) sm[e] = 0.0;
  if (tid == 0) {
    for (int q = 0; q < S; ++q) {
      bar_init(&full[q], 1);
      bar_init(&empty[q], kWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == kWarps) {  // ------------------------------------------------- producer
    if (lane == 0)
      for (int lt = 0; lt < T; ++lt) {
        const int q = lt % S;
        if (lt >= S) bar_wait_backoff(&empty[q], static_cast<uint32_t>(((lt / S) & 1) ^ 1));
        const int j = j0 + lt * kNB;
        const int nv = min(kNB, j1 - j);
        bar_expect(&full[q], static_cast<uint32_t>(nv * (rc + a.ldy) * 8));
        double* st = sm + static_cast<size_t>(q) * SL;
        for (int c = 0; c < nv; ++c)
          bulk_g2s(st + c * kXP, a.X + static_cast<int64_t>(j + c) * a.ldx + r0, static_cast<uint32_t>(rc * 8),
                   &full[q]);
        if (YP == a.ldy) {
          bulk_g2s(st + kNB * kXP, a.Y + static_cast<int64_t>(j) * a.ldy, static_cast<uint32_t>(nv * a.ldy * 8),
                   &full[q]);
        } else {  // row by row into the padded pitch
          for (int c = 0; c < nv; ++c)
            bulk_g2s(st + kNB * kXP + c * YP, a.Y + static_cast<int64_t>(j + c) * a.ldy,
                     static_cast<uint32_t>(a.ldy * 8), &full[q]);
        }
      }
    return;
  }
  double acc[2][2][NT][2];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) acc[h][e][nt][0] = acc[h][e][nt][1] = 0.0;
  const int rw = warp * 32 + 2 * gq;
#pragma unroll 1
  for (int lt = 0; lt < T; ++lt) {
    const int q = lt % S;
    bar_wait(&full[q], static_cast<uint32_t>((lt / S) & 1));
    const double* xs = sm + static_cast<size_t>(q) * SL;
    const double* ys = xs + kNB * kXP;
    const int nv = min(kNB, j1 - (j0 + lt * kNB));
#pragma unroll
    for (int ks = 0; ks < kNB / 4; ++ks) {
      const int k = 4 * ks + tq;
      double b[NT];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int c = nt * 8 + gq;
        b[nt] = (k < nv && c < a.pc) ? ys[k * YP + c] : 0.0;
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double2 x2 = *reinterpret_cast<const double2*>(xs + k * kXP + rw + 16 * h);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          mma884(acc[h][0][nt][0], acc[h][0][nt][1], x2.x, b[nt]);
          mma884(acc[h][1][nt][0], acc[h][1][nt][1], x2.y, b[nt]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) bar_arrive(&empty[q]);
  }
  double* zb = a.Z + blockIdx.y * a.zstride;
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int row = warp * 32 + 16 * h + 2 * gq + e;
      if (row >= rc) continue;
      double* zo = zb + static_cast<int64_t>(r0 + row) * a.ldz;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int c = nt * 8 + 2 * tq;
        if (c + 1 < a.pc) {
          zo[c] = acc[h][e][nt][0];
          zo[c + 1] = acc[h][e][nt][1];
        } else if (c < a.pc) {
          zo[c] = acc[h][e][nt][0];
        }
      }
    }
}

struct Plan {
  int splits = 0, cols_per_split = 0, stages = 0;
  size_t smem = 0;
};

inline Plan plan(const DenseX& X, int64_t ldy) {
  Plan pl;
  const int row_blocks = static_cast<int>(ceil_div(X.ld, kR));
  int s = std::max(1, sm_count() / row_blocks);
  pl.cols_per_split = static_cast<int>(ceil_div(ceil_div(X.n, s), kNB) * kNB);
  pl.splits = static_cast<int>(ceil_div(X.n, pl.cols_per_split));
  pl.stages = 6;
  while (pl.stages > 2 && smem_bytes(ldy, pl.stages) > 227 * 1024) --pl.stages;
  pl.smem = smem_bytes(ldy, pl.stages);
  return pl;
}

template <int NT>
void launch(const DenseX& X, const double* Y, int64_t ldy, int pc, double* Z, int64_t ldz, GramWork& work,
            cudaStream_t st) {
  const Plan pl = plan(X, ldy);
  if (pc > 8 * NT) throw Error(kContractViolation, "xy_tma: pc > 8 NT");
  Args a;
  a.X = X.x;
  a.ldx = X.ld;
  a.n = X.n;
  a.rows_total = static_cast<int>(X.ld);
  a.Y = Y;
  a.ldy = ldy;
  a.pc = pc;
  a.cols_per_split = pl.cols_per_split;
  a.stages = pl.stages;
  const size_t stride = static_cast<size_t>(X.ld) * pc;
  if (pl.splits == 1) {
    a.Z = Z;
    a.ldz = ldz;
    a.zstride = 0;
  } else {
    if (work.part_elems < stride * pl.splits) throw Error(kContractViolation, "xy_tma: workspace too small");
    a.Z = work.part;
    a.ldz = pc;
    a.zstride = stride;
  }
  static bool attr = false;
  if (!attr) {
    GAPLRA_CUDA_CHECK(cudaFuncSetAttribute(k_xy_tma<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr = true;
  }
  dim3 grid(static_cast<unsigned>(ceil_div(X.ld, kR)), pl.splits);
  k_xy_tma<NT><<<grid, kThreads, pl.smem, st>>>(a);
  GAPLRA_LAUNCH_CHECK();
  if (pl.splits > 1) {
    k_sum_splits<<<sm_count() * 4, 256, 0, st>>>(work.part, pl.splits, stride, static_cast<int>(X.ld), pc, pc, Z, ldz);
    GAPLRA_LAUNCH_CHECK();
  }
}

// applies to pc >= 2 with an even Y leading dimension (16-byte bulk copies of Y rows)
inline bool applies(int pc, int64_t ldy) {
  static const int mode = getenv("GAPLRA_XY_TMA") ? atoi(getenv("GAPLRA_XY_TMA")) : 1;
  return mode != 0 && pc >= 2 && ldy % 2 == 0;
}


}  // namespace xyt

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

// X validation at matrix creation (sparse_matrix.cpp:29 rejects non-finite
// entries): flags[0] |= 1 on a non-finite entry in rows < d, |= 2 on a
// non-zero pad row (rows d..ld-1 must be zero: the kernels read whole columns).
__global__ void k_check_dense(const double* __restrict__ X, int64_t ldx, int d, int n, int* __restrict__ flags) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  int bad = 0;
  for (int j = warp; j < n; j += nwarps) {
    const double* col = X + static_cast<int64_t>(j) * ldx;
    for (int i = lane; i < ldx; i += 32) {
      const double v = col[i];
      if (i < d) bad |= isfinite(v) ? 0 : 1;
      else bad |= v == 0.0 ? 0 : 2;
    }
  }
  bad = __reduce_or_sync(0xffffffffu, bad);
  if (lane == 0 && bad) atomicOr(flags, bad);
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

// the row-major block leading dimension the runtime uses (ldp_of: p rounded to even, 1 for p = 1)
static int64_t ldp_even(int p) { return p == 1 ? 1 : (p + 1) / 2 * 2; }

size_t gram_work_elems(const DenseX& X, int p) {
  size_t need = 0;
  if (p == 1 && p1::applies(X)) need = static_cast<size_t>(p1::ctas(X)) * X.ld;
  if (p <= 64 && xyt::applies(p, ldp_even(p))) {
    const xyt::Plan xp = xyt::plan(X, ldp_even(p));
    if (xp.splits > 1) need = std::max(need, static_cast<size_t>(xp.splits) * X.ld * p);
  }
  if (p > 32 && p <= 64 && use_mma(p)) {  // launch_xtw's one-launch wide form
    const MmaPlan m = mma_plan(X);
    if (m.rs > 1) need = std::max(need, static_cast<size_t>(m.rs) * X.n * p);
  }
  for (int c0 = 0; c0 < p; c0 += 32) {
    const int pc = std::min(32, p - c0);
    const fused::Plan fp = fused::plan(X, pc);
    if (fp.g) {  // (the two-pass needs below still apply: H = Xᵀ C runs launch_xtw alone)
      const int ncl = fused::clusters_for(X, pc, fp);
      if (ncl > 1) need = std::max(need, static_cast<size_t>(ncl) * X.ld * pc);
    }
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

bool gram_p1_applies(const DenseX& X) { return p1::applies(X); }

// Z == nullptr: y = Xᵀ w only (no workspace)
void launch_gram_p1(const DenseX& X, const double* W, int64_t ldw, double* Y, int64_t ldy, double* Z, int64_t ldz,
                    GramWork& work, cudaStream_t st) {
  if (!p1::applies(X)) throw Error(kContractViolation, "gram_p1: layout does not apply");
  const int nblk = p1::ctas(X);
  if (Z && work.part_elems < static_cast<size_t>(nblk) * X.ld) throw Error(kContractViolation, "gram_p1: workspace");
  const int64_t cpc = (ceil_div(X.n, nblk) + 1) / 2 * 2;
  const int grid = static_cast<int>(ceil_div(X.n, cpc));
  auto go = [&](auto kern) { kern<<<grid, p1::kThreads, 0, st>>>(X.x, X.ld, X.n, W, ldw, Y, ldy, work.part, cpc); };
  auto go_wide = [&](auto kern) {
    const int smem = static_cast<int>(X.ld * sizeof(double));
    GAPLRA_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<grid, p1::kThreads, smem, st>>>(X.x, X.ld, X.n, W, ldw, Y, ldy, work.part, cpc);
  };
  if (Z) {
    if (X.ld <= 1024) go(p1::k_gram_p1<1, true>);
    else if (X.ld <= 2048) go(p1::k_gram_p1<2, true>);
    else if (X.ld <= 4096) go(p1::k_gram_p1<4, true>);
    else go_wide(p1::k_gram_p1_wide<true>);
  } else {
    if (X.ld <= 1024) go(p1::k_gram_p1<1, false>);
    else if (X.ld <= 2048) go(p1::k_gram_p1<2, false>);
    else if (X.ld <= 4096) go(p1::k_gram_p1<4, false>);
    else go_wide(p1::k_gram_p1_wide<false>);
  }
  GAPLRA_LAUNCH_CHECK();
  if (!Z) return;
  p1::k_p1_sum<<<static_cast<int>(ceil_div(X.ld, 256)), 256, 0, st>>>(work.part, grid, X.ld, Z, ldz);
  GAPLRA_LAUNCH_CHECK();
}

bool gram_fused_applies(const DenseX& X, int p) {
  for (int c0 = 0; c0 < p; c0 += 32)
    if (!fused::plan(X, std::min(32, p - c0)).g) return false;
  return true;
}

void launch_gram_fused(const DenseX& X, const double* W, int64_t ldw, int p, double* Y, int64_t ldy, double* Z,
                       int64_t ldz, GramWork& work, cudaStream_t st) {
  for (int c0 = 0; c0 < p; c0 += 32) {
    const int pc = std::min(32, p - c0);
    const fused::Plan pl = fused::plan(X, pc);
    if (!pl.g) throw Error(kContractViolation, "gram_fused: layout does not apply");
    const double* w = W + c0;
    double* y = Y + c0;
    double* z = Z + c0;
    switch ((pc + 7) / 8 * 1000 + pl.r) {
      case 1128: fused::launch_chunk<1, 128>(X, w, ldw, pc, y, ldy, z, ldz, work, st, pl); break;
      case 1256: fused::launch_chunk<1, 256>(X, w, ldw, pc, y, ldy, z, ldz, work, st, pl); break;
      case 2128: fused::launch_chunk<2, 128>(X, w, ldw, pc, y, ldy, z, ldz, work, st, pl); break;
      case 2256: fused::launch_chunk<2, 256>(X, w, ldw, pc, y, ldy, z, ldz, work, st, pl); break;
      case 3128: fused::launch_chunk<3, 128>(X, w, ldw, pc, y, ldy, z, ldz, work, st, pl); break;
      case 3256: fused::launch_chunk<3, 256>(X, w, ldw, pc, y, ldy, z, ldz, work, st, pl); break;
      case 4128: fused::launch_chunk<4, 128>(X, w, ldw, pc, y, ldy, z, ldz, work, st, pl); break;
      default: fused::launch_chunk<4, 256>(X, w, ldw, pc, y, ldy, z, ldz, work, st, pl); break;
    }
  }
}

void launch_xtw(const DenseX& X, const double* W, int64_t ldw, int p, double* Y, int64_t ldy, GramWork& work,
                cudaStream_t st) {
  // GAPLRA_XTW_WIDE=1: 32 < p <= 64 in one launch (each X fragment feeds 8 n-tiles,
  // X read once).  Measured slower at C5 p = 64 (81.4 vs 76.5 ms per pass): 160
  // registers leave one CTA per SM, so the two 32-column launches stay the default
  static const int wide = getenv("GAPLRA_XTW_WIDE") ? atoi(getenv("GAPLRA_XTW_WIDE")) : 0;
  if (wide && p > 32 && p <= 64 && use_mma(p)) {
    const MmaPlan m = mma_plan(X);
    switch ((p + 7) / 8) {
      case 5: xtw_mma_chunk<5>(X, W, ldw, p, Y, ldy, work, st, m.rs, m.rows_per_split); break;
      case 6: xtw_mma_chunk<6>(X, W, ldw, p, Y, ldy, work, st, m.rs, m.rows_per_split); break;
      case 7: xtw_mma_chunk<7>(X, W, ldw, p, Y, ldy, work, st, m.rs, m.rows_per_split); break;
      default: xtw_mma_chunk<8>(X, W, ldw, p, Y, ldy, work, st, m.rs, m.rows_per_split); break;
    }
    return;
  }
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
  // all p <= 64 columns in one TMA-fed pass (C5 p = 64: X read once, not in two 32-column chunks)
  if (p <= 64 && xyt::applies(p, ldy)) {
    switch ((p + 7) / 8) {
      case 1: xyt::launch<1>(X, Y, ldy, p, Z, ldz, work, st); break;
      case 2: xyt::launch<2>(X, Y, ldy, p, Z, ldz, work, st); break;
      case 3: xyt::launch<3>(X, Y, ldy, p, Z, ldz, work, st); break;
      case 4: xyt::launch<4>(X, Y, ldy, p, Z, ldz, work, st); break;
      case 5: xyt::launch<5>(X, Y, ldy, p, Z, ldz, work, st); break;
      case 6: xyt::launch<6>(X, Y, ldy, p, Z, ldz, work, st); break;
      case 7: xyt::launch<7>(X, Y, ldy, p, Z, ldz, work, st); break;
      default: xyt::launch<8>(X, Y, ldy, p, Z, ldz, work, st); break;
    }
    return;
  }
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

void check_dense(const DenseX& X, int* flags, cudaStream_t st) {
  GAPLRA_CUDA_CHECK(cudaMemsetAsync(flags, 0, sizeof(int), st));
  k_check_dense<<<sm_count() * 8, 256, 0, st>>>(X.x, X.ld, X.d, X.n, flags);
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
