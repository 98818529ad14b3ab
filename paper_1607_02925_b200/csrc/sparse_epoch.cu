// Block-parallel SVRG epoch for CSC X (the C4 path).
//
// The sequential recurrence (k_svrg_epoch_sparse, SPEC.md:362 in lazy form
// W = α Ŵ + β C) couples step j to an earlier step l only through
// K_jl = x_jᵀ x_l, which is non-zero only when the two sampled columns share
// rows.  For a block of Bs steps starting at s0 with Ŵ₀ = Ŵ at the block start:
//
//   u_l   = r_l / α_{l+1}                      (Ŵ ← Ŵ + u_l x_l after step l)
//   t_j   = α_j (x_jᵀŴ₀ + Σ_{l<j} K_jl u_l) + β_j x_jᵀC
//   u_j   = b_j + κ Σ_{l<j} K_jl u_l,   b_j = ηn(α_j x_jᵀŴ₀ + β_j x_jᵀC − Y_{i_j}) / α_{j+1},
//   κ     = ηn α_j / α_{j+1} = ηn / ρ
//
// which is exact in exact arithmetic (only the rounding order differs from the
// step-by-step form).  Per block, one cooperative kernel does
//   (A) all CTAs: b_j (one warp per step, lane = column) and per-row entry
//       lists (atomic slot per row, touched-row list);
//   (B) CTA 0: sort each shared row's entries by step, emit the coupled pairs,
//       group them by target step in a fixed order, dependency levels by
//       fixed-point iteration, then u level by level (in shared memory);
//   (C) all CTAs: one warp per touched row applies its updates in step order
//       (one write per row: deterministic, no atomics), resets the row slot.
// A block whose row lists or pair list overflow the fixed capacities is done
// serially by CTA 0 (exact step-by-step), so any conflict density is correct.
// Data written in one phase and read by other SMs in a later phase (W, b, u)
// is read with ld.global.cg (L2), on top of grid.sync's GPU-scope fence.
#include <cooperative_groups.h>

#include <algorithm>

#include "common.cuh"
#include "svrg.cuh"

namespace cg = cooperative_groups;

namespace gaplra_cuda {

namespace {

constexpr int kSpThreads = 512;
constexpr int kSpWarps = kSpThreads / 32;
constexpr int kRowCap = 16;      // entries of one row within a block
constexpr int kPairCap = 16384;  // coupled (l, j) contributions within a block
constexpr int kSpMaxBs = 1024;

struct SpArgs {
  SparseEpochArgs e;
  int bs;                  // steps per block (power of two <= kSpMaxBs)
  int max_col_nnz;
  double* b;               // [bs][p] (global)
  int* rowcnt;             // [d], zero between blocks
  int2* rowent;            // [d][kRowCap]  (step j, CSC entry index)
  int* touched;            // [bs * max_col_nnz]
  int4* pairs;             // [kPairCap]: (target j, source l, entry of j, entry of l)
  int* counters;           // [2][4] per block parity: touched rows, pairs, overflow flag
  double* u_glob;          // [bs][p]
  int* csr;                // [bs + 1 + kPairCap]: grouped pair indices (global scratch)
};

__device__ __forceinline__ double ldv(const double* p) { return __ldg(p); }

__global__ void __launch_bounds__(kSpThreads, 1) k_sparse_epoch_blocked(SpArgs A) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double smem[];
  const SparseEpochArgs& a = A.e;
  const int p = a.p, bs = A.bs;
  double* u = smem;                                  // [bs][p]
  double* rp = u + static_cast<size_t>(bs) * p;       // [bs + 1] ρ^j
  double* gm = rp + bs + 1;                           // [bs + 1] γ_j
  int* lev = reinterpret_cast<int*>(gm + bs + 1);     // [bs]
  int* cnt = lev + bs;                                // [bs + 1]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gwarp = blockIdx.x * kSpWarps + warp, nwarps = gridDim.x * kSpWarps;
  if (tid == 0) {
    rp[0] = 1.0;
    gm[0] = 0.0;
    for (int j = 1; j <= bs; ++j) {
      rp[j] = rp[j - 1] * a.rho;
      gm[j] = fma(a.rho, gm[j - 1], 1.0);
    }
  }
  __syncthreads();
  const double kappa = a.eta_n / a.rho;
  double al = 1.0, be = 0.0;  // α, β at the block start (identical in every thread)
  const int64_t nblk = (a.m + bs - 1) / bs;
  for (int64_t blk = 0; blk < nblk; ++blk) {
    const int64_t s0 = blk * bs;
    const int bt = static_cast<int>(a.m - s0 < bs ? a.m - s0 : bs);
    int* ctr = A.counters + (blk & 1) * 4;  // this block's counters (the other parity is reset in (B))
    if (al < 1e-150) {  // fold α into Ŵ (rare)
      for (int64_t e = static_cast<int64_t>(blockIdx.x) * kSpThreads + tid; e < static_cast<int64_t>(a.d) * p;
           e += static_cast<int64_t>(gridDim.x) * kSpThreads) {
        const int64_t row = e / p, c = e - row * p;
        a.W[row * a.ldw + c] *= al;
      }
      al = 1.0;
      grid.sync();
    }
    // ---------------------------------------------------------------- (A)
    for (int j = gwarp; j < bt; j += nwarps) {
      const int i = a.idx[s0 + j];
      const int64_t e0 = a.colptr[i], e1 = a.colptr[i + 1];
      if (lane < p) {
        double dw = 0.0, dc = 0.0;
        for (int64_t e = e0; e < e1; ++e) {
          const int64_t row = a.rowidx[e];
          const double v = ldv(a.val + e);
          dw = fma(v, __ldcg(a.W + row * a.ldw + lane), dw);
          dc = fma(v, a.C[row * a.ldw + lane], dc);
        }
        const double aj = al * rp[j], bj = fma(rp[j], be, gm[j]);
        const double t = fma(aj, dw, bj * dc);
        A.b[static_cast<size_t>(j) * p + lane] =
            a.eta_n * (t - a.Y[static_cast<int64_t>(i) * a.ldy + lane]) / (al * rp[j + 1]);
      }
      for (int64_t e = e0 + lane; e < e1; e += 32) {
        const int row = a.rowidx[e];
        const int slot = atomicAdd(&A.rowcnt[row], 1);
        if (slot == 0) A.touched[atomicAdd(&ctr[0], 1)] = row;
        if (slot < kRowCap)
          A.rowent[static_cast<int64_t>(row) * kRowCap + slot] = make_int2(j, static_cast<int>(e));
        else
          ctr[2] = 1;
      }
    }
    grid.sync();
    // ---------------------------------------------------------------- (B)
    if (blockIdx.x == 0) {
      if (tid < 4) A.counters[((blk + 1) & 1) * 4 + tid] = 0;  // next block's counters
      const int nt = ctr[0];
      // sort shared rows by step and emit the coupled pairs
      for (int k = tid; k < nt; k += kSpThreads) {
        const int row = A.touched[k];
        const int c = min(A.rowcnt[row], kRowCap);
        if (c < 2) continue;
        int2* ent = A.rowent + static_cast<int64_t>(row) * kRowCap;
        for (int x = 1; x < c; ++x) {  // insertion sort by step
          const int2 v = ent[x];
          int y = x - 1;
          while (y >= 0 && ent[y].x > v.x) {
            ent[y + 1] = ent[y];
            --y;
          }
          ent[y + 1] = v;
        }
        for (int x = 1; x < c; ++x)
          for (int y = 0; y < x; ++y) {
            const int slot = atomicAdd(&ctr[1], 1);
            if (slot < kPairCap)
              A.pairs[slot] = make_int4(ent[x].x, ent[y].x, ent[x].y, ent[y].y);
            else
              ctr[2] = 1;
          }
      }
      __syncthreads();
      const bool overflow = ctr[2] != 0;
      if (!overflow) {
        const int np = ctr[1];
        // group pair indices by target step: counts, exclusive scan, fill, then
        // sort every group by (source step, entry) — a fixed summation order
        for (int j = tid; j <= bt; j += kSpThreads) cnt[j] = 0;
        __syncthreads();
        for (int k = tid; k < np; k += kSpThreads) atomicAdd(&cnt[A.pairs[k].x + 1], 1);
        __syncthreads();
        if (tid == 0)
          for (int j = 1; j <= bt; ++j) cnt[j] += cnt[j - 1];
        __syncthreads();
        int* grp = A.csr;  // [np] pair indices grouped by target
        for (int j = tid; j < bt; j += kSpThreads) lev[j] = cnt[j];  // fill cursor
        __syncthreads();
        for (int k = tid; k < np; k += kSpThreads) grp[atomicAdd(&lev[A.pairs[k].x], 1)] = k;
        __syncthreads();
        for (int j = tid; j < bt; j += kSpThreads) {
          const int g0 = cnt[j], g1 = cnt[j + 1];
          for (int x = g0 + 1; x < g1; ++x) {
            const int v = grp[x];
            const int4 pv = A.pairs[v];
            int y = x - 1;
            while (y >= g0) {
              const int4 py = A.pairs[grp[y]];
              if (py.y < pv.y || (py.y == pv.y && py.w <= pv.w)) break;
              grp[y + 1] = grp[y];
              --y;
            }
            grp[y + 1] = v;
          }
          lev[j] = 0;
        }
        __syncthreads();
        // dependency levels: lev_j = max(0, max_l lev_l + 1), fixed point from below
        for (;;) {
          int changed = 0;
          for (int j = tid; j < bt; j += kSpThreads) {
            int L = 0;
            for (int x = cnt[j]; x < cnt[j + 1]; ++x) L = max(L, lev[A.pairs[grp[x]].y] + 1);
            if (L != lev[j]) {
              lev[j] = L;
              changed = 1;
            }
          }
          if (!__syncthreads_or(changed)) break;
        }
        int maxlev = 0;
        for (int j = tid; j < bt; j += kSpThreads) maxlev = max(maxlev, lev[j]);
        maxlev = __reduce_max_sync(0xffffffffu, maxlev);
        __shared__ int wmax[kSpWarps];
        if (lane == 0) wmax[warp] = maxlev;
        __syncthreads();
        maxlev = 0;
        for (int w = 0; w < kSpWarps; ++w) maxlev = max(maxlev, wmax[w]);
        // solve level by level
        for (int L = 0; L <= maxlev; ++L) {
          for (int e = tid; e < bt * p; e += kSpThreads) {
            const int j = e / p, c = e - j * p;
            if (lev[j] != L) continue;
            double acc = 0.0;
            for (int x = cnt[j]; x < cnt[j + 1]; ++x) {
              const int4 pv = A.pairs[grp[x]];
              acc = fma(ldv(a.val + pv.z) * ldv(a.val + pv.w), u[pv.y * p + c], acc);
            }
            u[e] = fma(kappa, acc, __ldcg(A.b + e));
          }
          __syncthreads();
        }
      } else {
        // exact serial fallback: step by step with immediate updates (rows of
        // this block are untouched by (C) below: counters[2] tells it to skip)
        for (int j = 0; j < bt; ++j) {
          const int i = a.idx[s0 + j];
          const int64_t e0 = a.colptr[i], e1 = a.colptr[i + 1];
          if (warp == 0 && lane < p) {
            double dw = 0.0, dc = 0.0;
            for (int64_t e = e0; e < e1; ++e) {
              const int64_t row = a.rowidx[e];
              const double v = ldv(a.val + e);
              dw = fma(v, __ldcg(a.W + row * a.ldw + lane), dw);
              dc = fma(v, a.C[row * a.ldw + lane], dc);
            }
            const double aj = al * rp[j], bj = fma(rp[j], be, gm[j]);
            const double r = a.eta_n * (fma(aj, dw, bj * dc) - a.Y[static_cast<int64_t>(i) * a.ldy + lane]);
            const double sc = r / (al * rp[j + 1]);
            for (int64_t e = e0; e < e1; ++e) {
              const int64_t row = a.rowidx[e];
              a.W[row * a.ldw + lane] = fma(sc, ldv(a.val + e), a.W[row * a.ldw + lane]);
            }
          }
          __syncwarp();
        }
      }
      for (int e = tid; e < bt * p; e += kSpThreads) A.u_glob[e] = u[e];
    }
    grid.sync();
    // ---------------------------------------------------------------- (C)
    const bool overflow = ctr[2] != 0;
    const int nt = ctr[0];
    for (int k = gwarp; k < nt; k += nwarps) {
      const int row = A.touched[k];
      const int c = min(A.rowcnt[row], kRowCap);
      if (!overflow && lane < p) {
        const int2* ent = A.rowent + static_cast<int64_t>(row) * kRowCap;
        double w = __ldcg(a.W + static_cast<int64_t>(row) * a.ldw + lane);
        for (int x = 0; x < c; ++x) w = fma(ldv(a.val + ent[x].y), __ldcg(A.u_glob + ent[x].x * p + lane), w);
        a.W[static_cast<int64_t>(row) * a.ldw + lane] = w;
      }
      __syncwarp();
      if (lane == 0) A.rowcnt[row] = 0;
    }
    al *= rp[bt];
    be = fma(rp[bt], be, gm[bt]);
    grid.sync();
  }
  if (blockIdx.x == 0 && tid < 8) A.counters[tid] = 0;  // the last block's counters (all reads were before its sync)
  // W = α Ŵ + β C
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * kSpThreads + tid; e < static_cast<int64_t>(a.d) * p;
       e += static_cast<int64_t>(gridDim.x) * kSpThreads) {
    const int64_t row = e / p, c = e - row * p;
    double* w = a.W + row * a.ldw + c;
    *w = fma(al, *w, be * a.C[row * a.ldw + c]);
  }
}

}  // namespace

int sparse_block_steps(int d, double col_nnz, int p) {
  // expected coupled pairs in a block of bs steps: (bs·nnz)² / (2d); keep it
  // near 4096, the shared u tile bs·p doubles within 128 KB
  int bs = kSpMaxBs;
  while (bs > 32 && ((bs * col_nnz) * (bs * col_nnz) / (2.0 * d) > 4096.0 || bs * p > 16384)) bs /= 2;
  return bs;
}

size_t sparse_scratch_ints(int d, int bs, int max_col_nnz) {
  return static_cast<size_t>(d)                    // rowcnt
         + 2 * static_cast<size_t>(d) * kRowCap      // rowent (int2)
         + static_cast<size_t>(bs) * max_col_nnz     // touched
         + 4 * static_cast<size_t>(kPairCap)         // pairs (int4)
         + 8                                         // counters
         + static_cast<size_t>(kPairCap) + bs + 1;   // grouped pair indices
}

bool sparse_blocked_supported(int p) { return p >= 1 && p <= 32; }

void launch_svrg_epoch_sparse_blocked(const SparseEpochArgs& a, int bs, int max_col_nnz, double* dbuf, int* ibuf,
                                      cudaStream_t st) {
  SpArgs A;
  A.e = a;
  A.bs = bs;
  A.max_col_nnz = max_col_nnz;
  A.b = dbuf;
  A.u_glob = dbuf + static_cast<size_t>(A.bs) * a.p;
  int* q = ibuf;
  A.rowcnt = q;
  q += a.d;
  A.rowent = reinterpret_cast<int2*>(q);
  q += 2 * static_cast<size_t>(a.d) * kRowCap;
  A.touched = q;
  q += static_cast<size_t>(A.bs) * max_col_nnz;
  A.pairs = reinterpret_cast<int4*>(q);
  q += 4 * static_cast<size_t>(kPairCap);
  A.counters = q;
  q += 8;
  A.csr = q;
  const size_t smem = (static_cast<size_t>(A.bs) * a.p + 2 * (A.bs + 1)) * sizeof(double) +
                      (2 * static_cast<size_t>(A.bs) + 1) * sizeof(int);
  GAPLRA_CUDA_CHECK(cudaFuncSetAttribute(k_sparse_epoch_blocked, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem)));
  int per_sm = 0;
  GAPLRA_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sparse_epoch_blocked, kSpThreads, smem));
  if (per_sm < 1) throw Error(kDeviceError, "sparse epoch: kernel does not fit an SM");
  int sms = 0, dev = 0;
  GAPLRA_CUDA_CHECK(cudaGetDevice(&dev));
  GAPLRA_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  void* args[] = {&A};
  GAPLRA_CUDA_CHECK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_sparse_epoch_blocked), dim3(sms),
                                                dim3(kSpThreads), args, smem, st));
  GAPLRA_LAUNCH_CHECK();
}

}  // namespace gaplra_cuda
