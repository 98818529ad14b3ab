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
//   (A2) all CTAs: sort each shared row's entries by step, emit the coupled
//       pairs (key: target, source, entry; value: the K contribution);
//   (B) CTA 0: group the pairs by target step in a fixed order (counting sort
//       + per-group insertion sort) and solve u = b + κKu by in-place sweeps
//       until nothing changes (K is nilpotent), all in shared memory;
//   (C) all CTAs: one warp per touched row applies its updates in step order
//       (one write per row: deterministic, no atomics), resets the row slot.
// A block whose row lists or pair list overflow the fixed capacities is done
// serially by CTA 0 (exact step-by-step), so any conflict density is correct.
// Data written in one phase and read by other SMs in a later phase (W, b, u)
// is read with ld.global.cg (L2), on top of grid.sync's GPU-scope fence.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "svrg.cuh"

namespace cg = cooperative_groups;

namespace gaplra_cuda {

namespace {

constexpr int kSpThreads = 512;
constexpr int kSpWarps = kSpThreads / 32;
constexpr int kRowCap = 16;      // entries of one row within a block
constexpr int kPairCap = 16384;  // coupled (l, j) contributions within a block (global list)
constexpr int kSpMaxBs = 1024;
constexpr int kSpMaxEntries = 8192;  // bs·p: the u tile and the per-thread b registers

struct SpArgs {
  SparseEpochArgs e;
  int bs;                  // steps per block (power of two <= kSpMaxBs)
  int max_col_nnz;
  double* b;               // [bs][p] (global)
  int* rowcnt;             // [d], zero between blocks
  int2* rowent;            // [d][kRowCap]  (step j, CSC entry index)
  int* touched;            // [bs * max_col_nnz]
  unsigned long long* pkey;  // [kPairCap]: target j << 42 | source l << 32 | entry of l
  double* pval;              // [kPairCap]: val(entry of j) * val(entry of l)
  int* counters;           // [2][4] per block parity: touched rows, pairs, overflow flag
  double* u_glob;          // [bs][p]
  int spair_cap;           // pairs that fit the shared tile of CTA 0
  unsigned long long* dbg;  // GAPLRA_EPOCH_TIMING: ns per phase (A, A2, B, C) summed over blocks
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
  return t;
}

__device__ __forceinline__ double ldv(const double* p) { return __ldg(p); }

__global__ void __launch_bounds__(kSpThreads, 1) k_sparse_epoch_blocked(SpArgs A) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double smem[];
  const SparseEpochArgs& a = A.e;
  const int p = a.p, bs = A.bs;
  double* u = smem;                                  // [bs][p]
  double* rp = u + static_cast<size_t>(bs) * p;       // [bs + 1] ρ^j
  double* gm = rp + bs + 1;                           // [bs + 1] γ_j
  double* sv = gm + bs + 1;                           // [spair_cap] pair values
  unsigned long long* sk = reinterpret_cast<unsigned long long*>(sv + A.spair_cap);  // [spair_cap] keys
  int* lev = reinterpret_cast<int*>(sk + A.spair_cap);  // [bs] scan temporaries / fill cursors
  int* cnt = lev + bs;                                  // [bs + 1] group bounds
  int* perm = cnt + bs + 1;                             // [spair_cap] pair indices grouped by target
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
  unsigned long long tph[4] = {0, 0, 0, 0}, tlast = gtimer();
  auto mark = [&](int k) {
    if (A.dbg && blockIdx.x == 0 && tid == 0) {
      const unsigned long long now = gtimer();
      tph[k] += now - tlast;
      tlast = now;
    }
  };
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
    mark(0);
    // --------------------------------------------------------------- (A2)
    // every CTA: sort the entries of shared rows by step and emit the coupled
    // pairs with their contribution val_j(row) · val_l(row)
    {
      const int nt = ctr[0];
      for (int k = blockIdx.x * kSpThreads + tid; k < nt; k += gridDim.x * kSpThreads) {
        const int row = A.touched[k];
        const int c = min(A.rowcnt[row], kRowCap);
        if (c < 2) continue;
        int2 ent[kRowCap];
        const int2* src = A.rowent + static_cast<int64_t>(row) * kRowCap;
        for (int x = 0; x < c; ++x) ent[x] = src[x];
        for (int x = 1; x < c; ++x) {  // insertion sort by step
          const int2 v = ent[x];
          int y = x - 1;
          while (y >= 0 && ent[y].x > v.x) {
            ent[y + 1] = ent[y];
            --y;
          }
          ent[y + 1] = v;
        }
        int2* dst = A.rowent + static_cast<int64_t>(row) * kRowCap;
        for (int x = 0; x < c; ++x) dst[x] = ent[x];  // (C) applies the row's updates in step order
        for (int x = 1; x < c; ++x) {
          const double vj = ldv(a.val + ent[x].y);
          for (int y = 0; y < x; ++y) {
            const int slot = atomicAdd(&ctr[1], 1);
            if (slot < kPairCap) {
              A.pkey[slot] = (static_cast<unsigned long long>(ent[x].x) << 42) |
                             (static_cast<unsigned long long>(ent[y].x) << 32) | static_cast<unsigned>(ent[y].y);
              A.pval[slot] = vj * ldv(a.val + ent[y].y);
            } else {
              ctr[2] = 1;
            }
          }
        }
      }
    }
    grid.sync();
    mark(1);
    // ---------------------------------------------------------------- (B)
    if (blockIdx.x == 0) {
      if (tid < 4) A.counters[((blk + 1) & 1) * 4 + tid] = 0;  // next block's counters
      const int np = __ldcg(&ctr[1]);
      const bool overflow = __ldcg(&ctr[2]) != 0 || np > A.spair_cap;
      if (!overflow) {
        // pairs into shared memory, grouped by target step (counting sort),
        // every group sorted by (source step, entry): a fixed summation order
        for (int k = tid; k < np; k += kSpThreads) {
          sk[k] = __ldcg(A.pkey + k);
          sv[k] = __ldcg(A.pval + k);
        }
        for (int j = tid; j <= bt; j += kSpThreads) cnt[j] = 0;
        __syncthreads();
        for (int k = tid; k < np; k += kSpThreads) atomicAdd(&cnt[static_cast<int>(sk[k] >> 42) + 1], 1);
        __syncthreads();
        // inclusive scan of cnt[1..bt] (bt <= 1024): warp scans + warp totals
        __shared__ int wsum[kSpWarps];
        {
          const int per = (bt + kSpThreads - 1) / kSpThreads;  // 1 or 2 entries per thread
          const int j0 = 1 + tid * per;
          int loc = 0;
          for (int q = 0; q < per; ++q)
            if (j0 + q <= bt) loc += cnt[j0 + q];
          int inc = loc;
          for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += v;
          }
          if (lane == 31) wsum[warp] = inc;
          __syncthreads();
          int off = 0;
          for (int w = 0; w < warp; ++w) off += wsum[w];
          int run = off + inc - loc;
          for (int q = 0; q < per; ++q)
            if (j0 + q <= bt) {
              run += cnt[j0 + q];
              lev[j0 + q - 1] = run;  // end of group j0+q-1 (temporary)
            }
        }
        __syncthreads();
        for (int j = tid; j < bt; j += kSpThreads) cnt[j + 1] = lev[j];
        if (tid == 0) cnt[0] = 0;
        __syncthreads();
        for (int j = tid; j < bt; j += kSpThreads) lev[j] = cnt[j];  // fill cursors
        __syncthreads();
        for (int k = tid; k < np; k += kSpThreads) perm[atomicAdd(&lev[static_cast<int>(sk[k] >> 42)], 1)] = k;
        __syncthreads();
        for (int j = tid; j < bt; j += kSpThreads) {
          const int g0 = cnt[j], g1 = cnt[j + 1];
          for (int x = g0 + 1; x < g1; ++x) {
            const int v = perm[x];
            const unsigned long long kv = sk[v];
            int y = x - 1;
            while (y >= g0 && sk[perm[y]] > kv) {
              perm[y + 1] = perm[y];
              --y;
            }
            perm[y + 1] = v;
          }
        }
        __syncthreads();
        // u = b + κ K u by in-place fixed-point sweeps: the coupling is strictly
        // lower triangular (nilpotent), so the sweeps stop changing after
        // depth + 1 and the last sweep recomputes every u_j from its final
        // predecessors in the fixed group order
        constexpr int kOwn = kSpMaxEntries / kSpThreads;  // (j, c) entries per thread
        double bown[kOwn];
        const int ne = bt * p;
#pragma unroll
        for (int q = 0; q < kOwn; ++q) {
          const int e = tid + q * kSpThreads;
          bown[q] = e < ne ? __ldcg(A.b + e) : 0.0;
          if (e < ne) u[e] = bown[q];
        }
        __syncthreads();
        if (np > 0) {
          for (;;) {
            int changed = 0;
#pragma unroll
            for (int q = 0; q < kOwn; ++q) {
              const int e = tid + q * kSpThreads;
              if (e >= ne) break;
              const int j = e / p, c = e - j * p;
              const int g0 = cnt[j], g1 = cnt[j + 1];
              if (g0 == g1) continue;
              double acc = 0.0;
              for (int x = g0; x < g1; ++x) {
                const int k = perm[x];
                acc = fma(sv[k], u[static_cast<int>((sk[k] >> 32) & 0x3ff) * p + c], acc);
              }
              const double nu = fma(kappa, acc, bown[q]);
              if (nu != u[e]) {
                u[e] = nu;
                changed = 1;
              }
            }
            if (!__syncthreads_or(changed)) break;
          }
        }
        for (int e = tid; e < ne; e += kSpThreads) A.u_glob[e] = u[e];
      } else {
        if (tid == 0) ctr[2] = 1;  // (C) skips the block's row updates
        // exact serial fallback: step by step with immediate updates
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
    }
    grid.sync();
    mark(2);
    // ---------------------------------------------------------------- (C)
    const bool overflow = __ldcg(&ctr[2]) != 0;
    const int nt = __ldcg(&ctr[0]);
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
    mark(3);
  }
  if (A.dbg && blockIdx.x == 0 && tid == 0)
    for (int k = 0; k < 4; ++k) A.dbg[k] = tph[k];
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
  // near 4096, the shared u tile bs·p <= kSpMaxEntries doubles
  int bs = kSpMaxBs;
  while (bs > 32 && ((bs * col_nnz) * (bs * col_nnz) / (2.0 * d) > 4096.0 || bs * p > kSpMaxEntries)) bs /= 2;
  return bs;
}

size_t sparse_scratch_ints(int d, int bs, int max_col_nnz) {
  return static_cast<size_t>(d)                    // rowcnt
         + 2 * static_cast<size_t>(d) * kRowCap      // rowent (int2)
         + static_cast<size_t>(bs) * max_col_nnz     // touched
         + 4 * static_cast<size_t>(kPairCap)         // pair keys (u64) + values (f64)
         + 8;                                        // counters
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
  A.pkey = reinterpret_cast<unsigned long long*>(q);
  q += 2 * static_cast<size_t>(kPairCap);
  A.pval = reinterpret_cast<double*>(q);
  q += 2 * static_cast<size_t>(kPairCap);
  A.counters = q;
  q += 8;
  const size_t base = (static_cast<size_t>(A.bs) * a.p + 2 * (A.bs + 1)) * sizeof(double) +
                      (2 * static_cast<size_t>(A.bs) + 1) * sizeof(int);
  // shared pair tile: a power of two up to 8192 pairs within ~200 KB in total
  int cap = 8192;
  while (cap > 256 && base + static_cast<size_t>(cap) * 20 > 200 * 1024) cap >>= 1;
  A.spair_cap = cap;
  static const bool timing = getenv("GAPLRA_EPOCH_TIMING") != nullptr;
  static unsigned long long* dbg = nullptr;
  A.dbg = nullptr;
  if (timing) {
    if (!dbg) GAPLRA_CUDA_CHECK(cudaMalloc(&dbg, 4 * sizeof(unsigned long long)));
    A.dbg = dbg;
  }
  const size_t smem = base + static_cast<size_t>(cap) * 20;
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
  if (A.dbg) {
    unsigned long long h[4];
    GAPLRA_CUDA_CHECK(cudaMemcpyAsync(h, A.dbg, sizeof(h), cudaMemcpyDeviceToHost, st));
    GAPLRA_CUDA_CHECK(cudaStreamSynchronize(st));
    const double nbk = static_cast<double>((a.m + bs - 1) / bs);
    fprintf(stderr, "{\"sparse_epoch\": {\"bs\": %d, \"blocks\": %.0f, \"us_per_block\": [%.2f, %.2f, %.2f, %.2f]}}\n", bs,
            nbk, h[0] / nbk / 1e3, h[1] / nbk / 1e3, h[2] / nbk / 1e3, h[3] / nbk / 1e3);
  }
}

}  // namespace gaplra_cuda
