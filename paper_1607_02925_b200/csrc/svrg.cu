// SVRG epoch kernels for the block solve of (λI − XXᵀ)W = B.
//
// Spec (restated in oracle/oracle.cpp svrg_epoch): for each of
// m = 2n sampled indices i (shared by all p columns),
//     r = ηn (x_iᵀ W − Y_i),   W ← ρ W + C + x_i rᵀ,   ρ = 1 − ηλ,  C = η(X Xᵀ W̃ + B)
// with Y = Xᵀ W̃ from the anchor.  The device evaluates it in exact-arithmetic-
// equivalent s-step blocks of b steps:
//     P_j = x_{i_j}ᵀ W_0,  K_jl = x_{i_j}ᵀ x_{i_l},  H_i = x_iᵀ C (precomputed pass)
//     r_j = ηn (ρ^j P_j + γ_j H_{i_j} + Σ_{l<j} ρ^{j−1−l} K_jl r_l − Y_{i_j})
//     W_b = ρ^b W_0 + γ_b C + Σ_l ρ^{b−1−l} x_{i_l} r_lᵀ,      γ_j = Σ_{t<j} ρ^t
// Dense kernel: one thread-block cluster per group of ≤ PC columns; the G CTAs
// of a cluster split the d rows, keep their W and C row slices resident in
// shared memory for the whole epoch, stage the b sampled column slices, and
// all-reduce the b·PC + b(b−1)/2 partial dots through distributed shared
// memory (fixed rank order ⇒ deterministic, identical in every CTA).
#include <cooperative_groups.h>

#include <algorithm>

#include "common.cuh"
#include "svrg.cuh"

namespace cg = cooperative_groups;

namespace gaplra_cuda {

namespace {

constexpr int kEpochThreads = 256;

struct Smem {
  int rows, rows_pad, pc_pad, entries;
  size_t off_x, off_w, off_c, off_part, off_full, off_coef, off_pow, off_gam, off_idx, total;
};

template <int PC, int B>
__host__ __device__ inline Smem smem_layout(int rows) {
  Smem s;
  s.rows = rows;
  s.rows_pad = rows + 4;  // odd-ish pitch keeps column slices on distinct banks
  s.pc_pad = PC;
  s.entries = B * PC + B * (B - 1) / 2;
  size_t o = 0;
  s.off_x = o;
  o += static_cast<size_t>(B) * s.rows_pad;
  s.off_w = o;
  o += static_cast<size_t>(rows) * PC;
  s.off_c = o;
  o += static_cast<size_t>(rows) * PC;
  s.off_part = o;
  o += 2 * static_cast<size_t>(s.entries);
  s.off_full = o;
  o += s.entries;
  s.off_coef = o;
  o += static_cast<size_t>(B) * PC;
  s.off_pow = o;
  o += B + 1;
  s.off_gam = o;
  o += B + 1;
  s.off_idx = o;
  o += B;  // ints stored in double slots
  s.total = o * sizeof(double);
  return s;
}

template <int PC, int B>
__global__ void __launch_bounds__(kEpochThreads, 1) k_svrg_epoch_dense(EpochArgs a) {
  extern __shared__ __align__(16) double sm[];
  cg::cluster_group cluster = cg::this_cluster();
  const int G = static_cast<int>(cluster.num_blocks());
  const int g = static_cast<int>(cluster.block_rank());
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c0 = blockIdx.y * PC;
  const int pc = min(PC, a.p - c0);
  const Smem L = smem_layout<PC, B>(a.rows_per_cta);
  const int r0 = g * a.rows_per_cta;
  const int rc = max(0, min(a.rows_per_cta, a.d_pad - r0));

  double* Xs = sm + L.off_x;
  double* Ws = sm + L.off_w;
  double* Cs = sm + L.off_c;
  double* part = sm + L.off_part;
  double* full = sm + L.off_full;
  double* coef = sm + L.off_coef;
  double* rpow = sm + L.off_pow;
  double* gam = sm + L.off_gam;
  int* idxs = reinterpret_cast<int*>(sm + L.off_idx);

  // Resident W / C row slices (row-major r x PC, zero beyond pc).
  for (int e = tid; e < rc * PC; e += kEpochThreads) {
    const int r = e / PC, c = e - (e / PC) * PC;
    const int64_t gr = static_cast<int64_t>(r0 + r) * a.ldw + c0 + c;
    Ws[e] = c < pc ? a.W[gr] : 0.0;
    Cs[e] = c < pc ? a.C[gr] : 0.0;
  }
  if (tid == 0) {
    rpow[0] = 1.0;
    gam[0] = 0.0;
    for (int j = 1; j <= B; ++j) {
      rpow[j] = rpow[j - 1] * a.rho;
      gam[j] = gam[j - 1] + rpow[j - 1];
    }
  }
  __syncthreads();

  int par = 0;
  for (int64_t s0 = 0; s0 < a.m; s0 += B, par ^= 1) {
    const int bt = a.m - s0 < B ? static_cast<int>(a.m - s0) : B;
    if (tid < bt) idxs[tid] = a.idx[s0 + tid];
    __syncthreads();
    // Stage the sampled column slices x_{i_j}[r0 : r0 + rc).
    for (int e = tid; e < bt * rc; e += kEpochThreads) {
      const int j = e / rc, r = e - (e / rc) * rc;
      Xs[j * L.rows_pad + r] = __ldg(a.X + static_cast<int64_t>(idxs[j]) * a.ldx + r0 + r);
    }
    __syncthreads();
    // Local partial dots: P[j][c] (bt*PC entries) then K[j][l], l < j.
    const int np = bt * PC;
    const int ne = np + bt * (bt - 1) / 2;
    double* mypart = part + par * L.entries;
    for (int ent = warp; ent < ne; ent += kEpochThreads / 32) {
      double s = 0.0;
      if (ent < np) {
        const int j = ent / PC, c = ent - (ent / PC) * PC;
        const double* xj = Xs + j * L.rows_pad;
        for (int r = lane; r < rc; r += 32) s = fma(xj[r], Ws[r * PC + c], s);
      } else {
        int k = ent - np, j = 1;
        while (k >= j) {
          k -= j;
          ++j;
        }
        const double* xj = Xs + j * L.rows_pad;
        const double* xl = Xs + k * L.rows_pad;
        for (int r = lane; r < rc; r += 32) s = fma(xj[r], xl[r], s);
      }
      s = warp_sum(s);
      if (lane == 0) mypart[ent] = s;
    }
    cluster.sync();
    for (int ent = tid; ent < ne; ent += kEpochThreads) {
      double s = 0.0;
      for (int q = 0; q < G; ++q) s += cluster.map_shared_rank(mypart, q)[ent];
      full[ent] = s;
    }
    __syncthreads();
    // Recurrence for the bt coefficients of each column (thread = column).
    if (tid < pc) {
      const int c = tid;
      const double* K = full + np;
      for (int j = 0; j < bt; ++j) {
        const int64_t i = idxs[j];
        double v = fma(rpow[j], full[j * PC + c], gam[j] * a.H[i * a.ldy + c0 + c]) - a.Y[i * a.ldy + c0 + c];
        const double* Kj = K + j * (j - 1) / 2;
        for (int l = 0; l < j; ++l) v = fma(rpow[j - 1 - l] * Kj[l], coef[l * PC + c], v);
        coef[j * PC + c] = a.eta_n * v;
      }
      for (int l = 0; l < bt; ++l) coef[l * PC + c] *= rpow[bt - 1 - l];
    }
    __syncthreads();
    // W_b = ρ^b W_0 + γ_b C + Σ_l x_{i_l} coef_l   on the owned rows.
    const double rb = rpow[bt], gb = gam[bt];
    for (int e = tid; e < rc * PC; e += kEpochThreads) {
      const int r = e / PC, c = e - (e / PC) * PC;
      if (c >= pc) continue;
      double w = fma(rb, Ws[e], gb * Cs[e]);
      for (int l = 0; l < bt; ++l) w = fma(Xs[l * L.rows_pad + r], coef[l * PC + c], w);
      Ws[e] = w;
    }
    __syncthreads();
  }
  for (int e = tid; e < rc * PC; e += kEpochThreads) {
    const int r = e / PC, c = e - (e / PC) * PC;
    if (c < pc) a.W[static_cast<int64_t>(r0 + r) * a.ldw + c0 + c] = Ws[e];
  }
  cluster.sync();  // keep shared memory alive until every peer finished its DSMEM reads
}

// Sparse (CSC) epoch, lazy form W = α Ŵ + β C (O(nnz(x_i)) per step).  One
// warp per group of 32 columns; lane = column; steps strictly sequential.
__global__ void k_svrg_epoch_sparse(SparseEpochArgs a) {
  const int c = blockIdx.x * 32 + threadIdx.x;
  if (c >= a.p) return;
  double al = 1.0, be = 0.0;
  for (int64_t s = 0; s < a.m; ++s) {
    const int i = a.idx[s];
    const int64_t e0 = a.colptr[i], e1 = a.colptr[i + 1];
    double dw = 0.0, dc = 0.0;
    for (int64_t e = e0; e < e1; ++e) {
      const int64_t row = a.rowidx[e];
      dw = fma(a.val[e], a.W[row * a.ldw + c], dw);
      dc = fma(a.val[e], a.C[row * a.ldw + c], dc);
    }
    const double t = fma(al, dw, be * dc);
    const double r = a.eta_n * (t - a.Y[static_cast<int64_t>(i) * a.ldy + c]);
    al = a.rho * al;
    be = fma(a.rho, be, 1.0);
    if (al < 1e-150) {
      for (int row = 0; row < a.d; ++row) a.W[static_cast<int64_t>(row) * a.ldw + c] *= al;
      al = 1.0;
    }
    const double sc = r / al;
    for (int64_t e = e0; e < e1; ++e) {
      const int64_t row = a.rowidx[e];
      a.W[row * a.ldw + c] = fma(sc, a.val[e], a.W[row * a.ldw + c]);
    }
  }
  for (int row = 0; row < a.d; ++row) {
    double* w = a.W + static_cast<int64_t>(row) * a.ldw + c;
    *w = fma(al, *w, be * a.C[static_cast<int64_t>(row) * a.ldw + c]);
  }
}

// ---------------------------------------------------------------------------
// Anchor epilogue: M = λW̃ − Z − B (per-column |M_c|^2 partials), C = η(Z + B).
// W or Z may be null (= 0).  Grid-stride over rows, fixed-order reductions.
// ---------------------------------------------------------------------------
constexpr int kAnchorThreads = 256;
constexpr int kAnchorMaxP = 64;

__global__ void __launch_bounds__(kAnchorThreads) k_anchor(const double* __restrict__ W, const double* __restrict__ Z,
                                                           const double* __restrict__ Bm, int64_t ld, int d, int p,
                                                           double lambda, double eta, double* __restrict__ C,
                                                           double* __restrict__ part) {
  __shared__ double red[32];
  const int rows_per = static_cast<int>(ceil_div(d, gridDim.x));
  const int r0 = blockIdx.x * rows_per;
  const int r1 = min(r0 + rows_per, d);
  for (int c = 0; c < p; ++c) {
    double s = 0.0;
    for (int r = r0 + threadIdx.x; r < r1; r += kAnchorThreads) {
      const int64_t o = static_cast<int64_t>(r) * ld + c;
      const double w = W ? W[o] : 0.0;
      const double z = Z ? Z[o] : 0.0;
      const double b = Bm[o];
      const double mm = (lambda * w - z) - b;
      s = fma(mm, mm, s);
      if (C) C[o] = eta * (z + b);
    }
    s = block_sum(s, red);
    if (threadIdx.x == 0) part[blockIdx.x * kAnchorMaxP + c] = s;
  }
}

__global__ void k_anchor_final(const double* __restrict__ part, int nparts, int p, const double* __restrict__ bnorm,
                               double* __restrict__ out_colnorm, double* __restrict__ out_max) {
  __shared__ double vals[kAnchorMaxP];
  const int c = threadIdx.x;
  if (c < p) {
    double s = 0.0;
    for (int k = 0; k < nparts; ++k) s += part[k * kAnchorMaxP + c];
    const double nrm = sqrt(s);
    if (out_colnorm) out_colnorm[c] = nrm;
    const double b = bnorm ? bnorm[c] : 1.0;
    vals[c] = nrm / (b > 0.0 ? b : 1.0);
  }
  __syncthreads();
  if (c == 0) {
    double m = 0.0;
    bool bad = false;
    for (int k = 0; k < p; ++k) {
      if (!(vals[k] == vals[k]) || isinf(vals[k])) bad = true;
      m = fmax(m, vals[k]);
    }
    *out_max = bad ? __longlong_as_double(0x7ff8000000000000ll) : m;
  }
}

}  // namespace

EpochConfig choose_epoch_config(int d_pad, int p) {
  EpochConfig cfg;
  cfg.cluster = d_pad <= 4096 ? 8 : 16;
  cfg.pc = 8;
  cfg.b = 16;
  cfg.rows_per_cta = static_cast<int>(ceil_div(ceil_div(d_pad, cfg.cluster), 4) * 4);
  cfg.groups = static_cast<int>(ceil_div(p, cfg.pc));
  cfg.smem = smem_layout<8, 16>(cfg.rows_per_cta).total;
  return cfg;
}

void launch_svrg_epoch_dense(const EpochArgs& a, const EpochConfig& cfg, cudaStream_t st) {
  auto kern = k_svrg_epoch_dense<8, 16>;
  if (cfg.pc != 8 || cfg.b != 16) throw Error(kContractViolation, "epoch: unsupported config");
  if (cfg.smem > 227 * 1024) throw Error(kContractViolation, "epoch: d too large for the cluster row split");
  GAPLRA_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(cfg.smem)));
  if (cfg.cluster > 8)
    GAPLRA_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(cfg.cluster, cfg.groups, 1);
  lc.blockDim = dim3(kEpochThreads, 1, 1);
  lc.dynamicSmemBytes = cfg.smem;
  lc.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cfg.cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  EpochArgs args = a;
  args.rows_per_cta = cfg.rows_per_cta;
  GAPLRA_CUDA_CHECK(cudaLaunchKernelEx(&lc, kern, args));
}

void launch_svrg_epoch_sparse(const SparseEpochArgs& a, cudaStream_t st) {
  k_svrg_epoch_sparse<<<ceil_div(a.p, 32), 32, 0, st>>>(a);
  GAPLRA_LAUNCH_CHECK();
}

int anchor_parts(int d) { return static_cast<int>(std::min<int64_t>(ceil_div(d, 256), 148)); }

void launch_anchor(const double* W, const double* Z, const double* Bm, int64_t ld, int d, int p, double lambda,
                   double eta, double* C, double* part, const double* bnorm, double* colnorm, double* out_max,
                   cudaStream_t st) {
  if (p > kAnchorMaxP) throw Error(kContractViolation, "anchor: p > 64");
  const int parts = anchor_parts(d);
  k_anchor<<<parts, kAnchorThreads, 0, st>>>(W, Z, Bm, ld, d, p, lambda, eta, C, part);
  GAPLRA_LAUNCH_CHECK();
  k_anchor_final<<<1, kAnchorMaxP, 0, st>>>(part, parts, p, bnorm, colnorm, out_max);
  GAPLRA_LAUNCH_CHECK();
}

}  // namespace gaplra_cuda
