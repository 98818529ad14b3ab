// SVRG epoch kernels for the block solve of (λI − XXᵀ)W = B.
//
// Spec (restated in oracle/oracle.cpp svrg_epoch): for each of
// m = 2n sampled indices i (shared by all p columns),
//     r = ηn (x_iᵀ W − Y_i),   W ← ρ W + C + x_i rᵀ,   ρ = 1 − ηλ,  C = η(X Xᵀ W̃ + B)
// with Y = Xᵀ W̃ from the anchor.  The device evaluates it in exact-arithmetic-
// equivalent s-step blocks of b steps:
//     P_j = x_{i_j}ᵀ W_0,   H_i = x_iᵀ C (one precomputed pass per epoch)
//     v_j = ηn (ρ^j P_j + γ_j H_{i_j} − Y_{i_j}),   γ_j = Σ_{t<j} ρ^t
//     (I − L) r = v,   L_jl = ηn ρ^{j−1−l} x_{i_j}ᵀ x_{i_l}  (l < j)
//     W_b = ρ^b W_0 + γ_b C + Σ_l ρ^{b−1−l} x_{i_l} r_lᵀ
// L depends only on the index stream and X, so T = (I − L)⁻¹ is computed for
// every block of the epoch up front by k_block_gram_t (fully parallel, DMMA
// fp64 Gram of the b sampled columns).  The sequential part, k_svrg_chain,
// then needs per block only: the partial dots P over the CTA's rows, ONE
// cluster all-reduce through distributed shared memory, r = T v, and the W
// update on its rows.  One thread-block cluster (G CTAs splitting d rows,
// W/C row slices resident in shared memory for the whole epoch) per group of
// PC right-hand-side columns; sampled column slices and T are streamed one
// block ahead by TMA bulk copies (cp.async.bulk + mbarrier).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "svrg.cuh"
#include "rng.cuh"

namespace cg = cooperative_groups;

#ifndef V3_PROD1
#define V3_PROD1 2
#endif
#ifndef V3_SLEEP
#define V3_SLEEP 128
#endif

namespace gaplra_cuda {

namespace {

// ---------------------------------------------------------------------------
// PTX helpers: mbarrier + TMA 1D bulk copies + cp.async (LDGSTS) + DMMA.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Producer-side wait: producers run stages ahead, so a failed poll backs off
// instead of spinning (a spinning warp takes issue slots from the consumers
// on its SM sub-partition).
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  for (;;) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return;
    __nanosleep(V3_SLEEP);
  }
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// Bulk shared::cta -> shared::cluster copy completing on the receiver's mbarrier.
__device__ __forceinline__ void dsmem_bulk_copy(uint32_t remote_dst, uint32_t local_src, uint32_t bytes,
                                                uint32_t remote_bar) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   remote_dst),
               "r"(local_src), "r"(bytes), "r"(remote_bar)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ---- global-memory (L2) all-reduce among the CTAs of a column group (XG
// chains: no thread-block cluster, so a group may span any CTAs; C5's 8 groups
// of 16 CTAs exceed the 7 sixteen-CTA clusters that fit at once).  Block u's
// partials go to slot u % kXgSlots; each peer publishes with a release and one
// counter increment; a reader waits for G * (uses of the slot) arrivals and
// reads the partials through L2 (ld.cg: the slot's previous use may sit in L1).
// No gpu-scope fence / acquire in the loops: on this part those invalidate L1
// (CCTL.IVALL), which stalled the row warps' shared-memory traffic (an
// acquire-spinning reducer made the p = 1 update 4x slower).  The publisher's
// red.release orders the warp's stores (issued before it, the lanes joined by
// __syncwarp) ahead of the count; the reader polls relaxed and reads L2 after.
// Slot reuse: a CTA publishes block u + 1 only after it received every peer's
// block u - 1, so no peer still reads slot u + 1 - kXgSlots >= 4 blocks back.
constexpr int kXgSlots = 8;
__device__ __forceinline__ void xg_publish(unsigned* count) {
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(count) : "memory");
}
__device__ __forceinline__ void xg_wait(const unsigned* count, unsigned need) {
  unsigned v;
  for (;;) {
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(count) : "memory");
    if (v >= need) break;
  }
}
__device__ __forceinline__ double ld_cg(const double* p) {
  double v;
  asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_cg(double* p, double v) {
  asm volatile("st.global.cg.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// ---- flag-in-data ("LL") exchange cells: a partial travels as one 16-byte
// cell {lo32, flag, hi32, flag}; 8-byte halves are written and read atomically,
// so a reader that sees both flags equal to the expected value has the whole
// double — no fence, no counter, one L2 store + one L2 load on the critical
// path (the counter protocol above pays a MEMBAR.GPU + a counter round trip +
// the partial loads).  flag = 1 + (uses of the slot so far); the cells are
// zeroed before every launch, so a stale cell never matches.
__device__ __forceinline__ void ll_store(uint4* cell, double v, uint32_t flag) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(cell), "r"(__double2loint(v)), "r"(flag),
               "r"(__double2hiint(v)), "r"(flag)
               : "memory");
}
__device__ __forceinline__ uint4 ll_load(const uint4* cell) {
  uint4 w;
  asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
               : "l"(cell)
               : "memory");
  return w;
}
// Sum over the G peers of entry e = lane & 15 of a 16-entry slot ([G][16]
// cells): lanes 0-15 take peers q, q + 1 and lanes 16-31 peers q + 2, q + 3 of
// every four, (sa + sb) per half then half 0 + half 1 — the same fixed order as
// the counter form.  Up to 16 cells per lane are polled at once.
__device__ __forceinline__ double ll_gather16(const uint4* slot, int G, int lane, uint32_t flag) {
  const int e = lane & 15, hq = (lane >> 4) * 2;
  double sa = 0.0, sb = 0.0;
#pragma unroll 1
  for (int q0 = 0; q0 < G; q0 += 32) {
    uint4 w[16];
    unsigned pend = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int peer = q0 + 4 * (k >> 1) + hq + (k & 1);
      if (peer < G) {
        w[k] = ll_load(slot + peer * 16 + e);
        pend |= 1u << k;
      } else {
        w[k] = make_uint4(0u, flag, 0u, flag);
      }
    }
    while (pend) {
#pragma unroll
      for (int k = 0; k < 16; ++k)
        if (pend >> k & 1u) {
          if (w[k].y == flag && w[k].w == flag)
            pend &= ~(1u << k);
          else
            w[k] = ll_load(slot + (q0 + 4 * (k >> 1) + hq + (k & 1)) * 16 + e);
        }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      sa += __hiloint2double(static_cast<int>(w[2 * i].z), static_cast<int>(w[2 * i].x));
      sb += __hiloint2double(static_cast<int>(w[2 * i + 1].z), static_cast<int>(w[2 * i + 1].x));
    }
  }
  const double sv = sa + sb;
  return sv + __shfl_down_sync(0xffffffffu, sv, 16);
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// ---------------------------------------------------------------------------
// k_block_prep: everything of s-step block t that does not depend on W.
//   K_t   = X_{B_t}ᵀ X_{B_t}   (strict lower part), Kx_t = X_{B_t}ᵀ X_{B_{t−1}}
//   T_t   = (I − L_t)⁻¹,  L_jl = ηn ρ^{j−1−l} K_jl
//   TT_t  = diag(ρ^{b−1−j}) T_t diag(ηn ρ^l)          (coef = TT P̂ + U)
//   M_t   = TT_t Kx_t                                  (lookahead correction)
//   (U_t = diag(ρ^{b−1−j}) T_t q is formed later by k_block_u: it needs the
//   epoch's Y and H, the rest depends only on the index stream and X, so
//   k_block_prep of epoch e+1 runs beside the chain of epoch e)
// with W = Ŵ + β C tracked lazily (β_t = γ_{tB} = Σ_{k<tB} ρ^k), so C never has
// to be resident.  Gram by DMMA m8n8k4 fp64, warps split the d rows, fixed
// order reductions.  Slab per block: [TT | M | U(group 0) | U(group 1) | ...].
// ---------------------------------------------------------------------------
constexpr int kPrepThreads = 256;
constexpr int kMaxP = 64;

// 16x16 (B x B) product C = A·Bm by 256 threads (thread = entry), smem operands.
template <int B>
__device__ __forceinline__ void mat_mul_bb(const double (*A)[B + 1], const double (*Bm)[B + 1], double (*Cm)[B + 1],
                                           int tid) {
  for (int e = tid; e < B * B; e += kPrepThreads) {
    const int i = e / B, j = e % B;
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int k = 0; k < B; k += 2) {
      s0 = fma(A[i][k], Bm[k][j], s0);
      s1 = fma(A[i][k + 1], Bm[k + 1][j], s1);
    }
    Cm[i][j] = s0 + s1;
  }
}

// Column ring of k_block_prep: 32 columns (16 of block t, 16 of block t−1) ×
// kPrepKC rows per stage, filled by one producer warp with cp.async.bulk.
// Pitch ≡ 4 (mod 16) doubles: the m8n8k4 fragment LDS (lane → column lane>>2,
// row lane&3) touches 16 distinct bank pairs per half warp.
constexpr int kPrepKC = 64;
constexpr int kPrepPitch = kPrepKC + 4;
constexpr int kPrepStages = 4;
// LA = 2 (two-block lookahead chain): a third group of 16 columns, block t−2,
// for the second cross-Gram Kxx_t = X_{B_t}ᵀ X_{B_{t−2}}
template <int LA>
__host__ __device__ constexpr int prep_cols() { return 16 * (LA + 1); }
template <int LA>
__host__ __device__ constexpr size_t prep_ring_bytes() { return size_t(kPrepStages) * prep_cols<LA>() * kPrepPitch * sizeof(double); }
// cp.async.bulk takes warp-uniform operands, so one warp issues its lanes'
// copies one after another (~50 cycles each): 4 producer warps, one per SM
// sub-partition, 8 columns each.
constexpr int kPrepProducers = 4;
constexpr int kPrepCtas = 2;  // CTAs per SM: one's serial tail overlaps the other's Gram loop
// the consumers' per-warp partial Grams live after the ring (dynamic smem)
template <int LA>
__host__ __device__ constexpr size_t prep_red_bytes() {
  return size_t(kPrepThreads / 32) * (3 + 4 * LA) * 64 * sizeof(double);
}

__device__ __forceinline__ void prep_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kPrepThreads) : "memory"); }

template <int B, int LA>
__global__ void __launch_bounds__(kPrepThreads + 32 * kPrepProducers, kPrepCtas) k_block_prep(EpochArgs a) {
  static_assert(B == 16, "T = (I+L)(I+L^2)(I+L^4)(I+L^8) and the 32-column ring assume B = 16");
  static_assert(LA == 1 || LA == 2, "one- or two-block lookahead");
  constexpr int G8 = B / 8;
  constexpr int NW = G8 * (G8 + 1) / 2;  // within-block lower tiles
  constexpr int NX = G8 * G8;            // cross tiles per previous block
  constexpr int NT = NW + LA * NX;
  constexpr int NCOL = prep_cols<LA>();
  constexpr int CPP = NCOL / kPrepProducers;  // ring columns per producer warp
  constexpr int NWARP = kPrepThreads / 32;
  constexpr int RPW = kPrepKC / NWARP;  // rows of a chunk per consumer warp
  static_assert(RPW % 4 == 0, "whole m8n8k4 k-steps per warp");
  static_assert(prep_red_bytes<LA>() == size_t(NWARP) * NT * 64 * sizeof(double), "red layout");
  extern __shared__ __align__(128) double ring[];
  auto red = reinterpret_cast<double (*)[NT][64]>(ring + size_t(kPrepStages) * NCOL * kPrepPitch);
  __shared__ double K[B][B + 1];
  __shared__ double Kx[B][B + 1];
  __shared__ double Kxx[LA == 2 ? B : 1][B + 1];
  __shared__ double T[B][B + 1];
  __shared__ double TT[B][B + 1];
  __shared__ double rp[B + 1], gm[B + 1];
  __shared__ __align__(8) uint64_t full[kPrepStages], empty[kPrepStages];
  static_assert(prep_red_bytes<LA>() >= 4 * B * (B + 1) * sizeof(double), "P aliases red");
  // L, L², L⁴, L⁸ then the running products; red is dead once K/Kx are reduced
  auto P = reinterpret_cast<double (*)[B][B + 1]>(&red[0][0][0]);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nblocks = (a.m + B - 1) / B;
  // Grid-stride blocks: CTA c+1 reads block t+1's "previous" columns while CTA
  // c reads the same columns as block t's current ones, so one of the two
  // requests hits L2 (a contiguous range per CTA would re-read them after
  // ~148 MB of other traffic, i.e. from DRAM).
  const int64_t t_begin = blockIdx.x, t_step = gridDim.x, t_end = nblocks;
  const int nkc = (a.d_pad + kPrepKC - 1) / kPrepKC;
  if (threadIdx.x == 0) {
    rp[0] = 1.0;
    gm[0] = 0.0;
    for (int j = 1; j <= B; ++j) {
      rp[j] = rp[j - 1] * a.rho;
      gm[j] = gm[j - 1] + rp[j - 1];
    }
    for (int s = 0; s < kPrepStages; ++s) {
      mbar_init(&full[s], kPrepProducers);
      mbar_init(&empty[s], NWARP);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp < kPrepProducers) {  // ------------------------------------- producers
    // producer warp w stages ring columns [CPP w, CPP (w+1)): 0..15 block t,
    // 16..31 block t−1, (LA = 2) 32..47 block t−2
    const int rc = warp * CPP + lane;
    int stage = 0;
    uint32_t phase = 0;
    auto col_of = [&](int64_t t) {  // this lane's ring column of block t (zeros when masked)
      const double* col = a.zcol;
      if (t < t_end && lane < CPP) {
        const int64_t s0 = t * B;
        const int bt = static_cast<int>(a.m - s0 < B ? a.m - s0 : B);
        if (rc < B) {
          if (rc < bt) col = a.X + static_cast<int64_t>(a.idx[s0 + rc]) * a.ldx;
        } else if (rc < 2 * B) {
          if (t > 0) col = a.X + static_cast<int64_t>(a.idx[s0 - B + (rc - B)]) * a.ldx;
        } else if (t > 1) {
          col = a.X + static_cast<int64_t>(a.idx[s0 - 2 * B + (rc - 2 * B)]) * a.ldx;
        }
      }
      return col;
    };
    const double* ncol = col_of(t_begin);
    for (int64_t t = t_begin; t < t_end; t += t_step) {
      const double* col = ncol;
      ncol = col_of(t + t_step);  // next block's index load off the refill path
      for (int kc = 0; kc < nkc; ++kc) {
        const int k0 = kc * kPrepKC;
        const int len = a.d_pad - k0 < kPrepKC ? a.d_pad - k0 : kPrepKC;
        const uint32_t bytes = static_cast<uint32_t>(len) * sizeof(double);
        mbar_wait_backoff(&empty[stage], phase ^ 1);
        if (lane == 0) mbar_expect_tx(&full[stage], bytes * CPP);
        __syncwarp();
        if (lane < CPP)
          tma_load_1d(ring + (static_cast<size_t>(stage) * NCOL + rc) * kPrepPitch, col + k0, bytes, &full[stage]);
        if (++stage == kPrepStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    return;
  }
  // -------------------------------------------------------------- consumers
  const int ct = threadIdx.x - 32 * kPrepProducers, cw = warp - kPrepProducers;
  const int fr = lane >> 2, fc = lane & 3;
  int stage = 0;
  uint32_t phase = 0;
  for (int64_t t = t_begin; t < t_end; t += t_step) {
    const int64_t s0 = t * B;
    const int bt = static_cast<int>(a.m - s0 < B ? a.m - s0 : B);
    const bool has_prev = t > 0;
    double acc[NT][2];
#pragma unroll
    for (int qq = 0; qq < NT; ++qq) acc[qq][0] = acc[qq][1] = 0.0;
    for (int kc = 0; kc < nkc; ++kc) {
      const int len = a.d_pad - kc * kPrepKC < kPrepKC ? a.d_pad - kc * kPrepKC : kPrepKC;
      mbar_wait(&full[stage], phase);
      const double* sb = ring + static_cast<size_t>(stage) * NCOL * kPrepPitch + fr * kPrepPitch + fc;
#pragma unroll
      for (int ks = 0; ks < RPW / 4; ++ks) {
        const int kk = cw * RPW + ks * 4;
        if (kk < len) {
          double f[G8], fp[LA][G8];
#pragma unroll
          for (int g = 0; g < G8; ++g) {
            f[g] = sb[g * 8 * kPrepPitch + kk];
#pragma unroll
            for (int q = 0; q < LA; ++q) fp[q][g] = sb[((q + 1) * B + g * 8) * kPrepPitch + kk];
          }
          int qq = 0;
#pragma unroll
          for (int gj = 0; gj < G8; ++gj)
#pragma unroll
            for (int gl = 0; gl <= gj; ++gl, ++qq) dmma(acc[qq][0], acc[qq][1], f[gj], f[gl]);
#pragma unroll
          for (int q = 0; q < LA; ++q)
#pragma unroll
            for (int gj = 0; gj < G8; ++gj)
#pragma unroll
              for (int gl = 0; gl < G8; ++gl, ++qq) dmma(acc[qq][0], acc[qq][1], f[gj], fp[q][gl]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == kPrepStages) {
        stage = 0;
        phase ^= 1;
      }
    }
#pragma unroll
    for (int qq = 0; qq < NT; ++qq) {
      red[cw][qq][2 * lane] = acc[qq][0];
      red[cw][qq][2 * lane + 1] = acc[qq][1];
    }
    prep_sync();
    for (int e = ct; e < NT * 64; e += kPrepThreads) {
      const int qq = e / 64, o = e % 64;
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < NWARP; ++w) s += red[w][qq][o];
      const int ln = o >> 1;
      const int mi = ln >> 2, ni = 2 * (ln & 3) + (o & 1);
      if (qq < NW) {
        int gj = 0, rem = qq;
        while (rem > gj) {
          rem -= gj + 1;
          ++gj;
        }
        K[gj * 8 + mi][rem * 8 + ni] = s;
      } else if (qq < NW + NX) {
        const int x = qq - NW;
        Kx[(x / G8) * 8 + mi][(x % G8) * 8 + ni] = s;
      } else if constexpr (LA == 2) {
        const int x = qq - NW - NX;
        Kxx[(x / G8) * 8 + mi][(x % G8) * 8 + ni] = s;
      }
    }
    prep_sync();
    // L_jl = ηn ρ^{j−1−l} K_jl (l < j < bt), nilpotent: T = (I+L)(I+L²)(I+L⁴)(I+L⁸)
    for (int e = ct; e < B * B; e += kPrepThreads) {
      const int j = e / B, l = e % B;
      P[0][j][l] = (l < j && j < bt) ? a.eta_n * rp[j - 1 - l] * K[j][l] : 0.0;
    }
    prep_sync();
    mat_mul_bb<B>(P[0], P[0], P[1], ct);  // L²
    prep_sync();
    mat_mul_bb<B>(P[1], P[1], P[2], ct);  // L⁴
    prep_sync();
    mat_mul_bb<B>(P[2], P[2], P[3], ct);  // L⁸
    prep_sync();
    for (int e = ct; e < B * B; e += kPrepThreads) {  // T = I + L, P[k] += I
      const int j = e / B, l = e % B;
      const double id = j == l ? 1.0 : 0.0;
      T[j][l] = P[0][j][l] + id;
      P[1][j][l] += id;
      P[2][j][l] += id;
      P[3][j][l] += id;
    }
    prep_sync();
    mat_mul_bb<B>(T, P[1], P[0], ct);  // (I+L)(I+L²)
    prep_sync();
    mat_mul_bb<B>(P[0], P[2], P[1], ct);  // ·(I+L⁴)
    prep_sync();
    mat_mul_bb<B>(P[1], P[3], T, ct);  // ·(I+L⁸)
    prep_sync();
    for (int e = ct; e < B * B; e += kPrepThreads) {
      const int j = e / B, l = e % B;
      TT[j][l] = (j < bt && l <= j) ? rp[bt - 1 - j] * T[j][l] * (a.eta_n * rp[l]) : 0.0;
    }
    prep_sync();
    double* slab = a.slab + t * a.slab_len;
    // TT and M are stored transposed ([l][j]): consumers index them with j
    // varying across lanes (bank-conflict free).
    for (int e = ct; e < B * B; e += kPrepThreads) {
      const int j = e / B, l = e % B;
      slab[l * B + j] = TT[j][l];
      double s = 0.0;
      if (has_prev)
#pragma unroll
        for (int k = 0; k < B; ++k) s = fma(TT[j][k], Kx[k][l], s);
      slab[B * B + l * B + j] = s;
      if constexpr (LA == 2) {  // M2_t = TT_t Kxx_t (the ρ^{b_{t−1}} scale is applied by the chain)
        double s2 = 0.0;
        if (t > 1)
#pragma unroll
          for (int k = 0; k < B; ++k) s2 = fma(TT[j][k], Kxx[k][l], s2);
        slab[2 * B * B + l * B + j] = s2;
      }
    }
    prep_sync();
  }
}

// ---------------------------------------------------------------------------
// k_svrg_chain: the sequential recurrence with one-block lookahead.
// State per CTA: V = ρ^{b_t} Ŵ_t on its rows (W = Ŵ + βC, β folded into U).
// Iteration t (all quantities for the cluster's PC columns):
//   (b) Â_{t+1} partial = X_{B_{t+1}}ᵀ V_t on own rows (needs only V_t);
//       st.async into every peer's receive slot
//   (d) wait for Â_t (pushed one iteration earlier); Â_t = Σ_q slot_q (fixed order)
//   (a) coef_t = TT_t Â_t + M_t coef_{t−1} + U_t            (local, redundant)
//   (c) Ŵ_{t+1} = V_t + X_{B_t} coef_t;  V_{t+1} = ρ^{b_{t+1}} Ŵ_{t+1}
// so the cluster all-reduce of Â_{t+1} overlaps (d), (a), (c) of block t and
// (b) of block t+1.  X slices and the
// block slab stream through an S-stage TMA ring (cp.async.bulk + mbarrier).
// ---------------------------------------------------------------------------
constexpr int kChainThreads = 256;
constexpr int kMaxCluster = 16;
// Â_u lives in receive slot u mod 4.  A CTA pushes Â_{t+1} at the start of
// its iteration t, after it received Â_{t−1} from every peer, i.e. after every
// peer started iteration t−2 and so finished reading Â_{t−3} (same slot).
constexpr int kRecvSlots = 4;

struct ChainSmem {
  int rows_pad, stages;
  size_t stage_len, off_stage, off_v, off_recv, off_a, off_coef, off_rprev, off_idx, off_red, off_bar, total;
};

// rows_pad ≡ 2 (mod 16) doubles by default (DMMA / scalar phases: fragment
// loads across 8 slices are conflict-free); PAD16 gives rows_pad ≡ 0 (mod 16)
// for k_svrg_chain_v3, whose lane-permuted slice loads are then conflict-free.
template <int PC, int B, bool PAD16 = false>
__host__ __device__ inline ChainSmem chain_smem(int rows, int stages) {
  ChainSmem s;
  s.rows_pad = PAD16 ? (rows + 15) / 16 * 16 : (rows + 1) / 2 * 2 + 2;
  s.stages = stages;
  s.stage_len = static_cast<size_t>(B) * s.rows_pad + 2 * B * B + B * PC;  // X slices | TT | M | U
  size_t o = 0;
  s.off_stage = o;
  o += s.stage_len * stages;
  s.off_v = o;
  o += static_cast<size_t>(s.rows_pad) * PC;  // row-major [r][PC] or column-major [c][RP]
  s.off_recv = o;
  o += kRecvSlots * kMaxCluster * B * PC;
  s.off_a = o;
  o += B * PC;
  s.off_coef = o;
  o += B * PC;
  s.off_rprev = o;
  o += B * PC;
  s.off_idx = o;
  o += 0;
  s.off_red = o;
  o += (kChainThreads / 32) * (B / 8) * 64;
  s.off_bar = o;
  o += 20;  // full[8] | empty[8] | rbar[4]
  s.total = o * sizeof(double);
  return s;
}

__device__ __forceinline__ uint32_t mapa(uint32_t local_smem_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_smem_addr), "r"(rank));
  return r;
}
// Remote (DSMEM) 8-byte store that completes 8 transaction bytes on the
// receiver's mbarrier: no fence / cluster barrier on the critical path.
__device__ __forceinline__ void st_async_f64(uint32_t remote_addr, double v, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(remote_addr),
               "l"(__double_as_longlong(v)), "r"(remote_bar)
               : "memory");
}

__device__ __forceinline__ void st_async_f64x2(uint32_t remote_addr, double v0, double v1, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];" ::"r"(remote_addr),
               "l"(__double_as_longlong(v0)), "l"(__double_as_longlong(v1)), "r"(remote_bar)
               : "memory");
}

__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kChainThreads) : "memory"); }

// Producer side of the chain kernels: block t's X slices (rows [r0, r0+rc) of
// the bt sampled columns) and its slab part stream into stage t mod S.  The
// bulk copies take warp-uniform operands (one warp issues its lanes' copies in
// turn), so kChainProducers warps share the columns.
constexpr int kChainProducers = 4;


template <int PC, int B, int NP = kChainProducers>
__device__ __forceinline__ void chain_produce(const EpochArgs& a, int pw, int lane, int nb, int last_bt, int S, int rc,
                                              int r0, int RP, int grp, double* stages, size_t stage_len,
                                              uint64_t* full, uint64_t* empty, int head = 2 * B * B) {
  constexpr int CPP = B / NP;  // columns per producer warp
  static_assert(B % NP == 0 && CPP <= 31, "producers cover the B columns; lane 31 issues the slab");
  int s = 0;
  uint32_t eph = 0;  // parity of the next empty-barrier completion per wrap
  const int j0 = pw * CPP;
  // this lane's sampled column of block u, loaded one block ahead: the index
  // load's L2 latency stays off the refill path (empty -> TMA issue)
  auto col_of = [&](int u) {
    const int bu = u == nb - 1 ? last_bt : B;
    return u < nb && lane < CPP && j0 + lane < bu ? __ldg(a.idx + static_cast<int64_t>(u) * B + j0 + lane) : 0;
  };
  int ncol = col_of(0);
  for (int t = 0; t < nb; ++t) {
    const int col = ncol;
    ncol = col_of(t + 1);
    if (t >= S) mbar_wait_backoff(&empty[s], eph);
    const int bt = t == nb - 1 ? last_bt : B;
    double* st = stages + static_cast<size_t>(s) * stage_len;
    const int mine = rc > 0 ? max(0, min(CPP, bt - j0)) : 0;
    if (lane == 0) {
      fence_proxy_async();
      mbar_expect_tx(&full[s], static_cast<uint32_t>(mine * rc + (pw == 0 ? head + B * PC : 0)) * 8u);
    }
    __syncwarp();
    if (lane < mine) {
      const int j = j0 + lane;
      tma_load_1d(st + j * RP, a.X + static_cast<int64_t>(col) * a.ldx + r0, rc * 8u, &full[s]);
    }
    // L2 prefetch of the same slices a.prefetch blocks ahead: the index
    // stream is known for the whole epoch, so the ring's TMA loads hit L2
    // instead of paying the DRAM latency with only S blocks in flight
    if (a.prefetch > 0 && t + a.prefetch < nb && rc > 0 && lane < CPP) {
      const int64_t tp = t + a.prefetch;
      const int btp = tp == nb - 1 ? last_bt : B;
      const int j = j0 + lane;
      if (j < btp) {
        const double* src = a.X + static_cast<int64_t>(__ldg(a.idx + tp * B + j)) * a.ldx + r0;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(static_cast<uint32_t>(rc * 8u))
                     : "memory");
      }
    }
    if (pw == 0 && lane == 31) {
      const double* slab = a.slab + static_cast<int64_t>(t) * a.slab_len;
      tma_load_1d(st + B * RP, slab, static_cast<uint32_t>(head) * 8u, &full[s]);
      tma_load_1d(st + B * RP + head, slab + head + static_cast<size_t>(grp) * B * PC, B * PC * 8u, &full[s]);
    }
    if (++s == S) {
      s = 0;
      if (t >= S) eph ^= 1u;
    }
  }
}

template <int PC, int B, bool SCALAR>
__global__ void __launch_bounds__(kChainThreads + 32 * kChainProducers, 1) k_svrg_chain(EpochArgs a) {
  extern __shared__ __align__(128) double sm[];
  cg::cluster_group cluster = cg::this_cluster();
  const int G = static_cast<int>(cluster.num_blocks());
  const int g = static_cast<int>(cluster.block_rank());
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int grp = blockIdx.y;
  const int c0 = grp * PC;
  const int pc = min(PC, a.p - c0);
  const ChainSmem L = chain_smem<PC, B>(a.rows_per_cta, a.stages);
  const int S = L.stages;
  const int r0 = g * a.rows_per_cta;
  const int rc = max(0, min(a.rows_per_cta, a.d_pad - r0));
  const int RP = L.rows_pad;
  double* V = sm + L.off_v;
  double* recv = sm + L.off_recv;  // [kRecvSlots][kMaxCluster][B*PC]
  double* Ahat = sm + L.off_a;
  double* coef = sm + L.off_coef;
  double* rprev = sm + L.off_rprev;
  double* red = sm + L.off_red;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + L.off_bar);  // [S] TMA landed
  uint64_t* empty = full + 4;                                     // [S] consumers done
  uint64_t* rbar = full + 8;                                      // [4] all-reduce slots
  // stage of block t is t mod S; callers track it incrementally (no 64-bit
  // division on the critical path)
  auto stage_at = [&](int s_idx) { return sm + L.off_stage + static_cast<size_t>(s_idx) * L.stage_len; };

  const int nb = static_cast<int>((a.m + B - 1) / B);
  const int last_bt = static_cast<int>(a.m - static_cast<int64_t>(nb - 1) * B);
  auto bt_of = [&](int t) { return t == nb - 1 ? last_bt : B; };
  double rho_b = 1.0, rho_last = 1.0;  // ρ^B and ρ^{b of the last block}
  for (int j = 0; j < B; ++j) rho_b *= a.rho;
  for (int j = 0; j < last_bt; ++j) rho_last *= a.rho;
  // V row slice: row-major [r][PC] for the DMMA phases, column-major [c][RP]
  // (lane-consecutive rows, conflict-free) for the scalar phases.
  auto vix = [&](int r, int c) { return SCALAR ? c * RP + r : r * PC + c; };
  for (int e = tid; e < rc * PC; e += blockDim.x) {
    const int r = e / PC, c = e - (e / PC) * PC;
    V[vix(r, c)] = c < pc ? a.W[static_cast<int64_t>(r0 + r) * a.ldw + c0 + c] : 0.0;
  }
  for (int e = tid; e < B * PC; e += blockDim.x) rprev[e] = 0.0;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], kChainProducers);
      mbar_init(&empty[s], kChainThreads / 32);  // one arrival per consumer warp
    }
    for (int q = 0; q < kRecvSlots; ++q) mbar_init(&rbar[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster.sync();  // barriers initialised cluster-wide before any push / TMA

  if (warp >= kChainThreads / 32) {
    chain_produce<PC, B>(a, warp - kChainThreads / 32, lane, nb, last_bt, S, rc, r0, RP, grp, sm + L.off_stage,
                         L.stage_len, full, empty);
  } else {
    // ===== 8 consumer warps
    // stage index / full-barrier parity of the block being waited for
    int ws = 0;
    uint32_t wph = 0;
    auto wait_next = [&]() {  // blocks are waited for in order 0, 1, 2, ...
      mbar_wait(&full[ws], wph);
      if (++ws == S) {
        ws = 0;
        wph ^= 1u;
      }
    };
    // Scalar form: warp w owns steps j = w, w + 8 (lanes stride the rows),
    // xor-shuffle sums leave the totals in every lane, lane q < G st.async's
    // its copy to rank q.
    auto dots_push_scalar = [&](const double* xb, int bt, int u) {
      const int par = u & (kRecvSlots - 1);
      constexpr int NWC = kChainThreads / 32;
      const uint32_t rb = mapa(smem_u32(&rbar[par]), lane < G ? lane : 0);
      const uint32_t rslot = mapa(smem_u32(recv + (par * kMaxCluster + g) * B * PC), lane < G ? lane : 0);
      for (int j0 = warp; j0 < bt; j0 += 2 * NWC) {
        const int j1 = j0 + NWC;
        const bool two = j1 < bt;
        double s0[PC], s1[PC];
#pragma unroll
        for (int c = 0; c < PC; ++c) s0[c] = s1[c] = 0.0;
        const double* x0 = xb + j0 * RP;
        const double* x1 = xb + (two ? j1 : j0) * RP;
#pragma unroll 2
        for (int r = lane; r < rc; r += 32) {
          const double u0 = x0[r], u1 = x1[r];
#pragma unroll
          for (int c = 0; c < PC; ++c) {
            const double v = V[c * RP + r];
            s0[c] = fma(u0, v, s0[c]);
            s1[c] = fma(u1, v, s1[c]);
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int c = 0; c < PC; ++c) {
            s0[c] += __shfl_xor_sync(0xffffffffu, s0[c], o);
            s1[c] += __shfl_xor_sync(0xffffffffu, s1[c], o);
          }
        if (lane < G) {
#pragma unroll
          for (int c = 0; c < PC; ++c) {
            st_async_f64(rslot + (j0 * PC + c) * 8u, s0[c], rb);
            if (two) st_async_f64(rslot + (j1 * PC + c) * 8u, s1[c], rb);
          }
        }
      }
    };
    // Partial Â = X_Bᵀ V over the owned rows (DMMA: M = j, N = columns, K =
    // rows split over the 8 warps), fixed-order cross-warp sum, then st.async
    // of every entry into slot g of every peer (completing on its rbar).
    auto dots_push = [&](const double* xb, int bt, int u) {
      if constexpr (SCALAR) {
        dots_push_scalar(xb, bt, u);
        return;
      }
      const int par = u & (kRecvSlots - 1);
      const int gq = lane >> 2, tq = lane & 3;
      constexpr int NA = 4;  // independent accumulation chains per tile
      double acc[NA][B / 8][2];
#pragma unroll
      for (int q = 0; q < NA; ++q)
#pragma unroll
        for (int mt = 0; mt < B / 8; ++mt) acc[q][mt][0] = acc[q][mt][1] = 0.0;
      const int nks = rc / 4;
      constexpr int WS = kChainThreads / 32;
      int ks = warp;
      for (; ks + (NA - 1) * WS < nks; ks += NA * WS) {
#pragma unroll
        for (int q = 0; q < NA; ++q) {
          const int r = 4 * (ks + q * WS) + tq;
          const double bv = gq < PC ? V[r * PC + gq] : 0.0;
#pragma unroll
          for (int mt = 0; mt < B / 8; ++mt) dmma(acc[q][mt][0], acc[q][mt][1], xb[(8 * mt + gq) * RP + r], bv);
        }
      }
      for (; ks < nks; ks += WS) {
        const int r = 4 * ks + tq;
        const double bv = gq < PC ? V[r * PC + gq] : 0.0;
#pragma unroll
        for (int mt = 0; mt < B / 8; ++mt) dmma(acc[0][mt][0], acc[0][mt][1], xb[(8 * mt + gq) * RP + r], bv);
      }
#pragma unroll
      for (int mt = 0; mt < B / 8; ++mt) {
        red[(warp * (B / 8) + mt) * 64 + 2 * lane] = (acc[0][mt][0] + acc[1][mt][0]) + (acc[2][mt][0] + acc[3][mt][0]);
        red[(warp * (B / 8) + mt) * 64 + 2 * lane + 1] =
            (acc[0][mt][1] + acc[1][mt][1]) + (acc[2][mt][1] + acc[3][mt][1]);
      }
      consumers_sync();
      const uint32_t slot = smem_u32(recv + (par * kMaxCluster + g) * B * PC);
      const uint32_t rbl = smem_u32(&rbar[par]);
      for (int e = tid; e < bt * PC; e += kChainThreads) {
        const int j = e / PC, c = e - (e / PC) * PC;
        // C fragment position of (j, c): tile j/8, lane 4*(j%8) + c/2, element c%2
        const int o = ((j >> 3) * 64) + 2 * (4 * (j & 7) + (c >> 1)) + (c & 1);
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < kChainThreads / 32; ++w) s += red[w * (B / 8) * 64 + o];
        for (int q = 0; q < G; ++q) st_async_f64(mapa(slot, q) + e * 8u, s, mapa(rbl, q));
      }
    };
    auto arm_recv = [&](int u) {
      mbar_expect_tx(&rbar[u & (kRecvSlots - 1)], static_cast<uint32_t>(G * bt_of(u) * PC * 8));
    };
    auto recv_sum = [&](int u) {
      const int par = u & (kRecvSlots - 1);
      mbar_wait(&rbar[par], static_cast<uint32_t>((u >> 2) & 1));
      const int n = bt_of(u) * PC;
      for (int e = tid; e < n; e += kChainThreads) {
        double s = 0.0;
        for (int q = 0; q < G; ++q) s += recv[(par * kMaxCluster + q) * B * PC + e];
        Ahat[e] = s;
      }
    };
    if (nb > 0) {  // push Â_0 = X_{B_0}ᵀ Ŵ_0, then V_0 = ρ^{b_0} Ŵ_0
      if (tid == 0) arm_recv(0);
      wait_next();
      dots_push(stage_at(0), bt_of(0), 0);
      consumers_sync();
      double rb = 1.0;
      for (int j = 0; j < bt_of(0); ++j) rb *= a.rho;
      for (int e = tid; e < rc * PC; e += kChainThreads) {
        const int r = e / PC, c = e - (e / PC) * PC;
        V[vix(r, c)] *= rb;
      }
    }
    long long tacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long tp = clock64();
    auto tick = [&](int k) {
      if (a.dbg) {
        long long now;
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(now)::"memory");
        tacc[k] += now - tp;
        tp = now;
      }
    };
    int cs = 0;  // stage of block t
    for (int t = 0; t < nb; ++t) {
      const int bt = bt_of(t);
      const bool more = t + 1 < nb;
      const int ns = cs + 1 == S ? 0 : cs + 1;  // stage of block t + 1
      if (tid == 0 && more) arm_recv(t + 1);
      if (more) wait_next();
      tick(0);
      consumers_sync();  // V_t complete
      tick(1);
      // (b) lookahead partials of block t+1 → every peer
      if (more) {
        if (!(a.skip & 2)) {
          dots_push(stage_at(ns), bt_of(t + 1), t + 1);
        } else if (tid < G) {  // ablation: push zeros only
          const int par = (t + 1) & (kRecvSlots - 1);
          const uint32_t slot = mapa(smem_u32(recv + (par * kMaxCluster + g) * B * PC), tid);
          const uint32_t rb = mapa(smem_u32(&rbar[par]), tid);
          for (int e = 0; e < bt_of(t + 1) * PC; ++e) st_async_f64(slot + e * 8u, 0.0, rb);
        }
      }
      tick(2);
      // (d) Â_t
      recv_sum(t);
      tick(3);
      consumers_sync();  // Â_t, coef_{t−1} visible; V reads of (b) done
      tick(4);
      const double* xb = stage_at(cs);
      const double* TT = xb + B * RP;
      const double* M = TT + B * B;
      const double* Ub = M + B * B;
      // (a) coef_t = TT Â + M coef_{t−1} + U  — warps 0/1 own row tiles j in [8w, 8w+8),
      //     DMMA m8n8k4 (A = TT/M rows, B = Â / coef_{t−1} columns padded to 8)
      if (SCALAR && !(a.skip & 1)) {
        // thread (j, c): coef = U + Σ_l TT[j][l] Â[l][c] + M[j][l] coef_prev[l][c]
        for (int e = tid; e < bt * PC; e += kChainThreads) {
          const int j = e / PC, c = e - (e / PC) * PC;
          double s0 = Ub[e], s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
          for (int l = 0; l < B; l += 2) {
            s0 = fma(TT[l * B + j], Ahat[l * PC + c], s0);
            s1 = fma(TT[(l + 1) * B + j], Ahat[(l + 1) * PC + c], s1);
            s2 = fma(M[l * B + j], rprev[l * PC + c], s2);
            s3 = fma(M[(l + 1) * B + j], rprev[(l + 1) * PC + c], s3);
          }
          coef[e] = (s0 + s1) + (s2 + s3);
        }
        for (int e = bt * PC + tid; e < B * PC; e += kChainThreads) coef[e] = 0.0;
      } else if (!SCALAR && warp < B / 8 && !(a.skip & 1)) {
        const int gq = lane >> 2, tq = lane & 3, j = warp * 8 + gq;
        double cA[B / 4][2], cR[B / 4][2];  // independent accumulation chains
#pragma unroll
        for (int ks = 0; ks < B / 4; ++ks) {
          const int l = 4 * ks + tq;
          cA[ks][0] = cA[ks][1] = cR[ks][0] = cR[ks][1] = 0.0;
          dmma(cA[ks][0], cA[ks][1], TT[l * B + j], gq < PC ? Ahat[l * PC + gq] : 0.0);
          dmma(cR[ks][0], cR[ks][1], M[l * B + j], gq < PC ? rprev[l * PC + gq] : 0.0);
        }
        double c0 = 2 * tq < PC ? Ub[j * PC + 2 * tq] : 0.0;
        double c1 = 2 * tq + 1 < PC ? Ub[j * PC + 2 * tq + 1] : 0.0;
#pragma unroll
        for (int ks = 0; ks < B / 4; ++ks) {
          c0 += cA[ks][0] + cR[ks][0];
          c1 += cA[ks][1] + cR[ks][1];
        }
        if (2 * tq < PC) coef[j * PC + 2 * tq] = c0;
        if (2 * tq + 1 < PC) coef[j * PC + 2 * tq + 1] = c1;
      }
      tick(5);
      consumers_sync();  // coef_t visible
      tick(6);
      // (c) Ŵ_{t+1} = V_t + X_{B_t} coef_t ; V_{t+1} = ρ^{b_{t+1}} Ŵ_{t+1}   (thread = row)
      const double rn = !more ? 1.0 : (t + 1 == nb - 1 ? rho_last : rho_b);
      if (SCALAR && !(a.skip & 4)) {
        // thread = row: V[c][r] = rn (V[c][r] + Σ_l X_B[l][r] coef[l][c])
        for (int r = tid; r < rc; r += kChainThreads) {
          double w[PC], w2[PC];
#pragma unroll
          for (int c = 0; c < PC; ++c) {
            w[c] = V[c * RP + r];
            w2[c] = 0.0;
          }
#pragma unroll
          for (int l = 0; l < B; l += 2) {
            const double x = xb[l * RP + r], x2 = xb[(l + 1) * RP + r];
#pragma unroll
            for (int c = 0; c < PC; ++c) {
              w[c] = fma(x, coef[l * PC + c], w[c]);
              w2[c] = fma(x2, coef[(l + 1) * PC + c], w2[c]);
            }
          }
#pragma unroll
          for (int c = 0; c < PC; ++c) V[c * RP + r] = (w[c] + w2[c]) * rn;
        }
      } else if (!SCALAR && !(a.skip & 4)) {
        // DMMA: rows in tiles of 8 (M), columns padded to 8 (N), K = the b steps
        const int gq = lane >> 2, tq = lane & 3;
        double bc[B / 4];
#pragma unroll
        for (int ks = 0; ks < B / 4; ++ks) bc[ks] = gq < PC ? coef[(4 * ks + tq) * PC + gq] : 0.0;
        constexpr int WS = kChainThreads / 32, NT = 4;
        const int ntiles = (rc + 7) / 8;
        for (int rt0 = warp; rt0 < ntiles; rt0 += NT * WS) {
          double c[NT][2][2];  // [tile][chain][elem]: two K chains per tile, tiles interleaved
#pragma unroll
          for (int u = 0; u < NT; ++u) {
            const int r = 8 * (rt0 + u * WS) + gq;
            const bool live = rt0 + u * WS < ntiles && r < rc;
            c[u][0][0] = live && 2 * tq < PC ? V[r * PC + 2 * tq] : 0.0;
            c[u][0][1] = live && 2 * tq + 1 < PC ? V[r * PC + 2 * tq + 1] : 0.0;
            c[u][1][0] = c[u][1][1] = 0.0;
          }
#pragma unroll
          for (int ks = 0; ks < B / 4; ++ks)
#pragma unroll
            for (int u = 0; u < NT; ++u) {
              const int r = 8 * (rt0 + u * WS) + gq;
              const double av = (rt0 + u * WS < ntiles && r < rc) ? xb[(4 * ks + tq) * RP + r] : 0.0;
              dmma(c[u][ks & 1][0], c[u][ks & 1][1], av, bc[ks]);
            }
#pragma unroll
          for (int u = 0; u < NT; ++u) {
            const int r = 8 * (rt0 + u * WS) + gq;
            if (rt0 + u * WS < ntiles && r < rc) {
              if (2 * tq < PC) V[r * PC + 2 * tq] = (c[u][0][0] + c[u][1][0]) * rn;
              if (2 * tq + 1 < PC) V[r * PC + 2 * tq + 1] = (c[u][0][1] + c[u][1][1]) * rn;
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[cs]);  // stage t fully consumed (its lookahead use was at t−1)
      for (int e = tid; e < B * PC; e += kChainThreads) rprev[e] = coef[e];
      tick(7);
      cs = ns;
    }
    if (a.dbg && tid == 0) {
      const int cta = blockIdx.y * gridDim.x + blockIdx.x;
      for (int k = 0; k < 8; ++k) a.dbg[cta * 8 + k] = tacc[k];
    }
    consumers_sync();
    const double beta = -expm1(static_cast<double>(a.m) * log1p(a.rho - 1.0)) / (1.0 - a.rho);
    for (int e = tid; e < rc * PC; e += kChainThreads) {
      const int r = e / PC, c = e - (e / PC) * PC;
      if (c < pc) {
        const int64_t o = static_cast<int64_t>(r0 + r) * a.ldw + c0 + c;
        a.W[o] = fma(beta, a.C[o], V[vix(r, c)]);
      }
    }
  }
  cluster.sync();
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


int sm_count_dev() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

constexpr int kBlock = 16;

template <int PC>
size_t chain_smem_bytes(int rows, int stages) {
  return std::max(chain_smem<PC, kBlock>(rows, stages).total, chain_smem<PC, kBlock, true>(rows, stages).total);
}

size_t smem_for(int pc, int rows, int stages) {
  switch (pc) {
    case 1: return chain_smem_bytes<1>(rows, stages);
    case 2: return chain_smem_bytes<2>(rows, stages);
    case 3: return chain_smem_bytes<3>(rows, stages);
    case 4: return chain_smem_bytes<4>(rows, stages);
    case 6: return chain_smem_bytes<6>(rows, stages);
    default: return chain_smem_bytes<8>(rows, stages);
  }
}

int round_pc(int pc) {
  if (pc <= 4) return pc;
  if (pc <= 6) return 6;
  return 8;
}
// next smaller supported PC (round_pc(pc - 1) would map 8 back to 8)
int shrink_pc(int pc) { return pc == 8 ? 6 : (pc == 6 ? 4 : std::max(1, pc - 1)); }

}  // namespace

int slab_head(const EpochConfig& cfg) { return (cfg.la == 2 ? 3 : 2) * kBlock * kBlock; }

size_t xg_slot_elems(const EpochConfig& cfg) {  // doubles; x 2 for the 16-byte flag-in-data cells
  if (cfg.nclusters > 1) return 2 * static_cast<size_t>(kXgSlots) * cfg.nclusters * cfg.cluster * kBlock * cfg.pc;
  return cfg.xg ? 2 * static_cast<size_t>(kXgSlots) * cfg.groups * cfg.cluster * kBlock * cfg.pc : 0;
}
size_t xg_count_elems(const EpochConfig& cfg) { return cfg.xg ? static_cast<size_t>(kXgSlots) * cfg.groups : 0; }

int64_t epoch_slab_len(const EpochConfig& cfg) {
  return slab_head(cfg) + static_cast<int64_t>(kBlock) * cfg.pc * cfg.groups;
}

size_t epoch_slab_elems(int64_t m, const EpochConfig& cfg) {
  return static_cast<size_t>(ceil_div(m, kBlock)) * epoch_slab_len(cfg);
}

// U_t[j][c] = ρ^{b−1−j} Σ_l T_jl q_l[c] with q_l = ηn((ρ^l β_t + γ_l) H[i_l][c] − Y[i_l][c]).
// Since TT_jl = ρ^{b−1−j} T_jl ηn ρ^l:  U_t[j][c] = Σ_l TT_jl q'_l[c],
// q'_l = (β_t + γ_l / ρ^l) H[i_l][c] − Y[i_l][c] / ρ^l.   One CTA per block.
constexpr int kBlockUThreads = 128;
__global__ void __launch_bounds__(kBlockUThreads) k_block_u(EpochArgs a) {
  constexpr int B = kBlock;
  __shared__ double q[B][kMaxP];
  __shared__ double TTs[B * B];
  __shared__ double rinv[B], gr[B];
  const int64_t nblocks = (a.m + B - 1) / B;
  if (threadIdx.x == 0) {
    double rp = 1.0, gm = 0.0;
    for (int l = 0; l < B; ++l) {
      rinv[l] = 1.0 / rp;
      gr[l] = gm / rp;
      gm += rp;
      rp *= a.rho;
    }
  }
  const double one_minus_rho = 1.0 - a.rho;
  const double lr = log1p(a.rho - 1.0);
  for (int64_t t = blockIdx.x; t < nblocks; t += gridDim.x) {
    __syncthreads();
    const int64_t s0 = t * B;
    const int bt = static_cast<int>(a.m - s0 < B ? a.m - s0 : B);
    const double beta = -expm1(static_cast<double>(s0) * lr) / one_minus_rho;
    double* slab = a.slab + t * a.slab_len;
    for (int e = threadIdx.x; e < B * B; e += kBlockUThreads) TTs[e] = slab[e];  // transposed: TT[l*B + j]
    for (int e = threadIdx.x; e < B * a.p; e += kBlockUThreads) {
      const int l = e / a.p, c = e - (e / a.p) * a.p;
      double v = 0.0;
      if (l < bt) {
        const int64_t i = a.idx[s0 + l];
        v = fma(beta + gr[l], a.H[i * a.ldy + c], -a.Y[i * a.ldy + c] * rinv[l]);
      }
      q[l][c] = v;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < B * a.groups * a.pc; e += kBlockUThreads) {
      const int grp = e / (B * a.pc), rem = e - grp * (B * a.pc);
      const int j = rem / a.pc, cc = rem - (rem / a.pc) * a.pc;
      const int c = grp * a.pc + cc;
      double s = 0.0;
      if (j < bt && c < a.p) {
#pragma unroll
        for (int l = 0; l < B; ++l) s = fma(TTs[l * B + j], q[l][c], s);
      }
      slab[a.slab_head + e] = s;
    }
  }
}

void launch_block_u(const EpochArgs& a, const EpochConfig& cfg, cudaStream_t st) {
  EpochArgs args = a;
  args.pc = cfg.pc;
  args.groups = cfg.groups;
  args.slab_len = epoch_slab_len(cfg);
  args.slab_head = slab_head(cfg);
  const int64_t nblocks = ceil_div(a.m, kBlock);
  const int grid = static_cast<int>(std::min<int64_t>(nblocks, sm_count_dev() * 16));
  k_block_u<<<grid, kBlockUThreads, 0, st>>>(args);
  GAPLRA_LAUNCH_CHECK();
}

void launch_block_prep(const EpochArgs& a, const EpochConfig& cfg, cudaStream_t st) {
  if (a.p > kMaxP) throw Error(kContractViolation, "epoch: p > 64");
  EpochArgs args = a;
  args.pc = cfg.pc;
  args.groups = cfg.groups;
  args.slab_len = epoch_slab_len(cfg);
  args.slab_head = slab_head(cfg);
  const int64_t nblocks = ceil_div(a.m, kBlock);
  const int grid = static_cast<int>(std::min<int64_t>(nblocks, sm_count_dev() * kPrepCtas));
  constexpr size_t smem1 = prep_ring_bytes<1>() + prep_red_bytes<1>();
  constexpr size_t smem2 = prep_ring_bytes<2>() + prep_red_bytes<2>();
  static const bool attr = [] {
    GAPLRA_CUDA_CHECK(cudaFuncSetAttribute(k_block_prep<kBlock, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem1)));
    GAPLRA_CUDA_CHECK(cudaFuncSetAttribute(k_block_prep<kBlock, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem2)));
    return true;
  }();
  (void)attr;
  if (cfg.la == 2)
    k_block_prep<kBlock, 2><<<grid, kPrepThreads + 32 * kPrepProducers, smem2, st>>>(args);
  else
    k_block_prep<kBlock, 1><<<grid, kPrepThreads + 32 * kPrepProducers, smem1, st>>>(args);
  GAPLRA_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
// k_svrg_chain_v3: warp-specialised chain, the form measured fastest with
// tools/chain_skeleton.cu (p = 1: 1408 vs 1903 cycles per block for the
// 8-consumer form).  7 warps:
//   warps 0..3  rows: thread = rows 2·tid, 2·tid+1 (LDS.128 per slice),
//               V in registers; per block t: load block t+1's slice rows,
//               products with V_t, select-free warp halving, red; barrier
//               (rows); push Â_{t+1} (16-byte st.async); wait coef_t; update
//   warp 4      reducer: wait Â_t, fixed-order slot sum, coef_t = TT_t Â_t +
//               pre_t, signal the rows, then pre_{t+1} = M_{t+1} coef_t + U_{t+1}
//               — concurrently with the rows' products of block t+1
//   warps 5, 6  producers (8 slices each; warp 5 also the slab part)
// The coef hand-off alternates two named barriers (even / odd blocks), so the
// reducer can never arrive twice on one barrier phase.
// ---------------------------------------------------------------------------
// GAPLRA_EPOCH_TIMING: clock stamps of one all-reduce loop (blocks 1000..1007 of CTA 0), per hop:
// 0 rows: products done, 1 pusher: woken, 2 pusher: copies issued, 3 reducer: all partials in,
// 4 reducer: coef handed to the rows, 5 rows: coef received (update starts)
// Compiled in only with -DGAPLRA_HOP_TIMING: in the default build the stamps' clock reads (asm volatile with
// a memory clobber) sat in the rows' hot loop and cost the C3 p = 1 chain 13 %.
__device__ long long g_hop[8 * 8];
__device__ __forceinline__ void hop_stamp(const EpochArgs& a, int blk, int k) {
#ifdef GAPLRA_HOP_TIMING
  if (a.dbg && blockIdx.x == 0 && blockIdx.y == 0 && blk >= 1000 && blk < 1008) {
    long long now;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(now)::"memory");
    g_hop[(blk - 1000) * 8 + k] = now;
  }
#else
  (void)a;
  (void)blk;
  (void)k;
#endif
}
constexpr int kV3Rows = 4;       // row warps
// producer warps: 4 at PC = 1 (each issues its lanes' bulk copies one after
// another, so more warps raise the feed; PC > 1 needs the registers)
__host__ __device__ constexpr int v3_producers(int pc) { return pc == 1 ? V3_PROD1 : 2; }
// reducer warps: 2 once the block has more than 32 entries per column group
// (they split the entries; measured p = 20 / PC = 3: one reducer warp was busy
// 2818 of 2900 cycles per block)
__host__ __device__ constexpr int v3_reducers(int pc) { return pc >= 2 ? 2 : 1; }
// + one push warp: sums the row warps' partials and bulk-copies Â_{t+1} to the
// peers, so the rows go straight from products(t+1) to update(t)
__host__ __device__ constexpr int v3_threads(int pc) { return 32 * (kV3Rows + v3_reducers(pc) + 1 + v3_producers(pc)); }
// RR layout (PC = 1, 256 rows): three warpgroups — rows (warps 0-3, registers
// raised to 232 by setmaxnreg), reducer + pusher + 2 idle (warps 4-7), four
// producers (warps 8-11, lowered to 40) — so four producer warps feed the ring
// without capping the rows' register-resident update
constexpr int kV3RRThreads = 384;
template <bool RR>
__host__ __device__ constexpr int v3_block(int pc) { return RR ? kV3RRThreads : v3_threads(pc); }
// layouts the warp-specialised chain runs: 256 rows per CTA (H = 1, PC <= 3) or
// 512 rows (H = 2, PC = 1: only there do three 512-row stages fit beside the
// receive slots; with two, the stage re-read by the update would stall the ring)
inline bool v3_supports(int pc, int rows) { return pc <= 3 && (rows <= 256 || (rows <= 512 && pc == 1)); }

// H: 256-row halves per row thread (rows 2·tid + {0,1} + 256·h): 256·H rows per CTA.
// XG: plain CTAs (gridDim.x of them) exchanging the partials through L2
// instead of a DSMEM cluster, so the rows spread over more SMs than a cluster
// holds (p = 1: 128 rows per CTA, 32 CTAs at C2, 64 at C5).
template <int PC, int B, int H = 1, bool RR = false, bool XG = false>
__global__ void __launch_bounds__(v3_block<RR>(PC), 1) k_svrg_chain_v3(EpochArgs a) {
  static_assert(B == 16, "lane permutation j = i ^ (lane >> 1) covers 16 slices");
  static_assert(!RR || PC == 1, "RR layout: PC = 1");
  static_assert(!XG || (PC == 1 && RR), "L2 exchange: the p = 1 RR layout");
  constexpr int NPROD = RR ? 4 : v3_producers(PC);
  constexpr bool XREG = PC == 1 && H == 1;  // update from the products' registers (else re-read the stage)
  extern __shared__ __align__(128) double sm[];
  const int G = XG ? static_cast<int>(gridDim.x) : static_cast<int>(cg::this_cluster().num_blocks());
  const int g = XG ? static_cast<int>(blockIdx.x) : static_cast<int>(cg::this_cluster().block_rank());
  // PAIRED clusters (p = 1, a.ncl == 2): the rows are split over two clusters; each cluster all-reduces over
  // DSMEM as usual, then CTA g of one cluster swaps its cluster sum with CTA g of the other through L2
  // (flag-in-data cells, one writer and one reader per cell: no hot line), and adds them in cluster order.
  const int ncl = XG ? 1 : a.ncl;
  const int cl = ncl > 1 ? static_cast<int>(blockIdx.x) / G : 0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NV = B * PC;
  double* xg_slots = XG ? a.xg_slot : nullptr;  // [kXgSlots][G][NV]
  unsigned* xg_cnt = XG ? a.xg_count : nullptr;
  constexpr int NRD = v3_reducers(PC);
  constexpr int EPW = (NV + NRD - 1) / NRD;  // entries per reducer warp
  static_assert(EPW <= 32, "one entry per reducer lane");
  const int grp = blockIdx.y;
  const int c0 = grp * PC;
  const int pc = min(PC, a.p - c0);
  const ChainSmem L = chain_smem<PC, B, true>(a.rows_per_cta, a.stages);
  static_assert(2 * kV3Rows * NV + 6 * NV <= kChainThreads / 32 * (B / 8) * 64, "red[2] + coef + ahat + pre + outv fit");
  const int S = L.stages;
  const int r0 = (cl * G + g) * a.rows_per_cta;
  const int rc = max(0, min(a.rows_per_cta, a.d_pad - r0));
  const int RP = L.rows_pad;
  double* recv = sm + L.off_recv;  // [kRecvSlots][kMaxCluster][NV]
  double* red = sm + L.off_red;    // [2][kV3Rows][NV] (block parity)
  double* coef = red + 2 * kV3Rows * NV;  // [2][NV]
  double* Ahat = coef + 2 * NV;       // [NV]
  double* pre = Ahat + NV;            // [NV]
  double* outv = pre + NV;            // [2][NV] this CTA's summed partials, bulk-copied to every peer
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + L.off_bar);  // [S <= 4]
  uint64_t* empty = full + 8;                                     // [S <= 8]
  uint64_t* rbar = full + 16;                                      // [kRecvSlots]
  auto stage_at = [&](int s_idx) { return sm + L.off_stage + static_cast<size_t>(s_idx) * L.stage_len; };
  const int nb = static_cast<int>((a.m + B - 1) / B);
  const int last_bt = static_cast<int>(a.m - static_cast<int64_t>(nb - 1) * B);
  auto bt_of = [&](int t) { return t == nb - 1 ? last_bt : B; };
  double rho_b = 1.0, rho_last = 1.0;
  for (int j = 0; j < B; ++j) rho_b *= a.rho;
  for (int j = 0; j < last_bt; ++j) rho_last *= a.rho;
#pragma unroll 1
  for (size_t e = tid; e < L.off_v; e += blockDim.x) sm[e] = 0.0;  // pad rows / unwritten slices read as 0
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], NPROD);
      mbar_init(&empty[s], kV3Rows + NRD);
    }
    for (int q = 0; q < kRecvSlots; ++q) mbar_init(&rbar[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if constexpr (XG)
    __syncthreads();
  else
    cg::this_cluster().sync();
  // GAPLRA_EPOCH_TIMING: cycles per block; rows (tid 0) in slots 0..5, reducer (lane 0) in 6..7
  long long tacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tp;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(tp)::"memory");
  auto tick = [&](int kk) {
#ifdef GAPLRA_V3_TICKS  // the p <= 3 chain's phase ticks: off by default (3 % on the p = 1 chain)
    if (a.dbg) {
      long long now;
      asm volatile("mov.u64 %0, %%clock64;" : "=l"(now)::"memory");
      tacc[kk] += now - tp;
      tp = now;
    }
#else
    (void)kk;
#endif
  };

  constexpr int kFirstProd = RR ? 8 : kV3Rows + NRD + 1;
  if (warp >= kFirstProd) {  // ------------------------------------------- producers
    if constexpr (RR) asm volatile("setmaxnreg.dec.sync.aligned.u32 40;" ::: "memory");
    chain_produce<PC, B, NPROD>(a, warp - kFirstProd, lane, nb, last_bt, S, rc, r0, RP, grp, sm + L.off_stage,
                                L.stage_len, full, empty);
  } else if (RR && warp > kV3Rows + NRD) {  // ----------------------------- idle (RR)
  } else if (warp == kV3Rows + NRD) {  // ---------------------------------- pusher
    // Â_u: wait for the rows' red(u) (named barrier 5 / 6 by parity; the rows
    // cannot arrive for u + 2 first, since products(u + 2) follows update(u),
    // which needs Â_u from every peer, this one included), fixed-order sum of
    // the 4 warp partials into outv[u & 1], one bulk copy per peer
    for (int u = 0; u < nb; ++u) {
      if (u & 1)
        asm volatile("bar.sync 6, %0;" ::"n"(32 * (kV3Rows + 1)) : "memory");
      else
        asm volatile("bar.sync 5, %0;" ::"n"(32 * (kV3Rows + 1)) : "memory");
      if (lane == 0) hop_stamp(a, u, 1);
      if (!XG && lane < G && !(PC == 1 && a.push_async)) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      __syncwarp();
      const double* rb = red + (u & 1) * kV3Rows * NV;
      double* ov = outv + (u & 1) * NV;
      if constexpr (XG) {
        if (a.xg_ll) {  // one flag-in-data cell per entry: no fence, no counter
          uint4* dst = reinterpret_cast<uint4*>(xg_slots) + (static_cast<size_t>(u % kXgSlots) * G + g) * NV;
          for (int e = lane; e < NV; e += 32)
            ll_store(dst + e, (rb[e] + rb[NV + e]) + (rb[2 * NV + e] + rb[3 * NV + e]),
                     static_cast<uint32_t>(u / kXgSlots + 1));
          continue;
        }
        // partial -> L2 slot, then one release-increment
        double* dst = xg_slots + (static_cast<size_t>(u % kXgSlots) * G + g) * NV;
        for (int e = lane; e < NV; e += 32) st_cg(dst + e, (rb[e] + rb[NV + e]) + (rb[2 * NV + e] + rb[3 * NV + e]));
        __syncwarp();
        if (lane == 0) xg_publish(xg_cnt + u % kXgSlots);
        continue;
      }
      if constexpr (PC == 1) {
        // p = 1: 16 entries.  Each half-warp sums entry e = lane & 15 and stores it straight from the register
        // into every second peer's receive slot (st.async: the store itself completes 8 bytes on the peer's
        // barrier).  The staged bulk copy (sum -> shared -> fence.proxy.async -> one copy per peer) took ~1400
        // cycles from the pusher's wake-up to the copies being issued.
        if (a.push_async) {
          const int e = lane & 15, par = u & (kRecvSlots - 1);
          const double sum = (rb[e] + rb[NV + e]) + (rb[2 * NV + e] + rb[3 * NV + e]);
          const uint32_t dst = smem_u32(recv + (par * kMaxCluster + g) * NV + e), bar = smem_u32(&rbar[par]);
          for (int q = lane >> 4; q < G; q += 2) st_async_f64(mapa(dst, q), sum, mapa(bar, q));
          if (lane == 0) hop_stamp(a, u, 2);
          continue;
        }
      }
      for (int e = lane; e < NV; e += 32) ov[e] = (rb[e] + rb[NV + e]) + (rb[2 * NV + e] + rb[3 * NV + e]);
      fence_proxy_async();
      __syncwarp();
      if (lane < G) {
        const int par = u & (kRecvSlots - 1);
        dsmem_bulk_copy(mapa(smem_u32(recv + (par * kMaxCluster + g) * NV), lane), smem_u32(ov), NV * 8u,
                        mapa(smem_u32(&rbar[par]), lane));
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      if (lane == 0) hop_stamp(a, u, 2);
    }
    if (!XG && lane < G) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  } else if (warp >= kV3Rows) {  // ------------------------------------------ reducers
    const int rw = warp - kV3Rows;
    const int me = rw * EPW + lane;  // this lane's entry
    const bool mine = lane < EPW && me < NV;
    auto red_sync = [&]() {
      if constexpr (NRD > 1)
        asm volatile("bar.sync 4, %0;" ::"n"(32 * NRD) : "memory");
      else
        __syncwarp();
    };
    auto arm = [&](int u) {
      if (!XG && rw == 0 && lane == 0)
        mbar_expect_tx(&rbar[u & (kRecvSlots - 1)], static_cast<uint32_t>(G * NV * 8));  // full vectors
    };
    bool fast_done = false;
    if constexpr (PC == 1 && !XG) {
      if (a.ncl == 1 && a.fast_reducer) {
        fast_done = true;
        // p = 1, one cluster: the reducer warp is the chain's critical resource (the rows waited at the coef
        // barrier a third of the time), so everything that does not depend on Â_t is in registers BEFORE the
        // wait: this lane's columns of TT_t and M_{t+1} and U_{t+1}.  After the wait: 16 batched peer loads,
        // one shared round trip for Â, 16 FMAs -> coef_t to the rows; then pre_{t+1} from coef_t.  Same
        // sums, fixed orders of their own (results differ from the generic path below in the last bits).
        // lane = (entry e = lane & 15, half h = lane >> 4): the two half-warps split the peers of the sum and the
        // l-range of both matvecs (8 products each, joined by one shuffle), which halves the warp's shared loads
        const int e = lane & 15, h = lane >> 4, l0 = 8 * h;
        constexpr int HB = B / 2;
        double TTc[HB], Mn[HB], pre_r = 0.0;
        auto load_col = [&](const double* src, double (&dst)[HB]) {
#pragma unroll
          for (int l = 0; l < HB; ++l) dst[l] = src[(l0 + l) * B + e];
        };
        auto join = [](double v) { return v + __shfl_xor_sync(0xffffffffu, v, 16); };
        if (nb > 0) {
          arm(0);
          mbar_wait(&full[0], 0);
          const double* sl0 = stage_at(0) + B * RP;
          load_col(sl0, TTc);
          pre_r = sl0[2 * B * B + e];
        }
        int cs = 0;
        uint32_t cph = 0;
#pragma unroll 1
        for (int t = 0; t < nb; ++t) {
          const bool more = t + 1 < nb;
          const int ns = cs + 1 == S ? 0 : cs + 1;
          const uint32_t nph = ns == 0 ? cph ^ 1u : cph;
          if (more) arm(t + 1);
          const int par = t & (kRecvSlots - 1);
          double Un = 0.0;
          if (more) {  // stage t + 1 is complete (the rows' products of t + 1 ran before their update of t)
            mbar_wait(&full[ns], nph);
            const double* sn = stage_at(ns) + B * RP;
            load_col(sn + B * B, Mn);
            Un = sn[2 * B * B + e];
          }
          tick(7);
          const int nv = bt_of(t);
          mbar_wait(&rbar[par], static_cast<uint32_t>((t >> 2) & 1));
          tick(6);
          if (lane == 0) hop_stamp(a, t, 3);
          double sv;
          {
            // half h sums peers h G/2 .. (h + 1) G/2 - 1 in a fixed tree; total = lower + upper
            const int gh = G >> 1;
            const double* sl = recv + par * kMaxCluster * NV + h * gh * NV + e;
            double x[kMaxCluster / 2];
#pragma unroll
            for (int q = 0; q < kMaxCluster / 2; ++q) x[q] = q < gh ? sl[q * NV] : 0.0;
            const double part = ((x[0] + x[1]) + (x[2] + x[3])) + ((x[4] + x[5]) + (x[6] + x[7]));
            sv = join(e < nv ? part : 0.0);  // (the shuffle outside the select: every lane takes part)
          }
          if (h == 0) Ahat[e] = sv;
          __syncwarp();
          double* cf = coef + (t & 1) * NV;
          double cv;
          {
            double s0 = 0.0, s1 = 0.0;
#pragma unroll
            for (int l = 0; l < HB; l += 2) {
              s0 = fma(TTc[l], Ahat[l0 + l], s0);
              s1 = fma(TTc[l + 1], Ahat[l0 + l + 1], s1);
            }
            cv = pre_r + join(s0 + s1);
          }
          if (h == 0) cf[e] = cv;
          if (t & 1)
            asm volatile("bar.arrive 3, %0;" ::"n"(32 * (kV3Rows + NRD)) : "memory");
          else
            asm volatile("bar.arrive 2, %0;" ::"n"(32 * (kV3Rows + NRD)) : "memory");
          __syncwarp();
          if (lane == 0) {
            hop_stamp(a, t, 4);
            mbar_arrive(&empty[cs]);  // TT_t (in registers since before the wait): the stage is free for the reducer
          }
          if (more) {
            double s0 = 0.0, s1 = 0.0;
#pragma unroll
            for (int l = 0; l < HB; l += 2) {
              s0 = fma(Mn[l], cf[l0 + l], s0);
              s1 = fma(Mn[l + 1], cf[l0 + l + 1], s1);
            }
            pre_r = Un + join(s0 + s1);
            load_col(stage_at(ns) + B * RP, TTc);  // TT_{t+1}
          }
          cs = ns;
          cph = nph;
        }
        if (a.dbg && lane == 0) {
          const int cta = blockIdx.y * gridDim.x + blockIdx.x;
          for (int kk = 6; kk < 8; ++kk) a.dbg[cta * 8 + kk] = tacc[kk];
        }
      }
    }
    if (!fast_done) {
    if (nb > 0) {
      arm(0);
      mbar_wait(&full[0], 0);
      const double* Ub = stage_at(0) + B * RP + 2 * B * B;
      if (mine) pre[me] = Ub[me];
    }
    int cs = 0;
    uint32_t cph = 0;  // full-barrier parity of stage cs
#pragma unroll 1
    for (int t = 0; t < nb; ++t) {
      const bool more = t + 1 < nb;
      const int ns = cs + 1 == S ? 0 : cs + 1;
      const uint32_t nph = ns == 0 ? cph ^ 1u : cph;
      if (more) arm(t + 1);
      const int par = t & (kRecvSlots - 1);
      tick(7);
      const int nv = bt_of(t) * PC;
      if constexpr (XG) {
       if (a.xg_ll) {
        const double sv = ll_gather16(reinterpret_cast<const uint4*>(xg_slots) + static_cast<size_t>(t % kXgSlots) * G * NV,
                                      G, lane, static_cast<uint32_t>(t / kXgSlots + 1));
        tick(6);
        if (lane < 16) Ahat[lane] = lane < nv ? sv : 0.0;
        __syncwarp();
       } else {
        // NV = 16 entries; lane e and e + 16 split the peers (q mod 4 in {0,1} / {2,3}),
        // (s0 + s1) + (s2 + s3) in the same order as the DSMEM form
        if (lane == 0) xg_wait(xg_cnt + t % kXgSlots, static_cast<unsigned>(G) * (t / kXgSlots + 1));
        __syncwarp();
        tick(6);
        const int e = lane & 15, hq = (lane >> 4) * 2;
        const double* sl = xg_slots + static_cast<size_t>(t % kXgSlots) * G * NV + e;
        double sa = 0.0, sb = 0.0;
#pragma unroll 4
        for (int q = 0; q < G; q += 4) {
          sa += ld_cg(sl + (q + hq) * NV);
          sb += ld_cg(sl + (q + hq + 1) * NV);
        }
        double sv = sa + sb;
        const double other = __shfl_down_sync(0xffffffffu, sv, 16);
        if (lane < 16) Ahat[e] = e < nv ? sv + other : 0.0;
        __syncwarp();
       }
      } else {
        mbar_wait(&rbar[par], static_cast<uint32_t>((t >> 2) & 1));
        tick(6);
        if (rw == 0 && lane == 0) hop_stamp(a, t, 3);
      }
      if (!XG && mine) {
        const int e = me;
        double s = 0.0;
        if (e < nv) {
          const double* sl = recv + par * kMaxCluster * NV + e;
          double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll 1
          for (int q = 0; q < G; q += 4) {
            s0 += sl[q * NV];
            s1 += sl[(q + 1) * NV];
            s2 += sl[(q + 2) * NV];
            s3 += sl[(q + 3) * NV];
          }
          s = (s0 + s1) + (s2 + s3);
        }
        if constexpr (PC == 1) {
          if (ncl == 2) {  // swap cluster sums with the partner CTA (same rank, other cluster)
            const uint32_t flag = static_cast<uint32_t>(t / kXgSlots + 1);
            uint4* cells = reinterpret_cast<uint4*>(a.xg_slot) + static_cast<size_t>(t % kXgSlots) * 2 * G * NV;
            ll_store(cells + (cl * G + g) * NV + e, s, flag);
            const uint4* theirs = cells + ((cl ^ 1) * G + g) * NV + e;
            uint4 w = ll_load(theirs);
            while (w.y != flag || w.w != flag) w = ll_load(theirs);
            const double o = __hiloint2double(static_cast<int>(w.z), static_cast<int>(w.x));
            s = cl == 0 ? s + o : o + s;
          }
        }
        Ahat[e] = s;
      }
      red_sync();  // Â_t complete
      const double* TT = stage_at(cs) + B * RP;
      double* cf = coef + (t & 1) * NV;
      if (mine) {
        const int e = me;
        const int j = e / PC, c = e - (e / PC) * PC;
        double s0 = pre[e], s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
        for (int l = 0; l < B; l += 4) {
          s0 = fma(TT[l * B + j], Ahat[l * PC + c], s0);
          s1 = fma(TT[(l + 1) * B + j], Ahat[(l + 1) * PC + c], s1);
          s2 = fma(TT[(l + 2) * B + j], Ahat[(l + 2) * PC + c], s2);
          s3 = fma(TT[(l + 3) * B + j], Ahat[(l + 3) * PC + c], s3);
        }
        cf[e] = (s0 + s1) + (s2 + s3);
      }
      // coef_t ready for the rows (even / odd barrier)
      if (t & 1)
        asm volatile("bar.arrive 3, %0;" ::"n"(32 * (kV3Rows + NRD)) : "memory");
      else
        asm volatile("bar.arrive 2, %0;" ::"n"(32 * (kV3Rows + NRD)) : "memory");
      __syncwarp();
      if (rw == 0 && lane == 0) hop_stamp(a, t, 4);
      if (lane == 0) mbar_arrive(&empty[cs]);  // TT_t was the reducers' last use of stage t
      if (more) {  // pre_{t+1} = M_{t+1} coef_t + U_{t+1}
        red_sync();  // coef_t complete (the other reducer's half); its Â reads done
        mbar_wait(&full[ns], nph);
        const double* M = stage_at(ns) + B * RP + B * B;
        const double* Ub = M + B * B;
        if (mine) {
          const int e = me;
          const int j = e / PC, c = e - (e / PC) * PC;
          double s0 = Ub[e], s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
          for (int l = 0; l < B; l += 4) {
            s0 = fma(M[l * B + j], cf[l * PC + c], s0);
            s1 = fma(M[(l + 1) * B + j], cf[(l + 1) * PC + c], s1);
            s2 = fma(M[(l + 2) * B + j], cf[(l + 2) * PC + c], s2);
            s3 = fma(M[(l + 3) * B + j], cf[(l + 3) * PC + c], s3);
          }
          pre[e] = (s0 + s1) + (s2 + s3);
        }
        __syncwarp();
      }
      cs = ns;
      cph = nph;
    }
    if (a.dbg && lane == 0 && rw == 0) {
      const int cta = blockIdx.y * gridDim.x + blockIdx.x;
      for (int kk = 6; kk < 8; ++kk) a.dbg[cta * 8 + kk] = tacc[kk];
    }
    }  // !fast_done
  } else {  // --------------------------------------------------------------- rows
    if constexpr (RR) asm volatile("setmaxnreg.inc.sync.aligned.u32 232;" ::: "memory");
    const int pm = lane >> 1;  // product order j = i ^ pm
    const int ra = 2 * tid;    // rows ra + 256 h, ra + 1 + 256 h
    bool own0[H], own1[H];
    double v0[H][PC], v1[H][PC];
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const int rh = ra + 256 * h;
      own0[h] = rh < rc;
      own1[h] = rh + 1 < rc;
#pragma unroll
      for (int c = 0; c < PC; ++c) {
        v0[h][c] = own0[h] && c < pc ? a.W[static_cast<int64_t>(r0 + rh) * a.ldw + c0 + c] : 0.0;
        v1[h][c] = own1[h] && c < pc ? a.W[static_cast<int64_t>(r0 + rh + 1) * a.ldw + c0 + c] : 0.0;
      }
    }
    int ws = 0;
    uint32_t wph = 0;
    auto wait_stage = [&]() {  // blocks are waited for in order 0, 1, 2, ...
      mbar_wait(&full[ws], wph);
      const int s = ws;
      if (++ws == S) {
        ws = 0;
        wph ^= 1u;
      }
      return s;
    };
    auto load_rows = [&](const double* xb, double2 (&xr)[H][B]) {
#pragma unroll
      for (int h = 0; h < H; ++h)
#pragma unroll
        for (int i = 0; i < B; ++i)
          xr[h][i] = *reinterpret_cast<const double2*>(xb + (i ^ pm) * RP + ra + 256 * h);
    };
    auto products = [&](const double2 (&xr)[H][B], int u) {
      double val[B][PC];
#pragma unroll
      for (int i = 0; i < B; ++i)
#pragma unroll
        for (int c = 0; c < PC; ++c) {
          double sv = fma(xr[0][i].x, v0[0][c], xr[0][i].y * v1[0][c]);
#pragma unroll
          for (int h = 1; h < H; ++h) sv = fma(xr[h][i].x, v0[h][c], fma(xr[h][i].y, v1[h][c], sv));
          val[i][c] = sv;
        }
#pragma unroll
      for (int o = 16, n = B / 2; o >= 2; o >>= 1, n >>= 1)
#pragma unroll
        for (int i = 0; i < n; ++i)
#pragma unroll
          for (int c = 0; c < PC; ++c) val[i][c] += __shfl_xor_sync(0xffffffffu, val[i + n][c], o);
#pragma unroll
      for (int c = 0; c < PC; ++c) val[0][c] += __shfl_xor_sync(0xffffffffu, val[0][c], 1);
      double* rb = red + (u & 1) * kV3Rows * NV;
      if (!(lane & 1))
#pragma unroll
        for (int c = 0; c < PC; ++c) rb[warp * NV + pm * PC + c] = val[0][c];
      if (u & 1)  // red(u) complete for the pusher (barrier 5 / 6 by parity)
        asm volatile("bar.arrive 6, %0;" ::"n"(32 * (kV3Rows + 1)) : "memory");
      else
        asm volatile("bar.arrive 5, %0;" ::"n"(32 * (kV3Rows + 1)) : "memory");
      if (tid == 0) hop_stamp(a, u, 0);
    };
    auto update = [&](const double2 (&xr)[H][B], int t, double rn) {
      if (t & 1)
        asm volatile("bar.sync 3, %0;" ::"n"(32 * (kV3Rows + NRD)) : "memory");
      else
        asm volatile("bar.sync 2, %0;" ::"n"(32 * (kV3Rows + NRD)) : "memory");
      tick(4);
      if (tid == 0) hop_stamp(a, t, 5);
      const double* cf = coef + (t & 1) * NV;
#pragma unroll
      for (int h = 0; h < H; ++h) {
        double a0[PC], a1[PC];
#pragma unroll
        for (int c = 0; c < PC; ++c) a0[c] = a1[c] = 0.0;
#pragma unroll
        for (int i = 0; i < B; i += 2)
#pragma unroll
          for (int c = 0; c < PC; ++c) {
            const double k0 = cf[(i ^ pm) * PC + c], k1 = cf[((i + 1) ^ pm) * PC + c];
            v0[h][c] = fma(xr[h][i].x, k0, v0[h][c]);
            v1[h][c] = fma(xr[h][i].y, k0, v1[h][c]);
            a0[c] = fma(xr[h][i + 1].x, k1, a0[c]);
            a1[c] = fma(xr[h][i + 1].y, k1, a1[c]);
          }
#pragma unroll
        for (int c = 0; c < PC; ++c) {
          v0[h][c] = own0[h] ? (v0[h][c] + a0[c]) * rn : 0.0;
          v1[h][c] = own1[h] ? (v1[h][c] + a1[c]) * rn : 0.0;
        }
      }
    };
    double2 xa[H][B], xn[H][B];
    if (nb > 0) {  // Â_0 = X_{B_0}ᵀ Ŵ_0, then V_0 = ρ^{b_0} Ŵ_0
      const int s = wait_stage();
      load_rows(stage_at(s), xa);
      if (!XREG) {
        // stage 0 stays until its update; released below
      } else {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
      products(xa, 0);
      double rb = 1.0;
      for (int j = 0; j < bt_of(0); ++j) rb *= a.rho;
#pragma unroll
      for (int h = 0; h < H; ++h)
#pragma unroll
        for (int c = 0; c < PC; ++c) {
          v0[h][c] *= rb;
          v1[h][c] *= rb;
        }
    }
    // block t: products of t+1 (stage ns) then the update of t
    auto step = [&](int t, double2 (&xr)[H][B], double2 (&xq)[H][B]) {
      const bool more = t + 1 < nb;
      if (more) {
        tick(5);
        const int s = wait_stage();
        tick(0);
        load_rows(stage_at(s), xq);
        if (XREG) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[s]);
        }
        products(xq, t + 1);
        tick(1);
      }
      const double rn = !more ? 1.0 : (t + 1 == nb - 1 ? rho_last : rho_b);
      if (XREG) {
        update(xr, t, rn);
      } else {
        const int cs = t % S;
        double2 xt[H][B];
        load_rows(stage_at(cs), xt);
        update(xt, t, rn);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[cs]);
      }
      // the next products' red writes follow the coef barrier, which every row
      // thread passes after its push reads
    };
    if (XREG) {
      int t = 0;
#pragma unroll 1
      for (; t + 1 < nb; t += 2) {
        step(t, xa, xn);
        step(t + 1, xn, xa);
      }
      if (t < nb) step(t, xa, xn);
    } else {
#pragma unroll 1
      for (int t = 0; t < nb; ++t) step(t, xa, xn);
    }
    if (a.dbg && tid == 0) {
      const int cta = blockIdx.y * gridDim.x + blockIdx.x;
      for (int kk = 0; kk < 6; ++kk) a.dbg[cta * 8 + kk] = tacc[kk];
    }
    const double beta = -expm1(static_cast<double>(a.m) * log1p(a.rho - 1.0)) / (1.0 - a.rho);
#pragma unroll
    for (int h = 0; h < H; ++h)
#pragma unroll
      for (int c = 0; c < PC; ++c)
        if (c < pc) {
          const int rh = ra + 256 * h;
          if (own0[h]) {
            const int64_t o = static_cast<int64_t>(r0 + rh) * a.ldw + c0 + c;
            a.W[o] = fma(beta, a.C[o], v0[h][c]);
          }
          if (own1[h]) {
            const int64_t o = static_cast<int64_t>(r0 + rh + 1) * a.ldw + c0 + c;
            a.W[o] = fma(beta, a.C[o], v1[h][c]);
          }
        }
  }
  if constexpr (!XG) cg::this_cluster().sync();
}

// ---------------------------------------------------------------------------
// k_svrg_chain_v4: the chain on the FP64 tensor path for PC = 8 right-hand
// sides per cluster (C2: 3 clusters instead of 7 x PC 3).  Same algebra,
// lookahead and slab as v3; the products and the update are DMMA m8n8k4 in
// the transposed form, with Vᵀ (8 columns x the warp's 64 rows) kept as the
// update's C fragments in registers:
//   update    Vᵀ += coefᵀ X_Bᵀ   M = column, N = rows (8 per tile), K = slices
//   products  Âᵀ = Vᵀ X_B        M = column, N = slices, K = rows; the A
//             fragment of k-step (tile, u) is element u of the tile's C
//             fragment (lane tq <-> row 8 tile + 2 tq + u), so V never leaves
//             the registers
// Slice pitch RP ≡ 4 (mod 16) doubles: the update's LDS.64 B fragments and the
// products' LDS.128 (rows 2tq, 2tq+1, slices permuted 0 2 1 3 4 6 5 7) are
// bank-conflict free; coef is stored [slice][12].  Warps: 8 rows (ROWS / 8
// rows each), 4 reducers (each owns two right-hand-side columns: lane = (column, step), so Â -> coef -> pre
// of a column stay inside one warp and the reducers never wait for each other; measured and rejected: TT / M
// columns preloaded into registers before the all-reduce wait — C2 14.9 vs 14.6 ms, the extra shared loads
// queue behind the row warps' — and both matvecs as DMMAs in one reducer warp — C2 16.7 ms, C5 258 vs 238 ms,
// one warp's dependent DMMA chains are slower than 128 lanes of FMAs), 1 pusher (sums the row
// warps' partials, bulk-copies Â_{t+1} to the 16 peers), 2 producers.
// ROWS = 256 (C2, C3) or 512 (C5: d = 8192 on 16-CTA clusters; a 512-row
// stage is 71 KB, so the ring has 2 stages next to the 64 KB receive slots).
// ---------------------------------------------------------------------------
namespace v4 {
constexpr int PC = 8, B = 16, NV = B * PC;
constexpr int kRows = 8, kRed = 4, kProd = 2;
constexpr int kThreads = 32 * (kRows + kRed + 1 + kProd);
constexpr int CP = 12;  // coef pitch (doubles)
constexpr int RCP = 18;                // red: column-major [c][RCP] partials (pitch 18: the rows' stores are <= 2-way
                                       // conflicted, the pusher's reads along j conflict free)
constexpr int NVR = PC * RCP;          // one row warp's red vector

struct Smem {
  int rp, stages;
  size_t stage_len, off_recv, off_red, off_outv, off_cf, off_ahat, off_pre, off_bar, total;
};
__host__ __device__ inline int span(int rows) { return rows <= 128 ? 128 : (rows <= 256 ? 256 : 512); }
__host__ __device__ inline Smem smem(int rows, int stages, bool xg = false) {
  Smem L;
  L.rp = span(rows) + 4;  // the 8 row warps always span 128, 256 or 512 rows (pad rows are zero)
  L.stages = stages;
  L.stage_len = static_cast<size_t>(B) * L.rp + 2 * B * B + B * PC;
  size_t o = L.stage_len * stages;
  L.off_recv = o;
  if (!xg) o += static_cast<size_t>(kRecvSlots) * kMaxCluster * NV;  // XG: partials arrive through L2
  L.off_red = o;
  o += 2 * kRows * NVR;
  L.off_outv = o;
  o += 2 * NV;
  L.off_cf = o;
  o += 2 * B * CP;
  L.off_ahat = o;
  o += NV;
  L.off_pre = o;
  o += NV;
  L.off_bar = o;
  o += 16;
  L.total = o * sizeof(double);
  return L;
}
// 512-row layout (C5, L2 exchange): a block's 16 slices are two half-stages
// of 8 (33 KB each) in a ring of kHalves, with the slab part (TT | M | U) in
// its own ring of kSlabs.  The update releases a block's first half after its
// first two k-steps, so the ring holds blocks t and t + 1 plus one half in
// flight and the feed overlaps the chain (two 71 KB full stages did not: the
// rows waited ~2000 cycles per block for the refill).
constexpr int kHalves = 5, kSlabs = 3, kSlabLen = 2 * B * B + B * PC;
__host__ __device__ inline Smem smem_half() {
  Smem L;
  L.rp = 512 + 4;
  L.stages = 0;
  L.stage_len = static_cast<size_t>(B / 2) * L.rp;  // one half-stage
  size_t o = L.stage_len * kHalves + static_cast<size_t>(kSlabs) * kSlabLen;
  L.off_recv = o;  // XG only: no receive slots
  L.off_red = o;
  o += 2 * kRows * NVR;
  L.off_outv = o;
  o += 2 * NV;
  L.off_cf = o;
  o += 2 * B * CP;
  L.off_ahat = o;
  o += NV;
  L.off_pre = o;
  o += NV;
  L.off_bar = o;
  o += 24;  // fullH[5] emptyH[5] fullS[3] emptyS[3]
  L.total = o * sizeof(double);
  return L;
}
}  // namespace v4

// Producer of the half-stage ring: warp h streams half h (slices 8h .. 8h+7)
// of every block; warp 0 also the block's slab part.
__device__ __forceinline__ void chain_produce_half(const EpochArgs& a, int h, int lane, int nb, int last_bt, int rc,
                                                   int r0, int RP, int grp, double* halves, size_t half_len,
                                                   double* slabs, uint64_t* fullH, uint64_t* emptyH, uint64_t* fullS,
                                                   uint64_t* emptyS) {
  using namespace v4;
  auto col_of = [&](int u) {
    const int bu = u == nb - 1 ? last_bt : B;
    return u < nb && lane < B / 2 && 8 * h + lane < bu ? __ldg(a.idx + static_cast<int64_t>(u) * B + 8 * h + lane) : 0;
  };
  int ncol = col_of(0);
  for (int t = 0; t < nb; ++t) {
    const int col = ncol;
    ncol = col_of(t + 1);
    const int k = 2 * t + h, slot = k % kHalves, use = k / kHalves;
    if (use > 0) mbar_wait_backoff(&emptyH[slot], static_cast<uint32_t>((use - 1) & 1));
    const int ss = t % kSlabs, su = t / kSlabs;
    if (h == 0 && su > 0) mbar_wait_backoff(&emptyS[ss], static_cast<uint32_t>((su - 1) & 1));
    const int bt = t == nb - 1 ? last_bt : B;
    const int mine = rc > 0 ? max(0, min(B / 2, bt - 8 * h)) : 0;
    double* dst = halves + static_cast<size_t>(slot) * half_len;
    if (lane == 0) {
      fence_proxy_async();
      mbar_expect_tx(&fullH[slot], static_cast<uint32_t>(mine * rc) * 8u);
      if (h == 0) mbar_expect_tx(&fullS[ss], static_cast<uint32_t>(kSlabLen) * 8u);
    }
    __syncwarp();
    if (lane < mine) tma_load_1d(dst + lane * RP, a.X + static_cast<int64_t>(col) * a.ldx + r0, rc * 8u, &fullH[slot]);
    if (h == 0 && lane == 31) {
      const double* slab = a.slab + static_cast<int64_t>(t) * a.slab_len;
      double* sd = slabs + static_cast<size_t>(ss) * kSlabLen;
      tma_load_1d(sd, slab, 2 * B * B * 8u, &fullS[ss]);
      tma_load_1d(sd + 2 * B * B, slab + 2 * B * B + static_cast<size_t>(grp) * B * PC, B * PC * 8u, &fullS[ss]);
    }
  }
}

template <int ROWS, bool XG>
__global__ void __launch_bounds__(v4::kThreads, 1) k_svrg_chain_v4(EpochArgs a) {
  using namespace v4;
  constexpr int kRW = ROWS / kRows, kTiles = kRW / 8;  // rows and 8-row tiles per row warp
  constexpr bool HALF = ROWS > 256;                    // half-stage ring (512 rows, L2 exchange)
  static_assert(!HALF || XG, "the 512-row layout exchanges through L2");
  extern __shared__ __align__(128) double sm[];
  // peers: the cluster (DSMEM exchange) or, XG, the gridDim.x plain CTAs of this group (L2 exchange)
  const int G = XG ? static_cast<int>(gridDim.x) : static_cast<int>(cg::this_cluster().num_blocks());
  const int g = XG ? static_cast<int>(blockIdx.x) : static_cast<int>(cg::this_cluster().block_rank());
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int grp = blockIdx.y;
  const int c0 = grp * PC;
  const int pc = min(PC, a.p - c0);
  const Smem L = HALF ? smem_half() : smem(ROWS, a.stages, XG);
  const int S = L.stages, RP = L.rp;
  double* halves = sm;                                             // HALF: [kHalves][8][RP]
  double* slabs = sm + L.stage_len * kHalves;                      // HALF: [kSlabs][kSlabLen]
  double* xg_slots = XG ? a.xg_slot + static_cast<size_t>(blockIdx.y) * kXgSlots * G * NV : nullptr;  // [slot][G][NV]
  unsigned* xg_cnt = XG ? a.xg_count + static_cast<size_t>(blockIdx.y) * kXgSlots : nullptr;
  const int r0 = g * a.rows_per_cta;
  const int rc = max(0, min(a.rows_per_cta, a.d_pad - r0));
  double* recv = sm + L.off_recv;  // [kRecvSlots][kMaxCluster][NV]
  double* red = sm + L.off_red;    // [2][kRows][NV]
  double* outv = sm + L.off_outv;  // [2][NV]
  double* cfb = sm + L.off_cf;     // [2][B][CP]
  double* Ahat = sm + L.off_ahat;  // [NV]
  // (sm + L.off_pre: a second NV-entry tile, unused by the column-owner reducers)
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + L.off_bar);  // [S <= 4]
  uint64_t* empty = full + 4;                                     // [S]
  uint64_t* rbar = full + 8;                                      // [kRecvSlots]
  uint64_t* fullH = full;                                         // HALF: [kHalves]
  uint64_t* emptyH = full + kHalves;                              // HALF: [kHalves]
  uint64_t* fullS = full + 2 * kHalves;                           // HALF: [kSlabs]
  uint64_t* emptyS = fullS + kSlabs;                              // HALF: [kSlabs]
  auto stage_at = [&](int s_idx) { return sm + static_cast<size_t>(s_idx) * L.stage_len; };
  auto slab_tt = [&](int t) {  // TT_t (then M_t, U_t)
    return HALF ? slabs + static_cast<size_t>(t % kSlabs) * kSlabLen : stage_at(t % S) + B * RP;
  };
  const int nb = static_cast<int>((a.m + B - 1) / B);
  const int last_bt = static_cast<int>(a.m - static_cast<int64_t>(nb - 1) * B);
  auto bt_of = [&](int t) { return t == nb - 1 ? last_bt : B; };
  double rho_b = 1.0, rho_last = 1.0;
  for (int j = 0; j < B; ++j) rho_b *= a.rho;
  for (int j = 0; j < last_bt; ++j) rho_last *= a.rho;
#pragma unroll 1
  for (size_t e = tid; e < L.off_recv; e += blockDim.x) sm[e] = 0.0;  // pad rows / unwritten slices read as 0
  for (int e = tid; e < 2 * B * CP; e += blockDim.x) cfb[e] = 0.0;
  if (tid == 0) {
    if constexpr (HALF) {
      for (int q = 0; q < kHalves; ++q) {
        mbar_init(&fullH[q], 1);
        mbar_init(&emptyH[q], kRows);
      }
      for (int q = 0; q < kSlabs; ++q) {
        mbar_init(&fullS[q], 1);
        mbar_init(&emptyS[q], kRed);
      }
    } else {
      for (int s = 0; s < S; ++s) {
        mbar_init(&full[s], kProd);
        mbar_init(&empty[s], kRows + kRed);
      }
      for (int q = 0; q < kRecvSlots; ++q) mbar_init(&rbar[q], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if constexpr (XG)
    __syncthreads();
  else
    cg::this_cluster().sync();
  // GAPLRA_EPOCH_TIMING: cycles per block; rows (tid 0): 0 wait stage, 1 products,
  // 2 wait coef, 3 update; reducer (warp 4 lane 0): 4 wait Â, 5 reduce + coef,
  // 6 pre; pusher (lane 0): 7 wait red + push
  long long tacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tp = clock64();
  auto tick = [&](int kk) {
#ifndef GAPLRA_NO_TICKS
    if (a.dbg) {
      long long now;
      asm volatile("mov.u64 %0, %%clock64;" : "=l"(now)::"memory");
      tacc[kk] += now - tp;
      tp = now;
    }
#else
    (void)kk;
#endif
  };
  auto bar_red_arrive = [](int u) {  // rows -> pusher, red(u) written (barrier 5 / 6 by parity)
    if (u & 1)
      asm volatile("bar.arrive 6, %0;" ::"n"(32 * (kRows + 1)) : "memory");
    else
      asm volatile("bar.arrive 5, %0;" ::"n"(32 * (kRows + 1)) : "memory");
  };

  if (warp >= kRows + kRed + 1) {  // ------------------------------------------ producers
    if constexpr (HALF)
      chain_produce_half(a, warp - kRows - kRed - 1, lane, nb, last_bt, rc, r0, RP, grp, halves, L.stage_len, slabs,
                         fullH, emptyH, fullS, emptyS);
    else
      chain_produce<PC, B, kProd>(a, warp - kRows - kRed - 1, lane, nb, last_bt, S, rc, r0, RP, grp, sm,
                                  L.stage_len, full, empty);
  } else if (warp == kRows + kRed) {  // ---------------------------------------- pusher
    // Â_u partials of the 4 row warps -> fixed-order sum -> outv[u & 1] ->
    // one bulk copy per peer (lane q -> peer q).  The rows cannot arrive for
    // u + 2 on this barrier before this warp's sync for u: products(u + 2)
    // follows update(u), which needs Â_u from every peer, including this one.
    for (int u = 0; u < nb; ++u) {
      tick(7);
      if (u & 1)
        asm volatile("bar.sync 6, %0;" ::"n"(32 * (kRows + 1)) : "memory");
      else
        asm volatile("bar.sync 5, %0;" ::"n"(32 * (kRows + 1)) : "memory");
      if (!XG && lane < G && a.push_async != 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      __syncwarp();
      const double* rb = red + (u & 1) * kRows * NVR;
      double* ov = outv + (u & 1) * NV;
      // exchanged vector: entry en = c * 16 + j (column-major), read from the padded red [c][RCP]
      if constexpr (XG) {
        if (a.xg_ll == 2) {  // GAPLRA_V4_LL=1: flag-in-data cells, no fence and no counter
          uint4* cells = reinterpret_cast<uint4*>(a.xg_slot) + static_cast<size_t>(blockIdx.y) * kXgSlots * G * NV +
                         (static_cast<size_t>(u % kXgSlots) * G + g) * NV;
#pragma unroll
          for (int q = 0; q < NV / 32; ++q) {
            const int e = q * 32 + lane, er = (e >> 4) * RCP + (e & 15);
            double sum = 0.0;
#pragma unroll
            for (int w = 0; w < kRows; w += 2) sum += rb[w * NVR + er] + rb[(w + 1) * NVR + er];
            ll_store(cells + e, sum, static_cast<uint32_t>(u / kXgSlots + 1));
          }
          continue;
        }
        // partial -> L2 slot, then one release-increment
        double* dst = xg_slots + (static_cast<size_t>(u % kXgSlots) * G + g) * NV;
#pragma unroll
        for (int q = 0; q < NV / 32; ++q) {
          const int e = q * 32 + lane, er = (e >> 4) * RCP + (e & 15);
          double sum = 0.0;
#pragma unroll
          for (int w = 0; w < kRows; w += 2) sum += rb[w * NVR + er] + rb[(w + 1) * NVR + er];
          st_cg(dst + e, sum);
        }
        __syncwarp();
        if (lane == 0) xg_publish(xg_cnt + u % kXgSlots);
        continue;
      }
      if (a.push_async == 2) {  // GAPLRA_PUSH_ASYNC=2: measured not faster here (C2 15.5 vs 15.3 ms, C3 29.6 vs 29.0:
                                // 16 KB per block to the peers is DSMEM-bandwidth-bound either way)
        // straight from registers: lane sums entries (2 lane, 2 lane + 1) + 64 k and stores each pair into every
        // peer's receive slot with one 16-byte st.async (it completes 16 bytes on the peer's barrier); no
        // staging in shared memory, no async-proxy fence, no bulk-copy issue
        const int par = u & (kRecvSlots - 1);
        const uint32_t dst0 = smem_u32(recv + (par * kMaxCluster + g) * NV), bar0 = smem_u32(&rbar[par]);
#pragma unroll
        for (int k = 0; k < NV / 64; ++k) {
          const int e = 64 * k + 2 * lane, er = (e >> 4) * RCP + (e & 15);
          double s0 = 0.0, s1 = 0.0;
#pragma unroll
          for (int w = 0; w < kRows; w += 2) {
            const double2 x = *reinterpret_cast<const double2*>(rb + w * NVR + er);
            const double2 y = *reinterpret_cast<const double2*>(rb + (w + 1) * NVR + er);
            s0 += x.x + y.x;
            s1 += x.y + y.y;
          }
          for (int q = 0; q < G; ++q) st_async_f64x2(mapa(dst0 + e * 8u, q), s0, s1, mapa(bar0, q));
        }
        continue;
      }
#pragma unroll
      for (int q = 0; q < NV / 32; ++q) {
        const int e = q * 32 + lane, er = (e >> 4) * RCP + (e & 15);
        double sum = 0.0;
#pragma unroll
        for (int w = 0; w < kRows; w += 2) sum += rb[w * NVR + er] + rb[(w + 1) * NVR + er];
        ov[e] = sum;
      }
      fence_proxy_async();
      __syncwarp();
      if (lane < G) {
        const int par = u & (kRecvSlots - 1);
        dsmem_bulk_copy(mapa(smem_u32(recv + (par * kMaxCluster + g) * NV), lane), smem_u32(ov), NV * 8u,
                        mapa(smem_u32(&rbar[par]), lane));
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
    if (!XG && lane < G) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    tick(7);
    if (a.dbg && lane == 0) a.dbg[(blockIdx.y * gridDim.x + blockIdx.x) * 8 + 7] = tacc[7];
  } else if (warp >= kRows) {  // --------------------------------------------- reducers
    // warp rw owns columns 2 rw, 2 rw + 1: lane = (c = 2 rw + (lane >> 4), j = lane & 15), exchanged entry
    // e = c * 16 + j = 32 rw + lane.  Â[:, c], coef[:, c] and pre[:, c] live in this warp (a private 32-entry
    // tile + registers), so there is no barrier among the reducer warps.
    const int rw = warp - kRows;
    const int e = rw * 32 + lane;
    const int j = lane & 15, c = 2 * rw + (lane >> 4), hb = lane & 16;
    double* aw = Ahat + rw * 32;  // this warp's Â (then coef) tile: [column half][16]
    auto arm = [&](int u) {
      if (!XG && rw == 0 && lane == 0)
        mbar_expect_tx(&rbar[u & (kRecvSlots - 1)], static_cast<uint32_t>(G * NV * 8));
    };
    double pre_r = 0.0;
    if (nb > 0) {
      arm(0);
      mbar_wait(HALF ? &fullS[0] : &full[0], 0);
      pre_r = slab_tt(0)[2 * B * B + j * PC + c];
    }
    int cs = 0;
    uint32_t cph = 0;
#pragma unroll 1
    for (int t = 0; t < nb; ++t) {
      const bool more = t + 1 < nb;
      const int ns = cs + 1 == S ? 0 : cs + 1;
      const uint32_t nph = ns == 0 ? cph ^ 1u : cph;
      if (more) arm(t + 1);
      const int par = t & (kRecvSlots - 1);
      tick(6);
      if constexpr (XG) {
        // one poller per CTA (four pollers per CTA slowed the exchange: C5 coef wait 534 -> 879 cycles), then
        // the reducer warps meet once on a named barrier
        if (a.xg_ll != 2) {
          if (rw == 0 && lane == 0) xg_wait(xg_cnt + t % kXgSlots, static_cast<unsigned>(G) * (t / kXgSlots + 1));
          asm volatile("bar.sync 4, %0;" ::"n"(32 * kRed) : "memory");  // every peer's partial of block t is in L2
        }
      } else {
        mbar_wait(&rbar[par], static_cast<uint32_t>((t >> 2) & 1));
      }
      tick(4);
      double sacc = 0.0;
      if (j < bt_of(t)) {
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        if constexpr (XG) {
          if (a.xg_ll == 2) {  // poll this entry's cell of every peer (8 in flight), same summation order
            const uint4* cl = reinterpret_cast<const uint4*>(a.xg_slot) +
                              static_cast<size_t>(blockIdx.y) * kXgSlots * G * NV +
                              static_cast<size_t>(t % kXgSlots) * G * NV + e;
            const uint32_t flag = static_cast<uint32_t>(t / kXgSlots + 1);
#pragma unroll 1
            for (int q0 = 0; q0 < G; q0 += 8) {
              uint4 w[8];
#pragma unroll
              for (int k = 0; k < 8; ++k) w[k] = ll_load(cl + (q0 + k) * NV);
              unsigned pend = 0xffu;
              while (pend) {
#pragma unroll
                for (int k = 0; k < 8; ++k)
                  if (pend >> k & 1u) {
                    if (w[k].y == flag && w[k].w == flag)
                      pend &= ~(1u << k);
                    else
                      w[k] = ll_load(cl + (q0 + k) * NV);
                  }
              }
              auto val = [](const uint4& x) { return __hiloint2double(static_cast<int>(x.z), static_cast<int>(x.x)); };
              s0 += val(w[0]);
              s1 += val(w[1]);
              s2 += val(w[2]);
              s3 += val(w[3]);
              s0 += val(w[4]);
              s1 += val(w[5]);
              s2 += val(w[6]);
              s3 += val(w[7]);
            }
          } else {
          const double* sl = xg_slots + static_cast<size_t>(t % kXgSlots) * G * NV + e;
          // all G loads in flight (L2 latency, not a loop-carried chain, sets the cost)
#pragma unroll 4
          for (int q = 0; q < G; q += 4) {
            s0 += ld_cg(sl + q * NV);
            s1 += ld_cg(sl + (q + 1) * NV);
            s2 += ld_cg(sl + (q + 2) * NV);
            s3 += ld_cg(sl + (q + 3) * NV);
          }
          }
        } else {
          const double* sl = recv + par * kMaxCluster * NV + e;
#pragma unroll 4
          for (int q = 0; q < G; q += 4) {
            s0 += sl[q * NV];
            s1 += sl[(q + 1) * NV];
            s2 += sl[(q + 2) * NV];
            s3 += sl[(q + 3) * NV];
          }
        }
        sacc = (s0 + s1) + (s2 + s3);
      }
      aw[lane] = sacc;
      __syncwarp();  // Â[:, c] of both columns complete
      const double* TT = slab_tt(t);
      double* cf = cfb + (t & 1) * B * CP;
      double cv;
      {
        double s0 = pre_r, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
        for (int l = 0; l < B; l += 4) {
          s0 = fma(TT[l * B + j], aw[hb + l], s0);
          s1 = fma(TT[(l + 1) * B + j], aw[hb + l + 1], s1);
          s2 = fma(TT[(l + 2) * B + j], aw[hb + l + 2], s2);
          s3 = fma(TT[(l + 3) * B + j], aw[hb + l + 3], s3);
        }
        cv = (s0 + s1) + (s2 + s3);
        cf[j * CP + c] = cv;
      }
      if (t & 1)
        asm volatile("bar.arrive 3, %0;" ::"n"(32 * (kRows + kRed)) : "memory");
      else
        asm volatile("bar.arrive 2, %0;" ::"n"(32 * (kRows + kRed)) : "memory");
      tick(5);
      __syncwarp();  // every lane's Â reads done
      aw[lane] = cv;  // coef[:, c] for pre_{t+1}
      if (lane == 0) mbar_arrive(HALF ? &emptyS[t % kSlabs] : &empty[cs]);  // TT_t: the reducers' last use
      if (more) {  // pre_{t+1} = M_{t+1} coef_t + U_{t+1}
        __syncwarp();
        if constexpr (HALF)
          mbar_wait(&fullS[(t + 1) % kSlabs], static_cast<uint32_t>(((t + 1) / kSlabs) & 1));
        else
          mbar_wait(&full[ns], nph);
        const double* M = slab_tt(t + 1) + B * B;
        const double* Ub = M + B * B;
        double s0 = Ub[j * PC + c], s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
        for (int l = 0; l < B; l += 4) {
          s0 = fma(M[l * B + j], aw[hb + l], s0);
          s1 = fma(M[(l + 1) * B + j], aw[hb + l + 1], s1);
          s2 = fma(M[(l + 2) * B + j], aw[hb + l + 2], s2);
          s3 = fma(M[(l + 3) * B + j], aw[hb + l + 3], s3);
        }
        pre_r = (s0 + s1) + (s2 + s3);
        __syncwarp();  // the tile is free for the next Â
      }
      cs = ns;
      cph = nph;
    }
    tick(6);
    if (a.dbg && warp == kRows && lane == 0)
      for (int kk = 4; kk < 7; ++kk) a.dbg[(blockIdx.y * gridDim.x + blockIdx.x) * 8 + kk] = tacc[kk];
  } else {  // --------------------------------------------------------------- rows
    const int perm = ((gq & 1) << 1) | ((gq >> 1) & 1) | (gq & 4);  // 0 2 1 3 4 6 5 7
    const int rw0 = warp * kRW;  // this warp's first row (of the CTA's slice)
    double v[kTiles][2];          // Vᵀ C fragments: column gq, rows rw0 + 8 tile + 2 tq + {0, 1}
#pragma unroll
    for (int tl = 0; tl < kTiles; ++tl)
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int r = rw0 + 8 * tl + 2 * tq + u;
        v[tl][u] = (r < rc && gq < pc) ? a.W[static_cast<int64_t>(r0 + r) * a.ldw + c0 + gq] : 0.0;
      }
    int ws = 0;
    uint32_t wph = 0;
    auto wait_stage = [&]() {
      mbar_wait(&full[ws], wph);
      const int s = ws;
      if (++ws == S) {
        ws = 0;
        wph ^= 1u;
      }
      return s;
    };
    auto half_ptr = [&](int k) { return halves + static_cast<size_t>(k % kHalves) * L.stage_len; };
    auto wait_half = [&](int k) { mbar_wait(&fullH[k % kHalves], static_cast<uint32_t>((k / kHalves) & 1)); };
    // Âᵀ partial over the warp's rows: 2 slice tiles (slices 0-7 at xb0, 8-15 at
    // xb1), K = the rows; HALF: half kw (then kw + 1) is waited for just before use
    auto products = [&](const double* xb0, const double* xb1, int u_blk, int kw) {
      // (four accumulator chains per slice tile measured slower: products 1366 ->
      // 1703 cycles per block at C5)
      double acc[2][2][2];  // [slice tile][chain][elem]
#pragma unroll
      for (int n2 = 0; n2 < 2; ++n2)
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) acc[n2][ch][0] = acc[n2][ch][1] = 0.0;
#pragma unroll
      for (int n2 = 0; n2 < 2; ++n2) {
        if constexpr (HALF) wait_half(kw + n2);
        const double* xb = n2 ? xb1 : xb0;
#pragma unroll
        for (int tl = 0; tl < kTiles; ++tl) {
          const double2 xv = *reinterpret_cast<const double2*>(xb + perm * RP + rw0 + 8 * tl + 2 * tq);
#ifdef GAPLRA_CHAIN_ABLATE
          if (a.skip & 2) continue;  // GAPLRA_EPOCH_SKIP ablation (results invalid)
#endif
          dmma(acc[n2][tl & 1][0], acc[n2][tl & 1][1], v[tl][0], xv.x);
          dmma(acc[n2][tl & 1][0], acc[n2][tl & 1][1], v[tl][1], xv.y);
        }
      }
      // C fragment (column gq, slices 8 n2 + perm(2 tq), 8 n2 + perm(2 tq + 1)) -> red(u_blk) in [j PC + c]
      double* rb = red + (u_blk & 1) * kRows * NVR + warp * NVR;
      const int pa = ((2 * tq) & 1) << 1 | (((2 * tq) >> 1) & 1) | ((2 * tq) & 4);
      const int pb = ((2 * tq + 1) & 1) << 1 | (((2 * tq + 1) >> 1) & 1) | ((2 * tq + 1) & 4);
#pragma unroll
      for (int n2 = 0; n2 < 2; ++n2) {
        rb[gq * RCP + 8 * n2 + pa] = acc[n2][0][0] + acc[n2][1][0];
        rb[gq * RCP + 8 * n2 + pb] = acc[n2][0][1] + acc[n2][1][1];
      }
      bar_red_arrive(u_blk);
    };
    // Vᵀ = rn (Vᵀ + coefᵀ X_Bᵀ); HALF: each half-stage is released after its two k-steps
    auto update = [&](const double* xb0, const double* xb1, int t, double rn) {
      const double* xb = xb0;
      tick(1);
      if (t & 1)
        asm volatile("bar.sync 3, %0;" ::"n"(32 * (kRows + kRed)) : "memory");
      else
        asm volatile("bar.sync 2, %0;" ::"n"(32 * (kRows + kRed)) : "memory");
      tick(2);
      const double* cf = cfb + (t & 1) * B * CP;
      double af[4];
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) af[ks] = cf[(4 * ks + tq) * CP + gq];
      if constexpr (kTiles <= 4) {
        double bx[4][kTiles];
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
#pragma unroll
          for (int tl = 0; tl < kTiles; ++tl) bx[ks][tl] = xb[(4 * ks + tq) * RP + rw0 + 8 * tl + gq];
#ifdef GAPLRA_CHAIN_ABLATE
        if (!(a.skip & 4))
#endif
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)
#pragma unroll
            for (int tl = 0; tl < kTiles; ++tl) dmma(v[tl][0], v[tl][1], af[ks], bx[ks][tl]);
      } else {  // 512 rows: two k-steps of B fragments in flight (register budget of 480 threads;
                // a k-step software pipeline measured no faster: update 1821 vs 1803 cycles)
#pragma unroll
        for (int k2 = 0; k2 < 4; k2 += 2) {
          const double* xh = k2 ? xb1 : xb0;  // slices 4 (k2 + ks) + tq = 8 (k2 / 2) + 4 ks + tq
          double bx[2][kTiles];
#pragma unroll
          for (int ks = 0; ks < 2; ++ks)
#pragma unroll
            for (int tl = 0; tl < kTiles; ++tl) bx[ks][tl] = xh[(4 * ks + tq) * RP + rw0 + 8 * tl + gq];
#pragma unroll
          for (int ks = 0; ks < 2; ++ks)
#pragma unroll
            for (int tl = 0; tl < kTiles; ++tl) dmma(v[tl][0], v[tl][1], af[k2 + ks], bx[ks][tl]);
          if constexpr (HALF) {  // this half's slices are in registers / consumed
            __syncwarp();
            if (lane == 0) mbar_arrive(&emptyH[(2 * t + k2 / 2) % kHalves]);
          }
        }
      }
#pragma unroll
      for (int tl = 0; tl < kTiles; ++tl) {
        v[tl][0] *= rn;
        v[tl][1] *= rn;
      }
    };
    if (nb > 0) {  // Â_0 = X_{B_0}ᵀ Ŵ_0, then V_0 = ρ^{b_0} Ŵ_0
      if constexpr (HALF) {
        products(half_ptr(0), half_ptr(1), 0, 0);
      } else {
        const int s = wait_stage();
        products(stage_at(s), stage_at(s) + 8 * RP, 0, 0);
      }
      double rb0 = 1.0;
      for (int jj = 0; jj < bt_of(0); ++jj) rb0 *= a.rho;
#pragma unroll
      for (int tl = 0; tl < kTiles; ++tl) {
        v[tl][0] *= rb0;
        v[tl][1] *= rb0;
      }
    }
    int cs = 0;
#pragma unroll 1
    for (int t = 0; t < nb; ++t) {
      const bool more = t + 1 < nb;
      if (more) {
        tick(3);
        if constexpr (HALF) {
          tick(0);
          products(half_ptr(2 * t + 2), half_ptr(2 * t + 3), t + 1, 2 * t + 2);
        } else {
          const int s = wait_stage();
          tick(0);
          products(stage_at(s), stage_at(s) + 8 * RP, t + 1, 0);
        }
      }
      const double rn = !more ? 1.0 : (t + 1 == nb - 1 ? rho_last : rho_b);
      if constexpr (HALF) {
        update(half_ptr(2 * t), half_ptr(2 * t + 1), t, rn);
      } else {
        update(stage_at(cs), stage_at(cs) + 8 * RP, t, rn);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[cs]);
        cs = cs + 1 == S ? 0 : cs + 1;
      }
    }
    tick(3);
    if (a.dbg && tid == 0)
      for (int kk = 0; kk < 4; ++kk) a.dbg[(blockIdx.y * gridDim.x + blockIdx.x) * 8 + kk] = tacc[kk];
    const double beta = -expm1(static_cast<double>(a.m) * log1p(a.rho - 1.0)) / (1.0 - a.rho);
    if (gq < pc)
#pragma unroll
      for (int tl = 0; tl < kTiles; ++tl)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int r = rw0 + 8 * tl + 2 * tq + u;
          if (r < rc) {
            const int64_t o = static_cast<int64_t>(r0 + r) * a.ldw + c0 + gq;
            a.W[o] = fma(beta, a.C[o], v[tl][u]);
          }
        }
  }
  if constexpr (!XG) cg::this_cluster().sync();  // no CTA leaves while a peer may still copy into it
}

// ---------------------------------------------------------------------------
// k_chain_p1_la2: the p = 1 chain with a TWO-block lookahead.
// With V_t = ρ^{b_t} Ŵ_t (V_{−1} = V_{−2} = Ŵ_0) and Â'_t = X_{B_t}ᵀ V_{t−2}:
//   P̂_t = X_{B_t}ᵀ Ŵ_t = ρ^{b_{t−1}} (Â'_t + Kxx_t coef_{t−2}) + Kx_t coef_{t−1}
//   coef_t = TT_t P̂_t + U_t
//          = ρ^{b_{t−1}} (TT_t Â'_t + M2_t coef_{t−2}) + M_t coef_{t−1} + U_t
// (M = TT Kx, M2 = TT Kxx from k_block_prep<16, 2>; b_{−1} = 0) — the same
// recurrence as the one-block chains in exact arithmetic.  The rows push Â'_{t+2}
// (products with V_t) at iteration t, so the all-reduce has two blocks of
// slack: enough for the L2 exchange (XG) as well as DSMEM, and the rows can be
// spread thinner (more SMs pull X).  Warps: 4 rows (2 rows per thread; the
// update re-reads the stage), 1 reducer (lane = entry), 1 pusher, 4 producers.
// Ring of S >= 5 stages (blocks t, t+1, t+2 live), 8 receive slots (re-armed
// after use), coef in 4 buffers; named barriers 1-4 hand coef_t to the rows,
// 5-8 hand the rows' partials of block u to the pusher (by t, u mod 4).
// ---------------------------------------------------------------------------
namespace la2 {
constexpr int B = 16, kRows = 4, kProd = 4, kSlots = 8;
constexpr int kThreads = 32 * (kRows + 2 + kProd);
constexpr int kHead = 3 * B * B;  // TT | M | M2
struct Smem {
  int rp, stages;
  size_t stage_len, off_recv, off_red, off_cf, off_ahat, off_outv, off_bar, total;
};
__host__ __device__ inline Smem smem(int rows, int stages, bool xg) {
  Smem L;
  L.rp = (rows + 15) / 16 * 16;  // ≡ 0 (mod 16): the lane-permuted LDS.128 are conflict free
  L.stages = stages;
  L.stage_len = static_cast<size_t>(B) * L.rp + kHead + B;  // slices | TT M M2 | U
  size_t o = L.stage_len * stages;
  L.off_recv = o;
  if (!xg) o += static_cast<size_t>(kSlots) * kMaxCluster * B;
  L.off_red = o;
  o += 4 * kRows * B;
  L.off_cf = o;
  o += 4 * B;
  L.off_ahat = o;
  o += B;
  L.off_outv = o;
  o += 4 * B;
  L.off_bar = o;
  o += 32;  // full[<=12] | empty[<=12] | rbar[8]
  L.total = o * sizeof(double);
  return L;
}
}  // namespace la2

template <bool XG>
__global__ void __launch_bounds__(la2::kThreads, 1) k_chain_p1_la2(EpochArgs a) {
  using namespace la2;
  extern __shared__ __align__(128) double sm[];
  const int G = XG ? static_cast<int>(gridDim.x) : static_cast<int>(cg::this_cluster().num_blocks());
  const int g = XG ? static_cast<int>(blockIdx.x) : static_cast<int>(cg::this_cluster().block_rank());
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const Smem L = smem(a.rows_per_cta, a.stages, XG);
  const int S = L.stages, RP = L.rp;
  const int r0 = g * a.rows_per_cta;
  const int rc = max(0, min(a.rows_per_cta, a.d_pad - r0));
  double* recv = sm + L.off_recv;  // [kSlots][kMaxCluster][B]
  double* red = sm + L.off_red;    // [4][kRows][B]
  double* cf = sm + L.off_cf;      // [4][B]: coef_t in cf[t & 3]
  double* Ahat = sm + L.off_ahat;  // [B]
  double* outv = sm + L.off_outv;  // [4][B]
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + L.off_bar);
  uint64_t* empty = full + 12;
  uint64_t* rbar = full + 24;
  double* xg_slots = XG ? a.xg_slot : nullptr;  // [kSlots][G][B]
  unsigned* xg_cnt = XG ? a.xg_count : nullptr;  // [kSlots]
  auto stage_at = [&](int t) { return sm + static_cast<size_t>(t % S) * L.stage_len; };
  const int nb = static_cast<int>((a.m + B - 1) / B);
  const int last_bt = static_cast<int>(a.m - static_cast<int64_t>(nb - 1) * B);
  auto bt_of = [&](int t) { return t == nb - 1 ? last_bt : B; };
  double rho_b = 1.0, rho_last = 1.0;
  for (int j = 0; j < B; ++j) rho_b *= a.rho;
  for (int j = 0; j < last_bt; ++j) rho_last *= a.rho;
  auto rho_of = [&](int t) { return t < 0 ? 1.0 : (t == nb - 1 ? rho_last : rho_b); };  // ρ^{b_t}
#pragma unroll 1
  for (size_t e = tid; e < L.off_recv; e += blockDim.x) sm[e] = 0.0;  // pad rows / unwritten slices read as 0
  for (int e = tid; e < 4 * B; e += blockDim.x) cf[e] = 0.0;        // coef_{−1} = coef_{−2} = 0
  if (tid == 0) {
    for (int q = 0; q < S; ++q) {
      mbar_init(&full[q], kProd);
      mbar_init(&empty[q], kRows + 1);
    }
    for (int q = 0; q < kSlots; ++q) mbar_init(&rbar[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if constexpr (XG)
    __syncthreads();
  else
    cg::this_cluster().sync();
  long long tacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tp;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(tp)::"memory");
  auto tick = [&](int kk) {
#ifndef GAPLRA_NO_TICKS
    if (a.dbg) {
      long long now;
      asm volatile("mov.u64 %0, %%clock64;" : "=l"(now)::"memory");
      tacc[kk] += now - tp;
      tp = now;
    }
#else
    (void)kk;
#endif
  };
  auto red_arrive = [](int u) {  // rows -> pusher: red(u) written (barriers 5..8)
    switch (u & 3) {
      case 0: asm volatile("bar.arrive 5, %0;" ::"n"(32 * (kRows + 1)) : "memory"); break;
      case 1: asm volatile("bar.arrive 6, %0;" ::"n"(32 * (kRows + 1)) : "memory"); break;
      case 2: asm volatile("bar.arrive 7, %0;" ::"n"(32 * (kRows + 1)) : "memory"); break;
      default: asm volatile("bar.arrive 8, %0;" ::"n"(32 * (kRows + 1)) : "memory"); break;
    }
  };
  auto red_sync = [](int u) {
    switch (u & 3) {
      case 0: asm volatile("bar.sync 5, %0;" ::"n"(32 * (kRows + 1)) : "memory"); break;
      case 1: asm volatile("bar.sync 6, %0;" ::"n"(32 * (kRows + 1)) : "memory"); break;
      case 2: asm volatile("bar.sync 7, %0;" ::"n"(32 * (kRows + 1)) : "memory"); break;
      default: asm volatile("bar.sync 8, %0;" ::"n"(32 * (kRows + 1)) : "memory"); break;
    }
  };
  auto coef_arrive = [](int t) {  // reducer -> rows: coef_t in cf[t & 3] (barriers 1..4)
    switch (t & 3) {
      case 0: asm volatile("bar.arrive 1, %0;" ::"n"(32 * (kRows + 1)) : "memory"); break;
      case 1: asm volatile("bar.arrive 2, %0;" ::"n"(32 * (kRows + 1)) : "memory"); break;
      case 2: asm volatile("bar.arrive 3, %0;" ::"n"(32 * (kRows + 1)) : "memory"); break;
      default: asm volatile("bar.arrive 4, %0;" ::"n"(32 * (kRows + 1)) : "memory"); break;
    }
  };
  auto coef_sync = [](int t) {
    switch (t & 3) {
      case 0: asm volatile("bar.sync 1, %0;" ::"n"(32 * (kRows + 1)) : "memory"); break;
      case 1: asm volatile("bar.sync 2, %0;" ::"n"(32 * (kRows + 1)) : "memory"); break;
      case 2: asm volatile("bar.sync 3, %0;" ::"n"(32 * (kRows + 1)) : "memory"); break;
      default: asm volatile("bar.sync 4, %0;" ::"n"(32 * (kRows + 1)) : "memory"); break;
    }
  };

  if (warp >= kRows + 2) {  // ------------------------------------------- producers
    chain_produce<1, B, kProd>(a, warp - kRows - 2, lane, nb, last_bt, S, rc, r0, RP, 0, sm, L.stage_len, full,
                               empty, kHead);
  } else if (warp == kRows + 1) {  // -------------------------------------- pusher
    for (int u = 0; u < nb; ++u) {
      red_sync(u);
      if (!XG && lane < G) asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");  // outv[u & 3] free
      __syncwarp();
      const double* rb = red + (u & 3) * kRows * B;
      const int e = lane & 15;
      const double sum = (rb[e] + rb[B + e]) + (rb[2 * B + e] + rb[3 * B + e]);
      if constexpr (XG) {
        if (a.xg_ll) {
          if (lane < B)
            ll_store(reinterpret_cast<uint4*>(xg_slots) + (static_cast<size_t>(u % kSlots) * G + g) * B + e, sum,
                     static_cast<uint32_t>(u / kSlots + 1));
        } else {
          if (lane < B) st_cg(xg_slots + (static_cast<size_t>(u % kSlots) * G + g) * B + e, sum);
          __syncwarp();
          if (lane == 0) xg_publish(xg_cnt + u % kSlots);
        }
      } else {
        double* ov = outv + (u & 3) * B;
        if (lane < B) ov[e] = sum;
        fence_proxy_async();
        __syncwarp();
        if (lane < G) {
          const int q = u % kSlots;
          dsmem_bulk_copy(mapa(smem_u32(recv + (q * kMaxCluster + g) * B), lane), smem_u32(ov), B * 8u,
                          mapa(smem_u32(&rbar[q]), lane));
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
    }
    if (!XG && lane < G) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  } else if (warp == kRows) {  // ----------------------------------------- reducer
    const int j = lane & 15;
    if (!XG && lane == 0)
      for (int q = 0; q < kSlots && q < nb; ++q) mbar_expect_tx(&rbar[q], static_cast<uint32_t>(G * B * 8));
#pragma unroll 1
    for (int t = 0; t < nb; ++t) {
      tick(7);
      mbar_wait(&full[t % S], static_cast<uint32_t>((t / S) & 1));
      const double* sl = stage_at(t) + B * RP;  // TT, M, M2 transposed ([l][j]), then U
      const double rprev = rho_of(t - 1);
      const double* c1 = cf + ((t - 1) & 3) * B;
      const double* c2 = cf + ((t - 2) & 3) * B;
      double pre;
      {
        double s0 = sl[3 * B * B + j], s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
        for (int l = 0; l < B; l += 2) {
          s0 = fma(sl[B * B + l * B + j], c1[l], s0);
          s1 = fma(sl[B * B + (l + 1) * B + j], c1[l + 1], s1);
          s2 = fma(sl[2 * B * B + l * B + j], c2[l], s2);
          s3 = fma(sl[2 * B * B + (l + 1) * B + j], c2[l + 1], s3);
        }
        pre = (s0 + s1) + rprev * (s2 + s3);
      }
      tick(6);
      const int bt = bt_of(t);
      if constexpr (XG) {
       if (a.xg_ll) {
        const double sv = ll_gather16(reinterpret_cast<const uint4*>(xg_slots) + static_cast<size_t>(t % kSlots) * G * B,
                                      G, lane, static_cast<uint32_t>(t / kSlots + 1));
        tick(5);
        if (lane < B) Ahat[j] = j < bt ? sv : 0.0;
       } else {
        if (lane == 0) xg_wait(xg_cnt + t % kSlots, static_cast<unsigned>(G) * (t / kSlots + 1));
        __syncwarp();
        tick(5);
        const int hq = (lane >> 4) * 2;
        const double* ps = xg_slots + static_cast<size_t>(t % kSlots) * G * B + j;
        double sa = 0.0, sb = 0.0;
#pragma unroll 4
        for (int q = 0; q < G; q += 4) {
          sa += ld_cg(ps + (q + hq) * B);
          sb += ld_cg(ps + (q + hq + 1) * B);
        }
        const double sv = sa + sb;
        const double other = __shfl_down_sync(0xffffffffu, sv, 16);
        if (lane < B) Ahat[j] = j < bt ? sv + other : 0.0;
       }
      } else {
        mbar_wait(&rbar[t % kSlots], static_cast<uint32_t>((t / kSlots) & 1));
        tick(5);
        if (lane < B) {
          const double* ps = recv + (t % kSlots) * kMaxCluster * B + j;
          double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll 1
          for (int q = 0; q < G; q += 4) {
            s0 += ps[q * B];
            s1 += ps[(q + 1) * B];
            s2 += ps[(q + 2) * B];
            s3 += ps[(q + 3) * B];
          }
          Ahat[j] = j < bt ? (s0 + s1) + (s2 + s3) : 0.0;
        }
      }
      __syncwarp();
      if (lane < B) {
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
        for (int l = 0; l < B; l += 4) {
          s0 = fma(sl[l * B + j], Ahat[l], s0);
          s1 = fma(sl[(l + 1) * B + j], Ahat[l + 1], s1);
          s2 = fma(sl[(l + 2) * B + j], Ahat[l + 2], s2);
          s3 = fma(sl[(l + 3) * B + j], Ahat[l + 3], s3);
        }
        cf[(t & 3) * B + j] = fma(rprev, (s0 + s1) + (s2 + s3), pre);
      }
      __syncwarp();
      coef_arrive(t);
      tick(4);
      if (lane == 0) {
        if (!XG && t + kSlots < nb) mbar_expect_tx(&rbar[t % kSlots], static_cast<uint32_t>(G * B * 8));
        mbar_arrive(&empty[t % S]);  // TT, M, M2, U of block t: the reducer's last use
      }
    }
    if (a.dbg && lane == 0) {
      const int cta = blockIdx.y * gridDim.x + blockIdx.x;
      for (int kk = 4; kk < 8; ++kk) a.dbg[cta * 8 + kk] = tacc[kk];
    }
  } else {  // --------------------------------------------------------------- rows
    const int pm = lane >> 1;  // product order j = i ^ pm (select-free warp halving)
    const int ra = 2 * tid;    // rows ra, ra + 1 of the CTA's slice
    const bool own0 = ra < rc, own1 = ra + 1 < rc;
    double v0 = own0 ? a.W[static_cast<int64_t>(r0 + ra) * a.ldw] : 0.0;
    double v1 = own1 ? a.W[static_cast<int64_t>(r0 + ra + 1) * a.ldw] : 0.0;
    auto wait_stage = [&](int t) { mbar_wait(&full[t % S], static_cast<uint32_t>((t / S) & 1)); };
    auto load_rows = [&](const double* xb, double2 (&xr)[B]) {
#pragma unroll
      for (int i = 0; i < B; ++i) xr[i] = *reinterpret_cast<const double2*>(xb + (i ^ pm) * RP + ra);
    };
    auto products = [&](const double2 (&xr)[B], int u) {
      double val[B];
#pragma unroll
      for (int i = 0; i < B; ++i) val[i] = fma(xr[i].x, v0, xr[i].y * v1);
#pragma unroll
      for (int o = 16, n = B / 2; o >= 2; o >>= 1, n >>= 1)
#pragma unroll
        for (int i = 0; i < n; ++i) val[i] += __shfl_xor_sync(0xffffffffu, val[i + n], o);
      val[0] += __shfl_xor_sync(0xffffffffu, val[0], 1);
      if (!(lane & 1)) red[(u & 3) * kRows * B + warp * B + pm] = val[0];
      red_arrive(u);
    };
    auto update = [&](const double2 (&xr)[B], int t, double rn) {
      tick(1);
      coef_sync(t);
      tick(2);
      const double* c = cf + (t & 3) * B;
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int i = 0; i < B; i += 2) {
        const double k0 = c[i ^ pm], k1 = c[(i + 1) ^ pm];
        v0 = fma(xr[i].x, k0, v0);
        v1 = fma(xr[i].y, k0, v1);
        a0 = fma(xr[i + 1].x, k1, a0);
        a1 = fma(xr[i + 1].y, k1, a1);
      }
      v0 = own0 ? (v0 + a0) * rn : 0.0;
      v1 = own1 ? (v1 + a1) * rn : 0.0;
    };
    double2 xr[B];
    // Â'_0 = X_{B_0}ᵀ Ŵ_0 and Â'_1 = X_{B_1}ᵀ Ŵ_0 (V_{−2} = V_{−1} = Ŵ_0), then V_0 = ρ^{b_0} Ŵ_0
    for (int u = 0; u < 2 && u < nb; ++u) {
      wait_stage(u);
      load_rows(stage_at(u), xr);
      products(xr, u);
    }
    {
      const double r = rho_of(0);
      v0 *= r;
      v1 *= r;
    }
#pragma unroll 1
    for (int t = 0; t < nb; ++t) {
      if (t + 2 < nb) {
        tick(3);
        wait_stage(t + 2);
        tick(0);
        load_rows(stage_at(t + 2), xr);
        products(xr, t + 2);  // with V_t
      }
      load_rows(stage_at(t), xr);
      update(xr, t, t + 1 < nb ? rho_of(t + 1) : 1.0);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[t % S]);
    }
    if (a.dbg && tid == 0) {
      const int cta = blockIdx.y * gridDim.x + blockIdx.x;
      for (int kk = 0; kk < 4; ++kk) a.dbg[cta * 8 + kk] = tacc[kk];
    }
    const double beta = -expm1(static_cast<double>(a.m) * log1p(a.rho - 1.0)) / (1.0 - a.rho);
    if (own0) {
      const int64_t o = static_cast<int64_t>(r0 + ra) * a.ldw;
      a.W[o] = fma(beta, a.C[o], v0);
    }
    if (own1) {
      const int64_t o = static_cast<int64_t>(r0 + ra + 1) * a.ldw;
      a.W[o] = fma(beta, a.C[o], v1);
    }
  }
  if constexpr (!XG) cg::this_cluster().sync();
}

// Clusters of `cluster` one-SM CTAs that can be resident at once (a cluster
// lives inside one GPC, so this is below SMs / cluster when GPCs are uneven).
int max_active_clusters(int cluster) {
  static int cached[17] = {0};
  if (cluster < 1 || cluster > 16) return 1;
  if (cached[cluster]) return cached[cluster];
  auto kern = k_svrg_chain_v3<1, kBlock>;
  const int smem = 200 * 1024;  // any CTA of the chain takes a whole SM
  GAPLRA_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  GAPLRA_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(cluster, 64, 1);
  lc.blockDim = dim3(v3_threads(1), 1, 1);
  lc.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &lc) != cudaSuccess || n < 1) {
    (void)cudaGetLastError();
    n = std::max(1, sm_count_dev() / cluster);
  }
  cached[cluster] = n;
  return n;
}

EpochConfig choose_epoch_config(int d_pad, int p) {
  // Candidate layouts: clusters of 16 or 8 CTAs splitting the d rows, PC RHS
  // columns per cluster.  Prefer one the warp-specialised chain (v3) runs:
  // PC <= 3 and <= 256 rows per CTA (C2: 16 x 256 rows, PC 3; C3: 8 x 256,
  // PC 2); otherwise the largest cluster.  GAPLRA_CLUSTER=8|16 forces the size.
  static const int env_cluster = getenv("GAPLRA_CLUSTER") ? atoi(getenv("GAPLRA_CLUSTER")) : 0;
  auto make = [&](int cluster) {
    EpochConfig cfg;
    cfg.b = kBlock;
    cfg.cluster = cluster;
    const int max_clusters = max_active_clusters(cfg.cluster);
    static const int env_pc = getenv("GAPLRA_CHAIN_PC") ? atoi(getenv("GAPLRA_CHAIN_PC")) : 0;  // experiments
    cfg.pc = round_pc(env_pc > 0 ? std::min(env_pc, p) : static_cast<int>(ceil_div(p, max_clusters)));
    cfg.rows_per_cta = static_cast<int>(ceil_div(ceil_div(d_pad, cfg.cluster), 4) * 4);
    const size_t cap = 227 * 1024;
    for (;;) {
      cfg.stages = 4;
      while (cfg.stages > 2 && smem_for(cfg.pc, cfg.rows_per_cta, cfg.stages) > cap) --cfg.stages;
      if (smem_for(cfg.pc, cfg.rows_per_cta, cfg.stages) <= cap || cfg.pc == 1) break;
      cfg.pc = shrink_pc(cfg.pc);
    }
    cfg.groups = static_cast<int>(ceil_div(p, cfg.pc));
    cfg.smem = smem_for(cfg.pc, cfg.rows_per_cta, cfg.stages);
    return cfg;
  };
  if (env_cluster == 8 || env_cluster == 16) return make(env_cluster);
  // the DMMA chain v4 (PC = 8, <= 256 rows per CTA) for p >= 4: C2 runs 3
  // clusters of 16 CTAs instead of 7 x PC 3 (epoch 17.7 -> 14.2 ms);
  // GAPLRA_CHAIN_V4=0 keeps the scalar chains
  static const int env_v4 = getenv("GAPLRA_CHAIN_V4") ? atoi(getenv("GAPLRA_CHAIN_V4")) : 1;
  static const int env_pc = getenv("GAPLRA_CHAIN_PC") ? atoi(getenv("GAPLRA_CHAIN_PC")) : 0;
  // (d <= 1024 keeps v3: with <= 128 rows per CTA half of v4's row warps idle;
  // C1 measured 0.31 s with v4 against 0.28 s)
  if (env_v4 && env_pc == 0 && p >= 4 && d_pad > 1024 && d_pad <= 16 * 512) {
    EpochConfig cfg;
    cfg.b = kBlock;
    cfg.cluster = d_pad <= 8 * 256 ? 8 : 16;
    // GAPLRA_V4_ROWS=128: rows spread thinner (C2: 3 groups x 32 plain CTAs over L2; C3: 16-CTA clusters)
    static const int env_v4_rows = getenv("GAPLRA_V4_ROWS") ? atoi(getenv("GAPLRA_V4_ROWS")) : 0;
    if (env_v4_rows == 128) cfg.cluster = static_cast<int>(ceil_div(ceil_div(d_pad, 128), 4) * 4);
    cfg.pc = 8;
    cfg.rows_per_cta = static_cast<int>(ceil_div(ceil_div(d_pad, cfg.cluster), 4) * 4);
    cfg.groups = static_cast<int>(ceil_div(p, 8));
    cfg.stages = 3;
    while (cfg.stages > 2 && v4::smem(cfg.rows_per_cta, cfg.stages).total > 227 * 1024) --cfg.stages;
    cfg.smem = v4::smem(cfg.rows_per_cta, cfg.stages).total;
    // more groups than resident clusters (C5: 8 groups of 16 CTAs, 7 sixteen-CTA
    // clusters fit): plain CTAs exchanging through L2, one wave on 128 SMs.
    // GAPLRA_CHAIN_XG=0 never, 2 always (where the CTAs fit one wave)
    static const int env_xg = getenv("GAPLRA_CHAIN_XG") ? atoi(getenv("GAPLRA_CHAIN_XG")) : 1;
    // (512 rows per CTA always exchange through L2: the half-stage ring and
    // the 64 KB of DSMEM receive slots do not fit together)
    if (cfg.cluster <= 16 && cfg.groups <= max_active_clusters(cfg.cluster) && env_xg != 2 && cfg.rows_per_cta <= 256)
      return cfg;
    if ((env_xg || cfg.rows_per_cta > 256) && cfg.groups * cfg.cluster <= sm_count_dev()) {
      cfg.xg = 1;
      cfg.stages = 3;
      while (cfg.stages > 2 && v4::smem(cfg.rows_per_cta, cfg.stages, true).total > 227 * 1024) --cfg.stages;
      cfg.smem = cfg.rows_per_cta > 256 ? v4::smem_half().total : v4::smem(cfg.rows_per_cta, cfg.stages, true).total;
      return cfg;
    }
  }
  // p = 1 with the two-block lookahead chain (k_chain_p1_la2): GAPLRA_P1_LA2=1,
  // GAPLRA_LA2_ROWS rows per CTA (128), GAPLRA_LA2_XG=1 forces the L2 exchange
  // (otherwise a DSMEM cluster when the CTAs fit one: <= 16)
  static const int env_la2 = getenv("GAPLRA_P1_LA2") ? atoi(getenv("GAPLRA_P1_LA2")) : 0;
  static const int env_la2_rows = getenv("GAPLRA_LA2_ROWS") ? atoi(getenv("GAPLRA_LA2_ROWS")) : 128;
  static const int env_la2_xg = getenv("GAPLRA_LA2_XG") ? atoi(getenv("GAPLRA_LA2_XG")) : 0;
  if (p == 1 && env_la2 && env_pc == 0 && d_pad > 1024 && d_pad <= 8192) {
    EpochConfig cfg;
    cfg.b = kBlock;
    cfg.pc = 1;
    cfg.groups = 1;
    cfg.la = 2;
    const int want = std::max(32, std::min(256, env_la2_rows));
    cfg.cluster = static_cast<int>(ceil_div(ceil_div(d_pad, want), 4) * 4);
    cfg.rows_per_cta = static_cast<int>(ceil_div(ceil_div(d_pad, cfg.cluster), 4) * 4);
    cfg.xg = (env_la2_xg || cfg.cluster > 16) ? 1 : 0;
    if (cfg.cluster <= sm_count_dev() && (cfg.xg || max_active_clusters(cfg.cluster) >= 1)) {
      cfg.stages = 6;
      while (cfg.stages > 5 && la2::smem(cfg.rows_per_cta, cfg.stages, cfg.xg).total > 227 * 1024) --cfg.stages;
      cfg.smem = la2::smem(cfg.rows_per_cta, cfg.stages, cfg.xg).total;
      if (cfg.smem <= 227 * 1024) return cfg;
    }
  }
  // p = 1, 1024 < d <= 8192, GAPLRA_P1_XG=1 (experiment, off by default): the
  // rows spread over d / 128 plain CTAs that exchange through L2 (C2 32, C3
  // 16, C5 64 SMs).  Measured slower than the one-cluster layout (C2 18.0 vs
  // 8.8 ms, C3 30.4 vs 15.1, C5 267 (197 at 256 rows) vs 143 ms per epoch):
  // the L2 hop (publisher MEMBAR.GPU ~700 cycles + poll + loads) puts ~2000
  // cycles per block on the reducer's critical path, where the DSMEM
  // all-reduce costs ~500 (ncu: profiles/r02_ncu_v3xg.json).  GAPLRA_P1_XG_ROWS
  // sets the rows per CTA.
  static const int env_xg1 = getenv("GAPLRA_P1_XG") ? atoi(getenv("GAPLRA_P1_XG")) : 0;
  static const int env_xg_rows = getenv("GAPLRA_P1_XG_ROWS") ? atoi(getenv("GAPLRA_P1_XG_ROWS")) : 128;
  if (p == 1 && env_xg1 && env_pc == 0 && d_pad > 1024 && d_pad <= 8192) {
    EpochConfig cfg;
    cfg.b = kBlock;
    cfg.pc = 1;
    cfg.groups = 1;
    cfg.xg = 1;
    const int want = std::max(16, std::min(256, env_xg_rows));
    cfg.cluster = static_cast<int>(ceil_div(ceil_div(d_pad, want), 4) * 4);  // the peer sum runs 4 at a time
    cfg.rows_per_cta = static_cast<int>(ceil_div(ceil_div(d_pad, cfg.cluster), 4) * 4);
    if (cfg.cluster <= sm_count_dev()) {
      cfg.stages = 4;
      cfg.smem = chain_smem<1, kBlock, true>(cfg.rows_per_cta, cfg.stages).total;
      return cfg;
    }
  }
  // p = 1, 2048 < d <= 8192, GAPLRA_P1_PAIR=1 (experiment, off by default): two paired 16-CTA clusters.  The rows
  // per CTA halve (C5 256, C2 128) and the cross-cluster hop is a pairwise L2 swap of flag-in-data cells (one
  // writer, one reader per cell).  Measured slower: the swap alone costs ~1200 cycles per block on the
  // reducer's chain (C2 17.0 vs 9.1 ms, C5 177 vs 146 ms per epoch).
  static const int env_pair = getenv("GAPLRA_P1_PAIR") ? atoi(getenv("GAPLRA_P1_PAIR")) : 0;
  if (p == 1 && env_pair && env_pc == 0 && env_cluster == 0 && d_pad > 2048 && d_pad <= 8192 &&
      max_active_clusters(16) >= 2) {
    EpochConfig cfg = make(16);
    cfg.nclusters = 2;
    cfg.rows_per_cta = static_cast<int>(ceil_div(ceil_div(d_pad, 32), 4) * 4);
    cfg.stages = 4;
    cfg.smem = smem_for(cfg.pc, cfg.rows_per_cta, cfg.stages);
    return cfg;
  }
  const EpochConfig c16 = make(16), c8 = make(8);
  auto v3_ok = [](const EpochConfig& c) { return v3_supports(c.pc, c.rows_per_cta); };
  if (d_pad < 1024) return c8;
  // 8 peers instead of 16 when 8 CTAs cover the rows at <= 256 each (C3 p = 1:
  // 16.3 vs 17.5 ms per epoch: the all-reduce and its slot sum halve)
  if (v3_ok(c8) && c8.rows_per_cta <= 256) return c8;
  if (v3_ok(c16)) return c16;
  if (v3_ok(c8)) return c8;
  return c16;
}

// GAPLRA_XG_LL=0: the counter protocol for the p = 1 L2-exchange chains (default: flag-in-data cells)
int xg_ll_mode() {
  static const int v = getenv("GAPLRA_XG_LL") ? atoi(getenv("GAPLRA_XG_LL")) : 1;
  return v;
}

template <int PC>
void launch_chain_pc(const EpochArgs& a, const EpochConfig& cfg, cudaStream_t st) {
  // GAPLRA_CHAIN_MODE: 0 auto (the warp-specialised v3 where it fits: PC <= 3
  // and <= 256 rows per CTA; else scalar smem phases for PC <= 2, DMMA phases
  // above), 1 DMMA, 2 scalar smem, 3 v3.  Measured r01 on C2 (ms per epoch,
  // p = 1 / p = 20 at PC = 3): v3 9.9 / 17.6; scalar 19.1 / 29.4; DMMA 25.1 / 28.0.
  static const int env_mode = getenv("GAPLRA_CHAIN_MODE") ? atoi(getenv("GAPLRA_CHAIN_MODE")) : 0;
  const bool v3_fits = v3_supports(PC, cfg.rows_per_cta);
  const int mode = env_mode ? env_mode : (v3_fits ? 3 : (PC <= 2 ? 2 : 1));
  const bool v3 = mode == 3 && v3_fits;
  auto kern = mode == 1 ? k_svrg_chain<PC, kBlock, false> : k_svrg_chain<PC, kBlock, true>;
  if constexpr (PC <= 3) {
    if (v3) kern = k_svrg_chain_v3<PC, kBlock, 1>;
    if constexpr (PC == 1) {
      static const int env_rr = getenv("GAPLRA_CHAIN_RR") ? atoi(getenv("GAPLRA_CHAIN_RR")) : 1;
      if (v3 && env_rr && cfg.rows_per_cta <= 256) kern = k_svrg_chain_v3<1, kBlock, 1, true>;
    }
  }
  if constexpr (PC == 1) {
    static const int env_rr2 = getenv("GAPLRA_CHAIN_RR") ? atoi(getenv("GAPLRA_CHAIN_RR")) : 1;
    if (v3 && cfg.rows_per_cta > 256) kern = env_rr2 ? k_svrg_chain_v3<1, kBlock, 2, true> : k_svrg_chain_v3<1, kBlock, 2>;
  }
  int stages = cfg.stages;
  size_t smem = cfg.smem;
  // the DMMA chain v4 at PC = 8 (rows <= 512 per CTA); GAPLRA_CHAIN_MODE=4 forces it
  const bool use_v4 = PC == 8 && cfg.rows_per_cta <= 512 && (env_mode == 0 || env_mode == 4);
  const bool xg = cfg.xg != 0;
  if (use_v4) {
    stages = 2;
    for (int sN = 4; sN > 2; --sN)
      if (v4::smem(cfg.rows_per_cta, sN, xg).total <= 227 * 1024) {
        stages = sN;
        break;
      }
    smem = v4::smem(cfg.rows_per_cta, stages, xg).total;
    if (cfg.rows_per_cta > 256) {  // half-stage ring, L2 exchange
      if (!xg) throw Error(kContractViolation, "epoch: 512-row chain layout needs the L2 exchange");
      smem = v4::smem_half().total;
      kern = k_svrg_chain_v4<512, true>;
    } else {
      if (cfg.rows_per_cta <= 128)
        kern = xg ? k_svrg_chain_v4<128, true> : k_svrg_chain_v4<128, false>;
      else
        kern = xg ? k_svrg_chain_v4<256, true> : k_svrg_chain_v4<256, false>;
    }
  } else if (xg) {
    if constexpr (PC == 1) {
      if (!v3 || cfg.rows_per_cta > 256) throw Error(kContractViolation, "epoch: p = 1 L2-exchange layout needs v3 RR");
      kern = k_svrg_chain_v3<1, kBlock, 1, true, true>;
    } else {
      throw Error(kContractViolation, "epoch: L2-exchange layout needs the v4 chain or p = 1");
    }
  }
  if (v3 && !use_v4) {  // pitch ≡ 0 (mod 16) layout; up to GAPLRA_CHAIN_STAGES (<= 8) stages as fit
    static const int max_st = getenv("GAPLRA_CHAIN_STAGES") ? std::min(8, atoi(getenv("GAPLRA_CHAIN_STAGES"))) : 4;
    stages = 2;
    for (int sN = max_st; sN > 2; --sN)
      if (chain_smem<PC, kBlock, true>(cfg.rows_per_cta, sN).total <= 227 * 1024) {
        stages = sN;
        break;
      }
    smem = chain_smem<PC, kBlock, true>(cfg.rows_per_cta, stages).total;
  }
  GAPLRA_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  if (cfg.cluster > 8 && !xg)
    GAPLRA_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(cfg.cluster * std::max(1, cfg.nclusters), cfg.groups, 1);
  bool rr = false;
  if constexpr (PC == 1)
    rr = kern == k_svrg_chain_v3<1, kBlock, 1, true> || kern == k_svrg_chain_v3<1, kBlock, 2, true> ||
         kern == k_svrg_chain_v3<1, kBlock, 1, true, true>;
  lc.blockDim = dim3(use_v4 ? v4::kThreads
                            : (rr ? kV3RRThreads : (v3 ? v3_threads(PC) : kChainThreads + 32 * kChainProducers)),
                     1, 1);
  lc.dynamicSmemBytes = smem;
  lc.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cfg.cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  lc.attrs = attr;
  lc.numAttrs = xg ? 0 : 1;  // XG: plain CTAs (all co-resident: groups x cluster <= SMs, one CTA per SM)
  if (xg) {
    if (!a.xg_slot || !a.xg_count) throw Error(kContractViolation, "epoch: XG layout without exchange buffers");
    GAPLRA_CUDA_CHECK(cudaMemsetAsync(a.xg_count, 0, xg_count_elems(cfg) * sizeof(unsigned), st));
    if (xg_ll_mode() && !use_v4) GAPLRA_CUDA_CHECK(cudaMemsetAsync(a.xg_slot, 0, xg_slot_elems(cfg) * sizeof(double), st));
  }
  if (cfg.nclusters > 1) {
    if constexpr (PC == 1) {
      if (!a.xg_slot) throw Error(kContractViolation, "epoch: paired clusters without exchange buffers");
      if (use_v4 || xg) throw Error(kContractViolation, "epoch: paired clusters are a p = 1 layout");
      GAPLRA_CUDA_CHECK(cudaMemsetAsync(a.xg_slot, 0, xg_slot_elems(cfg) * sizeof(double), st));
    } else {
      throw Error(kContractViolation, "epoch: paired clusters are a p = 1 layout");
    }
  }
  EpochArgs args = a;
  static const int env_push = getenv("GAPLRA_PUSH_ASYNC") ? atoi(getenv("GAPLRA_PUSH_ASYNC")) : 1;
  args.push_async = env_push;  // p = 1 DSMEM chains: st.async push (0: staged bulk copies)
  static const int env_fr = getenv("GAPLRA_FAST_REDUCER") ? atoi(getenv("GAPLRA_FAST_REDUCER")) : 1;
  args.fast_reducer = env_fr;  // p = 1 DSMEM chains: register-preloaded reducer (0: the generic reducer loop)
  args.ncl = std::max(1, cfg.nclusters);
  args.xg_ll = xg && !use_v4 ? xg_ll_mode() : 0;
  static const int env_v4_ll = getenv("GAPLRA_V4_LL") ? atoi(getenv("GAPLRA_V4_LL")) : 0;
  if (xg && use_v4 && env_v4_ll) {  // experiment: flag-in-data cells for the v4 L2 exchange
    args.xg_ll = 2;
    GAPLRA_CUDA_CHECK(cudaMemsetAsync(a.xg_slot, 0, xg_slot_elems(cfg) * sizeof(double), st));
  }
  args.rows_per_cta = cfg.rows_per_cta;
  args.stages = stages;
  args.pc = cfg.pc;
  args.groups = cfg.groups;
  args.slab_len = epoch_slab_len(cfg);
  GAPLRA_CUDA_CHECK(cudaLaunchKernelEx(&lc, kern, args));
  GAPLRA_LAUNCH_CHECK();
}

void launch_chain_la2(const EpochArgs& a, const EpochConfig& cfg, cudaStream_t st) {
  const bool xg = cfg.xg != 0;
  auto kern = xg ? k_chain_p1_la2<true> : k_chain_p1_la2<false>;
  const size_t smem = la2::smem(cfg.rows_per_cta, cfg.stages, xg).total;
  GAPLRA_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  if (!xg && cfg.cluster > 8)
    GAPLRA_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(cfg.cluster, 1, 1);
  lc.blockDim = dim3(la2::kThreads, 1, 1);
  lc.dynamicSmemBytes = smem;
  lc.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cfg.cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  lc.attrs = attr;
  lc.numAttrs = xg ? 0 : 1;
  if (xg) {
    if (!a.xg_slot || !a.xg_count) throw Error(kContractViolation, "epoch: XG layout without exchange buffers");
    GAPLRA_CUDA_CHECK(cudaMemsetAsync(a.xg_count, 0, xg_count_elems(cfg) * sizeof(unsigned), st));
    if (xg_ll_mode()) GAPLRA_CUDA_CHECK(cudaMemsetAsync(a.xg_slot, 0, xg_slot_elems(cfg) * sizeof(double), st));
  }
  EpochArgs args = a;
  args.xg_ll = xg ? xg_ll_mode() : 0;
  args.rows_per_cta = cfg.rows_per_cta;
  args.stages = cfg.stages;
  args.pc = 1;
  args.groups = 1;
  args.slab_len = epoch_slab_len(cfg);
  args.slab_head = slab_head(cfg);
  GAPLRA_CUDA_CHECK(cudaLaunchKernelEx(&lc, kern, args));
  GAPLRA_LAUNCH_CHECK();
}

void launch_svrg_epoch_dense(const EpochArgs& a, const EpochConfig& cfg, cudaStream_t st) {
  if (cfg.smem > 227 * 1024) throw Error(kContractViolation, "epoch: d too large for the cluster row split");
  if (cfg.la == 2) {
    launch_chain_la2(a, cfg, st);
    return;
  }
  switch (cfg.pc) {
    case 1: launch_chain_pc<1>(a, cfg, st); break;
    case 2: launch_chain_pc<2>(a, cfg, st); break;
    case 3: launch_chain_pc<3>(a, cfg, st); break;
    case 4: launch_chain_pc<4>(a, cfg, st); break;
    case 6: launch_chain_pc<6>(a, cfg, st); break;
    default: launch_chain_pc<8>(a, cfg, st); break;
  }
}

void read_chain_hops(long long* out) { GAPLRA_CUDA_CHECK(cudaMemcpyFromSymbol(out, g_hop, sizeof(long long) * 64)); }

void launch_svrg_epoch_sparse(const SparseEpochArgs& a, cudaStream_t st) {
  k_svrg_epoch_sparse<<<ceil_div(a.p, 32), 32, 0, st>>>(a);
  GAPLRA_LAUNCH_CHECK();
}

namespace {
__device__ __forceinline__ uint64_t splitmix_dev(uint64_t& x) {  // rng.cpp:9-16 (the host derive_seed)
  uint64_t z = (x += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t derive_seed_dev(uint64_t root, uint64_t tag) {
  uint64_t x = root ^ (0xA0761D6478BD642Full * (tag + 1));
  const uint64_t a = splitmix_dev(x);
  const uint64_t b = splitmix_dev(x);
  return a ^ ((b << 32) | (b >> 32));
}
__global__ void k_epoch_control(const double* __restrict__ res, EpochCtl* __restrict__ ctl, double* __restrict__ hist,
                                int hist_cap, double tol, double slack, int cap, uint64_t root, int64_t solve_id,
                                cudaGraphConditionalHandle cond) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int e = ctl->e + 1;
  const double r = *res;
  if (e < hist_cap) hist[e] = r;
  int status = 0;
  if (!isfinite(r)) {
    status = 2;
  } else if (r <= tol) {
    status = 1;
  } else if (slack > 0.0 && e >= 1 && r > slack * ctl->best) {
    status = 3;
  } else {
    ctl->best = fmin(ctl->best, r);
    if (e >= cap) status = 4;
  }
  ctl->e = e;
  ctl->status = status;
  ctl->next_seed = derive_seed_dev(root, kTagSvrg ^ (static_cast<uint64_t>(solve_id) << 20) ^
                                             static_cast<uint64_t>(e + 1));
  cudaGraphSetConditional(cond, status == 0 ? 1u : 0u);
}
}  // namespace

void launch_epoch_control(const double* res, EpochCtl* ctl, double* hist, int hist_cap, double tol, double slack,
                          int cap, uint64_t root, int64_t solve_id, unsigned long long cond, cudaStream_t st) {
  k_epoch_control<<<1, 32, 0, st>>>(res, ctl, hist, hist_cap, tol, slack, cap, root, solve_id,
                                    static_cast<cudaGraphConditionalHandle>(cond));
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
