// Skeleton of the SVRG chain's per-block loop (16-CTA cluster, 256 threads,
// thread = row) with independent switches, to price each ingredient:
//   F_TMA   : stage ring fed by cp.async.bulk (16 slices x rc rows + 4 KB slab)
//   F_XCHG  : all-to-all st.async of 16 partials, waited one block later
//   F_COMP  : 16 LDS + products + 16-value warp halving + update FMAs
//   F_WARP0 : warp 0 sums 16 slots and a 16x16 coef between two barriers
// Prints cycles per block for each combination.
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
namespace cg = cooperative_groups;
constexpr int F_TMA = 1, F_XCHG = 2, F_COMP = 4, F_WARP0 = 8, F_LDG = 16, F_NOFENCE = 32, F_ONECOPY = 64, F_PRODW = 128;
constexpr int RC = 256, RP = 256, B = 16;

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
  uint32_t o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}
__device__ __forceinline__ void mwait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bsync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

template <int F, int S>
__global__ void __cluster_dims__(16, 1, 1) __launch_bounds__(384, 1) k(const double* X, const int* idx, int nb, long long* out) {
  extern __shared__ __align__(128) double sm[];
  double* stage = sm;                           // [S][B*RP + 512]
  double* recv = sm + S * (B * RP + 512);       // [4][16][16]
  double* red = recv + 4 * 16 * 16;             // [8][16]
  double* coef = red + 128;                     // [16]
  double* ahat = coef + 16;
  uint64_t* full = reinterpret_cast<uint64_t*>(ahat + 16);
  uint64_t* rbar = full + S;
  uint64_t* empty = rbar + 4;
  cg::cluster_group cl = cg::this_cluster();
  const int g = cl.block_rank(), tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, pm = lane >> 1;
  const size_t SL = B * RP + 512;
  if (tid == 0) {
    for (int i = 0; i < S; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 4;" ::"r"(su32(&full[i])));
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&rbar[i])));
    for (int i = 0; i < S; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(su32(&empty[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int e = tid; e < S * SL; e += 256) stage[e] = 0.001 * (e & 7);
  __syncthreads();
  auto issue = [&](int u) {  // warps 4..7, lanes 0..3: 4 slices each; warp 4 lane 31 the slab
    const int iw = (F & F_PRODW) ? warp - 8 : warp - 4, s = u % S;
    if (!(F & F_NOFENCE)) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (F & F_ONECOPY) {  // one contiguous 32 KB + slab copy per block from warp 4 lane 0
      if (iw == 0 && lane == 0) {
        expect(&full[s], (16 * RC + 512) * 8);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(stage + s * SL)),
                     "l"(X + static_cast<int64_t>(idx[u * B]) * 4096), "r"(16 * RC * 8), "r"(su32(&full[s])) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(stage + s * SL + B * RP)),
                     "l"(X), "r"(512 * 8), "r"(su32(&full[s])) : "memory");
      } else if (lane == 0) expect(&full[s], 0);
      return;
    }
    if (lane == 0) expect(&full[s], (4 * RC + (iw == 0 ? 512 : 0)) * 8);
    __syncwarp();
    if (lane < 4) {
      const int j = iw * 4 + lane;
      const double* src = X + static_cast<int64_t>(idx[u * B + j]) * 4096 + g * RC;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(stage + s * SL + j * RP)),
                   "l"(src), "r"(RC * 8), "r"(su32(&full[s])) : "memory");
    }
    if (iw == 0 && lane == 31)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(stage + s * SL + B * RP)),
                   "l"(X), "r"(512 * 8), "r"(su32(&full[s])) : "memory");
  };
  if ((F & F_TMA) && !(F & F_PRODW) && warp >= 4 && warp < 8)
    for (int u = 0; u < S && u < nb; ++u) issue(u);
  cl.sync();
  if (warp >= 8) {  // producer warps (F_PRODW)
    if (F & F_PRODW)
      for (int u = 0; u < nb; ++u) {
        if (u >= S) mwait(&empty[u % S], ((u / S) - 1) & 1);
        issue(u);
      }
    cl.sync();
    return;
  }
  double v = 1.0 + tid * 1e-6, xr[B];
  for (int i = 0; i < B; ++i) xr[i] = 0;
  // LDG feed: rows of block u+3 in flight while block u+1 is used
  double q1[B], q2[B], q3[B];
  auto ldg_block = [&](int u, double (&q)[B]) {
    for (int i = 0; i < B; ++i)
      q[i] = u < nb ? __ldcs(X + static_cast<int64_t>(__ldg(idx + u * B + (i ^ pm))) * 4096 + g * RC + tid) : 0.0;
  };
  if (F & F_LDG) { ldg_block(1, q1); ldg_block(2, q2); ldg_block(3, q3); }
  if ((F & F_XCHG) && tid == 0) expect(&rbar[0], 16 * 16 * 8);
  if (F & F_XCHG) {  // push block 0
    const uint32_t slot = su32(recv + g * 16), rb = su32(&rbar[0]);
    const int e = tid >> 4, q = tid & 15;
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(mapa(slot, q) + e * 8),
                 "l"(__double_as_longlong(v)), "r"(mapa(rb, q)) : "memory");
  }
  long long t0 = clock64();
  for (int t = 0; t < nb; ++t) {
    const bool more = t + 1 < nb;
    if ((F & F_XCHG) && tid == 0 && more) expect(&rbar[(t + 1) & 3], 16 * 16 * 8);
    if ((F & F_TMA) && !(F & F_PRODW) && warp >= 4 && t >= 1 && t - 1 + S < nb) issue(t - 1 + S);
    if ((F & F_PRODW) && t >= 1 && lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[(t - 1) % S])) : "memory");
    const double* xb = stage + ((t + 1) % S) * SL;
    if ((F & F_TMA) && more) mwait(&full[(t + 1) % S], ((t + 1) / S) & 1);
    if (F & F_COMP) {
      double xn[B], val[B];
      if (F & F_LDG) {
        for (int i = 0; i < B; ++i) { xn[i] = q1[i]; q1[i] = q2[i]; q2[i] = q3[i]; }
        ldg_block(t + 4, q3);
      } else
        for (int i = 0; i < B; ++i) xn[i] = xb[(i ^ pm) * RP + tid];
      for (int i = 0; i < B; ++i) val[i] = xn[i] * v;
      for (int o = 16, n = B / 2; o >= 2; o >>= 1, n >>= 1)
        for (int i = 0; i < n; ++i) val[i] += __shfl_xor_sync(0xffffffffu, val[i + n], o);
      val[0] += __shfl_xor_sync(0xffffffffu, val[0], 1);
      if (!(lane & 1)) red[warp * 16 + pm] = val[0];
      for (int i = 0; i < B; ++i) {
        const double tmp = xr[i];
        xr[i] = xn[i];
        xn[i] = tmp;
      }
    }
    bsync();
    if ((F & F_XCHG) && more) {
      const int par = (t + 1) & 3, e = tid >> 4, q = tid & 15;
      const uint32_t slot = su32(recv + (par * 16 + g) * 16), rb = su32(&rbar[par]);
      double s = 0;
      for (int w = 0; w < 8; ++w) s += red[w * 16 + e];
      asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(mapa(slot, q) + e * 8),
                   "l"(__double_as_longlong(s)), "r"(mapa(rb, q)) : "memory");
    }
    if (warp == 0) {
      if (F & F_XCHG) mwait(&rbar[t & 3], (t >> 2) & 1);
      if (F & F_WARP0) {
        if (lane < 16) {
          double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
          const double* sl = recv + (t & 3) * 256 + lane;
          for (int q = 0; q < 16; q += 4) {
            s0 += sl[q * 16];
            s1 += sl[(q + 1) * 16];
            s2 += sl[(q + 2) * 16];
            s3 += sl[(q + 3) * 16];
          }
          ahat[lane] = (s0 + s1) + (s2 + s3);
        }
        __syncwarp();
        if (lane < 16) {
          double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
          const double* TT = stage + (t % S) * SL + B * RP;
          for (int l = 0; l < 16; l += 4) {
            s0 = fma(TT[l * 16 + lane], ahat[l], s0);
            s1 = fma(TT[(l + 1) * 16 + lane], ahat[l + 1], s1);
            s2 = fma(TT[(l + 2) * 16 + lane], ahat[l + 2], s2);
            s3 = fma(TT[(l + 3) * 16 + lane], ahat[l + 3], s3);
          }
          coef[lane] = ((s0 + s1) + (s2 + s3)) * 1e-3;
        }
      }
    }
    bsync();
    if (F & F_COMP) {
      double w2 = 0;
      for (int i = 0; i < B; i += 2) {
        v = fma(xr[i], coef[i ^ pm], v);
        w2 = fma(xr[i + 1], coef[(i + 1) ^ pm], w2);
      }
      v = (v + w2) * 0.999;
    }
  }
  long long t1 = clock64();
  if (tid == 0 && g == 0) out[0] = (t1 - t0) / nb;
  if (v == 12345.0) out[1] = 1;
  cl.sync();
}

template <int F, int S = 4>
void run(const double* X, const int* idx, int nb, long long* d, const char* tag = "") {
  const size_t smem = (S * (B * RP + 512) + 4 * 256 + 128 + 32) * 8 + 256;
  cudaFuncSetAttribute(k<F, S>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k<F, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  k<F, S><<<16, (F & F_PRODW) ? 384 : 256, smem>>>(X, idx, nb, d);
  printf("%s S=%d ", tag, S);
  long long h = -1;
  cudaError_t e = cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("{\"tma\": %d, \"xchg\": %d, \"comp\": %d, \"warp0\": %d, \"cycles_per_block\": %lld, \"err\": \"%s\"}\n", !!(F & F_TMA),
         !!(F & F_XCHG), !!(F & F_COMP), !!(F & F_WARP0), h, cudaGetErrorString(e));
  fflush(stdout);
}
int main_old(double** pX, int** pidx, long long** pd) {
  const int n = 100000, nb = 12500;
  double* X;
  int* idx;
  long long* d;
  cudaMalloc(&X, static_cast<size_t>(n) * 4096 * 8);
  cudaMemset(X, 0, static_cast<size_t>(n) * 4096 * 8);
  cudaMalloc(&idx, nb * 16 * 4);
  int* h = new int[nb * 16];
  uint64_t st = 88172645463325252ull;
  for (int i = 0; i < nb * 16; ++i) {
    st ^= st << 13; st ^= st >> 7; st ^= st << 17;
    h[i] = static_cast<int>(st % n);
  }
  cudaMemcpy(idx, h, nb * 16 * 4, cudaMemcpyHostToDevice);
  int* idx_small;  // 2000 columns = 64 MB: L2-resident
  cudaMalloc(&idx_small, nb * 16 * 4);
  for (int i = 0; i < nb * 16; ++i) h[i] %= 2000;
  cudaMemcpy(idx_small, h, nb * 16 * 4, cudaMemcpyHostToDevice);
  cudaMalloc(&d, 256);
  *pX = X; *pidx = idx; *pd = d;
  return 0;
  run<F_TMA, 4>(X, idx, nb, d, "tma");
  run<F_TMA | F_NOFENCE, 4>(X, idx, nb, d, "tma-nofence");
  run<F_TMA | F_ONECOPY, 4>(X, idx, nb, d, "tma-onecopy");
  run<F_TMA | F_PRODW, 4>(X, idx, nb, d, "tma-prodwarps");
  run<F_TMA | F_PRODW | F_XCHG | F_COMP | F_WARP0, 4>(X, idx, nb, d, "prodw-all");
  run<F_TMA | F_XCHG | F_COMP | F_WARP0, 4>(X, idx, nb, d, "inline-all");
  run<F_TMA | F_NOFENCE | F_XCHG | F_COMP | F_WARP0, 4>(X, idx, nb, d, "inline-nofence-all");
  return 0;
}

// ---- reducer-warp skeleton: warps 0..7 rows, warp 8 reducer (d + a), warp 9 producer
template <int S, bool NOX = false>
__global__ void __cluster_dims__(16, 1, 1) __launch_bounds__(320, 1) k3(const double* X, const int* idx, int nb, long long* out) {
  extern __shared__ __align__(128) double sm[];
  const size_t SL = B * RP + 512;
  double* stage = sm;
  double* recv = sm + S * SL;          // [4][16][16]
  double* red = recv + 4 * 256;        // [8][16]
  double* coef = red + 128;            // [2][16]
  double* ahat = coef + 32;            // [16]
  uint64_t* full = reinterpret_cast<uint64_t*>(ahat + 16);
  uint64_t* empty = full + S;
  uint64_t* rbar = empty + S;
  cg::cluster_group cl = cg::this_cluster();
  const int g = cl.block_rank(), tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, pm = lane >> 1;
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 9;" ::"r"(su32(&empty[i])));
    }
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&rbar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int e = tid; e < S * SL; e += 320) stage[e] = 0.001 * (e & 7);
  for (int e = tid; e < 32; e += 320) coef[e] = 0.0;
  __syncthreads();
  cl.sync();
  long long t0 = clock64();
  long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tp = clock64();
  auto tk = [&](int k) {
    long long now;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(now)::"memory");
    ph[k] += now - tp;
    tp = now;
  };
  if (warp == 9) {  // producer: 16 slices + slab per block, one warp
    for (int u = 0; u < nb; ++u) {
      const int s = u % S;
      if (u >= S) mwait(&empty[s], ((u / S) - 1) & 1);
      if (lane == 0) expect(&full[s], NOX ? 0 : (16 * RC + 512) * 8);
      __syncwarp();
      if (NOX) continue;
      if (lane < 16) {
        const double* src = X + static_cast<int64_t>(idx[u * B + lane]) * 4096 + g * RC;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(stage + s * SL + lane * RP)),
                     "l"(src), "r"(RC * 8), "r"(su32(&full[s])) : "memory");
      }
      if (lane == 31)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(stage + s * SL + B * RP)),
                     "l"(X), "r"(512 * 8), "r"(su32(&full[s])) : "memory");
    }
  } else if (warp == 8) {  // reducer: Â_t -> coef_t (double-buffered), arrive on the coef barrier
    if (lane == 0) expect(&rbar[0], 16 * 16 * 8);
    for (int t = 0; t < nb; ++t) {
      if (lane == 0 && t + 1 < nb) expect(&rbar[(t + 1) & 3], 16 * 16 * 8);
      tk(0);
      mwait(&full[t % S], (t / S) & 1);
      tk(1);
      mwait(&rbar[t & 3], (t >> 2) & 1);
      tk(2);
      if (lane < 16) {
        double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
        const double* sl = recv + (t & 3) * 256 + lane;
        for (int q = 0; q < 16; q += 4) {
          s0 += sl[q * 16];
          s1 += sl[(q + 1) * 16];
          s2 += sl[(q + 2) * 16];
          s3 += sl[(q + 3) * 16];
        }
        ahat[lane] = (s0 + s1) + (s2 + s3);
      }
      __syncwarp();
      tk(3);
      if (lane < 16) {
        double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
        const double* TT = stage + (t % S) * SL + B * RP;
        for (int l = 0; l < 16; l += 4) {
          s0 = fma(TT[l * 16 + lane], ahat[l], s0);
          s1 = fma(TT[(l + 1) * 16 + lane], ahat[l + 1], s1);
          s2 = fma(TT[(l + 2) * 16 + lane], ahat[l + 2], s2);
          s3 = fma(TT[(l + 3) * 16 + lane], ahat[l + 3], s3);
        }
        coef[(t & 1) * 16 + lane] = ((s0 + s1) + (s2 + s3)) * 1e-3;
      }
      tk(4);
      asm volatile("bar.arrive 2, 288;" ::: "memory");  // coef_t ready
      __syncwarp();
      tk(5);
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[t % S])) : "memory");
    }
  } else {  // row warps
    double v = 1.0 + tid * 1e-6, xr[B];
    {  // Â_0 push
      mwait(&full[0], 0);
      if (tid == 0) {}
      const int e = tid >> 4, q = tid & 15;
      asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(mapa(su32(recv + g * 16), q) + e * 8),
                   "l"(__double_as_longlong(v)), "r"(mapa(su32(&rbar[0]), q)) : "memory");
      for (int i = 0; i < B; ++i) xr[i] = stage[(i ^ pm) * RP + tid];
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[0])) : "memory");
    }
    for (int t = 0; t < nb; ++t) {
      const bool more = t + 1 < nb;
      double xn[B];
      tk(0);
      if (more) {
        mwait(&full[(t + 1) % S], ((t + 1) / S) & 1);
        tk(1);
        const double* xb = stage + ((t + 1) % S) * SL;
        double val[B];
        for (int i = 0; i < B; ++i) xn[i] = xb[(i ^ pm) * RP + tid];
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[(t + 1) % S])) : "memory");
        for (int i = 0; i < B; ++i) val[i] = xn[i] * v;
        for (int o = 16, n = B / 2; o >= 2; o >>= 1, n >>= 1)
          for (int i = 0; i < n; ++i) val[i] += __shfl_xor_sync(0xffffffffu, val[i + n], o);
        val[0] += __shfl_xor_sync(0xffffffffu, val[0], 1);
        if (!(lane & 1)) red[warp * 16 + pm] = val[0];
        tk(2);
        asm volatile("bar.sync 1, 256;" ::: "memory");
        tk(3);
        const int par = (t + 1) & 3, e = tid >> 4, q = tid & 15;
        double s = 0;
        for (int w = 0; w < 8; ++w) s += red[w * 16 + e];
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(mapa(su32(recv + (par * 16 + g) * 16), q) + e * 8),
                     "l"(__double_as_longlong(s)), "r"(mapa(su32(&rbar[par]), q)) : "memory");
      }
      tk(4);
      asm volatile("bar.sync 2, 288;" ::: "memory");  // coef_t ready (reducer arrives)
      tk(5);
      double w2 = 0;
      const double* cf = coef + (t & 1) * 16;
      for (int i = 0; i < B; i += 2) {
        v = fma(xr[i], cf[i ^ pm], v);
        w2 = fma(xr[i + 1], cf[(i + 1) ^ pm], w2);
      }
      v = (v + w2) * 0.999;
      for (int i = 0; i < B; ++i) xr[i] = xn[i];
      tk(6);
    }
    if (v == 12345.0) out[1] = 1;
  }
  long long t1 = clock64();
  if (tid == 0 && g == 0) out[0] = (t1 - t0) / nb;
  if ((tid == 0 || tid == 256) && g == 0)
    for (int k = 0; k < 8; ++k) out[2 + (tid == 256 ? 8 : 0) + k] = ph[k] / nb;
  cl.sync();
}
template <int S, bool NOX = false>
void run3(const double* X, const int* idx, int nb, long long* d) {
  const size_t smem = (S * (B * RP + 512) + 4 * 256 + 128 + 64) * 8 + 256;
  cudaError_t e1 = cudaFuncSetAttribute(k3<S, NOX>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaError_t e2 = cudaFuncSetAttribute(k3<S, NOX>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  k3<S, NOX><<<16, 320, smem>>>(X, idx, nb, d);
  printf("attr %s %s launch %s smem %zu\n", cudaGetErrorString(e1), cudaGetErrorString(e2), cudaGetErrorString(cudaGetLastError()), smem);
  long long h = -1;
  cudaError_t e = cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("reducer-warp nox=%d S=%d cycles_per_block %lld err %s\n", (int)NOX, S, h, cudaGetErrorString(e));
  long long hp[16];
  cudaMemcpy(hp, d + 2, 16 * 8, cudaMemcpyDeviceToHost);
  printf("  row warp0 [top, wait_full, load+products, bar1, push, bar2(coef), update]:");
  for (int k = 0; k < 7; ++k) printf(" %lld", hp[k]);
  printf("\n  reducer [top, wait_full, wait_rbar, sum, coef, arrive]:");
  for (int k = 0; k < 6; ++k) printf(" %lld", hp[8 + k]);
  printf("\n");
  fflush(stdout);
}

// ---- k4: 4 row warps x 2 rows/thread (LDS.128), warp 4 reducer, warp 5 producer
template <int S, int NP = 1>
__global__ void __cluster_dims__(16, 1, 1) __launch_bounds__(256, 1) k4(const double* X, const int* idx, int nb, long long* out) {
  extern __shared__ __align__(128) double sm[];
  const size_t SL = B * RP + 512;
  double* stage = sm;
  double* recv = sm + S * SL;          // [4][16][16]
  double* red = recv + 4 * 256;        // [4][16]
  double* coef = red + 64;             // [2][16]
  double* ahat = coef + 32;            // [16]
  uint64_t* full = reinterpret_cast<uint64_t*>(ahat + 16);
  uint64_t* empty = full + S;
  uint64_t* rbar = empty + S;
  cg::cluster_group cl = cg::this_cluster();
  const int g = cl.block_rank(), tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, pm = lane >> 1;
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[i])), "r"(NP));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 5;" ::"r"(su32(&empty[i])));
    }
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&rbar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int e = tid; e < S * SL; e += blockDim.x) stage[e] = 0.001 * (e & 7);
  for (int e = tid; e < 32; e += blockDim.x) coef[e] = 0.0;
  __syncthreads();
  cl.sync();
  long long t0 = clock64();
  long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tp = clock64();
  auto tk = [&](int k) {
    long long now;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(now)::"memory");
    ph[k] += now - tp;
    tp = now;
  };
  if (warp >= 5) {
    const int pw = warp - 5, per = 16 / NP;
    for (int u = 0; u < nb; ++u) {
      const int s = u % S;
      if (u >= S) mwait(&empty[s], ((u / S) - 1) & 1);
      if (lane == 0) expect(&full[s], (per * RC + (pw == 0 ? 512 : 0)) * 8);
      __syncwarp();
      if (lane < per) {
        const int jj = pw * per + lane;
        const double* src = X + static_cast<int64_t>(idx[u * B + jj]) * 4096 + g * RC;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(stage + s * SL + jj * RP)),
                     "l"(src), "r"(RC * 8), "r"(su32(&full[s])) : "memory");
      }
      if (lane == 31 && pw == 0)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(stage + s * SL + B * RP)),
                     "l"(X), "r"(512 * 8), "r"(su32(&full[s])) : "memory");
    }
  } else if (warp == 4) {
    if (lane == 0) expect(&rbar[0], 16 * 16 * 8);
    for (int t = 0; t < nb; ++t) {
      if (lane == 0 && t + 1 < nb) expect(&rbar[(t + 1) & 3], 16 * 16 * 8);
      tk(0);
      mwait(&full[t % S], (t / S) & 1);
      tk(1);
      mwait(&rbar[t & 3], (t >> 2) & 1);
      tk(2);
      double a = 0;
      if (lane < 16) {
        double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
        const double* sl = recv + (t & 3) * 256 + lane;
        for (int q = 0; q < 16; q += 4) {
          s0 += sl[q * 16];
          s1 += sl[(q + 1) * 16];
          s2 += sl[(q + 2) * 16];
          s3 += sl[(q + 3) * 16];
        }
        a = (s0 + s1) + (s2 + s3);
      }
      tk(3);
      {  // coef via shuffles of Â (no smem round trip)
        double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
        const double* TT = stage + (t % S) * SL + B * RP;
        const int j = lane & 15;
        for (int l = 0; l < 16; l += 4) {
          s0 = fma(TT[l * 16 + j], __shfl_sync(0xffffffffu, a, l), s0);
          s1 = fma(TT[(l + 1) * 16 + j], __shfl_sync(0xffffffffu, a, l + 1), s1);
          s2 = fma(TT[(l + 2) * 16 + j], __shfl_sync(0xffffffffu, a, l + 2), s2);
          s3 = fma(TT[(l + 3) * 16 + j], __shfl_sync(0xffffffffu, a, l + 3), s3);
        }
        if (lane < 16) coef[(t & 1) * 16 + lane] = ((s0 + s1) + (s2 + s3)) * 1e-3;
      }
      tk(4);
      asm volatile("bar.arrive 2, 160;" ::: "memory");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[t % S])) : "memory");
      tk(5);
    }
  } else {  // 4 row warps, rows 2 tid, 2 tid + 1
    double v0 = 1.0 + tid * 1e-6, v1 = 1.0 - tid * 1e-6;
    double2 xa[B], xb2[B];
    mwait(&full[0], 0);
    for (int i = 0; i < B; ++i) xa[i] = *reinterpret_cast<const double2*>(stage + (i ^ pm) * RP + 2 * tid);
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[0])) : "memory");
    for (int rep = tid; rep < 256; rep += 128) {
      const int e = rep >> 4, q = rep & 15;
      asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(mapa(su32(recv + g * 16), q) + e * 8),
                   "l"(__double_as_longlong(v0)), "r"(mapa(su32(&rbar[0]), q)) : "memory");
    }
    auto step = [&](int t, double2 (&xr)[B], double2 (&xn)[B]) {
      const bool more = t + 1 < nb;
      tk(0);
      if (more) {
        mwait(&full[(t + 1) % S], ((t + 1) / S) & 1);
        tk(1);
        const double* xb = stage + ((t + 1) % S) * SL;
        double val[B];
        for (int i = 0; i < B; ++i) xn[i] = *reinterpret_cast<const double2*>(xb + (i ^ pm) * RP + 2 * tid);
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[(t + 1) % S])) : "memory");
        for (int i = 0; i < B; ++i) val[i] = fma(xn[i].x, v0, xn[i].y * v1);
        for (int o = 16, n = B / 2; o >= 2; o >>= 1, n >>= 1)
          for (int i = 0; i < n; ++i) val[i] += __shfl_xor_sync(0xffffffffu, val[i + n], o);
        val[0] += __shfl_xor_sync(0xffffffffu, val[0], 1);
        if (!(lane & 1)) red[warp * 16 + pm] = val[0];
        tk(2);
        asm volatile("bar.sync 1, 128;" ::: "memory");
        tk(3);
        const int par = (t + 1) & 3;
        for (int rep = tid; rep < 256; rep += 128) {
          const int e = rep >> 4, q = rep & 15;
          const double s = (red[e] + red[16 + e]) + (red[32 + e] + red[48 + e]);
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(mapa(su32(recv + (par * 16 + g) * 16), q) + e * 8),
                       "l"(__double_as_longlong(s)), "r"(mapa(su32(&rbar[par]), q)) : "memory");
        }
      }
      tk(4);
      asm volatile("bar.sync 2, 160;" ::: "memory");
      tk(5);
      const double* cf = coef + (t & 1) * 16;
      double a0 = 0, a1 = 0;
      for (int i = 0; i < B; ++i) {
        const double c = cf[i ^ pm];
        v0 = fma(xr[i].x, c, v0);
        v1 = fma(xr[i].y, c, v1);
      }
      v0 = (v0 + a0) * 0.999;
      v1 = (v1 + a1) * 0.999;
      tk(6);
    };
    int t = 0;
    for (; t + 1 < nb; t += 2) {
      step(t, xa, xb2);
      step(t + 1, xb2, xa);
    }
    if (t < nb) step(t, xa, xb2);
    if (v0 + v1 == 12345.0) out[1] = 1;
  }
  long long t1 = clock64();
  if (tid == 0 && g == 0) out[0] = (t1 - t0) / nb;
  if ((tid == 0 || tid == 128) && g == 0)
    for (int k = 0; k < 8; ++k) out[2 + (tid == 128 ? 8 : 0) + k] = ph[k] / nb;
  cl.sync();
}
template <int S, int NP = 1>
void run4(const double* X, const int* idx, int nb, long long* d) {
  const size_t smem = (S * (B * RP + 512) + 4 * 256 + 64 + 64) * 8 + 256;
  cudaFuncSetAttribute(k4<S, NP>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k4<S, NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  k4<S, NP><<<16, 160 + 32 * NP, smem>>>(X, idx, nb, d);
  long long h = -1;
  cudaError_t e = cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("k4 S=%d NP=%d cycles_per_block %lld err %s\n", S, NP, h, cudaGetErrorString(e));
  long long hp[16];
  cudaMemcpy(hp, d + 2, 16 * 8, cudaMemcpyDeviceToHost);
  printf("  row warp0 [top, wait_full, load+products, bar1, push, bar2(coef), update]:");
  for (int k = 0; k < 7; ++k) printf(" %lld", hp[k]);
  printf("\n  reducer [top, wait_full, wait_rbar, sum, coef, arrive]:");
  for (int k = 0; k < 6; ++k) printf(" %lld", hp[8 + k]);
  printf("\n");
  fflush(stdout);
}

int main() {
  double* X; int* idx; long long* d;
  main_old(&X, &idx, &d);
  run3<4>(X, idx, 12500, d);
  run4<4, 1>(X, idx, 12500, d);
  run4<4, 2>(X, idx, 12500, d);
  run4<4, 4>(X, idx, 12500, d);
  run4<5, 2>(X, idx, 12500, d);
  return 0;
}
