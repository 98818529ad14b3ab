// Microbenchmark of the chain's cluster exchange: 16 CTAs, 256 threads, every
// block (iteration) each CTA pushes NV doubles to every peer with st.async
// (8 B or 16 B messages, issued by all threads or by one warp) and waits for
// its own NV x 16 incoming values on an mbarrier.  Prints cycles/iteration.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
  uint32_t o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(su32(b)), "r"(ph) : "memory");
}
template <int NV, int MODE>
__global__ void __cluster_dims__(16, 1, 1) __launch_bounds__(256, 1) k(int iters, long long* out) {
  __shared__ __align__(16) double recv[4][16][NV];
  __shared__ double own[4][16][(NV + 15) / 16];
  __shared__ __align__(16) double outv[4][NV];
  __shared__ __align__(8) uint64_t bar[4], bar2[4];
  cg::cluster_group cl = cg::this_cluster();
  const int g = cl.block_rank(), tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])));
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar2[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cl.sync();
  long long t0 = clock64();
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    const int par = it & 3;
    constexpr int OWN = (NV + 15) / 16;  // entries owned per CTA (reduce-scatter)
    if (tid == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[par])), "r"((MODE == 3 ? 1 : 16) * NV * 8) : "memory");
      if (MODE == 3)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar2[par])), "r"(16 * OWN * 8) : "memory");
    }
    asm volatile("bar.sync 1, 256;" ::: "memory");
    const uint32_t slot = su32(&recv[par][g][0]), rb = su32(&bar[par]);
    if (MODE == 0) {  // all threads, 8-byte messages
      for (int i = tid; i < NV * 16; i += 256) {
        const int e = i >> 4, q = i & 15;
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(mapa(slot, q) + e * 8),
                     "l"(__double_as_longlong(acc + e)), "r"(mapa(rb, q)) : "memory");
      }
    } else if (MODE == 1) {  // all threads, 16-byte messages
      for (int i = tid; i < NV * 8; i += 256) {
        const int e = (i >> 4) * 2, q = i & 15;
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(mapa(slot, q) + e * 8),
                     "d"(acc + e), "d"(acc), "r"(mapa(rb, q)) : "memory");
      }
    } else if (MODE == 2) {  // warp 0 only, 16 lanes = peers, 16-byte messages
      if (tid < 16)
        for (int e = 0; e < NV; e += 2)
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(mapa(slot, tid) + e * 8),
                       "d"(acc + e), "d"(acc), "r"(mapa(rb, tid)) : "memory");
    }
    else if (MODE == 3) {  // reduce-scatter to the owner, owner all-gathers the totals
      const uint32_t o2 = su32(&own[par][g][0]), b2 = su32(&bar2[par]);
      if (tid < NV) {  // entry e -> owner e % 16, position e / 16
        const int q = tid & 15, k = tid >> 4;
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(mapa(o2, q) + k * 8),
                     "l"(__double_as_longlong(acc + tid)), "r"(mapa(b2, q)) : "memory");
      }
      wait(&bar2[par], (it >> 2) & 1);
      if (tid < 16 * OWN) {  // thread (k, q): total of owned entry k -> peer q
        const int k = tid >> 4, q = tid & 15, e = k * 16 + g;
        double s = 0;
        for (int p = 0; p < 16; ++p) s += own[par][p][k];
        if (e < NV)
          for (int pp = 0; pp < 1; ++pp)
            asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(mapa(slot, q) + e * 8),
                         "l"(__double_as_longlong(s)), "r"(mapa(rb, q)) : "memory");
      }
    }
    else if (MODE == 4 || MODE == 5) {  // bulk smem -> remote smem copy per peer
      if (tid < NV) outv[par][tid] = acc + tid;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("bar.sync 1, 256;" ::: "memory");
      const int lanes = MODE == 4 ? 16 : 2;  // MODE 4: warp 0 lanes 0..15; MODE 5: 2 lanes in each of 8 warps
      const int w = tid >> 5, l = tid & 31;
      if (l < lanes && (MODE == 4 ? w == 0 : true)) {
        const int q = MODE == 4 ? l : w * 2 + l;
        asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(mapa(slot, q)),
                     "r"(su32(&outv[par][0])), "r"(NV * 8), "r"(mapa(rb, q)) : "memory");
      }
    }
    wait(&bar[par], (it >> 2) & 1);
    acc += recv[par][(g + 1) & 15][tid % NV];
  }
  long long t1 = clock64();
  if (tid == 0 && g == 0) out[0] = (t1 - t0) / iters;
  if (acc == 12345.0) out[1] = 1;
  cl.sync();
}
template <int NV, int MODE>
void run(long long* d) {
  k<NV, MODE><<<16, 256>>>(20000, d);
  long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("{\"nv\": %d, \"mode\": %d, \"cycles_per_exchange\": %lld}\n", NV, MODE, h);
  fflush(stdout);
}
int main() {
  long long* d;
  cudaMalloc(&d, 16);
#define ALLOW(N, M) cudaFuncSetAttribute(k<N, M>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)
  ALLOW(1, 0); ALLOW(2, 0); ALLOW(4, 0); ALLOW(8, 0); ALLOW(16, 3); ALLOW(48, 3);
  run<1, 0>(d); run<2, 0>(d); run<4, 0>(d); run<8, 0>(d);
  cudaFuncSetAttribute(k<16, 0>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k<16, 1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k<16, 2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k<48, 0>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k<48, 1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k<48, 2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  run<16, 0>(d); run<16, 1>(d); run<16, 2>(d);
  run<48, 0>(d); run<48, 1>(d); run<48, 2>(d);
  run<16, 3>(d); run<48, 3>(d);
  ALLOW(16, 4); ALLOW(48, 4); ALLOW(16, 5); ALLOW(48, 5); ALLOW(2, 4);
  run<2, 4>(d); run<16, 4>(d); run<48, 4>(d); run<16, 5>(d); run<48, 5>(d);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
