// Latency / throughput calibration for the chain kernel's building blocks.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void lat(double* out, long long* cyc, int iters) {
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = i * 1e-3;
  __syncthreads();
  double a = threadIdx.x * 1e-6 + 1.0, b = 0.999;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) a = fma(a, b, 1e-9);  // dependent DFMA
  long long t1 = clock64();
  int idx = threadIdx.x & 7;
  for (int i = 0; i < iters; ++i) idx = (int)sm[idx] & 7;  // dependent LDS (+cvt)
  long long t2 = clock64();
  double s = a;
  for (int i = 0; i < iters; ++i) s += __shfl_xor_sync(0xffffffffu, s, 1);  // dependent shfl+add
  long long t3 = clock64();
  double c0 = 0, c1 = 0;
  for (int i = 0; i < iters; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  long long t4 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = (t1 - t0) / iters; cyc[1] = (t2 - t1) / iters; cyc[2] = (t3 - t2) / iters; cyc[3] = (t4 - t3) / iters;
  }
  out[threadIdx.x] = a + idx + s + c0 + c1;
}
__global__ void __cluster_dims__(16, 1, 1) cl16(long long* cyc, int iters, double* out) {
  __shared__ double buf[64];
  cg::cluster_group cl = cg::this_cluster();
  buf[threadIdx.x % 64] = threadIdx.x;
  cl.sync();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) cl.sync();
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = (t1 - t0) / iters;
  out[blockIdx.x] = buf[0];
}
int main() {
  double* out; long long* cyc; long long h[4];
  cudaMalloc(&out, 4096 * 8); cudaMalloc(&cyc, 64);
  for (int threads : {32, 256}) {
    lat<<<1, threads>>>(out, cyc, 4096); cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, 32, cudaMemcpyDeviceToHost);
    printf("{\"threads\": %d, \"dfma_dep\": %lld, \"lds_dep\": %lld, \"shfl_dadd_dep\": %lld, \"dmma_dep\": %lld}\n", threads, h[0], h[1], h[2], h[3]);
  }
  cudaFuncSetAttribute(cl16, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cl16<<<16, 256>>>(cyc, 2000, out); cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("{\"cluster16_sync\": %lld, \"err\": \"%s\"}\n", h[0], cudaGetErrorString(e));
}
