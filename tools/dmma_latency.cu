// DMMA m8n8k4 latency / throughput probe: one CTA per SM, W warps, C independent
// accumulator chains per warp; prints cycles per mma per chain and per SMSP.
#include <cstdio>
#include <cuda_runtime.h>
template <int C>
__global__ void k(double* out, int iters, long long* cyc) {
  double a = threadIdx.x * 1e-3, b = 0.5;
  double c[C][2];
#pragma unroll
  for (int i = 0; i < C; ++i) c[i][0] = c[i][1] = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < C; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < C; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
template <int C>
void run(int warps) {
  double* out; long long* cyc; cudaMalloc(&out, 8); cudaMalloc(&cyc, 8);
  const int iters = 2000;
  k<C><<<148, 32 * warps>>>(out, iters, cyc);
  cudaDeviceSynchronize();
  long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  const double per = double(h) / iters;  // cycles per iteration (C mma per warp)
  const double smsp_warps = warps / 4.0 < 1 ? 1 : warps / 4.0;
  printf("chains/warp %2d warps %2d: %.1f cycles per iter, %.1f cycles per mma per SMSP\n", C, warps, per,
         per / (C * smsp_warps));
  cudaFree(out); cudaFree(cyc);
}
int main() {
  for (int w : {1, 4, 8, 16, 32}) { run<1>(w); run<2>(w); run<4>(w); run<8>(w); }
  return 0;
}
