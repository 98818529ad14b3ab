// Microbenchmarks that set the roofline denominators and the kernel design:
// FP64 DFMA and DMMA (mma.sync m8n8k4 f64) throughput, L2 re-read bandwidth,
// HBM streaming read bandwidth, cluster barrier + DSMEM latency.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

namespace cg = cooperative_groups;

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 0.5;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void read_kernel(const double2* __restrict__ in, size_t n2, int reps, double* out) {
  double acc = 0;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) {
      double2 v = __ldcg(in + i);
      acc += v.x + v.y;
    }
  if (acc == 12345.678) out[0] = acc;
}

__global__ void __cluster_dims__(8, 1, 1) cluster_sync_kernel(int iters, long long* cycles, double* out) {
  __shared__ double buf[64];
  cg::cluster_group cl = cg::this_cluster();
  buf[threadIdx.x % 64] = threadIdx.x;
  cl.sync();
  long long t0 = clock64();
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    double* remote = cl.map_shared_rank(buf, (cl.block_rank() + 1) % 8);
    acc += remote[threadIdx.x % 64];
    cl.sync();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) cycles[0] = (t1 - t0) / iters;
  if (acc == 12345.678) out[0] = acc;
}

float time_it(void (*launch)(void*), void* arg, int reps) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  launch(arg);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a));
  for (int i = 0; i < reps; ++i) launch(arg);
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms;
  CK(cudaEventElapsedTime(&ms, a, b));
  return ms / reps;
}

struct Args {
  double* out;
  const double2* buf;
  size_t n2;
  int iters, reps, grid, block;
};

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  const int sms = prop.multiProcessorCount;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"l2_bytes\": %d}\n", prop.name, sms, prop.l2CacheSize);
  double* out;
  CK(cudaMalloc(&out, 64));
  Args A{};
  A.out = out;

  // DFMA: grid = sms*4 blocks x 256 threads, 16 independent chains per thread.
  A.iters = 20000;
  A.grid = sms * 4;
  A.block = 256;
  float ms = time_it([](void* p) {
    Args* a = (Args*)p;
    dfma_kernel<<<a->grid, a->block>>>(a->out, a->iters, 0.999999, 1e-7);
  }, &A, 5);
  double fl = 2.0 * 16 * (double)A.iters * A.grid * A.block;
  printf("{\"dfma_tflops\": %.2f, \"ms\": %.3f}\n", fl / ms / 1e9, ms);

  A.iters = 20000;
  ms = time_it([](void* p) {
    Args* a = (Args*)p;
    dmma_kernel<<<a->grid, a->block>>>(a->out, a->iters);
  }, &A, 5);
  fl = 2.0 * 256 * 8 * (double)A.iters * A.grid * (A.block / 32);
  printf("{\"dmma_tflops\": %.2f, \"ms\": %.3f}\n", fl / ms / 1e9, ms);

  // L2 re-read bandwidth: 64 MB buffer read 20x; HBM: 4 GB buffer read once.
  for (size_t mb : {32, 64, 96, 4096}) {
    size_t bytes = mb << 20;
    double2* buf;
    CK(cudaMalloc(&buf, bytes));
    CK(cudaMemset(buf, 0, bytes));
    A.buf = buf;
    A.n2 = bytes / 16;
    A.reps = mb <= 96 ? 20 : 1;
    A.grid = sms * 8;
    A.block = 512;
    ms = time_it([](void* p) {
      Args* a = (Args*)p;
      read_kernel<<<a->grid, a->block>>>(a->buf, a->n2, a->reps, a->out);
    }, &A, 5);
    printf("{\"read_buffer_mb\": %zu, \"gbs\": %.1f}\n", mb, (double)bytes * A.reps / ms / 1e6);
    CK(cudaFree(buf));
  }

  long long* cyc;
  CK(cudaMalloc(&cyc, 8));
  cluster_sync_kernel<<<sms / 8 * 8, 64>>>(1000, cyc, out);
  CK(cudaDeviceSynchronize());
  long long hc;
  CK(cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost));
  printf("{\"cluster8_sync_plus_dsmem_cycles\": %lld}\n", hc);
  return 0;
}
