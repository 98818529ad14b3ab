// Shared device helpers for the sm_100a kernels of the shift-and-invert path.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

namespace gaplra_cuda {

// ---- status codes (mirror include/gaplra_cuda.h) ---------------------------
enum Status : int {
  kOk = 0,
  kContractViolation = 1,
  kRankDeficient = 2,
  kIndefiniteShift = 3,
  kSolverStalled = 4,
  kShiftOutOfRange = 5,
  kShiftTuningStalled = 6,
  kNoPreconditioningNeeded = 7,
  kDeviceError = 8,
  kOutOfMemory = 9,
  kNoUsableGap = 10,
  kDegenerateProgress = 11,
};

struct Error : std::runtime_error {
  int code;
  int payload;
  Error(int c, const std::string& what, int pl = 0) : std::runtime_error(what), code(c), payload(pl) {}
};

#define GAPLRA_CUDA_CHECK(expr)                                                              \
  do {                                                                                       \
    cudaError_t _e = (expr);                                                                 \
    if (_e != cudaSuccess) {                                                                 \
      throw ::gaplra_cuda::Error(_e == cudaErrorMemoryAllocation ? ::gaplra_cuda::kOutOfMemory \
                                                                 : ::gaplra_cuda::kDeviceError, \
                                 std::string(#expr) + ": " + cudaGetErrorString(_e) + " (" +  \
                                     __FILE__ + ":" + std::to_string(__LINE__) + ")");          \
    }                                                                                        \
  } while (0)

// Every kernel launch of the library goes through this check, which also
// counts it (gaplra_launch_count in the C ABI).
unsigned long long& launch_counter();
#define GAPLRA_LAUNCH_CHECK()                          \
  do {                                                 \
    ++::gaplra_cuda::launch_counter();                 \
    GAPLRA_CUDA_CHECK(cudaGetLastError());             \
  } while (0)

constexpr int kWarp = 32;

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// 256-bit read-only streaming load of 4 consecutive doubles (LDG.E.ENL2.256).
// `p` must be 32-byte aligned.
__device__ __forceinline__ void ldg4(const double* p, double& a, double& b, double& c, double& d) {
  asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
               : "l"(p));
}

__device__ __forceinline__ double2 ldg2(const double* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block-wide sum (fixed butterfly + fixed warp order).  `red`
// needs blockDim.x/32 doubles of shared memory.  Result broadcast to all.
__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (wid == 0) {
    t = lane < nw ? red[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) red[0] = t;
  }
  __syncthreads();
  return red[0];
}

__device__ __forceinline__ double block_max(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  if (wid == 0) {
    double t = lane < nw ? red[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t = fmax(t, __shfl_xor_sync(0xffffffffu, t, o));
    if (lane == 0) red[0] = t;
  }
  __syncthreads();
  return red[0];
}

}  // namespace gaplra_cuda
