// Seeded index streams for the SVRG epochs (see rng.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace gaplra_cuda {

// Seed tags pinned in DESIGN.md §2.3 (the oracle uses the same values).
constexpr uint64_t kTagGauss = 0x6761757373ull;  // reference's own "gauss" (orthonormalize.cpp:17)
constexpr uint64_t kTagSvrg = 0x73767267ull;
constexpr uint64_t kTagEstA = 0x65737461ull;
constexpr uint64_t kTagEstD = 0x65737464ull;
constexpr uint64_t kTagSubspace = 0x73756273ull;

uint64_t derive_seed(uint64_t root, uint64_t tag);
uint64_t svrg_stream_seed(uint64_t root, int64_t solve_id, int epoch);

// out[k] = Rng(seed).uniform_index(n) for k < m (int32, n < 2^31).
// `rejects` is one device unsigned int of scratch.  dseed (optional): read the
// seed from device memory at run time (the device-resident epoch loop).
void launch_index_stream(uint64_t seed, uint64_t n, int64_t m, int32_t* out, unsigned int* rejects,
                         cudaStream_t st, const uint64_t* dseed = nullptr);

}  // namespace gaplra_cuda
