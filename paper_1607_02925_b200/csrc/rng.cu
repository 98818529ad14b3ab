// Device replay of the reference's SVRG index stream, bit-exact.
//
// The stream is Rng(seed).uniform_index(n) repeated m times
// (proj/core/src/rng.cpp:23-38 xoshiro256++ seeded by splitmix64, and
// rng.cpp:61-69 rejection sampling draw % n with limit = n * floor((2^64-1)/n)).
// xoshiro256's state transition is linear over GF(2), so the state after k
// steps is T^k s0 for a 256x256 bit matrix T.  The host precomputes
// J_l = T^(chunk * 2^l); thread t jumps to state T^(t*chunk) s0 by applying
// J_l for every set bit l of t, then emits its `chunk` draws.  Rejected draws
// (probability < n / 2^64 per draw) are counted; if any occurred anywhere, a
// fix-up kernel regenerates the stream serially, so the output is exact in
// every case.
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "common.cuh"
#include "rng.cuh"

namespace gaplra_cuda {

namespace {

struct State {
  uint64_t s[4];
};

__host__ __device__ inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

__host__ __device__ inline uint64_t splitmix(uint64_t& x) {
  x += 0x9E3779B97F4A7C15ull;
  uint64_t z = x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__host__ __device__ inline State seed_state(uint64_t seed) {
  State st;
  uint64_t t = seed;
  for (int i = 0; i < 4; ++i) st.s[i] = splitmix(t);
  return st;
}

__host__ __device__ inline uint64_t next(State& st) {
  uint64_t* s = st.s;
  const uint64_t out = rotl(s[0] + s[3], 23) + s[0];
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl(s[3], 45);
  return out;
}

// Column-major GF(2) matrix: cols[i] = image of basis state e_i.
struct BitMat {
  State cols[256];
};

State apply(const BitMat& m, const State& v) {
  State o{{0, 0, 0, 0}};
  for (int i = 0; i < 256; ++i)
    if ((v.s[i >> 6] >> (i & 63)) & 1ull)
      for (int w = 0; w < 4; ++w) o.s[w] ^= m.cols[i].s[w];
  return o;
}

BitMat compose(const BitMat& a, const BitMat& b) {  // a ∘ b
  BitMat o;
  for (int i = 0; i < 256; ++i) o.cols[i] = apply(a, b.cols[i]);
  return o;
}

BitMat step_matrix() {
  BitMat m;
  for (int i = 0; i < 256; ++i) {
    State e{{0, 0, 0, 0}};
    e.s[i >> 6] = 1ull << (i & 63);
    next(e);
    m.cols[i] = e;
  }
  return m;
}

BitMat power(BitMat base, uint64_t e) {
  BitMat r;
  for (int i = 0; i < 256; ++i) {
    State v{{0, 0, 0, 0}};
    v.s[i >> 6] = 1ull << (i & 63);
    r.cols[i] = v;
  }
  while (e) {
    if (e & 1) r = compose(base, r);
    base = compose(base, base);
    e >>= 1;
  }
  return r;
}

__global__ void k_index_stream(uint64_t seed, uint64_t n, int64_t m, int chunk, int levels,
                               const uint64_t* __restrict__ cols, int32_t* __restrict__ out,
                               unsigned int* __restrict__ rejects, const uint64_t* __restrict__ dseed) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t begin = t * chunk;
  if (begin >= m) return;
  if (dseed) seed = *dseed;  // device-resident epoch loop: the seed of the epoch being prepared
  State st = seed_state(seed);
  for (int l = 0; l < levels; ++l) {
    if (!((t >> l) & 1)) continue;
    const uint64_t* mc = cols + static_cast<size_t>(l) * 256 * 4;
    uint64_t o0 = 0, o1 = 0, o2 = 0, o3 = 0;
#pragma unroll 4
    for (int i = 0; i < 256; ++i) {
      const uint64_t mask = 0ull - ((st.s[i >> 6] >> (i & 63)) & 1ull);
      o0 ^= mask & __ldg(mc + 4 * i + 0);
      o1 ^= mask & __ldg(mc + 4 * i + 1);
      o2 ^= mask & __ldg(mc + 4 * i + 2);
      o3 ^= mask & __ldg(mc + 4 * i + 3);
    }
    st.s[0] = o0;
    st.s[1] = o1;
    st.s[2] = o2;
    st.s[3] = o3;
  }
  const uint64_t limit = n * (~0ull / n);
  const int64_t end = begin + chunk < m ? begin + chunk : m;
  unsigned int rej = 0;
  for (int64_t k = begin; k < end; ++k) {
    const uint64_t draw = next(st);
    if (draw >= limit) {
      ++rej;
      out[k] = -1;
    } else {
      out[k] = static_cast<int32_t>(draw % n);
    }
  }
  if (rej) atomicAdd(rejects, rej);
}

// Exact serial regeneration, only taken when some draw was rejected.
__global__ void k_index_fixup(uint64_t seed, uint64_t n, int64_t m, int32_t* __restrict__ out,
                              const unsigned int* __restrict__ rejects, const uint64_t* __restrict__ dseed) {
  if (*rejects == 0 || threadIdx.x != 0 || blockIdx.x != 0) return;
  if (dseed) seed = *dseed;
  State st = seed_state(seed);
  const uint64_t limit = n * (~0ull / n);
  for (int64_t k = 0; k < m; ++k) {
    uint64_t draw;
    do {
      draw = next(st);
    } while (draw >= limit);
    out[k] = static_cast<int32_t>(draw % n);
  }
}

constexpr int kChunk = 512;
constexpr int kLevels = 24;  // streams up to 512 * 2^24 = 8.6e9 draws

std::mutex g_mu;
std::unordered_map<int, uint64_t*> g_tables;  // device -> J_0..J_{L-1}

const uint64_t* jump_table() {
  int dev = 0;
  GAPLRA_CUDA_CHECK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_tables.find(dev);
  if (it != g_tables.end()) return it->second;
  std::vector<uint64_t> host(static_cast<size_t>(kLevels) * 256 * 4);
  BitMat j = power(step_matrix(), kChunk);
  for (int l = 0; l < kLevels; ++l) {
    std::memcpy(host.data() + static_cast<size_t>(l) * 256 * 4, j.cols, sizeof(j.cols));
    j = compose(j, j);
  }
  uint64_t* d = nullptr;
  GAPLRA_CUDA_CHECK(cudaMalloc(&d, host.size() * sizeof(uint64_t)));
  GAPLRA_CUDA_CHECK(cudaMemcpy(d, host.data(), host.size() * sizeof(uint64_t), cudaMemcpyHostToDevice));
  g_tables[dev] = d;
  return d;
}

}  // namespace

uint64_t derive_seed(uint64_t root, uint64_t tag) {  // rng.cpp:71-76
  uint64_t x = root ^ (0xA0761D6478BD642Full * (tag + 1));
  const uint64_t a = splitmix(x);
  const uint64_t b = splitmix(x);
  return a ^ rotl(b, 32);
}

uint64_t svrg_stream_seed(uint64_t root, int64_t solve_id, int epoch) {
  return derive_seed(root, kTagSvrg ^ (static_cast<uint64_t>(solve_id) << 20) ^ static_cast<uint64_t>(epoch));
}

void launch_index_stream(uint64_t seed, uint64_t n, int64_t m, int32_t* out, unsigned int* rejects,
                         cudaStream_t st, const uint64_t* dseed) {
  if (m <= 0) return;
  if (n == 0 || ceil_div(m, kChunk) > (int64_t{1} << kLevels)) throw Error(kContractViolation, "index stream size");
  const uint64_t* table = jump_table();
  const int64_t threads = ceil_div(m, kChunk);
  GAPLRA_CUDA_CHECK(cudaMemsetAsync(rejects, 0, sizeof(unsigned int), st));
  k_index_stream<<<ceil_div(threads, 128), 128, 0, st>>>(seed, n, m, kChunk, kLevels, table, out, rejects, dseed);
  GAPLRA_LAUNCH_CHECK();
  k_index_fixup<<<1, 32, 0, st>>>(seed, n, m, out, rejects, dseed);
  GAPLRA_LAUNCH_CHECK();
}

}  // namespace gaplra_cuda
