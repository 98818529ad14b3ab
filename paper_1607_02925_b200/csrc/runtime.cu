// Native runtime of the B200 shift-and-invert path: context / resident X /
// workspaces, and the drivers that sequence the device kernels — block SVRG
// solve, Alg. 3 estimate,
// tune_shift, subspace_iterate,
// restricted_projection and the ShiftedInverse pipeline —
// behind the C ABI of include/gaplra_cuda.h.  Every pinned choice (seeds,
// stopping rules, W0 = 0, last iterate) matches oracle/oracle.cpp; see
// DESIGN.md §2.  There is no CPU compute path: every numeric step is a kernel.
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "../../include/gaplra_cuda.h"
#include "common.cuh"
#include "gram.cuh"
#include "linalg.cuh"
#include "rng.cuh"
#include "svrg.cuh"

namespace gaplra_cuda {

unsigned long long& launch_counter() {
  static unsigned long long n = 0;
  return n;
}

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  T* ensure(size_t k) {
    if (k <= n && p) return p;
    release();
    GAPLRA_CUDA_CHECK(cudaMalloc(&p, std::max<size_t>(k, 1) * sizeof(T)));
    // cudaMemset runs on the legacy stream, which does not order against the
    // context's non-blocking stream: complete it before the buffer is used.
    GAPLRA_CUDA_CHECK(cudaMemset(p, 0, std::max<size_t>(k, 1) * sizeof(T)));
    GAPLRA_CUDA_CHECK(cudaDeviceSynchronize());
    n = k;
    return p;
  }
};

inline int64_t ldp_of(int p) { return p == 1 ? 1 : (p + 1) / 2 * 2; }
inline int64_t round4(int64_t d) { return (d + 3) / 4 * 4; }

// ---------------------------------------------------------------------------
// Host Rng (bit-exact with rng.cpp) for gaussian_init: S0 is generated on the
// host because device libm (log/sin/cos) differs in the last ulp.
// ---------------------------------------------------------------------------
struct HostRng {
  uint64_t s[4];
  double spare = 0.0;
  bool has = false;
  static uint64_t sm(uint64_t& x) {
    x += 0x9E3779B97F4A7C15ull;
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  static uint64_t rl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  explicit HostRng(uint64_t seed) {
    uint64_t t = seed;
    for (auto& w : s) w = sm(t);
  }
  uint64_t next() {
    const uint64_t out = rl(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rl(s[3], 45);
    return out;
  }
  double u01() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double normal() {
    if (has) {
      has = false;
      return spare;
    }
    double u1;
    do {
      u1 = u01();
    } while (u1 <= 0.0);
    const double u2 = u01();
    const double radius = std::sqrt(-2.0 * std::log(u1));
    const double angle = 2.0 * M_PI * u2;
    spare = radius * std::sin(angle);
    has = true;
    return radius * std::cos(angle);
  }
};

void gaussian_init_host(int d, int p, uint64_t seed, double* out_rowmajor, int64_t ld) {
  if (p < 1 || p > d) throw Error(kContractViolation, "gaussian_init: requires 1 <= p <= d");
  HostRng r(derive_seed(seed, kTagGauss));
  for (int i = 0; i < d; ++i)
    for (int c = 0; c < p; ++c) out_rowmajor[static_cast<int64_t>(i) * ld + c] = r.normal();
}

// ---------------------------------------------------------------------------
struct Matrix {
  int kind = 0;  // 0 dense, 1 csc
  int d = 0, n = 0;
  int64_t ld = 0, nnz = 0;
  DBuf<double> xbuf;
  const double* x = nullptr;
  DBuf<int64_t> colptr, rowptr;
  DBuf<int32_t> rowidx, colidx;
  DBuf<double> val, rval;
  double maxn2 = -1.0, fro2 = -1.0;
  int max_col_nnz = 0;  // CSC: largest column (sizes the blocked sparse epoch's scratch)
  int device = 0;
  DenseX dense() const {
    DenseX X;
    X.x = x;
    X.ld = ld;
    X.d = d;
    X.n = n;
    return X;
  }
  SparseX sparse() const {
    SparseX S;
    S.d = d;
    S.n = n;
    S.nnz = nnz;
    S.colptr = colptr.p;
    S.rowidx = rowidx.p;
    S.val = val.p;
    S.rowptr = rowptr.p;
    S.colidx = colidx.p;
    S.rval = rval.p;
    return S;
  }
  int64_t d_pad() const { return kind == 0 ? ld : round4(d); }
};

// Live per-kernel-class timing (CUDA events on the launching stream), with the
// algorithmic bytes / flops of each launch for the roofline report.
enum ProfClass {
  kProfGram = 0,  // X(XᵀW) pass, p > 1
  kProfEpoch,     // SVRG epoch chain, p > 1
  kProfHPass,
  kProfIndex,
  kProfQr,
  kProfAnchor,
  kProfBlockGram,
  kProfGramP1,   // X(Xᵀv) pass, p = 1 (Alg. 3 / tuning)
  kProfEpochP1,  // SVRG epoch chain, p = 1
  kProfBlockU,   // per-epoch U coefficients of the s-step blocks (needs Y, H)
  kProfClasses
};
constexpr int kEpochBlock = 16;  // s-step block (svrg.cu kBlock)

struct ProfPending {
  int cls;
  cudaEvent_t a, b;
};

struct Context {
  int device = 0;
  cudaStream_t own = nullptr, st = nullptr;
  std::string err;
  gaplra_ledger led{};
  // workspaces
  DBuf<double> gw, ybuf, hbuf, zbuf, cbuf, wbuf, bbuf, sbuf, tbuf, qrs, small, apart, bnorm, scal, tmp, tmat, zcol;
  DBuf<int32_t> idx, idx2;  // index streams of even / odd epochs
  DBuf<double> tmat2;        // slab of odd epochs (tmat: even)
  DBuf<unsigned int> rej, rej2;
  DBuf<double> ghist, gctl;  // device-resident epoch loop: residual history, control block
  DBuf<double> qrc;      // rank completion: the iterate before QR, with replaced columns
  const double* qr_in = nullptr;
  DBuf<double> xgs;      // L2-exchange chains (EpochConfig::xg): partial slots
  DBuf<unsigned> xgc;    //   and their arrival counters
  DBuf<double> spd;  // blocked sparse epoch: b, u
  DBuf<int> spi;     // blocked sparse epoch: row lists, pairs, counters
  DBuf<double> spl;  // level-scheduled sparse epoch: symbolic plan + b, u (bytes / 8)
  // Side stream for the next epoch's W-independent precompute (index stream +
  // k_block_prep), run beside the current epoch's chain on the SMs the chain
  // leaves idle.  Events order it against the main stream.
  cudaStream_t aux = nullptr;
  cudaEvent_t pre_done[2] = {nullptr, nullptr}, chain_done[2] = {nullptr, nullptr}, u_done = nullptr;
  cudaStream_t aux_stream() {
    if (!aux) {
      // lowest priority: when chain e and prep e+1 become ready together (a graph
      // launches its branches in no fixed order), the chain's CTAs are dispatched
      // first and the prep fills the SMs it leaves idle
      int lo = 0, hi = 0;
      GAPLRA_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      GAPLRA_CUDA_CHECK(cudaStreamCreateWithPriority(&aux, cudaStreamNonBlocking, lo));
      for (int i = 0; i < 2; ++i) {
        GAPLRA_CUDA_CHECK(cudaEventCreateWithFlags(&pre_done[i], cudaEventDisableTiming));
        GAPLRA_CUDA_CHECK(cudaEventCreateWithFlags(&chain_done[i], cudaEventDisableTiming));
      }
      GAPLRA_CUDA_CHECK(cudaEventCreateWithFlags(&u_done, cudaEventDisableTiming));
    }
    return aux;
  }
  DBuf<int> status;
  double* pin = nullptr;  // pinned host scalars
  int* pin_i = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  bool profiling = false;
  gaplra_profile prof{};
  std::vector<ProfPending> pending;
  std::vector<cudaEvent_t> spare;
  cudaEvent_t fence_ev[64] = {};
  cudaEvent_t fence_event(int i) {
    if (!fence_ev[i]) GAPLRA_CUDA_CHECK(cudaEventCreate(&fence_ev[i]));
    return fence_ev[i];
  }
  cudaEvent_t new_event() {
    if (!spare.empty()) {
      cudaEvent_t e = spare.back();
      spare.pop_back();
      return e;
    }
    cudaEvent_t e;
    GAPLRA_CUDA_CHECK(cudaEventCreate(&e));
    return e;
  }
  void resolve() {
    for (auto& p : pending) {
      float ms = 0.f;
      if (cudaEventSynchronize(p.b) == cudaSuccess && cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess)
        prof.ms[p.cls] += ms;
      spare.push_back(p.a);
      spare.push_back(p.b);
    }
    pending.clear();
  }
  ~Context() {
    resolve();
    for (auto e : spare) cudaEventDestroy(e);
    if (pin) cudaFreeHost(pin);
    if (pin_i) cudaFreeHost(pin_i);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (aux) {
      cudaStreamSynchronize(aux);
      for (int i = 0; i < 2; ++i) {
        cudaEventDestroy(pre_done[i]);
        cudaEventDestroy(chain_done[i]);
      }
      cudaEventDestroy(u_done);
      cudaStreamDestroy(aux);
    }
    if (own) cudaStreamDestroy(own);
  }
  unsigned long long host_syncs = 0;  // host waits on the device (gaplra_host_syncs)
  void sync() {
    ++host_syncs;
    GAPLRA_CUDA_CHECK(cudaStreamSynchronize(st));
    if (!pending.empty()) resolve();
  }
  double read_scalar(const double* dptr) {
    GAPLRA_CUDA_CHECK(cudaMemcpyAsync(pin, dptr, sizeof(double), cudaMemcpyDeviceToHost, st));
    sync();
    return pin[0];
  }
};

// RAII: time one launch (or launch group) of class `cls` when profiling.
struct Prof {
  Context& c;
  int cls;
  cudaEvent_t a = nullptr;
  double bytes, flops;
  cudaStream_t s;
  Prof(Context& cc, int k, double by, double fl, cudaStream_t st = nullptr)
      : c(cc), cls(k), bytes(by), flops(fl), s(st ? st : cc.st) {
    if (!c.profiling) {
      if (fence_mask() >> cls & 1) cudaEventRecord(c.fence_event(2 * cls), s);
      return;
    }
    a = c.new_event();
    cudaEventRecord(a, s);
  }
  // GAPLRA_FENCE_CLASSES=mask (experiment): timing events around the kernels of the given profile classes
  // even with profiling off (an event record keeps the neighbouring kernels of a stream from overlapping)
  static unsigned fence_mask() {
    static const unsigned m = getenv("GAPLRA_FENCE_CLASSES") ? static_cast<unsigned>(strtoul(getenv("GAPLRA_FENCE_CLASSES"), nullptr, 0)) : 0u;
    return m;
  }
  ~Prof() {
    if (!c.profiling && (fence_mask() >> cls & 1)) cudaEventRecord(c.fence_event(2 * cls + 1), s);
    if (!c.profiling) return;
    cudaEvent_t b = c.new_event();
    cudaEventRecord(b, s);
    c.pending.push_back({cls, a, b});
    c.prof.count[cls] += 1;
    c.prof.bytes[cls] += bytes;
    c.prof.flops[cls] += flops;
  }
};

struct Timer {
  Context& c;
  double* acc;
  cudaEvent_t a, b;
  Timer(Context& cc, double* out) : c(cc), acc(out) {
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, c.st);
  }
  ~Timer() {
    cudaEventRecord(b, c.st);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    if (acc) *acc += ms;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
};

// ---------------------------------------------------------------------------
// Units
// ---------------------------------------------------------------------------
// max_j |x_j|^2 and |X|_F^2 (deterministic, cached on the matrix)
void col_norms(Context& c, Matrix& X) {
  if (X.maxn2 >= 0.0) return;
  DBuf<double> nb;
  double* norms = nb.ensure(static_cast<size_t>(X.n));
  double* s = c.scal.ensure(8) + 4;
  if (X.kind == 0)
    col_norm2_dense(X.dense(), norms, c.st);
  else
    col_norm2_sparse(X.sparse(), norms, c.st);
  reduce_sum_max(norms, X.n, s, c.st);
  GAPLRA_CUDA_CHECK(cudaMemcpyAsync(c.pin, s, 2 * sizeof(double), cudaMemcpyDeviceToHost, c.st));
  c.sync();
  X.fro2 = c.pin[0];
  X.maxn2 = c.pin[1];
}

// Z (d_pad x ldz) = X (Xᵀ W); Y (n x ldy) = Xᵀ W.
void gram_block_dev(Context& c, const Matrix& X, int p, const double* W, int64_t ldw, double* Z, int64_t ldz,
                    double* Y, int64_t ldy) {
  if (!Y) {
    ldy = ldp_of(p);
    Y = c.ybuf.ensure(static_cast<size_t>(X.n) * ldy);
  }
  const double xbytes = X.kind == 0 ? 8.0 * X.d * X.n : 12.0 * X.nnz + 8.0 * (X.n + 1);
  Prof prof(c, p > 1 ? kProfGram : kProfGramP1, xbytes, 4.0 * X.nnz * p);
  if (X.kind == 0) {
    const DenseX D = X.dense();
    GramWork w;
    w.part_elems = gram_work_elems(D, p);
    w.part = w.part_elems ? c.gw.ensure(w.part_elems) : nullptr;
    if (gram_fused_applies(D, p)) {  // one pass over X (d <= 4096)
      launch_gram_fused(D, W, ldw, p, Y, ldy, Z, ldz, w, c.st);
    } else if (p == 1 && gram_p1_applies(D)) {  // one pass, 1024 < d <= 8192
      launch_gram_p1(D, W, ldw, Y, ldy, Z, ldz, w, c.st);
    } else {
      launch_xtw(D, W, ldw, p, Y, ldy, w, c.st);
      launch_xy(D, Y, ldy, p, Z, ldz, w, c.st);
    }
  } else {
    const SparseX S = X.sparse();
    launch_xtw_sparse(S, W, ldw, p, Y, ldy, c.st);
    launch_xy_sparse(S, Y, ldy, p, Z, ldz, c.st);
  }
  c.led.gram_applies += p;
}

// QR (two-pass MGS) in place on a row-major device block; throws RankDeficient.
void qr_dev(Context& c, double* Y, int64_t ldy, int d, int p, bool count = true) {
  if (d < p || p < 1) throw Error(kContractViolation, "qr_orthonormalize: need 1 <= cols <= rows");
  double* scratch = c.qrs.ensure(static_cast<size_t>(p) * round4(d));
  int* status = c.status.ensure(2);
  {
    Prof prof(c, kProfQr, 8.0 * d * p * 2, 4.0 * d * p * p);
    launch_qr_mgs2(Y, ldy, d, p, scratch, status, c.st);
  }
  GAPLRA_CUDA_CHECK(cudaMemcpyAsync(c.pin_i, status, 2 * sizeof(int), cudaMemcpyDeviceToHost, c.st));
  c.sync();
  if (count) c.led.qr_factorizations++;
  if (c.pin_i[0] == kRankDeficient)
    throw Error(kRankDeficient, "qr_orthonormalize: column " + std::to_string(c.pin_i[1]) +
                                    " is numerically dependent on earlier columns",
                c.pin_i[1]);
}

struct SvrgResult {
  int epochs = 0;
  std::vector<double> history;
};

struct SvrgParams {
  double eta, tol, slack, hint;
  int64_t m;
  int cap;
  uint64_t root;
};

SvrgParams resolve(Context& c, Matrix& X, double lambda, const gaplra_svrg_params& prm) {
  if (!(prm.tol > 0.0)) throw Error(kContractViolation, "solve_svrg: tol must be > 0");
  SvrgParams s;
  col_norms(c, X);
  s.hint = prm.lambda1_hint;
  if (prm.eta > 0.0) {
    s.eta = prm.eta;
  } else {
    s.eta = 1.0 / (4.0 * (lambda + static_cast<double>(X.n) * X.maxn2));
    // stability cap (oracle.cpp svrg_setup): eta <= (lambda - hint) / (|X|_F^2 hint)
    if (prm.lambda1_hint > 0.0) {
      if (!(lambda > prm.lambda1_hint))
        throw Error(kIndefiniteShift, "solve_svrg: lambda must exceed the lambda_1 hint");
      if (X.fro2 > 0.0) s.eta = std::min(s.eta, (lambda - prm.lambda1_hint) / (X.fro2 * prm.lambda1_hint));
    }
  }
  s.m = prm.m > 0 ? prm.m : 2 * static_cast<int64_t>(X.n);
  s.cap = prm.epoch_cap > 0 ? prm.epoch_cap : static_cast<int>(std::ceil(200.0 * std::log(1.0 / prm.tol)));
  s.tol = prm.tol;
  s.slack = prm.monotone_slack;
  s.root = prm.root_seed;
  return s;
}

// Dense epochs in two halves.
//  epoch_pre_dev: the W-independent part — index stream and k_block_prep (TT, M
//    of every 16-step block) — into the buffers of `parity` on stream `s`;
//  epoch_run_dev: H = XᵀC, U (k_block_u), the chain, on the main stream.
// svrg_solve_dev runs epoch e+1's pre on the side stream beside epoch e's chain.
struct EpochPre {
  int32_t* idx = nullptr;
  double* slab = nullptr;
  EpochConfig cfg{};
  int64_t m = 0;
};

EpochPre epoch_pre_dev(Context& c, Matrix& X, int p, double eta, double lambda, uint64_t stream_seed, int64_t m,
                       int parity, cudaStream_t s, const uint64_t* dseed = nullptr) {
  EpochPre pre;
  pre.m = m;
  pre.idx = (parity ? c.idx2 : c.idx).ensure(static_cast<size_t>(m));
  {
    Prof prof(c, kProfIndex, 4.0 * m, 0.0, s);
    launch_index_stream(stream_seed, static_cast<uint64_t>(X.n), m, pre.idx, (parity ? c.rej2 : c.rej).ensure(1), s,
                        dseed);
  }
  if (X.kind != 0) return pre;
  const double col_nnz = static_cast<double>(X.nnz) / X.n;
  EpochArgs a{};
  a.X = X.x;
  a.ldx = X.ld;
  a.d_pad = static_cast<int>(X.ld);
  a.n = X.n;
  a.idx = pre.idx;
  a.m = m;
  a.p = p;
  a.rho = 1.0 - eta * lambda;
  a.eta_n = eta * static_cast<double>(X.n);
  pre.cfg = choose_epoch_config(a.d_pad, p);
  pre.slab = (parity ? c.tmat2 : c.tmat).ensure(epoch_slab_elems(m, pre.cfg));
  a.slab = pre.slab;
  a.zcol = c.zcol.ensure(static_cast<size_t>(X.ld));
  Prof prof(c, kProfBlockGram, 8.0 * X.d * m, 3.0 * kEpochBlock * col_nnz * m, s);
  launch_block_prep(a, pre.cfg, s);
  return pre;
}

void epoch_run_dev(Context& c, Matrix& X, int p, double* W, const double* C, const double* Y, double eta,
                   double lambda, const EpochPre& pre) {
  const int64_t ld = ldp_of(p);
  const int64_t m = pre.m;
  const double col_nnz = static_cast<double>(X.nnz) / X.n;
  const double col_bytes = X.kind == 0 ? 8.0 * X.d : 12.0 * col_nnz;
  const double rho = 1.0 - eta * lambda;
  const double eta_n = eta * static_cast<double>(X.n);
  if (X.kind == 0) {
    double* H = c.hbuf.ensure(static_cast<size_t>(X.n) * ld);
    GramWork w;
    const DenseX D = X.dense();
    w.part_elems = gram_work_elems(D, p);
    w.part = w.part_elems ? c.gw.ensure(w.part_elems) : nullptr;
    {
      Prof prof(c, kProfHPass, 8.0 * X.d * X.n, 2.0 * X.nnz * p);
      if (p == 1 && gram_p1_applies(D))
        launch_gram_p1(D, C, ld, H, ld, nullptr, 0, w, c.st);
      else
        launch_xtw(D, C, ld, p, H, ld, w, c.st);
    }
    EpochArgs a{};
    a.X = X.x;
    a.ldx = X.ld;
    a.d_pad = static_cast<int>(X.ld);
    a.n = X.n;
    a.idx = pre.idx;
    a.m = m;
    a.W = W;
    a.C = C;
    a.ldw = ld;
    a.Y = Y;
    a.H = H;
    a.ldy = ld;
    a.p = p;
    a.rho = rho;
    a.eta_n = eta_n;
    const EpochConfig& cfg = pre.cfg;
    a.slab = pre.slab;
    a.zcol = c.zcol.ensure(static_cast<size_t>(X.ld));
    if (cfg.xg || cfg.nclusters > 1) {
      a.xg_slot = c.xgs.ensure(xg_slot_elems(cfg));
      a.xg_count = c.xgc.ensure(xg_count_elems(cfg));
    }
    {
      Prof prof(c, kProfBlockU, 16.0 * m * p, 2.0 * kEpochBlock * m * p);
      launch_block_u(a, cfg, c.st);
    }
    if (c.u_done) GAPLRA_CUDA_CHECK(cudaEventRecord(c.u_done, c.st));
    static const bool timing = getenv("GAPLRA_EPOCH_TIMING") != nullptr;
    static const int skip = getenv("GAPLRA_EPOCH_SKIP") ? atoi(getenv("GAPLRA_EPOCH_SKIP")) : 0;
    a.skip = skip;
    static const int prefetch = getenv("GAPLRA_CHAIN_PREFETCH") ? atoi(getenv("GAPLRA_CHAIN_PREFETCH")) : 0;
    a.prefetch = prefetch;
    DBuf<long long> dbg;
    if (timing) {
      a.dbg = dbg.ensure(static_cast<size_t>(cfg.cluster) * cfg.nclusters * cfg.groups * 8);
      fprintf(stderr, "{\"epoch_layout\": {\"d_pad\": %d, \"p\": %d, \"cluster\": %d, \"pc\": %d, \"groups\": %d, "
              "\"rows_per_cta\": %d, \"stages\": %d, \"smem\": %zu}}\n", a.d_pad, p, cfg.cluster, cfg.pc, cfg.groups,
              cfg.rows_per_cta, cfg.stages, cfg.smem);
    }
    {
      Prof prof(c, p > 1 ? kProfEpoch : kProfEpochP1, col_bytes * m, 4.0 * col_nnz * p * m);
      launch_svrg_epoch_dense(a, cfg, c.st);
    }
    if (timing) {
      std::vector<long long> h(static_cast<size_t>(cfg.cluster) * cfg.nclusters * cfg.groups * 8);
      GAPLRA_CUDA_CHECK(cudaMemcpyAsync(h.data(), dbg.p, h.size() * sizeof(long long), cudaMemcpyDeviceToHost, c.st));
      c.sync();
      const double nbk = static_cast<double>(ceil_div(m, cfg.b));
      fprintf(stderr, "{\"epoch_phase_cycles_per_block\": [");
      for (int k = 0; k < 8; ++k) fprintf(stderr, "%s%.0f", k ? ", " : "", h[k] / nbk);
      fprintf(stderr, "], \"mean_over_ctas\": [");
      const size_t nct = h.size() / 8;
      for (int k = 0; k < 8; ++k) {
        double sum = 0;
        for (size_t q = 0; q < nct; ++q) sum += static_cast<double>(h[q * 8 + k]);
        fprintf(stderr, "%s%.0f", k ? ", " : "", sum / nct / nbk);
      }
      fprintf(stderr, "], \"cluster\": %d, \"pc\": %d, \"groups\": %d, \"stages\": %d}\n", cfg.cluster, cfg.pc,
              cfg.groups, cfg.stages);
#ifdef GAPLRA_HOP_TIMING
      if (p == 1 && m >= 1008 * kEpochBlock) {
        long long hp[64];
        read_chain_hops(hp);
        fprintf(stderr, "{\"chain_hops_block_1002\": {\"rows_products_done\": 0, \"pusher_woken\": %lld, \"copies_issued\": %lld, "
                "\"reducer_all_in\": %lld, \"coef_handed\": %lld, \"rows_coef_received\": %lld, \"next_products_done\": %lld}}\n",
                hp[2 * 8 + 1] - hp[2 * 8], hp[2 * 8 + 2] - hp[2 * 8], hp[2 * 8 + 3] - hp[2 * 8], hp[2 * 8 + 4] - hp[2 * 8],
                hp[2 * 8 + 5] - hp[2 * 8], hp[3 * 8] - hp[2 * 8]);
      }
#endif
    }
  } else {
    SparseEpochArgs a{};
    a.d = X.d;
    a.n = X.n;
    a.p = p;
    a.colptr = X.colptr.p;
    a.rowidx = X.rowidx.p;
    a.val = X.val.p;
    a.idx = pre.idx;
    a.m = m;
    a.W = W;
    a.C = C;
    a.ldw = ld;
    a.Y = Y;
    a.ldy = ld;
    a.rho = rho;
    a.eta_n = eta_n;
    static const bool blocked = !(getenv("GAPLRA_SPARSE_BLOCKED") && atoi(getenv("GAPLRA_SPARSE_BLOCKED")) == 0);
    Prof prof(c, p > 1 ? kProfEpoch : kProfEpochP1, col_bytes * m, 4.0 * col_nnz * p * m);
    // GAPLRA_SPARSE_LEVELS=0: the fixed-point block kernel of sparse_epoch.cu instead of the level-scheduled one
    static const bool levels = !(getenv("GAPLRA_SPARSE_LEVELS") && atoi(getenv("GAPLRA_SPARSE_LEVELS")) == 0);
    if (blocked && levels && sparse_levels_supported(p) && X.max_col_nnz > 0) {
      const SparseLevelPlan plan = sparse_levels_plan(X.d, m, col_nnz, X.max_col_nnz);
      void* scratch = c.spl.ensure((plan.bytes + 7) / 8);
      launch_svrg_epoch_sparse_levels(a, plan, scratch, c.st);
    } else if (blocked && sparse_blocked_supported(p) && X.max_col_nnz > 0) {
      const int bs = sparse_block_steps(X.d, col_nnz, p);
      double* db = c.spd.ensure(2 * static_cast<size_t>(bs) * p);
      const size_t ni = sparse_scratch_ints(X.d, bs, X.max_col_nnz);
      int* ib = c.spi.ensure(ni);
      // row counts and counters must start at zero (the layout depends on d)
      GAPLRA_CUDA_CHECK(cudaMemsetAsync(ib, 0, ni * sizeof(int), c.st));
      launch_svrg_epoch_sparse_blocked(a, bs, X.max_col_nnz, db, ib, c.st);
    } else {
      launch_svrg_epoch_sparse(a, c.st);
    }
  }
}

// One stochastic epoch on device blocks (ld = ldp(p)): W in/out, C, Y given;
// H = Xᵀ C computed here (dense only).  Everything on the main stream.
void epoch_dev(Context& c, Matrix& X, int p, double* W, const double* C, const double* Y, double eta,
               double lambda, uint64_t stream_seed, int64_t m) {
  const EpochPre pre = epoch_pre_dev(c, X, p, eta, lambda, stream_seed, m, 0, c.st);
  epoch_run_dev(c, X, p, W, C, Y, eta, lambda, pre);
}

// Device-resident epoch loop (north star item 5): epochs 1, 2, ... of a dense
// solve as one CUDA graph with a WHILE node, so the host does not read a
// residual per epoch.  Entered after the host ran epoch 0 and evaluated the
// anchor of epoch 1 (all buffers exist; epoch 1's index stream and slab are in
// the parity-1 buffers).  Body (one iteration = epoch e):
//   H pass, k_block_u (parity-1 "cur" buffers) -> fork: chain e ‖ index stream +
//   k_block_prep of epoch e+1 into the parity-0 "nxt" buffers (seed from the
//   device) -> join -> copy nxt -> cur -> anchor of epoch e+1 (gram pass +
//   k_anchor) -> k_epoch_control (the host loop's tests, history, next seed,
//   loop condition).
// Returns the device control block after the graph; the caller turns its
// status into the host loop's outcome.  One sync per solve instead of one per epoch.
struct GraphEpochs {
  EpochCtl ctl{};
  std::vector<double> hist;
};
GraphEpochs run_epochs_graph(Context& c, Matrix& X, int p, double* W, double* Z, double* C, double* Y,
                             const double* B, double* part, double* bn, double* res, double lambda,
                             const SvrgParams& prm, int64_t solve_id, const EpochPre& cur, double best) {
  const int64_t ld = ldp_of(p), dp = X.d_pad();
  const int hist_cap = prm.cap + 2;
  double* hist = c.ghist.ensure(static_cast<size_t>(hist_cap));
  EpochCtl* ctl = reinterpret_cast<EpochCtl*>(c.gctl.ensure(4));
  uint64_t* dseed = reinterpret_cast<uint64_t*>(&ctl->next_seed);
  EpochCtl h0{};
  h0.best = best;
  h0.e = 1;
  h0.status = 0;
  h0.next_seed = svrg_stream_seed(prm.root, solve_id, 2);
  GAPLRA_CUDA_CHECK(cudaMemcpyAsync(ctl, &h0, sizeof(h0), cudaMemcpyHostToDevice, c.st));
  // buffers of the prep (parity 0) and their sizes, allocated before capture
  const EpochConfig cfg = cur.cfg;
  const size_t slab_elems = epoch_slab_elems(prm.m, cfg);
  double* slab_nxt = c.tmat.ensure(slab_elems);
  int32_t* idx_nxt = c.idx.ensure(static_cast<size_t>(prm.m));
  c.rej.ensure(1);
  cudaStream_t aux = c.aux_stream();
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ge = nullptr;
  GAPLRA_CUDA_CHECK(cudaGraphCreate(&g, 0));
  struct GraphGuard {
    cudaGraph_t& g;
    cudaGraphExec_t& ge;
    ~GraphGuard() {
      if (ge) cudaGraphExecDestroy(ge);
      if (g) cudaGraphDestroy(g);
    }
  } guard{g, ge};
  cudaGraphConditionalHandle cond;
  GAPLRA_CUDA_CHECK(cudaGraphConditionalHandleCreate(&cond, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams np{};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = cond;
  np.conditional.type = cudaGraphCondTypeWhile;
  np.conditional.size = 1;
  cudaGraphNode_t node;
  GAPLRA_CUDA_CHECK(cudaGraphAddNode(&node, g, nullptr, 0, &np));
  cudaGraph_t body = np.conditional.phGraph_out[0];
  static const bool gdebug = getenv("GAPLRA_GRAPH_DEBUG") != nullptr;
  const auto t_cap0 = std::chrono::steady_clock::now();
  GAPLRA_CUDA_CHECK(cudaStreamBeginCaptureToGraph(c.st, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  const unsigned long long launches0 = launch_counter();
  try {
    epoch_run_dev(c, X, p, W, C, Y, prm.eta, lambda, cur);  // records c.u_done after k_block_u
    GAPLRA_CUDA_CHECK(cudaStreamWaitEvent(aux, c.u_done, 0));
    const EpochPre nxt = epoch_pre_dev(c, X, p, prm.eta, lambda, 0, prm.m, 0, aux, dseed);
    GAPLRA_CUDA_CHECK(cudaEventRecord(c.pre_done[0], aux));
    // The join with the side stream comes AFTER the anchor's gram pass, as in the host loop (there the main
    // stream waits for the prep only before the next H pass): at C5 the prep on the 20 SMs the chain leaves
    // takes about as long as the chain, and joining before the gram pass put it on the critical path
    // (step 9.39 s in the graph against 8.69 s in the host loop).  GAPLRA_GRAPH_JOIN=early restores that.
    static const bool join_early = getenv("GAPLRA_GRAPH_JOIN") && std::string(getenv("GAPLRA_GRAPH_JOIN")) == "early";
    auto join_and_rotate = [&]() {
      GAPLRA_CUDA_CHECK(cudaStreamWaitEvent(c.st, c.pre_done[0], 0));
      launch_copy(nxt.idx, cur.idx, static_cast<size_t>(prm.m) * sizeof(int32_t), c.st);
      if (nxt.slab) launch_copy(nxt.slab, cur.slab, slab_elems * sizeof(double), c.st);
    };
    if (join_early) join_and_rotate();
    gram_block_dev(c, X, p, W, ld, Z, ld, Y, ld);
    launch_anchor(W, Z, B, ld, static_cast<int>(dp), p, lambda, prm.eta, C, part, bn, nullptr, res, c.st);
    if (!join_early) join_and_rotate();
    launch_epoch_control(res, ctl, hist, hist_cap, prm.tol, prm.slack, prm.cap, prm.root, solve_id, cond, c.st);
  } catch (...) {
    cudaGraph_t tmp = nullptr;
    cudaStreamEndCapture(c.st, &tmp);
    throw;
  }
  cudaGraph_t captured = nullptr;
  GAPLRA_CUDA_CHECK(cudaStreamEndCapture(c.st, &captured));
  const unsigned long long per_body = launch_counter() - launches0;  // kernels of one iteration (counted at capture)
  (void)slab_nxt;
  (void)idx_nxt;
  // events last recorded inside the capture cannot be waited on outside it: re-record them
  GAPLRA_CUDA_CHECK(cudaEventRecord(c.pre_done[0], aux));
  GAPLRA_CUDA_CHECK(cudaEventRecord(c.u_done, c.st));
  const auto t_cap1 = std::chrono::steady_clock::now();
  GAPLRA_CUDA_CHECK(cudaGraphInstantiate(&ge, g, 0));
  const auto t_inst = std::chrono::steady_clock::now();
  cudaEvent_t ga = nullptr, gb = nullptr;
  if (gdebug) {
    cudaEventCreate(&ga);
    cudaEventCreate(&gb);
    cudaEventRecord(ga, c.st);
  }
  GAPLRA_CUDA_CHECK(cudaGraphLaunch(ge, c.st));
  if (gdebug) cudaEventRecord(gb, c.st);
  GraphEpochs out;
  GAPLRA_CUDA_CHECK(cudaMemcpyAsync(&out.ctl, ctl, sizeof(EpochCtl), cudaMemcpyDeviceToHost, c.st));
  c.sync();
  if (gdebug) {
    float gms = 0.f;
    cudaEventElapsedTime(&gms, ga, gb);
    fprintf(stderr, "{\"graph\": {\"capture_ms\": %.3f, \"instantiate_ms\": %.3f, \"run_ms\": %.3f, \"epochs\": %d, "
            "\"ms_per_epoch\": %.3f, \"kernels_per_epoch\": %llu}}\n",
            std::chrono::duration<double, std::milli>(t_cap1 - t_cap0).count(),
            std::chrono::duration<double, std::milli>(t_inst - t_cap1).count(), gms, out.ctl.e - 1,
            gms / std::max(1, out.ctl.e - 1), per_body);
    cudaEventDestroy(ga);
    cudaEventDestroy(gb);
  }
  if (out.ctl.e > 2) launch_counter() += per_body * static_cast<unsigned long long>(out.ctl.e - 2);  // executions
  const int last = std::min(out.ctl.e, hist_cap - 1);
  if (last >= 2) {
    out.hist.resize(static_cast<size_t>(last - 1));
    GAPLRA_CUDA_CHECK(cudaMemcpy(out.hist.data(), hist + 2, out.hist.size() * sizeof(double), cudaMemcpyDeviceToHost));
  }
  return out;
}

// Block solve (λI − XXᵀ)W = B with W0 = 0; B, W device blocks with ld = ldp(p).
// warm = true: W holds the initial guess on entry, else W0 = 0.
SvrgResult svrg_solve_dev(Context& c, Matrix& X, double lambda, int p, const double* B, double* W,
                          const gaplra_svrg_params& prm_in, int64_t solve_id, SvrgResult* partial = nullptr,
                          bool warm = false) {
  const SvrgParams prm = resolve(c, X, lambda, prm_in);
  const int64_t ld = ldp_of(p), dp = X.d_pad();
  const size_t blk = static_cast<size_t>(dp) * ld;
  double* Z = c.zbuf.ensure(blk);
  double* C = c.cbuf.ensure(blk);
  double* Y = c.ybuf.ensure(static_cast<size_t>(X.n) * ld);
  double* part = c.apart.ensure(static_cast<size_t>(anchor_parts(static_cast<int>(dp))) * 64);
  double* bn = c.bnorm.ensure(64);
  double* res = c.scal.ensure(8) + 1;
  // |B_c| via the anchor kernel with W = Z = 0, λ = 0  (M = −B).
  launch_anchor(nullptr, nullptr, B, ld, static_cast<int>(dp), p, 0.0, 0.0, nullptr, part, nullptr, bn, res, c.st);
  if (!warm) GAPLRA_CUDA_CHECK(cudaMemsetAsync(W, 0, blk * sizeof(double), c.st));
  SvrgResult local;
  SvrgResult& out = partial ? *partial : local;
  out = SvrgResult{};
  double best = INFINITY;
  // epoch e+1's index stream + k_block_prep run on the side stream beside
  // epoch e's chain (dense X); GAPLRA_OVERLAP=0 keeps everything on one stream
  // GAPLRA_OVERLAP: 0 serial; 1 epoch e+1's prep starts once chain
  // e−1 is done; 2 it also waits for epoch e's k_block_u (prep then shares the
  // SMs with chain e only, not with the H pass / block_u, whose CTAs it starved;
  // default: C5 p = 64 epoch 434 -> 377 ms, p = 1 210 -> 169 ms, C2 / C3 1-3 % faster)
  static const int overlap_mode = getenv("GAPLRA_OVERLAP") ? atoi(getenv("GAPLRA_OVERLAP")) : 2;
  static const bool overlap = overlap_mode != 0;
  const bool side = overlap && X.kind == 0;
  EpochPre next;
  bool have_next = false;
  struct AuxJoin {  // the main stream never runs ahead of side-stream writes into shared buffers
    Context& c;
    bool used = false;
    ~AuxJoin() {
      if (used)
        for (int i = 0; i < 2; ++i) cudaStreamWaitEvent(c.st, c.pre_done[i], 0);
    }
  } join{c};
  for (int e = 0;; ++e) {
    const bool zero = e == 0 && !warm;
    if (!zero) gram_block_dev(c, X, p, W, ld, Z, ld, Y, ld);
    else GAPLRA_CUDA_CHECK(cudaMemsetAsync(Y, 0, static_cast<size_t>(X.n) * ld * sizeof(double), c.st));
    launch_anchor(zero ? nullptr : W, zero ? nullptr : Z, B, ld, static_cast<int>(dp), p, lambda, prm.eta, C, part,
                  bn, nullptr, res, c.st);
    const double r = c.read_scalar(res);
    out.history.push_back(r);
    if (!std::isfinite(r)) throw Error(kSolverStalled, "solve_svrg: non-finite residual (indefinite shift?)");
    if (r <= prm.tol) break;
    if (prm.slack > 0.0 && e >= 1 && r > prm.slack * best)
      throw Error(kSolverStalled, "solve_svrg: residual grew above slack x best (epoch " + std::to_string(e) + ")");
    best = std::min(best, r);
    if (e >= prm.cap) throw Error(kSolverStalled, "solve_svrg: epoch cap reached");
    // from epoch 1 on, the loop runs on the device (GAPLRA_GRAPH=0: host loop)
    static const bool graph_env = !(getenv("GAPLRA_GRAPH") && atoi(getenv("GAPLRA_GRAPH")) == 0);
    static const bool timing_env = getenv("GAPLRA_EPOCH_TIMING") != nullptr;
    // Epochs of >= ~1 TFLOP stay on the host loop: one scalar read per 0.3 s epoch is free, and at C5 p = 64
    // (prep on the SMs the chain leaves ~ as long as the chain) the graph ran the step 8 % slower
    // (9.39 vs 8.69 s).  GAPLRA_GRAPH_MAX_TFLOP moves the threshold.
    static const double graph_max_tflop = getenv("GAPLRA_GRAPH_MAX_TFLOP") ? atof(getenv("GAPLRA_GRAPH_MAX_TFLOP")) : 1.0;
    const bool small_epochs = 4.0 * static_cast<double>(X.d) * p * static_cast<double>(prm.m) < graph_max_tflop * 1e12;
    if (e == 1 && have_next && side && overlap_mode == 2 && graph_env && small_epochs && !timing_env && !c.profiling) {
      GAPLRA_CUDA_CHECK(cudaStreamWaitEvent(c.st, c.pre_done[1], 0));
      const GraphEpochs ge = run_epochs_graph(c, X, p, W, Z, C, Y, B, part, bn, res, lambda, prm, solve_id, next, best);
      const int runs = ge.ctl.e - 1;  // epochs 1 .. e-1 ran in the graph, each followed by one anchor
      // the captured anchor's gram pass counted its p applies once, at capture time
      c.led.gram_applies += static_cast<uint64_t>(p) * static_cast<uint64_t>(std::max(0, runs - 1));
      out.epochs += runs;
      c.led.epochs += static_cast<uint64_t>(runs);
      c.led.solver_column_samples += static_cast<uint64_t>(runs) * static_cast<uint64_t>(prm.m);
      for (double v : ge.hist) out.history.push_back(v);
      have_next = false;
      switch (ge.ctl.status) {
        case 1: break;
        case 2: throw Error(kSolverStalled, "solve_svrg: non-finite residual (indefinite shift?)");
        case 3:
          throw Error(kSolverStalled,
                      "solve_svrg: residual grew above slack x best (epoch " + std::to_string(ge.ctl.e) + ")");
        case 4: throw Error(kSolverStalled, "solve_svrg: epoch cap reached");
        default: throw Error(kDeviceError, "solve_svrg: device epoch loop ended without a status");
      }
      break;
    }
    const int parity = e & 1;
    EpochPre pre;
    if (have_next) {
      pre = next;
      GAPLRA_CUDA_CHECK(cudaStreamWaitEvent(c.st, c.pre_done[parity], 0));
    } else {
      pre = epoch_pre_dev(c, X, p, prm.eta, lambda, svrg_stream_seed(prm.root, solve_id, e), prm.m, parity, c.st);
    }
    epoch_run_dev(c, X, p, W, C, Y, prm.eta, lambda, pre);
    have_next = false;
    if (side && e + 1 <= prm.cap) {
      cudaStream_t aux = c.aux_stream();
      join.used = true;
      GAPLRA_CUDA_CHECK(cudaEventRecord(c.chain_done[parity], c.st));
      // buffers of parity e+1 were last read by epoch e−1's chain
      GAPLRA_CUDA_CHECK(cudaStreamWaitEvent(aux, c.chain_done[parity ^ 1], 0));
      if (overlap_mode == 2) GAPLRA_CUDA_CHECK(cudaStreamWaitEvent(aux, c.u_done, 0));
      next = epoch_pre_dev(c, X, p, prm.eta, lambda, svrg_stream_seed(prm.root, solve_id, e + 1), prm.m, parity ^ 1,
                           aux);
      GAPLRA_CUDA_CHECK(cudaEventRecord(c.pre_done[parity ^ 1], aux));
      have_next = true;
    }
    out.epochs++;
    c.led.epochs++;
    c.led.solver_column_samples += static_cast<uint64_t>(prm.m);
  }
  c.led.linear_solves++;
  return out;
}

// ---------------------------------------------------------------------------
// Operators and the subspace engine.
// ---------------------------------------------------------------------------
struct Op {
  virtual ~Op() = default;
  // out = op(in), device blocks with ld = ldp(p); `guess` (optional, may be
  // consumed) warm-starts iterative operators
  virtual void apply(const double* in, double* out, int p, const double* guess = nullptr) = 0;
};

struct GramOp : Op {
  Context& c;
  Matrix& X;
  GramOp(Context& cc, Matrix& xx) : c(cc), X(xx) {}
  void apply(const double* in, double* out, int p, const double* = nullptr) override {
    gram_block_dev(c, X, p, in, ldp_of(p), out, ldp_of(p), nullptr, 0);
    c.led.operator_applies += p;
  }
};

struct InverseOp : Op {
  Context& c;
  Matrix& X;
  double lambda;
  gaplra_svrg_params prm;
  int64_t* counter;
  InverseOp(Context& cc, Matrix& xx, double lam, const gaplra_svrg_params& pr, int64_t* sc)
      : c(cc), X(xx), lambda(lam), prm(pr), counter(sc) {}
  void apply(const double* in, double* out, int p, const double* guess = nullptr) override {
    if (guess)
      GAPLRA_CUDA_CHECK(cudaMemcpyAsync(out, guess, static_cast<size_t>(X.d_pad()) * ldp_of(p) * sizeof(double),
                                        cudaMemcpyDeviceToDevice, c.st));
    svrg_solve_dev(c, X, lambda, p, in, out, prm, (*counter)++, nullptr, guess != nullptr);
    c.led.operator_applies += p;
  }
};

// solve_cg, the pinned block form of oracle.cpp cg_solve:
// one CG recurrence per column, all columns stepped together; W0 = 0 or the
// warm guess (R0 = B - D W0); stop before an iteration when max_c |r_c|/|b_c|
// <= tol; IndefiniteShift on p_cᵀ D p_c <= 0 with r_c != 0; frozen columns
// (r_c = 0) take alpha = beta = 0; cap = max_iter > 0 ? max_iter : d + 10.
// Per iteration: one X·(XᵀP) pass, six small kernels, one read of the p
// residual norms (the stopping test).
struct CgResult {
  int iterations = 0;
  std::vector<double> history;
};

// P u = u - U (Uᵀ u) for a row-major d x p device block (project_out,
// linear_operator.cpp:66-81: all coefficients first, then one subtraction);
// U: d_pad x ldp(m) row-major, m <= 64.
void project_out_dev(Context& c, const double* U, int m, double* v, int64_t ldv, int d, int p) {
  if (m <= 0) return;
  double* G = c.small.ensure(static_cast<size_t>(64) * 64 * 4 + 8) + 3 * 64 * 64;
  double* part = c.tmp.ensure(static_cast<size_t>(small_gram_parts(d)) * 64 * 64 + 8);
  launch_small_gram(U, ldp_of(m), m, v, ldv, p, d, part, G, c.st);  // m x p coefficients
  launch_small_mul(U, ldp_of(m), m, G, p, p, d, 1.0, -1.0, v, ldv, c.st);
}

// With a deflation basis U (m columns) the system is lambda I - P X Xᵀ P,
// P = I - U Uᵀ (Alg. 7's X_{-(s-1)}); for iterates in range(P)
// that is one project_out after each gram pass (oracle.cpp cg_solve).
CgResult cg_solve_dev(Context& c, Matrix& X, double lambda, int p, const double* B, double* W, double tol,
                      int max_iter, bool warm, CgResult* partial = nullptr, const double* U = nullptr, int m = 0) {
  if (p < 1 || p > 64) throw Error(kContractViolation, "solve_cg: need 1 <= p <= 64");
  if (!(tol > 0.0)) throw Error(kContractViolation, "solve_cg: tol must be > 0");
  const int d = X.d;
  const int64_t ld = ldp_of(p), dp = X.d_pad();
  const size_t blk = static_cast<size_t>(dp) * ld;
  const int cap = max_iter > 0 ? max_iter : d + 10;
  DBuf<double> rb, pb, qb, zb, vb;
  double* R = rb.ensure(blk);
  double* P = pb.ensure(blk);
  double* Q = qb.ensure(blk);
  double* Zg = zb.ensure(blk);
  double* v = vb.ensure(5 * 64);
  double *rr = v, *rr_new = v + 64, *pq = v + 128, *alpha = v + 192, *bn2 = v + 256;
  // sized for project_out_dev's use of the same workspace (a smaller c.tmp
  // would be reallocated under `part` inside the loop)
  double* part = c.tmp.ensure(static_cast<size_t>(small_gram_parts(d)) * 64 * 64 + 8);
  int* status = c.status.ensure(2);
  GAPLRA_CUDA_CHECK(cudaMemsetAsync(status, 0, 2 * sizeof(int), c.st));
  launch_col_dots(B, ld, B, ld, d, p, part, bn2, c.st);
  std::vector<double> bnorm(p);
  GAPLRA_CUDA_CHECK(cudaMemcpyAsync(c.pin, bn2, p * sizeof(double), cudaMemcpyDeviceToHost, c.st));
  c.sync();
  for (int k = 0; k < p; ++k) bnorm[k] = std::sqrt(c.pin[k]);
  if (warm) {  // R = B - D W0: Q = lambda W0 - X Xᵀ W0, then R = 1 * B - Q
    gram_block_dev(c, X, p, W, ld, Zg, ld, nullptr, 0);
    project_out_dev(c, U, m, Zg, ld, d, p);
    launch_cg_dq(W, Zg, lambda, Q, ld, d, p, c.st);
    launch_cg_dq(B, Q, 1.0, R, ld, d, p, c.st);
  } else {
    GAPLRA_CUDA_CHECK(cudaMemsetAsync(W, 0, blk * sizeof(double), c.st));
    GAPLRA_CUDA_CHECK(cudaMemcpyAsync(R, B, blk * sizeof(double), cudaMemcpyDeviceToDevice, c.st));
  }
  GAPLRA_CUDA_CHECK(cudaMemcpyAsync(P, R, blk * sizeof(double), cudaMemcpyDeviceToDevice, c.st));
  launch_col_dots(R, ld, R, ld, d, p, part, rr, c.st);
  CgResult out;
  auto residual = [&](const double* rrd) {
    GAPLRA_CUDA_CHECK(cudaMemcpyAsync(c.pin, rrd, p * sizeof(double), cudaMemcpyDeviceToHost, c.st));
    GAPLRA_CUDA_CHECK(cudaMemcpyAsync(c.pin_i, status, sizeof(int), cudaMemcpyDeviceToHost, c.st));
    c.sync();
    double worst = 0.0;
    for (int k = 0; k < p; ++k) {
      const double rk = std::sqrt(c.pin[k]) / (bnorm[k] > 0.0 ? bnorm[k] : 1.0);
      worst = std::isfinite(rk) ? std::max(worst, rk) : rk;
    }
    return worst;
  };
  try {
    for (int it = 0;; ++it) {
      const double r = residual(rr);
      if (c.pin_i[0]) throw Error(kIndefiniteShift, "solve_cg: nonpositive curvature pᵀ(lambda I - X Xᵀ)p <= 0");
      out.history.push_back(r);
      if (!std::isfinite(r)) throw Error(kSolverStalled, "solve_cg: non-finite residual");
      if (r <= tol) break;
      if (it >= cap) throw Error(kSolverStalled, "solve_cg: iteration cap reached");
      gram_block_dev(c, X, p, P, ld, Zg, ld, nullptr, 0);
      project_out_dev(c, U, m, Zg, ld, d, p);
      launch_cg_dq(P, Zg, lambda, Q, ld, d, p, c.st);
      launch_col_dots(P, ld, Q, ld, d, p, part, pq, c.st);
      launch_cg_alpha(rr, pq, p, alpha, status, c.st);
      launch_cg_xr(alpha, P, Q, W, R, ld, d, p, c.st);
      launch_col_dots(R, ld, R, ld, d, p, part, rr_new, c.st);
      launch_cg_dir(rr, rr_new, R, P, ld, d, p, c.st);
      GAPLRA_CUDA_CHECK(cudaMemcpyAsync(rr, rr_new, p * sizeof(double), cudaMemcpyDeviceToDevice, c.st));
      out.iterations++;
    }
  } catch (...) {
    if (partial) *partial = out;
    throw;
  }
  c.led.linear_solves++;
  return out;
}

// solve_accelerated_svrg, the device form of oracle.cpp
// accsvrg_solve: Catalyst outer loop (kappa = sqrt(h mu), extrapolation
// beta = (1 - sqrt q)/(1 + sqrt q), q = mu/(mu + kappa)) around block SVRG
// solves of (lambda + kappa) I - X Xᵀ, inner tol max(tol/10, res/10), stream
// ids (solve_id << 10) | k, warm-started at the current iterate.
SvrgResult accsvrg_solve_dev(Context& c, Matrix& X, double lambda, int p, const double* B, double* W,
                             const gaplra_svrg_params& prm, int64_t solve_id, bool warm) {
  const double h = prm.lambda1_hint;
  if (!(h > 0.0) || !(lambda > h))
    throw Error(kContractViolation, "solve_accelerated_svrg: needs lambda1_hint h > 0 and lambda > h");
  const double mu = lambda - h, kappa = std::sqrt(h * mu), q = mu / (mu + kappa);
  const double beta = (1.0 - std::sqrt(q)) / (1.0 + std::sqrt(q));
  const int cap = prm.epoch_cap > 0 ? prm.epoch_cap : static_cast<int>(std::ceil(200.0 * std::log(1.0 / prm.tol)));
  const int d = X.d;
  const int64_t ld = ldp_of(p), dp = X.d_pad();
  const size_t blk = static_cast<size_t>(dp) * ld;
  DBuf<double> xb, yb, rb, zb, qb, nb;
  double* xc = xb.ensure(blk);
  double* yc = yb.ensure(blk);
  double* rhs = rb.ensure(blk);
  double* Zg = zb.ensure(blk);
  double* Q = qb.ensure(blk);
  double* xn = nb.ensure(blk);
  if (warm)
    GAPLRA_CUDA_CHECK(cudaMemcpyAsync(xc, W, blk * sizeof(double), cudaMemcpyDeviceToDevice, c.st));
  else
    GAPLRA_CUDA_CHECK(cudaMemsetAsync(xc, 0, blk * sizeof(double), c.st));
  GAPLRA_CUDA_CHECK(cudaMemcpyAsync(yc, xc, blk * sizeof(double), cudaMemcpyDeviceToDevice, c.st));
  double* part = c.tmp.ensure(static_cast<size_t>(small_gram_parts(d)) * 64 + 8);
  double* nv = c.scal.ensure(8 + 2 * 64) + 8;
  launch_col_dots(B, ld, B, ld, d, p, part, nv, c.st);
  GAPLRA_CUDA_CHECK(cudaMemcpyAsync(c.pin, nv, p * sizeof(double), cudaMemcpyDeviceToHost, c.st));
  c.sync();
  std::vector<double> bnorm(p);
  for (int k = 0; k < p; ++k) bnorm[k] = std::sqrt(c.pin[k]);
  SvrgResult out;
  for (int k = 0;; ++k) {
    gram_block_dev(c, X, p, xc, ld, Zg, ld, nullptr, 0);
    launch_cg_dq(xc, Zg, lambda, Q, ld, d, p, c.st);  // Q = D x
    launch_cg_dq(B, Q, 1.0, rhs, ld, d, p, c.st);     // r = b - D x (in rhs)
    launch_col_dots(rhs, ld, rhs, ld, d, p, part, nv, c.st);
    GAPLRA_CUDA_CHECK(cudaMemcpyAsync(c.pin, nv, p * sizeof(double), cudaMemcpyDeviceToHost, c.st));
    c.sync();
    double r = 0.0;
    for (int j = 0; j < p; ++j) {
      const double rj = std::sqrt(c.pin[j]) / (bnorm[j] > 0.0 ? bnorm[j] : 1.0);
      r = std::isfinite(rj) ? std::max(r, rj) : rj;
    }
    out.history.push_back(r);
    if (!std::isfinite(r)) throw Error(kSolverStalled, "solve_accelerated_svrg: non-finite residual");
    if (r <= prm.tol) break;
    if (k >= cap) throw Error(kSolverStalled, "solve_accelerated_svrg: outer cap reached");
    launch_axpby(1.0, B, kappa, yc, rhs, ld, d, p, c.st);  // b + kappa y
    gaplra_svrg_params pin = prm;
    pin.tol = std::max(0.1 * prm.tol, 0.1 * r);
    pin.epoch_cap = 0;
    GAPLRA_CUDA_CHECK(cudaMemcpyAsync(xn, xc, blk * sizeof(double), cudaMemcpyDeviceToDevice, c.st));
    const SvrgResult in = svrg_solve_dev(c, X, lambda + kappa, p, rhs, xn, pin, (solve_id << 10) | (k & 1023), nullptr,
                                         true);
    out.epochs += in.epochs;
    launch_axpby(1.0 + beta, xn, -beta, xc, yc, ld, d, p, c.st);  // y = x' + beta (x' - x)
    GAPLRA_CUDA_CHECK(cudaMemcpyAsync(xc, xn, blk * sizeof(double), cudaMemcpyDeviceToDevice, c.st));
  }
  GAPLRA_CUDA_CHECK(cudaMemcpyAsync(W, xc, blk * sizeof(double), cudaMemcpyDeviceToDevice, c.st));
  return out;
}

// inverse_operator(accsvrg, lambda)
struct AccOp : Op {
  Context& c;
  Matrix& X;
  double lambda;
  gaplra_svrg_params prm;
  int64_t* counter;
  AccOp(Context& cc, Matrix& xx, double lam, const gaplra_svrg_params& pr, int64_t* sc)
      : c(cc), X(xx), lambda(lam), prm(pr), counter(sc) {}
  void apply(const double* in, double* out, int p, const double* guess = nullptr) override {
    if (guess)
      GAPLRA_CUDA_CHECK(cudaMemcpyAsync(out, guess, static_cast<size_t>(X.d_pad()) * ldp_of(p) * sizeof(double),
                                        cudaMemcpyDeviceToDevice, c.st));
    accsvrg_solve_dev(c, X, lambda, p, in, out, prm, (*counter)++, guess != nullptr);
    c.led.operator_applies += p;
  }
};

// inverse_operator(cg, lambda)
struct CgOp : Op {
  Context& c;
  Matrix& X;
  double lambda, tol;
  const double* U;  // deflated system (m = 0: none)
  int m;
  CgOp(Context& cc, Matrix& xx, double lam, double t, const double* u = nullptr, int mm = 0)
      : c(cc), X(xx), lambda(lam), tol(t), U(u), m(mm) {}
  void apply(const double* in, double* out, int p, const double* guess = nullptr) override {
    if (guess)
      GAPLRA_CUDA_CHECK(cudaMemcpyAsync(out, guess, static_cast<size_t>(X.d_pad()) * ldp_of(p) * sizeof(double),
                                        cudaMemcpyDeviceToDevice, c.st));
    cg_solve_dev(c, X, lambda, p, in, out, tol, 0, guess != nullptr, nullptr, U, m);
    c.led.operator_applies += p;
  }
};

// DeflatedOperator::apply (linear_operator.cpp:56-64) on device blocks: P C P.
struct DeflatedOp : Op {
  Context& c;
  Op& base;
  const double* U;
  int m, d;
  int64_t dp;
  DBuf<double> work;
  DeflatedOp(Context& cc, Op& b, const double* u, int mm, int dd, int64_t dpp)
      : c(cc), base(b), U(u), m(mm), d(dd), dp(dpp) {}
  void apply(const double* in, double* out, int p, const double* guess = nullptr) override {
    if (m <= 0) {
      base.apply(in, out, p, guess);
      return;
    }
    const int64_t ld = ldp_of(p);
    double* w = work.ensure(static_cast<size_t>(dp) * ld);
    GAPLRA_CUDA_CHECK(cudaMemcpyAsync(w, in, static_cast<size_t>(dp) * ld * sizeof(double), cudaMemcpyDeviceToDevice,
                                      c.st));
    project_out_dev(c, U, m, w, ld, d, p);
    base.apply(w, out, p, guess);
    project_out_dev(c, U, m, out, ld, d, p);
  }
};

// S0 = QR(gaussian_init(d, p, seed)), redraw once with seed + 1.
void orth_init(Context& c, int d, int64_t dp, int p, uint64_t seed, double* S) {
  const int64_t ld = ldp_of(p);
  std::vector<double> h(static_cast<size_t>(dp) * ld, 0.0);
  for (int attempt = 0; attempt < 2; ++attempt) {
    gaussian_init_host(d, p, seed + attempt, h.data(), ld);
    GAPLRA_CUDA_CHECK(cudaMemcpyAsync(S, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice, c.st));
    try {
      qr_dev(c, S, ld, d, p, /*count=*/false);
      return;
    } catch (const Error& e) {
      if (e.code != kRankDeficient || attempt == 1) throw;
    }
  }
}

// |S Sᵀ − S' S'ᵀ|_F = sqrt(2) |S' − S (Sᵀ S')|_F ; G = Sᵀ S' is left in c.small
double projector_diff_dev(Context& c, const double* S, const double* S2, int d, int p) {
  const int64_t ld = ldp_of(p);
  double* G = c.small.ensure(static_cast<size_t>(64) * 64 * 4 + 8);
  double* part = c.tmp.ensure(static_cast<size_t>(small_gram_parts(d)) * 64 * 64 + 8);
  launch_small_gram(S, ld, p, S2, ld, p, d, part, G, c.st);
  double* R = c.tbuf.ensure(static_cast<size_t>(round4(d)) * ld);
  GAPLRA_CUDA_CHECK(cudaMemcpyAsync(R, S2, static_cast<size_t>(d) * ld * sizeof(double), cudaMemcpyDeviceToDevice, c.st));
  launch_small_mul(S, ld, p, G, p, p, d, 1.0, -1.0, R, ld, c.st);
  double* out = c.scal.ensure(8) + 2;
  launch_frob2(R, ld, d, p, part, out, c.st);
  return std::sqrt(2.0 * c.read_scalar(out));
}

// guess = Q (Qᵀ Y) G  with G = S_oldᵀ Q already in c.small (oracle.cpp warm_guess)
void warm_guess_dev(Context& c, const double* Q, const double* Y, int d, int p, double* guess) {
  const int64_t ld = ldp_of(p);
  double* G = c.small.p;
  double* R = G + 64 * 64;
  double* RG = R + 64 * 64;
  double* part = c.tmp.ensure(static_cast<size_t>(small_gram_parts(d)) * 64 * 64 + 8);
  launch_small_gram(Q, ld, p, Y, ld, p, d, part, R, c.st);
  launch_small_mul(R, p, p, G, p, p, p, 0.0, 1.0, RG, p, c.st);
  launch_small_mul(Q, ld, p, RG, p, p, d, 0.0, 1.0, guess, ld, c.st);
}

// Rank completion of an iterate (oracle.cpp qr_complete): a
// dependent column j of C·S (operator range of dimension < p) is replaced by
// gaussian_init(d, 1, derive_seed(seed, j + 64·attempt)) and the QR redone (the same
// draws every iteration, so a completed iterate is a fixed point and the
// projector early stop still fires).
constexpr uint64_t kTagComplete = 0x636f6d70ull;  // "comp"
void qr_complete_dev(Context& c, double* Q, int64_t ld, int d, int p, uint64_t seed) {
  const size_t blk = static_cast<size_t>(round4(d)) * ld;
  double* orig = nullptr;
  std::vector<double> h(static_cast<size_t>(d));
  for (int attempt = 0;; ++attempt) {
    try {
      qr_dev(c, Q, ld, d, p, /*count=*/false);
      return;
    } catch (const Error& e) {
      if (e.code != kRankDeficient || attempt >= p) throw;
      if (!orig) {  // the block before QR: the caller's copy in c.sbuf (op output) is not touched
        orig = c.qrc.ensure(blk);
        GAPLRA_CUDA_CHECK(cudaMemcpyAsync(orig, c.qr_in, blk * sizeof(double), cudaMemcpyDeviceToDevice, c.st));
      }
      gaussian_init_host(d, 1, derive_seed(seed, static_cast<uint64_t>(e.payload + 64 * attempt)), h.data(), 1);
      GAPLRA_CUDA_CHECK(cudaMemcpy2DAsync(orig + e.payload, ld * sizeof(double), h.data(), sizeof(double),
                                          sizeof(double), d, cudaMemcpyHostToDevice, c.st));
      GAPLRA_CUDA_CHECK(cudaMemcpyAsync(Q, orig, blk * sizeof(double), cudaMemcpyDeviceToDevice, c.st));
      c.sync();  // h is reused by the next attempt
    }
  }
}

// Alg. 1 with projector early stop and warm-started solves; final S in `S`.
int subspace_iterate_dev(Context& c, Op& op, int d, int64_t dp, int p, int L, uint64_t seed, double conv_tol,
                         double* S) {
  const int64_t ld = ldp_of(p);
  const size_t blk = static_cast<size_t>(dp) * ld;
  orth_init(c, d, dp, p, seed, S);
  DBuf<double> qb, gb;
  double* Yb = c.sbuf.ensure(blk);
  double* Q = qb.ensure(blk);
  double* guess = gb.ensure(blk);
  bool have_guess = false;
  int it = 0;
  for (int l = 1; l <= L; ++l) {
    op.apply(S, Yb, p, have_guess ? guess : nullptr);
    GAPLRA_CUDA_CHECK(cudaMemcpyAsync(Q, Yb, blk * sizeof(double), cudaMemcpyDeviceToDevice, c.st));
    c.qr_in = Yb;
    qr_complete_dev(c, Q, ld, d, p, derive_seed(seed, kTagComplete));
    c.led.qr_factorizations++;
    it = l;
    const double diff = projector_diff_dev(c, S, Q, d, p);
    const bool stop = conv_tol > 0.0 && diff <= conv_tol;
    warm_guess_dev(c, Q, Yb, d, p, guess);
    have_guess = true;
    GAPLRA_CUDA_CHECK(cudaMemcpyAsync(S, Q, blk * sizeof(double), cudaMemcpyDeviceToDevice, c.st));
    if (stop) break;
  }
  c.led.outer_iterations += it;
  return it;
}

// Alg. 3, k = 1 (Rayleigh quotient of the iterate, relative-change early stop).
double estimate_top_dev(Context& c, Op& op, int d, int64_t dp, double eps_prime, uint64_t seed, double rq_tol,
                        int* iters) {
  const int L = static_cast<int>(std::ceil(4.0 / eps_prime * std::log(d / eps_prime)));
  DBuf<double> s, y, q, gs;
  double* S = s.ensure(static_cast<size_t>(dp));
  double* Yb = y.ensure(static_cast<size_t>(dp));
  double* Q = q.ensure(static_cast<size_t>(dp));
  double* guess = gs.ensure(static_cast<size_t>(dp));
  orth_init(c, d, dp, 1, seed, S);
  double* G = c.small.ensure(static_cast<size_t>(64) * 64 * 4 + 8);
  double* part = c.tmp.ensure(static_cast<size_t>(small_gram_parts(d)) * 64 * 64 + 8);
  double* th = G + 3 * 64 * 64;
  double prev = 0.0, theta = 0.0;
  bool have_guess = false;
  int it = 0;
  for (int l = 1; l <= L + 1; ++l) {
    op.apply(S, Yb, 1, have_guess ? guess : nullptr);
    it = l;
    launch_small_gram(S, 1, 1, Yb, 1, 1, d, part, th, c.st);
    theta = c.read_scalar(th);
    if (l > 1 && std::fabs(theta - prev) <= rq_tol * std::fabs(theta)) break;
    if (l == L + 1) break;
    GAPLRA_CUDA_CHECK(cudaMemcpyAsync(Q, Yb, static_cast<size_t>(dp) * sizeof(double), cudaMemcpyDeviceToDevice, c.st));
    qr_dev(c, Q, 1, d, 1);
    launch_small_gram(S, 1, 1, Q, 1, 1, d, part, G, c.st);  // G = s_oldᵀ q
    warm_guess_dev(c, Q, Yb, d, 1, guess);
    have_guess = true;
    std::swap(S, Q);
    prev = theta;
  }
  if (iters) *iters = it;
  return theta;
}

// Alg. 3 for any k (oracle.cpp estimate_eigs): Ritz values of the k-column
// iterate (H = Sᵀ C S symmetrised, Jacobi), descending; early stop when
// every value changes by <= rq_tol relative; k = 1 is estimate_top_dev.
std::vector<double> estimate_eigs_dev(Context& c, Op& op, int d, int64_t dp, int k, double eps_prime, uint64_t seed,
                                      double rq_tol, int* iters) {
  if (k < 1 || k > 64) throw Error(kContractViolation, "estimate_eigenvalues: need 1 <= k <= 64");
  const int L = static_cast<int>(std::ceil(4.0 / eps_prime * std::log(d / eps_prime)));
  const int64_t ld = ldp_of(k);
  const size_t blk = static_cast<size_t>(dp) * ld;
  DBuf<double> s, y, q, gs, hb;
  double* S = s.ensure(blk);
  double* Yb = y.ensure(blk);
  double* Q = q.ensure(blk);
  double* guess = gs.ensure(blk);
  double* H = hb.ensure(static_cast<size_t>(k) * k + k + static_cast<size_t>(k) * k);
  double* vals = H + k * k;
  double* vecs = vals + k;
  orth_init(c, d, dp, k, seed, S);
  double* G = c.small.ensure(static_cast<size_t>(64) * 64 * 4 + 8);
  double* part = c.tmp.ensure(static_cast<size_t>(small_gram_parts(d)) * 64 * 64 + 8);
  std::vector<double> theta(k, 0.0), prev(k, 0.0);
  bool have_guess = false;
  int it = 0;
  for (int l = 1; l <= L + 1; ++l) {
    op.apply(S, Yb, k, have_guess ? guess : nullptr);
    it = l;
    launch_small_gram(S, ld, k, Yb, ld, k, d, part, H, c.st);
    launch_symmetrize(H, k, c.st);
    launch_jacobi(H, k, vals, vecs, c.st);
    GAPLRA_CUDA_CHECK(cudaMemcpyAsync(c.pin, vals, k * sizeof(double), cudaMemcpyDeviceToHost, c.st));
    c.sync();
    for (int a = 0; a < k; ++a) theta[a] = c.pin[a];
    bool stop = l > 1;
    for (int a = 0; a < k && stop; ++a) stop = std::fabs(theta[a] - prev[a]) <= rq_tol * std::fabs(theta[a]);
    if (stop || l == L + 1) break;
    GAPLRA_CUDA_CHECK(cudaMemcpyAsync(Q, Yb, blk * sizeof(double), cudaMemcpyDeviceToDevice, c.st));
    c.qr_in = Yb;
    qr_complete_dev(c, Q, ld, d, k, derive_seed(seed, kTagComplete));
    c.led.qr_factorizations++;
    launch_small_gram(S, ld, k, Q, ld, k, d, part, G, c.st);  // G = S_oldᵀ Q
    warm_guess_dev(c, Q, Yb, d, k, guess);
    have_guess = true;
    std::swap(S, Q);
    prev = theta;
  }
  if (iters) *iters = it;
  return theta;
}

// Alg. 4 / Alg. 5 (oracle.cpp detect_multiplicative_gap / detect_additive_gap)
int detect_multiplicative_gap_host(const double* est, int count, int s, int p) {
  const double f = 1.0 - 1.0 / (static_cast<double>(p) * p);
  for (int i = 0; i + 1 < count; ++i)
    if (est[i + 1] <= est[i] * f) return s + i;
  return -1;
}
int detect_additive_gap_host(const double* inv, int count, int s, int k, double delta) {
  if (count < 1 || !(inv[0] >= delta / 27.0 && inv[0] <= delta / 5.0))
    throw Error(kShiftOutOfRange, "detect_additive_gap: inverse estimate outside [delta/27, delta/5] (Eq. 5)");
  for (int i = 0; i + 1 < count; ++i)
    if (inv[i + 1] - inv[i] >= 5.0 * delta / 9.0) return s + i;
  return k;
}

gaplra_svrg_params prm_from(const gaplra_si_config& cfg, double tol) {
  gaplra_svrg_params p{};
  p.eta = 0.0;
  p.m = 0;
  p.tol = tol;
  p.epoch_cap = cfg.epoch_cap;
  p.monotone_slack = cfg.monotone_slack;
  p.root_seed = cfg.seed;
  p.lambda1_hint = 0.0;
  return p;
}

void tune_shift_dev(Context& c, Matrix& X, double delta, const gaplra_si_config& cfg, int64_t* counter,
                    gaplra_si_report& rep, const double* U = nullptr, int m = 0) {
  if (!(delta > 0.0)) throw Error(kContractViolation, "tune_shift: delta must be > 0");
  const int d = X.d;
  const int64_t dp = X.d_pad();
  GramOp a0(c, X);
  DeflatedOp a(c, a0, U, m, d, dp);  // A_{-(s-1)}
  const double l1 = estimate_top_dev(c, a, d, dp, 0.25, derive_seed(cfg.seed, kTagEstA), cfg.rq_tol, nullptr);
  rep.lambda1_hat = l1;
  rep.tune_steps = 0;
  if (l1 < 3.0 * delta && !cfg.force)
    throw Error(kNoPreconditioningNeeded, "tune_shift: lambda1_hat < 3 delta (no preconditioning needed)");
  double lambda = 1.5 * l1;
  const double ratio = l1 / delta;
  const int cap = (ratio > 1.0 ? static_cast<int>(std::ceil(4.0 * std::log2(ratio))) : 0) + 5;
  gaplra_svrg_params prm = prm_from(cfg, cfg.tol_tune);
  // lambda_1 upper estimates (oracle.cpp tune_shift): l1_hat >= (3/4) lambda_1, then
  // lambda_1 <= 2 lambda_t - lambda_{t-1}
  double hint = l1 / 0.75, prev_lambda = lambda;
  for (int t = 0; t < cap; ++t) {
    if (t > 0) hint = 2.0 * lambda - prev_lambda;
    prm.lambda1_hint = hint;
    InverseOp dinv(c, X, lambda, prm, counter);
    CgOp dcg(c, X, lambda, cfg.tol_tune, U, m);
    // a deflated shifted system is solved by CG (oracle.cpp tune_shift)
    DeflatedOp op(c, cfg.backend == 1 || m > 0 ? static_cast<Op&>(dcg) : static_cast<Op&>(dinv), U, m, d, dp);
    const double est = estimate_top_dev(c, op, d, dp, 1.0 / 9.0, derive_seed(cfg.seed, kTagEstD + t), cfg.rq_tol,
                                        nullptr);
    const double inv = 1.0 / std::max(est, 1e-300);
    if (rep.tune_steps < 64) {
      rep.tune_lambda[rep.tune_steps] = lambda;
      rep.tune_inv[rep.tune_steps] = inv;
    }
    rep.tune_steps++;
    if (inv >= delta / 27.0 && inv <= delta / 5.0) {
      rep.lambda = lambda;
      rep.lambda1_hint = lambda - (8.0 / 9.0) * inv;
      return;
    }
    prev_lambda = lambda;
    lambda = lambda - (4.0 / 9.0) * inv;
  }
  rep.lambda = lambda;
  throw Error(kShiftTuningStalled, "tune_shift: no estimate landed in [delta/27, delta/5]");
}

// W (d_pad x ldp(k)) = S U_k, ritz[k] (host) from H = Sᵀ X Xᵀ S.
void restricted_projection_dev(Context& c, Matrix& X, const double* S, int p, int k, double* W, double* ritz_host) {
  const int d = X.d;
  const int64_t dp = X.d_pad(), ld = ldp_of(p);
  if (k < 1 || k > p || p > kJacobiMax) throw Error(kContractViolation, "restricted_projection: need 1 <= k <= p <= 64");
  DBuf<double> z;
  double* Z = z.ensure(static_cast<size_t>(dp) * ld);
  gram_block_dev(c, X, p, S, ld, Z, ld, nullptr, 0);
  double* H = c.small.ensure(static_cast<size_t>(64) * 64 * 4 + 8);
  double* part = c.tmp.ensure(static_cast<size_t>(small_gram_parts(d)) * 64 * 64 + 8);
  launch_small_gram(S, ld, p, Z, ld, p, d, part, H, c.st);
  DBuf<double> vv;  // (H lives in c.small)
  double* vals = vv.ensure(static_cast<size_t>(p) + static_cast<size_t>(p) * p);
  double* vecs = vals + p;
  launch_jacobi(H, p, vals, vecs, c.st);
  launch_small_mul(S, ld, p, vecs, p, k, d, 0.0, 1.0, W, ldp_of(k), c.st);
  GAPLRA_CUDA_CHECK(cudaMemcpyAsync(ritz_host, vals, k * sizeof(double), cudaMemcpyDeviceToHost, c.st));
  c.sync();
}

// error_report, the pinned form of oracle.cpp
// orc_error_report: frobenius = sqrt(max(0, |X|_F^2 - |XᵀW|_F^2)) (one Xᵀ W
// pass); spectral = power method on P X Xᵀ P (P = I - W Wᵀ) from
// P g / |P g|, g = gaussian_init(d, 1, derive_seed(seed, "errs")), `iters`
// gram passes at p = 1.
constexpr uint64_t kTagErr = 0x65727273ull;  // "errs"

void error_report_dev(Context& c, Matrix& X, int k, const double* W, int iters, uint64_t seed, double* frob,
                      double* spec) {
  const int d = X.d;
  const int64_t dp = X.d_pad(), ldk = ldp_of(k);
  col_norms(c, X);
  double fy = 0.0;
  double* out = c.scal.ensure(8) + 5;
  if (k > 0) {
    const int64_t ldy = ldk;
    double* Y = c.ybuf.ensure(static_cast<size_t>(X.n) * ldy);
    if (X.kind == 0) {
      const DenseX D = X.dense();
      GramWork w;
      w.part_elems = gram_work_elems(D, k);
      w.part = w.part_elems ? c.gw.ensure(w.part_elems) : nullptr;
      launch_xtw(D, W, ldk, k, Y, ldy, w, c.st);
    } else {
      launch_xtw_sparse(X.sparse(), W, ldk, k, Y, ldy, c.st);
    }
    double* part = c.tmp.ensure(static_cast<size_t>(small_gram_parts(X.n)) + 8);
    launch_frob2(Y, ldy, X.n, k, part, out, c.st);
    fy = c.read_scalar(out);
  }
  *frob = std::sqrt(std::max(X.fro2 - fy, 0.0));
  DBuf<double> vb, zb;
  double* v = vb.ensure(static_cast<size_t>(dp));
  double* z = zb.ensure(static_cast<size_t>(dp));
  double* G = c.small.ensure(static_cast<size_t>(64) * 64 * 4 + 8);
  double* part = c.tmp.ensure(static_cast<size_t>(small_gram_parts(d)) * 64 * 64 + 8);
  std::vector<double> h(static_cast<size_t>(dp), 0.0);
  gaussian_init_host(d, 1, derive_seed(seed, kTagErr), h.data(), 1);
  GAPLRA_CUDA_CHECK(cudaMemcpyAsync(v, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice, c.st));
  auto project = [&](double* u) {  // u -= W (Wᵀ u)
    if (k == 0) return;
    launch_small_gram(W, ldk, k, u, 1, 1, d, part, G, c.st);
    launch_small_mul(W, ldk, k, G, 1, 1, d, 1.0, -1.0, u, 1, c.st);
  };
  auto normalize = [&](double* u) {
    launch_frob2(u, 1, d, 1, part, out, c.st);
    launch_scale_inv_sqrt(u, 1, d, 1, out, c.st);
    return c.read_scalar(out);
  };
  project(v);
  double theta = 0.0;
  if (normalize(v) > 0.0) {
    for (int it = 0; it < iters; ++it) {
      gram_block_dev(c, X, 1, v, 1, z, 1, nullptr, 0);
      project(z);
      launch_small_gram(v, 1, 1, z, 1, 1, d, part, out + 1, c.st);
      theta = c.read_scalar(out + 1);
      std::swap(v, z);
      if (normalize(v) == 0.0) break;
    }
  }
  *spec = std::sqrt(std::max(theta, 0.0));
}

// principal_angles, oracle.cpp orc_principal_angles:
// Q = qr_orthonormalize(S), Gᵀ = Qᵀ U (p x k), H = G Gᵀ, Jacobi, cos = sqrt(clamp).
void principal_angles_dev(Context& c, int d, int k, const double* U, int p, double* S, double* cos_host) {
  const int64_t ldu = ldp_of(k), lds = ldp_of(p);
  if (k < 1 || p < 1 || k > 64 || p > 64 || k > d || p > d)
    throw Error(kContractViolation, "principal_angles: need 1 <= k, p <= min(d, 64)");
  qr_dev(c, S, lds, d, p, /*count=*/false);
  double* G = c.small.ensure(static_cast<size_t>(64) * 64 * 4 + 8);
  double* H = G + 64 * 64;
  double* part = c.tmp.ensure(static_cast<size_t>(small_gram_parts(std::max(d, p))) * 64 * 64 + 8);
  launch_small_gram(S, lds, p, U, ldu, k, d, part, G, c.st);  // Gᵀ: p x k, ld = k
  launch_small_gram(G, k, k, G, k, k, p, part, H, c.st);      // H = G Gᵀ: k x k
  DBuf<double> vv;
  double* vals = vv.ensure(static_cast<size_t>(k) + static_cast<size_t>(k) * k);
  launch_jacobi(H, k, vals, vals + k, c.st);
  GAPLRA_CUDA_CHECK(cudaMemcpyAsync(c.pin, vals, k * sizeof(double), cudaMemcpyDeviceToHost, c.st));
  c.sync();
  for (int a = 0; a < k; ++a) cos_host[a] = std::sqrt(std::min(std::max(c.pin[a], 0.0), 1.0));
}

// approximate — Alg. 7, the device form of oracle.cpp
// approximate with the same pins: per interval {s..k} on A_{-(s-1)}, Alg. 3 at
// eps' = 1/(9p^2) -> Alg. 4; a multiplicative gap q gives PlainPower on
// {s..q} (width q-s+1, L = ceil(4 p^4 ln(kd/eps_int))); otherwise tune_shift
// on the deflated operators, Alg. 3 on D_{-(s-1)} at eps' = 1/(9p) -> Alg. 5
// -> ShiftedInverse (width q-s+1 or p-s+1 at q = k, L = ceil(4 k ln(kd/eps_int)));
// NoPreconditioningNeeded -> PlainPower with width p-s+1, q = k.  Deflated
// shifted systems are solved by CG; the first interval's by the configured
// backend.  Finally restricted_projection(A, basis, k).
constexpr uint64_t kTagInterval = 0x696e7476ull;  // "intv"
constexpr uint64_t kTagGapBudget = 0x67617062ull;  // "gapb"

// find_gap_budget (oracle.cpp find_gap_budget): Alg. 3 on A with p + 1 columns
// at eps' = 1/100, Delta0 = lambda_hat_k - lambda_hat_{p+1}, Delta = Delta0 / 1.5.
double find_gap_budget_dev(Context& c, Matrix& X, int k, int p, uint64_t seed, double rq_tol) {
  if (k < 1 || p <= k || p + 1 > 64 || p + 1 > X.d)
    throw Error(kContractViolation, "find_gap_budget: need 1 <= k < p, p + 1 <= min(d, 64)");
  GramOp a(c, X);
  const std::vector<double> est =
      estimate_eigs_dev(c, a, X.d, X.d_pad(), p + 1, 0.01, derive_seed(seed, kTagGapBudget), rq_tol, nullptr);
  const double d0 = est[k - 1] - est[p];
  if (!(d0 > 1e-14 * est[0])) throw Error(kNoUsableGap, "find_gap_budget: no gap between lambda_k and lambda_{p+1}");
  return d0 / 1.5;
}

void approximate_dev(Context& c, Matrix& X, const gaplra_si_config& cfg, double* W, double* ritz_host,
                     gaplra_ap_report& rep) {
  const int d = X.d, k = cfg.k, p = cfg.p;
  const int64_t dp = X.d_pad();
  if (k < 1 || p <= k || p >= d || p > 64) throw Error(kContractViolation, "approximate: need 1 <= k < p < d, p <= 64");
  gaplra_si_config cfg_d = cfg;
  if (!(cfg_d.delta > 0.0)) cfg_d.delta = find_gap_budget_dev(c, X, k, p, cfg.seed, cfg.rq_tol);
  rep.delta = cfg_d.delta;
  const gaplra_si_config& cfgd = cfg_d;
  const double eps_int = cfg.eps / (3.0 * std::max(cfg.mu, 1.0) * k * d);
  const double lg = std::log(k * static_cast<double>(d) / eps_int);
  auto capped = [&](double L) {
    const int l = static_cast<int>(std::min(std::ceil(L), 1e9));
    return cfg.max_outer > 0 ? std::min(l, cfg.max_outer) : l;
  };
  DBuf<double> ubs[2], sb;
  int cur = 0;
  double* U = nullptr;
  int m = 0;
  int64_t solves = 0;
  int s = 1;
  for (int j = 0; s <= k; ++j) {
    if (j >= k) throw Error(kDegenerateProgress, "approximate: more intervals than target indices (DegenerateProgress)");
    gaplra_si_config cj = cfg;
    cj.seed = derive_seed(cfg.seed, kTagInterval + static_cast<uint64_t>(j));
    GramOp a0(c, X);
    DeflatedOp a(c, a0, U, m, d, dp);
    const int cnt = k - s + 1;
    const std::vector<double> est =
        estimate_eigs_dev(c, a, d, dp, cnt, 1.0 / (9.0 * p * p), derive_seed(cj.seed, kTagEstA), cfg.rq_tol, nullptr);
    int q = detect_multiplicative_gap_host(est.data(), cnt, s, p);
    int strategy = 0, width = 0, iters = 0;
    double shift = 0.0;
    double* S = nullptr;
    auto plain = [&](int wdt) {
      strategy = 0;
      width = wdt;
      S = sb.ensure(static_cast<size_t>(dp) * ldp_of(wdt));
      iters = subspace_iterate_dev(c, a, d, dp, wdt, capped(4.0 * std::pow(static_cast<double>(p), 4) * lg),
                                   derive_seed(cj.seed, kTagSubspace), cfg.conv_tol, S);
    };
    if (q >= 0) {
      plain(q - s + 1);
    } else {
      gaplra_si_report tr;
      std::memset(&tr, 0, sizeof(tr));
      bool shifted = true;
      try {
        tune_shift_dev(c, X, cfgd.delta, cj, &solves, tr, U, m);
      } catch (const Error& e) {
        if (e.code != kNoPreconditioningNeeded) throw;
        shifted = false;
      }
      if (!shifted) {
        q = k;
        plain(p - s + 1);
      } else {
        shift = tr.lambda;
        gaplra_svrg_params prm = prm_from(cj, cfg.tol_solve);
        prm.lambda1_hint = tr.lambda1_hint;
        InverseOp dinv(c, X, shift, prm, &solves);
        CgOp dcg(c, X, shift, cfg.tol_solve, U, m);
        DeflatedOp dd(c, cfg.backend == 1 || m > 0 ? static_cast<Op&>(dcg) : static_cast<Op&>(dinv), U, m, d, dp);
        const std::vector<double> dest = estimate_eigs_dev(c, dd, d, dp, cnt, 1.0 / (9.0 * p),
                                                           derive_seed(cj.seed, kTagEstD), cfg.rq_tol, nullptr);
        std::vector<double> inv(cnt);
        for (int i = 0; i < cnt; ++i) inv[i] = 1.0 / std::max(dest[i], 1e-300);
        q = detect_additive_gap_host(inv.data(), cnt, s, k, cfgd.delta);
        strategy = 1;
        width = q < k ? q - s + 1 : p - s + 1;
        S = sb.ensure(static_cast<size_t>(dp) * ldp_of(width));
        iters = subspace_iterate_dev(c, dd, d, dp, width, capped(4.0 * k * lg), derive_seed(cj.seed, kTagSubspace),
                                     cfg.conv_tol, S);
      }
    }
    // deflation_basis_extend (oracle.cpp basis_extend): project, QR, append;
    // a new column in span(U) is a duplicated eigendirection
    project_out_dev(c, U, m, S, ldp_of(width), d, width);
    try {
      qr_dev(c, S, ldp_of(width), d, width, /*count=*/false);
    } catch (const Error& e) {
      if (e.code != kRankDeficient || m == 0) throw;
      throw Error(kDegenerateProgress, std::string("approximate: deflation_basis_extend: ") + e.what(), e.payload);
    }
    const int m2 = m + width;
    if (m2 > 64) throw Error(kContractViolation, "approximate: basis wider than 64 columns");
    double* U2 = ubs[cur ^ 1].ensure(static_cast<size_t>(dp) * ldp_of(m2));
    GAPLRA_CUDA_CHECK(cudaMemsetAsync(U2, 0, static_cast<size_t>(dp) * ldp_of(m2) * sizeof(double), c.st));
    if (m > 0)
      GAPLRA_CUDA_CHECK(cudaMemcpy2DAsync(U2, ldp_of(m2) * sizeof(double), U, ldp_of(m) * sizeof(double),
                                          m * sizeof(double), d, cudaMemcpyDeviceToDevice, c.st));
    GAPLRA_CUDA_CHECK(cudaMemcpy2DAsync(U2 + m, ldp_of(m2) * sizeof(double), S, ldp_of(width) * sizeof(double),
                                        width * sizeof(double), d, cudaMemcpyDeviceToDevice, c.st));
    cur ^= 1;
    U = U2;
    m = m2;
    if (rep.n_intervals < 64) {
      const int t = rep.n_intervals;
      rep.s[t] = s;
      rep.q[t] = q;
      rep.strategy[t] = strategy;
      rep.width[t] = width;
      rep.iterations[t] = iters;
      rep.shift[t] = shift;
    }
    rep.n_intervals++;
    s = q + 1;
  }
  restricted_projection_dev(c, X, U, m, k, W, ritz_host);
}

int outer_cap(const gaplra_si_config& cfg, int d) {
  if (cfg.max_outer > 0) return cfg.max_outer;
  const double eps_int = cfg.eps / (3.0 * std::max(cfg.mu, 1.0) * cfg.k * d);
  return static_cast<int>(std::ceil(4.0 * cfg.k * std::log(cfg.k * static_cast<double>(d) / eps_int)));
}

// ---------------------------------------------------------------------------
// Host <-> device block helpers for the C ABI (host row-major, ld = p).
// ---------------------------------------------------------------------------
void upload_block(Context& c, const double* h, int rows, int p, double* dbuf, int64_t ld) {
  GAPLRA_CUDA_CHECK(cudaMemcpy2DAsync(dbuf, ld * sizeof(double), h, p * sizeof(double), p * sizeof(double), rows,
                                      cudaMemcpyHostToDevice, c.st));
}
void download_block(Context& c, const double* dbuf, int64_t ld, int rows, int p, double* h) {
  GAPLRA_CUDA_CHECK(cudaMemcpy2DAsync(h, p * sizeof(double), dbuf, ld * sizeof(double), p * sizeof(double), rows,
                                      cudaMemcpyDeviceToHost, c.st));
}

bool all_finite(const double* v, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (!std::isfinite(v[i])) return false;
  return true;
}

}  // namespace gaplra_cuda

using namespace gaplra_cuda;

struct gaplra_ctx {
  Context c;
};
struct gaplra_matrix {
  Matrix m;
  gaplra_ctx* owner;
};

namespace {

template <class F>
int guard(gaplra_ctx* ctx, F&& f) {
  try {
    if (ctx) GAPLRA_CUDA_CHECK(cudaSetDevice(ctx->c.device));
    f();
    if (ctx) ctx->c.err.clear();
    return GAPLRA_OK;
  } catch (const Error& e) {
    if (ctx) ctx->c.err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    if (ctx) ctx->c.err = e.what();
    return GAPLRA_DEVICE_ERROR;
  }
}

void require(bool ok, const char* what) {
  if (!ok) throw Error(kContractViolation, what);
}

}  // namespace

extern "C" {

int gaplra_version(void) { return 1; }

int gaplra_ctx_create(int device, gaplra_ctx** out) {
  if (!out) return GAPLRA_CONTRACT_VIOLATION;
  *out = nullptr;
  gaplra_ctx* ctx = new gaplra_ctx();
  int rc = guard(nullptr, [&] {
    int count = 0;
    GAPLRA_CUDA_CHECK(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) throw Error(kDeviceError, "no such CUDA device");
    ctx->c.device = device;
    GAPLRA_CUDA_CHECK(cudaSetDevice(device));
    int lo = 0, hi = 0;
    GAPLRA_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    GAPLRA_CUDA_CHECK(cudaStreamCreateWithPriority(&ctx->c.own, cudaStreamNonBlocking, hi));  // main: highest
    ctx->c.st = ctx->c.own;
    GAPLRA_CUDA_CHECK(cudaMallocHost(&ctx->c.pin, 64 * sizeof(double)));
    GAPLRA_CUDA_CHECK(cudaMallocHost(&ctx->c.pin_i, 64 * sizeof(int)));
  });
  if (rc != GAPLRA_OK) {
    delete ctx;
    return rc;
  }
  *out = ctx;
  return GAPLRA_OK;
}

int gaplra_ctx_destroy(gaplra_ctx* ctx) {
  if (!ctx) return GAPLRA_OK;
  cudaSetDevice(ctx->c.device);
  cudaStreamSynchronize(ctx->c.st);
  delete ctx;
  return GAPLRA_OK;
}

const char* gaplra_last_error(const gaplra_ctx* ctx) { return ctx ? ctx->c.err.c_str() : "null context"; }

int gaplra_ctx_set_stream(gaplra_ctx* ctx, void* s) {
  if (!ctx) return GAPLRA_CONTRACT_VIOLATION;
  ctx->c.st = s ? static_cast<cudaStream_t>(s) : ctx->c.own;
  return GAPLRA_OK;
}

int gaplra_ctx_synchronize(gaplra_ctx* ctx) {
  if (!ctx) return GAPLRA_CONTRACT_VIOLATION;
  return guard(ctx, [&] { ctx->c.sync(); });
}

int gaplra_ledger_get(const gaplra_ctx* ctx, gaplra_ledger* out) {
  if (!ctx || !out) return GAPLRA_CONTRACT_VIOLATION;
  *out = ctx->c.led;
  return GAPLRA_OK;
}

int gaplra_ledger_reset(gaplra_ctx* ctx) {
  if (!ctx) return GAPLRA_CONTRACT_VIOLATION;
  ctx->c.led = gaplra_ledger{};
  return GAPLRA_OK;
}

unsigned long long gaplra_launch_count(void) { return launch_counter(); }

unsigned long long gaplra_host_syncs(const gaplra_ctx* ctx) { return ctx ? ctx->c.host_syncs : 0ull; }

int gaplra_profile_enable(gaplra_ctx* ctx, int on) {
  if (!ctx) return GAPLRA_CONTRACT_VIOLATION;
  return guard(ctx, [&] {
    ctx->c.sync();
    ctx->c.profiling = on != 0;
  });
}

int gaplra_profile_get(gaplra_ctx* ctx, gaplra_profile* out) {
  if (!ctx || !out) return GAPLRA_CONTRACT_VIOLATION;
  return guard(ctx, [&] {
    ctx->c.sync();
    *out = ctx->c.prof;
  });
}

int gaplra_profile_reset(gaplra_ctx* ctx) {
  if (!ctx) return GAPLRA_CONTRACT_VIOLATION;
  return guard(ctx, [&] {
    ctx->c.sync();
    ctx->c.prof = gaplra_profile{};
  });
}

int gaplra_matrix_dense(gaplra_ctx* ctx, int d, int n, const double* x, int64_t ldx, int on_device,
                        gaplra_matrix** out) {
  if (!ctx || !out) return GAPLRA_CONTRACT_VIOLATION;
  *out = nullptr;
  gaplra_matrix* M = new gaplra_matrix();
  M->owner = ctx;
  int rc = guard(ctx, [&] {
    require(d > 0 && n > 0 && x && ldx >= d, "matrix_dense: bad dimensions");
    Matrix& m = M->m;
    m.kind = 0;
    m.d = d;
    m.n = n;
    m.nnz = static_cast<int64_t>(d) * n;
    m.device = ctx->c.device;
    if (on_device) {
      // the kernels size W, Z and the per-CTA row split by ld: a borrowed X must
      // use the library's own layout, ld = round4(d), with zero pad rows
      require(ldx == round4(d), "matrix_dense: borrowed device X needs ldx == round_up(d, 4) (zero pad rows)");
      m.ld = ldx;
      m.x = x;
    } else {
      m.ld = round4(d);
      double* buf = m.xbuf.ensure(static_cast<size_t>(m.ld) * n);
      GAPLRA_CUDA_CHECK(cudaMemcpy2DAsync(buf, m.ld * sizeof(double), x, ldx * sizeof(double), d * sizeof(double), n,
                                          cudaMemcpyHostToDevice, ctx->c.st));
      m.x = buf;
    }
    // one device read of X: finite entries (sparse_matrix.cpp:29) and zero pad rows
    int* flags = ctx->c.status.ensure(2);
    check_dense(m.dense(), flags, ctx->c.st);
    GAPLRA_CUDA_CHECK(cudaMemcpyAsync(ctx->c.pin_i, flags, sizeof(int), cudaMemcpyDeviceToHost, ctx->c.st));
    ctx->c.sync();
    require(!(ctx->c.pin_i[0] & 1), "matrix_dense: X has a non-finite entry");
    require(!(ctx->c.pin_i[0] & 2), "matrix_dense: borrowed X has non-zero pad rows (rows d..ldx-1 must be zero)");
  });
  if (rc != GAPLRA_OK) {
    delete M;
    return rc;
  }
  *out = M;
  return GAPLRA_OK;
}

int gaplra_matrix_csc(gaplra_ctx* ctx, int d, int n, const int64_t* colptr, const int32_t* rowidx, const double* val,
                      int on_device, gaplra_matrix** out) {
  if (!ctx || !out) return GAPLRA_CONTRACT_VIOLATION;
  *out = nullptr;
  gaplra_matrix* M = new gaplra_matrix();
  M->owner = ctx;
  int rc = guard(ctx, [&] {
    require(d > 0 && n > 0 && colptr, "matrix_csc: bad dimensions");
    Matrix& m = M->m;
    m.kind = 1;
    m.d = d;
    m.n = n;
    m.device = ctx->c.device;
    std::vector<int64_t> cp(static_cast<size_t>(n) + 1);
    if (on_device)
      GAPLRA_CUDA_CHECK(cudaMemcpy(cp.data(), colptr, cp.size() * sizeof(int64_t), cudaMemcpyDeviceToHost));
    else
      std::memcpy(cp.data(), colptr, cp.size() * sizeof(int64_t));
    const int64_t nnz = cp[n];
    require(cp[0] == 0 && nnz >= 0, "matrix_csc: colptr must start at 0");
    std::vector<int32_t> ri(static_cast<size_t>(nnz));
    std::vector<double> v(static_cast<size_t>(nnz));
    if (on_device) {
      GAPLRA_CUDA_CHECK(cudaMemcpy(ri.data(), rowidx, nnz * sizeof(int32_t), cudaMemcpyDeviceToHost));
      GAPLRA_CUDA_CHECK(cudaMemcpy(v.data(), val, nnz * sizeof(double), cudaMemcpyDeviceToHost));
    } else {
      std::memcpy(ri.data(), rowidx, nnz * sizeof(int32_t));
      std::memcpy(v.data(), val, nnz * sizeof(double));
    }
    // Validation as SparseColumnsMatrix's ctor (sparse_matrix.cpp:10-37).
    for (int j = 0; j < n; ++j) {
      require(cp[j + 1] >= cp[j], "matrix_csc: colptr not monotone");
      int prev = -1;
      for (int64_t e = cp[j]; e < cp[j + 1]; ++e) {
        require(ri[e] >= 0 && ri[e] < d, "matrix_csc: row index out of range");
        require(ri[e] > prev, "matrix_csc: indices not strictly increasing");
        require(std::isfinite(v[e]), "matrix_csc: non-finite value");
        prev = ri[e];
      }
    }
    // CSR copy (row access) for the gather form of Z = X Y.
    std::vector<int64_t> rp(static_cast<size_t>(d) + 1, 0);
    for (int64_t e = 0; e < nnz; ++e) rp[ri[e] + 1]++;
    for (int r = 0; r < d; ++r) rp[r + 1] += rp[r];
    std::vector<int32_t> ci(static_cast<size_t>(nnz));
    std::vector<double> rv(static_cast<size_t>(nnz));
    std::vector<int64_t> fill(rp.begin(), rp.end() - 1);
    for (int j = 0; j < n; ++j)
      for (int64_t e = cp[j]; e < cp[j + 1]; ++e) {
        const int64_t o = fill[ri[e]]++;
        ci[o] = j;
        rv[o] = v[e];
      }
    m.nnz = nnz;
    m.ld = round4(d);
    for (int j = 0; j < n; ++j) m.max_col_nnz = std::max(m.max_col_nnz, static_cast<int>(cp[j + 1] - cp[j]));
    auto up = [&](auto& buf, const auto& hv) {
      buf.ensure(hv.size());
      GAPLRA_CUDA_CHECK(cudaMemcpy(buf.p, hv.data(), hv.size() * sizeof(hv[0]), cudaMemcpyHostToDevice));
    };
    up(m.colptr, cp);
    up(m.rowidx, ri);
    up(m.val, v);
    up(m.rowptr, rp);
    up(m.colidx, ci);
    up(m.rval, rv);
  });
  if (rc != GAPLRA_OK) {
    delete M;
    return rc;
  }
  *out = M;
  return GAPLRA_OK;
}

int gaplra_matrix_destroy(gaplra_matrix* x) {
  if (!x) return GAPLRA_OK;
  cudaSetDevice(x->m.device);
  delete x;
  return GAPLRA_OK;
}

int gaplra_matrix_info(const gaplra_matrix* x, int* d, int* n, int64_t* nnz, int64_t* ld) {
  if (!x) return GAPLRA_CONTRACT_VIOLATION;
  if (d) *d = x->m.d;
  if (n) *n = x->m.n;
  if (nnz) *nnz = x->m.nnz;
  if (ld) *ld = x->m.ld;
  return GAPLRA_OK;
}

int gaplra_gram_block(gaplra_ctx* ctx, const gaplra_matrix* x, int p, const double* w, double* z, double* y) {
  if (!ctx || !x) return GAPLRA_CONTRACT_VIOLATION;
  return guard(ctx, [&] {
    Context& c = ctx->c;
    const Matrix& X = const_cast<gaplra_matrix*>(x)->m;
    require(p >= 1 && w && z, "gram_block: bad arguments");
    require(all_finite(w, static_cast<size_t>(X.d) * p), "gram_apply: non-finite input");
    const int64_t ld = ldp_of(p), dp = X.d_pad();
    DBuf<double> wd, zd, yd;
    wd.ensure(static_cast<size_t>(dp) * ld);
    zd.ensure(static_cast<size_t>(dp) * ld);
    yd.ensure(static_cast<size_t>(X.n) * ld);
    upload_block(c, w, X.d, p, wd.p, ld);
    gram_block_dev(c, X, p, wd.p, ld, zd.p, ld, yd.p, ld);
    download_block(c, zd.p, ld, X.d, p, z);
    if (y) download_block(c, yd.p, ld, X.n, p, y);
    c.sync();
  });
}

int gaplra_gram_apply(gaplra_ctx* ctx, const gaplra_matrix* x, const double* v, double* out) {
  const int rc = gaplra_gram_block(ctx, x, 1, v, out, nullptr);
  if (rc == GAPLRA_OK && ctx) ctx->c.led.operator_applies++;
  return rc;
}

int gaplra_gram_block_device(gaplra_ctx* ctx, const gaplra_matrix* x, int p, const double* w, int64_t ldw, double* z,
                             int64_t ldz, double* y, int64_t ldy) {
  if (!ctx || !x) return GAPLRA_CONTRACT_VIOLATION;
  return guard(ctx, [&] {
    require(p >= 1 && w && z, "gram_block_device: bad arguments");
    require(p == 1 || (ldw % 2 == 0 && ldz % 2 == 0 && (!y || ldy % 2 == 0)), "gram_block_device: ld must be even");
    gram_block_dev(ctx->c, x->m, p, w, ldw, z, ldz, y, ldy);
  });
}

int gaplra_index_stream(gaplra_ctx* ctx, uint64_t seed, uint64_t n, int64_t m, int32_t* out) {
  if (!ctx) return GAPLRA_CONTRACT_VIOLATION;
  return guard(ctx, [&] {
    require(n >= 1 && n < (1ull << 31) && m >= 0 && (m == 0 || out), "index_stream: bad arguments");
    Context& c = ctx->c;
    int32_t* d = c.idx.ensure(static_cast<size_t>(std::max<int64_t>(m, 1)));
    launch_index_stream(seed, n, m, d, c.rej.ensure(1), c.st);
    if (m) GAPLRA_CUDA_CHECK(cudaMemcpyAsync(out, d, m * sizeof(int32_t), cudaMemcpyDeviceToHost, c.st));
    c.sync();
  });
}

int gaplra_gaussian_init(int d, int p, uint64_t seed, double* out) {
  if (!out) return GAPLRA_CONTRACT_VIOLATION;
  return guard(nullptr, [&] { gaussian_init_host(d, p, seed, out, p); });
}

int gaplra_qr_orthonormalize(gaplra_ctx* ctx, int d, int p, const double* y, double* q, int* bad_col) {
  if (!ctx) return GAPLRA_CONTRACT_VIOLATION;
  if (bad_col) *bad_col = -1;
  return guard(ctx, [&] {
    require(y && q && p >= 1 && d >= p, "qr_orthonormalize: need 1 <= cols <= rows");
    require(all_finite(y, static_cast<size_t>(d) * p), "qr_orthonormalize: non-finite entry");
    Context& c = ctx->c;
    const int64_t ld = ldp_of(p);
    DBuf<double> b;
    b.ensure(static_cast<size_t>(round4(d)) * ld);
    upload_block(c, y, d, p, b.p, ld);
    try {
      qr_dev(c, b.p, ld, d, p, /*count=*/false);
    } catch (const Error& e) {
      if (e.code == kRankDeficient && bad_col) *bad_col = e.payload;
      throw;
    }
    download_block(c, b.p, ld, d, p, q);
    c.sync();
  });
}

int gaplra_orthonormality_defect(gaplra_ctx* ctx, int d, int p, const double* q, double* defect) {
  if (!ctx || !q || !defect) return GAPLRA_CONTRACT_VIOLATION;
  return guard(ctx, [&] {
    require(p >= 1 && p <= 64, "orthonormality_defect: 1 <= p <= 64");
    Context& c = ctx->c;
    const int64_t ld = ldp_of(p);
    DBuf<double> b;
    b.ensure(static_cast<size_t>(round4(d)) * ld);
    upload_block(c, q, d, p, b.p, ld);
    double* G = c.small.ensure(static_cast<size_t>(64) * 64 * 4 + 8);
    double* part = c.tmp.ensure(static_cast<size_t>(small_gram_parts(d)) * 64 * 64 + 8);
    launch_small_gram(b.p, ld, p, b.p, ld, p, d, part, G, c.st);
    std::vector<double> h(static_cast<size_t>(p) * p);
    GAPLRA_CUDA_CHECK(cudaMemcpyAsync(h.data(), G, h.size() * sizeof(double), cudaMemcpyDeviceToHost, c.st));
    c.sync();
    double worst = 0.0;
    for (int i = 0; i < p; ++i)
      for (int j = 0; j < p; ++j) worst = std::max(worst, std::fabs(h[i * p + j] - (i == j ? 1.0 : 0.0)));
    *defect = worst;
  });
}

int gaplra_jacobi_eigh(gaplra_ctx* ctx, int n, const double* h, double* vals, double* vecs) {
  if (!ctx) return GAPLRA_CONTRACT_VIOLATION;
  return guard(ctx, [&] {
    require(h && vals && vecs && n >= 1 && n <= kJacobiMax, "jacobi_eigh: need a square matrix with n <= 64");
    Context& c = ctx->c;
    DBuf<double> b;
    b.ensure(static_cast<size_t>(n) * n * 2 + n);
    GAPLRA_CUDA_CHECK(cudaMemcpyAsync(b.p, h, static_cast<size_t>(n) * n * sizeof(double), cudaMemcpyHostToDevice, c.st));
    double* dv = b.p + n * n;
    double* dvec = dv + n;
    launch_jacobi(b.p, n, dv, dvec, c.st);
    GAPLRA_CUDA_CHECK(cudaMemcpyAsync(vals, dv, n * sizeof(double), cudaMemcpyDeviceToHost, c.st));
    GAPLRA_CUDA_CHECK(cudaMemcpyAsync(vecs, dvec, static_cast<size_t>(n) * n * sizeof(double), cudaMemcpyDeviceToHost, c.st));
    c.sync();
  });
}

int gaplra_svrg_epoch(gaplra_ctx* ctx, const gaplra_matrix* x, int p, double* w, const double* y, const double* cc,
                      double eta, double lambda, uint64_t stream_seed, int64_t m) {
  if (!ctx || !x) return GAPLRA_CONTRACT_VIOLATION;
  return guard(ctx, [&] {
    require(p >= 1 && w && y && cc && m >= 0, "svrg_epoch: bad arguments");
    Context& c = ctx->c;
    Matrix& X = const_cast<gaplra_matrix*>(x)->m;
    const int64_t ld = ldp_of(p), dp = X.d_pad();
    DBuf<double> wd, cd, yd;
    wd.ensure(static_cast<size_t>(dp) * ld);
    cd.ensure(static_cast<size_t>(dp) * ld);
    yd.ensure(static_cast<size_t>(X.n) * ld);
    upload_block(c, w, X.d, p, wd.p, ld);
    upload_block(c, cc, X.d, p, cd.p, ld);
    upload_block(c, y, X.n, p, yd.p, ld);
    epoch_dev(c, X, p, wd.p, cd.p, yd.p, eta, lambda, stream_seed, m);
    download_block(c, wd.p, ld, X.d, p, w);
    c.sync();
  });
}

int gaplra_svrg_solve(gaplra_ctx* ctx, const gaplra_matrix* x, double lambda, int p, const double* b, double* w,
                      const gaplra_svrg_params* prm, int64_t solve_id, int* epochs, double* history, int hist_cap,
                      int* hist_len) {
  if (!ctx || !x || !prm) return GAPLRA_CONTRACT_VIOLATION;
  return guard(ctx, [&] {
    require(p >= 1 && p <= 64 && b && w, "solve_svrg: bad arguments");
    require(all_finite(b, static_cast<size_t>(x->m.d) * p), "solve_svrg: non-finite right-hand side");
    Context& c = ctx->c;
    Matrix& X = const_cast<gaplra_matrix*>(x)->m;
    const int64_t ld = ldp_of(p), dp = X.d_pad();
    DBuf<double> bd, wd;
    bd.ensure(static_cast<size_t>(dp) * ld);
    wd.ensure(static_cast<size_t>(dp) * ld);
    upload_block(c, b, X.d, p, bd.p, ld);
    SvrgResult r;
    auto report = [&] {
      if (epochs) *epochs = r.epochs;
      if (hist_len) *hist_len = static_cast<int>(r.history.size());
      if (history)
        for (int i = 0; i < std::min<int>(hist_cap, static_cast<int>(r.history.size())); ++i) history[i] = r.history[i];
    };
    try {
      r = svrg_solve_dev(c, X, lambda, p, bd.p, wd.p, *prm, solve_id, &r);
    } catch (...) {
      report();
      throw;
    }
    download_block(c, wd.p, ld, X.d, p, w);
    c.sync();
    report();
  });
}

int gaplra_estimate_top(gaplra_ctx* ctx, const gaplra_matrix* x, int inverse, double lambda, double eps_prime,
                        uint64_t seed, double rq_tol, const gaplra_svrg_params* prm, int64_t* solve_counter,
                        double* value, int* iterations) {
  if (!ctx || !x || !value) return GAPLRA_CONTRACT_VIOLATION;
  return guard(ctx, [&] {
    require(eps_prime > 0.0 && eps_prime < 1.0, "estimate_eigenvalues: eps' in (0, 1)");
    Context& c = ctx->c;
    Matrix& X = const_cast<gaplra_matrix*>(x)->m;
    int64_t local = 0;
    if (inverse) {
      require(prm != nullptr, "estimate_top: inverse needs svrg params");
      InverseOp op(c, X, lambda, *prm, solve_counter ? solve_counter : &local);
      *value = estimate_top_dev(c, op, X.d, X.d_pad(), eps_prime, seed, rq_tol, iterations);
    } else {
      GramOp op(c, X);
      *value = estimate_top_dev(c, op, X.d, X.d_pad(), eps_prime, seed, rq_tol, iterations);
    }
  });
}

int gaplra_tune_shift(gaplra_ctx* ctx, const gaplra_matrix* x, double delta, const gaplra_si_config* cfg,
                      int64_t* solve_counter, gaplra_si_report* rep) {
  if (!ctx || !x || !cfg || !rep) return GAPLRA_CONTRACT_VIOLATION;
  std::memset(rep, 0, sizeof(*rep));
  return guard(ctx, [&] {
    int64_t local = 0;
    Timer t(ctx->c, &rep->ms_tune);
    tune_shift_dev(ctx->c, const_cast<gaplra_matrix*>(x)->m, delta, *cfg, solve_counter ? solve_counter : &local, *rep);
  });
}

int gaplra_restricted_projection(gaplra_ctx* ctx, const gaplra_matrix* x, int p, const double* s, int k, double* w,
                                 double* ritz) {
  if (!ctx || !x) return GAPLRA_CONTRACT_VIOLATION;
  return guard(ctx, [&] {
    require(s && w && ritz && k >= 1 && k <= p && p <= 64, "restricted_projection: bad arguments");
    Context& c = ctx->c;
    Matrix& X = const_cast<gaplra_matrix*>(x)->m;
    const int64_t ld = ldp_of(p), dp = X.d_pad();
    DBuf<double> sd, wd;
    sd.ensure(static_cast<size_t>(dp) * ld);
    wd.ensure(static_cast<size_t>(dp) * ldp_of(k));
    upload_block(c, s, X.d, p, sd.p, ld);
    restricted_projection_dev(c, X, sd.p, p, k, wd.p, ritz);
    download_block(c, wd.p, ldp_of(k), X.d, k, w);
    c.sync();
  });
}

int gaplra_shift_invert(gaplra_ctx* ctx, const gaplra_matrix* x, const gaplra_si_config* cfg, double* w, double* ritz,
                        double* s, gaplra_si_report* rep) {
  if (!ctx || !x || !cfg || !rep) return GAPLRA_CONTRACT_VIOLATION;
  std::memset(rep, 0, sizeof(*rep));
  return guard(ctx, [&] {
    Context& c = ctx->c;
    Matrix& X = const_cast<gaplra_matrix*>(x)->m;
    require(cfg->k >= 1 && cfg->p > cfg->k && cfg->p < X.d && cfg->p <= 64, "shift_invert: need 1 <= k < p < d, p <= 64");
    require(w && ritz, "shift_invert: null output");
    const gaplra_ledger before = c.led;
    Timer total(c, &rep->ms_total);
    int64_t solves = 0;
    if (cfg->lambda > 0.0) {
      rep->lambda = cfg->lambda;
      rep->lambda1_hint = cfg->lambda1_hint;
    } else {
      Timer t(c, &rep->ms_tune);
      tune_shift_dev(c, X, cfg->delta, *cfg, &solves, *rep);
    }
    const int p = cfg->p, k = cfg->k;
    const int64_t ld = ldp_of(p), dp = X.d_pad();
    DBuf<double> sb, wb;
    double* S = sb.ensure(static_cast<size_t>(dp) * ld);
    {
      Timer t(c, &rep->ms_subspace);
      gaplra_svrg_params prm = prm_from(*cfg, cfg->tol_solve);
      prm.lambda1_hint = rep->lambda1_hint;
      InverseOp dinv(c, X, rep->lambda, prm, &solves);
      CgOp dcg(c, X, rep->lambda, cfg->tol_solve);
      AccOp dacc(c, X, rep->lambda, prm, &solves);
      Op& op = cfg->backend == 1 ? static_cast<Op&>(dcg) : cfg->backend == 2 ? static_cast<Op&>(dacc) : static_cast<Op&>(dinv);
      rep->outer_cap = outer_cap(*cfg, X.d);
      rep->outer_iterations = subspace_iterate_dev(c, op, X.d, dp, p, rep->outer_cap,
                                                   derive_seed(cfg->seed, kTagSubspace), cfg->conv_tol, S);
    }
    double* W = wb.ensure(static_cast<size_t>(dp) * ldp_of(k));
    {
      Timer t(c, &rep->ms_rayleigh_ritz);
      restricted_projection_dev(c, X, S, p, k, W, ritz);
    }
    download_block(c, W, ldp_of(k), X.d, k, w);
    if (s) download_block(c, S, ld, X.d, p, s);
    c.sync();
    gaplra_ledger& L = rep->ledger;
    L.gram_applies = c.led.gram_applies - before.gram_applies;
    L.operator_applies = c.led.operator_applies - before.operator_applies;
    L.qr_factorizations = c.led.qr_factorizations - before.qr_factorizations;
    L.linear_solves = c.led.linear_solves - before.linear_solves;
    L.solver_column_samples = c.led.solver_column_samples - before.solver_column_samples;
    L.epochs = c.led.epochs - before.epochs;
    L.outer_iterations = c.led.outer_iterations - before.outer_iterations;
  });
}

int gaplra_cg_solve(gaplra_ctx* ctx, const gaplra_matrix* x, double lambda, int p, const double* b, double* w,
                    double tol, int max_iter, int* iterations, double* history, int hist_cap, int* hist_len) {
  if (!ctx || !x) return GAPLRA_CONTRACT_VIOLATION;
  return guard(ctx, [&] {
    require(p >= 1 && p <= 64 && b && w && tol > 0.0, "solve_cg: bad arguments");
    require(all_finite(b, static_cast<size_t>(x->m.d) * p), "solve_cg: non-finite right-hand side");
    Context& c = ctx->c;
    Matrix& X = const_cast<gaplra_matrix*>(x)->m;
    const int64_t ld = ldp_of(p), dp = X.d_pad();
    DBuf<double> bd, wd;
    bd.ensure(static_cast<size_t>(dp) * ld);
    wd.ensure(static_cast<size_t>(dp) * ld);
    GAPLRA_CUDA_CHECK(cudaMemsetAsync(bd.p, 0, static_cast<size_t>(dp) * ld * sizeof(double), c.st));
    upload_block(c, b, X.d, p, bd.p, ld);
    CgResult r;
    auto report = [&] {
      if (iterations) *iterations = r.iterations;
      if (hist_len) *hist_len = static_cast<int>(r.history.size());
      if (history)
        for (int i = 0; i < std::min<int>(hist_cap, static_cast<int>(r.history.size())); ++i) history[i] = r.history[i];
    };
    try {
      r = cg_solve_dev(c, X, lambda, p, bd.p, wd.p, tol, max_iter, false, &r);
    } catch (...) {
      report();
      throw;
    }
    download_block(c, wd.p, ld, X.d, p, w);
    c.sync();
    report();
  });
}

int gaplra_error_report(gaplra_ctx* ctx, const gaplra_matrix* x, int k, const double* w, int iters, uint64_t seed,
                        double* frob, double* spec) {
  if (!ctx || !x || !frob || !spec) return GAPLRA_CONTRACT_VIOLATION;
  return guard(ctx, [&] {
    Context& c = ctx->c;
    Matrix& X = const_cast<gaplra_matrix*>(x)->m;
    require(k >= 0 && k <= 64 && k <= X.d && (k == 0 || w) && iters >= 0, "error_report: bad arguments");
    const int64_t ldk = ldp_of(std::max(k, 1)), dp = X.d_pad();
    DBuf<double> wd;
    wd.ensure(static_cast<size_t>(dp) * ldk);
    GAPLRA_CUDA_CHECK(cudaMemsetAsync(wd.p, 0, static_cast<size_t>(dp) * ldk * sizeof(double), c.st));
    if (k > 0) upload_block(c, w, X.d, k, wd.p, ldk);
    error_report_dev(c, X, k, wd.p, iters, seed, frob, spec);
  });
}

int gaplra_principal_angles(gaplra_ctx* ctx, int d, int k, const double* u, int p, const double* s, double* cosines) {
  if (!ctx || !u || !s || !cosines) return GAPLRA_CONTRACT_VIOLATION;
  return guard(ctx, [&] {
    Context& c = ctx->c;
    const int64_t dp = round4(d);
    DBuf<double> ud, sd;
    ud.ensure(static_cast<size_t>(dp) * ldp_of(k));
    sd.ensure(static_cast<size_t>(dp) * ldp_of(p));
    GAPLRA_CUDA_CHECK(cudaMemsetAsync(ud.p, 0, static_cast<size_t>(dp) * ldp_of(k) * sizeof(double), c.st));
    GAPLRA_CUDA_CHECK(cudaMemsetAsync(sd.p, 0, static_cast<size_t>(dp) * ldp_of(p) * sizeof(double), c.st));
    upload_block(c, u, d, k, ud.p, ldp_of(k));
    upload_block(c, s, d, p, sd.p, ldp_of(p));
    principal_angles_dev(c, d, k, ud.p, p, sd.p, cosines);
  });
}

int gaplra_detect_multiplicative_gap(const double* est, int count, int s, int p, int* q) {
  if (!est || !q || count < 1 || p < 1) return GAPLRA_CONTRACT_VIOLATION;
  *q = detect_multiplicative_gap_host(est, count, s, p);
  return GAPLRA_OK;
}

int gaplra_detect_additive_gap(gaplra_ctx* ctx, const double* inv, int count, int s, int k, double delta, int* q) {
  if (!inv || !q) return GAPLRA_CONTRACT_VIOLATION;
  return guard(ctx, [&] { *q = detect_additive_gap_host(inv, count, s, k, delta); });
}

int gaplra_estimate_eigenvalues(gaplra_ctx* ctx, const gaplra_matrix* x, int inverse, double lambda, int k,
                                double eps_prime, uint64_t seed, double rq_tol, const gaplra_svrg_params* prm,
                                double* values, int* iterations) {
  if (!ctx || !x || !values) return GAPLRA_CONTRACT_VIOLATION;
  return guard(ctx, [&] {
    require(eps_prime > 0.0 && eps_prime < 1.0 && k >= 1 && k <= 64 && (!inverse || prm),
            "estimate_eigenvalues: bad arguments");
    Context& c = ctx->c;
    Matrix& X = const_cast<gaplra_matrix*>(x)->m;
    int64_t sc = 0;
    std::vector<double> v;
    if (inverse) {
      InverseOp op(c, X, lambda, *prm, &sc);
      v = estimate_eigs_dev(c, op, X.d, X.d_pad(), k, eps_prime, seed, rq_tol, iterations);
    } else {
      GramOp op(c, X);
      v = estimate_eigs_dev(c, op, X.d, X.d_pad(), k, eps_prime, seed, rq_tol, iterations);
    }
    std::copy(v.begin(), v.end(), values);
  });
}

int gaplra_approximate(gaplra_ctx* ctx, const gaplra_matrix* x, const gaplra_si_config* cfg, double* w, double* ritz,
                       gaplra_ap_report* rep) {
  if (!ctx || !x || !cfg || !w || !ritz || !rep) return GAPLRA_CONTRACT_VIOLATION;
  std::memset(rep, 0, sizeof(*rep));
  return guard(ctx, [&] {
    Context& c = ctx->c;
    Matrix& X = const_cast<gaplra_matrix*>(x)->m;
    const gaplra_ledger before = c.led;
    Timer total(c, &rep->ms_total);
    DBuf<double> wb;
    double* W = wb.ensure(static_cast<size_t>(X.d_pad()) * ldp_of(cfg->k));
    approximate_dev(c, X, *cfg, W, ritz, *rep);
    download_block(c, W, ldp_of(cfg->k), X.d, cfg->k, w);
    c.sync();
    gaplra_ledger& L = rep->ledger;
    L.gram_applies = c.led.gram_applies - before.gram_applies;
    L.operator_applies = c.led.operator_applies - before.operator_applies;
    L.qr_factorizations = c.led.qr_factorizations - before.qr_factorizations;
    L.linear_solves = c.led.linear_solves - before.linear_solves;
    L.solver_column_samples = c.led.solver_column_samples - before.solver_column_samples;
    L.epochs = c.led.epochs - before.epochs;
    L.outer_iterations = c.led.outer_iterations - before.outer_iterations;
  });
}

int gaplra_find_gap_budget(gaplra_ctx* ctx, const gaplra_matrix* x, int k, int p, uint64_t seed, double rq_tol,
                           double* delta) {
  if (!ctx || !x || !delta) return GAPLRA_CONTRACT_VIOLATION;
  return guard(ctx, [&] { *delta = find_gap_budget_dev(ctx->c, const_cast<gaplra_matrix*>(x)->m, k, p, seed, rq_tol); });
}

int gaplra_accsvrg_solve(gaplra_ctx* ctx, const gaplra_matrix* x, double lambda, int p, const double* b, double* w,
                         const gaplra_svrg_params* prm, int64_t solve_id, int* epochs, double* history, int hist_cap,
                         int* hist_len) {
  if (!ctx || !x || !prm) return GAPLRA_CONTRACT_VIOLATION;
  return guard(ctx, [&] {
    require(p >= 1 && p <= 64 && b && w && prm->tol > 0.0, "solve_accelerated_svrg: bad arguments");
    require(all_finite(b, static_cast<size_t>(x->m.d) * p), "solve_accelerated_svrg: non-finite right-hand side");
    Context& c = ctx->c;
    Matrix& X = const_cast<gaplra_matrix*>(x)->m;
    const int64_t ld = ldp_of(p), dp = X.d_pad();
    DBuf<double> bd, wd;
    bd.ensure(static_cast<size_t>(dp) * ld);
    wd.ensure(static_cast<size_t>(dp) * ld);
    GAPLRA_CUDA_CHECK(cudaMemsetAsync(bd.p, 0, static_cast<size_t>(dp) * ld * sizeof(double), c.st));
    upload_block(c, b, X.d, p, bd.p, ld);
    const SvrgResult r = accsvrg_solve_dev(c, X, lambda, p, bd.p, wd.p, *prm, solve_id, false);
    download_block(c, wd.p, ld, X.d, p, w);
    c.sync();
    if (epochs) *epochs = r.epochs;
    if (hist_len) *hist_len = static_cast<int>(r.history.size());
    if (history)
      for (int i = 0; i < std::min<int>(hist_cap, static_cast<int>(r.history.size())); ++i) history[i] = r.history[i];
  });
}

}  // extern "C"
