// TEST INFRASTRUCTURE ONLY — CPU oracle for the shift-and-invert hot path.
// See oracle.h for the contract and the reference file:line each piece follows.
// Build: oracle/Makefile (g++ -O2, -ffp-contract=off, no -march: the reference
// objects contain no FMA, SURVEY.md §8(c) "FP semantics").

#include "oracle.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <numeric>
#include <stdexcept>
#include <thread>
#include <vector>

namespace {

// ---------------------------------------------------------------------------
// Rng — xoshiro256++ seeded by splitmix64 (rng.cpp:9-76).
// ---------------------------------------------------------------------------
inline uint64_t sm64(uint64_t& x) {
  x += 0x9E3779B97F4A7C15ull;
  uint64_t z = x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
inline uint64_t rotl64(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }

struct Rng {
  uint64_t s[4];
  double spare = 0.0;
  bool has_spare = false;
  explicit Rng(uint64_t seed) {
    uint64_t t = seed;
    for (auto& w : s) w = sm64(t);
  }
  uint64_t next() {
    const uint64_t out = rotl64(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    return out;
  }
  double uniform01() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double normal() {  // Box-Muller with one cached spare (rng.cpp:44-59)
    if (has_spare) {
      has_spare = false;
      return spare;
    }
    double u1;
    do {
      u1 = uniform01();
    } while (u1 <= 0.0);
    const double u2 = uniform01();
    const double radius = std::sqrt(-2.0 * std::log(u1));
    const double angle = 2.0 * M_PI * u2;
    spare = radius * std::sin(angle);
    has_spare = true;
    return radius * std::cos(angle);
  }
  uint64_t uniform_index(uint64_t n) {  // rejection sampling (rng.cpp:61-69)
    const uint64_t limit = n * (~uint64_t{0} / n);
    uint64_t draw;
    do {
      draw = next();
    } while (draw >= limit);
    return draw % n;
  }
};

uint64_t derive_seed(uint64_t root, uint64_t tag) {  // rng.cpp:71-76
  uint64_t x = root ^ (0xA0761D6478BD642Full * (tag + 1));
  const uint64_t a = sm64(x);
  const uint64_t b = sm64(x);
  return a ^ rotl64(b, 32);
}

// Seed tags pinned by this restatement.  "gauss" is the
// reference's own tag (orthonormalize.cpp:17).
constexpr uint64_t kTagGauss = 0x6761757373ull;
constexpr uint64_t kTagSvrg = 0x73767267ull;      // "svrg"
constexpr uint64_t kTagEstA = 0x65737461ull;      // "esta"
constexpr uint64_t kTagEstD = 0x65737464ull;      // "estd" (+ tuning step)
constexpr uint64_t kTagSubspace = 0x73756273ull;  // "subs"

uint64_t svrg_stream_seed(uint64_t root, int64_t solve_id, int epoch) {
  return derive_seed(root, kTagSvrg ^ (static_cast<uint64_t>(solve_id) << 20) ^
                               static_cast<uint64_t>(epoch));
}

struct Status : std::runtime_error {
  int code;
  int payload;
  Status(int c, int pl = 0) : std::runtime_error("status"), code(c), payload(pl) {}
};

// ---------------------------------------------------------------------------
// Thread helper: run f(c) for c in [0, count) over nthreads threads.
// Work items are independent (block columns), so results are identical for
// any thread count.
// ---------------------------------------------------------------------------
void parallel_for(int count, int nthreads, const std::function<void(int)>& f) {
  if (nthreads <= 1 || count <= 1) {
    for (int c = 0; c < count; ++c) f(c);
    return;
  }
  nthreads = std::min(nthreads, count);
  std::vector<std::thread> ts;
  for (int t = 0; t < nthreads; ++t)
    ts.emplace_back([&, t] {
      for (int c = t; c < count; c += nthreads) f(c);
    });
  for (auto& th : ts) th.join();
}

// ---------------------------------------------------------------------------
// Column-major d x p block (column c contiguous).
// ---------------------------------------------------------------------------
struct Block {
  int d = 0, p = 0;
  std::vector<double> a;
  Block() = default;
  Block(int d_, int p_) : d(d_), p(p_), a(static_cast<size_t>(d_) * p_, 0.0) {}
  double* col(int c) { return a.data() + static_cast<size_t>(c) * d; }
  const double* col(int c) const { return a.data() + static_cast<size_t>(c) * d; }
  double& at(int i, int c) { return a[static_cast<size_t>(c) * d + i]; }
  double at(int i, int c) const { return a[static_cast<size_t>(c) * d + i]; }
  static Block from_rowmajor(int d, int p, const double* r) {
    Block b(d, p);
    for (int i = 0; i < d; ++i)
      for (int c = 0; c < p; ++c) b.at(i, c) = r[static_cast<size_t>(i) * p + c];
    return b;
  }
  void to_rowmajor(double* r) const {
    for (int i = 0; i < d; ++i)
      for (int c = 0; c < p; ++c) r[static_cast<size_t>(i) * p + c] = at(i, c);
  }
};

// ---------------------------------------------------------------------------
// X access mirroring SparseColumnsMatrix (sparse_matrix.cpp).  Dense X is
// treated as dense-as-sparse: entries with |x| > 0, rows ascending
// (from_dense, sparse_matrix.cpp:39-49).
// ---------------------------------------------------------------------------
struct Mat {
  const orc_mat* m;
  explicit Mat(const orc_mat* mm) : m(mm) {}
  int d() const { return m->d; }
  int n() const { return m->n; }
  template <class F>
  void for_col(int j, F&& f) const {
    if (m->kind == 0) {
      const double* x = m->x + static_cast<size_t>(j) * m->d;
      for (int i = 0; i < m->d; ++i) {
        const double v = x[i];
        if (std::fabs(v) > 0.0) f(i, v);
      }
    } else {
      for (int64_t e = m->colptr[j]; e < m->colptr[j + 1]; ++e) f(m->rowidx[e], m->val[e]);
    }
  }
  double column_dot(int j, const double* v) const {  // sparse_matrix.cpp:101-105
    double acc = 0.0;
    for_col(j, [&](int i, double x) { acc += x * v[i]; });
    return acc;
  }
  void column_axpy(int j, double alpha, double* y) const {  // :107-109
    for_col(j, [&](int i, double x) { y[i] += alpha * x; });
  }
  double column_norm_squared(int j) const {  // :111-115
    double acc = 0.0;
    for_col(j, [&](int, double x) { acc += x * x; });
    return acc;
  }
  void spmv_transpose(const double* v, double* out) const {  // :80-91
    for (int j = 0; j < n(); ++j) out[j] = column_dot(j, v);
  }
  void spmv(const double* v, double* out) const {  // :66-78
    std::fill(out, out + d(), 0.0);
    for (int j = 0; j < n(); ++j) {
      const double a = v[j];
      if (a == 0.0) continue;
      for_col(j, [&](int i, double x) { out[i] += a * x; });
    }
  }
};

bool all_finite(const double* v, size_t len) {
  for (size_t i = 0; i < len; ++i)
    if (!std::isfinite(v[i])) return false;
  return true;
}

// Y (n x p, column-major) = X^T W ; Z = X Y.  One gram_apply per column.
void gram_block(const Mat& x, const Block& w, Block& z, std::vector<double>* y, int nthreads) {
  const int n = x.n(), p = w.p;
  z = Block(x.d(), p);
  std::vector<double> ylocal;
  std::vector<double>& yy = y ? *y : ylocal;
  yy.assign(static_cast<size_t>(n) * p, 0.0);
  parallel_for(p, nthreads, [&](int c) {
    double* yc = yy.data() + static_cast<size_t>(c) * n;
    x.spmv_transpose(w.col(c), yc);
    x.spmv(yc, z.col(c));
  });
}

// ---------------------------------------------------------------------------
// qr_orthonormalize: two-pass MGS (orthonormalize.cpp:25-79), column-major.
// ---------------------------------------------------------------------------
constexpr double kRankTol = 1e-13;

void qr_inplace(Block& q) {
  const int d = q.d, p = q.p;
  if (d < p || p == 0) throw Status(ORC_CONTRACT_VIOLATION);
  if (!all_finite(q.a.data(), q.a.size())) throw Status(ORC_CONTRACT_VIOLATION);
  double scale = 0.0;
  for (int j = 0; j < p; ++j) {
    double nrm = 0.0;
    const double* cj = q.col(j);
    for (int i = 0; i < d; ++i) nrm += cj[i] * cj[i];
    scale = std::max(scale, std::sqrt(nrm));
  }
  if (scale == 0.0) throw Status(ORC_RANK_DEFICIENT, 0);
  std::vector<double> col(d);
  for (int j = 0; j < p; ++j) {
    std::memcpy(col.data(), q.col(j), sizeof(double) * d);
    for (int pass = 0; pass < 2; ++pass) {
      for (int prev = 0; prev < j; ++prev) {
        const double* qp = q.col(prev);
        double proj = 0.0;
        for (int i = 0; i < d; ++i) proj += qp[i] * col[i];
        for (int i = 0; i < d; ++i) col[i] -= proj * qp[i];
      }
    }
    double nrm = 0.0;
    for (int i = 0; i < d; ++i) nrm += col[i] * col[i];
    nrm = std::sqrt(nrm);
    if (!(nrm > kRankTol * scale)) throw Status(ORC_RANK_DEFICIENT, j);
    const double inv = 1.0 / nrm;
    double* qj = q.col(j);
    for (int i = 0; i < d; ++i) qj[i] = col[i] * inv;
  }
}

Block gaussian_init(int d, int p, uint64_t seed) {  // orthonormalize.cpp:12-21
  if (p < 1 || p > d) throw Status(ORC_CONTRACT_VIOLATION);
  Rng rng(derive_seed(seed, kTagGauss));
  Block b(d, p);
  for (int i = 0; i < d; ++i)
    for (int c = 0; c < p; ++c) b.at(i, c) = rng.normal();  // row-major fill order
  return b;
}

// ---------------------------------------------------------------------------
// jacobi_eigh (jacobi.cpp:13-109), on a row-major n x n buffer.
// ---------------------------------------------------------------------------
void jacobi(int n, const double* in, double* vals, double* vecs) {
  std::vector<double> a(in, in + static_cast<size_t>(n) * n), v(static_cast<size_t>(n) * n, 0.0);
  auto A = [&](int i, int j) -> double& { return a[static_cast<size_t>(i) * n + j]; };
  auto V = [&](int i, int j) -> double& { return v[static_cast<size_t>(i) * n + j]; };
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) {
      const double m = 0.5 * (A(i, j) + A(j, i));
      A(i, j) = m;
      A(j, i) = m;
    }
  for (int i = 0; i < n; ++i) V(i, i) = 1.0;
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0, diag = 0.0;
    for (int i = 0; i < n; ++i) {
      diag += A(i, i) * A(i, i);
      for (int j = i + 1; j < n; ++j) off += 2.0 * A(i, j) * A(i, j);
    }
    if (off <= 1e-14 * 1e-14 * std::max(diag, 1e-300)) break;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = A(p, q);
        if (apq == 0.0) continue;
        const double app = A(p, p), aqq = A(q, q);
        const double tau = (aqq - app) / (2.0 * apq);
        const double t = (tau >= 0.0) ? 1.0 / (tau + std::sqrt(1.0 + tau * tau))
                                      : 1.0 / (tau - std::sqrt(1.0 + tau * tau));
        const double c = 1.0 / std::sqrt(1.0 + t * t);
        const double s = t * c;
        for (int i = 0; i < n; ++i) {
          const double aip = A(i, p), aiq = A(i, q);
          A(i, p) = c * aip - s * aiq;
          A(i, q) = s * aip + c * aiq;
        }
        for (int i = 0; i < n; ++i) {
          const double api = A(p, i), aqi = A(q, i);
          A(p, i) = c * api - s * aqi;
          A(q, i) = s * api + c * aqi;
        }
        for (int i = 0; i < n; ++i) {
          const double vip = V(i, p), viq = V(i, q);
          V(i, p) = c * vip - s * viq;
          V(i, q) = s * vip + c * viq;
        }
      }
  }
  std::vector<int> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int i, int j) { return A(i, i) > A(j, j); });
  for (int j = 0; j < n; ++j) {
    vals[j] = A(order[j], order[j]);
    for (int i = 0; i < n; ++i) vecs[static_cast<size_t>(i) * n + j] = V(i, order[j]);
  }
  for (int j = 0; j < n; ++j) {  // sign convention (jacobi.cpp:16-31)
    int arg = 0;
    double best = 0.0;
    for (int i = 0; i < n; ++i) {
      const double av = std::fabs(vecs[static_cast<size_t>(i) * n + j]);
      if (av > best) {
        best = av;
        arg = i;
      }
    }
    if (vecs[static_cast<size_t>(arg) * n + j] < 0.0)
      for (int i = 0; i < n; ++i) vecs[static_cast<size_t>(i) * n + j] = -vecs[static_cast<size_t>(i) * n + j];
  }
}

// ---------------------------------------------------------------------------
// SVRG — block form sharing one index stream.
// ---------------------------------------------------------------------------
struct SvrgSetup {
  double eta, rho, eta_n, lambda;
  int64_t m;
  int cap;
};

SvrgSetup svrg_setup(const Mat& x, double lambda, const orc_svrg_params* prm) {
  SvrgSetup s;
  s.lambda = lambda;
  double maxn2 = 0.0;
  if (prm->eta > 0.0) {
    s.eta = prm->eta;
  } else {
    double fro2 = 0.0;  // frobenius_norm_squared (sparse_matrix.cpp:117-121)
    for (int j = 0; j < x.n(); ++j) {
      const double c = x.column_norm_squared(j);
      maxn2 = std::max(maxn2, c);
      fro2 += c;
    }
    const double L = static_cast<double>(x.n()) * maxn2;
    s.eta = 1.0 / (4.0 * (lambda + L));
    // Stability cap: within an epoch the error's second moment
    // contracts only if eta < 2 (lambda - lambda_1) / (|X|_F^2 lambda_1); use
    // half of it with the caller's lambda_1 upper estimate (the
    // ShiftedSystem hint "used for step sizing").
    if (prm->lambda1_hint > 0.0) {
      if (!(lambda > prm->lambda1_hint)) throw Status(ORC_INDEFINITE_SHIFT);
      if (fro2 > 0.0) s.eta = std::min(s.eta, (lambda - prm->lambda1_hint) / (fro2 * prm->lambda1_hint));
    }
  }
  s.rho = 1.0 - s.eta * lambda;
  s.eta_n = s.eta * static_cast<double>(x.n());
  s.m = prm->m > 0 ? prm->m : 2 * static_cast<int64_t>(x.n());
  s.cap = prm->epoch_cap > 0 ? prm->epoch_cap
                             : static_cast<int>(std::ceil(200.0 * std::log(1.0 / prm->tol)));
  return s;
}

void index_stream(uint64_t seed, int n, int64_t m, std::vector<int32_t>& idx) {
  idx.resize(m);
  Rng rng(seed);
  for (int64_t s = 0; s < m; ++s) idx[s] = static_cast<int32_t>(rng.uniform_index(static_cast<uint64_t>(n)));
}

// W (column-major d x p) in/out; Y column-major n x p; C column-major d x p.
// Dense X: direct form  w = rho*w + C; w += r x_i.
// Sparse X: lazy form   W = a*What + b*C  (identical in exact arithmetic; the
// O(d) rho*W + C sweep per step would make C4 epochs O(d m p)).
void svrg_epoch(const Mat& x, Block& w, const std::vector<double>& y, const Block& cblk,
                const SvrgSetup& st, const std::vector<int32_t>& idx, int nthreads) {
  const int d = x.d(), n = x.n(), p = w.p;
  const int64_t m = static_cast<int64_t>(idx.size());
  if (x.m->kind == 0) {
    parallel_for(p, nthreads, [&](int c) {
      double* wc = w.col(c);
      const double* cc = cblk.col(c);
      const double* yc = y.data() + static_cast<size_t>(c) * n;
      for (int64_t s = 0; s < m; ++s) {
        const int i = idx[s];
        const double t = x.column_dot(i, wc);
        const double r = st.eta_n * (t - yc[i]);
        for (int k = 0; k < d; ++k) wc[k] = st.rho * wc[k] + cc[k];
        x.column_axpy(i, r, wc);
      }
    });
  } else {
    parallel_for(p, nthreads, [&](int c) {
      double* wc = w.col(c);
      const double* cc = cblk.col(c);
      const double* yc = y.data() + static_cast<size_t>(c) * n;
      double a = 1.0, b = 0.0;
      for (int64_t s = 0; s < m; ++s) {
        const int i = idx[s];
        const double t = a * x.column_dot(i, wc) + b * x.column_dot(i, cc);
        const double r = st.eta_n * (t - yc[i]);
        a = st.rho * a;
        b = st.rho * b + 1.0;
        if (a < 1e-150) {
          for (int k = 0; k < d; ++k) wc[k] *= a;
          a = 1.0;
        }
        x.column_axpy(i, r / a, wc);
      }
      for (int k = 0; k < d; ++k) wc[k] = a * wc[k] + b * cc[k];
    });
  }
}

struct SolveResult {
  int epochs = 0;
  std::vector<double> history;
};

// Block solve (lambda I - X X^T) W = B with W0 = 0.  Epoch loop:
//   anchor (skipped at e = 0: W = 0 => Y = 0, Z = 0), M = lambda W - Z - B,
//   res = max_c |M_c| / |B_c|; stop if res <= tol; stall on non-finite,
//   non-monotone (> slack * previous) or cap; else C = eta (Z + B) and run m
//   steps on the stream derive_seed(root, TAG_SVRG ^ (solve_id << 20) ^ e).
SolveResult svrg_solve(const Mat& x, double lambda, const Block& b, Block& w,
                       const orc_svrg_params* prm, int64_t solve_id, orc_ledger* led,
                       int nthreads, const Block* guess = nullptr) {
  const int d = x.d(), n = x.n(), p = b.p;
  const SvrgSetup st = svrg_setup(x, lambda, prm);
  const bool warm = guess != nullptr;
  w = warm ? *guess : Block(d, p);
  std::vector<double> bnorm(p);
  for (int c = 0; c < p; ++c) {
    double acc = 0.0;
    for (int i = 0; i < d; ++i) acc += b.at(i, c) * b.at(i, c);
    bnorm[c] = std::sqrt(acc);
  }
  SolveResult res;
  std::vector<double> y(static_cast<size_t>(n) * p, 0.0);
  Block z(d, p), cblk(d, p);
  std::vector<int32_t> idx;
  double best = INFINITY;
  for (int e = 0;; ++e) {
    if (e > 0 || warm) {
      gram_block(x, w, z, &y, nthreads);
      if (led) led->gram_applies += p;
    }
    double r = 0.0;
    for (int c = 0; c < p; ++c) {
      double acc = 0.0;
      for (int i = 0; i < d; ++i) {
        const double mm = (lambda * w.at(i, c) - z.at(i, c)) - b.at(i, c);
        acc += mm * mm;
      }
      const double rc = std::sqrt(acc) / (bnorm[c] > 0.0 ? bnorm[c] : 1.0);
      r = std::max(r, rc);
      if (!std::isfinite(rc)) r = rc;
    }
    res.history.push_back(r);
    if (!std::isfinite(r)) throw Status(ORC_SOLVER_STALLED);
    if (r <= prm->tol) break;
    // Divergence guard (SPEC.md:359 asks for monotone epochs within 5%; the
    // full-gradient residual of plain SVRG fluctuates by up to ~20% per epoch
    // at small gaps, so the pinned rule is: stall when the residual exceeds
    // slack x the best residual seen so far — DESIGN.md §2.2).
    if (prm->monotone_slack > 0.0 && e >= 1 && r > prm->monotone_slack * best)
      throw Status(ORC_SOLVER_STALLED);
    best = std::min(best, r);
    if (e >= st.cap) throw Status(ORC_SOLVER_STALLED);
    for (int c = 0; c < p; ++c)
      for (int i = 0; i < d; ++i) cblk.at(i, c) = st.eta * (z.at(i, c) + b.at(i, c));
    index_stream(svrg_stream_seed(prm->root_seed, solve_id, e), n, st.m, idx);
    svrg_epoch(x, w, y, cblk, st, idx, nthreads);
    res.epochs++;
    if (led) {
      led->epochs++;
      led->solver_column_samples += static_cast<uint64_t>(st.m);
    }
  }
  if (led) led->linear_solves++;
  return res;
}

// solve_accelerated_svrg (design :363): a Catalyst outer
// loop around solve_svrg.  mu = lambda - h (h = prm->lambda1_hint, required),
// kappa = sqrt(h mu), q = mu / (mu + kappa), beta = (1 - sqrt q) / (1 + sqrt q).
// x = guess or 0, y = x; per outer step k: the residual of the original system
// r = b - D x (one gram pass), stop when max_c |r_c| / |b_c| <= tol; else
// x' = solve_svrg((lambda + kappa) I - X Xᵀ, b + kappa y) warm-started at x,
// inner tol max(tol / 10, res / 10), stream ids (solve_id << 10) | k; then
// y = x' + beta (x' - x), x = x'.  Outer cap ceil(200 ln(1/tol)).
SolveResult accsvrg_solve(const Mat& x, double lambda, const Block& b, Block& w, const orc_svrg_params* prm,
                          int64_t solve_id, orc_ledger* led, int nthreads, const Block* guess = nullptr) {
  const int d = x.d(), p = b.p;
  const double h = prm->lambda1_hint;
  if (!(h > 0.0) || !(lambda > h)) throw Status(ORC_CONTRACT_VIOLATION);
  const double mu = lambda - h, kappa = std::sqrt(h * mu), q = mu / (mu + kappa);
  const double beta = (1.0 - std::sqrt(q)) / (1.0 + std::sqrt(q));
  const int cap = prm->epoch_cap > 0 ? prm->epoch_cap : static_cast<int>(std::ceil(200.0 * std::log(1.0 / prm->tol)));
  std::vector<double> bnorm(p);
  for (int c = 0; c < p; ++c) {
    double acc = 0.0;
    for (int i = 0; i < d; ++i) acc += b.at(i, c) * b.at(i, c);
    bnorm[c] = std::sqrt(acc);
  }
  Block xc = guess ? *guess : Block(d, p), yc = xc, z, rhs(d, p), xn;
  SolveResult res;
  for (int k = 0;; ++k) {
    gram_block(x, xc, z, nullptr, nthreads);
    if (led) led->gram_applies += p;
    double r = 0.0;
    for (int c = 0; c < p; ++c) {
      double acc = 0.0;
      for (int i = 0; i < d; ++i) {
        const double rr = b.at(i, c) - (lambda * xc.at(i, c) - z.at(i, c));
        acc += rr * rr;
      }
      const double rc = std::sqrt(acc) / (bnorm[c] > 0.0 ? bnorm[c] : 1.0);
      r = std::isfinite(rc) ? std::max(r, rc) : rc;
    }
    res.history.push_back(r);
    if (!std::isfinite(r)) throw Status(ORC_SOLVER_STALLED);
    if (r <= prm->tol) break;
    if (k >= cap) throw Status(ORC_SOLVER_STALLED);
    for (int c = 0; c < p; ++c)
      for (int i = 0; i < d; ++i) rhs.at(i, c) = b.at(i, c) + kappa * yc.at(i, c);
    orc_svrg_params pin = *prm;
    pin.tol = std::max(0.1 * prm->tol, 0.1 * r);
    pin.epoch_cap = 0;
    const SolveResult in = svrg_solve(x, lambda + kappa, rhs, xn, &pin, (solve_id << 10) | (k & 1023), led, nthreads,
                                      &xc);
    res.epochs += in.epochs;
    for (int c = 0; c < p; ++c)
      for (int i = 0; i < d; ++i) {
        const double xv = xn.at(i, c);
        yc.at(i, c) = xv + beta * (xv - xc.at(i, c));
        xc.at(i, c) = xv;
      }
  }
  w = xc;
  return res;
}

// ---------------------------------------------------------------------------
// Operators for the subspace engine.
// ---------------------------------------------------------------------------
struct BlockOp {
  virtual ~BlockOp() = default;
  // `guess` (optional): warm start for operators that iterate
  virtual void apply(const Block& in, Block& out, const Block* guess = nullptr) = 0;
};

struct GramOp : BlockOp {
  Mat x;
  orc_ledger* led;
  int nthreads;
  GramOp(const Mat& xx, orc_ledger* l, int nt) : x(xx), led(l), nthreads(nt) {}
  void apply(const Block& in, Block& out, const Block* = nullptr) override {
    gram_block(x, in, out, nullptr, nthreads);
    if (led) {
      led->gram_applies += in.p;
      led->operator_applies += in.p;
    }
  }
};

// inverse_operator(svrg, lambda) with an empty deflation basis.
struct InverseOp : BlockOp {
  Mat x;
  double lambda;
  orc_svrg_params prm;
  int64_t* solve_counter;
  orc_ledger* led;
  int nthreads;
  InverseOp(const Mat& xx, double lam, const orc_svrg_params& pr, int64_t* sc, orc_ledger* l, int nt)
      : x(xx), lambda(lam), prm(pr), solve_counter(sc), led(l), nthreads(nt) {}
  void apply(const Block& in, Block& out, const Block* guess = nullptr) override {
    svrg_solve(x, lambda, in, out, &prm, (*solve_counter)++, led, nthreads, guess);
    if (led) led->operator_applies += in.p;
  }
};

// project_out (linear_operator.cpp:66-81): one-pass CGS, all coefficients
// first, then subtracted in basis order; per column of a block.
void project_out_block(const Block& basis, Block& v) {
  const int m = basis.p, d = basis.d;
  if (m == 0) return;
  std::vector<double> coeffs(m);
  for (int c = 0; c < v.p; ++c) {
    for (int j = 0; j < m; ++j) {
      double acc = 0.0;
      for (int i = 0; i < d; ++i) acc += basis.at(i, j) * v.at(i, c);
      coeffs[j] = acc;
    }
    for (int j = 0; j < m; ++j) {
      const double cj = coeffs[j];
      if (cj == 0.0) continue;
      for (int i = 0; i < d; ++i) v.at(i, c) -= cj * basis.at(i, j);
    }
  }
}

// solve_cg: block CG on (lambda I - X X^T) W = B, one
// independent recurrence per column, all columns stepped together.  Pinned:
// W0 = 0 (or the warm guess, R0 = B - D W0), stop before an iteration when
// max_c |r_c| / |b_c| <= tol, IndefiniteShift when p_c^T D p_c <= 0 for a
// column with r_c != 0, a column with r_c = 0 is frozen (alpha = beta = 0),
// cap = max_iter > 0 ? max_iter : d + 10 iterations -> SolverStalled.
// Dots are sequential row sums; D p = lambda p - X (X^T p) is one gram_block.
struct CgResult {
  int iterations = 0;
  std::vector<double> history;
};

// With a deflation basis U the system is lambda I - P X Xᵀ P (P = I - U Uᵀ;
// SPEC.md:114, Alg. 7's X_{-(s-1)}): for iterates in range(P) that is
// p -> lambda p - P (X Xᵀ p), i.e. one project_out after each gram pass.
CgResult cg_solve(const Mat& x, double lambda, const Block& b, Block& w, double tol, int max_iter,
                  orc_ledger* led, int nthreads, const Block* guess = nullptr, const Block* basis = nullptr) {
  const int d = x.d(), p = b.p;
  const int cap = max_iter > 0 ? max_iter : d + 10;
  auto coldot = [&](const Block& u, const Block& v, int c) {
    double acc = 0.0;
    for (int i = 0; i < d; ++i) acc += u.at(i, c) * v.at(i, c);
    return acc;
  };
  std::vector<double> bnorm(p), rr(p), pq(p), alpha(p), beta(p);
  for (int c = 0; c < p; ++c) bnorm[c] = std::sqrt(coldot(b, b, c));
  Block r = b, z, q(d, p);
  if (guess) {
    w = *guess;
    gram_block(x, w, z, nullptr, nthreads);
    if (basis) project_out_block(*basis, z);
    if (led) led->gram_applies += p;
    for (int c = 0; c < p; ++c)
      for (int i = 0; i < d; ++i) r.at(i, c) = b.at(i, c) - (lambda * w.at(i, c) - z.at(i, c));
  } else {
    w = Block(d, p);
  }
  Block pd = r;
  for (int c = 0; c < p; ++c) rr[c] = coldot(r, r, c);
  CgResult res;
  for (int it = 0;; ++it) {
    double worst = 0.0;
    for (int c = 0; c < p; ++c) worst = std::max(worst, std::sqrt(rr[c]) / (bnorm[c] > 0.0 ? bnorm[c] : 1.0));
    res.history.push_back(worst);
    if (!std::isfinite(worst)) throw Status(ORC_SOLVER_STALLED);
    if (worst <= tol) break;
    if (it >= cap) throw Status(ORC_SOLVER_STALLED);
    gram_block(x, pd, z, nullptr, nthreads);
    if (basis) project_out_block(*basis, z);
    if (led) led->gram_applies += p;
    for (int c = 0; c < p; ++c)
      for (int i = 0; i < d; ++i) q.at(i, c) = lambda * pd.at(i, c) - z.at(i, c);
    for (int c = 0; c < p; ++c) {
      pq[c] = coldot(pd, q, c);
      if (rr[c] > 0.0 && !(pq[c] > 0.0)) throw Status(ORC_INDEFINITE_SHIFT);
      alpha[c] = rr[c] > 0.0 ? rr[c] / pq[c] : 0.0;
    }
    for (int c = 0; c < p; ++c)
      for (int i = 0; i < d; ++i) {
        w.at(i, c) += alpha[c] * pd.at(i, c);
        r.at(i, c) -= alpha[c] * q.at(i, c);
      }
    for (int c = 0; c < p; ++c) {
      const double rn = coldot(r, r, c);
      beta[c] = rr[c] > 0.0 ? rn / rr[c] : 0.0;
      rr[c] = rn;
    }
    for (int c = 0; c < p; ++c)
      for (int i = 0; i < d; ++i) pd.at(i, c) = r.at(i, c) + beta[c] * pd.at(i, c);
    res.iterations++;
  }
  if (led) led->linear_solves++;
  return res;
}

// inverse_operator(accsvrg, lambda) (backend = accsvrg)
struct AccOp : BlockOp {
  Mat x;
  double lambda;
  orc_svrg_params prm;
  int64_t* solve_counter;
  orc_ledger* led;
  int nthreads;
  AccOp(const Mat& xx, double lam, const orc_svrg_params& pr, int64_t* sc, orc_ledger* l, int nt)
      : x(xx), lambda(lam), prm(pr), solve_counter(sc), led(l), nthreads(nt) {}
  void apply(const Block& in, Block& out, const Block* guess = nullptr) override {
    accsvrg_solve(x, lambda, in, out, &prm, (*solve_counter)++, led, nthreads, guess);
    if (led) led->operator_applies += in.p;
  }
};

// inverse_operator(cg, lambda) (backend = cg)
struct CgOp : BlockOp {
  Mat x;
  double lambda, tol;
  int max_iter;
  orc_ledger* led;
  int nthreads;
  const Block* basis;  // deflated system (nullptr: none)
  CgOp(const Mat& xx, double lam, double t, int mi, orc_ledger* l, int nt, const Block* u = nullptr)
      : x(xx), lambda(lam), tol(t), max_iter(mi), led(l), nthreads(nt), basis(u && u->p > 0 ? u : nullptr) {}
  void apply(const Block& in, Block& out, const Block* guess = nullptr) override {
    cg_solve(x, lambda, in, out, tol, max_iter, led, nthreads, guess, basis);
    if (led) led->operator_applies += in.p;
  }
};

// G = Aᵀ B (p x q, row-major), sequential row sums
std::vector<double> gram_ab(const Block& a, const Block& b) {
  std::vector<double> g(static_cast<size_t>(a.p) * b.p, 0.0);
  for (int i = 0; i < a.p; ++i)
    for (int j = 0; j < b.p; ++j) {
      double acc = 0.0;
      for (int r = 0; r < a.d; ++r) acc += a.at(r, i) * b.at(r, j);
      g[static_cast<size_t>(i) * b.p + j] = acc;
    }
  return g;
}

// Warm start for the next solve D⁻¹ S_new: in the converged
// limit D⁻¹ S_new = S_new (S_newᵀ Y)(S_oldᵀ S_new), with Y = D⁻¹ S_old.
Block warm_guess(const Block& s_new, const Block& y, const std::vector<double>& g_old_new) {
  const int p = s_new.p;
  const std::vector<double> r = gram_ab(s_new, y);
  std::vector<double> rg(static_cast<size_t>(p) * p, 0.0);
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < p; ++j) {
      double acc = 0.0;
      for (int k = 0; k < p; ++k) acc += r[static_cast<size_t>(i) * p + k] * g_old_new[static_cast<size_t>(k) * p + j];
      rg[static_cast<size_t>(i) * p + j] = acc;
    }
  Block w(s_new.d, p);
  for (int r0 = 0; r0 < s_new.d; ++r0)
    for (int j = 0; j < p; ++j) {
      double acc = 0.0;
      for (int k = 0; k < p; ++k) acc += s_new.at(r0, k) * rg[static_cast<size_t>(k) * p + j];
      w.at(r0, j) = acc;
    }
  return w;
}

// ||S S^T - S' S'^T||_F = sqrt(2) |S' - S (S^T S')|_F (stable form).
double projector_diff(const Block& s, const Block& s2, std::vector<double>* g_out = nullptr) {
  const int d = s.d, p = s.p;
  std::vector<double> g = gram_ab(s, s2);
  if (g_out) *g_out = g;
  double tot = 0.0;
  for (int b = 0; b < p; ++b)
    for (int i = 0; i < d; ++i) {
      double r = s2.at(i, b);
      for (int a = 0; a < p; ++a) r -= s.at(i, a) * g[static_cast<size_t>(a) * p + b];
      tot += r * r;
    }
  return std::sqrt(2.0 * tot);
}

Block orth_init(int d, int p, uint64_t seed) {
  // S0 = QR(gaussian_init(d, p, seed)); on RankDeficient redraw once with
  // seed + 1.
  try {
    Block s = gaussian_init(d, p, seed);
    qr_inplace(s);
    return s;
  } catch (const Status& st) {
    if (st.code != ORC_RANK_DEFICIENT) throw;
    Block s = gaussian_init(d, p, seed + 1);
    qr_inplace(s);
    return s;
  }
}

// Rank completion of an iterate: when the operator's range
// has dimension < p (X of exact rank < p, SPEC.md:541's "perfect recovery
// regime"), C·S is rank deficient and MGS2 stops at the first dependent column
// j; that column is replaced by a fresh Gaussian direction
// gaussian_init(d, 1, derive_seed(seed, j + 64·attempt)) and the QR redone (the same
// draws every iteration, so a completed iterate is a fixed point and the
// projector early stop still fires) —
// columns before j are unchanged, the new one lies outside range(C), S stays
// orthonormal.  Only S⁰ keeps the SPEC's redraw-once rule.
constexpr uint64_t kTagComplete = 0x636f6d70ull;  // "comp"
void qr_complete(Block& q, uint64_t seed) {
  Block orig = q;
  for (int attempt = 0;; ++attempt) {
    try {
      qr_inplace(q);
      return;
    } catch (const Status& st) {
      if (st.code != ORC_RANK_DEFICIENT || attempt >= q.p) throw;
      const Block g = gaussian_init(q.d, 1, derive_seed(seed, static_cast<uint64_t>(st.payload + 64 * attempt)));
      for (int i = 0; i < q.d; ++i) orig.at(i, st.payload) = g.at(i, 0);
      q = orig;
    }
  }
}

// Alg. 1 with projector-difference early stop.
Block subspace_iterate(BlockOp& op, int d, int p, int L, uint64_t seed, double conv_tol,
                       int* iters, orc_ledger* led) {
  Block s = orth_init(d, p, seed);
  Block y, guess;
  bool have_guess = false;
  int it = 0;
  std::vector<double> g;
  for (int l = 1; l <= L; ++l) {
    op.apply(s, y, have_guess ? &guess : nullptr);
    Block q = y;
    qr_complete(q, derive_seed(seed, kTagComplete));
    if (led) led->qr_factorizations++;
    it = l;
    const double diff = projector_diff(s, q, &g);
    const bool stop = conv_tol > 0.0 && diff <= conv_tol;
    guess = warm_guess(q, y, g);
    have_guess = true;
    s = q;
    if (stop) break;
  }
  if (iters) *iters = it;
  if (led) led->outer_iterations += it;
  return s;
}

// Alg. 3 for k = 1: L = ceil(4/eps' ln(d/eps')); the
// estimate is the Rayleigh quotient s^T C s of the current iterate, with an
// early stop when it changes by <= rq_tol relative.
double estimate_top(BlockOp& op, int d, double eps_prime, uint64_t seed, double rq_tol, int* iters,
                    orc_ledger* led) {
  const int L = static_cast<int>(std::ceil(4.0 / eps_prime * std::log(d / eps_prime)));
  Block s = orth_init(d, 1, seed);
  Block y, guess;
  bool have_guess = false;
  double prev = 0.0, theta = 0.0;
  int it = 0;
  for (int l = 1; l <= L + 1; ++l) {
    op.apply(s, y, have_guess ? &guess : nullptr);
    it = l;
    double acc = 0.0;
    for (int i = 0; i < d; ++i) acc += s.at(i, 0) * y.at(i, 0);
    theta = acc;
    if (l > 1 && std::fabs(theta - prev) <= rq_tol * std::fabs(theta)) break;
    if (l == L + 1) break;
    Block q = y;
    qr_inplace(q);
    if (led) led->qr_factorizations++;
    guess = warm_guess(q, y, gram_ab(s, q));
    have_guess = true;
    s = q;
    prev = theta;
  }
  if (iters) *iters = it;
  return theta;
}

// DeflatedOperator::apply (linear_operator.cpp:56-64) on a block: P C P with
// P = I - basis basisᵀ; for an inverse operator this is inverse_operator's
// "apply(v) = P solve(lambda, P v)".
struct DeflatedOp : BlockOp {
  BlockOp& base;
  const Block& basis;
  DeflatedOp(BlockOp& b, const Block& u) : base(b), basis(u) {}
  void apply(const Block& in, Block& out, const Block* guess = nullptr) override {
    Block work = in;
    project_out_block(basis, work);
    base.apply(work, out, guess);
    project_out_block(basis, out);
  }
};

// Alg. 3 for any k: subspace iteration on k columns, the
// estimates are the Ritz values (eigenvalues of Sᵀ C S = z_iᵀ C z_i for the
// Ritz vectors z_i, descending), early stop when every one changes by
// <= rq_tol relative.  For k = 1 this is estimate_top.
std::vector<double> estimate_eigs(BlockOp& op, int d, int k, double eps_prime, uint64_t seed, double rq_tol,
                                  int* iters, orc_ledger* led) {
  const int L = static_cast<int>(std::ceil(4.0 / eps_prime * std::log(d / eps_prime)));
  Block s = orth_init(d, k, seed);
  Block y, guess;
  bool have_guess = false;
  std::vector<double> prev(k, 0.0), theta(k, 0.0), vecs(static_cast<size_t>(k) * k);
  int it = 0;
  for (int l = 1; l <= L + 1; ++l) {
    op.apply(s, y, have_guess ? &guess : nullptr);
    it = l;
    std::vector<double> h = gram_ab(s, y);
    for (int a = 0; a < k; ++a)
      for (int b = a + 1; b < k; ++b) {
        const double m = 0.5 * (h[static_cast<size_t>(a) * k + b] + h[static_cast<size_t>(b) * k + a]);
        h[static_cast<size_t>(a) * k + b] = h[static_cast<size_t>(b) * k + a] = m;
      }
    jacobi(k, h.data(), theta.data(), vecs.data());
    bool stop = l > 1;
    for (int a = 0; a < k && stop; ++a) stop = std::fabs(theta[a] - prev[a]) <= rq_tol * std::fabs(theta[a]);
    if (stop || l == L + 1) break;
    Block q = y;
    qr_complete(q, derive_seed(seed, kTagComplete));
    if (led) led->qr_factorizations++;
    guess = warm_guess(q, y, gram_ab(s, q));
    have_guess = true;
    s = q;
    prev = theta;
  }
  if (iters) *iters = it;
  return theta;
}

// Alg. 4: smallest global q in {s..s+count-2} with
// est[q+1] <= est[q] (1 - p^-2); -1 when none (est[i] = lambda_hat_{s+i}).
int detect_multiplicative_gap(const double* est, int count, int s, int p) {
  const double f = 1.0 - 1.0 / (static_cast<double>(p) * p);
  for (int i = 0; i + 1 < count; ++i)
    if (est[i + 1] <= est[i] * f) return s + i;
  return -1;
}

// Alg. 5: requires inv[0] = lambda~_s^-1 in [delta/27,
// delta/5] (Eq. 5) else ShiftOutOfRange; q = min{i : inv_{i+1} - inv_i >=
// 5 delta / 9} over the consecutive estimates, else k.
int detect_additive_gap(const double* inv, int count, int s, int k, double delta) {
  if (count < 1 || !(inv[0] >= delta / 27.0 && inv[0] <= delta / 5.0)) throw Status(ORC_SHIFT_OUT_OF_RANGE);
  for (int i = 0; i + 1 < count; ++i)
    if (inv[i + 1] - inv[i] >= 5.0 * delta / 9.0) return s + i;
  return k;
}

orc_svrg_params make_prm(const orc_si_config* cfg, double tol) {
  orc_svrg_params prm;
  prm.eta = 0.0;
  prm.m = 0;
  prm.tol = tol;
  prm.epoch_cap = cfg->epoch_cap;
  prm.monotone_slack = cfg->monotone_slack;
  prm.root_seed = cfg->seed;
  prm.lambda1_hint = 0.0;
  return prm;
}

// tune_shift — Alg. 6 with the window
// [Delta/27, Delta/5] and estimate -> test -> update order.
void tune_shift(const Mat& x, double delta, const orc_si_config* cfg, int64_t* solve_counter,
                orc_si_report* rep, int nthreads, const Block* basis = nullptr) {
  const int d = x.d();
  const Block none(d, 0);
  const Block& u = basis ? *basis : none;
  GramOp a0(x, &rep->ledger, nthreads);
  DeflatedOp a(a0, u);  // A_{-(s-1)} (Alg. 6 on the deflated matrix)
  const double l1 = estimate_top(a, d, 0.25, derive_seed(cfg->seed, kTagEstA), cfg->rq_tol,
                                 nullptr, &rep->ledger);
  rep->lambda1_hat = l1;
  rep->tune_steps = 0;
  if (l1 < 3.0 * delta && !cfg->force) throw Status(ORC_NO_PRECONDITIONING_NEEDED);
  double lambda = 1.5 * l1;
  const double ratio = l1 / delta;
  const int cap = (ratio > 1.0 ? static_cast<int>(std::ceil(4.0 * std::log2(ratio))) : 0) + 5;
  orc_svrg_params prm = make_prm(cfg, cfg->tol_tune);
  // lambda_1 upper estimates: Alg. 3 at eps' = 1/4 gives lambda1_hat >= (3/4) lambda_1;
  // after an update lambda_t = lambda_{t-1} - (4/9) inv_{t-1} with inv <= (9/8)(lambda_{t-1} -
  // lambda_1), lambda_1 <= 2 lambda_t - lambda_{t-1}.
  double hint = l1 / 0.75, prev_lambda = lambda;
  for (int t = 0; t < cap; ++t) {
    if (t > 0) hint = 2.0 * lambda - prev_lambda;
    prm.lambda1_hint = hint;
    InverseOp dinv(x, lambda, prm, solve_counter, &rep->ledger, nthreads);
    CgOp dcg(x, lambda, cfg->tol_tune, 0, &rep->ledger, nthreads, &u);
    // a deflated shifted system is solved by CG (the SVRG epoch samples the
    // undeflated columns of X)
    const bool cg = cfg->backend == 1 || u.p > 0;
    DeflatedOp op(cg ? static_cast<BlockOp&>(dcg) : static_cast<BlockOp&>(dinv), u);
    const double est = estimate_top(op, d, 1.0 / 9.0, derive_seed(cfg->seed, kTagEstD + t),
                                    cfg->rq_tol, nullptr, &rep->ledger);
    const double inv = 1.0 / std::max(est, 1e-300);
    if (rep->tune_steps < 64) {
      rep->tune_lambda[rep->tune_steps] = lambda;
      rep->tune_inv[rep->tune_steps] = inv;
    }
    rep->tune_steps++;
    if (inv >= delta / 27.0 && inv <= delta / 5.0) {
      rep->lambda = lambda;
      rep->lambda1_hint = lambda - (8.0 / 9.0) * inv;
      return;
    }
    prev_lambda = lambda;
    lambda = lambda - (4.0 / 9.0) * inv;
  }
  rep->lambda = lambda;
  throw Status(ORC_SHIFT_TUNING_STALLED);
}

// restricted_projection — Alg. 2: H = S^T (X X^T S) with
// DenseMatrix::gram_with's loop order (dense_matrix.cpp:80-93), jacobi_eigh,
// W = S U_k with DenseMatrix::multiply's order (dense_matrix.cpp:65-78).
void restricted_projection(const Mat& x, const Block& s, int k, Block& w, std::vector<double>& ritz,
                           orc_ledger* led, int nthreads) {
  const int d = s.d, p = s.p;
  Block z;
  gram_block(x, s, z, nullptr, nthreads);
  if (led) led->gram_applies += p;
  std::vector<double> h(static_cast<size_t>(p) * p, 0.0);
  for (int kk = 0; kk < d; ++kk)
    for (int i = 0; i < p; ++i) {
      const double a = s.at(kk, i);
      if (a == 0.0) continue;
      for (int j = 0; j < p; ++j) h[static_cast<size_t>(i) * p + j] += a * z.at(kk, j);
    }
  std::vector<double> vals(p), vecs(static_cast<size_t>(p) * p);
  jacobi(p, h.data(), vals.data(), vecs.data());
  w = Block(d, k);
  for (int i = 0; i < d; ++i)
    for (int kk = 0; kk < p; ++kk) {
      const double a = s.at(i, kk);
      if (a == 0.0) continue;
      for (int j = 0; j < k; ++j) w.at(i, j) += a * vecs[static_cast<size_t>(kk) * p + j];
    }
  ritz.assign(vals.begin(), vals.begin() + k);
}

// deflation_basis_extend: project the new block against the
// current basis (project_out), QR it, append; RankDeficient against a non-empty
// basis -> DegenerateProgress.
Block basis_extend(const Block& cur, const Block& nb) {
  Block q = nb;
  project_out_block(cur, q);
  try {
    qr_inplace(q);
  } catch (const Status& e) {
    if (e.code != ORC_RANK_DEFICIENT || cur.p == 0) throw;
    throw Status(ORC_DEGENERATE_PROGRESS, e.payload);
  }
  Block out(cur.d, cur.p + q.p);
  std::copy(cur.a.begin(), cur.a.end(), out.a.begin());
  std::copy(q.a.begin(), q.a.end(), out.a.begin() + cur.a.size());
  return out;
}

// approximate — Alg. 7 with every SPEC
// design decision: eps_int = eps / (3 mu k d); per interval {s..k} on the
// deflated A_{-(s-1)}: Alg. 3 at eps' = 1/(9p^2) -> Alg. 4; a multiplicative
// gap q gives PlainPower on {s..q} (width q-s+1, L = ceil(4 p^4 ln(kd/eps_int)));
// otherwise Alg. 6 tune_shift, Alg. 3 on D_{-(s-1)} at eps' = 1/(9p) -> Alg. 5
// -> ShiftedInverse on {s..q} with width q-s+1 (q < k) or p-s+1 (q = k) and
// L = ceil(4 k ln(kd/eps_int)).  NoPreconditioningNeeded from tune_shift
// (lambda_hat_s < 3 delta) routes the interval to PlainPower with width
// p-s+1 and q = k (plain power converges there without a shift).  Every
// subspace iteration stops early at conv_tol and is capped at max_outer when
// > 0.  Seeds: interval j uses derive_seed(seed, "intv" + j) as its root.
// Final: restricted_projection(A, basis (d x p), k).
constexpr uint64_t kTagInterval = 0x696e7476ull;  // "intv"
constexpr uint64_t kTagGapBudget = 0x67617062ull;  // "gapb"

// find_gap_budget (procedure pinned here):
// Alg. 3 on A with p + 1 columns at eps' = 1/100 (seed derive_seed(seed,
// "gapb")), Delta0 = lambda_hat_k - lambda_hat_{p+1}; NoUsableGap when
// Delta0 <= 1e-14 lambda_hat_1; Delta = Delta0 / 1.5 (the contract Delta <=
// lambda_k - lambda_{p+1} <= 2 Delta then holds while the two estimates are
// within the +-1/3 band of the true gap).
double find_gap_budget(const Mat& x, int k, int p, uint64_t seed, double rq_tol, orc_ledger* led, int nthreads) {
  GramOp a(x, led, nthreads);
  const std::vector<double> est = estimate_eigs(a, x.d(), p + 1, 0.01, derive_seed(seed, kTagGapBudget), rq_tol,
                                                nullptr, led);
  const double d0 = est[k - 1] - est[p];
  if (!(d0 > 1e-14 * est[0])) throw Status(ORC_NO_USABLE_GAP);
  return d0 / 1.5;
}

void approximate(const Mat& x, const orc_si_config* cfg, Block& w, std::vector<double>& ritz, orc_ap_report* rep,
                 int nthreads) {
  const int d = x.d(), k = cfg->k, p = cfg->p;
  const double eps_int = cfg->eps / (3.0 * std::max(cfg->mu, 1.0) * k * d);
  const double lg = std::log(k * static_cast<double>(d) / eps_int);
  auto capped = [&](double L) {
    const int l = static_cast<int>(std::min(std::ceil(L), 1e9));
    return cfg->max_outer > 0 ? std::min(l, cfg->max_outer) : l;
  };
  orc_si_config c2 = *cfg;
  if (!(c2.delta > 0.0)) c2.delta = find_gap_budget(x, k, p, cfg->seed, cfg->rq_tol, &rep->ledger, nthreads);
  rep->delta = c2.delta;
  cfg = &c2;
  Block basis(d, 0);
  int64_t solves = 0;
  int s = 1;
  for (int j = 0; s <= k; ++j) {
    if (j >= k) throw Status(ORC_DEGENERATE_PROGRESS);
    orc_si_config cj = *cfg;
    cj.seed = derive_seed(cfg->seed, kTagInterval + static_cast<uint64_t>(j));
    GramOp a0(x, &rep->ledger, nthreads);
    DeflatedOp a(a0, basis);
    const int cnt = k - s + 1;
    const std::vector<double> est = estimate_eigs(a, d, cnt, 1.0 / (9.0 * p * p), derive_seed(cj.seed, kTagEstA),
                                                  cfg->rq_tol, nullptr, &rep->ledger);
    int q = detect_multiplicative_gap(est.data(), cnt, s, p);
    int strategy = 0, width = 0, iters = 0;
    double shift = 0.0;
    Block S;
    auto plain = [&](int wdt) {
      strategy = 0;
      width = wdt;
      S = subspace_iterate(a, d, wdt, capped(4.0 * std::pow(static_cast<double>(p), 4) * lg),
                           derive_seed(cj.seed, kTagSubspace), cfg->conv_tol, &iters, &rep->ledger);
    };
    if (q >= 0) {
      plain(q - s + 1);
    } else {
      orc_si_report tr;
      std::memset(&tr, 0, sizeof(tr));
      bool shifted = true;
      try {
        tune_shift(x, cfg->delta, &cj, &solves, &tr, nthreads, &basis);
      } catch (const Status& e) {
        if (e.code != ORC_NO_PRECONDITIONING_NEEDED) throw;
        shifted = false;
      }
      auto add = [&](const orc_ledger& l) {
        rep->ledger.gram_applies += l.gram_applies;
        rep->ledger.operator_applies += l.operator_applies;
        rep->ledger.qr_factorizations += l.qr_factorizations;
        rep->ledger.linear_solves += l.linear_solves;
        rep->ledger.solver_column_samples += l.solver_column_samples;
        rep->ledger.epochs += l.epochs;
        rep->ledger.outer_iterations += l.outer_iterations;
      };
      add(tr.ledger);
      if (!shifted) {
        q = k;
        plain(p - s + 1);
      } else {
        shift = tr.lambda;
        orc_svrg_params prm = make_prm(&cj, cfg->tol_solve);
        prm.lambda1_hint = tr.lambda1_hint;
        InverseOp dinv(x, shift, prm, &solves, &rep->ledger, nthreads);
        CgOp dcg(x, shift, cfg->tol_solve, 0, &rep->ledger, nthreads, &basis);
        const bool cg = cfg->backend == 1 || basis.p > 0;
        DeflatedOp dd(cg ? static_cast<BlockOp&>(dcg) : static_cast<BlockOp&>(dinv), basis);
        const std::vector<double> dest = estimate_eigs(dd, d, cnt, 1.0 / (9.0 * p), derive_seed(cj.seed, kTagEstD),
                                                       cfg->rq_tol, nullptr, &rep->ledger);
        std::vector<double> inv(cnt);
        for (int i = 0; i < cnt; ++i) inv[i] = 1.0 / std::max(dest[i], 1e-300);
        q = detect_additive_gap(inv.data(), cnt, s, k, cfg->delta);
        strategy = 1;
        width = q < k ? q - s + 1 : p - s + 1;
        S = subspace_iterate(dd, d, width, capped(4.0 * k * lg), derive_seed(cj.seed, kTagSubspace), cfg->conv_tol,
                             &iters, &rep->ledger);
      }
    }
    basis = basis_extend(basis, S);
    if (rep->n_intervals < 64) {
      const int t = rep->n_intervals;
      rep->s[t] = s;
      rep->q[t] = q;
      rep->strategy[t] = strategy;
      rep->width[t] = width;
      rep->iterations[t] = iters;
      rep->shift[t] = shift;
    }
    rep->n_intervals++;
    s = q + 1;
  }
  restricted_projection(x, basis, k, w, ritz, &rep->ledger, nthreads);
}

int outer_cap(const orc_si_config* cfg, int d) {
  if (cfg->max_outer > 0) return cfg->max_outer;
  const double eps_int = cfg->eps / (3.0 * std::max(cfg->mu, 1.0) * cfg->k * d);
  return static_cast<int>(std::ceil(4.0 * cfg->k * std::log(cfg->k * static_cast<double>(d) / eps_int)));
}

bool valid(const orc_mat* x) {
  if (!x || x->d <= 0 || x->n <= 0) return false;
  if (x->kind == 0) return x->x != nullptr;
  return x->kind == 1 && x->colptr && x->rowidx && x->val;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return ORC_OK;
  } catch (const Status& s) {
    return s.code;
  } catch (...) {
    return ORC_CONTRACT_VIOLATION;
  }
}

}  // namespace

extern "C" {

uint64_t orc_derive_seed(uint64_t root, uint64_t tag) { return derive_seed(root, tag); }

void orc_next_u64(uint64_t seed, int64_t count, uint64_t* out) {
  Rng r(seed);
  for (int64_t i = 0; i < count; ++i) out[i] = r.next();
}

void orc_uniform_index(uint64_t seed, uint64_t n, int64_t count, uint64_t* out) {
  Rng r(seed);
  for (int64_t i = 0; i < count; ++i) out[i] = r.uniform_index(n);
}

void orc_normal(uint64_t seed, int64_t count, double* out) {
  Rng r(seed);
  for (int64_t i = 0; i < count; ++i) out[i] = r.normal();
}

int orc_gaussian_init(int d, int p, uint64_t seed, double* out) {
  return guarded([&] { gaussian_init(d, p, seed).to_rowmajor(out); });
}

int orc_qr(int d, int p, const double* in, double* out, int* bad_col) {
  try {
    Block b = Block::from_rowmajor(d, p, in);
    qr_inplace(b);
    b.to_rowmajor(out);
    return ORC_OK;
  } catch (const Status& s) {
    if (bad_col) *bad_col = s.payload;
    return s.code;
  }
}

int orc_jacobi(int n, const double* in, double* vals, double* vecs) {
  return guarded([&] { jacobi(n, in, vals, vecs); });
}

double orc_max_col_norm2(const orc_mat* x) {
  Mat m(x);
  double best = 0.0;
  for (int j = 0; j < m.n(); ++j) best = std::max(best, m.column_norm_squared(j));
  return best;
}

int orc_gram_block(const orc_mat* x, int p, const double* w, double* z, double* y, int nthreads) {
  if (!valid(x) || p < 1) return ORC_CONTRACT_VIOLATION;
  return guarded([&] {
    Mat m(x);
    Block wb = Block::from_rowmajor(x->d, p, w), zb;
    if (!all_finite(wb.a.data(), wb.a.size())) throw Status(ORC_CONTRACT_VIOLATION);
    std::vector<double> yy;
    gram_block(m, wb, zb, &yy, nthreads);
    zb.to_rowmajor(z);
    if (y)
      for (int j = 0; j < x->n; ++j)
        for (int c = 0; c < p; ++c) y[static_cast<size_t>(j) * p + c] = yy[static_cast<size_t>(c) * x->n + j];
  });
}

int orc_svrg_epoch(const orc_mat* x, int p, double* w, const double* y, const double* c, double eta,
                   double lambda, uint64_t stream_seed, int64_t m, uint64_t* idx_out, int nthreads) {
  if (!valid(x) || p < 1 || m < 0) return ORC_CONTRACT_VIOLATION;
  return guarded([&] {
    Mat mm(x);
    const int d = x->d, n = x->n;
    Block wb = Block::from_rowmajor(d, p, w), cb = Block::from_rowmajor(d, p, c);
    std::vector<double> yy(static_cast<size_t>(n) * p);
    for (int j = 0; j < n; ++j)
      for (int cc = 0; cc < p; ++cc) yy[static_cast<size_t>(cc) * n + j] = y[static_cast<size_t>(j) * p + cc];
    SvrgSetup st;
    st.eta = eta;
    st.lambda = lambda;
    st.rho = 1.0 - eta * lambda;
    st.eta_n = eta * static_cast<double>(n);
    st.m = m;
    st.cap = 0;
    std::vector<int32_t> idx;
    index_stream(stream_seed, n, m, idx);
    if (idx_out)
      for (int64_t s = 0; s < m; ++s) idx_out[s] = static_cast<uint64_t>(idx[s]);
    svrg_epoch(mm, wb, yy, cb, st, idx, nthreads);
    wb.to_rowmajor(w);
  });
}

int orc_svrg_solve(const orc_mat* x, double lambda, int p, const double* b, double* w,
                   const orc_svrg_params* prm, int64_t solve_id, int* epochs, double* history,
                   int hist_cap, int* hist_len, int nthreads) {
  if (!valid(x) || p < 1 || !prm || !(prm->tol > 0.0)) return ORC_CONTRACT_VIOLATION;
  SolveResult res;
  int code = guarded([&] {
    Mat m(x);
    Block bb = Block::from_rowmajor(x->d, p, b), wb;
    if (!all_finite(bb.a.data(), bb.a.size())) throw Status(ORC_CONTRACT_VIOLATION);
    try {
      res = svrg_solve(m, lambda, bb, wb, prm, solve_id, nullptr, nthreads);
    } catch (const Status&) {
      wb.to_rowmajor(w);
      throw;
    }
    wb.to_rowmajor(w);
  });
  if (epochs) *epochs = res.epochs;
  if (hist_len) *hist_len = static_cast<int>(res.history.size());
  if (history)
    for (int i = 0; i < std::min<int>(hist_cap, static_cast<int>(res.history.size())); ++i)
      history[i] = res.history[i];
  return code;
}

int orc_estimate_top(const orc_mat* x, int inverse, double lambda, double eps_prime, uint64_t seed,
                     double rq_tol, const orc_svrg_params* prm, int64_t* solve_counter, double* value,
                     int* iterations, orc_ledger* ledger, int nthreads) {
  if (!valid(x)) return ORC_CONTRACT_VIOLATION;
  return guarded([&] {
    Mat m(x);
    int64_t local = 0;
    if (inverse) {
      InverseOp op(m, lambda, *prm, solve_counter ? solve_counter : &local, ledger, nthreads);
      *value = estimate_top(op, x->d, eps_prime, seed, rq_tol, iterations, ledger);
    } else {
      GramOp op(m, ledger, nthreads);
      *value = estimate_top(op, x->d, eps_prime, seed, rq_tol, iterations, ledger);
    }
  });
}

int orc_tune_shift(const orc_mat* x, double delta, const orc_si_config* cfg, int64_t* solve_counter,
                   orc_si_report* rep, int nthreads) {
  if (!valid(x) || !(delta > 0.0)) return ORC_CONTRACT_VIOLATION;
  return guarded([&] { tune_shift(Mat(x), delta, cfg, solve_counter, rep, nthreads); });
}

int orc_restricted_projection(const orc_mat* x, int p, const double* s, int k, double* w, double* ritz,
                              int nthreads) {
  if (!valid(x) || k < 1 || k > p) return ORC_CONTRACT_VIOLATION;
  return guarded([&] {
    Block sb = Block::from_rowmajor(x->d, p, s), wb;
    std::vector<double> r;
    restricted_projection(Mat(x), sb, k, wb, r, nullptr, nthreads);
    wb.to_rowmajor(w);
    std::copy(r.begin(), r.end(), ritz);
  });
}

int orc_shift_invert(const orc_mat* x, const orc_si_config* cfg, double* w, double* ritz, double* s_out,
                     orc_si_report* rep, int nthreads) {
  if (!valid(x) || !cfg || cfg->k < 1 || cfg->p <= cfg->k || cfg->p >= x->d) return ORC_CONTRACT_VIOLATION;
  std::memset(rep, 0, sizeof(*rep));
  return guarded([&] {
    Mat m(x);
    int64_t solves = 0;
    if (cfg->lambda > 0.0) {
      rep->lambda = cfg->lambda;
      rep->lambda1_hint = cfg->lambda1_hint;
    } else {
      tune_shift(m, cfg->delta, cfg, &solves, rep, nthreads);
    }
    orc_svrg_params prm = make_prm(cfg, cfg->tol_solve);
    prm.lambda1_hint = rep->lambda1_hint;
    InverseOp dinv(m, rep->lambda, prm, &solves, &rep->ledger, nthreads);
    CgOp dcg(m, rep->lambda, cfg->tol_solve, 0, &rep->ledger, nthreads);
    AccOp dacc(m, rep->lambda, prm, &solves, &rep->ledger, nthreads);
    BlockOp& op = cfg->backend == 1   ? static_cast<BlockOp&>(dcg)
                  : cfg->backend == 2 ? static_cast<BlockOp&>(dacc)
                                      : static_cast<BlockOp&>(dinv);
    rep->outer_cap = outer_cap(cfg, x->d);
    Block s = subspace_iterate(op, x->d, cfg->p, rep->outer_cap, derive_seed(cfg->seed, kTagSubspace),
                               cfg->conv_tol, &rep->outer_iterations, &rep->ledger);
    Block wb;
    std::vector<double> r;
    restricted_projection(m, s, cfg->k, wb, r, &rep->ledger, nthreads);
    wb.to_rowmajor(w);
    std::copy(r.begin(), r.end(), ritz);
    if (s_out) s.to_rowmajor(s_out);
  });
}

double orc_sin_theta(int d, int k, const double* u, int q, const double* qm) {
  // R = U - Q (Q^T U); sin theta_max = sqrt(lambda_max(R^T R)).
  std::vector<double> g(static_cast<size_t>(q) * k, 0.0);
  for (int a = 0; a < q; ++a)
    for (int b = 0; b < k; ++b) {
      double acc = 0.0;
      for (int i = 0; i < d; ++i) acc += qm[static_cast<size_t>(i) * q + a] * u[static_cast<size_t>(i) * k + b];
      g[static_cast<size_t>(a) * k + b] = acc;
    }
  std::vector<double> r(static_cast<size_t>(d) * k);
  for (int i = 0; i < d; ++i)
    for (int b = 0; b < k; ++b) {
      double v = u[static_cast<size_t>(i) * k + b];
      for (int a = 0; a < q; ++a) v -= qm[static_cast<size_t>(i) * q + a] * g[static_cast<size_t>(a) * k + b];
      r[static_cast<size_t>(i) * k + b] = v;
    }
  std::vector<double> h(static_cast<size_t>(k) * k, 0.0);
  for (int a = 0; a < k; ++a)
    for (int b = 0; b < k; ++b) {
      double acc = 0.0;
      for (int i = 0; i < d; ++i) acc += r[static_cast<size_t>(i) * k + a] * r[static_cast<size_t>(i) * k + b];
      h[static_cast<size_t>(a) * k + b] = acc;
    }
  std::vector<double> vals(k), vecs(static_cast<size_t>(k) * k);
  jacobi(k, h.data(), vals.data(), vecs.data());
  return std::sqrt(std::max(vals[0], 0.0));
}

int orc_detect_multiplicative_gap(const double* est, int count, int s, int p) {
  return detect_multiplicative_gap(est, count, s, p);
}

int orc_detect_additive_gap(const double* inv, int count, int s, int k, double delta, int* q) {
  return guarded([&] { *q = detect_additive_gap(inv, count, s, k, delta); });
}

int orc_estimate_eigenvalues(const orc_mat* x, int inverse, double lambda, int k, double eps_prime, uint64_t seed,
                             double rq_tol, const orc_svrg_params* prm, double* values, int* iterations,
                             int nthreads) {
  if (!valid(x) || k < 1 || k > x->d || !(eps_prime > 0.0 && eps_prime < 1.0)) return ORC_CONTRACT_VIOLATION;
  return guarded([&] {
    Mat m(x);
    int64_t sc = 0;
    std::vector<double> v;
    if (inverse) {
      InverseOp op(m, lambda, *prm, &sc, nullptr, nthreads);
      v = estimate_eigs(op, x->d, k, eps_prime, seed, rq_tol, iterations, nullptr);
    } else {
      GramOp op(m, nullptr, nthreads);
      v = estimate_eigs(op, x->d, k, eps_prime, seed, rq_tol, iterations, nullptr);
    }
    std::copy(v.begin(), v.end(), values);
  });
}

int orc_find_gap_budget(const orc_mat* x, int k, int p, uint64_t seed, double rq_tol, double* delta, int nthreads) {
  if (!valid(x) || k < 1 || p <= k || p + 1 > x->d || !delta) return ORC_CONTRACT_VIOLATION;
  return guarded([&] { *delta = find_gap_budget(Mat(x), k, p, seed, rq_tol, nullptr, nthreads); });
}

int orc_approximate(const orc_mat* x, const orc_si_config* cfg, double* w, double* ritz, orc_ap_report* rep,
                    int nthreads) {
  if (!valid(x) || !cfg || cfg->k < 1 || cfg->p <= cfg->k || cfg->p >= x->d) return ORC_CONTRACT_VIOLATION;
  std::memset(rep, 0, sizeof(*rep));
  return guarded([&] {
    Block wb;
    std::vector<double> r;
    approximate(Mat(x), cfg, wb, r, rep, nthreads);
    wb.to_rowmajor(w);
    std::copy(r.begin(), r.end(), ritz);
  });
}

int orc_accsvrg_solve(const orc_mat* x, double lambda, int p, const double* b, double* w,
                      const orc_svrg_params* prm, int64_t solve_id, int* epochs, double* history, int hist_cap,
                      int* hist_len, int nthreads) {
  if (!valid(x) || p < 1 || !prm || !(prm->tol > 0.0)) return ORC_CONTRACT_VIOLATION;
  SolveResult res;
  int code = guarded([&] {
    Block bb = Block::from_rowmajor(x->d, p, b), wb;
    res = accsvrg_solve(Mat(x), lambda, bb, wb, prm, solve_id, nullptr, nthreads);
    wb.to_rowmajor(w);
  });
  if (epochs) *epochs = res.epochs;
  if (hist_len) *hist_len = static_cast<int>(res.history.size());
  if (history)
    for (int i = 0; i < std::min<int>(hist_cap, static_cast<int>(res.history.size())); ++i) history[i] = res.history[i];
  return code;
}

int orc_cg_solve(const orc_mat* x, double lambda, int p, const double* b, double* w, double tol, int max_iter,
                 int* iterations, double* history, int hist_cap, int* hist_len, int nthreads) {
  if (!valid(x) || p < 1 || !(tol > 0.0)) return ORC_CONTRACT_VIOLATION;
  return guarded([&] {
    Block bb = Block::from_rowmajor(x->d, p, b), wb;
    CgResult r;
    try {
      r = cg_solve(Mat(x), lambda, bb, wb, tol, max_iter, nullptr, nthreads);
    } catch (...) {
      if (iterations) *iterations = -1;
      throw;
    }
    wb.to_rowmajor(w);
    if (iterations) *iterations = r.iterations;
    if (hist_len) {
      *hist_len = static_cast<int>(r.history.size());
      for (int i = 0; i < std::min(hist_cap, *hist_len); ++i) history[i] = r.history[i];
    }
  });
}

// error_report: frobenius = sqrt(max(0, |X|_F^2 - |W^T X|_F^2))
// (sequential sums: column j of X^T W is spmv_transpose of column c of W);
// spectral = power method on P X X^T P, P = I - W W^T: v0 = P g / |P g| with
// g = gaussian_init(d, 1, derive_seed(seed, "errs")), then `iters` times
// z = P X X^T v, theta = v^T z, v = z / |z|; spectral = sqrt(max(theta, 0)).
int orc_error_report(const orc_mat* x, int k, const double* w, int iters, uint64_t seed, double* frob,
                     double* spec) {
  if (!valid(x) || k < 0 || k > x->d) return ORC_CONTRACT_VIOLATION;
  return guarded([&] {
    Mat m(x);
    const int d = x->d, n = x->n;
    double fx = 0.0;
    for (int j = 0; j < n; ++j) fx += m.column_norm_squared(j);
    Block wb = Block::from_rowmajor(d, k, w);
    std::vector<double> yc(n);
    double fy = 0.0;
    for (int c = 0; c < k; ++c) {
      m.spmv_transpose(wb.col(c), yc.data());
      for (int j = 0; j < n; ++j) fy += yc[j] * yc[j];
    }
    *frob = std::sqrt(std::max(fx - fy, 0.0));
    auto project = [&](std::vector<double>& v) {
      for (int c = 0; c < k; ++c) {
        double a = 0.0;
        for (int i = 0; i < d; ++i) a += wb.at(i, c) * v[i];
        for (int i = 0; i < d; ++i) v[i] -= a * wb.at(i, c);
      }
    };
    auto normalize = [&](std::vector<double>& v) {
      double a = 0.0;
      for (int i = 0; i < d; ++i) a += v[i] * v[i];
      a = std::sqrt(a);
      if (a > 0.0)
        for (int i = 0; i < d; ++i) v[i] /= a;
      return a;
    };
    constexpr uint64_t kTagErr = 0x65727273ull;  // "errs"
    Block g = gaussian_init(d, 1, derive_seed(seed, kTagErr));
    std::vector<double> v(g.a.begin(), g.a.end()), t(n), z(d);
    project(v);
    double theta = 0.0;
    if (normalize(v) > 0.0) {
      for (int it = 0; it < iters; ++it) {
        m.spmv_transpose(v.data(), t.data());
        m.spmv(t.data(), z.data());
        project(z);
        theta = 0.0;
        for (int i = 0; i < d; ++i) theta += v[i] * z[i];
        v = z;
        if (normalize(v) == 0.0) break;
      }
    }
    *spec = std::sqrt(std::max(theta, 0.0));
  });
}

// principal_angles: Q = qr_orthonormalize(S); G = U^T Q
// (k x p, sequential sums); cosines = sqrt(clamp(eig(G G^T), 0, 1)), descending
// (jacobi_eigh order), one per column of U.
int orc_principal_angles(int d, int k, const double* u, int p, const double* s, double* cosines) {
  if (k < 1 || p < 1 || k > d || p > d) return ORC_CONTRACT_VIOLATION;
  return guarded([&] {
    Block q = Block::from_rowmajor(d, p, s);
    qr_inplace(q);
    Block ub = Block::from_rowmajor(d, k, u);
    const std::vector<double> g = gram_ab(ub, q);  // k x p
    std::vector<double> h(static_cast<size_t>(k) * k, 0.0);
    for (int a = 0; a < k; ++a)
      for (int b = 0; b < k; ++b) {
        double acc = 0.0;
        for (int j = 0; j < p; ++j) acc += g[static_cast<size_t>(a) * p + j] * g[static_cast<size_t>(b) * p + j];
        h[static_cast<size_t>(a) * k + b] = acc;
      }
    std::vector<double> vals(k), vecs(static_cast<size_t>(k) * k);
    jacobi(k, h.data(), vals.data(), vecs.data());
    for (int a = 0; a < k; ++a) cosines[a] = std::sqrt(std::min(std::max(vals[a], 0.0), 1.0));
  });
}

}  // extern "C"
