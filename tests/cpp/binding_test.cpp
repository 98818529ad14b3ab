// TEST INFRASTRUCTURE: the reference-side C++ binding (include/gaplra_device.hpp)
// compiled against the reference's own headers and sources
// (/root/reference/proj/core, never copied; recipe: oracle/Makefile
// `binding`) and linked with libgaplra_cuda.so.
//
//   binding_test nogpu   no CUDA device: the binding must surface the failure
//                        as a gaplra::Error subtype (DeviceFailure)
//   binding_test gpu     DeviceGramOperator against the reference
//                        GramOperator (same X, same vectors, same ledger),
//                        apply_block, solve_svrg's residual, and the error
//                        mapping with payloads (SolverStalled history,
//                        RankDeficient column, ContractViolation)
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <random>
#include <string>
#include <vector>

#include "gaplra_device.hpp"

using namespace gaplra;

static int fails = 0;
#define EXPECT(cond, ...)                       \
  do {                                          \
    if (!(cond)) {                              \
      std::fprintf(stderr, "FAIL %s: ", #cond); \
      std::fprintf(stderr, __VA_ARGS__);        \
      std::fprintf(stderr, "\n");               \
      ++fails;                                  \
    }                                           \
  } while (0)

static SparseColumnsMatrix random_x(int d, int n, int z, unsigned seed) {
  std::mt19937_64 g(seed);
  std::normal_distribution<double> nd(0.0, 1.0);
  std::vector<std::vector<SparseEntry>> cols(static_cast<size_t>(n));
  for (int j = 0; j < n; ++j) {
    std::vector<int> rows;
    while (static_cast<int>(rows.size()) < z) {
      const int r = static_cast<int>(g() % static_cast<uint64_t>(d));
      bool dup = false;
      for (int q : rows) dup |= q == r;
      if (!dup) rows.push_back(r);
    }
    std::sort(rows.begin(), rows.end());
    for (int r : rows) cols[static_cast<size_t>(j)].push_back({r, nd(g) / std::sqrt(static_cast<double>(n))});
  }
  return SparseColumnsMatrix(d, n, std::move(cols));
}

static double rel(const std::vector<double>& a, const std::vector<double>& b) {
  double m = 0.0, s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) {
    m = std::max(m, std::fabs(a[i] - b[i]));
    s = std::max(s, std::fabs(b[i]));
  }
  return m / std::max(s, 1e-300);
}

static int run_nogpu() {
  try {
    device::Context ctx(0);
  } catch (const device::DeviceFailure& e) {
    std::printf("binding nogpu ok: DeviceFailure(%d): %s\n", e.status(), e.what());
    return 0;
  } catch (const Error& e) {
    std::printf("unexpected gaplra::Error: %s\n", e.what());
    return 1;
  }
  std::printf("a CUDA device is present: nothing to check in nogpu mode\n");
  return 0;
}

static int run_gpu() {
  device::Context ctx(0);
  const int d = 300, n = 1000;
  const SparseColumnsMatrix x = random_x(d, n, 10, 7);
  CostLedger led_ref, led_dev;
  GramOperator ref(x, &led_ref);
  device::DeviceGramOperator dev(ctx, x, &led_dev);
  EXPECT(dev.dim() == ref.dim(), "dim");
  std::mt19937_64 g(3);
  std::normal_distribution<double> nd(0.0, 1.0);
  // apply: the plugin interface, vector by vector (linear_operator.cpp:23-29)
  for (int t = 0; t < 4; ++t) {
    std::vector<double> v(static_cast<size_t>(d)), a, b;
    for (double& e : v) e = nd(g);
    ref.apply(v, a);
    dev.apply(v, b);
    EXPECT(rel(b, a) <= 1e-13, "apply rel %.3e", rel(b, a));
  }
  // apply_block: p applies in one pass, row-major d x p
  const int p = 5;
  DenseMatrix w(d, p);
  for (double& e : w.entries()) e = nd(g);
  const DenseMatrix z = dev.apply_block(w);
  for (int c = 0; c < p; ++c) {
    std::vector<double> col = w.column(c), a;
    ref.apply(col, a);
    EXPECT(rel(z.column(c), a) <= 1e-13, "apply_block col %d rel %.3e", c, rel(z.column(c), a));
  }
  EXPECT(led_dev.gram_applies.load() == 4 + p && led_ref.gram_applies.load() == 4 + p &&
             led_dev.operator_applies.load() == led_ref.operator_applies.load(),
         "ledger dev %llu ref %llu", (unsigned long long)led_dev.gram_applies.load(),
         (unsigned long long)led_ref.gram_applies.load());
  // solve_svrg at a definite shift: residual of (lambda I - X Xᵀ) W = B by the reference operator
  double l1 = 0.0;
  {
    std::vector<double> q(static_cast<size_t>(d), 1.0), a;
    for (int it = 0; it < 200; ++it) {
      ref.apply(q, a);
      double nrm = 0.0;
      for (double e : a) nrm += e * e;
      nrm = std::sqrt(nrm);
      l1 = nrm;
      for (int i = 0; i < d; ++i) q[static_cast<size_t>(i)] = a[static_cast<size_t>(i)] / nrm;
    }
  }
  const double lam = 1.5 * l1;
  DenseMatrix bm(d, 2);
  for (double& e : bm.entries()) e = nd(g);
  const device::SolverReport rep = device::solve_svrg(dev, lam, bm, 1e-10, 11);
  EXPECT(rep.epochs >= 1 && !rep.residual_history.empty(), "solve report");
  for (int c = 0; c < 2; ++c) {
    std::vector<double> wc = rep.solution.column(c), a;
    ref.apply(wc, a);
    std::vector<double> r(static_cast<size_t>(d));
    double rn = 0.0, bn = 0.0;
    for (int i = 0; i < d; ++i) {
      const double bi = bm(i, c);
      r[static_cast<size_t>(i)] = lam * wc[static_cast<size_t>(i)] - a[static_cast<size_t>(i)] - bi;
      rn += r[static_cast<size_t>(i)] * r[static_cast<size_t>(i)];
      bn += bi * bi;
    }
    EXPECT(std::sqrt(rn / bn) <= 1e-8, "solve residual col %d %.3e", c, std::sqrt(rn / bn));
  }
  // SolverStalled carries the residual history (errors.hpp:46-58)
  try {
    device::solve_svrg(dev, 0.25 * l1, bm, 1e-10, 11);
    EXPECT(false, "indefinite shift did not throw");
  } catch (const SolverStalled& e) {
    EXPECT(!e.residual_history().empty(), "SolverStalled without history");
  }
  // RankDeficient carries the column (errors.hpp:23-31)
  {
    DenseMatrix y(d, 3);
    for (int i = 0; i < d; ++i) {
      y(i, 0) = nd(g);
      y(i, 1) = nd(g);
      y(i, 2) = 2.0 * y(i, 0) - y(i, 1);
    }
    DenseMatrix q(d, 3);
    int bad = -1;
    const int rc = gaplra_qr_orthonormalize(ctx.get(), d, 3, y.entries().data(), q.entries().data(), &bad);
    try {
      device::check(ctx.get(), rc, bad);
      EXPECT(false, "rank-deficient QR did not throw");
    } catch (const RankDeficient& e) {
      EXPECT(e.column() == 2, "RankDeficient column %d", e.column());
    }
  }
  // a non-finite dense X is a ContractViolation at construction (sparse_matrix.cpp:29)
  {
    std::vector<double> xd(static_cast<size_t>(8) * 5, 1.0);
    xd[13] = std::numeric_limits<double>::quiet_NaN();
    try {
      device::DeviceGramOperator bad(ctx, 8, 5, xd.data(), 8);
      EXPECT(false, "non-finite X accepted");
    } catch (const ContractViolation&) {
    }
  }
  std::printf(fails ? "binding gpu FAILED (%d)\n" : "binding gpu ok\n", fails);
  return fails ? 1 : 0;
}

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
  try {
    return gpu ? run_gpu() : run_nogpu();
  } catch (const std::exception& e) {
    std::printf("uncaught: %s\n", e.what());
    return 2;
  }
}
