// gaplra_device.hpp — the reference-side C++ binding of libgaplra_cuda.so.
//
// Header-only, layered on the C ABI (gaplra_cuda.h).  It keeps the reference's
// own C++ API (proj/core/include/gaplra/*.hpp must be on the include path):
//
//   gaplra::device::Context              one CUDA device + stream (gaplra_ctx)
//   gaplra::device::DeviceGramOperator   a gaplra::LinearOperator
//                                        (linear_operator.hpp:34-48) whose
//                                        apply is GramOperator::apply
//                                        (linear_operator.cpp:23-29) on X
//                                        resident in HBM, CostLedger included
//   gaplra::device::solve_svrg           the svrg backend of inverse_operator
//                                        (SPEC.md:327-335,345-348), block form
//   gaplra::device::shift_invert         Alg. 7's ShiftedInverse branch
//   gaplra::device::check                status -> the reference's exception
//                                        types (errors.hpp:10-98), payloads
//                                        (RankDeficient column, SolverStalled
//                                        residual history, ShiftTuningStalled
//                                        (λ, λ̃⁻¹) history) carried over
//
// No numeric work happens here: every call is one C-ABI call.
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "gaplra/dense_matrix.hpp"
#include "gaplra/errors.hpp"
#include "gaplra/linear_operator.hpp"
#include "gaplra/sparse_matrix.hpp"
#include "gaplra_cuda.h"

namespace gaplra {
namespace device {

// SPEC.md:425's signal (tune_shift: lambda_1 < 3 Delta) — errors.hpp has no class for it.
class NoPreconditioningNeeded : public Error {
 public:
  explicit NoPreconditioningNeeded(const std::string& what) : Error(what) {}
};

// CUDA failure or device memory exhausted (no reference counterpart).
class DeviceFailure : public Error {
 public:
  DeviceFailure(const std::string& what, int status) : Error(what), status_(status) {}
  int status() const { return status_; }
  bool out_of_memory() const { return status_ == GAPLRA_OUT_OF_MEMORY; }

 private:
  int status_;
};

// Rethrows a gaplra_status as the reference's exception type.
inline void check(const gaplra_ctx* ctx, int rc, int payload = -1, std::vector<double> residual_history = {},
                  std::vector<std::pair<double, double>> tune_history = {}) {
  if (rc == GAPLRA_OK) return;
  const std::string msg = gaplra_last_error(ctx);
  switch (rc) {
    case GAPLRA_CONTRACT_VIOLATION: throw ContractViolation(msg);
    case GAPLRA_RANK_DEFICIENT: throw RankDeficient(msg, payload);
    case GAPLRA_INDEFINITE_SHIFT: throw IndefiniteShift(msg);
    case GAPLRA_SOLVER_STALLED: throw SolverStalled(msg, std::move(residual_history));
    case GAPLRA_SHIFT_OUT_OF_RANGE: throw ShiftOutOfRange(msg, 0.0, 0.0);
    case GAPLRA_SHIFT_TUNING_STALLED: throw ShiftTuningStalled(msg, std::move(tune_history));
    case GAPLRA_NO_USABLE_GAP: throw NoUsableGap(msg);
    case GAPLRA_DEGENERATE_PROGRESS: throw DegenerateProgress(msg);
    case GAPLRA_NO_PRECONDITIONING_NEEDED: throw NoPreconditioningNeeded(msg);
    default: throw DeviceFailure(msg, rc);  // GAPLRA_DEVICE_ERROR / GAPLRA_OUT_OF_MEMORY
  }
}

class Context {
 public:
  explicit Context(int device = 0) {
    const int rc = gaplra_ctx_create(device, &c_);
    if (rc != GAPLRA_OK) throw DeviceFailure("gaplra_ctx_create failed (no CUDA device?)", rc);
  }
  ~Context() { gaplra_ctx_destroy(c_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  gaplra_ctx* get() const { return c_; }

 private:
  gaplra_ctx* c_ = nullptr;
};

// X resident in HBM; borrows nothing from the host after construction
// (GramOperator borrows X, linear_operator.hpp:53-60: here the device copy is
// owned instead).  CSC straight from the reference's column storage.
class DeviceGramOperator final : public LinearOperator {
 public:
  DeviceGramOperator(const Context& ctx, const SparseColumnsMatrix& x, CostLedger* ledger = nullptr)
      : c_(ctx.get()), d_(x.d()), ledger_(ledger) {
    std::vector<int64_t> cp(static_cast<size_t>(x.n()) + 1, 0);
    std::vector<int32_t> ri;
    std::vector<double> v;
    ri.reserve(static_cast<size_t>(x.nnz()));
    v.reserve(static_cast<size_t>(x.nnz()));
    for (int j = 0; j < x.n(); ++j) {
      for (const SparseEntry& e : x.column(j)) {
        ri.push_back(e.index);
        v.push_back(e.value);
      }
      cp[static_cast<size_t>(j) + 1] = static_cast<int64_t>(ri.size());
    }
    check(c_, gaplra_matrix_csc(c_, x.d(), x.n(), cp.data(), ri.data(), v.data(), 0, &m_));
  }
  // Dense X, column-major d x n with leading dimension ldx (host buffer, copied).
  DeviceGramOperator(const Context& ctx, int d, int n, const double* x_colmajor, int64_t ldx,
                     CostLedger* ledger = nullptr)
      : c_(ctx.get()), d_(d), ledger_(ledger) {
    check(c_, gaplra_matrix_dense(c_, d, n, x_colmajor, ldx, 0, &m_));
  }
  ~DeviceGramOperator() override { gaplra_matrix_destroy(m_); }
  DeviceGramOperator(const DeviceGramOperator&) = delete;
  DeviceGramOperator& operator=(const DeviceGramOperator&) = delete;

  int dim() const override { return d_; }
  // = GramOperator::apply (linear_operator.cpp:23-29), ledger included
  void apply(const std::vector<double>& in, std::vector<double>& out) const override {
    if (static_cast<int>(in.size()) != d_) throw ContractViolation("DeviceGramOperator::apply: length mismatch");
    out.resize(static_cast<size_t>(d_));
    check(c_, gaplra_gram_apply(c_, m_, in.data(), out.data()));
    count(1);
  }
  // p applies in one X·(XᵀW) pass; W row-major d x p (DenseMatrix layout)
  DenseMatrix apply_block(const DenseMatrix& w) const {
    if (w.rows() != d_) throw ContractViolation("DeviceGramOperator::apply_block: row mismatch");
    DenseMatrix z(w.rows(), w.cols());
    check(c_, gaplra_gram_block(c_, m_, w.cols(), w.entries().data(), z.entries().data(), nullptr));
    count(static_cast<uint64_t>(w.cols()));
    return z;
  }
  gaplra_ctx* context() const { return c_; }
  const gaplra_matrix* matrix() const { return m_; }

 private:
  void count(uint64_t k) const {
    if (!ledger_) return;
    ledger_->gram_applies.fetch_add(k, std::memory_order_relaxed);
    ledger_->operator_applies.fetch_add(k, std::memory_order_relaxed);
  }
  gaplra_ctx* c_;
  gaplra_matrix* m_ = nullptr;
  int d_;
  CostLedger* ledger_;
};

struct SolverReport {
  DenseMatrix solution;
  int epochs = 0;
  std::vector<double> residual_history;
};

// solve_svrg(sys, B, tol, seed) for a d x p block sharing one index stream.
inline SolverReport solve_svrg(const DeviceGramOperator& a, double lambda, const DenseMatrix& b, double tol,
                               uint64_t seed = 0, int64_t solve_id = 0, double lambda1_hint = 0.0) {
  SolverReport r{DenseMatrix(b.rows(), b.cols()), 0, std::vector<double>(8192)};
  gaplra_svrg_params prm = {0.0, 0, tol, 0, 10.0, seed, lambda1_hint};
  int len = 0;
  const int rc = gaplra_svrg_solve(a.context(), a.matrix(), lambda, b.cols(), b.entries().data(),
                                   r.solution.entries().data(), &prm, solve_id, &r.epochs, r.residual_history.data(),
                                   static_cast<int>(r.residual_history.size()), &len);
  r.residual_history.resize(static_cast<size_t>(len));
  check(a.context(), rc, -1, r.residual_history);
  return r;
}

struct ShiftInvertResult {
  DenseMatrix W, S;
  std::vector<double> ritz;
  gaplra_si_report report;
};

inline std::vector<std::pair<double, double>> tune_history(const gaplra_si_report& rep) {
  std::vector<std::pair<double, double>> h;
  for (int i = 0; i < rep.tune_steps && i < 64; ++i) h.emplace_back(rep.tune_lambda[i], rep.tune_inv[i]);
  return h;
}

// Alg. 7's ShiftedInverse branch on I = {1..k}: tune_shift -> subspace_iterate -> Alg. 2
inline ShiftInvertResult shift_invert(const DeviceGramOperator& a, const gaplra_si_config& cfg) {
  ShiftInvertResult r{DenseMatrix(a.dim(), cfg.k), DenseMatrix(a.dim(), cfg.p),
                      std::vector<double>(static_cast<size_t>(cfg.k)), gaplra_si_report{}};
  const int rc = gaplra_shift_invert(a.context(), a.matrix(), &cfg, r.W.entries().data(), r.ritz.data(),
                                     r.S.entries().data(), &r.report);
  check(a.context(), rc, -1, {}, tune_history(r.report));
  return r;
}

}  // namespace device
}  // namespace gaplra
