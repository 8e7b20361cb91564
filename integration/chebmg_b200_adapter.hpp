// chebmg_b200_adapter.hpp -- the reference-side binding of libchebmg_b200.so.
//
// This is the header a maintainer of the reference (/root/reference/proj)
// drops next to <chebmg/...> to route the hot path to B200.  It is compiled
// against the UNMODIFIED reference headers by oracle/Makefile (target
// _ref/libchebmg_adapter.so, with the test entry points of
// oracle/adapter_driver.cpp) and exercised by tests/test_adapter_gpu.py.
// Two depths:
//
//  1. Operator level -- B200Operator satisfies chebmg::LinearOperatorLike
//     (operators.hpp:19-26) over host Vecs; the reference's own templates
//     (chebyshev_smooth, v_cycle-style drivers, pcg, pgmres, stationary_solve)
//     run unchanged with every apply executed on the GPU.  device_preconditioner
//     turns a library preconditioner (GPU V-cycle / p-MG cycle) into a
//     chebmg::Preconditioner (krylov.hpp:39).
//  2. Driver level -- dispatch_driver_b200 replaces detail::dispatch_driver
//     (harness.hpp:152-168): the hierarchy, the V-cycle and the Krylov loop stay
//     on the device; run_case_with_b200 is run_case_with (harness.hpp:230-258)
//     with that one call swapped.
#ifndef CHEBMG_B200_ADAPTER_HPP
#define CHEBMG_B200_ADAPTER_HPP

#include <chebmg/harness.hpp>
#include <chebmg/krylov.hpp>
#include <chebmg/multigrid.hpp>
#include <chebmg/operators.hpp>
#include <chebmg/problem.hpp>

#include <algorithm>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "chebmg_b200.h"

namespace chebmg_b200 {

// cmg_status -> the reference's exception types (chebmg_b200.h header comment)
inline void check(int rc) {
  if (rc == CMG_OK) return;
  const std::string msg = cmg_last_error();
  if (rc == CMG_EINVAL) throw std::invalid_argument(msg);
  if (rc == CMG_ERANGE) throw std::out_of_range(msg);
  throw std::runtime_error(msg);
}

// RAII device buffer
class DeviceVec {
 public:
  DeviceVec(cmg_ctx* ctx, std::size_t n) : ctx_(ctx), n_(n) {
    check(cmg_malloc(ctx_, n_ * sizeof(double), reinterpret_cast<void**>(&p_)));
  }
  ~DeviceVec() {
    if (p_) cmg_free(ctx_, p_);
  }
  DeviceVec(const DeviceVec&) = delete;
  DeviceVec& operator=(const DeviceVec&) = delete;
  double* get() const { return p_; }
  std::size_t size() const { return n_; }

 private:
  cmg_ctx* ctx_;
  std::size_t n_;
  double* p_ = nullptr;
};

// Host <-> device vector layout of an operator: identity for FD (vec_len ==
// rows); for SEM the owned-slot map (cmg_sem_slot_map_host: canonical index
// per slot, -1 = padding).
class Layout {
 public:
  Layout(cmg_ctx* ctx, cmg_op* op, std::vector<std::int64_t> slot_map = {})
      : ctx_(ctx), rows_(cmg_op_rows(op)), len_(cmg_op_vec_len(op)), map_(std::move(slot_map)), stage_(len_) {
    if (map_.empty() && len_ != rows_) throw std::invalid_argument("Layout: slot map required (vec_len != rows)");
  }
  std::size_t rows() const { return rows_; }
  std::size_t len() const { return len_; }

  void upload(const chebmg::Vec& v, double* d) const {
    if (map_.empty()) {
      check(cmg_upload(ctx_, d, v.data(), len_ * sizeof(double)));
      return;
    }
    for (std::size_t q = 0; q < len_; ++q) stage_[q] = map_[q] >= 0 ? v[map_[q]] : 0.0;
    check(cmg_upload(ctx_, d, stage_.data(), len_ * sizeof(double)));
  }
  void download(const double* d, chebmg::Vec& v) const {
    v.resize(rows_);
    if (map_.empty()) {
      check(cmg_download(ctx_, v.data(), d, len_ * sizeof(double)));
      return;
    }
    check(cmg_download(ctx_, stage_.data(), d, len_ * sizeof(double)));
    for (std::size_t q = 0; q < len_; ++q)
      if (map_[q] >= 0) v[map_[q]] = stage_[q];
  }

 private:
  cmg_ctx* ctx_;
  std::size_t rows_, len_;
  std::vector<std::int64_t> map_;
  mutable std::vector<double> stage_;
};

// LinearOperatorLike (operators.hpp:19-26) over host Vecs; apply() runs the
// B200 kernel and counts one application on the device operator, so the
// reference's matvec accounting (fine_matvecs) is unchanged.
class B200Operator {
 public:
  B200Operator(cmg_ctx* ctx, cmg_op* op, std::vector<std::int64_t> slot_map = {})
      : op_(op), L_(ctx, op, std::move(slot_map)), dx_(ctx, L_.len()), dy_(ctx, L_.len()) {}
  std::size_t rows() const { return L_.rows(); }
  std::size_t cols() const { return L_.rows(); }
  void apply(const chebmg::Vec& x, chebmg::Vec& y) const {
    L_.upload(x, dx_.get());
    check(cmg_op_apply(op_, dx_.get(), dy_.get()));
    L_.download(dy_.get(), y);
  }
  chebmg::Vec diagonal() const {
    check(cmg_op_diagonal(op_, dy_.get()));
    chebmg::Vec d;
    L_.download(dy_.get(), d);
    return d;
  }
  std::size_t applications() const { return cmg_op_applications(op_); }
  void reset_applications() const { cmg_op_reset_applications(op_); }
  const Layout& layout() const { return L_; }
  cmg_op* handle() const { return op_; }

 private:
  cmg_op* op_;
  Layout L_;
  DeviceVec dx_, dy_;
};
static_assert(chebmg::LinearOperatorLike<B200Operator>);

// A library preconditioner (cmg_precond_fd_vcycle / cmg_precond_pmg) as the
// reference's Preconditioner (krylov.hpp:39): z = M v with host vectors.
inline chebmg::Preconditioner device_preconditioner(cmg_ctx* ctx, cmg_precond* M, const Layout& L) {
  auto dv = std::make_shared<DeviceVec>(ctx, L.len());
  auto dz = std::make_shared<DeviceVec>(ctx, L.len());
  return [M, &L, dv, dz](const chebmg::Vec& v) {
    L.upload(v, dv->get());
    check(cmg_precond_apply(M, dv->get(), dz->get()));
    chebmg::Vec z;
    L.download(dz->get(), z);
    return z;
  };
}

// The reference's Hierarchy (multigrid.hpp:21-48) built on the device.
class B200Hierarchy {
 public:
  B200Hierarchy(cmg_ctx* ctx, const chebmg::Domain& dom, std::size_t factor, std::size_t eigen_iterations,
                std::uint64_t eigen_seed)
      : ctx_(ctx), domain(dom) {
    check(cmg_fd_hierarchy_create(ctx, dom.n, dom.Lx, dom.Ly, factor, eigen_iterations, eigen_seed, &h_));
    lambda_tilde = cmg_fd_hierarchy_lambda_tilde(h_);
  }
  ~B200Hierarchy() {
    if (h_) cmg_fd_hierarchy_destroy(h_);
  }
  B200Hierarchy(const B200Hierarchy&) = delete;
  B200Hierarchy& operator=(const B200Hierarchy&) = delete;
  cmg_fd_hier* handle() const { return h_; }
  cmg_op* op() const { return cmg_fd_hierarchy_op(h_); }
  std::size_t fine_dim() const { return cmg_op_rows(op()); }
  cmg_ctx* ctx() const { return ctx_; }

  chebmg::Domain domain;
  double lambda_tilde = 0.0;

 private:
  cmg_ctx* ctx_;
  cmg_fd_hier* h_ = nullptr;
};

inline cmg_cycle_config to_c(const chebmg::CycleConfig& cc) {
  return cmg_cycle_config{{static_cast<int>(cc.smoother.family), cc.smoother.lambda_tilde,
                           cc.smoother.lambda_max_multiplier, cc.smoother.lambda_min_multiplier},
                          cc.k_pre, cc.k_post};
}

// detail::dispatch_driver (harness.hpp:152-168) on the device: the V-cycle
// preconditioner and the pcg / pgmres / stationary loop run in the library;
// b crosses the boundary once, the report comes back with the reference's
// fields and status strings.
inline chebmg::SolveReport dispatch_driver_b200(const chebmg::CaseConfig& cfg, const B200Hierarchy& h,
                                                const chebmg::CycleConfig& cycle_cfg, const chebmg::Vec& b) {
  cmg_ctx* ctx = h.ctx();
  const cmg_cycle_config cc = to_c(cycle_cfg);
  cmg_precond* M = nullptr;
  check(cmg_precond_fd_vcycle(h.handle(), &cc, &M));
  const std::size_t n = b.size();
  DeviceVec db(ctx, n), dx(ctx, n);
  check(cmg_upload(ctx, db.get(), b.data(), n * sizeof(double)));
  std::vector<double> hist(cfg.maxit + 2);
  cmg_solve_report r{};
  r.residual_history = hist.data();
  r.history_capacity = hist.size();
  const cmg_solve_options o{cfg.tol, cfg.maxit, cfg.restart, 1, 0};
  int rc = CMG_OK;
  switch (cfg.driver) {
    case chebmg::Driver::pcg: rc = cmg_pcg(h.op(), M, db.get(), nullptr, dx.get(), &o, &r); break;
    case chebmg::Driver::pgmres: rc = cmg_pgmres(h.op(), M, db.get(), nullptr, dx.get(), &o, &r); break;
    case chebmg::Driver::mg_solver:
      rc = cmg_stationary_solve(h.op(), M, db.get(), cfg.tol, cfg.maxit, dx.get(), &r);
      break;
  }
  cmg_precond_destroy(M);
  check(rc);
  chebmg::SolveReport rep;
  rep.iterations = r.iterations;
  rep.fine_matvecs = r.fine_matvecs;
  rep.rho = r.rho;
  rep.converged = r.converged != 0;
  rep.status = r.status;
  rep.wall_time_sec = r.wall_time_sec;
  rep.residual_history.assign(hist.begin(), hist.begin() + std::min(r.history_len, hist.size()));
  return rep;
}

// run_case_with (harness.hpp:230-258) with dispatch_driver swapped for the
// device driver; the harness logic around it (problem, lambda_min tuning,
// candidate table, C estimate) is the reference's own.
inline chebmg::CaseResult run_case_with_b200(const chebmg::CaseConfig& cfg, const B200Hierarchy& h) {
  cfg.validate();
  chebmg::CaseResult res;
  res.cfg = cfg;
  res.lambda_tilde = h.lambda_tilde;
  if (cfg.cycle == chebmg::Cycle::one_sided && cfg.driver == chebmg::Driver::pcg)
    res.note = "pcg with an asymmetric one-sided preconditioner";
  auto smoother = [&](double lmin_mult) {
    chebmg::ChebyshevConfig s;
    s.family = cfg.family;
    s.lambda_tilde = h.lambda_tilde;
    s.lambda_max_multiplier = cfg.lambda_max_multiplier;
    s.lambda_min_multiplier = lmin_mult;
    return s;
  };
  double lmin_mult = cfg.lambda_min_multiplier;
  if (cfg.family == chebmg::Family::first_opt_lambda) {  // tune_lambda_min_empirical (harness.hpp:172-225)
    const chebmg::Vec b_tune = chebmg::random_vector(h.fine_dim(), cfg.seeds.tuning);
    std::vector<chebmg::TuneRow> rows;
    for (double cand : chebmg::default_tuning_candidates()) {
      const chebmg::CycleConfig cc{smoother(cand), cfg.k_pre(), cfg.k_post()};
      rows.push_back(chebmg::TuneRow{cand, dispatch_driver_b200(cfg, h, cc, b_tune)});
    }
    const std::size_t best = chebmg::select_tuned(rows);
    if (best == rows.size())
      throw std::runtime_error("tune_lambda_min_empirical: all candidates failed for case " + cfg.id());
    lmin_mult = rows[best].candidate;
    res.tuned_lambda_min = lmin_mult;
  }
  const chebmg::Problem prob = chebmg::build_problem(h.domain, cfg.seeds.rhs);
  const chebmg::CycleConfig cc{smoother(lmin_mult), cfg.k_pre(), cfg.k_post()};
  res.report = dispatch_driver_b200(cfg, h, cc, prob.b);
  if (cfg.estimate_c) {
    double C = 0.0;
    std::size_t steps = 0;
    check(cmg_fd_estimate_C(h.handle(), 20, cfg.seeds.eigen, 1, &C, nullptr, nullptr, &steps));
    res.C_est = C;
  }
  return res;
}

}  // namespace chebmg_b200

#endif
