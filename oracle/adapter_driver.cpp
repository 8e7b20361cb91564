// adapter_driver.cpp -- TEST INFRASTRUCTURE: C entry points that run the
// UNMODIFIED reference templates over the B200 library through the
// reference-side binding integration/chebmg_b200_adapter.hpp.  Built by
// oracle/Makefile against /root/reference/proj/include into
// oracle/_ref/libchebmg_adapter.so (git-ignored, travels to the GPU box);
// called by tests/test_adapter_gpu.py.  Nothing here computes: the reference
// templates do, with every operator / preconditioner apply on the GPU.
#include <chebmg_b200_adapter.hpp>
#include <chebmg/smoothers.hpp>

#include <cstring>
#include <memory>
#include <string>

using namespace chebmg;
using chebmg_b200::B200Hierarchy;
using chebmg_b200::B200Operator;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

Family fam(int f) {
  switch (f) {
    case 0: return Family::first;
    case 1: return Family::first_opt_lambda;
    case 2: return Family::fourth;
    default: return Family::fourth_opt;
  }
}

struct Out {
  double* hist;
  std::size_t cap;
  std::size_t* hist_len;
  std::size_t* its;
  std::size_t* mv;
  int* converged;
  char* status;
};

void put(const SolveReport& r, const Out& o) {
  *o.hist_len = r.residual_history.size();
  for (std::size_t i = 0; i < r.residual_history.size() && i < o.cap; ++i) o.hist[i] = r.residual_history[i];
  *o.its = r.iterations;
  *o.mv = r.fine_matvecs;
  *o.converged = r.converged ? 1 : 0;
  std::snprintf(o.status, 128, "%s", r.status.c_str());
}

// one context per process (device 0, legacy stream)
cmg_ctx* ctx0() {
  static cmg_ctx* c = [] {
    cmg_ctx* x = nullptr;
    chebmg_b200::check(cmg_ctx_create(0, nullptr, &x));
    return x;
  }();
  return c;
}

}  // namespace

extern "C" {

const char* ad_last_error() { return g_err.c_str(); }

// chebyshev_smooth (smoothers.hpp:156-172) -- the reference template -- over the
// GPU stencil; inv_diag from B200Operator::diagonal through the reference's
// jacobi_inverse_diagonal.  x in/out (host).
int ad_fd_smooth(std::size_t n, double Lx, int family, std::size_t order, double lambda_tilde, const double* b,
                 double* x, int x_is_zero, std::size_t* apps) {
  return guarded([&] {
    cmg_op* op = nullptr;
    chebmg_b200::check(cmg_fd_op_create(ctx0(), n, Lx, 1.0, &op));
    {
      B200Operator A(ctx0(), op);
      const Vec inv = jacobi_inverse_diagonal(A.diagonal());
      ChebyshevConfig cfg;
      cfg.family = fam(family);
      cfg.lambda_tilde = lambda_tilde;
      const std::size_t m = A.rows();
      Vec bv(b, b + m), xv(x, x + m);
      const std::size_t a0 = A.applications();
      chebyshev_smooth(A, inv, cfg, order, bv, xv, x_is_zero != 0);
      *apps = A.applications() - a0;
      std::memcpy(x, xv.data(), m * sizeof(double));
    }
    cmg_op_destroy(op);
  });
}

// The reference's pcg / pgmres (krylov.hpp:75-264) over B200Operator, with the
// GPU V-cycle as the reference Preconditioner; b = build_problem(rhs_seed 1234).
int ad_fd_solve_templates(std::size_t n, double Lx, std::size_t factor, int family, std::size_t kpre,
                          std::size_t kpost, int driver, double tol, double* x_out, double* hist, std::size_t cap,
                          std::size_t* hist_len, std::size_t* its, std::size_t* mv, int* converged, char* status) {
  return guarded([&] {
    const Domain dom(Lx, 1.0, n);
    B200Hierarchy h(ctx0(), dom, factor, 30, 7);
    B200Operator A(ctx0(), h.op());
    const CycleConfig cc{ChebyshevConfig{fam(family), 1, h.lambda_tilde, 1.03, 0.1}, kpre, kpost};
    const cmg_cycle_config c = chebmg_b200::to_c(cc);
    cmg_precond* Md = nullptr;
    chebmg_b200::check(cmg_precond_fd_vcycle(h.handle(), &c, &Md));
    {
      const Preconditioner M = chebmg_b200::device_preconditioner(ctx0(), Md, A.layout());
      const Problem prob = build_problem(dom, 1234);
      const Vec x0(prob.b.size(), 0.0);
      SolveOptions o;
      o.tol = tol;
      A.reset_applications();
      auto res = driver == 0 ? pcg(A, M, prob.b, x0, o) : pgmres(A, M, prob.b, x0, o);
      std::memcpy(x_out, res.first.data(), res.first.size() * sizeof(double));
      put(res.second, Out{hist, cap, hist_len, its, mv, converged, status});
    }
    cmg_precond_destroy(Md);
  });
}

// run_case_with_b200 (the harness with dispatch_driver_b200), driver 0 pcg, 1 pgmres, 2 mg_solver
int ad_fd_run_case_b200(std::size_t n, double Lx, std::size_t factor, int family, std::size_t k, int cycle,
                        int driver, double tol, double* hist, std::size_t cap, std::size_t* hist_len,
                        std::size_t* its, std::size_t* mv, int* converged, char* status, double* tuned) {
  return guarded([&] {
    CaseConfig cfg;
    cfg.Lx = Lx;
    cfg.n = n;
    cfg.factor = factor;
    cfg.family = fam(family);
    cfg.k = k;
    cfg.cycle = cycle == 0 ? Cycle::full : Cycle::one_sided;
    cfg.driver = driver == 0 ? Driver::pcg : (driver == 1 ? Driver::pgmres : Driver::mg_solver);
    cfg.tol = tol;
    B200Hierarchy h(ctx0(), Domain(Lx, 1.0, n), factor, cfg.eigen_iterations, cfg.seeds.eigen);
    const CaseResult r = chebmg_b200::run_case_with_b200(cfg, h);
    put(r.report, Out{hist, cap, hist_len, its, mv, converged, status});
    *tuned = r.tuned_lambda_min ? *r.tuned_lambda_min : -1.0;
  });
}

// ---- SEM: the reference templates over a GPU SEM level (owned-slot layout mapped
// to the canonical ordering by B200Operator) ----
struct AdPmg {
  cmg_pmg* p = nullptr;
  std::unique_ptr<B200Operator> A;
};

void* ad_pmg_create(int E, int geometry, double eps, int smoother) {
  try {
    auto* h = new AdPmg;
    cmg_sem_desc d{7, E, E, E, geometry, eps, 0, 1};
    const int orders[3] = {7, 3, 1};
    chebmg_b200::check(cmg_pmg_create(ctx0(), &d, 3, orders, smoother, 30, 7, &h->p));
    std::vector<std::int64_t> map(cmg_sem_local_slots(&d));
    chebmg_b200::check(cmg_sem_slot_map_host(&d, map.data()));
    h->A = std::make_unique<B200Operator>(ctx0(), cmg_pmg_op(h->p, 0), std::move(map));
    return h;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ad_pmg_destroy(void* hp) {
  auto* h = static_cast<AdPmg*>(hp);
  if (!h) return;
  h->A.reset();
  cmg_pmg_destroy(h->p);
  delete h;
}

double ad_pmg_lambda(void* hp, int level) { return cmg_pmg_lambda_tilde(static_cast<AdPmg*>(hp)->p, level); }

// chebyshev_smooth template over the GPU fine SEM operator (canonical host vectors)
int ad_pmg_smooth(void* hp, int family, std::size_t order, double lambda_tilde, const double* b, double* x,
                  int x_is_zero, std::size_t* apps) {
  auto* h = static_cast<AdPmg*>(hp);
  return guarded([&] {
    const B200Operator& A = *h->A;
    const Vec inv = jacobi_inverse_diagonal(A.diagonal());
    ChebyshevConfig cfg;
    cfg.family = fam(family);
    cfg.lambda_tilde = lambda_tilde;
    const std::size_t m = A.rows();
    Vec bv(b, b + m), xv(x, x + m);
    const std::size_t a0 = A.applications();
    chebyshev_smooth(A, inv, cfg, order, bv, xv, x_is_zero != 0);
    *apps = A.applications() - a0;
    std::memcpy(x, xv.data(), m * sizeof(double));
  });
}

// the reference's pgmres / pcg over the GPU SEM operator with the GPU p-MG cycle
int ad_pmg_solve(void* hp, int driver, int family, std::size_t kpre, std::size_t kpost, const double* b,
                 double tol, double* x_out, double* hist, std::size_t cap, std::size_t* hist_len,
                 std::size_t* its, std::size_t* mv, int* converged, char* status) {
  auto* h = static_cast<AdPmg*>(hp);
  return guarded([&] {
    const B200Operator& A = *h->A;
    const cmg_cycle_config c{{family, cmg_pmg_lambda_tilde(h->p, 0), 1.03, 0.1}, kpre, kpost};
    cmg_precond* Md = nullptr;
    chebmg_b200::check(cmg_precond_pmg(h->p, &c, &Md));
    {
      const Preconditioner M = chebmg_b200::device_preconditioner(ctx0(), Md, A.layout());
      const std::size_t m = A.rows();
      const Vec bv(b, b + m), x0(m, 0.0);
      SolveOptions o;
      o.tol = tol;
      A.reset_applications();
      auto res = driver == 0 ? pcg(A, M, bv, x0, o) : pgmres(A, M, bv, x0, o);
      std::memcpy(x_out, res.first.data(), m * sizeof(double));
      put(res.second, Out{hist, cap, hist_len, its, mv, converged, status});
    }
    cmg_precond_destroy(Md);
  });
}

}  // extern "C"
