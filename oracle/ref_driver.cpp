// ref_driver.cpp -- C entry points around the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile straight from the
// reference headers where they lie (-I /root/reference/proj/include); output
// goes only to oracle/_ref/libchebmg_ref.so (git-ignored).  Nothing here
// re-implements reference arithmetic: every numeric result comes from the
// reference's own templates (chebyshev_smooth, v_cycle, pcg, pgmres,
// run_case_with, estimate_C).  For the SEM path, which the reference lacks,
// the oracle's C SEM operator (oracle_sem.c) is wrapped in a class satisfying
// the reference's LinearOperatorLike concept (operators.hpp:19-26) so that the
// reference's smoother and Krylov templates drive it -- the CPU baseline the
// survey prescribes.
#include <chebmg/cholesky.hpp>
#include <chebmg/harness.hpp>
#include <chebmg/io.hpp>
#include <chebmg/krylov.hpp>
#include <chebmg/lanczos.hpp>
#include <chebmg/multigrid.hpp>
#include <chebmg/problem.hpp>
#include <chebmg/smoothers.hpp>

#include <algorithm>
#include <memory>
#include <cstring>
#include <sstream>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

extern "C" {
#include "oracle.h"
}

using namespace chebmg;

namespace {

int classify(const std::exception& e) {
  if (dynamic_cast<const std::out_of_range*>(&e)) return 2;
  if (dynamic_cast<const std::invalid_argument*>(&e)) return 1;
  return 3;
}

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return classify(e);
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

void fill_report(const SolveReport& rep, double* hist, std::size_t hist_cap, std::size_t* hist_len,
                 std::size_t* its, std::size_t* mv, int* converged, char* status, double* rho,
                 double* wall) {
  *hist_len = rep.residual_history.size();
  for (std::size_t i = 0; i < rep.residual_history.size() && i < hist_cap; ++i)
    hist[i] = rep.residual_history[i];
  *its = rep.iterations;
  *mv = rep.fine_matvecs;
  *converged = rep.converged ? 1 : 0;
  std::snprintf(status, 128, "%s", rep.status.c_str());
  *rho = rep.rho;
  *wall = rep.wall_time_sec;
}

// LinearOperatorLike adapter over the oracle's C SEM operator.
class SemOperator {
 public:
  explicit SemOperator(orc_op* op, const orc_sem* s) : op_(op), s_(s) {}
  std::size_t rows() const { return op_->n; }
  std::size_t cols() const { return op_->n; }
  void apply(const Vec& x, Vec& y) const { orc_op_apply(op_, x.data(), y.data()); }
  Vec diagonal() const {
    Vec d(op_->n);
    orc_sem_diagonal(s_, d.data());
    return d;
  }
  std::size_t applications() const { return op_->count; }
  void reset_applications() const { op_->count = 0; }

 private:
  orc_op* op_;
  const orc_sem* s_;
};
static_assert(LinearOperatorLike<SemOperator>);

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_random_vector(std::size_t n, std::uint64_t seed, double* out) {
  const Vec v = random_vector(n, seed);
  std::memcpy(out, v.data(), n * sizeof(double));
}

double ref_dot(std::size_t n, const double* a, const double* b) {
  return dot(Vec(a, a + n), Vec(b, b + n));
}

void ref_fd_build_problem(std::size_t n, double Lx, double Ly, std::uint64_t seed, double* u,
                          double* b) {
  const Problem p = build_problem(Domain(Lx, Ly, n), seed);
  std::memcpy(u, p.u_exact.data(), p.u_exact.size() * sizeof(double));
  std::memcpy(b, p.b.data(), p.b.size() * sizeof(double));
}

void ref_fd_stencil_apply(std::size_t n, double Lx, double Ly, const double* x, double* y) {
  const StencilOperator A(Domain(Lx, Ly, n));
  Vec xv(x, x + A.rows()), yv(A.rows());
  A.apply(xv, yv);
  std::memcpy(y, yv.data(), yv.size() * sizeof(double));
}

void ref_fd_prolong(std::size_t n, std::size_t nc, const double* xc, double* y) {
  const Prolongation P(n, nc);
  Vec xv(xc, xc + P.coarse_dim()), yv(P.fine_dim());
  P.apply(xv, yv);
  std::memcpy(y, yv.data(), yv.size() * sizeof(double));
}

void ref_fd_restrict(std::size_t n, std::size_t nc, const double* x, double* yc) {
  const Prolongation P(n, nc);
  Vec xv(x, x + P.fine_dim()), yv(P.coarse_dim());
  P.apply_transpose(xv, yv);
  std::memcpy(yc, yv.data(), yv.size() * sizeof(double));
}

void* ref_hier_create(std::size_t n, double Lx, double Ly, std::size_t factor,
                      std::size_t eigen_iterations, std::uint64_t eigen_seed) {
  try {
    return new Hierarchy(build_hierarchy(Domain(Lx, Ly, n), factor, eigen_iterations, eigen_seed));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_hier_destroy(void* h) { delete static_cast<Hierarchy*>(h); }
double ref_hier_lambda(void* h) { return static_cast<Hierarchy*>(h)->lambda_tilde; }
std::size_t ref_hier_bandwidth(void* h) { return static_cast<Hierarchy*>(h)->coarse->bandwidth(); }
std::size_t ref_hier_coarse_nnz(void* h) { return static_cast<Hierarchy*>(h)->Ac.nonzeros(); }

void ref_hier_coarse_solve(void* hp, const double* rc, double* ec) {
  auto* h = static_cast<Hierarchy*>(hp);
  Vec r(rc, rc + h->P.coarse_dim()), e(h->P.coarse_dim());
  h->coarse->solve(r, e);
  std::memcpy(ec, e.data(), e.size() * sizeof(double));
}

void ref_hier_coarse_apply(void* hp, const double* xc, double* yc) {
  auto* h = static_cast<Hierarchy*>(hp);
  Vec x(xc, xc + h->P.coarse_dim()), y(h->P.coarse_dim());
  h->Ac.apply(x, y);
  std::memcpy(yc, y.data(), y.size() * sizeof(double));
}

int ref_smooth(void* hp, int family, std::size_t order, double lambda_tilde, double lmax_mult,
               double lmin_mult, const double* b, double* x, int x_is_zero, std::size_t* apps) {
  auto* h = static_cast<Hierarchy*>(hp);
  return guarded([&] {
    ChebyshevConfig cfg;
    cfg.family = fam(family);
    cfg.lambda_tilde = lambda_tilde;
    cfg.lambda_max_multiplier = lmax_mult;
    cfg.lambda_min_multiplier = lmin_mult;
    const std::size_t n = h->fine_dim();
    Vec bv(b, b + n), xv(x, x + n);
    const std::size_t a0 = h->A.applications();
    chebyshev_smooth(h->A, h->inv_diag, cfg, order, bv, xv, x_is_zero != 0);
    *apps = h->A.applications() - a0;
    std::memcpy(x, xv.data(), n * sizeof(double));
  });
}

int ref_v_cycle(void* hp, int family, double lmax_mult, double lmin_mult, std::size_t k_pre,
                std::size_t k_post, const double* b, double* x, int x_is_zero, std::size_t* apps) {
  auto* h = static_cast<Hierarchy*>(hp);
  return guarded([&] {
    ChebyshevConfig s;
    s.family = fam(family);
    s.lambda_tilde = h->lambda_tilde;
    s.lambda_max_multiplier = lmax_mult;
    s.lambda_min_multiplier = lmin_mult;
    const std::size_t n = h->fine_dim();
    Vec bv(b, b + n), xv(x, x + n);
    const std::size_t a0 = h->A.applications();
    v_cycle(*h, CycleConfig{s, k_pre, k_post}, bv, xv, x_is_zero != 0);
    *apps = h->A.applications() - a0;
    std::memcpy(x, xv.data(), n * sizeof(double));
  });
}

// driver: 0 pcg, 1 pgmres, 2 mg_solver (stationary)
int ref_solve(void* hp, int driver, int family, double lmax_mult, double lmin_mult,
              std::size_t k_pre, std::size_t k_post, const double* b, const double* x0, double tol,
              std::size_t maxit, std::size_t restart, double* x_out, double* hist,
              std::size_t hist_cap, std::size_t* hist_len, std::size_t* its, std::size_t* mv,
              int* converged, char* status, double* rho, double* wall) {
  auto* h = static_cast<Hierarchy*>(hp);
  return guarded([&] {
    ChebyshevConfig s;
    s.family = fam(family);
    s.lambda_tilde = h->lambda_tilde;
    s.lambda_max_multiplier = lmax_mult;
    s.lambda_min_multiplier = lmin_mult;
    const CycleConfig cc{s, k_pre, k_post};
    const Preconditioner M = [&](const Vec& v) { return preconditioner_apply(*h, cc, v); };
    const std::size_t n = h->fine_dim();
    const Vec bv(b, b + n), x0v(x0, x0 + n);
    SolveOptions o;
    o.tol = tol;
    o.maxit = maxit;
    o.restart = restart;
    SolveReport rep;
    Vec x(n, 0.0);
    if (driver == 0) {
      auto res = pcg(h->A, M, bv, x0v, o);
      x = res.first;
      rep = res.second;
    } else if (driver == 1) {
      auto res = pgmres(h->A, M, bv, x0v, o);
      x = res.first;
      rep = res.second;
    } else {
      rep = detail::stationary_solve(h->A, M, bv, tol, maxit);
    }
    std::memcpy(x_out, x.data(), n * sizeof(double));
    fill_report(rep, hist, hist_cap, hist_len, its, mv, converged, status, rho, wall);
  });
}

// run_case (harness.hpp:253-258) with the hierarchy reused across calls
int ref_run_case_with(void* hp, double Lx, std::size_t n, std::size_t factor, int family,
                      std::size_t k, int cycle, int driver, double tol, std::size_t restart,
                      std::size_t maxit, double* hist, std::size_t hist_cap, std::size_t* hist_len,
                      std::size_t* its, std::size_t* mv, int* converged, char* status, double* rho,
                      double* wall, double* lambda_tilde, double* tuned_lmin) {
  auto* h = static_cast<Hierarchy*>(hp);
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
    cfg.restart = restart;
    cfg.maxit = maxit;
    const CaseResult r = run_case_with(cfg, *h);
    fill_report(r.report, hist, hist_cap, hist_len, its, mv, converged, status, rho, wall);
    *lambda_tilde = r.lambda_tilde;
    *tuned_lmin = r.tuned_lambda_min ? *r.tuned_lambda_min : -1.0;
  });
}

double ref_estimate_C(void* hp, std::size_t m, std::uint64_t seed) {
  auto* h = static_cast<Hierarchy*>(hp);
  return estimate_C(*h, m, seed).C;
}

// ---- SEM: reference templates driving the oracle's restated SEM operator ----

// Chebyshev-Jacobi smoothing sweep on one SEM level through the reference's
// chebyshev_smooth (smoothers.hpp:156-172).
int ref_sem_smooth(void* pmg, int level, int family, std::size_t order, double lmax_mult,
                   double lmin_mult, const double* b, double* x, int x_is_zero, std::size_t* apps) {
  auto* p = static_cast<orc_pmg*>(pmg);
  return guarded([&] {
    orc_sem* s = orc_pmg_sem(p, level);
    SemOperator A(orc_pmg_op(p, level), s);
    const Vec inv_diag = jacobi_inverse_diagonal(A.diagonal());
    ChebyshevConfig cfg;
    cfg.family = fam(family);
    cfg.lambda_tilde = orc_pmg_lambda_tilde(p, level);
    cfg.lambda_max_multiplier = lmax_mult;
    cfg.lambda_min_multiplier = lmin_mult;
    const std::size_t n = A.rows();
    Vec bv(b, b + n), xv(x, x + n);
    const std::size_t a0 = A.applications();
    chebyshev_smooth(A, inv_diag, cfg, order, bv, xv, x_is_zero != 0);
    *apps = A.applications() - a0;
    std::memcpy(x, xv.data(), n * sizeof(double));
  });
}

// Bench helper: a reusable smoother context (inverse diagonal computed once,
// smoothers.hpp:174-181) so repeated sweeps time only chebyshev_smooth.
struct SemSweep {
  orc_pmg* p;
  int level;
  SemOperator A;
  Vec inv_diag;
};

void* ref_sem_sweep_create(void* pmg, int level) {
  auto* p = static_cast<orc_pmg*>(pmg);
  SemOperator A(orc_pmg_op(p, level), orc_pmg_sem(p, level));
  auto* s = new SemSweep{p, level, A, jacobi_inverse_diagonal(A.diagonal())};
  return s;
}
void ref_sem_sweep_destroy(void* s) { delete static_cast<SemSweep*>(s); }

// `reps` sweeps of chebyshev_smooth (reference template) on the stored operator
int ref_sem_sweep_run(void* sp, int family, std::size_t order, double lambda_tilde, const double* b,
                      double* x, int x_is_zero, int reps) {
  auto* s = static_cast<SemSweep*>(sp);
  return guarded([&] {
    ChebyshevConfig cfg;
    cfg.family = fam(family);
    cfg.lambda_tilde = lambda_tilde;
    const std::size_t n = s->A.rows();
    Vec bv(b, b + n), xv(x, x + n);
    for (int r = 0; r < reps; ++r) chebyshev_smooth(s->A, s->inv_diag, cfg, order, bv, xv, x_is_zero != 0);
    std::memcpy(x, xv.data(), n * sizeof(double));
  });
}

// Bench context for the reference CPU arm: ONE SEM level at full size (no
// hierarchy, no coarse factorisation), b = the PAPER.md RHS, a seeded warm x,
// inv_diag = jacobi_inverse_diagonal, lambda_tilde from the reference's
// estimate_lambda_max (setup, untimed; a few iterations suffice for timing).
struct SemBench {
  orc_sem* s;
  SemOperator A;
  Vec inv_diag, b, x;
  double lambda;
};

void* ref_sem_bench_create(int N, int E, int geometry, double eps, std::size_t eig_iters, std::uint64_t seed) {
  try {
    orc_sem* s = orc_sem_create(N, E, E, E, geometry, eps);
    if (!s) throw std::invalid_argument("orc_sem_create failed");
    SemOperator A(orc_sem_op(s), s);
    auto* c = new SemBench{s, A, jacobi_inverse_diagonal(A.diagonal()), Vec(A.rows()), random_vector(A.rows(), 11),
                           0.0};
    orc_sem_rhs(s, c->b.data());
    c->lambda = estimate_lambda_max(c->A, c->inv_diag, eig_iters, seed);
    return c;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

std::size_t ref_sem_bench_n(void* h) { return static_cast<SemBench*>(h)->A.rows(); }
double ref_sem_bench_lambda(void* h) { return static_cast<SemBench*>(h)->lambda; }

// one warm chebyshev_smooth sweep (smoothers.hpp:156-172) in place on x
int ref_sem_bench_sweep(void* h, int family, std::size_t order) {
  auto* c = static_cast<SemBench*>(h);
  return guarded([&] {
    ChebyshevConfig cfg;
    cfg.family = fam(family);
    cfg.lambda_tilde = c->lambda;
    chebyshev_smooth(c->A, c->inv_diag, cfg, order, c->b, c->x, false);
  });
}

void ref_sem_bench_destroy(void* h) {
  auto* c = static_cast<SemBench*>(h);
  if (!c) return;
  orc_sem_destroy(c->s);
  delete c;
}

// p-MG preconditioned PGMRES / PCG through the reference's Krylov templates
// (krylov.hpp:75-264); the preconditioner is the restated multilevel V-cycle.
int ref_sem_solve(void* pmg, int driver, int family, double lmax_mult, double lmin_mult,
                  std::size_t k_pre, std::size_t k_post, const double* b, double tol,
                  std::size_t maxit, std::size_t restart, double* x_out, double* hist,
                  std::size_t hist_cap, std::size_t* hist_len, std::size_t* its, std::size_t* mv,
                  int* converged, char* status, double* rho, double* wall) {
  auto* p = static_cast<orc_pmg*>(pmg);
  return guarded([&] {
    SemOperator A(orc_pmg_op(p, 0), orc_pmg_sem(p, 0));
    const std::size_t n = A.rows();
    const Preconditioner M = [&](const Vec& v) {
      Vec z(n, 0.0);
      if (orc_pmg_v_cycle(p, family, lmax_mult, lmin_mult, k_pre, k_post, v.data(), z.data(), 1))
        throw std::invalid_argument("pmg v-cycle: invalid smoother configuration");
      return z;
    };
    const Vec bv(b, b + n), x0(n, 0.0);
    SolveOptions o;
    o.tol = tol;
    o.maxit = maxit;
    o.restart = restart;
    std::pair<Vec, SolveReport> res =
        driver == 0 ? pcg(A, M, bv, x0, o) : pgmres(A, M, bv, x0, o);
    std::memcpy(x_out, res.first.data(), n * sizeof(double));
    fill_report(res.second, hist, hist_cap, hist_len, its, mv, converged, status, rho, wall);
  });
}

// ---- SEM p-multigrid on the reference's own templates ----
//
// The reference's CPU path for the north-star solve, as literally as the
// reference allows: its pgmres/pcg (krylov.hpp:75-264) drive A; the
// preconditioner is its v_cycle (multigrid.hpp:69-90) generalised to several
// p-levels -- chebyshev_smooth (smoothers.hpp:156-172), residual_into
// (:83-91), axpy, the x = corr assign rule -- with jacobi_inverse_diagonal
// (:174-181), estimate_lambda_max (:61-79) and, on the coarsest level, the
// reference's BandedCholesky (cholesky.hpp:18-91) of the assembled operator
// (CsrMatrix::from_triplets, operators.hpp:80-103).  Only the pieces the
// reference has no code for come from the restatement: the SEM operator and
// its diagonal, the p-transfers, and (for ASM/RAS) the Schwarz smoother with
// its generic-S Chebyshev recurrence.
struct RefPmg {
  orc_pmg* p = nullptr;
  int nl = 0, smoother = 0;
  std::vector<SemOperator> A;
  std::vector<Vec> inv_diag;
  std::vector<double> lambda;
  std::vector<orc_schwarz_ctx> sch;
  std::unique_ptr<BandedCholesky> coarse;

  void vcycle(int l, const ChebyshevConfig& base, std::size_t kpre, std::size_t kpost, const Vec& b, Vec& x,
              bool x_is_zero) const {
    const SemOperator& Al = A[l];
    const std::size_t n = Al.rows();
    if (l == nl - 1) {  // exact coarse solve (multigrid.hpp:78)
      if (x_is_zero) {
        coarse->solve(b, x);
      } else {
        Vec r(n), e(n);
        detail::residual_into(Al, b, x, false, r);
        coarse->solve(r, e);
        axpy(1.0, e, x);
      }
      return;
    }
    ChebyshevConfig cfg = base;
    cfg.lambda_tilde = lambda[l];
    auto smooth = [&](std::size_t k, Vec& xv, bool xz) {
      if (smoother == 0) {
        chebyshev_smooth(Al, inv_diag[l], cfg, k, b, xv, xz);
      } else {  // Schwarz S: the restated generic-S recurrence (no reference code)
        orc_smoother S{nullptr, orc_sem_schwarz_apply_cb, const_cast<orc_schwarz_ctx*>(&sch[l])};
        orc_cheb_config c{static_cast<int>(cfg.family), cfg.lambda_tilde, cfg.lambda_max_multiplier,
                          cfg.lambda_min_multiplier};
        orc_op* op = orc_pmg_op(p, l);
        if (orc_chebyshev_smooth(op, &S, &c, k, b.data(), xv.data(), xz ? 1 : 0))
          throw std::invalid_argument("schwarz smoother: invalid configuration");
      }
    };
    if (kpre > 0) {
      smooth(kpre, x, x_is_zero);
      x_is_zero = false;
    }
    Vec r(n);
    detail::residual_into(Al, b, x, x_is_zero, r);
    const std::size_t nc = A[l + 1].rows();
    Vec rc(nc), ec(nc, 0.0), corr(n);
    orc_sem_restrict(orc_pmg_sem(p, l), orc_pmg_sem(p, l + 1), r.data(), rc.data());
    vcycle(l + 1, base, kpre, kpost, rc, ec, true);
    orc_sem_prolong(orc_pmg_sem(p, l), orc_pmg_sem(p, l + 1), ec.data(), corr.data());
    if (x_is_zero) {
      x = corr;
    } else {
      axpy(1.0, corr, x);
    }
    if (kpost > 0) smooth(kpost, x, false);
  }
};

extern "C" {

// levels/diagonals/transfers from the restatement, everything else reference
void* ref_pmg_create(int nlevels, const int* orders, int Ex, int Ey, int Ez, int geometry, double eps,
                     int smoother, std::size_t eig_iters, std::uint64_t seed) {
  try {
    auto* R = new RefPmg;
    R->p = orc_pmg_create_ex(nlevels, orders, Ex, Ey, Ez, geometry, eps, smoother, eig_iters, seed,
                             ORC_PMG_NO_LAMBDA | ORC_PMG_NO_COARSE);
    if (!R->p) throw std::invalid_argument("orc_pmg_create_ex failed");
    R->nl = nlevels;
    R->smoother = smoother;
    R->sch.resize(nlevels);
    for (int l = 0; l < nlevels; ++l) {
      R->A.emplace_back(orc_pmg_op(R->p, l), orc_pmg_sem(R->p, l));
      R->inv_diag.push_back(jacobi_inverse_diagonal(R->A[l].diagonal()));
      R->sch[l] = orc_schwarz_ctx{orc_pmg_sem(R->p, l), smoother == 2};
    }
    R->lambda.assign(nlevels, 0.0);
    for (int l = 0; l + 1 < nlevels; ++l) {
      if (smoother == 0) {
        R->lambda[l] = estimate_lambda_max(R->A[l], R->inv_diag[l], eig_iters, seed);
      } else {
        orc_smoother S{nullptr, orc_sem_schwarz_apply_cb, &R->sch[l]};
        R->lambda[l] = orc_estimate_lambda_max(orc_pmg_op(R->p, l), &S, eig_iters, seed);
      }
      R->A[l].reset_applications();
    }
    orc_sem* c = orc_pmg_sem(R->p, nlevels - 1);
    const std::size_t cnt = orc_sem_local_triplets(c, nullptr, nullptr, nullptr);
    std::vector<std::int64_t> rr(cnt), cc(cnt);
    std::vector<double> vv(cnt);
    orc_sem_local_triplets(c, rr.data(), cc.data(), vv.data());
    std::vector<std::tuple<std::size_t, std::size_t, double>> trip(cnt);
    for (std::size_t t = 0; t < cnt; ++t) trip[t] = {std::size_t(rr[t]), std::size_t(cc[t]), vv[t]};
    const std::size_t nc = orc_sem_n(c);
    R->coarse = std::make_unique<BandedCholesky>(CsrMatrix::from_triplets(nc, nc, std::move(trip)));
    return R;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_pmg_destroy(void* h) {
  auto* R = static_cast<RefPmg*>(h);
  if (R) orc_pmg_destroy(R->p);
  delete R;
}

void* ref_pmg_levels(void* h) { return static_cast<RefPmg*>(h)->p; }
double ref_pmg_lambda(void* h, int l) { return static_cast<RefPmg*>(h)->lambda[l]; }
std::size_t ref_pmg_coarse_bandwidth(void* h) { return static_cast<RefPmg*>(h)->coarse->bandwidth(); }

int ref_pmg_coarse_solve(void* h, const double* b, double* x) {
  auto* R = static_cast<RefPmg*>(h);
  return guarded([&] {
    const std::size_t n = R->coarse->size();
    Vec bv(b, b + n), xv(n);
    R->coarse->solve(bv, xv);
    std::memcpy(x, xv.data(), n * sizeof(double));
  });
}

// preconditioner_apply (multigrid.hpp:94-98): one V-cycle from x = 0
int ref_pmg_v_cycle(void* h, int family, double lmax_mult, double lmin_mult, std::size_t k_pre,
                    std::size_t k_post, const double* b, double* x) {
  auto* R = static_cast<RefPmg*>(h);
  return guarded([&] {
    ChebyshevConfig s;
    s.family = fam(family);
    s.lambda_max_multiplier = lmax_mult;
    s.lambda_min_multiplier = lmin_mult;
    const std::size_t n = R->A[0].rows();
    Vec bv(b, b + n), xv(n, 0.0);
    R->vcycle(0, s, k_pre, k_post, bv, xv, true);
    std::memcpy(x, xv.data(), n * sizeof(double));
  });
}

// Chebyshev sweep on one level (Jacobi: chebyshev_smooth template)
int ref_pmg_smooth(void* h, int level, int family, std::size_t order, double lmax_mult, double lmin_mult,
                   const double* b, double* x, int x_is_zero, std::size_t* apps) {
  auto* R = static_cast<RefPmg*>(h);
  return guarded([&] {
    ChebyshevConfig cfg;
    cfg.family = fam(family);
    cfg.lambda_tilde = R->lambda[level];
    cfg.lambda_max_multiplier = lmax_mult;
    cfg.lambda_min_multiplier = lmin_mult;
    const std::size_t n = R->A[level].rows();
    Vec bv(b, b + n), xv(x, x + n);
    const std::size_t a0 = R->A[level].applications();
    chebyshev_smooth(R->A[level], R->inv_diag[level], cfg, order, bv, xv, x_is_zero != 0);
    *apps = R->A[level].applications() - a0;
    std::memcpy(x, xv.data(), n * sizeof(double));
  });
}

// pgmres (driver 1) / pcg (driver 0) with the reference-template p-MG V-cycle, x0 = 0
int ref_pmg_solve(void* h, int driver, int family, double lmax_mult, double lmin_mult, std::size_t k_pre,
                  std::size_t k_post, const double* b, double tol, std::size_t maxit, std::size_t restart,
                  double* x_out, double* hist, std::size_t hist_cap, std::size_t* hist_len, std::size_t* its,
                  std::size_t* mv, int* converged, char* status, double* rho, double* wall) {
  auto* R = static_cast<RefPmg*>(h);
  return guarded([&] {
    ChebyshevConfig s;
    s.family = fam(family);
    s.lambda_max_multiplier = lmax_mult;
    s.lambda_min_multiplier = lmin_mult;
    const SemOperator& A = R->A[0];
    const std::size_t n = A.rows();
    const Preconditioner M = [&](const Vec& v) {
      Vec z(n, 0.0);
      R->vcycle(0, s, k_pre, k_post, v, z, true);
      return z;
    };
    const Vec bv(b, b + n), x0(n, 0.0);
    SolveOptions o;
    o.tol = tol;
    o.maxit = maxit;
    o.restart = restart;
    std::pair<Vec, SolveReport> res = driver == 0 ? pcg(A, M, bv, x0, o) : pgmres(A, M, bv, x0, o);
    std::memcpy(x_out, res.first.data(), n * sizeof(double));
    fill_report(res.second, hist, hist_cap, hist_len, its, mv, converged, status, rho, wall);
  });
}

}  // extern "C"

// ---- io.hpp text formats (checker for paper_2210_03179_b200/io.py) ----

static std::size_t put(const std::string& s, char* out, std::size_t cap) {
  if (cap) {
    const std::size_t n = std::min(s.size(), cap - 1);
    std::memcpy(out, s.data(), n);
    out[n] = '\0';
  }
  return s.size();
}

std::size_t ref_format_shortest(double v, char* out, std::size_t cap) {
  return put(format_shortest(v), out, cap);
}

// The reference's own sweep (harness.hpp:297-337) on a config text
// (io.hpp:525-563), emitted as CSV without the wall-time column.
int ref_sweep_csv(const char* config_text, char* out, std::size_t cap, std::size_t* len) {
  return guarded([&] {
    std::istringstream is(config_text);
    const SweepSpec spec = sweep_spec_from_config(Config::parse(is));
    const SweepResult sr = sweep(spec);
    std::ostringstream os;
    CsvOptions o;
    o.include_timing = false;
    write_csv(os, sr.rows, o);
    *len = put(os.str(), out, cap);
  });
}

std::size_t ref_beta_table_csv(char* out, std::size_t cap) {
  std::ostringstream os;
  write_beta_table_csv(os);
  return put(os.str(), out, cap);
}

// One CSV row (io.hpp:71-84) of a CaseResult assembled from plain fields;
// C_est / tuned < 0 mean "absent".
std::size_t ref_csv_row(double Lx, std::size_t factor, int family, std::size_t k, int cycle, int driver,
                        std::size_t its, std::size_t mv, double rho, double C_est, double lambda_tilde,
                        double lmin_mult, double tuned, int converged, double wall_sec, int timing,
                        char* out, std::size_t cap) {
  CaseResult r;
  r.cfg.Lx = Lx;
  r.cfg.factor = factor;
  r.cfg.family = fam(family);
  r.cfg.k = k;
  r.cfg.cycle = cycle == 0 ? Cycle::full : Cycle::one_sided;
  r.cfg.driver = driver == 0 ? Driver::pcg : driver == 1 ? Driver::pgmres : Driver::mg_solver;
  r.cfg.lambda_min_multiplier = lmin_mult;
  r.report.iterations = its;
  r.report.fine_matvecs = mv;
  r.report.rho = rho;
  r.report.converged = converged != 0;
  r.report.wall_time_sec = wall_sec;
  r.lambda_tilde = lambda_tilde;
  if (C_est >= 0) r.C_est = C_est;
  if (tuned >= 0) r.tuned_lambda_min = tuned;
  CsvOptions o;
  o.include_timing = timing != 0;
  std::ostringstream os;
  write_csv_row(os, r, o);
  return put(os.str(), out, cap);
}

}  // extern "C"
