// capi.cpp -- extern "C" ABI (include/chebmg_b200.h) and the host-side
// control flow of the hot path: Chebyshev smoother (smoothers.hpp:95-172),
// two-level FD V-cycle (multigrid.hpp:69-98), PCG / PGMRES / stationary
// drivers (krylov.hpp:75-264, harness.hpp:118-150).  All vector arithmetic is
// launched on the device; the host keeps only the reference's scalar
// decisions (convergence / breakdown tests) and reads back one small status
// block per Krylov iteration.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numbers>
#include <string>
#include <vector>

#include "cmg_objects.hpp"

namespace {
thread_local std::string g_last_error;
}
namespace cmg {
std::atomic<unsigned long long> g_kernel_launches{0};
void set_last_error(const std::string& m) { g_last_error = m; }
}

using namespace cmg;

namespace {

template <class F>
int guard(F&& f) {
  try {
    f();
    return CMG_OK;
  } catch (const cmg::Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return CMG_ERUNTIME;
  }
}

[[noreturn]] void fail(int code, const std::string& msg) { throw cmg::Error(code, msg); }

double read_scalar(cmg_ctx* c, const double* dev) {
  CMG_CUDA(cudaMemcpyAsync(c->hpin, dev, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  return c->hpin[0];
}

// ------------------------------------------------------------------ FD operator
struct FdOp final : cmg_op {
  FdGrid g;
  double dval;
  FdOp(cmg_ctx* c, std::size_t nn, double Lx, double Ly) {
    if (nn < 2) fail(CMG_EINVAL, "Domain: n must be at least 2");                     // domain.hpp:18
    if (Lx <= 0.0 || Ly <= 0.0) fail(CMG_EINVAL, "Domain: side lengths must be positive");  // :19
    ctx = c;
    const double hx = Lx / static_cast<double>(nn), hy = Ly / static_cast<double>(nn);
    g.m = static_cast<int>(nn - 1);
    g.ihx2 = 1.0 / (hx * hx);
    g.ihy2 = 1.0 / (hy * hy);
    dval = 2.0 * (g.ihx2 + g.ihy2);
    n = len = static_cast<std::size_t>(g.m) * g.m;
  }
  void apply(const double* x, double* y) override {
    fd_apply(g, x, y, ctx->stream);
    ++count;
  }
  void residual(const double* b, const double* x, double* r) override {
    fd_residual(g, b, x, r, nullptr, ctx->stream);
    ++count;
  }
  void diagonal(double* d) override { launch_set(len, dval, d, ctx->stream); }
  void cheb4_init(const double* b, const double* x, bool xz, const double* invd, double c0,
                  double* r, double* d) override {
    fd_cheb4_init(g, b, x, xz, invd, c0, r, d, ctx->stream);
    if (!xz) ++count;
  }
  void cheb4_step(double beta, double c1, double c2, bool xz, const double* invd,
                  const double* r_in, double* x, double* r, const double* d, double* d_out,
                  double beta_last) override {
    fd_cheb4_step(g, beta, c1, c2, xz, invd, r_in, x, r, d, d_out, beta_last, ctx->stream);
    ++count;
  }
  void cheb1_init(const double* b, const double* x, bool xz, const double* invd, double theta,
                  double* z, double* d) override {
    fd_cheb1_init(g, b, x, xz, invd, theta, z, d, ctx->stream);
    if (!xz) ++count;
  }
  void cheb1_step(double c1, double c2, bool xz, const double* invd, double* x, double* z,
                  const double* d, double* d_out, double beta_last) override {
    fd_cheb1_step(g, c1, c2, xz, invd, x, z, d, d_out, beta_last, ctx->stream);
    ++count;
  }
};

}  // namespace

// ------------------------------------------------------------------ generic smoother steps
void cmg_op::cheb4_init(const double* b, const double* x, bool xz, const double* invd, double c0,
                        double* r, double* d) {
  if (xz)
    CMG_CUDA(cudaMemcpyAsync(r, b, len * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  else
    residual(b, x, r);
  launch_scal_copy(len, nullptr, c0, invd, d, ctx->stream);  // d = (c0 * invD)
  launch_mul(len, r, d, ctx->stream);                         // d *= r
}

void cmg_op::cheb4_step(double beta, double c1, double c2, bool xz, const double* invd,
                        const double* r_in, double* x, double* r, const double* d, double* d_out,
                        double beta_last) {
  (void)beta; (void)c1; (void)c2; (void)xz; (void)invd; (void)r_in; (void)x; (void)r; (void)d;
  (void)d_out; (void)beta_last;
  fail(CMG_ERUNTIME, "operator has no fused 4th-kind step");
}
void cmg_op::cheb1_init(const double* b, const double* x, bool xz, const double* invd,
                        double theta, double* z, double* d) {
  (void)b; (void)x; (void)xz; (void)invd; (void)theta; (void)z; (void)d;
  fail(CMG_ERUNTIME, "operator has no fused 1st-kind init");
}
void cmg_op::cheb1_step(double c1, double c2, bool xz, const double* invd, double* x, double* z,
                        const double* d, double* d_out, double beta_last) {
  (void)c1; (void)c2; (void)xz; (void)invd; (void)x; (void)z; (void)d; (void)d_out; (void)beta_last;
  fail(CMG_ERUNTIME, "operator has no fused 1st-kind step");
}

// ------------------------------------------------------------------ smoother (smoothers.hpp)
namespace cmg {

static bool is_fourth(int f) { return f == CMG_FOURTH || f == CMG_FOURTH_OPT; }

void validate_cheb(const cmg_cheb_config& c) {  // smoothers.hpp:51-56
  if (c.family < 0 || c.family > 3) fail(CMG_EINVAL, "unknown smoother family");
  const double lmax = c.lambda_max_multiplier * c.lambda_tilde;
  const double lmin = c.lambda_min_multiplier * c.lambda_tilde;
  if (c.lambda_tilde <= 0.0) fail(CMG_EINVAL, "ChebyshevConfig: lambda_tilde must be positive");
  if (lmax <= 0.0) fail(CMG_EINVAL, "ChebyshevConfig: lambda_max must be positive");
  if (!is_fourth(c.family) && !(0.0 < lmin && lmin < lmax))
    fail(CMG_EINVAL, "ChebyshevConfig: need 0 < lambda_min < lambda_max");
}

void chebyshev_smooth(cmg_op* A, const double* invd, const cmg_cheb_config& cfg,
                      std::size_t order, const double* b, double* x, bool x_is_zero) {
  if (order == 0) return;  // smoothers.hpp:159
  validate_cheb(cfg);
  A->ensure_scratch();
  double* r = A->s_r.p;
  double* d = A->s_d.p;
  double* d2 = A->s_d2.p;
  const double lmax = cfg.lambda_max_multiplier * cfg.lambda_tilde;
  if (is_fourth(cfg.family)) {  // smoothers.hpp:126-148
    const double* beta = nullptr;
    if (cfg.family == CMG_FOURTH_OPT) {
      beta = host_beta_row(order);
      if (!beta)
        fail(CMG_ERANGE, "beta_coefficients: order " + std::to_string(order) +
                             " outside tabulated range 1..20");
    }
    const double inv_lmax = 1.0 / lmax;
    A->cheb4_init(b, x, x_is_zero, invd, (4.0 / 3.0) * inv_lmax, r, d);
    bool xz = x_is_zero;
    const double bk = beta ? beta[order - 1] : 1.0;
    for (std::size_t it = 1; it < order; ++it) {
      const double bi = beta ? beta[it - 1] : 1.0;
      const double fi = static_cast<double>(it);
      const double c1 = (2.0 * fi - 1.0) / (2.0 * fi + 3.0);
      const double c2 = (8.0 * fi + 4.0) / (2.0 * fi + 3.0) * inv_lmax;
      // the last step also applies the final x += beta_k d' (same rounding order)
      A->cheb4_step(bi, c1, c2, xz, invd, r, x, r, d, d2, it + 1 == order ? bk : 0.0);
      std::swap(d, d2);
      xz = false;
    }
    if (order == 1) vec_final_update(A->len, bk, xz, d, x, A->ctx->stream);
  } else {  // smoothers.hpp:95-120
    const double lmin = cfg.lambda_min_multiplier * cfg.lambda_tilde;
    const double theta = 0.5 * (lmax + lmin);
    const double delta = 0.5 * (lmax - lmin);
    const double sigma = theta / delta;
    double rho_prev = 1.0 / sigma;
    A->cheb1_init(b, x, x_is_zero, invd, theta, r, d);
    bool xz = x_is_zero;
    for (std::size_t it = 1; it < order; ++it) {
      const double rho = 1.0 / (2.0 * sigma - rho_prev);
      const double c1 = rho * rho_prev;
      const double c2 = 2.0 * rho / delta;
      A->cheb1_step(c1, c2, xz, invd, x, r, d, d2, it + 1 == order ? 1.0 : 0.0);
      std::swap(d, d2);
      rho_prev = rho;
      xz = false;
    }
    if (order == 1) vec_final_update(A->len, 1.0, xz, d, x, A->ctx->stream);
  }
  // keep the op's canonical scratch pointers stable for the next call
  if (d != A->s_d.p) std::swap(A->s_d.p, A->s_d2.p);
}

// smoothers.hpp:95-148 with the diagonal S replaced by an operator (Schwarz):
// same recurrences and coefficients as chebyshev_smooth, unfused.
void chebyshev_smooth_S(cmg_op* A, SApply S, void* sctx, const cmg_cheb_config& cfg, std::size_t order,
                        const double* b, double* x, bool x_is_zero, SUpdate U) {
  if (order == 0) return;
  validate_cheb(cfg);
  A->ensure_scratch();
  cmg_ctx* c = A->ctx;
  cudaStream_t s = c->stream;
  const std::size_t L = A->len;
  double* r = A->s_r.p;
  double* d = A->s_d.p;
  double* t = A->s_t.p;
  double* sv = c->workspace(7, L);
  const double lmax = cfg.lambda_max_multiplier * cfg.lambda_tilde;
  if (x_is_zero) CMG_CUDA(cudaMemcpyAsync(r, b, L * sizeof(double), cudaMemcpyDeviceToDevice, s));
  else A->residual(b, x, r);
  bool xz = x_is_zero;
  if (is_fourth(cfg.family)) {  // smoothers.hpp:126-148
    const double* beta = nullptr;
    if (cfg.family == CMG_FOURTH_OPT) {
      beta = host_beta_row(order);
      if (!beta)
        fail(CMG_ERANGE, "beta_coefficients: order " + std::to_string(order) + " outside tabulated range 1..20");
    }
    const double inv_lmax = 1.0 / lmax;
    S(sctx, r, sv);
    launch_scal_copy(L, nullptr, (4.0 / 3.0) * inv_lmax, sv, d, s);
    for (std::size_t it = 1; it < order; ++it) {
      const double bi = beta ? beta[it - 1] : 1.0;
      const double fi = static_cast<double>(it);
      const double c1 = (2.0 * fi - 1.0) / (2.0 * fi + 3.0);
      const double c2 = (8.0 * fi + 4.0) / (2.0 * fi + 3.0) * inv_lmax;
      if (U) {
        // x += beta d ; r -= A d in the operator's fused step epilogue (its d
        // update reduced to a copy, c1 = 1, c2 = 0), then the S update
        double* d2 = d == A->s_d.p ? A->s_d2.p : A->s_d.p;
        A->cheb4_step(bi, 1.0, 0.0, xz, d, r, x, r, d, d2, 0.0);
        d = d2;
        xz = false;
        U(sctx, 4, r, c1, c2, d, r, nullptr, 0);
        continue;
      }
      if (xz) launch_scal_copy(L, nullptr, bi, d, x, s);
      else launch_axpy(L, bi, d, x, s);
      xz = false;
      A->apply(d, t);
      launch_axpy(L, -1.0, t, r, s);
      S(sctx, r, sv);
      launch_lincomb(L, c1, d, c2, sv, d, s);
    }
    vec_final_update(L, beta ? beta[order - 1] : 1.0, xz, d, x, s);
    if (d != A->s_d.p) std::swap(A->s_d.p, A->s_d2.p);
  } else {  // smoothers.hpp:95-120
    const double lmin = cfg.lambda_min_multiplier * cfg.lambda_tilde;
    const double theta = 0.5 * (lmax + lmin), delta = 0.5 * (lmax - lmin), sigma = theta / delta;
    double rho_prev = 1.0 / sigma;
    S(sctx, r, sv);  // z = S r (r holds the residual); keep z in r
    CMG_CUDA(cudaMemcpyAsync(r, sv, L * sizeof(double), cudaMemcpyDeviceToDevice, s));
    launch_scal_copy(L, nullptr, 1.0 / theta, r, d, s);
    for (std::size_t it = 1; it < order; ++it) {
      const double rho = 1.0 / (2.0 * sigma - rho_prev);
      if (U) {  // x += d joins the S update (it reads d at the same slot)
        A->apply(d, t);
        U(sctx, 1, t, rho * rho_prev, 2.0 * rho / delta, d, r, x, xz ? 1 : 0);
        xz = false;
        rho_prev = rho;
        continue;
      }
      if (xz) CMG_CUDA(cudaMemcpyAsync(x, d, L * sizeof(double), cudaMemcpyDeviceToDevice, s));
      else launch_axpy(L, 1.0, d, x, s);
      xz = false;
      A->apply(d, t);
      S(sctx, t, sv);
      launch_axpy(L, -1.0, sv, r, s);
      launch_lincomb(L, rho * rho_prev, d, 2.0 * rho / delta, r, d, s);
      rho_prev = rho;
    }
    vec_final_update(L, 1.0, xz, d, x, s);
  }
}

// smoothers.hpp:61-79 with S an operator
double estimate_lambda_max_S(cmg_op* A, SApply S, void* sctx, std::size_t iterations, std::uint64_t seed) {
  if (iterations < 1) fail(CMG_EINVAL, "estimate_lambda_max: iterations must be >= 1");
  cmg_ctx* c = A->ctx;
  std::vector<double> v0(A->n);
  host_random_vector(A->n, seed, v0.data());
  DBuf v(A->len), w(A->len), t(A->len);
  v.zero(c->stream);
  w.zero(c->stream);
  t.zero(c->stream);
  A->upload_canonical(v0.data(), v.p);
  double* nrm = c->dscal + S_TMP0;
  for (std::size_t it = 0; it < iterations; ++it) {
    A->apply(v.p, t.p);
    S(sctx, t.p, w.p);
    A->norm2(w.p, nrm);
    launch_div_scalar_dev(A->len, w.p, nrm, v.p, c->stream);
  }
  A->apply(v.p, t.p);
  S(sctx, t.p, w.p);
  A->dot(v.p, w.p, c->dscal + S_TMP0);
  A->dot(v.p, v.p, c->dscal + S_TMP1);
  CMG_CUDA(cudaMemcpyAsync(c->hpin, c->dscal + S_TMP0, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  return c->hpin[0] / c->hpin[1];
}

// smoothers.hpp:61-79
double estimate_lambda_max(cmg_op* A, const double* invd, std::size_t iterations,
                           std::uint64_t seed) {
  if (iterations < 1) fail(CMG_EINVAL, "estimate_lambda_max: iterations must be >= 1");
  cmg_ctx* c = A->ctx;
  int* zf = c->dflag + 8;
  CMG_CUDA(cudaMemsetAsync(zf, 0, sizeof(int), c->stream));
  A->flag_zero_entries(invd, zf);  // smoothers.hpp:66-67 (padding slots excluded)
  int hz = 0;
  CMG_CUDA(cudaMemcpyAsync(&hz, zf, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  if (hz) fail(CMG_EINVAL, "estimate_lambda_max: zero diagonal entry");
  std::vector<double> v0(A->n);
  host_random_vector(A->n, seed, v0.data());
  DBuf v(A->len), w(A->len);
  v.zero(c->stream);
  w.zero(c->stream);
  A->upload_canonical(v0.data(), v.p);
  double* nrm = c->dscal + S_TMP0;
  for (std::size_t it = 0; it < iterations; ++it) {
    A->apply(v.p, w.p);
    launch_mul(A->len, invd, w.p, c->stream);
    A->norm2(w.p, nrm);
    launch_div_scalar_dev(A->len, w.p, nrm, v.p, c->stream);
  }
  A->apply(v.p, w.p);
  launch_mul(A->len, invd, w.p, c->stream);
  A->dot(v.p, w.p, c->dscal + S_TMP0);
  A->dot(v.p, v.p, c->dscal + S_TMP1);
  CMG_CUDA(cudaMemcpyAsync(c->hpin, c->dscal + S_TMP0, 2 * sizeof(double), cudaMemcpyDeviceToHost,
                           c->stream));
  c->sync();
  return c->hpin[0] / c->hpin[1];
}

}  // namespace cmg

// ------------------------------------------------------------------ FD hierarchy
struct cmg_fd_hier {
  cmg_ctx* ctx = nullptr;
  std::size_t nfine = 0, factor = 0;
  double Lx = 1.0, Ly = 1.0;
  int mf = 0, mc = 0;
  std::unique_ptr<FdOp> A;
  DBuf invd;
  double lambda_tilde = 0.0;
  DBuf S, Dg, rc, ec, t1, t2, r;  // coarse FDM data + scratch
};

namespace {

void fd_coarse_solve(cmg_fd_hier* h, const double* rc, double* ec) {
  // A_c^{-1} = (S x S) D^{-1} (S x S)^T  (fast diagonalisation)
  const int mc = h->mc;
  cudaStream_t s = h->ctx->stream;
  mode_product(0, mc, mc, 1, mc, (long)mc * mc, h->S.p, mc, true, rc, h->t1.p, nullptr, s);
  mode_product(1, mc, mc, 1, mc, (long)mc * mc, h->S.p, mc, true, h->t1.p, h->t2.p, h->Dg.p, s);
  mode_product(0, mc, mc, 1, mc, (long)mc * mc, h->S.p, mc, false, h->t2.p, h->t1.p, nullptr, s);
  mode_product(1, mc, mc, 1, mc, (long)mc * mc, h->S.p, mc, false, h->t1.p, ec, nullptr, s);
}

// multigrid.hpp:69-90
void fd_v_cycle(cmg_fd_hier* h, const cmg_cycle_config& cfg, const double* b, double* x,
                bool x_is_zero) {
  cudaStream_t s = h->ctx->stream;
  if (cfg.k_pre > 0) {
    chebyshev_smooth(h->A.get(), h->invd.p, cfg.smoother, cfg.k_pre, b, x, x_is_zero);
    x_is_zero = false;
  }
  if (x_is_zero) {
    fd_restrict(h->mf, h->mc, (int)h->factor, b, h->rc.p, s);
  } else {
    h->A->residual(b, x, h->r.p);
    fd_restrict(h->mf, h->mc, (int)h->factor, h->r.p, h->rc.p, s);
  }
  fd_coarse_solve(h, h->rc.p, h->ec.p);
  fd_prolong(h->mf, h->mc, (int)h->factor, h->ec.p, x, x_is_zero, s);
  if (cfg.k_post > 0)
    chebyshev_smooth(h->A.get(), h->invd.p, cfg.smoother, cfg.k_post, b, x, false);
}

// preconditioner_apply: one V-cycle from x = 0 (multigrid.hpp:94-98).  The FD
// cycle is a fixed chain of small launches (≈11 at the n=256 config, each a few
// microseconds), so each (v, z) pair it is applied to -- PGMRES walks V_j -> Z_j
// -- is captured once into a CUDA graph and replayed as one launch.  Replays
// re-add the captured operator applications and kernel launches so the
// counters read exactly as for direct launches.  CMG_FD_GRAPHS=0 disables.
struct VCyclePrecond final : cmg_precond {
  cmg_fd_hier* h = nullptr;
  cmg_cycle_config cfg{};
  struct Captured {
    const double* v;
    double* z;
    cudaGraphExec_t exec;
    std::size_t applications;
    unsigned long long launches;
  };
  std::vector<Captured> graphs;
  cudaStream_t cap = nullptr;
  int use_graphs = -1;

  ~VCyclePrecond() override {
    for (auto& g : graphs) cudaGraphExecDestroy(g.exec);
    if (cap) cudaStreamDestroy(cap);
  }

  void apply(const double* v, double* z) override {
    if (use_graphs < 0) {
      const char* env = std::getenv("CMG_FD_GRAPHS");
      use_graphs = (env && std::atoi(env) == 0) ? 0 : 1;
    }
    if (!use_graphs || graphs.size() >= 128) {
      fd_v_cycle(h, cfg, v, z, true);
      return;
    }
    const Captured* g = nullptr;
    for (const auto& c : graphs)
      if (c.v == v && c.z == z) g = &c;
    if (!g) g = capture(v, z);
    CMG_CUDA(cudaGraphLaunch(g->exec, ctx->stream));
    h->A->count += g->applications;
    g_kernel_launches += g->launches;
  }

  const Captured* capture(const double* v, double* z) {
    // everything that may throw or allocate happens before the capture
    if (cfg.k_pre > 0 || cfg.k_post > 0) validate_cheb(cfg.smoother);
    if (cfg.smoother.family == CMG_FOURTH_OPT && std::max(cfg.k_pre, cfg.k_post) > 0 &&
        !host_beta_row(std::max(cfg.k_pre, cfg.k_post)))
      fail(CMG_ERANGE, "beta_coefficients: order outside tabulated range 1..20");
    h->A->ensure_scratch();
    if (!cap) CMG_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    CMG_CUDA(cudaStreamSynchronize(ctx->stream));  // scratch initialisation done
    const std::size_t a0 = h->A->count;
    const unsigned long long l0 = g_kernel_launches.load();
    cudaStream_t user = ctx->stream;
    ctx->stream = cap;
    cudaGraph_t graph = nullptr;
    CMG_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
    try {
      fd_v_cycle(h, cfg, v, z, true);
    } catch (...) {
      cudaStreamEndCapture(cap, &graph);
      if (graph) cudaGraphDestroy(graph);
      ctx->stream = user;
      throw;
    }
    ctx->stream = user;
    CMG_CUDA(cudaStreamEndCapture(cap, &graph));
    cudaGraphExec_t exec = nullptr;
    const cudaError_t err = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    CMG_CUDA(err);
    Captured c{v, z, exec, h->A->count - a0, g_kernel_launches.load() - l0};
    h->A->count = a0;  // captured, not executed
    g_kernel_launches -= c.launches;
    graphs.push_back(c);
    return &graphs.back();
  }
};

// Sturm-count bisection for the extreme eigenvalues of the Lanczos tridiagonal
// (lanczos.hpp:49-83); host arithmetic, m <= a few dozen.
double tridiag_spectral_radius(const std::vector<double>& a, const std::vector<double>& b) {
  const std::size_t n = a.size();
  if (n == 0) fail(CMG_EINVAL, "tridiag_spectral_radius: empty matrix");
  double lo = a[0], hi = a[0];
  for (std::size_t i = 0; i < n; ++i) {
    const double off = (i > 0 ? std::abs(b[i - 1]) : 0.0) + (i + 1 < n ? std::abs(b[i]) : 0.0);
    lo = std::min(lo, a[i] - off);
    hi = std::max(hi, a[i] + off);
  }
  auto below = [&](double x) {
    std::size_t cnt = 0;
    double d = a[0] - x;
    cnt += d < 0.0;
    for (std::size_t i = 1; i < n; ++i) {
      if (d == 0.0) d = 1e-300;
      d = a[i] - x - b[i - 1] * b[i - 1] / d;
      cnt += d < 0.0;
    }
    return cnt;
  };
  const double scale = std::max(std::abs(lo), std::abs(hi)) + 1e-300;
  auto extreme = [&](bool largest) {
    double l = lo, u = hi;
    for (int it = 0; it < 200 && (u - l) > 1e-15 * scale; ++it) {
      const double mid = 0.5 * (l + u);
      const std::size_t c = below(mid);
      const bool keep_upper = largest ? (c == n) : (c == 0);
      if (keep_upper == largest) u = mid; else l = mid;
    }
    return 0.5 * (l + u);
  };
  return std::max(std::abs(extreme(true)), std::abs(extreme(false)));
}

// Lanczos estimate of the approximation constant C (lanczos.hpp:97-155) on the
// device.  The exact fine solve the reference does with a banded Cholesky of
// fine_csr (lanczos.hpp:21-37) is a fast-diagonalisation solve here: the
// 5-point operator is I (x) T/hx^2 + T (x) I/hy^2 with T = tridiag(-1,2,-1),
// whose eigenvectors are the discrete sines -> 4 mode products per solve.
void fd_estimate_C(cmg_fd_hier* h, std::size_t m, std::uint64_t seed, bool reorth,
                   std::vector<double>& alpha, std::vector<double>& beta, double* C) {
  if (m < 1) fail(CMG_EINVAL, "estimate_C: need at least one iteration");
  cmg_ctx* c = h->ctx;
  cudaStream_t s = c->stream;
  FdOp* A = h->A.get();
  const int mf = h->mf;
  const std::size_t n = A->len;
  // fine sine basis and eigenvalue grid
  std::vector<double> Sf((std::size_t)mf * mf), lam(mf), Dg(n);
  const double pi = std::numbers::pi, nrm = std::sqrt(2.0 / (mf + 1));
  for (int i = 0; i < mf; ++i) {
    lam[i] = 2.0 - 2.0 * std::cos((i + 1) * pi / (mf + 1));
    for (int k = 0; k < mf; ++k) Sf[(std::size_t)i * mf + k] = nrm * std::sin((double)(i + 1) * (k + 1) * pi / (mf + 1));
  }
  for (int a = 0; a < mf; ++a)
    for (int b = 0; b < mf; ++b) Dg[(std::size_t)a * mf + b] = lam[b] * A->g.ihx2 + lam[a] * A->g.ihy2;
  DBuf S(Sf.size()), D(n), t1(n), t2(n), u1(n), u2(n), r(n), Q(m * n), sc(2);
  CMG_CUDA(cudaMemcpyAsync(S.p, Sf.data(), Sf.size() * sizeof(double), cudaMemcpyHostToDevice, s));
  CMG_CUDA(cudaMemcpyAsync(D.p, Dg.data(), n * sizeof(double), cudaMemcpyHostToDevice, s));
  auto fine_solve = [&](const double* rhs, double* out) {
    mode_product(0, mf, mf, 1, mf, (long)n, S.p, mf, true, rhs, u1.p, nullptr, s);
    mode_product(1, mf, mf, 1, mf, (long)n, S.p, mf, true, u1.p, u2.p, D.p, s);
    mode_product(0, mf, mf, 1, mf, (long)n, S.p, mf, false, u2.p, u1.p, nullptr, s);
    mode_product(1, mf, mf, 1, mf, (long)n, S.p, mf, false, u1.p, out, nullptr, s);
  };
  const double lambda_hat = estimate_lambda_max(A, h->invd.p, 200, seed ^ 0x9e3779b97f4a7c15ull);
  auto project_f = [&](double* u) {  // u -= P A_c^{-1} P^T A u
    A->apply(u, t1.p);
    fd_restrict(h->mf, h->mc, (int)h->factor, t1.p, h->rc.p, s);
    fd_coarse_solve(h, h->rc.p, h->ec.p);
    fd_prolong(h->mf, h->mc, (int)h->factor, h->ec.p, t2.p, true, s);
    launch_axpy(n, -1.0, t2.p, u, s);
  };
  auto op_inv = [&](const double* q, double* out) {  // lambda_hat * A^{-1} (D q)
    launch_scal_copy(n, nullptr, A->dval, q, t1.p, s);
    fine_solve(t1.p, t2.p);
    launch_scal_copy(n, nullptr, lambda_hat, t2.p, out, s);
  };
  double* d0 = sc.p;
  auto reortho = [&](std::size_t nq) {
    for (std::size_t i = 0; i < nq; ++i) {
      launch_dot(Q.p + i * n, r.p, n, c->dpart, d0, s);
      launch_axpy_dev(n, d0, -1.0, Q.p + i * n, r.p, nullptr, s);
    }
  };
  std::vector<double> q0(n);
  host_random_vector(n, seed, q0.data());
  CMG_CUDA(cudaMemcpyAsync(Q.p, q0.data(), n * sizeof(double), cudaMemcpyHostToDevice, s));
  project_f(Q.p);
  launch_norm2(Q.p, n, c->dpart, d0, s);
  launch_scal_copy(n, d0, 0.0, Q.p, Q.p, s);  // scal(1/||q||, q)
  alpha.clear();
  beta.clear();
  op_inv(Q.p, r.p);
  project_f(r.p);
  launch_dot(Q.p, r.p, n, c->dpart, d0, s);
  alpha.push_back(read_scalar(c, d0));
  launch_axpy_dev(n, d0, -1.0, Q.p, r.p, nullptr, s);
  if (reorth) reortho(1);
  launch_norm2(r.p, n, c->dpart, sc.p + 1, s);
  double bk = read_scalar(c, sc.p + 1);
  for (std::size_t k = 2; k <= m && bk != 0.0; ++k) {
    beta.push_back(bk);
    double* qk = Q.p + (k - 1) * n;
    launch_scal_copy(n, sc.p + 1, 0.0, r.p, qk, s);  // q_k = r / beta
    op_inv(qk, r.p);
    project_f(r.p);
    launch_axpy_dev(n, sc.p + 1, -1.0, Q.p + (k - 2) * n, r.p, nullptr, s);
    launch_dot(qk, r.p, n, c->dpart, d0, s);
    alpha.push_back(read_scalar(c, d0));
    launch_axpy_dev(n, d0, -1.0, qk, r.p, nullptr, s);
    if (reorth) reortho(k);
    launch_norm2(r.p, n, c->dpart, sc.p + 1, s);
    bk = read_scalar(c, sc.p + 1);
  }
  *C = tridiag_spectral_radius(alpha, beta);
}

struct IdentityPrecond final : cmg_precond {
  std::size_t len = 0;
  void apply(const double* v, double* z) override {
    CMG_CUDA(cudaMemcpyAsync(z, v, len * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  }
};

struct CallbackPrecond final : cmg_precond {
  cmg_precond_fn fn = nullptr;
  void* user = nullptr;
  void apply(const double* v, double* z) override { fn(user, v, z); }
};

// ------------------------------------------------------------------ Krylov (krylov.hpp)
struct Report {
  std::size_t iterations = 0, mv0 = 0;
  std::vector<double> hist;
  bool converged = false;
  std::string status;
  double rho = 1.0;
};

void finish(cmg_op* A, Report& R, cmg_solve_report* rep, double t0) {
  if (!R.converged && R.status.empty()) R.status = "maxit reached";
  if (R.iterations > 0) {  // convergence_rate, krylov.hpp:30-37
    R.rho = std::exp(std::log(R.hist.back() / R.hist.front()) / static_cast<double>(R.iterations));
  }
  rep->iterations = R.iterations;
  rep->fine_matvecs = A->count - R.mv0;
  rep->rho = R.rho;
  rep->converged = R.converged ? 1 : 0;
  std::snprintf(rep->status, sizeof rep->status, "%s", R.status.c_str());
  rep->history_len = R.hist.size();
  if (rep->residual_history)
    for (std::size_t i = 0; i < R.hist.size() && i < rep->history_capacity; ++i)
      rep->residual_history[i] = R.hist[i];
  rep->wall_time_sec =
      std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count() - t0;
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

bool device_all_zero(cmg_ctx* c, std::size_t n, const double* x) {
  // all_zero(x0) (krylov.hpp:53-57): any nonzero -> flag
  int* f = c->dflag + 9;
  CMG_CUDA(cudaMemsetAsync(f, 0, sizeof(int), c->stream));
  launch_any_nonzero(n, x, f, c->stream);
  int h = 0;
  CMG_CUDA(cudaMemcpyAsync(&h, f, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  return h == 0;
}

void pgmres(cmg_op* A, cmg_precond* M, const double* b, const double* x0, double* x_out,
            const cmg_solve_options& o, cmg_solve_report* rep) {
  const double t0 = now_s();
  if (o.restart < 1) fail(CMG_EINVAL, "pgmres: restart must be >= 1");
  cmg_ctx* c = A->ctx;
  cudaStream_t s = c->stream;
  const std::size_t L = A->len;
  const int m = static_cast<int>(o.restart);
  Report R;
  R.mv0 = A->count;
  WBuf xb = wsbuf(c, 0, L), r = wsbuf(c, 1, L), V = wsbuf(c, 2, (m + 1) * L), Z = wsbuf(c, 3, m * L),
       w = wsbuf(c, 4, L), rt = wsbuf(c, 5, L), xj = wsbuf(c, 6, L);
  xb.zero(s); r.zero(s); w.zero(s); rt.zero(s); xj.zero(s);
  bool x0zero = true;
  if (x0) {
    CMG_CUDA(cudaMemcpyAsync(xb.p, x0, L * sizeof(double), cudaMemcpyDeviceToDevice, s));
    x0zero = device_all_zero(c, L, x0);
  }
  double* dsc = c->dscal;
  if (x0zero) CMG_CUDA(cudaMemcpyAsync(r.p, b, L * sizeof(double), cudaMemcpyDeviceToDevice, s));
  else A->residual(b, xb.p, r.p);
  A->norm2(r.p, dsc + S_R0);
  const double r0 = read_scalar(c, dsc + S_R0);
  R.hist.push_back(r0);
  if (r0 == 0.0) {
    R.converged = true;
    R.status = "zero initial residual";
    CMG_CUDA(cudaMemcpyAsync(x_out, xb.p, L * sizeof(double), cudaMemcpyDeviceToDevice, s));
    finish(A, R, rep, t0);
    return;
  }
  // scalars of the Arnoldi cycle: the context's fixed slots up to restart 63,
  // else a workspace sized for m (any restart >= 1, krylov.hpp:148)
  double *coef = dsc + S_COEF, *coef2 = dsc + S_COEF2, *H = dsc + S_H, *Hs = dsc + S_HS, *g = dsc + S_G,
         *y = dsc + S_Y;
  if (m > 63) {
    const std::size_t nh = static_cast<std::size_t>(m + 1) * m;
    WBuf sc = wsbuf(c, 8, 2 * (m + 1) + 2 * nh + (m + 1) + m);
    coef = sc.p;
    coef2 = coef + (m + 1);
    H = coef2 + (m + 1);
    Hs = H + nh;
    g = Hs + nh;
    y = g + (m + 1);
  }
  // global working copy of the least-squares solve, used when it exceeds shared memory
  double* lsq_work = wsbuf(c, 9, gmres_lsq_work(m)).p;
  const bool fuse_ok = m <= 63;
  bool done = false;
  while (!done && R.iterations < o.maxit) {
    A->norm2(r.p, dsc + S_BETA);  // beta = norm2(r)
    launch_scal_copy(L, dsc + S_BETA, 0.0, r.p, V.p, s);  // V0 = r * (1/beta)
    CMG_CUDA(cudaMemsetAsync(H, 0, sizeof(double) * (m + 1) * m, s));
    const double window_start = R.hist.back();
    int j = 0;
    for (; j < m && R.iterations < o.maxit; ++j) {
      double* Vj = V.p + (std::size_t)j * L;
      double* Zj = Z.p + (std::size_t)j * L;
      M->apply(Vj, Zj);
      A->apply(Zj, w.p);
      // CGS(2) (krylov.hpp:186-195): project, subtract, [project again, subtract];
      // the first subtraction and the second projection share one pass over V
      static const bool fuse_cgs = [] {
        const char* env = std::getenv("CMG_CGS_FUSE");
        return !(env && std::atoi(env) == 0);
      }();
      A->mdot(V.p, L, j + 1, w.p, coef);
      if (o.reorthogonalize && !(fuse_cgs && fuse_ok)) {
        launch_cgs_update(V.p, L, j + 1, coef, w.p, L, H + j, m, s);
        A->mdot(V.p, L, j + 1, w.p, coef2);
        launch_cgs_update(V.p, L, j + 1, coef2, w.p, L, H + j, m, s);
      } else if (o.reorthogonalize) {
        A->cgs_mdot(V.p, L, j + 1, coef, w.p, coef2, H + j, m);
        launch_cgs_update(V.p, L, j + 1, coef2, w.p, L, H + j, m, s);
      } else {
        launch_cgs_update(V.p, L, j + 1, coef, w.p, L, H + j, m, s);
      }
      double* hj1 = H + (std::size_t)(j + 1) * m + j;
      A->norm2(w.p, hj1);
      launch_normalize_if_pos(L, w.p, hj1, V.p + (std::size_t)(j + 1) * L, s);
      launch_gmres_lsq(H, m, j, 0.0, dsc + S_BETA, Hs, g, y, lsq_work, s);
      launch_form_iterate(xb.p, Z.p, L, j + 1, y, xj.p, L, s);
      A->residual(b, xj.p, rt.p);
      A->norm2(rt.p, dsc + S_RT);
      CMG_CUDA(cudaMemcpyAsync(c->hpin, dsc + S_RT, sizeof(double), cudaMemcpyDeviceToHost, s));
      CMG_CUDA(cudaMemcpyAsync(c->hpin + 1, hj1, sizeof(double), cudaMemcpyDeviceToHost, s));
      c->sync();
      const double rt_norm = c->hpin[0], hj1v = c->hpin[1];
      ++R.iterations;
      R.hist.push_back(rt_norm);
      if (rt_norm / r0 <= o.tol) {
        std::swap(xb.p, xj.p);
        R.converged = true;
        done = true;
        ++j;
        break;
      }
      if (j + 1 == m || R.iterations == o.maxit) {
        std::swap(xb.p, xj.p);
        std::swap(r.p, rt.p);
      }
      if (hj1v == 0.0) {
        if (!(j + 1 == m || R.iterations == o.maxit)) std::swap(xb.p, xj.p);
        R.status = "breakdown: Arnoldi produced a zero vector";
        done = true;
        break;
      }
    }
    if (done) break;
    if (R.hist.back() >= window_start && R.iterations < o.maxit) {
      R.status = "stagnation: no residual decrease over a restart cycle";
      break;
    }
  }
  CMG_CUDA(cudaMemcpyAsync(x_out, xb.p, L * sizeof(double), cudaMemcpyDeviceToDevice, s));
  c->sync();
  finish(A, R, rep, t0);
}

void pcg(cmg_op* A, cmg_precond* M, const double* b, const double* x0, double* x_out,
         const cmg_solve_options& o, cmg_solve_report* rep) {
  const double t0 = now_s();
  cmg_ctx* c = A->ctx;
  cudaStream_t s = c->stream;
  const std::size_t L = A->len;
  Report R;
  R.mv0 = A->count;
  WBuf xb = wsbuf(c, 0, L), r = wsbuf(c, 1, L), z = wsbuf(c, 2, L), p = wsbuf(c, 3, L),
       Ap = wsbuf(c, 4, L), rt = wsbuf(c, 5, L);
  xb.zero(s); r.zero(s); z.zero(s); p.zero(s); Ap.zero(s); rt.zero(s);
  double* dsc = c->dscal;
  int* stop = c->dflag;
  if (o.enforce_spd_preconditioner) {  // krylov.hpp:60-68
    std::vector<double> hu(A->n), hv(A->n);
    host_random_vector(A->n, 0x5eedu, hu.data());
    host_random_vector(A->n, 0xfeedu, hv.data());
    DBuf u(L), v(L), Mu(L), Mv(L);
    u.zero(s); v.zero(s); Mu.zero(s); Mv.zero(s);
    A->upload_canonical(hu.data(), u.p);
    A->upload_canonical(hv.data(), v.p);
    M->apply(v.p, Mv.p);
    A->dot(u.p, Mv.p, dsc + S_TMP0);
    M->apply(u.p, Mu.p);
    A->dot(v.p, Mu.p, dsc + S_TMP1);
    CMG_CUDA(cudaMemcpyAsync(c->hpin, dsc + S_TMP0, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    c->sync();
    const double a = c->hpin[0], bb = c->hpin[1];
    const double scale = std::fabs(a) + std::fabs(bb) + 1.0;
    if (std::fabs(a - bb) > 1e-10 * scale)
      fail(CMG_EINVAL, "pcg: preconditioner failed the symmetry probe");
  }
  bool x0zero = true;
  if (x0) {
    CMG_CUDA(cudaMemcpyAsync(xb.p, x0, L * sizeof(double), cudaMemcpyDeviceToDevice, s));
    x0zero = device_all_zero(c, L, x0);
  }
  if (x0zero) CMG_CUDA(cudaMemcpyAsync(r.p, b, L * sizeof(double), cudaMemcpyDeviceToDevice, s));
  else A->residual(b, xb.p, r.p);
  A->norm2(r.p, dsc + S_R0);
  const double r0 = read_scalar(c, dsc + S_R0);
  R.hist.push_back(r0);
  if (r0 == 0.0) {
    R.converged = true;
    R.status = "zero initial residual";
    CMG_CUDA(cudaMemcpyAsync(x_out, xb.p, L * sizeof(double), cudaMemcpyDeviceToDevice, s));
    finish(A, R, rep, t0);
    return;
  }
  M->apply(r.p, z.p);
  CMG_CUDA(cudaMemcpyAsync(p.p, z.p, L * sizeof(double), cudaMemcpyDeviceToDevice, s));
  A->dot(r.p, z.p, dsc + S_RZ);
  CMG_CUDA(cudaMemsetAsync(stop, 0, sizeof(int), s));
  if (read_scalar(c, dsc + S_RZ) <= 0.0) {
    R.status = "indefinite preconditioner: <r, Mr> <= 0";
  } else {
    for (std::size_t it = 1; it <= o.maxit; ++it) {
      A->apply(p.p, Ap.p);
      A->dot(p.p, Ap.p, dsc + S_PAP);
      launch_pcg_alpha(dsc + S_RZ, dsc + S_PAP, dsc + S_ALPHA, stop, s);
      launch_axpy_dev(L, dsc + S_ALPHA, 1.0, p.p, xb.p, stop, s);
      launch_axpy_dev(L, dsc + S_ALPHA, -1.0, Ap.p, r.p, stop, s);
      A->residual(b, xb.p, rt.p);
      A->norm2(rt.p, dsc + S_RT);
      int hstop = 0;
      CMG_CUDA(cudaMemcpyAsync(c->hpin, dsc + S_RT, sizeof(double), cudaMemcpyDeviceToHost, s));
      CMG_CUDA(cudaMemcpyAsync(&hstop, stop, sizeof(int), cudaMemcpyDeviceToHost, s));
      c->sync();
      if (hstop == 2) {  // pAp <= 0: the reference breaks before the residual matvec
        --A->count;
        R.status = "breakdown: <p, Ap> <= 0";
        break;
      }
      const double rt_norm = c->hpin[0];
      R.iterations = it;
      R.hist.push_back(rt_norm);
      if (rt_norm / r0 <= o.tol) {
        R.converged = true;
        break;
      }
      M->apply(r.p, z.p);
      A->dot(r.p, z.p, dsc + S_RZNEW);
      launch_pcg_beta(dsc + S_RZNEW, dsc + S_RZ, dsc + S_PBETA, stop, s);
      launch_xpby_dev(L, z.p, dsc + S_PBETA, p.p, stop, s);
      CMG_CUDA(cudaMemcpyAsync(&hstop, stop, sizeof(int), cudaMemcpyDeviceToHost, s));
      c->sync();
      if (hstop == 3) {
        R.status = "indefinite preconditioner: <r, Mr> <= 0";
        break;
      }
    }
  }
  CMG_CUDA(cudaMemcpyAsync(x_out, xb.p, L * sizeof(double), cudaMemcpyDeviceToDevice, s));
  c->sync();
  finish(A, R, rep, t0);
}

// harness.hpp:118-150
void stationary(cmg_op* A, cmg_precond* M, const double* b, double tol, std::size_t maxit,
                double* x_out, cmg_solve_report* rep) {
  const double t0 = now_s();
  cmg_ctx* c = A->ctx;
  cudaStream_t s = c->stream;
  const std::size_t L = A->len;
  Report R;
  R.mv0 = A->count;
  WBuf x = wsbuf(c, 0, L), r = wsbuf(c, 1, L), z = wsbuf(c, 2, L);
  x.zero(s); z.zero(s);
  CMG_CUDA(cudaMemcpyAsync(r.p, b, L * sizeof(double), cudaMemcpyDeviceToDevice, s));
  double* dsc = c->dscal;
  A->norm2(r.p, dsc + S_R0);
  const double r0 = read_scalar(c, dsc + S_R0);
  R.hist.push_back(r0);
  if (r0 == 0.0) {
    R.converged = true;
    R.status = "zero initial residual";
  } else {
    for (std::size_t it = 1; it <= maxit; ++it) {
      M->apply(r.p, z.p);
      launch_axpy(L, 1.0, z.p, x.p, s);
      A->residual(b, x.p, r.p);
      A->norm2(r.p, dsc + S_RT);
      const double rn = read_scalar(c, dsc + S_RT);
      R.iterations = it;
      R.hist.push_back(rn);
      if (rn / r0 <= tol) {
        R.converged = true;
        break;
      }
    }
  }
  if (x_out) CMG_CUDA(cudaMemcpyAsync(x_out, x.p, L * sizeof(double), cudaMemcpyDeviceToDevice, s));
  c->sync();
  finish(A, R, rep, t0);
}

cmg_solve_options opts_or_default(const cmg_solve_options* o) {
  cmg_solve_options d{1e-6, 500, 30, 1, 0};  // krylov.hpp:41-49
  return o ? *o : d;
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

const char* cmg_last_error(void) { return g_last_error.c_str(); }
const char* cmg_version(void) { return "chebmg_b200 0.1 (sm_100a)"; }

int cmg_ctx_create(int device, void* stream, cmg_ctx** out) {
  return guard([&] {
    auto c = std::make_unique<cmg_ctx>();
    c->device = device;
    CMG_CUDA(cudaSetDevice(device));
    // NULL selects the legacy default stream, so work stays ordered with a
    // host framework (e.g. torch) that also uses the default stream.
    c->stream = static_cast<cudaStream_t>(stream);
    CMG_CUDA(cudaMalloc(&c->dscal, S_END * sizeof(double)));
    CMG_CUDA(cudaMemset(c->dscal, 0, S_END * sizeof(double)));
    CMG_CUDA(cudaMalloc(&c->dflag, 16 * sizeof(int)));
    CMG_CUDA(cudaMemset(c->dflag, 0, 16 * sizeof(int)));
    CMG_CUDA(cudaMalloc(&c->dpart, (std::size_t)kRedBlocks * 64 * sizeof(double)));
    CMG_CUDA(cudaMallocHost(&c->hpin, 64 * sizeof(double)));
    *out = c.release();
  });
}

int cmg_ctx_destroy(cmg_ctx* c) {
  return guard([&] {
    if (!c) return;
    cudaStreamSynchronize(c->stream);
    cudaFree(c->dscal);
    cudaFree(c->dflag);
    cudaFree(c->dpart);
    cudaFreeHost(c->hpin);
    if (c->own_stream) cudaStreamDestroy(c->stream);
    delete c;
  });
}

int cmg_ctx_synchronize(cmg_ctx* c) { return guard([&] { c->sync(); }); }
uint64_t cmg_ctx_kernel_launches(const cmg_ctx*) { return g_kernel_launches.load(); }

int cmg_malloc(cmg_ctx*, size_t bytes, void** d) {
  return guard([&] { CMG_CUDA(cudaMalloc(d, bytes)); });
}
int cmg_free(cmg_ctx*, void* d) { return guard([&] { CMG_CUDA(cudaFree(d)); }); }
int cmg_upload(cmg_ctx* c, void* dst, const void* src, size_t bytes) {
  return guard([&] {
    CMG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->stream));
    c->sync();
  });
}
int cmg_download(cmg_ctx* c, void* dst, const void* src, size_t bytes) {
  return guard([&] {
    CMG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream));
    c->sync();
  });
}

int cmg_random_vector_host(size_t n, uint64_t seed, double* out) {
  return guard([&] { host_random_vector(n, seed, out); });
}
int cmg_dot(cmg_ctx* c, size_t n, const double* a, const double* b, double* out) {
  return guard([&] {
    launch_dot(a, b, n, c->dpart, c->dscal + S_TMP0, c->stream);
    *out = read_scalar(c, c->dscal + S_TMP0);
  });
}
int cmg_norm2(cmg_ctx* c, size_t n, const double* a, double* out) {
  return guard([&] {
    launch_norm2(a, n, c->dpart, c->dscal + S_TMP0, c->stream);
    *out = read_scalar(c, c->dscal + S_TMP0);
  });
}
int cmg_axpy(cmg_ctx* c, size_t n, double alpha, const double* x, double* y) {
  return guard([&] { launch_axpy(n, alpha, x, y, c->stream); });
}

int cmg_fd_op_create(cmg_ctx* c, size_t n, double Lx, double Ly, cmg_op** out) {
  return guard([&] { *out = new FdOp(c, n, Lx, Ly); });
}
int cmg_op_destroy(cmg_op* op) {
  return guard([&] { delete op; });
}
size_t cmg_op_rows(const cmg_op* op) { return op->n; }
size_t cmg_op_vec_len(const cmg_op* op) { return op->len; }
int cmg_op_apply(cmg_op* op, const double* x, double* y) {
  return guard([&] { op->apply(x, y); });
}
int cmg_op_diagonal(cmg_op* op, double* d) {
  return guard([&] { op->diagonal(d); });
}
size_t cmg_op_applications(const cmg_op* op) { return op->count; }
void cmg_op_reset_applications(cmg_op* op) { op->count = 0; }

int cmg_fd_build_problem_host(size_t n, double Lx, double Ly, uint64_t seed, double* u,
                              double* b) {
  return guard([&] {
    if (n < 2) fail(CMG_EINVAL, "Domain: n must be at least 2");
    if (Lx <= 0.0 || Ly <= 0.0) fail(CMG_EINVAL, "Domain: side lengths must be positive");
    host_fd_build_problem(n, Lx, Ly, seed, u, b);
  });
}

int cmg_jacobi_inverse_diagonal(cmg_ctx* c, size_t n, const double* diag, double* inv) {
  return guard([&] {
    int* zf = c->dflag + 10;
    CMG_CUDA(cudaMemsetAsync(zf, 0, sizeof(int), c->stream));
    launch_recip(n, diag, inv, zf, c->stream);
    int h = 0;
    CMG_CUDA(cudaMemcpyAsync(&h, zf, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    if (h) fail(CMG_EINVAL, "jacobi_inverse_diagonal: zero diagonal entry");
  });
}

int cmg_estimate_lambda_max(cmg_op* A, const double* invd, size_t iterations, uint64_t seed,
                            double* out) {
  return guard([&] { *out = estimate_lambda_max(A, invd, iterations, seed); });
}

int cmg_chebyshev_smooth(cmg_op* A, const double* invd, const cmg_cheb_config* cfg, size_t order,
                         const double* b, double* x, int x_is_zero) {
  return guard([&] { chebyshev_smooth(A, invd, *cfg, order, b, x, x_is_zero != 0); });
}

int cmg_beta_coefficients(size_t k, double* out) {
  return guard([&] {
    const double* row = host_beta_row(k);
    if (!row)
      fail(CMG_ERANGE, "beta_coefficients: order " + std::to_string(k) +
                           " outside tabulated range 1..20");
    std::memcpy(out, row, k * sizeof(double));
  });
}

namespace {
std::unique_ptr<cmg_fd_hier> fd_hier_build(cmg_ctx* c, size_t n, double Lx, double Ly, size_t factor) {
  if (factor < 2 || n % factor != 0)
    fail(CMG_EINVAL, "build_hierarchy: factor must divide n");  // multigrid.hpp:39-40
  if (n / factor < 2)
    fail(CMG_EINVAL, "interp_1d: coarse resolution must divide n and leave interior points");
  auto h = std::make_unique<cmg_fd_hier>();
  h->ctx = c;
  h->nfine = n;
  h->factor = factor;
  h->Lx = Lx;
  h->Ly = Ly;
  h->A = std::make_unique<FdOp>(c, n, Lx, Ly);
  h->mf = h->A->g.m;
  h->mc = static_cast<int>(n / factor - 1);
  const std::size_t nf = h->A->len, nc = (std::size_t)h->mc * h->mc;
  cudaStream_t s = c->stream;
  h->invd.alloc(nf);
  launch_set(nf, 1.0 / h->A->dval, h->invd.p, s);  // jacobi_inverse_diagonal(A.diagonal())
  std::vector<double> S, lam;
  host_fd_coarse_eig((int)n, (int)factor, S, lam);
  const double hx = Lx / static_cast<double>(n), hy = Ly / static_cast<double>(n);
  std::vector<double> Dg(nc);
  for (int a = 0; a < h->mc; ++a)
    for (int bb = 0; bb < h->mc; ++bb) Dg[(std::size_t)a * h->mc + bb] = lam[bb] / (hx * hx) + lam[a] / (hy * hy);
  h->S.alloc(nc);
  h->Dg.alloc(nc);
  CMG_CUDA(cudaMemcpyAsync(h->S.p, S.data(), nc * sizeof(double), cudaMemcpyHostToDevice, s));
  CMG_CUDA(cudaMemcpyAsync(h->Dg.p, Dg.data(), nc * sizeof(double), cudaMemcpyHostToDevice, s));
  h->rc.alloc(nc); h->ec.alloc(nc); h->t1.alloc(nc); h->t2.alloc(nc); h->r.alloc(nf);
  h->r.zero(s);
  c->sync();  // host vectors S, Dg go out of scope
  return h;
}
}  // namespace

int cmg_fd_hierarchy_create(cmg_ctx* c, size_t n, double Lx, double Ly, size_t factor,
                            size_t eigen_iterations, uint64_t eigen_seed, cmg_fd_hier** out) {
  return guard([&] {
    auto h = fd_hier_build(c, n, Lx, Ly, factor);
    h->lambda_tilde = estimate_lambda_max(h->A.get(), h->invd.p, eigen_iterations, eigen_seed);
    h->A->count = 0;  // multigrid.hpp:46
    c->sync();
    *out = h.release();
  });
}

int cmg_fd_hierarchy_clone(const cmg_fd_hier* src, cmg_ctx* c, cmg_fd_hier** out) {
  return guard([&] {
    auto h = fd_hier_build(c, src->nfine, src->Lx, src->Ly, src->factor);
    h->lambda_tilde = src->lambda_tilde;  // same operator: reuse the estimate
    *out = h.release();
  });
}

int cmg_fd_hierarchy_destroy(cmg_fd_hier* h) {
  return guard([&] { delete h; });
}
double cmg_fd_hierarchy_lambda_tilde(const cmg_fd_hier* h) { return h->lambda_tilde; }
cmg_op* cmg_fd_hierarchy_op(cmg_fd_hier* h) { return h->A.get(); }
const double* cmg_fd_hierarchy_inv_diag(cmg_fd_hier* h) { return h->invd.p; }
size_t cmg_fd_hierarchy_coarse_dim(const cmg_fd_hier* h) { return (size_t)h->mc * h->mc; }

int cmg_fd_prolong(cmg_fd_hier* h, const double* xc, double* y) {
  return guard([&] { fd_prolong(h->mf, h->mc, (int)h->factor, xc, y, true, h->ctx->stream); });
}
int cmg_fd_restrict(cmg_fd_hier* h, const double* x, double* yc) {
  return guard([&] { fd_restrict(h->mf, h->mc, (int)h->factor, x, yc, h->ctx->stream); });
}
int cmg_fd_coarse_solve(cmg_fd_hier* h, const double* rc, double* ec) {
  return guard([&] { fd_coarse_solve(h, rc, ec); });
}
int cmg_fd_estimate_C(cmg_fd_hier* h, size_t m, uint64_t seed, int reorthogonalize, double* C,
                      double* alpha, double* beta, size_t* steps) {
  return guard([&] {
    std::vector<double> a, b;
    fd_estimate_C(h, m, seed, reorthogonalize != 0, a, b, C);
    if (alpha) std::copy(a.begin(), a.end(), alpha);
    if (beta) std::copy(b.begin(), b.end(), beta);
    if (steps) *steps = a.size();
  });
}
int cmg_fd_v_cycle(cmg_fd_hier* h, const cmg_cycle_config* cfg, const double* b, double* x,
                   int x_is_zero) {
  return guard([&] { fd_v_cycle(h, *cfg, b, x, x_is_zero != 0); });
}
int cmg_fd_preconditioner_apply(cmg_fd_hier* h, const cmg_cycle_config* cfg, const double* v,
                                double* z) {
  return guard([&] { fd_v_cycle(h, *cfg, v, z, true); });
}

int cmg_precond_fd_vcycle(cmg_fd_hier* h, const cmg_cycle_config* cfg, cmg_precond** out) {
  return guard([&] {
    auto p = std::make_unique<VCyclePrecond>();
    p->ctx = h->ctx;
    p->h = h;
    p->cfg = *cfg;
    *out = p.release();
  });
}
int cmg_precond_identity(cmg_ctx* c, cmg_precond** out) {
  return guard([&] {
    auto p = std::make_unique<IdentityPrecond>();
    p->ctx = c;
    *out = p.release();
  });
}
int cmg_precond_callback(cmg_ctx* c, cmg_precond_fn fn, void* user, cmg_precond** out) {
  return guard([&] {
    auto p = std::make_unique<CallbackPrecond>();
    p->ctx = c;
    p->fn = fn;
    p->user = user;
    *out = p.release();
  });
}
int cmg_precond_destroy(cmg_precond* M) {
  return guard([&] { delete M; });
}
int cmg_precond_apply(cmg_precond* M, const double* v, double* z) {
  return guard([&] { M->apply(v, z); });
}

static void bind_identity_len(cmg_op* A, cmg_precond* M) {
  if (auto* ip = dynamic_cast<IdentityPrecond*>(M)) ip->len = A->len;
}

int cmg_pcg(cmg_op* A, cmg_precond* M, const double* b, const double* x0, double* x,
            const cmg_solve_options* o, cmg_solve_report* rep) {
  return guard([&] {
    bind_identity_len(A, M);
    if (M->variable())
      fail(CMG_EINVAL,
           "pcg: the preconditioner is not a fixed linear operator (deformed-mesh coarse CG above "
           "CMG_COARSE_DENSE_MAX); use pgmres");
    pcg(A, M, b, x0, x, opts_or_default(o), rep);
  });
}
int cmg_pgmres(cmg_op* A, cmg_precond* M, const double* b, const double* x0, double* x,
               const cmg_solve_options* o, cmg_solve_report* rep) {
  return guard([&] {
    bind_identity_len(A, M);
    pgmres(A, M, b, x0, x, opts_or_default(o), rep);
  });
}
int cmg_stationary_solve(cmg_op* A, cmg_precond* M, const double* b, double tol, size_t maxit,
                         double* x, cmg_solve_report* rep) {
  return guard([&] {
    bind_identity_len(A, M);
    stationary(A, M, b, tol, maxit, x, rep);
  });
}

}  // extern "C"
