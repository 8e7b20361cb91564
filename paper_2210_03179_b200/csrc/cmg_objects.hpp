// cmg_objects.hpp -- host-side objects behind the opaque C-ABI handles.
#pragma once

#include "cmg_internal.hpp"
#include "../../include/chebmg_b200.h"

#include <memory>
#include <string>
#include <vector>

namespace cmg {

// device buffer owned by a C++ object
struct DBuf {
  double* p = nullptr;
  std::size_t n = 0;
  DBuf() = default;
  explicit DBuf(std::size_t count) { alloc(count); }
  void alloc(std::size_t count) {
    release();
    n = count;
    if (count) CMG_CUDA(cudaMalloc(&p, count * sizeof(double)));
  }
  void zero(cudaStream_t s) {
    if (n) CMG_CUDA(cudaMemsetAsync(p, 0, n * sizeof(double), s));
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  ~DBuf() { release(); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
};

// NCCL communicator wrapper (comm.cpp).  Only the SEM shared-face halo and
// the Krylov inner-product reductions use it (BASELINE.json north_star).
struct Comm {
  void* nccl = nullptr;  // ncclComm_t
  int rank = 0, nranks = 1;
  // side stream for face exchanges that overlap element kernels, and the
  // events that order it against the compute stream (created with the comm)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_ready = nullptr, ev_halo = nullptr, ev_contrib = nullptr;
  ~Comm();
  // in-place sum over ranks of `count` doubles (device)
  void allreduce_sum(double* buf, std::size_t count, cudaStream_t s);
  // gather `count` doubles from every rank into recv[rank*count ...] (device)
  void allgather(const double* send, double* recv, std::size_t count, cudaStream_t s);
  // grouped point-to-point: send to / receive from neighbours (peer < 0: none)
  void sendrecv(const double* send_up, std::size_t n_up, double* recv_down, std::size_t n_down,
                int up, int down, cudaStream_t s);
  void exchange(const double* send_a, std::size_t na, int peer_a, double* recv_a,
                const double* send_b, std::size_t nb, int peer_b, double* recv_b, cudaStream_t s);
  // one group, both directions: n_up doubles go up (and arrive from below in
  // recv_lo), n_dn go down (and arrive from above in recv_hi)
  void shift(const double* send_up, double* recv_lo, std::size_t n_up, const double* send_dn, double* recv_hi,
             std::size_t n_dn, int up, int down, cudaStream_t s);
};

}  // namespace cmg

// Scratch scalar slots in ctx->dscal
enum : int {
  S_R0 = 0, S_BETA, S_RT, S_TMP0, S_TMP1, S_RZ, S_RZNEW, S_PAP, S_ALPHA, S_PBETA,
  S_COEF = 64,          // restart+1 CGS coefficients
  S_COEF2 = 128,        // second CGS pass (restart+1 <= 64)
  S_H = 256,            // (m+1)*m Hessenberg
  S_HS = S_H + 4160,    // copy
  S_G = S_HS + 4160,    // m+1
  S_Y = S_G + 80,       // m
  S_CG = S_Y + 80,      // coarse CG scalars (8)
  S_END = S_CG + 16
};

struct cmg_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  double* dscal = nullptr;   // S_END doubles
  int* dflag = nullptr;      // 16 ints
  double* dpart = nullptr;   // reduction partials: kRedBlocks * 64
  double* hpin = nullptr;    // pinned readback area: 64 doubles
  std::unique_ptr<cmg::Comm> comm;
  int rank = 0, nranks = 1;
  // Krylov workspace cache: grown on demand, reused across solves (a PGMRES(30)
  // basis at E=64^3 is 44 GB -- allocating it per solve would dominate).
  std::vector<std::unique_ptr<cmg::DBuf>> ws;
  double* workspace(int slot, std::size_t n) {
    if (static_cast<int>(ws.size()) <= slot) ws.resize(slot + 1);
    if (!ws[slot]) ws[slot] = std::make_unique<cmg::DBuf>();
    if (ws[slot]->n < n) ws[slot]->alloc(n);
    return ws[slot]->p;
  }
  void sync() { CMG_CUDA(cudaStreamSynchronize(stream)); }
};

namespace cmg {
// view of a workspace slot with the DBuf interface used by the drivers
struct WBuf {
  double* p;
  std::size_t n;
  void zero(cudaStream_t s) {
    if (n) CMG_CUDA(cudaMemsetAsync(p, 0, n * sizeof(double), s));
  }
};
inline WBuf wsbuf(cmg_ctx* c, int slot, std::size_t n) { return WBuf{c->workspace(slot, n), n}; }
}  // namespace cmg

// LinearOperatorLike on device vectors (operators.hpp:19-26).  `n` is the
// number of unknowns (rows()), `len` the storage length of a device vector.
struct cmg_op {
  cmg_ctx* ctx = nullptr;
  std::size_t n = 0, len = 0;
  std::size_t count = 0;  // applications() counter, operators.hpp:56,63
  cmg::DBuf s_r, s_d, s_d2, s_t;  // smoother scratch (smoothers.hpp:103,131)
  virtual ~cmg_op() = default;

  void ensure_scratch() {
    if (s_r.n != len) {
      s_r.alloc(len); s_d.alloc(len); s_d2.alloc(len); s_t.alloc(len);
      s_r.zero(ctx->stream); s_d.zero(ctx->stream); s_d2.zero(ctx->stream); s_t.zero(ctx->stream);
    }
  }

  // y = A x ; counts one application
  virtual void apply(const double* x, double* y) = 0;
  // r = b - A x ; counts one application
  virtual void residual(const double* b, const double* x, double* r) {
    apply(x, r);
    cmg::launch_sub(len, b, r, r, ctx->stream);
  }
  virtual void diagonal(double* d) = 0;
  // Fused Chebyshev-Jacobi steps (smoothers.hpp:95-148).  Defaults compose
  // unfused kernels; FD and SEM operators override with one fused kernel.
  virtual void cheb4_init(const double* b, const double* x, bool x_is_zero, const double* invd,
                          double c0, double* r, double* d);
  // beta_last > 0 marks the LAST step of a sweep: the final x += beta_k d'
  // (smoothers.hpp:146-147 / :119) is fused in and r, d' are not written back.
  virtual void cheb4_step(double beta, double c1, double c2, bool x_zero, const double* invd,
                          const double* r_in, double* x, double* r, const double* d, double* d_out,
                          double beta_last = 0.0);
  virtual void cheb1_init(const double* b, const double* x, bool x_is_zero, const double* invd,
                          double theta, double* z, double* d);
  virtual void cheb1_step(double c1, double c2, bool x_zero, const double* invd, double* x,
                          double* z, const double* d, double* d_out, double beta_last = 0.0);
  // Inner products over the operator's vector space (distributed ops reduce
  // across ranks); results land in device memory.
  virtual void dot(const double* a, const double* b, double* out_dev) {
    cmg::launch_dot(a, b, len, ctx->dpart, out_dev, ctx->stream);
  }
  virtual void norm2(const double* a, double* out_dev) {
    cmg::launch_norm2(a, len, ctx->dpart, out_dev, ctx->stream);
  }
  virtual void mdot(const double* V, std::size_t ldv, int nv, const double* w, double* out_dev) {
    cmg::launch_mdot(V, ldv, nv, w, len, ctx->dpart, out_dev, ctx->stream);
  }
  // one CGS pass followed by the next pass's projections (krylov.hpp:186-195):
  // w -= V coef_in ; hcol += coef_in ; out = V^T w.  Same results as the
  // update and mdot issued separately; fused when nv <= kCgsFuseMax.
  virtual void cgs_mdot(const double* V, std::size_t ldv, int nv, const double* coef_in, double* w,
                        double* out_dev, double* hcol, int hstride) {
    if (nv <= cmg::kCgsFuseMax) {
      cmg::launch_cgs_mdot(V, ldv, nv, coef_in, w, len, hcol, hstride, ctx->dpart, out_dev, ctx->stream);
    } else {
      cmg::launch_cgs_update(V, ldv, nv, coef_in, w, len, hcol, hstride, ctx->stream);
      mdot(V, ldv, nv, w, out_dev);
    }
  }
  // set *flag if any unknown's entry of v is exactly zero (storage padding excluded)
  virtual void flag_zero_entries(const double* v, int* flag) {
    cmg::launch_any_zero(len, v, flag, ctx->stream);
  }
  // host canonical vector -> device storage layout (identity for FD)
  virtual void upload_canonical(const double* host, double* dev) {
    CMG_CUDA(cudaMemcpyAsync(dev, host, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  }
  virtual void download_canonical(const double* dev, double* host) {
    CMG_CUDA(cudaMemcpyAsync(host, dev, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
  }
};

struct cmg_precond {
  cmg_ctx* ctx = nullptr;
  virtual ~cmg_precond() = default;
  virtual void apply(const double* v, double* z) = 0;
  // true when M is not one fixed linear operator (an inner solve stopped by a
  // tolerance): PCG's theory then does not hold, only flexible-form PGMRES does
  virtual bool variable() const { return false; }
};

namespace cmg {
void set_last_error(const std::string& m);
// generic drivers (capi.cpp)
void chebyshev_smooth(cmg_op* A, const double* invd, const cmg_cheb_config& cfg,
                      std::size_t order, const double* b, double* x, bool x_is_zero);
double estimate_lambda_max(cmg_op* A, const double* invd, std::size_t iterations,
                           std::uint64_t seed);
void validate_cheb(const cmg_cheb_config& c);

// host setup (host_setup.cpp)
void host_random_vector(std::size_t n, std::uint64_t seed, double* out);
void host_fd_build_problem(std::size_t n, double Lx, double Ly, std::uint64_t seed, double* u,
                           double* b);
// FD coarse separable eigenbasis: S (mc x mc row-major, columns = eigenvectors,
// S^T M S = I) and lambda (mc) of K s = lambda M s, M = P1^T P1, K = P1^T T P1
void host_fd_coarse_eig(int n, int f, std::vector<double>& S, std::vector<double>& lam);
const double* host_beta_row(std::size_t k);  // nullptr outside 1..20
void host_gll(int N, double* xi, double* w);
void host_deriv_matrix(int N, const double* xi, double* D);
void host_interp_matrix(int Nf, int Nc, double* J);
// generalized symmetric eigenproblem A s = lam B s with B SPD (dense, n small)
void host_sym_geneig(int n, const double* A, const double* B, double* S, double* lam);
void host_node_coords(int geometry, double eps, const double* xi, int Ex, int Ey, int Ez, int ex, int ey,
                      int ez, int i, int j, int k, double* X, double* Y, double* Z);
void host_element_lengths(int geometry, double eps, int N, const double* xi, int Ex, int Ey, int Ez, int ex,
                          int ey, int ez, double* L);
void host_fdm_1d(int N, const double* w, const double* D, double Ll, double L, double Lr, int dl, int d0,
                 int dN, int dr, double* S, double* lam);
// Chebyshev smoothing / power iteration with a general smoother operator S
// (S(in, out): out = S in) -- the Schwarz path
using SApply = void (*)(void* ctx, const double* in, double* out);
// optional fused recurrence update (same arithmetic as S followed by the
// vector updates):  kind 4: d = c1 d + c2 S in ;  kind 1: x += d (x = d if x_zero),
// r -= S in, d = c1 d + c2 r
using SUpdate = void (*)(void* ctx, int kind, const double* in, double c1, double c2, double* d, double* r,
                         double* x, int x_zero);
void chebyshev_smooth_S(cmg_op* A, SApply S, void* sctx, const cmg_cheb_config& cfg, std::size_t order,
                        const double* b, double* x, bool x_is_zero, SUpdate U = nullptr);
double estimate_lambda_max_S(cmg_op* A, SApply S, void* sctx, std::size_t iterations, std::uint64_t seed);
}  // namespace cmg
