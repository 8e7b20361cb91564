// cmg_internal.hpp -- shared declarations for the chebmg-b200 native library.
//
// Layering:
//   capi.cpp         extern "C" ABI (include/chebmg_b200.h) + host drivers
//                    (smoother / V-cycle / PCG / PGMRES control flow)
//   host_setup.cpp   setup-time host math (GLL, FDM eigenbases, RNG, RHS)
//   k_blas.cu        deterministic reductions, Krylov vector kernels
//   k_fd.cu          2D five-point FD kernels (fused stencil + Chebyshev)
//   k_sem.cu         SEM kernels (fused Ax + QQ^T + Chebyshev, transfers, FDM)
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace cmg {

// ---------------------------------------------------------------- errors
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
enum : int { OK = 0, EINVAL_ = 1, ERANGE_ = 2, ERUNTIME_ = 3, ECUDA_ = 4, ENCCL_ = 5 };

[[noreturn]] inline void throw_cuda(cudaError_t e, const char* what, const char* file, int line) {
  throw Error(ECUDA_, std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" +
                          std::to_string(line) + ")");
}
#define CMG_CUDA(x)                                              \
  do {                                                           \
    cudaError_t e_ = (x);                                        \
    if (e_ != cudaSuccess) ::cmg::throw_cuda(e_, #x, __FILE__, __LINE__); \
  } while (0)
// Every kernel launch wrapper reports through CMG_LAUNCH_CHECK (one per
// launched kernel) so cmg_ctx_kernel_launches() is an exact count.
extern std::atomic<unsigned long long> g_kernel_launches;
#define CMG_LAUNCH_CHECK()                 \
  do {                                     \
    ::cmg::g_kernel_launches.fetch_add(1, std::memory_order_relaxed); \
    CMG_CUDA(cudaGetLastError());          \
  } while (0)

// ---------------------------------------------------------------- reductions
// Deterministic two-stage reductions: a fixed grid of kRedBlocks blocks writes
// one partial per block (fixed intra-block tree), then a single block sums the
// partials in a fixed tree.  Same inputs -> same bits, run to run.
constexpr int kRedThreads = 256;
constexpr int kRedBlocks = 592;  // 4 x 148 SMs

// out[0] = sum_i a[i]*b[i]
void launch_dot(const double* a, const double* b, std::size_t n, double* partials, double* out,
                cudaStream_t s);
// out[l] = sum_i V[l*ldv + i] * w[i], l < nv  (CGS coefficients), partials >= nv*kRedBlocks
void launch_mdot(const double* V, std::size_t ldv, int nv, const double* w, std::size_t n,
                 double* partials, double* out, cudaStream_t s);
// out[0] = sqrt(sum a^2)
void launch_norm2(const double* a, std::size_t n, double* partials, double* out, cudaStream_t s);
// Finalise partial sums written by fused kernels: out[0] = sum(partials[0..np))
void launch_finalize(const double* partials, int np, double* out, int do_sqrt, cudaStream_t s);

// ---------------------------------------------------------------- vector ops
void launch_axpy(std::size_t n, double alpha, const double* x, double* y, cudaStream_t s);
// y += (*alpha_dev) * x   (sign = +1/-1 applied to alpha)
void launch_axpy_dev(std::size_t n, const double* alpha_dev, double sign, const double* x,
                     double* y, const int* stop_flag, cudaStream_t s);
void launch_scal_copy(std::size_t n, const double* inv_dev_or_null, double host_scale,
                      const double* x, double* y, cudaStream_t s);
void launch_sub(std::size_t n, const double* b, const double* t, double* r, cudaStream_t s);  // r=b-t
void launch_xpby_dev(std::size_t n, const double* z, const double* beta_dev, double* p,
                     const int* stop_flag, cudaStream_t s);  // p = z + beta p
void launch_set(std::size_t n, double v, double* x, cudaStream_t s);
void launch_recip(std::size_t n, const double* d, double* inv, int* zero_flag, cudaStream_t s);
void launch_mul(std::size_t n, const double* a, double* x, cudaStream_t s);  // x[i] *= a[i]
void launch_div_scalar_dev(std::size_t n, const double* x, const double* s_dev, double* y,
                           cudaStream_t s);  // y = x / *s
void launch_any_zero(std::size_t n, const double* d, int* flag, cudaStream_t s);
void launch_any_nonzero(std::size_t n, const double* d, int* flag, cudaStream_t s);
// out = c1 d + c2 s   (Chebyshev direction update with a general smoother)
void launch_lincomb(std::size_t n, double c1, const double* d, double c2, const double* s, double* out,
                    cudaStream_t st);

// ---------------------------------------------------------------- Krylov helpers
// CGS: w -= sum_l coef[l] V_l ; h[l*hstride] += coef[l]
void launch_cgs_update(const double* V, std::size_t ldv, int nv, const double* coef, double* w,
                       std::size_t n, double* hcol, int hstride, cudaStream_t s);
// fused CGS pass (nv <= kCgsFuseMax): w -= V coef_in, h += coef_in, out = V^T w_new;
// bit-identical to launch_cgs_update followed by launch_mdot
constexpr int kCgsFuseMax = 32;
void launch_cgs_mdot(const double* V, std::size_t ldv, int nv, const double* coef_in, double* w, std::size_t n,
                     double* hcol, int hstride, double* partials, double* out, cudaStream_t s);
// V_{j+1} = w / h  if h > 0  (krylov.hpp:197-200)
void launch_normalize_if_pos(std::size_t n, const double* w, const double* h, double* v,
                             cudaStream_t s);
// Givens least squares on a copy of H (krylov.hpp:203-227): one thread
std::size_t gmres_lsq_work(int m);  // doubles of global workspace for restart m
void launch_gmres_lsq(const double* H, int m, int j, double, const double* beta_dev, double* Hs, double* g,
                      double* y, double* gwork, cudaStream_t s);
// xj = x + sum_l y_l Z_l  (krylov.hpp:228-229)
void launch_form_iterate(const double* x, const double* Z, std::size_t ldz, int nz,
                         const double* y, double* xj, std::size_t n, cudaStream_t s);
// PCG scalar step: alpha = rz/pAp with breakdown flags (krylov.hpp:96-113)
void launch_pcg_alpha(const double* rz, const double* pAp, double* alpha, int* stop_flag,
                      cudaStream_t s);
void launch_pcg_beta(const double* rz_new, double* rz, double* beta, int* stop_flag,
                     cudaStream_t s);

// ---------------------------------------------------------------- FD kernels (k_fd.cu)
struct FdGrid {
  int m;           // interior points per dim (n-1)
  double ihx2, ihy2;
};
// y = A x
void fd_apply(const FdGrid& g, const double* x, double* y, cudaStream_t s);
// r = b - A x   (+ optional partials of r^2 for a fused norm)
void fd_residual(const FdGrid& g, const double* b, const double* x, double* r, double* partials,
                 cudaStream_t s);
// 4th-kind init: r = b - A x (or b when x_is_zero) ; d = c0 * invD * r
void fd_cheb4_init(const FdGrid& g, const double* b, const double* x, bool x_is_zero,
                   const double* invd, double c0, double* r, double* d, cudaStream_t s);
// one 4th-kind step: x += beta d ; r -= A d ; d_out = c1 d + c2 invD r
void fd_cheb4_step(const FdGrid& g, double beta, double c1, double c2, bool x_zero,
                   const double* invd, const double* r_in, double* x, double* r, const double* d,
                   double* d_out, double beta_last, cudaStream_t s);
// 1st-kind init: z = invD (b - A x) ; d = z / theta
void fd_cheb1_init(const FdGrid& g, const double* b, const double* x, bool x_is_zero,
                   const double* invd, double theta, double* z, double* d, cudaStream_t s);
// one 1st-kind step: x += d ; z -= invD A d ; d_out = c1 d + c2 z
void fd_cheb1_step(const FdGrid& g, double c1, double c2, bool x_zero, const double* invd,
                   double* x, double* z, const double* d, double* d_out, double beta_last,
                   cudaStream_t s);
// x += beta d  (or x = beta d when x_zero)
void vec_final_update(std::size_t n, double beta, bool x_zero, const double* d, double* x,
                      cudaStream_t s);
// rc = P^T r  (gather form)
void fd_restrict(int mf, int mc, int f, const double* r, double* rc, cudaStream_t s);
// x (+)= P ec
void fd_prolong(int mf, int mc, int f, const double* ec, double* x, bool assign, cudaStream_t s);
// fused: r = b - A x then rc = P^T r (r kept for nothing: computed on the fly)
// mode product along one dim of a (n0,n1,n2) array with strides (1,s1,s2):
//   out[..o..] = sum_m M[o*ld + m] (or M[m*ld + o] when transpose) * in[..m..]
void mode_product_s0(int dim, int n0, int n1, int n2, long s0, long s1, long s2, const double* M,
                     int ld, bool transpose, const double* in, double* out, const double* div,
                     cudaStream_t s);
void mode_product(int dim, int n0, int n1, int n2, long s1, long s2, const double* M, int ld,
                  bool transpose, const double* in, double* out, const double* div_or_null,
                  cudaStream_t s);

}  // namespace cmg
