// k_fd.cu -- 2D five-point finite-difference kernels (sm_100a).
//
// Every Chebyshev step is ONE kernel: the stencil apply of the search
// direction is fused with the recurrence (x, r, d updated in one pass,
// 48 B/DOF of algorithmic HBM traffic -- DESIGN.md §4.1).
//
// Compiled with --fmad=false and written in the reference's operand order
// (operators.hpp:43-57, smoothers.hpp:95-148, transfer.hpp:61-88) so the
// smoother sweep and the transfers are bit-identical to the reference CPU
// path; tests/test_fd_gpu.py checks that with exact equality.
#include "cmg_internal.hpp"

namespace cmg {

namespace {

constexpr int BX = 32, BY = 8;

__device__ __forceinline__ double stencil(const double* __restrict__ x, int ix, int iy, int m,
                                          double c, double ihx2, double ihy2) {
  const long id = (long)iy * m + ix;
  double v = c * x[id];
  if (ix > 0) v -= ihx2 * x[id - 1];
  if (ix + 1 < m) v -= ihx2 * x[id + 1];
  if (iy > 0) v -= ihy2 * x[id - m];
  if (iy + 1 < m) v -= ihy2 * x[id + m];
  return v;
}

__global__ void k_fd_apply(int m, double ihx2, double ihy2, const double* __restrict__ x,
                           double* __restrict__ y) {
  const int ix = blockIdx.x * BX + threadIdx.x, iy = blockIdx.y * BY + threadIdx.y;
  if (ix >= m || iy >= m) return;
  const double c = 2.0 * (ihx2 + ihy2);
  y[(long)iy * m + ix] = stencil(x, ix, iy, m, c, ihx2, ihy2);
}

// r = b - A x ; optional per-block partials of r^2 (deterministic block order)
__global__ void k_fd_residual(int m, double ihx2, double ihy2, const double* __restrict__ b,
                              const double* __restrict__ x, double* __restrict__ r,
                              double* __restrict__ partials) {
  const int ix = blockIdx.x * BX + threadIdx.x, iy = blockIdx.y * BY + threadIdx.y;
  double rv = 0.0;
  if (ix < m && iy < m) {
    const double c = 2.0 * (ihx2 + ihy2);
    const long id = (long)iy * m + ix;
    rv = b[id] - stencil(x, ix, iy, m, c, ihx2, ihy2);
    r[id] = rv;
  }
  if (partials) {
    __shared__ double sh[BX * BY];
    const int t = threadIdx.y * BX + threadIdx.x;
    sh[t] = rv * rv;
    __syncthreads();
    for (int s = BX * BY / 2; s > 0; s >>= 1) {
      if (t < s) sh[t] += sh[t + s];
      __syncthreads();
    }
    if (t == 0) partials[blockIdx.y * gridDim.x + blockIdx.x] = sh[0];
  }
}

// smoothers.hpp:83-91 + :133-134
__global__ void k_fd_cheb4_init(int m, double ihx2, double ihy2, const double* __restrict__ b,
                                const double* __restrict__ x, int x_is_zero,
                                const double* __restrict__ invd, double c0, double* __restrict__ r,
                                double* __restrict__ d) {
  const int ix = blockIdx.x * BX + threadIdx.x, iy = blockIdx.y * BY + threadIdx.y;
  if (ix >= m || iy >= m) return;
  const long id = (long)iy * m + ix;
  const double c = 2.0 * (ihx2 + ihy2);
  const double rv = x_is_zero ? b[id] : b[id] - stencil(x, ix, iy, m, c, ihx2, ihy2);
  r[id] = rv;
  d[id] = c0 * invd[id] * rv;
}

// smoothers.hpp:136-145, one fused pass per step
__global__ void k_fd_cheb4_step(int m, double ihx2, double ihy2, double beta, double c1, double c2,
                                int x_zero, const double* __restrict__ invd,
                                const double* __restrict__ r_in, double* __restrict__ x,
                                double* __restrict__ r, const double* __restrict__ d,
                                double* __restrict__ d_out, double beta_last) {
  const int ix = blockIdx.x * BX + threadIdx.x, iy = blockIdx.y * BY + threadIdx.y;
  if (ix >= m || iy >= m) return;
  const long id = (long)iy * m + ix;
  const double c = 2.0 * (ihx2 + ihy2);
  const double dv = d[id];
  const double xv = x_zero ? beta * dv : x[id] + beta * dv;
  const double t = stencil(d, ix, iy, m, c, ihx2, ihy2);
  const double rv = r_in[id] + -1.0 * t;
  const double dn = c1 * dv + c2 * invd[id] * rv;
  if (beta_last > 0.0) {  // last step: fused final x += beta_k d (smoothers.hpp:146-147)
    x[id] = xv + beta_last * dn;
  } else {
    x[id] = xv;
    r[id] = rv;
    d_out[id] = dn;
  }
}

// smoothers.hpp:104-107
__global__ void k_fd_cheb1_init(int m, double ihx2, double ihy2, const double* __restrict__ b,
                                const double* __restrict__ x, int x_is_zero,
                                const double* __restrict__ invd, double theta,
                                double* __restrict__ z, double* __restrict__ d) {
  const int ix = blockIdx.x * BX + threadIdx.x, iy = blockIdx.y * BY + threadIdx.y;
  if (ix >= m || iy >= m) return;
  const long id = (long)iy * m + ix;
  const double c = 2.0 * (ihx2 + ihy2);
  double zv = x_is_zero ? b[id] : b[id] - stencil(x, ix, iy, m, c, ihx2, ihy2);
  zv *= invd[id];
  z[id] = zv;
  d[id] = zv / theta;
}

// smoothers.hpp:109-118
__global__ void k_fd_cheb1_step(int m, double ihx2, double ihy2, double c1, double c2, int x_zero,
                                const double* __restrict__ invd, double* __restrict__ x,
                                double* __restrict__ z, const double* __restrict__ d,
                                double* __restrict__ d_out, double beta_last) {
  const int ix = blockIdx.x * BX + threadIdx.x, iy = blockIdx.y * BY + threadIdx.y;
  if (ix >= m || iy >= m) return;
  const long id = (long)iy * m + ix;
  const double c = 2.0 * (ihx2 + ihy2);
  const double dv = d[id];
  const double xv = x_zero ? 1.0 * dv : x[id] + 1.0 * dv;
  const double t = stencil(d, ix, iy, m, c, ihx2, ihy2);
  const double zv = z[id] - invd[id] * t;
  const double dn = c1 * dv + c2 * zv;
  if (beta_last > 0.0) {  // last step: fused final x += d (smoothers.hpp:119)
    x[id] = xv + beta_last * dn;
  } else {
    x[id] = xv;
    z[id] = zv;
    d_out[id] = dn;
  }
}

__global__ void k_final_update(std::size_t n, double beta, int x_zero, const double* __restrict__ d,
                               double* __restrict__ x) {
  for (std::size_t i = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x; i < n;
       i += (std::size_t)gridDim.x * blockDim.x)
    x[i] = x_zero ? beta * d[i] : x[i] + beta * d[i];
}

// interp_1d weight of coarse interior node cj (1-based) at fine node i (1-based), transfer.hpp:20-46
__device__ __forceinline__ double w1d(int i, int cj, int f) {
  const int j0 = i / f;
  const double t = (double)(i % f) / (double)f;
  if (j0 == cj) return 1.0 - t;
  if (j0 + 1 == cj && t > 0.0) return t;
  return 0.0;
}

// P^T in gather form, summing in the reference's fine row-major scatter order
__global__ void k_fd_restrict(int mf, int mc, int f, const double* __restrict__ r,
                              double* __restrict__ rc) {
  const int cx = blockIdx.x * blockDim.x + threadIdx.x, cy = blockIdx.y;
  if (cx >= mc || cy >= mc) return;
  const int cjx = cx + 1, cjy = cy + 1;
  double s = 0.0;
  for (int gy = cjy * f - f + 1; gy <= cjy * f + f - 1; ++gy) {
    if (gy < 1 || gy > mf) continue;
    const double wy = w1d(gy, cjy, f);
    for (int gx = cjx * f - f + 1; gx <= cjx * f + f - 1; ++gx) {
      if (gx < 1 || gx > mf) continue;
      const double wx = w1d(gx, cjx, f);
      s += wy * wx * r[(long)(gy - 1) * mf + (gx - 1)];
    }
  }
  rc[(long)cy * mc + cx] = s;
}

// x (+)= P ec   (transfer.hpp:61-71 ; multigrid.hpp:83-87)
__global__ void k_fd_prolong(int mf, int mc, int f, const double* __restrict__ ec,
                             double* __restrict__ x, int assign) {
  const int ix = blockIdx.x * BX + threadIdx.x, iy = blockIdx.y * BY + threadIdx.y;
  if (ix >= mf || iy >= mf) return;
  const int gx = ix + 1, gy = iy + 1;
  int cyi[2], cxi[2];
  double wy[2], wx[2];
  int ny = 0, nx = 0;
  {
    const int j0 = gy / f;
    const double t = (double)(gy % f) / (double)f;
    if (j0 >= 1 && j0 <= mc) { cyi[ny] = j0 - 1; wy[ny] = 1.0 - t; if (wy[ny] != 0.0) ++ny; }
    if (j0 + 1 <= mc && t > 0.0) { cyi[ny] = j0; wy[ny] = t; ++ny; }
  }
  {
    const int j0 = gx / f;
    const double t = (double)(gx % f) / (double)f;
    if (j0 >= 1 && j0 <= mc) { cxi[nx] = j0 - 1; wx[nx] = 1.0 - t; if (wx[nx] != 0.0) ++nx; }
    if (j0 + 1 <= mc && t > 0.0) { cxi[nx] = j0; wx[nx] = t; ++nx; }
  }
  double s = 0.0;
  for (int a = 0; a < ny; ++a)
    for (int b = 0; b < nx; ++b) s += wy[a] * wx[b] * ec[(long)cyi[a] * mc + cxi[b]];
  const long id = (long)iy * mf + ix;
  x[id] = assign ? s : x[id] + 1.0 * s;
}

// Strided small-GEMM "mode product": contract dimension `dim` of a 3D array.
// out[o, r] = sum_m Mop(o, m) in[m, r]; Mop = M (row-major, ld) or M^T.
// 16x16 output tile per 256-thread block (one output per thread, 64 blocks at
// the n=256 coarse grid), k in tiles of TK (64 or 128, one staging round for
// every coarse grid up to 128) accumulated in ascending order.
// Loads and stores walk whichever of (k, r) is unit-stride so both stay
// coalesced for every contracted dimension.
constexpr int TM = 16, TR = 16;
template <int TK>
__global__ void __launch_bounds__(256) k_mode_product(int nd, int na, int nb, long sd, long sa, long sb,
                                                      const double* __restrict__ M, int ld, int transpose,
                                                      const double* __restrict__ in, double* __restrict__ out,
                                                      const double* __restrict__ div) {
  __shared__ double Ms[TM][TK + 1];
  __shared__ double Bs[TK][TR + 1];
  const int o0 = blockIdx.y * TM, r0 = blockIdx.x * TR;
  const int R = na * nb;
  const bool kfast = sd == 1;  // contracted dimension is the unit-stride one
  const int t = threadIdx.x;
  const int oo = kfast ? t % TM : t / TR, ro = kfast ? t / TM : t % TR;
  double acc = 0.0;
  for (int k0 = 0; k0 < nd; k0 += TK) {
    // All global loads of the stage are issued before any shared store: the
    // launch is load-latency bound (one dependent load->store pair per
    // element serialised ~16 DRAM round trips).
    constexpr int LM = TM * TK / 256, LB = TK * TR / 256;
    double vm[LM], vb[LB];
#pragma unroll
    for (int i = 0; i < LM; ++i) {
      const int e = t + i * 256;
      const int mo = transpose ? e % TM : e / TK, mk = transpose ? e / TM : e % TK;
      const int o = o0 + mo, k = k0 + mk;
      vm[i] = (o < nd && k < nd) ? (transpose ? M[(long)k * ld + o] : M[(long)o * ld + k]) : 0.0;
    }
#pragma unroll
    for (int i = 0; i < LB; ++i) {
      const int e = t + i * 256;
      const int kk = kfast ? e % TK : e / TR, rr = kfast ? e / TK : e % TR;
      const int k = k0 + kk, r = r0 + rr;
      vb[i] = (k < nd && r < R) ? in[(long)k * sd + (long)(r % na) * sa + (long)(r / na) * sb] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < LM; ++i) {
      const int e = t + i * 256;
      Ms[transpose ? e % TM : e / TK][transpose ? e / TM : e % TK] = vm[i];
    }
#pragma unroll
    for (int i = 0; i < LB; ++i) {
      const int e = t + i * 256;
      Bs[kfast ? e % TK : e / TR][kfast ? e / TK : e % TR] = vb[i];
    }
    __syncthreads();
    const int kn = min(TK, nd - k0);
#pragma unroll 8
    for (int kk = 0; kk < kn; ++kk) acc += Ms[oo][kk] * Bs[kk][ro];
    __syncthreads();
  }
  const int o = o0 + oo, r = r0 + ro;
  if (o >= nd || r >= R) return;
  const long idx = (long)o * sd + (long)(r % na) * sa + (long)(r / na) * sb;
  out[idx] = div ? acc / div[idx] : acc;
}

inline dim3 grid2d(int m) { return dim3((m + BX - 1) / BX, (m + BY - 1) / BY); }

}  // namespace

void fd_apply(const FdGrid& g, const double* x, double* y, cudaStream_t s) {
  k_fd_apply<<<grid2d(g.m), dim3(BX, BY), 0, s>>>(g.m, g.ihx2, g.ihy2, x, y);
  CMG_LAUNCH_CHECK();
}

void fd_residual(const FdGrid& g, const double* b, const double* x, double* r, double* partials,
                 cudaStream_t s) {
  k_fd_residual<<<grid2d(g.m), dim3(BX, BY), 0, s>>>(g.m, g.ihx2, g.ihy2, b, x, r, partials);
  CMG_LAUNCH_CHECK();
}

int fd_residual_partials(const FdGrid& g) {
  const dim3 gr = grid2d(g.m);
  return (int)(gr.x * gr.y);
}

void fd_cheb4_init(const FdGrid& g, const double* b, const double* x, bool x_is_zero,
                   const double* invd, double c0, double* r, double* d, cudaStream_t s) {
  k_fd_cheb4_init<<<grid2d(g.m), dim3(BX, BY), 0, s>>>(g.m, g.ihx2, g.ihy2, b, x, x_is_zero, invd,
                                                       c0, r, d);
  CMG_LAUNCH_CHECK();
}

void fd_cheb4_step(const FdGrid& g, double beta, double c1, double c2, bool x_zero,
                   const double* invd, const double* r_in, double* x, double* r, const double* d,
                   double* d_out, double beta_last, cudaStream_t s) {
  k_fd_cheb4_step<<<grid2d(g.m), dim3(BX, BY), 0, s>>>(g.m, g.ihx2, g.ihy2, beta, c1, c2, x_zero,
                                                       invd, r_in, x, r, d, d_out, beta_last);
  CMG_LAUNCH_CHECK();
}

void fd_cheb1_init(const FdGrid& g, const double* b, const double* x, bool x_is_zero,
                   const double* invd, double theta, double* z, double* d, cudaStream_t s) {
  k_fd_cheb1_init<<<grid2d(g.m), dim3(BX, BY), 0, s>>>(g.m, g.ihx2, g.ihy2, b, x, x_is_zero, invd,
                                                       theta, z, d);
  CMG_LAUNCH_CHECK();
}

void fd_cheb1_step(const FdGrid& g, double c1, double c2, bool x_zero, const double* invd,
                   double* x, double* z, const double* d, double* d_out, double beta_last,
                   cudaStream_t s) {
  k_fd_cheb1_step<<<grid2d(g.m), dim3(BX, BY), 0, s>>>(g.m, g.ihx2, g.ihy2, c1, c2, x_zero, invd,
                                                       x, z, d, d_out, beta_last);
  CMG_LAUNCH_CHECK();
}

void vec_final_update(std::size_t n, double beta, bool x_zero, const double* d, double* x,
                      cudaStream_t s) {
  std::size_t g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  k_final_update<<<(int)g, 256, 0, s>>>(n, beta, x_zero, d, x);
  CMG_LAUNCH_CHECK();
}

void fd_restrict(int mf, int mc, int f, const double* r, double* rc, cudaStream_t s) {
  k_fd_restrict<<<dim3((mc + 63) / 64, mc), 64, 0, s>>>(mf, mc, f, r, rc);
  CMG_LAUNCH_CHECK();
}

void fd_prolong(int mf, int mc, int f, const double* ec, double* x, bool assign, cudaStream_t s) {
  k_fd_prolong<<<grid2d(mf), dim3(BX, BY), 0, s>>>(mf, mc, f, ec, x, assign);
  CMG_LAUNCH_CHECK();
}

void mode_product(int dim, int n0, int n1, int n2, long s1, long s2, const double* M, int ld,
                  bool transpose, const double* in, double* out, const double* div,
                  cudaStream_t s) {
  mode_product_s0(dim, n0, n1, n2, 1, s1, s2, M, ld, transpose, in, out, div, s);
}

void mode_product_s0(int dim, int n0, int n1, int n2, long s0, long s1, long s2, const double* M, int ld,
                     bool transpose, const double* in, double* out, const double* div, cudaStream_t s) {
  const int n[3] = {n0, n1, n2};
  const long st[3] = {s0, s1, s2};
  const int a = dim == 0 ? 1 : 0, b = dim == 2 ? 1 : 2;
  const int nd = n[dim];
  const int R = n[a] * n[b];
  dim3 grid((R + TR - 1) / TR, (nd + TM - 1) / TM);
  if (nd <= 64)  // the SEM p=1 boxes: half the staging footprint, more resident blocks
    k_mode_product<64><<<grid, 256, 0, s>>>(nd, n[a], n[b], st[dim], st[a], st[b], M, ld, transpose,
                                            in, out, div);
  else
    k_mode_product<128><<<grid, 256, 0, s>>>(nd, n[a], n[b], st[dim], st[a], st[b], M, ld, transpose,
                                             in, out, div);
  CMG_LAUNCH_CHECK();
}

}  // namespace cmg
