// k_blas.cu -- deterministic reductions and Krylov vector kernels.
//
// Compiled with --fmad=false: the scalar Krylov kernels (Givens least
// squares, CGS updates, iterate formation) then round exactly like the
// reference's sequential C++ (krylov.hpp:144-264, no -march in its CMake),
// so the only difference from the reference is the summation ORDER of the
// inner products (fixed two-stage tree here, left-to-right there).
#include <cstdlib>
#include "cmg_internal.hpp"

namespace cmg {

namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// fixed-order block reduction; result valid in thread 0
__device__ __forceinline__ double block_sum(double v, double* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double r = 0.0;
  if (warp == 0) {
    r = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0.0;
    r = warp_sum(r);
  }
  __syncthreads();
  return r;
}

int red_grid(std::size_t n) {
  std::size_t g = (n + kRedThreads - 1) / kRedThreads;
  if (g < 1) g = 1;
  if (g > (std::size_t)kRedBlocks) g = kRedBlocks;
  return (int)g;
}

__global__ void k_dot_partials(const double* __restrict__ a, const double* __restrict__ b,
                               std::size_t n, double* __restrict__ partials) {
  __shared__ double sh[32];
  double s = 0.0;
  for (std::size_t i = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x; i < n;
       i += (std::size_t)gridDim.x * blockDim.x)
    s += a[i] * b[i];
  s = block_sum(s, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

__global__ void k_finalize(const double* __restrict__ partials, int np, double* out, int do_sqrt,
                           int nvec) {
  // block l reduces partials[l*np .. l*np+np)
  __shared__ double sh[32];
  const double* p = partials + (std::size_t)blockIdx.x * np;
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) s += p[i];
  s = block_sum(s, sh);
  if (threadIdx.x == 0) out[blockIdx.x] = do_sqrt ? sqrt(s) : s;
  (void)nvec;
}

template <int CH>
__global__ void k_mdot_partials(const double* __restrict__ V, std::size_t ldv, int nv, int l0,
                                const double* __restrict__ w, std::size_t n,
                                double* __restrict__ partials) {
  __shared__ double sh[CH][8];
  double acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = 0.0;
  const int cnt = min(CH, nv - l0);
  for (std::size_t i = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x; i < n;
       i += (std::size_t)gridDim.x * blockDim.x) {
    const double wi = w[i];
#pragma unroll
    for (int c = 0; c < CH; ++c)
      if (c < cnt) acc[c] += V[(std::size_t)(l0 + c) * ldv + i] * wi;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const double v = warp_sum(acc[c]);
    if (lane == 0) sh[c][warp] = v;
  }
  __syncthreads();
  if (threadIdx.x < cnt) {
    double s = 0.0;
    for (int wv = 0; wv < (int)(blockDim.x >> 5); ++wv) s += sh[threadIdx.x][wv];
    partials[(std::size_t)(l0 + threadIdx.x) * gridDim.x + blockIdx.x] = s;
  }
}

__global__ void k_axpy(std::size_t n, double alpha, const double* __restrict__ x,
                       double* __restrict__ y) {
  for (std::size_t i = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x; i < n;
       i += (std::size_t)gridDim.x * blockDim.x)
    y[i] += alpha * x[i];
}

__global__ void k_axpy_dev(std::size_t n, const double* alpha, double sign,
                           const double* __restrict__ x, double* __restrict__ y, const int* stop) {
  if (stop && *stop) return;
  const double a = sign * *alpha;
  for (std::size_t i = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x; i < n;
       i += (std::size_t)gridDim.x * blockDim.x)
    y[i] += a * x[i];
}

__global__ void k_scal_copy(std::size_t n, const double* inv_dev, double host_scale,
                            const double* __restrict__ x, double* __restrict__ y) {
  // y = x * (1 / *inv_dev)  or  y = x * host_scale     (core.hpp:49-51: x[i] *= alpha)
  const double a = inv_dev ? 1.0 / *inv_dev : host_scale;
  for (std::size_t i = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x; i < n;
       i += (std::size_t)gridDim.x * blockDim.x)
    y[i] = x[i] * a;
}

__global__ void k_sub(std::size_t n, const double* __restrict__ b, const double* __restrict__ t,
                      double* __restrict__ r) {
  for (std::size_t i = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x; i < n;
       i += (std::size_t)gridDim.x * blockDim.x)
    r[i] = b[i] - t[i];
}

__global__ void k_xpby(std::size_t n, const double* __restrict__ z, const double* beta,
                       double* __restrict__ p, const int* stop) {
  if (stop && *stop) return;
  const double bt = *beta;
  for (std::size_t i = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x; i < n;
       i += (std::size_t)gridDim.x * blockDim.x)
    p[i] = z[i] + bt * p[i];
}

__global__ void k_set(std::size_t n, double v, double* x) {
  for (std::size_t i = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x; i < n;
       i += (std::size_t)gridDim.x * blockDim.x)
    x[i] = v;
}

__global__ void k_recip(std::size_t n, const double* __restrict__ d, double* __restrict__ inv,
                        int* zero_flag) {
  for (std::size_t i = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x; i < n;
       i += (std::size_t)gridDim.x * blockDim.x) {
    const double v = d[i];
    if (v == 0.0 && zero_flag) atomicExch(zero_flag, 1);
    inv[i] = 1.0 / v;
  }
}

__global__ void k_mul(std::size_t n, const double* __restrict__ a, double* __restrict__ x) {
  for (std::size_t i = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x; i < n;
       i += (std::size_t)gridDim.x * blockDim.x)
    x[i] *= a[i];
}

__global__ void k_div_scalar(std::size_t n, const double* __restrict__ x, const double* s,
                             double* __restrict__ y) {
  const double d = *s;
  for (std::size_t i = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x; i < n;
       i += (std::size_t)gridDim.x * blockDim.x)
    y[i] = x[i] / d;
}

__global__ void k_any_zero(std::size_t n, const double* __restrict__ d, int* flag) {
  for (std::size_t i = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x; i < n;
       i += (std::size_t)gridDim.x * blockDim.x)
    if (d[i] == 0.0) atomicExch(flag, 1);
}

// w += sum_l (-coef[l]) V_l   in the reference's sequential axpy order
__global__ void k_cgs_update(const double* __restrict__ V, std::size_t ldv, int nv,
                             const double* __restrict__ coef, double* __restrict__ w, std::size_t n,
                             double* hcol, int hstride) {
  __shared__ double c[64];
  for (int l = threadIdx.x; l < nv; l += blockDim.x) c[l] = coef[l];
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0)
    for (int l = 0; l < nv; ++l) hcol[(std::size_t)l * hstride] += c[l];
  for (std::size_t i = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x; i < n;
       i += (std::size_t)gridDim.x * blockDim.x) {
    double v = w[i];
    for (int l = 0; l < nv; ++l) v += -c[l] * V[(std::size_t)l * ldv + i];
    w[i] = v;
  }
}

// Fused CGS pass: w -= V coef (k_cgs_update's arithmetic) and the partial
// sums of V^T w_new with k_mdot_partials' grid/block/reduction structure, so
// the coefficients are bit-identical to the unfused pair while V is streamed
// from HBM once instead of twice (the second read of each V_li hits cache).
template <int MAXV>
__global__ void __launch_bounds__(kRedThreads) k_cgs_mdot(const double* __restrict__ V, std::size_t ldv,
                                                          int nv, const double* __restrict__ coef,
                                                          double* __restrict__ w, std::size_t n, double* hcol,
                                                          int hstride, double* __restrict__ partials) {
  __shared__ double c[MAXV];
  __shared__ double sh[MAXV][kRedThreads / 32];
  for (int l = threadIdx.x; l < nv; l += blockDim.x) c[l] = coef[l];
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0)
    for (int l = 0; l < nv; ++l) hcol[(std::size_t)l * hstride] += c[l];
  double acc[MAXV];
#pragma unroll
  for (int q = 0; q < MAXV; ++q) acc[q] = 0.0;
  for (std::size_t i = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x; i < n;
       i += (std::size_t)gridDim.x * blockDim.x) {
    double v = w[i];
    if constexpr (MAXV <= 16) {  // the basis entries stay in registers for both uses
      double vv[MAXV];
#pragma unroll
      for (int q = 0; q < MAXV; ++q) vv[q] = q < nv ? V[(std::size_t)q * ldv + i] : 0.0;
#pragma unroll
      for (int q = 0; q < MAXV; ++q)
        if (q < nv) v += -c[q] * vv[q];
      w[i] = v;
#pragma unroll
      for (int q = 0; q < MAXV; ++q)
        if (q < nv) acc[q] += vv[q] * v;
    } else {
      for (int l = 0; l < nv; ++l) v += -c[l] * V[(std::size_t)l * ldv + i];
      w[i] = v;
#pragma unroll
      for (int q = 0; q < MAXV; ++q)
        if (q < nv) acc[q] += V[(std::size_t)q * ldv + i] * v;
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < MAXV; ++q) {
    if (q < nv) {
      const double s = warp_sum(acc[q]);
      if (lane == 0) sh[q][warp] = s;
    }
  }
  __syncthreads();
  if (threadIdx.x < nv) {
    double s = 0.0;
    for (int wv = 0; wv < (int)(blockDim.x >> 5); ++wv) s += sh[threadIdx.x][wv];
    partials[(std::size_t)threadIdx.x * gridDim.x + blockIdx.x] = s;
  }
}

__global__ void k_normalize_if_pos(std::size_t n, const double* __restrict__ w, const double* h,
                                   double* __restrict__ v) {
  const double hv = *h;
  if (!(hv > 0.0)) return;
  const double a = 1.0 / hv;
  for (std::size_t i = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x; i < n;
       i += (std::size_t)gridDim.x * blockDim.x)
    v[i] = w[i] * a;
}

// krylov.hpp:203-227, one thread, reference operation order
// One warp, H staged in shared memory; lane l owns columns l and l+32 of every
// rotation, so each entry sees exactly the reference's operations in the
// reference's order (krylov.hpp:203-227) -- only the schedule is parallel.
// Working copy in dynamic shared memory ((j+2)(j+1) + 2j + 3 doubles), or in
// `gwork` (global) when that exceeds the shared-memory opt-in (restart > ~165).
__global__ void k_gmres_lsq(const double* __restrict__ H, int m, int j, const double* beta,
                            double* Hs, double* g, double* y, double* gwork) {
  extern __shared__ double lsq_smem[];
  double* sh = gwork ? gwork : lsq_smem;
  double* sg = sh + (std::size_t)(j + 2) * (j + 1);
  double* sy = sg + (j + 2);
  const int lane = threadIdx.x;
  const int ld = j + 1;  // columns 0..j
  for (int i = lane; i < (j + 2) * ld; i += 32) sh[i] = H[(i / ld) * m + (i % ld)];
  for (int i = lane; i <= j + 1; i += 32) sg[i] = 0.0;
  __syncwarp();
  if (lane == 0) sg[0] = *beta;
  __syncwarp();
#define HS(i, jj) sh[(i) * ld + (jj)]
  for (int c = 0; c <= j; ++c) {
    for (int rr = c + 1; rr <= j + 1; ++rr) {
      const double a11 = HS(c, c), a21 = HS(rr, c);
      __syncwarp();
      if (a21 == 0.0) continue;  // warp-uniform
      const double den = sqrt(a11 * a11 + a21 * a21);
      const double cs = a11 / den, sn = a21 / den;
      for (int cc = c + lane; cc <= j; cc += 32) {
        const double t1 = HS(c, cc), t2 = HS(rr, cc);
        HS(c, cc) = cs * t1 + sn * t2;
        HS(rr, cc) = -sn * t1 + cs * t2;
      }
      if (lane == 0) {
        const double t1 = sg[c], t2 = sg[rr];
        sg[c] = cs * t1 + sn * t2;
        sg[rr] = -sn * t1 + cs * t2;
      }
      __syncwarp();
    }
  }
  if (lane == 0) {
    for (int bi = j; bi >= 0; --bi) {
      double s = sg[bi];
      for (int cc = bi + 1; cc <= j; ++cc) s -= HS(bi, cc) * sy[cc];
      sy[bi] = s / HS(bi, bi);
    }
  }
  __syncwarp();
  for (int i = lane; i <= j; i += 32) y[i] = sy[i];
  for (int i = lane; i <= m; i += 32) g[i] = i <= j + 1 ? sg[i] : 0.0;
  for (int i = lane; i < (m + 1) * m; i += 32) {
    const int r = i / m, cc = i % m;
    Hs[i] = (r <= j + 1 && cc <= j) ? HS(r, cc) : H[i];
  }
#undef HS
}

__global__ void k_form_iterate(const double* __restrict__ x, const double* __restrict__ Z,
                               std::size_t ldz, int nz, const double* __restrict__ y,
                               double* __restrict__ xj, std::size_t n) {
  __shared__ double c[64];
  for (int l = threadIdx.x; l < nz; l += blockDim.x) c[l] = y[l];
  __syncthreads();
  for (std::size_t i = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x; i < n;
       i += (std::size_t)gridDim.x * blockDim.x) {
    double v = x[i];
    for (int l = 0; l < nz; ++l) v += c[l] * Z[(std::size_t)l * ldz + i];
    xj[i] = v;
  }
}

__global__ void k_pcg_alpha(const double* rz, const double* pAp, double* alpha, int* stop) {
  if (*stop) return;
  if (*pAp <= 0.0) {
    *stop = 2;  // breakdown: <p, Ap> <= 0
    return;
  }
  *alpha = *rz / *pAp;
}

__global__ void k_pcg_beta(const double* rz_new, double* rz, double* beta, int* stop) {
  if (*stop) return;
  if (*rz_new <= 0.0) {
    *stop = 3;  // indefinite preconditioner
    return;
  }
  *beta = *rz_new / *rz;
  *rz = *rz_new;
}

inline int vgrid(std::size_t n) {
  std::size_t g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace

void launch_dot(const double* a, const double* b, std::size_t n, double* partials, double* out,
                cudaStream_t s) {
  const int g = red_grid(n);
  k_dot_partials<<<g, kRedThreads, 0, s>>>(a, b, n, partials);
  CMG_LAUNCH_CHECK();
  k_finalize<<<1, kRedThreads, 0, s>>>(partials, g, out, 0, 1);
  CMG_LAUNCH_CHECK();
}

void launch_norm2(const double* a, std::size_t n, double* partials, double* out, cudaStream_t s) {
  const int g = red_grid(n);
  k_dot_partials<<<g, kRedThreads, 0, s>>>(a, a, n, partials);
  CMG_LAUNCH_CHECK();
  k_finalize<<<1, kRedThreads, 0, s>>>(partials, g, out, 1, 1);
  CMG_LAUNCH_CHECK();
}

void launch_finalize(const double* partials, int np, double* out, int do_sqrt, cudaStream_t s) {
  k_finalize<<<1, kRedThreads, 0, s>>>(partials, np, out, do_sqrt, 1);
  CMG_LAUNCH_CHECK();
}

void launch_mdot(const double* V, std::size_t ldv, int nv, const double* w, std::size_t n,
                 double* partials, double* out, cudaStream_t s) {
  const int g = red_grid(n);
  for (int c0 = 0; c0 < nv; c0 += 64) {  // the partials buffer holds 64 vectors; each dot is independent
    const int nc = nv - c0 < 64 ? nv - c0 : 64;
    const double* Vc = V + (std::size_t)c0 * ldv;
    for (int l0 = 0; l0 < nc; l0 += 16) {
      k_mdot_partials<16><<<g, kRedThreads, 0, s>>>(Vc, ldv, nc, l0, w, n, partials);
      CMG_LAUNCH_CHECK();
    }
    k_finalize<<<nc, kRedThreads, 0, s>>>(partials, g, out + c0, 0, nc);
    CMG_LAUNCH_CHECK();
  }
}

void launch_axpy(std::size_t n, double alpha, const double* x, double* y, cudaStream_t s) {
  k_axpy<<<vgrid(n), 256, 0, s>>>(n, alpha, x, y);
  CMG_LAUNCH_CHECK();
}
void launch_axpy_dev(std::size_t n, const double* alpha_dev, double sign, const double* x,
                     double* y, const int* stop_flag, cudaStream_t s) {
  k_axpy_dev<<<vgrid(n), 256, 0, s>>>(n, alpha_dev, sign, x, y, stop_flag);
  CMG_LAUNCH_CHECK();
}
void launch_scal_copy(std::size_t n, const double* inv_dev, double host_scale, const double* x,
                      double* y, cudaStream_t s) {
  k_scal_copy<<<vgrid(n), 256, 0, s>>>(n, inv_dev, host_scale, x, y);
  CMG_LAUNCH_CHECK();
}
void launch_sub(std::size_t n, const double* b, const double* t, double* r, cudaStream_t s) {
  k_sub<<<vgrid(n), 256, 0, s>>>(n, b, t, r);
  CMG_LAUNCH_CHECK();
}
void launch_xpby_dev(std::size_t n, const double* z, const double* beta_dev, double* p,
                     const int* stop_flag, cudaStream_t s) {
  k_xpby<<<vgrid(n), 256, 0, s>>>(n, z, beta_dev, p, stop_flag);
  CMG_LAUNCH_CHECK();
}
void launch_set(std::size_t n, double v, double* x, cudaStream_t s) {
  k_set<<<vgrid(n), 256, 0, s>>>(n, v, x);
  CMG_LAUNCH_CHECK();
}
void launch_recip(std::size_t n, const double* d, double* inv, int* zero_flag, cudaStream_t s) {
  k_recip<<<vgrid(n), 256, 0, s>>>(n, d, inv, zero_flag);
  CMG_LAUNCH_CHECK();
}
void launch_mul(std::size_t n, const double* a, double* x, cudaStream_t s) {
  k_mul<<<vgrid(n), 256, 0, s>>>(n, a, x);
  CMG_LAUNCH_CHECK();
}
void launch_div_scalar_dev(std::size_t n, const double* x, const double* s_dev, double* y,
                           cudaStream_t s) {
  k_div_scalar<<<vgrid(n), 256, 0, s>>>(n, x, s_dev, y);
  CMG_LAUNCH_CHECK();
}
void launch_any_zero(std::size_t n, const double* d, int* flag, cudaStream_t s) {
  k_any_zero<<<vgrid(n), 256, 0, s>>>(n, d, flag);
  CMG_LAUNCH_CHECK();
}
namespace {
__global__ void k_lincomb(std::size_t n, double c1, const double* __restrict__ d, double c2,
                          const double* __restrict__ s, double* __restrict__ out) {
  for (std::size_t i = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x; i < n;
       i += (std::size_t)gridDim.x * blockDim.x)
    out[i] = c1 * d[i] + c2 * s[i];
}
}  // namespace
void launch_lincomb(std::size_t n, double c1, const double* d, double c2, const double* s, double* out,
                    cudaStream_t st) {
  k_lincomb<<<vgrid(n), 256, 0, st>>>(n, c1, d, c2, s, out);
  CMG_LAUNCH_CHECK();
}

namespace {
__global__ void k_any_nonzero(std::size_t n, const double* __restrict__ d, int* flag) {
  for (std::size_t i = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x; i < n;
       i += (std::size_t)gridDim.x * blockDim.x)
    if (d[i] != 0.0) atomicExch(flag, 1);
}
}  // namespace
void launch_any_nonzero(std::size_t n, const double* d, int* flag, cudaStream_t s) {
  k_any_nonzero<<<vgrid(n), 256, 0, s>>>(n, d, flag);
  CMG_LAUNCH_CHECK();
}

void launch_cgs_update(const double* V, std::size_t ldv, int nv, const double* coef, double* w,
                       std::size_t n, double* hcol, int hstride, cudaStream_t s) {
  for (int l0 = 0; l0 < nv; l0 += 64) {  // chunks continue each entry's sequential axpy order
    const int nc = nv - l0 < 64 ? nv - l0 : 64;
    k_cgs_update<<<vgrid(n), 256, 0, s>>>(V + (std::size_t)l0 * ldv, ldv, nc, coef + l0, w, n,
                                          hcol + (std::size_t)l0 * hstride, hstride);
    CMG_LAUNCH_CHECK();
  }
}
void launch_cgs_mdot(const double* V, std::size_t ldv, int nv, const double* coef, double* w, std::size_t n,
                    double* hcol, int hstride, double* partials, double* out, cudaStream_t s) {
  const int g = red_grid(n);
  if (nv <= 8) k_cgs_mdot<8><<<g, kRedThreads, 0, s>>>(V, ldv, nv, coef, w, n, hcol, hstride, partials);
  else if (nv <= 16) k_cgs_mdot<16><<<g, kRedThreads, 0, s>>>(V, ldv, nv, coef, w, n, hcol, hstride, partials);
  else k_cgs_mdot<32><<<g, kRedThreads, 0, s>>>(V, ldv, nv, coef, w, n, hcol, hstride, partials);
  CMG_LAUNCH_CHECK();
  k_finalize<<<nv, kRedThreads, 0, s>>>(partials, g, out, 0, nv);
  CMG_LAUNCH_CHECK();
}
void launch_normalize_if_pos(std::size_t n, const double* w, const double* h, double* v,
                             cudaStream_t s) {
  k_normalize_if_pos<<<vgrid(n), 256, 0, s>>>(n, w, h, v);
  CMG_LAUNCH_CHECK();
}
std::size_t gmres_lsq_work(int m) { return (std::size_t)(m + 1) * m + 2 * (std::size_t)m + 1; }

void launch_gmres_lsq(const double* H, int m, int j, double, const double* beta_dev, double* Hs,
                      double* g, double* y, double* gwork, cudaStream_t s) {
  static constexpr std::size_t kMaxSmem = 227 * 1024;
  static bool configured = false;
  // CMG_LSQ_SMEM_MAX (bytes, test knob): below it the working copy lives in shared memory
  static const std::size_t smem_max = [] {
    const char* env = std::getenv("CMG_LSQ_SMEM_MAX");
    return env ? std::min<std::size_t>(kMaxSmem, std::strtoull(env, nullptr, 10)) : kMaxSmem;
  }();
  if (!configured) {
    CMG_CUDA(cudaFuncSetAttribute(k_gmres_lsq, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxSmem));
    configured = true;
  }
  const std::size_t bytes = gmres_lsq_work(j + 1) * sizeof(double);
  if (bytes <= smem_max) k_gmres_lsq<<<1, 32, bytes, s>>>(H, m, j, beta_dev, Hs, g, y, nullptr);
  else k_gmres_lsq<<<1, 32, 0, s>>>(H, m, j, beta_dev, Hs, g, y, gwork);
  CMG_LAUNCH_CHECK();
}
// xj = x + sum_l y_l Z_l, per entry in ascending l; more than 64 columns run as
// consecutive chunks continuing from the stored partial sum (same operations,
// same order, same bits)
void launch_form_iterate(const double* x, const double* Z, std::size_t ldz, int nz,
                         const double* y, double* xj, std::size_t n, cudaStream_t s) {
  for (int l0 = 0; l0 < nz || l0 == 0; l0 += 64) {
    const int nc = nz - l0 < 64 ? nz - l0 : 64;
    k_form_iterate<<<vgrid(n), 256, 0, s>>>(l0 == 0 ? x : xj, Z + (std::size_t)l0 * ldz, ldz, nc, y + l0, xj, n);
    CMG_LAUNCH_CHECK();
  }
}
void launch_pcg_alpha(const double* rz, const double* pAp, double* alpha, int* stop_flag,
                      cudaStream_t s) {
  k_pcg_alpha<<<1, 1, 0, s>>>(rz, pAp, alpha, stop_flag);
  CMG_LAUNCH_CHECK();
}
void launch_pcg_beta(const double* rz_new, double* rz, double* beta, int* stop_flag,
                     cudaStream_t s) {
  k_pcg_beta<<<1, 1, 0, s>>>(rz_new, rz, beta, stop_flag);
  CMG_LAUNCH_CHECK();
}

}  // namespace cmg
