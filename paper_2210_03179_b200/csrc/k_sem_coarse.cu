// k_sem_coarse.cu -- dense direct solve of the p=1 coarse problem on a
// deformed mesh (the box mesh uses the separable FDM solve instead).
//
// The p=1 operator couples every vertex to its 27 lattice neighbours, so its
// entries are recovered from 27 matrix-free applications with "colour" probe
// vectors (vertex (ix,iy,iz) has colour (ix%3, iy%3, iz%3); two vertices of
// one colour are never neighbours).  The rows are scattered into a dense
// column-major matrix and factored once by Cholesky; the inverse is formed
// once, and every coarse solve is a pass of column dot products over the
// rank's slab of it (or, CMG_COARSE_INV=0, two triangular solves) -- exact,
// like the reference's banded Cholesky (cholesky.hpp:18-91), and deterministic.
#include <algorithm>

#include "sem_kernels.hpp"
#include "sem_layout.hpp"

namespace cmg {

namespace {

// p=1 slot layout: one owned vertex per element at slot 2*e (sem_nos(1) == 2);
// vertex (ex+1, ey+1, ez+1) is an unknown iff ex < nx, ey < ny, ez_global < nz
__global__ void k_probe(int Ex, int Ey, int Ezl, int z0, int nx, int ny, int nz, int cx, int cy, int cz,
                        double* __restrict__ v) {
  const long E = (long)Ex * Ey * Ezl;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < E; e += (long)gridDim.x * blockDim.x) {
    const int ex = (int)(e % Ex), ey = (int)((e / Ex) % Ey), ez = z0 + (int)(e / ((long)Ex * Ey));
    const bool on = ex < nx && ey < ny && ez < nz && ex % 3 == cx && ey % 3 == cy && ez % 3 == cz;
    v[2 * e] = on ? 1.0 : 0.0;
    v[2 * e + 1] = 0.0;
  }
}

__device__ __forceinline__ int probe_offset(int i, int c) {
  const int r = ((c - i % 3) % 3 + 3) % 3;
  return r == 0 ? 0 : (r == 1 ? 1 : -1);
}

// rows[(ex + nx*(ey + ny*lz))*27 + o] = A(i, i + offset_o) from the colour-c probe
__global__ void k_probe_extract(int Ex, int Ey, int Ezl, int z0, int nx, int ny, int nz, int cx, int cy, int cz,
                                const double* __restrict__ y, double* __restrict__ rows) {
  const long E = (long)Ex * Ey * Ezl;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < E; e += (long)gridDim.x * blockDim.x) {
    const int ex = (int)(e % Ex), ey = (int)((e / Ex) % Ey), lz = (int)(e / ((long)Ex * Ey));
    const int ez = z0 + lz;
    if (ex >= nx || ey >= ny || ez >= nz) continue;
    const int dx = probe_offset(ex, cx), dy = probe_offset(ey, cy), dz = probe_offset(ez, cz);
    const int o = (dx + 1) + 3 * ((dy + 1) + 3 * (dz + 1));
    rows[(ex + (long)nx * (ey + (long)ny * lz)) * 27 + o] = y[2 * e];
  }
}

// dense column-major A (n x n, n = nx*ny*nz) from the gathered 27-entry rows
__global__ void k_dense_build(int nx, int ny, int nz, const double* __restrict__ rows, double* __restrict__ A) {
  const long n = (long)nx * ny * nz;
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < n * 27; t += (long)gridDim.x * blockDim.x) {
    const long i = t / 27;
    const int o = (int)(t - i * 27);
    const int ix = (int)(i % nx), iy = (int)((i / nx) % ny), iz = (int)(i / ((long)nx * ny));
    const int jx = ix + o % 3 - 1, jy = iy + (o / 3) % 3 - 1, jz = iz + o / 9 - 1;
    if (jx < 0 || jx >= nx || jy < 0 || jy >= ny || jz < 0 || jz >= nz) continue;
    const long j = jx + (long)nx * (jy + (long)ny * jz);
    A[i + j * n] = rows[i * 27 + o];
  }
}

// dense vector (unknown order) <-> p=1 slot array over the full element grid
__global__ void k_slots_to_dense(int Ex, int Ey, int nx, int ny, int nz, const double* __restrict__ full,
                                 double* __restrict__ b) {
  const long n = (long)nx * ny * nz;
  for (long u = blockIdx.x * (long)blockDim.x + threadIdx.x; u < n; u += (long)gridDim.x * blockDim.x) {
    const int ix = (int)(u % nx), iy = (int)((u / nx) % ny), iz = (int)(u / ((long)nx * ny));
    b[u] = full[2 * (ix + (long)Ex * (iy + (long)Ey * iz))];
  }
}

__global__ void k_dense_to_slots(int Ex, int Ey, int Ezl, int z0, int nx, int ny, int nz,
                                 const double* __restrict__ x, double* __restrict__ ec) {
  const long E = (long)Ex * Ey * Ezl;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < E; e += (long)gridDim.x * blockDim.x) {
    const int ex = (int)(e % Ex), ey = (int)((e / Ex) % Ey), ez = z0 + (int)(e / ((long)Ex * Ey));
    const bool on = ex < nx && ey < ny && ez < nz;
    ec[2 * e] = on ? x[ex + (long)nx * (ey + (long)ny * ez)] : 0.0;
    ec[2 * e + 1] = 0.0;
  }
}

// lower triangle -> upper (potri leaves only the lower half of the symmetric
// inverse); 32x32 tiles through shared memory so both sides are coalesced
__global__ void k_symmetrize(long n, double* __restrict__ A) {
  __shared__ double T[32][33];
  const int bi = blockIdx.x, bj = blockIdx.y;  // tile (row block bi, column block bj), bi >= bj
  if (bi < bj) return;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (int c = ty; c < 32; c += 8) {
    const long i = (long)bi * 32 + tx, j = (long)bj * 32 + c;
    T[c][tx] = (i < n && j < n) ? A[i + j * n] : 0.0;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const long i = (long)bi * 32 + r, j = (long)bj * 32 + tx;  // write A[j, i] = A[i, j], i > j
    if (i < n && j < n && i > j) A[j + i * n] = T[tx][r];
  }
}

// y[c] = sum_k A[k, c] b[k] for the columns of a column slab: one block per
// column, fixed per-thread strides and a fixed reduction tree, so every y[c]
// is the same bits whichever slab (rank) computes it.  Eight independent
// loads in flight per thread (ncu: the 4-load, column-looping version sat at
// 67% of DRAM bandwidth on long-scoreboard stalls).
__global__ void __launch_bounds__(256) k_coldot(long n, const double* __restrict__ A, const double* __restrict__ b,
                                                double* __restrict__ y) {
  __shared__ double red[8];
  const long c = blockIdx.x;
  const double* col = A + c * n;
  double acc[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  long k = threadIdx.x;
  for (; k + 7 * 256 < n; k += 8 * 256) {
    double a[8], v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      a[u] = __ldcs(col + k + u * 256);  // streamed once: keep b in L2 instead
      v[u] = __ldg(b + k + u * 256);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] += a[u] * v[u];
  }
  for (; k < n; k += 256) acc[0] += col[k] * b[k];
  double v = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) y[c] = ((red[0] + red[1]) + (red[2] + red[3])) + ((red[4] + red[5]) + (red[6] + red[7]));
}

inline unsigned grid_for(long n) { return (unsigned)std::min<long>((n + 255) / 256, 148L * 16); }

}  // namespace

void coarse_symmetrize(long n, double* A, cudaStream_t s) {
  const unsigned t = (unsigned)((n + 31) / 32);
  k_symmetrize<<<dim3(t, t), dim3(32, 8), 0, s>>>(n, A);
  CMG_LAUNCH_CHECK();
}
void coarse_coldot(long n, long ncols, const double* A, const double* b, double* y, cudaStream_t s) {
  if (ncols <= 0) return;
  k_coldot<<<(unsigned)ncols, 256, 0, s>>>(n, A, b, y);
  CMG_LAUNCH_CHECK();
}

void coarse_probe(const CoarseGrid& g, int cx, int cy, int cz, double* v, cudaStream_t s) {
  k_probe<<<grid_for((long)g.Ex * g.Ey * g.Ezl), 256, 0, s>>>(g.Ex, g.Ey, g.Ezl, g.z0, g.nx, g.ny, g.nz, cx, cy, cz,
                                                               v);
  CMG_LAUNCH_CHECK();
}
void coarse_probe_extract(const CoarseGrid& g, int cx, int cy, int cz, const double* y, double* rows,
                          cudaStream_t s) {
  k_probe_extract<<<grid_for((long)g.Ex * g.Ey * g.Ezl), 256, 0, s>>>(g.Ex, g.Ey, g.Ezl, g.z0, g.nx, g.ny, g.nz,
                                                                       cx, cy, cz, y, rows);
  CMG_LAUNCH_CHECK();
}
void coarse_dense_build(const CoarseGrid& g, const double* rows, double* A, cudaStream_t s) {
  k_dense_build<<<grid_for((long)g.nx * g.ny * g.nz * 27), 256, 0, s>>>(g.nx, g.ny, g.nz, rows, A);
  CMG_LAUNCH_CHECK();
}
void coarse_slots_to_dense(const CoarseGrid& g, const double* full, double* b, cudaStream_t s) {
  k_slots_to_dense<<<grid_for((long)g.nx * g.ny * g.nz), 256, 0, s>>>(g.Ex, g.Ey, g.nx, g.ny, g.nz, full, b);
  CMG_LAUNCH_CHECK();
}
void coarse_dense_to_slots(const CoarseGrid& g, const double* x, double* ec, cudaStream_t s) {
  k_dense_to_slots<<<grid_for((long)g.Ex * g.Ey * g.Ezl), 256, 0, s>>>(g.Ex, g.Ey, g.Ezl, g.z0, g.nx, g.ny, g.nz,
                                                                        x, ec);
  CMG_LAUNCH_CHECK();
}

}  // namespace cmg
