// k_schwarz.cu -- Chebyshev-Schwarz smoother kernels (PAPER.md:560-629,
// SURVEY App. A8): overlapping (N+3)^3 extended-element subdomains solved
// exactly by fast diagonalisation, combined additively (ASM, post-weighted)
// or restrictively (RAS).  The definition matches oracle/oracle_schwarz.c.
#include "sem_kernels.hpp"
#include "sem_layout.hpp"

namespace cmg {

namespace {

template <int N>
__device__ __forceinline__ int owner1d_s(int g, int ne, int& oe) {
  if (g <= 0 || g >= N * ne) return -1;
  oe = (g - 1) / N;
  return (g - 1) - oe * N;
}

// one block per element: gather r on the extended box, FDM solve, write the
// local solution (RAS: the element's own (N+1)^3 nodes; ASM: all (N+3)^3).
// Each mode product is a set of line contractions: a thread loads one
// (N+3)-line of the box into registers once and produces the whole output
// line, with the 1D eigenbasis rows broadcast from shared memory (every
// output still sums its N+3 terms in ascending order).
template <int N>
__global__ void __launch_bounds__(128) k_schwarz_local(SchwarzArgs A) {
  constexpr int PB = N + 3, PB2 = PB * PB, PB3 = PB2 * PB, N1 = N + 1, NOS = sem_nos(N);
  __shared__ double u[PB3], t[PB3];
  __shared__ double S[3][PB2], lam[3][PB];
  const long e = blockIdx.x;
  const int ex = (int)(e % A.Ex), ey = (int)((e / A.Ex) % A.Ey), ez = (int)(e / ((long)A.Ex * A.Ey));
  for (int d = 0; d < 3; ++d) {
    const int id = A.sidx[e * 3 + d];
    for (int q = threadIdx.x; q < PB2; q += blockDim.x) S[d][q] = A.S[(long)id * PB2 + q];
    for (int q = threadIdx.x; q < PB; q += blockDim.x) lam[d][q] = A.lam[(long)id * PB + q];
  }
  for (int q = threadIdx.x; q < PB3; q += blockDim.x) {
    const int a = q % PB, b = (q / PB) % PB, c = q / PB2;
    int oex = 0, oey = 0, oez = 0;
    const int ax = owner1d_s<N>(ex * N + a - 1, A.Ex, oex);
    const int ay = owner1d_s<N>(ey * N + b - 1, A.Ey, oey);
    const int az = owner1d_s<N>(ez * N + c - 1, A.Ez, oez);
    double v = 0.0;
    if (ax >= 0 && ay >= 0 && az >= 0)
      v = A.r[((long)oex + (long)A.Ex * ((long)oey + (long)A.Ey * oez)) * NOS + sem_pos(N, ax, ay, az)];
    u[q] = v;
  }
  __syncthreads();
  // line l of dimension dim: the other two indices (p, q) = (l % PB, l / PB)
  auto line_base = [](int dim, int l) {
    const int p = l % PB, q = l / PB;
    return dim == 0 ? PB * (p + PB * q) : (dim == 1 ? p + PB2 * q : p + PB * q);
  };
  constexpr int STRIDE[3] = {1, PB, PB2};
  // forward: (Sz^T x Sy^T x Sx^T) u; the eigenvalue division fused into the last pass
  double* in = u;
  double* out = t;
#pragma unroll 1
  for (int dim = 0; dim < 3; ++dim) {
    for (int l = threadIdx.x; l < PB2; l += blockDim.x) {
      const int base = line_base(dim, l), st = STRIDE[dim];
      double v[PB];
#pragma unroll
      for (int m = 0; m < PB; ++m) v[m] = in[base + m * st];
#pragma unroll 2
      for (int o = 0; o < PB; ++o) {
        double acc = 0.0;
#pragma unroll
        for (int m = 0; m < PB; ++m) acc += S[dim][m * PB + o] * v[m];
        const int q = base + o * st;
        if (dim == 2) {
          const int a = q % PB, b = (q / PB) % PB, c = q / PB2;
          acc /= (lam[0][a] + lam[1][b] + lam[2][c]);
        }
        out[q] = acc;
      }
    }
    __syncthreads();
    double* tmp = in;
    in = out;
    out = tmp;
  }
  // backward: (Sz x Sy x Sx)
#pragma unroll 1
  for (int dim = 0; dim < 3; ++dim) {
    for (int l = threadIdx.x; l < PB2; l += blockDim.x) {
      const int base = line_base(dim, l), st = STRIDE[dim];
      double v[PB];
#pragma unroll
      for (int m = 0; m < PB; ++m) v[m] = in[base + m * st];
#pragma unroll 2
      for (int o = 0; o < PB; ++o) {
        double acc = 0.0;
#pragma unroll
        for (int m = 0; m < PB; ++m) acc += S[dim][o * PB + m] * v[m];
        out[base + o * st] = acc;
      }
    }
    __syncthreads();
    double* tmp = in;
    in = out;
    out = tmp;
  }
  if (A.ras) {
    for (int q = threadIdx.x; q < N1 * N1 * N1; q += blockDim.x) {
      const int i = q % N1, j = (q / N1) % N1, k = q / (N1 * N1);
      A.Lout[e * (N1 * N1 * N1) + q] = in[(i + 1) + PB * ((j + 1) + PB * (k + 1))];
    }
  } else {
    for (int q = threadIdx.x; q < PB3; q += blockDim.x) A.Lout[e * PB3 + q] = in[q];
  }
}

// ASM: every owned slot sums the extended local solutions covering it (fixed
// ascending-element order, oracle_schwarz.c) and applies W = 1/count
template <int N>
__global__ void k_asm_gather(SchwarzArgs A, double* __restrict__ y) {
  constexpr int PB = N + 3, PB3 = PB * PB * PB, NOS = sem_nos(N);
  const long n = (long)A.Ex * A.Ey * A.Ez * NOS;
  for (long q = blockIdx.x * (long)blockDim.x + threadIdx.x; q < n; q += (long)gridDim.x * blockDim.x) {
    const long e = q / NOS;
    int a, b, c;
    if (!sem_abc(N, (int)(q - e * NOS), a, b, c)) {
      y[q] = 0.0;
      continue;
    }
    const int ex = (int)(e % A.Ex), ey = (int)((e / A.Ex) % A.Ey), ez = (int)(e / ((long)A.Ex * A.Ey));
    const int gx = ex * N + a + 1, gy = ey * N + b + 1, gz = ez * N + c + 1;
    if (gx >= N * A.Ex || gy >= N * A.Ey || gz >= N * A.Ez) {
      y[q] = 0.0;
      continue;
    }
    double acc = 0.0;
    int cnt = 0;
    // candidate elements along each dim: e' with e'N - 1 <= g <= e'N + N + 1
    for (int cz = gz / N - 2; cz <= gz / N + 1; ++cz) {
      if (cz < 0 || cz >= A.Ez || !(cz * N - 1 <= gz && gz <= cz * N + N + 1)) continue;
      for (int cy = gy / N - 2; cy <= gy / N + 1; ++cy) {
        if (cy < 0 || cy >= A.Ey || !(cy * N - 1 <= gy && gy <= cy * N + N + 1)) continue;
        for (int cx = gx / N - 2; cx <= gx / N + 1; ++cx) {
          if (cx < 0 || cx >= A.Ex || !(cx * N - 1 <= gx && gx <= cx * N + N + 1)) continue;
          const long e2 = cx + (long)A.Ex * (cy + (long)A.Ey * cz);
          const int la = gx - cx * N + 1, lb = gy - cy * N + 1, lc = gz - cz * N + 1;
          acc += A.Lout[e2 * PB3 + la + PB * (lb + PB * lc)];
          ++cnt;
        }
      }
    }
    y[q] = acc * (1.0 / (double)cnt);
  }
}

}  // namespace

void sem_schwarz_local(const SchwarzArgs& a, cudaStream_t s) {
  const long E = (long)a.Ex * a.Ey * a.Ez;
#define X(n) \
  if (a.N == n) { k_schwarz_local<n><<<(unsigned)E, 128, 0, s>>>(a); CMG_LAUNCH_CHECK(); return; }
  X(2) X(3) X(4) X(5) X(7)
#undef X
  throw Error(EINVAL_, "Schwarz smoother: unsupported order");
}

void sem_asm_gather(const SchwarzArgs& a, double* y, cudaStream_t s) {
  const long n = (long)a.Ex * a.Ey * a.Ez * sem_nos(a.N);
  unsigned g = (unsigned)std::min<long>((n + 255) / 256, 148 * 16);
#define X(nn) \
  if (a.N == nn) { k_asm_gather<nn><<<g, 256, 0, s>>>(a, y); CMG_LAUNCH_CHECK(); return; }
  X(2) X(3) X(4) X(5) X(7)
#undef X
  throw Error(EINVAL_, "Schwarz smoother: unsupported order");
}

}  // namespace cmg
