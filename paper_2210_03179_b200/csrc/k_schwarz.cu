// k_schwarz.cu -- Chebyshev-Schwarz smoother kernels (PAPER.md:560-629,
// SURVEY App. A8): overlapping (N+3)^3 extended-element subdomains solved
// exactly by fast diagonalisation, combined additively (ASM, post-weighted)
// or restrictively (RAS).  The definition matches oracle/oracle_schwarz.c,
// and so does the rounding: this file is built with --fmad=false and every
// mode-product output is one __fma_rn chain over ascending m, as the oracle's
// fma() chain, so the CUDA-core local solves are bit-identical to it (the
// opt-in DMMA variant, CMG_SCHWARZ_MMA=1, is not).
#include <cstdlib>

#include "sem_kernels.hpp"
#include "sem_layout.hpp"

namespace cmg {

namespace {

// element coordinates of a local element index (< 2^31): two 32-bit divisions
// instead of the 64-bit ones `long % int` compiles to (a software routine)
__device__ __forceinline__ void elem_xyz(long e, int Ex, int Ey, int& ex, int& ey, int& ez) {
  const unsigned u = (unsigned)e, q = u / (unsigned)Ex;
  ex = (int)(u - q * (unsigned)Ex);
  ez = (int)(q / (unsigned)Ey);
  ey = (int)(q - (unsigned)ez * (unsigned)Ey);
}


template <int N>
__device__ __forceinline__ int owner1d_s(int g, int ne, int& oe) {
  if (g <= 0 || g >= N * ne) return -1;
  oe = (g - 1) / N;
  return (g - 1) - oe * N;
}

// r at global box node (ex*N+a-1, ey*N+b-1, ez*N+c-1) of element (ex, ey, ez):
// owned slots, or the neighbouring slab's planes (SchwarzArgs ghost layouts)
template <int N>
__device__ __forceinline__ double box_value(const SchwarzArgs& A, int ex, int ey, int ez, int a, int b, int c) {
  constexpr int NOS = sem_nos(N);
  int oex = 0, oey = 0, oez = 0;
  const int ax = owner1d_s<N>(ex * N + a - 1, A.Ex, oex);
  const int ay = owner1d_s<N>(ey * N + b - 1, A.Ey, oey);
  const int az = owner1d_s<N>(ez * N + c - 1, A.Ez, oez);
  if (ax < 0 || ay < 0 || az < 0) return 0.0;
  const long col = oex + (long)A.Ex * oey;
  if (oez < A.z0) return A.rlo[(col * 2 + (az - (N - 2))) * (N * N) + ay * N + ax];
  if (oez >= A.z0 + A.Ezl) return A.rhi[col * (N * N) + ay * N + ax];
  return A.r[(col + (long)A.Ex * A.Ey * (oez - A.z0)) * NOS + sem_pos(N, ax, ay, az)];
}

// one block per element: gather r on the extended box, FDM solve, write the
// local solution (RAS: the element's own (N+1)^3 nodes; ASM: all (N+3)^3).
// Each mode product is a set of line contractions: a thread loads one
// (N+3)-line of the box into registers once and produces the whole output
// line, with the 1D eigenbasis rows broadcast from shared memory (every
// output still sums its N+3 terms in ascending order).
template <int N>
__global__ void __launch_bounds__(64) k_schwarz_local(SchwarzArgs A) {
  constexpr int PB = N + 3, PB2 = PB * PB, PB3 = PB2 * PB, N1 = N + 1, NOS = sem_nos(N);
  // box stored with an odd x pitch: lines along x (stride PX between threads)
  // then hit distinct shared-memory banks
  constexpr int PX = PB | 1, PS = PX * PB;
  __shared__ double u[PS * PB], t[PS * PB];
  __shared__ __align__(16) double S[3][PB2];
  __shared__ double lam[3][PB];
  const long e = blockIdx.x;
  int ex, ey, ez;
  elem_xyz(e, A.Ex, A.Ey, ex, ey, ez);
  ez += A.z0;
  for (int d = 0; d < 3; ++d) {
    const int id = A.sidx[e * 3 + d];
    for (int q = threadIdx.x; q < PB2; q += blockDim.x) S[d][q] = A.S[(long)id * PB2 + q];
    for (int q = threadIdx.x; q < PB; q += blockDim.x) lam[d][q] = A.lam[(long)id * PB + q];
  }
  for (int q = threadIdx.x; q < PB3; q += blockDim.x) {
    const int a = q % PB, b = (q / PB) % PB, c = q / PB2;
    u[a + PX * b + PS * c] = box_value<N>(A, ex, ey, ez, a, b, c);
  }
  __syncthreads();
  // line l of dimension dim: the other two indices (p, q) = (l % PB, l / PB)
  auto line_base = [](int dim, int l) {
    const int p = l % PB, q = l / PB;
    return dim == 0 ? PX * p + PS * q : (dim == 1 ? p + PS * q : p + PX * q);
  };
  auto stride_of = [](int dim) { return dim == 0 ? 1 : (dim == 1 ? PX : PS); };
  // Two lines per thread share every eigenbasis load (the broadcast loads of
  // S dominate the shared-memory traffic), and S is read two entries at a time
  // when PB is even.  Every output still sums its PB terms in ascending order.
  constexpr int HALF = (PB2 + 1) / 2;
  constexpr bool PAIR = PB % 2 == 0;
  double* in = u;
  double* out = t;
  // forward: (Sz^T x Sy^T x Sx^T) u; the eigenvalue division fused into the last pass
#pragma unroll 1
  for (int dim = 0; dim < 3; ++dim) {
    const double* Sd = S[dim];
    for (int l = threadIdx.x; l < HALF; l += blockDim.x) {
      const int l2 = l + HALF;
      const bool two = l2 < PB2;
      const int b1 = line_base(dim, l), b2 = line_base(dim, two ? l2 : l), st = stride_of(dim);
      double v1[PB], v2[PB];
#pragma unroll
      for (int m = 0; m < PB; ++m) {
        v1[m] = in[b1 + m * st];
        v2[m] = in[b2 + m * st];
      }
      if constexpr (PAIR) {
#pragma unroll 1
        for (int o = 0; o < PB; o += 2) {
          double a0 = 0.0, a1 = 0.0, c0 = 0.0, c1 = 0.0;
#pragma unroll
          for (int m = 0; m < PB; ++m) {
            const double2 sp = *reinterpret_cast<const double2*>(Sd + m * PB + o);
            a0 = __fma_rn(sp.x, v1[m], a0);
            a1 = __fma_rn(sp.y, v1[m], a1);
            c0 = __fma_rn(sp.x, v2[m], c0);
            c1 = __fma_rn(sp.y, v2[m], c1);
          }
          if (dim == 2) {
            a0 /= (lam[0][l % PB] + lam[1][l / PB] + lam[2][o]);
            a1 /= (lam[0][l % PB] + lam[1][l / PB] + lam[2][o + 1]);
            c0 /= (lam[0][l2 % PB] + lam[1][l2 / PB] + lam[2][o]);
            c1 /= (lam[0][l2 % PB] + lam[1][l2 / PB] + lam[2][o + 1]);
          }
          out[b1 + o * st] = a0;
          out[b1 + (o + 1) * st] = a1;
          if (two) {
            out[b2 + o * st] = c0;
            out[b2 + (o + 1) * st] = c1;
          }
        }
      } else {
#pragma unroll 1
        for (int o = 0; o < PB; ++o) {
          double a0 = 0.0, c0 = 0.0;
#pragma unroll
          for (int m = 0; m < PB; ++m) {
            const double sv = Sd[m * PB + o];
            a0 = __fma_rn(sv, v1[m], a0);
            c0 = __fma_rn(sv, v2[m], c0);
          }
          if (dim == 2) {
            a0 /= (lam[0][l % PB] + lam[1][l / PB] + lam[2][o]);
            c0 /= (lam[0][l2 % PB] + lam[1][l2 / PB] + lam[2][o]);
          }
          out[b1 + o * st] = a0;
          if (two) out[b2 + o * st] = c0;
        }
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
    const double* Sd = S[dim];
    for (int l = threadIdx.x; l < HALF; l += blockDim.x) {
      const int l2 = l + HALF;
      const bool two = l2 < PB2;
      const int b1 = line_base(dim, l), b2 = line_base(dim, two ? l2 : l), st = stride_of(dim);
      double v1[PB], v2[PB];
#pragma unroll
      for (int m = 0; m < PB; ++m) {
        v1[m] = in[b1 + m * st];
        v2[m] = in[b2 + m * st];
      }
#pragma unroll 1
      for (int o = 0; o < PB; ++o) {
        double a0 = 0.0, c0 = 0.0;
        if constexpr (PAIR) {
#pragma unroll
          for (int m = 0; m < PB; m += 2) {
            const double2 sp = *reinterpret_cast<const double2*>(Sd + o * PB + m);
            a0 = __fma_rn(sp.x, v1[m], a0);
            a0 = __fma_rn(sp.y, v1[m + 1], a0);
            c0 = __fma_rn(sp.x, v2[m], c0);
            c0 = __fma_rn(sp.y, v2[m + 1], c0);
          }
        } else {
#pragma unroll
          for (int m = 0; m < PB; ++m) {
            const double sv = Sd[o * PB + m];
            a0 = __fma_rn(sv, v1[m], a0);
            c0 = __fma_rn(sv, v2[m], c0);
          }
        }
        out[b1 + o * st] = a0;
        if (two) out[b2 + o * st] = c0;
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
      A.Lout[e * (N1 * N1 * N1) + q] = in[(i + 1) + PX * (j + 1) + PS * (k + 1)];
    }
  } else {
    for (int q = threadIdx.x; q < PB3; q += blockDim.x) {
      const int a = q % PB, b = (q / PB) % PB, c = q / PB2;
      A.Lout[e * PB3 + q] = in[a + PX * b + PS * c];
    }
  }
}

// Same local solve with the contraction loops interchanged: a thread streams
// the eigenbasis ROW m (S[m][0..PB) forward, the row of a transposed copy
// backward, both broadcast as 16-byte loads) against the m-th value of its two
// lines and keeps all 2*PB accumulators live, so 2*PB independent fma chains
// are in flight instead of 4 (k_schwarz_local is latency-bound: one DFMA
// chain of PB terms per output pair).  Each output is still one fma chain over
// ascending m: bitwise identical to k_schwarz_local and the restatement.
template <int N>
__global__ void __launch_bounds__(64) k_schwarz_local_il(SchwarzArgs A) {
  constexpr int PB = N + 3, PB2 = PB * PB, PB3 = PB2 * PB, N1 = N + 1;
  static_assert(PB % 2 == 0, "interchanged loops read eigenbasis rows in pairs");
  constexpr int PX = PB | 1, PS = PX * PB;
  __shared__ double u[PS * PB], t[PS * PB];
  __shared__ __align__(16) double S[3][PB2];   // S[d][m*PB + o]: forward  out[o] += S[m][o] in[m]
  __shared__ __align__(16) double ST[3][PB2];  // ST[d][m*PB + o] = S[d][o*PB + m]: backward
  __shared__ double lam[3][PB];
  const long e = blockIdx.x;
  int ex, ey, ez;
  elem_xyz(e, A.Ex, A.Ey, ex, ey, ez);
  ez += A.z0;
  for (int d = 0; d < 3; ++d) {
    const int id = A.sidx[e * 3 + d];
    for (int q = threadIdx.x; q < PB2; q += blockDim.x) {
      const double v = A.S[(long)id * PB2 + q];
      S[d][q] = v;
      ST[d][(q % PB) * PB + q / PB] = v;
    }
    for (int q = threadIdx.x; q < PB; q += blockDim.x) lam[d][q] = A.lam[(long)id * PB + q];
  }
  for (int q = threadIdx.x; q < PB3; q += blockDim.x) {
    const int a = q % PB, b = (q / PB) % PB, c = q / PB2;
    u[a + PX * b + PS * c] = box_value<N>(A, ex, ey, ez, a, b, c);
  }
  __syncthreads();
  constexpr int HALF = (PB2 + 1) / 2;
  double* in = u;
  double* out = t;
#pragma unroll 1
  for (int pass = 0; pass < 6; ++pass) {
    const int dim = pass % 3;
    const double* Sd = pass < 3 ? S[dim] : ST[dim];
    const int st = dim == 0 ? 1 : (dim == 1 ? PX : PS);
    for (int l = threadIdx.x; l < HALF; l += blockDim.x) {
      const int l2 = l + HALF;
      const bool two = l2 < PB2;
      const int p1 = l % PB, q1 = l / PB, p2 = (two ? l2 : l) % PB, q2 = (two ? l2 : l) / PB;
      const int b1 = dim == 0 ? PX * p1 + PS * q1 : (dim == 1 ? p1 + PS * q1 : p1 + PX * q1);
      const int b2 = dim == 0 ? PX * p2 + PS * q2 : (dim == 1 ? p2 + PS * q2 : p2 + PX * q2);
      double a[PB], c[PB];
#pragma unroll
      for (int o = 0; o < PB; ++o) a[o] = c[o] = 0.0;
#pragma unroll 1
      for (int m = 0; m < PB; ++m) {  // not unrolled: keeps the 2*PB accumulators, not 5*PB loads, live
        const double v1 = in[b1 + m * st], v2 = in[b2 + m * st];
#pragma unroll
        for (int o = 0; o < PB; o += 2) {
          const double2 sp = *reinterpret_cast<const double2*>(Sd + m * PB + o);
          a[o] = __fma_rn(sp.x, v1, a[o]);
          a[o + 1] = __fma_rn(sp.y, v1, a[o + 1]);
          c[o] = __fma_rn(sp.x, v2, c[o]);
          c[o + 1] = __fma_rn(sp.y, v2, c[o + 1]);
        }
      }
#pragma unroll
      for (int o = 0; o < PB; ++o) {
        out[b1 + o * st] = a[o];
        if (two) out[b2 + o * st] = c[o];
      }
    }
    __syncthreads();
    if (pass == 2) {  // the eigenvalue division as its own elementwise sweep (a division's slow
                      // path is a call: kept away from the 2*PB live accumulators)
      for (int q = threadIdx.x; q < PB3; q += blockDim.x) {
        const int x = q % PB, y = (q / PB) % PB, z = q / PB2;
        out[x + PX * y + PS * z] /= (lam[0][x] + lam[1][y] + lam[2][z]);
      }
      __syncthreads();
    }
    double* tmp = in;
    in = out;
    out = tmp;
  }
  if (A.ras) {
    for (int q = threadIdx.x; q < N1 * N1 * N1; q += blockDim.x) {
      const int i = q % N1, j = (q / N1) % N1, k = q / (N1 * N1);
      A.Lout[e * (N1 * N1 * N1) + q] = in[(i + 1) + PX * (j + 1) + PS * (k + 1)];
    }
  } else {
    for (int q = threadIdx.x; q < PB3; q += blockDim.x) {
      const int a = q % PB, b = (q / PB) % PB, c = q / PB2;
      A.Lout[e * PB3 + q] = in[a + PX * b + PS * c];
    }
  }
}

// Low orders (N <= 4, the p=3 level of the (7,3,1) Schwarz schedule): a box
// has only (N+3)^2 <= 49 lines per pass, so one element per block left most
// threads idle.  EPB elements share a block, one line per thread; every
// output is formed by exactly the same expression sequence as above, so the
// two kernels give identical bits.
template <int N, int EPB>
__global__ void __launch_bounds__(EPB * (N + 3) * (N + 3)) k_schwarz_local_small(SchwarzArgs A, long E) {
  constexpr int PB = N + 3, PB2 = PB * PB, PB3 = PB2 * PB, N1 = N + 1;
  constexpr int PX = PB | 1, PS = PX * PB, BOX = PS * PB;
  constexpr bool PAIR = PB % 2 == 0;
  __shared__ double u[EPB][BOX], t[EPB][BOX];
  __shared__ __align__(16) double S[EPB][3][PB2];
  __shared__ double lam[EPB][3][PB];
  const int le = threadIdx.x / PB2, l = threadIdx.x - le * PB2;
  const long e = blockIdx.x * (long)EPB + le;
  const bool on = e < E;
  if (on) {
    int ex, ey, ez;
  elem_xyz(e, A.Ex, A.Ey, ex, ey, ez);
  ez += A.z0;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const int id = A.sidx[e * 3 + d];
      S[le][d][l] = A.S[(long)id * PB2 + l];
      if (l < PB) lam[le][d][l] = A.lam[(long)id * PB + l];
    }
    const int a = l % PB, b = l / PB;
#pragma unroll
    for (int c = 0; c < PB; ++c) u[le][a + PX * b + PS * c] = box_value<N>(A, ex, ey, ez, a, b, c);
  }
  __syncthreads();
  double* in = u[le];
  double* out = t[le];
  const int p = l % PB, q = l / PB;
#pragma unroll 1
  for (int pass = 0; pass < 6; ++pass) {
    const int dim = pass % 3;
    const double* Sd = S[le][dim];
    const int b1 = dim == 0 ? PX * p + PS * q : (dim == 1 ? p + PS * q : p + PX * q);
    const int st = dim == 0 ? 1 : (dim == 1 ? PX : PS);
    if (on) {
      double v[PB];
#pragma unroll
      for (int m = 0; m < PB; ++m) v[m] = in[b1 + m * st];
      if (pass < 3) {  // forward: S^T along dim; the eigenvalue division fused into the last pass
        if constexpr (PAIR) {
#pragma unroll
          for (int o = 0; o < PB; o += 2) {
            double a0 = 0.0, a1 = 0.0;
#pragma unroll
            for (int m = 0; m < PB; ++m) {
              const double2 sp = *reinterpret_cast<const double2*>(Sd + m * PB + o);
              a0 = __fma_rn(sp.x, v[m], a0);
              a1 = __fma_rn(sp.y, v[m], a1);
            }
            if (pass == 2) {
              a0 /= (lam[le][0][p] + lam[le][1][q] + lam[le][2][o]);
              a1 /= (lam[le][0][p] + lam[le][1][q] + lam[le][2][o + 1]);
            }
            out[b1 + o * st] = a0;
            out[b1 + (o + 1) * st] = a1;
          }
        } else {
#pragma unroll
          for (int o = 0; o < PB; ++o) {
            double a0 = 0.0;
#pragma unroll
            for (int m = 0; m < PB; ++m) a0 = __fma_rn(Sd[m * PB + o], v[m], a0);
            if (pass == 2) a0 /= (lam[le][0][p] + lam[le][1][q] + lam[le][2][o]);
            out[b1 + o * st] = a0;
          }
        }
      } else {  // backward: S along dim
#pragma unroll
        for (int o = 0; o < PB; ++o) {
          double a0 = 0.0;
          if constexpr (PAIR) {
#pragma unroll
            for (int m = 0; m < PB; m += 2) {
              const double2 sp = *reinterpret_cast<const double2*>(Sd + o * PB + m);
              a0 = __fma_rn(sp.x, v[m], a0);
              a0 = __fma_rn(sp.y, v[m + 1], a0);
            }
          } else {
#pragma unroll
            for (int m = 0; m < PB; ++m) a0 = __fma_rn(Sd[o * PB + m], v[m], a0);
          }
          out[b1 + o * st] = a0;
        }
      }
    }
    __syncthreads();
    double* tmp = in;
    in = out;
    out = tmp;
  }
  if (!on) return;
  if (A.ras) {
    for (int r = l; r < N1 * N1 * N1; r += PB2) {
      const int i = r % N1, j = (r / N1) % N1, k = r / (N1 * N1);
      A.Lout[e * (N1 * N1 * N1) + r] = in[(i + 1) + PX * (j + 1) + PS * (k + 1)];
    }
  } else {
    for (int r = l; r < PB3; r += PB2) {
      const int a = r % PB, b = (r / PB) % PB, c = r / PB2;
      A.Lout[e * PB3 + r] = in[a + PX * b + PS * c];
    }
  }
}

// FP64 tensor-core variant of the same local solve.  Each of the six mode
// products is a small GEMM  out[o, line] = sum_m M(o, m) in[m, line]  with
// M = S^T (forward) or S (backward), (N+3) x (N+3) padded to 16 x 12, and the
// (N+3)^2 lines as the N dimension; mma.sync m8n8k4 f64 (DMMA) replaces the
// per-line register contractions whose broadcast eigenbasis loads saturated
// the shared-memory pipe.  4 warps per element split the 8-line column tiles.
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int N>
__global__ void __launch_bounds__(128) k_schwarz_local_mma(SchwarzArgs A) {
  constexpr int PB = N + 3, PB2 = PB * PB, PB3 = PB2 * PB, N1 = N + 1, NOS = sem_nos(N);
  constexpr int PX = PB | 1, PS = PX * PB;
  constexpr int MT = (PB + 7) / 8, KT = (PB + 3) / 4, NT = (PB2 + 7) / 8;
  __shared__ double u[PS * PB], t[PS * PB];
  __shared__ double S[3][PB2];
  __shared__ double lam[3][PB];
  const long e = blockIdx.x;
  int ex, ey, ez;
  elem_xyz(e, A.Ex, A.Ey, ex, ey, ez);
  ez += A.z0;
  for (int d = 0; d < 3; ++d) {
    const int id = A.sidx[e * 3 + d];
    for (int q = threadIdx.x; q < PB2; q += blockDim.x) S[d][q] = A.S[(long)id * PB2 + q];
    for (int q = threadIdx.x; q < PB; q += blockDim.x) lam[d][q] = A.lam[(long)id * PB + q];
  }
  for (int q = threadIdx.x; q < PB3; q += blockDim.x) {
    const int a = q % PB, b = (q / PB) % PB, c = q / PB2;
    u[a + PX * b + PS * c] = box_value<N>(A, ex, ey, ez, a, b, c);
  }
  __syncthreads();
  auto line_base = [](int dim, int l) {
    const int p = l % PB, q = l / PB;
    return dim == 0 ? PX * p + PS * q : (dim == 1 ? p + PS * q : p + PX * q);
  };
  auto stride_of = [](int dim) { return dim == 0 ? 1 : (dim == 1 ? PX : PS); };
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tg = lane & 3;  // fragment row group / thread in group
  double* in = u;
  double* out = t;
#pragma unroll 1
  for (int pass = 0; pass < 6; ++pass) {
    const int dim = pass % 3;
    const bool fwd = pass < 3;
    const int st = stride_of(dim);
    // A fragments (row o, col m) of M for every (m-tile, k-step)
    double af[MT][KT];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int kt = 0; kt < KT; ++kt) {
        const int o = mt * 8 + g, m = kt * 4 + tg;
        af[mt][kt] = (o < PB && m < PB) ? (fwd ? S[dim][m * PB + o] : S[dim][o * PB + m]) : 0.0;
      }
    for (int nt = warp; nt < NT; nt += 4) {
      double bf[KT];
      const int lb = nt * 8 + g;  // this thread's B column (line)
#pragma unroll
      for (int kt = 0; kt < KT; ++kt) {
        const int m = kt * 4 + tg;
        bf[kt] = (lb < PB2 && m < PB) ? in[line_base(dim, lb) + m * st] : 0.0;
      }
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int kt = 0; kt < KT; ++kt) dmma_8x8x4(d0, d1, af[mt][kt], bf[kt]);
        const int o = mt * 8 + g;
        if (o < PB) {
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int l = nt * 8 + 2 * tg + i;
            if (l < PB2) {
              double v = i ? d1 : d0;
              if (pass == 2) v /= (lam[0][l % PB] + lam[1][l / PB] + lam[2][o]);
              out[line_base(dim, l) + o * st] = v;
            }
          }
        }
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
      A.Lout[e * (N1 * N1 * N1) + q] = in[(i + 1) + PX * (j + 1) + PS * (k + 1)];
    }
  } else {
    for (int q = threadIdx.x; q < PB3; q += blockDim.x) {
      const int a = q % PB, b = (q / PB) % PB, c = q / PB2;
      A.Lout[e * PB3 + q] = in[a + PX * b + PS * c];
    }
  }
}

// ASM: every owned slot sums the extended local solutions covering it (fixed
// ascending-element order, oracle_schwarz.c) and applies W = 1/count.  The
// result sv is stored (u.kind 0) or consumed by the Chebyshev update
// (kind 4: d = c1 d + c2 sv; kind 1: r -= sv, d = c1 d + c2 r).
__device__ __forceinline__ void asm_emit(const AsmUpdate& u, double* __restrict__ y, long q, double sv) {
  if (u.kind == 0) {
    y[q] = sv;
  } else if (u.kind == 4) {
    u.d[q] = u.c1 * u.d[q] + u.c2 * sv;
  } else {
    if (u.x) u.x[q] = u.x_zero ? u.d[q] : u.x[q] + u.d[q];
    const double rv = u.r[q] - sv;
    u.r[q] = rv;
    u.d[q] = u.c1 * u.d[q] + u.c2 * rv;
  }
}

template <int N>
__global__ void k_asm_gather(SchwarzArgs A, double* __restrict__ y, AsmUpdate u) {
  constexpr int PB = N + 3, PB2 = PB * PB, PB3 = PB2 * PB, NOS = sem_nos(N);
  const long n = (long)A.Ex * A.Ey * A.Ezl * NOS;
  for (long q = blockIdx.x * (long)blockDim.x + threadIdx.x; q < n; q += (long)gridDim.x * blockDim.x) {
    const long e = q / NOS;
    int a, b, c;
    if (!sem_abc(N, (int)(q - e * NOS), a, b, c)) {
      asm_emit(u, y, q, 0.0);
      continue;
    }
    int ex, ey, ez;
  elem_xyz(e, A.Ex, A.Ey, ex, ey, ez);
  ez += A.z0;
    const int gx = ex * N + a + 1, gy = ey * N + b + 1, gz = ez * N + c + 1;
    if (gx >= N * A.Ex || gy >= N * A.Ey || gz >= N * A.Ez) {
      asm_emit(u, y, q, 0.0);
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
          const long col = cx + (long)A.Ex * cy;
          const int la = gx - cx * N + 1, lb = gy - cy * N + 1, lc = gz - cz * N + 1;
          if (cz < A.z0) acc += A.Llo[col * PB2 + la + PB * lb];  // lc == N+2
          else if (cz >= A.z0 + A.Ezl) acc += A.Lhi[(col * 2 + lc) * PB2 + la + PB * lb];  // lc 0, 1
          else acc += A.Lout[(col + (long)A.Ex * A.Ey * (cz - A.z0)) * PB3 + la + PB * (lb + PB * lc)];
          ++cnt;
        }
      }
    }
    asm_emit(u, y, q, acc * (1.0 / (double)cnt));
  }
}

// Faces for the neighbouring slabs, in the SchwarzArgs ghost layouts.  what 0:
// r planes az = N-2, N-1 of the top layer (up) and az = 0 of the bottom layer
// (dn); what 1: ASM Lout plane z = N+2 of the top layer (up) and z = 0, 1 of
// the bottom layer (dn).
template <int N>
__global__ void k_schwarz_pack(SchwarzArgs A, int what, double* __restrict__ up, double* __restrict__ dn) {
  constexpr int PB = N + 3, PB2 = PB * PB, PB3 = PB2 * PB, NOS = sem_nos(N), NN = N * N;
  const long cols = (long)A.Ex * A.Ey, top = cols * (A.Ezl - 1);
  const int pu = what == 0 ? 2 * NN : PB2, pd = what == 0 ? NN : 2 * PB2;
  const long n = cols * (pu + pd);
  for (long q = blockIdx.x * (long)blockDim.x + threadIdx.x; q < n; q += (long)gridDim.x * blockDim.x) {
    const bool isup = q < cols * pu;
    const long k = isup ? q : q - cols * pu;
    const int per = isup ? pu : pd;
    const long col = k / per;
    const int i = (int)(k - col * per);
    const long e = (isup ? top : 0) + col;
    double v;
    if (what == 0) {  // i = plane * NN + ay * N + ax
      const int pl = i / NN, ay = (i % NN) / N, ax = i % N;
      v = A.r[e * NOS + sem_pos(N, ax, ay, isup ? N - 2 + pl : 0)];
    } else {          // i = plane * PB2 + b * PB + a
      const int pl = i / PB2;
      v = A.Lout[e * PB3 + (isup ? N + 2 : pl) * PB2 + i % PB2];
    }
    (isup ? up : dn)[k] = v;
  }
}

}  // namespace

void sem_schwarz_pack(const SchwarzArgs& a, int what, double* up, double* dn, cudaStream_t s) {
  const long n = schwarz_ghost_up(a, what) + schwarz_ghost_dn(a, what);
  const unsigned g = (unsigned)std::min<long>((n + 255) / 256, 148 * 8);
#define X(nn) \
  if (a.N == nn) { k_schwarz_pack<nn><<<g, 256, 0, s>>>(a, what, up, dn); CMG_LAUNCH_CHECK(); return; }
  X(2) X(3) X(4) X(5) X(7)
#undef X
  throw Error(EINVAL_, "Schwarz smoother: unsupported order");
}

void sem_schwarz_local(const SchwarzArgs& a, cudaStream_t s) {
  const long E = (long)a.Ex * a.Ey * a.Ezl;
  // CUDA-core line contractions by default; the DMMA variant is opt-in
  // (CMG_SCHWARZ_MMA=1): measured 826 vs 562 us per apply at E=32^3 -- the
  // fragment index math and the dependent m8n8k4 chains cost more than the
  // shared-memory traffic they remove (profiles/r01/schwarz_summary.txt)
  static const bool use_mma = [] {
    const char* env = std::getenv("CMG_SCHWARZ_MMA");
    return env && std::atoi(env) == 1;
  }();
  // interchanged-loop local solve, opt-in (CMG_SCHWARZ_IL=1): measured 636 vs
  // 570 us per apply at E=32^3 and RAS (1,1) 23.8 vs 23.0 ms (profiles/r02/
  // schwarz_il_ab.txt) -- 96 registers, so fewer resident blocks, and the
  // per-m row loads are no cheaper than the per-output ones they replace
  static const bool il = [] {
    const char* env = std::getenv("CMG_SCHWARZ_IL");
    return env && std::atoi(env) == 1;
  }();
  // low orders: several elements per block (CMG_SCHWARZ_SMALL=0 keeps one per block)
  static const bool small = [] {
    const char* env = std::getenv("CMG_SCHWARZ_SMALL");
    return !(env && std::atoi(env) == 0);
  }();
#define XS(n, epb)                                                                              \
  if (a.N == n && small && !use_mma) {                                                          \
    k_schwarz_local_small<n, epb><<<(unsigned)((E + epb - 1) / epb), epb * (n + 3) * (n + 3), 0, s>>>(a, E); \
    CMG_LAUNCH_CHECK();                                                                         \
    return;                                                                                     \
  }
  XS(2, 8) XS(3, 8) XS(4, 4)
#undef XS
#define X(n)                                                                  \
  if (a.N == n) {                                                             \
    if (use_mma) k_schwarz_local_mma<n><<<(unsigned)E, 128, 0, s>>>(a);      \
    else if (il && (n + 3) % 2 == 0) k_schwarz_local_il<(n + 3) % 2 == 0 ? n : 5><<<(unsigned)E, 64, 0, s>>>(a); \
    else k_schwarz_local<n><<<(unsigned)E, 64, 0, s>>>(a);                    \
    CMG_LAUNCH_CHECK();                                                       \
    return;                                                                   \
  }
  X(2) X(3) X(4) X(5) X(7)
#undef X
  throw Error(EINVAL_, "Schwarz smoother: unsupported order");
}

void sem_asm_gather(const SchwarzArgs& a, double* y, cudaStream_t s, const AsmUpdate& u) {
  const long n = (long)a.Ex * a.Ey * a.Ezl * sem_nos(a.N);
  unsigned g = (unsigned)std::min<long>((n + 255) / 256, 148 * 16);
#define X(nn) \
  if (a.N == nn) { k_asm_gather<nn><<<g, 256, 0, s>>>(a, y, u); CMG_LAUNCH_CHECK(); return; }
  X(2) X(3) X(4) X(5) X(7)
#undef X
  throw Error(EINVAL_, "Schwarz smoother: unsupported order");
}

}  // namespace cmg
