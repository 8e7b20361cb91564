// k_sem.cu -- spectral-element kernels for sm_100a (fp64).
//
// Hot path: the Chebyshev-Jacobi step on a p-level, i.e. the matrix-free
// operator A = Q^T A_L Q (sum-factorised tensor contractions with six
// geometric factors per node) fused with the direct
// stiffness summation and the three-term recurrence (smoothers.hpp:126-148
// with S = invD).  See sem_kernels.hpp for the K1/K2 split that makes QQ^T
// deterministic and partition-independent, and sem_layout.hpp for the
// interior-first slot order that makes both kernels' vector traffic
// contiguous per element.
//
// K1 (element kernel, AX mode) for the high orders is k_sem_k1.cuh (line
// contractions with the GLL matrix in constant memory, TMA-staged geometric
// factors and epilogue operands); the low orders (coarse p-levels) use
// k_sem_k1_ax below (several elements per block, k-split columns).
#include <cstdlib>

#include "sem_kernels.hpp"
#include "sem_layout.hpp"

namespace cmg {

void host_interp_matrix(int Nf, int Nc, double* J);  // host_setup.cpp

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
struct SemC {
  static constexpr int N1 = N + 1;
  static constexpr int NP = N1 * N1 * N1;
  static constexpr int NOS = sem_nos(N);
  static constexpr int NINT = sem_nint(N);
  static constexpr int NSH = sem_nshared(N);
  // k-split across threads: order 3 keeps whole columns per thread (the p=3 smoother
  // step 280 -> 266 us at E=64^3, TTS -0.9%, profiles/r02/ab_k1ax3_ks.txt)
  static constexpr int KS = (N1 % 2 == 0 && N >= 5) ? 2 : 1;
  static constexpr int KN = N1 / KS;                          // k values per thread
  static constexpr int TPE = N1 * N1 * KS;                    // threads per element
  static constexpr int EPB = (128 / TPE) > 0 ? (128 / TPE) : 1;  // elements per block
  static constexpr int NT = EPB * TPE;
  // interior operand block copied per element (16-byte multiple)
  static constexpr int NINT_PAD = ((NINT * 8 + 15) / 16) * 16 / 8;
};

// ---------------------------------------------------------------- async-copy helpers
// (sm_90+ PTX; SASS on sm_100a: UBLKCP / SYNCS.* / LDGSTS)
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// shared -> global bulk copy (TMA engine), completion tracked by a bulk group
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
// make this thread's generic-proxy shared-memory writes visible to the async (TMA) proxy
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// commit the issued bulk stores and wait until their shared-memory source has been read
__device__ __forceinline__ void bulk_store_wait_read() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// Block-wide wait until *flag >= v (a peer GPU's stream memop writes the epoch after
// its producing kernel; acquire at system scope, then the CTA barrier orders every
// thread's later reads of the peer buffer after it).  Called by all threads.
__device__ __forceinline__ void block_wait_flag(const unsigned* flag, unsigned v) {
  if (threadIdx.x == 0) {
    unsigned x;
    while (true) {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(x) : "l"(flag) : "memory");
      if ((int)(x - v) >= 0) break;
      __nanosleep(128);
    }
  }
  __syncthreads();
}

// owner of local node index l (0..N) along one dimension of element coordinate ec:
// returns the owned-slot coordinate in the owner (oe) or -1 for a Dirichlet node
template <int N>
__device__ __forceinline__ int owner1d(int ec, int l, int ne, int& oe) {
  const int g = ec * N + l;
  if (g <= 0 || g >= N * ne) return -1;
  oe = (g - 1) / N;
  return (g - 1) - oe * N;
}

// ---------------------------------------------------------------- arithmetic contract
// This file is compiled with --fmad=false (Makefile): the only fused
// multiply-adds are the explicit __fma_rn calls, placed exactly where
// oracle/oracle_sem.c calls C99 fma(), so the local operator, its diagonal,
// the p-transfers and the Chebyshev epilogues round identically on the GPU
// and in the CPU restatement (bitwise):
//   1D contraction  v = 0; for m ascending: v = fma(D_m, u_m, v)
//   geometry        w_a = fma(g_c, u_t, fma(g_b, u_s, g_a * u_r))
//   divergence      out = v_t + (v_r + v_s)       (three separate chains)
//   everything else: the reference's operand order without contraction.
__device__ __forceinline__ double geo3(double ga, double gb, double gc, double ur, double us, double ut) {
  return __fma_rn(gc, ut, __fma_rn(gb, us, ga * ur));
}

// ---------------------------------------------------------------- epilogues
template <int EPI>
struct EpiOps {  // slot-vector operands read for interior nodes, in smem order
  static constexpr int n = (EPI == EPI_CHEB4 || EPI == EPI_CHEB1 || EPI == EPI_SUPD1) ? 3
                           : (EPI == EPI_CHEB4_INIT || EPI == EPI_CHEB1_INIT || EPI == EPI_SUPD4) ? 2
                           : (EPI == EPI_RESID || EPI == EPI_ADD) ? 1 : 0;
};

template <int EPI>
__device__ __forceinline__ const double* epi_op(const SemArgs& A, int q) {
  if constexpr (EPI == EPI_CHEB4) return q == 0 ? A.x : (q == 1 ? A.r_in : A.invd);
  else if constexpr (EPI == EPI_CHEB1) return q == 0 ? A.x : (q == 1 ? A.r : A.invd);
  else if constexpr (EPI == EPI_CHEB4_INIT || EPI == EPI_CHEB1_INIT) return q == 0 ? A.b : A.invd;
  else if constexpr (EPI == EPI_RESID) return A.b;
  else if constexpr (EPI == EPI_SUPD4) return q == 0 ? A.invd : A.d;
  else if constexpr (EPI == EPI_SUPD1) return q == 0 ? A.r_in : (q == 1 ? A.invd : A.d);
  else return A.y;
}

// o0..o2: the operands at this slot (prefetched or loaded); w = (A u) at the node
template <int EPI>
__device__ __forceinline__ void epilogue(const SemArgs& A, long slot, double w, double dv, double o0,
                                         double o1, double o2) {
  if constexpr (EPI == EPI_STORE) {
    A.y[slot] = w;
  } else if constexpr (EPI == EPI_ADD) {
    A.y[slot] = o0 + w;
  } else if constexpr (EPI == EPI_RESID) {
    A.r[slot] = o0 - w;
  } else if constexpr (EPI == EPI_CHEB4) {
    // smoothers.hpp:138-144: x += beta d ; r -= A d ; d = c1 d + c2 invD r
    const double xv = A.x_zero ? A.beta * dv : o0 + A.beta * dv;
    const double rv = o1 - w;
    const double dn = A.c1 * dv + A.c2 * o2 * rv;
    if (A.beta_last > 0.0) {  // last step: fused final x += beta_k d (smoothers.hpp:146-147)
      A.x[slot] = xv + A.beta_last * dn;
    } else {
      A.x[slot] = xv;
      A.r[slot] = rv;
      A.d_out[slot] = dn;
    }
  } else if constexpr (EPI == EPI_CHEB1) {
    // smoothers.hpp:109-118: x += d ; z -= invD A d ; d = c1 d + c2 z
    const double xv = A.x_zero ? dv : o0 + dv;
    const double zv = o1 - o2 * w;
    const double dn = A.c1 * dv + A.c2 * zv;
    if (A.beta_last > 0.0) {  // last step: fused final x += d (smoothers.hpp:119)
      A.x[slot] = xv + A.beta_last * dn;
    } else {
      A.x[slot] = xv;
      A.r[slot] = zv;
      A.d_out[slot] = dn;
    }
  } else if constexpr (EPI == EPI_CHEB4_INIT) {
    const double rv = o0 - w;
    A.r[slot] = rv;
    A.d_out[slot] = A.c0 * o1 * rv;
  } else if constexpr (EPI == EPI_CHEB1_INIT) {
    const double zv = (o0 - w) * o1;
    A.r[slot] = zv;
    A.d_out[slot] = zv / A.theta;
  } else if constexpr (EPI == EPI_SUPD4) {
    A.d_out[slot] = A.c1 * o1 + A.c2 * (o0 * w);
  } else if constexpr (EPI == EPI_SUPD1) {
    if (A.x) A.x[slot] = A.x_zero ? o2 : A.x[slot] + o2;  // x += d (the pre-update d)
    const double rv = o0 - o1 * w;
    A.r[slot] = rv;
    A.d_out[slot] = A.c1 * o2 + A.c2 * rv;
  }
}

// ---------------------------------------------------------------- K1 (AX mode)
template <int N, int EPI>
struct K1Smem {
  using C = SemC<N>;
  static constexpr int NOPS = EpiOps<EPI>::n;
  static constexpr std::size_t g_off = 0;                                            // [EPB][6][NP]
  static constexpr std::size_t u_off = g_off + (std::size_t)C::EPB * 6 * C::NP;      // [EPB][NP]
  static constexpr std::size_t o_off = u_off + (((std::size_t)C::EPB * C::NP + 1) & ~(std::size_t)1);  // [EPB][NOPS][NINT_PAD], 16B-aligned
  static constexpr std::size_t d_off = o_off + (std::size_t)C::EPB * NOPS * C::NINT_PAD;  // [N1][N1+1]
  static constexpr std::size_t bar_off = d_off + (std::size_t)C::N1 * (C::N1 + 1);
  static constexpr std::size_t bytes = (bar_off + 1) * sizeof(double);
};

// GLL derivative matrices per order in constant memory: with compile-time
// indices every D entry becomes a DFMA constant-bank operand (no LDS).
__constant__ double c_D[8][64];

template <int N, int EPI>
__global__ void __launch_bounds__(SemC<N>::NT) k_sem_k1_ax(SemArgs A) {
  using C = SemC<N>;
  using S = K1Smem<N, EPI>;
  constexpr int N1 = C::N1, NP = C::NP, NOS = C::NOS, TPE = C::TPE, EPB = C::EPB, KN = C::KN;
  constexpr int NOPS = S::NOPS, NIP = C::NINT_PAD;
  extern __shared__ __align__(128) double sm[];
  double* sG = sm + S::g_off;
  double* su = sm + S::u_off;
  double* so = sm + S::o_off;
  double (*sD)[N1 + 1] = reinterpret_cast<double (*)[N1 + 1]>(sm + S::d_off);
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(sm + S::bar_off);
  const int le = threadIdx.x / TPE;
  const int t = threadIdx.x - le * TPE;
  const int i = t % N1, j = (t / N1) % N1, kh = t / (N1 * N1);
  const int kb = kh * KN;
  const long e0 = A.e_begin + (long)blockIdx.x * EPB;
  const long e = e0 + le;
  const bool active = e < A.e_end;
  const int nact = (int)min((long)EPB, A.e_end - e0);
  // 1. one thread streams geometric factors + interior operand blocks with TMA
  if (threadIdx.x == 0) {
    const bool skip_x = (EPI == EPI_CHEB4 || EPI == EPI_CHEB1) && A.x_zero;
    unsigned bytes = (unsigned)(nact * 6 * NP * sizeof(double));
    if constexpr (NOPS > 0 && C::NINT > 0) bytes += (unsigned)(nact * (NOPS - (skip_x ? 1 : 0)) * NIP * 8);
    mbar_init(bar, 1);
    mbar_expect_tx(bar, bytes);
    for (int q = 0; q < nact; ++q) {
      bulk_g2s(sG + (std::size_t)q * 6 * NP, A.G + (e0 + q) * 6 * NP, 6 * NP * sizeof(double), bar);
      if constexpr (NOPS > 0 && C::NINT > 0) {
#pragma unroll
        for (int op = 0; op < NOPS; ++op) {
          if (op == 0 && skip_x) continue;
          bulk_g2s(so + ((std::size_t)q * NOPS + op) * NIP, epi_op<EPI>(A, op) + (e0 + q) * NOS, NIP * 8, bar);
        }
      }
    }
  }
  for (int q = threadIdx.x; q < N1 * N1; q += blockDim.x) sD[q / N1][q % N1] = A.D[q];
  int ex = 0, ey = 0, ez = 0;
  if (active) elem_xyz(e, A.Ex, A.Ey, ex, ey, ez);
  // 2. gather Q u (owner slots / halo / Dirichlet zero) into shared memory
  double* ue = su + (std::size_t)le * NP;
  double ucol[KN];  // this thread's own column (all of it when KS == 1)
  {
    int oex = 0, oey = 0;
    const int ax = owner1d<N>(ex, i, A.Ex, oex);
    const int ay = owner1d<N>(ey, j, A.Ey, oey);
#pragma unroll
    for (int kk = 0; kk < KN; ++kk) {
      const int k = kb + kk;
      double v = 0.0;
      if (active && ax >= 0 && ay >= 0) {
        int oez = 0;
        const int az = owner1d<N>(A.z0 + ez, k, A.Ez, oez);
        if (az >= 0) {
          const int lz = oez - A.z0;
          if (lz < 0)
            v = A.halo_lo[((long)oex + (long)A.Ex * oey) * (N * N) + ax + N * ay];
          else
            v = A.u[((long)oex + (long)A.Ex * ((long)oey + (long)A.Ey * lz)) * NOS + sem_pos(N, ax, ay, az)];
        }
      }
      ue[(k * N1 + j) * N1 + i] = v;
      ucol[kk] = v;
    }
  }
  __syncthreads();
  mbar_wait(bar, 0);
  // 3. gradient + geometric factors: w_r, w_s, w_t overwrite G_rr, G_rs, G_rt in place
  double* Ge = sG + (std::size_t)le * 6 * NP;
  if constexpr (C::KS == 1) {
    // Whole columns per thread: the k-direction contractions use the thread's own
    // column from registers and D from constant memory (compile-time k, m), the
    // i/j rows of D sit in registers; w_t never leaves registers.  Same chains,
    // same operands as the generic path below (same bits), half the shared traffic.
    double Di[N1], Dj[N1], DiT[N1], DjT[N1], wtc[KN];
#pragma unroll
    for (int m = 0; m < N1; ++m) {
      Di[m] = sD[i][m];
      Dj[m] = sD[j][m];
      DiT[m] = sD[m][i];
      DjT[m] = sD[m][j];
    }
#pragma unroll
    for (int k = 0; k < N1; ++k) {
      const int l = (k * N1 + j) * N1 + i;
      double ur = 0.0, us = 0.0, ut = 0.0;
#pragma unroll
      for (int m = 0; m < N1; ++m) {
        ur = __fma_rn(Di[m], ue[(k * N1 + j) * N1 + m], ur);
        us = __fma_rn(Dj[m], ue[(k * N1 + m) * N1 + i], us);
        ut = __fma_rn(c_D[N][k * N1 + m], ucol[m], ut);
      }
      const double g0 = Ge[l], g1 = Ge[NP + l], g2 = Ge[2 * NP + l];
      const double g3 = Ge[3 * NP + l], g4 = Ge[4 * NP + l], g5 = Ge[5 * NP + l];
      Ge[l] = geo3(g0, g1, g2, ur, us, ut);
      Ge[NP + l] = geo3(g1, g3, g4, ur, us, ut);
      wtc[k] = geo3(g2, g4, g5, ur, us, ut);
    }
    __syncthreads();
    if (!active) return;
    const bool ij_interior = (i >= 1 && i < N && j >= 1 && j < N);
    const double* soe = so + (std::size_t)le * NOPS * NIP;
#pragma unroll
    for (int k = 0; k < N1; ++k) {
      double vr = 0.0, vs = 0.0, vt = 0.0;
#pragma unroll
      for (int m = 0; m < N1; ++m) {
        vr = __fma_rn(DiT[m], Ge[(k * N1 + j) * N1 + m], vr);
        vs = __fma_rn(DjT[m], Ge[NP + (k * N1 + m) * N1 + i], vs);
        vt = __fma_rn(c_D[N][m * N1 + k], wtc[m], vt);
      }
      const double v = vt + (vr + vs);
      if (ij_interior && k >= 1 && k < N) {
        const int p = (i - 1) + (N - 1) * ((j - 1) + (N - 1) * (k - 1));
        double o0 = 0.0, o1 = 0.0, o2 = 0.0;
        if constexpr (NOPS > 0) o0 = soe[p];
        if constexpr (NOPS > 1) o1 = soe[NIP + p];
        if constexpr (NOPS > 2) o2 = soe[2 * NIP + p];
        epilogue<EPI>(A, e * NOS + p, v, ucol[k], o0, o1, o2);
      } else {
        A.shell[e * A.nshell + A.lut[(k * N1 + j) * N1 + i]] = v;
      }
    }
  } else {
#pragma unroll
  for (int kk = 0; kk < KN; ++kk) {
    const int k = kb + kk;
    const int l = (k * N1 + j) * N1 + i;
    double ur = 0.0, us = 0.0, ut = 0.0;
#pragma unroll
    for (int m = 0; m < N1; ++m) {
      ur = __fma_rn(sD[i][m], ue[(k * N1 + j) * N1 + m], ur);
      us = __fma_rn(sD[j][m], ue[(k * N1 + m) * N1 + i], us);
      ut = __fma_rn(sD[k][m], ue[(m * N1 + j) * N1 + i], ut);
    }
    const double g0 = Ge[l], g1 = Ge[NP + l], g2 = Ge[2 * NP + l];
    const double g3 = Ge[3 * NP + l], g4 = Ge[4 * NP + l], g5 = Ge[5 * NP + l];
    Ge[l] = geo3(g0, g1, g2, ur, us, ut);
    Ge[NP + l] = geo3(g1, g3, g4, ur, us, ut);
    Ge[2 * NP + l] = geo3(g2, g4, g5, ur, us, ut);
  }
  __syncthreads();
  if (!active) return;
  // 4. divergence + epilogue (interior nodes finished, shell nodes to the shell buffer)
  const bool ij_interior = (i >= 1 && i < N && j >= 1 && j < N);
  const double* soe = so + (std::size_t)le * NOPS * NIP;
#pragma unroll
  for (int kk = 0; kk < KN; ++kk) {
    const int k = kb + kk;
    double vr = 0.0, vs = 0.0, vt = 0.0;
#pragma unroll
    for (int m = 0; m < N1; ++m) {
      vr = __fma_rn(sD[m][i], Ge[(k * N1 + j) * N1 + m], vr);
      vs = __fma_rn(sD[m][j], Ge[NP + (k * N1 + m) * N1 + i], vs);
      vt = __fma_rn(sD[m][k], Ge[2 * NP + (m * N1 + j) * N1 + i], vt);
    }
    const double v = vt + (vr + vs);
    if (ij_interior && k >= 1 && k < N) {
      const int p = (i - 1) + (N - 1) * ((j - 1) + (N - 1) * (k - 1));
      const double dv = ue[(k * N1 + j) * N1 + i];
      double o0 = 0.0, o1 = 0.0, o2 = 0.0;
      if constexpr (NOPS > 0) o0 = soe[p];
      if constexpr (NOPS > 1) o1 = soe[NIP + p];
      if constexpr (NOPS > 2) o2 = soe[2 * NIP + p];
      epilogue<EPI>(A, e * NOS + p, v, dv, o0, o1, o2);
    } else {
      A.shell[e * A.nshell + A.lut[(k * N1 + j) * N1 + i]] = v;
    }
  }
  }
}

// ---------------------------------------------------------------- K1 (AX mode, line contractions)

// Line-blocked layout: one block = one element, (N+1)^2 threads.  Each
// contraction is done by a thread owning a whole line of N+1 nodes along the
// contracted direction: N+1 shared loads, (N+1)^2 DFMAs with constant D,
// N+1 stores -- one shared access per output instead of 2(N+1).  Rows are
// padded to N+2 doubles (conflict-free line loads).
template <int N, int EPI, bool GS = true>
struct K3Smem {
  static constexpr int N1 = N + 1, NP = N1 * N1 * N1, NPP = N1 * N1 * (N1 + 1);
  static constexpr int NOPS = EpiOps<EPI>::n, NIP = SemC<N>::NINT_PAD;
  static constexpr std::size_t g_off = 0;                                  // [6][NP]  (TMA)
  static constexpr std::size_t g_len = GS ? (std::size_t)6 * NP : 0;       // 0: factors read to registers
  static constexpr std::size_t o_off = g_off + g_len;                      // [NOPS][NIP] (TMA)
  static constexpr std::size_t u_off = o_off + (std::size_t)NOPS * NIP;    // [NPP] u, later v
  static constexpr std::size_t r_off = u_off + NPP;                        // [NPP] u_r -> w_r
  static constexpr std::size_t s_off = r_off + NPP;                        // [NPP] u_s -> w_s
  static constexpr std::size_t bar_off = (s_off + NPP + 1) & ~(std::size_t)1;
  static constexpr std::size_t bytes = (bar_off + 1) * sizeof(double);
};

#include "k_sem_k1.cuh"

// ---------------------------------------------------------------- K1 (LVEC mode: assemble an L-vector)
template <int N, int EPI>
__global__ void k_sem_k1_lvec(SemArgs A) {
  constexpr int N1 = N + 1, NP = N1 * N1 * N1, NOS = sem_nos(N);
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const long e = A.e_begin + t / NP;
  if (e >= A.e_end) return;
  const int l = (int)(t % NP);
  const int i = l % N1, j = (l / N1) % N1, k = l / (N1 * N1);
  const double v = A.lvec[e * NP + l];
  if (i >= 1 && i < N && j >= 1 && j < N && k >= 1 && k < N) {
    const long slot = e * NOS + (i - 1) + (N - 1) * ((j - 1) + (N - 1) * (k - 1));
    double o0 = 0.0, o1 = 0.0, o2 = 0.0;
    if constexpr (EpiOps<EPI>::n > 0) o0 = epi_op<EPI>(A, 0)[slot];
    if constexpr (EpiOps<EPI>::n > 1) o1 = epi_op<EPI>(A, 1)[slot];
    if constexpr (EpiOps<EPI>::n > 2) o2 = epi_op<EPI>(A, 2)[slot];
    epilogue<EPI>(A, slot, v, 0.0, o0, o1, o2);
  } else {
    A.shell[e * A.nshell + A.lut[l]] = v;
  }
}

// ---------------------------------------------------------------- K2
// Contributor table per shared slot s (sem.cpp): the packed (a,b,c) and up to 8
// (shell offset, direction) entries in the fixed (dz, dy, dx) order, so every
// contribution load is independent (no lut -> shell dependency).

constexpr int k2_eb(int N) { return sem_nshared(N) >= 256 ? 1 : 256 / sem_nshared(N); }

// One owned shared node: sum its <= 8 shell contributions in the fixed
// (dz, dy, dx) order, then the step's epilogue.  Returns without work for
// padding slots.
//
// A single-launch step that ran this per owned node inside the element kernel
// (elements claimed in decreasing order, per-element "shell written" flags)
// was measured at E=64^3: 21.9 vs 34.1 GDOF-step/s for the K1 + K2 pair --
// waiting for the +x neighbour's flag cost 1.15 ms and the in-block node work
// 0.7 ms per step, against 0.47 ms for the separate K2 launch.
template <int N, int EPI>
__device__ __forceinline__ void k2_node(const SemArgs& A, long e, int ex, int ey, int ez, int s) {
  constexpr int N1 = N + 1, NOS = sem_nos(N), NINT = sem_nint(N);
  // host-built table (sem.cpp, L1-resident): [count, a|b<<8|c<<16, (offset, dx|dy<<1|dz<<2) x count],
  // offset = shell position relative to this element's shell block
  const int* tab = A.k2tab + s * K2TAB_STRIDE;
  const int head = __ldg(tab);
  const int n = head & 0xff, a = (head >> 8) & 0xff, b = (head >> 16) & 0xff, c = head >> 24;
  // padding (far domain boundary) is not an unknown
  if (ex * N + a + 1 >= N * A.Ex || ey * N + b + 1 >= N * A.Ey || (A.z0 + ez) * N + c + 1 >= N * A.Ez) return;
  // the epilogue operands first: their loads are independent of the contributions,
  // so all of a thread's loads are in flight together (K2 is memory-latency bound)
  const long slot = e * NOS + NINT + s;
  double dv = 0.0, o0 = 0.0, o1 = 0.0, o2 = 0.0;
  if constexpr (EPI == EPI_CHEB4 || EPI == EPI_CHEB1) {
    dv = A.d[slot];
    if (!A.x_zero) o0 = A.x[slot];
    o1 = epi_op<EPI>(A, 1)[slot];
    o2 = A.invd[slot];
  } else {
    if constexpr (EpiOps<EPI>::n > 0) o0 = epi_op<EPI>(A, 0)[slot];
    if constexpr (EpiOps<EPI>::n > 1) o1 = epi_op<EPI>(A, 1)[slot];
    if constexpr (EpiOps<EPI>::n > 2) o2 = epi_op<EPI>(A, 2)[slot];
  }
  const double* sh = A.shell + e * A.nshell;
  const bool top = ez + 1 >= A.Ezl;  // the dz=1 contributions come from the halo
  double vals[8];
#pragma unroll
  for (int cidx = 0; cidx < 8; ++cidx) {
    if (cidx < n) {
      const int p = __ldg(tab + 1 + cidx);
      const int off = p & 0x0fffffff, f = (unsigned)p >> 28;
      if (top && (f & 4)) {
        // halo: k=0 face of the layer above, indexed by (ex', ey', i', j')
        const int dx = f & 1, dy = (f >> 1) & 1;
        const int i2 = (a + 1) - dx * N, j2 = (b + 1) - dy * N;
        vals[cidx] = __ldcg(A.contrib_hi + ((long)(ex + dx) + (long)A.Ex * (ey + dy)) * (N1 * N1) + i2 + N1 * j2);
      } else {
        vals[cidx] = sh[off];
      }
    }
  }
  double sum = 0.0;
#pragma unroll
  for (int cidx = 0; cidx < 8; ++cidx)
    if (cidx < n) sum += vals[cidx];
  epilogue<EPI>(A, slot, sum, dv, o0, o1, o2);
}

template <int N, int EPI>
__global__ void k_sem_k2(SemArgs A) {
  // block = K2EB consecutive elements of one (ey, ez) row, one thread per owned
  // shared slot: element coordinates come from the grid, no integer division
  constexpr int NSH = sem_nshared(N);
  const int q = threadIdx.x / NSH;
  const int s = threadIdx.x - q * NSH;
  const int ex = blockIdx.x * k2_eb(N) + q, ey = blockIdx.y, ez = blockIdx.z + A.k2_z0;
  // top-layer blocks (dispatched last: blockIdx.z is the slowest grid index) read the
  // upper rank's contributions: wait for them here instead of on the stream
  if (A.k2_wait && ez == A.Ezl - 1) block_wait_flag(A.k2_wait, A.k2_wait_v);
  if (q >= k2_eb(N) || ex >= A.Ex) return;
  const long e = ex + (long)A.Ex * (ey + (long)A.Ey * ez);
  k2_node<N, EPI>(A, e, ex, ey, ez, s);
}

template <int N, int MODE, int EPI>
void launch_k1(const SemArgs& a, cudaStream_t s) {
  using C = SemC<N>;
  const long ne = a.e_end - a.e_begin;
  if (ne <= 0) return;
  if constexpr (MODE == SEM_AX && N >= 5 && (N + 1) % 2 == 0) {
    // line-contraction kernels (k_sem_k1.cuh), two threads per line.  Default:
    // geometric factors read to registers (k_sem_k1_greg) -- 36.4 vs 33.8
    // GDOF-step/s for the TMA/shared-memory-staged factors (k_sem_k1_lines,
    // CMG_K1_GREG=0) at E=64^3.  Also measured and dropped: 4 threads per line
    // (30.4), 6 or 10 blocks/SM register caps (35.1 / 34.8), a persistent
    // software-pipelined element loop (26.0; spills at its register cap).
    static int greg = -1;
    if (greg < 0) {
      const char* env = std::getenv("CMG_K1_GREG");
      greg = (env && std::atoi(env) == 0) ? 0 : 1;
      CMG_CUDA(cudaFuncSetAttribute(k_sem_k1_greg<N, EPI, 2, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)K3Smem<N, EPI, false>::bytes));
      CMG_CUDA(cudaFuncSetAttribute(k_sem_k1_lines<N, EPI, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)K3Smem<N, EPI>::bytes));
    }
    // L2 prefetch of the element's factors at block start: 1765 vs 1849 us per
    // K1 in isolation (ncu); +0.3% on the power-capped sweep
    static const int pf = [] {
      const char* env = std::getenv("CMG_K1_PREFETCH");
      return (env && std::atoi(env) == 0) ? 0 : 1;
    }();
    constexpr unsigned nt = (N + 1) * (N + 1) * 2;
    SemArgs b = a;
    b.prefetch_g = pf;
    const long LE = (long)a.Ex * a.Ey;  // [e_begin, e_end) is whole element layers
    b.k1_z0 = (int)(a.e_begin / LE);
    const dim3 grid((unsigned)a.Ex, (unsigned)a.Ey, (unsigned)(ne / LE));
    if (greg) k_sem_k1_greg<N, EPI, 2, 8><<<grid, nt, K3Smem<N, EPI, false>::bytes, s>>>(b);
    else k_sem_k1_lines<N, EPI, 2><<<grid, nt, K3Smem<N, EPI>::bytes, s>>>(b);
  } else if constexpr (MODE == SEM_AX) {
    if constexpr (N == 3) {
      // order 3: the register-factor line kernel, one element (one warp) per
      // block, as an A/B knob against the packed low-order kernel below --
      // measured slower (E=64^3 solve 0.308-0.311 vs 0.304 s), so opt-in
      static const int g3 = [] {
        const char* env = std::getenv("CMG_K1_GREG3");
        if (env && std::atoi(env) == 1) {
          CMG_CUDA(cudaFuncSetAttribute(k_sem_k1_greg<3, EPI, 2, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)K3Smem<3, EPI, false>::bytes));
          return 1;
        }
        return 0;
      }();
      if (g3) {
        SemArgs b = a;
        const long LE = (long)a.Ex * a.Ey;
        b.k1_z0 = (int)(a.e_begin / LE);
        const dim3 grid((unsigned)a.Ex, (unsigned)a.Ey, (unsigned)(ne / LE));
        k_sem_k1_greg<3, EPI, 2, 16><<<grid, 32, K3Smem<3, EPI, false>::bytes, s>>>(b);
        CMG_LAUNCH_CHECK();
        return;
      }
    }
    // low orders (coarse p-levels): several elements per block, k-split columns
    constexpr std::size_t smem = K1Smem<N, EPI>::bytes;
    static bool configured = false;
    if (!configured) {
      CMG_CUDA(cudaFuncSetAttribute(k_sem_k1_ax<N, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      configured = true;
    }
    const long blocks = (ne + C::EPB - 1) / C::EPB;
    k_sem_k1_ax<N, EPI><<<(unsigned)blocks, C::NT, smem, s>>>(a);
  } else {
    const long threads = ne * C::NP;
    k_sem_k1_lvec<N, EPI><<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(a);
  }
  CMG_LAUNCH_CHECK();
}

template <int N, int EPI>
void launch_k2(const SemArgs& a, cudaStream_t s) {
  const long ne = a.e_end - a.e_begin;
  if (ne <= 0) return;
  const long per_layer = (long)a.Ex * a.Ey;  // [e_begin, e_end) is whole layers
  SemArgs b = a;
  b.k2_z0 = (int)(a.e_begin / per_layer);
  const dim3 grid((unsigned)((a.Ex + k2_eb(N) - 1) / k2_eb(N)), (unsigned)a.Ey, (unsigned)(ne / per_layer));
  k_sem_k2<N, EPI><<<grid, k2_eb(N) * sem_nshared(N), 0, s>>>(b);
  CMG_LAUNCH_CHECK();
}

template <int N, int MODE>
void dispatch_k1_epi(const SemArgs& a, int epi, cudaStream_t s) {
  switch (epi) {
    case EPI_STORE: return launch_k1<N, MODE, EPI_STORE>(a, s);
    case EPI_ADD: return launch_k1<N, MODE, EPI_ADD>(a, s);
    case EPI_RESID: return launch_k1<N, MODE, EPI_RESID>(a, s);
    case EPI_CHEB4: return launch_k1<N, MODE, EPI_CHEB4>(a, s);
    case EPI_CHEB1: return launch_k1<N, MODE, EPI_CHEB1>(a, s);
    case EPI_CHEB4_INIT: return launch_k1<N, MODE, EPI_CHEB4_INIT>(a, s);
    case EPI_CHEB1_INIT: return launch_k1<N, MODE, EPI_CHEB1_INIT>(a, s);
  }
  throw Error(EINVAL_, "sem_k1: bad epilogue");
}

template <int N>
void dispatch_k1(const SemArgs& a, int mode, int epi, cudaStream_t s) {
  if (mode == SEM_AX) dispatch_k1_epi<N, SEM_AX>(a, epi, s);
  else if (epi == EPI_STORE) launch_k1<N, SEM_LVEC, EPI_STORE>(a, s);
  else if (epi == EPI_ADD) launch_k1<N, SEM_LVEC, EPI_ADD>(a, s);
  else if (epi == EPI_SUPD4) launch_k1<N, SEM_LVEC, EPI_SUPD4>(a, s);
  else if (epi == EPI_SUPD1) launch_k1<N, SEM_LVEC, EPI_SUPD1>(a, s);
  else throw Error(EINVAL_, "sem_k1: LVEC mode supports STORE/ADD/SUPD");
}

template <int N>
void dispatch_k2(const SemArgs& a, int epi, cudaStream_t s) {
  switch (epi) {
    case EPI_STORE: return launch_k2<N, EPI_STORE>(a, s);
    case EPI_ADD: return launch_k2<N, EPI_ADD>(a, s);
    case EPI_RESID: return launch_k2<N, EPI_RESID>(a, s);
    case EPI_CHEB4: return launch_k2<N, EPI_CHEB4>(a, s);
    case EPI_CHEB1: return launch_k2<N, EPI_CHEB1>(a, s);
    case EPI_CHEB4_INIT: return launch_k2<N, EPI_CHEB4_INIT>(a, s);
    case EPI_CHEB1_INIT: return launch_k2<N, EPI_CHEB1_INIT>(a, s);
    case EPI_SUPD4: return launch_k2<N, EPI_SUPD4>(a, s);
    case EPI_SUPD1: return launch_k2<N, EPI_SUPD1>(a, s);
  }
  throw Error(EINVAL_, "sem_k2: bad epilogue");
}

// ---------------------------------------------------------------- pointwise
__global__ void k_cheb4_init_zero(std::size_t n, const double* __restrict__ b,
                                  const double* __restrict__ invd, double c0, double* __restrict__ r,
                                  double* __restrict__ d) {
  for (std::size_t q = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x; q < n;
       q += (std::size_t)gridDim.x * blockDim.x) {
    const double rv = b[q];
    r[q] = rv;
    d[q] = c0 * invd[q] * rv;
  }
}

__global__ void k_cheb1_init_zero(std::size_t n, const double* __restrict__ b,
                                  const double* __restrict__ invd, double theta,
                                  double* __restrict__ z, double* __restrict__ d) {
  for (std::size_t q = blockIdx.x * (std::size_t)blockDim.x + threadIdx.x; q < n;
       q += (std::size_t)gridDim.x * blockDim.x) {
    const double zv = b[q] * invd[q];
    z[q] = zv;
    d[q] = zv / theta;
  }
}

inline unsigned vgrid(std::size_t n) {
  std::size_t g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  return (unsigned)(g < 1 ? 1 : g);
}

// ---------------------------------------------------------------- halo packing
__global__ void k_pack_top(SemArgs A, const double* __restrict__ u, double* __restrict__ buf) {
  const int N = A.N;
  const long n = (long)A.Ex * A.Ey * N * N;
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int ab = (int)(t % (N * N));
  const long exy = t / (N * N);
  const long e = exy + (long)A.Ex * A.Ey * (A.Ezl - 1);
  // the c = N-1 plane: last N^2 shared slots, (b, a) lexicographic
  buf[t] = u[e * sem_nos(N) + sem_nint(N) + (N - 1) * (2 * N - 1) + ab];
}

__global__ void k_pack_contrib_bottom(SemArgs A, double* __restrict__ buf) {
  const int N1 = A.N + 1;
  const long n = (long)A.Ex * A.Ey * N1 * N1;
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int ij = (int)(t % (N1 * N1));
  const long e = t / (N1 * N1);  // layer 0
  buf[t] = A.shell[e * A.nshell + A.lut[ij]];  // k = 0 plane: lut index (0*N1 + j)*N1 + i = ij
}

// ---------------------------------------------------------------- geometry (setup)
__device__ double kr_right(double eps, double x) { return (x <= 0.5) ? (2.0 - eps) * x : 1.0 + eps * (x - 1.0); }
__device__ double kr_left(double eps, double x) { return 1.0 - kr_right(eps, 1.0 - x); }
__device__ double kr_step(double a, double b, double x) {
  if (x <= 0.0) return a;
  if (x >= 1.0) return b;
  return a + (b - a) * (x * x * x * (x * (6.0 * x - 15.0) + 10.0));
}

// Kershaw map (same definition as oracle/oracle_sem.c)
__device__ void kershaw(double eps, double x, double y, double z, double& X, double& Y, double& Z) {
  X = x;
  int layer = (int)(x * 6.0);
  if (layer > 5) layer = 5;
  const double lam = (x - layer / 6.0) * 6.0;
  switch (layer) {
    case 0: Y = kr_left(eps, y); Z = kr_left(eps, z); break;
    case 1:
    case 4:
      Y = kr_step(kr_left(eps, y), kr_right(eps, y), lam);
      Z = kr_step(kr_left(eps, z), kr_right(eps, z), lam);
      break;
    case 2:
      Y = kr_step(kr_right(eps, y), kr_left(eps, y), lam / 2.0);
      Z = kr_step(kr_right(eps, z), kr_left(eps, z), lam / 2.0);
      break;
    case 3:
      Y = kr_step(kr_right(eps, y), kr_left(eps, y), (1.0 + lam) / 2.0);
      Z = kr_step(kr_right(eps, z), kr_left(eps, z), (1.0 + lam) / 2.0);
      break;
    default: Y = kr_right(eps, y); Z = kr_right(eps, z); break;
  }
}

// one block per element, one thread per node
__global__ void k_geometry(SemGeom g, double* __restrict__ G, double* __restrict__ Lrhs,
                           double* __restrict__ Lmass) {
  extern __shared__ double smg[];
  const int N = g.N, N1 = N + 1, NP = N1 * N1 * N1;
  double* X = smg;
  double* Y = smg + NP;
  double* Z = smg + 2 * NP;
  const long e = blockIdx.x;
  const int ex = (int)(e % g.Ex), ey = (int)((e / g.Ex) % g.Ey), ez = g.z0 + (int)(e / ((long)g.Ex * g.Ey));
  for (int l = threadIdx.x; l < NP; l += blockDim.x) {
    const int i = l % N1, j = (l / N1) % N1, k = l / (N1 * N1);
    const double x = ((double)ex + 0.5 * (g.xi[i] + 1.0)) / (double)g.Ex;
    const double y = ((double)ey + 0.5 * (g.xi[j] + 1.0)) / (double)g.Ey;
    const double z = ((double)ez + 0.5 * (g.xi[k] + 1.0)) / (double)g.Ez;
    double u = x, v = y, w = z;
    if (g.geometry == 1) kershaw(g.eps, x, y, z, u, v, w);
    X[l] = u - 0.5;
    Y[l] = v - 0.5;
    Z[l] = w - 0.5;
  }
  __syncthreads();
  for (int l = threadIdx.x; l < NP; l += blockDim.x) {
    const int i = l % N1, j = (l / N1) % N1, k = l / (N1 * N1);
    double Jm[3][3];
    const double* Cc[3] = {X, Y, Z};
    for (int c = 0; c < 3; ++c) {
      double dr = 0, ds = 0, dt = 0;
      for (int m = 0; m < N1; ++m) {
        dr += g.D[i * N1 + m] * Cc[c][m + N1 * (j + N1 * k)];
        ds += g.D[j * N1 + m] * Cc[c][i + N1 * (m + N1 * k)];
        dt += g.D[k * N1 + m] * Cc[c][i + N1 * (j + N1 * m)];
      }
      Jm[c][0] = dr; Jm[c][1] = ds; Jm[c][2] = dt;
    }
    const double det = Jm[0][0] * (Jm[1][1] * Jm[2][2] - Jm[1][2] * Jm[2][1]) -
                       Jm[0][1] * (Jm[1][0] * Jm[2][2] - Jm[1][2] * Jm[2][0]) +
                       Jm[0][2] * (Jm[1][0] * Jm[2][1] - Jm[1][1] * Jm[2][0]);
    double Ji[3][3];
    Ji[0][0] = (Jm[1][1] * Jm[2][2] - Jm[1][2] * Jm[2][1]) / det;
    Ji[0][1] = (Jm[0][2] * Jm[2][1] - Jm[0][1] * Jm[2][2]) / det;
    Ji[0][2] = (Jm[0][1] * Jm[1][2] - Jm[0][2] * Jm[1][1]) / det;
    Ji[1][0] = (Jm[1][2] * Jm[2][0] - Jm[1][0] * Jm[2][2]) / det;
    Ji[1][1] = (Jm[0][0] * Jm[2][2] - Jm[0][2] * Jm[2][0]) / det;
    Ji[1][2] = (Jm[0][2] * Jm[1][0] - Jm[0][0] * Jm[1][2]) / det;
    Ji[2][0] = (Jm[1][0] * Jm[2][1] - Jm[1][1] * Jm[2][0]) / det;
    Ji[2][1] = (Jm[0][1] * Jm[2][0] - Jm[0][0] * Jm[2][1]) / det;
    Ji[2][2] = (Jm[0][0] * Jm[1][1] - Jm[0][1] * Jm[1][0]) / det;
    const double W = g.w[i] * g.w[j] * g.w[k] * det;
    const int pa[6] = {0, 0, 0, 1, 1, 2}, pb[6] = {0, 1, 2, 1, 2, 2};
    for (int q = 0; q < 6; ++q) {
      const int a = pa[q], b = pb[q];
      G[(e * 6 + q) * NP + l] = W * (Ji[a][0] * Ji[b][0] + Ji[a][1] * Ji[b][1] + Ji[a][2] * Ji[b][2]);
    }
    if (Lmass) Lmass[e * NP + l] = W;
    if (Lrhs) {
      const double pi = 3.141592653589793238462643383279502884;
      const double f = 3.0 * pi * pi * sin(pi * X[l]) * sin(pi * Y[l]) * sin(pi * Z[l]);
      Lrhs[e * NP + l] = W * f;
    }
  }
}

// App. A5 diagonal, one block per element
__global__ void k_local_diag(int N, const double* __restrict__ G, const double* __restrict__ D,
                             double* __restrict__ Ld) {
  const int N1 = N + 1, NP = N1 * N1 * N1;
  const long e = blockIdx.x;
  const double* Ge = G + e * 6 * NP;
  for (int l = threadIdx.x; l < NP; l += blockDim.x) {
    const int i = l % N1, j = (l / N1) % N1, k = l / (N1 * N1);
    double v = 0;
    for (int m = 0; m < N1; ++m) {
      v += D[m * N1 + i] * D[m * N1 + i] * Ge[m + N1 * (j + N1 * k)];
      v += D[m * N1 + j] * D[m * N1 + j] * Ge[3 * NP + i + N1 * (m + N1 * k)];
      v += D[m * N1 + k] * D[m * N1 + k] * Ge[5 * NP + i + N1 * (j + N1 * m)];
    }
    v += 2.0 * D[i * N1 + i] * D[j * N1 + j] * Ge[NP + l];
    v += 2.0 * D[i * N1 + i] * D[k * N1 + k] * Ge[2 * NP + l];
    v += 2.0 * D[j * N1 + j] * D[k * N1 + k] * Ge[4 * NP + l];
    Ld[e * NP + l] = v;
  }
}

__device__ __forceinline__ bool slot_valid(const SemArgs& A, long q) {
  const int N = A.N;
  const long NOS = sem_nos(N);
  const long e = q / NOS;
  int a, b, c;
  if (!sem_abc(N, (int)(q - e * NOS), a, b, c)) return false;
  int ex, ey, ez;
  elem_xyz(e, A.Ex, A.Ey, ex, ey, ez);
  return ex * N + a + 1 < N * A.Ex && ey * N + b + 1 < N * A.Ey && (A.z0 + ez) * N + c + 1 < N * A.Ez;
}

__global__ void k_inverse_diag(SemArgs A, const double* __restrict__ d, double* __restrict__ inv,
                               int* zero_flag) {
  const long n = A.E * (long)sem_nos(A.N);
  for (long q = blockIdx.x * (long)blockDim.x + threadIdx.x; q < n; q += (long)gridDim.x * blockDim.x) {
    if (slot_valid(A, q)) {
      const double v = d[q];
      if (v == 0.0) atomicExch(zero_flag, 1);
      inv[q] = 1.0 / v;
    } else {
      inv[q] = 0.0;
    }
  }
}

__global__ void k_flag_zero_valid(SemArgs A, const double* __restrict__ v, int* flag) {
  const long n = A.E * (long)sem_nos(A.N);
  for (long q = blockIdx.x * (long)blockDim.x + threadIdx.x; q < n; q += (long)gridDim.x * blockDim.x)
    if (v[q] == 0.0 && slot_valid(A, q)) atomicExch(flag, 1);
}

__global__ void k_slot_mask(SemArgs A, double* __restrict__ m) {
  const long n = A.E * (long)sem_nos(A.N);
  for (long q = blockIdx.x * (long)blockDim.x + threadIdx.x; q < n; q += (long)gridDim.x * blockDim.x)
    m[q] = slot_valid(A, q) ? 1.0 : 0.0;
}

// ---------------------------------------------------------------- p-transfers
// tepb(NF) elements per 128-thread block (smem staging per element): for the
// small low-order elements each thread then keeps several independent loads in
// flight (prolong/restrict 3->1: 130/108 vs 220/212 us at E=64^3); the order-7
// elements already fill the threads and keep one element per block (more
// blocks per SM: 704/568 vs 857/775 us with four).
constexpr int tepb(int NF) { return NF >= 5 ? 1 : 4; }

template <int NF, int NCO>
__global__ void __launch_bounds__(128) k_prolong(SemArgs F, SemArgs Cc, const double* __restrict__ J,
                                                 const double* __restrict__ xc, double* __restrict__ yf, int add) {
  constexpr int TEPB = tepb(NF);
  constexpr int F1 = NF + 1, C1 = NCO + 1, NOF = NF * NF * NF;
  constexpr int NOSF = sem_nos(NF), NOSC = sem_nos(NCO);
  constexpr int UC = C1 * C1 * C1, T1 = F1 * C1 * C1, T2 = F1 * F1 * C1;
  __shared__ double sJ[F1 * C1];
  __shared__ double uc[TEPB][UC];
  __shared__ double t1[TEPB][T1];
  __shared__ double t2[TEPB][T2];
  __shared__ int sxyz[TEPB][3];  // element coordinates (the divisions done once per element)
  const long e0 = (long)blockIdx.x * TEPB, E = F.e_end;
  for (int q = threadIdx.x; q < F1 * C1; q += blockDim.x) sJ[q] = J[q];
  if (threadIdx.x < TEPB) {
    const long e = e0 + threadIdx.x;
    elem_xyz(e, F.Ex, F.Ey, sxyz[threadIdx.x][0], sxyz[threadIdx.x][1], sxyz[threadIdx.x][2]);
  }
  __syncthreads();
  for (int qq = threadIdx.x; qq < TEPB * UC; qq += blockDim.x) {
    const int le = qq / UC, q = qq - le * UC;
    const long e = e0 + le;
    double v = 0.0;
    if (e < E) {
      const int ex = sxyz[le][0], ey = sxyz[le][1], ez = sxyz[le][2];
      const int a = q % C1, b = (q / C1) % C1, c = q / (C1 * C1);
      int oex = 0, oey = 0, oez = 0;
      const int ax = owner1d<NCO>(ex, a, Cc.Ex, oex);
      const int ay = owner1d<NCO>(ey, b, Cc.Ey, oey);
      const int az = owner1d<NCO>(Cc.z0 + ez, c, Cc.Ez, oez);
      if (ax >= 0 && ay >= 0 && az >= 0) {
        const int lz = oez - Cc.z0;
        if (lz < 0)
          v = Cc.halo_lo[((long)oex + (long)Cc.Ex * oey) * (NCO * NCO) + ax + NCO * ay];
        else
          v = xc[((long)oex + (long)Cc.Ex * ((long)oey + (long)Cc.Ey * lz)) * NOSC + sem_pos(NCO, ax, ay, az)];
      }
    }
    uc[le][q] = v;
  }
  __syncthreads();
  for (int qq = threadIdx.x; qq < TEPB * T1; qq += blockDim.x) {  // contract x
    const int le = qq / T1, q = qq - le * T1;
    const int i = q % F1, b = (q / F1) % C1, c = q / (F1 * C1);
    double v = 0.0;
    for (int m = 0; m < C1; ++m) v = __fma_rn(sJ[i * C1 + m], uc[le][m + C1 * (b + C1 * c)], v);
    t1[le][q] = v;
  }
  __syncthreads();
  for (int qq = threadIdx.x; qq < TEPB * T2; qq += blockDim.x) {  // contract y
    const int le = qq / T2, q = qq - le * T2;
    const int i = q % F1, j = (q / F1) % F1, c = q / (F1 * F1);
    double v = 0.0;
    for (int m = 0; m < C1; ++m) v = __fma_rn(sJ[j * C1 + m], t1[le][i + F1 * (m + C1 * c)], v);
    t2[le][q] = v;
  }
  __syncthreads();
  for (int qq = threadIdx.x; qq < TEPB * NOF; qq += blockDim.x) {  // contract z at owned fine nodes
    const int le = qq / NOF, q = qq - le * NOF;
    const long e = e0 + le;
    if (e >= E) continue;
    const int ex = sxyz[le][0], ey = sxyz[le][1], ez = sxyz[le][2];
    const int a = q % NF, b = (q / NF) % NF, c = q / (NF * NF);
    const int i = a + 1, j = b + 1, k = c + 1;
    if (ex * NF + i >= NF * F.Ex || ey * NF + j >= NF * F.Ey || (F.z0 + ez) * NF + k >= NF * F.Ez) continue;
    double v = 0.0;
    for (int m = 0; m < C1; ++m) v = __fma_rn(sJ[k * C1 + m], t2[le][i + F1 * (j + F1 * m)], v);
    const long slot = e * NOSF + sem_pos(NF, a, b, c);
    yf[slot] = add ? yf[slot] + v : v;
  }
}

// ---------------------------------------------------------------- p-transfers, one warp per element
// The order-7 <-> 3 transfers as warp-level line contractions, the K1 recipe:
// J (8x4) sits in __constant__ memory and every index into it is a
// compile-time constant (a DFMA constant-bank operand, no shared traffic), a
// lane owns whole lines of the contracted direction, a warp owns an element
// (only __syncwarp between the three contractions, ~10 elements in flight
// per scheduler), the element's contiguous fine block is read / written with
// coalesced lane-strided accesses (slot <-> node by sem_pos / sem_abc).  Every output is the same ascending fma chain as k_prolong /
// k_restrict_local (bitwise identical; r01: 704 / 568 us per launch at E=64^3).
__constant__ double c_J73[8 * 4];          // J[i*4 + m] = l^3_m(xi^7_i)  (host_interp_matrix(7, 3))

constexpr int kTW = 4;  // warps (elements) per block

template <int NF, int NCO>
__global__ void __launch_bounds__(32 * kTW) k_restrict_w(SemArgs F, const double* __restrict__ xf,
                                                       double* __restrict__ Lc) {
  static_assert(NF == 7 && NCO == 3, "warp transfer kernels are instantiated for 7 -> 3");
  constexpr int F1 = 8, C1 = 4, P = 9, NOSF = sem_nos(NF);
  // uf (64 lines of 8 along x, node (i,j,k) at (k*8 + j)*P + i) | t1 (32 lines of 8); t2 aliases uf.
  // Local nodes with i, j or k = 0 are not the element's own (zero in the restatement's
  // input): the m = 0 terms are skipped -- fma(J, +0, +0) = +0, so every chain still
  // rounds identically -- and all-zero lines give +0 outputs, so uf needs no zeroing.
  // one 64-line buffer per warp: uf, then t1 (lines 0..31) and t2 (lines 32..47) once the
  // x step has pulled its two uf lines into registers (18 KB per block, 12 blocks per SM)
  __shared__ double sm[kTW][64 * P];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long e = (long)blockIdx.x * kTW + w;
  if (e >= F.e_end) return;
  double* uf = sm[w];
  double* t1 = sm[w];
  double* t2 = sm[w] + 32 * P;
  const double* xe = xf + e * NOSF;
#pragma unroll
  for (int r = 0; r < (NOSF + 31) / 32; ++r) {
    const int q = lane + 32 * r;
    int a, b, c;  // arithmetic inverse of the slot layout
    if (q < NOSF && sem_abc(NF, q, a, b, c)) uf[((c + 1) * F1 + (b + 1)) * P + (a + 1)] = __ldg(xe + q);
  }
  __syncwarp();
  // J^T along x: line (j, k) -> t1[(a*8 + k)*P + j], a = 0..3
  double u2[2][F1];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int L = lane + 32 * h, j = L & 7, k = L >> 3;
#pragma unroll
    for (int m = 1; m < F1; ++m) u2[h][m] = (j == 0 || k == 0) ? 0.0 : uf[(k * F1 + j) * P + m];
  }
  __syncwarp();  // uf fully read: t1 / t2 reuse its storage
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int L = lane + 32 * h, j = L & 7, k = L >> 3;
    const bool zero = j == 0 || k == 0;
#pragma unroll
    for (int a = 0; a < C1; ++a) {
      double v = 0.0;
      if (!zero) {
#pragma unroll
        for (int m = 1; m < F1; ++m) v = __fma_rn(c_J73[m * C1 + a], u2[h][m], v);
      }
      t1[(a * F1 + k) * P + j] = v;
    }
  }
  __syncwarp();
  // J^T along y: line (a, k) -> t2[(a*4 + b)*P + k]  (t1[., j = 0, .] = +0)
  {
    const int a = lane >> 3, k = lane & 7;
    double u[F1];
#pragma unroll
    for (int m = 1; m < F1; ++m) u[m] = t1[(a * F1 + k) * P + m];
#pragma unroll
    for (int b = 0; b < C1; ++b) {
      double v = 0.0;
      if (k != 0) {
#pragma unroll
        for (int m = 1; m < F1; ++m) v = __fma_rn(c_J73[m * C1 + b], u[m], v);
      }
      t2[(a * C1 + b) * P + k] = v;
    }
  }
  __syncwarp();
  // J^T along z: line (a, b) -> Lc[a + 4(b + 4c)]  (t2[., ., k = 0] = +0)
  if (lane < C1 * C1) {
    const int a = lane & 3, b = lane >> 2;
    double u[F1];
#pragma unroll
    for (int m = 1; m < F1; ++m) u[m] = t2[(a * C1 + b) * P + m];
#pragma unroll
    for (int c = 0; c < C1; ++c) {
      double v = 0.0;
#pragma unroll
      for (int m = 1; m < F1; ++m) v = __fma_rn(c_J73[m * C1 + c], u[m], v);
      Lc[e * 64 + a + C1 * (b + C1 * c)] = v;
    }
  }
}

template <int NF, int NCO>
__global__ void __launch_bounds__(32 * kTW) k_prolong_w(SemArgs F, SemArgs Cc, const double* __restrict__ xc,
                                                      double* __restrict__ yf, int add) {
  static_assert(NF == 7 && NCO == 3, "warp transfer kernels are instantiated for 7 -> 3");
  constexpr int F1 = 8, C1 = 4, P = 5, NOSF = sem_nos(NF), NOSC = sem_nos(NCO);
  // per warp: t1 (32 lines of 4) | t2 (64 lines of 4); uc (16 lines of 4) aliases t2
  __shared__ double sm[kTW][32 * P + 64 * P];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long e = (long)blockIdx.x * kTW + w;
  if (e >= F.e_end) return;
  double* t1 = sm[w];
  double* t2 = t1 + 32 * P;
  double* uc = t2;
  double* ye = yf + e * NOSF;
  int ex, ey, ez;
  elem_xyz(e, F.Ex, F.Ey, ex, ey, ez);
  // this lane's fine outputs: lines (i, j) = (L & 7, L >> 3), L = lane, lane + 32, nodes k = 1..7;
  // their old values are loaded first (add) so the loads overlap the gather and contractions
  double old[2][F1 - 1];
  bool line_ok[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int L = lane + 32 * h, i = L & 7, j = L >> 3;
    line_ok[h] = i != 0 && j != 0 && ex * NF + i < NF * F.Ex && ey * NF + j < NF * F.Ey;
#pragma unroll
    for (int k = 1; k < F1; ++k)
      old[h][k - 1] = (add && line_ok[h]) ? ye[sem_pos(NF, (i - 1) & 7, (j - 1) & 7, k - 1)] : 0.0;
  }
  // gather the element's coarse nodal values: uc[(c*4 + b)*P + a]
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int q = lane + 32 * r, a = q & 3, b = (q >> 2) & 3, c = q >> 4;
    int oex = 0, oey = 0, oez = 0;
    const int ax = owner1d<NCO>(ex, a, Cc.Ex, oex);
    const int ay = owner1d<NCO>(ey, b, Cc.Ey, oey);
    const int az = owner1d<NCO>(Cc.z0 + ez, c, Cc.Ez, oez);
    double v = 0.0;
    if (ax >= 0 && ay >= 0 && az >= 0) {
      const int lz = oez - Cc.z0;
      if (lz < 0)
        v = Cc.halo_lo[((long)oex + (long)Cc.Ex * oey) * (NCO * NCO) + ax + NCO * ay];
      else
        v = __ldg(xc + ((long)oex + (long)Cc.Ex * ((long)oey + (long)Cc.Ey * lz)) * NOSC + sem_pos(NCO, ax, ay, az));
    }
    uc[(c * C1 + b) * P + a] = v;
  }
  __syncwarp();
  // J along x: line (b, c) -> t1[(i*4 + c)*P + b]
  if (lane < C1 * C1) {
    const int b = lane & 3, c = lane >> 2;
    double u[C1];
#pragma unroll
    for (int m = 0; m < C1; ++m) u[m] = uc[(c * C1 + b) * P + m];
#pragma unroll
    for (int i = 0; i < F1; ++i) {
      double v = 0.0;
#pragma unroll
      for (int m = 0; m < C1; ++m) v = __fma_rn(c_J73[i * C1 + m], u[m], v);
      t1[(i * C1 + c) * P + b] = v;
    }
  }
  __syncwarp();
  // J along y: line (i, c) -> t2[(j*8 + i)*P + c]
  {
    const int i = lane >> 2, c = lane & 3;
    double u[C1];
#pragma unroll
    for (int m = 0; m < C1; ++m) u[m] = t1[(i * C1 + c) * P + m];
    __syncwarp();  // uc (aliased by t2) fully consumed by the x step
#pragma unroll
    for (int j = 0; j < F1; ++j) {
      double v = 0.0;
#pragma unroll
      for (int m = 0; m < C1; ++m) v = __fma_rn(c_J73[j * C1 + m], u[m], v);
      t2[(j * F1 + i) * P + c] = v;
    }
  }
  __syncwarp();
  // J along z at the owned fine nodes (i, j, k >= 1), written straight to the fine block
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if (!line_ok[h]) continue;
    const int L = lane + 32 * h, i = L & 7, j = L >> 3;
    double u[C1];
#pragma unroll
    for (int m = 0; m < C1; ++m) u[m] = t2[(j * F1 + i) * P + m];
#pragma unroll
    for (int k = 1; k < F1; ++k) {
      if ((F.z0 + ez) * NF + k >= NF * F.Ez) continue;  // padding (far boundary)
      double v = 0.0;
#pragma unroll
      for (int m = 0; m < C1; ++m) v = __fma_rn(c_J73[k * C1 + m], u[m], v);
      ye[sem_pos(NF, i - 1, j - 1, k - 1)] = add ? old[h][k - 1] + v : v;
    }
  }
}

// constant tables of the warp transfer kernels (once per device)
void upload_transfer_tables() {
  static bool done[64] = {};
  int dev = 0;
  CMG_CUDA(cudaGetDevice(&dev));
  if (dev < 64 && done[dev]) return;
  double J[8 * 4];
  host_interp_matrix(7, 3, J);
  CMG_CUDA(cudaMemcpyToSymbol(c_J73, J, sizeof J));
  if (dev < 64) done[dev] = true;
}

// High orders (NF >= 5): the element's owned fine slots are ONE contiguous
// block of NOS doubles (sem_layout.hpp), so the read-modify-write of the fine
// vector is a TMA bulk load at block start (overlapping the coarse gather and
// the x/y contractions) and a single bulk store of the finished block -- full
// sectors both ways instead of 343 scattered 8-byte accesses.  Padding slots
// keep their value (add) or are written 0.  Same arithmetic, same bits as
// k_prolong (r01: 704 us at E=64^3, ~30% of HBM).
template <int NF, int NCO>
__global__ void __launch_bounds__(128) k_prolong_tma(SemArgs F, SemArgs Cc, const double* __restrict__ J,
                                                     const double* __restrict__ xc, double* __restrict__ yf,
                                                     int add) {
  constexpr int F1 = NF + 1, C1 = NCO + 1, NOF = NF * NF * NF;
  constexpr int NOSF = sem_nos(NF), NOSC = sem_nos(NCO);
  constexpr int UC = C1 * C1 * C1, T1 = F1 * C1 * C1, T2 = F1 * F1 * C1;
  static_assert((NOSF * 8) % 16 == 0, "bulk copies need 16-byte multiples");
  __shared__ __align__(128) double sy[NOSF];
  __shared__ double sJ[F1 * C1];
  __shared__ double uc[UC];
  __shared__ double t1[T1];
  __shared__ double t2[T2];
  __shared__ __align__(8) unsigned long long bar;
  const long e = blockIdx.x;
  double* ye = yf + e * NOSF;
  if (add && threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_expect_tx(&bar, NOSF * 8);
    bulk_g2s(sy, ye, NOSF * 8, &bar);
  }
  if (!add)
    for (int q = threadIdx.x; q < NOSF; q += blockDim.x) sy[q] = 0.0;
  for (int q = threadIdx.x; q < F1 * C1; q += blockDim.x) sJ[q] = J[q];
  int ex, ey, ez;
  elem_xyz(e, F.Ex, F.Ey, ex, ey, ez);
  for (int q = threadIdx.x; q < UC; q += blockDim.x) {
    const int a = q % C1, b = (q / C1) % C1, c = q / (C1 * C1);
    int oex = 0, oey = 0, oez = 0;
    const int ax = owner1d<NCO>(ex, a, Cc.Ex, oex);
    const int ay = owner1d<NCO>(ey, b, Cc.Ey, oey);
    const int az = owner1d<NCO>(Cc.z0 + ez, c, Cc.Ez, oez);
    double v = 0.0;
    if (ax >= 0 && ay >= 0 && az >= 0) {
      const int lz = oez - Cc.z0;
      if (lz < 0)
        v = Cc.halo_lo[((long)oex + (long)Cc.Ex * oey) * (NCO * NCO) + ax + NCO * ay];
      else
        v = xc[((long)oex + (long)Cc.Ex * ((long)oey + (long)Cc.Ey * lz)) * NOSC + sem_pos(NCO, ax, ay, az)];
    }
    uc[q] = v;
  }
  __syncthreads();
  for (int q = threadIdx.x; q < T1; q += blockDim.x) {  // contract x
    const int i = q % F1, b = (q / F1) % C1, c = q / (F1 * C1);
    double v = 0.0;
    for (int m = 0; m < C1; ++m) v = __fma_rn(sJ[i * C1 + m], uc[m + C1 * (b + C1 * c)], v);
    t1[q] = v;
  }
  __syncthreads();
  for (int q = threadIdx.x; q < T2; q += blockDim.x) {  // contract y
    const int i = q % F1, j = (q / F1) % F1, c = q / (F1 * F1);
    double v = 0.0;
    for (int m = 0; m < C1; ++m) v = __fma_rn(sJ[j * C1 + m], t1[i + F1 * (m + C1 * c)], v);
    t2[q] = v;
  }
  __syncthreads();
  if (add) mbar_wait(&bar, 0);
  for (int q = threadIdx.x; q < NOF; q += blockDim.x) {  // contract z at owned fine nodes
    const int a = q % NF, b = (q / NF) % NF, c = q / (NF * NF);
    const int i = a + 1, j = b + 1, k = c + 1;
    if (ex * NF + i >= NF * F.Ex || ey * NF + j >= NF * F.Ey || (F.z0 + ez) * NF + k >= NF * F.Ez) continue;
    double v = 0.0;
    for (int m = 0; m < C1; ++m) v = __fma_rn(sJ[k * C1 + m], t2[i + F1 * (j + F1 * m)], v);
    const int pos = sem_pos(NF, a, b, c);
    sy[pos] = add ? sy[pos] + v : v;
  }
  fence_proxy_async_smem();
  __syncthreads();
  if (threadIdx.x == 0) {
    bulk_s2g(ye, sy, NOSF * 8);
    bulk_store_wait_read();
  }
}

// Restriction for NF >= 5: the element's owned fine block arrives by one TMA
// bulk load; same contractions and bits as k_restrict_local.
template <int NF, int NCO>
__global__ void __launch_bounds__(128) k_restrict_tma(SemArgs F, const double* __restrict__ J,
                                                      const double* __restrict__ xf, double* __restrict__ Lc) {
  constexpr int F1 = NF + 1, C1 = NCO + 1, CP = C1 * C1 * C1, NOSF = sem_nos(NF);
  constexpr int UF = F1 * F1 * F1, T1 = C1 * F1 * F1, T2 = C1 * C1 * F1;
  static_assert((NOSF * 8) % 16 == 0, "bulk copies need 16-byte multiples");
  __shared__ __align__(128) double sx[NOSF];
  __shared__ double sJ[F1 * C1];
  __shared__ double uf[UF];
  __shared__ double t1[T1];
  __shared__ double t2[T2];
  __shared__ __align__(8) unsigned long long bar;
  const long e = blockIdx.x;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_expect_tx(&bar, NOSF * 8);
    bulk_g2s(sx, xf + e * NOSF, NOSF * 8, &bar);
  }
  for (int q = threadIdx.x; q < F1 * C1; q += blockDim.x) sJ[q] = J[q];
  __syncthreads();
  mbar_wait(&bar, 0);
  for (int q = threadIdx.x; q < UF; q += blockDim.x) {
    const int i = q % F1, j = (q / F1) % F1, k = q / (F1 * F1);
    uf[q] = (i >= 1 && j >= 1 && k >= 1) ? sx[sem_pos(NF, i - 1, j - 1, k - 1)] : 0.0;  // padding slots are zero
  }
  __syncthreads();
  for (int q = threadIdx.x; q < T1; q += blockDim.x) {  // J^T along x
    const int a = q % C1, j = (q / C1) % F1, k = q / (C1 * F1);
    double v = 0.0;
    for (int m = 0; m < F1; ++m) v = __fma_rn(sJ[m * C1 + a], uf[m + F1 * (j + F1 * k)], v);
    t1[q] = v;
  }
  __syncthreads();
  for (int q = threadIdx.x; q < T2; q += blockDim.x) {
    const int a = q % C1, b = (q / C1) % C1, k = q / (C1 * C1);
    double v = 0.0;
    for (int m = 0; m < F1; ++m) v = __fma_rn(sJ[m * C1 + b], t1[a + C1 * (m + F1 * k)], v);
    t2[q] = v;
  }
  __syncthreads();
  for (int q = threadIdx.x; q < CP; q += blockDim.x) {
    const int a = q % C1, b = (q / C1) % C1, c = q / (C1 * C1);
    double v = 0.0;
    for (int m = 0; m < F1; ++m) v = __fma_rn(sJ[m * C1 + c], t2[a + C1 * (b + C1 * m)], v);
    Lc[e * CP + q] = v;
  }
}

template <int NF, int NCO>
__global__ void __launch_bounds__(128) k_restrict_local(SemArgs F, const double* __restrict__ J,
                                                        const double* __restrict__ xf, double* __restrict__ Lc) {
  constexpr int TEPB = tepb(NF);
  constexpr int F1 = NF + 1, C1 = NCO + 1, CP = C1 * C1 * C1, NOSF = sem_nos(NF);
  constexpr int UF = F1 * F1 * F1, T1 = C1 * F1 * F1, T2 = C1 * C1 * F1;
  __shared__ double sJ[F1 * C1];
  __shared__ double uf[TEPB][UF];
  __shared__ double t1[TEPB][T1];
  __shared__ double t2[TEPB][T2];
  const long e0 = (long)blockIdx.x * TEPB, E = F.e_end;
  for (int q = threadIdx.x; q < F1 * C1; q += blockDim.x) sJ[q] = J[q];
  for (int qq = threadIdx.x; qq < TEPB * UF; qq += blockDim.x) {
    const int le = qq / UF, q = qq - le * UF;
    const long e = e0 + le;
    const int i = q % F1, j = (q / F1) % F1, k = q / (F1 * F1);
    double v = 0.0;
    if (e < E && i >= 1 && j >= 1 && k >= 1) v = xf[e * NOSF + sem_pos(NF, i - 1, j - 1, k - 1)];
    uf[le][q] = v;  // padding slots are zero
  }
  __syncthreads();
  for (int qq = threadIdx.x; qq < TEPB * T1; qq += blockDim.x) {  // J^T along x
    const int le = qq / T1, q = qq - le * T1;
    const int a = q % C1, j = (q / C1) % F1, k = q / (C1 * F1);
    double v = 0.0;
    for (int m = 0; m < F1; ++m) v = __fma_rn(sJ[m * C1 + a], uf[le][m + F1 * (j + F1 * k)], v);
    t1[le][q] = v;
  }
  __syncthreads();
  for (int qq = threadIdx.x; qq < TEPB * T2; qq += blockDim.x) {
    const int le = qq / T2, q = qq - le * T2;
    const int a = q % C1, b = (q / C1) % C1, k = q / (C1 * C1);
    double v = 0.0;
    for (int m = 0; m < F1; ++m) v = __fma_rn(sJ[m * C1 + b], t1[le][a + C1 * (m + F1 * k)], v);
    t2[le][q] = v;
  }
  __syncthreads();
  for (int qq = threadIdx.x; qq < TEPB * CP; qq += blockDim.x) {
    const int le = qq / CP, q = qq - le * CP;
    const long e = e0 + le;
    if (e >= E) continue;
    const int a = q % C1, b = (q / C1) % C1, c = q / (C1 * C1);
    double v = 0.0;
    for (int m = 0; m < F1; ++m) v = __fma_rn(sJ[m * C1 + c], t2[le][a + C1 * (b + C1 * m)], v);
    Lc[e * CP + q] = v;
  }
}

// ---------------------------------------------------------------- layer dots
// partials[(v*L + layer)*LCH + chunk]
constexpr int LCH = 32;
// MAXC: 8 in general, 1 for the single dots (norms, <v, w>): one accumulator
// leaves the registers to unroll the stride loop so several loads are in
// flight per thread. Either way each accumulator sums its terms in ascending
// q and the block reduction is the same, so the partials keep their bits.
template <int MAXC, int UNR = (MAXC == 1 ? 4 : 1)>
__global__ void k_layer_dots(const double* __restrict__ V, std::size_t ldv, int nv,
                             const double* __restrict__ w, long layer_len, int nlayers,
                             double* __restrict__ partials) {
  const int layer = blockIdx.y, chunk = blockIdx.x, v0 = blockIdx.z * 8;
  const int cnt = min(8, nv - v0);
  __shared__ double sh[MAXC][8];
  double acc[MAXC];
#pragma unroll
  for (int c = 0; c < MAXC; ++c) acc[c] = 0.0;
  const long base = (long)layer * layer_len;
  const long step = (long)LCH * blockDim.x;
  long q = (long)chunk * blockDim.x + threadIdx.x;
  if constexpr (MAXC > 1 && UNR > 1) {
    // UNR strides' loads issued together; each accumulator still adds its terms in
    // ascending q, so the partials keep their bits
    for (; q + (UNR - 1) * step < layer_len; q += UNR * step) {
      double wv[UNR], vv[UNR][MAXC];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        wv[u] = w[base + q + u * step];
#pragma unroll
        for (int c = 0; c < MAXC; ++c)
          vv[u][c] = c < cnt ? V[(std::size_t)(v0 + c) * ldv + base + q + u * step] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u)
#pragma unroll
        for (int c = 0; c < MAXC; ++c)
          if (c < cnt) acc[c] += vv[u][c] * wv[u];
    }
  }
#pragma unroll(MAXC == 1 ? 4 : 1)
  for (; q < layer_len; q += step) {
    const double wv = w[base + q];
#pragma unroll
    for (int c = 0; c < MAXC; ++c)
      if (c < cnt) acc[c] += V[(std::size_t)(v0 + c) * ldv + base + q] * wv;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < MAXC; ++c) {
    double v = acc[c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) sh[c][warp] = v;
  }
  __syncthreads();
  if (threadIdx.x < cnt) {
    double s = 0.0;
    for (int wv = 0; wv < (int)(blockDim.x >> 5); ++wv) s += sh[threadIdx.x][wv];
    partials[((long)(v0 + threadIdx.x) * nlayers + layer) * LCH + chunk] = s;
  }
}

// Fused CGS pass over the layered layout: w -= V coef (k_cgs_update's
// arithmetic) and the per-layer partials of V^T w_new with k_layer_dots' exact
// chunking and reduction order -- coefficients are bit-identical to the
// unfused update + layer dots, V is streamed from HBM once.
// MAXV: compile-time bound on nv (8/16/32) so the accumulators of short bases
// do not cost the registers of long ones.
template <int MAXV, int UNR = 1>
__global__ void __launch_bounds__(256) k_layer_cgs_dots(const double* __restrict__ V, std::size_t ldv, int nv,
                                                        const double* __restrict__ coef, double* __restrict__ w,
                                                        long layer_len, int nlayers, double* hcol, int hstride,
                                                        double* __restrict__ partials) {
  const int layer = blockIdx.y, chunk = blockIdx.x;
  __shared__ double c[MAXV];
  __shared__ double sh[MAXV][8];
  for (int l = threadIdx.x; l < nv; l += blockDim.x) c[l] = coef[l];
  __syncthreads();
  if (layer == 0 && chunk == 0 && threadIdx.x == 0)
    for (int l = 0; l < nv; ++l) hcol[(std::size_t)l * hstride] += c[l];
  double acc[MAXV];
#pragma unroll
  for (int q = 0; q < MAXV; ++q) acc[q] = 0.0;
  const long base = (long)layer * layer_len;
  const long step = (long)LCH * blockDim.x;
  long q0 = (long)chunk * blockDim.x + threadIdx.x;
  if constexpr (UNR > 1 && MAXV <= 16) {
    // UNR strides at once: all their loads in flight together; per entry the same
    // update chain, per accumulator the same ascending-q order (same bits)
    for (; q0 + (UNR - 1) * step < layer_len; q0 += UNR * step) {
      double v[UNR], vv[UNR][MAXV];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const std::size_t i = base + q0 + u * step;
        v[u] = w[i];
#pragma unroll
        for (int l = 0; l < MAXV; ++l) vv[u][l] = l < nv ? V[(std::size_t)l * ldv + i] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
#pragma unroll
        for (int l = 0; l < MAXV; ++l)
          if (l < nv) v[u] = __dadd_rn(v[u], __dmul_rn(-c[l], vv[u][l]));
        w[base + q0 + u * step] = v[u];
#pragma unroll
        for (int l = 0; l < MAXV; ++l)
          if (l < nv) acc[l] += vv[u][l] * v[u];
      }
    }
  }
  for (long q = q0; q < layer_len; q += step) {
    const std::size_t i = base + q;
    double v = w[i];
    if constexpr (MAXV <= 16) {  // the basis entries stay in registers for both uses
      double vv[MAXV];
#pragma unroll
      for (int l = 0; l < MAXV; ++l) vv[l] = l < nv ? V[(std::size_t)l * ldv + i] : 0.0;
      // unfused multiply-add, as k_cgs_update (k_blas.cu is built with --fmad=false)
#pragma unroll
      for (int l = 0; l < MAXV; ++l)
        if (l < nv) v = __dadd_rn(v, __dmul_rn(-c[l], vv[l]));
      w[i] = v;
#pragma unroll
      for (int l = 0; l < MAXV; ++l)
        if (l < nv) acc[l] += vv[l] * v;
    } else {
      for (int l = 0; l < nv; ++l) v = __dadd_rn(v, __dmul_rn(-c[l], V[(std::size_t)l * ldv + i]));
      w[i] = v;
#pragma unroll
      for (int l = 0; l < MAXV; ++l)
        if (l < nv) acc[l] += V[(std::size_t)l * ldv + i] * v;
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int l = 0; l < MAXV; ++l) {
    if (l < nv) {
      double v = acc[l];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
      if (lane == 0) sh[l][warp] = v;
    }
  }
  __syncthreads();
  if (threadIdx.x < nv) {
    double s = 0.0;
    for (int wv = 0; wv < (int)(blockDim.x >> 5); ++wv) s += sh[threadIdx.x][wv];
    partials[((long)threadIdx.x * nlayers + layer) * LCH + chunk] = s;
  }
}

__global__ void k_layer_reduce(const double* __restrict__ partials, int nv, int nlayers,
                               double* __restrict__ out) {
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long)nv * nlayers) return;
  double s = 0.0;
  for (int c = 0; c < LCH; ++c) s += partials[t * LCH + c];
  out[t] = s;  // out[v*nlayers + layer]
}

// One GPU: k_layer_reduce and k_layer_finalize in one launch, block per vector --
// each layer's chunk sum in k_layer_reduce's order, then the layers in
// k_layer_finalize's ascending order, so the result has the same bits.
__global__ void k_layer_reduce_final(const double* __restrict__ partials, int nlayers, double* __restrict__ out,
                                     int do_sqrt) {
  extern __shared__ double lsum[];
  const int v = blockIdx.x;
  for (int l = threadIdx.x; l < nlayers; l += blockDim.x) {
    const double* p = partials + ((long)v * nlayers + l) * LCH;
    double s = 0.0;
    for (int c = 0; c < LCH; ++c) s += p[c];
    lsum[l] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int l = 0; l < nlayers; ++l) s += lsum[l];
    out[v] = do_sqrt ? sqrt(s) : s;
  }
}

__global__ void k_layer_finalize(const double* __restrict__ g, int nv, const int* __restrict__ lpr,
                                 int nranks, double* __restrict__ out, int do_sqrt) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  double s = 0.0;
  long off = 0;
  for (int r = 0; r < nranks; ++r) {
    const int L = lpr[r];
    for (int l = 0; l < L; ++l) s += g[off + (long)v * L + l];
    off += (long)nv * L;
  }
  out[v] = do_sqrt ? sqrt(s) : s;
}

}  // namespace

// ====================================================================== host launchers
#define CMG_ORDERS(X) X(1) X(2) X(3) X(4) X(5) X(7)

void sem_k1(const SemArgs& a, int mode, int epi, cudaStream_t s) {
#define X(n) if (a.N == n) return dispatch_k1<n>(a, mode, epi, s);
  CMG_ORDERS(X)
#undef X
  throw Error(EINVAL_, "SEM order must be one of 1,2,3,4,5,7");
}

void sem_k2(const SemArgs& a, int epi, cudaStream_t s) {
#define X(n) if (a.N == n) return dispatch_k2<n>(a, epi, s);
  CMG_ORDERS(X)
#undef X
  throw Error(EINVAL_, "SEM order must be one of 1,2,3,4,5,7");
}

void sem_set_derivative(int N, const double* D_host) {
  CMG_CUDA(cudaMemcpyToSymbol(c_D, D_host, (N + 1) * (N + 1) * sizeof(double), (std::size_t)N * 64 * sizeof(double)));
}

void sem_cheb4_init_zero(std::size_t n, const double* b, const double* invd, double c0, double* r,
                         double* d, cudaStream_t s) {
  k_cheb4_init_zero<<<vgrid(n), 256, 0, s>>>(n, b, invd, c0, r, d);
  CMG_LAUNCH_CHECK();
}

void sem_cheb1_init_zero(std::size_t n, const double* b, const double* invd, double theta,
                         double* z, double* d, cudaStream_t s) {
  k_cheb1_init_zero<<<vgrid(n), 256, 0, s>>>(n, b, invd, theta, z, d);
  CMG_LAUNCH_CHECK();
}

void sem_pack_top(const SemArgs& a, const double* u, double* buf, cudaStream_t s) {
  const long n = (long)a.Ex * a.Ey * a.N * a.N;
  k_pack_top<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(a, u, buf);
  CMG_LAUNCH_CHECK();
}

void sem_pack_contrib_bottom(const SemArgs& a, double* buf, cudaStream_t s) {
  const long n = (long)a.Ex * a.Ey * (a.N + 1) * (a.N + 1);
  k_pack_contrib_bottom<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(a, buf);
  CMG_LAUNCH_CHECK();
}

void sem_geometry(const SemGeom& g, double* G, double* Lrhs, double* Lmass, cudaStream_t s) {
  const long E = (long)g.Ex * g.Ey * g.Ezl;
  const int NP = (g.N + 1) * (g.N + 1) * (g.N + 1);
  k_geometry<<<(unsigned)E, 128, 3 * NP * sizeof(double), s>>>(g, G, Lrhs, Lmass);
  CMG_LAUNCH_CHECK();
}

void sem_local_diag(int N, long E, const double* G, const double* D, double* Ldiag, cudaStream_t s) {
  k_local_diag<<<(unsigned)E, 128, 0, s>>>(N, G, D, Ldiag);
  CMG_LAUNCH_CHECK();
}

void sem_inverse_diag(const SemArgs& a, const double* diag, double* invd, int* zero_flag,
                      cudaStream_t s) {
  const std::size_t n = (std::size_t)a.E * sem_nos(a.N);
  k_inverse_diag<<<vgrid(n), 256, 0, s>>>(a, diag, invd, zero_flag);
  CMG_LAUNCH_CHECK();
}

void sem_flag_zero_valid(const SemArgs& a, const double* v, int* flag, cudaStream_t s) {
  const std::size_t n = (std::size_t)a.E * sem_nos(a.N);
  k_flag_zero_valid<<<vgrid(n), 256, 0, s>>>(a, v, flag);
  CMG_LAUNCH_CHECK();
}

void sem_slot_mask(const SemArgs& a, double* mask, cudaStream_t s) {
  const std::size_t n = (std::size_t)a.E * sem_nos(a.N);
  k_slot_mask<<<vgrid(n), 256, 0, s>>>(a, mask);
  CMG_LAUNCH_CHECK();
}

// CMG_TRANSFER_KERNEL: 2 (default) warp-per-element kernels for 7 <-> 3,
// 1 the block kernels with TMA bulk copies (order >= 5), 0 the plain block kernels
static int transfer_kernel() {
  static const int k = [] {
    const char* env = std::getenv("CMG_TRANSFER_KERNEL");
    return env ? std::atoi(env) : 2;
  }();
  return k;
}

template <int NF, int NCO>
static void prolong_t(const SemArgs& f, const SemArgs& c, const double* J, const double* xc, double* yf,
                      bool add, cudaStream_t s) {
  SemArgs ff = f;
  ff.e_end = f.E;
  const bool tma = transfer_kernel() == 1;
  if constexpr (NF == 7 && NCO == 3) {
    if (transfer_kernel() == 2) {
      upload_transfer_tables();
      k_prolong_w<7, 3><<<(unsigned)((f.E + kTW - 1) / kTW), 32 * kTW, 0, s>>>(ff, c, xc, yf, add ? 1 : 0);
      CMG_LAUNCH_CHECK();
      return;
    }
  }
  if (NF >= 5 && tma)
    k_prolong_tma<NF, NCO><<<(unsigned)f.E, 128, 0, s>>>(ff, c, J, xc, yf, add ? 1 : 0);
  else
    k_prolong<NF, NCO><<<(unsigned)((f.E + tepb(NF) - 1) / tepb(NF)), 128, 0, s>>>(ff, c, J, xc, yf, add ? 1 : 0);
  CMG_LAUNCH_CHECK();
}

template <int NF, int NCO>
static void restrict_t(const SemArgs& f, const double* J, const double* xf, double* Lc, cudaStream_t s) {
  SemArgs ff = f;
  ff.e_end = f.E;
  const bool tma = transfer_kernel() == 1;
  if constexpr (NF == 7 && NCO == 3) {
    if (transfer_kernel() == 2) {
      upload_transfer_tables();
      k_restrict_w<7, 3><<<(unsigned)((f.E + kTW - 1) / kTW), 32 * kTW, 0, s>>>(ff, xf, Lc);
      CMG_LAUNCH_CHECK();
      return;
    }
  }
  if (NF >= 5 && tma)
    k_restrict_tma<NF, NCO><<<(unsigned)f.E, 128, 0, s>>>(ff, J, xf, Lc);
  else
    k_restrict_local<NF, NCO><<<(unsigned)((f.E + tepb(NF) - 1) / tepb(NF)), 128, 0, s>>>(ff, J, xf, Lc);
  CMG_LAUNCH_CHECK();
}

#define CMG_PAIRS(X) X(7, 3) X(7, 5) X(5, 3) X(3, 1) X(7, 1) X(5, 1) X(4, 2) X(2, 1) X(3, 2) X(4, 1)

void sem_prolong(const SemArgs& f, const SemArgs& c, const double* J, const double* xc, double* yf,
                 bool add, cudaStream_t s) {
#define X(a, b) if (f.N == a && c.N == b) return prolong_t<a, b>(f, c, J, xc, yf, add, s);
  CMG_PAIRS(X)
#undef X
  throw Error(EINVAL_, "unsupported p-multigrid order pair");
}

void sem_restrict_local(const SemArgs& f, int Nc, const double* J, const double* xf, double* Lc,
                        cudaStream_t s) {
#define X(a, b) if (f.N == a && Nc == b) return restrict_t<a, b>(f, J, xf, Lc, s);
  CMG_PAIRS(X)
#undef X
  throw Error(EINVAL_, "unsupported p-multigrid order pair");
}

static void layer_reduce_launch(const double* partials, int nv, int nlayers, double* out, double* final_out,
                                int do_sqrt, cudaStream_t s) {
  if (final_out) {
    k_layer_reduce_final<<<(unsigned)nv, 128, (std::size_t)nlayers * sizeof(double), s>>>(partials, nlayers,
                                                                                         final_out, do_sqrt);
  } else {
    const long t = (long)nv * nlayers;
    k_layer_reduce<<<(unsigned)((t + 127) / 128), 128, 0, s>>>(partials, nv, nlayers, out);
  }
  CMG_LAUNCH_CHECK();
}

void sem_layer_dots(const double* V, std::size_t ldv, int nv, const double* w, long layer_len,
                    int nlayers, double* partials, double* out, cudaStream_t s, double* final_out, int do_sqrt) {
  dim3 grid(LCH, nlayers, (nv + 7) / 8);
  // CMG_DOTS_UNROLL: strides per load batch of the multi-dots (E=64^3 solve, 8 launches:
  // 1 -> 11.2 ms at 3.4 TB/s, 2 -> 8.6 ms, 4 -> 6.6 ms at 5.8 TB/s; profiles/r02/ab_dots.txt)
  static const int unr = [] {
    const char* env = std::getenv("CMG_DOTS_UNROLL");
    return env ? std::atoi(env) : 4;
  }();
  if (nv == 1)
    k_layer_dots<1><<<grid, 256, 0, s>>>(V, ldv, nv, w, layer_len, nlayers, partials);
  else if (unr >= 4)
    k_layer_dots<8, 4><<<grid, 256, 0, s>>>(V, ldv, nv, w, layer_len, nlayers, partials);
  else if (unr == 2)
    k_layer_dots<8, 2><<<grid, 256, 0, s>>>(V, ldv, nv, w, layer_len, nlayers, partials);
  else
    k_layer_dots<8, 1><<<grid, 256, 0, s>>>(V, ldv, nv, w, layer_len, nlayers, partials);
  CMG_LAUNCH_CHECK();
  layer_reduce_launch(partials, nv, nlayers, out, final_out, do_sqrt, s);
}

void sem_layer_cgs_dots(const double* V, std::size_t ldv, int nv, const double* coef, double* w, long layer_len,
                        int nlayers, double* hcol, int hstride, double* partials, double* out, cudaStream_t s,
                        double* final_out) {
  dim3 grid(LCH, nlayers, 1);
  // CMG_CGS_UNROLL: strides per load batch of the fused CGS pass (8 launches at E=64^3:
  // 1 -> 10.3 ms at 3.6 TB/s, 2 -> 7.2 ms at 5.2 TB/s; profiles/r02/ab_dots.txt)
  static const int unr = [] {
    const char* env = std::getenv("CMG_CGS_UNROLL");
    return env ? std::atoi(env) : 2;
  }();
  if (nv <= 8 && unr >= 3)
    k_layer_cgs_dots<8, 3><<<grid, 256, 0, s>>>(V, ldv, nv, coef, w, layer_len, nlayers, hcol, hstride, partials);
  else if (nv <= 8 && unr == 2)
    k_layer_cgs_dots<8, 2><<<grid, 256, 0, s>>>(V, ldv, nv, coef, w, layer_len, nlayers, hcol, hstride, partials);
  else if (nv <= 8) k_layer_cgs_dots<8><<<grid, 256, 0, s>>>(V, ldv, nv, coef, w, layer_len, nlayers, hcol, hstride, partials);
  else if (nv <= 16 && unr >= 2)
    k_layer_cgs_dots<16, 2><<<grid, 256, 0, s>>>(V, ldv, nv, coef, w, layer_len, nlayers, hcol, hstride, partials);
  else if (nv <= 16) k_layer_cgs_dots<16><<<grid, 256, 0, s>>>(V, ldv, nv, coef, w, layer_len, nlayers, hcol, hstride, partials);
  else k_layer_cgs_dots<32><<<grid, 256, 0, s>>>(V, ldv, nv, coef, w, layer_len, nlayers, hcol, hstride, partials);
  CMG_LAUNCH_CHECK();
  layer_reduce_launch(partials, nv, nlayers, out, final_out, 0, s);
}

void sem_layer_finalize(const double* gathered, int nv, const int* lpr, int nranks, double* out,
                        int do_sqrt, cudaStream_t s) {
  k_layer_finalize<<<(nv + 63) / 64, 64, 0, s>>>(gathered, nv, lpr, nranks, out, do_sqrt);
  CMG_LAUNCH_CHECK();
}

}  // namespace cmg
