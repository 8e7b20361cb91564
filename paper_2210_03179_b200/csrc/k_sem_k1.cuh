// k_sem_k1.cuh -- the fused SEM element kernel (K1, AX mode) used for the
// high p-levels.  Included by k_sem.cu (needs its helpers: SemC, EpiOps,
// epi_op, epilogue, owner1d, TMA/mbarrier wrappers, c_D, K3Smem).
//
// One element per block of 2(N+1)^2 threads.  Every tensor contraction is a
// "line contraction": the N+1 values of a line along the contracted direction
// are loaded once from shared memory and multiplied by the GLL derivative
// matrix held in __constant__ memory (no shared traffic for D).  Each line is
// split between two threads (half H of the outputs each); the phases between
// barriers are templates on H so every D index is a compile-time constant,
// and the barriers themselves stay in uniform control flow.
//   1. thread 0: TMA bulk copies of the element's 6 geometric factors
//      (24.6 KB at N=7) and of the interior blocks of the epilogue operands;
//   2. all threads: branch-free gather of Q u (all loads issued before any
//      store, so the element pays one memory latency, not KH);
//   3. gradient (r rows, s columns, t on the thread's column) -> G_e grad u;
//   4. divergence (r rows, s columns accumulate, t on the column) ->
//      epilogue: interior nodes finished in place, shell nodes to K2.
// The thread's own half of its column stays in registers between the phases
// (the gathered u values for the t-gradient and the epilogue, its w_t values
// for the t-divergence); only the partner's half goes through shared memory.
// (k_sem_k1_greg, the default, reads the factors into registers instead of 1.)

// Element of this K1 block.  The grid is (Ex, Ey, layers) from layer A.k1_z0 on,
// so the coordinates need no division (64-bit divisions by the runtime Ex, Ey
// were ~10% of K1's instructions).  With an in-kernel halo wait (A.k1_wait) the
// layers are rotated by one: layers 1.. come first and the layer-0 blocks, the
// only readers of the lower rank's halo, are dispatched last (z is the slowest
// grid index).
struct K1Elem {
  int ex, ey, ez;  // ez: local layer
  long e;
};
__device__ __forceinline__ K1Elem k1_element(const SemArgs& A) {
  int zb = blockIdx.z;
  if (A.k1_wait && ++zb == (int)gridDim.z) zb = 0;
  K1Elem r;
  r.ex = blockIdx.x;
  r.ey = blockIdx.y;
  r.ez = A.k1_z0 + zb;
  r.e = r.ex + (long)A.Ex * (r.ey + (long)A.Ey * r.ez);
  return r;
}
__device__ __forceinline__ void k1_halo_wait(const SemArgs& A, const K1Elem& el) {
  if (A.k1_wait && el.ez == 0) block_wait_flag(A.k1_wait, A.k1_wait_v);
}

template <int N, int EPI, int KS>
struct K1L {
  using S = K3Smem<N, EPI>;
  static constexpr int N1 = N + 1, NP = N1 * N1 * N1, NOS = sem_nos(N), NOPS = S::NOPS, NIP = S::NIP;
  static constexpr int R = N1 + 1, KH = N1 / KS;
  static_assert(N1 % KS == 0, "line split must divide N+1");
  // Shared-memory position of node (i,j,k) in the u/r/s line buffers.  A warp's
  // 32 threads own lines (ta, tb), ta in 0..7 and tb in 4 consecutive values,
  // and each LDS.64/STS.64 is one wavefront only if the 32 addresses are
  // distinct mod 32 doubles.  The padded layout (row pitch N+2) is conflict-free
  // along i and j but 2-way for the thread's own column (i = ta, j = tb), which
  // the gather, geometry, t-contraction and epilogue touch 28 loads + 16 stores
  // per element (ncu: 29% / 38% excess shared wavefronts, L1 data pipe 92-95%).
  // For N+1 = 8 the XOR-swizzled layout 72k + 8j + (i ^ j) is conflict-free in
  // all three directions (column 8(tb + k) + (ta ^ tb), j-lines 8(tb + m) +
  // (ta ^ m), i-lines 8(ta + tb) + (m ^ ta)); each row stays a permutation of
  // its 8 slots.  Measured: L1 pipe 95 -> 81%, K1 1.70 -> 1.64 ms, sweep +3.7%
  // (profiles/r02/ab_k1_swizzle_grid3.txt; before the division-free grid the
  // extra XOR address math cost more than it saved, ab_k1_xor_swizzle.log).
  static constexpr bool SWZ = (N1 == 8);
  __device__ static constexpr int idx(int i, int j, int k) {
    if constexpr (SWZ) return k * 72 + j * 8 + (i ^ j);
    else return ((k * N1 + j) * R + i);
  }

  template <int H>
  __device__ static void gather(const SemArgs& A, double* su, int ta, int tb, const K1Elem& el, double* own) {
    constexpr int O0 = H * KH;
    const int ex = el.ex, ey = el.ey, ez = el.ez;
    int oex = 0, oey = 0;
    const int ax = owner1d<N>(ex, ta, A.Ex, oex);
    const int ay = owner1d<N>(ey, tb, A.Ey, oey);
    const bool xy_ok = ax >= 0 && ay >= 0;
    const double* ptr[KH];
    bool ok[KH], from_halo[KH];
#pragma unroll
    for (int q = 0; q < KH; ++q) {
      int oez = 0;
      const int az = owner1d<N>(A.z0 + ez, O0 + q, A.Ez, oez);
      const int lz = oez - A.z0;
      ok[q] = xy_ok && az >= 0;
      const long own = ((long)oex + (long)A.Ex * ((long)oey + (long)A.Ey * lz)) * NOS +
                       sem_pos(N, xy_ok ? ax : 0, xy_ok ? ay : 0, az >= 0 ? az : 0);
      const long halo = ((long)oex + (long)A.Ex * oey) * (N * N) + ax + N * ay;
      from_halo[q] = lz < 0;
      ptr[q] = from_halo[q] ? A.halo_lo + halo : A.u + own;
    }
    double v[KH];
    // the halo may be written by a peer during this kernel (in-kernel wait): L2-only load for it
#pragma unroll
    for (int q = 0; q < KH; ++q) v[q] = ok[q] ? (from_halo[q] ? __ldcg(ptr[q]) : __ldg(ptr[q])) : 0.0;
#pragma unroll
    for (int q = 0; q < KH; ++q) {
      su[idx(ta, tb, O0 + q)] = v[q];
      own[q] = v[q];
    }
  }

  template <int H>
  __device__ static void gradient(const double* su, double* sr, double* ss, int ta, int tb, double* wt,
                                  const double* own) {
    constexpr int O0 = H * KH;
    double l[N1];
#pragma unroll
    for (int m = 0; m < N1; ++m) l[m] = su[idx(m, ta, tb)];
#pragma unroll
    for (int q = 0; q < KH; ++q) {
      double v = 0.0;
#pragma unroll
      for (int m = 0; m < N1; ++m) v = __fma_rn(c_D[N][(O0 + q) * N1 + m], l[m], v);
      sr[idx(O0 + q, ta, tb)] = v;
    }
#pragma unroll
    for (int m = 0; m < N1; ++m) l[m] = su[idx(ta, m, tb)];
#pragma unroll
    for (int q = 0; q < KH; ++q) {
      double v = 0.0;
#pragma unroll
      for (int m = 0; m < N1; ++m) v = __fma_rn(c_D[N][(O0 + q) * N1 + m], l[m], v);
      ss[idx(ta, O0 + q, tb)] = v;
    }
    // the thread's own column: its KH gathered values are still in registers
#pragma unroll
    for (int m = 0; m < N1; ++m) l[m] = (m >= O0 && m < O0 + KH) ? own[m - O0] : su[idx(ta, tb, m)];
#pragma unroll
    for (int q = 0; q < KH; ++q) {
      double v = 0.0;
#pragma unroll
      for (int m = 0; m < N1; ++m) v = __fma_rn(c_D[N][(O0 + q) * N1 + m], l[m], v);
      wt[q] = v;
    }
  }

  template <int H>
  __device__ static void geometry(const double* sG, double* sr, double* ss, int i, int j, double* wt) {
    constexpr int O0 = H * KH;
#pragma unroll
    for (int q = 0; q < KH; ++q) {
      const int k = O0 + q;
      const int l = (k * N1 + j) * N1 + i;
      const double ur = sr[idx(i, j, k)], us = ss[idx(i, j, k)], ut = wt[q];
      const double g0 = sG[l], g1 = sG[NP + l], g2 = sG[2 * NP + l];
      const double g3 = sG[3 * NP + l], g4 = sG[4 * NP + l], g5 = sG[5 * NP + l];
      sr[idx(i, j, k)] = geo3(g0, g1, g2, ur, us, ut);
      ss[idx(i, j, k)] = geo3(g1, g3, g4, ur, us, ut);
      wt[q] = geo3(g2, g4, g5, ur, us, ut);
    }
  }

  // same as geometry() with the factors read straight from HBM into registers
  // (coalesced: consecutive threads own consecutive i of one (j,k) row)
  template <int H>
  __device__ static void geometry_reg(const double* __restrict__ Ge, double* sr, double* ss, int i, int j,
                                      double* wt) {
    constexpr int O0 = H * KH;
    double g[6][KH];
#pragma unroll
    for (int q = 0; q < KH; ++q) {
      const int l = ((O0 + q) * N1 + j) * N1 + i;
#pragma unroll
      for (int f = 0; f < 6; ++f) g[f][q] = __ldg(Ge + f * NP + l);
    }
#pragma unroll
    for (int q = 0; q < KH; ++q) {
      const int k = O0 + q;
      const double ur = sr[idx(i, j, k)], us = ss[idx(i, j, k)], ut = wt[q];
      sr[idx(i, j, k)] = geo3(g[0][q], g[1][q], g[2][q], ur, us, ut);
      ss[idx(i, j, k)] = geo3(g[1][q], g[3][q], g[4][q], ur, us, ut);
      wt[q] = geo3(g[2][q], g[4][q], g[5][q], ur, us, ut);
    }
  }

  template <int H>
  __device__ static void div_r(const double* sr, double* su, int ta, int tb) {
    constexpr int O0 = H * KH;
    double l[N1];
#pragma unroll
    for (int m = 0; m < N1; ++m) l[m] = sr[idx(m, ta, tb)];
#pragma unroll
    for (int q = 0; q < KH; ++q) {
      double v = 0.0;
#pragma unroll
      for (int m = 0; m < N1; ++m) v = __fma_rn(c_D[N][m * N1 + (O0 + q)], l[m], v);
      su[idx(O0 + q, ta, tb)] = v;
    }
  }

  template <int H>
  __device__ static void div_s(const double* ss, double* su, double* sr, int ta, int tb, const double* wt) {
    constexpr int O0 = H * KH;
#pragma unroll
    for (int q = 0; q < KH; ++q) sr[idx(ta, tb, O0 + q)] = wt[q];  // publish w_t columns
    double l[N1];
#pragma unroll
    for (int m = 0; m < N1; ++m) l[m] = ss[idx(ta, m, tb)];
#pragma unroll
    for (int q = 0; q < KH; ++q) {
      double v = 0.0;
#pragma unroll
      for (int m = 0; m < N1; ++m) v = __fma_rn(c_D[N][m * N1 + (O0 + q)], l[m], v);
      su[idx(ta, O0 + q, tb)] += v;
    }
  }

  template <int H>
  __device__ static void finish(const SemArgs& A, const double* su, const double* sr, const double* so, int i,
                                int j, long e, const double* dvh, const double* wt) {
    constexpr int O0 = H * KH;
    const bool ij_interior = (i >= 1 && i < N && j >= 1 && j < N);
    double l[N1];
    // w_t of the column: the thread published its own KH values, the rest come from its partner
#pragma unroll
    for (int m = 0; m < N1; ++m) l[m] = (m >= O0 && m < O0 + KH) ? wt[m - O0] : sr[idx(i, j, m)];
#pragma unroll
    for (int q = 0; q < KH; ++q) {
      const int k = O0 + q;
      double v = 0.0;
#pragma unroll
      for (int m = 0; m < N1; ++m) v = __fma_rn(c_D[N][m * N1 + k], l[m], v);
      v += su[idx(i, j, k)];
      if (ij_interior && k >= 1 && k < N) {
        const int p = (i - 1) + (N - 1) * ((j - 1) + (N - 1) * (k - 1));
        double a0 = 0.0, a1 = 0.0, a2 = 0.0;
        if constexpr (NOPS > 0) a0 = so[p];
        if constexpr (NOPS > 1) a1 = so[NIP + p];
        if constexpr (NOPS > 2) a2 = so[2 * NIP + p];
        epilogue<EPI>(A, e * NOS + p, v, dvh[q], a0, a1, a2);
      } else {
        A.shell[e * A.nshell + A.lut[(k * N1 + j) * N1 + i]] = v;
      }
    }
  }
};

template <int N, int EPI, int KS>
__global__ void __launch_bounds__((N + 1) * (N + 1) * KS) k_sem_k1_lines(SemArgs A) {
  using L = K1L<N, EPI, KS>;
  using S = typename L::S;
  constexpr int N1 = N + 1, NP = N1 * N1 * N1, NOS = sem_nos(N), NOPS = S::NOPS, NIP = S::NIP, KH = L::KH;
  extern __shared__ __align__(128) double sm[];
  double* sG = sm + S::g_off;
  double* so = sm + S::o_off;
  double* su = sm + S::u_off;
  double* sr = sm + S::r_off;
  double* ss = sm + S::s_off;
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(sm + S::bar_off);
  const int t = threadIdx.x;
  const K1Elem el = k1_element(A);
  const long e = el.e;
  const int line = t % (N1 * N1);
  const int h = t / (N1 * N1);  // line part: warp-uniform for N1*N1 a multiple of 32
  const int ta = line % N1, tb = line / N1;
  if (t == 0) {  // 1. TMA
    const bool skip_x = (EPI == EPI_CHEB4 || EPI == EPI_CHEB1) && A.x_zero;
    unsigned bytes = 6 * NP * sizeof(double);
    if constexpr (NOPS > 0 && sem_nint(N) > 0) bytes += (NOPS - (skip_x ? 1 : 0)) * NIP * 8;
    mbar_init(bar, 1);
    mbar_expect_tx(bar, bytes);
    bulk_g2s(sG, A.G + e * 6 * NP, 6 * NP * sizeof(double), bar);
    if constexpr (NOPS > 0 && sem_nint(N) > 0) {
#pragma unroll
      for (int op = 0; op < NOPS; ++op) {
        if (op == 0 && skip_x) continue;
        bulk_g2s(so + (std::size_t)op * NIP, epi_op<EPI>(A, op) + e * NOS, NIP * 8, bar);
      }
    }
  }
  double wt[KH], dvh[KH];
// run a phase on this thread's line part with a compile-time part index (h < KS <= 4)
#define ON_PART(fn, ...)                                   \
  do {                                                     \
    switch (h) {                                           \
      case 0: L::template fn<0>(__VA_ARGS__); break;       \
      case 1: L::template fn<1 % KS>(__VA_ARGS__); break;  \
      case 2: L::template fn<2 % KS>(__VA_ARGS__); break;  \
      default: L::template fn<3 % KS>(__VA_ARGS__); break; \
    }                                                      \
  } while (0)
  k1_halo_wait(A, el);
  ON_PART(gather, A, su, ta, tb, el, dvh);
  __syncthreads();
  ON_PART(gradient, su, sr, ss, ta, tb, wt, dvh);
  __syncthreads();
  mbar_wait(bar, 0);
  ON_PART(geometry, sG, sr, ss, ta, tb, wt);
  __syncthreads();
  ON_PART(div_r, sr, su, ta, tb);
  __syncthreads();
  ON_PART(div_s, ss, su, sr, ta, tb, wt);
  __syncthreads();
  ON_PART(finish, A, su, sr, so, ta, tb, e, dvh, wt);
}

// Variant without the 24.6 KB shared-memory stage for the geometric factors:
// they are read into registers in the geometry phase, so a block needs only
// the u/r/s line buffers and the epilogue operands (~19 KB at N=7) and twice
// as many elements are resident per SM to hide the HBM latency.
template <int N, int EPI, int KS, int MINB>
__global__ void __launch_bounds__((N + 1) * (N + 1) * KS, MINB) k_sem_k1_greg(SemArgs A) {
  using L = K1L<N, EPI, KS>;
  using S = K3Smem<N, EPI, false>;
  constexpr int N1 = N + 1, NP = N1 * N1 * N1, NOPS = S::NOPS, NIP = S::NIP, KH = L::KH;
  constexpr bool HAS_OPS = NOPS > 0 && sem_nint(N) > 0;
  extern __shared__ __align__(128) double sm[];
  double* so = sm + S::o_off;
  double* su = sm + S::u_off;
  double* sr = sm + S::r_off;
  double* ss = sm + S::s_off;
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(sm + S::bar_off);
  const int t = threadIdx.x;
  const K1Elem el = k1_element(A);
  const long e = el.e;
  const int line = t % (N1 * N1);
  const int h = t / (N1 * N1);
  const int ta = line % N1, tb = line / N1;
  if constexpr (HAS_OPS) {
    if (t == 0) {  // TMA of the interior epilogue operands
      const bool skip_x = (EPI == EPI_CHEB4 || EPI == EPI_CHEB1) && A.x_zero;
      mbar_init(bar, 1);
      mbar_expect_tx(bar, (NOPS - (skip_x ? 1 : 0)) * NIP * 8);
#pragma unroll
      for (int op = 0; op < NOPS; ++op) {
        if (op == 0 && skip_x) continue;
        bulk_g2s(so + (std::size_t)op * NIP, epi_op<EPI>(A, op) + e * sem_nos(N), NIP * 8, bar);
      }
    }
  }
  const double* Ge = A.G + e * 6 * NP;
  if (A.prefetch_g) {
    // pull the element's factors toward L2 now: the geometry phase's register
    // loads then wait on L2 instead of HBM while gather/gradient run
    constexpr int LINES = 6 * NP * 8 / 128;
    for (int q = t; q < LINES; q += (N + 1) * (N + 1) * KS)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(Ge + q * 16));
  }
  double wt[KH], dvh[KH];
  k1_halo_wait(A, el);
  ON_PART(gather, A, su, ta, tb, el, dvh);
  __syncthreads();
  ON_PART(gradient, su, sr, ss, ta, tb, wt, dvh);
  __syncthreads();
  ON_PART(geometry_reg, Ge, sr, ss, ta, tb, wt);
  __syncthreads();
  ON_PART(div_r, sr, su, ta, tb);
  __syncthreads();
  ON_PART(div_s, ss, su, sr, ta, tb, wt);
  __syncthreads();
  if constexpr (HAS_OPS) mbar_wait(bar, 0);
  ON_PART(finish, A, su, sr, so, ta, tb, e, dvh, wt);
}

#undef ON_PART
