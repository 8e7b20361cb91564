// k_sem_k1.cuh -- the fused SEM element kernel (K1, AX mode) used for the
// high p-levels.  Included by k_sem.cu (needs its helpers: SemC, EpiOps,
// epi_op, epilogue, owner1d, TMA/mbarrier wrappers, c_D, K3Smem).
//
// One element per block of 2(N+1)^2 threads.  Every tensor contraction is a
// "line contraction": the N+1 values of a line along the contracted direction
// are loaded once from shared memory and multiplied by the GLL derivative
// matrix held in __constant__ memory (DFMA uniform-register operands, no
// shared traffic for D).  Each line is split between two threads (half H of
// the outputs each), H is a template parameter so every D index is a
// compile-time constant.
//   1. thread 0: TMA bulk copies of the element's 6 geometric factors
//      (24.6 KB at N=7) and of the interior blocks of the epilogue operands;
//   2. all threads: branch-free gather of Q u (all loads issued before any
//      store, so the element pays one memory latency, not KH);
//   3. gradient (r rows, s columns, t in registers) -> G_e grad u;
//   4. divergence (r rows, s columns accumulate, t in registers) ->
//      epilogue: interior nodes finished in place, shell nodes to K2.

template <int N, int EPI, int H>
__device__ __forceinline__ void k1_body(const SemArgs& A, double* sm, int line, long e) {
  using S = K3Smem<N, EPI>;
  constexpr int N1 = N + 1, NP = N1 * N1 * N1, NOS = sem_nos(N), NOPS = S::NOPS, NIP = S::NIP;
  constexpr int R = N1 + 1;
  constexpr int KH = N1 / 2, O0 = H * KH;
#define IDX(i, j, k) (((k) * N1 + (j)) * R + (i))
#define CD(a, b) c_D[N][(a) * N1 + (b)]
  double* sG = sm + S::g_off;
  double* so = sm + S::o_off;
  double* su = sm + S::u_off;
  double* sr = sm + S::r_off;
  double* ss = sm + S::s_off;
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(sm + S::bar_off);
  const int ta = line % N1, tb = line / N1;
  const int ex = (int)(e % A.Ex), ey = (int)((e / A.Ex) % A.Ey), ez = (int)(e / ((long)A.Ex * A.Ey));
  // 2. gather: thread (i,j,H) owns k in [O0, O0+KH)
  {
    const int i = ta, j = tb;
    int oex = 0, oey = 0;
    const int ax = owner1d<N>(ex, i, A.Ex, oex);
    const int ay = owner1d<N>(ey, j, A.Ey, oey);
    const bool xy_ok = ax >= 0 && ay >= 0;
    const double* ptr[KH];
    bool ok[KH];
#pragma unroll
    for (int q = 0; q < KH; ++q) {
      int oez = 0;
      const int az = owner1d<N>(A.z0 + ez, O0 + q, A.Ez, oez);
      const int lz = oez - A.z0;
      ok[q] = xy_ok && az >= 0;
      const long own = ((long)oex + (long)A.Ex * ((long)oey + (long)A.Ey * lz)) * NOS +
                       sem_pos(N, xy_ok ? ax : 0, xy_ok ? ay : 0, az >= 0 ? az : 0);
      const long halo = ((long)oex + (long)A.Ex * oey) * (N * N) + ax + N * ay;
      ptr[q] = (lz < 0) ? A.halo_lo + halo : A.u + own;
    }
    double v[KH];
#pragma unroll
    for (int q = 0; q < KH; ++q) v[q] = ok[q] ? __ldg(ptr[q]) : 0.0;
#pragma unroll
    for (int q = 0; q < KH; ++q) su[IDX(i, j, O0 + q)] = v[q];
  }
  __syncthreads();
  // 3. gradient
  double wt[KH], dvh[KH];
  {
    double l[N1];
#pragma unroll
    for (int m = 0; m < N1; ++m) l[m] = su[IDX(m, ta, tb)];
#pragma unroll
    for (int q = 0; q < KH; ++q) {
      double v = 0.0;
#pragma unroll
      for (int m = 0; m < N1; ++m) v += CD(O0 + q, m) * l[m];
      sr[IDX(O0 + q, ta, tb)] = v;
    }
#pragma unroll
    for (int m = 0; m < N1; ++m) l[m] = su[IDX(ta, m, tb)];
#pragma unroll
    for (int q = 0; q < KH; ++q) {
      double v = 0.0;
#pragma unroll
      for (int m = 0; m < N1; ++m) v += CD(O0 + q, m) * l[m];
      ss[IDX(ta, O0 + q, tb)] = v;
    }
#pragma unroll
    for (int m = 0; m < N1; ++m) l[m] = su[IDX(ta, tb, m)];
#pragma unroll
    for (int q = 0; q < KH; ++q) {
      double v = 0.0;
#pragma unroll
      for (int m = 0; m < N1; ++m) v += CD(O0 + q, m) * l[m];
      wt[q] = v;
      dvh[q] = l[O0 + q];
    }
  }
  __syncthreads();
  mbar_wait(bar, 0);
  {
    const int i = ta, j = tb;
#pragma unroll
    for (int q = 0; q < KH; ++q) {
      const int k = O0 + q;
      const int l = (k * N1 + j) * N1 + i;
      const double ur = sr[IDX(i, j, k)], us = ss[IDX(i, j, k)], ut = wt[q];
      const double g0 = sG[l], g1 = sG[NP + l], g2 = sG[2 * NP + l];
      const double g3 = sG[3 * NP + l], g4 = sG[4 * NP + l], g5 = sG[5 * NP + l];
      sr[IDX(i, j, k)] = g0 * ur + g1 * us + g2 * ut;
      ss[IDX(i, j, k)] = g1 * ur + g3 * us + g4 * ut;
      wt[q] = g2 * ur + g4 * us + g5 * ut;
    }
  }
  __syncthreads();
  // 4. divergence
  {
    double l[N1];
#pragma unroll
    for (int m = 0; m < N1; ++m) l[m] = sr[IDX(m, ta, tb)];
#pragma unroll
    for (int q = 0; q < KH; ++q) {
      double v = 0.0;
#pragma unroll
      for (int m = 0; m < N1; ++m) v += CD(m, O0 + q) * l[m];
      su[IDX(O0 + q, ta, tb)] = v;
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < KH; ++q) sr[IDX(ta, tb, O0 + q)] = wt[q];
  {
    double l[N1];
#pragma unroll
    for (int m = 0; m < N1; ++m) l[m] = ss[IDX(ta, m, tb)];
#pragma unroll
    for (int q = 0; q < KH; ++q) {
      double v = 0.0;
#pragma unroll
      for (int m = 0; m < N1; ++m) v += CD(m, O0 + q) * l[m];
      su[IDX(ta, O0 + q, tb)] += v;
    }
  }
  __syncthreads();
  const int i = ta, j = tb;
  const bool ij_interior = (i >= 1 && i < N && j >= 1 && j < N);
  double l[N1];
#pragma unroll
  for (int m = 0; m < N1; ++m) l[m] = sr[IDX(i, j, m)];
#pragma unroll
  for (int q = 0; q < KH; ++q) {
    const int k = O0 + q;
    double v = 0.0;
#pragma unroll
    for (int m = 0; m < N1; ++m) v += CD(m, O0 + q) * l[m];
    v += su[IDX(i, j, k)];
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
#undef IDX
#undef CD
}

template <int N, int EPI>
__global__ void __launch_bounds__((N + 1) * (N + 1) * 2) k_sem_k1_lines(SemArgs A) {
  using S = K3Smem<N, EPI>;
  constexpr int N1 = N + 1, NP = N1 * N1 * N1, NOS = sem_nos(N), NOPS = S::NOPS, NIP = S::NIP;
  extern __shared__ __align__(128) double sm[];
  const int t = threadIdx.x;
  const long e = A.e_begin + blockIdx.x;
  if (t == 0) {  // 1. TMA
    double* sG = sm + S::g_off;
    double* so = sm + S::o_off;
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(sm + S::bar_off);
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
  const int line = t % (N1 * N1);
  if (t < N1 * N1) k1_body<N, EPI, 0>(A, sm, line, e);  // warp-uniform split
  else k1_body<N, EPI, 1>(A, sm, line, e);
}
