/*
 * oracle_schwarz.c -- CPU restatement (TEST INFRASTRUCTURE ONLY) of the
 * Chebyshev-Schwarz smoother of PAPER.md:560-629.
 * PARITY UNPINNED BY THE REFERENCE (no reference implementation exists).
 *
 * Definition used (the spec leaves the 1D extension open; this is ours and
 * the GPU path implements the same one):
 *  - extended subdomain of element e: its (N+1) GLL nodes plus one node of
 *    each neighbour per direction -> pbar = N+3 nodes per direction
 *    (PAPER.md:579-583); global 1D indices [eN-1, eN+N+1].
 *  - box approximation: element lengths per direction = mean length of the
 *    four element edges in that direction; 1D stiffness/mass of the
 *    3-element patch (left neighbour, element, right neighbour) with GLL
 *    (lumped) mass, restricted to the pbar extended nodes; homogeneous
 *    Dirichlet beyond.  Extended nodes that are global Dirichlet nodes are
 *    decoupled (identity row/col), which leaves the reduced solve exact.
 *  - FDM: A_* S = B_* S Lambda, S^T B_* S = I, Abar^{-1} =
 *    (Sz x Sy x Sx) D^{-1} (Sz x Sy x Sx)^T, D = I x I x Lx + I x Ly x I + Lz x I x I
 *    (PAPER.md:587-613).  Each mode-product output is one fma() chain over
 *    ascending m -- the rounding of the GPU's k_schwarz_local (__fma_rn), so
 *    the local solves compare bit for bit.
 *  - ASM: S r = W_asm (sum_e R_e^T Abar_e^{-1} R_e r), W_asm = 1 / (number of
 *    extended subdomains covering the node) -- post-multiplied.
 *  - RAS: S r = W_mult (sum_e Q_e^T [Abar_e^{-1} R_e r restricted to the
 *    element's own nodes]), W_mult = 1 / (element multiplicity) -- overlap
 *    values are not added back.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

#define NMAX 16
#define PB (NMAX + 3)

void orc_kershaw_map(double eps, double x, double y, double z, double* X, double* Y, double* Z);
void orc_sem_node_coords(int geometry, double eps, int N, const double* xi, int Ex, int Ey, int Ez,
                         int ex, int ey, int ez, int i, int j, int k, double* X, double* Y,
                         double* Z);

/* cyclic Jacobi eigen-solver for a symmetric n x n matrix (row-major, destroyed);
 * eigenvectors in columns of V */
void orc_sym_eig(int n, double* A, double* lam, double* V) {
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) V[i * n + j] = (i == j) ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, diag = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        if (i != j) off += A[i * n + j] * A[i * n + j];
        else diag += A[i * n + i] * A[i * n + i];
      }
    if (off <= 1e-30 * diag) break;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = A[p * n + q];
        if (apq == 0.0) continue;
        const double app = A[p * n + p], aqq = A[q * n + q];
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {
          const double akp = A[k * n + p], akq = A[k * n + q];
          A[k * n + p] = c * akp - s * akq;
          A[k * n + q] = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          const double apk = A[p * n + k], aqk = A[q * n + k];
          A[p * n + k] = c * apk - s * aqk;
          A[q * n + k] = s * apk + c * aqk;
        }
        for (int k = 0; k < n; ++k) {
          const double vkp = V[k * n + p], vkq = V[k * n + q];
          V[k * n + p] = c * vkp - s * vkq;
          V[k * n + q] = s * vkp + c * vkq;
        }
      }
  }
  for (int i = 0; i < n; ++i) lam[i] = A[i * n + i];
}

/* A s = lam B s with B SPD: B = L L^T, C = L^{-1} A L^{-T} (symmetrised),
 * C Q = Q Lambda (cyclic Jacobi), S = L^{-T} Q so that S^T B S = I.  Same
 * operation sequence as the GPU library's setup (csrc/host_setup.cpp
 * host_sym_geneig), so the eigenbases -- and with them the local solves --
 * are bit-identical. */
static void sym_geneig(int n, const double* A, const double* B, double* S, double* lam) {
  double L[PB * PB], Li[PB * PB], C[PB * PB], Q[PB * PB];
  memset(L, 0, sizeof L);
  memset(Li, 0, sizeof Li);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j <= i; ++j) {
      double s = B[i * n + j];
      for (int k = 0; k < j; ++k) s -= L[i * n + k] * L[j * n + k];
      if (i == j)
        L[i * n + i] = sqrt(s);
      else
        L[i * n + j] = s / L[j * n + j];
    }
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      double s = (i == j) ? 1.0 : 0.0;
      for (int k = 0; k < i; ++k) s -= L[i * n + k] * Li[k * n + j];
      Li[i * n + j] = s / L[i * n + i];
    }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double s = 0.0;
      for (int k = 0; k < n; ++k)
        for (int l = 0; l < n; ++l) s += Li[i * n + k] * A[k * n + l] * Li[j * n + l];
      C[i * n + j] = s;
    }
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) C[i * n + j] = C[j * n + i] = 0.5 * (C[i * n + j] + C[j * n + i]);
  orc_sym_eig(n, C, lam, Q);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double s = 0.0;
      for (int k = 0; k < n; ++k) s += Li[k * n + i] * Q[k * n + j];
      S[i * n + j] = s;
    }
}

/* 1D extended operators for one direction.
 * L = element length, Ll/Lr = neighbour lengths (ignored when that side is absent),
 * dl/dr = 1 if the extended node at index 0 / pbar-1 is a global Dirichlet node,
 * d0/dN = 1 if the element's own node 0 / N is a global Dirichlet node.
 * Output: S (pbar x pbar, column eigenvectors, S^T B S = I) and lam (pbar). */
void orc_fdm_1d(int N, const double* xi, const double* w, const double* D, double Ll, double L,
                double Lr, int dl, int d0, int dN, int dr, double* S, double* lam) {
  (void)xi;
  const int n1 = N + 1, pb = N + 3, np = 3 * N + 1;
  double K[(3 * NMAX + 1) * (3 * NMAX + 1)], M[3 * NMAX + 1];
  memset(K, 0, sizeof K);
  memset(M, 0, sizeof M);
  const double Ls[3] = {Ll, L, Lr};
  for (int el = 0; el < 3; ++el) {
    const double h = Ls[el];
    for (int a = 0; a < n1; ++a) {
      M[el * N + a] += 0.5 * h * w[a];
      for (int b = 0; b < n1; ++b) {
        double kab = 0.0;
        for (int m = 0; m < n1; ++m) kab += D[m * n1 + a] * w[m] * D[m * n1 + b];
        K[(el * N + a) * np + (el * N + b)] += (2.0 / h) * kab;
      }
    }
  }
  /* restrict to patch indices N-1 .. 2N+1; Dirichlet-eliminated nodes decoupled */
  int dirm[PB];
  memset(dirm, 0, sizeof dirm);
  if (dl) dirm[0] = 1;
  if (d0) { dirm[0] = 1; dirm[1] = 1; }
  if (dN) { dirm[pb - 1] = 1; dirm[pb - 2] = 1; }
  if (dr) dirm[pb - 1] = 1;
  double A[PB * PB], B[PB * PB];
  memset(B, 0, sizeof B);
  for (int a = 0; a < pb; ++a) {
    B[a * pb + a] = dirm[a] ? 1.0 : M[N - 1 + a];
    for (int b = 0; b < pb; ++b)
      A[a * pb + b] = (dirm[a] || dirm[b]) ? (a == b ? 1.0 : 0.0) : K[(N - 1 + a) * np + (N - 1 + b)];
  }
  sym_geneig(pb, A, B, S, lam);
}

/* element edge-length box approximation */
static void elem_lengths(int geometry, double eps, int N, const double* xi, int Ex, int Ey, int Ez,
                         int ex, int ey, int ez, double* L) {
  double P[8][3];
  for (int v = 0; v < 8; ++v) {
    const int i = (v & 1) ? N : 0, j = (v & 2) ? N : 0, k = (v & 4) ? N : 0;
    orc_sem_node_coords(geometry, eps, N, xi, Ex, Ey, Ez, ex, ey, ez, i, j, k, &P[v][0], &P[v][1], &P[v][2]);
  }
  for (int d = 0; d < 3; ++d) {
    const int bit = 1 << d;
    double s = 0.0;
    for (int v = 0; v < 8; ++v)
      if (!(v & bit)) {
        const double dx = P[v | bit][0] - P[v][0], dy = P[v | bit][1] - P[v][1], dz = P[v | bit][2] - P[v][2];
        s += sqrt(dx * dx + dy * dy + dz * dz);
      }
    L[d] = 0.25 * s;
  }
}

/* internal accessor (oracle_sem.c layout) */
typedef struct {
  int N, n1, np, Ex, Ey, Ez, E, Mx, My, Mz;
  size_t n;
  int geometry;
  double eps;
  double xi[NMAX + 1], w[NMAX + 1], D[(NMAX + 1) * (NMAX + 1)];
} sem_view;

void orc_sem_view(const orc_sem* s, int* N, int* Ex, int* Ey, int* Ez, int* geometry, double* eps,
                  double* xi, double* w, double* D);

void orc_sem_schwarz(const orc_sem* s, int ras, const double* r, double* out) {
  int N, Ex, Ey, Ez, geometry;
  double eps, xi[NMAX + 1], w[NMAX + 1], D[(NMAX + 1) * (NMAX + 1)];
  orc_sem_view(s, &N, &Ex, &Ey, &Ez, &geometry, &eps, xi, w, D);
  const int pb = N + 3, n1 = N + 1;
  const int Mx = N * Ex - 1, My = N * Ey - 1, Mz = N * Ez - 1;
  const size_t n = (size_t)Mx * My * Mz;
  const int ne[3] = {Ex, Ey, Ez};
  double* acc = calloc(n, sizeof(double));
  double* cnt = calloc(n, sizeof(double));
  double Sd[3][PB * PB], lamd[3][PB];
  double u[PB * PB * PB], t[PB * PB * PB];
  for (int e = 0; e < Ex * Ey * Ez; ++e) {
    const int ec[3] = {e % Ex, (e / Ex) % Ey, e / (Ex * Ey)};
    double L[3], Ln[3], Rn[3];
    elem_lengths(geometry, eps, N, xi, Ex, Ey, Ez, ec[0], ec[1], ec[2], L);
    for (int d = 0; d < 3; ++d) {
      int nb[3] = {ec[0], ec[1], ec[2]};
      double Lt[3];
      Ln[d] = L[d];
      Rn[d] = L[d];
      if (ec[d] > 0) {
        nb[d] = ec[d] - 1;
        elem_lengths(geometry, eps, N, xi, Ex, Ey, Ez, nb[0], nb[1], nb[2], Lt);
        Ln[d] = Lt[d];
      }
      nb[d] = ec[d];
      if (ec[d] + 1 < ne[d]) {
        nb[d] = ec[d] + 1;
        elem_lengths(geometry, eps, N, xi, Ex, Ey, Ez, nb[0], nb[1], nb[2], Lt);
        Rn[d] = Lt[d];
      }
      const int g0 = ec[d] * N; /* global 1D index of own node 0 */
      const int gmax = N * ne[d];
      const int dl = (g0 - 1) <= 0, d0 = g0 == 0, dN = g0 + N == gmax, dr = (g0 + N + 1) >= gmax;
      orc_fdm_1d(N, xi, w, D, Ln[d], L[d], Rn[d], dl, d0, dN, dr, Sd[d], lamd[d]);
    }
    /* R_e r on the extended box */
    for (int c = 0; c < pb; ++c)
      for (int b = 0; b < pb; ++b)
        for (int a = 0; a < pb; ++a) {
          const int gx = ec[0] * N + a - 1, gy = ec[1] * N + b - 1, gz = ec[2] * N + c - 1;
          const int in = gx >= 1 && gx <= Mx && gy >= 1 && gy <= My && gz >= 1 && gz <= Mz;
          u[a + pb * (b + pb * c)] = in ? r[((size_t)(gz - 1) * My + (gy - 1)) * Mx + (gx - 1)] : 0.0;
        }
    /* forward: t = (Sz^T x Sy^T x Sx^T) u */
    for (int dim = 0; dim < 3; ++dim) {
      const double* S = Sd[dim];
      for (int c = 0; c < pb; ++c)
        for (int b = 0; b < pb; ++b)
          for (int a = 0; a < pb; ++a) {
            double v = 0.0;
            for (int m = 0; m < pb; ++m) {
              const int o = dim == 0 ? a : (dim == 1 ? b : c);
              const int idx = dim == 0 ? m + pb * (b + pb * c) : (dim == 1 ? a + pb * (m + pb * c) : a + pb * (b + pb * m));
              v = fma(S[m * pb + o], u[idx], v);
            }
            t[a + pb * (b + pb * c)] = v;
          }
      memcpy(u, t, sizeof(double) * pb * pb * pb);
    }
    for (int c = 0; c < pb; ++c)
      for (int b = 0; b < pb; ++b)
        for (int a = 0; a < pb; ++a) u[a + pb * (b + pb * c)] /= (lamd[0][a] + lamd[1][b] + lamd[2][c]);
    for (int dim = 0; dim < 3; ++dim) {
      const double* S = Sd[dim];
      for (int c = 0; c < pb; ++c)
        for (int b = 0; b < pb; ++b)
          for (int a = 0; a < pb; ++a) {
            double v = 0.0;
            for (int m = 0; m < pb; ++m) {
              const int o = dim == 0 ? a : (dim == 1 ? b : c);
              const int idx = dim == 0 ? m + pb * (b + pb * c) : (dim == 1 ? a + pb * (m + pb * c) : a + pb * (b + pb * m));
              v = fma(S[o * pb + m], u[idx], v);
            }
            t[a + pb * (b + pb * c)] = v;
          }
      memcpy(u, t, sizeof(double) * pb * pb * pb);
    }
    /* scatter */
    for (int c = 0; c < pb; ++c)
      for (int b = 0; b < pb; ++b)
        for (int a = 0; a < pb; ++a) {
          if (ras && (a < 1 || a > n1 || b < 1 || b > n1 || c < 1 || c > n1)) continue;
          const int gx = ec[0] * N + a - 1, gy = ec[1] * N + b - 1, gz = ec[2] * N + c - 1;
          if (!(gx >= 1 && gx <= Mx && gy >= 1 && gy <= My && gz >= 1 && gz <= Mz)) continue;
          const size_t g = ((size_t)(gz - 1) * My + (gy - 1)) * Mx + (gx - 1);
          acc[g] += u[a + pb * (b + pb * c)];
          cnt[g] += 1.0;
        }
  }
  for (size_t g = 0; g < n; ++g) out[g] = acc[g] * (1.0 / cnt[g]);
  free(acc);
  free(cnt);
}

void orc_sem_schwarz_apply_cb(void* ctx, const double* r, double* out) {
  const orc_schwarz_ctx* c = ctx;
  orc_sem_schwarz(c->s, c->ras, r, out);
}
