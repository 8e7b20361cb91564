/*
 * oracle_sem.c -- CPU restatement (TEST INFRASTRUCTURE ONLY) of the
 * spectral-element p-multigrid pieces named by BASELINE.json:north_star.
 *
 * PARITY UNPINNED BY THE REFERENCE: /root/reference has no SEM code
 * (SURVEY.md §0, §2a).  This file restates PAPER.md:540-634 and SURVEY.md
 * Appendix A with textbook SEM (Deville-Fischer-Mund): GLL basis, box /
 * Kershaw geometry, matrix-free A_e with six geometric factors, direct
 * stiffness summation Q^T over a canonical lexicographic global numbering,
 * Jacobi diagonal, tensor-product p-transfers, rediscretised coarse levels,
 * an exact banded-Cholesky p=1 solve, and the reference's V-cycle control
 * flow (multigrid.hpp:69-90) generalised to many levels.  It is pinned by
 * analytic tests (tests/test_oracle_sem.py): GLL quadrature exactness, D on
 * polynomials, symmetry / SPD, constant null-space of A_e, P^T = transpose of
 * P, and the separable p=1 operator.
 *
 * Canonical global vector: interior GLL nodes (Dirichlet nodes eliminated as
 * in domain.hpp:9-11), index ((gz-1)*My + (gy-1))*Mx + (gx-1), Mx = N*Ex-1.
 * Local node (i,j,k) of element e=(ex,ey,ez) is global (ex*N+i, ey*N+j, ez*N+k).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

#define NMAX 16

/* ---- A1: GLL nodes/weights (Newton on (1-x^2) L_N'(x)), derivative matrix ---- */
static void legendre(int N, double x, double* LN, double* LNm1) {
  double p0 = 1.0, p1 = x;
  if (N == 0) {
    *LN = 1.0;
    *LNm1 = 0.0;
    return;
  }
  for (int k = 2; k <= N; ++k) {
    const double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / (double)k;
    p0 = p1;
    p1 = p2;
  }
  *LN = p1;
  *LNm1 = p0;
}

void orc_gll(int N, double* xi, double* w) {
  const double pi = 3.141592653589793238462643383279502884;
  for (int j = 0; j <= N; ++j) {
    double x = -cos(pi * (double)j / (double)N);
    if (j > 0 && j < N) {
      for (int it = 0; it < 100; ++it) {
        /* Newton on q(x) = L_{N+1}(x) - L_{N-1}(x) (zeros = GLL interior nodes) */
        double LN, LNm1;
        legendre(N, x, &LN, &LNm1);
        const double LNp1 = ((2.0 * N + 1.0) * x * LN - N * LNm1) / (N + 1.0);
        const double q = LNp1 - LNm1;
        const double dq = (2.0 * N + 1.0) * LN; /* d/dx(L_{N+1}-L_{N-1}) = (2N+1) L_N */
        const double dx = q / dq;
        x -= dx;
        if (fabs(dx) < 1e-16) break;
      }
    }
    xi[j] = x;
  }
  xi[0] = -1.0;
  xi[N] = 1.0;
  /* symmetrise */
  for (int j = 0; j <= N / 2; ++j) {
    const double a = 0.5 * (xi[N - j] - xi[j]);
    xi[j] = -a;
    xi[N - j] = a;
  }
  if (N % 2 == 0) xi[N / 2] = 0.0;
  for (int j = 0; j <= N; ++j) {
    double LN, LNm1;
    legendre(N, xi[j], &LN, &LNm1);
    w[j] = 2.0 / ((double)N * (N + 1.0) * LN * LN);
  }
}

void orc_deriv_matrix(int N, const double* xi, double* D) {
  const int n1 = N + 1;
  double LN[NMAX + 1];
  for (int j = 0; j <= N; ++j) {
    double tmp;
    legendre(N, xi[j], &LN[j], &tmp);
  }
  for (int i = 0; i <= N; ++i)
    for (int j = 0; j <= N; ++j) {
      double v = 0.0;
      if (i != j)
        v = LN[i] / (LN[j] * (xi[i] - xi[j]));
      else if (i == 0)
        v = -0.25 * N * (N + 1.0);
      else if (i == N)
        v = 0.25 * N * (N + 1.0);
      D[i * n1 + j] = v;
    }
}

/* J[i*(Nc+1)+j] = l^c_j(xi^f_i) (Lagrange basis of the coarse GLL nodes) */
void orc_interp_matrix(int Nf, int Nc, double* J) {
  double xf[NMAX + 1], wf[NMAX + 1], xc[NMAX + 1], wc[NMAX + 1];
  orc_gll(Nf, xf, wf);
  orc_gll(Nc, xc, wc);
  for (int i = 0; i <= Nf; ++i)
    for (int j = 0; j <= Nc; ++j) {
      double v = 1.0;
      for (int m = 0; m <= Nc; ++m)
        if (m != j) v *= (xf[i] - xc[m]) / (xc[j] - xc[m]);
      J[i * (Nc + 1) + j] = v;
    }
}

/* ---- A2: geometry ---- */
/* Kershaw map on [0,1]^3 (CEED benchmark family); x untouched */
static double kr_right(double eps, double x) { return (x <= 0.5) ? (2.0 - eps) * x : 1.0 + eps * (x - 1.0); }
static double kr_left(double eps, double x) { return 1.0 - kr_right(eps, 1.0 - x); }
static double kr_step(double a, double b, double x) {
  if (x <= 0.0) return a;
  if (x >= 1.0) return b;
  return a + (b - a) * (x * x * x * (x * (6.0 * x - 15.0) + 10.0));
}

void orc_kershaw_map(double eps, double x, double y, double z, double* X, double* Y, double* Z) {
  *X = x;
  int layer = (int)(x * 6.0);
  if (layer > 5) layer = 5;
  const double lambda = (x - layer / 6.0) * 6.0;
  switch (layer) {
    case 0:
      *Y = kr_left(eps, y);
      *Z = kr_left(eps, z);
      break;
    case 1:
    case 4:
      *Y = kr_step(kr_left(eps, y), kr_right(eps, y), lambda);
      *Z = kr_step(kr_left(eps, z), kr_right(eps, z), lambda);
      break;
    case 2:
      *Y = kr_step(kr_right(eps, y), kr_left(eps, y), lambda / 2.0);
      *Z = kr_step(kr_right(eps, z), kr_left(eps, z), lambda / 2.0);
      break;
    case 3:
      *Y = kr_step(kr_right(eps, y), kr_left(eps, y), (1.0 + lambda) / 2.0);
      *Z = kr_step(kr_right(eps, z), kr_left(eps, z), (1.0 + lambda) / 2.0);
      break;
    default:
      *Y = kr_right(eps, y);
      *Z = kr_right(eps, z);
      break;
  }
}

typedef struct {
  orc_op base;
  orc_sem* s;
} sem_op;

struct orc_sem {
  int N, n1, np; /* order, N+1, (N+1)^3 */
  int Ex, Ey, Ez, E;
  int Mx, My, Mz; /* interior nodes per dim */
  size_t n;       /* Mx*My*Mz */
  int geometry;
  double eps;
  double xi[NMAX + 1], w[NMAX + 1], D[(NMAX + 1) * (NMAX + 1)];
  double* G;     /* E * 6 * np: rr, rs, rt, ss, st, tt */
  double* B;     /* E * np: mass */
  double* X;     /* E * 3 * np coordinates */
  int64_t* map;  /* E * np -> global or -1 */
  sem_op op;
  double *uL, *wL; /* scratch np */
};

void orc_sem_node_coords(int geometry, double eps, int N, const double* xi, int Ex, int Ey, int Ez,
                         int ex, int ey, int ez, int i, int j, int k, double* X, double* Y,
                         double* Z) {
  /* box [-1/2,1/2]^3, uniform elements, trilinear map at GLL points */
  (void)N;
  const double x = ((double)ex + 0.5 * (xi[i] + 1.0)) / (double)Ex;
  const double y = ((double)ey + 0.5 * (xi[j] + 1.0)) / (double)Ey;
  const double z = ((double)ez + 0.5 * (xi[k] + 1.0)) / (double)Ez;
  double u = x, v = y, t = z;
  if (geometry == 1) orc_kershaw_map(eps, x, y, z, &u, &v, &t);
  *X = u - 0.5;
  *Y = v - 0.5;
  *Z = t - 0.5;
}

static void sem_apply(orc_op* self, const double* x, double* y);

orc_sem* orc_sem_create(int N, int Ex, int Ey, int Ez, int geometry, double eps) {
  if (N < 1 || N > NMAX - 1 || Ex < 1 || Ey < 1 || Ez < 1) return NULL;
  orc_sem* s = calloc(1, sizeof *s);
  s->N = N;
  s->n1 = N + 1;
  s->np = s->n1 * s->n1 * s->n1;
  s->Ex = Ex;
  s->Ey = Ey;
  s->Ez = Ez;
  s->E = Ex * Ey * Ez;
  s->Mx = N * Ex - 1;
  s->My = N * Ey - 1;
  s->Mz = N * Ez - 1;
  s->n = (size_t)s->Mx * s->My * s->Mz;
  s->geometry = geometry;
  s->eps = eps;
  orc_gll(N, s->xi, s->w);
  orc_deriv_matrix(N, s->xi, s->D);
  const int n1 = s->n1, np = s->np;
  s->G = malloc((size_t)s->E * 6 * np * sizeof(double));
  s->B = malloc((size_t)s->E * np * sizeof(double));
  s->X = malloc((size_t)s->E * 3 * np * sizeof(double));
  s->map = malloc((size_t)s->E * np * sizeof(int64_t));
  s->uL = malloc(np * sizeof(double));
  s->wL = malloc(np * sizeof(double));
  for (int e = 0; e < s->E; ++e) {
    const int ex = e % Ex, ey = (e / Ex) % Ey, ez = e / (Ex * Ey);
    double* Xe = s->X + (size_t)e * 3 * np;
    for (int k = 0; k < n1; ++k)
      for (int j = 0; j < n1; ++j)
        for (int i = 0; i < n1; ++i) {
          const int l = i + n1 * (j + n1 * k);
          orc_sem_node_coords(geometry, eps, N, s->xi, Ex, Ey, Ez, ex, ey, ez, i, j, k, &Xe[l],
                              &Xe[np + l], &Xe[2 * np + l]);
          const int gx = ex * N + i, gy = ey * N + j, gz = ez * N + k;
          const int dir = gx == 0 || gx == N * Ex || gy == 0 || gy == N * Ey || gz == 0 || gz == N * Ez;
          s->map[(size_t)e * np + l] =
              dir ? -1 : ((int64_t)(gz - 1) * s->My + (gy - 1)) * s->Mx + (gx - 1);
        }
    /* Jacobian by spectral differentiation of the nodal coordinates */
    double* Ge = s->G + (size_t)e * 6 * np;
    double* Be = s->B + (size_t)e * np;
    for (int k = 0; k < n1; ++k)
      for (int j = 0; j < n1; ++j)
        for (int i = 0; i < n1; ++i) {
          const int l = i + n1 * (j + n1 * k);
          double Jm[3][3];
          for (int c = 0; c < 3; ++c) {
            const double* xc = Xe + (size_t)c * np;
            double dr = 0, ds = 0, dt = 0;
            for (int m = 0; m < n1; ++m) {
              dr += s->D[i * n1 + m] * xc[m + n1 * (j + n1 * k)];
              ds += s->D[j * n1 + m] * xc[i + n1 * (m + n1 * k)];
              dt += s->D[k * n1 + m] * xc[i + n1 * (j + n1 * m)];
            }
            Jm[c][0] = dr;
            Jm[c][1] = ds;
            Jm[c][2] = dt;
          }
          const double det = Jm[0][0] * (Jm[1][1] * Jm[2][2] - Jm[1][2] * Jm[2][1]) -
                             Jm[0][1] * (Jm[1][0] * Jm[2][2] - Jm[1][2] * Jm[2][0]) +
                             Jm[0][2] * (Jm[1][0] * Jm[2][1] - Jm[1][1] * Jm[2][0]);
          /* inverse: Ji[a][c] = d r_a / d x_c */
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
          const double W = s->w[i] * s->w[j] * s->w[k] * det;
          const int pa[6] = {0, 0, 0, 1, 1, 2}, pb[6] = {0, 1, 2, 1, 2, 2};
          for (int q = 0; q < 6; ++q) {
            const int a = pa[q], b = pb[q];
            Ge[(size_t)q * np + l] = W * (Ji[a][0] * Ji[b][0] + Ji[a][1] * Ji[b][1] + Ji[a][2] * Ji[b][2]);
          }
          Be[l] = W;
        }
  }
  s->op.base.n = s->n;
  s->op.base.apply = sem_apply;
  s->op.base.count = 0;
  s->op.s = s;
  return s;
}

void orc_sem_destroy(orc_sem* s) {
  if (!s) return;
  free(s->G); free(s->B); free(s->X); free(s->map); free(s->uL); free(s->wL);
  free(s);
}

void orc_sem_view(const orc_sem* s, int* N, int* Ex, int* Ey, int* Ez, int* geometry, double* eps,
                  double* xi, double* w, double* D) {
  *N = s->N;
  *Ex = s->Ex;
  *Ey = s->Ey;
  *Ez = s->Ez;
  *geometry = s->geometry;
  *eps = s->eps;
  memcpy(xi, s->xi, sizeof(double) * s->n1);
  memcpy(w, s->w, sizeof(double) * s->n1);
  memcpy(D, s->D, sizeof(double) * s->n1 * s->n1);
}

size_t orc_sem_n(const orc_sem* s) { return s->n; }
orc_op* orc_sem_op(orc_sem* s) { return &s->op.base; }

void orc_sem_local_to_global_map(const orc_sem* s, int64_t* map) {
  memcpy(map, s->map, (size_t)s->E * s->np * sizeof(int64_t));
}

void orc_sem_geom(const orc_sem* s, double* G, double* B) {
  if (G) memcpy(G, s->G, (size_t)s->E * 6 * s->np * sizeof(double));
  if (B) memcpy(B, s->B, (size_t)s->E * s->np * sizeof(double));
}

/* ---- A3: local matrix-free operator ----
 * Arithmetic contract shared with the GPU kernels (paper_2210_03179_b200/csrc/
 * k_sem.cu "arithmetic contract"; that file is built with --fmad=false and
 * places __fma_rn exactly where this file calls fma()), so the two round
 * identically and the operator is compared bit for bit:
 *   1D contraction  v = 0; for m ascending: v = fma(D_m, u_m, v)
 *   geometry        w_a = fma(g_c, u_t, fma(g_b, u_s, g_a * u_r))
 *   divergence      out = v_t + (v_r + v_s)     (three separate chains)
 * The summation order is a choice of this restatement (the reference has no
 * SEM operator); any fixed order is an equally exact A_e. */
static double geo3(double ga, double gb, double gc, double ur, double us, double ut) {
  return fma(gc, ut, fma(gb, us, ga * ur));
}

static void local_ax(const orc_sem* s, const double* Ge, const double* u, double* out) {
  const int n1 = s->n1, np = s->np;
  const double* D = s->D;
  double wr[NMAX * NMAX * NMAX], ws[NMAX * NMAX * NMAX], wt[NMAX * NMAX * NMAX];
  for (int k = 0; k < n1; ++k)
    for (int j = 0; j < n1; ++j)
      for (int i = 0; i < n1; ++i) {
        const int l = i + n1 * (j + n1 * k);
        double ur = 0, us = 0, ut = 0;
        for (int m = 0; m < n1; ++m) {
          ur = fma(D[i * n1 + m], u[m + n1 * (j + n1 * k)], ur);
          us = fma(D[j * n1 + m], u[i + n1 * (m + n1 * k)], us);
          ut = fma(D[k * n1 + m], u[i + n1 * (j + n1 * m)], ut);
        }
        const double grr = Ge[l], grs = Ge[np + l], grt = Ge[2 * np + l];
        const double gss = Ge[3 * np + l], gst = Ge[4 * np + l], gtt = Ge[5 * np + l];
        wr[l] = geo3(grr, grs, grt, ur, us, ut);
        ws[l] = geo3(grs, gss, gst, ur, us, ut);
        wt[l] = geo3(grt, gst, gtt, ur, us, ut);
      }
  for (int k = 0; k < n1; ++k)
    for (int j = 0; j < n1; ++j)
      for (int i = 0; i < n1; ++i) {
        double vr = 0, vs = 0, vt = 0;
        for (int m = 0; m < n1; ++m) {
          vr = fma(D[m * n1 + i], wr[m + n1 * (j + n1 * k)], vr);
          vs = fma(D[m * n1 + j], ws[i + n1 * (m + n1 * k)], vs);
          vt = fma(D[m * n1 + k], wt[i + n1 * (j + n1 * m)], vt);
        }
        out[i + n1 * (j + n1 * k)] = vt + (vr + vs);
      }
}

/* A4: y = Q^T A_L Q x, Dirichlet rows/cols eliminated */
static void sem_apply(orc_op* self, const double* x, double* y) {
  orc_sem* s = ((sem_op*)self)->s;
  const int np = s->np;
  memset(y, 0, s->n * sizeof(double));
  for (int e = 0; e < s->E; ++e) {
    const int64_t* me = s->map + (size_t)e * np;
    for (int l = 0; l < np; ++l) s->uL[l] = me[l] >= 0 ? x[me[l]] : 0.0;
    local_ax(s, s->G + (size_t)e * 6 * np, s->uL, s->wL);
    for (int l = 0; l < np; ++l)
      if (me[l] >= 0) y[me[l]] += s->wL[l];
  }
}

/* Element matrices of the assembled operator as (row, col, value) triplets,
 * one per local pair of non-Dirichlet nodes (duplicates to be summed, as
 * CsrMatrix::from_triplets does, operators.hpp:80-103).  Returns the count;
 * NULL outputs only count. */
size_t orc_sem_local_triplets(const orc_sem* s, int64_t* rows, int64_t* cols, double* vals) {
  const int np = s->np;
  size_t cnt = 0;
  double* u = calloc(np, sizeof(double));
  double* w = malloc(np * sizeof(double));
  for (int e = 0; e < s->E; ++e) {
    const int64_t* me = s->map + (size_t)e * np;
    for (int b = 0; b < np; ++b) {
      if (me[b] < 0) continue;
      if (rows) {
        memset(u, 0, np * sizeof(double));
        u[b] = 1.0;
        local_ax(s, s->G + (size_t)e * 6 * np, u, w);
      }
      for (int a = 0; a < np; ++a) {
        if (me[a] < 0) continue;
        if (rows) {
          rows[cnt] = me[a];
          cols[cnt] = me[b];
          vals[cnt] = w[a];
        }
        ++cnt;
      }
    }
  }
  free(u);
  free(w);
  return cnt;
}

/* A5 */
void orc_sem_diagonal(const orc_sem* s, double* d) {
  const int n1 = s->n1, np = s->np;
  const double* D = s->D;
  memset(d, 0, s->n * sizeof(double));
  for (int e = 0; e < s->E; ++e) {
    const double* Ge = s->G + (size_t)e * 6 * np;
    const int64_t* me = s->map + (size_t)e * np;
    for (int k = 0; k < n1; ++k)
      for (int j = 0; j < n1; ++j)
        for (int i = 0; i < n1; ++i) {
          const int l = i + n1 * (j + n1 * k);
          if (me[l] < 0) continue;
          double v = 0;
          for (int m = 0; m < n1; ++m) {
            v += D[m * n1 + i] * D[m * n1 + i] * Ge[m + n1 * (j + n1 * k)];
            v += D[m * n1 + j] * D[m * n1 + j] * Ge[3 * np + i + n1 * (m + n1 * k)];
            v += D[m * n1 + k] * D[m * n1 + k] * Ge[5 * np + i + n1 * (j + n1 * m)];
          }
          v += 2.0 * D[i * n1 + i] * D[j * n1 + j] * Ge[np + l];
          v += 2.0 * D[i * n1 + i] * D[k * n1 + k] * Ge[2 * np + l];
          v += 2.0 * D[j * n1 + j] * D[k * n1 + k] * Ge[4 * np + l];
          d[me[l]] += v;
        }
  }
}

/* b = Q^T B_L f_L, f = 3 pi^2 sin(pi x) sin(pi y) sin(pi z) */
void orc_sem_rhs(const orc_sem* s, double* b) {
  const double pi = 3.141592653589793238462643383279502884;
  const int np = s->np;
  memset(b, 0, s->n * sizeof(double));
  for (int e = 0; e < s->E; ++e) {
    const double* Xe = s->X + (size_t)e * 3 * np;
    const int64_t* me = s->map + (size_t)e * np;
    for (int l = 0; l < np; ++l) {
      if (me[l] < 0) continue;
      const double f = 3.0 * pi * pi * sin(pi * Xe[l]) * sin(pi * Xe[np + l]) * sin(pi * Xe[2 * np + l]);
      b[me[l]] += s->B[(size_t)e * np + l] * f;
    }
  }
}

/* ---- A6: p-transfers (owner-selection prolongation, exact transpose); the
 * contractions follow the same fma chain as k_prolong / k_restrict_local ---- */
static void tensor3(int nf, int nc, const double* J, const double* in, double* out, int transpose) {
  /* out = (J (x) J (x) J) in   (transpose: (J^T (x) J^T (x) J^T) in) ; J is nf x nc */
  double t1[NMAX * NMAX * NMAX], t2[NMAX * NMAX * NMAX];
  const int a = transpose ? nf : nc; /* input extent */
  const int b = transpose ? nc : nf; /* output extent */
#define JM(o, i) (transpose ? J[(i) * nc + (o)] : J[(o) * nc + (i)])
  for (int k = 0; k < a; ++k)
    for (int j = 0; j < a; ++j)
      for (int i = 0; i < b; ++i) {
        double v = 0;
        for (int m = 0; m < a; ++m) v = fma(JM(i, m), in[m + a * (j + a * k)], v);
        t1[i + b * (j + a * k)] = v;
      }
  for (int k = 0; k < a; ++k)
    for (int j = 0; j < b; ++j)
      for (int i = 0; i < b; ++i) {
        double v = 0;
        for (int m = 0; m < a; ++m) v = fma(JM(j, m), t1[i + b * (m + a * k)], v);
        t2[i + b * (j + b * k)] = v;
      }
  for (int k = 0; k < b; ++k)
    for (int j = 0; j < b; ++j)
      for (int i = 0; i < b; ++i) {
        double v = 0;
        for (int m = 0; m < a; ++m) v = fma(JM(k, m), t2[i + b * (j + b * m)], v);
        out[i + b * (j + b * k)] = v;
      }
#undef JM
}

/* owner of a local node: the element whose local indices are all >= 1 */
static int owns(const orc_sem* s, int i, int j, int k) {
  (void)s;
  return i >= 1 && j >= 1 && k >= 1;
}

void orc_sem_prolong(const orc_sem* f, const orc_sem* c, const double* xc, double* yf) {
  const int nf1 = f->n1, nc1 = c->n1;
  double J[(NMAX + 1) * (NMAX + 1)], uc[NMAX * NMAX * NMAX], uf[NMAX * NMAX * NMAX];
  orc_interp_matrix(f->N, c->N, J);
  memset(yf, 0, f->n * sizeof(double));
  for (int e = 0; e < f->E; ++e) {
    const int64_t* mc = c->map + (size_t)e * c->np;
    const int64_t* mf = f->map + (size_t)e * f->np;
    for (int l = 0; l < c->np; ++l) uc[l] = mc[l] >= 0 ? xc[mc[l]] : 0.0;
    tensor3(nf1, nc1, J, uc, uf, 0);
    for (int k = 0; k < nf1; ++k)
      for (int j = 0; j < nf1; ++j)
        for (int i = 0; i < nf1; ++i) {
          const int l = i + nf1 * (j + nf1 * k);
          if (mf[l] >= 0 && owns(f, i, j, k)) yf[mf[l]] = uf[l];
        }
  }
}

void orc_sem_restrict(const orc_sem* f, const orc_sem* c, const double* xf, double* yc) {
  const int nf1 = f->n1, nc1 = c->n1;
  double J[(NMAX + 1) * (NMAX + 1)], uc[NMAX * NMAX * NMAX], uf[NMAX * NMAX * NMAX];
  orc_interp_matrix(f->N, c->N, J);
  memset(yc, 0, c->n * sizeof(double));
  for (int e = 0; e < f->E; ++e) {
    const int64_t* mc = c->map + (size_t)e * c->np;
    const int64_t* mf = f->map + (size_t)e * f->np;
    for (int k = 0; k < nf1; ++k)
      for (int j = 0; j < nf1; ++j)
        for (int i = 0; i < nf1; ++i) {
          const int l = i + nf1 * (j + nf1 * k);
          uf[l] = (mf[l] >= 0 && owns(f, i, j, k)) ? xf[mf[l]] : 0.0;
        }
    tensor3(nf1, nc1, J, uf, uc, 1);
    for (int l = 0; l < c->np; ++l)
      if (mc[l] >= 0) yc[mc[l]] += uc[l];
  }
}

/* ---- A8: Schwarz (ASM/RAS) smoother with FDM local solves -- see oracle_schwarz.c ---- */

/* ---- A6/A7/A9: p-multigrid hierarchy ---- */
struct orc_pmg {
  int nlevels;
  orc_sem* lev[8];
  double* inv_diag[8];
  double lambda_tilde[8];
  int smoother; /* 0 Jacobi, 1 ASM, 2 RAS */
  orc_schwarz_ctx sch[8];
  /* exact coarse solve: banded Cholesky of the assembled coarsest operator */
  size_t cn, cbw;
  double* cband;
};

#define CB(p, i, j) (p)->cband[(i) * ((p)->cbw + 1) + ((j) + (p)->cbw - (i))]

static int coarse_factor(orc_pmg* p) {
  orc_sem* s = p->lev[p->nlevels - 1];
  const int np = s->np;
  const size_t n = s->n;
  /* bandwidth: max |g1-g2| over element-local pairs */
  size_t bw = 0;
  for (int e = 0; e < s->E; ++e) {
    const int64_t* me = s->map + (size_t)e * np;
    for (int a = 0; a < np; ++a)
      for (int b = 0; b < np; ++b)
        if (me[a] >= 0 && me[b] >= 0) {
          const size_t d = (size_t)llabs(me[a] - me[b]);
          if (d > bw) bw = d;
        }
  }
  p->cn = n;
  p->cbw = bw;
  p->cband = calloc(n * (bw + 1), sizeof(double));
  double* u = calloc(np, sizeof(double));
  double* w = malloc(np * sizeof(double));
  for (int e = 0; e < s->E; ++e) {
    const int64_t* me = s->map + (size_t)e * np;
    for (int b = 0; b < np; ++b) {
      if (me[b] < 0) continue;
      memset(u, 0, np * sizeof(double));
      u[b] = 1.0;
      local_ax(s, s->G + (size_t)e * 6 * np, u, w);
      for (int a = 0; a < np; ++a)
        if (me[a] >= 0 && me[a] >= me[b]) CB(p, (size_t)me[a], (size_t)me[b]) += w[a];
    }
  }
  free(u);
  free(w);
  for (size_t i = 0; i < n; ++i) { /* cholesky.hpp:70-86 restated */
    const size_t j0 = i > bw ? i - bw : 0;
    for (size_t j = j0; j <= i; ++j) {
      double sum = CB(p, i, j);
      const size_t jb = j > bw ? j - bw : 0;
      const size_t k0 = j0 > jb ? j0 : jb;
      for (size_t k = k0; k < j; ++k) sum -= CB(p, i, k) * CB(p, j, k);
      if (j < i)
        CB(p, i, j) = sum / CB(p, j, j);
      else {
        if (sum <= 0.0) return -1;
        CB(p, i, i) = sqrt(sum);
      }
    }
  }
  return 0;
}

void orc_pmg_coarse_solve(orc_pmg* p, const double* b, double* x) {
  const size_t n = p->cn, bw = p->cbw; /* cholesky.hpp:44-58 */
  memcpy(x, b, n * sizeof(double));
  for (size_t i = 0; i < n; ++i) {
    const size_t j0 = i > bw ? i - bw : 0;
    double s = x[i];
    for (size_t j = j0; j < i; ++j) s -= CB(p, i, j) * x[j];
    x[i] = s / CB(p, i, i);
  }
  for (size_t ii = n; ii-- > 0;) {
    const size_t jmax = (n - 1 < ii + bw) ? n - 1 : ii + bw;
    double s = x[ii];
    for (size_t j = ii + 1; j <= jmax; ++j) s -= CB(p, j, ii) * x[j];
    x[ii] = s / CB(p, ii, ii);
  }
}

static orc_smoother level_smoother(orc_pmg* p, int l) {
  orc_smoother S;
  if (p->smoother == 0) {
    S.inv_diag = p->inv_diag[l];
    S.S_apply = NULL;
    S.S_ctx = NULL;
  } else {
    S.inv_diag = NULL;
    S.S_apply = orc_sem_schwarz_apply_cb;
    S.S_ctx = &p->sch[l];
  }
  return S;
}

orc_pmg* orc_pmg_create(int nlevels, const int* orders, int Ex, int Ey, int Ez, int geometry,
                        double eps, int smoother, size_t eigen_iterations, uint64_t eigen_seed) {
  return orc_pmg_create_ex(nlevels, orders, Ex, Ey, Ez, geometry, eps, smoother, eigen_iterations,
                           eigen_seed, 0);
}

/* flags: ORC_PMG_NO_LAMBDA skips the lambda estimates (left 0), ORC_PMG_NO_COARSE
 * the banded Cholesky of the coarsest level -- for oracle/ref_driver.cpp, which
 * owns both through the reference's own templates (estimate_lambda_max,
 * BandedCholesky) and only borrows the levels, diagonals and transfers. */
orc_pmg* orc_pmg_create_ex(int nlevels, const int* orders, int Ex, int Ey, int Ez, int geometry,
                           double eps, int smoother, size_t eigen_iterations, uint64_t eigen_seed,
                           int flags) {
  if (nlevels < 1 || nlevels > 8) return NULL;
  orc_pmg* p = calloc(1, sizeof *p);
  p->nlevels = nlevels;
  p->smoother = smoother;
  for (int l = 0; l < nlevels; ++l) {
    p->lev[l] = orc_sem_create(orders[l], Ex, Ey, Ez, geometry, eps);
    if (!p->lev[l]) {
      orc_pmg_destroy(p);
      return NULL;
    }
    const size_t n = p->lev[l]->n;
    p->inv_diag[l] = malloc(n * sizeof(double));
    orc_sem_diagonal(p->lev[l], p->inv_diag[l]);
    for (size_t i = 0; i < n; ++i) p->inv_diag[l][i] = 1.0 / p->inv_diag[l][i]; /* smoothers.hpp:174-181 */
    p->sch[l].s = p->lev[l];
    p->sch[l].ras = smoother == 2;
  }
  for (int l = 0; l + 1 < nlevels && !(flags & ORC_PMG_NO_LAMBDA); ++l) {
    orc_smoother S = level_smoother(p, l);
    p->lambda_tilde[l] = orc_estimate_lambda_max(&p->lev[l]->op.base, &S, eigen_iterations, eigen_seed);
    p->lev[l]->op.base.count = 0;
  }
  if (!(flags & ORC_PMG_NO_COARSE) && coarse_factor(p) != 0) {
    orc_pmg_destroy(p);
    return NULL;
  }
  return p;
}

void orc_pmg_destroy(orc_pmg* p) {
  if (!p) return;
  for (int l = 0; l < p->nlevels; ++l) {
    orc_sem_destroy(p->lev[l]);
    free(p->inv_diag[l]);
  }
  free(p->cband);
  free(p);
}

orc_op* orc_pmg_op(orc_pmg* p, int level) { return &p->lev[level]->op.base; }
orc_sem* orc_pmg_sem(orc_pmg* p, int level) { return p->lev[level]; }
double orc_pmg_lambda_tilde(const orc_pmg* p, int level) { return p->lambda_tilde[level]; }

/* multigrid.hpp:69-90 generalised to many levels */
static int vcycle_level(orc_pmg* p, int l, const orc_cheb_config* base, size_t k_pre,
                        size_t k_post, const double* b, double* x, int x_is_zero) {
  orc_sem* s = p->lev[l];
  const size_t n = s->n;
  if (l == p->nlevels - 1) {
    double* e = malloc(n * sizeof(double));
    if (x_is_zero) {
      orc_pmg_coarse_solve(p, b, x);
    } else {
      double* r = malloc(n * sizeof(double));
      orc_op_apply(&s->op.base, x, r);
      for (size_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
      orc_pmg_coarse_solve(p, r, e);
      orc_axpy(n, 1.0, e, x);
      free(r);
    }
    free(e);
    return 0;
  }
  orc_cheb_config cfg = *base;
  cfg.lambda_tilde = p->lambda_tilde[l];
  orc_smoother S = level_smoother(p, l);
  int rc = 0;
  if (k_pre > 0) {
    rc = orc_chebyshev_smooth(&s->op.base, &S, &cfg, k_pre, b, x, x_is_zero);
    if (rc) return rc;
    x_is_zero = 0;
  }
  double* r = malloc(n * sizeof(double));
  if (x_is_zero) {
    memcpy(r, b, n * sizeof(double));
  } else {
    orc_op_apply(&s->op.base, x, r);
    for (size_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
  }
  orc_sem* c = p->lev[l + 1];
  double* rc_ = malloc(c->n * sizeof(double));
  double* ec = calloc(c->n, sizeof(double));
  double* corr = malloc(n * sizeof(double));
  orc_sem_restrict(s, c, r, rc_);
  rc = vcycle_level(p, l + 1, base, k_pre, k_post, rc_, ec, 1);
  if (!rc) {
    orc_sem_prolong(s, c, ec, corr);
    if (x_is_zero)
      memcpy(x, corr, n * sizeof(double));
    else
      orc_axpy(n, 1.0, corr, x);
    if (k_post > 0) rc = orc_chebyshev_smooth(&s->op.base, &S, &cfg, k_post, b, x, 0);
  }
  free(r); free(rc_); free(ec); free(corr);
  return rc;
}

int orc_pmg_v_cycle(orc_pmg* p, int family, double lmax_mult, double lmin_mult, size_t k_pre,
                    size_t k_post, const double* b, double* x, int x_is_zero) {
  orc_cheb_config base = {family, 1.0, lmax_mult, lmin_mult};
  return vcycle_level(p, 0, &base, k_pre, k_post, b, x, x_is_zero);
}

typedef struct {
  orc_pmg* p;
  int family;
  double lmaxm, lminm;
  size_t kpre, kpost;
} pmg_prec_ctx;

static void pmg_prec(void* vctx, const double* v, double* z) { /* multigrid.hpp:94-98 */
  pmg_prec_ctx* c = vctx;
  memset(z, 0, c->p->lev[0]->n * sizeof(double));
  orc_pmg_v_cycle(c->p, c->family, c->lmaxm, c->lminm, c->kpre, c->kpost, v, z, 1);
}

/* p-MG preconditioned PCG (driver 0) / PGMRES (driver 1) with the restated
 * reference Krylov drivers (krylov.hpp:75-264); x0 = 0 */
void orc_pmg_solve(orc_pmg* p, int driver, int family, double lmaxm, double lminm, size_t kpre,
                   size_t kpost, const double* b, double tol, size_t maxit, size_t restart,
                   double* x, double* hist, orc_solve_report* rep) {
  pmg_prec_ctx c = {p, family, lmaxm, lminm, kpre, kpost};
  const size_t n = p->lev[0]->n;
  double* x0 = calloc(n, sizeof(double));
  orc_solve_options o = {tol, maxit, restart, 1};
  if (driver == 0)
    orc_pcg(&p->lev[0]->op.base, pmg_prec, &c, b, x0, &o, x, hist, rep);
  else
    orc_pgmres(&p->lev[0]->op.base, pmg_prec, &c, b, x0, &o, x, hist, rep);
  free(x0);
}
