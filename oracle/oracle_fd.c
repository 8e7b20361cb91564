/*
 * oracle_fd.c -- CPU restatement (TEST INFRASTRUCTURE ONLY) of the reference's
 * 2D five-point FD two-level path: stencil, manufactured problem, bilinear
 * transfer, Galerkin coarse operator, banded Cholesky, V-cycle and the
 * run_case driver.  Bit-identical to the compiled reference by construction
 * (same operation order); pinned in tests/test_oracle.py.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

/* ---- operators.hpp:33-57: StencilOperator::apply ---- */
typedef struct {
  orc_op base;
  size_t m;
  double inv_hx2, inv_hy2;
} fd_op;

static void fd_apply_raw(size_t m, double ihx2, double ihy2, const double* x, double* y) {
  const double c = 2.0 * (ihx2 + ihy2);
  for (size_t iy = 0; iy < m; ++iy) {
    for (size_t ix = 0; ix < m; ++ix) {
      const size_t id = iy * m + ix;
      double v = c * x[id];
      if (ix > 0) v -= ihx2 * x[id - 1];
      if (ix + 1 < m) v -= ihx2 * x[id + 1];
      if (iy > 0) v -= ihy2 * x[id - m];
      if (iy + 1 < m) v -= ihy2 * x[id + m];
      y[id] = v;
    }
  }
}

static void fd_apply(orc_op* self, const double* x, double* y) {
  fd_op* op = (fd_op*)self;
  fd_apply_raw(op->m, op->inv_hx2, op->inv_hy2, x, y);
}

static void fd_op_init(fd_op* op, size_t n, double Lx, double Ly) {
  const double hx = Lx / (double)n, hy = Ly / (double)n; /* domain.hpp:24-25 */
  op->m = n - 1;
  op->inv_hx2 = 1.0 / (hx * hx);
  op->inv_hy2 = 1.0 / (hy * hy);
  op->base.n = op->m * op->m;
  op->base.apply = fd_apply;
  op->base.count = 0;
}

void orc_fd_stencil_apply(size_t n, double Lx, double Ly, const double* x, double* y) {
  fd_op op;
  fd_op_init(&op, n, Lx, Ly);
  fd_apply(&op.base, x, y);
}

/* ---- problem.hpp:27-45 ---- */
void orc_fd_build_problem(size_t n, double Lx, double Ly, uint64_t seed, double* u, double* b) {
  const size_t m = n - 1;
  const double hx = Lx / (double)n, hy = Ly / (double)n;
  const double pi = 3.141592653589793238462643383279502884;
  orc_mt64 g;
  orc_mt64_seed(&g, seed);
  for (size_t iy = 0; iy < m; ++iy) {
    const double y = (double)(iy + 1) * hy;
    for (size_t ix = 0; ix < m; ++ix) {
      const double x = (double)(ix + 1) * hx;
      u[iy * m + ix] = sin(3.0 * pi * x / Lx) * sin(4.0 * pi * y / Ly) + orc_uniform_pm_half(&g);
    }
  }
  orc_fd_stencil_apply(n, Lx, Ly, u, b);
}

/* ---- transfer.hpp:20-46: interp_1d ---- */
typedef struct {
  size_t idx[2];
  double w[2];
  int nnz;
} interp_row;

static interp_row* interp_1d(size_t n, size_t nc) {
  const size_t ratio = n / nc;
  interp_row* rows = calloc(n - 1, sizeof(interp_row));
  for (size_t i = 1; i < n; ++i) {
    const size_t j0 = i / ratio;
    const double t = (double)(i % ratio) / (double)ratio;
    interp_row row;
    memset(&row, 0, sizeof row);
#define PUSH(cj, wv)                         \
  do {                                       \
    const double w_ = (wv);                  \
    if (w_ != 0.0) {                         \
      row.idx[row.nnz] = (cj) - 1;           \
      row.w[row.nnz] = w_;                   \
      ++row.nnz;                             \
    }                                        \
  } while (0)
    if (j0 >= 1 && j0 <= nc - 1) PUSH(j0, 1.0 - t);
    if (j0 + 1 <= nc - 1 && t > 0.0) PUSH(j0 + 1, t);
#undef PUSH
    rows[i - 1] = row;
  }
  return rows;
}

/* transfer.hpp:61-71 */
static void prolong_tab(size_t mf, size_t mc, const interp_row* tab, const double* x, double* y) {
  for (size_t iy = 0; iy < mf; ++iy) {
    const interp_row* ry = &tab[iy];
    for (size_t ix = 0; ix < mf; ++ix) {
      const interp_row* rx = &tab[ix];
      double s = 0.0;
      for (int a = 0; a < ry->nnz; ++a)
        for (int b = 0; b < rx->nnz; ++b) s += ry->w[a] * rx->w[b] * x[ry->idx[a] * mc + rx->idx[b]];
      y[iy * mf + ix] = s;
    }
  }
}

/* transfer.hpp:74-88 */
static void restrict_tab(size_t mf, size_t mc, const interp_row* tab, const double* x, double* y) {
  memset(y, 0, mc * mc * sizeof(double));
  for (size_t iy = 0; iy < mf; ++iy) {
    const interp_row* ry = &tab[iy];
    for (size_t ix = 0; ix < mf; ++ix) {
      const interp_row* rx = &tab[ix];
      const double v = x[iy * mf + ix];
      for (int a = 0; a < ry->nnz; ++a)
        for (int b = 0; b < rx->nnz; ++b) y[ry->idx[a] * mc + rx->idx[b]] += ry->w[a] * rx->w[b] * v;
    }
  }
}

void orc_fd_prolong(size_t n, size_t nc, const double* xc, double* y) {
  interp_row* tab = interp_1d(n, nc);
  prolong_tab(n - 1, nc - 1, tab, xc, y);
  free(tab);
}

void orc_fd_restrict(size_t n, size_t nc, const double* x, double* yc) {
  interp_row* tab = interp_1d(n, nc);
  restrict_tab(n - 1, nc - 1, tab, x, yc);
  free(tab);
}

/* ---- cholesky.hpp:18-91 over the Galerkin matrix of transfer.hpp:98-114 ---- */
struct orc_fd_hier {
  size_t n, nc, mf, mc, factor;
  double Lx, Ly;
  fd_op A;
  double* inv_diag;
  interp_row* tab;
  size_t bw;
  double* band; /* band[i*(bw+1) + (j + bw - i)] = L(i,j) */
  double lambda_tilde;
  double* scratch;
};

#define BAND(h, i, j) (h)->band[(i) * ((h)->bw + 1) + ((j) + (h)->bw - (i))]

/*
 * Galerkin A_c = P^T A P column by column (transfer.hpp:98-114).  The
 * reference applies P, A and P^T over the whole grid for every column; here
 * each column's three applies are restricted to the support of P e_j (plus the
 * stencil halo).  Every skipped term is an exact +0.0 contribution, and the
 * nonzero contributions accumulate in the same fine row-major order, so the
 * resulting entries are bit-identical to the reference's (checked against
 * oracle/_ref in tests/test_oracle.py).
 */
static void galerkin_band(struct orc_fd_hier* h) {
  const size_t mf = h->mf, mc = h->mc, nc2 = mc * mc, f = h->factor;
  double* pf = calloc(mf * mf, sizeof(double));
  double* apf = calloc(mf * mf, sizeof(double));
  double* col = calloc(nc2, sizeof(double));
  /* pass 1: values per column -> dense band with bw from pattern */
  /* bandwidth of P^T A P for tensor bilinear P with factor f is <= 2*mc+2 */
  const size_t bwmax = mc + 1;
  double* colvals = malloc(nc2 * (2 * bwmax + 1) * sizeof(double));
  size_t bw = 0;
  for (size_t j = 0; j < nc2; ++j) {
    const size_t cy = j / mc, cx = j % mc;
    /* fine support of P e_j: coarse node (cy+1, cx+1) covers fine (cj*f - f, cj*f + f) */
    const long fy0 = (long)((cy + 1) * f) - (long)f, fy1 = (long)((cy + 1) * f) + (long)f;
    const long fx0 = (long)((cx + 1) * f) - (long)f, fx1 = (long)((cx + 1) * f) + (long)f;
    /* fine interior index iy = gy - 1, support gy in (fy0, fy1) */
    long iy0 = fy0, iy1 = fy1 - 2, ix0 = fx0, ix1 = fx1 - 2; /* inclusive, interior indices */
    if (iy0 < 0) iy0 = 0;
    if (ix0 < 0) ix0 = 0;
    if (iy1 > (long)mf - 1) iy1 = (long)mf - 1;
    if (ix1 > (long)mf - 1) ix1 = (long)mf - 1;
    /* P e_j on the support (zero elsewhere; pf is kept all-zero between columns) */
    for (long iy = iy0; iy <= iy1; ++iy) {
      const interp_row* ry = &h->tab[iy];
      for (long ix = ix0; ix <= ix1; ++ix) {
        const interp_row* rx = &h->tab[ix];
        double s = 0.0;
        for (int a = 0; a < ry->nnz; ++a)
          for (int b = 0; b < rx->nnz; ++b)
            s += ry->w[a] * rx->w[b] * ((ry->idx[a] * mc + rx->idx[b]) == j ? 1.0 : 0.0);
        pf[iy * mf + ix] = s;
      }
    }
    /* A pf on support + halo */
    long ay0 = iy0 - 1 < 0 ? 0 : iy0 - 1, ay1 = iy1 + 1 > (long)mf - 1 ? (long)mf - 1 : iy1 + 1;
    long ax0 = ix0 - 1 < 0 ? 0 : ix0 - 1, ax1 = ix1 + 1 > (long)mf - 1 ? (long)mf - 1 : ix1 + 1;
    const double ihx2 = h->A.inv_hx2, ihy2 = h->A.inv_hy2, c = 2.0 * (ihx2 + ihy2);
    for (long iy = ay0; iy <= ay1; ++iy)
      for (long ix = ax0; ix <= ax1; ++ix) {
        const size_t id = (size_t)iy * mf + (size_t)ix;
        double v = c * pf[id];
        if (ix > 0) v -= ihx2 * pf[id - 1];
        if ((size_t)ix + 1 < mf) v -= ihx2 * pf[id + 1];
        if (iy > 0) v -= ihy2 * pf[id - mf];
        if ((size_t)iy + 1 < mf) v -= ihy2 * pf[id + mf];
        apf[id] = v;
      }
    /* P^T apf, accumulated in fine row-major order over the halo region */
    for (size_t i = 0; i < nc2; ++i) col[i] = 0.0;
    for (long iy = ay0; iy <= ay1; ++iy) {
      const interp_row* ry = &h->tab[iy];
      for (long ix = ax0; ix <= ax1; ++ix) {
        const interp_row* rx = &h->tab[ix];
        const double v = apf[(size_t)iy * mf + (size_t)ix];
        for (int a = 0; a < ry->nnz; ++a)
          for (int b = 0; b < rx->nnz; ++b) col[ry->idx[a] * mc + rx->idx[b]] += ry->w[a] * rx->w[b] * v;
      }
    }
    /* record column j entries within [j-bwmax, j+bwmax] */
    for (size_t i = 0; i < nc2; ++i) {
      if (col[i] != 0.0) {
        const size_t d = i > j ? i - j : j - i;
        if (d > bw) bw = d;
        if (d > bwmax) abort(); /* cannot happen for f >= 2 (coupling is nearest-neighbour) */
      }
    }
    for (long t = -(long)bwmax; t <= (long)bwmax; ++t) {
      const long i = (long)j + t;
      colvals[j * (2 * bwmax + 1) + (size_t)(t + (long)bwmax)] =
          (i >= 0 && i < (long)nc2) ? col[i] : 0.0;
    }
    /* reset scratch on the touched region */
    for (long iy = ay0; iy <= ay1; ++iy)
      for (long ix = ax0; ix <= ax1; ++ix) {
        pf[(size_t)iy * mf + (size_t)ix] = 0.0;
        apf[(size_t)iy * mf + (size_t)ix] = 0.0;
      }
  }
  h->bw = bw;
  h->band = calloc(nc2 * (bw + 1), sizeof(double));
  /* lower band: L(r,c) for c in [r-bw, r]; A(r,c) = column c entry at row r */
  for (size_t c = 0; c < nc2; ++c)
    for (size_t r = c; r < nc2 && r <= c + bw; ++r) BAND(h, r, c) = colvals[c * (2 * bwmax + 1) + (r - c + bwmax)];
  free(colvals);
  free(pf);
  free(apf);
  free(col);
}

static int band_factor(struct orc_fd_hier* h) { /* cholesky.hpp:70-86 */
  const size_t n = h->mc * h->mc, bw = h->bw;
  for (size_t i = 0; i < n; ++i) {
    const size_t j0 = i > bw ? i - bw : 0;
    for (size_t j = j0; j <= i; ++j) {
      double s = BAND(h, i, j);
      const size_t jb = j > bw ? j - bw : 0;
      const size_t k0 = j0 > jb ? j0 : jb;
      for (size_t k = k0; k < j; ++k) s -= BAND(h, i, k) * BAND(h, j, k);
      if (j < i) {
        BAND(h, i, j) = s / BAND(h, j, j);
      } else {
        if (s <= 0.0) return -1;
        BAND(h, i, i) = sqrt(s);
      }
    }
  }
  return 0;
}

void orc_fd_hier_coarse_solve(const orc_fd_hier* h, const double* b, double* x) {
  /* cholesky.hpp:44-58 */
  const size_t n = h->mc * h->mc, bw = h->bw;
  memcpy(x, b, n * sizeof(double));
  for (size_t i = 0; i < n; ++i) {
    const size_t j0 = i > bw ? i - bw : 0;
    double s = x[i];
    for (size_t j = j0; j < i; ++j) s -= BAND(h, i, j) * x[j];
    x[i] = s / BAND(h, i, i);
  }
  for (size_t ii = n; ii-- > 0;) {
    const size_t jmax = (n - 1 < ii + bw) ? n - 1 : ii + bw;
    double s = x[ii];
    for (size_t j = ii + 1; j <= jmax; ++j) s -= BAND(h, j, ii) * x[j];
    x[ii] = s / BAND(h, ii, ii);
  }
}

/* multigrid.hpp:36-48 */
orc_fd_hier* orc_fd_hier_create(size_t n, double Lx, double Ly, size_t factor,
                                size_t eigen_iterations, uint64_t eigen_seed) {
  if (factor < 2 || n % factor != 0) return NULL;
  if (n / factor < 2) return NULL; /* interp_1d:24-25 */
  orc_fd_hier* h = calloc(1, sizeof *h);
  h->n = n;
  h->nc = n / factor;
  h->factor = factor;
  h->Lx = Lx;
  h->Ly = Ly;
  h->mf = n - 1;
  h->mc = h->nc - 1;
  fd_op_init(&h->A, n, Lx, Ly);
  const size_t nf = h->mf * h->mf;
  h->inv_diag = malloc(nf * sizeof(double));
  const double dval = 2.0 * (h->A.inv_hx2 + h->A.inv_hy2); /* operators.hpp:59-61 */
  for (size_t i = 0; i < nf; ++i) h->inv_diag[i] = 1.0 / dval;  /* smoothers.hpp:174-181 */
  h->tab = interp_1d(n, h->nc);
  galerkin_band(h);
  if (band_factor(h) != 0) {
    orc_fd_hier_destroy(h);
    return NULL;
  }
  orc_smoother S = {h->inv_diag, NULL, NULL};
  h->lambda_tilde = orc_estimate_lambda_max(&h->A.base, &S, eigen_iterations, eigen_seed);
  h->A.base.count = 0;
  h->scratch = malloc(3 * nf * sizeof(double));
  return h;
}

void orc_fd_hier_destroy(orc_fd_hier* h) {
  if (!h) return;
  free(h->inv_diag);
  free(h->tab);
  free(h->band);
  free(h->scratch);
  free(h);
}

double orc_fd_hier_lambda_tilde(const orc_fd_hier* h) { return h->lambda_tilde; }
orc_op* orc_fd_hier_op(orc_fd_hier* h) { return &h->A.base; }
size_t orc_fd_hier_coarse_dim(const orc_fd_hier* h) { return h->mc * h->mc; }
size_t orc_fd_hier_bandwidth(const orc_fd_hier* h) { return h->bw; }

/* multigrid.hpp:69-90 */
int orc_fd_v_cycle(orc_fd_hier* h, const orc_cheb_config* s, size_t k_pre, size_t k_post,
                   const double* b, double* x, int x_is_zero) {
  const size_t nf = h->mf * h->mf, nc2 = h->mc * h->mc;
  orc_smoother S = {h->inv_diag, NULL, NULL};
  double* r = malloc(nf * sizeof(double));
  double* corr = malloc(nf * sizeof(double));
  double* rc = malloc(nc2 * sizeof(double));
  double* ec = malloc(nc2 * sizeof(double));
  int rc_ = 0;
  if (k_pre > 0) {
    rc_ = orc_chebyshev_smooth(&h->A.base, &S, s, k_pre, b, x, x_is_zero);
    if (rc_) goto out;
    x_is_zero = 0;
  }
  if (x_is_zero) {
    memcpy(r, b, nf * sizeof(double));
  } else {
    orc_op_apply(&h->A.base, x, r);
    for (size_t i = 0; i < nf; ++i) r[i] = b[i] - r[i];
  }
  restrict_tab(h->mf, h->mc, h->tab, r, rc);
  orc_fd_hier_coarse_solve(h, rc, ec);
  prolong_tab(h->mf, h->mc, h->tab, ec, corr);
  if (x_is_zero) {
    memcpy(x, corr, nf * sizeof(double));
  } else {
    orc_axpy(nf, 1.0, corr, x);
  }
  if (k_post > 0) rc_ = orc_chebyshev_smooth(&h->A.base, &S, s, k_post, b, x, 0);
out:
  free(r); free(corr); free(rc); free(ec);
  return rc_;
}

/* ---- harness.hpp:152-258 ---- */
typedef struct {
  orc_fd_hier* h;
  orc_cheb_config s;
  size_t k_pre, k_post;
} fd_prec_ctx;

static void fd_prec(void* ctx, const double* v, double* z) { /* multigrid.hpp:94-98 */
  fd_prec_ctx* c = ctx;
  memset(z, 0, c->h->A.base.n * sizeof(double));
  orc_fd_v_cycle(c->h, &c->s, c->k_pre, c->k_post, v, z, 1);
}

static void dispatch(const orc_case_config* cfg, fd_prec_ctx* pc, const double* b, double* hist,
                     double* x_out, orc_solve_report* rep) {
  const size_t n = pc->h->A.base.n;
  orc_solve_options o = {cfg->tol, cfg->maxit, cfg->restart, 1};
  double* x0 = calloc(n, sizeof(double));
  double* xs = x_out ? x_out : malloc(n * sizeof(double));
  if (cfg->driver == 0)
    orc_pcg(&pc->h->A.base, fd_prec, pc, b, x0, &o, xs, hist, rep);
  else if (cfg->driver == 1)
    orc_pgmres(&pc->h->A.base, fd_prec, pc, b, x0, &o, xs, hist, rep);
  else
    orc_stationary(&pc->h->A.base, fd_prec, pc, b, cfg->tol, cfg->maxit, hist, rep);
  free(x0);
  if (!x_out) free(xs);
}

int orc_fd_run_case_with(const orc_case_config* cfg, orc_fd_hier* h, double* hist,
                         double* x_out, orc_case_result* res) {
  if (cfg->k < 1 || cfg->factor < 2 || cfg->n % cfg->factor != 0 || !(cfg->tol > 0.0)) return -1;
  const size_t n = h->A.base.n;
  memset(res, 0, sizeof *res);
  res->lambda_tilde = h->lambda_tilde;
  res->tuned_lambda_min = NAN;
  fd_prec_ctx pc;
  pc.h = h;
  pc.s.family = cfg->family;
  pc.s.lambda_tilde = h->lambda_tilde;
  pc.s.lambda_max_multiplier = cfg->lambda_max_multiplier;
  pc.s.lambda_min_multiplier = cfg->lambda_min_multiplier;
  pc.k_pre = cfg->cycle == 0 ? cfg->k : 2 * cfg->k;
  pc.k_post = cfg->cycle == 0 ? cfg->k : 0;
  if (cfg->family == ORC_FIRST_OPT_LAMBDA) { /* harness.hpp:172-225 */
    double* bt = malloc(n * sizeof(double));
    double* th = malloc((cfg->maxit + 2) * sizeof(double));
    orc_random_vector(n, cfg->tuning_seed, bt);
    const double lo = log(0.0125), hi = log(0.4);
    int best = -1;
    size_t best_its = 0, best_mv = 0;
    double best_c = 0.0;
    for (int i = 0; i < 16; ++i) {
      const double cand = exp(lo + (hi - lo) * (double)i / 15.0);
      pc.s.lambda_min_multiplier = cand;
      orc_solve_report tr;
      dispatch(cfg, &pc, bt, th, NULL, &tr);
      if (!tr.converged) continue;
      if (best < 0 || tr.iterations < best_its || (tr.iterations == best_its && tr.fine_matvecs < best_mv)) {
        best = i;
        best_its = tr.iterations;
        best_mv = tr.fine_matvecs;
        best_c = cand;
      }
    }
    free(bt);
    free(th);
    if (best < 0) return -3;
    res->tuned_lambda_min = best_c;
    pc.s.lambda_min_multiplier = best_c;
  }
  double* u = malloc(n * sizeof(double));
  double* b = malloc(n * sizeof(double));
  orc_fd_build_problem(h->n, h->Lx, h->Ly, cfg->rhs_seed, u, b);
  dispatch(cfg, &pc, b, hist, x_out, &res->report);
  free(u);
  free(b);
  return 0;
}
