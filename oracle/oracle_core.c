/*
 * oracle_core.c -- CPU restatement (TEST INFRASTRUCTURE ONLY) of the
 * reference's core kernels, smoothers and Krylov drivers.
 * Arithmetic order follows the reference line by line so that this file is
 * bit-identical to the compiled reference (checked in tests/test_oracle.py).
 * Citations: /root/reference/proj/include/chebmg/<file>:<line>.
 */
#define _POSIX_C_SOURCE 199309L
#include "oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ---- core.hpp:18-32: std::mt19937_64 restated (parameters fixed by the C++ standard) ---- */
#define MT_N 312
#define MT_M 156
#define MT_UM 0xFFFFFFFF80000000ULL
#define MT_LM 0x000000007FFFFFFFULL

void orc_mt64_seed(orc_mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->mti = MT_N;
}

uint64_t orc_mt64_next(orc_mt64* g) {
  if (g->mti >= MT_N) {
    for (int i = 0; i < MT_N; ++i) {
      const uint64_t x = (g->mt[i] & MT_UM) | (g->mt[(i + 1) % MT_N] & MT_LM);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = g->mt[(i + MT_M) % MT_N] ^ xa;
    }
    g->mti = 0;
  }
  uint64_t y = g->mt[g->mti++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

double orc_uniform01(orc_mt64* g) { return (double)(orc_mt64_next(g) >> 11) * 0x1.0p-53; }
double orc_uniform_pm_half(orc_mt64* g) { return orc_uniform01(g) - 0.5; }

void orc_random_vector(size_t n, uint64_t seed, double* out) {
  orc_mt64 g;
  orc_mt64_seed(&g, seed);
  for (size_t i = 0; i < n; ++i) out[i] = orc_uniform_pm_half(&g);
}

/* core.hpp:37-55: sequential, left-to-right */
double orc_dot(size_t n, const double* a, const double* b) {
  double s = 0.0;
  for (size_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}
double orc_norm2(size_t n, const double* a) { return sqrt(orc_dot(n, a, a)); }
void orc_axpy(size_t n, double alpha, const double* x, double* y) {
  for (size_t i = 0; i < n; ++i) y[i] += alpha * x[i];
}
void orc_scal(size_t n, double alpha, double* x) {
  for (size_t i = 0; i < n; ++i) x[i] *= alpha;
}

void orc_op_apply(orc_op* op, const double* x, double* y) {
  op->apply(op, x, y);
  op->count++;
}

/* ---- beta_table.hpp:16-92: optimised 4th-kind weights, one row per order ----
 * Frozen data (also tabulated in PAPER.md:1085-1256 for k<=16). */
static const double kBetaRows[20][20] = {
  {1.12500000000000},
  {1.02387287570313, 1.26408905371085},
  {1.00842544782028, 1.08867839208730, 1.33753125909618},
  {1.00391310427285, 1.04035811188593, 1.14863498546254, 1.38268869241000},
  {1.00212930146164, 1.02173711549260, 1.07872433192603, 1.19810065292663, 1.41322542791682},
  {1.00128517255940, 1.01304293035233, 1.04678215124113, 1.11616489419675, 1.23829020218444,
   1.43524297106744},
  {1.00083464397912, 1.00843949430122, 1.03008707768713, 1.07408384092003, 1.15036186707366,
   1.27116474046139, 1.45186658649364},
  {1.00057246631197, 1.00577427662415, 1.02050187922941, 1.05019803444565, 1.10115572984941,
   1.18086042806856, 1.29838585382576, 1.46486073151099},
  {1.00040960072832, 1.00412439506106, 1.01460212148266, 1.03561113626671, 1.07139972529194,
   1.12688273710962, 1.20785219140729, 1.32121930716746, 1.47529642820699},
  {1.00030312229652, 1.00304840660796, 1.01077022715387, 1.02619011597640, 1.05231724933755,
   1.09255743207549, 1.15083376663972, 1.23172250870894, 1.34060802024460, 1.48386124407011},
  {1.00023058595209, 1.00231675024028, 1.00817245396304, 1.01982986566342, 1.03950210235324,
   1.06965042700541, 1.11305754295742, 1.17290876275564, 1.25288300576792, 1.35725579919519,
   1.49101672564139},
  {1.00017947200828, 1.00180189139619, 1.00634861907307, 1.01537864566306, 1.03056942830760,
   1.05376019693943, 1.08699862592072, 1.13259183097913, 1.19316273358172, 1.27171293675110,
   1.37169337969799, 1.49708418575562},
  {1.00014241921559, 1.00142906932629, 1.00503028986298, 1.01216910518495, 1.02414874342792,
   1.04238158880820, 1.06842008128700, 1.10399010936759, 1.15102748242645, 1.21171811910125,
   1.28854264865128, 1.38432619380991, 1.50229418757368},
  {1.00011490538261, 1.00115246376914, 1.00405357333264, 1.00979590573153, 1.01941300472994,
   1.03401425035436, 1.05480599606629, 1.08311420301813, 1.12040891660892, 1.16833095655446,
   1.22872122288238, 1.30365305707817, 1.39546814053678, 1.50681646209583},
  {1.00009404750752, 1.00094291696343, 1.00331449056444, 1.00800294833816, 1.01584236259140,
   1.02772083317705, 1.04459535422831, 1.06750761206125, 1.09760092545889, 1.13613855366157,
   1.18452361426236, 1.24432087304475, 1.31728069083392, 1.40536543893560, 1.51077872501845},
  {1.00007794828179, 1.00078126847253, 1.00274487974401, 1.00662291017015, 1.01309858836971,
   1.02289448329337, 1.03678321409983, 1.05559875719896, 1.08024848405560, 1.11172607131497,
   1.15112543431072, 1.19965584614973, 1.25865841744946, 1.32962412656664, 1.41421360695576,
   1.51427891730346},
  {1.00006532421835, 1.00065457229394, 1.00229877774486, 1.00554326911736, 1.01095500750169,
   1.01913015411687, 1.03070194811914, 1.04634897780009, 1.06680393215691, 1.09286292447318,
   1.12539548508825, 1.16535532700759, 1.21379199547431, 1.27186352115440, 1.34085020626151,
   1.42216968385262, 1.51739340276302},
  {1.00005528587929, 1.00055386596109, 1.00194441667431, 1.00468643017764, 1.00925575086302,
   1.01615026747724, 1.02589581483226, 1.03905234089533, 1.05622039735333, 1.07804801455226,
   1.10523802504393, 1.13855590385702, 1.17883819807934, 1.22700162343084, 1.28405291126305,
   1.35109949588951, 1.42936113938518, 1.52018259905167},
  {1.00004720363588, 1.00047281026427, 1.00165935774692, 1.00399768913685, 1.00789119418335,
   1.01376015830695, 1.02204625617210, 1.03321722811532, 1.04777177911575, 1.06624474173252,
   1.08921254649299, 1.11729904561317, 1.15118173868339, 1.19159845208034, 1.23935452739299,
   1.29533057810180, 1.36049087815687, 1.43589245099391, 1.52269493294403},
  {1.00004062325693, 1.00040683513747, 1.00142744315642, 1.00343771758074, 1.00678268540710,
   1.01182049995714, 1.01892591212711, 1.02849387004706, 1.04094327481330, 1.05672092105986,
   1.07630565244070, 1.10021276361009, 1.12899868202683, 1.16326596487872, 1.20366864864086,
   1.25091799126016, 1.30578864971467, 1.36912533874972, 1.44185001996246, 1.52496967411643},
};

const double* orc_beta_coefficients(size_t k) {
  if (k < 1 || k > 20) return NULL;
  return kBetaRows[k - 1];
}

/* ---- smoothers.hpp ---- */
static int is_fourth(int f) { return f == ORC_FOURTH || f == ORC_FOURTH_OPT; }

static int cfg_validate(const orc_cheb_config* c) { /* smoothers.hpp:51-56 */
  const double lmax = c->lambda_max_multiplier * c->lambda_tilde;
  const double lmin = c->lambda_min_multiplier * c->lambda_tilde;
  if (c->lambda_tilde <= 0.0) return -1;
  if (lmax <= 0.0) return -1;
  if (!is_fourth(c->family) && !(0.0 < lmin && lmin < lmax)) return -1;
  return 0;
}

/* smoothers.hpp:83-91 */
static void residual_into(orc_op* A, const double* b, const double* x, int x_is_zero, double* r) {
  const size_t n = A->n;
  if (x_is_zero) {
    memcpy(r, b, n * sizeof(double));
    return;
  }
  orc_op_apply(A, x, r);
  for (size_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
}

/* smoothers.hpp:95-120 */
static void smooth_first(orc_op* A, const orc_smoother* S, const double* b, double* x,
                         int x_is_zero, size_t k, double lmin, double lmax) {
  const size_t n = A->n;
  const double theta = 0.5 * (lmax + lmin);
  const double delta = 0.5 * (lmax - lmin);
  const double sigma = theta / delta;
  double rho_prev = 1.0 / sigma;
  double* z = malloc(n * sizeof(double));
  double* d = malloc(n * sizeof(double));
  double* t = malloc(n * sizeof(double));
  double* st = S->inv_diag ? NULL : malloc(n * sizeof(double));
  residual_into(A, b, x, x_is_zero, z);
  if (S->inv_diag) {
    for (size_t i = 0; i < n; ++i) z[i] *= S->inv_diag[i];
  } else {
    memcpy(t, z, n * sizeof(double));
    S->S_apply(S->S_ctx, t, z);
  }
  for (size_t i = 0; i < n; ++i) d[i] = z[i] / theta;
  for (size_t it = 1; it < k; ++it) {
    orc_axpy(n, 1.0, d, x);
    orc_op_apply(A, d, t);
    if (S->inv_diag) {
      for (size_t i = 0; i < n; ++i) z[i] -= S->inv_diag[i] * t[i];
    } else {
      S->S_apply(S->S_ctx, t, st);
      for (size_t i = 0; i < n; ++i) z[i] -= st[i];
    }
    const double rho = 1.0 / (2.0 * sigma - rho_prev);
    const double c1 = rho * rho_prev;
    const double c2 = 2.0 * rho / delta;
    for (size_t i = 0; i < n; ++i) d[i] = c1 * d[i] + c2 * z[i];
    rho_prev = rho;
  }
  orc_axpy(n, 1.0, d, x);
  free(z); free(d); free(t); free(st);
}

/* smoothers.hpp:126-148 */
static void smooth_fourth(orc_op* A, const orc_smoother* S, const double* b, double* x,
                          int x_is_zero, size_t k, double lmax, const double* beta) {
  const size_t n = A->n;
  const double inv_lmax = 1.0 / lmax;
  double* r = malloc(n * sizeof(double));
  double* d = malloc(n * sizeof(double));
  double* t = malloc(n * sizeof(double));
  double* sr = S->inv_diag ? NULL : malloc(n * sizeof(double));
  residual_into(A, b, x, x_is_zero, r);
  if (S->inv_diag) {
    for (size_t i = 0; i < n; ++i) d[i] = (4.0 / 3.0) * inv_lmax * S->inv_diag[i] * r[i];
  } else {
    S->S_apply(S->S_ctx, r, sr);
    for (size_t i = 0; i < n; ++i) d[i] = (4.0 / 3.0) * inv_lmax * sr[i];
  }
  for (size_t it = 1; it < k; ++it) {
    const double bi = beta ? beta[it - 1] : 1.0;
    orc_axpy(n, bi, d, x);
    orc_op_apply(A, d, t);
    orc_axpy(n, -1.0, t, r);
    const double fi = (double)it;
    const double c1 = (2.0 * fi - 1.0) / (2.0 * fi + 3.0);
    const double c2 = (8.0 * fi + 4.0) / (2.0 * fi + 3.0) * inv_lmax;
    if (S->inv_diag) {
      for (size_t i = 0; i < n; ++i) d[i] = c1 * d[i] + c2 * S->inv_diag[i] * r[i];
    } else {
      S->S_apply(S->S_ctx, r, sr);
      for (size_t i = 0; i < n; ++i) d[i] = c1 * d[i] + c2 * sr[i];
    }
  }
  const double bk = beta ? beta[k - 1] : 1.0;
  orc_axpy(n, bk, d, x);
  free(r); free(d); free(t); free(sr);
}

/* smoothers.hpp:156-172 */
int orc_chebyshev_smooth(orc_op* A, const orc_smoother* S, const orc_cheb_config* cfg,
                         size_t order, const double* b, double* x, int x_is_zero) {
  if (order == 0) return 0;
  if (cfg_validate(cfg)) return -1;
  const double lmax = cfg->lambda_max_multiplier * cfg->lambda_tilde;
  if (is_fourth(cfg->family)) {
    const double* beta = NULL;
    if (cfg->family == ORC_FOURTH_OPT) {
      beta = orc_beta_coefficients(order);
      if (!beta) return -2;
    }
    smooth_fourth(A, S, b, x, x_is_zero, order, lmax, beta);
  } else {
    const double lmin = cfg->lambda_min_multiplier * cfg->lambda_tilde;
    smooth_first(A, S, b, x, x_is_zero, order, lmin, lmax);
  }
  return 0;
}

/* smoothers.hpp:61-79 */
double orc_estimate_lambda_max(orc_op* A, const orc_smoother* S, size_t iterations,
                               uint64_t seed) {
  const size_t n = A->n;
  double* v = malloc(n * sizeof(double));
  double* w = malloc(n * sizeof(double));
  double* t = S->inv_diag ? NULL : malloc(n * sizeof(double));
  orc_random_vector(n, seed, v);
  for (size_t it = 0; it <= iterations; ++it) {
    if (S->inv_diag) {
      orc_op_apply(A, v, w);
      for (size_t i = 0; i < n; ++i) w[i] *= S->inv_diag[i];
    } else {
      orc_op_apply(A, v, t);
      S->S_apply(S->S_ctx, t, w);
    }
    if (it == iterations) break;
    const double nrm = orc_norm2(n, w);
    for (size_t i = 0; i < n; ++i) v[i] = w[i] / nrm;
  }
  const double lam = orc_dot(n, v, w) / orc_dot(n, v, v);
  free(v); free(w); free(t);
  return lam;
}

/* ---- krylov.hpp ---- */
static double now_sec(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

static int all_zero(size_t n, const double* v) { /* krylov.hpp:53-57 */
  for (size_t i = 0; i < n; ++i)
    if (v[i] != 0.0) return 0;
  return 1;
}

static void finish_report(orc_solve_report* rep, const double* hist) { /* krylov.hpp:30-37 */
  if (!rep->converged && rep->status[0] == 0) snprintf(rep->status, sizeof rep->status, "maxit reached");
  if (rep->iterations > 0) {
    const double r0 = hist[0], rN = hist[rep->hist_len - 1];
    rep->rho = exp(log(rN / r0) / (double)rep->iterations);
  }
}

/* krylov.hpp:75-137 (symmetry probe omitted: it is an opt-in option) */
void orc_pcg(orc_op* A, orc_prec_fn M, void* Mctx, const double* b, const double* x0,
             const orc_solve_options* o, double* x, double* hist, orc_solve_report* rep) {
  const double t0 = now_sec();
  const size_t n = A->n;
  const size_t mv0 = A->count;
  memset(rep, 0, sizeof *rep);
  rep->rho = 1.0;
  memcpy(x, x0, n * sizeof(double));
  double* r = malloc(n * sizeof(double));
  double* z = malloc(n * sizeof(double));
  double* p = malloc(n * sizeof(double));
  double* Ap = malloc(n * sizeof(double));
  double* rt = malloc(n * sizeof(double));
  residual_into(A, b, x, all_zero(n, x0), r);
  const double r0_norm = orc_norm2(n, r);
  hist[rep->hist_len++] = r0_norm;
  if (r0_norm == 0.0) {
    rep->converged = 1;
    snprintf(rep->status, sizeof rep->status, "zero initial residual");
    rep->fine_matvecs = A->count - mv0;
    goto out;
  }
  M(Mctx, r, z);
  memcpy(p, z, n * sizeof(double));
  double rz = orc_dot(n, r, z);
  for (size_t it = 1; it <= o->maxit; ++it) {
    if (rz <= 0.0) {
      snprintf(rep->status, sizeof rep->status, "indefinite preconditioner: <r, Mr> <= 0");
      break;
    }
    orc_op_apply(A, p, Ap);
    const double pAp = orc_dot(n, p, Ap);
    if (pAp <= 0.0) {
      snprintf(rep->status, sizeof rep->status, "breakdown: <p, Ap> <= 0");
      break;
    }
    const double alpha = rz / pAp;
    orc_axpy(n, alpha, p, x);
    orc_axpy(n, -alpha, Ap, r);
    residual_into(A, b, x, 0, rt);
    const double rt_norm = orc_norm2(n, rt);
    rep->iterations = it;
    hist[rep->hist_len++] = rt_norm;
    if (rt_norm / r0_norm <= o->tol) {
      rep->converged = 1;
      break;
    }
    M(Mctx, r, z);
    const double rz_new = orc_dot(n, r, z);
    if (rz_new <= 0.0) {
      snprintf(rep->status, sizeof rep->status, "indefinite preconditioner: <r, Mr> <= 0");
      break;
    }
    const double beta = rz_new / rz;
    for (size_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
    rz = rz_new;
  }
  finish_report(rep, hist);
  rep->fine_matvecs = A->count - mv0;
out:
  rep->wall_time_sec = now_sec() - t0;
  free(r); free(z); free(p); free(Ap); free(rt);
}

/* krylov.hpp:144-264 */
void orc_pgmres(orc_op* A, orc_prec_fn M, void* Mctx, const double* b, const double* x0,
                const orc_solve_options* o, double* x, double* hist, orc_solve_report* rep) {
  const double t0 = now_sec();
  const size_t n = A->n;
  const size_t m = o->restart;
  const size_t mv0 = A->count;
  memset(rep, 0, sizeof *rep);
  rep->rho = 1.0;
  memcpy(x, x0, n * sizeof(double));
  double* r = malloc(n * sizeof(double));
  residual_into(A, b, x, all_zero(n, x0), r);
  const double r0_norm = orc_norm2(n, r);
  hist[rep->hist_len++] = r0_norm;
  if (r0_norm == 0.0) {
    rep->converged = 1;
    snprintf(rep->status, sizeof rep->status, "zero initial residual");
    rep->fine_matvecs = A->count - mv0;
    rep->wall_time_sec = now_sec() - t0;
    free(r);
    return;
  }
  double* V = malloc((m + 1) * n * sizeof(double));
  double* Z = malloc(m * n * sizeof(double));
  double* H = malloc((m + 1) * m * sizeof(double));
  double* Hs = malloc((m + 1) * m * sizeof(double));
  double* y = calloc(m, sizeof(double));
  double* g = calloc(m + 1, sizeof(double));
  double* coef = malloc((m + 1) * sizeof(double));
  double* w = malloc(n * sizeof(double));
  double* rt = malloc(n * sizeof(double));
  double* xj = malloc(n * sizeof(double));
#define Hh(i, j) H[(i) * m + (j)]
#define HS(i, j) Hs[(i) * m + (j)]
  int done = 0;
  while (!done && rep->iterations < o->maxit) {
    const double beta = orc_norm2(n, r);
    memcpy(V, r, n * sizeof(double));
    orc_scal(n, 1.0 / beta, V);
    size_t nV = 1;
    memset(H, 0, (m + 1) * m * sizeof(double));
    const double window_start_res = hist[rep->hist_len - 1];
    size_t j = 0;
    for (; j < m && rep->iterations < o->maxit; ++j) {
      M(Mctx, V + j * n, Z + j * n);
      orc_op_apply(A, Z + j * n, w);
      for (size_t i = 0; i <= j; ++i) Hh(i, j) = 0.0;
      const int passes = o->reorthogonalize ? 2 : 1;
      for (int pass = 0; pass < passes; ++pass) {
        for (size_t i = 0; i <= j; ++i) coef[i] = orc_dot(n, V + i * n, w);
        for (size_t i = 0; i <= j; ++i) {
          orc_axpy(n, -coef[i], V + i * n, w);
          Hh(i, j) += coef[i];
        }
      }
      Hh(j + 1, j) = orc_norm2(n, w);
      if (Hh(j + 1, j) > 0.0) {
        memcpy(V + nV * n, w, n * sizeof(double));
        orc_scal(n, 1.0 / Hh(j + 1, j), V + nV * n);
        nV++;
      }
      memcpy(Hs, H, (m + 1) * m * sizeof(double));
      memset(g, 0, (m + 1) * sizeof(double));
      g[0] = beta;
      for (size_t c = 0; c <= j; ++c) {
        for (size_t rr = c + 1; rr <= j + 1; ++rr) {
          const double a11 = HS(c, c), a21 = HS(rr, c);
          if (a21 == 0.0) continue;
          const double den = sqrt(a11 * a11 + a21 * a21);
          const double cs = a11 / den, sn = a21 / den;
          for (size_t cc = c; cc <= j; ++cc) {
            const double t1 = HS(c, cc), t2 = HS(rr, cc);
            HS(c, cc) = cs * t1 + sn * t2;
            HS(rr, cc) = -sn * t1 + cs * t2;
          }
          const double t1 = g[c], t2 = g[rr];
          g[c] = cs * t1 + sn * t2;
          g[rr] = -sn * t1 + cs * t2;
        }
      }
      for (size_t bi = j + 1; bi-- > 0;) {
        double s = g[bi];
        for (size_t cc = bi + 1; cc <= j; ++cc) s -= HS(bi, cc) * y[cc];
        y[bi] = s / HS(bi, bi);
      }
      memcpy(xj, x, n * sizeof(double));
      for (size_t i = 0; i <= j; ++i) orc_axpy(n, y[i], Z + i * n, xj);
      residual_into(A, b, xj, 0, rt);
      const double rt_norm = orc_norm2(n, rt);
      ++rep->iterations;
      hist[rep->hist_len++] = rt_norm;
      if (rt_norm / r0_norm <= o->tol) {
        memcpy(x, xj, n * sizeof(double));
        rep->converged = 1;
        done = 1;
        ++j;
        break;
      }
      if (j + 1 == m || rep->iterations == o->maxit) {
        memcpy(x, xj, n * sizeof(double));
        memcpy(r, rt, n * sizeof(double));
      }
      if (Hh(j + 1, j) == 0.0) {
        memcpy(x, xj, n * sizeof(double));
        snprintf(rep->status, sizeof rep->status, "breakdown: Arnoldi produced a zero vector");
        done = 1;
        break;
      }
    }
    if (done) break;
    if (hist[rep->hist_len - 1] >= window_start_res && rep->iterations < o->maxit) {
      snprintf(rep->status, sizeof rep->status,
               "stagnation: no residual decrease over a restart cycle");
      break;
    }
  }
#undef Hh
#undef HS
  finish_report(rep, hist);
  rep->fine_matvecs = A->count - mv0;
  rep->wall_time_sec = now_sec() - t0;
  free(r); free(V); free(Z); free(H); free(Hs); free(y); free(g); free(coef);
  free(w); free(rt); free(xj);
}

/* harness.hpp:118-150 */
void orc_stationary(orc_op* A, orc_prec_fn M, void* Mctx, const double* b, double tol,
                    size_t maxit, double* hist, orc_solve_report* rep) {
  const double t0 = now_sec();
  const size_t mv0 = A->count;
  const size_t n = A->n;
  memset(rep, 0, sizeof *rep);
  rep->rho = 1.0;
  double* x = calloc(n, sizeof(double));
  double* r = malloc(n * sizeof(double));
  double* t = malloc(n * sizeof(double));
  double* z = malloc(n * sizeof(double));
  memcpy(r, b, n * sizeof(double));
  const double r0 = orc_norm2(n, r);
  hist[rep->hist_len++] = r0;
  if (r0 == 0.0) {
    rep->converged = 1;
    snprintf(rep->status, sizeof rep->status, "zero initial residual");
    goto out;
  }
  for (size_t it = 1; it <= maxit; ++it) {
    M(Mctx, r, z);
    orc_axpy(n, 1.0, z, x);
    orc_op_apply(A, x, t);
    for (size_t i = 0; i < n; ++i) r[i] = b[i] - t[i];
    rep->iterations = it;
    hist[rep->hist_len++] = orc_norm2(n, r);
    if (hist[rep->hist_len - 1] / r0 <= tol) {
      rep->converged = 1;
      break;
    }
  }
  if (!rep->converged) snprintf(rep->status, sizeof rep->status, "maxit reached");
  if (rep->iterations > 0) rep->rho = exp(log(hist[rep->hist_len - 1] / hist[0]) / (double)rep->iterations);
  rep->fine_matvecs = A->count - mv0;
  rep->wall_time_sec = now_sec() - t0;
out:
  free(x); free(r); free(t); free(z);
}
