/*
 * oracle.h -- CPU restatement of the reference chebmg hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in paper_2210_03179_b200/ links or calls
 * this; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load liboracle.so, and only as the checker or the
 * CPU baseline.
 *
 * Parity status: the FD path restated here is PINNED bit-for-bit against the
 * compiled reference (oracle/_ref/libchebmg_ref.so built from
 * /root/reference/proj/include) and against the committed golden fixtures in
 * tests/golden/ (see tests/test_oracle.py).  The SEM path has no reference
 * implementation: it is a restatement of PAPER.md:540-634 + SURVEY.md App. A,
 * "parity unpinned" by the reference; it is pinned instead by analytic
 * properties (GLL exactness, symmetry, manufactured solutions, separable
 * p=1 operator) and is driven through the reference's own smoother / Krylov
 * templates in oracle/ref_driver.cpp.
 *
 * Every function cites the reference file:line it follows
 * (paths relative to /root/reference/proj/include/chebmg/).
 */
#ifndef CHEBMG_ORACLE_H
#define CHEBMG_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------- core.hpp ---------------- */
typedef struct {
  uint64_t mt[312];
  int mti;
} orc_mt64;

void orc_mt64_seed(orc_mt64* g, uint64_t seed);
uint64_t orc_mt64_next(orc_mt64* g);
double orc_uniform01(orc_mt64* g);         /* core.hpp:18-20 */
double orc_uniform_pm_half(orc_mt64* g);   /* core.hpp:23-25 */
void orc_random_vector(size_t n, uint64_t seed, double* out); /* core.hpp:27-32 */
double orc_dot(size_t n, const double* a, const double* b);    /* core.hpp:37-41 */
double orc_norm2(size_t n, const double* a);                   /* core.hpp:43 */
void orc_axpy(size_t n, double alpha, const double* x, double* y); /* core.hpp:45-47 */
void orc_scal(size_t n, double alpha, double* x);              /* core.hpp:49-51 */

/* ---------------- generic operator (operators.hpp:19-26) ---------------- */
typedef struct orc_op orc_op;
struct orc_op {
  size_t n;
  void (*apply)(orc_op* self, const double* x, double* y);
  size_t count; /* applications() counter, operators.hpp:56,63 */
};
void orc_op_apply(orc_op* op, const double* x, double* y);

/* ---------------- beta_table.hpp ---------------- */
/* returns pointer to beta_1..beta_k, or NULL if k outside 1..20 (beta_table.hpp:86-92) */
const double* orc_beta_coefficients(size_t k);

/* ---------------- smoothers.hpp ---------------- */
enum { ORC_FIRST = 0, ORC_FIRST_OPT_LAMBDA = 1, ORC_FOURTH = 2, ORC_FOURTH_OPT = 3 };

typedef struct {
  int family;
  double lambda_tilde;
  double lambda_max_multiplier; /* 1.03 default, smoothers.hpp:45 */
  double lambda_min_multiplier; /* 0.1 default, smoothers.hpp:46 */
} orc_cheb_config;

/* Smoother S: either a diagonal (inv_diag != NULL; exact reference arithmetic)
 * or a general operator apply (S_apply(S_ctx, r, out): out = S r). */
typedef struct {
  const double* inv_diag;
  void (*S_apply)(void* ctx, const double* r, double* out);
  void* S_ctx;
} orc_smoother;

/* returns 0 ok, -1 invalid config (ChebyshevConfig::validate, smoothers.hpp:51-56),
 * -2 order outside beta table (beta_table.hpp:87-89) */
int orc_chebyshev_smooth(orc_op* A, const orc_smoother* S, const orc_cheb_config* cfg,
                         size_t order, const double* b, double* x, int x_is_zero);
/* smoothers.hpp:61-79 */
double orc_estimate_lambda_max(orc_op* A, const orc_smoother* S, size_t iterations,
                               uint64_t seed);

/* ---------------- krylov.hpp ---------------- */
typedef void (*orc_prec_fn)(void* ctx, const double* v, double* z);

typedef struct {
  double tol;
  size_t maxit;
  size_t restart;
  int reorthogonalize;
} orc_solve_options;

typedef struct {
  size_t iterations;
  size_t fine_matvecs;
  double rho;
  int converged;
  char status[128];
  double wall_time_sec;
  size_t hist_len;
} orc_solve_report;

/* hist must hold maxit+1 doubles */
void orc_pcg(orc_op* A, orc_prec_fn M, void* Mctx, const double* b, const double* x0,
             const orc_solve_options* o, double* x_out, double* hist, orc_solve_report* rep);
void orc_pgmres(orc_op* A, orc_prec_fn M, void* Mctx, const double* b, const double* x0,
                const orc_solve_options* o, double* x_out, double* hist, orc_solve_report* rep);
/* harness.hpp:118-150 */
void orc_stationary(orc_op* A, orc_prec_fn M, void* Mctx, const double* b, double tol,
                    size_t maxit, double* hist, orc_solve_report* rep);

/* ---------------- FD path (domain/operators/problem/transfer/cholesky/multigrid) ---- */
typedef struct orc_fd_hier orc_fd_hier;

void orc_fd_stencil_apply(size_t n, double Lx, double Ly, const double* x, double* y);
void orc_fd_build_problem(size_t n, double Lx, double Ly, uint64_t seed, double* u, double* b);
void orc_fd_prolong(size_t n, size_t nc, const double* xc, double* y);
void orc_fd_restrict(size_t n, size_t nc, const double* x, double* yc);

/* returns NULL on invalid factor (multigrid.hpp:39-40) */
orc_fd_hier* orc_fd_hier_create(size_t n, double Lx, double Ly, size_t factor,
                                size_t eigen_iterations, uint64_t eigen_seed);
void orc_fd_hier_destroy(orc_fd_hier* h);
double orc_fd_hier_lambda_tilde(const orc_fd_hier* h);
orc_op* orc_fd_hier_op(orc_fd_hier* h);
size_t orc_fd_hier_coarse_dim(const orc_fd_hier* h);
size_t orc_fd_hier_bandwidth(const orc_fd_hier* h);
void orc_fd_hier_coarse_solve(const orc_fd_hier* h, const double* rc, double* ec);
int orc_fd_v_cycle(orc_fd_hier* h, const orc_cheb_config* s, size_t k_pre, size_t k_post,
                   const double* b, double* x, int x_is_zero);

/* Case driver: mirrors run_case (harness.hpp:230-258) for the FD problem.
 * driver: 0 pcg, 1 pgmres, 2 mg_solver. cycle: 0 full, 1 one_sided. */
typedef struct {
  double Lx;
  size_t n, factor;
  int family;
  size_t k;
  int cycle;
  int driver;
  double tol;
  size_t restart, maxit;
  uint64_t rhs_seed, eigen_seed, tuning_seed;
  double lambda_max_multiplier, lambda_min_multiplier;
  size_t eigen_iterations;
} orc_case_config;

typedef struct {
  orc_solve_report report;
  double lambda_tilde;
  double tuned_lambda_min; /* NaN unless first_opt_lambda */
} orc_case_result;

int orc_fd_run_case_with(const orc_case_config* cfg, orc_fd_hier* h, double* hist,
                         double* x_out, orc_case_result* res);

/* ---------------- SEM path (restated spec, parity unpinned) ---------------- */
typedef struct orc_sem orc_sem;

void orc_gll(int N, double* xi, double* w);                   /* A1 */
void orc_deriv_matrix(int N, const double* xi, double* D);     /* A1, D[i*(N+1)+j] = l_j'(xi_i) */
void orc_interp_matrix(int Nf, int Nc, double* J);             /* A6, J[(Nf+1) x (Nc+1)] */

/* geometry: 0 = box, 1 = Kershaw(eps) */
orc_sem* orc_sem_create(int N, int Ex, int Ey, int Ez, int geometry, double eps);
void orc_sem_destroy(orc_sem* s);
size_t orc_sem_n(const orc_sem* s);                            /* interior unknowns */
orc_op* orc_sem_op(orc_sem* s);
void orc_sem_diagonal(const orc_sem* s, double* d);            /* A5 */
void orc_sem_rhs(const orc_sem* s, double* b);
void orc_sem_local_to_global_map(const orc_sem* s, int64_t* map); /* A4, -1 = Dirichlet */
void orc_sem_geom(const orc_sem* s, double* G /* E*6*(N+1)^3 */, double* B /* E*(N+1)^3 */);
/* p-transfer between two meshes of the same element grid: A6 */
void orc_sem_prolong(const orc_sem* fine, const orc_sem* coarse, const double* xc, double* yf);
void orc_sem_restrict(const orc_sem* fine, const orc_sem* coarse, const double* xf, double* yc);
/* Schwarz smoother (A8): ras = 0 ASM, 1 RAS */
void orc_sem_schwarz(const orc_sem* s, int ras, const double* r, double* out);
void orc_sem_schwarz_apply_cb(void* ctx, const double* r, double* out); /* ctx = orc_schwarz_ctx */
typedef struct { const orc_sem* s; int ras; } orc_schwarz_ctx;

/* p-multigrid hierarchy (A6/A7/A9) */
typedef struct orc_pmg orc_pmg;
/* smoother: 0 Jacobi, 1 ASM, 2 RAS */
orc_pmg* orc_pmg_create(int nlevels, const int* orders, int Ex, int Ey, int Ez, int geometry,
                        double eps, int smoother, size_t eigen_iterations, uint64_t eigen_seed);
enum { ORC_PMG_NO_LAMBDA = 1, ORC_PMG_NO_COARSE = 2 };
orc_pmg* orc_pmg_create_ex(int nlevels, const int* orders, int Ex, int Ey, int Ez, int geometry,
                           double eps, int smoother, size_t eigen_iterations, uint64_t eigen_seed,
                           int flags);
size_t orc_sem_local_triplets(const orc_sem* s, int64_t* rows, int64_t* cols, double* vals);
void orc_pmg_destroy(orc_pmg* p);
orc_op* orc_pmg_op(orc_pmg* p, int level);
orc_sem* orc_pmg_sem(orc_pmg* p, int level);
double orc_pmg_lambda_tilde(const orc_pmg* p, int level);
int orc_pmg_v_cycle(orc_pmg* p, int family, double lmax_mult, double lmin_mult, size_t k_pre,
                    size_t k_post, const double* b, double* x, int x_is_zero);
void orc_pmg_coarse_solve(orc_pmg* p, const double* rc, double* ec);
void orc_pmg_solve(orc_pmg* p, int driver, int family, double lmaxm, double lminm, size_t kpre,
                   size_t kpost, const double* b, double tol, size_t maxit, size_t restart,
                   double* x, double* hist, orc_solve_report* rep);
void orc_kershaw_map(double eps, double x, double y, double z, double* X, double* Y, double* Z);

#ifdef __cplusplus
}
#endif

#endif
