/*
 * chebmg_b200.h -- C ABI of the B200-native Chebyshev-smoothed V-cycle
 * preconditioner path (libchebmg_b200.so).
 *
 * This is the drop-in boundary for the reference's C++ template layer
 * (/root/reference/proj/include/chebmg).  Each entry point
 * names the reference interface it replaces.  Conventions:
 *   - every function returns int status (cmg_status); cmg_last_error()
 *     returns the message of the calling thread's last failure.  Status
 *     codes map to the reference's exceptions: CMG_EINVAL <->
 *     std::invalid_argument, CMG_ERANGE <-> std::out_of_range,
 *     CMG_ERUNTIME <-> std::runtime_error.  Numerical breakdowns are NOT
 *     errors: they are reported in cmg_solve_report.status exactly like
 *     SolveReport::status (krylov.hpp:18-26).
 *   - vectors are DEVICE pointers (double*) on the context's device unless a
 *     parameter is suffixed _host.  All work is stream-ordered on the
 *     context's stream; calls that return host scalars synchronise it.
 *   - one host thread per context (the reference is single-threaded,
 *     core.hpp:34-35).
 *   - SEM vectors use the "owned-slot" layout: E * N^3 slots,
 *     element-blocked; cmg_sem_* helpers convert to/from the canonical
 *     lexicographic interior ordering.  cmg_op_rows() is the number of
 *     unknowns, cmg_op_vec_len() the storage length of a device vector.
 */
#ifndef CHEBMG_B200_H
#define CHEBMG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  CMG_OK = 0,
  CMG_EINVAL = 1,   /* std::invalid_argument */
  CMG_ERANGE = 2,   /* std::out_of_range     */
  CMG_ERUNTIME = 3, /* std::runtime_error    */
  CMG_ECUDA = 4,
  CMG_ENCCL = 5
} cmg_status;

/* smoothers.hpp:14 Family */
typedef enum { CMG_FIRST = 0, CMG_FIRST_OPT_LAMBDA = 1, CMG_FOURTH = 2, CMG_FOURTH_OPT = 3 } cmg_family;

typedef struct cmg_ctx cmg_ctx;
typedef struct cmg_op cmg_op;           /* LinearOperatorLike (operators.hpp:19-26) */
typedef struct cmg_fd_hier cmg_fd_hier; /* Hierarchy (multigrid.hpp:21-31) */
typedef struct cmg_pmg cmg_pmg;         /* SEM p-multigrid hierarchy (no reference) */
typedef struct cmg_precond cmg_precond; /* Preconditioner (krylov.hpp:39) */

/* ---------------- context / memory ---------------- */
const char* cmg_last_error(void);
const char* cmg_version(void);
/* stream: a cudaStream_t (NULL = the legacy default stream) */
int cmg_ctx_create(int device, void* stream, cmg_ctx** out);
int cmg_ctx_destroy(cmg_ctx* ctx);
int cmg_ctx_synchronize(cmg_ctx* ctx);
/* number of kernels this library launched on ctx so far (evidence counter) */
uint64_t cmg_ctx_kernel_launches(const cmg_ctx* ctx);
int cmg_malloc(cmg_ctx* ctx, size_t bytes, void** dptr);
int cmg_free(cmg_ctx* ctx, void* dptr);
int cmg_upload(cmg_ctx* ctx, void* dst, const void* src_host, size_t bytes);
int cmg_download(cmg_ctx* ctx, void* dst_host, const void* src, size_t bytes);

/* ---------------- core.hpp:27-55 ---------------- */
/* host: std::mt19937_64 stream of core.hpp:18-32 (bit-identical) */
int cmg_random_vector_host(size_t n, uint64_t seed, double* out_host);
int cmg_dot(cmg_ctx* ctx, size_t n, const double* a, const double* b, double* out_host);
int cmg_norm2(cmg_ctx* ctx, size_t n, const double* a, double* out_host);
int cmg_axpy(cmg_ctx* ctx, size_t n, double alpha, const double* x, double* y);

/* ---------------- operators.hpp / domain.hpp / problem.hpp ---------------- */
/* StencilOperator(Domain(Lx, Ly, n)) -- operators.hpp:33-72, domain.hpp:17-20 */
int cmg_fd_op_create(cmg_ctx* ctx, size_t n, double Lx, double Ly, cmg_op** out);
int cmg_op_destroy(cmg_op* op);
size_t cmg_op_rows(const cmg_op* op);
size_t cmg_op_vec_len(const cmg_op* op);
int cmg_op_apply(cmg_op* op, const double* x, double* y);       /* operators.hpp:43-57 */
int cmg_op_diagonal(cmg_op* op, double* d);                      /* operators.hpp:59-61 */
size_t cmg_op_applications(const cmg_op* op);                    /* operators.hpp:63 */
void cmg_op_reset_applications(cmg_op* op);                      /* operators.hpp:64 */
/* build_problem (problem.hpp:27-45) on the host, bit-identical: u_host, b_host of (n-1)^2 */
int cmg_fd_build_problem_host(size_t n, double Lx, double Ly, uint64_t seed, double* u_host,
                              double* b_host);

/* ---------------- smoothers.hpp ---------------- */
typedef struct {
  int family;                   /* cmg_family */
  double lambda_tilde;
  double lambda_max_multiplier; /* reference default 1.03 (smoothers.hpp:45) */
  double lambda_min_multiplier; /* reference default 0.1  (smoothers.hpp:46) */
} cmg_cheb_config;

/* smoothers.hpp:174-181 (CMG_EINVAL on a zero entry) */
int cmg_jacobi_inverse_diagonal(cmg_ctx* ctx, size_t n, const double* diag, double* inv);
/* smoothers.hpp:61-79 */
int cmg_estimate_lambda_max(cmg_op* A, const double* inv_diag, size_t iterations, uint64_t seed,
                            double* out_host);
/* smoothers.hpp:156-172 */
int cmg_chebyshev_smooth(cmg_op* A, const double* inv_diag, const cmg_cheb_config* cfg,
                         size_t order, const double* b, double* x, int x_is_zero);
/* beta_coefficients (beta_table.hpp:86-92): copies beta_1..beta_k; CMG_ERANGE outside 1..20 */
int cmg_beta_coefficients(size_t k, double* out_host);

/* ---------------- multigrid.hpp ---------------- */
typedef struct {
  cmg_cheb_config smoother;
  size_t k_pre, k_post;
} cmg_cycle_config;

/* build_hierarchy (multigrid.hpp:36-48); the exact coarse solve is a
 * separable fast-diagonalisation solve of A_c = P^T A P. */
int cmg_fd_hierarchy_create(cmg_ctx* ctx, size_t n, double Lx, double Ly, size_t factor,
                            size_t eigen_iterations, uint64_t eigen_seed, cmg_fd_hier** out);
/* Same hierarchy on another context (stream), lambda_tilde copied instead of
 * re-estimated: independent scratch for concurrent solves (harness.hpp:186-201). */
int cmg_fd_hierarchy_clone(const cmg_fd_hier* src, cmg_ctx* ctx, cmg_fd_hier** out);
int cmg_fd_hierarchy_destroy(cmg_fd_hier* h);
double cmg_fd_hierarchy_lambda_tilde(const cmg_fd_hier* h);
cmg_op* cmg_fd_hierarchy_op(cmg_fd_hier* h);
const double* cmg_fd_hierarchy_inv_diag(cmg_fd_hier* h);
size_t cmg_fd_hierarchy_coarse_dim(const cmg_fd_hier* h);
int cmg_fd_prolong(cmg_fd_hier* h, const double* xc, double* y);          /* transfer.hpp:61-71 */
int cmg_fd_restrict(cmg_fd_hier* h, const double* x, double* yc);         /* transfer.hpp:74-88 */
int cmg_fd_coarse_solve(cmg_fd_hier* h, const double* rc, double* ec);    /* cholesky.hpp:44-58 */
int cmg_fd_v_cycle(cmg_fd_hier* h, const cmg_cycle_config* cfg, const double* b, double* x,
                   int x_is_zero);                                        /* multigrid.hpp:69-90 */
int cmg_fd_preconditioner_apply(cmg_fd_hier* h, const cmg_cycle_config* cfg, const double* v,
                                double* z);                               /* multigrid.hpp:94-98 */
/* Lanczos approximation constant C (lanczos.hpp:97-155, CEstimate :39-44).
 * alpha needs room for m doubles, beta for m-1 (either may be NULL);
 * *steps receives the Lanczos steps taken (alpha.size()). */
int cmg_fd_estimate_C(cmg_fd_hier* h, size_t m, uint64_t seed, int reorthogonalize, double* C,
                      double* alpha, double* beta, size_t* steps);

/* ---------------- krylov.hpp ---------------- */
typedef struct {
  double tol;
  size_t maxit;
  size_t restart;
  int reorthogonalize;
  int enforce_spd_preconditioner;
} cmg_solve_options;

typedef struct {
  size_t iterations;
  size_t fine_matvecs;
  double rho;
  int converged;
  char status[128];
  double wall_time_sec;
  double* residual_history; /* host buffer supplied by the caller (may be NULL) */
  size_t history_capacity;
  size_t history_len;       /* full length, even if > capacity */
} cmg_solve_report;

typedef void (*cmg_precond_fn)(void* user, const double* v, double* z);
int cmg_precond_fd_vcycle(cmg_fd_hier* h, const cmg_cycle_config* cfg, cmg_precond** out);
int cmg_precond_identity(cmg_ctx* ctx, cmg_precond** out);
int cmg_precond_callback(cmg_ctx* ctx, cmg_precond_fn fn, void* user, cmg_precond** out);
int cmg_precond_destroy(cmg_precond* M);
int cmg_precond_apply(cmg_precond* M, const double* v, double* z);

/* pcg / pgmres (krylov.hpp:75-137, 144-264); x0 may equal NULL (zeros) */
int cmg_pcg(cmg_op* A, cmg_precond* M, const double* b, const double* x0, double* x,
            const cmg_solve_options* opts, cmg_solve_report* rep);
int cmg_pgmres(cmg_op* A, cmg_precond* M, const double* b, const double* x0, double* x,
               const cmg_solve_options* opts, cmg_solve_report* rep);
/* detail::stationary_solve (harness.hpp:118-150) */
int cmg_stationary_solve(cmg_op* A, cmg_precond* M, const double* b, double tol, size_t maxit,
                         double* x, cmg_solve_report* rep);

/* ---------------- SEM (no reference implementation) ---------------- */
typedef struct {
  int order;              /* N (GLL points per dim N+1) */
  int ex, ey, ez;         /* global element grid */
  int geometry;           /* 0 box [-1/2,1/2]^3, 1 Kershaw(eps) */
  double eps;
  int rank, nranks;       /* z-slab partition of ez (contiguous element layers) */
} cmg_sem_desc;

/* geometric-factor SEM operator A = Q^T A_L Q with Dirichlet elimination */
int cmg_sem_op_create(cmg_ctx* ctx, const cmg_sem_desc* desc, cmg_op** out);
/* local element layer range of this rank: [z0, z1) */
int cmg_sem_partition(const cmg_sem_desc* desc, int* z0, int* z1);
/* canonical interior index of each owned slot (-1 for padding) -- gs map, host */
int cmg_sem_slot_map_host(const cmg_sem_desc* desc, int64_t* map_host);
/* canonical global index of each local node of each local element (-1 Dirichlet), host */
int cmg_sem_gs_map_host(const cmg_sem_desc* desc, int64_t* map_host);
size_t cmg_sem_local_slots(const cmg_sem_desc* desc);
/* RHS b = Q^T B f into a device slot vector */
int cmg_sem_rhs(cmg_op* op, double* b);
/* host tables the device operators are built from: GLL
 * nodes xi[N+1], weights w[N+1], derivative matrix D[(N+1)^2] (row-major,
 * D[i*(N+1)+j] = l_j'(xi_i)); interpolation J[(Nf+1)*(Nc+1)]; the 1D Schwarz
 * FDM basis S[(N+3)^2] / lam[N+3] of an extended element.  No device needed. */
int cmg_sem_basis_host(int N, double* xi, double* w, double* D);
int cmg_sem_interp_host(int Nf, int Nc, double* J);
int cmg_sem_fdm1d_host(int N, double Ll, double L, double Lr, int dl, int d0, int dN, int dr, double* S,
                       double* lam);

/* p-multigrid hierarchy: orders e.g. {7,3,1}; smoother 0 Chebyshev-Jacobi, 1 ASM, 2 RAS */
int cmg_pmg_create(cmg_ctx* ctx, const cmg_sem_desc* fine, int nlevels, const int* orders,
                   int smoother, size_t eigen_iterations, uint64_t eigen_seed, cmg_pmg** out);
int cmg_pmg_destroy(cmg_pmg* p);
cmg_op* cmg_pmg_op(cmg_pmg* p, int level);
double cmg_pmg_lambda_tilde(const cmg_pmg* p, int level);
const double* cmg_pmg_inv_diag(cmg_pmg* p, int level);
int cmg_pmg_prolong(cmg_pmg* p, int level, const double* xc, double* yf);   /* level+1 -> level */
int cmg_pmg_restrict(cmg_pmg* p, int level, const double* xf, double* yc);  /* level -> level+1 */
int cmg_pmg_coarse_solve(cmg_pmg* p, const double* rc, double* ec);
int cmg_pmg_schwarz_apply(cmg_pmg* p, int level, const double* r, double* out);
int cmg_pmg_smooth(cmg_pmg* p, int level, const cmg_cheb_config* cfg, size_t order,
                   const double* b, double* x, int x_is_zero);
int cmg_pmg_v_cycle(cmg_pmg* p, const cmg_cycle_config* cfg, const double* b, double* x,
                    int x_is_zero);
int cmg_precond_pmg(cmg_pmg* p, const cmg_cycle_config* cfg, cmg_precond** out);

/* ---------------- multi-GPU (one process per GPU) ---------------- */
/* 128-byte ncclUniqueId produced on rank 0 by cmg_nccl_unique_id, broadcast
 * by the caller (e.g. torch.distributed), then passed to every rank. */
int cmg_nccl_unique_id(unsigned char out_host[128]);
int cmg_ctx_attach_nccl(cmg_ctx* ctx, const unsigned char id_host[128], int rank, int nranks);

#ifdef __cplusplus
}
#endif

#endif /* CHEBMG_B200_H */
