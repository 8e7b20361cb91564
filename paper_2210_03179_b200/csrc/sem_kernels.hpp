// sem_kernels.hpp -- launch interface of the SEM kernels (k_sem.cu).
//
// Vector layout ("owned slots"): element e = ex + Ex*(ey + Ey*ez)
// (ez local to the rank's z-slab) owns the GLL nodes with local indices
// (a+1, b+1, c+1), a,b,c in [0,N); slot = e*N^3 + a + N*(b + N*c).  Slots on
// the far domain boundary are padding (kept zero).  A node with some local
// index 0 is owned by the -x/-y/-z neighbour; Dirichlet nodes are eliminated.
//
// QQ^T (direct stiffness summation) is split in two deterministic kernels:
//   K1 (element kernel): computes the local contribution at all (N+1)^3 nodes
//       of each element; nodes interior to the element (all indices in
//       1..N-1, single contributor) are finished in place with the fused
//       epilogue; the "shell" nodes are written to a shell buffer.
//   K2 (shared-node kernel): every owned node with some local index == N sums
//       its <= 8 contributions in a FIXED (dz,dy,dx) order -- the same order on
//       every partition, so results are bitwise independent of the GPU count --
//       and applies the same epilogue.
#pragma once

#include "cmg_internal.hpp"

namespace cmg {

enum SemMode : int { SEM_AX = 0, SEM_LVEC = 1 };
enum SemEpi : int {
  EPI_STORE = 0,      // y = w
  EPI_RESID = 1,      // r = b - w
  EPI_CHEB4 = 2,      // x += beta d ; r = r_in - w ; d_out = c1 d + c2 invd r
  EPI_CHEB1 = 3,      // x += d ; z -= invd w ; d_out = c1 d + c2 z
  EPI_CHEB4_INIT = 4, // r = b - w ; d_out = c0 invd r
  EPI_CHEB1_INIT = 5, // z = invd (b - w) ; d_out = z / theta
  EPI_ADD = 6,        // y += w
  // Chebyshev-Schwarz (RAS) updates fused into the assembly of the local
  // solutions (L-vector mode), invd = 1/multiplicity:
  EPI_SUPD4 = 7,      // d_out = c1 d + c2 (invd w)             (4th kind: d = c1 d + c2 S r)
  EPI_SUPD1 = 8       // [x += d] ; r = r_in - invd w ; d_out = c1 d + c2 r (1st kind: r -= S t; d = c1 d + c2 r)
};

// K2 contributor table row: [count | a<<8 | b<<16 | c<<24], then per contribution
// (shell offset relative to the owner's block) | (dx | dy<<1 | dz<<2) << 28
constexpr int K2TAB_STRIDE = 9;

struct SemArgs {
  int N = 7;
  int Ex = 1, Ey = 1, Ezl = 1;  // local element grid (Ezl element layers on this rank)
  int Ez = 1, z0 = 0;           // global layers, first global layer of this rank
  long E = 1;                   // local elements
  const double* G = nullptr;    // [E][6][(N+1)^3]
  const double* D = nullptr;    // (N+1)^2
  const int* lut = nullptr;     // local node -> shell index (-1 interior)
  const int* shared = nullptr;  // shared-owned slot list (slot-local index)
  int nshared = 0, nshell = 0;
  double* shell = nullptr;      // [E][nshell]
  const double* u = nullptr;    // AX input (slots)
  const double* lvec = nullptr; // LVEC input [E][(N+1)^3]
  const double* halo_lo = nullptr;    // [Ex*Ey*N*N] slots c=N-1 of the layer below (other rank)
  const double* contrib_hi = nullptr; // [Ex*Ey*(N+1)^2] k=0 contributions of the layer above
  // epilogue operands (slot vectors)
  double* y = nullptr;
  const double* b = nullptr;
  double* x = nullptr;
  double* r = nullptr;
  const double* r_in = nullptr;
  const double* d = nullptr;
  double* d_out = nullptr;
  const double* invd = nullptr;
  double beta = 1, c1 = 0, c2 = 0, c0 = 0, theta = 1;
  double beta_last = 0;  // > 0: last sweep step, final x += beta_k d' fused, r/d' not stored
  int x_zero = 0;
  const int* k2tab = nullptr;  // K2 contributor table [nshared][K2TAB_STRIDE] (sem.cpp)
  // element range [e_begin, e_end) processed by this launch (for overlap splits;
  // K2 needs whole element layers)
  long e_begin = 0, e_end = 0;
  int k2_z0 = 0;  // first local layer of a K2 launch (set by the launcher)
  int k1_z0 = 0;  // first local layer of a K1 line-kernel launch (grid = Ex x Ey x layers; set by the launcher)
  int prefetch_g = 0;  // K1: L2 prefetch of the element's geometric factors at block start
  // in-kernel waits on a peer's "ready" epoch (multi-GPU face exchanges over peer
  // memory): K1 runs its blocks layer 1.. first and only the layer-0 blocks, which
  // read halo_lo, wait for *k1_wait >= k1_wait_v; in K2 only the top-layer blocks,
  // which read contrib_hi, wait for *k2_wait >= k2_wait_v.  nullptr: no wait (the
  // launcher's stream already waited).
  const unsigned* k1_wait = nullptr;
  unsigned k1_wait_v = 0;
  const unsigned* k2_wait = nullptr;
  unsigned k2_wait_v = 0;
};

// upload the order-N GLL derivative matrix to constant memory (once per order)
void sem_set_derivative(int N, const double* D_host);
// K1 over elements [e_begin, e_end) and K2 over the same elements
void sem_k1(const SemArgs& a, int mode, int epi, cudaStream_t s);
void sem_k2(const SemArgs& a, int epi, cudaStream_t s);

// pointwise epilogues over all slots (x_is_zero smoother inits)
void sem_cheb4_init_zero(std::size_t n, const double* b, const double* invd, double c0, double* r,
                         double* d, cudaStream_t s);
void sem_cheb1_init_zero(std::size_t n, const double* b, const double* invd, double theta,
                         double* z, double* d, cudaStream_t s);

// halo packing
void sem_pack_top(const SemArgs& a, const double* u, double* buf, cudaStream_t s);
void sem_pack_contrib_bottom(const SemArgs& a, double* buf, cudaStream_t s);

// setup: geometric factors (and optional RHS L-vector B f), per element
struct SemGeom {
  int N, Ex, Ey, Ez, z0, Ezl;
  int geometry;  // 0 box, 1 Kershaw
  double eps;
  const double* xi;  // GLL nodes (device)
  const double* w;   // weights (device)
  const double* D;   // derivative matrix (device)
};
void sem_geometry(const SemGeom& g, double* G, double* Lrhs, double* Lmass, cudaStream_t s);
// local diagonal of A_e into an L-vector
void sem_local_diag(int N, long E, const double* G, const double* D, double* Ldiag, cudaStream_t s);
// invd = valid ? 1/diag : 0  ; flags zero diagonal entries on valid slots
void sem_inverse_diag(const SemArgs& a, const double* diag, double* invd, int* zero_flag,
                      cudaStream_t s);
// slot validity mask (1.0 valid, 0.0 padding)
void sem_slot_mask(const SemArgs& a, double* mask, cudaStream_t s);
// *flag = 1 if some valid slot of v is exactly zero
void sem_flag_zero_valid(const SemArgs& a, const double* v, int* flag, cudaStream_t s);

// p-transfers between two levels on the same element grid
// prolong: y_f (=|+=) J^{(x)3} x_c at owned fine slots; coarse gather uses halo_lo (coarse)
void sem_prolong(const SemArgs& fine, const SemArgs& coarse, const double* J, const double* xc,
                 double* yf, bool add, cudaStream_t s);
// restrict (first half): coarse L-vector = J^T^{(x)3} (fine owned values, zero elsewhere)
void sem_restrict_local(const SemArgs& fine, int Nc, const double* J, const double* xf,
                        double* Lc, cudaStream_t s);

// per-layer partial inner products: out[v*Ezl + l] = sum over layer l of V_v . w
// final_out != nullptr (one GPU, nlayers <= 4096): the per-layer sums and their
// z-ordered total in one launch straight into final_out[v] (sqrt'ed if do_sqrt),
// same bits as out + sem_layer_finalize
void sem_layer_dots(const double* V, std::size_t ldv, int nv, const double* w, long layer_len,
                    int nlayers, double* partials, double* out, cudaStream_t s, double* final_out = nullptr,
                    int do_sqrt = 0);
// fused CGS pass (nv <= 32): w -= V coef, hcol += coef, then the per-layer V^T w
void sem_layer_cgs_dots(const double* V, std::size_t ldv, int nv, const double* coef, double* w, long layer_len,
                        int nlayers, double* hcol, int hstride, double* partials, double* out, cudaStream_t s,
                        double* final_out = nullptr);
// final sum over all global layers (gathered [rank][v][layer_local] blocks) in z order
void sem_layer_finalize(const double* gathered, int nv, const int* layers_per_rank, int nranks,
                        double* out, int do_sqrt, cudaStream_t s);

// dense direct p=1 coarse solve (deformed meshes), k_sem_coarse.cu
struct CoarseGrid {
  int Ex, Ey, Ezl, z0;  // p=1 element grid of this rank's slab
  int nx, ny, nz;       // global interior vertices per direction (unknowns nx*ny*nz)
};
// colour probe vector (vertices with (ix%3, iy%3, iz%3) == (cx, cy, cz)) in slot layout
void coarse_probe(const CoarseGrid& g, int cx, int cy, int cz, double* v, cudaStream_t s);
// rows[local row][27] entries A(i, i+o) read off the probe's image y
void coarse_probe_extract(const CoarseGrid& g, int cx, int cy, int cz, const double* y, double* rows,
                          cudaStream_t s);
// dense column-major A from the gathered rows (A zeroed by the caller)
void coarse_dense_build(const CoarseGrid& g, const double* rows, double* A, cudaStream_t s);
void coarse_slots_to_dense(const CoarseGrid& g, const double* full, double* b, cudaStream_t s);
void coarse_dense_to_slots(const CoarseGrid& g, const double* x, double* ec, cudaStream_t s);
// n x n lower triangle -> full symmetric (column-major)
void coarse_symmetrize(long n, double* A, cudaStream_t s);
// y[c] = A[:, c] . b for the ncols columns of a column-major n x ncols slab (deterministic)
void coarse_coldot(long n, long ncols, const double* A, const double* b, double* y, cudaStream_t s);

// Schwarz (ASM/RAS) with FDM local solves
// On a z-slab partition (layers z0 .. z0+Ezl-1 of Ez) the extended boxes of
// the first / last owned layer reach two node planes into the layer below and
// one into the layer above; those planes arrive in rlo / rhi.  ASM also sums
// the boxes of the neighbouring layers: one Lout plane of the layer below
// (Llo) and two of the layer above (Lhi).  Ghost layouts:
//   rlo [Ex*Ey][2][N][N] (az = N-2, N-1)     rhi [Ex*Ey][N][N] (az = 0)
//   Llo [Ex*Ey][PB][PB]  (box z = N+2)       Lhi [Ex*Ey][2][PB][PB] (box z = 0, 1)
struct SchwarzArgs {
  int N = 7, Ex = 1, Ey = 1, Ez = 1;  // Ez: global element layers
  int z0 = 0, Ezl = 1;                // owned layers
  const double* S = nullptr;    // unique 1D eigenbases [nu][pb*pb] (columns, S^T B S = I)
  const double* lam = nullptr;  // [nu][pb]
  const int* sidx = nullptr;    // [E][3] index of each element's x/y/z basis
  const double* r = nullptr;    // input residual (slots)
  double* Lout = nullptr;       // local solutions (ras: (N+1)^3 per element; asm: (N+3)^3)
  const double* rlo = nullptr;
  const double* rhi = nullptr;
  const double* Llo = nullptr;
  const double* Lhi = nullptr;
  int ras = 1;
};
void sem_schwarz_local(const SchwarzArgs& a, cudaStream_t s);
// ASM: y = W sum_e R_e^T Lout_e  (W = 1/number of covering subdomains)
// optional fused Chebyshev update of the ASM result sv (kind 0: y = sv;
// 4: d = c1 d + c2 sv; 1: r -= sv, d = c1 d + c2 r)
struct AsmUpdate {
  int kind = 0;
  double c1 = 0, c2 = 0;
  double* d = nullptr;
  double* r = nullptr;
  double* x = nullptr;  // kind 1: x += d first (x = d if x_zero)
  int x_zero = 0;
};
void sem_asm_gather(const SchwarzArgs& a, double* y, cudaStream_t s, const AsmUpdate& u = AsmUpdate{});
// pack the faces the neighbouring slabs need: r planes (what = 0) before the
// local solves, ASM Lout planes (what = 1) after them
void sem_schwarz_pack(const SchwarzArgs& a, int what, double* up, double* dn, cudaStream_t s);
// ghost sizes in doubles: up-going (= rlo / Llo) and down-going (= rhi / Lhi)
inline long schwarz_ghost_up(const SchwarzArgs& a, int what) {
  const long pb = a.N + 3;
  return (long)a.Ex * a.Ey * (what == 0 ? 2L * a.N * a.N : pb * pb);
}
inline long schwarz_ghost_dn(const SchwarzArgs& a, int what) {
  const long pb = a.N + 3;
  return (long)a.Ex * a.Ey * (what == 0 ? (long)a.N * a.N : 2 * pb * pb);
}

}  // namespace cmg
