// host_setup.cpp -- setup-time host math (never on the solve path).
//
// Compiled with g++ -O2 and no -march / -ffast-math so that the seeded
// inputs (core.hpp:18-32 RNG, problem.hpp:27-45 RHS) are bit-identical to the
// reference's, and the small dense eigen-decompositions are reproducible.
#include <cmath>
#include <cstring>
#include <numbers>
#include <random>
#include <vector>

#include "cmg_objects.hpp"

namespace cmg {

// core.hpp:18-32
void host_random_vector(std::size_t n, std::uint64_t seed, double* out) {
  std::mt19937_64 gen(seed);
  for (std::size_t i = 0; i < n; ++i) out[i] = static_cast<double>(gen() >> 11) * 0x1.0p-53 - 0.5;
}

// problem.hpp:27-45 (b = A u through the same stencil arithmetic, operators.hpp:43-57)
void host_fd_build_problem(std::size_t n, double Lx, double Ly, std::uint64_t seed, double* u,
                           double* b) {
  const std::size_t m = n - 1;
  const double hx = Lx / static_cast<double>(n), hy = Ly / static_cast<double>(n);
  const double pi = std::numbers::pi;
  std::mt19937_64 gen(seed);
  for (std::size_t iy = 0; iy < m; ++iy) {
    const double y = static_cast<double>(iy + 1) * hy;
    for (std::size_t ix = 0; ix < m; ++ix) {
      const double x = static_cast<double>(ix + 1) * hx;
      u[iy * m + ix] = std::sin(3.0 * pi * x / Lx) * std::sin(4.0 * pi * y / Ly) +
                       (static_cast<double>(gen() >> 11) * 0x1.0p-53 - 0.5);
    }
  }
  const double ihx2 = 1.0 / (hx * hx), ihy2 = 1.0 / (hy * hy);
  const double c = 2.0 * (ihx2 + ihy2);
  for (std::size_t iy = 0; iy < m; ++iy)
    for (std::size_t ix = 0; ix < m; ++ix) {
      const std::size_t id = iy * m + ix;
      double v = c * u[id];
      if (ix > 0) v -= ihx2 * u[id - 1];
      if (ix + 1 < m) v -= ihx2 * u[id + 1];
      if (iy > 0) v -= ihy2 * u[id - m];
      if (iy + 1 < m) v -= ihy2 * u[id + m];
      b[id] = v;
    }
}

// Optimised 4th-kind weights (beta_table.hpp:16-79; PAPER.md:1085-1256 for k<=16).
static const double kBeta[20][20] = {
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

const double* host_beta_row(std::size_t k) {
  if (k < 1 || k > 20) return nullptr;
  return kBeta[k - 1];
}

// 1D linear-interpolation weight of coarse interior node cj at fine node i
// (both 1-based), transfer.hpp:20-46
static double w1d(long i, long cj, long f) {
  const long j0 = i / f;
  const double t = static_cast<double>(i % f) / static_cast<double>(f);
  if (j0 == cj) return 1.0 - t;
  if (j0 + 1 == cj && t > 0.0) return t;
  return 0.0;
}

// A_c = P^T A P is separable: M = P1^T P1 and K = P1^T T P1 are
// symmetric tridiagonal Toeplitz (every coarse hat lies inside the fine
// interior), so both are diagonalised by the discrete sine basis.
void host_fd_coarse_eig(int n, int f, std::vector<double>& S, std::vector<double>& lam) {
  const long mf = n - 1, mc = n / f - 1;
  // entries of M and K for a column c=1 vs c and c+1 (Toeplitz: one column suffices)
  auto Pcol = [&](long cj, std::vector<double>& col) {
    col.assign(mf, 0.0);
    for (long i = 1; i <= mf; ++i) col[i - 1] = w1d(i, cj, f);
  };
  std::vector<double> p1, p2, tp1;
  const long c0 = mc >= 3 ? 2 : 1;  // interior column (unaffected by truncation)
  Pcol(c0, p1);
  tp1.assign(mf, 0.0);
  for (long i = 0; i < mf; ++i)
    tp1[i] = 2.0 * p1[i] - (i > 0 ? p1[i - 1] : 0.0) - (i + 1 < mf ? p1[i + 1] : 0.0);
  double aM = 0, aK = 0, bM = 0, bK = 0;
  for (long i = 0; i < mf; ++i) {
    aM += p1[i] * p1[i];
    aK += p1[i] * tp1[i];
  }
  if (mc >= 2) {
    Pcol(c0 + 1, p2);
    for (long i = 0; i < mf; ++i) {
      bM += p2[i] * p1[i];
      bK += p2[i] * tp1[i];
    }
  }
  S.assign(mc * mc, 0.0);
  lam.assign(mc, 0.0);
  const double pi = std::numbers::pi;
  for (long k = 1; k <= mc; ++k) {
    const double th = static_cast<double>(k) * pi / static_cast<double>(mc + 1);
    const double lm = aM + 2.0 * bM * std::cos(th), lk = aK + 2.0 * bK * std::cos(th);
    lam[k - 1] = lk / lm;
    const double nrm = std::sqrt(lm * 0.5 * static_cast<double>(mc + 1));
    for (long c = 1; c <= mc; ++c) S[(c - 1) * mc + (k - 1)] = std::sin(static_cast<double>(c) * th) / nrm;
  }
}

// ---- SEM basis ----
static void legendre(int N, double x, double* LN, double* LNm1) {
  double p0 = 1.0, p1 = x;
  if (N == 0) {
    *LN = 1.0;
    *LNm1 = 0.0;
    return;
  }
  for (int k = 2; k <= N; ++k) {
    const double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / static_cast<double>(k);
    p0 = p1;
    p1 = p2;
  }
  *LN = p1;
  *LNm1 = p0;
}

void host_gll(int N, double* xi, double* w) {
  const double pi = std::numbers::pi;
  for (int j = 0; j <= N; ++j) {
    double x = -std::cos(pi * j / N);
    if (j > 0 && j < N) {
      for (int it = 0; it < 100; ++it) {
        double LN, LNm1;
        legendre(N, x, &LN, &LNm1);
        const double LNp1 = ((2.0 * N + 1.0) * x * LN - N * LNm1) / (N + 1.0);
        const double dx = (LNp1 - LNm1) / ((2.0 * N + 1.0) * LN);
        x -= dx;
        if (std::fabs(dx) < 1e-16) break;
      }
    }
    xi[j] = x;
  }
  xi[0] = -1.0;
  xi[N] = 1.0;
  for (int j = 0; j <= N / 2; ++j) {
    const double a = 0.5 * (xi[N - j] - xi[j]);
    xi[j] = -a;
    xi[N - j] = a;
  }
  if (N % 2 == 0) xi[N / 2] = 0.0;
  for (int j = 0; j <= N; ++j) {
    double LN, LNm1;
    legendre(N, xi[j], &LN, &LNm1);
    w[j] = 2.0 / (static_cast<double>(N) * (N + 1.0) * LN * LN);
  }
}

void host_deriv_matrix(int N, const double* xi, double* D) {
  const int n1 = N + 1;
  std::vector<double> LN(n1);
  for (int j = 0; j <= N; ++j) {
    double t;
    legendre(N, xi[j], &LN[j], &t);
  }
  for (int i = 0; i <= N; ++i)
    for (int j = 0; j <= N; ++j) {
      double v = 0.0;
      if (i != j) v = LN[i] / (LN[j] * (xi[i] - xi[j]));
      else if (i == 0) v = -0.25 * N * (N + 1.0);
      else if (i == N) v = 0.25 * N * (N + 1.0);
      D[i * n1 + j] = v;
    }
}

void host_interp_matrix(int Nf, int Nc, double* J) {
  std::vector<double> xf(Nf + 1), wf(Nf + 1), xc(Nc + 1), wc(Nc + 1);
  host_gll(Nf, xf.data(), wf.data());
  host_gll(Nc, xc.data(), wc.data());
  for (int i = 0; i <= Nf; ++i)
    for (int j = 0; j <= Nc; ++j) {
      double v = 1.0;
      for (int m = 0; m <= Nc; ++m)
        if (m != j) v *= (xf[i] - xc[m]) / (xc[j] - xc[m]);
      J[i * (Nc + 1) + j] = v;
    }
}

// ---- geometry on the host (Schwarz box approximation only; the device computes the factors) ----
static double kr_right(double eps, double x) { return (x <= 0.5) ? (2.0 - eps) * x : 1.0 + eps * (x - 1.0); }
static double kr_left(double eps, double x) { return 1.0 - kr_right(eps, 1.0 - x); }
static double kr_step(double a, double b, double x) {
  if (x <= 0.0) return a;
  if (x >= 1.0) return b;
  return a + (b - a) * (x * x * x * (x * (6.0 * x - 15.0) + 10.0));
}

void host_node_coords(int geometry, double eps, const double* xi, int Ex, int Ey, int Ez, int ex, int ey,
                      int ez, int i, int j, int k, double* X, double* Y, double* Z) {
  const double x = (ex + 0.5 * (xi[i] + 1.0)) / Ex, y = (ey + 0.5 * (xi[j] + 1.0)) / Ey,
               z = (ez + 0.5 * (xi[k] + 1.0)) / Ez;
  double u = x, v = y, w = z;
  if (geometry == 1) {  // Kershaw map, as k_sem.cu / oracle_sem.c
    int layer = static_cast<int>(x * 6.0);
    if (layer > 5) layer = 5;
    const double lam = (x - layer / 6.0) * 6.0;
    switch (layer) {
      case 0: v = kr_left(eps, y); w = kr_left(eps, z); break;
      case 1:
      case 4:
        v = kr_step(kr_left(eps, y), kr_right(eps, y), lam);
        w = kr_step(kr_left(eps, z), kr_right(eps, z), lam);
        break;
      case 2:
        v = kr_step(kr_right(eps, y), kr_left(eps, y), lam / 2.0);
        w = kr_step(kr_right(eps, z), kr_left(eps, z), lam / 2.0);
        break;
      case 3:
        v = kr_step(kr_right(eps, y), kr_left(eps, y), (1.0 + lam) / 2.0);
        w = kr_step(kr_right(eps, z), kr_left(eps, z), (1.0 + lam) / 2.0);
        break;
      default: v = kr_right(eps, y); w = kr_right(eps, z); break;
    }
  }
  *X = u - 0.5;
  *Y = v - 0.5;
  *Z = w - 0.5;
}

// box approximation of an element: mean length of its 4 edges per direction
void host_element_lengths(int geometry, double eps, int N, const double* xi, int Ex, int Ey, int Ez, int ex,
                          int ey, int ez, double* L) {
  double P[8][3];
  for (int v = 0; v < 8; ++v)
    host_node_coords(geometry, eps, xi, Ex, Ey, Ez, ex, ey, ez, (v & 1) ? N : 0, (v & 2) ? N : 0,
                     (v & 4) ? N : 0, &P[v][0], &P[v][1], &P[v][2]);
  for (int d = 0; d < 3; ++d) {
    const int bit = 1 << d;
    double s = 0.0;
    for (int v = 0; v < 8; ++v)
      if (!(v & bit)) {
        const double dx = P[v | bit][0] - P[v][0], dy = P[v | bit][1] - P[v][1], dz = P[v | bit][2] - P[v][2];
        s += std::sqrt(dx * dx + dy * dy + dz * dz);
      }
    L[d] = 0.25 * s;
  }
}

// 1D extended-element operators of the Schwarz subdomain (PAPER.md:579-617,
// definition in oracle/oracle_schwarz.c): 3-element patch stiffness / GLL mass
// restricted to the N+3 extended nodes, Dirichlet-eliminated nodes decoupled.
void host_fdm_1d(int N, const double* w, const double* D, double Ll, double L, double Lr, int dl, int d0,
                 int dN, int dr, double* S, double* lam) {
  const int n1 = N + 1, pb = N + 3, np = 3 * N + 1;
  std::vector<double> K(np * np, 0.0), M(np, 0.0);
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
  std::vector<double> A(pb * pb), B(pb * pb, 0.0);
  std::vector<int> dir(pb, 0);
  if (dl) dir[0] = 1;
  if (d0) dir[0] = dir[1] = 1;
  if (dN) dir[pb - 1] = dir[pb - 2] = 1;
  if (dr) dir[pb - 1] = 1;
  for (int a = 0; a < pb; ++a) {
    B[a * pb + a] = dir[a] ? 1.0 : M[N - 1 + a];
    for (int b = 0; b < pb; ++b)
      A[a * pb + b] = (dir[a] || dir[b]) ? (a == b ? 1.0 : 0.0) : K[(N - 1 + a) * np + (N - 1 + b)];
  }
  host_sym_geneig(pb, A.data(), B.data(), S, lam);
}

// cyclic Jacobi on a symmetric matrix (destroyed); eigenvectors in columns of V
static void sym_eig(int n, double* A, double* lam, double* V) {
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) V[i * n + j] = (i == j) ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, dg = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) (i != j ? off : dg) += A[i * n + j] * A[i * n + j];
    if (off <= 1e-30 * dg) break;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = A[p * n + q];
        if (apq == 0.0) continue;
        const double theta = (A[q * n + q] - A[p * n + p]) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
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

// A s = lam B s, B SPD: B = L L^T, C = L^{-1} A L^{-T}, S = L^{-T} Q  (S^T B S = I)
void host_sym_geneig(int n, const double* A, const double* B, double* S, double* lam) {
  std::vector<double> L(n * n, 0.0), C(n * n), Q(n * n), Li(n * n, 0.0);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j <= i; ++j) {
      double s = B[i * n + j];
      for (int k = 0; k < j; ++k) s -= L[i * n + k] * L[j * n + k];
      if (i == j) {
        if (s <= 0) throw Error(ERUNTIME_, "host_sym_geneig: B not positive definite");
        L[i * n + i] = std::sqrt(s);
      } else {
        L[i * n + j] = s / L[j * n + j];
      }
    }
  for (int j = 0; j < n; ++j)  // Li = L^{-1}
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
  sym_eig(n, C.data(), lam, Q.data());
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double s = 0.0;
      for (int k = 0; k < n; ++k) s += Li[k * n + i] * Q[k * n + j];
      S[i * n + j] = s;
    }
}

}  // namespace cmg
