// sem.cpp -- host side of the spectral-element p-multigrid path.
//
// SemLevel is the LinearOperatorLike for one p-level on one rank's z-slab of
// elements (operators.hpp:19-26 shape): apply / residual / diagonal and the
// fused Chebyshev-Jacobi steps all run as K1 + K2 kernel pairs (k_sem.cu),
// with the NCCL face halo (input top face up, bottom-face contributions down)
// between them when the mesh is partitioned.  Inner products are reduced per
// element layer and summed in global z order on every rank, so every result
// is bitwise identical for 1, 2, 4 or 8 GPUs.
//
// Pmg is the p-multigrid hierarchy with the reference's
// V-cycle control flow (multigrid.hpp:69-90) applied recursively.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <tuple>
#include <string>
#include <vector>

#include <cuda.h>
#include <cusolverDn.h>

#include "cmg_objects.hpp"
#include "sem_kernels.hpp"
#include "sem_layout.hpp"

using namespace cmg;

namespace {

[[noreturn]] void fail(int code, const std::string& m) { throw cmg::Error(code, m); }

// Stream-ordered 32-bit memory operations (driver API, resolved at run time
// through the runtime's entry-point query; the library links cudart statically)
using MemOpFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
struct StreamMemOps {
  MemOpFn wait = nullptr, write = nullptr;
};
const StreamMemOps& memops() {
  static const StreamMemOps ops = [] {
    StreamMemOps o;
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      o.wait = reinterpret_cast<MemOpFn>(f);
    f = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      o.write = reinterpret_cast<MemOpFn>(f);
    return o;
  }();
  return ops;
}
bool stream_mem_ops() { return memops().wait && memops().write; }

// Every rank must take the same branch before a collective setup step: the
// per-process conditions (environment knobs, driver stream-memory-op support)
// are agreed first with one allreduce, so no rank returns early while the
// others block in the following allgather.
bool all_ranks_agree(cmg_ctx* ctx, bool local) {
  cudaStream_t s = ctx->stream;
  DBuf d(1);
  const double v = local ? 1.0 : 0.0;
  CMG_CUDA(cudaMemcpyAsync(d.p, &v, sizeof(double), cudaMemcpyHostToDevice, s));
  ctx->comm->allreduce_sum(d.p, 1, s);
  double total = 0.0;
  CMG_CUDA(cudaMemcpyAsync(&total, d.p, sizeof(double), cudaMemcpyDeviceToHost, s));
  CMG_CUDA(cudaStreamSynchronize(s));
  return total == static_cast<double>(ctx->comm->nranks);
}
// exchanges smaller than this many doubles stay on NCCL (CMG_PEER_MIN)
std::size_t peer_min_doubles() {
  static const std::size_t v = [] {
    const char* env = std::getenv("CMG_PEER_MIN");
    return env ? static_cast<std::size_t>(std::atol(env)) : static_cast<std::size_t>(32768);
  }();
  return v;
}
// the stream waits until *flag >= v (v counts up)
void stream_wait(cudaStream_t s, const unsigned* flag, unsigned v) {
  if (memops().wait(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(flag), v,
                    CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
    fail(CMG_ERUNTIME, "sem: cuStreamWaitValue32 failed");
}
// *flag = v once the stream's preceding work is complete (with a memory barrier)
void stream_write(cudaStream_t s, unsigned* flag, unsigned v) {
  if (memops().write(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(flag), v,
                     CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
    fail(CMG_ERUNTIME, "sem: cuStreamWriteValue32 failed");
}

// Two-way neighbour exchange over peer memory (the pattern of SemLevel's face
// halo, for the Schwarz ghost planes): every rank packs the part its upper
// neighbour needs and the part its lower neighbour needs into one IPC-exported,
// double-buffered buffer; consumers read them through NVLink after a
// stream-ordered "ready" flag and acknowledge so the producer may reuse the
// buffer two exchanges later.  Collective setup; all ranks fall back to NCCL
// together if any mapping fails.
struct PeerShift {
  bool on = false;
  std::size_t nu = 0, nd = 0;
  DBuf buf;                        // local [2][nu + nd]
  unsigned* flags = nullptr;       // local: ready from below, ready from above, ack from above, ack from below
  const double* buf_dn = nullptr;  // rank below's buf (mapped)
  const double* buf_up = nullptr;  // rank above's buf (mapped)
  unsigned* flags_dn = nullptr;
  unsigned* flags_up = nullptr;
  std::vector<void*> opened;
  unsigned epoch = 0;
  int up = -1, down = -1;
  PeerShift() = default;
  PeerShift(const PeerShift&) = delete;
  PeerShift& operator=(const PeerShift&) = delete;
  ~PeerShift() {
    for (void* p : opened) cudaIpcCloseMemHandle(p);
    if (flags) cudaFree(flags);
  }

  void setup(cmg_ctx* ctx, int rank, int nranks, std::size_t n_up, std::size_t n_dn) {
    if (nranks < 2) return;
    const char* env = std::getenv("CMG_PEER_HALO");
    const bool local = !(env && std::atoi(env) == 0) && stream_mem_ops() && n_up + n_dn >= peer_min_doubles();
    if (!all_ranks_agree(ctx, local)) return;
    cudaStream_t s = ctx->stream;
    nu = n_up;
    nd = n_dn;
    up = rank + 1 < nranks ? rank + 1 : -1;
    down = rank > 0 ? rank - 1 : -1;
    buf.alloc(2 * (nu + nd));
    buf.zero(s);
    CMG_CUDA(cudaMalloc(&flags, 4 * sizeof(unsigned)));
    CMG_CUDA(cudaMemsetAsync(flags, 0, 4 * sizeof(unsigned), s));
    constexpr int HB = 2 * sizeof(cudaIpcMemHandle_t);
    constexpr int HD = (HB + 7) / 8;
    std::vector<unsigned char> mine(HD * 8, 0);
    cudaIpcMemHandle_t h[2];
    CMG_CUDA(cudaIpcGetMemHandle(&h[0], buf.p));
    CMG_CUDA(cudaIpcGetMemHandle(&h[1], flags));
    std::memcpy(mine.data(), h, HB);
    DBuf dmine(HD), dall(static_cast<std::size_t>(HD) * nranks);
    CMG_CUDA(cudaMemcpyAsync(dmine.p, mine.data(), HD * 8, cudaMemcpyHostToDevice, s));
    ctx->comm->allgather(dmine.p, dall.p, HD, s);
    std::vector<unsigned char> all(static_cast<std::size_t>(HD) * 8 * nranks);
    CMG_CUDA(cudaMemcpyAsync(all.data(), dall.p, all.size(), cudaMemcpyDeviceToHost, s));
    CMG_CUDA(cudaStreamSynchronize(s));
    bool ok = true;
    auto open = [&](int r, int which) -> void* {
      cudaIpcMemHandle_t hh;
      std::memcpy(&hh, all.data() + static_cast<std::size_t>(r) * HD * 8 + which * sizeof(cudaIpcMemHandle_t),
                  sizeof(hh));
      void* p = nullptr;
      if (cudaIpcOpenMemHandle(&p, hh, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        ok = false;
        return nullptr;
      }
      opened.push_back(p);
      return p;
    };
    if (down >= 0) {
      buf_dn = static_cast<const double*>(open(down, 0));
      flags_dn = static_cast<unsigned*>(open(down, 1));
    }
    if (up >= 0) {
      buf_up = static_cast<const double*>(open(up, 0));
      flags_up = static_cast<unsigned*>(open(up, 1));
    }
    const double mine_ok = ok ? 1.0 : 0.0;
    CMG_CUDA(cudaMemcpyAsync(dmine.p, &mine_ok, sizeof(double), cudaMemcpyHostToDevice, s));
    ctx->comm->allreduce_sum(dmine.p, 1, s);
    double total = 0.0;
    CMG_CUDA(cudaMemcpyAsync(&total, dmine.p, sizeof(double), cudaMemcpyDeviceToHost, s));
    CMG_CUDA(cudaStreamSynchronize(s));
    on = total == static_cast<double>(nranks);
  }
  // where to pack this exchange's up-going and down-going parts (waits until
  // both consumers are done with the buffer from two exchanges ago)
  double* begin(cudaStream_t s) {
    const unsigned k = ++epoch;
    if (k > 2) {
      if (up >= 0) stream_wait(s, flags + 2, k - 2);
      if (down >= 0) stream_wait(s, flags + 3, k - 2);
    }
    return buf.p + (k & 1) * (nu + nd);
  }
  // after the pack: publish it, wait for the neighbours' packs, return their parts
  void post(cudaStream_t s, const double** lo, const double** hi) {
    const unsigned k = epoch;
    if (up >= 0) stream_write(s, flags_up + 0, k);
    if (down >= 0) stream_write(s, flags_dn + 1, k);
    if (down >= 0) {
      stream_wait(s, flags + 0, k);
      *lo = buf_dn + (k & 1) * (nu + nd);
    }
    if (up >= 0) {
      stream_wait(s, flags + 1, k);
      *hi = buf_up + (k & 1) * (nu + nd) + nu;
    }
  }
  // after the kernel that read the neighbours' parts
  void done(cudaStream_t s) {
    const unsigned k = epoch;
    if (down >= 0) stream_write(s, flags_dn + 2, k);
    if (up >= 0) stream_write(s, flags_up + 3, k);
  }
};

template <class F>
int guard(F&& f) {
  try {
    f();
    return CMG_OK;
  } catch (const cmg::Error& e) {
    cmg::set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    cmg::set_last_error(e.what());
    return CMG_ERUNTIME;
  }
}

struct IBuf {
  int* p = nullptr;
  void upload(const std::vector<int>& h) {
    if (p) cudaFree(p);
    CMG_CUDA(cudaMalloc(&p, std::max<std::size_t>(1, h.size()) * sizeof(int)));
    if (!h.empty()) CMG_CUDA(cudaMemcpy(p, h.data(), h.size() * sizeof(int), cudaMemcpyHostToDevice));
  }
  ~IBuf() {
    if (p) cudaFree(p);
  }
};

void validate_desc(const cmg_sem_desc& d) {
  if (d.order < 1 || d.order > 7 || d.order == 6)
    fail(CMG_EINVAL, "sem: order must be one of 1,2,3,4,5,7");
  if (d.ex < 1 || d.ey < 1 || d.ez < 1) fail(CMG_EINVAL, "sem: element counts must be positive");
  if (d.nranks < 1 || d.rank < 0 || d.rank >= d.nranks) fail(CMG_EINVAL, "sem: bad rank/nranks");
  if (d.nranks > d.ez) fail(CMG_EINVAL, "sem: more ranks than element layers");
  if (d.geometry != 0 && d.geometry != 1) fail(CMG_EINVAL, "sem: geometry must be 0 (box) or 1 (Kershaw)");
  if (d.geometry == 1 && !(d.eps > 0.0 && d.eps <= 1.0)) fail(CMG_EINVAL, "sem: Kershaw eps must be in (0,1]");
}

// z-slab partition (contiguous element layers)
void partition(const cmg_sem_desc& d, int& z0, int& z1) {
  z0 = static_cast<int>((static_cast<long>(d.rank) * d.ez) / d.nranks);
  z1 = static_cast<int>((static_cast<long>(d.rank + 1) * d.ez) / d.nranks);
}

long canonical_of_slot(const cmg_sem_desc& d, int z0, long q) {
  const int N = d.order;
  const long NOS = sem_nos(N);
  const long e = q / NOS;
  int a, b, c;
  if (!sem_abc(N, static_cast<int>(q - e * NOS), a, b, c)) return -1;  // pad slot
  const int ex = static_cast<int>(e % d.ex), ey = static_cast<int>((e / d.ex) % d.ey);
  const int ez = z0 + static_cast<int>(e / (static_cast<long>(d.ex) * d.ey));
  const long gx = static_cast<long>(ex) * N + a + 1, gy = static_cast<long>(ey) * N + b + 1,
             gz = static_cast<long>(ez) * N + c + 1;
  const long Mx = static_cast<long>(N) * d.ex - 1, My = static_cast<long>(N) * d.ey - 1,
             Mz = static_cast<long>(N) * d.ez - 1;
  if (gx > Mx || gy > My || gz > Mz) return -1;
  return ((gz - 1) * My + (gy - 1)) * Mx + (gx - 1);
}

}  // namespace

// ============================================================== SemLevel
struct SemLevel final : cmg_op {
  cmg_sem_desc desc{};
  int N = 7, Ex = 1, Ey = 1, Ez = 1, z0 = 0, z1 = 1, Ezl = 1;
  long E = 0;
  int nshell = 0, nshared = 0;
  DBuf G, Dm, xi, w, shell, halo_lo, halo_send, contrib_hi, contrib_send, diagv, mask, Lrhs;
  DBuf lpart, lout, lgath;
  IBuf lut, shared, lpr, k2tab;
  std::vector<int> lpr_h;

  SemLevel(cmg_ctx* c, const cmg_sem_desc& d) {
    validate_desc(d);
    ctx = c;
    desc = d;
    N = d.order;
    Ex = d.ex;
    Ey = d.ey;
    Ez = d.ez;
    partition(d, z0, z1);
    Ezl = z1 - z0;
    if (d.nranks > 1) {
      if (d.ez % d.nranks != 0) fail(CMG_EINVAL, "sem: ez must be divisible by nranks");
      if (!ctx->comm || ctx->nranks != d.nranks || ctx->rank != d.rank)
        fail(CMG_EINVAL, "sem: context has no matching NCCL communicator (cmg_ctx_attach_nccl)");
    }
    E = static_cast<long>(Ex) * Ey * Ezl;
    len = static_cast<std::size_t>(E * sem_nos(N));
    n = static_cast<std::size_t>((static_cast<long>(N) * Ex - 1) * (static_cast<long>(N) * Ey - 1) *
                                 (static_cast<long>(N) * Ez - 1));
    const int N1 = N + 1, NP = N1 * N1 * N1;
    // shell LUT and shared-owned list
    // Shell layout, grouped by the direction (dx,dy,dz) = (i==0, j==0, k==0) of
    // the node's owner and, inside a group, in the owner's shared-slot order:
    // K2's threads (one per owned shared slot) then read each neighbour's
    // contributions as contiguous runs, and the (0,0,0) group is the element's
    // own shared slots in slot order.
    std::vector<int> lut_h(NP, -1), sh_h;
    nshell = 0;
    static const bool lex_shell = [] {
      const char* env = std::getenv("CMG_SHELL_LEX");
      return env && std::atoi(env) == 1;
    }();
    if (lex_shell) {  // lexicographic shell order (A/B knob)
      for (int k = 0; k < N1; ++k)
        for (int j = 0; j < N1; ++j)
          for (int i = 0; i < N1; ++i)
            if (!(i >= 1 && i < N && j >= 1 && j < N && k >= 1 && k < N)) lut_h[(k * N1 + j) * N1 + i] = nshell++;
    } else {
      const int nsh = sem_nshared(N);
      for (int dz = 0; dz < 2; ++dz)
        for (int dy = 0; dy < 2; ++dy)
          for (int dx = 0; dx < 2; ++dx)
            for (int s2 = 0; s2 < nsh; ++s2) {
              int a2, b2, c2;
              sem_shared_abc(N, s2, a2, b2, c2);
              const int io = a2 + 1, jo = b2 + 1, ko = c2 + 1;  // owner-local indices
              if (io > N || jo > N || ko > N) continue;         // pad slot
              if ((dx && io != N) || (dy && jo != N) || (dz && ko != N)) continue;
              const int i = io - dx * N, j = jo - dy * N, k = ko - dz * N;
              lut_h[(k * N1 + j) * N1 + i] = nshell++;
            }
    }
    if (nshell != NP - (N - 1) * (N - 1) * (N - 1)) fail(CMG_ERUNTIME, "sem: shell layout size mismatch");
    for (int c2 = 0; c2 < N; ++c2)
      for (int b2 = 0; b2 < N; ++b2)
        for (int a2 = 0; a2 < N; ++a2)
          if (a2 == N - 1 || b2 == N - 1 || c2 == N - 1) sh_h.push_back(a2 + N * (b2 + N * c2));
    nshared = static_cast<int>(sh_h.size());
    lut.upload(lut_h);
    shared.upload(sh_h);
    // K2 contributor table: per shared slot s (interior-first order) its packed
    // (a,b,c) and its <= 8 contributions in fixed (dz,dy,dx) order, each as the
    // shell offset relative to the owner's shell block plus the direction bits
    {
      const int nsh = sem_nshared(N);
      std::vector<int> tab(static_cast<std::size_t>(nsh) * K2TAB_STRIDE, 0);
      for (int s2 = 0; s2 < nsh; ++s2) {
        int a2, b2, c2;
        sem_shared_abc(N, s2, a2, b2, c2);
        int* row = tab.data() + static_cast<std::size_t>(s2) * K2TAB_STRIDE;
        const int i = a2 + 1, j = b2 + 1, k = c2 + 1;
        int cnt = 0;
        if (i <= N && j <= N && k <= N) {  // the pad slot has no contributions
          for (int dz = 0; dz < (k == N ? 2 : 1); ++dz)
            for (int dy = 0; dy < (j == N ? 2 : 1); ++dy)
              for (int dx = 0; dx < (i == N ? 2 : 1); ++dx) {
                const int li = i - dx * N, lj = j - dy * N, lk = k - dz * N;
                const long off = (dx + static_cast<long>(Ex) * (dy + static_cast<long>(Ey) * dz)) * nshell +
                                 lut_h[(lk * N1 + lj) * N1 + li];
                if (off > 0x0fffffffL) fail(CMG_EINVAL, "sem: element rows too long for the K2 table");
                row[1 + cnt++] = static_cast<int>(off) | ((dx | (dy << 1) | (dz << 2)) << 28);
              }
        }
        row[0] = cnt | (a2 << 8) | (b2 << 16) | (c2 << 24);
      }
      k2tab.upload(tab);
    }
    // basis
    std::vector<double> xih(N1), wh(N1), Dh(N1 * N1);
    host_gll(N, xih.data(), wh.data());
    host_deriv_matrix(N, xih.data(), Dh.data());
    xi.alloc(N1);
    w.alloc(N1);
    Dm.alloc(N1 * N1);
    CMG_CUDA(cudaMemcpy(xi.p, xih.data(), N1 * sizeof(double), cudaMemcpyHostToDevice));
    CMG_CUDA(cudaMemcpy(w.p, wh.data(), N1 * sizeof(double), cudaMemcpyHostToDevice));
    CMG_CUDA(cudaMemcpy(Dm.p, Dh.data(), N1 * N1 * sizeof(double), cudaMemcpyHostToDevice));
    sem_set_derivative(N, Dh.data());
    cudaStream_t s = ctx->stream;
    // geometry on the device (setup)
    G.alloc(static_cast<std::size_t>(E) * 6 * NP);
    Lrhs.alloc(static_cast<std::size_t>(E) * NP);
    SemGeom g{N, Ex, Ey, Ez, z0, Ezl, d.geometry, d.eps, xi.p, w.p, Dm.p};
    sem_geometry(g, G.p, Lrhs.p, nullptr, s);
    shell.alloc(static_cast<std::size_t>(E) * nshell);
    halo_lo.alloc(static_cast<std::size_t>(Ex) * Ey * N * N);
    halo_send.alloc(static_cast<std::size_t>(Ex) * Ey * N * N);
    contrib_hi.alloc(static_cast<std::size_t>(Ex) * Ey * N1 * N1);
    contrib_send.alloc(static_cast<std::size_t>(Ex) * Ey * N1 * N1);
    halo_lo.zero(s);
    contrib_hi.zero(s);
    peer_setup();
    // assembled diagonal (App. A5) and the padding mask
    {
      DBuf Ld(static_cast<std::size_t>(E) * NP);
      sem_local_diag(N, E, G.p, Dm.p, Ld.p, s);
      diagv.alloc(len);
      diagv.zero(s);
      SemArgs a = args();
      a.lvec = Ld.p;
      a.y = diagv.p;
      run(SEM_LVEC, EPI_STORE, a);
      ctx->sync();
    }
    mask.alloc(len);
    sem_slot_mask(args(), mask.p, s);
    // per-layer reduction buffers (up to 64 vectors)
    lpart.alloc(static_cast<std::size_t>(64) * Ezl * 32);
    lout.alloc(static_cast<std::size_t>(64) * Ezl);
    lgath.alloc(static_cast<std::size_t>(64) * Ez);
    lpr_h.assign(d.nranks, 0);
    for (int r = 0; r < d.nranks; ++r) {
      cmg_sem_desc dr = d;
      dr.rank = r;
      int a0, a1;
      partition(dr, a0, a1);
      lpr_h[r] = a1 - a0;
    }
    lpr.upload(lpr_h);
    ctx->sync();
  }

  SemArgs args() const {
    SemArgs a;
    a.N = N;
    a.Ex = Ex;
    a.Ey = Ey;
    a.Ezl = Ezl;
    a.Ez = Ez;
    a.z0 = z0;
    a.E = E;
    a.G = G.p;
    a.D = Dm.p;
    a.lut = lut.p;
    a.shared = shared.p;
    a.nshared = nshared;
    a.nshell = nshell;
    a.k2tab = k2tab.p;
    a.shell = shell.p;
    a.halo_lo = halo_lo.p;
    a.contrib_hi = contrib_hi.p;
    a.e_begin = 0;
    a.e_end = E;
    return a;
  }

  bool distributed() const { return desc.nranks > 1; }
  int up() const { return desc.rank + 1 < desc.nranks ? desc.rank + 1 : -1; }
  int down() const { return desc.rank > 0 ? desc.rank - 1 : -1; }

  // input face halo: my top layer (c=N-1 slots) goes up, the layer below comes in
  void exchange_halo(const double* u) {
    if (!distributed()) return;
    SemArgs a = args();
    sem_pack_top(a, u, halo_send.p, ctx->stream);
    ctx->comm->sendrecv(halo_send.p, halo_send.n, halo_lo.p, halo_lo.n, up(), down(), ctx->stream);
  }
  // shell contributions of my bottom face go down, the layer above's come in
  void exchange_contrib() {
    if (!distributed()) return;
    SemArgs a = args();
    sem_pack_contrib_bottom(a, contrib_send.p, ctx->stream);
    ctx->comm->sendrecv(contrib_send.p, contrib_send.n, contrib_hi.p, contrib_hi.n, down(), up(),
                        ctx->stream);
  }

  // ---- face exchange over peer memory (no NCCL on the operator path) ----
  // Each rank IPC-exports double-buffered pack buffers and four flags; K1 of
  // the rank above reads my packed top layer straight through NVLink and K2
  // of the rank below reads my bottom-face contributions the same way.  The
  // handshake is stream-ordered memory operations on the flags (no spinning
  // kernels): a pack is followed by a flag write into the consumer's memory,
  // the consumer's stream waits for it before the kernel that reads the peer
  // buffer, then acknowledges so the producer may reuse that buffer two
  // exchanges later.  Epochs count exchanges, identical on every rank (SPMD).
  struct PeerHalo {
    bool on = false;
    std::size_t hn = 0, cn = 0;          // doubles per halo / contribution buffer
    DBuf hsend, csend;                    // local [2][hn], [2][cn] (IPC-exported)
    unsigned* flags = nullptr;            // local [4]: halo ready, halo ack, contrib ready, contrib ack
    const double* hsend_dn = nullptr;     // rank below's hsend (mapped)
    const double* csend_up = nullptr;     // rank above's csend (mapped)
    unsigned* flags_dn = nullptr;         // rank below's flags (mapped)
    unsigned* flags_up = nullptr;         // rank above's flags (mapped)
    std::vector<void*> opened;            // IPC mappings to close
    unsigned hepoch = 0, cepoch = 0;
    ~PeerHalo() {
      for (void* p : opened) cudaIpcCloseMemHandle(p);
      if (flags) cudaFree(flags);
    }
  };
  PeerHalo peer;

  void peer_setup() {
    if (!distributed()) return;
    const char* env = std::getenv("CMG_PEER_HALO");
    const bool local = !(env && std::atoi(env) == 0) && stream_mem_ops() &&
                       static_cast<std::size_t>(Ex) * Ey * N * N >= peer_min_doubles();  // small levels: NCCL
    if (!all_ranks_agree(ctx, local)) return;
    cudaStream_t s = ctx->stream;
    peer.hn = static_cast<std::size_t>(Ex) * Ey * N * N;
    peer.cn = static_cast<std::size_t>(Ex) * Ey * (N + 1) * (N + 1);
    peer.hsend.alloc(2 * peer.hn);
    peer.csend.alloc(2 * peer.cn);
    peer.hsend.zero(s);
    peer.csend.zero(s);
    CMG_CUDA(cudaMalloc(&peer.flags, 4 * sizeof(unsigned)));
    CMG_CUDA(cudaMemsetAsync(peer.flags, 0, 4 * sizeof(unsigned), s));
    // exchange the three IPC handles of every rank (packed into doubles for the allgather)
    constexpr int HB = 3 * sizeof(cudaIpcMemHandle_t);
    constexpr int HD = (HB + 7) / 8;
    std::vector<unsigned char> mine(HD * 8, 0);
    cudaIpcMemHandle_t h[3];
    CMG_CUDA(cudaIpcGetMemHandle(&h[0], peer.hsend.p));
    CMG_CUDA(cudaIpcGetMemHandle(&h[1], peer.csend.p));
    CMG_CUDA(cudaIpcGetMemHandle(&h[2], peer.flags));
    std::memcpy(mine.data(), h, HB);
    const int R = desc.nranks;
    DBuf dmine(HD), dall(static_cast<std::size_t>(HD) * R);
    CMG_CUDA(cudaMemcpyAsync(dmine.p, mine.data(), HD * 8, cudaMemcpyHostToDevice, s));
    ctx->comm->allgather(dmine.p, dall.p, HD, s);
    std::vector<unsigned char> all(static_cast<std::size_t>(HD) * 8 * R);
    CMG_CUDA(cudaMemcpyAsync(all.data(), dall.p, all.size(), cudaMemcpyDeviceToHost, s));
    CMG_CUDA(cudaStreamSynchronize(s));
    bool ok = true;
    auto open = [&](int rank, int which) -> void* {
      cudaIpcMemHandle_t hh;
      std::memcpy(&hh, all.data() + static_cast<std::size_t>(rank) * HD * 8 + which * sizeof(cudaIpcMemHandle_t),
                  sizeof(hh));
      void* p = nullptr;
      if (cudaIpcOpenMemHandle(&p, hh, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        ok = false;
        return nullptr;
      }
      peer.opened.push_back(p);
      return p;
    };
    if (down() >= 0) {
      peer.hsend_dn = static_cast<const double*>(open(down(), 0));
      peer.flags_dn = static_cast<unsigned*>(open(down(), 2));
    }
    if (up() >= 0) {
      peer.csend_up = static_cast<const double*>(open(up(), 1));
      peer.flags_up = static_cast<unsigned*>(open(up(), 2));
    }
    // all ranks switch together (and only once every mapping exists), else all keep NCCL
    const double mine_ok = ok ? 1.0 : 0.0;
    CMG_CUDA(cudaMemcpyAsync(dmine.p, &mine_ok, sizeof(double), cudaMemcpyHostToDevice, s));
    ctx->comm->allreduce_sum(dmine.p, 1, s);
    double total = 0.0;
    CMG_CUDA(cudaMemcpyAsync(&total, dmine.p, sizeof(double), cudaMemcpyDeviceToHost, s));
    CMG_CUDA(cudaStreamSynchronize(s));
    peer.on = total == static_cast<double>(R);
  }

  // In-kernel waits for the peer exchanges (CMG_PEER_KWAIT, default on): the
  // element work that does not read the neighbour's data runs while it is in
  // flight, without splitting K1/K2 into extra launches.  K1's rotated grid is
  // implemented by the line kernels (order >= 5); other orders wait on the stream.
  static bool kwait() {
    static const bool on = [] {
      const char* env = std::getenv("CMG_PEER_KWAIT");
      return !(env && std::atoi(env) == 0);
    }();
    return on;
  }
  bool kwait_k1() const { return kwait() && N >= 5 && (N + 1) % 2 == 0; }

  void run_peer(int mode, int epi, SemArgs& a) {
    cudaStream_t s = ctx->stream;
    SemArgs b = a;
    if (mode == SEM_AX) {  // input halo: my top layer up, the rank below's into my K1
      const unsigned k = ++peer.hepoch;
      const double* hs = peer.hsend.p + (k & 1) * peer.hn;
      if (up() >= 0) {
        if (k > 2) stream_wait(s, peer.flags + 1, k - 2);  // rank above done with this buffer
        sem_pack_top(a, a.u, const_cast<double*>(hs), s);
        stream_write(s, peer.flags_up + 0, k);
      }
      if (down() >= 0) {
        b.halo_lo = peer.hsend_dn + (k & 1) * peer.hn;
        if (kwait_k1()) {  // only the layer-0 blocks (dispatched last) wait, inside K1
          b.k1_wait = peer.flags + 0;
          b.k1_wait_v = k;
        } else {
          stream_wait(s, peer.flags + 0, k);
        }
      }
      sem_k1(b, mode, epi, s);
      b.k1_wait = nullptr;
      if (down() >= 0) stream_write(s, peer.flags_dn + 1, k);
    } else {
      sem_k1(b, mode, epi, s);
    }
    // shell contributions of my bottom face down, the rank above's into my K2
    const unsigned k = ++peer.cepoch;
    const double* cs = peer.csend.p + (k & 1) * peer.cn;
    if (down() >= 0) {
      if (k > 2) stream_wait(s, peer.flags + 3, k - 2);  // rank below done with this buffer
      sem_pack_contrib_bottom(a, const_cast<double*>(cs), s);
      stream_write(s, peer.flags_dn + 2, k);
    }
    if (up() >= 0) {
      b.contrib_hi = peer.csend_up + (k & 1) * peer.cn;
      if (kwait()) {  // only the top-layer blocks (dispatched last) wait, inside K2
        b.k2_wait = peer.flags + 2;
        b.k2_wait_v = k;
      } else {
        stream_wait(s, peer.flags + 2, k);
      }
    }
    sem_k2(b, epi, s);
    if (up() >= 0) stream_write(s, peer.flags_up + 3, k);
  }

  void run(int mode, int epi, SemArgs& a) {
    if (peer.on) {
      run_peer(mode, epi, a);
      return;
    }
    // split-launch overlap of the face exchanges (below), opt-in: measured 67.5
    // vs 68.3 GDOF-step/s without it at 2 GPUs -- the extra launch tails of the
    // one-layer K1/K2 pieces cost more than the hidden NCCL latency
    static const bool overlap = [] {
      const char* env = std::getenv("CMG_SEM_OVERLAP");
      return env && std::atoi(env) == 1;
    }();
    if (!distributed() || Ezl < 2 || !overlap) {
      if (mode == SEM_AX) exchange_halo(a.u);
      sem_k1(a, mode, epi, ctx->stream);
      exchange_contrib();
      sem_k2(a, epi, ctx->stream);
      return;
    }
    // Partitioned: both face exchanges run on the communicator's side stream,
    // hidden behind element work that does not need them --
    //   input halo   || K1 on layers 1..Ezl-1  (only layer 0 reads the halo)
    //   contributions || K2 on layers 0..Ezl-2 (only the top layer reads them)
    cudaStream_t s = ctx->stream;
    Comm& cm = *ctx->comm;
    const long LE = static_cast<long>(Ex) * Ey;
    SemArgs lo = a, hi = a;
    lo.e_begin = 0, lo.e_end = LE;
    hi.e_begin = LE, hi.e_end = E;
    if (mode == SEM_AX) {
      sem_pack_top(a, a.u, halo_send.p, s);
      CMG_CUDA(cudaEventRecord(cm.ev_ready, s));
      CMG_CUDA(cudaStreamWaitEvent(cm.side, cm.ev_ready, 0));
      cm.sendrecv(halo_send.p, halo_send.n, halo_lo.p, halo_lo.n, up(), down(), cm.side);
      CMG_CUDA(cudaEventRecord(cm.ev_halo, cm.side));
    }
    sem_k1(hi, mode, epi, s);
    if (mode == SEM_AX) CMG_CUDA(cudaStreamWaitEvent(s, cm.ev_halo, 0));
    sem_k1(lo, mode, epi, s);
    sem_pack_contrib_bottom(a, contrib_send.p, s);
    CMG_CUDA(cudaEventRecord(cm.ev_ready, s));
    CMG_CUDA(cudaStreamWaitEvent(cm.side, cm.ev_ready, 0));
    cm.sendrecv(contrib_send.p, contrib_send.n, contrib_hi.p, contrib_hi.n, down(), up(), cm.side);
    CMG_CUDA(cudaEventRecord(cm.ev_contrib, cm.side));
    SemArgs below = a, top = a;
    below.e_begin = 0, below.e_end = E - LE;
    top.e_begin = E - LE, top.e_end = E;
    sem_k2(below, epi, s);
    CMG_CUDA(cudaStreamWaitEvent(s, cm.ev_contrib, 0));
    sem_k2(top, epi, s);
  }

  void apply(const double* x, double* y) override {
    SemArgs a = args();
    a.u = x;
    a.y = y;
    run(SEM_AX, EPI_STORE, a);
    ++count;
  }
  void residual(const double* b, const double* x, double* r) override {
    SemArgs a = args();
    a.u = x;
    a.b = b;
    a.r = r;
    run(SEM_AX, EPI_RESID, a);
    ++count;
  }
  void flag_zero_entries(const double* v, int* flag) override {
    sem_flag_zero_valid(args(), v, flag, ctx->stream);
  }
  void diagonal(double* d) override {
    CMG_CUDA(cudaMemcpyAsync(d, diagv.p, len * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  }
  void cheb4_init(const double* b, const double* x, bool xz, const double* invd, double c0,
                  double* r, double* d) override {
    if (xz) {
      sem_cheb4_init_zero(len, b, invd, c0, r, d, ctx->stream);
      return;
    }
    SemArgs a = args();
    a.u = x;
    a.b = b;
    a.r = r;
    a.d_out = d;
    a.invd = invd;
    a.c0 = c0;
    run(SEM_AX, EPI_CHEB4_INIT, a);
    ++count;
  }
  void cheb4_step(double beta, double c1, double c2, bool xz, const double* invd,
                  const double* r_in, double* x, double* r, const double* d, double* d_out,
                  double beta_last) override {
    SemArgs a = args();
    a.u = d;
    a.d = d;
    a.d_out = d_out;
    a.x = x;
    a.r = r;
    a.r_in = r_in;
    a.invd = invd;
    a.beta = beta;
    a.c1 = c1;
    a.c2 = c2;
    a.beta_last = beta_last;
    a.x_zero = xz ? 1 : 0;
    run(SEM_AX, EPI_CHEB4, a);
    ++count;
  }
  void cheb1_init(const double* b, const double* x, bool xz, const double* invd, double theta,
                  double* z, double* d) override {
    if (xz) {
      sem_cheb1_init_zero(len, b, invd, theta, z, d, ctx->stream);
      return;
    }
    SemArgs a = args();
    a.u = x;
    a.b = b;
    a.r = z;
    a.d_out = d;
    a.invd = invd;
    a.theta = theta;
    run(SEM_AX, EPI_CHEB1_INIT, a);
    ++count;
  }
  void cheb1_step(double c1, double c2, bool xz, const double* invd, double* x, double* z,
                  const double* d, double* d_out, double beta_last) override {
    SemArgs a = args();
    a.u = d;
    a.d = d;
    a.d_out = d_out;
    a.x = x;
    a.r = z;
    a.invd = invd;
    a.c1 = c1;
    a.c2 = c2;
    a.beta_last = beta_last;
    a.x_zero = xz ? 1 : 0;
    run(SEM_AX, EPI_CHEB1, a);
    ++count;
  }

  // deterministic, partition-independent inner products (sem_kernels.hpp)
  void layer_reduce(const double* V, std::size_t ldv, int nv, const double* w, double* out,
                    bool do_sqrt) {
    if (nv > 64) fail(CMG_EINVAL, "sem: too many vectors in one reduction");
    const long layer_len = static_cast<long>(Ex) * Ey * sem_nos(N);
    if (!distributed() && Ezl <= 4096) {  // per-layer sums and their z-ordered total in one launch
      sem_layer_dots(V, ldv, nv, w, layer_len, Ezl, lpart.p, lout.p, ctx->stream, out, do_sqrt ? 1 : 0);
      return;
    }
    sem_layer_dots(V, ldv, nv, w, layer_len, Ezl, lpart.p, lout.p, ctx->stream);
    const double* g = lout.p;
    if (distributed()) {
      ctx->comm->allgather(lout.p, lgath.p, static_cast<std::size_t>(nv) * Ezl, ctx->stream);
      g = lgath.p;
    }
    sem_layer_finalize(g, nv, lpr.p, desc.nranks, out, do_sqrt ? 1 : 0, ctx->stream);
  }
  void dot(const double* a, const double* b, double* out) override { layer_reduce(a, 0, 1, b, out, false); }
  void norm2(const double* a, double* out) override { layer_reduce(a, 0, 1, a, out, true); }
  void mdot(const double* V, std::size_t ldv, int nv, const double* w, double* out) override {
    for (int c0 = 0; c0 < nv; c0 += 64)  // each inner product is reduced independently
      layer_reduce(V + static_cast<std::size_t>(c0) * ldv, ldv, std::min(64, nv - c0), w, out + c0, false);
  }
  void cgs_mdot(const double* V, std::size_t ldv, int nv, const double* coef_in, double* w, double* out,
                double* hcol, int hstride) override {
    if (nv > 32) {
      launch_cgs_update(V, ldv, nv, coef_in, w, len, hcol, hstride, ctx->stream);
      layer_reduce(V, ldv, nv, w, out, false);
      return;
    }
    const long layer_len = static_cast<long>(Ex) * Ey * sem_nos(N);
    if (!distributed() && Ezl <= 4096) {
      sem_layer_cgs_dots(V, ldv, nv, coef_in, w, layer_len, Ezl, hcol, hstride, lpart.p, lout.p, ctx->stream, out);
      return;
    }
    sem_layer_cgs_dots(V, ldv, nv, coef_in, w, layer_len, Ezl, hcol, hstride, lpart.p, lout.p, ctx->stream);
    const double* g = lout.p;
    if (distributed()) {
      ctx->comm->allgather(lout.p, lgath.p, static_cast<std::size_t>(nv) * Ezl, ctx->stream);
      g = lgath.p;
    }
    sem_layer_finalize(g, nv, lpr.p, desc.nranks, out, 0, ctx->stream);
  }

  std::vector<long> slot_map() const {
    std::vector<long> m(len);
    for (std::size_t q = 0; q < len; ++q) m[q] = canonical_of_slot(desc, z0, static_cast<long>(q));
    return m;
  }
  void upload_canonical(const double* host, double* dev) override {
    std::vector<double> h(len, 0.0);
    const auto m = slot_map();
    for (std::size_t q = 0; q < len; ++q)
      if (m[q] >= 0) h[q] = host[m[q]];
    CMG_CUDA(cudaMemcpyAsync(dev, h.data(), len * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    ctx->sync();
  }
  void download_canonical(const double* dev, double* host) override {
    std::vector<double> h(len);
    CMG_CUDA(cudaMemcpyAsync(h.data(), dev, len * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
    const auto m = slot_map();
    for (std::size_t q = 0; q < len; ++q)
      if (m[q] >= 0) host[m[q]] = h[q];
  }

  void rhs(double* b) {
    SemArgs a = args();
    a.lvec = Lrhs.p;
    a.y = b;
    CMG_CUDA(cudaMemsetAsync(b, 0, len * sizeof(double), ctx->stream));
    run(SEM_LVEC, EPI_STORE, a);
  }
};

// ============================================================== p-multigrid
struct cmg_pmg {
  cmg_ctx* ctx = nullptr;
  int nlevels = 0;
  int smoother = 0;
  std::vector<std::unique_ptr<SemLevel>> lev;
  std::vector<std::unique_ptr<DBuf>> invd, J, Lc, vr, vb, vx;
  std::vector<double> lambda;
  // coarse FDM (p=1 box): S_d, lam_d per dimension, D grid over the full p=1 slot array
  DBuf Sx, Sy, Sz, Dg, cfull, t1, t2;
  DBuf cg_r, cg_z, cg_p, cg_Ap;  // deformed-mesh coarse CG
  // Schwarz smoother data per smoothed level
  struct Schwarz {
    DBuf S, lam, Lout, wmult;
    DBuf rsend, rlo, rhi, Lsend, Llo, Lhi;  // slab faces (partitioned levels, NCCL path)
    PeerShift rpeer, Lpeer;                 // the same faces through peer memory (default)
    IBuf sidx;
    cmg_pmg* p = nullptr;
    int level = 0;
  };
  std::vector<std::unique_ptr<Schwarz>> sch;
  int cnx = 0, cny = 0, cnz = 0;
  // dense Cholesky factor of the deformed-mesh p=1 operator (k_sem_coarse.cu)
  cusolverDnHandle_t sol = nullptr;
  DBuf cS;                        // explicit inverse: this rank's column slab [cu0, cu1)
  long cu0 = 0, cu1 = 0;
  bool cinv = false;
  DBuf cA, cwork, cb, cx;
  int* cinfo = nullptr;
  int cn = 0;
  ~cmg_pmg() {
    if (sol) cusolverDnDestroy(sol);
    if (cinfo) cudaFree(cinfo);
  }
};

namespace {

void pmg_restrict(cmg_pmg* p, int l, const double* xf, double* yc) {
  SemLevel* f = p->lev[l].get();
  SemLevel* c = p->lev[l + 1].get();
  sem_restrict_local(f->args(), c->N, p->J[l]->p, xf, p->Lc[l]->p, p->ctx->stream);
  SemArgs a = c->args();
  a.lvec = p->Lc[l]->p;
  a.y = yc;
  c->run(SEM_LVEC, EPI_STORE, a);
}

void pmg_prolong(cmg_pmg* p, int l, const double* xc, double* yf, bool add) {
  SemLevel* f = p->lev[l].get();
  SemLevel* c = p->lev[l + 1].get();
  c->exchange_halo(xc);
  sem_prolong(f->args(), c->args(), p->J[l]->p, xc, yf, add, p->ctx->stream);
}

// exact p=1 solve on the box: A_1^{-1} = (Sz x Sy x Sx) D^{-1} (Sz x Sy x Sx)^T
void pmg_fdm_box(cmg_pmg* p, const double* rc, double* ec) {
  SemLevel* c = p->lev.back().get();
  cudaStream_t s = p->ctx->stream;
  if (c->N != 1) fail(CMG_EINVAL, "pmg: the coarsest level must be p=1");
  const long full = static_cast<long>(c->Ex) * c->Ey * c->Ez * sem_nos(1);
  const double* in = rc;
  if (c->distributed()) {
    p->ctx->comm->allgather(rc, p->cfull.p, c->len, s);
    in = p->cfull.p;
  }
  const int nx = p->cnx, ny = p->cny, nz = p->cnz;
  const long s0 = sem_nos(1), s1 = s0 * c->Ex, s2 = s1 * c->Ey;
  if (nx < 1 || ny < 1 || nz < 1) {  // no interior p=1 unknowns
    CMG_CUDA(cudaMemsetAsync(ec, 0, c->len * sizeof(double), s));
    return;
  }
  CMG_CUDA(cudaMemsetAsync(p->t1.p, 0, full * sizeof(double), s));
  CMG_CUDA(cudaMemsetAsync(p->t2.p, 0, full * sizeof(double), s));
  mode_product_s0(0, nx, ny, nz, s0, s1, s2, p->Sx.p, nx, true, in, p->t1.p, nullptr, s);
  mode_product_s0(1, nx, ny, nz, s0, s1, s2, p->Sy.p, ny, true, p->t1.p, p->t2.p, nullptr, s);
  mode_product_s0(2, nx, ny, nz, s0, s1, s2, p->Sz.p, nz, true, p->t2.p, p->t1.p, p->Dg.p, s);
  mode_product_s0(0, nx, ny, nz, s0, s1, s2, p->Sx.p, nx, false, p->t1.p, p->t2.p, nullptr, s);
  mode_product_s0(1, nx, ny, nz, s0, s1, s2, p->Sy.p, ny, false, p->t2.p, p->t1.p, nullptr, s);
  if (c->distributed()) {
    mode_product_s0(2, nx, ny, nz, s0, s1, s2, p->Sz.p, nz, false, p->t1.p, p->t2.p, nullptr, s);
    CMG_CUDA(cudaMemcpyAsync(ec, p->t2.p + static_cast<long>(c->z0) * s2, c->len * sizeof(double),
                             cudaMemcpyDeviceToDevice, s));
  } else {
    CMG_CUDA(cudaMemsetAsync(ec, 0, c->len * sizeof(double), s));
    mode_product_s0(2, nx, ny, nz, s0, s1, s2, p->Sz.p, nz, false, p->t1.p, ec, nullptr, s);
  }
}

// Deformed mesh: assemble the p=1 operator from 27 colour probes (k_sem_coarse.cu)
// into a dense matrix and Cholesky-factor it once (cuSOLVER), when it has at
// most CMG_COARSE_DENSE_MAX (default 46340, i.e. < 2^31 entries) unknowns;
// larger coarse problems keep the CG below.  Partitioned: every rank gathers
// all rows and factors redundantly (the coarse solve is replicated anyway).
void coarse_dense_setup(cmg_pmg* p) {
  SemLevel* C = p->lev.back().get();
  const long n = static_cast<long>(p->cnx) * p->cny * p->cnz;
  long cap = 46340;
  if (const char* env = std::getenv("CMG_COARSE_DENSE_MAX")) cap = std::min(cap, std::atol(env));
  if (n < 1 || n > cap) return;
  cudaStream_t s = p->ctx->stream;
  const CoarseGrid g{C->Ex, C->Ey, C->Ezl, C->z0, p->cnx, p->cny, p->cnz};
  const long rows_local = static_cast<long>(p->cnx) * p->cny * C->Ezl;
  DBuf v(C->len), y(C->len), rl(rows_local * 27), rg;
  rl.zero(s);
  const std::size_t cnt0 = C->count;
  for (int cz = 0; cz < 3; ++cz)
    for (int cy = 0; cy < 3; ++cy)
      for (int cx = 0; cx < 3; ++cx) {
        coarse_probe(g, cx, cy, cz, v.p, s);
        C->apply(v.p, y.p);
        coarse_probe_extract(g, cx, cy, cz, y.p, rl.p, s);
      }
  C->count = cnt0;
  const double* rows = rl.p;
  if (C->distributed()) {
    rg.alloc(static_cast<std::size_t>(rows_local) * 27 * C->desc.nranks);
    p->ctx->comm->allgather(rl.p, rg.p, static_cast<std::size_t>(rows_local) * 27, s);
    rows = rg.p;
  }
  p->cA.alloc(static_cast<std::size_t>(n) * n);
  p->cA.zero(s);
  coarse_dense_build(g, rows, p->cA.p, s);
  if (cusolverDnCreate(&p->sol) != CUSOLVER_STATUS_SUCCESS) fail(CMG_ERUNTIME, "pmg: cusolverDnCreate failed");
  cusolverDnSetStream(p->sol, s);
  int lwork = 0;
  if (cusolverDnDpotrf_bufferSize(p->sol, CUBLAS_FILL_MODE_LOWER, static_cast<int>(n), p->cA.p, static_cast<int>(n),
                                  &lwork) != CUSOLVER_STATUS_SUCCESS)
    fail(CMG_ERUNTIME, "pmg: potrf buffer size failed");
  p->cwork.alloc(std::max(lwork, 1));
  CMG_CUDA(cudaMalloc(&p->cinfo, sizeof(int)));
  if (cusolverDnDpotrf(p->sol, CUBLAS_FILL_MODE_LOWER, static_cast<int>(n), p->cA.p, static_cast<int>(n), p->cwork.p,
                       lwork, p->cinfo) != CUSOLVER_STATUS_SUCCESS)
    fail(CMG_ERUNTIME, "pmg: coarse potrf failed");
  int info = 0;
  CMG_CUDA(cudaMemcpyAsync(&info, p->cinfo, sizeof(int), cudaMemcpyDeviceToHost, s));
  CMG_CUDA(cudaStreamSynchronize(s));
  if (info != 0) fail(CMG_ERUNTIME, "pmg: coarse p=1 operator not positive definite");
  p->cb.alloc(n);
  p->cn = static_cast<int>(n);
  // Default: form the inverse from the factor once (potri) and apply it as
  // column dot products per coarse solve -- a bandwidth-bound pass instead of
  // two latency-bound triangular solves.  CMG_COARSE_INV=0 keeps potrs.
  const char* inv_env = std::getenv("CMG_COARSE_INV");
  if (inv_env && std::atoi(inv_env) == 0) return;
  int lw2 = 0;
  if (cusolverDnDpotri_bufferSize(p->sol, CUBLAS_FILL_MODE_LOWER, static_cast<int>(n), p->cA.p, static_cast<int>(n),
                                  &lw2) != CUSOLVER_STATUS_SUCCESS)
    fail(CMG_ERUNTIME, "pmg: potri buffer size failed");
  if (static_cast<std::size_t>(lw2) > p->cwork.n) p->cwork.alloc(lw2);
  if (cusolverDnDpotri(p->sol, CUBLAS_FILL_MODE_LOWER, static_cast<int>(n), p->cA.p, static_cast<int>(n), p->cwork.p,
                       lw2, p->cinfo) != CUSOLVER_STATUS_SUCCESS)
    fail(CMG_ERUNTIME, "pmg: coarse potri failed");
  CMG_CUDA(cudaMemcpyAsync(&info, p->cinfo, sizeof(int), cudaMemcpyDeviceToHost, s));
  CMG_CUDA(cudaStreamSynchronize(s));
  if (info != 0) fail(CMG_ERUNTIME, "pmg: coarse inverse failed");
  // Keep only the columns of the (symmetric) inverse whose unknowns this rank
  // owns: p=1 unknown (ix, iy, iz) lives in element layer iz, so a z-slab's
  // unknowns are one contiguous column range and each rank reads n x (its
  // unknowns) per coarse solve instead of the whole matrix.
  coarse_symmetrize(n, p->cA.p, s);
  const long layer = static_cast<long>(p->cnx) * p->cny;
  p->cu0 = std::min<long>(n, layer * C->z0);
  p->cu1 = std::min<long>(n, layer * (C->z0 + C->Ezl));
  if (p->cu0 == 0 && p->cu1 == n) {  // one rank: the slab is the whole matrix
    std::swap(p->cS.p, p->cA.p);
    std::swap(p->cS.n, p->cA.n);
  } else {
    p->cS.alloc(static_cast<std::size_t>(n) * std::max<long>(p->cu1 - p->cu0, 1));
    CMG_CUDA(cudaMemcpyAsync(p->cS.p, p->cA.p + p->cu0 * n,
                             static_cast<std::size_t>(n) * (p->cu1 - p->cu0) * sizeof(double),
                             cudaMemcpyDeviceToDevice, s));
    CMG_CUDA(cudaStreamSynchronize(s));
  }
  p->cA.release();
  p->cinv = true;
  p->cx.alloc(n);
}

// p=1 solve.  Box: the FDM solve is exact.  Deformed (Kershaw) mesh: the
// rediscretised p=1 operator is not separable, so the coarse solve is CG on
// A_1 preconditioned by the box FDM, run to a relative residual of 1e-13
// (numerically exact; the paper's single CPU BoomerAMG V-cycle, PAPER.md:618-622,
// is replaced by this all-GPU solve -- no CPU fallback).
void pmg_coarse_solve(cmg_pmg* p, const double* rc, double* ec) {
  SemLevel* c = p->lev.back().get();
  if (c->desc.geometry == 0) {
    pmg_fdm_box(p, rc, ec);
    return;
  }
  if (p->cn > 0) {  // dense Cholesky solve (coarse_dense_setup)
    cudaStream_t s = p->ctx->stream;
    const double* in = rc;
    if (c->distributed()) {
      p->ctx->comm->allgather(rc, p->cfull.p, c->len, s);
      in = p->cfull.p;
    }
    const CoarseGrid g{c->Ex, c->Ey, c->Ezl, c->z0, p->cnx, p->cny, p->cnz};
    coarse_slots_to_dense(g, in, p->cb.p, s);
    if (p->cinv) {  // x = A^{-1} b on this rank's unknowns: one HBM pass over its column slab
      coarse_coldot(p->cn, p->cu1 - p->cu0, p->cS.p, p->cb.p, p->cx.p + p->cu0, s);
      coarse_dense_to_slots(g, p->cx.p, ec, s);
      return;
    }
    if (cusolverDnDpotrs(p->sol, CUBLAS_FILL_MODE_LOWER, p->cn, 1, p->cA.p, p->cn, p->cb.p, p->cn, p->cinfo) !=
        CUSOLVER_STATUS_SUCCESS)
      fail(CMG_ERUNTIME, "pmg: coarse potrs failed");
    coarse_dense_to_slots(g, p->cb.p, ec, s);
    return;
  }
  cmg_ctx* ctx = p->ctx;
  cudaStream_t s = ctx->stream;
  const std::size_t L = c->len;
  double* x = ec;
  double* r = p->cg_r.p;
  double* z = p->cg_z.p;
  double* pp = p->cg_p.p;
  double* Ap = p->cg_Ap.p;
  double* sc = ctx->dscal + S_CG;
  int* stop = ctx->dflag + 12;
  const std::size_t cnt0 = c->count;
  CMG_CUDA(cudaMemsetAsync(x, 0, L * sizeof(double), s));
  CMG_CUDA(cudaMemcpyAsync(r, rc, L * sizeof(double), cudaMemcpyDeviceToDevice, s));
  CMG_CUDA(cudaMemsetAsync(stop, 0, sizeof(int), s));
  c->norm2(r, sc + 0);  // r0
  pmg_fdm_box(p, r, z);
  CMG_CUDA(cudaMemcpyAsync(pp, z, L * sizeof(double), cudaMemcpyDeviceToDevice, s));
  c->dot(r, z, sc + 1);  // rz
  CMG_CUDA(cudaMemcpyAsync(ctx->hpin, sc, sizeof(double), cudaMemcpyDeviceToHost, s));
  ctx->sync();
  const double r0 = ctx->hpin[0];
  if (r0 == 0.0) return;
  double last = r0;
  for (int it = 1; it <= 2000; ++it) {
    c->apply(pp, Ap);
    c->dot(pp, Ap, sc + 2);
    launch_pcg_alpha(sc + 1, sc + 2, sc + 3, stop, s);
    launch_axpy_dev(L, sc + 3, 1.0, pp, x, stop, s);
    launch_axpy_dev(L, sc + 3, -1.0, Ap, r, stop, s);
    if (it % 8 == 0) {
      // run to the rounding floor: stop below 1e-15 r0 or once 8 more
      // iterations no longer halve the (recursive) residual
      c->norm2(r, sc + 5);
      CMG_CUDA(cudaMemcpyAsync(ctx->hpin, sc + 5, sizeof(double), cudaMemcpyDeviceToHost, s));
      ctx->sync();
      const double rn = ctx->hpin[0];
      if (rn <= 1e-15 * r0 || (rn <= 1e-11 * r0 && rn > 0.5 * last)) break;
      last = rn;
    }
    pmg_fdm_box(p, r, z);
    c->dot(r, z, sc + 4);
    launch_pcg_beta(sc + 4, sc + 1, sc + 6, stop, s);
    launch_xpby_dev(L, z, sc + 6, pp, stop, s);
  }
  c->count = cnt0;  // coarse-level applications are not fine matvecs
}

// ---- Schwarz (ASM / RAS) smoother, PAPER.md:560-629 ----
void schwarz_setup(cmg_pmg* p, int l) {
  SemLevel* L = p->lev[l].get();
  if (L->N < 2) fail(CMG_EINVAL, "pmg: Schwarz smoothers need order >= 2");
  auto sc = std::make_unique<cmg_pmg::Schwarz>();
  sc->p = p;
  sc->level = l;
  const int N = L->N, N1 = N + 1, pb = N + 3;
  std::vector<double> xi(N1), w(N1), D(N1 * N1);
  host_gll(N, xi.data(), w.data());
  host_deriv_matrix(N, xi.data(), D.data());
  const int ne[3] = {L->Ex, L->Ey, L->Ez};
  // element box lengths of the owned layers and one neighbouring layer each side
  const long cols = static_cast<long>(L->Ex) * L->Ey;
  const int zl = std::max(L->z0 - 1, 0), zh = std::min(L->z1 + 1, L->Ez);
  std::vector<double> Lel(static_cast<std::size_t>(cols) * (zh - zl) * 3);
  auto lel = [&](const int* c) { return &Lel[((c[2] - zl) * cols + c[0] + static_cast<long>(L->Ex) * c[1]) * 3]; };
  for (int ez = zl; ez < zh; ++ez)
    for (int ey = 0; ey < L->Ey; ++ey)
      for (int ex = 0; ex < L->Ex; ++ex) {
        const int c[3] = {ex, ey, ez};
        host_element_lengths(L->desc.geometry, L->desc.eps, N, xi.data(), L->Ex, L->Ey, L->Ez, ex, ey, ez, lel(c));
      }
  // 1D FDM bases, deduplicated on (Ll, L, Lr, boundary flags)
  std::map<std::tuple<double, double, double, int>, int> uniq;
  std::vector<double> Sall, lall;
  std::vector<int> sidx(static_cast<std::size_t>(L->E) * 3);
  std::vector<double> Sd(pb * pb), ld(pb);
  for (long e = 0; e < L->E; ++e) {
    const int ec[3] = {static_cast<int>(e % L->Ex), static_cast<int>((e / L->Ex) % L->Ey),
                       L->z0 + static_cast<int>(e / cols)};
    for (int d = 0; d < 3; ++d) {
      int lo[3] = {ec[0], ec[1], ec[2]}, hi[3] = {ec[0], ec[1], ec[2]};
      --lo[d];
      ++hi[d];
      const double Lc = lel(ec)[d];
      const double Ll = ec[d] > 0 ? lel(lo)[d] : Lc;
      const double Lr = ec[d] + 1 < ne[d] ? lel(hi)[d] : Lc;
      const int g0 = ec[d] * N, gmax = N * ne[d];
      const int dl = (g0 - 1) <= 0, d0 = g0 == 0, dN = g0 + N == gmax, dr = (g0 + N + 1) >= gmax;
      const int flags = dl | (d0 << 1) | (dN << 2) | (dr << 3);
      const auto key = std::make_tuple(Ll, Lc, Lr, flags);
      auto it = uniq.find(key);
      if (it == uniq.end()) {
        host_fdm_1d(N, w.data(), D.data(), Ll, Lc, Lr, dl, d0, dN, dr, Sd.data(), ld.data());
        it = uniq.emplace(key, static_cast<int>(uniq.size())).first;
        Sall.insert(Sall.end(), Sd.begin(), Sd.end());
        lall.insert(lall.end(), ld.begin(), ld.end());
      }
      sidx[e * 3 + d] = it->second;
    }
  }
  sc->S.alloc(Sall.size());
  sc->lam.alloc(lall.size());
  CMG_CUDA(cudaMemcpy(sc->S.p, Sall.data(), Sall.size() * sizeof(double), cudaMemcpyHostToDevice));
  CMG_CUDA(cudaMemcpy(sc->lam.p, lall.data(), lall.size() * sizeof(double), cudaMemcpyHostToDevice));
  sc->sidx.upload(sidx);
  const bool ras = p->smoother == 2;
  sc->Lout.alloc(static_cast<std::size_t>(L->E) * (ras ? N1 * N1 * N1 : pb * pb * pb));
  if (ras) {  // W = 1 / element multiplicity (assembled count of local copies)
    DBuf ones(static_cast<std::size_t>(L->E) * N1 * N1 * N1), cnt(L->len);
    launch_set(ones.n, 1.0, ones.p, p->ctx->stream);
    cnt.zero(p->ctx->stream);
    SemArgs a = L->args();
    a.lvec = ones.p;
    a.y = cnt.p;
    L->run(SEM_LVEC, EPI_STORE, a);
    sc->wmult.alloc(L->len);
    sem_inverse_diag(L->args(), cnt.p, sc->wmult.p, p->ctx->dflag + 13, p->ctx->stream);
    p->ctx->sync();
  }
  if (L->distributed()) {
    SchwarzArgs g;
    g.N = N;
    g.Ex = L->Ex;
    g.Ey = L->Ey;
    const long ru = schwarz_ghost_up(g, 0), rd = schwarz_ghost_dn(g, 0);
    sc->rsend.alloc(ru + rd);
    sc->rlo.alloc(ru);
    sc->rhi.alloc(rd);
    sc->rlo.zero(p->ctx->stream);
    sc->rhi.zero(p->ctx->stream);
    sc->rpeer.setup(p->ctx, L->desc.rank, L->desc.nranks, ru, rd);
    if (!ras) {
      const long lu = schwarz_ghost_up(g, 1), ld = schwarz_ghost_dn(g, 1);
      sc->Lsend.alloc(lu + ld);
      sc->Llo.alloc(lu);
      sc->Lhi.alloc(ld);
      sc->Llo.zero(p->ctx->stream);
      sc->Lhi.zero(p->ctx->stream);
      sc->Lpeer.setup(p->ctx, L->desc.rank, L->desc.nranks, lu, ld);
    }
  }
  if (static_cast<int>(p->sch.size()) <= l) p->sch.resize(l + 1);
  p->sch[l] = std::move(sc);
}

// CMG_SCHWARZ_FUSE=0: S stored, then separate vector updates
bool fused_supd() {
  static const bool on = [] {
    const char* env = std::getenv("CMG_SCHWARZ_FUSE");
    return !(env && std::atoi(env) == 0);
  }();
  return on;
}

// local solves of S applied to r on level l (exchanging the neighbour slabs'
// planes when partitioned); returns the args for the assembly
SchwarzArgs schwarz_local(cmg_pmg::Schwarz* sc, const double* r) {
  cmg_pmg* p = sc->p;
  SemLevel* L = p->lev[sc->level].get();
  cudaStream_t s = p->ctx->stream;
  SchwarzArgs a;
  a.N = L->N;
  a.Ex = L->Ex;
  a.Ey = L->Ey;
  a.Ez = L->Ez;
  a.z0 = L->z0;
  a.Ezl = L->Ezl;
  a.S = sc->S.p;
  a.lam = sc->lam.p;
  a.sidx = sc->sidx.p;
  a.r = r;
  a.Lout = sc->Lout.p;
  a.ras = p->smoother == 2;
  const bool part = L->distributed();
  if (part) {  // r planes of the neighbouring slabs
    const long ru = schwarz_ghost_up(a, 0), rd = schwarz_ghost_dn(a, 0);
    if (sc->rpeer.on) {  // read in place from the neighbours' pack buffers (NVLink)
      double* send = sc->rpeer.begin(s);
      sem_schwarz_pack(a, 0, send, send + ru, s);
      sc->rpeer.post(s, &a.rlo, &a.rhi);
    } else {  // NCCL, one group
      sem_schwarz_pack(a, 0, sc->rsend.p, sc->rsend.p + ru, s);
      p->ctx->comm->shift(sc->rsend.p, sc->rlo.p, ru, sc->rsend.p + ru, sc->rhi.p, rd, L->up(), L->down(), s);
      a.rlo = sc->rlo.p;
      a.rhi = sc->rhi.p;
    }
  }
  sem_schwarz_local(a, s);
  if (part && sc->rpeer.on) sc->rpeer.done(s);
  if (part && !a.ras) {  // ASM also sums the neighbouring layers' boxes
    const long lu = schwarz_ghost_up(a, 1), ld = schwarz_ghost_dn(a, 1);
    if (sc->Lpeer.on) {  // released by asm_done() after the gather
      double* send = sc->Lpeer.begin(s);
      sem_schwarz_pack(a, 1, send, send + lu, s);
      sc->Lpeer.post(s, &a.Llo, &a.Lhi);
    } else {
      sem_schwarz_pack(a, 1, sc->Lsend.p, sc->Lsend.p + lu, s);
      p->ctx->comm->shift(sc->Lsend.p, sc->Llo.p, lu, sc->Lsend.p + lu, sc->Lhi.p, ld, L->up(), L->down(), s);
      a.Llo = sc->Llo.p;
      a.Lhi = sc->Lhi.p;
    }
  }
  return a;
}

// after the ASM gather that read the neighbours' box planes
void asm_done(cmg_pmg::Schwarz* sc) {
  if (sc->Lpeer.on) sc->Lpeer.done(sc->p->ctx->stream);
}

// out = S_ASM r or S_RAS r on level l
void schwarz_apply(void* vctx, const double* r, double* out) {
  auto* sc = static_cast<cmg_pmg::Schwarz*>(vctx);
  cmg_pmg* p = sc->p;
  SemLevel* L = p->lev[sc->level].get();
  cudaStream_t s = p->ctx->stream;
  const SchwarzArgs a = schwarz_local(sc, r);
  if (a.ras) {
    SemArgs b = L->args();
    b.lvec = sc->Lout.p;
    b.y = out;
    L->run(SEM_LVEC, EPI_STORE, b);
    launch_mul(L->len, sc->wmult.p, out, s);
  } else {
    sem_asm_gather(a, out, s);
    asm_done(sc);
  }
}

// Chebyshev-Schwarz recurrence updates (chebyshev_smooth_S).  RAS: the
// 1/multiplicity scaling and the vector update run in the epilogue of the
// assembly of the local solutions (EPI_SUPD4 / EPI_SUPD1), so S r is never
// stored.  ASM: the same updates applied where the box solutions are summed.
void schwarz_update(void* vctx, int kind, const double* in, double c1, double c2, double* d, double* r, double* x,
                    int x_zero) {
  auto* sc = static_cast<cmg_pmg::Schwarz*>(vctx);
  cmg_pmg* p = sc->p;
  SemLevel* L = p->lev[sc->level].get();
  cudaStream_t s = p->ctx->stream;
  if (p->smoother == 2) {
    schwarz_local(sc, in);
    SemArgs b = L->args();
    b.lvec = sc->Lout.p;
    b.invd = sc->wmult.p;
    b.d = d;
    b.d_out = d;
    b.c1 = c1;
    b.c2 = c2;
    if (kind == 1) {
      b.r_in = r;
      b.r = r;
      b.x = x;
      b.x_zero = x_zero;
    }
    L->run(SEM_LVEC, kind == 4 ? EPI_SUPD4 : EPI_SUPD1, b);
    return;
  }
  const SchwarzArgs a = schwarz_local(sc, in);
  AsmUpdate u;
  u.kind = kind;
  u.c1 = c1;
  u.c2 = c2;
  u.d = d;
  u.r = r;
  u.x = x;
  u.x_zero = x_zero;
  sem_asm_gather(a, nullptr, s, u);
  asm_done(sc);
}

void pmg_smooth(cmg_pmg* p, int l, const cmg_cheb_config& cfg, std::size_t order, const double* b,
                double* x, bool xz) {
  if (p->smoother == 0) chebyshev_smooth(p->lev[l].get(), p->invd[l]->p, cfg, order, b, x, xz);
  else chebyshev_smooth_S(p->lev[l].get(), schwarz_apply, p->sch[l].get(), cfg, order, b, x, xz,
                          fused_supd() ? schwarz_update : nullptr);
}

// multigrid.hpp:69-90, recursively over the p-levels
void pmg_vcycle(cmg_pmg* p, int l, const cmg_cycle_config& cc, const double* b, double* x, bool xz) {
  SemLevel* L = p->lev[l].get();
  cudaStream_t s = p->ctx->stream;
  if (l == p->nlevels - 1) {
    if (xz) {
      pmg_coarse_solve(p, b, x);
    } else {
      L->residual(b, x, p->vr[l]->p);
      pmg_coarse_solve(p, p->vr[l]->p, p->vx[l]->p);
      launch_axpy(L->len, 1.0, p->vx[l]->p, x, s);
    }
    return;
  }
  cmg_cheb_config cfg = cc.smoother;
  cfg.lambda_tilde = p->lambda[l];
  if (cc.k_pre > 0) {
    pmg_smooth(p, l, cfg, cc.k_pre, b, x, xz);
    xz = false;
  }
  const double* r = b;
  if (!xz) {
    L->residual(b, x, p->vr[l]->p);
    r = p->vr[l]->p;
  }
  double* bc = p->vb[l + 1]->p;
  double* xc = p->vx[l + 1]->p;
  pmg_restrict(p, l, r, bc);
  CMG_CUDA(cudaMemsetAsync(xc, 0, p->lev[l + 1]->len * sizeof(double), s));
  pmg_vcycle(p, l + 1, cc, bc, xc, true);
  pmg_prolong(p, l, xc, x, !xz);
  if (cc.k_post > 0) pmg_smooth(p, l, cfg, cc.k_post, b, x, false);
}

// preconditioner_apply for the p-MG hierarchy (multigrid.hpp:94-98).  One V-cycle
// is ~55 launches; on one GPU each (v, z) pair it is applied to (PGMRES walks
// V_j -> Z_j, the same buffers in every solve) is captured once into a CUDA
// graph and replayed as one launch, the captured operator applications and
// kernel launches re-added to the counters.  Not captured: partitioned
// hierarchies (their peer-memory handshakes carry per-call epochs), the
// tolerance-stopped CG coarse solve and the cuSOLVER triangular solves.  The
// first apply runs directly (lazy workspaces and kernel attributes), a failed
// capture falls back to direct launches.  CMG_SEM_GRAPHS=0 disables.
struct PmgPrecond final : cmg_precond {
  cmg_pmg* p = nullptr;
  cmg_cycle_config cfg{};
  struct Captured {
    const double* v;
    double* z;
    cudaGraphExec_t exec;
    std::vector<std::size_t> counts;  // operator applications per level
    unsigned long long launches;
  };
  std::vector<Captured> graphs;
  std::vector<const double*> ws_seen;  // context workspace slots when the graphs were captured
  cudaStream_t cap = nullptr;
  bool warm = false, broken = false;

  std::vector<const double*> ws_now() const {
    std::vector<const double*> v;
    for (const auto& w : p->ctx->ws) v.push_back(w ? w->p : nullptr);
    return v;
  }

  ~PmgPrecond() override {
    for (auto& g : graphs) cudaGraphExecDestroy(g.exec);
    if (cap) cudaStreamDestroy(cap);
  }
  // deformed mesh above CMG_COARSE_DENSE_MAX: the coarse solve is the
  // tolerance-stopped CG (pmg_coarse_solve), so each V-cycle is a slightly
  // different operator
  bool variable() const override { return p->lev.back()->desc.geometry != 0 && p->cn == 0; }

  bool graph_ok() const {
    static const bool on = [] {
      const char* env = std::getenv("CMG_SEM_GRAPHS");
      return !(env && std::atoi(env) == 0);
    }();
    if (!on || broken || graphs.size() >= 128) return false;
    for (const auto& l : p->lev)
      if (l->distributed()) return false;
    const SemLevel* c = p->lev.back().get();
    return c->desc.geometry == 0 || (p->cn > 0 && p->cinv);
  }
  void direct(const double* v, double* z) {
    CMG_CUDA(cudaMemsetAsync(z, 0, p->lev[0]->len * sizeof(double), p->ctx->stream));
    pmg_vcycle(p, 0, cfg, v, z, true);
  }
  void apply(const double* v, double* z) override {
    if (!warm || !graph_ok()) {
      direct(v, z);
      warm = true;
      return;
    }
    if (ws_now() != ws_seen) {  // a context workspace (Schwarz scratch) was reallocated: recapture
      for (auto& c : graphs) cudaGraphExecDestroy(c.exec);
      graphs.clear();
      ws_seen = ws_now();
    }
    const Captured* g = nullptr;
    for (const auto& c : graphs)
      if (c.v == v && c.z == z) g = &c;
    if (!g) g = capture(v, z);
    if (!g) {
      direct(v, z);
      return;
    }
    CMG_CUDA(cudaGraphLaunch(g->exec, p->ctx->stream));
    for (std::size_t l = 0; l < p->lev.size(); ++l) p->lev[l]->count += g->counts[l];
    g_kernel_launches += g->launches;
  }
  const Captured* capture(const double* v, double* z) {
    if (!cap) CMG_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    CMG_CUDA(cudaStreamSynchronize(p->ctx->stream));
    std::vector<std::size_t> c0;
    for (const auto& l : p->lev) c0.push_back(l->count);
    const unsigned long long l0 = g_kernel_launches.load();
    cudaStream_t user = p->ctx->stream;
    p->ctx->stream = cap;
    cudaGraph_t graph = nullptr;
    bool ok = cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
    if (ok) {
      try {
        direct(v, z);
      } catch (...) {
        ok = false;
      }
      ok = (cudaStreamEndCapture(cap, &graph) == cudaSuccess) && ok && graph;
    }
    p->ctx->stream = user;
    cudaGraphExec_t exec = nullptr;
    if (ok) ok = cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess;
    if (graph) cudaGraphDestroy(graph);
    Captured c{v, z, exec, {}, g_kernel_launches.load() - l0};
    for (std::size_t l = 0; l < p->lev.size(); ++l) {
      c.counts.push_back(p->lev[l]->count - c0[l]);
      p->lev[l]->count = c0[l];  // captured, not executed
    }
    g_kernel_launches -= c.launches;
    if (!ok) {
      cudaGetLastError();
      broken = true;
      return nullptr;
    }
    graphs.push_back(std::move(c));
    ws_seen = ws_now();
    return &graphs.back();
  }
};

SemLevel* as_sem(cmg_op* op) {
  auto* s = dynamic_cast<SemLevel*>(op);
  if (!s) fail(CMG_EINVAL, "operator is not a SEM operator");
  return s;
}

}  // namespace

// ============================================================== C ABI
extern "C" {

int cmg_sem_partition(const cmg_sem_desc* d, int* z0, int* z1) {
  return guard([&] {
    validate_desc(*d);
    partition(*d, *z0, *z1);
  });
}

size_t cmg_sem_local_slots(const cmg_sem_desc* d) {
  int z0, z1;
  partition(*d, z0, z1);
  return static_cast<size_t>(d->ex) * d->ey * (z1 - z0) * sem_nos(d->order);
}

int cmg_sem_basis_host(int N, double* xi, double* w, double* D) {
  return guard([&] {
    if (N < 1 || N > 7) fail(CMG_EINVAL, "sem_basis_host: order must be 1..7");
    host_gll(N, xi, w);
    host_deriv_matrix(N, xi, D);
  });
}

int cmg_sem_interp_host(int Nf, int Nc, double* J) {
  return guard([&] {
    if (Nf < 1 || Nf > 7 || Nc < 1 || Nc > Nf) fail(CMG_EINVAL, "sem_interp_host: need 1 <= Nc <= Nf <= 7");
    host_interp_matrix(Nf, Nc, J);
  });
}

int cmg_sem_fdm1d_host(int N, double Ll, double L, double Lr, int dl, int d0, int dN, int dr, double* S,
                       double* lam) {
  return guard([&] {
    if (N < 2 || N > 7) fail(CMG_EINVAL, "sem_fdm1d_host: order must be 2..7");
    std::vector<double> xi(N + 1), w(N + 1), D((N + 1) * (N + 1));
    host_gll(N, xi.data(), w.data());
    host_deriv_matrix(N, xi.data(), D.data());
    host_fdm_1d(N, w.data(), D.data(), Ll, L, Lr, dl, d0, dN, dr, S, lam);
  });
}

int cmg_sem_slot_map_host(const cmg_sem_desc* d, int64_t* map) {
  return guard([&] {
    validate_desc(*d);
    int z0, z1;
    partition(*d, z0, z1);
    const std::size_t len = cmg_sem_local_slots(d);
    for (std::size_t q = 0; q < len; ++q) map[q] = canonical_of_slot(*d, z0, static_cast<long>(q));
  });
}

int cmg_sem_gs_map_host(const cmg_sem_desc* d, int64_t* map) {
  return guard([&] {
    validate_desc(*d);
    int z0, z1;
    partition(*d, z0, z1);
    const int N = d->order, N1 = N + 1;
    const long NP = static_cast<long>(N1) * N1 * N1;
    const long Mx = static_cast<long>(N) * d->ex - 1, My = static_cast<long>(N) * d->ey - 1;
    const long E = static_cast<long>(d->ex) * d->ey * (z1 - z0);
    for (long e = 0; e < E; ++e) {
      const int ex = static_cast<int>(e % d->ex), ey = static_cast<int>((e / d->ex) % d->ey);
      const int ez = z0 + static_cast<int>(e / (static_cast<long>(d->ex) * d->ey));
      for (int k = 0; k < N1; ++k)
        for (int j = 0; j < N1; ++j)
          for (int i = 0; i < N1; ++i) {
            const long gx = static_cast<long>(ex) * N + i, gy = static_cast<long>(ey) * N + j,
                       gz = static_cast<long>(ez) * N + k;
            const bool dir = gx == 0 || gx == static_cast<long>(N) * d->ex || gy == 0 ||
                             gy == static_cast<long>(N) * d->ey || gz == 0 || gz == static_cast<long>(N) * d->ez;
            map[e * NP + (k * N1 + j) * N1 + i] = dir ? -1 : ((gz - 1) * My + (gy - 1)) * Mx + (gx - 1);
          }
    }
  });
}

int cmg_sem_op_create(cmg_ctx* c, const cmg_sem_desc* d, cmg_op** out) {
  return guard([&] { *out = new SemLevel(c, *d); });
}

int cmg_sem_rhs(cmg_op* op, double* b) {
  return guard([&] { as_sem(op)->rhs(b); });
}

int cmg_pmg_create(cmg_ctx* ctx, const cmg_sem_desc* fine, int nlevels, const int* orders,
                   int smoother, size_t eigen_iterations, uint64_t eigen_seed, cmg_pmg** out) {
  return guard([&] {
    if (nlevels < 2 || nlevels > 6) fail(CMG_EINVAL, "pmg: need 2..6 levels");
    if (orders[0] != fine->order) fail(CMG_EINVAL, "pmg: orders[0] must equal the fine order");
    for (int l = 1; l < nlevels; ++l)
      if (orders[l] >= orders[l - 1]) fail(CMG_EINVAL, "pmg: orders must decrease");
    if (orders[nlevels - 1] != 1) fail(CMG_EINVAL, "pmg: the coarsest level must be p=1");
    if (smoother < 0 || smoother > 2) fail(CMG_EINVAL, "pmg: smoother must be 0 (Jacobi), 1 (ASM) or 2 (RAS)");
    auto p = std::make_unique<cmg_pmg>();
    p->ctx = ctx;
    p->nlevels = nlevels;
    p->smoother = smoother;
    cudaStream_t s = ctx->stream;
    for (int l = 0; l < nlevels; ++l) {
      cmg_sem_desc d = *fine;
      d.order = orders[l];
      p->lev.push_back(std::make_unique<SemLevel>(ctx, d));
      SemLevel* L = p->lev.back().get();
      auto iv = std::make_unique<DBuf>(L->len);
      int* zf = ctx->dflag + 11;
      CMG_CUDA(cudaMemsetAsync(zf, 0, sizeof(int), s));
      sem_inverse_diag(L->args(), L->diagv.p, iv->p, zf, s);
      p->invd.push_back(std::move(iv));
      for (auto* v : {&p->vr, &p->vb, &p->vx}) {
        v->push_back(std::make_unique<DBuf>(L->len));
        v->back()->zero(s);
      }
    }
    for (int l = 0; l + 1 < nlevels; ++l) {
      const int Nf = orders[l], Nc = orders[l + 1];
      std::vector<double> Jh((Nf + 1) * (Nc + 1));
      host_interp_matrix(Nf, Nc, Jh.data());
      p->J.push_back(std::make_unique<DBuf>(Jh.size()));
      CMG_CUDA(cudaMemcpy(p->J.back()->p, Jh.data(), Jh.size() * sizeof(double), cudaMemcpyHostToDevice));
      p->Lc.push_back(std::make_unique<DBuf>(static_cast<std::size_t>(p->lev[l]->E) * (Nc + 1) * (Nc + 1) *
                                             (Nc + 1)));
    }
    // coarse separable eigenbases (p=1 on the uniform box: K = tridiag(-1,2,-1)/h, M = h I)
    SemLevel* C = p->lev.back().get();
    auto eig1d = [&](int ne, DBuf& S, std::vector<double>& lam) {
      const int m = ne - 1;
      lam.assign(std::max(m, 1), 0.0);
      S.alloc(std::max(m * m, 1));
      if (m < 1) return;
      const double h = 1.0 / ne;
      std::vector<double> K(m * m, 0.0), M(m * m, 0.0), Sh(m * m);
      for (int i = 0; i < m; ++i) {
        K[i * m + i] = 2.0 / h;
        if (i > 0) K[i * m + i - 1] = -1.0 / h;
        if (i + 1 < m) K[i * m + i + 1] = -1.0 / h;
        M[i * m + i] = h;
      }
      host_sym_geneig(m, K.data(), M.data(), Sh.data(), lam.data());
      CMG_CUDA(cudaMemcpy(S.p, Sh.data(), m * m * sizeof(double), cudaMemcpyHostToDevice));
    };
    std::vector<double> lx, ly, lz;
    eig1d(C->Ex, p->Sx, lx);
    eig1d(C->Ey, p->Sy, ly);
    eig1d(C->Ez, p->Sz, lz);
    p->cnx = C->Ex - 1;
    p->cny = C->Ey - 1;
    p->cnz = C->Ez - 1;
    const long full = static_cast<long>(C->Ex) * C->Ey * C->Ez * sem_nos(1);
    std::vector<double> Dh(full, 1.0);
    for (int k = 0; k < p->cnz; ++k)
      for (int j = 0; j < p->cny; ++j)
        for (int i = 0; i < p->cnx; ++i)
          Dh[sem_nos(1) * (i + static_cast<long>(C->Ex) * (j + static_cast<long>(C->Ey) * k))] = lx[i] + ly[j] + lz[k];
    p->Dg.alloc(full);
    CMG_CUDA(cudaMemcpy(p->Dg.p, Dh.data(), full * sizeof(double), cudaMemcpyHostToDevice));
    p->cfull.alloc(full);
    p->t1.alloc(full);
    p->t2.alloc(full);
    p->cfull.zero(s);
    for (DBuf* b : {&p->cg_r, &p->cg_z, &p->cg_p, &p->cg_Ap}) {
      b->alloc(C->len);
      b->zero(s);
    }
    if (C->desc.geometry != 0) coarse_dense_setup(p.get());
    // lambda_tilde per smoothed level (smoothers.hpp:61-79; S = invD or the Schwarz operator)
    p->lambda.assign(nlevels, 0.0);
    for (int l = 0; l + 1 < nlevels; ++l) {
      if (smoother == 0) {
        p->lambda[l] = estimate_lambda_max(p->lev[l].get(), p->invd[l]->p, eigen_iterations, eigen_seed);
      } else {
        schwarz_setup(p.get(), l);
        p->lambda[l] = estimate_lambda_max_S(p->lev[l].get(), schwarz_apply, p->sch[l].get(), eigen_iterations,
                                             eigen_seed);
      }
      // a non-positive Rayleigh quotient means an indefinite level operator, e.g.
      // a Kershaw map whose kinks (y, z = 1/2) fall inside elements at small eps
      if (!(p->lambda[l] > 0.0))
        fail(CMG_EINVAL, "pmg: level " + std::to_string(l) +
                             " operator is not positive definite (deformed mesh invalid at this resolution?)");
      p->lev[l]->count = 0;
    }
    ctx->sync();
    *out = p.release();
  });
}

int cmg_pmg_destroy(cmg_pmg* p) {
  return guard([&] { delete p; });
}
cmg_op* cmg_pmg_op(cmg_pmg* p, int level) { return p->lev.at(level).get(); }
double cmg_pmg_lambda_tilde(const cmg_pmg* p, int level) { return p->lambda.at(level); }
const double* cmg_pmg_inv_diag(cmg_pmg* p, int level) { return p->invd.at(level)->p; }

int cmg_pmg_prolong(cmg_pmg* p, int level, const double* xc, double* yf) {
  return guard([&] { pmg_prolong(p, level, xc, yf, false); });
}
int cmg_pmg_restrict(cmg_pmg* p, int level, const double* xf, double* yc) {
  return guard([&] { pmg_restrict(p, level, xf, yc); });
}
int cmg_pmg_coarse_solve(cmg_pmg* p, const double* rc, double* ec) {
  return guard([&] { pmg_coarse_solve(p, rc, ec); });
}
int cmg_pmg_schwarz_apply(cmg_pmg* p, int level, const double* r, double* out) {
  return guard([&] {
    if (p->smoother == 0 || level < 0 || level >= static_cast<int>(p->sch.size()) || !p->sch[level])
      fail(CMG_EINVAL, "pmg: no Schwarz smoother on this level");
    schwarz_apply(p->sch[level].get(), r, out);
  });
}
int cmg_pmg_smooth(cmg_pmg* p, int level, const cmg_cheb_config* cfg, size_t order, const double* b,
                   double* x, int x_is_zero) {
  return guard([&] { pmg_smooth(p, level, *cfg, order, b, x, x_is_zero != 0); });
}
int cmg_pmg_v_cycle(cmg_pmg* p, const cmg_cycle_config* cfg, const double* b, double* x, int x_is_zero) {
  return guard([&] { pmg_vcycle(p, 0, *cfg, b, x, x_is_zero != 0); });
}
int cmg_precond_pmg(cmg_pmg* p, const cmg_cycle_config* cfg, cmg_precond** out) {
  return guard([&] {
    auto m = std::make_unique<PmgPrecond>();
    m->ctx = p->ctx;
    m->p = p;
    m->cfg = *cfg;
    *out = m.release();
  });
}

}  // extern "C"
