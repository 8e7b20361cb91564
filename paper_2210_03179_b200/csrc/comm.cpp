// comm.cpp -- NCCL plumbing for the element-partitioned SEM path.
//
// One process per GPU; the communicator is created from a unique id that the
// caller broadcasts (torch.distributed in the Python host layer).  NCCL is
// bound at run time with dlopen: if the hosting process already loaded a
// libnccl.so.2 (e.g. torch's), that instance is reused, otherwise the system
// library is loaded.  Only the types/enums of nccl.h are used at compile time.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "cmg_objects.hpp"

namespace {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

NcclApi& nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("/usr/lib/x86_64-linux-gnu/libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) return;
#define SYM(name) api.name = reinterpret_cast<decltype(api.name)>(dlsym(h, "nccl" #name))
    SYM(GetUniqueId); SYM(CommInitRank); SYM(CommDestroy); SYM(AllReduce); SYM(AllGather);
    SYM(Send); SYM(Recv); SYM(GroupStart); SYM(GroupEnd); SYM(GetErrorString);
#undef SYM
    api.ok = api.GetUniqueId && api.CommInitRank && api.AllReduce && api.AllGather && api.Send &&
             api.Recv && api.GroupStart && api.GroupEnd;
  });
  if (!api.ok) throw cmg::Error(cmg::ENCCL_, "NCCL (libnccl.so.2) could not be loaded");
  return api;
}

}  // namespace

#define CMG_NCCL(x)                                                                            \
  do {                                                                                         \
    ncclResult_t r_ = (x);                                                                     \
    if (r_ != ncclSuccess)                                                                     \
      throw ::cmg::Error(::cmg::ENCCL_,                                                        \
                         std::string(#x) + ": " +                                              \
                             (nccl_api().GetErrorString ? nccl_api().GetErrorString(r_) : "nccl error")); \
  } while (0)

namespace cmg {

Comm::~Comm() {
  if (nccl) nccl_api().CommDestroy(static_cast<ncclComm_t>(nccl));
  for (cudaEvent_t e : {ev_ready, ev_halo, ev_contrib})
    if (e) cudaEventDestroy(e);
  if (side) cudaStreamDestroy(side);
}

void Comm::allreduce_sum(double* buf, std::size_t count, cudaStream_t s) {
  if (nranks == 1) return;
  CMG_NCCL(nccl_api().AllReduce(buf, buf, count, ncclDouble, ncclSum, static_cast<ncclComm_t>(nccl), s));
}

void Comm::allgather(const double* send, double* recv, std::size_t count, cudaStream_t s) {
  if (nranks == 1) {
    if (send != recv)
      CMG_CUDA(cudaMemcpyAsync(recv, send, count * sizeof(double), cudaMemcpyDeviceToDevice, s));
    return;
  }
  CMG_NCCL(nccl_api().AllGather(send, recv, count, ncclDouble, static_cast<ncclComm_t>(nccl), s));
}

void Comm::sendrecv(const double* send_up, std::size_t n_up, double* recv_down,
                    std::size_t n_down, int up, int down, cudaStream_t s) {
  auto c = static_cast<ncclComm_t>(nccl);
  auto& api = nccl_api();
  CMG_NCCL(api.GroupStart());
  if (up >= 0 && n_up) CMG_NCCL(api.Send(send_up, n_up, ncclDouble, up, c, s));
  if (down >= 0 && n_down) CMG_NCCL(api.Recv(recv_down, n_down, ncclDouble, down, c, s));
  CMG_NCCL(api.GroupEnd());
}

void Comm::exchange(const double* send_a, std::size_t na, int peer_a, double* recv_a,
                    const double* send_b, std::size_t nb, int peer_b, double* recv_b,
                    cudaStream_t s) {
  auto c = static_cast<ncclComm_t>(nccl);
  auto& api = nccl_api();
  CMG_NCCL(api.GroupStart());
  if (peer_a >= 0 && na) {
    CMG_NCCL(api.Send(send_a, na, ncclDouble, peer_a, c, s));
    CMG_NCCL(api.Recv(recv_a, na, ncclDouble, peer_a, c, s));
  }
  if (peer_b >= 0 && nb) {
    CMG_NCCL(api.Send(send_b, nb, ncclDouble, peer_b, c, s));
    CMG_NCCL(api.Recv(recv_b, nb, ncclDouble, peer_b, c, s));
  }
  CMG_NCCL(api.GroupEnd());
}

void Comm::shift(const double* send_up, double* recv_lo, std::size_t n_up, const double* send_dn,
                 double* recv_hi, std::size_t n_dn, int up, int down, cudaStream_t s) {
  auto c = static_cast<ncclComm_t>(nccl);
  auto& api = nccl_api();
  CMG_NCCL(api.GroupStart());
  if (up >= 0) {
    CMG_NCCL(api.Send(send_up, n_up, ncclDouble, up, c, s));
    CMG_NCCL(api.Recv(recv_hi, n_dn, ncclDouble, up, c, s));
  }
  if (down >= 0) {
    CMG_NCCL(api.Send(send_dn, n_dn, ncclDouble, down, c, s));
    CMG_NCCL(api.Recv(recv_lo, n_up, ncclDouble, down, c, s));
  }
  CMG_NCCL(api.GroupEnd());
}

}  // namespace cmg

extern "C" {

int cmg_nccl_unique_id(unsigned char out[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  try {
    ncclUniqueId id;
    CMG_NCCL(nccl_api().GetUniqueId(&id));
    std::memcpy(out, &id, 128);
    return CMG_OK;
  } catch (const cmg::Error& e) {
    cmg::set_last_error(e.what());
    return e.code;
  }
}

int cmg_ctx_attach_nccl(cmg_ctx* ctx, const unsigned char id_bytes[128], int rank, int nranks) {
  try {
    CMG_CUDA(cudaSetDevice(ctx->device));
    auto comm = std::make_unique<cmg::Comm>();
    comm->rank = rank;
    comm->nranks = nranks;
    if (nranks > 1) {
      ncclUniqueId id;
      std::memcpy(&id, id_bytes, 128);
      ncclComm_t c;
      CMG_NCCL(nccl_api().CommInitRank(&c, nranks, id, rank));
      comm->nccl = c;
      CMG_CUDA(cudaStreamCreateWithFlags(&comm->side, cudaStreamNonBlocking));
      for (cudaEvent_t* e : {&comm->ev_ready, &comm->ev_halo, &comm->ev_contrib})
        CMG_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    }
    ctx->rank = rank;
    ctx->nranks = nranks;
    ctx->comm = std::move(comm);
    return CMG_OK;
  } catch (const cmg::Error& e) {
    cmg::set_last_error(e.what());
    return e.code;
  }
}

}  // extern "C"
