// gs_nccl.cu -- the engine's own NCCL communicator behind the gs_comm hooks.
//
// The reference has no distributed code; the exchanged quantities are the barycenter's log-sum
// (barycenter.cpp:75-78, allreduce SUM), its marginal error (barycenter.cpp:86, allreduce MAX)
// and, for row partitions, the neighbour rows of T_{k-1} each Chebyshev step reads
// (heat.cpp:124-130 over sparse.cpp:85-99). Those are issued here as NCCL calls on the engine's
// stream, so a captured sweep graph contains them (gs_comm::flags = GS_COMM_GRAPH_SAFE) and no
// Python or host callback runs inside the sweep loop. NCCL is resolved with dlopen at run time:
// the library builds and loads without it, and shares the process's libnccl.so.2 when torch (or
// anyone else) already loaded it.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "gs_internal.cuh"

namespace {

struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.why = "libnccl.so.2 not found";
      return;
    }
    auto sym = [&](const char* name) { return dlsym(h, name); };
    a.GetUniqueId = (decltype(a.GetUniqueId))sym("ncclGetUniqueId");
    a.CommInitRank = (decltype(a.CommInitRank))sym("ncclCommInitRank");
    a.CommDestroy = (decltype(a.CommDestroy))sym("ncclCommDestroy");
    a.AllReduce = (decltype(a.AllReduce))sym("ncclAllReduce");
    a.Send = (decltype(a.Send))sym("ncclSend");
    a.Recv = (decltype(a.Recv))sym("ncclRecv");
    a.GroupStart = (decltype(a.GroupStart))sym("ncclGroupStart");
    a.GroupEnd = (decltype(a.GroupEnd))sym("ncclGroupEnd");
    a.GetErrorString = (decltype(a.GetErrorString))sym("ncclGetErrorString");
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllReduce && a.Send && a.Recv &&
           a.GroupStart && a.GroupEnd;
    if (!a.ok) a.why = "libnccl.so.2 lacks a required symbol";
  });
  return a;
}

struct NcclComm {
  gs_comm hooks;  // first member: a gs_comm* is a NcclComm*
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  int64_t calls = 0;
};

int nccl_allreduce(void* user, double* buf, int64_t count, int op, void* stream) {
  NcclComm* c = static_cast<NcclComm*>(user);
  ++c->calls;
  if (count <= 0) return 0;
  const ncclResult_t r = api().AllReduce(buf, buf, (size_t)count, ncclFloat64, op == 0 ? ncclSum : ncclMax,
                                         c->comm, (cudaStream_t)stream);
  return r == ncclSuccess ? 0 : 1;
}

// one group of point-to-point transfers with the ranks that have bytes to exchange: a
// Cuthill-McKee / bisection row split talks to its neighbours only
int nccl_alltoallv(void* user, const void* sendbuf, const int64_t* send_bytes, void* recvbuf,
                   const int64_t* recv_bytes, int nranks, void* stream) {
  NcclComm* c = static_cast<NcclComm*>(user);
  ++c->calls;
  const NcclApi& A = api();
  cudaStream_t s = (cudaStream_t)stream;
  if (A.GroupStart() != ncclSuccess) return 1;
  int64_t so = 0, ro = 0;
  ncclResult_t r = ncclSuccess;
  for (int q = 0; q < nranks && r == ncclSuccess; ++q) {
    if (send_bytes[q] > 0)
      r = A.Send(static_cast<const char*>(sendbuf) + so, (size_t)send_bytes[q], ncclUint8, q, c->comm, s);
    if (r == ncclSuccess && recv_bytes[q] > 0)
      r = A.Recv(static_cast<char*>(recvbuf) + ro, (size_t)recv_bytes[q], ncclUint8, q, c->comm, s);
    so += send_bytes[q];
    ro += recv_bytes[q];
  }
  const ncclResult_t e = A.GroupEnd();
  return (r == ncclSuccess && e == ncclSuccess) ? 0 : 1;
}

}  // namespace

extern "C" int gs_nccl_unique_id(void* id_out) {
  const NcclApi& A = api();
  if (!A.ok) return GS_ERR_NCCL;
  ncclUniqueId id;
  if (A.GetUniqueId(&id) != ncclSuccess) return GS_ERR_NCCL;
  static_assert(sizeof(ncclUniqueId) == GS_NCCL_UNIQUE_ID_BYTES, "ncclUniqueId size");
  memcpy(id_out, &id, sizeof id);
  return GS_OK;
}

extern "C" int gs_nccl_comm_create(gs_ctx* ctx, const void* id, int nranks, int rank, gs_comm** out) {
  *out = nullptr;
  const NcclApi& A = api();
  if (!A.ok) {
    ctx->err = "NcclError: " + A.why;
    return GS_ERR_NCCL;
  }
  if (nranks < 1 || rank < 0 || rank >= nranks) return gs_fail(ctx, ERRC_INVALID_ARGUMENT, "nccl rank / size");
  GS_CUDA(ctx, cudaSetDevice(ctx->device));
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof uid);
  NcclComm* c = new NcclComm();
  const ncclResult_t r = A.CommInitRank(&c->comm, nranks, uid, rank);
  if (r != ncclSuccess) {
    ctx->err = std::string("NcclError: ncclCommInitRank: ") + (A.GetErrorString ? A.GetErrorString(r) : "");
    delete c;
    return GS_ERR_NCCL;
  }
  c->nranks = nranks;
  c->rank = rank;
  c->hooks.allreduce = nccl_allreduce;
  c->hooks.alltoallv = nccl_alltoallv;
  c->hooks.user = c;
  c->hooks.flags = GS_COMM_GRAPH_SAFE;
  *out = &c->hooks;
  return GS_OK;
}

extern "C" void gs_nccl_comm_destroy(gs_comm* comm) {
  if (!comm) return;
  NcclComm* c = reinterpret_cast<NcclComm*>(comm);
  if (c->comm && api().ok) api().CommDestroy(c->comm);
  delete c;
}

extern "C" int64_t gs_nccl_comm_calls(const gs_comm* comm) {
  return comm ? reinterpret_cast<const NcclComm*>(comm)->calls : 0;
}
