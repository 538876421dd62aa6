// NCCL transport of the partitioned matvec: grouped point-to-point
// ghost exchanges (ncclSend / ncclRecv, an all-to-allv over NVLink / NVSwitch), an
// in-place allreduce of the straddling boxes' partial multipoles, and an allgather
// of the owned potential ranges (replicated output mode).  Everything is enqueued
// on the matvec stream: no host synchronisation inside a matvec.
//
// libnccl.so.2 is resolved at run time (dlopen).  In a process that already has
// PyTorch's NCCL mapped, RTLD_NOLOAD returns that same library, so one NCCL
// instance serves both torch.distributed and this library.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "fmm_internal.h"

namespace kifmm {

namespace {

struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& api() {
  static NcclApi A;
  static std::once_flag once;
  std::call_once(once, [] {
    // KIFMM_NCCL_LIB: an explicit library path (test seam: tests/native/nccl_shim.cpp runs
    // this transport with several processes on one GPU)
    void* h = nullptr;
    if (const char* p = std::getenv("KIFMM_NCCL_LIB")) {
      h = dlopen(p, RTLD_NOW | RTLD_LOCAL);
      if (!h) { A.err = std::string("dlopen(") + p + ") failed: " + dlerror(); return; }
    }
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) { A.err = std::string("dlopen(libnccl.so.2) failed: ") + dlerror(); return; }
    auto sym = [&](const char* name) -> void* { return dlsym(h, name); };
    A.GetUniqueId = (decltype(A.GetUniqueId))sym("ncclGetUniqueId");
    A.CommInitRank = (decltype(A.CommInitRank))sym("ncclCommInitRank");
    A.CommDestroy = (decltype(A.CommDestroy))sym("ncclCommDestroy");
    A.Send = (decltype(A.Send))sym("ncclSend");
    A.Recv = (decltype(A.Recv))sym("ncclRecv");
    A.AllReduce = (decltype(A.AllReduce))sym("ncclAllReduce");
    A.GroupStart = (decltype(A.GroupStart))sym("ncclGroupStart");
    A.GroupEnd = (decltype(A.GroupEnd))sym("ncclGroupEnd");
    A.GetErrorString = (decltype(A.GetErrorString))sym("ncclGetErrorString");
    A.ok = A.GetUniqueId && A.CommInitRank && A.CommDestroy && A.Send && A.Recv && A.AllReduce && A.GroupStart &&
           A.GroupEnd && A.GetErrorString;
    if (!A.ok) A.err = "libnccl.so.2 lacks a required symbol";
  });
  return A;
}

int check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return 0;
  set_error(std::string(what) + ": " + api().GetErrorString(r));
  return -5;
}

#define KIFMM_NCCL(call)                         \
  do {                                           \
    if (int rc_ = check((call), #call)) return rc_; \
  } while (0)

// inside ncclGroupStart / ncclGroupEnd: an error closes the group before returning, so
// the thread is not left with an open NCCL group (the first error's message is kept)
#define KIFMM_NCCL_IN_GROUP(call)                \
  do {                                           \
    if (int rc_ = check((call), #call)) {        \
      const std::string msg_ = last_error();     \
      api().GroupEnd();                          \
      set_error(msg_);                           \
      return rc_;                                \
    }                                            \
  } while (0)

int need_comm(Plan& P) {
  if (!P.nccl_comm) {
    set_error("plan has nranks > 1 but no NCCL communicator (loopback plans run through fmm_matvec_group)");
    return -5;
  }
  return 0;
}

}  // namespace

int nccl_unique_id(void* id128) {
  NcclApi& A = api();
  if (!A.ok) { set_error(A.err); return -5; }
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  KIFMM_NCCL(A.GetUniqueId(&id));
  std::memcpy(id128, &id, sizeof(id));
  return 0;
}

int nccl_comm_init(Plan& P, const void* id128) {
  NcclApi& A = api();
  if (!A.ok) { set_error(A.err); return -5; }
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  ncclComm_t c = nullptr;
  KIFMM_NCCL(A.CommInitRank(&c, P.dist.nranks, id, P.dist.rank));
  P.nccl_comm = c;
  return 0;
}

void nccl_comm_destroy(Plan& P) {
  if (P.nccl_comm && api().ok) api().CommDestroy((ncclComm_t)P.nccl_comm);
  P.nccl_comm = nullptr;
}

// all-to-allv of ghost rows: to peer s the rows [send_off[s], send_off[s+1]) of the
// send buffer, from peer s into [recv_off[s], recv_off[s+1]) of the receive buffer
int nccl_exchange(Plan& P, Exchange& X, cudaStream_t st) {
  if (int rc = need_comm(P)) return rc;
  NcclApi& A = api();
  ncclComm_t c = (ncclComm_t)P.nccl_comm;
  const int R = P.dist.nranks;
  KIFMM_NCCL(A.GroupStart());
  for (int s = 0; s < R; ++s) {
    if (s == P.dist.rank) continue;
    const size_t ns = (size_t)(X.send_off[s + 1] - X.send_off[s]) * X.row;
    const size_t nr = (size_t)(X.recv_off[s + 1] - X.recv_off[s]) * X.row;
    if (ns) KIFMM_NCCL_IN_GROUP(A.Send(X.d_send + (size_t)X.send_off[s] * X.row, ns, ncclFloat64, s, c, st));
    if (nr) KIFMM_NCCL_IN_GROUP(A.Recv(X.d_recv + (size_t)X.recv_off[s] * X.row, nr, ncclFloat64, s, c, st));
  }
  KIFMM_NCCL(A.GroupEnd());
  return 0;
}

int nccl_allreduce_sum(Plan& P, double* buf, size_t count, cudaStream_t st) {
  if (count == 0) return 0;  // identical on every rank (the straddling set is global)
  if (int rc = need_comm(P)) return rc;
  KIFMM_NCCL(api().AllReduce(buf, buf, count, ncclFloat64, ncclSum, (ncclComm_t)P.nccl_comm, st));
  return 0;
}

// every rank's owned sorted range [bnd[r], bnd[r+1]) of buf to every other rank
int nccl_allgather_ranges(Plan& P, double* buf, cudaStream_t st) {
  if (int rc = need_comm(P)) return rc;
  NcclApi& A = api();
  ncclComm_t c = (ncclComm_t)P.nccl_comm;
  const DistPlan& D = P.dist;
  const size_t mine = (size_t)(D.own_hi - D.own_lo);
  KIFMM_NCCL(A.GroupStart());
  for (int s = 0; s < D.nranks; ++s) {
    if (s == D.rank) continue;
    const size_t theirs = (size_t)(D.bnd[s + 1] - D.bnd[s]);
    if (mine) KIFMM_NCCL_IN_GROUP(A.Send(buf + D.own_lo, mine, ncclFloat64, s, c, st));
    if (theirs) KIFMM_NCCL_IN_GROUP(A.Recv(buf + D.bnd[s], theirs, ncclFloat64, s, c, st));
  }
  KIFMM_NCCL(A.GroupEnd());
  return 0;
}

}  // namespace kifmm
