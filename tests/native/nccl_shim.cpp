// A stand-in libnccl.so.2 for running the library's PRODUCTION NCCL transport
// (paper_1211_2517_b200/csrc/nccl_transport.cpp) with several ranks as separate processes
// on ONE GPU (test infrastructure; selected with KIFMM_NCCL_LIB=<path of this .so>).
//
// It implements the nine entry points the transport resolves: ncclGetUniqueId,
// ncclCommInitRank, ncclCommDestroy, ncclGroupStart, ncclGroupEnd, ncclSend, ncclRecv,
// ncclAllReduce (double, sum), ncclGetErrorString.  Data moves device to device through
// CUDA IPC (cuIpcGetMemHandle / cuIpcOpenMemHandle on the base allocation of each send
// buffer); ranks rendezvous on a POSIX shared-memory segment named by the unique id with a
// host barrier.  Every collective first synchronises the caller's stream on the host, so
// no GPU kernel ever waits on another process (kernels that spin on each other across
// processes on one GPU are not safe on this driver; B200_PROFILING.md) — the ranks'
// kernels simply time-slice.  The allreduce sums in rank order on the host: every rank
// gets the bitwise-same result, as NCCL's ring would.
#include <cuda.h>
#include <fcntl.h>
#include <nccl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <thread>
#include <vector>

namespace {

constexpr int kMaxRanks = 16;

struct SendDesc {
  CUipcMemHandle h;
  uint64_t off;    // bytes from the allocation base
  uint64_t bytes;  // 0: nothing for this peer
};

struct RankSlot {
  SendDesc to[kMaxRanks];  // this rank's send to each peer (group op) / its buffer (allreduce: to[0])
};

struct Shared {
  std::atomic<uint32_t> magic;
  std::atomic<int> arrived;
  std::atomic<int> generation;
  int nranks;
  RankSlot slot[kMaxRanks];
};

struct Comm {
  std::string name;
  int nranks = 0, rank = 0;
  Shared* sh = nullptr;
  std::map<std::string, CUdeviceptr> opened;  // IPC handle bytes -> mapped base
};

struct Pending {
  bool send;
  void* ptr;
  size_t count;
  ncclDataType_t type;
  int peer;
  Comm* comm;
  CUstream stream;
};

thread_local int g_group = 0;
thread_local std::vector<Pending> g_pending;

size_t type_size(ncclDataType_t t) {
  switch (t) {
    case ncclFloat64: case ncclInt64: case ncclUint64: return 8;
    case ncclFloat32: case ncclInt32: case ncclUint32: return 4;
    case ncclFloat16: return 2;
    default: return 1;
  }
}

void barrier(Comm* c) {
  Shared* s = c->sh;
  const int gen = s->generation.load();
  if (s->arrived.fetch_add(1) + 1 == c->nranks) {
    s->arrived.store(0);
    s->generation.fetch_add(1);
  } else {
    while (s->generation.load() == gen) std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}

ncclResult_t describe(const void* ptr, size_t bytes, SendDesc* d) {
  std::memset(d, 0, sizeof(*d));
  d->bytes = bytes;
  if (!bytes) return ncclSuccess;
  CUdeviceptr base = 0;
  size_t size = 0;
  if (cuMemGetAddressRange(&base, &size, (CUdeviceptr)ptr) != CUDA_SUCCESS) return ncclInvalidArgument;
  if (cuIpcGetMemHandle(&d->h, base) != CUDA_SUCCESS) return ncclUnhandledCudaError;
  d->off = (CUdeviceptr)ptr - base;
  return ncclSuccess;
}

ncclResult_t open_peer(Comm* c, const SendDesc& d, CUdeviceptr* out) {
  std::string key(reinterpret_cast<const char*>(&d.h), sizeof(d.h));
  auto it = c->opened.find(key);
  if (it == c->opened.end()) {
    CUdeviceptr p = 0;
    if (cuIpcOpenMemHandle(&p, d.h, CU_IPC_MEM_LAZY_ENABLE_PEER_ACCESS) != CUDA_SUCCESS) return ncclUnhandledCudaError;
    it = c->opened.emplace(key, p).first;
  }
  *out = it->second + d.off;
  return ncclSuccess;
}

// the grouped send / recv of one comm: publish sends, barrier, pull receives, barrier
ncclResult_t run_group(Comm* c, const std::vector<Pending>& ops) {
  RankSlot& me = c->sh->slot[c->rank];
  std::memset(&me, 0, sizeof(me));
  for (const Pending& p : ops) {
    // (stream 0 is the legacy default stream: synchronised like any other)
    if (cuStreamSynchronize(p.stream) != CUDA_SUCCESS) return ncclUnhandledCudaError;
    if (p.send && describe(p.ptr, p.count * type_size(p.type), &me.to[p.peer]) != ncclSuccess)
      return ncclUnhandledCudaError;
  }
  barrier(c);
  ncclResult_t rc = ncclSuccess;
  for (const Pending& p : ops) {
    if (p.send) continue;
    const SendDesc& d = c->sh->slot[p.peer].to[c->rank];
    const size_t bytes = p.count * type_size(p.type);
    if (d.bytes != bytes) { rc = ncclInvalidUsage; continue; }  // mismatched send / recv sizes
    CUdeviceptr src = 0;
    // on the receiver's stream, then waited for: a device-to-device cuMemcpy returns before
    // the copy completes, and the sender may reuse its buffer after the next barrier
    if (bytes && (open_peer(c, d, &src) != ncclSuccess ||
                  cuMemcpyDtoDAsync((CUdeviceptr)p.ptr, src, bytes, p.stream) != CUDA_SUCCESS ||
                  cuStreamSynchronize(p.stream) != CUDA_SUCCESS))
      rc = ncclUnhandledCudaError;
  }
  barrier(c);  // the senders' buffers are free again
  return rc;
}

}  // namespace

extern "C" {

const char* ncclGetErrorString(ncclResult_t r) {
  switch (r) {
    case ncclSuccess: return "no error";
    case ncclUnhandledCudaError: return "unhandled cuda error (shim)";
    case ncclSystemError: return "system error (shim)";
    case ncclInvalidArgument: return "invalid argument (shim)";
    case ncclInvalidUsage: return "invalid usage (shim)";
    default: return "error (shim)";
  }
}

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
  static std::atomic<int> counter{0};
  std::memset(id, 0, sizeof(*id));
  const auto t = std::chrono::steady_clock::now().time_since_epoch().count();
  std::snprintf(id->internal, sizeof(id->internal), "/kifmm_shim_%d_%d_%lld", (int)getpid(), counter++,
                (long long)(t % 1000000007LL));
  return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* comm, int nranks, ncclUniqueId id, int rank) {
  if (nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks) return ncclInvalidArgument;
  Comm* c = new Comm;
  c->name.assign(id.internal, strnlen(id.internal, sizeof(id.internal)));
  c->nranks = nranks;
  c->rank = rank;
  int fd = -1;
  if (rank == 0) {
    fd = shm_open(c->name.c_str(), O_CREAT | O_RDWR, 0600);
    if (fd < 0 || ftruncate(fd, sizeof(Shared)) != 0) { delete c; return ncclSystemError; }
  } else {
    for (int tries = 0; tries < 60000 && fd < 0; ++tries) {  // rank 0 creates the segment
      fd = shm_open(c->name.c_str(), O_RDWR, 0600);
      if (fd < 0) std::this_thread::sleep_for(std::chrono::milliseconds(1));
    }
    if (fd < 0) { delete c; return ncclSystemError; }
  }
  void* m = mmap(nullptr, sizeof(Shared), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (m == MAP_FAILED) { delete c; return ncclSystemError; }
  c->sh = static_cast<Shared*>(m);
  if (rank == 0) {
    c->sh->arrived.store(0);
    c->sh->generation.store(0);
    c->sh->nranks = nranks;
    c->sh->magic.store(0x5348494du);
  } else {
    while (c->sh->magic.load() != 0x5348494du) std::this_thread::sleep_for(std::chrono::microseconds(100));
  }
  barrier(c);
  *comm = reinterpret_cast<ncclComm_t>(c);
  return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t comm) {
  Comm* c = reinterpret_cast<Comm*>(comm);
  if (!c) return ncclSuccess;
  barrier(c);
  for (auto& kv : c->opened) cuIpcCloseMemHandle(kv.second);
  const bool last = c->rank == 0;
  munmap(c->sh, sizeof(Shared));
  if (last) shm_unlink(c->name.c_str());
  delete c;
  return ncclSuccess;
}

ncclResult_t ncclGroupStart() {
  ++g_group;
  return ncclSuccess;
}

ncclResult_t ncclGroupEnd() {
  if (g_group <= 0) return ncclInvalidUsage;
  if (--g_group > 0) return ncclSuccess;
  std::vector<Pending> ops;
  ops.swap(g_pending);
  if (ops.empty()) return ncclSuccess;
  // one group per comm here (the transport never mixes comms in a group)
  return run_group(ops[0].comm, ops);
}

ncclResult_t ncclSend(const void* buf, size_t count, ncclDataType_t type, int peer, ncclComm_t comm,
                      cudaStream_t stream) {
  if (g_group <= 0) return ncclInvalidUsage;  // the transport always groups point-to-point calls
  g_pending.push_back(Pending{true, const_cast<void*>(buf), count, type, peer, reinterpret_cast<Comm*>(comm),
                              reinterpret_cast<CUstream>(stream)});
  return ncclSuccess;
}

ncclResult_t ncclRecv(void* buf, size_t count, ncclDataType_t type, int peer, ncclComm_t comm, cudaStream_t stream) {
  if (g_group <= 0) return ncclInvalidUsage;
  g_pending.push_back(
      Pending{false, buf, count, type, peer, reinterpret_cast<Comm*>(comm), reinterpret_cast<CUstream>(stream)});
  return ncclSuccess;
}

ncclResult_t ncclAllReduce(const void* sendbuff, void* recvbuff, size_t count, ncclDataType_t type, ncclRedOp_t op,
                           ncclComm_t comm, cudaStream_t stream) {
  if (type != ncclFloat64 || op != ncclSum) return ncclInvalidArgument;
  Comm* c = reinterpret_cast<Comm*>(comm);
  if (cuStreamSynchronize(reinterpret_cast<CUstream>(stream)) != CUDA_SUCCESS) return ncclUnhandledCudaError;
  const size_t bytes = count * 8;
  RankSlot& me = c->sh->slot[c->rank];
  std::memset(&me, 0, sizeof(me));
  if (describe(sendbuff, bytes, &me.to[0]) != ncclSuccess) return ncclUnhandledCudaError;
  barrier(c);
  std::vector<double> sum(count, 0.0), part(count);
  ncclResult_t rc = ncclSuccess;
  for (int r = 0; r < c->nranks && bytes; ++r) {  // rank order: the same sum on every rank
    CUdeviceptr src = (CUdeviceptr)sendbuff;
    if (r != c->rank && open_peer(c, c->sh->slot[r].to[0], &src) != ncclSuccess) { rc = ncclUnhandledCudaError; break; }
    if (cuMemcpyDtoH(part.data(), src, bytes) != CUDA_SUCCESS) { rc = ncclUnhandledCudaError; break; }
    for (size_t i = 0; i < count; ++i) sum[i] += part[i];
  }
  barrier(c);  // every rank has read every buffer before any is overwritten
  // on the caller's stream and waited for (a pageable host-to-device cuMemcpy may return
  // before the DMA lands)
  const CUstream s = reinterpret_cast<CUstream>(stream);
  if (rc == ncclSuccess && bytes &&
      (cuMemcpyHtoDAsync((CUdeviceptr)recvbuff, sum.data(), bytes, s) != CUDA_SUCCESS ||
       cuStreamSynchronize(s) != CUDA_SUCCESS))
    rc = ncclUnhandledCudaError;
  return rc;
}

}  // extern "C"
