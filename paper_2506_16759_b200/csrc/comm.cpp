// In-library NCCL communicator (SURVEY §8(b) h2_comm_*, §8(e) per-level all-gathers over NVLink).
// libnccl.so.2 is loaded at run time (dlopen): in a process that already imported torch this is
// torch's NCCL; libh2 has no link-time NCCL dependency and builds without a GPU.  The per-level
// exchange of Algorithm 1 under sharding (§IV-B: ranks, skeleton indices I~,
// the next level's Omega rows) is an in-place all-gather of variable byte segments, issued as one
// NCCL group of P broadcasts (segment r rooted at rank r), stream-ordered on the build stream:
// no host staging, no host synchronisation.
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <string>

#include "comm.hpp"
#include "common.cuh"

namespace h2 {
namespace {

struct Nccl {
  void* so = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
  std::string why;
};

Nccl& nccl() {
  static Nccl N;
  static std::once_flag once;
  std::call_once(once, [] {
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      N.so = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (N.so) break;
    }
    if (!N.so) {
      N.why = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [](const char* s) { return dlsym(N.so, s); };
    N.getUniqueId = reinterpret_cast<decltype(N.getUniqueId)>(sym("ncclGetUniqueId"));
    N.commInitRank = reinterpret_cast<decltype(N.commInitRank)>(sym("ncclCommInitRank"));
    N.commDestroy = reinterpret_cast<decltype(N.commDestroy)>(sym("ncclCommDestroy"));
    N.broadcast = reinterpret_cast<decltype(N.broadcast)>(sym("ncclBroadcast"));
    N.send = reinterpret_cast<decltype(N.send)>(sym("ncclSend"));
    N.recv = reinterpret_cast<decltype(N.recv)>(sym("ncclRecv"));
    N.groupStart = reinterpret_cast<decltype(N.groupStart)>(sym("ncclGroupStart"));
    N.groupEnd = reinterpret_cast<decltype(N.groupEnd)>(sym("ncclGroupEnd"));
    N.errorString = reinterpret_cast<decltype(N.errorString)>(sym("ncclGetErrorString"));
    if (!N.getUniqueId || !N.commInitRank || !N.commDestroy || !N.broadcast || !N.send || !N.recv || !N.groupStart || !N.groupEnd)
      N.why = "libnccl.so.2 lacks a required symbol";
  });
  if (!N.why.empty()) throw Error(H2_ERR_NCCL, N.why);
  return N;
}

void check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    const char* s = nccl().errorString ? nccl().errorString(r) : "?";
    throw Error(H2_ERR_NCCL, std::string(what) + ": " + s);
  }
}

}  // namespace

void nccl_unique_id(void* id128) {
  static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id is 128 bytes");
  ncclUniqueId id;
  check(nccl().getUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(id128, &id, sizeof id);
}

void* nccl_comm_init(const void* id128, int rank, int nranks) {
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof id);
  ncclComm_t c = nullptr;
  check(nccl().commInitRank(&c, nranks, id, rank), "ncclCommInitRank");
  return c;
}

void nccl_comm_free(void* c) {
  if (c) nccl().commDestroy(static_cast<ncclComm_t>(c));
}

void nccl_allgatherv(void* c, int nranks, void* buf, const int64_t* counts, const int64_t* displs, cudaStream_t st) {
  Nccl& N = nccl();
  char* b = static_cast<char*>(buf);
  check(N.groupStart(), "ncclGroupStart");
  for (int r = 0; r < nranks; ++r)
    if (counts[r] > 0)
      check(N.broadcast(b + displs[r], b + displs[r], (size_t)counts[r], ncclInt8, r, static_cast<ncclComm_t>(c), st),
            "ncclBroadcast");
  check(N.groupEnd(), "ncclGroupEnd");
}

// all-to-all of byte segments (the column-split sketch exchange, S§8(e)): one NCCL group of
// point-to-point sends / receives to and from every other rank; the own segment is a device copy
void nccl_alltoallv(void* c, int rank, int nranks, const void* send, const int64_t* scounts, const int64_t* sdispls,
                    void* recv, const int64_t* rcounts, const int64_t* rdispls, cudaStream_t st) {
  Nccl& N = nccl();
  const char* sb = static_cast<const char*>(send);
  char* rb = static_cast<char*>(recv);
  if (scounts[rank] > 0)
    H2_CUDA(cudaMemcpyAsync(rb + rdispls[rank], sb + sdispls[rank], (size_t)scounts[rank], cudaMemcpyDeviceToDevice, st));
  check(N.groupStart(), "ncclGroupStart");
  for (int r = 0; r < nranks; ++r) {
    if (r == rank) continue;
    if (scounts[r] > 0)
      check(N.send(sb + sdispls[r], (size_t)scounts[r], ncclInt8, r, static_cast<ncclComm_t>(c), st), "ncclSend");
    if (rcounts[r] > 0)
      check(N.recv(rb + rdispls[r], (size_t)rcounts[r], ncclInt8, r, static_cast<ncclComm_t>(c), st), "ncclRecv");
  }
  check(N.groupEnd(), "ncclGroupEnd");
}

}  // namespace h2
