// comm.cpp -- NCCL over NVLink/NVSwitch for the multi-GPU dual PCG.
//
// NCCL is loaded at run time (dlopen) only when a context is set up with world > 1, so the
// single-GPU library has no NCCL dependency.  The caller (bench.py / torchrun) creates the
// 128-byte unique id on rank 0 with ieti_nccl_unique_id() and broadcasts it through
// torch.distributed; every rank then calls ieti_setup() with it (collective).
// All collectives are issued on the library stream and are captured into the PCG graphs.
#include "internal.h"

#include <dlfcn.h>

#include <cstring>
#include <stdexcept>
#include <string>

#include "nccl.h"

#ifndef IETI_NCCL_PATH
#define IETI_NCCL_PATH "libnccl.so.2"
#endif

namespace {
struct NcclApi {
  void *h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
  std::string err;

  bool load() {
    if (h) return true;
    h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen(IETI_NCCL_PATH, RTLD_NOW | RTLD_GLOBAL);
    if (!h) { err = std::string("cannot load NCCL: ") + dlerror(); return false; }
#define SYM(name)                                                              \
  *(void **)(&name) = dlsym(h, "nccl" #name);                                  \
  if (!name) { err = "NCCL symbol missing: nccl" #name; return false; }
    SYM(GetUniqueId) SYM(CommInitRank) SYM(CommDestroy) SYM(AllGather) SYM(AllReduce) SYM(Send) SYM(Recv)
    SYM(GroupStart) SYM(GroupEnd) SYM(GetErrorString)
#undef SYM
    return true;
  }
};
NcclApi &api() {
  static NcclApi a;
  return a;
}
}  // namespace

static void nck(ncclResult_t r, const char *what) {
  if (r != ncclSuccess)
    throw CommError(std::string("NCCL ") + what + ": " + (api().GetErrorString ? api().GetErrorString(r) : "?"));
}

int comm_unique_id(void *out128, std::string &err) {
  if (!api().load()) { err = api().err; return -1; }
  ncclUniqueId id;
  if (api().GetUniqueId(&id) != ncclSuccess) { err = "ncclGetUniqueId failed"; return -1; }
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  memcpy(out128, &id, 128);
  return 0;
}

void Comm::init(const void *uid128, int rank_, int world_, bool force) {
  rank = rank_;
  world = world_;
  if (world <= 1 && !force) return;
  if (!uid128) throw CommError("world > 1 needs nccl_unique_id");
  if (!api().load()) throw CommError(api().err);
  ncclUniqueId id;
  memcpy(&id, uid128, 128);
  ncclComm_t c = nullptr;
  nck(api().CommInitRank(&c, world, id, rank), "CommInitRank");
  comm = c;
}

void Comm::destroy() {
  if (comm) api().CommDestroy((ncclComm_t)comm);
  comm = nullptr;
}

void Comm::allgather(const double *send, double *recv, size_t count, cudaStream_t s) {
  nck(api().AllGather(send, recv, count, ncclDouble, (ncclComm_t)comm, s), "AllGather");
}

void Comm::allreduce_sum(double *buf, size_t count, cudaStream_t s) {
  nck(api().AllReduce(buf, buf, count, ncclDouble, ncclSum, (ncclComm_t)comm, s), "AllReduce");
}

void Comm::exchange(const std::vector<int> &peers, const double *send, const std::vector<int> &send_ptr,
                    double *recv, const std::vector<int> &recv_ptr, cudaStream_t s) {
  nck(api().GroupStart(), "GroupStart");
  for (size_t i = 0; i < peers.size(); ++i) {
    const int ns = send_ptr[i + 1] - send_ptr[i], nr = recv_ptr[i + 1] - recv_ptr[i];
    if (ns) nck(api().Send(send + send_ptr[i], ns, ncclDouble, peers[i], (ncclComm_t)comm, s), "Send");
    if (nr) nck(api().Recv(recv + recv_ptr[i], nr, ncclDouble, peers[i], (ncclComm_t)comm, s), "Recv");
  }
  nck(api().GroupEnd(), "GroupEnd");
}
