// comm.cpp -- NCCL over NVLink/NVSwitch for the multi-GPU dual PCG.
//
// NCCL is loaded at run time (dlopen) only when a context is set up with world > 1, so the
// single-GPU library has no NCCL dependency.  The caller (bench.py / torchrun) creates the
// 128-byte unique id on rank 0 with ieti_nccl_unique_id() and broadcasts it through
// torch.distributed; every rank then calls ieti_setup() with it (collective).
// All collectives are issued on the library stream and are captured into the PCG graphs.
#include "internal.h"

#include <dlfcn.h>

#include <cstdint>
#include <cstdlib>

#include <condition_variable>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

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

// ---- in-process loopback group (IETI_LOOPBACK=1, tests only) ------------------------------
// Several ranks of one process (one host thread each, all on one GPU) exchange through device
// copies, ordered by a host barrier: no kernel ever waits for another rank.  Eager calls only
// (the PCG graphs are not captured in this mode).
struct LoopGroup {
  int world = 0, arrived = 0;
  unsigned long long gen = 0;
  std::mutex m;
  std::condition_variable cv;
  std::vector<const double *> send;
  std::vector<const std::vector<int> *> peers, ptr;
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const unsigned long long g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};
static std::map<std::string, std::shared_ptr<LoopGroup>> &loop_registry() {
  static std::map<std::string, std::shared_ptr<LoopGroup>> r;
  return r;
}
static std::mutex loop_registry_m;

static void cck(cudaError_t e, const char *what) {
  if (e != cudaSuccess) throw CommError(std::string("loopback ") + what + ": " + cudaGetErrorString(e));
}

static void nck(ncclResult_t r, const char *what) {
  if (r != ncclSuccess)
    throw CommError(std::string("NCCL ") + what + ": " + (api().GetErrorString ? api().GetErrorString(r) : "?"));
}

int comm_unique_id(void *out128, std::string &err) {
  const char *lb = getenv("IETI_LOOPBACK");
  if (lb && lb[0] == '1') {                         // loopback group key: any unique 128 bytes
    static unsigned long long counter = 0;
    memset(out128, 0, 128);
    const unsigned long long v = ++counter ^ (unsigned long long)(uintptr_t)&counter;
    memcpy(out128, &v, sizeof(v));
    return 0;
  }
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
  const char *lb = getenv("IETI_LOOPBACK");
  if (world > 1 && lb && lb[0] == '1') {
    if (!uid128) throw CommError("loopback group needs an id");
    const std::string key((const char *)uid128, 128);
    std::lock_guard<std::mutex> g(loop_registry_m);
    auto &sp = loop_registry()[key];
    if (!sp) {
      sp = std::make_shared<LoopGroup>();
      sp->world = world;
      sp->send.assign(world, nullptr);
      sp->peers.assign(world, nullptr);
      sp->ptr.assign(world, nullptr);
    }
    loop = sp;
    comm = this;                                   // non-null: the collective paths are active
    return;
  }
  if (!uid128) throw CommError("world > 1 needs nccl_unique_id");
  if (!api().load()) throw CommError(api().err);
  ncclUniqueId id;
  memcpy(&id, uid128, 128);
  ncclComm_t c = nullptr;
  nck(api().CommInitRank(&c, world, id, rank), "CommInitRank");
  comm = c;
}

void Comm::destroy() {
  if (loop) {
    loop.reset();
    comm = nullptr;
    return;
  }
  if (comm) api().CommDestroy((ncclComm_t)comm);
  comm = nullptr;
}

void Comm::allgather(const double *send, double *recv, size_t count, cudaStream_t s) {
  if (loop) {
    cck(cudaStreamSynchronize(s), "sync");
    loop->send[rank] = send;
    loop->barrier();
    for (int q = 0; q < world; ++q)
      cck(cudaMemcpyAsync(recv + (size_t)q * count, loop->send[q], count * sizeof(double), cudaMemcpyDeviceToDevice, s),
          "allgather copy");
    cck(cudaStreamSynchronize(s), "sync");
    loop->barrier();
    return;
  }
  nck(api().AllGather(send, recv, count, ncclDouble, (ncclComm_t)comm, s), "AllGather");
}

void Comm::allreduce_sum(double *buf, size_t count, cudaStream_t s) {
  if (loop) {
    cck(cudaStreamSynchronize(s), "sync");
    loop->send[rank] = buf;
    loop->barrier();
    std::vector<double> acc(count, 0.0), tmp(count);
    for (int q = 0; q < world; ++q) {                 // rank order: every rank gets the same sum
      cck(cudaMemcpy(tmp.data(), loop->send[q], count * sizeof(double), cudaMemcpyDeviceToHost), "allreduce read");
      for (size_t i = 0; i < count; ++i) acc[i] += tmp[i];
    }
    loop->barrier();
    // ordered on s and complete before the barrier (a pageable legacy-stream copy may return
    // before its DMA lands)
    cck(cudaMemcpyAsync(buf, acc.data(), count * sizeof(double), cudaMemcpyHostToDevice, s), "allreduce write");
    cck(cudaStreamSynchronize(s), "sync");
    loop->barrier();
    return;
  }
  nck(api().AllReduce(buf, buf, count, ncclDouble, ncclSum, (ncclComm_t)comm, s), "AllReduce");
}

void Comm::exchange(const std::vector<int> &peers, const double *send, const std::vector<int> &send_ptr,
                    double *recv, const std::vector<int> &recv_ptr, cudaStream_t s) {
  if (loop) {
    cck(cudaStreamSynchronize(s), "sync");
    loop->send[rank] = send;
    loop->peers[rank] = &peers;
    loop->ptr[rank] = &send_ptr;
    loop->barrier();
    for (size_t i = 0; i < peers.size(); ++i) {
      const int q = peers[i], nr = recv_ptr[i + 1] - recv_ptr[i];
      if (!nr) continue;
      const std::vector<int> &pq = *loop->peers[q], &sq = *loop->ptr[q];
      size_t jq = 0;
      while (jq < pq.size() && pq[jq] != rank) ++jq;
      if (jq == pq.size() || sq[jq + 1] - sq[jq] != nr) throw CommError("loopback exchange: inconsistent plans");
      cck(cudaMemcpyAsync(recv + recv_ptr[i], loop->send[q] + sq[jq], nr * sizeof(double), cudaMemcpyDeviceToDevice, s),
          "exchange copy");
    }
    cck(cudaStreamSynchronize(s), "sync");
    loop->barrier();
    return;
  }
  nck(api().GroupStart(), "GroupStart");
  for (size_t i = 0; i < peers.size(); ++i) {
    const int ns = send_ptr[i + 1] - send_ptr[i], nr = recv_ptr[i + 1] - recv_ptr[i];
    if (ns) nck(api().Send(send + send_ptr[i], ns, ncclDouble, peers[i], (ncclComm_t)comm, s), "Send");
    if (nr) nck(api().Recv(recv + recv_ptr[i], nr, ncclDouble, peers[i], (ncclComm_t)comm, s), "Recv");
  }
  nck(api().GroupEnd(), "GroupEnd");
}
