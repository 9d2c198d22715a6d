// TEST INFRASTRUCTURE: a minimal stand-in for libnccl.so.2 that lets several processes share ONE
// GPU (real NCCL refuses duplicate GPUs in a communicator), so the product's NCCL transport code
// (libpjds: dist.cpp post_nccl, message schedule, comm stream + events) runs unchanged in a
// multi-process test on a single B200.
//
// Semantics (enough for grouped point-to-point): ncclSend/ncclRecv inside ncclGroupStart/End are
// recorded; ncclGroupEnd synchronises the stream, publishes every send buffer through CUDA IPC in a
// POSIX shared-memory mailbox (slot per (src, dst, message index)), then completes every receive by
// a device-to-device copy from the peer's buffer, and finally waits until its own sends have been
// consumed.  All sends are published before any receive blocks, so a group cannot deadlock.
// Message k from a to b is matched with the k-th receive b posts from a -- NCCL's ordering rule.
#include <cuda.h>
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

extern "C" {
typedef enum { ncclSuccess = 0, ncclUnhandledCudaError = 1, ncclSystemError = 2, ncclInternalError = 3,
               ncclInvalidArgument = 4, ncclInvalidUsage = 5 } ncclResult_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef enum { ncclInt8 = 0, ncclUint8 = 1, ncclInt32 = 2, ncclUint32 = 3, ncclInt64 = 4, ncclUint64 = 5,
               ncclFloat16 = 6, ncclFloat32 = 7, ncclFloat64 = 8, ncclBfloat16 = 9 } ncclDataType_t;
struct FakeComm;
typedef FakeComm* ncclComm_t;
}

namespace {

constexpr int kMaxRanks = 8;
constexpr int kMaxMsgs = 256;  // per (src, dst) pair and group

struct Slot {
  std::atomic<uint64_t> posted;    // group sequence number the message belongs to
  std::atomic<uint64_t> consumed;  // group sequence number the receiver finished copying
  cudaIpcMemHandle_t handle;
  uint64_t offset, bytes;
};
struct Mailbox {
  Slot slot[kMaxRanks][kMaxRanks][kMaxMsgs];
};

struct Op {
  bool send;
  void* buf;
  size_t bytes;
  int peer;
  cudaStream_t stream;
};

}  // namespace

struct FakeComm {
  std::string name;
  int rank = 0, nranks = 1;
  Mailbox* mb = nullptr;
  uint64_t seq_send[8] = {}, seq_recv[8] = {};  // groups with traffic on each directed pair
};

namespace {
thread_local std::vector<std::pair<FakeComm*, Op>> g_ops;
thread_local int g_depth = 0;

size_t tsize(ncclDataType_t t) {
  switch (t) {
    case ncclInt8: case ncclUint8: return 1;
    case ncclFloat16: case ncclBfloat16: return 2;
    case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
    default: return 8;
  }
}

ncclResult_t run_group() {
  if (g_ops.empty()) return ncclSuccess;
  FakeComm* c = g_ops[0].first;
  for (auto& po : g_ops)
    if (cudaStreamSynchronize(po.second.stream) != cudaSuccess) return ncclUnhandledCudaError;
  int sent[kMaxRanks] = {}, recvd[kMaxRanks] = {};
  // a directed pair's sequence number advances once per group that carries messages on it, on
  // both ends, so ranks that skip a group (nothing to exchange) stay in step
  uint64_t sseq[kMaxRanks], rseq[kMaxRanks];
  bool has_s[kMaxRanks] = {}, has_r[kMaxRanks] = {};
  for (auto& po : g_ops) (po.second.send ? has_s : has_r)[po.second.peer] = true;
  for (int p = 0; p < kMaxRanks; ++p) {
    sseq[p] = has_s[p] ? ++c->seq_send[p] : 0;
    rseq[p] = has_r[p] ? ++c->seq_recv[p] : 0;
  }
  // publish sends
  for (auto& po : g_ops) {
    const Op& o = po.second;
    if (!o.send) continue;
    Slot& s = c->mb->slot[c->rank][o.peer][sent[o.peer]++];
    CUdeviceptr base = 0;
    size_t size = 0;
    if (cuMemGetAddressRange(&base, &size, (CUdeviceptr)o.buf) != CUDA_SUCCESS) return ncclUnhandledCudaError;
    if (cudaIpcGetMemHandle(&s.handle, (void*)base) != cudaSuccess) return ncclUnhandledCudaError;
    s.offset = (uint64_t)((CUdeviceptr)o.buf - base);
    s.bytes = o.bytes;
    s.posted.store(sseq[o.peer], std::memory_order_release);
  }
  // complete receives
  for (auto& po : g_ops) {
    const Op& o = po.second;
    if (o.send) continue;
    Slot& s = c->mb->slot[o.peer][c->rank][recvd[o.peer]++];
    while (s.posted.load(std::memory_order_acquire) != rseq[o.peer]) std::this_thread::yield();
    if (s.bytes != o.bytes) {
      std::fprintf(stderr, "fake nccl: size mismatch %d->%d: %llu vs %zu\n", o.peer, c->rank,
                   (unsigned long long)s.bytes, o.bytes);
      return ncclInvalidUsage;
    }
    void* peer = nullptr;
    if (cudaIpcOpenMemHandle(&peer, s.handle, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return ncclUnhandledCudaError;
    cudaError_t e = cudaMemcpy(o.buf, (char*)peer + s.offset, o.bytes, cudaMemcpyDeviceToDevice);
    cudaIpcCloseMemHandle(peer);
    if (e != cudaSuccess) return ncclUnhandledCudaError;
    s.consumed.store(rseq[o.peer], std::memory_order_release);
  }
  // our send buffers may be reused once every receiver has copied them
  for (int p = 0; p < c->nranks; ++p)
    for (int k = 0; k < sent[p]; ++k)
      while (c->mb->slot[c->rank][p][k].consumed.load(std::memory_order_acquire) != sseq[p]) std::this_thread::yield();
  g_ops.clear();
  return ncclSuccess;
}

}  // namespace

extern "C" {

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
  std::memset(id, 0, sizeof(*id));
  std::random_device rd;
  std::snprintf(id->internal, sizeof(id->internal), "/pjds_fake_nccl_%08x%08x", rd(), rd());
  return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* comm, int nranks, ncclUniqueId id, int rank) {
  if (nranks > kMaxRanks || rank < 0 || rank >= nranks) return ncclInvalidArgument;
  cuInit(0);
  int fd = shm_open(id.internal, O_CREAT | O_RDWR, 0600);
  if (fd < 0) return ncclSystemError;
  if (ftruncate(fd, sizeof(Mailbox)) != 0) { close(fd); return ncclSystemError; }
  void* p = mmap(nullptr, sizeof(Mailbox), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) return ncclSystemError;
  auto* c = new FakeComm();
  c->rank = rank;
  c->nranks = nranks;
  c->mb = (Mailbox*)p;
  c->name = id.internal;
  *comm = c;
  return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t comm) {
  if (comm) {
    munmap(comm->mb, sizeof(Mailbox));
    if (comm->rank == 0) shm_unlink(comm->name.c_str());
    delete comm;
  }
  return ncclSuccess;
}

ncclResult_t ncclGroupStart() {
  ++g_depth;
  return ncclSuccess;
}

ncclResult_t ncclGroupEnd() {
  if (--g_depth > 0) return ncclSuccess;
  return run_group();
}

ncclResult_t ncclSend(const void* buf, size_t count, ncclDataType_t t, int peer, ncclComm_t comm, cudaStream_t s) {
  g_ops.push_back({comm, Op{true, const_cast<void*>(buf), count * tsize(t), peer, s}});
  return g_depth ? ncclSuccess : run_group();
}

ncclResult_t ncclRecv(void* buf, size_t count, ncclDataType_t t, int peer, ncclComm_t comm, cudaStream_t s) {
  g_ops.push_back({comm, Op{false, buf, count * tsize(t), peer, s}});
  return g_depth ? ncclSuccess : run_group();
}

const char* ncclGetErrorString(ncclResult_t r) {
  static const char* names[] = {"success", "unhandled cuda error", "system error", "internal error",
                                "invalid argument", "invalid usage"};
  return (r >= 0 && r <= 5) ? names[r] : "unknown";
}

}  // extern "C"
