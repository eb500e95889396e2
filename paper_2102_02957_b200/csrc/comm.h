// comm.h — the communicator of one rank (C1-C5 of SURVEY §2.3): the only place the library's
// collectives go through.  Two implementations:
//   * NcclComm: one process per GPU, NCCL loaded at run time (dlopen), so single-GPU use needs
//     no NCCL and the process shares whichever libnccl.so.2 torch already loaded.  Waits on a
//     stream that has NCCL work poll ncclCommGetAsyncError with a timeout (a dead peer returns
//     SV_ENCCL instead of hanging every rank).
//   * LocalComm: an in-process "virtual world" of G ranks whose shards live on ONE device, each
//     rank driven by its own host thread (sv_world_create / sv_create_local).  Barriers are CUDA
//     events exchanged through a host barrier (stream-ordered, no device-side waiting), reductions
//     are summed on the host in rank order, send/recv are device-to-device copies.  It runs the
//     same exchange kernels, plans and readouts as the NCCL path, so a one-GPU box can test them.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <string>

namespace sv {

struct Nccl {
  // opaque NCCL types
  typedef void* Comm;
  struct UniqueId {
    char internal[128];
  };
  enum DType { Int8 = 0, Uint8 = 1, Int32 = 2, Uint32 = 3, Int64 = 4, Uint64 = 5, F16 = 6, F32 = 7, F64 = 8 };
  int (*GetUniqueId)(void* id) = nullptr;
  int (*CommInitRank)(Comm* comm, int nranks, UniqueId id, int rank) = nullptr;
  int (*CommDestroy)(Comm) = nullptr;
  int (*CommAbort)(Comm) = nullptr;
  int (*CommGetAsyncError)(Comm, int*) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  int (*AllGather)(const void*, void*, size_t, int, Comm, cudaStream_t) = nullptr;
  int (*Send)(const void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  int (*Recv)(void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
  void* handle = nullptr;
};

// Load NCCL once; returns nullptr (and fills err) if unavailable.
Nccl* nccl(std::string& err);

// Element types of the reductions (values of Nccl::DType).
enum CommType { kU8 = Nccl::Uint8, kU64 = Nccl::Uint64, kF32 = Nccl::F32, kF64 = Nccl::F64 };

// One rank's view of the world.  Every call returns 0 or a negative SV_E* code with a message in
// err().  All calls are collective in the same order on every rank except send / recv, which
// pair up between two ranks (inside group_start / group_end they are matched as a batch).
class Comm {
 public:
  virtual ~Comm() = default;
  int rank() const { return rank_; }
  int world() const { return world_; }
  const std::string& err() const { return err_; }
  virtual bool local() const = 0;  // in-process virtual world (shards on one device)
  // in-place sum over ranks of `count` elements of `type`, stream-ordered on st
  virtual int allreduce_sum(void* buf, size_t count, CommType type, cudaStream_t st) = 0;
  // recv[r * bytes ...] = rank r's send (device buffers), stream-ordered on st
  virtual int allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) = 0;
  // stream-ordered barrier: work queued on st after it starts after every rank's work queued on its
  // own stream before it (NCCL: a 1-element all-reduce; local: events)
  virtual int barrier(cudaStream_t st) = 0;
  virtual int group_start() = 0;
  virtual int group_end() = 0;
  virtual int send(const void* p, size_t bytes, int peer, cudaStream_t st) = 0;
  virtual int recv(void* p, size_t bytes, int peer, cudaStream_t st) = 0;
  // block until st is idle; NCCL: poll the communicator's async error, abort it after timeout_s
  virtual int wait(cudaStream_t st) = 0;
  // device pointers of every rank's shard as usable from this rank's device (local worlds: the
  // pointers themselves; NCCL worlds use CUDA IPC in api.cpp).  Collective.
  virtual int share_pointers(void* mine, void** all) = 0;

 protected:
  int fail(int code, const std::string& msg) {
    err_ = msg;
    return code;
  }
  int rank_ = 0, world_ = 1;
  std::string err_;
};

// NCCL communicator of rank `rank` in a world of `world` processes (uid128: ncclGetUniqueId of
// rank 0).  scratch: 16 bytes of device memory the barrier reduces.  Returns nullptr + err.
Comm* make_nccl_comm(int world, int rank, const void* uid128, void* scratch, std::string& err);

// In-process virtual worlds (sv_world_create): ranks of one world share its state.
struct LocalWorld;
LocalWorld* local_world_create(int world);
void local_world_release(LocalWorld* w);  // reference counted: the world and every rank handle
int local_world_size(const LocalWorld* w);
Comm* make_local_comm(LocalWorld* w, int rank, std::string& err);

// Seconds a collective may wait for its peers before it fails with SV_ENCCL (SV_COMM_TIMEOUT_S,
// default 600).
double comm_timeout_s();

}  // namespace sv
