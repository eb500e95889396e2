// comm.h — NCCL loaded at run time (dlopen) so single-GPU use needs no NCCL and the process
// shares whichever libnccl.so.2 torch already loaded.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
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
// ncclCommInitRank with a 128-byte unique id.
int nccl_comm_init(Nccl* n, Nccl::Comm* comm, int nranks, const void* uid128, int rank);

}  // namespace sv
