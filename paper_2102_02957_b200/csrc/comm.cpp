// comm.cpp — run-time binding of the NCCL entry points the library uses (C5 bootstrap, C1/C2
// grouped send/recv, C3 all-reduce, C4 all-gather of SURVEY §2.3).
#include "comm.h"

#include <dlfcn.h>

#include <cstring>
#include <mutex>

namespace sv {

namespace {
std::mutex g_mu;
Nccl g_nccl;
bool g_tried = false;
std::string g_err;

template <typename F>
bool sym(void* h, const char* name, F& out) {
  out = reinterpret_cast<F>(dlsym(h, name));
  return out != nullptr;
}
}  // namespace

Nccl* nccl(std::string& err) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_tried) {
    g_tried = true;
    // Prefer an already-loaded NCCL (torch's), then the default search path.
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      g_err = std::string("cannot load libnccl.so.2: ") + dlerror();
    } else {
      bool ok = sym(h, "ncclGetUniqueId", g_nccl.GetUniqueId) && sym(h, "ncclCommInitRank", g_nccl.CommInitRank) &&
                sym(h, "ncclCommDestroy", g_nccl.CommDestroy) && sym(h, "ncclAllReduce", g_nccl.AllReduce) &&
                sym(h, "ncclAllGather", g_nccl.AllGather) && sym(h, "ncclSend", g_nccl.Send) &&
                sym(h, "ncclRecv", g_nccl.Recv) && sym(h, "ncclGroupStart", g_nccl.GroupStart) &&
                sym(h, "ncclGroupEnd", g_nccl.GroupEnd) && sym(h, "ncclGetErrorString", g_nccl.GetErrorString);
      if (!ok) {
        g_err = "libnccl.so.2 lacks a required symbol";
      } else {
        g_nccl.handle = h;
      }
    }
  }
  if (!g_nccl.handle) {
    err = g_err;
    return nullptr;
  }
  return &g_nccl;
}

int nccl_comm_init(Nccl* n, Nccl::Comm* comm, int nranks, const void* uid128, int rank) {
  Nccl::UniqueId id;
  std::memcpy(id.internal, uid128, 128);
  return n->CommInitRank(comm, nranks, id, rank);
}

}  // namespace sv
