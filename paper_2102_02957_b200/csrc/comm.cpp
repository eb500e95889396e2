// comm.cpp — the two communicators of comm.h: NCCL (one process per GPU; C1/C2 grouped
// send/recv, C3 all-reduce, C4 all-gather, C5 bootstrap of SURVEY §2.3) and the in-process
// virtual world (G ranks on one device, one host thread each).
#include "comm.h"

#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/sv.h"

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

double now_s() {
  using namespace std::chrono;
  return duration<double>(steady_clock::now().time_since_epoch()).count();
}

size_t type_size(CommType t) {
  switch (t) {
    case kU8:
      return 1;
    case kF32:
      return 4;
    default:
      return 8;
  }
}
}  // namespace

double comm_timeout_s() {
  static const double t = [] {
    const char* e = std::getenv("SV_COMM_TIMEOUT_S");
    const double v = e ? std::atof(e) : 0.0;
    return v > 0 ? v : 600.0;
  }();
  return t;
}

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
                sym(h, "ncclCommDestroy", g_nccl.CommDestroy) && sym(h, "ncclCommAbort", g_nccl.CommAbort) &&
                sym(h, "ncclCommGetAsyncError", g_nccl.CommGetAsyncError) && sym(h, "ncclAllReduce", g_nccl.AllReduce) &&
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

// ============================================================================ NCCL
namespace {

class NcclComm final : public Comm {
 public:
  NcclComm(Nccl* n, Nccl::Comm c, int world, int rank, void* scratch) : n_(n), c_(c), scratch_(scratch) {
    world_ = world;
    rank_ = rank;
  }
  ~NcclComm() override {
    if (c_) (aborted_ ? (void)0 : (void)n_->CommDestroy(c_));
  }
  bool local() const override { return false; }
  int allreduce_sum(void* buf, size_t count, CommType type, cudaStream_t st) override {
    return chk(n_->AllReduce(buf, buf, count, (int)type, 0 /* ncclSum */, c_, st), "ncclAllReduce");
  }
  int allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) override {
    return chk(n_->AllGather(send, recv, bytes, Nccl::Uint8, c_, st), "ncclAllGather");
  }
  int barrier(cudaStream_t st) override {
    return chk(n_->AllReduce(scratch_, scratch_, 1, Nccl::F32, 0, c_, st), "ncclAllReduce (barrier)");
  }
  int group_start() override { return chk(n_->GroupStart(), "ncclGroupStart"); }
  int group_end() override { return chk(n_->GroupEnd(), "ncclGroupEnd"); }
  int send(const void* p, size_t bytes, int peer, cudaStream_t st) override {
    return chk(n_->Send(p, bytes, Nccl::Uint8, peer, c_, st), "ncclSend");
  }
  int recv(void* p, size_t bytes, int peer, cudaStream_t st) override {
    return chk(n_->Recv(p, bytes, Nccl::Uint8, peer, c_, st), "ncclRecv");
  }
  // Poll the stream and the communicator's asynchronous error: a failed or vanished peer makes
  // NCCL kernels spin forever, so after comm_timeout_s() (or on an async error) the communicator
  // is aborted, which also releases the stream, and the call fails with SV_ENCCL.
  int wait(cudaStream_t st) override {
    if (aborted_) return fail(SV_ENCCL, "communicator was aborted after an earlier failure");
    const double t0 = now_s(), limit = comm_timeout_s();
    int spins = 0;
    for (;;) {
      const cudaError_t e = cudaStreamQuery(st);
      if (e == cudaSuccess) return SV_OK;
      if (e != cudaErrorNotReady) return fail(SV_ECUDA, std::string("stream failed: ") + cudaGetErrorString(e));
      int ae = 0;
      if (n_->CommGetAsyncError(c_, &ae) == 0 && ae != 0 && ae != 7 /* ncclInProgress */) {
        abort_comm();
        return fail(SV_ENCCL, std::string("NCCL asynchronous error: ") + n_->GetErrorString(ae));
      }
      if (now_s() - t0 > limit) {
        abort_comm();
        return fail(SV_ENCCL, "NCCL collective did not complete within SV_COMM_TIMEOUT_S = " + std::to_string(limit) +
                                  " s (a peer failed or stopped calling); communicator aborted");
      }
      if (++spins > 200) std::this_thread::sleep_for(std::chrono::microseconds(50));
      else std::this_thread::yield();
    }
  }
  int share_pointers(void*, void**) override { return fail(SV_EINVAL, "internal: NCCL worlds map peers with CUDA IPC"); }

 private:
  int chk(int r, const char* what) {
    if (r == 0) return SV_OK;
    return fail(SV_ENCCL, std::string(what) + ": " + n_->GetErrorString(r));
  }
  void abort_comm() {
    if (!aborted_ && c_) n_->CommAbort(c_);
    aborted_ = true;
  }
  Nccl* n_;
  Nccl::Comm c_;
  void* scratch_;
  bool aborted_ = false;
};

}  // namespace

Comm* make_nccl_comm(int world, int rank, const void* uid128, void* scratch, std::string& err) {
  Nccl* n = nccl(err);
  if (!n) return nullptr;
  Nccl::UniqueId id;
  std::memcpy(id.internal, uid128, 128);
  Nccl::Comm c = nullptr;
  const int r = n->CommInitRank(&c, world, id, rank);
  if (r != 0) {
    err = std::string("ncclCommInitRank: ") + n->GetErrorString(r);
    return nullptr;
  }
  return new NcclComm(n, c, world, rank, scratch);
}

// ============================================================================ local world
struct LocalWorld {
  explicit LocalWorld(int g) : G(g), host(g), ev(g, nullptr), ptrs(g, nullptr) {}
  const int G;
  std::mutex mu;
  std::condition_variable cv;
  int refs = 1;
  int arrived = 0;
  uint64_t gen = 0;
  bool broken = false;                          // a barrier timed out: every later call fails
  std::vector<std::vector<unsigned char>> host;  // per-rank staging of reductions / gathers
  std::vector<cudaEvent_t> ev;                   // per-rank barrier events
  std::vector<void*> ptrs;
  struct Post {
    const void* p;
    size_t bytes;
    cudaEvent_t ready;
  };
  std::map<std::pair<int, int>, std::deque<Post>> posts;         // (src, dst) -> sends not yet received
  std::map<std::pair<int, int>, std::deque<cudaEvent_t>> dones;  // (src, dst) -> receives completed
};

LocalWorld* local_world_create(int world) { return new LocalWorld(world); }

void local_world_release(LocalWorld* w) {
  if (!w) return;
  bool last = false;
  {
    std::lock_guard<std::mutex> lk(w->mu);
    last = --w->refs == 0;
  }
  if (last) {
    for (cudaEvent_t e : w->ev)
      if (e) cudaEventDestroy(e);
    delete w;
  }
}

int local_world_size(const LocalWorld* w) { return w ? w->G : 0; }

namespace {

class LocalComm final : public Comm {
 public:
  LocalComm(LocalWorld* w, int rank) : w_(w) {
    world_ = w->G;
    rank_ = rank;
    std::lock_guard<std::mutex> lk(w->mu);
    w->refs++;
  }
  ~LocalComm() override { local_world_release(w_); }
  bool local() const override { return true; }

  int allreduce_sum(void* buf, size_t count, CommType type, cudaStream_t st) override {
    const size_t bytes = count * type_size(type);
    std::vector<unsigned char> sum(bytes);
    if (int rc = post_host(buf, bytes, st)) return rc;
    {  // every rank sums all contributions in rank order: identical bits on every rank
      std::lock_guard<std::mutex> lk(w_->mu);
      for (size_t i = 0; i < count; i++) {
        if (type == kF64) {
          double s = 0.0;
          for (int r = 0; r < world_; r++) s += reinterpret_cast<const double*>(w_->host[r].data())[i];
          reinterpret_cast<double*>(sum.data())[i] = s;
        } else if (type == kF32) {
          float s = 0.0f;
          for (int r = 0; r < world_; r++) s += reinterpret_cast<const float*>(w_->host[r].data())[i];
          reinterpret_cast<float*>(sum.data())[i] = s;
        } else if (type == kU64) {
          uint64_t s = 0;
          for (int r = 0; r < world_; r++) s += reinterpret_cast<const uint64_t*>(w_->host[r].data())[i];
          reinterpret_cast<uint64_t*>(sum.data())[i] = s;
        } else {
          unsigned char s = 0;
          for (int r = 0; r < world_; r++) s = (unsigned char)(s + w_->host[r][i]);
          sum[i] = s;
        }
      }
    }
    if (int rc = host_barrier()) return rc;  // everyone has read the staging
    if (cudaMemcpyAsync(buf, sum.data(), bytes, cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      return fail(SV_ECUDA, "local all-reduce: copy back failed");
    return SV_OK;
  }

  int allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) override {
    if (int rc = post_host(send, bytes, st)) return rc;
    std::vector<unsigned char> all(bytes * world_);
    {
      std::lock_guard<std::mutex> lk(w_->mu);
      for (int r = 0; r < world_; r++) std::memcpy(all.data() + r * bytes, w_->host[r].data(), bytes);
    }
    if (int rc = host_barrier()) return rc;
    if (cudaMemcpyAsync(recv, all.data(), all.size(), cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      return fail(SV_ECUDA, "local all-gather: copy failed");
    return SV_OK;
  }

  int barrier(cudaStream_t st) override {
    cudaEvent_t mine;
    {
      std::lock_guard<std::mutex> lk(w_->mu);
      if (!w_->ev[rank_] && cudaEventCreateWithFlags(&w_->ev[rank_], cudaEventDisableTiming) != cudaSuccess)
        return fail(SV_ECUDA, "local barrier: event creation failed");
      mine = w_->ev[rank_];
    }
    if (cudaEventRecord(mine, st) != cudaSuccess) return fail(SV_ECUDA, "local barrier: event record failed");
    if (int rc = host_barrier()) return rc;
    for (int r = 0; r < world_; r++) {
      cudaEvent_t e;
      {
        std::lock_guard<std::mutex> lk(w_->mu);
        e = w_->ev[r];
      }
      if (r != rank_ && cudaStreamWaitEvent(st, e, 0) != cudaSuccess) return fail(SV_ECUDA, "local barrier: wait failed");
    }
    return host_barrier();  // every rank has captured every event before any is recorded again
  }

  int group_start() override {
    in_group_ = true;
    return SV_OK;
  }
  int group_end() override {
    in_group_ = false;
    return flush();
  }
  int send(const void* p, size_t bytes, int peer, cudaStream_t st) override {
    ops_.push_back({true, const_cast<void*>(p), bytes, peer, st});
    return in_group_ ? SV_OK : flush();
  }
  int recv(void* p, size_t bytes, int peer, cudaStream_t st) override {
    ops_.push_back({false, p, bytes, peer, st});
    return in_group_ ? SV_OK : flush();
  }

  int wait(cudaStream_t st) override {
    const cudaError_t e = cudaStreamSynchronize(st);
    return e == cudaSuccess ? SV_OK : fail(SV_ECUDA, std::string("stream failed: ") + cudaGetErrorString(e));
  }

  int share_pointers(void* mine, void** all) override {
    {
      std::lock_guard<std::mutex> lk(w_->mu);
      w_->ptrs[rank_] = mine;
    }
    if (int rc = host_barrier()) return rc;
    {
      std::lock_guard<std::mutex> lk(w_->mu);
      for (int r = 0; r < world_; r++) all[r] = w_->ptrs[r];
    }
    return host_barrier();
  }

 private:
  struct Op {
    bool is_send;
    void* p;
    size_t bytes;
    int peer;
    cudaStream_t st;
  };

  // Generation-counted barrier of the world's host threads, with the communicator timeout.
  int host_barrier() {
    std::unique_lock<std::mutex> lk(w_->mu);
    if (w_->broken) return fail(SV_ENCCL, "local world is broken (an earlier barrier timed out)");
    const uint64_t g = w_->gen;
    if (++w_->arrived == world_) {
      w_->arrived = 0;
      w_->gen++;
      w_->cv.notify_all();
      return SV_OK;
    }
    const bool ok = w_->cv.wait_for(lk, std::chrono::duration<double>(comm_timeout_s()),
                                    [&] { return w_->gen != g || w_->broken; });
    if (!ok || w_->broken) {
      w_->broken = true;
      w_->cv.notify_all();
      return fail(SV_ENCCL, "local world: a rank did not reach the barrier within SV_COMM_TIMEOUT_S");
    }
    return SV_OK;
  }

  // copy this rank's device contribution into its host slot, then wait for every rank's
  int post_host(const void* dev, size_t bytes, cudaStream_t st) {
    std::vector<unsigned char> tmp(bytes);
    if (cudaMemcpyAsync(tmp.data(), dev, bytes, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      return fail(SV_ECUDA, "local collective: device-to-host copy failed");
    {
      std::lock_guard<std::mutex> lk(w_->mu);
      w_->host[rank_].swap(tmp);
    }
    return host_barrier();
  }

  template <typename Pred>
  int wait_for(std::unique_lock<std::mutex>& lk, Pred pred, const char* what) {
    if (!w_->cv.wait_for(lk, std::chrono::duration<double>(comm_timeout_s()), [&] { return pred() || w_->broken; }) ||
        w_->broken) {
      w_->broken = true;
      w_->cv.notify_all();
      return fail(SV_ENCCL, std::string("local world: ") + what + " timed out");
    }
    return SV_OK;
  }

  // Execute the queued sends / receives: post every send (pointer + ready event), then serve every
  // receive as a device-to-device copy from the sender's buffer, then wait until every send has
  // been received (its buffer may change afterwards).  Posts before waits: no pairwise deadlock.
  int flush() {
    std::vector<Op> ops;
    ops.swap(ops_);
    for (const Op& o : ops) {
      if (!o.is_send) continue;
      cudaEvent_t e;
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess || cudaEventRecord(e, o.st) != cudaSuccess)
        return fail(SV_ECUDA, "local send: event failed");
      std::lock_guard<std::mutex> lk(w_->mu);
      w_->posts[{rank_, o.peer}].push_back({o.p, o.bytes, e});
      w_->cv.notify_all();
    }
    for (const Op& o : ops) {
      if (o.is_send) continue;
      LocalWorld::Post x{};
      {
        std::unique_lock<std::mutex> lk(w_->mu);
        auto& q = w_->posts[{o.peer, rank_}];
        if (int rc = wait_for(lk, [&] { return !q.empty(); }, "receive")) return rc;
        x = q.front();
        q.pop_front();
      }
      if (x.bytes != o.bytes) return fail(SV_EINVAL, "local recv: size does not match the matching send");
      cudaEvent_t d;
      if (cudaStreamWaitEvent(o.st, x.ready, 0) != cudaSuccess ||
          cudaMemcpyAsync(o.p, x.p, o.bytes, cudaMemcpyDeviceToDevice, o.st) != cudaSuccess ||
          cudaEventCreateWithFlags(&d, cudaEventDisableTiming) != cudaSuccess || cudaEventRecord(d, o.st) != cudaSuccess)
        return fail(SV_ECUDA, "local recv: copy failed");
      cudaEventDestroy(x.ready);
      std::lock_guard<std::mutex> lk(w_->mu);
      w_->dones[{o.peer, rank_}].push_back(d);
      w_->cv.notify_all();
    }
    for (const Op& o : ops) {
      if (!o.is_send) continue;
      cudaEvent_t d;
      {
        std::unique_lock<std::mutex> lk(w_->mu);
        auto& q = w_->dones[{rank_, o.peer}];
        if (int rc = wait_for(lk, [&] { return !q.empty(); }, "send completion")) return rc;
        d = q.front();
        q.pop_front();
      }
      if (cudaStreamWaitEvent(o.st, d, 0) != cudaSuccess) return fail(SV_ECUDA, "local send: wait failed");
      cudaEventDestroy(d);
    }
    return SV_OK;
  }

  LocalWorld* w_;
  bool in_group_ = false;
  std::vector<Op> ops_;
};

}  // namespace

Comm* make_local_comm(LocalWorld* w, int rank, std::string& err) {
  if (!w || rank < 0 || rank >= w->G) {
    err = "bad local world or rank";
    return nullptr;
  }
  return new LocalComm(w, rank);
}

}  // namespace sv
