// api.cpp — the C ABI (include/sv.h): handle, sharded state store, executor, readout.
//
// Layers: L1 this file (validation, errors, handle) -> L2 host planner (blocking.cpp,
// plan.cpp, compile.cpp) -> L3 sharded store + scheduler (this file: pi/sigma maps, stream,
// program upload, step execution) -> L4 kernels (kernels.cu) and L5 comm (comm.cpp, NCCL +
// CUDA IPC peer memory).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "comm.h"
#include "common.h"
#include "compile.h"
#include "jit.h"
#include "kernels.cuh"

using namespace sv;

namespace {

thread_local std::string g_last_error;

// NVTX ranges (header-only NVTX3: free unless a tool such as Nsight Systems is attached) around
// every circuit, section launch, exchange and readout, so a timeline shows the step structure.
struct Nvtx {
  explicit Nvtx(const char* fmt, ...) __attribute__((format(printf, 2, 3))) {
    char buf[160];
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    nvtxRangePushA(buf);
  }
  ~Nvtx() { nvtxRangePop(); }
  Nvtx(const Nvtx&) = delete;
  Nvtx& operator=(const Nvtx&) = delete;
};

double now_ms() {
  using namespace std::chrono;
  return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
};

struct PinBuf {
  void* p = nullptr;
  size_t cap = 0;
};

// Bit-permutation evaluated with byte tables: f(x) = OR_j T_j[byte_j(x)].
struct BitPerm {
  std::vector<uint64_t> t;  // nbytes * 256
  int nbytes = 0;
  void build(const std::vector<int>& dst_of_src_bit) {  // bit i of x goes to bit dst[i]
    const int n = (int)dst_of_src_bit.size();
    nbytes = (n + 7) / 8;
    t.assign((size_t)nbytes * 256, 0);
    for (int j = 0; j < nbytes; j++)
      for (int v = 0; v < 256; v++) {
        uint64_t o = 0;
        for (int b = 0; b < 8; b++)
          if (((v >> b) & 1) && 8 * j + b < n) o |= 1ull << dst_of_src_bit[8 * j + b];
        t[(size_t)j * 256 + v] = o;
      }
  }
  uint64_t operator()(uint64_t x) const {
    uint64_t o = 0;
    for (int j = 0; j < nbytes; j++) o |= t[(size_t)j * 256 + ((x >> (8 * j)) & 255)];
    return o;
  }
};

}  // namespace

struct sv_state {
  int n = 0, c = 0, nL = 0, g = 0, rank = 0, world = 1, device = 0;
  bool dbl = true;
  size_t amp = 16;
  void* sv = nullptr;
  bool own_sv = false;
  cudaStream_t st = nullptr;
  bool own_stream = false;
  std::vector<int> pi, sigma;

  DevBuf d_prog, d_coef, d_aux, d_scratch, d_small, d_tmp, d_tmp2, d_stage;
  PinBuf h_stage, h_stage2;
  cudaEvent_t ev_upload = nullptr;
  bool upload_pending = false;

  Comm* comm = nullptr;            // NCCL (one process per GPU) or an in-process local world
  std::vector<void*> peers;       // peer shard pointers mapped in this process (self = sv)
  std::vector<void*> ipc_opened;  // to close
  bool p2p = false;
  // cross-GPU exchange engine (exchange(), lazy): receive slots mapped by every peer, a push /
  // transport stream and an unpack stream (both high priority), and the pipeline's events
  DevBuf d_xrecv, d_xsend;
  std::vector<void*> peer_xrecv;  // every rank's receive slots (peer path)
  std::vector<void*> xrecv_opened;
  bool xrecv_shared = false;
  uint64_t xslot = 0;             // amplitudes per slot
  cudaStream_t st_x = nullptr, st_u = nullptr, st_p = nullptr;
  cudaEvent_t ev_start = nullptr, ev_pushed[3] = {}, ev_unpacked[3] = {}, ev_landed[4] = {}, ev_done = nullptr;
  cudaEvent_t ev_packed[2] = {}, ev_prev[4] = {};

  Program prog;
  sv_stats_t stats{};
  std::string err;
  bool basis_pending = false;  // state is exactly |basis_index> (set by sv_reset)
  uint64_t basis_index = 0;
  bool virt = false;  // ... and not written yet: the next circuit's first section generates it

  // optional per-launch device timing (sv_set_timing)
  struct TRec {
    cudaEvent_t a, b;
    int kind;  // 0 section, 1 exchange, 2 gate, 3 section with a generated input (write only)
    double bytes, flops;
  };
  bool timing = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<TRec> trecs;
};

namespace {

int fail(sv_state* h, int code, const std::string& msg) {
  if (h) h->err = msg;
  g_last_error = msg;
  return code;
}
int fail(sv_state* h, const Status& s) { return fail(h, s.code, s.msg); }

#define CUDA_TRY(h, expr)                                                                        \
  do {                                                                                           \
    cudaError_t _e = (expr);                                                                     \
    if (_e != cudaSuccess)                                                                       \
      return fail(h, SV_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));              \
  } while (0)

#define COMM_TRY(h, expr)                                                                        \
  do {                                                                                           \
    int _r = (expr);                                                                             \
    if (_r != 0) return fail(h, _r, (h)->comm->err());                                           \
  } while (0)

int ensure_dev(sv_state* h, DevBuf& b, size_t bytes) {
  if (b.cap >= bytes) return SV_OK;
  if (b.p) {
    CUDA_TRY(h, cudaStreamSynchronize(h->st));
    CUDA_TRY(h, cudaFree(b.p));
    b.p = nullptr;
    b.cap = 0;
  }
  size_t cap = std::max<size_t>(bytes, 4096);
  cap = (cap + 4095) & ~size_t(4095);
  cudaError_t e = cudaMalloc(&b.p, cap);
  if (e != cudaSuccess) return fail(h, SV_ECAPACITY, std::string("device scratch allocation failed: ") + cudaGetErrorString(e));
  b.cap = cap;
  return SV_OK;
}

int ensure_pin(sv_state* h, PinBuf& b, size_t bytes) {
  if (b.cap >= bytes) return SV_OK;
  if (b.p) {
    CUDA_TRY(h, cudaStreamSynchronize(h->st));
    CUDA_TRY(h, cudaFreeHost(b.p));
    b.p = nullptr;
    b.cap = 0;
  }
  size_t cap = std::max<size_t>(bytes, 1 << 16);
  CUDA_TRY(h, cudaMallocHost(&b.p, cap));
  b.cap = cap;
  return SV_OK;
}

// memory index of logical index x: bit q of x -> bit sigma[pi[q]]
BitPerm mu_of(const sv_state* h) {
  std::vector<int> dst(h->n);
  for (int q = 0; q < h->n; q++) dst[q] = h->sigma[h->pi[q]];
  BitPerm p;
  p.build(dst);
  return p;
}
BitPerm mu_inv_of(const sv_state* h) {
  std::vector<int> dst(h->n);
  for (int q = 0; q < h->n; q++) dst[h->sigma[h->pi[q]]] = q;
  BitPerm p;
  p.build(dst);
  return p;
}

int barrier(sv_state* h, cudaStream_t st = nullptr) {
  if (h->world == 1) return SV_OK;
  COMM_TRY(h, h->comm->barrier(st ? st : h->st));
  return SV_OK;
}

// Block until the handle's stream is idle; on several ranks through the communicator, which fails
// (SV_ENCCL) instead of hanging when a peer is gone (comm.h).
int sync_stream(sv_state* h) {
  if (h->world == 1 || !h->comm) {
    CUDA_TRY(h, cudaStreamSynchronize(h->st));
    return SV_OK;
  }
  COMM_TRY(h, h->comm->wait(h->st));
  return SV_OK;
}

// Section launches an exchange runs quarter by quarter around itself (the executor's pipeline
// plan, apply_circuit): the split bits are out of the tile of every one of them.
struct XPipe {
  int ns = 0, sbit[2] = {0, 0};
  std::vector<size_t> pre, post;  // indices into h->prog.launches
};
int exchange(sv_state* h, std::vector<ExPair> pairs, uint32_t flags, const XPipe& xp);

int upload_program(sv_state* h) {
  const size_t ib = h->prog.ints.size() * sizeof(int);
  const size_t ncoef = h->prog.coefs.size() / 2, naux = h->prog.aux.size() / 2;
  const size_t cb = ncoef * h->amp, ab = naux * h->amp;
  if (ib + cb + ab == 0) return SV_OK;
  if (h->upload_pending) CUDA_TRY(h, cudaEventSynchronize(h->ev_upload));  // staging reuse
  const size_t c_at = (ib + 15) & ~size_t(15), a_at = (c_at + cb + 15) & ~size_t(15);
  if (int rc = ensure_pin(h, h->h_stage, a_at + ab + 64)) return rc;
  if (int rc = ensure_dev(h, h->d_prog, ib + 16)) return rc;
  if (int rc = ensure_dev(h, h->d_coef, cb + 16)) return rc;
  if (int rc = ensure_dev(h, h->d_aux, ab + 16)) return rc;
  char* s = (char*)h->h_stage.p;
  std::memcpy(s, h->prog.ints.data(), ib);
  auto put = [&](char* dst, const std::vector<double>& src, size_t n) {
    if (h->dbl) {
      std::memcpy(dst, src.data(), n * 16);
    } else {  // round to nearest fp32 on upload
      float* f = (float*)dst;
      for (size_t i = 0; i < 2 * n; i++) f[i] = (float)src[i];
    }
  };
  put(s + c_at, h->prog.coefs, ncoef);
  put(s + a_at, h->prog.aux, naux);
  if (ib) CUDA_TRY(h, cudaMemcpyAsync(h->d_prog.p, s, ib, cudaMemcpyHostToDevice, h->st));
  if (cb) CUDA_TRY(h, cudaMemcpyAsync(h->d_coef.p, s + c_at, cb, cudaMemcpyHostToDevice, h->st));
  if (ab) CUDA_TRY(h, cudaMemcpyAsync(h->d_aux.p, s + a_at, ab, cudaMemcpyHostToDevice, h->st));
  CUDA_TRY(h, cudaEventRecord(h->ev_upload, h->st));
  h->upload_pending = true;
  return SV_OK;
}

int gate_step(sv_state* h, const sv_gate& gm) {
  GateArgs a{};
  a.q0 = gm.q0;
  a.q1 = gm.q1;
  auto code = [&](int mb) { return mb >= h->nL ? 200 + ((h->rank >> (mb - h->nL)) & 1) : mb; };
  switch (gm.kind) {
    case SV_U1:
      a.type = SV_OP_U1;
      std::memcpy(a.m, gm.m, 8 * sizeof(double));
      break;
    case SV_U2:
      a.type = SV_OP_U2;
      std::memcpy(a.m, gm.m, 32 * sizeof(double));
      break;
    case SV_D1:
    case SV_D2: {
      a.type = SV_OP_DIAG;
      a.q0 = code(gm.q0);
      a.q1 = gm.kind == SV_D2 ? code(gm.q1) : 200;
      for (int i = 0; i < 8; i++) a.m[i] = (i % 2 == 0) ? 1.0 : 0.0;
      std::memcpy(a.m, gm.m, (gm.kind == SV_D2 ? 8 : 4) * sizeof(double));
      break;
    }
    case SV_SWAP:
      a.type = 7;
      break;
    default:
      return fail(h, SV_EMALFORMED, "internal: bad gate step");
  }
  CUDA_TRY(h, launch_gate(h->dbl, h->sv, h->nL, a, h->st));
  h->stats.kernel_launches++;
  return SV_OK;
}

cudaEvent_t ev_get(sv_state* h) {
  if (!h->ev_pool.empty()) {
    cudaEvent_t e = h->ev_pool.back();
    h->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

cudaEvent_t tstart(sv_state* h) {
  if (!h->timing) return nullptr;
  cudaEvent_t e = ev_get(h);
  cudaEventRecord(e, h->st);
  return e;
}

void tend(sv_state* h, cudaEvent_t a, int kind, double bytes, double flops) {
  if (!a) return;
  cudaEvent_t b = ev_get(h);
  cudaEventRecord(b, h->st);
  h->trecs.push_back({a, b, kind, bytes, flops});
}

int materialize_at(sv_state* h, int64_t vidx);

// One section launch (generated kernel, else the interpreter), optionally restricted to the tiles
// whose out bits match split_a / split_b (kernels.cuh).
int launch_one(sv_state* h, const Launch& L, int split_a = 0, int split_b = 0, int64_t vidx = -1) {
  Nvtx r("sv section T=%d phases=%d ops=%d%s", L.T, L.n_phases, L.n_ops, split_a ? " (quarter)" : "");
  const int* pdev = (const int*)h->d_prog.p + L.int_off;
  const char* cdev = (const char*)h->d_coef.p + L.coef_off * h->amp;
  const char* adev = (const char*)h->d_aux.p + L.aux_off * h->amp;
  cudaError_t je = cudaSuccess;
  if (vidx != -1 && !split_a && !split_b && jit_virtual_input_ok(L, h->dbl)) {
    // The input is a basis state and a section is a linear map applied tile by tile: every tile but
    // the one holding the amplitude is zero in and zero out.  Clear the shard and run that tile.
    CUDA_TRY(h, cudaMemsetAsync(h->sv, 0, h->amp << h->nL, h->st));
    if (vidx < 0) return SV_OK;  // the amplitude is on another GPU: this shard stays zero
    const SvSecHeader* H = reinterpret_cast<const SvSecHeader*>(h->prog.ints.data() + L.int_off);
    int64_t tile = 0;
    for (int j = 0; j < H->n_out; j++) tile |= (int64_t)((vidx >> H->out_bits[j]) & 1) << j;
    if (jit_launch_section(h->dbl, h->sv, h->prog.ints.data() + L.int_off, h->prog.coefs.data() + 2 * L.coef_off, L,
                           cdev, adev, h->st, &je, 0, 0, vidx, tile)) {
      CUDA_TRY(h, je);
      h->stats.jit_launches++;
      h->stats.kernel_launches++;
      return SV_OK;
    }
    if (int rc = materialize_at(h, vidx)) return rc;  // no generated kernel after all
    return launch_one(h, L, split_a, split_b, -1);
  }
  if (jit_launch_section(h->dbl, h->sv, h->prog.ints.data() + L.int_off, h->prog.coefs.data() + 2 * L.coef_off, L,
                         cdev, adev, h->st, &je, split_a, split_b, vidx)) {
    CUDA_TRY(h, je);
    h->stats.jit_launches++;
    h->stats.kernel_launches++;
    return SV_OK;
  } else if (vidx != -1) {  // no generated kernel after all: write the basis state, then run normally
    if (int rc = materialize_at(h, vidx)) return rc;
    return launch_one(h, L, split_a, split_b, -1);
  } else {
    CUDA_TRY(h, launch_section(h->dbl, h->sv, pdev, L.int_count, cdev, L.coef_count, adev, L.T, L.n_out, L.n_phases,
                               L.flags, L.n_sets, h->st, split_a, split_b));
    h->stats.interp_launches++;
  }
  h->stats.kernel_launches++;
  return SV_OK;
}

int drain_timing(sv_state* h) {
  if (h->trecs.empty()) return SV_OK;
  CUDA_TRY(h, cudaEventSynchronize(h->trecs.back().b));
  static const bool dbg = std::getenv("SV_DEBUG_TIMING") != nullptr;  // per-launch times (analysis aid)
  for (auto& r : h->trecs) {
    float ms = 0.f;
    CUDA_TRY(h, cudaEventElapsedTime(&ms, r.a, r.b));
    if (dbg) std::fprintf(stderr, "[sv] rank %d kind %d %.3f ms\n", h->rank, r.kind, ms);
    if (r.kind == 0 || r.kind == 3) {
      h->stats.timed_sections++;
      h->stats.section_ms += ms;
      h->stats.section_bytes += r.bytes;
      h->stats.section_flops += r.flops;
      if (r.kind == 3) {
        h->stats.timed_input_sections++;
        h->stats.input_section_ms += ms;
        h->stats.input_section_bytes += r.bytes;
        h->stats.input_section_flops += r.flops;
      }
    } else if (r.kind == 1) {
      h->stats.exchange_ms += ms;
    } else {
      h->stats.gate_ms += ms;
    }
    h->ev_pool.push_back(r.a);
    h->ev_pool.push_back(r.b);
  }
  h->trecs.clear();
  return SV_OK;
}

// physical swap of memory bits m1 <-> m2 (both local), one pass over half of the shard
int swap_step(sv_state* h, int m1, int m2) {
  GateArgs a{};
  a.type = 7;
  a.q0 = m1;
  a.q1 = m2;
  CUDA_TRY(h, launch_gate(h->dbl, h->sv, h->nL, a, h->st));
  h->stats.kernel_launches++;
  return SV_OK;
}

int check_handle(sv_state* h) {
  if (!h) return fail(nullptr, SV_EINVAL, "null handle");
  CUDA_TRY(h, cudaSetDevice(h->device));
  return SV_OK;
}

// Memory index of logical basis index k under the layout (pi, sigma).
uint64_t basis_memory_index(const sv_state* h, uint64_t k, const std::vector<int>& sigma) {
  uint64_t x = 0;
  for (int q = 0; q < h->n; q++) x |= ((k >> q) & 1ull) << sigma[h->pi[q]];
  return x;
}

// Write the pending basis state |basis_index> (sv_reset defers it) at its memory index under sigma.
int materialize(sv_state* h, const std::vector<int>& sigma) {
  if (!h->virt) return SV_OK;
  const uint64_t x = basis_memory_index(h, h->basis_index, sigma);
  const int64_t off = (int)(x >> h->nL) == h->rank ? (int64_t)(x & ((1ull << h->nL) - 1)) : -1;
  CUDA_TRY(h, launch_set_basis(h->dbl, h->sv, h->nL, off, h->st));
  h->stats.kernel_launches += off >= 0 ? 1 : 0;
  h->virt = false;
  return SV_OK;
}

int materialize_at(sv_state* h, int64_t vidx) {  // shard offset (or -2: the amplitude is elsewhere)
  CUDA_TRY(h, launch_set_basis(h->dbl, h->sv, h->nL, vidx >= 0 ? vidx : -1, h->st));
  h->stats.kernel_launches += vidx >= 0 ? 1 : 0;
  h->virt = false;
  return SV_OK;
}

int ready(sv_state* h) {  // a call that reads the state: valid handle, state written
  if (int rc = check_handle(h)) return rc;
  return materialize(h, h->sigma);
}

// Sum `count` values of dtype over all ranks in place (device buffer).
int allreduce(sv_state* h, void* buf, size_t count, CommType type) {
  if (h->world == 1) return SV_OK;
  COMM_TRY(h, h->comm->allreduce_sum(buf, count, type, h->st));
  return SV_OK;
}

// Map every rank's buffer `mine` (allocation base_alloc + base_off) into this process: CUDA IPC
// handles all-gathered over the communicator (NCCL worlds), plain pointers (local worlds).
// *ok: every rank mapped every peer (agreed across ranks).
int share_buffer(sv_state* h, void* mine_ptr, void* base_alloc, size_t base_off, std::vector<void*>& out,
                 std::vector<void*>& opened, bool* ok_all) {
  out.assign(h->world, nullptr);
  if (h->comm->local()) {  // one process, one device: the other ranks' buffers are plain pointers
    COMM_TRY(h, h->comm->share_pointers(mine_ptr, out.data()));
    *ok_all = true;
    return SV_OK;
  }
  struct Rec {
    cudaIpcMemHandle_t hd;
    uint64_t off;
    int32_t ok;
    char pad[128 - sizeof(cudaIpcMemHandle_t) - 12];
  };
  static_assert(sizeof(Rec) == 128, "rec size");
  Rec mine{};
  mine.ok = cudaIpcGetMemHandle(&mine.hd, base_alloc) == cudaSuccess ? 1 : 0;
  cudaGetLastError();
  mine.off = base_off;
  if (int rc = ensure_dev(h, h->d_tmp, sizeof(Rec) * (h->world + 1))) return rc;
  CUDA_TRY(h, cudaMemcpyAsync((char*)h->d_tmp.p + sizeof(Rec) * h->world, &mine, sizeof(Rec), cudaMemcpyHostToDevice, h->st));
  COMM_TRY(h, h->comm->allgather((char*)h->d_tmp.p + sizeof(Rec) * h->world, h->d_tmp.p, sizeof(Rec), h->st));
  std::vector<Rec> all(h->world);
  CUDA_TRY(h, cudaMemcpyAsync(all.data(), h->d_tmp.p, sizeof(Rec) * h->world, cudaMemcpyDeviceToHost, h->st));
  if (int rc_ = sync_stream(h)) return rc_;
  int ok = 1;
  for (auto& r : all) ok &= r.ok;
  out[h->rank] = mine_ptr;
  for (int r = 0; ok && r < h->world; r++) {
    if (r == h->rank) continue;
    void* p = nullptr;
    if (cudaIpcOpenMemHandle(&p, all[r].hd, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      ok = 0;
      break;
    }
    opened.push_back(p);
    out[r] = (char*)p + all[r].off;
  }
  // agree across ranks
  float f = ok ? 0.f : 1.f;
  CUDA_TRY(h, cudaMemcpyAsync(h->d_small.p, &f, sizeof(float), cudaMemcpyHostToDevice, h->st));
  if (int rc = allreduce(h, h->d_small.p, 1, kF32)) return rc;
  CUDA_TRY(h, cudaMemcpyAsync(&f, h->d_small.p, sizeof(float), cudaMemcpyDeviceToHost, h->st));
  if (int rc_ = sync_stream(h)) return rc_;
  CUDA_TRY(h, cudaMemsetAsync(h->d_small.p, 0, 16, h->st));
  *ok_all = (f == 0.f);
  return SV_OK;
}

int setup_p2p(sv_state* h, void* base_alloc, size_t base_off) {
  bool ok = false;
  if (int rc = share_buffer(h, h->sv, base_alloc, base_off, h->peers, h->ipc_opened, &ok)) return rc;
  h->p2p = ok;
  return SV_OK;
}

// ------------------------------------------------------------------------ cross-GPU exchange
// The exchange of k local memory bits m_i with rank bits b_i (one grouped step, §8(e); the paper's
// chunk_swap across processes, pipelined through buffers as in its Fig. 5).
// In every XOR round t of the subcube, this rank's block mu = mine ^ t (elements whose m-bits equal
// mu) is replaced by the partner's block `mine`, element j of one block pairing with element j of
// the other (j: compact index over the remaining local bits).  Blocks are strided whenever an m-bit
// is low, so they travel packed:
//   peer path (CUDA IPC / local world): the copy engines move each piece into the partner's
//     receive slot over NVLink — as strided 2-D copies straight from the state when the block's
//     runs are >= SV_XRUN bytes, else after a small-grid kernel packed it into a local send slot
//     (SV_XCE=0: that kernel stores into the peer's slot itself) — then the copy engines (runs >=
//     SV_XRUN bytes) or an unpack kernel scatter the slot into place;
//   NCCL path (SV_EXCHANGE_NCCL, the comparator of P:420's send/recv): pack into a local send slot,
//     grouped ncclSend / ncclRecv, unpack.
// Pieces alternate between two slots: the transport of piece q (stream st_x) overlaps the unpack of
// piece q - 1 (stream st_u); one stream-ordered barrier per piece (peer path) certifies that piece
// q has landed everywhere and that piece q - 1 is unpacked everywhere, which frees its slot for
// piece q + 1 (a barrier at the start orders the first push after the previous exchange's
// unpacks).  With the next section's first launch
// L0 (pipelined exchange + section) the pieces are grouped by up to two of its out-of-tile bits and
// each quarter of its tiles starts on the compute stream as soon as that quarter has landed, while
// the next quarter is still on NVLink.
// Exchange tuning (measured: docs DESIGN §7): 132 CTAs for the pack / push / unpack kernels (264 or
// 528 no faster alone, slower overlapped), receive slots of 1 GiB (4 GiB no faster).  SV_XPIPE=0
// runs the exchange without overlapping its neighbouring sections (a comparator line).
constexpr unsigned kXGrid = 132;
// most section launches run quarter by quarter on either side of an exchange (SV_XCHAIN overrides).
// Longer chains measured no faster (QV33 on 2 GPUs 942 / 940 / 940 ms at 1 / 4 / 16;
// the FP64-bound sections are power-capped, the HBM-bound ones share HBM with the copies).
size_t x_chain() {
  const char* e = std::getenv("SV_XCHAIN");
  return e ? std::strtoull(e, nullptr, 10) : 1;
}
constexpr uint64_t kXSlotBytes = 1ull << 30;
unsigned x_grid() { return kXGrid; }
uint64_t x_slot_bytes() { return kXSlotBytes; }
// SV_XCE=0: the peer path pushes with a small-grid kernel (remote stores) instead of packing into a
// local send slot and copying it to the peer with the copy engines (default)
bool x_ce() {
  static const bool on = [] {
    const char* e = std::getenv("SV_XCE");
    return !(e && e[0] == '0');
  }();
  return on;
}
// Copy engines for both ends of a piece when the exchanged block's contiguous runs are at least
// SV_XRUN bytes (default 1024; 0 disables): the rows go straight from the state into the peer's
// slot (no pack kernel, no send slot) and from the slot into place (no unpack kernel; SV_XCEU=0
// keeps the unpack kernel).  Measured: QFT34 on 2 GPUs 317.9 -> 286.0 ms per step.
uint64_t x_run_bytes() {
  const char* e = std::getenv("SV_XRUN");
  return e ? std::strtoull(e, nullptr, 10) : 1024;
}
bool x_ce_unpack() {
  const char* e = std::getenv("SV_XCEU");
  return !(e && e[0] == '0');
}
// In-place form (SV_XINPLACE=1, opt-in): with copy engines at both ends, one rank of each pair
// receives in place — its partner writes straight into its state once its own piece has left — so
// only the other rank unpacks (the roles alternate between groups of pieces); three receive slots.
// It halves the unpack traffic but serialises each in-place copy behind its piece's barrier:
// measured within +-2% of the default (QV33 faster on one box, QFT weak and QV28 slower).
bool x_inplace() {
  const char* e = std::getenv("SV_XINPLACE");
  return e && e[0] == '1';
}
bool x_pipe() {
  static const bool on = [] {
    const char* e = std::getenv("SV_XPIPE");
    return !(e && e[0] == '0');
  }();
  return on;
}

int ensure_exchange_engine(sv_state* h, uint64_t slot_amps, bool nccl_path) {
  if (!h->st_x) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    CUDA_TRY(h, cudaStreamCreateWithPriority(&h->st_x, cudaStreamNonBlocking, hi));
    CUDA_TRY(h, cudaStreamCreateWithPriority(&h->st_u, cudaStreamNonBlocking, hi));
    CUDA_TRY(h, cudaStreamCreateWithPriority(&h->st_p, cudaStreamNonBlocking, hi));
    for (cudaEvent_t* e : {&h->ev_start, &h->ev_done, &h->ev_pushed[0], &h->ev_pushed[1], &h->ev_pushed[2],
                           &h->ev_unpacked[0], &h->ev_unpacked[1], &h->ev_unpacked[2], &h->ev_landed[0], &h->ev_landed[1], &h->ev_landed[2], &h->ev_landed[3],
                           &h->ev_packed[0], &h->ev_packed[1], &h->ev_prev[0], &h->ev_prev[1], &h->ev_prev[2],
                           &h->ev_prev[3]})
      CUDA_TRY(h, cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  }
  if (h->xslot < slot_amps) {  // collective: every rank grows its slots at the same exchange
    for (void* p : h->xrecv_opened) cudaIpcCloseMemHandle(p);
    h->xrecv_opened.clear();
    h->xrecv_shared = false;
    if (int rc = ensure_dev(h, h->d_xrecv, 3 * slot_amps * h->amp)) return rc;  // 3 for the in-place form
    h->xslot = slot_amps;
  }
  if (nccl_path || x_ce())
    if (int rc = ensure_dev(h, h->d_xsend, 2 * h->xslot * h->amp)) return rc;
  if (nccl_path) return SV_OK;
  if (!h->xrecv_shared) {
    bool ok = false;
    if (int rc = share_buffer(h, h->d_xrecv.p, h->d_xrecv.p, 0, h->peer_xrecv, h->xrecv_opened, &ok)) return rc;
    if (!ok) return fail(h, SV_ECUDA, "exchange slots could not be mapped by every peer");
    h->xrecv_shared = true;
  }
  return SV_OK;
}

int exchange(sv_state* h, std::vector<ExPair> pairs, uint32_t flags, const XPipe& xp) {
  Nvtx r("sv exchange k=%zu pre=%zu post=%zu", pairs.size(), xp.pre.size(), xp.post.size());
  std::sort(pairs.begin(), pairs.end(), [](const ExPair& a, const ExPair& b) { return a.m < b.m; });
  const int k = (int)pairs.size();
  if (k < 1 || k > 8) return fail(h, SV_EINVAL, "internal: exchange of 1..8 bits expected");
  int m[8], bsel[8], mine = 0;
  for (int i = 0; i < k; i++) {
    m[i] = pairs[i].m;
    bsel[i] = pairs[i].b - h->nL;
    mine |= ((h->rank >> bsel[i]) & 1) << i;
  }
  const bool nccl_path = (flags & SV_EXCHANGE_NCCL) || !h->p2p;
  const int ns = xp.ns;
  const int* sbit = xp.sbit;
  const int P = 1 << ns;
  const uint64_t qblock = 1ull << (h->nL - k - ns);  // elements per (quarter, partner)
  const uint64_t slot = std::min<uint64_t>(qblock, std::max<uint64_t>(1, x_slot_bytes() / h->amp));
  if (int rc = ensure_exchange_engine(h, slot, nccl_path)) return rc;
  h->stats.bytes_sent += (uint64_t)((1ull << k) - 1) * (1ull << (h->nL - k)) * h->amp;
  h->stats.exchanges += k;
  h->stats.exchange_batches++;
  // quarter p of a chain launch: the split bits fixed to p's bits (tile-expansion specs in the
  // launch's ascending out-bit order)
  auto run_quarter = [&](size_t li, int p) -> int {
    const Launch& L = h->prog.launches[li];
    const SvSecHeader* H = reinterpret_cast<const SvSecHeader*>(h->prog.ints.data() + L.int_off);
    int js[2] = {0, 0}, vs[2] = {0, 0}, sp[2] = {0, 0};
    for (int i = 0; i < ns; i++) {
      for (int j = 0; j < H->n_out; j++)
        if (H->out_bits[j] == sbit[i]) js[i] = j;
      vs[i] = (p >> i) & 1;
    }
    if (ns == 2 && js[0] > js[1]) std::swap(js[0], js[1]), std::swap(vs[0], vs[1]);
    for (int i = 0; i < ns; i++) sp[i] = (1 << 16) | (vs[i] << 8) | js[i];
    const double amps = (double)(1ull << h->nL) / P;
    cudaEvent_t ts = tstart(h);
    if (int rc = launch_one(h, L, sp[0], sp[1])) return rc;
    tend(h, ts, 0, 2.0 * amps * (double)h->amp, L.flops_per_amp * amps);
    return SV_OK;
  };

  // the exchange streams start after everything queued so far on the compute stream; the chain
  // before it (xp.pre) then runs quarter by quarter there, the exchange of quarter p starting as
  // soon as the chain has written quarter p
  CUDA_TRY(h, cudaEventRecord(h->ev_start, h->st));
  CUDA_TRY(h, cudaStreamWaitEvent(h->st_x, h->ev_start, 0));
  CUDA_TRY(h, cudaStreamWaitEvent(h->st_u, h->ev_start, 0));
  CUDA_TRY(h, cudaStreamWaitEvent(h->st_p, h->ev_start, 0));
  const bool pre = !xp.pre.empty();
  if (pre) {
    for (int p = 0; p < P; p++) {
      for (size_t li : xp.pre)
        if (int rc = run_quarter(li, p)) return rc;
      CUDA_TRY(h, cudaEventRecord(h->ev_prev[p], h->st));
    }
  }
  const bool ce = !nccl_path && x_ce();
  int lo = m[0];
  for (int i = 0; i < ns; i++) lo = std::min(lo, sbit[i]);
  const uint64_t xrun = x_run_bytes();
  const bool direct = ce && xrun > 0 && (1ull << lo) * h->amp >= xrun;  // gather by copy engine
  const uint64_t min_run = direct ? (xrun + h->amp - 1) / h->amp : 0;
  const bool ce_unpack = !nccl_path && x_ce_unpack();
  cudaEvent_t t0 = nullptr;  // recorded where the first piece starts (after quarter 0 of Lp)
  char* recv = (char*)h->d_xrecv.p;
  char* send = (char*)h->d_xsend.p;
  // every rank is done with everything before this exchange — its unpacks of the previous one
  // included — before any push lands in a peer's slot
  if (!nccl_path)
    if (int rc = barrier(h, h->st_x)) return rc;
  int pos[11], val[11], pval[11];
  bool inplace = direct && ce_unpack && x_inplace();
  if (inplace) {  // every piece has the row shape the copy engines take (checked on piece 0)
    int np = 0, zero[11] = {};
    for (int i = 0; i < k; i++) pos[np++] = m[i];
    for (int i = 0; i < ns; i++) pos[np++] = sbit[i];
    int nc = 0;
    inplace = copy_bits_ce_xx(h->sv, zero, h->sv, zero, 0, std::min(slot, qblock), np, pos, h->amp, min_run, h->st_x,
                              &nc, true) == cudaSuccess;
  }
  const bool single_group = P * ((1 << k) - 1) == 1;
  uint64_t q = 0;
  for (int p = 0; p < P; p++) {
    if (pre) {  // quarter p of the chain before is written before it is packed / sent
      CUDA_TRY(h, cudaStreamWaitEvent(h->st_p, h->ev_prev[p], 0));
      CUDA_TRY(h, cudaStreamWaitEvent(h->st_x, h->ev_prev[p], 0));
    }
    if (h->timing && p == 0) {  // the exchange's span: from its first piece to its last unpack
      t0 = ev_get(h);
      CUDA_TRY(h, cudaEventRecord(t0, ce && !direct ? h->st_p : h->st_x));
    }
    for (int t = 1; t < (1 << k); t++) {  // XOR schedule: every round is a perfect matching of ranks
      const int mu = mine ^ t;
      int partner = h->rank;
      for (int i = 0; i < k; i++) partner = (partner & ~(1 << bsel[i])) | (((mu >> i) & 1) << bsel[i]);
      int nins = 0;
      for (int i = 0; i < k; i++) {
        pos[nins] = m[i];
        pval[nins] = (mine >> i) & 1;  // the partner's block that mine replaces (in-place form)
        val[nins++] = (mu >> i) & 1;
      }
      for (int i = 0; i < ns; i++) {
        pos[nins] = sbit[i];
        pval[nins] = (p >> i) & 1;
        val[nins++] = (p >> i) & 1;
      }
      for (uint64_t off = 0; off < qblock; off += slot, q++) {
        const uint64_t cnt = std::min<uint64_t>(slot, qblock - off);
        const int b = (int)(q & 1);
        if (inplace) {
          // Roles per group of pieces (alternating, so each rank unpacks about half): the stager
          // copies its rows into the partner's slot before the piece's barrier; after it (the
          // stager's rows have left) the partner copies its rows straight into the stager's state
          // and then unpacks its slot.  Slot q % 3 is free: its previous unpack (piece q - 3) was
          // waited for before the previous barrier.
          const bool lower = h->rank < partner;
          const bool stager = lower ^ (single_group ? off >= qblock / 2 : (((p * ((1 << k) - 1)) + t - 1) & 1) != 0);
          const int b3 = (int)(q % 3);
          int nc = 0;
          if (stager) {
            char* dst = (char*)h->peer_xrecv[partner] + (size_t)b3 * slot * h->amp;
            CUDA_TRY(h, copy_bits_ce(true, h->sv, dst, off, cnt, nins, pos, val, h->amp, min_run, h->st_x, &nc));
          }
          if (q >= 2) CUDA_TRY(h, cudaStreamWaitEvent(h->st_x, h->ev_unpacked[(q - 2) % 3], 0));
          if (int rc = barrier(h, h->st_x)) return rc;
          if (!stager) {
            CUDA_TRY(h, copy_bits_ce_xx(h->sv, val, h->peers[partner], pval, off, cnt, nins, pos, h->amp, min_run,
                                        h->st_x, &nc, false));
            CUDA_TRY(h, cudaEventRecord(h->ev_pushed[b3], h->st_x));
            CUDA_TRY(h, cudaStreamWaitEvent(h->st_u, h->ev_pushed[b3], 0));
            CUDA_TRY(h, copy_bits_ce(false, h->sv, recv + (size_t)b3 * slot * h->amp, off, cnt, nins, pos, val, h->amp,
                                     min_run, h->st_u, &nc));
            CUDA_TRY(h, cudaEventRecord(h->ev_unpacked[b3], h->st_u));
          }
          continue;
        }
        if (nccl_path) {
          if (q >= 2) CUDA_TRY(h, cudaStreamWaitEvent(h->st_x, h->ev_unpacked[b], 0));  // my slot b is free
          char* sb = send + (size_t)b * slot * h->amp;
          CUDA_TRY(h, launch_pack_bits(h->dbl, true, h->sv, sb, off, cnt, nins, pos, val, 1ull << h->nL, h->st_x, x_grid()));
          COMM_TRY(h, h->comm->group_start());
          COMM_TRY(h, h->comm->send(sb, cnt * h->amp, partner, h->st_x));
          COMM_TRY(h, h->comm->recv(recv + (size_t)b * slot * h->amp, cnt * h->amp, partner, h->st_x));
          COMM_TRY(h, h->comm->group_end());
        } else {
          // One barrier per piece: after it every push of piece q has landed AND every rank's
          // unpack of piece q - 1 is done (each rank's exchange stream waited for its own first),
          // so piece q + 1 may be pushed into the slot piece q - 1 used.
          char* dst = (char*)h->peer_xrecv[partner] + (size_t)b * slot * h->amp;
          int nc = 0;
          cudaError_t de = cudaErrorNotSupported;
          if (direct)  // rows of the block straight from the state into the peer's slot
            de = copy_bits_ce(true, h->sv, dst, off, cnt, nins, pos, val, h->amp, min_run, h->st_x, &nc);
          if (de != cudaErrorNotSupported) {
            CUDA_TRY(h, de);
            h->stats.kernel_launches -= 1;  // no pack kernel for this piece
          } else if (ce) {  // pack on its own stream, copy engine over NVLink: no SM holds the transfer
            char* sb = send + (size_t)b * slot * h->amp;
            if (q >= 2) CUDA_TRY(h, cudaStreamWaitEvent(h->st_p, h->ev_pushed[b], 0));  // send slot b copied
            CUDA_TRY(h, launch_pack_bits(h->dbl, true, h->sv, sb, off, cnt, nins, pos, val, 1ull << h->nL, h->st_p, x_grid()));
            CUDA_TRY(h, cudaEventRecord(h->ev_packed[b], h->st_p));
            CUDA_TRY(h, cudaStreamWaitEvent(h->st_x, h->ev_packed[b], 0));
            CUDA_TRY(h, cudaMemcpyAsync(dst, sb, cnt * h->amp, cudaMemcpyDeviceToDevice, h->st_x));
          } else {
            CUDA_TRY(h, launch_pack_bits(h->dbl, true, h->sv, dst, off, cnt, nins, pos, val, 1ull << h->nL, h->st_x, x_grid()));
          }
          if (q >= 1) CUDA_TRY(h, cudaStreamWaitEvent(h->st_x, h->ev_unpacked[b ^ 1], 0));
          if (int rc = barrier(h, h->st_x)) return rc;
        }
        h->stats.kernel_launches += 2;
        CUDA_TRY(h, cudaEventRecord(h->ev_pushed[b], h->st_x));
        CUDA_TRY(h, cudaStreamWaitEvent(h->st_u, h->ev_pushed[b], 0));
        {
          int nc = 0;
          cudaError_t ue = cudaErrorNotSupported;
          if (ce_unpack)
            ue = copy_bits_ce(false, h->sv, recv + (size_t)b * slot * h->amp, off, cnt, nins, pos, val, h->amp,
                              (std::max<uint64_t>(xrun, 1024) + h->amp - 1) / h->amp, h->st_u, &nc);
          if (ue != cudaErrorNotSupported) {
            CUDA_TRY(h, ue);
            h->stats.kernel_launches -= 1;
          } else {
            CUDA_TRY(h, launch_pack_bits(h->dbl, false, h->sv, recv + (size_t)b * slot * h->amp, off, cnt, nins, pos, val,
                                         1ull << h->nL, h->st_u, x_grid()));
          }
        }
        CUDA_TRY(h, cudaEventRecord(h->ev_unpacked[b], h->st_u));
      }
    }
    if (inplace) {  // the partners' in-place copies of quarter p have landed after one more barrier
      if (int rc = barrier(h, h->st_x)) return rc;
      CUDA_TRY(h, cudaEventRecord(h->ev_done, h->st_x));
      CUDA_TRY(h, cudaStreamWaitEvent(h->st_u, h->ev_done, 0));
    }
    if (!xp.post.empty()) {  // quarter p of the chain after: its tiles have every exchanged element now
      CUDA_TRY(h, cudaEventRecord(h->ev_landed[p], h->st_u));
      CUDA_TRY(h, cudaStreamWaitEvent(h->st, h->ev_landed[p], 0));
      for (size_t li : xp.post)
        if (int rc = run_quarter(li, p)) return rc;
    }
  }
  if (h->timing) {
    cudaEvent_t t1 = ev_get(h);
    CUDA_TRY(h, cudaEventRecord(t1, h->st_u));
    h->trecs.push_back({t0, t1, 1, 0.0, 0.0});
  }
  // the compute stream continues after both exchange streams
  CUDA_TRY(h, cudaEventRecord(h->ev_done, h->st_u));
  CUDA_TRY(h, cudaStreamWaitEvent(h->st, h->ev_done, 0));
  CUDA_TRY(h, cudaEventRecord(h->ev_done, h->st_x));
  CUDA_TRY(h, cudaStreamWaitEvent(h->st, h->ev_done, 0));
  h->stats.sections += xp.pre.size() + xp.post.size();
  return SV_OK;
}

}  // namespace

// ====================================================================== ABI
extern "C" {

int sv_abi_version(void) { return 3; }

const char* sv_last_error(sv_handle h) { return h ? h->err.c_str() : g_last_error.c_str(); }

void sv_free(void* p) { std::free(p); }

int sv_nccl_unique_id(void* out128) {
  if (!out128) return fail(nullptr, SV_EINVAL, "null output");
  std::string e;
  Nccl* n = nccl(e);
  if (!n) return fail(nullptr, SV_ENCCL, e);
  int r = n->GetUniqueId(out128);
  if (r != 0) return fail(nullptr, SV_ENCCL, n->GetErrorString(r));
  return SV_OK;
}

int sv_create(int n_qubits, int chunk_bits, sv_precision prec, sv_handle* out) {
  return sv_create_dist(n_qubits, chunk_bits, prec, 0, 1, nullptr, nullptr, 0, nullptr, out);
}

namespace {
// Shared by sv_create_dist (NCCL world, one process per GPU) and sv_create_local (in-process world
// on one device): `local` non-null selects the latter.
int create_common(int n_qubits, int chunk_bits, sv_precision prec, int rank, int world, const void* uid,
                  LocalWorld* local, void* ext_dev_buf, size_t ext_bytes, void* cuda_stream, sv_handle* out) {
  if (!out) return fail(nullptr, SV_EINVAL, "null output handle");
  *out = nullptr;
  if (world < 1 || (world & (world - 1))) return fail(nullptr, SV_EINVAL, "world must be a power of two");
  if (rank < 0 || rank >= world) return fail(nullptr, SV_EINVAL, "rank out of range");
  if (prec != SV_FP32 && prec != SV_FP64) return fail(nullptr, SV_EINVAL, "bad precision");
  const int g = __builtin_ctz((unsigned)world);
  if (n_qubits < 1 || n_qubits > 40) return fail(nullptr, SV_EINVAL, "n_qubits must be in [1, 40]");
  if (n_qubits - g < 1) return fail(nullptr, SV_EINVAL, "more GPUs than amplitudes");
  if (chunk_bits < 1 || chunk_bits > n_qubits - g)
    return fail(nullptr, SV_EINVAL, "chunk_bits must satisfy 1 <= c <= n - log2(world)");
  if (world > 1 && !uid && !local) return fail(nullptr, SV_EINVAL, "world > 1 needs an NCCL unique id");

  auto* h = new sv_state();
  h->n = n_qubits;
  h->c = chunk_bits;
  h->g = g;
  h->nL = n_qubits - g;
  h->rank = rank;
  h->world = world;
  h->dbl = prec == SV_FP64;
  h->amp = h->dbl ? 16 : 8;
  h->pi.resize(h->n);
  h->sigma.resize(h->n);
  std::iota(h->pi.begin(), h->pi.end(), 0);
  std::iota(h->sigma.begin(), h->sigma.end(), 0);
  auto bail = [&](int rc) {
    sv_destroy(h);
    return rc;
  };
  cudaError_t e = cudaGetDevice(&h->device);
  if (e != cudaSuccess) return bail(fail(nullptr, SV_ECUDA, std::string("no CUDA device: ") + cudaGetErrorString(e)));
  const size_t bytes = h->amp << h->nL;
  if (ext_dev_buf) {
    if (ext_bytes < bytes) return bail(fail(nullptr, SV_ECAPACITY, "ext_dev_buf smaller than the shard"));
    h->sv = ext_dev_buf;
  } else {
    e = cudaMalloc(&h->sv, bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      h->sv = nullptr;
      return bail(fail(nullptr, SV_ECAPACITY, "shard of " + std::to_string(bytes) + " bytes does not fit: " +
                                                  cudaGetErrorString(e)));
    }
    h->own_sv = true;
  }
  if (cuda_stream) {
    h->st = (cudaStream_t)cuda_stream;
  } else {
    if (cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking) != cudaSuccess)
      return bail(fail(nullptr, SV_ECUDA, "stream creation failed"));
    h->own_stream = true;
  }
  if (cudaEventCreateWithFlags(&h->ev_upload, cudaEventDisableTiming) != cudaSuccess)
    return bail(fail(nullptr, SV_ECUDA, "event creation failed"));
  if (int rc = ensure_dev(h, h->d_small, 4096)) return bail(fail(nullptr, rc, h->err));
  if (cudaMemsetAsync(h->d_small.p, 0, 4096, h->st) != cudaSuccess) return bail(fail(nullptr, SV_ECUDA, "memset"));
  if (world > 1) {
    std::string er;
    h->comm = local ? make_local_comm(local, rank, er) : make_nccl_comm(world, rank, uid, h->d_small.p, er);
    if (!h->comm) return bail(fail(nullptr, SV_ENCCL, er));
    // allocation base of the shard for CUDA IPC
    void* base = h->sv;
    size_t off = 0;
    if (!h->own_sv && !local) {
      typedef int (*GetRange)(unsigned long long*, size_t*, unsigned long long);
      void* lib = dlopen("libcuda.so.1", RTLD_NOW | RTLD_NOLOAD);
      GetRange fn = lib ? (GetRange)dlsym(lib, "cuMemGetAddressRange_v2") : nullptr;
      unsigned long long b = 0;
      size_t sz = 0;
      if (fn && fn(&b, &sz, (unsigned long long)h->sv) == 0) {
        base = (void*)b;
        off = (size_t)((char*)h->sv - (char*)base);
      }
    }
    if (int rc = setup_p2p(h, base, off)) return bail(fail(nullptr, rc, h->err));
  }
  if (int rc = sv_reset(h, 0)) return bail(rc);
  *out = h;
  return SV_OK;
}
}  // namespace

int sv_create_dist(int n_qubits, int chunk_bits, sv_precision prec, int rank, int world, const void* uid,
                   void* ext_dev_buf, size_t ext_bytes, void* cuda_stream, sv_handle* out) {
  return create_common(n_qubits, chunk_bits, prec, rank, world, uid, nullptr, ext_dev_buf, ext_bytes, cuda_stream, out);
}

int sv_world_create(int world, sv_world* out) {
  if (!out) return fail(nullptr, SV_EINVAL, "null output");
  *out = nullptr;
  if (world < 1 || world > 64 || (world & (world - 1))) return fail(nullptr, SV_EINVAL, "world must be a power of two <= 64");
  *out = reinterpret_cast<sv_world>(local_world_create(world));
  return SV_OK;
}

int sv_world_destroy(sv_world w) {
  local_world_release(reinterpret_cast<LocalWorld*>(w));
  return SV_OK;
}

int sv_create_local(int n_qubits, int chunk_bits, sv_precision prec, sv_world w, int rank, void* cuda_stream,
                    sv_handle* out) {
  if (!w) return fail(nullptr, SV_EINVAL, "null world");
  LocalWorld* lw = reinterpret_cast<LocalWorld*>(w);
  return create_common(n_qubits, chunk_bits, prec, rank, local_world_size(lw), nullptr, lw, nullptr, 0, cuda_stream,
                       out);
}

int sv_destroy(sv_handle h) {
  if (!h) return SV_OK;
  cudaSetDevice(h->device);
  if (h->st) cudaStreamSynchronize(h->st);
  for (void* p : h->ipc_opened) cudaIpcCloseMemHandle(p);
  delete h->comm;
  for (DevBuf* b : {&h->d_prog, &h->d_coef, &h->d_aux, &h->d_scratch, &h->d_small, &h->d_tmp, &h->d_tmp2, &h->d_stage})
    if (b->p) cudaFree(b->p);
  for (PinBuf* b : {&h->h_stage, &h->h_stage2})
    if (b->p) cudaFreeHost(b->p);
  if (h->own_sv && h->sv) cudaFree(h->sv);
  if (h->ev_upload) cudaEventDestroy(h->ev_upload);
  for (auto& r : h->trecs) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (cudaEvent_t e : h->ev_pool) cudaEventDestroy(e);
  for (void* p : h->xrecv_opened) cudaIpcCloseMemHandle(p);
  for (cudaEvent_t e : {h->ev_start, h->ev_done, h->ev_pushed[0], h->ev_pushed[1], h->ev_pushed[2], h->ev_unpacked[0],
                        h->ev_unpacked[1], h->ev_unpacked[2],
                        h->ev_landed[0], h->ev_landed[1], h->ev_landed[2], h->ev_landed[3], h->ev_packed[0],
                        h->ev_packed[1], h->ev_prev[0], h->ev_prev[1], h->ev_prev[2], h->ev_prev[3]})
    if (e) cudaEventDestroy(e);
  if (h->st_x) cudaStreamDestroy(h->st_x);
  if (h->st_u) cudaStreamDestroy(h->st_u);
  if (h->st_p) cudaStreamDestroy(h->st_p);
  for (DevBuf* b : {&h->d_xrecv, &h->d_xsend})
    if (b->p) cudaFree(b->p);
  if (h->own_stream && h->st) cudaStreamDestroy(h->st);
  cudaGetLastError();
  delete h;
  return SV_OK;
}

int sv_reset(sv_handle h, uint64_t k) {
  if (int rc = check_handle(h)) return rc;
  if (h->n < 64 && (k >> h->n)) return fail(h, SV_EINVAL, "basis index out of range");
  std::iota(h->pi.begin(), h->pi.end(), 0);
  std::iota(h->sigma.begin(), h->sigma.end(), 0);
  // Deferred: the next circuit's first section generates |k> in its load (no memset pass, no read
  // pass), or the first call that reads the state writes it (materialize).
  h->basis_pending = true;  // the next circuit may choose its memory layout freely (NEXT-2)
  h->basis_index = k;
  h->virt = true;
  return SV_OK;
}

int sv_synchronize(sv_handle h) {
  if (int rc = check_handle(h)) return rc;
  if (int rc_ = sync_stream(h)) return rc_;
  return SV_OK;
}

int sv_apply_circuit(sv_handle h, const sv_gate* gates, size_t n_gates, uint32_t flags) {
  if (int rc = check_handle(h)) return rc;
  Nvtx r("sv_apply_circuit n=%d gates=%zu rank=%d/%d", h->n, n_gates, h->rank, h->world);
  if (n_gates && !gates) return fail(h, SV_EINVAL, "null gate array");
  const double t0 = now_ms();
  std::vector<int> pi = h->pi, sigma = h->sigma;
  std::vector<Step> steps;
  PlanCounters ctr;
  PlanLayout lay;
  lay.low_bits = h->dbl ? 3 : 4;  // 128-byte runs
  apply_tile_prefs(lay);
  lay.free_initial = h->basis_pending && !(flags & SV_UNBLOCKED);
  std::vector<int> sigma0;
  Status s = make_plan(gates, n_gates, h->n, h->c, h->g, pi, sigma, flags, steps, ctr, lay, &sigma0);
  if (!s.good()) return fail(h, s);
  if (!lay.free_initial) sigma0 = h->sigma;
  if (!h->virt && lay.free_initial && sigma0 != h->sigma) {
    // relocate the single nonzero amplitude of |k> to its place under the chosen layout
    const uint64_t from = basis_memory_index(h, h->basis_index, h->sigma);
    const uint64_t to = basis_memory_index(h, h->basis_index, sigma0);
    const uint64_t lm = (1ull << h->nL) - 1;
    if ((int)(from >> h->nL) == h->rank) CUDA_TRY(h, launch_set_amp(h->dbl, h->sv, (int64_t)(from & lm), 0.0, h->st));
    if ((int)(to >> h->nL) == h->rank) CUDA_TRY(h, launch_set_amp(h->dbl, h->sv, (int64_t)(to & lm), 1.0, h->st));
    h->stats.kernel_launches += 2;
  }
  h->basis_pending = false;
  h->prog.clear();
  const int T_default = lay.tile_default;
  std::vector<size_t> launch_end(steps.size(), 0);  // one past the last launch of each step
  for (size_t i = 0; i < steps.size(); i++) {
    const Step& st = steps[i];
    if (st.type == Step::SECTION && h->nL >= SV_R_BITS) {
      const Status cs =
          compile_section_split(st.gates, h->nL, h->rank, h->g, T_default, lay.low_bits, st.swaps, h->prog);
      if (!cs.good()) return fail(h, cs);
      if (h->prog.launches.back().T > 13)
        return fail(h, SV_ECAPACITY, "a section needs a tile larger than shared memory (lower chunk_bits)");
    }
    launch_end[i] = h->prog.launches.size();
  }
  h->stats.pass_ms = now_ms() - t0;
  // A deferred basis state (sv_reset) is generated by the first section's load when the plan
  // starts with a section run by a generated kernel; else it is written now.
  int64_t vidx = -1;  // -1: read the state; >= 0 the shard offset of the one amplitude; -2 none here
  if (h->virt) {
    if (!steps.empty() && steps[0].type == Step::SECTION && !h->prog.launches.empty() &&
        jit_virtual_input_ok(h->prog.launches[0], h->dbl)) {
      const uint64_t x = basis_memory_index(h, h->basis_index, sigma0);
      vidx = (int)(x >> h->nL) == h->rank ? (int64_t)(x & ((1ull << h->nL) - 1)) : -2;
      h->virt = false;
    } else if (int rc = materialize(h, sigma0)) {
      return rc;
    }
  }
  jit_prepare(h->prog, h->dbl, vidx != -1);  // run-time specialised kernels (jit.h): compile what is missing
  if (int rc = upload_program(h)) return rc;
  // Pipeline plan (§8(e), the paper's overlap of exchange and computation): each
  // exchange takes up to two split bits — local memory bits it does not exchange that lie outside
  // the tile of the section launches next to it — and runs the launches on either side whose tiles
  // all avoid those bits quarter by quarter around itself: the chain before it writes quarter p,
  // quarter p travels, the chain after it computes on quarter p while quarter p + 1 travels.
  std::vector<XPipe> xps(steps.size());
  std::vector<char> by_exchange(h->prog.launches.size(), 0);
  if (x_pipe() && h->nL >= SV_R_BITS) {
    std::vector<size_t> launch_begin(steps.size());
    for (size_t i = 0; i < steps.size(); i++) launch_begin[i] = i ? launch_end[i - 1] : 0;
    auto hdr = [&](size_t li) { return reinterpret_cast<const SvSecHeader*>(h->prog.ints.data() + h->prog.launches[li].int_off); };
    auto out_has = [&](size_t li, int b) {
      if (h->prog.launches[li].T < SV_R_BITS) return false;
      const SvSecHeader* H = hdr(li);
      for (int j = 0; j < H->n_out; j++)
        if (H->out_bits[j] == b) return true;
      return false;
    };
    size_t claimed = vidx != -1 ? 1 : 0;  // launches before this index are taken (or the generated input)
    for (size_t i = 0; i < steps.size(); i++) {
      if (steps[i].type != Step::EXCHANGE || i + 1 >= steps.size() || steps[i + 1].type != Step::SECTION) continue;
      const size_t l0 = launch_begin[i + 1];
      if (l0 >= launch_end[i + 1] || h->prog.launches[l0].T < SV_R_BITS) continue;
      uint64_t mmask = 0;
      for (const ExPair& e : steps[i].ex) mmask |= 1ull << e.m;
      // the chain before: launches of the sections right before the exchange, not yet taken
      std::vector<size_t> cand_pre;
      for (size_t j = i; j-- > 0 && steps[j].type == Step::SECTION;)
        for (size_t li = launch_end[j]; li-- > launch_begin[j];) cand_pre.push_back(li);
      const bool has_lp = !cand_pre.empty() && cand_pre[0] >= claimed;
      XPipe& xp = xps[i];
      const SvSecHeader* H0 = hdr(l0);
      for (int with_lp = has_lp; with_lp >= 0 && xp.ns == 0; with_lp--)  // common bits first, else the chain after only
        for (int j = H0->n_out - 1; j >= 0 && xp.ns < 2; j--) {  // highest out bits of the first launch
          const int b = H0->out_bits[j];
          if ((mmask >> b) & 1) continue;
          if (with_lp && !out_has(cand_pre[0], b)) continue;
          xp.sbit[xp.ns++] = b;
        }
      if (h->nL - (int)steps[i].ex.size() - xp.ns < 0) xp.ns = 0;
      auto fits = [&](size_t li) {
        for (int q = 0; q < xp.ns; q++)
          if (!out_has(li, xp.sbit[q])) return false;
        return true;
      };
      if (xp.ns > 0) {
        for (size_t li : cand_pre) {
          if (li < claimed || xp.pre.size() >= x_chain() || !fits(li)) break;
          xp.pre.push_back(li);
        }
        std::reverse(xp.pre.begin(), xp.pre.end());
        for (size_t j = i + 1; j < steps.size() && steps[j].type == Step::SECTION && xp.post.size() < x_chain(); j++) {
          bool all = true;
          for (size_t li = launch_begin[j]; li < launch_end[j]; li++) {
            if (!fits(li) || xp.post.size() >= x_chain()) {
              all = false;
              break;
            }
            xp.post.push_back(li);
          }
          if (!all) break;
        }
      }
      for (size_t li : xp.pre) by_exchange[li] = 1;
      for (size_t li : xp.post) by_exchange[li] = 1;
      if (!xp.post.empty()) claimed = xp.post.back() + 1;
    }
  }
  size_t si = 0;
  for (size_t i = 0; i < steps.size(); i++) {
    const Step& st = steps[i];
    switch (st.type) {
      case Step::EXCHANGE: {
        if (int rc = exchange(h, st.ex, flags, xps[i])) return rc;
        break;
      }
      case Step::SECTION: {
        if (h->nL < SV_R_BITS) {  // shards of < 16 amplitudes: per-gate kernels (no tile to block)
          for (const sv_gate& gm : st.gates)
            if (int rc = gate_step(h, gm)) return rc;
          for (const auto& sw : st.swaps)
            if (int rc = swap_step(h, sw.first, sw.second)) return rc;
          break;
        }
        for (; si < launch_end[i]; si++) {
          const Launch& L = h->prog.launches[si];
          const bool gen_input = si == 0 && vidx != -1;  // the deferred basis state: a write-only pass
          if (by_exchange[si]) continue;  // run by the neighbouring exchange, quarter by quarter
          cudaEvent_t t = tstart(h);
          if (int rc = launch_one(h, L, 0, 0, si == 0 ? vidx : -1)) return rc;
          const double amps = (double)(1ull << h->nL);
          // a generated input: the shard is cleared (write-only bytes) and one tile computed
          const double fl = gen_input ? (vidx >= 0 ? L.flops_per_amp * (double)(1ull << L.T) : 0.0) : L.flops_per_amp * amps;
          tend(h, t, gen_input ? 3 : 0, (gen_input ? 1.0 : 2.0) * amps * (double)h->amp, fl);
          h->stats.sections++;
        }
        break;
      }
      case Step::GATE: {
        cudaEvent_t t = tstart(h);
        if (int rc = gate_step(h, st.gates[0])) return rc;
        tend(h, t, 2, 0.0, 0.0);
        break;
      }
      case Step::COMPACT: {  // standalone memory-bit swap passes that keep the next tile coalesced
        cudaEvent_t t = tstart(h);
        for (const auto& sw : st.swaps)
          if (int rc = swap_step(h, sw.first, sw.second)) return rc;
        tend(h, t, 2, 0.0, 0.0);
        h->stats.compactions += st.swaps.size();
        break;
      }
    }
  }
  h->pi = pi;
  h->sigma = sigma;
  h->stats.circuits++;
  h->stats.gates += n_gates;
  h->stats.chunk_swaps += ctr.chunk_swaps;
  h->stats.store_swaps += ctr.store_swaps;
  h->stats.apply_ms = now_ms() - t0;
  return SV_OK;
}

int sv_get_permutation(sv_handle h, int32_t* out) {
  if (!h || !out) return fail(h, SV_EINVAL, "null argument");
  for (int q = 0; q < h->n; q++) out[q] = h->pi[q];
  return SV_OK;
}

int sv_stats_get(sv_handle h, sv_stats_t* out) {
  if (!h || !out) return fail(h, SV_EINVAL, "null argument");
  if (int rc = drain_timing(h)) return rc;
  *out = h->stats;
  const JitCounters jc = jit_counters();
  out->jit_compiled = jc.compiled;
  out->jit_compile_ms = jc.compile_ms;
  return SV_OK;
}

int sv_stats(sv_handle h, sv_stats_t* out) { return sv_stats_get(h, out); }

int sv_stats_reset(sv_handle h) {
  if (!h) return fail(h, SV_EINVAL, "null handle");
  if (int rc = drain_timing(h)) return rc;
  h->stats = sv_stats_t{};
  return SV_OK;
}

int sv_set_timing(sv_handle h, int enable) {
  if (!h) return fail(h, SV_EINVAL, "null handle");
  h->timing = enable != 0;
  return SV_OK;
}

int sv_norm(sv_handle h, double* out) {
  if (int rc = ready(h)) return rc;
  Nvtx r("sv_norm");
  if (!out) return fail(h, SV_EINVAL, "null output");
  if (int rc = ensure_dev(h, h->d_scratch, norm_scratch_doubles() * sizeof(double))) return rc;
  CUDA_TRY(h, launch_norm(h->dbl, h->sv, h->nL, (double*)h->d_scratch.p, (double*)h->d_small.p + 8, h->st));
  h->stats.kernel_launches += 2;
  if (int rc = allreduce(h, (double*)h->d_small.p + 8, 1, kF64)) return rc;
  CUDA_TRY(h, cudaMemcpyAsync(out, (double*)h->d_small.p + 8, sizeof(double), cudaMemcpyDeviceToHost, h->st));
  if (int rc_ = sync_stream(h)) return rc_;
  return SV_OK;
}

int sv_probabilities(sv_handle h, const int32_t* qubits, int nq, double* host_out) {
  if (int rc = ready(h)) return rc;
  Nvtx r("sv_probabilities nq=%d", nq);
  if (nq < 0 || nq > 24 || (nq && (!qubits || !host_out))) return fail(h, SV_EINVAL, "bad qubit list (nq <= 24)");
  uint64_t seen = 0;
  std::vector<int> loc_bits, loc_pos;
  int rank_part = 0;
  for (int i = 0; i < nq; i++) {
    const int q = qubits[i];
    if (q < 0 || q >= h->n || ((seen >> q) & 1)) return fail(h, SV_EINVAL, "bad or duplicate qubit");
    seen |= 1ull << q;
    const int mb = h->sigma[h->pi[q]];
    if (mb < h->nL) {
      loc_bits.push_back(mb);
      loc_pos.push_back(i);
    } else {
      rank_part |= ((h->rank >> (mb - h->nL)) & 1) << i;
    }
  }
  const int nl = (int)loc_bits.size();
  const size_t bins_l = size_t(1) << nl, bins = size_t(1) << nq;
  if (int rc = ensure_dev(h, h->d_scratch, std::max(marginal_scratch_doubles(nl), norm_scratch_doubles()) * sizeof(double))) return rc;
  if (int rc = ensure_dev(h, h->d_tmp, bins * sizeof(double))) return rc;
  CUDA_TRY(h, launch_marginal(h->dbl, h->sv, h->nL, loc_bits.data(), nl, (double*)h->d_scratch.p, (double*)h->d_tmp.p, h->st));
  h->stats.kernel_launches += 2;
  if (h->world == 1) {
    CUDA_TRY(h, cudaMemcpyAsync(host_out, h->d_tmp.p, bins * sizeof(double), cudaMemcpyDeviceToHost, h->st));
    if (int rc_ = sync_stream(h)) return rc_;
    return SV_OK;
  }
  std::vector<double> loc(bins_l);
  CUDA_TRY(h, cudaMemcpyAsync(loc.data(), h->d_tmp.p, bins_l * sizeof(double), cudaMemcpyDeviceToHost, h->st));
  if (int rc_ = sync_stream(h)) return rc_;
  std::vector<double> full(bins, 0.0);
  for (size_t y = 0; y < bins_l; y++) {
    size_t o = rank_part;
    for (int j = 0; j < nl; j++) o |= ((y >> j) & 1) << loc_pos[j];
    full[o] = loc[y];
  }
  CUDA_TRY(h, cudaMemcpyAsync(h->d_tmp.p, full.data(), bins * sizeof(double), cudaMemcpyHostToDevice, h->st));
  if (int rc = allreduce(h, h->d_tmp.p, bins, kF64)) return rc;
  CUDA_TRY(h, cudaMemcpyAsync(host_out, h->d_tmp.p, bins * sizeof(double), cudaMemcpyDeviceToHost, h->st));
  if (int rc_ = sync_stream(h)) return rc_;
  return SV_OK;
}

int sv_get_amplitudes(sv_handle h, const uint64_t* idx, size_t cnt, void* host_out) {
  if (int rc = ready(h)) return rc;
  if (cnt == 0) return SV_OK;
  if (!idx || !host_out) return fail(h, SV_EINVAL, "null argument");
  const BitPerm mu = mu_of(h);
  const uint64_t lmask = (1ull << h->nL) - 1;
  const size_t chunk = 1 << 20;
  if (int rc = ensure_pin(h, h->h_stage2, chunk * sizeof(uint64_t))) return rc;
  if (int rc = ensure_dev(h, h->d_tmp, chunk * sizeof(uint64_t))) return rc;
  if (int rc = ensure_dev(h, h->d_tmp2, chunk * h->amp)) return rc;
  for (size_t b = 0; b < cnt; b += chunk) {
    const size_t m = std::min(chunk, cnt - b);
    if (int rc_ = sync_stream(h)) return rc_;  // staging reuse
    uint64_t* offs = (uint64_t*)h->h_stage2.p;
    for (size_t i = 0; i < m; i++) {
      const uint64_t x = idx[b + i];
      if (h->n < 64 && (x >> h->n)) return fail(h, SV_EINVAL, "amplitude index out of range");
      const uint64_t mem = mu(x);
      offs[i] = (int)(mem >> h->nL) == h->rank ? (mem & lmask) : ~0ull;
    }
    CUDA_TRY(h, cudaMemcpyAsync(h->d_tmp.p, offs, m * sizeof(uint64_t), cudaMemcpyHostToDevice, h->st));
    CUDA_TRY(h, launch_gather(h->dbl, h->sv, (const uint64_t*)h->d_tmp.p, m, h->d_tmp2.p, h->st));
    h->stats.kernel_launches++;
    if (int rc = allreduce(h, h->d_tmp2.p, 2 * m, h->dbl ? kF64 : kF32)) return rc;
    CUDA_TRY(h, cudaMemcpyAsync((char*)host_out + b * h->amp, h->d_tmp2.p, m * h->amp, cudaMemcpyDeviceToHost, h->st));
  }
  if (int rc_ = sync_stream(h)) return rc_;
  return SV_OK;
}

int sv_get_state(sv_handle h, void* host_out) {
  if (int rc = ready(h)) return rc;
  if (h->rank == 0 && !host_out) return fail(h, SV_EINVAL, "null output");
  const BitPerm inv = mu_inv_of(h);
  const size_t piece = std::min<size_t>(size_t(1) << h->nL, (size_t(256) << 20) / h->amp);
  const size_t shard = size_t(1) << h->nL;
  if (int rc = ensure_pin(h, h->h_stage2, piece * h->amp)) return rc;
  if (h->world > 1)
    if (int rc = ensure_dev(h, h->d_stage, piece * h->amp)) return rc;
  for (int src = 0; src < h->world; src++) {
    for (size_t off = 0; off < shard; off += piece) {
      const size_t cnt = std::min(piece, shard - off);
      const void* dev = (char*)h->sv + off * h->amp;
      if (src != 0) {
        if (h->rank == src) {
          COMM_TRY(h, h->comm->send(dev, cnt * h->amp, 0, h->st));
        } else if (h->rank == 0) {
          COMM_TRY(h, h->comm->recv(h->d_stage.p, cnt * h->amp, src, h->st));
          dev = h->d_stage.p;
        }
      }
      if (h->rank != 0) continue;
      CUDA_TRY(h, cudaMemcpyAsync(h->h_stage2.p, dev, cnt * h->amp, cudaMemcpyDeviceToHost, h->st));
      if (int rc_ = sync_stream(h)) return rc_;
      const uint64_t mbase = ((uint64_t)src << h->nL) + off;
      const char* in = (const char*)h->h_stage2.p;
      char* o = (char*)host_out;
      for (size_t i = 0; i < cnt; i++) std::memcpy(o + inv(mbase + i) * h->amp, in + i * h->amp, h->amp);
    }
  }
  if (int rc_ = sync_stream(h)) return rc_;
  return SV_OK;
}

static uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  uint64_t z = x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

int sv_sample(sv_handle h, size_t shots, uint64_t seed, uint64_t* host_out) {
  if (int rc = ready(h)) return rc;
  Nvtx r("sv_sample shots=%zu", shots);
  if (shots == 0) return SV_OK;
  if (!host_out) return fail(h, SV_EINVAL, "null output");
  const int B = std::min(12, h->nL);
  const size_t nblk = size_t(1) << (h->nL - B);
  if (int rc = ensure_dev(h, h->d_tmp, nblk * sizeof(double) + 64)) return rc;
  CUDA_TRY(h, launch_block_sums(h->dbl, h->sv, h->nL, B, (double*)h->d_tmp.p, h->st));
  h->stats.kernel_launches++;
  std::vector<double> bs(nblk);
  CUDA_TRY(h, cudaMemcpyAsync(bs.data(), h->d_tmp.p, nblk * sizeof(double), cudaMemcpyDeviceToHost, h->st));
  if (int rc_ = sync_stream(h)) return rc_;
  std::vector<double> cum(nblk);
  double tot = 0.0;
  for (size_t i = 0; i < nblk; i++) {
    tot += bs[i];
    cum[i] = tot;
  }
  std::vector<double> totals(h->world, 0.0);
  totals[h->rank] = tot;
  if (h->world > 1) {
    CUDA_TRY(h, cudaMemcpyAsync(h->d_tmp.p, totals.data(), h->world * sizeof(double), cudaMemcpyHostToDevice, h->st));
    if (int rc = allreduce(h, h->d_tmp.p, h->world, kF64)) return rc;
    CUDA_TRY(h, cudaMemcpyAsync(totals.data(), h->d_tmp.p, h->world * sizeof(double), cudaMemcpyDeviceToHost, h->st));
    if (int rc_ = sync_stream(h)) return rc_;
  }
  double before = 0.0;
  for (int r = 0; r < h->rank; r++) before += totals[r];
  const double mine_end = before + tot;
  // A u at or above the total mass (rounding) goes to the last nonzero outcome: the last block
  // with mass on the last rank that has mass (never a zero-probability index).
  int last_nz_rank = -1;
  for (int r = 0; r < h->world; r++)
    if (totals[r] > 0.0) last_nz_rank = r;
  const bool tail_here = h->rank == last_nz_rank;
  size_t tail_blk = 0;
  for (size_t i = 0; i < nblk; i++)
    if (bs[i] > 0.0) tail_blk = i;
  // u_s, sorted; this rank takes the shots in [before, mine_end) (and the tail, see above)
  std::vector<std::pair<double, size_t>> us(shots);
  for (size_t s = 0; s < shots; s++) us[s] = {(double)(splitmix64(seed ^ (uint64_t)s) >> 11) * 0x1.0p-53, s};
  std::sort(us.begin(), us.end());
  std::vector<int64_t> items;
  std::vector<double> resid;
  std::vector<size_t> who;
  size_t bi = 0;
  for (auto& pr : us) {
    const double u = pr.first;
    if (u < before || (u >= mine_end && !tail_here)) continue;
    double r = u - before, r2;
    if (u >= mine_end) {  // the tail: past every element of the last block with mass
      bi = std::max(bi, tail_blk);
      r2 = bs[bi];
    } else {
      while (bi + 1 < nblk && cum[bi] <= r) bi++;
      r2 = r - (bi ? cum[bi - 1] : 0.0);
    }
    if (!items.empty() && items[items.size() - 3] == (int64_t)bi) {
      items.back()++;
    } else {
      items.push_back((int64_t)bi);
      items.push_back((int64_t)resid.size());
      items.push_back(1);
    }
    resid.push_back(r2);
    who.push_back(pr.second);
  }
  std::vector<uint64_t> res(shots, 0);
  const size_t nit = items.size() / 3, nsh = resid.size();
  if (nsh) {
    if (int rc = ensure_dev(h, h->d_tmp2, items.size() * 8 + nsh * 8 + nsh * 8 + 64)) return rc;
    char* d = (char*)h->d_tmp2.p;
    int64_t* d_items = (int64_t*)d;
    double* d_res = (double*)(d + items.size() * 8);
    uint64_t* d_off = (uint64_t*)(d + items.size() * 8 + nsh * 8);
    CUDA_TRY(h, cudaMemcpyAsync(d_items, items.data(), items.size() * 8, cudaMemcpyHostToDevice, h->st));
    CUDA_TRY(h, cudaMemcpyAsync(d_res, resid.data(), nsh * 8, cudaMemcpyHostToDevice, h->st));
    CUDA_TRY(h, launch_sample_resolve(h->dbl, h->sv, B, d_items, (int)nit, d_res, d_off, h->st));
    h->stats.kernel_launches++;
    std::vector<uint64_t> offs(nsh);
    CUDA_TRY(h, cudaMemcpyAsync(offs.data(), d_off, nsh * 8, cudaMemcpyDeviceToHost, h->st));
    if (int rc_ = sync_stream(h)) return rc_;
    const BitPerm inv = mu_inv_of(h);
    for (size_t i = 0; i < nsh; i++) res[who[i]] = inv(((uint64_t)h->rank << h->nL) | offs[i]);
  }
  if (h->world > 1) {
    if (int rc = ensure_dev(h, h->d_tmp, shots * 8)) return rc;
    CUDA_TRY(h, cudaMemcpyAsync(h->d_tmp.p, res.data(), shots * 8, cudaMemcpyHostToDevice, h->st));
    if (int rc = allreduce(h, h->d_tmp.p, shots, kU64)) return rc;
    CUDA_TRY(h, cudaMemcpyAsync(res.data(), h->d_tmp.p, shots * 8, cudaMemcpyDeviceToHost, h->st));
    if (int rc_ = sync_stream(h)) return rc_;
  }
  std::memcpy(host_out, res.data(), shots * 8);
  return SV_OK;
}

int sv_block_circuit(const sv_gate* gates, size_t n_gates, int n, int c, const int32_t* pi0, uint32_t flags,
                     sv_gate** out, size_t* n_out, int32_t* pi_final) {
  if (!out || !n_out || (n_gates && !gates)) return fail(nullptr, SV_EINVAL, "null argument");
  std::vector<int> pi(n > 0 ? n : 0);
  if (n < 1 || n > 63) return fail(nullptr, SV_EINVAL, "n out of range");
  for (int q = 0; q < n; q++) pi[q] = pi0 ? pi0[q] : q;
  std::vector<sv_gate> tokens;
  Status s = block_pass(gates, n_gates, n, c, pi, flags, tokens);
  if (!s.good()) return fail(nullptr, s);
  sv_gate* buf = (sv_gate*)std::malloc(sizeof(sv_gate) * std::max<size_t>(tokens.size(), 1));
  if (!buf) return fail(nullptr, SV_ECAPACITY, "out of host memory");
  if (!tokens.empty()) std::memcpy(buf, tokens.data(), sizeof(sv_gate) * tokens.size());
  *out = buf;
  *n_out = tokens.size();
  if (pi_final)
    for (int q = 0; q < n; q++) pi_final[q] = pi[q];
  return SV_OK;
}

int sv_plan_circuit(const sv_gate* gates, size_t n_gates, int n, int c, int world_log2, const int32_t* pi0,
                    const int32_t* sigma0, uint32_t flags, sv_gate** out, size_t* n_out, int32_t* pi_final,
                    int32_t* sigma_final) {
  if (!out || !n_out || (n_gates && !gates)) return fail(nullptr, SV_EINVAL, "null argument");
  if (n < 1 || n > 63) return fail(nullptr, SV_EINVAL, "n out of range");
  std::vector<int> pi(n), sigma(n);
  for (int q = 0; q < n; q++) {
    pi[q] = pi0 ? pi0[q] : q;
    sigma[q] = sigma0 ? sigma0[q] : q;
  }
  std::vector<Step> steps;
  PlanCounters ctr;
  PlanLayout lay;
  apply_tile_prefs(lay);  // fp64 tile policy (as sv_apply_circuit on an fp64 state)
  lay.free_initial = (flags & SV_FREE_LAYOUT) && !(flags & SV_UNBLOCKED);
  Status s = make_plan(gates, n_gates, n, c, world_log2, pi, sigma, flags, steps, ctr, lay);
  if (!s.good()) return fail(nullptr, s);
  std::vector<sv_gate> recs;
  sv_gate mk;
  std::memset(&mk, 0, sizeof(mk));
  for (size_t i = 0; i < steps.size(); i++) {
    const Step& st = steps[i];
    if (st.type == Step::EXCHANGE) {
      for (const ExPair& p : st.ex) {
        sv_gate r = mk;
        r.kind = SV_EXCHANGE;
        r.q0 = p.m;
        r.q1 = p.b;
        r.pad = (int32_t)i;
        recs.push_back(r);
      }
    } else if (st.type == Step::COMPACT) {  // physical memory-bit swaps: SWAP records outside sections
      for (const auto& sw : st.swaps) {
        sv_gate r = mk;
        r.kind = SV_SWAP;
        r.q0 = sw.first;
        r.q1 = sw.second;
        r.pad = (int32_t)i;
        recs.push_back(r);
      }
    } else {
      sv_gate b = mk;
      b.kind = SV_BEGIN;
      b.q0 = b.q1 = -1;
      b.pad = (int32_t)i;
      recs.push_back(b);
      for (const sv_gate& gm : st.gates) recs.push_back(gm);
      b.kind = SV_END;
      recs.push_back(b);
      for (const auto& sw : st.swaps) {  // swaps fused into the section's store, right after it
        sv_gate r = mk;
        r.kind = SV_SWAP;
        r.q0 = sw.first;
        r.q1 = sw.second;
        r.pad = (int32_t)i;
        recs.push_back(r);
      }
    }
  }
  sv_gate* buf = (sv_gate*)std::malloc(sizeof(sv_gate) * std::max<size_t>(recs.size(), 1));
  if (!buf) return fail(nullptr, SV_ECAPACITY, "out of host memory");
  if (!recs.empty()) std::memcpy(buf, recs.data(), sizeof(sv_gate) * recs.size());
  *out = buf;
  *n_out = recs.size();
  for (int q = 0; q < n; q++) {
    if (pi_final) pi_final[q] = pi[q];
    if (sigma_final) sigma_final[q] = sigma[q];
  }
  return SV_OK;
}

}  // extern "C"

extern "C" int sv_compile_circuit(const sv_gate* gates, size_t n_gates, int n, int c, int world_log2, int rank,
                                  sv_precision prec, const int32_t* pi0, const int32_t* sigma0, uint32_t flags,
                                  int64_t** steps_out, size_t* n_steps,
                                  int32_t** ints_out, size_t* n_ints, double** coefs_out, size_t* n_coefs,
                                  double** aux_out, size_t* n_aux, int32_t* pi_final, int32_t* sigma_final) {
  if (!steps_out || !n_steps || !ints_out || !n_ints || !coefs_out || !n_coefs || !aux_out || !n_aux ||
      (n_gates && !gates))
    return fail(nullptr, SV_EINVAL, "null argument");
  if (n < 1 || n > 63 || world_log2 < 0 || world_log2 >= n) return fail(nullptr, SV_EINVAL, "bad n / world");
  const int nL = n - world_log2;
  std::vector<int> pi(n), sigma(n);
  for (int q = 0; q < n; q++) {
    pi[q] = pi0 ? pi0[q] : q;
    sigma[q] = sigma0 ? sigma0[q] : q;
  }
  std::vector<Step> steps;
  PlanCounters ctr;
  PlanLayout lay;
  lay.low_bits = prec == SV_FP64 ? 3 : 4;
  apply_tile_prefs(lay);
  lay.free_initial = (flags & SV_FREE_LAYOUT) && !(flags & SV_UNBLOCKED);
  Status s = make_plan(gates, n_gates, n, c, world_log2, pi, sigma, flags, steps, ctr, lay);
  if (!s.good()) return fail(nullptr, s);
  Program prog;
  std::vector<int64_t> rec;
  auto put = [&](std::initializer_list<int64_t> v) {
    int64_t r[12] = {0};
    int i = 0;
    for (int64_t x : v) r[i++] = x;
    rec.insert(rec.end(), r, r + 12);
  };
  for (size_t i = 0; i < steps.size(); i++) {
    const Step& st = steps[i];
    if (st.type == Step::EXCHANGE) {
      for (const ExPair& p : st.ex) put({0, p.m, p.b, (int64_t)i});
    } else if (st.type == Step::COMPACT) {
      for (const auto& sw : st.swaps) put({3, sw.first, sw.second});
    } else if (st.type == Step::GATE || nL < SV_R_BITS) {
      for (const sv_gate& gm : st.gates) put({2, gm.kind, gm.q0, gm.q1, gm.pad});
      for (const auto& sw : st.swaps) put({3, sw.first, sw.second});
    } else {
      const size_t first = prog.launches.size();
      const Status cs =
          compile_section_split(st.gates, nL, rank, world_log2, lay.tile_default, lay.low_bits, st.swaps, prog);
      if (!cs.good()) return fail(nullptr, cs);
      for (size_t k = first; k < prog.launches.size(); k++) {
        const Launch& L = prog.launches[k];
        put({1, (int64_t)L.int_off, (int64_t)L.int_count, (int64_t)L.coef_off, (int64_t)L.coef_count, L.T, L.n_out,
             L.flags, (int64_t)L.aux_off, (int64_t)L.aux_count});
      }
    }
  }
  auto dup = [](const void* src, size_t bytes) {
    void* p = std::malloc(bytes ? bytes : 1);
    if (p && bytes) std::memcpy(p, src, bytes);
    return p;
  };
  *steps_out = (int64_t*)dup(rec.data(), rec.size() * sizeof(int64_t));
  *n_steps = rec.size() / 12;
  *ints_out = (int32_t*)dup(prog.ints.data(), prog.ints.size() * sizeof(int));
  *n_ints = prog.ints.size();
  *coefs_out = (double*)dup(prog.coefs.data(), prog.coefs.size() * sizeof(double));
  *n_coefs = prog.coefs.size() / 2;
  *aux_out = (double*)dup(prog.aux.data(), prog.aux.size() * sizeof(double));
  *n_aux = prog.aux.size() / 2;
  for (int q = 0; q < n; q++) {
    if (pi_final) pi_final[q] = pi[q];
    if (sigma_final) sigma_final[q] = sigma[q];
  }
  return SV_OK;
}

extern "C" int sv_jit_compile_circuit(const sv_gate* gates, size_t n_gates, int n, int c, int world_log2, int rank,
                                      sv_precision prec, uint32_t flags, const char* dump_dir, int* n_kernels,
                                      double* compile_ms) {
  if (n_gates && !gates) return fail(nullptr, SV_EINVAL, "null gate array");
  if (n < 1 || n > 63 || world_log2 < 0 || world_log2 >= n) return fail(nullptr, SV_EINVAL, "bad n / world");
  const int nL = n - world_log2;
  std::vector<int> pi(n), sigma(n);
  for (int q = 0; q < n; q++) pi[q] = sigma[q] = q;
  std::vector<Step> steps;
  PlanCounters ctr;
  PlanLayout lay;
  lay.low_bits = prec == SV_FP64 ? 3 : 4;
  apply_tile_prefs(lay);
  lay.free_initial = (flags & SV_FREE_LAYOUT) && !(flags & SV_UNBLOCKED);
  Status s = make_plan(gates, n_gates, n, c, world_log2, pi, sigma, flags, steps, ctr, lay);
  if (!s.good()) return fail(nullptr, s);
  Program prog;
  for (const Step& st : steps) {
    if (st.type != Step::SECTION || nL < SV_R_BITS) continue;
    Status cs = compile_section_split(st.gates, nL, rank, world_log2, lay.tile_default, lay.low_bits, st.swaps, prog);
    if (!cs.good()) return fail(nullptr, cs);
  }
  int k = 0;
  double total = 0.0;
  for (const Launch& L : prog.launches) {
    double ms = 0.0;
    Status js = jit_compile_only(prog.ints.data() + L.int_off, L, prec == SV_FP64, dump_dir, k, &ms);
    if (!js.good()) return fail(nullptr, js);
    total += ms;
    k++;
  }
  if (n_kernels) *n_kernels = k;
  if (compile_ms) *compile_ms = total;
  return SV_OK;
}

extern "C" int sv_jit_mode(int mode) { return jit_set_mode(mode); }

extern "C" int sv_jit_wait(void) {
  jit_wait();
  return SV_OK;
}
