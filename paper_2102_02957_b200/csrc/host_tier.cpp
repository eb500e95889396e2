// host_tier.cpp — NEXT-4: the state resident in (pinned) host memory, the GPU as a cache of
// 2^d-amplitude chunks ("for all chunks: fetch, apply the section, evict";
// chunks beyond GPU memory kept in host memory).
//
// The top n - d qubits index host chunks the way rank bits index GPUs: the same planner (two-level
// when it moves less, Belady victims) maps the blocked circuit onto memory bits, every section is
// one streaming pass of all chunks through the GPU (H2D / section kernel / D2H on three streams,
// two device buffers, so PCIe both ways and the kernel overlap), and an exchange of a local bit
// with a chunk bit is a bit permutation of the host array (data movement in the memory tier, done
// by host threads).  Readouts stream the chunks through the same reduction kernels.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "../../include/sv.h"
#include "common.h"
#include "compile.h"
#include "jit.h"
#include "kernels.cuh"
#include "program.h"

namespace sv {
namespace {

struct RankProg {  // one chunk index's programs (rank-bit constants differ) and their device copies
  Program prog;
  void* d_ints = nullptr;
  void* d_coef = nullptr;
  void* d_aux = nullptr;
  size_t cap_i = 0, cap_c = 0, cap_a = 0;
};

thread_local std::string t_host_err;

}  // namespace
}  // namespace sv

struct sv_host_state {
  int n = 0, c = 0, d = 0, gh = 0, device = 0;
  bool dbl = true;
  size_t amp = 16;
  void* host = nullptr;
  void* dbuf[2] = {nullptr, nullptr};
  double* d_red = nullptr;  // reduction scratch + output
  size_t red_cap = 0;
  cudaStream_t s_in = nullptr, s_cmp = nullptr, s_out = nullptr;
  cudaEvent_t ev_in[2] = {}, ev_cmp[2] = {}, ev_out[2] = {};
  std::vector<int> pi, sigma;
  std::vector<sv::RankProg> rp;
  std::string err;
};

namespace sv {
namespace {

int hfail(sv_host_state* h, int code, const std::string& msg) {
  if (h) h->err = msg;
  t_host_err = msg;
  return code;
}
#define HCUDA(h, expr)                                                                       \
  do {                                                                                       \
    cudaError_t e_ = (expr);                                                                 \
    if (e_ != cudaSuccess) return hfail(h, SV_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

size_t chunk_amps(const sv_host_state* h) { return size_t(1) << h->d; }

// Swap memory bits m (local, < d) and b of the host array: for every index with bit m = 1 and bit
// b = 0, exchange it with its partner (runs of 2^min(m, b) contiguous amplitudes), host threads.
void host_bit_swap(sv_host_state* h, int m, int b) {
  if (m == b) return;
  const int lo = std::min(m, b), hi = std::max(m, b);
  const uint64_t N = 1ull << h->n, run = 1ull << lo, runs = N >> (lo + 2);  // blocks with lo = 1, hi = 0
  const size_t bytes = run * h->amp;
  const unsigned nth = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  auto work = [&](unsigned t) {
    std::vector<char> tmp(bytes);
    for (uint64_t i = t; i < runs; i += nth) {
      // i enumerates indices with bits lo and hi removed (in units of runs)
      uint64_t x = i << lo;  // bits >= lo
      const uint64_t l1 = x & ((1ull << lo) - 1);
      x = ((x - l1) << 1) | l1;
      const uint64_t l2 = x & ((1ull << hi) - 1);
      x = ((x - l2) << 1) | l2;
      const uint64_t a = x | (1ull << lo), c = x | (1ull << hi);  // (lo = 1, hi = 0) <-> (lo = 0, hi = 1)
      char* pa = (char*)h->host + a * h->amp;
      char* pc = (char*)h->host + c * h->amp;
      std::memcpy(tmp.data(), pa, bytes);
      std::memcpy(pa, pc, bytes);
      std::memcpy(pc, tmp.data(), bytes);
    }
  };
  std::vector<std::thread> th;
  for (unsigned t = 1; t < nth; t++) th.emplace_back(work, t);
  work(0);
  for (auto& t : th) t.join();
}

int upload_rank(sv_host_state* h, RankProg& r) {
  const Program& p = r.prog;
  const size_t ib = p.ints.size() * sizeof(int), cb = p.coefs.size() / 2 * h->amp, ab = p.aux.size() / 2 * h->amp;
  auto grow = [&](void*& ptr, size_t& cap, size_t need) -> int {
    if (need <= cap) return SV_OK;
    if (ptr) HCUDA(h, cudaFree(ptr));
    ptr = nullptr;
    cap = std::max<size_t>(need, 4096);
    HCUDA(h, cudaMalloc(&ptr, cap));
    return SV_OK;
  };
  if (int rc = grow(r.d_ints, r.cap_i, ib + 16)) return rc;
  if (int rc = grow(r.d_coef, r.cap_c, cb + 16)) return rc;
  if (int rc = grow(r.d_aux, r.cap_a, ab + 16)) return rc;
  auto conv = [&](const std::vector<double>& src) {
    std::vector<char> out(src.size() / 2 * h->amp);
    if (h->dbl) {
      std::memcpy(out.data(), src.data(), out.size());
    } else {
      float* f = (float*)out.data();
      for (size_t i = 0; i < src.size(); i++) f[i] = (float)src[i];
    }
    return out;
  };
  if (ib) HCUDA(h, cudaMemcpy(r.d_ints, p.ints.data(), ib, cudaMemcpyHostToDevice));
  if (cb) {
    auto c = conv(p.coefs);
    HCUDA(h, cudaMemcpy(r.d_coef, c.data(), cb, cudaMemcpyHostToDevice));
  }
  if (ab) {
    auto a = conv(p.aux);
    HCUDA(h, cudaMemcpy(r.d_aux, a.data(), ab, cudaMemcpyHostToDevice));
  }
  return SV_OK;
}

// One streaming pass: every chunk r through the GPU with `per_chunk(r, buffer, stream)`; write back
// unless read_only.
template <typename F>
int stream_chunks(sv_host_state* h, bool read_only, F per_chunk) {
  const int R = 1 << h->gh;
  const size_t bytes = chunk_amps(h) * h->amp;
  for (int r = 0; r < R; r++) {
    const int b = r & 1;
    if (r >= 2) HCUDA(h, cudaStreamWaitEvent(h->s_in, h->ev_out[b], 0));  // buffer b is free again
    HCUDA(h, cudaMemcpyAsync(h->dbuf[b], (char*)h->host + (size_t)r * bytes, bytes, cudaMemcpyHostToDevice, h->s_in));
    HCUDA(h, cudaEventRecord(h->ev_in[b], h->s_in));
    HCUDA(h, cudaStreamWaitEvent(h->s_cmp, h->ev_in[b], 0));
    if (int rc = per_chunk(r, h->dbuf[b], h->s_cmp)) return rc;
    HCUDA(h, cudaEventRecord(h->ev_cmp[b], h->s_cmp));
    HCUDA(h, cudaStreamWaitEvent(h->s_out, h->ev_cmp[b], 0));
    if (!read_only)
      HCUDA(h, cudaMemcpyAsync((char*)h->host + (size_t)r * bytes, h->dbuf[b], bytes, cudaMemcpyDeviceToHost, h->s_out));
    HCUDA(h, cudaEventRecord(h->ev_out[b], h->s_out));
  }
  HCUDA(h, cudaStreamSynchronize(h->s_out));
  HCUDA(h, cudaStreamSynchronize(h->s_cmp));
  return SV_OK;
}

int ensure_red(sv_host_state* h, size_t doubles) {
  if (doubles <= h->red_cap) return SV_OK;
  if (h->d_red) HCUDA(h, cudaFree(h->d_red));
  h->d_red = nullptr;
  HCUDA(h, cudaMalloc(&h->d_red, doubles * sizeof(double)));
  h->red_cap = doubles;
  return SV_OK;
}

uint64_t mu_of(const sv_host_state* h, uint64_t x) {
  uint64_t m = 0;
  for (int q = 0; q < h->n; q++) m |= ((x >> q) & 1ull) << h->sigma[h->pi[q]];
  return m;
}

}  // namespace
}  // namespace sv

using namespace sv;

extern "C" int sv_host_create(int n, int c, sv_precision prec, int device_bits, sv_host_handle* out) {
  if (!out) return hfail(nullptr, SV_EINVAL, "null output");
  *out = nullptr;
  if (n < 2 || n > 40 || device_bits < SV_R_BITS || device_bits >= n || c < 1 || c > device_bits)
    return hfail(nullptr, SV_EINVAL, "need 4 <= device_bits < n <= 40 and 1 <= chunk_bits <= device_bits");
  auto* h = new sv_host_state();
  h->n = n;
  h->c = c;
  h->d = device_bits;
  h->gh = n - device_bits;
  h->dbl = prec == SV_FP64;
  h->amp = h->dbl ? 16 : 8;
  h->pi.resize(n);
  h->sigma.resize(n);
  std::iota(h->pi.begin(), h->pi.end(), 0);
  std::iota(h->sigma.begin(), h->sigma.end(), 0);
  auto bail = [&](int rc) {
    sv_host_destroy(h);
    return rc;
  };
  if (cudaGetDevice(&h->device) != cudaSuccess) return bail(hfail(nullptr, SV_ECUDA, "no CUDA device"));
  const size_t total = (size_t(1) << n) * h->amp, chunk = chunk_amps(h) * h->amp;
  if (cudaMallocHost(&h->host, total) != cudaSuccess) return bail(hfail(nullptr, SV_ECAPACITY, "pinned host allocation failed"));
  for (int b = 0; b < 2; b++)
    if (cudaMalloc(&h->dbuf[b], chunk) != cudaSuccess) return bail(hfail(nullptr, SV_ECAPACITY, "device chunk buffers"));
  for (cudaStream_t* s : {&h->s_in, &h->s_cmp, &h->s_out})
    if (cudaStreamCreateWithFlags(s, cudaStreamNonBlocking) != cudaSuccess) return bail(hfail(nullptr, SV_ECUDA, "streams"));
  for (int b = 0; b < 2; b++)
    for (cudaEvent_t* e : {&h->ev_in[b], &h->ev_cmp[b], &h->ev_out[b]})
      if (cudaEventCreateWithFlags(e, cudaEventDisableTiming) != cudaSuccess) return bail(hfail(nullptr, SV_ECUDA, "events"));
  h->rp.resize(size_t(1) << h->gh);
  if (int rc = sv_host_reset(h, 0)) return bail(rc);
  *out = h;
  return SV_OK;
}

extern "C" int sv_host_destroy(sv_host_handle h) {
  if (!h) return SV_OK;
  cudaSetDevice(h->device);
  for (cudaStream_t s : {h->s_in, h->s_cmp, h->s_out})
    if (s) cudaStreamSynchronize(s);
  for (auto& r : h->rp)
    for (void* p : {r.d_ints, r.d_coef, r.d_aux})
      if (p) cudaFree(p);
  for (void* p : h->dbuf)
    if (p) cudaFree(p);
  if (h->d_red) cudaFree(h->d_red);
  if (h->host) cudaFreeHost(h->host);
  for (int b = 0; b < 2; b++)
    for (cudaEvent_t e : {h->ev_in[b], h->ev_cmp[b], h->ev_out[b]})
      if (e) cudaEventDestroy(e);
  for (cudaStream_t s : {h->s_in, h->s_cmp, h->s_out})
    if (s) cudaStreamDestroy(s);
  cudaGetLastError();
  delete h;
  return SV_OK;
}

extern "C" int sv_host_reset(sv_host_handle h, uint64_t k) {
  if (!h) return hfail(nullptr, SV_EINVAL, "null handle");
  if (k >> h->n) return hfail(h, SV_EINVAL, "basis index out of range");
  std::iota(h->pi.begin(), h->pi.end(), 0);
  std::iota(h->sigma.begin(), h->sigma.end(), 0);
  std::memset(h->host, 0, (size_t(1) << h->n) * h->amp);
  if (h->dbl)
    ((double*)h->host)[2 * k] = 1.0;
  else
    ((float*)h->host)[2 * k] = 1.0f;
  return SV_OK;
}

extern "C" int sv_host_apply_circuit(sv_host_handle h, const sv_gate* gates, size_t n_gates, uint32_t flags) {
  if (!h) return hfail(nullptr, SV_EINVAL, "null handle");
  if (n_gates && !gates) return hfail(h, SV_EINVAL, "null gate array");
  if (flags & (SV_UNBLOCKED | SV_EXCHANGE_NCCL)) return hfail(h, SV_EINVAL, "host tier: blocked path only");
  HCUDA(h, cudaSetDevice(h->device));
  std::vector<int> pi = h->pi, sigma = h->sigma;
  std::vector<Step> steps;
  PlanCounters ctr;
  PlanLayout lay;
  lay.low_bits = h->dbl ? 3 : 4;
  apply_tile_prefs(lay);
  Status s = make_plan(gates, n_gates, h->n, h->c, h->gh, pi, sigma, flags, steps, ctr, lay);
  if (!s.good()) return hfail(h, s.code, s.msg);
  const int R = 1 << h->gh;
  std::vector<size_t> launch_end(steps.size(), 0);
  for (auto& r : h->rp) r.prog.clear();
  for (size_t i = 0; i < steps.size(); i++) {
    if (steps[i].type == Step::SECTION)
      for (int r = 0; r < R; r++) {
        Status cs = compile_section_split(steps[i].gates, h->d, r, h->gh, lay.tile_default, lay.low_bits,
                                          steps[i].swaps, h->rp[r].prog);
        if (!cs.good()) return hfail(h, cs.code, cs.msg);
        if (h->rp[r].prog.launches.size() != h->rp[0].prog.launches.size())
          return hfail(h, SV_EMALFORMED, "internal: chunk programs differ in launch count");
      }
    launch_end[i] = h->rp[0].prog.launches.size();
  }
  for (int r = 0; r < R; r++) {
    jit_prepare(h->rp[r].prog, h->dbl);
    if (int rc = upload_rank(h, h->rp[r])) return rc;
  }
  size_t li = 0;
  for (size_t i = 0; i < steps.size(); i++) {
    const Step& st = steps[i];
    if (st.type == Step::EXCHANGE) {
      for (const ExPair& p : st.ex) host_bit_swap(h, p.m, p.b);
    } else if (st.type == Step::COMPACT) {
      for (const auto& sw : st.swaps) host_bit_swap(h, sw.first, sw.second);
    } else if (st.type == Step::SECTION) {
      for (; li < launch_end[i]; li++) {
        const size_t at = li;
        int rc = stream_chunks(h, false, [&](int r, void* buf, cudaStream_t stm) -> int {
          RankProg& rp = h->rp[r];
          const Launch& L = rp.prog.launches[at];
          const int* pdev = (const int*)rp.d_ints + L.int_off;
          const char* cdev = (const char*)rp.d_coef + L.coef_off * h->amp;
          const char* adev = (const char*)rp.d_aux + L.aux_off * h->amp;
          cudaError_t je = cudaSuccess;
          if (!jit_launch_section(h->dbl, buf, rp.prog.ints.data() + L.int_off, rp.prog.coefs.data() + 2 * L.coef_off,
                                  L, cdev, adev, stm, &je))
            je = launch_section(h->dbl, buf, pdev, L.int_count, cdev, L.coef_count, adev, L.T, L.n_out, L.n_phases,
                                L.flags, L.n_sets, stm);
          HCUDA(h, je);
          return SV_OK;
        });
        if (rc) return rc;
      }
    } else {
      return hfail(h, SV_EMALFORMED, "internal: unexpected step in the host tier");
    }
  }
  h->pi = pi;
  h->sigma = sigma;
  return SV_OK;
}

extern "C" int sv_host_get_state(sv_host_handle h, void* host_out) {
  if (!h || !host_out) return hfail(h, SV_EINVAL, "null argument");
  const uint64_t N = 1ull << h->n;
  for (uint64_t x = 0; x < N; x++)  // logical order: a_logical[x] = mem[mu(x)]
    std::memcpy((char*)host_out + x * h->amp, (const char*)h->host + mu_of(h, x) * h->amp, h->amp);
  return SV_OK;
}

extern "C" int sv_host_norm(sv_host_handle h, double* out) {
  if (!h || !out) return hfail(h, SV_EINVAL, "null argument");
  HCUDA(h, cudaSetDevice(h->device));
  const int R = 1 << h->gh;
  if (int rc = ensure_red(h, norm_scratch_doubles() + R)) return rc;
  double* outs = h->d_red + norm_scratch_doubles();
  int rc = stream_chunks(h, true, [&](int r, void* buf, cudaStream_t stm) -> int {
    HCUDA(h, launch_norm(h->dbl, buf, h->d, h->d_red, outs + r, stm));
    return SV_OK;
  });
  if (rc) return rc;
  std::vector<double> part(R);
  HCUDA(h, cudaMemcpy(part.data(), outs, R * sizeof(double), cudaMemcpyDeviceToHost));
  double t = 0;
  for (double v : part) t += v;  // R per-chunk sums
  *out = t;
  return SV_OK;
}

extern "C" int sv_host_probabilities(sv_host_handle h, const int32_t* qubits, int nq, double* host_out) {
  if (!h || nq < 0 || nq > 24 || (nq && (!qubits || !host_out))) return hfail(h, SV_EINVAL, "bad arguments");
  HCUDA(h, cudaSetDevice(h->device));
  const int R = 1 << h->gh, bins = 1 << nq;
  // logical qubit i -> memory bit; local ones are reduced on the GPU per chunk, chunk bits fix the bin
  std::vector<int> loc, loc_i;
  std::vector<int> mb(nq);
  for (int i = 0; i < nq; i++) {
    if (qubits[i] < 0 || qubits[i] >= h->n) return hfail(h, SV_EINVAL, "qubit out of range");
    mb[i] = h->sigma[h->pi[qubits[i]]];
    if (mb[i] < h->d) {
      loc.push_back(mb[i]);
      loc_i.push_back(i);
    }
  }
  const int nl = (int)loc.size();
  const size_t lbins = size_t(1) << nl;
  if (int rc = ensure_red(h, std::max(marginal_scratch_doubles(nl), norm_scratch_doubles()) + R * lbins)) return rc;
  double* outs = h->d_red + std::max(marginal_scratch_doubles(nl), norm_scratch_doubles());
  int rc = stream_chunks(h, true, [&](int r, void* buf, cudaStream_t stm) -> int {
    HCUDA(h, launch_marginal(h->dbl, buf, h->d, loc.data(), nl, h->d_red, outs + r * lbins, stm));
    return SV_OK;
  });
  if (rc) return rc;
  std::vector<double> part(R * lbins);
  HCUDA(h, cudaMemcpy(part.data(), outs, part.size() * sizeof(double), cudaMemcpyDeviceToHost));
  std::fill(host_out, host_out + bins, 0.0);
  for (int r = 0; r < R; r++) {
    int ybase = 0;  // bin bits of the chunk-index (non-local) qubits
    for (int i = 0; i < nq; i++)
      if (mb[i] >= h->d) ybase |= (int)(((uint64_t)r >> (mb[i] - h->d)) & 1) << i;
    for (size_t y = 0; y < lbins; y++) {
      int yy = ybase;
      for (int j = 0; j < nl; j++) yy |= (int)((y >> j) & 1) << loc_i[j];
      host_out[yy] += part[r * lbins + y];
    }
  }
  return SV_OK;
}

extern "C" const char* sv_host_last_error(sv_host_handle h) { return h ? h->err.c_str() : t_host_err.c_str(); }
