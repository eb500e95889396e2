// jit.cpp — run-time specialised section kernels (see jit.h).
//
// The generated kernel is the interpreter kernel of section.cu with its loops over phases and
// ops unrolled for one program: the same device building blocks (section_dev.cuh, embedded in
// libsv.so as text by build.py) with every slot, map entry and coefficient offset an immediate.
// NVRTC and the CUDA library API are reached through dlopen / the static runtime, so libsv.so
// still loads on a host without a GPU or without NVRTC (the interpreter then runs).
#include "jit.h"

#include <dlfcn.h>
#include <sys/stat.h>
#include <unistd.h>
#include <nvrtc.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <cstring>
#include <deque>
#include <iterator>
#include <memory>
#include <mutex>
#include <sstream>
#include <thread>
#include <unordered_map>
#include <vector>

#include "program.h"

namespace sv {
namespace {

#include "jit_headers.inc"  // kJitHeaderNames[], kJitHeaderTexts[], kJitHeaderCount (build.py)

// ------------------------------------------------------------------------------------ NVRTC
struct Nvrtc {
  bool ok = false;
  decltype(&nvrtcCreateProgram) create = nullptr;
  decltype(&nvrtcDestroyProgram) destroy = nullptr;
  decltype(&nvrtcCompileProgram) compile = nullptr;
  decltype(&nvrtcGetProgramLogSize) log_size = nullptr;
  decltype(&nvrtcGetProgramLog) log = nullptr;
  decltype(&nvrtcGetCUBINSize) cubin_size = nullptr;
  decltype(&nvrtcGetCUBIN) cubin = nullptr;
  decltype(&nvrtcAddNameExpression) add_name = nullptr;
  decltype(&nvrtcGetLoweredName) lowered = nullptr;
};

Nvrtc load_nvrtc() {
  Nvrtc n;
  void* h = nullptr;
  for (const char* name : {"libnvrtc.so.12", "/usr/local/cuda/lib64/libnvrtc.so.12", "libnvrtc.so"})
    if ((h = dlopen(name, RTLD_NOW | RTLD_LOCAL))) break;
  if (!h) return n;
#define SV_SYM(field, sym) n.field = reinterpret_cast<decltype(n.field)>(dlsym(h, sym))
  SV_SYM(create, "nvrtcCreateProgram");
  SV_SYM(destroy, "nvrtcDestroyProgram");
  SV_SYM(compile, "nvrtcCompileProgram");
  SV_SYM(log_size, "nvrtcGetProgramLogSize");
  SV_SYM(log, "nvrtcGetProgramLog");
  SV_SYM(cubin_size, "nvrtcGetCUBINSize");
  SV_SYM(cubin, "nvrtcGetCUBIN");
  SV_SYM(add_name, "nvrtcAddNameExpression");
  SV_SYM(lowered, "nvrtcGetLoweredName");
#undef SV_SYM
  n.ok = n.create && n.destroy && n.compile && n.log_size && n.log && n.cubin_size && n.cubin && n.add_name &&
         n.lowered;
  return n;
}

Nvrtc& nvrtc() {
  static Nvrtc n = load_nvrtc();
  return n;
}

enum Mode { kOff = 0, kSync = 1, kAsync = 2 };
std::atomic<int> g_mode{-1};
Mode mode() {
  int m = g_mode.load();
  if (m < 0) {
    const char* e = std::getenv("SV_JIT");
    m = (!e || !*e || !std::strcmp(e, "sync") || !std::strcmp(e, "1")) ? kSync : !std::strcmp(e, "async") ? kAsync : kOff;
    int expect = -1;
    g_mode.compare_exchange_strong(expect, m);
    m = g_mode.load();
  }
  return (Mode)m;
}

// ------------------------------------------------------------------------------------ source
// Pipelined variant (gen_source_pipelined): two warp groups per CTA work on alternate tiles of
// a persistent CTA with three tile buffers in shared memory, each group loading its next tile
// with cp.async while it computes the current one.
constexpr int kPipeSetsBytes = 2 * 5 * SV_MAX_SETS;  // per-CTA factor slots (both groups), in amplitudes
bool pipelined(const Launch& L, bool dbl) {
  static const bool on = [] {
    const char* e = std::getenv("SV_PIPE");  // opt-in: measured slower than two CTAs per SM
    return e && e[0] == '1';
  }();
  const size_t amp = dbl ? 16 : 8;
  return on && !(L.flags & SV_FLAG_XRANK) && L.T >= 9 && L.T <= 12 &&
         3 * (amp << L.T) + kPipeSetsBytes * amp + 64 <= 227 * 1024;
}

// Persistent grid + L2 prefetch of each CTA's next tile for the plain generated kernel (SV_L2PF=1)
bool l2_prefetch(const Launch& L, bool dbl) {
  static const bool on = [] {
    const char* e = std::getenv("SV_L2PF");
    return e && e[0] == '1';
  }();
  return on && !pipelined(L, dbl) && !(L.flags & SV_FLAG_XRANK) && L.T >= SV_R_BITS;
}

size_t smem_bytes(const Launch& L, bool dbl) {
  const size_t amp = dbl ? 16 : 8;
  if (pipelined(L, dbl)) return 3 * (amp << L.T) + kPipeSetsBytes * amp + 64;
  const bool no_smem = L.n_phases == 1 && (L.flags & SV_FLAG_FIRST_DIRECT) && (L.flags & SV_FLAG_LAST_DIRECT);
  if (L.n_sets) return (amp << L.T) + 5 * SV_MAX_SETS * amp;
  return no_smem ? 0 : amp << L.T;
}

// Resident CTAs per SM the generated kernel is register-budgeted for (launch bounds): 512 threads
// per SM at 128 registers (SV_JIT_THREADS_SM overrides the target for tiles below 12 bits).
// Sections without dense 2-qubit gates (QFT-like: butterflies and phases) need fewer registers
// and run 640 threads per SM (QFT30 29.7 -> 29.3 ms); U2 sections would spill there.
int resident_ctas(int T, int nt, bool dense) {
  static const int target = [] {
    const char* e = std::getenv("SV_JIT_THREADS_SM");
    return e ? std::max(32, std::atoi(e)) : 0;
  }();
  if (T > 12) return 1;
  if (T == 12) return 2;
  const int t = target ? target : (dense ? 512 : 640);
  return std::max(1, std::min(16, t / nt));
}

bool has_dense(const int* p) {
  const SvSecHeader* H = reinterpret_cast<const SvSecHeader*>(p);
  const SvOp* ops = reinterpret_cast<const SvOp*>(p + H->op_off);
  for (int i = 0; i < H->n_ops; i++)
    if (ops[i].type == SV_OP_U2 || ops[i].type == SV_OP_U1) return true;
  return false;
}

// Coefficients as a __grid_constant__ kernel parameter when they fit the 32 KiB parameter space
// (FMAs then read them from the parameter bank); else from the module's __constant__ bank.
constexpr size_t kParamCoefMax = 31 * 1024;
bool coef_in_param(const Launch& L, bool dbl) { return L.coef_count * (dbl ? 16 : 8) <= kParamCoefMax; }
std::string coef_param_decl_impl(const Launch& L, bool dbl) {
  if (coef_in_param(L, dbl))
    return "const __grid_constant__ CoefParam<V, " + std::to_string(L.coef_count ? L.coef_count : 1) + "> P";
  return "const CoefBank<V> P";
}

struct Gen {
  std::ostringstream o;
  int T = 0, ntl = 0;

  template <typename X>
  void arr(const char* type, const char* name, const X* v, int n) {
    o << "    constexpr " << type << " " << name << "[" << (n > 0 ? n : 1) << "] = {";
    if (n == 0) o << "0";
    for (int i = 0; i < n; i++) o << (i ? ", " : "") << v[i];
    o << "};\n";
  }
  // HBM element offset of register 0 (b) and of every register k (RO[k]) under map m
  int nl = 64;  // memory bits >= nl are rank bits (fused exchange, SV_FLAG_XRANK)
  bool xrank = false;
  bool virt = false;  // the tile's input is generated: 1 at shard offset vidx, 0 elsewhere
  void hbm(const SvMap& m) {
    long long ro[16];
    int gk[16], tmb[16];
    uint32_t trank = 0;  // thread bits on the rank bit
    for (int k = 0; k < 16; k++) {
      ro[k] = 0;
      gk[k] = 0;
      for (int s = 0; s < SV_R_BITS; s++)
        if ((k >> s) & 1) {
          if (m.rmb[s] >= nl)
            gk[k] = 1;
          else
            ro[k] |= 1ll << m.rmb[s];
        }
    }
    for (int j = 0; j < ntl; j++) {
      tmb[j] = m.tmb[j] >= nl ? 63 : m.tmb[j];  // 63: contributes nothing below (masked)
      if (m.tmb[j] >= nl) trank |= 1u << j;
    }
    arr("int", "TMB", tmb, ntl);
    arr("long long", "RO", ro, 16);
    o << "    uint64_t b = tile_off;\n"
      << "#pragma unroll\n    for (int j = 0; j < " << ntl << "; j++) if (TMB[j] != 63) b |= (uint64_t)((tid >> j) & 1) << TMB[j];\n";
    if (xrank) {  // which GPU's shard each register lives on (the rank bit's value)
      arr("int", "GK", gk, 16);
      o << "    const int gs = (tid & " << trank << ") ? 1 : 0;\n";
    }
  }
  // swizzled smem offset of register 0 (x) and XOR offsets W[k] for thread-bit words tw, slot words rw
  void smem(const int* tw, const int* rw) {
    int w[16];
    for (int k = 0; k < 16; k++) {
      w[k] = 0;
      for (int s = 0; s < SV_R_BITS; s++)
        if ((k >> s) & 1) w[k] ^= rw[s];
    }
    arr("int", "TW", tw, ntl);
    arr("int", "W", w, 16);
    o << "    int x = 0;\n#pragma unroll\n    for (int j = 0; j < " << ntl
      << "; j++) x ^= ((tid >> j) & 1) ? TW[j] : 0;\n";
  }
  // DIAGSET op with its structure specialised (section_dev.cuh diagset_c); false: not applicable
  bool diagset_c(const int* p, const SvOp& op, const std::string& nthr) {
    if (op.type != SV_OP_DIAGSET) return false;
    const int d = op.a, flags = p[d];
    const int set = (flags >> 8) & 255, tabm = (flags >> 16) & 31;
    if (set == 255 || p[d + 9] != p[d + 8]) return false;  // per-warp CTA terms or mixed terms
    int ctam = 0;
    for (int i = 0; i < 5; i++)
      if (p[d + 3 + i] > p[d + 2 + i]) ctam |= 1 << i;
    o << "    diagset_c<" << (flags & 1) << ", " << set << ", " << tabm << ", " << ctam << ">(v, " << d << ", "
      << op.coef << ", tid, " << nthr << ", aux, ctaf, P);\n";
    return true;
  }
  void lds() { o << "#pragma unroll\n    for (int k = 0; k < 16; k++) v[k] = sm[x ^ W[k]];\n"; }
  void sts() { o << "#pragma unroll\n    for (int k = 0; k < 16; k++) sm[x ^ W[k]] = v[k];\n"; }
  void ldg() {
    if (virt) {
      o << "#pragma unroll\n    for (int k = 0; k < 16; k++) { v[k].x = (long long)(b + RO[k]) == vidx ? 1 : 0; v[k].y = 0; }\n";
      return;
    }
    if (xrank)
      o << "#pragma unroll\n    for (int k = 0; k < 16; k++) v[k] = ((gs ^ GK[k]) ? psi_hi : psi)[b + RO[k]];\n";
    else
      o << "#pragma unroll\n    for (int k = 0; k < 16; k++) v[k] = psi[b + RO[k]];\n";
  }
  void stg() {
    if (xrank)
      o << "#pragma unroll\n    for (int k = 0; k < 16; k++) ((gs ^ GK[k]) ? psi_hi : psi)[b + RO[k]] = v[k];\n";
    else
      o << "#pragma unroll\n    for (int k = 0; k < 16; k++) psi[b + RO[k]] = v[k];\n";
  }
};

std::string gen_source_pipelined(const int* p, const Launch& L, bool dbl);

std::string gen_source(const int* p, const Launch& L, bool dbl, bool virt = false) {
  if (pipelined(L, dbl)) return gen_source_pipelined(p, L, dbl);
  const SvSecHeader* H = reinterpret_cast<const SvSecHeader*>(p);
  Gen g;
  g.virt = virt;
  g.xrank = (H->flags & SV_FLAG_XRANK) != 0;
  g.nl = g.xrank ? H->nl : 64;
  g.T = H->T;
  g.ntl = H->T - SV_R_BITS;
  const int nt = 1 << g.ntl;
  const bool first = H->flags & SV_FLAG_FIRST_DIRECT, last = H->flags & SV_FLAG_LAST_DIRECT;
  const int nph = H->n_phases;
  const bool persist = l2_prefetch(L, dbl);
  auto& o = g.o;
  o << "#include \"section_dev.cuh\"\nusing namespace sv;\ntypedef " << (dbl ? "double2" : "float2") << " V;\n";
  o << "extern \"C\" __global__ void __launch_bounds__(" << nt << ", " << resident_ctas(H->T, nt, has_dense(p))
    << ") sv_sec(V* __restrict__ psi, V* __restrict__ psi_hi, const V* __restrict__ aux, int split_a, int split_b, "
    << "long long vidx, "
    << coef_param_decl_impl(L, dbl) << ") {\n";
  o << "  extern __shared__ __align__(16) unsigned char smem_raw[];\n"
    << "  V* sm = reinterpret_cast<V*>(smem_raw);\n"
    << "  V* ctaf = reinterpret_cast<V*>(smem_raw + (sizeof(V) << " << H->T << "));\n"
    << "  (void)sm; (void)ctaf; (void)aux; (void)vidx; (void)psi_hi;\n"
    << "  const int tid = threadIdx.x;\n";
  g.arr("int", "OB", H->out_bits, H->n_out);
  o << "  auto tile_of = [&](uint64_t t) {\n    uint64_t r = 0;\n#pragma unroll\n    for (int j = 0; j < "
    << H->n_out << "; j++) r |= ((t >> j) & 1ull) << OB[j];\n    return r;\n  };\n";
  if (persist) {
    // L2 prefetch of the CTA's next tile: one request per 128-byte line (lanes / registers whose
    // memory bits below G are zero), through the map the tile is read with
    const SvMap& m0 = first ? H->din : H->load;
    const int G = dbl ? 3 : 4;
    uint32_t lead_mask = 0;
    int rskip = 0;
    for (int j = 0; j < g.ntl; j++)
      if (m0.tmb[j] < G) lead_mask |= 1u << j;
    for (int s2 = 0; s2 < SV_R_BITS; s2++)
      if (m0.rmb[s2] < G) rskip |= 1 << s2;
    g.arr("int", "PTMB", m0.tmb, g.ntl);
    long long ro[16];
    for (int k = 0; k < 16; k++) {
      ro[k] = 0;
      for (int s2 = 0; s2 < SV_R_BITS; s2++)
        if ((k >> s2) & 1) ro[k] |= 1ll << m0.rmb[s2];
    }
    g.arr("long long", "PRO", ro, 16);
    o << "  const bool lead = (tid & " << lead_mask << ") == 0;\n"
      << "  uint64_t pb = 0;\n#pragma unroll\n  for (int j = 0; j < " << g.ntl
      << "; j++) pb |= (uint64_t)((tid >> j) & 1) << PTMB[j];\n"
      << "  constexpr unsigned long long NTILES = 1ull << " << H->n_out << ";\n"
      << "#pragma unroll 1\n"
      << "  for (uint64_t bid = blockIdx.x; bid < NTILES; bid += gridDim.x) {\n"
      << "  const uint64_t tile_off = tile_of(bid);\n"
      << "  if (lead && bid + gridDim.x < NTILES) {\n"
      << "    const V* q = psi + (tile_of(bid + gridDim.x) | pb);\n#pragma unroll\n"
      << "    for (int k = 0; k < 16; k++)\n"
      << "      if (!(k & " << rskip << ")) asm volatile(\"prefetch.global.L2 [%0];\" ::\"l\"(q + PRO[k]));\n"
      << "  }\n";
  } else {
    o << "  {\n  const uint64_t tile_off = tile_of(expand_tile(blockIdx.x, split_a, split_b));\n";
  }
  if (H->n_sets > 0) {
    o << "  for (int f = tid; f < " << 5 * H->n_sets << "; f += " << nt << ") {\n"
      << "    const int d = c_prog[kH_SETS + f / 5], i = f % 5;\n"
      << "    ctaf[f] = cta_factor<V>(c_prog[d + 2 + i], c_prog[d + 3 + i], tile_off, P);\n  }\n"
      << "  __syncthreads();\n";
  }
  o << "  V v[16];\n";
  if (!first) {
    o << "  {  // load: lanes walk the lowest load memory bits, scatter into the swizzled tile\n";
    g.hbm(H->load);
    g.ldg();
    g.smem(H->load.tw, H->load.rw);
    g.sts();
    o << "    __syncthreads();\n  }\n";
  }
  const SvPhase* ph = reinterpret_cast<const SvPhase*>(p + H->phase_off);
  const SvOp* ops = reinterpret_cast<const SvOp*>(p + H->op_off);
  for (int k = 0; k < nph; k++) {
    const bool din = first && k == 0, dout = last && k == nph - 1;
    o << "  {  // phase " << k << "\n";
    if (din) {
      g.hbm(H->din);
      g.ldg();
    }
    if (!din || !dout) g.smem(ph[k].tw, ph[k].rw);
    if (!din) g.lds();
    for (int i = 0; i < ph[k].op_count; i++) {
      const SvOp& op = ops[ph[k].op_begin + i];
      if (!g.diagset_c(p, op, std::to_string(nt)))
        o << "    op_c<" << op.type << ", " << op.a << ", " << op.b << ", " << op.coef << ", " << op.extra
          << ">(v, tid, " << nt << ", tile_off, aux, ctaf, P);\n";
    }
    if (dout) {
      o << "    {\n";
      g.hbm(H->dout);
      g.stg();
      o << "    }\n";
    } else {
      g.sts();
      o << "    __syncthreads();\n";
    }
    o << "  }\n";
  }
  if (!last) {
    o << "  {  // gather in store order, lanes walk the lowest store memory bits\n";
    g.smem(H->store.tw, H->store.rw);
    g.lds();
    g.hbm(H->store);
    g.stg();
    o << "  }\n";
  }
  if (persist) o << "  __syncthreads();  // the next tile reuses shared memory\n";
  o << "  }\n}\n";
  (void)L;
  return o.str();
}

// Persistent CTA, two warp groups of 2^(T-4) threads, three tile buffers.  The CTA's tiles
// j = 0, 1, 2, ... (tile blockIdx.x + j * gridDim.x) alternate between the groups and tile j
// lives in buffer j % 3.  Buffer (j + 2) % 3 is released when the other group finishes tile
// j - 1 (done[] in shared memory), and the group computing tile j then issues the cp.async
// loads of its next tile j + 2 there: at the first phase boundary that sees the release, or at
// the end of tile j.  Phase barriers are named barriers of the group, so the two groups drift
// freely and one group's loads / shared-memory traffic overlap the other's arithmetic.
std::string gen_source_pipelined(const int* p, const Launch& L, bool dbl) {
  (void)L;
  const SvSecHeader* H = reinterpret_cast<const SvSecHeader*>(p);
  Gen g;
  g.T = H->T;
  g.ntl = H->T - SV_R_BITS;
  const int nt = 1 << g.ntl;
  const bool last = H->flags & SV_FLAG_LAST_DIRECT;
  const int nph = H->n_phases;
  auto& o = g.o;
  o << "#include \"section_dev.cuh\"\nusing namespace sv;\ntypedef " << (dbl ? "double2" : "float2") << " V;\n";
  o << "constexpr int NTG = " << nt << ", TILE = " << (1 << H->T) << ";\n";
  o << "extern \"C\" __global__ void __launch_bounds__(" << 2 * nt << ", " << std::max(1, 512 / (2 * nt))
    << ") sv_sec(V* __restrict__ psi, V* __restrict__ psi_hi, const V* __restrict__ aux, int split_a, int split_b, "
    << "long long vidx, "
    << coef_param_decl_impl(L, dbl) << ") {\n";
  o << "  extern __shared__ __align__(128) unsigned char smem_raw[];\n"
    << "  V* const bufs = reinterpret_cast<V*>(smem_raw);\n"
    << "  V* const ctaf_all = bufs + 3 * TILE;\n"
    << "  int* const done = reinterpret_cast<int*>(ctaf_all + " << kPipeSetsBytes << ");\n"
    << "  const int grp = threadIdx.x / NTG, tid = threadIdx.x % NTG, bar = 1 + grp;\n"
    << "  V* const ctaf = ctaf_all + grp * " << 5 * SV_MAX_SETS << ";\n"
    << "  (void)ctaf; (void)aux; (void)vidx; (void)psi_hi;\n"
    << "  constexpr unsigned long long NTILES = 1ull << " << H->n_out << ";\n";
  g.arr("int", "OB", H->out_bits, H->n_out);
  o << "  auto tile_of = [&](uint64_t t) {\n    uint64_t r = 0;\n#pragma unroll\n    for (int j = 0; j < "
    << H->n_out << "; j++) r |= ((t >> j) & 1ull) << OB[j];\n    return r;\n  };\n"
    << "  auto blk_of = [&](long long j) { return (uint64_t)blockIdx.x + (uint64_t)j * gridDim.x; };\n";
  {  // load map: thread part of the HBM offset and of the swizzled smem offset (tile-invariant)
    long long ro[16];
    int w[16];
    for (int k = 0; k < 16; k++) {
      ro[k] = 0;
      w[k] = 0;
      for (int s = 0; s < SV_R_BITS; s++)
        if ((k >> s) & 1) {
          ro[k] |= 1ll << H->load.rmb[s];
          w[k] ^= H->load.rw[s];
        }
    }
    g.arr("int", "LTMB", H->load.tmb, g.ntl);
    g.arr("int", "LTW", H->load.tw, g.ntl);
    g.arr("long long", "LRO", ro, 16);
    g.arr("int", "LW", w, 16);
  }
  o << "  uint64_t lb = 0;\n  int lx = 0;\n#pragma unroll\n  for (int j = 0; j < " << g.ntl
    << "; j++) {\n    lb |= (uint64_t)((tid >> j) & 1) << LTMB[j];\n    lx ^= ((tid >> j) & 1) ? LTW[j] : 0;\n  }\n";
  o << "  auto issue = [&](long long j) {\n    V* dst = bufs + (int)(j % 3) * TILE;\n"
    << "    const V* src = psi + (tile_of(blk_of(j)) | lb);\n#pragma unroll\n"
    << "    for (int k = 0; k < 16; k++) cp_async_v(dst + (lx ^ LW[k]), src + LRO[k]);\n    cp_async_commit();\n  };\n";
  o << "  if (threadIdx.x < 3) done[threadIdx.x] = (int)threadIdx.x - 3;  // tile -3 + b 'finished' in buffer b\n"
    << "  __syncthreads();\n"
    << "  long long j = grp;\n  if (blk_of(j) < NTILES) issue(j);\n"
    << "#pragma unroll 1\n"  // keep the tile body single: unrolling it doubles compile time and code
    << "  for (; blk_of(j) < NTILES; j += 2) {\n"
    << "    V* const sm = bufs + (int)(j % 3) * TILE;\n"
    << "    const bool want = blk_of(j + 2) < NTILES;\n"
    << "    int* const nxt_done = done + (int)((j + 2) % 3);\n"
    << "    bool issued = false;\n"
    << "    const uint64_t tile_off = tile_of(blk_of(j));\n";
  if (H->n_sets > 0) {
    o << "    for (int f = tid; f < " << 5 * H->n_sets << "; f += NTG) {\n"
      << "      const int d = c_prog[kH_SETS + f / 5], i = f % 5;\n"
      << "      ctaf[f] = cta_factor<V>(c_prog[d + 2 + i], c_prog[d + 3 + i], tile_off, P);\n    }\n";
  }
  o << "    cp_async_wait<0>();\n    group_sync<NTG>(bar);\n    V v[16];\n";
  const SvPhase* ph = reinterpret_cast<const SvPhase*>(p + H->phase_off);
  const SvOp* ops = reinterpret_cast<const SvOp*>(p + H->op_off);
  for (int k = 0; k < nph; k++) {
    const bool dout = last && k == nph - 1;
    o << "  {  // phase " << k << "\n";
    g.smem(ph[k].tw, ph[k].rw);
    g.lds();
    for (int i = 0; i < ph[k].op_count; i++) {
      const SvOp& op = ops[ph[k].op_begin + i];
      if (!g.diagset_c(p, op, "NTG"))
        o << "    op_c<" << op.type << ", " << op.a << ", " << op.b << ", " << op.coef << ", " << op.extra
          << ">(v, tid, NTG, tile_off, aux, ctaf, P);\n";
    }
    if (dout) {
      o << "    {\n";
      g.hbm(H->dout);
      g.stg();
      o << "    }\n";
    } else {
      g.sts();
      o << "    if (want && !issued) {\n"
        << "      if (group_sync_or<NTG>(bar, ld_volatile(nxt_done) >= j - 1)) {\n"
        << "        issue(j + 2);\n        issued = true;\n      }\n"
        << "    } else {\n      group_sync<NTG>(bar);\n    }\n";
    }
    o << "  }\n";
  }
  if (!last) {
    o << "  {  // gather in store order, lanes walk the lowest store memory bits\n";
    g.smem(H->store.tw, H->store.rw);
    g.lds();
    g.hbm(H->store);
    g.stg();
    o << "  }\n";
  }
  o << "    group_sync<NTG>(bar);  // every read of this buffer is done: release it\n"
    << "    if (tid == 0) st_release(done + (int)(j % 3), (int)j);\n"
    << "    if (want && !issued) {\n"
    << "      while (ld_volatile(nxt_done) < j - 1) {\n      }\n"
    << "      issue(j + 2);\n    }\n"
    << "  }\n}\n";
  return o.str();
}

// ------------------------------------------------------------------------------------ cache
struct Entry {
  std::atomic<int> state{0};  // 0 pending, 1 ready, 2 failed
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kern = nullptr;
  void* c_prog = nullptr;
  size_t c_prog_bytes = 0;
  void* c_coef = nullptr;
  size_t c_coef_bytes = 0;
  uint64_t occ = 0;  // resident CTAs on the device (pipelined variant's grid)
  std::string err;
};

struct Job {
  std::shared_ptr<Entry> e;
  std::string src;
  int dev;
  bool dbl;
};

std::mutex g_mu;
std::unordered_map<std::string, std::shared_ptr<Entry>> g_cache;
JitCounters g_ctr;

// NVRTC: source -> sm_100a cubin (+ the lowered names of the __constant__ arrays)
bool compile_cubin(const std::string& src, bool dbl, std::vector<char>& cubin, std::string& name_prog,
                   std::string& name_coef, std::string& err) {
  Nvrtc& N = nvrtc();
  if (!N.ok) {
    err = "NVRTC (libnvrtc.so.12) not found";
    return false;
  }
  nvrtcProgram prog = nullptr;
  if (N.create(&prog, src.c_str(), "sv_section_jit.cu", kJitHeaderCount, kJitHeaderTexts, kJitHeaderNames) !=
      NVRTC_SUCCESS) {
    err = "nvrtcCreateProgram failed";
    return false;
  }
  const char* sym_prog = "&sv::c_prog";
  const char* sym_coef = dbl ? "&sv::c_coef64" : "&sv::c_coef32";
  N.add_name(prog, sym_prog);
  N.add_name(prog, sym_coef);
  const char* opts[] = {"-arch=sm_100a", "-std=c++17", "-lineinfo", "-DSV_JIT_KERNEL=1"};
  const nvrtcResult rc = N.compile(prog, 4, opts);
  if (rc != NVRTC_SUCCESS) {
    size_t n = 0;
    N.log_size(prog, &n);
    std::string log(n, '\0');
    if (n) N.log(prog, &log[0]);
    err = "NVRTC compile failed: " + log.substr(0, 4000);
    N.destroy(&prog);
    return false;
  }
  size_t nc = 0;
  N.cubin_size(prog, &nc);
  cubin.resize(nc);
  N.cubin(prog, cubin.data());
  const char* lp = nullptr;
  const char* lc = nullptr;
  if (N.lowered(prog, sym_prog, &lp) == NVRTC_SUCCESS && lp) name_prog = lp;
  if (N.lowered(prog, sym_coef, &lc) == NVRTC_SUCCESS && lc) name_coef = lc;
  N.destroy(&prog);
  return true;
}

// On-disk cubin cache (SV_JIT_CACHE=<dir>, default $HOME/.cache/sv_jit; "0" disables): a kernel
// compiled once is reused by later processes.  Key: FNV-1a of the source, the embedded headers
// and the NVRTC options; file: [u32 len][name_prog][u32 len][name_coef][cubin].
std::string cache_dir() {
  static const std::string d = [] {
    const char* e = std::getenv("SV_JIT_CACHE");
    if (e) return std::string(e[0] == '0' && e[1] == '\0' ? "" : e);
    const char* home = std::getenv("HOME");
    return home ? std::string(home) + "/.cache/sv_jit" : std::string();
  }();
  return d;
}
std::string cache_path(const std::string& src, bool dbl) {
  const std::string dir = cache_dir();
  if (dir.empty()) return {};
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](const char* p, size_t n) {
    for (size_t i = 0; i < n; i++) h = (h ^ (unsigned char)p[i]) * 1099511628211ull;
  };
  mix(src.data(), src.size());
  for (int i = 0; i < kJitHeaderCount; i++) mix(kJitHeaderTexts[i], std::strlen(kJitHeaderTexts[i]));
  const char* tag = dbl ? "sm_100a/fp64/v1" : "sm_100a/fp32/v1";
  mix(tag, std::strlen(tag));
  char name[40];
  std::snprintf(name, sizeof(name), "/sv_%016llx.bin", (unsigned long long)h);
  return dir + name;
}
bool cache_load(const std::string& path, std::vector<char>& cubin, std::string& np, std::string& nc) {
  if (path.empty()) return false;
  std::ifstream f(path, std::ios::binary);
  if (!f) return false;
  std::vector<char> all((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  size_t at = 0;
  auto str = [&](std::string& out) {
    uint32_t n = 0;
    if (at + 4 > all.size()) return false;
    std::memcpy(&n, all.data() + at, 4);
    at += 4;
    if (at + n > all.size()) return false;
    out.assign(all.data() + at, n);
    at += n;
    return true;
  };
  if (!str(np) || !str(nc) || at >= all.size()) return false;
  cubin.assign(all.begin() + (long)at, all.end());
  return true;
}
void cache_store(const std::string& path, const std::vector<char>& cubin, const std::string& np,
                 const std::string& nc) {
  if (path.empty()) return;
  const std::string dir = cache_dir();
  for (size_t at = 1; at <= dir.size(); at++)  // mkdir -p
    if (at == dir.size() || dir[at] == '/') ::mkdir(dir.substr(0, at).c_str(), 0755);
  const std::string tmp = path + ".tmp" + std::to_string((long long)::getpid());
  {
    std::ofstream f(tmp, std::ios::binary);
    if (!f) return;
    const uint32_t a = (uint32_t)np.size(), b = (uint32_t)nc.size();
    f.write(reinterpret_cast<const char*>(&a), 4);
    f.write(np.data(), a);
    f.write(reinterpret_cast<const char*>(&b), 4);
    f.write(nc.data(), b);
    f.write(cubin.data(), (std::streamsize)cubin.size());
    if (!f) return;
  }
  std::rename(tmp.c_str(), path.c_str());
}

void build_entry(Entry& e, const std::string& src, int dev, bool dbl) {
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<char> cubin;
  std::string name_prog, name_coef;
  const std::string cpath = cache_path(src, dbl);
  const bool hit = cache_load(cpath, cubin, name_prog, name_coef);
  if (!hit && compile_cubin(src, dbl, cubin, name_prog, name_coef, e.err)) cache_store(cpath, cubin, name_prog, name_coef);
  if (!hit && cubin.empty()) {
    static std::once_flag once;
    std::call_once(once, [&] { std::fprintf(stderr, "[sv] JIT disabled for this kernel: %s\n", e.err.c_str()); });
    e.state = 2;
    return;
  }
  cudaSetDevice(dev);
  cudaError_t ce = cudaLibraryLoadData(&e.lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
  if (ce != cudaSuccess && hit) {  // a damaged cache entry: drop it and compile
    cudaGetLastError();
    std::remove(cpath.c_str());
    cubin.clear();
    if (compile_cubin(src, dbl, cubin, name_prog, name_coef, e.err)) {
      cache_store(cpath, cubin, name_prog, name_coef);
      ce = cudaLibraryLoadData(&e.lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
    }
  }
  if (ce == cudaSuccess) ce = cudaLibraryGetKernel(&e.kern, e.lib, "sv_sec");
  if (ce != cudaSuccess) {
    e.err = std::string("module load failed: ") + cudaGetErrorString(ce);
    cudaGetLastError();
    e.state = 2;
    return;
  }
  if (!name_prog.empty() && cudaLibraryGetGlobal(&e.c_prog, &e.c_prog_bytes, e.lib, name_prog.c_str()) != cudaSuccess)
    e.c_prog = nullptr;
  if (!name_coef.empty() && cudaLibraryGetGlobal(&e.c_coef, &e.c_coef_bytes, e.lib, name_coef.c_str()) != cudaSuccess)
    e.c_coef = nullptr;
  cudaGetLastError();
  const size_t amp = dbl ? 16 : 8;
  ce = cudaFuncSetAttribute(reinterpret_cast<const void*>(e.kern), cudaFuncAttributeMaxDynamicSharedMemorySize,
                            227 * 1024);  // the opt-in maximum; occupancy follows the launch size
  if (ce != cudaSuccess) {
    e.err = std::string("cudaFuncSetAttribute failed: ") + cudaGetErrorString(ce);
    cudaGetLastError();
    e.state = 2;
    return;
  }
  const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  {
    std::lock_guard<std::mutex> lk(g_mu);
    g_ctr.compiled++;
    g_ctr.compile_ms += ms;
  }
  e.state = 1;
}

// background compiler (mode async)
struct Worker {
  std::mutex mu;
  std::condition_variable cv, idle;
  std::deque<Job> q;
  bool stop = false, busy = false;
  std::thread th;
  Worker() {
    th = std::thread([this] {
      for (;;) {
        Job j;
        {
          std::unique_lock<std::mutex> lk(mu);
          cv.wait(lk, [this] { return stop || !q.empty(); });
          if (stop) return;
          j = std::move(q.front());
          q.pop_front();
          busy = true;
        }
        build_entry(*j.e, j.src, j.dev, j.dbl);
        {
          std::lock_guard<std::mutex> lk(mu);
          busy = false;
        }
        idle.notify_all();
      }
    });
  }
  ~Worker() {
    {
      std::lock_guard<std::mutex> lk(mu);
      stop = true;
    }
    cv.notify_all();
    if (th.joinable()) th.join();
  }
  void push(Job j) {
    {
      std::lock_guard<std::mutex> lk(mu);
      q.push_back(std::move(j));
    }
    cv.notify_one();
  }
  void wait() {
    std::unique_lock<std::mutex> lk(mu);
    idle.wait(lk, [this] { return q.empty() && !busy; });
  }
};

Worker& worker() {
  static Worker w;
  return w;
}

}  // namespace

std::string jit_source(const int* prog_host, const Launch& L, bool dbl) { return gen_source(prog_host, L, dbl); }

Status jit_compile_only(const int* prog_host, const Launch& L, bool dbl, const char* dump_dir, int index,
                        double* ms) {
  const auto t0 = std::chrono::steady_clock::now();
  const std::string src = gen_source(prog_host, L, dbl);
  std::vector<char> cubin;
  std::string np, nc, err;
  const bool ok = compile_cubin(src, dbl, cubin, np, nc, err);
  *ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  if (dump_dir) {
    const std::string base = std::string(dump_dir) + "/section_" + std::to_string(index);
    std::ofstream(base + ".cu") << src;
    if (ok) std::ofstream(base + ".cubin", std::ios::binary).write(cubin.data(), (std::streamsize)cubin.size());
  }
  if (!ok) return Status::err(nvrtc().ok ? SV_EMALFORMED : SV_EUNAVAILABLE, err);
  return Status::ok();
}

namespace {
std::string make_key(const int* prog_host, const Launch& L, bool dbl, int dev, bool virt = false) {
  std::string key(reinterpret_cast<const char*>(prog_host), L.int_count * sizeof(int));
  key.push_back(dbl ? 'd' : 'f');
  if (virt) key.push_back('v');
  key.append(reinterpret_cast<const char*>(&dev), sizeof(dev));
  return key;
}
}  // namespace

int jit_set_mode(int m) {
  const int prev = mode();
  if (m >= 0 && m <= 2) g_mode.store(m);
  return prev;
}

bool jit_virtual_input_ok(const Launch& L, bool dbl) {
  return mode() == kSync && L.T >= SV_R_BITS && !pipelined(L, dbl) && !l2_prefetch(L, dbl) &&
         !(L.flags & SV_FLAG_XRANK);
}

void jit_prepare(const Program& prog, bool dbl, bool virt_first) {
  const Mode m = mode();
  if (m == kOff) return;
  int dev = 0;
  cudaGetDevice(&dev);
  std::vector<std::pair<std::shared_ptr<Entry>, std::string>> todo;
  for (size_t li = 0; li < prog.launches.size(); li++) {
    const Launch& L = prog.launches[li];
    if (L.T < SV_R_BITS) continue;
    const bool virt = virt_first && li == 0;
    const int* p = prog.ints.data() + L.int_off;
    std::string key = make_key(p, L, dbl, dev, virt);
    std::shared_ptr<Entry> e;
    {
      std::lock_guard<std::mutex> lk(g_mu);
      if (g_cache.count(key)) continue;
      e = std::make_shared<Entry>();
      g_cache.emplace(std::move(key), e);
    }
    todo.emplace_back(e, gen_source(p, L, dbl, virt));
  }
  if (todo.empty()) return;
  if (m == kAsync) {
    for (auto& t : todo) worker().push(Job{t.first, std::move(t.second), dev, dbl});
    return;
  }
  // sync: compile the missing kernels in parallel (NVRTC is thread-safe per program)
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const unsigned nth = std::min<unsigned>(hw, (unsigned)todo.size());
  std::atomic<size_t> next{0};
  auto run = [&] {
    for (size_t i; (i = next.fetch_add(1)) < todo.size();) build_entry(*todo[i].first, todo[i].second, dev, dbl);
  };
  std::vector<std::thread> th;
  for (unsigned t = 1; t < nth; t++) th.emplace_back(run);
  run();
  for (auto& t : th) t.join();
}

bool jit_launch_section(bool dbl, void* sv, const int* prog_host, const double* coef_host, const Launch& L,
                        const int* prog_dev, const void* coef_dev, const void* aux_dev, cudaStream_t st,
                        cudaError_t* err, int split_a, int split_b, void* sv_hi, int64_t vidx) {
  *err = cudaSuccess;
  const Mode m = mode();
  if (m == kOff || L.T < SV_R_BITS) return false;
  if ((split_a || split_b) && (pipelined(L, dbl) || l2_prefetch(L, dbl))) return false;  // persistent variants
  int dev = 0;
  cudaGetDevice(&dev);
  const bool virt = vidx != -1;
  if (virt && !jit_virtual_input_ok(L, dbl)) return false;
  std::string key = make_key(prog_host, L, dbl, dev, virt);
  std::shared_ptr<Entry> e;
  bool fresh = false;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_cache.find(key);
    if (it == g_cache.end()) {
      e = std::make_shared<Entry>();
      g_cache.emplace(key, e);
      fresh = true;
    } else {
      e = it->second;
    }
  }
  if (fresh) {
    if (m == kSync)
      build_entry(*e, gen_source(prog_host, L, dbl, virt), dev, dbl);
    else
      worker().push(Job{e, gen_source(prog_host, L, dbl, virt), dev, dbl});
  }
  if (e->state.load() != 1) {
    std::lock_guard<std::mutex> lk(g_mu);
    g_ctr.fallbacks++;
    return false;
  }
  const size_t amp = dbl ? 16 : 8;
  if (e->c_prog) {
    if (L.int_count * sizeof(int) > e->c_prog_bytes) return false;
    *err = cudaMemcpyAsync(e->c_prog, prog_dev, L.int_count * sizeof(int), cudaMemcpyDeviceToDevice, st);
    if (*err != cudaSuccess) return true;
  }
  if (e->c_coef && L.coef_count && !coef_in_param(L, dbl)) {
    if (L.coef_count * amp > e->c_coef_bytes) return false;
    *err = cudaMemcpyAsync(e->c_coef, coef_dev, L.coef_count * amp, cudaMemcpyDeviceToDevice, st);
    if (*err != cudaSuccess) return true;
  }
  void* a0 = sv;
  void* a0h = sv_hi ? sv_hi : sv;
  void* a1 = const_cast<void*>(aux_dev);
  int a2 = split_a, a3 = split_b;
  // the coefficient parameter: the section's coefficients (fp64 on the host) in the state's precision
  thread_local std::vector<char> pbuf;
  const size_t nc = L.coef_count ? L.coef_count : 1;
  char empty_bank = 0;
  void* a4 = &empty_bank;  // CoefBank<V>: an empty struct parameter
  if (coef_in_param(L, dbl)) {
    pbuf.assign(nc * amp, 0);
    if (dbl) {
      std::memcpy(pbuf.data(), coef_host, L.coef_count * 16);
    } else {
      float* f = reinterpret_cast<float*>(pbuf.data());
      for (size_t i = 0; i < 2 * L.coef_count; i++) f[i] = (float)coef_host[i];
    }
    a4 = pbuf.data();
  }
  long long av = (long long)vidx;
  void* args[] = {&a0, &a0h, &a1, &a2, &a3, &av, a4};
  const unsigned threads = (pipelined(L, dbl) ? 2u : 1u) << (L.T - SV_R_BITS);
  unsigned grid = (unsigned)(1ull << (L.n_out - (split_a ? 1 : 0) - (split_b ? 1 : 0)));
  if (pipelined(L, dbl) || l2_prefetch(L, dbl)) {  // persistent: one wave of resident CTAs
    if (e->occ == 0) {
      int sms = 0, nb = 0;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, reinterpret_cast<const void*>(e->kern), (int)threads,
                                                        smem_bytes(L, dbl)) != cudaSuccess || nb < 1)
        nb = 1;
      cudaGetLastError();
      e->occ = (uint64_t)nb * (uint64_t)sms;
    }
    const uint64_t pairs = pipelined(L, dbl) ? ((1ull << L.n_out) + 1) / 2 : (1ull << L.n_out);  // two groups per CTA
    grid = (unsigned)std::min<uint64_t>(e->occ, std::max<uint64_t>(1, pairs));
  }
  *err = cudaLaunchKernel(reinterpret_cast<const void*>(e->kern), dim3(grid), dim3(threads), args,
                          smem_bytes(L, dbl), st);
  {
    std::lock_guard<std::mutex> lk(g_mu);
    g_ctr.hits++;
  }
  return true;
}

void jit_wait() {
  if (mode() == kAsync) worker().wait();
}

JitCounters jit_counters() {
  std::lock_guard<std::mutex> lk(g_mu);
  return g_ctr;
}

}  // namespace sv
