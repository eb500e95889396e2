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
#include <array>
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

typedef int CUresult_sv;  // CUresult (driver API) without including cuda.h

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
// SV_CHECK=1: generated kernels trap on any HBM index outside the shard or shared-memory index
// outside the tile (a debugging build of the section kernels; compute-sanitizer is closed on this
// pool, so the GPU suite is run once with it: DESIGN §12)
bool checked() {
  static const bool on = [] {
    const char* e = std::getenv("SV_CHECK");
    return e && e[0] == '1';
  }();
  return on;
}

size_t smem_bytes(const Launch& L, bool dbl) {
  const size_t amp = dbl ? 16 : 8;
  const bool no_smem = L.n_phases == 1 && (L.flags & SV_FLAG_FIRST_DIRECT) && (L.flags & SV_FLAG_LAST_DIRECT);
  if (L.n_sets) return (amp << L.T) + 5 * SV_MAX_SETS * amp;
  return no_smem ? 0 : amp << L.T;
}

// Resident CTAs per SM the generated kernel is register-budgeted for (launch bounds): 512 threads
// per SM at 128 registers.  Sections without dense gates (QFT-like: butterflies and phases) need
// fewer registers and run 640 threads per SM (QFT30 29.7 -> 29.3 ms); U2 sections would spill there.
// (The four-multiply form of a dense 2-qubit gate — 64 FP64 operations and 32 coefficient loads per
// 4 amplitudes instead of the Gauss form's 60 and 48 — was measured slower: QV33 1880 vs 1754 ms.)
// (384 threads per SM for dense sections, 168 registers: QV28 52.6 vs 46.8 ms, QV33 2015 vs 1744 ms —
// fewer warps lose more than the extra registers gain; 640 spills.)
int resident_ctas(int T, int nt, bool dense) {
  if (T > 12) return 1;
  if (T == 12) return 2;
  return std::max(1, std::min(16, (dense ? 512 : 640) / nt));
}

bool has_dense(const int* p) {
  const SvSecHeader* H = reinterpret_cast<const SvSecHeader*>(p);
  const SvOp* ops = reinterpret_cast<const SvOp*>(p + H->op_off);
  for (int i = 0; i < H->n_ops; i++)
    if (ops[i].type == SV_OP_U2 || ops[i].type == SV_OP_U1) return true;
  return false;
}

// Coefficients as a __grid_constant__ kernel parameter when they fit the 32 KiB parameter space
// (FMAs then read them from the parameter bank); else through a pointer to the handle's device
// copy of the section's coefficients (CoefPtr).
constexpr size_t kParamCoefMax = 31 * 1024;
bool coef_in_param(const Launch& L, bool dbl) { return L.coef_count * (dbl ? 16 : 8) <= kParamCoefMax; }
std::string coef_param_decl_impl(const Launch& L, bool dbl) {
  if (coef_in_param(L, dbl))
    return "const __grid_constant__ CoefParam<V, " + std::to_string(L.coef_count ? L.coef_count : 1) + "> P";
  return "const CoefPtr<V> P";
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
  bool virt = false;  // the tile's input is generated: 1 at shard offset vidx, 0 elsewhere
  void hbm(const SvMap& m) {
    long long ro[16];
    for (int k = 0; k < 16; k++) {
      ro[k] = 0;
      for (int s = 0; s < SV_R_BITS; s++)
        if ((k >> s) & 1) ro[k] |= 1ll << m.rmb[s];
    }
    arr("int", "TMB", m.tmb, ntl);
    arr("long long", "RO", ro, 16);
    o << "    uint64_t b = tile_off;\n"
      << "#pragma unroll\n    for (int j = 0; j < " << ntl << "; j++) b |= (uint64_t)((tid >> j) & 1) << TMB[j];\n";
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
  long long namps = 0;  // checked builds: amplitudes of the shard
  void chk_smem() {
    if (checked())
      o << "#pragma unroll\n    for (int k = 0; k < 16; k++) if ((unsigned)(x ^ W[k]) >= " << (1u << T) << "u) __trap();\n";
  }
  void chk_hbm() {
    if (checked())
      o << "#pragma unroll\n    for (int k = 0; k < 16; k++) if ((unsigned long long)(b + RO[k]) >= " << namps << "ull) __trap();\n";
  }
  void lds() {
    chk_smem();
    o << "#pragma unroll\n    for (int k = 0; k < 16; k++) v[k] = sm[x ^ W[k]];\n";
  }
  void sts() {
    chk_smem();
    o << "#pragma unroll\n    for (int k = 0; k < 16; k++) sm[x ^ W[k]] = v[k];\n";
  }
  void ldg() {
    if (virt) {
      o << "#pragma unroll\n    for (int k = 0; k < 16; k++) { v[k].x = (long long)(b + RO[k]) == vidx ? 1 : 0; v[k].y = 0; }\n";
      return;
    }
    chk_hbm();
    o << "#pragma unroll\n    for (int k = 0; k < 16; k++) v[k] = psi[b + RO[k]];\n";
  }
  void stg() {
    chk_hbm();
    o << "#pragma unroll\n    for (int k = 0; k < 16; k++) psi[b + RO[k]] = v[k];\n";
  }
};

// Per-CTA DIAGSET factors (out-of-tile terms, program.h): the product of each factor's terms is
// emitted as straight-line code with the masks and coefficient offsets as immediates, a balanced
// product tree per factor, one factor per warp (lane 0; warp-uniform branches).  The interpreter's
// loop over the terms (a dependent chain with a constant-bank load per term, 10 threads busy)
// stalled every warp of a QFT tile at the following barrier (ncu: barrier stalls dominant, ADU 28%).
void emit_cta_factors(std::ostringstream& o, const int* p, int nt) {
  const SvSecHeader* H = reinterpret_cast<const SvSecHeader*>(p);
  const int nf = 5 * H->n_sets, nw = std::max(1, nt / 32);
  o << "  if ((tid & 31) == 0) {\n    const V one = cone<V>();\n    (void)one;\n";
  for (int w = 0; w < nw && w < nf; w++) {
    o << "    if ((tid >> 5) == " << w << ") {\n";
    for (int f = w; f < nf; f += nw) {
      const int d = H->set_desc[f / 5], i = f % 5;
      const int b = p[d + 2 + i], e = p[d + 3 + i];
      std::vector<std::string> terms;
      for (int t = b; t < e; t += 3) {
        const unsigned long long M = (unsigned long long)(uint32_t)p[t] | ((unsigned long long)(uint32_t)p[t + 1] << 32);
        terms.push_back("((tile_off & " + std::to_string(M) + "ull) == " + std::to_string(M) + "ull ? P(" +
                        std::to_string(p[t + 2]) + ") : one)");
      }
      if (terms.empty()) {
        o << "      ctaf[" << f << "] = one;\n";
        continue;
      }
      // four interleaved accumulators: short dependency chains, few live registers (the tile's loads
      // are already in flight in 64 registers)
      const size_t na = std::min<size_t>(4, terms.size());
      o << "      {\n";
      for (size_t k = 0; k < na; k++) o << "        V a" << k << " = " << terms[k] << ";\n";
      for (size_t k = na; k < terms.size(); k++) {
        const std::string& t = terms[k];  // "((cond) ? P(i) : one)" -> multiply only where the bits are set
        const size_t q = t.find(" ? ");
        o << "        if (" << t.substr(1, q - 1) << ") a" << (k % na) << " = cmul(a" << (k % na) << ", "
          << t.substr(q + 3, t.find(" : ") - q - 3) << ");\n";
      }
      std::string r = "a0";
      if (na >= 2) r = "cmul(a0, a1)";
      if (na >= 3) r = "cmul(" + r + ", " + (na == 4 ? std::string("cmul(a2, a3)") : std::string("a2")) + ")";
      o << "        ctaf[" << f << "] = " << r << ";\n      }\n";
    }
    o << "    }\n";
  }
  o << "  }\n";
}

std::string gen_source(const int* p, const Launch& L, bool dbl, bool virt = false) {
  const SvSecHeader* H = reinterpret_cast<const SvSecHeader*>(p);
  Gen g;
  g.virt = virt;
  g.T = H->T;
  g.namps = 1ll << (H->T + H->n_out);
  g.ntl = H->T - SV_R_BITS;
  const int nt = 1 << g.ntl;
  const bool first = H->flags & SV_FLAG_FIRST_DIRECT, last = H->flags & SV_FLAG_LAST_DIRECT;
  const int nph = H->n_phases;
  auto& o = g.o;
  // the program itself goes into the module's constant bank (section_dev.cuh SV_JIT_PROG)
  o << "#define SV_JIT_PROG ";
  for (size_t i = 0; i < L.int_count; i++) o << (i ? "," : "") << p[i];
  o << "\n#include \"section_dev.cuh\"\nusing namespace sv;\ntypedef " << (dbl ? "double2" : "float2") << " V;\n";
  o << "extern \"C\" __global__ void __launch_bounds__(" << nt << ", " << resident_ctas(H->T, nt, has_dense(p))
    << ") sv_sec(V* __restrict__ psi, const V* __restrict__ aux, int split_a, int split_b, long long vidx, "
    << "unsigned long long blk0, " << coef_param_decl_impl(L, dbl) << ") {\n";
  o << "  extern __shared__ __align__(16) unsigned char smem_raw[];\n"
    << "  V* sm = reinterpret_cast<V*>(smem_raw);\n"
    << "  V* ctaf = reinterpret_cast<V*>(smem_raw + (sizeof(V) << " << H->T << "));\n"
    << "  (void)sm; (void)ctaf; (void)aux; (void)vidx;\n"
    << "  const int tid = threadIdx.x;\n";
  g.arr("int", "OB", H->out_bits, H->n_out);
  o << "  auto tile_of = [&](uint64_t t) {\n    uint64_t r = 0;\n#pragma unroll\n    for (int j = 0; j < "
    << H->n_out << "; j++) r |= ((t >> j) & 1ull) << OB[j];\n    return r;\n  };\n";
  o << "  {\n  const uint64_t tile_off = tile_of(expand_tile(blockIdx.x + blk0, split_a, split_b));\n";
  // The tile's HBM loads are issued first (phase 0's registers, or the load step's), so their
  // latency overlaps the per-CTA DIAGSET factors computed next.
  o << "  V v[16];\n";
  o << "  {  // " << (first ? "phase 0 reads HBM directly" : "load: lanes walk the lowest load memory bits") << "\n";
  g.hbm(first ? H->din : H->load);
  g.ldg();
  o << "  }\n";
  if (H->n_sets > 0) emit_cta_factors(o, p, nt);
  if (!first) {
    o << "  {  // scatter into the swizzled tile\n";
    g.smem(H->load.tw, H->load.rw);
    g.sts();
    o << "  }\n";
  }
  if (!first || H->n_sets > 0) o << "  __syncthreads();\n";
  const SvPhase* ph = reinterpret_cast<const SvPhase*>(p + H->phase_off);
  const SvOp* ops = reinterpret_cast<const SvOp*>(p + H->op_off);
  for (int k = 0; k < nph; k++) {
    const bool din = first && k == 0, dout = last && k == nph - 1;
    o << "  {  // phase " << k << "\n";
    if (!din || !dout) g.smem(ph[k].tw, ph[k].rw);
    if (!din) g.lds();
    for (int i = 0; i < ph[k].op_count; i++) {
      const SvOp& op = ops[ph[k].op_begin + i];
      if (!g.diagset_c(p, op, std::to_string(nt)))
        // dense gates of a phase fed straight from HBM take the split form (u2_slots SPLIT): with
        // the chained form ptxas interleaves the tile's loads with the first gate and leaves
        // HBM latency exposed
        o << "    op_c<" << op.type << ", " << op.a << ", " << op.b << ", " << op.coef << ", "
          << (op.type == SV_OP_U2 ? (din ? 1 : 0) : op.extra) << ">(v, tid, " << nt << ", tile_off, aux, ctaf, P);\n";
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
  o << "  }\n}\n";
  return o.str();
}

// ------------------------------------------------------------------------------- TMA variant
// Tile loads by the Tensor Memory Accelerator (cp.async.bulk.tensor, SASS UTMALDG) — an opt-in
// variant (SV_TMA), measured slower than the plain kernel (QFT30 7.39 vs 6.65 ms per
// section before the DIAGSET prologue fix; only 3 tiles per SM compute at a time).  The shard is
// described to the TMA as a tensor of up to 5 dimensions cut at the starts of the tile's runs of
// consecutive memory bits, so one box (2^w0 x ... amplitudes, rows of >= 128 bytes) is a whole
// tile, or 2^E boxes when more runs than dimensions remain (E "enumerated" tile bits).  A
// persistent CTA keeps a ring of S tile slots: while it computes tile j in slot j % S, the TMA
// fills the slots of tiles j + 1 .. j + S - 1 (mbarrier transaction counts), so HBM reads run
// continuously instead of in the load phase of each CTA (microbench: this gather pattern reaches
// 5.8 TB/s read + write with a 2-3 slot ring vs 5.2 TB/s for LDG at the section kernel's 7
// resident 32 KiB tiles per SM).  The box lands in "natural" order (tile position p at smem bit
// nat[p]); the first step reads it with lanes on the lowest memory bits (conflict-free) and, after
// a CTA barrier, writes the swizzled layout of the phases into the same slot.
struct TmaPlan {
  bool ok = false;
  int D = 0;                      // tensor dimensions (1..5)
  int lo[5] = {}, span[5] = {}, w[5] = {};  // dim d: memory bits [lo, lo + span); box: bits [lo, lo + w)
  int E = 0;                      // enumerated tile bits (2^E boxes per tile)
  int ebits[8] = {};
  int nat[16] = {};               // tile position -> smem index bit of the natural layout
  int boxbits = 0;
};

// SV_TMA (opt-in, measured slower — DESIGN §6): 0 off (default); 1 / 2: the TMA-fed slot ring for
// sections without dense gates / for every section with a tile of <= 11 bits
int tma_mode() {
  static const int m = [] {
    const char* e = std::getenv("SV_TMA");
    return e ? std::atoi(e) : 0;
  }();
  return m;
}
constexpr int kTmaSlots = 2;

TmaPlan tma_plan(const int* p, const Launch& L, bool dbl) {
  TmaPlan P;
  const SvSecHeader* H = reinterpret_cast<const SvSecHeader*>(p);
  const int T = H->T, nL = H->T + H->n_out;
  const int md = tma_mode();
  if (md == 0 || T < SV_R_BITS || T > 11) return P;
  if (md == 1 && has_dense(p)) return P;
  if (kTmaSlots * (size_t(dbl ? 16 : 8) << T) + 5 * SV_MAX_SETS * 16 + 64 > 227 * 1024) return P;
  (void)L;
  const int* tb = H->tile_bits;
  const int G = dbl ? 3 : 4;  // rows of >= 128 bytes
  if (tb[0] != 0) return P;
  std::vector<std::pair<int, int>> runs;  // (first bit, length)
  for (int j = 0; j < T; j++) {
    if (j == 0 || tb[j] != tb[j - 1] + 1)
      runs.push_back({tb[j], 1});
    else
      runs.back().second++;
  }
  if (runs[0].second < G) return P;
  std::vector<std::pair<int, int>> pieces;  // box limit: 256 elements per dimension
  for (size_t r = 0; r < runs.size(); r++) {
    int st = runs[r].first, len = runs[r].second;
    int cap = r == 0 ? 7 : 8;  // dim 0 counts 2 elements (re, im) per amplitude
    while (len > 0) {
      const int l = std::min(len, cap);
      pieces.push_back({st, l});
      st += l;
      len -= l;
      cap = 8;
    }
  }
  std::vector<int> order(pieces.size());
  for (size_t i = 0; i < order.size(); i++) order[i] = (int)i;
  std::stable_sort(order.begin() + 1, order.end(), [&](int a, int b) { return pieces[a].second > pieces[b].second; });
  std::vector<std::pair<int, int>> box;
  for (size_t i = 0; i < order.size() && box.size() < 5; i++) box.push_back(pieces[order[i]]);
  std::sort(box.begin(), box.end());
  int E = 0;
  for (size_t i = 0; i < order.size(); i++) {
    const auto& pc = pieces[order[i]];
    if (std::find(box.begin(), box.end(), pc) != box.end()) continue;
    for (int b = 0; b < pc.second; b++) {
      if (E >= 4) return P;  // at most 16 boxes per tile
      P.ebits[E++] = pc.first + b;
    }
  }
  std::sort(P.ebits, P.ebits + E);
  // dimension spans: from each box's first bit to the next box's (the top one to nL); a span the
  // tensor map cannot describe in one dimension (2^32 elements) gets an extra box-width-0 dimension
  std::vector<std::array<int, 3>> dims;  // lo, span, w
  for (size_t i = 0; i < box.size(); i++) {
    const int lo = box[i].first, hi = i + 1 < box.size() ? box[i + 1].first : nL;
    dims.push_back({lo, hi - lo, box[i].second});
  }
  for (size_t i = 0; i < dims.size(); i++) {
    const int lim = i == 0 ? 31 : 32;
    if (dims[i][1] > lim) {
      if (dims.size() >= 5) return P;
      const int cut = dims[i][0] + std::max(dims[i][2], dims[i][1] / 2);
      const std::array<int, 3> extra = {cut, dims[i][0] + dims[i][1] - cut, 0};
      dims[i][1] = cut - dims[i][0];
      dims.insert(dims.begin() + i + 1, extra);
      i = (size_t)-1;  // re-check from the start
    }
  }
  P.D = (int)dims.size();
  int acc = 0;
  for (int d = 0; d < P.D; d++) {
    P.lo[d] = dims[d][0];
    P.span[d] = dims[d][1];
    P.w[d] = dims[d][2];
    acc += P.w[d];
  }
  P.boxbits = acc;
  P.E = E;
  // natural layout: box bits in dimension order, then the enumerated bits
  for (int pos = 0; pos < T; pos++) {
    const int m = tb[pos];
    int bit = -1, base = 0;
    for (int d = 0; d < P.D; d++) {
      if (m >= P.lo[d] && m < P.lo[d] + P.w[d]) bit = base + (m - P.lo[d]);
      base += P.w[d];
    }
    for (int i = 0; i < E; i++)
      if (P.ebits[i] == m) bit = P.boxbits + i;
    if (bit < 0) return TmaPlan();
    P.nat[pos] = bit;
  }
  P.ok = true;
  return P;
}

// the 2^E boxes of the tile at amplitude offset `base`, each handed to `call`<D>(&tm, c[, ...])
void emit_tma_coords(std::ostringstream& o, const TmaPlan& TP, const char* base, const char* call) {
  o << "    const uint64_t a0 = " << base << ";\n";
  o << "#pragma unroll\n    for (int e = 0; e < " << (1 << TP.E) << "; e++) {\n      uint64_t a = a0;\n";
  for (int i = 0; i < TP.E; i++) o << "      if ((e >> " << i << ") & 1) a |= 1ull << " << TP.ebits[i] << ";\n";
  o << "      int c[5] = {0, 0, 0, 0, 0};\n";
  for (int d = 0; d < TP.D; d++) {
    const unsigned long long mask = (TP.span[d] >= 64) ? ~0ull : ((1ull << TP.span[d]) - 1);
    if (d == 0)
      o << "      c[0] = (int)(2 * (a & " << mask << "ull));\n";
    else
      o << "      c[" << d << "] = (int)((a >> " << TP.lo[d] << ") & " << mask << "ull);\n";
  }
  o << "      " << call << "<" << TP.D << ">(slots + s * TILE + e * BOX, &tm, c[0], c[1], c[2], c[3], c[4], &bar[s]);\n    }\n";
}

int tma_ctas_per_sm(const Launch& L, bool dbl) {
  const size_t bytes = kTmaSlots * (size_t(dbl ? 16 : 8) << L.T) + 5 * SV_MAX_SETS * (dbl ? 16 : 8) + 64;
  return (int)std::max<size_t>(1, std::min<size_t>(8, (228 * 1024) / (bytes + 1024)));
}
size_t tma_smem_bytes(const Launch& L, bool dbl) {
  return kTmaSlots * (size_t(dbl ? 16 : 8) << L.T) + 5 * SV_MAX_SETS * (dbl ? 16 : 8) + 64;
}

std::string gen_source_tma(const int* p, const Launch& L, bool dbl, const TmaPlan& TP) {
  const SvSecHeader* H = reinterpret_cast<const SvSecHeader*>(p);
  Gen g;
  g.T = H->T;
  g.namps = 1ll << (H->T + H->n_out);
  g.ntl = H->T - SV_R_BITS;
  const int nt = 1 << g.ntl;
  const bool first = H->flags & SV_FLAG_FIRST_DIRECT, last = H->flags & SV_FLAG_LAST_DIRECT;
  const int nph = H->n_phases;
  const int T = H->T;
  auto& o = g.o;
  int pos_of[64];
  std::fill(pos_of, pos_of + 64, -1);
  for (int j = 0; j < T; j++) pos_of[H->tile_bits[j]] = j;
  // natural-layout words of a boundary map (thread bit j / register slot s -> 1 << nat bit)
  auto nat_map = [&](const SvMap& m) {
    int tw[16], rw[SV_R_BITS];
    for (int j = 0; j < g.ntl; j++) tw[j] = 1 << TP.nat[pos_of[m.tmb[j]]];
    for (int s2 = 0; s2 < SV_R_BITS; s2++) rw[s2] = 1 << TP.nat[pos_of[m.rmb[s2]]];
    g.smem(tw, rw);
  };
  o << "#define SV_JIT_PROG ";
  for (size_t i = 0; i < L.int_count; i++) o << (i ? "," : "") << p[i];
  o << "\n#include \"section_dev.cuh\"\nusing namespace sv;\ntypedef " << (dbl ? "double2" : "float2") << " V;\n";
  o << "constexpr int S = " << kTmaSlots << ", TILE = " << (1 << T) << ", BOX = " << (1 << TP.boxbits) << ";\n";
  o << "extern \"C\" __global__ void __launch_bounds__(" << nt << ", " << tma_ctas_per_sm(L, dbl)
    << ") sv_sec(V* __restrict__ psi, const V* __restrict__ aux, int split_a, int split_b, long long vidx, "
    << "const __grid_constant__ SvTmap tm, unsigned long long ntiles, " << coef_param_decl_impl(L, dbl) << ") {\n";
  o << "  extern __shared__ __align__(1024) unsigned char smem_raw[];\n"
    << "  V* const slots = reinterpret_cast<V*>(smem_raw);\n"
    << "  V* const ctaf = reinterpret_cast<V*>(smem_raw + S * TILE * sizeof(V));\n"
    << "  uint64_t* const bar = reinterpret_cast<uint64_t*>(smem_raw + S * TILE * sizeof(V) + " << 5 * SV_MAX_SETS
    << " * sizeof(V));\n"
    << "  (void)ctaf; (void)aux; (void)vidx;\n"
    << "  const int tid = threadIdx.x;\n";
  g.arr("int", "OB", H->out_bits, H->n_out);
  o << "  auto tile_of = [&](uint64_t t) {\n    uint64_t r = 0;\n#pragma unroll\n    for (int j = 0; j < "
    << H->n_out << "; j++) r |= ((t >> j) & 1ull) << OB[j];\n    return r;\n  };\n";
  o << "  if (tid == 0) {\n    for (int s = 0; s < S; s++) mbar_init(&bar[s], 1);\n    mbar_init_fence();\n  }\n"
    << "  __syncthreads();\n";
  // the issue of one tile: 2^E boxes, coordinates from the tile's amplitude offset
  o << "  auto issue = [&](uint64_t b, int s) {\n"
    << "    fence_proxy_async();\n"
    << "    mbar_expect_tx(&bar[s], TILE * (uint32_t)sizeof(V));\n";
  emit_tma_coords(o, TP, "tile_of(expand_tile(b, split_a, split_b))", "tma_load");
  o << "  };\n";
  o << "  if (tid == 0)\n    for (int i = 0; i < S - 1; i++) {\n"
    << "      const uint64_t b = blockIdx.x + (uint64_t)i * gridDim.x;\n      if (b < ntiles) issue(b, i);\n    }\n";
  o << "  uint32_t j = 0;\n#pragma unroll 1\n"
    << "  for (uint64_t blk = blockIdx.x; blk < ntiles; blk += gridDim.x, j++) {\n"
    << "    const int s = (int)(j % S);\n"
    << "    if (tid == 0) {\n      const uint64_t bn = blk + (uint64_t)(S - 1) * gridDim.x;\n"
    << "      if (bn < ntiles) issue(bn, (int)((j + S - 1) % S));\n    }\n"
    << "    const uint64_t tile_off = tile_of(expand_tile(blk, split_a, split_b));\n"
    << "    V* const sm = slots + s * TILE;\n";
  if (H->n_sets > 0) {
    emit_cta_factors(o, p, nt);
    o << "    __syncthreads();\n";
  }
  o << "    mbar_wait_parity(&bar[s], (j / S) & 1);\n";
  o << "    V v[16];\n";
  const SvPhase* ph = reinterpret_cast<const SvPhase*>(p + H->phase_off);
  const SvOp* ops = reinterpret_cast<const SvOp*>(p + H->op_off);
  if (!first) {
    o << "    {  // the staged tile (natural order), lanes on the lowest load memory bits -> swizzled layout\n";
    nat_map(H->load);
    g.lds();
    o << "    }\n    __syncthreads();\n    {\n";
    g.smem(H->load.tw, H->load.rw);
    g.sts();
    o << "    __syncthreads();\n    }\n";
  }
  for (int k = 0; k < nph; k++) {
    const bool din = first && k == 0, dout = last && k == nph - 1;
    o << "    {  // phase " << k << "\n";
    if (din) {
      o << "    {\n";
      nat_map(H->din);
      g.lds();
      o << "    }\n";
    } else {
      g.smem(ph[k].tw, ph[k].rw);
      g.lds();
    }
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
      if (din) {  // every thread has read the natural layout before the slot is rewritten
        o << "    __syncthreads();\n";
        g.smem(ph[k].tw, ph[k].rw);
      }
      g.sts();
      o << "    __syncthreads();\n";
    }
    o << "    }\n";
  }
  if (!last) {
    o << "    {  // gather in store order, lanes walk the lowest store memory bits\n";
    g.smem(H->store.tw, H->store.rw);
    g.lds();
    g.hbm(H->store);
    g.stg();
    o << "    }\n";
  }
  o << "    __syncthreads();  // slot s is free for the tile S - 1 ahead\n  }\n}\n";
  return o.str();
}

// host side: encode the tensor map of a launch's tile gather over the shard at sv
typedef CUresult_sv (*EncodeTiledFn)(void*, int, unsigned, void*, const uint64_t*, const uint64_t*, const uint32_t*,
                                      const uint32_t*, int, int, int, int);
EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    cudaGetLastError();
    return reinterpret_cast<EncodeTiledFn>(f);
  }();
  return fn;
}
bool encode_tmap(const TmaPlan& P, bool dbl, void* sv, unsigned char (&out)[128]) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return false;
  uint64_t dims[5], strides[4];
  uint32_t box[5], es[5];
  const uint64_t amp = dbl ? 16 : 8;
  for (int d = 0; d < P.D; d++) {
    dims[d] = (d == 0 ? 2ull : 1ull) << P.span[d];
    box[d] = (d == 0 ? 2u : 1u) << P.w[d];
    es[d] = 1;
    if (d > 0) strides[d - 1] = amp << P.lo[d];
  }
  // CU_TENSOR_MAP_DATA_TYPE_FLOAT64 = 8, FLOAT32 = 7; interleave none = 0, swizzle none = 0,
  // L2 promotion 256B = 3, oob fill none = 0
  const int r = enc(out, dbl ? 8 : 7, (unsigned)P.D, sv, dims, strides, box, es, 0, 0, 3, 0);
  return r == 0;
}

// ------------------------------------------------------------------------------------ cache
struct Entry {
  std::atomic<int> state{0};  // 0 pending, 1 ready, 2 failed
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kern = nullptr;
  std::string err;
  bool tma = false;  // the TMA-fed persistent variant (gen_source_tma), with its tile plan
  TmaPlan tp;
  std::atomic<int> occ{0};  // resident CTAs on the device of the TMA variant (its persistent grid)
};

// The source of a launch's kernel; decides (once, at entry creation) between the TMA-fed
// persistent variant and the plain one.  A launch that generates its input (vidx) reads nothing.
std::string source_for(const int* p, const Launch& L, bool dbl, bool virt, Entry& e) {
  if (!virt) {
    e.tp = tma_plan(p, L, dbl);
    e.tma = e.tp.ok;
  }
  if (e.tma) return gen_source_tma(p, L, dbl, e.tp);
  return gen_source(p, L, dbl, virt);
}

struct Job {
  std::shared_ptr<Entry> e;
  std::string src;
  int dev;
  bool dbl;
};

std::mutex g_mu;
std::unordered_map<std::string, std::shared_ptr<Entry>> g_cache;
JitCounters g_ctr;

const char* const kNvrtcOpts[] = {"-arch=sm_100a", "-std=c++17", "-lineinfo", "-DSV_JIT_KERNEL=1"};
constexpr int kNvrtcNopts = 4;
constexpr const char* kAbiTag = "sv_sec/abi-4";  // bump when the generated kernel's parameters change

// NVRTC: source -> sm_100a cubin
bool compile_cubin(const std::string& src, std::vector<char>& cubin, std::string& err) {
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
  const nvrtcResult rc = N.compile(prog, kNvrtcNopts, kNvrtcOpts);
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
  N.destroy(&prog);
  return true;
}

// On-disk cubin cache (SV_JIT_CACHE=<dir>, default $HOME/.cache/sv_jit; "0" disables): a kernel
// compiled once is reused by later processes.  The key is a 128-bit hash (two FNV-1a streams) of
// everything that determines the cubin: the generated source, the embedded headers, the NVRTC
// options and version, the precision and an ABI tag.  The file stores the key again and the
// source length, both checked on load, so a foreign or stale file is recompiled, never launched.
std::string cache_dir() {
  static const std::string d = [] {
    const char* e = std::getenv("SV_JIT_CACHE");
    if (e) return std::string(e[0] == '0' && e[1] == '\0' ? "" : e);
    const char* home = std::getenv("HOME");
    return home ? std::string(home) + "/.cache/sv_jit" : std::string();
  }();
  return d;
}
struct CacheKey {
  uint64_t h1 = 1469598103934665603ull, h2 = 0x84222325cbf29ce4ull;
  void mix(const void* data, size_t n) {
    const unsigned char* p = static_cast<const unsigned char*>(data);
    for (size_t i = 0; i < n; i++) {
      h1 = (h1 ^ p[i]) * 1099511628211ull;
      h2 = (h2 ^ p[i]) * 0x100000001b3ull + 0x9E3779B97F4A7C15ull;
    }
  }
  void mix(const char* z) { mix(z, std::strlen(z) + 1); }
};
CacheKey cache_key(const std::string& src, bool dbl) {
  CacheKey k;
  k.mix(src.data(), src.size());
  for (int i = 0; i < kJitHeaderCount; i++) k.mix(kJitHeaderTexts[i]);
  for (int i = 0; i < kNvrtcNopts; i++) k.mix(kNvrtcOpts[i]);
  k.mix(kAbiTag);
  k.mix(dbl ? "fp64" : "fp32");
  int ver[2] = {0, 0};
  typedef nvrtcResult (*VerFn)(int*, int*);
  static VerFn vf = [] {
    void* h = dlopen("libnvrtc.so.12", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("/usr/local/cuda/lib64/libnvrtc.so.12", RTLD_NOW | RTLD_NOLOAD);
    return h ? reinterpret_cast<VerFn>(dlsym(h, "nvrtcVersion")) : nullptr;
  }();
  if (vf) vf(&ver[0], &ver[1]);
  k.mix(ver, sizeof(ver));
  return k;
}
std::string cache_path(const CacheKey& k) {
  const std::string dir = cache_dir();
  if (dir.empty()) return {};
  char name[64];
  std::snprintf(name, sizeof(name), "/sv_%016llx%016llx.bin", (unsigned long long)k.h1, (unsigned long long)k.h2);
  return dir + name;
}
// file: [u64 h1][u64 h2][u64 source length][cubin]
bool cache_load(const std::string& path, const CacheKey& k, size_t src_len, std::vector<char>& cubin) {
  if (path.empty()) return false;
  std::ifstream f(path, std::ios::binary);
  if (!f) return false;
  std::vector<char> all((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  if (all.size() <= 24) return false;
  uint64_t hdr[3];
  std::memcpy(hdr, all.data(), 24);
  if (hdr[0] != k.h1 || hdr[1] != k.h2 || hdr[2] != (uint64_t)src_len) return false;
  cubin.assign(all.begin() + 24, all.end());
  return true;
}
void cache_store(const std::string& path, const CacheKey& k, size_t src_len, const std::vector<char>& cubin) {
  if (path.empty()) return;
  const std::string dir = cache_dir();
  for (size_t at = 1; at <= dir.size(); at++)  // mkdir -p
    if (at == dir.size() || dir[at] == '/') ::mkdir(dir.substr(0, at).c_str(), 0755);
  const std::string tmp = path + ".tmp" + std::to_string((long long)::getpid()) + "_" +
                          std::to_string((unsigned long long)std::hash<std::thread::id>()(std::this_thread::get_id()));
  {
    std::ofstream f(tmp, std::ios::binary);
    if (!f) return;
    const uint64_t hdr[3] = {k.h1, k.h2, (uint64_t)src_len};
    f.write(reinterpret_cast<const char*>(hdr), 24);
    f.write(cubin.data(), (std::streamsize)cubin.size());
    if (!f) return;
  }
  std::rename(tmp.c_str(), path.c_str());
}

void build_entry(Entry& e, const std::string& src, int dev, bool dbl) {
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<char> cubin;
  const CacheKey key = cache_key(src, dbl);
  const std::string cpath = cache_path(key);
  const bool hit = cache_load(cpath, key, src.size(), cubin);
  if (!hit && compile_cubin(src, cubin, e.err)) cache_store(cpath, key, src.size(), cubin);
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
    if (compile_cubin(src, cubin, e.err)) {
      cache_store(cpath, key, src.size(), cubin);
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

// Mode sync: another thread (another rank of a local world, jit_prepare of another handle) may be
// compiling this entry right now; wait for it instead of falling back to the interpreter.
void wait_ready(const Entry& e) {
  while (e.state.load() == 0) std::this_thread::sleep_for(std::chrono::microseconds(200));
}

}  // namespace

std::string jit_source(const int* prog_host, const Launch& L, bool dbl) {
  Entry tmp;
  return source_for(prog_host, L, dbl, false, tmp);
}

Status jit_compile_only(const int* prog_host, const Launch& L, bool dbl, const char* dump_dir, int index,
                        double* ms) {
  const auto t0 = std::chrono::steady_clock::now();
  Entry tmp;
  const std::string src = source_for(prog_host, L, dbl, false, tmp);
  std::vector<char> cubin;
  std::string err;
  const bool ok = compile_cubin(src, cubin, err);
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
  (void)dbl;
  return mode() == kSync && L.T >= SV_R_BITS;
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
    todo.emplace_back(e, source_for(p, L, dbl, virt, *e));
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
                        const void* coef_dev, const void* aux_dev, cudaStream_t st, cudaError_t* err, int split_a,
                        int split_b, int64_t vidx, int64_t only_tile) {
  *err = cudaSuccess;
  const Mode m = mode();
  if (m == kOff || L.T < SV_R_BITS) return false;
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
    std::string src = source_for(prog_host, L, dbl, virt, *e);
    if (m == kSync)
      build_entry(*e, src, dev, dbl);
    else
      worker().push(Job{e, std::move(src), dev, dbl});
  } else if (m == kSync) {
    wait_ready(*e);
  }
  if (e->state.load() != 1) {
    std::lock_guard<std::mutex> lk(g_mu);
    g_ctr.fallbacks++;
    return false;
  }
  const size_t amp = dbl ? 16 : 8;
  void* a0 = sv;
  void* a1 = const_cast<void*>(aux_dev);
  int a2 = split_a, a3 = split_b;
  long long av = (long long)vidx;
  // the coefficient parameter: the section's coefficients (fp64 on the host) in the state's precision,
  // or a pointer to the handle's device copy (already in the state's precision)
  thread_local std::vector<char> pbuf;
  const size_t nc = L.coef_count ? L.coef_count : 1;
  const void* coef_ptr = coef_dev;
  void* a4 = &coef_ptr;
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
  const unsigned threads = 1u << (L.T - SV_R_BITS);
  const unsigned long long ntiles = 1ull << (L.n_out - (split_a ? 1 : 0) - (split_b ? 1 : 0));
  if (e->tma) {
    alignas(64) unsigned char tmap[128];
    if (!encode_tmap(e->tp, dbl, sv, tmap)) {
      *err = cudaErrorInvalidValue;
      return true;
    }
    if (e->occ <= 0) {  // resident CTAs on the device (first launch of this kernel)
      int nb = 0, sms = 0;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, reinterpret_cast<const void*>(e->kern), (int)threads,
                                                        tma_smem_bytes(L, dbl)) != cudaSuccess ||
          nb < 1)
        nb = 1;
      cudaGetLastError();
      e->occ = nb * sms;
    }
    unsigned long long nt = ntiles;
    void* args[] = {&a0, &a1, &a2, &a3, &av, tmap, &nt, a4};
    const unsigned grid = (unsigned)std::min<unsigned long long>(ntiles, (unsigned long long)e->occ);
    *err = cudaLaunchKernel(reinterpret_cast<const void*>(e->kern), dim3(grid), dim3(threads), args,
                            tma_smem_bytes(L, dbl), st);
  } else {
    unsigned long long blk0 = only_tile >= 0 ? (unsigned long long)only_tile : 0ull;
    void* args[] = {&a0, &a1, &a2, &a3, &av, &blk0, a4};
    *err = cudaLaunchKernel(reinterpret_cast<const void*>(e->kern), dim3(only_tile >= 0 ? 1u : (unsigned)ntiles),
                            dim3(threads), args, smem_bytes(L, dbl), st);
  }
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
