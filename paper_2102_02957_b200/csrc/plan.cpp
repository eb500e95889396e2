// plan.cpp — executor mapping of the blocked circuit onto memory bits (host C++).
//
// The paper executes chunk_swaps by moving amplitudes between chunks.
// Here every chunk_swap, and every SWAP inside a section, is a pure RELABEL of sigma (the map
// paper-physical qubit -> memory bit): mem[mu'(y)] = mem[mu(tau_ab(y))] exactly when sigma' is
// sigma with entries a and b exchanged (DESIGN "Executor mapping").  Data moves only when a
// section needs a qubit whose memory bit is a rank bit (>= nL); then that rank bit is
// physically exchanged with a local memory bit no gate of the section uses (the highest such
// bit, so exchanged blocks are contiguous), one grouped exchange per section.
#include <algorithm>
#include <cstring>

#include "common.h"

namespace sv {

namespace {

constexpr int kMaxTileBits = 13;  // one CTA tile: 2^13 amplitudes (128 KiB fp64)

sv_gate to_memory(const sv_gate& t, const std::vector<int>& sigma) {
  sv_gate r = t;
  r.q0 = sigma[t.q0];
  r.q1 = is_two(t.kind) ? sigma[t.q1] : -1;
  return r;
}

struct SectionMapper {
  int n, nL;
  std::vector<int>& sigma;
  std::vector<int> owner;  // owner[m] = paper qubit whose memory bit is m
  std::vector<Step>& steps;
  PlanCounters& ctr;

  SectionMapper(int n_, int nL_, std::vector<int>& s, std::vector<Step>& st, PlanCounters& c)
      : n(n_), nL(nL_), sigma(s), owner(n_), steps(st), ctr(c) {
    for (int p = 0; p < n; p++) owner[sigma[p]] = p;
  }

  void relabel(int a, int b) {  // paper qubits a, b exchange memory bits
    std::swap(sigma[a], sigma[b]);
    owner[sigma[a]] = a;
    owner[sigma[b]] = b;
  }

  void section(const std::vector<sv_gate>& sec) {
    // 1. memory bits the section's non-diagonal gates touch (SWAPs are relabels, walked virtually)
    std::vector<int> v = sigma;
    uint64_t need = 0;
    std::vector<int> rank_bits;  // in order of first use
    for (const sv_gate& t : sec) {
      if (t.kind == SV_SWAP) {
        std::swap(v[t.q0], v[t.q1]);
        continue;
      }
      if (is_diag(t.kind)) continue;
      int bits[2] = {v[t.q0], is_two(t.kind) ? v[t.q1] : -1};
      for (int b : bits) {
        if (b < 0) continue;
        if (!((need >> b) & 1) && b >= nL) rank_bits.push_back(b);
        need |= 1ull << b;
      }
    }
    // 2. bring needed rank bits onto local memory bits (one grouped exchange)
    if (!rank_bits.empty()) {
      Step ex;
      ex.type = Step::EXCHANGE;
      uint64_t taken = need;
      for (int b : rank_bits) {
        int m = nL - 1;
        while (m >= 0 && ((taken >> m) & 1)) m--;
        // m >= 0 is guaranteed: the section needs at most c <= nL local bits in total
        taken |= 1ull << m;
        ex.ex.push_back({m, b});
        relabel(owner[m], owner[b]);
      }
      ctr.exchanges += ex.ex.size();
      ctr.exchange_batches++;
      steps.push_back(std::move(ex));
    }
    // 3. translate the section to memory bits; SWAPs relabel sigma for everything after them
    std::vector<sv_gate> mem;
    for (const sv_gate& t : sec) {
      if (t.kind == SV_SWAP) {
        relabel(t.q0, t.q1);
        continue;
      }
      mem.push_back(to_memory(t, sigma));
    }
    if (mem.empty()) return;
    uint64_t act = 0;
    for (const sv_gate& m : mem)
      if (!is_diag(m.kind)) act |= qmask(m);
    if (__builtin_popcountll(act) <= kMaxTileBits) {
      push_section(std::move(mem));
      return;
    }
    // More active bits than one tile holds (chunk_bits > kMaxTileBits): split the section with
    // the same pass at c = kMaxTileBits on memory bits.  Its chunk_swaps are relabels of an
    // inner frame whose inverse keeps every gate on its own memory bit, so only the grouping is
    // used (each inner section's gates are the originals, by index).
    std::vector<sv_gate> in = mem;
    for (size_t i = 0; i < in.size(); i++) in[i].pad = (int32_t)i;
    std::vector<int> ipi(nL);
    for (int b = 0; b < nL; b++) ipi[b] = b;
    std::vector<sv_gate> toks;
    Status st = block_pass(in.data(), in.size(), nL, kMaxTileBits, ipi, 0, toks);
    if (!st.good()) {  // cannot happen for valid sections; keep the section whole
      push_section(std::move(mem));
      return;
    }
    std::vector<sv_gate> cur;
    for (const sv_gate& t : toks) {
      if (t.kind == SV_BEGIN) {
        cur.clear();
      } else if (t.kind == SV_END) {
        if (!cur.empty()) push_section(std::move(cur));
        cur.clear();
      } else if (t.kind != SV_CHUNK_SWAP) {
        cur.push_back(mem[t.pad]);
      }
    }
  }

  void push_section(std::vector<sv_gate> gates) {
    Step s;
    s.type = Step::SECTION;
    s.gates = std::move(gates);
    ctr.sections++;
    steps.push_back(std::move(s));
  }
};

}  // namespace

Status make_plan(const sv_gate* g, size_t count, int n, int c, int world_log2, std::vector<int>& pi,
                 std::vector<int>& sigma, uint32_t flags, std::vector<Step>& steps, PlanCounters& ctr) {
  const int nL = n - world_log2;
  if (world_log2 < 0 || nL < 1) return Status::err(SV_EINVAL, "world too large for n");
  if (c < 1 || c > nL) return Status::err(SV_EINVAL, "chunk_bits must satisfy 1 <= c <= n - log2(world)");
  if ((int)pi.size() != n || (int)sigma.size() != n) return Status::err(SV_EINVAL, "bad permutation length");
  if (Status s = validate_gates(g, count, n); !s.good()) return s;

  if (flags & SV_UNBLOCKED) {
    // Per-gate baseline: each gate is one step on memory bits mu(q) = sigma[pi[q]].
    for (size_t i = 0; i < count; i++) {
      sv_gate m = g[i];
      m.q0 = sigma[pi[g[i].q0]];
      m.q1 = is_two(g[i].kind) ? sigma[pi[g[i].q1]] : -1;
      m.pad = (int32_t)i;
      if (!is_diag(m.kind) && (m.q0 >= nL || (is_two(m.kind) && m.q1 >= nL)))
        return Status::err(SV_EINFEASIBLE,
                           "unblocked mode: gate " + std::to_string(i) + " acts on a global qubit (needs the pass)");
      Step s;
      s.type = Step::GATE;
      s.gates.push_back(m);
      steps.push_back(std::move(s));
    }
    return Status::ok();
  }

  std::vector<sv_gate> tokens;
  tokens.reserve(count * 2 + 16);
  if (Status s = block_pass(g, count, n, c, pi, flags, tokens); !s.good()) return s;

  SectionMapper mapper(n, nL, sigma, steps, ctr);
  std::vector<sv_gate> sec;
  bool inside = false;
  for (const sv_gate& t : tokens) {
    switch (t.kind) {
      case SV_CHUNK_SWAP:
        mapper.relabel(t.q0, t.q1);
        ctr.chunk_swaps++;
        break;
      case SV_BEGIN:
        sec.clear();
        inside = true;
        break;
      case SV_END:
        if (!inside) return Status::err(SV_EMALFORMED, "END without BEGIN");
        mapper.section(sec);
        inside = false;
        break;
      default:
        sec.push_back(t);
    }
  }
  return Status::ok();
}

}  // namespace sv
