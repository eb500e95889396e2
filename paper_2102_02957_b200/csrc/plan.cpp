// plan.cpp — executor mapping of the blocked circuit onto memory bits (host C++).
//
// The paper executes chunk_swaps by moving amplitudes between chunks.
// Here every chunk_swap, and every SWAP inside a section, is a pure RELABEL of sigma (the map
// paper-physical qubit -> memory bit): mem[mu'(y)] = mem[mu(tau_ab(y))] exactly when sigma' is
// sigma with entries a and b exchanged (DESIGN "Executor mapping").  Data moves only
//   * when a section needs a qubit whose memory bit is a rank bit (>= nL): that rank
//     bit is exchanged with a local memory bit no gate of the section uses (EXCHANGE step);
//   * to keep section tiles coalesced: every tile should contain the lowest memory bits.  The
//     planner looks one section ahead and fuses bit swaps into the current section's store so
//     the next section's qubits land on low memory bits (free: same addresses, permuted); when a
//     section still cannot hold its qubits plus the low bits, a standalone swap pass moves them
//     (COMPACT step).  A physical swap of memory bits plus the matching relabel of sigma leaves
//     the logical state unchanged, so none of this changes what the circuit computes.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "common.h"

namespace sv {

namespace {

constexpr int SV_R_BITS_PLAN = 4;  // register qubits per phase (program.h SV_R_BITS)

sv_gate to_memory(const sv_gate& t, const std::vector<int>& sigma) {
  sv_gate r = t;
  r.q0 = sigma[t.q0];
  r.q1 = is_two(t.kind) ? sigma[t.q1] : -1;
  return r;
}

struct Block {
  std::vector<std::pair<int, int>> relabels;  // chunk_swaps (paper qubits) before the section
  std::vector<sv_gate> gates;                  // section gates on paper qubits
};

struct Planner {
  int n, nL;
  const PlanLayout& L;
  std::vector<int>& sigma;
  std::vector<int> owner;  // owner[m] = paper qubit whose memory bit is m
  std::vector<Step>& steps;
  PlanCounters& ctr;

  Planner(int n_, int nL_, const PlanLayout& lay, std::vector<int>& s, std::vector<Step>& st, PlanCounters& c)
      : n(n_), nL(nL_), L(lay), sigma(s), owner(n_), steps(st), ctr(c) {
    for (int p = 0; p < n; p++) owner[sigma[p]] = p;
  }

  void relabel(int a, int b) {  // paper qubits a, b exchange memory bits
    std::swap(sigma[a], sigma[b]);
    owner[sigma[a]] = a;
    owner[sigma[b]] = b;
  }
  void swap_bits(int m1, int m2) { relabel(owner[m1], owner[m2]); }  // after a physical swap

  // Memory bits the block's non-diagonal gates touch under the map v (SWAPs walked virtually),
  // and the rank bits among them in order of first use.
  static uint64_t needed(const Block& b, std::vector<int> v, int nL, std::vector<int>* rank_bits) {
    uint64_t need = 0;
    for (const sv_gate& t : b.gates) {
      if (t.kind == SV_SWAP) {
        std::swap(v[t.q0], v[t.q1]);
        continue;
      }
      if (is_diag(t.kind)) continue;
      const int bits[2] = {v[t.q0], is_two(t.kind) ? v[t.q1] : -1};
      for (int bb : bits) {
        if (bb < 0) continue;
        if (rank_bits && !((need >> bb) & 1) && bb >= nL) rank_bits->push_back(bb);
        need |= 1ull << bb;
      }
    }
    return need;
  }

  void run(const std::vector<Block>& blocks) {
    for (size_t i = 0; i < blocks.size(); i++) {
      for (const auto& rl : blocks[i].relabels) relabel(rl.first, rl.second);
      section(blocks, i);
    }
  }

  void section(const std::vector<Block>& blocks, size_t i) {
    const Block& B = blocks[i];
    // 1. bring needed rank bits onto local memory bits (one grouped exchange)
    std::vector<int> rank_bits;
    uint64_t need = needed(B, sigma, nL, &rank_bits);
    if (!rank_bits.empty()) {
      Step ex;
      ex.type = Step::EXCHANGE;
      // Victim local bits, Belady-style (the paper's MPI-level blocking, NEXT-1): a relabel never
      // moves a qubit's memory bit, so walking the later blocks' relabels gives the next section
      // that needs each memory bit; evict the local bits needed furthest ahead (never: best),
      // among bits >= low_bits (the tile coalescing bits stay), higher bits first on ties.
      std::vector<size_t> next_use(nL, blocks.size());
      {
        std::vector<int> v = sigma;
        uint64_t seen = 0;
        for (size_t j = i + 1; j < blocks.size() && __builtin_popcountll(seen) < nL; j++) {
          for (const auto& rl : blocks[j].relabels) std::swap(v[rl.first], v[rl.second]);
          const uint64_t nj = needed(blocks[j], v, nL, nullptr);
          for (int m = 0; m < nL; m++)
            if (((nj >> m) & 1) && !((seen >> m) & 1)) {
              next_use[m] = j;
              seen |= 1ull << m;
            }
        }
      }
      const int nlow = std::min(L.low_bits, nL);
      uint64_t taken = need;
      for (int b : rank_bits) {
        int m = -1;
        for (int pass = 0; pass < 2 && m < 0; pass++)  // pass 1 may use the low bits if it must
          for (int cand = nL - 1; cand >= (pass ? 0 : nlow); cand--) {
            if ((taken >> cand) & 1) continue;
            if (m < 0 || next_use[cand] > next_use[m]) m = cand;
          }
        // m >= 0 is guaranteed: the section needs at most c <= nL local bits in total
        taken |= 1ull << m;
        ex.ex.push_back({m, b});
        swap_bits(m, b);
      }
      ctr.exchanges += ex.ex.size();
      ctr.exchange_batches++;
      steps.push_back(std::move(ex));
      need = needed(B, sigma, nL, nullptr);
    }
    // 2. coalescing: the tile must hold the section's bits and the low memory bits
    const int nlow = std::min(L.low_bits, nL);
    const uint64_t low = (1ull << nlow) - 1;
    int cnt = __builtin_popcountll(need);
    if (cnt <= L.max_tile && cnt + __builtin_popcountll(low & ~need) > L.max_tile) {
      Step cp;
      cp.type = Step::COMPACT;
      int over = cnt + __builtin_popcountll(low & ~need) - L.max_tile;
      for (int l = 0; l < nlow && over > 0; l++) {
        if ((need >> l) & 1) continue;
        int h = nL - 1;
        while (h >= nlow && !((need >> h) & 1)) h--;
        if (h < nlow) break;
        cp.swaps.push_back({l, h});
        swap_bits(l, h);
        need = (need & ~(1ull << h)) | (1ull << l);
        over--;
      }
      ctr.compactions += cp.swaps.size();
      if (!cp.swaps.empty()) steps.push_back(std::move(cp));
    }
    // 3. translate the section to memory bits; SWAPs relabel sigma for everything after them
    std::vector<sv_gate> mem;
    for (const sv_gate& t : B.gates) {
      if (t.kind == SV_SWAP) {
        relabel(t.q0, t.q1);
        continue;
      }
      mem.push_back(to_memory(t, sigma));
    }
    uint64_t act = 0;
    for (const sv_gate& m : mem)
      if (!is_diag(m.kind)) act |= qmask(m);
    // 4. look ahead: fuse swaps into this section's store that put the next section's qubits on
    //    the low memory bits (both bits of each swap lie in this section's tile)
    std::vector<std::pair<int, int>> sw;
    if (!mem.empty() && i + 1 < blocks.size() && __builtin_popcountll(act) <= L.max_tile) {
      const uint64_t tile = choose_tile(act, nL, L);
      std::vector<int> v = sigma;
      for (const auto& rl : blocks[i + 1].relabels) std::swap(v[rl.first], v[rl.second]);
      const uint64_t nxt = needed(blocks[i + 1], v, nL, nullptr) & ((nL >= 64) ? ~0ull : ((1ull << nL) - 1));
      if (__builtin_popcountll(nxt) <= L.max_tile) {
        uint64_t cand = nxt & tile & ~low;  // next-section bits we can pull down now
        // qubits of the next section's first gates (about its first register phase): leave them
        // off the low bits when others can go there, so that phase's lanes can walk the low bits
        // and read HBM directly
        uint64_t early = 0;
        {
          std::vector<int> w = v;
          for (const sv_gate& t : blocks[i + 1].gates) {
            if (t.kind == SV_SWAP) {
              std::swap(w[t.q0], w[t.q1]);
              continue;
            }
            if (is_diag(t.kind)) continue;
            uint64_t m = 1ull << w[t.q0];
            if (is_two(t.kind)) m |= 1ull << w[t.q1];
            if (__builtin_popcountll(early | m) > SV_R_BITS_PLAN) break;
            early |= m;
          }
        }
        for (int l = 0; l < nlow && cand; l++) {
          if (((nxt >> l) & 1) || !((tile >> l) & 1)) continue;
          const uint64_t pref = (cand & ~early) ? (cand & ~early) : cand;
          const int x = 63 - __builtin_clzll(pref);  // highest (late-used) candidate
          cand &= ~(1ull << x);
          sw.push_back({l, x});
        }
      }
    }
    if (mem.empty()) {
      return;
    }
    if (__builtin_popcountll(act) <= L.max_tile) {
      push_section(std::move(mem), sw);
    } else {
      // More active bits than one tile holds (chunk_bits > max_tile): split the section with the
      // same pass at c = max_tile - low_bits on memory bits (room for the coalescing bits).  Its chunk_swaps are relabels of an inner frame
      // whose inverse keeps every gate on its own memory bit, so only the grouping is used (each
      // inner section's gates are the originals, by index).
      std::vector<sv_gate> in = mem;
      for (size_t k = 0; k < in.size(); k++) in[k].pad = (int32_t)k;
      std::vector<int> ipi(nL);
      for (int b = 0; b < nL; b++) ipi[b] = b;
      std::vector<sv_gate> toks;
      Status st = block_pass(in.data(), in.size(), nL, std::max(2, L.max_tile - nlow), ipi, 0, toks);
      if (!st.good()) {  // cannot happen for valid sections; keep the section whole
        push_section(std::move(mem), {});
      } else {
        std::vector<sv_gate> cur;
        for (const sv_gate& t : toks) {
          if (t.kind == SV_BEGIN) {
            cur.clear();
          } else if (t.kind == SV_END) {
            if (!cur.empty()) push_section(std::move(cur), {});
            cur.clear();
          } else if (t.kind != SV_CHUNK_SWAP) {
            cur.push_back(mem[t.pad]);
          }
        }
      }
      sw.clear();
    }
    for (const auto& s : sw) swap_bits(s.first, s.second);
    ctr.store_swaps += sw.size();
  }

  void push_section(std::vector<sv_gate> gates, const std::vector<std::pair<int, int>>& sw) {
    Step s;
    s.type = Step::SECTION;
    s.gates = std::move(gates);
    s.swaps = sw;
    ctr.sections++;
    steps.push_back(std::move(s));
  }
};

}  // namespace

// One-level executor mapping: the pass at chunk c, sections mapped onto memory bits, exchanges
// when a section needs a rank bit (Belady victims, Planner::section).
Status plan_one_level(const sv_gate* g, size_t count, int n, int c, int world_log2, std::vector<int>& pi,
                      std::vector<int>& sigma, uint32_t flags, std::vector<Step>& steps, PlanCounters& ctr,
                      const PlanLayout& layout, std::vector<int>* sigma_initial) {
  const int nL = n - world_log2;
  std::vector<sv_gate> tokens;
  tokens.reserve(count * 2 + 16);
  if (Status s = block_pass(g, count, n, c, pi, flags, tokens); !s.good()) return s;

  std::vector<Block> blocks;
  Block cur;
  bool inside = false;
  std::vector<std::pair<int, int>> trailing;  // chunk_swaps after the last section
  for (const sv_gate& t : tokens) {
    switch (t.kind) {
      case SV_CHUNK_SWAP:
        cur.relabels.push_back({t.q0, t.q1});
        ctr.chunk_swaps++;
        break;
      case SV_BEGIN:
        inside = true;
        break;
      case SV_END:
        if (!inside) return Status::err(SV_EMALFORMED, "END without BEGIN");
        blocks.push_back(std::move(cur));
        cur = Block();
        inside = false;
        break;
      default:
        cur.gates.push_back(t);
    }
  }
  if (layout.free_initial && !blocks.empty()) {
    // NEXT-2 "free initial layout" (the paper's bit reordering): the state is a basis
    // state, so sigma can be chosen freely at no data cost.  Put the first section's qubits on
    // the lowest memory bits (its tile is then coalesced and no exchange is needed), keep every
    // other qubit's relative order, then undo the first block's chunk_swap relabels.
    std::vector<int> after = sigma;
    for (const auto& rl : blocks[0].relabels) std::swap(after[rl.first], after[rl.second]);
    const uint64_t need = Planner::needed(blocks[0], after, n, nullptr);
    std::vector<int> order(n);  // paper qubits: needed first, each group by current memory bit
    for (int p = 0; p < n; p++) order[p] = p;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
      const bool na = (need >> after[a]) & 1, nb = (need >> after[b]) & 1;
      if (na != nb) return na;
      return after[a] < after[b];
    });
    for (int i = 0; i < n; i++) after[order[i]] = i;
    for (auto it = blocks[0].relabels.rbegin(); it != blocks[0].relabels.rend(); ++it)
      std::swap(after[it->first], after[it->second]);
    sigma = after;
  }
  if (sigma_initial) *sigma_initial = sigma;
  Planner planner(n, nL, layout, sigma, steps, ctr);
  planner.run(blocks);
  for (const auto& rl : cur.relabels) planner.relabel(rl.first, rl.second);  // trailing chunk_swaps
  return Status::ok();
}

double exchange_volume(const std::vector<Step>& steps) {  // shard-equivalents sent per GPU
  double v = 0.0;
  for (const Step& st : steps)
    if (st.type == Step::EXCHANGE) v += 1.0 - std::ldexp(1.0, -(int)st.ex.size());
  return v;
}

// Two-level blocking (NEXT-1; the paper's own MPI-level use of the pass): an outer
// pass with chunk = the GPU shard (nL qubits) decides which qubits are global; its chunk_swaps are
// the cross-GPU exchanges (batched), and every outer block — whose non-diagonal gates are all on
// local qubits — is planned by the one-level mapping with the inner chunk c, which then never
// exchanges.  Outer positions are memory bits; tau tracks where the inner plans' physical moves
// (store swaps, compactions) put each of them.
Status plan_two_level(const sv_gate* g, size_t count, int n, int c, int world_log2, std::vector<int>& pi,
                      std::vector<int>& sigma, uint32_t flags, std::vector<Step>& steps, PlanCounters& ctr,
                      const PlanLayout& layout, std::vector<int>* sigma_initial) {
  const int nL = n - world_log2;
  std::vector<int> mem(n);  // logical -> memory bit at entry
  for (int q = 0; q < n; q++) mem[q] = sigma[pi[q]];
  std::vector<int> piO = mem;
  std::vector<sv_gate> tokens;
  tokens.reserve(count * 2 + 16);
  if (layout.free_initial) {
    // basis state: the first outer block's qubits start local (no exchange before it)
    std::vector<int> probe = piO;
    if (Status s = block_pass(g, count, n, nL, probe, 0, tokens); !s.good()) return s;
    std::vector<int> inv(n);
    for (int q = 0; q < n; q++) inv[piO[q]] = q;
    uint64_t first = 0;  // logical qubits of the first outer block's non-diagonal gates
    bool inside = false;
    std::vector<int> cur = piO, curinv = inv;
    for (const sv_gate& t : tokens) {
      if (t.kind == SV_CHUNK_SWAP) {  // the pass's relabel in outer positions
        const int a = curinv[t.q0], b = curinv[t.q1];
        std::swap(cur[a], cur[b]);
        curinv[cur[a]] = a;
        curinv[cur[b]] = b;
      } else if (t.kind == SV_BEGIN) {
        inside = true;
      } else if (t.kind == SV_END) {
        break;
      } else if (inside && !is_diag(t.kind)) {
        first |= 1ull << curinv[t.q0];
        if (is_two(t.kind)) first |= 1ull << curinv[t.q1];
      }
    }
    std::vector<int> order(n);
    for (int q = 0; q < n; q++) order[q] = q;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
      const bool fa = (first >> a) & 1, fb = (first >> b) & 1;
      if (fa != fb) return fa;
      return piO[a] < piO[b];
    });
    for (int i = 0; i < n; i++) piO[order[i]] = i;
    tokens.clear();
  }
  const std::vector<int> piO0 = piO;
  if (Status s = block_pass(g, count, n, nL, piO, 0, tokens); !s.good()) return s;

  std::vector<int> tau(n), init_tau(n);
  for (int p = 0; p < n; p++) tau[p] = init_tau[p] = p;
  bool first_block = true;
  Step batch;
  batch.type = Step::EXCHANGE;
  auto flush = [&]() {
    if (batch.ex.empty()) return;
    ctr.exchanges += batch.ex.size();
    ctr.exchange_batches++;
    steps.push_back(std::move(batch));
    batch = Step();
    batch.type = Step::EXCHANGE;
  };
  std::vector<sv_gate> blk;
  bool inside = false;
  for (const sv_gate& t : tokens) {
    if (t.kind == SV_CHUNK_SWAP) {
      if (t.q1 < nL || t.q0 >= nL) return Status::err(SV_EMALFORMED, "internal: outer chunk_swap not local/global");
      batch.ex.push_back({tau[t.q0], tau[t.q1]});
      ctr.chunk_swaps++;
    } else if (t.kind == SV_BEGIN) {
      flush();
      blk.clear();
      inside = true;
    } else if (t.kind == SV_END) {
      if (!inside) return Status::err(SV_EMALFORMED, "END without BEGIN");
      inside = false;
      for (sv_gate& x : blk) {
        x.q0 = tau[x.q0];
        if (is_two(x.kind)) x.q1 = tau[x.q1];
      }
      std::vector<int> pin(n), sin(n), sinit;
      for (int p = 0; p < n; p++) pin[p] = sin[p] = p;
      PlanLayout L2 = layout;
      L2.free_initial = layout.free_initial && first_block;
      if (Status s = plan_one_level(blk.data(), blk.size(), n, c, world_log2, pin, sin, flags & ~(uint32_t)SV_RESTORE_ORDER,
                                    steps, ctr, L2, &sinit);
          !s.good())
        return s;
      if (first_block && layout.free_initial) init_tau = sinit;  // block-start bit p lives at sinit[p]
      std::vector<int> rho(n);
      for (int x = 0; x < n; x++) rho[x] = sin[pin[x]];
      for (int p = 0; p < n; p++) tau[p] = rho[first_block && layout.free_initial ? p : tau[p]];
      first_block = false;
    } else {
      blk.push_back(t);
    }
  }
  flush();
  // logical q: outer position piO[q] -> memory bit tau[piO[q]]
  if (sigma_initial) {
    std::vector<int> s0(n);
    for (int q = 0; q < n; q++) s0[pi[q]] = init_tau[piO0[q]];
    *sigma_initial = s0;
  }
  pi = piO;
  sigma = tau;
  return Status::ok();
}

// Blocked plan: one-level, or — on several GPUs — the two-level plan when it moves fewer bytes
// across GPUs.  (Either plan's exchanges may pick any local bit: both exchange transports handle
// strided blocks — the peer kernel element-wise, the NCCL path by packing.)
Status plan_blocked(const sv_gate* g, size_t count, int n, int c, int world_log2, std::vector<int>& pi,
                    std::vector<int>& sigma, uint32_t flags, std::vector<Step>& steps, PlanCounters& ctr,
                    const PlanLayout& layout, std::vector<int>* sigma_initial) {
  if (world_log2 == 0 || (flags & SV_RESTORE_ORDER))
    return plan_one_level(g, count, n, c, world_log2, pi, sigma, flags, steps, ctr, layout, sigma_initial);
  std::vector<int> pi1 = pi, s1 = sigma, pi2 = pi, s2 = sigma, init1, init2;
  std::vector<Step> st1, st2;
  PlanCounters c1, c2;
  if (Status s = plan_one_level(g, count, n, c, world_log2, pi1, s1, flags, st1, c1, layout, &init1); !s.good())
    return s;
  Status s = plan_two_level(g, count, n, c, world_log2, pi2, s2, flags, st2, c2, layout, &init2);
  const bool use2 = s.good() && exchange_volume(st2) < exchange_volume(st1);
  if (use2) {
    pi = pi2, sigma = s2, ctr = c2;
    steps.insert(steps.end(), st2.begin(), st2.end());
    if (sigma_initial) *sigma_initial = init2;
  } else {
    pi = pi1, sigma = s1, ctr = c1;
    steps.insert(steps.end(), st1.begin(), st1.end());
    if (sigma_initial) *sigma_initial = init1;
  }
  return Status::ok();
}

Status make_plan(const sv_gate* g, size_t count, int n, int c, int world_log2, std::vector<int>& pi,
                 std::vector<int>& sigma, uint32_t flags, std::vector<Step>& steps, PlanCounters& ctr,
                 const PlanLayout& layout, std::vector<int>* sigma_initial) {
  const int nL = n - world_log2;
  if (world_log2 < 0 || nL < 1) return Status::err(SV_EINVAL, "world too large for n");
  if (c < 1 || c > nL) return Status::err(SV_EINVAL, "chunk_bits must satisfy 1 <= c <= n - log2(world)");
  if ((int)pi.size() != n || (int)sigma.size() != n) return Status::err(SV_EINVAL, "bad permutation length");
  if (Status s = validate_gates(g, count, n); !s.good()) return s;

  if (sigma_initial) *sigma_initial = sigma;
  if (flags & SV_UNBLOCKED) {
    // Per-gate baseline: each gate is one step on memory bits mu(q) = sigma[pi[q]].  On
    // several GPUs a non-diagonal gate on a global qubit is the paper's unblocked multi-GPU
    // baseline (NEXT-3): its rank bit is exchanged with a local bit the gate does not
    // use, the gate runs there, and a second exchange writes the halves back.  A SWAP of a local
    // and a global qubit is itself one exchange.
    for (size_t i = 0; i < count; i++) {
      sv_gate m = g[i];
      m.q0 = sigma[pi[g[i].q0]];
      m.q1 = is_two(g[i].kind) ? sigma[pi[g[i].q1]] : -1;
      m.pad = (int32_t)i;
      const bool r0 = m.q0 >= nL, r1 = is_two(m.kind) && m.q1 >= nL;
      if (is_diag(m.kind) || (!r0 && !r1)) {
        Step s;
        s.type = Step::GATE;
        s.gates.push_back(m);
        steps.push_back(std::move(s));
        continue;
      }
      if (m.kind == SV_SWAP && r0 != r1) {
        Step ex;
        ex.type = Step::EXCHANGE;
        ex.ex.push_back({r0 ? m.q1 : m.q0, r0 ? m.q0 : m.q1});
        ctr.exchanges++;
        ctr.exchange_batches++;
        steps.push_back(std::move(ex));
        continue;
      }
      Step in;
      in.type = Step::EXCHANGE;
      uint64_t used = 0;
      if (!r0) used |= 1ull << m.q0;
      if (is_two(m.kind) && !r1) used |= 1ull << m.q1;
      int* qs[2] = {&m.q0, &m.q1};
      for (int k = 0; k < 2; k++) {
        if (!(k == 0 ? r0 : r1)) continue;
        int v = nL - 1;
        while (v >= 0 && ((used >> v) & 1)) v--;
        if (v < 0) return Status::err(SV_EINFEASIBLE, "unblocked mode: no local bit to exchange into");
        used |= 1ull << v;
        in.ex.push_back({v, *qs[k]});
        *qs[k] = v;
      }
      ctr.exchanges += 2 * in.ex.size();
      ctr.exchange_batches += 2;
      Step gs;
      gs.type = Step::GATE;
      gs.gates.push_back(m);
      Step out = in;  // the same exchange again restores the layout (write back)
      steps.push_back(std::move(in));
      steps.push_back(std::move(gs));
      steps.push_back(std::move(out));
    }
    return Status::ok();
  }

  return plan_blocked(g, count, n, c, world_log2, pi, sigma, flags, steps, ctr, layout, sigma_initial);
}

}  // namespace sv
