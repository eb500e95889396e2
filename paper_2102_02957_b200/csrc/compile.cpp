// compile.cpp — section compiler: memory-frame section -> SvSecHeader/SvPhase/SvOp program.
//
// See program.h for the model.  Phase scheduling is a greedy in-order list schedule over the
// section's gates: a gate joins the current phase if no earlier deferred gate of this phase
// shares a tile position with it and its non-diagonal positions fit the R_BITS register slots;
// diagonal gates join whenever their dependencies allow (they act per amplitude).
// Reordering only qubit-disjoint gates is the same legality rule the pass uses.
//
// Diagonal fusion: inside a phase every diagonal gate is sunk as late as its tile positions
// allow (past non-diagonal gates on other positions), and each run of diagonal gates becomes one
// DIAGSET: the product of all its factors, decomposed into terms c^[S subset k][J subset tid]
// [O subset tile] over register slots S, thread bits J and out-of-tile bits O.  Terms on two
// slots are constants (a 16-entry table); the rest belong to the empty set or one slot and are
// tabulated per thread index on the host (constant and thread-bit terms) or evaluated once per
// warp (out-of-tile terms), so a QFT section's hundreds of controlled phases cost a few complex
// multiplies per amplitude.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <tuple>
#include <utility>

#include "common.h"
#include "compile.h"

namespace sv {

namespace {

typedef std::complex<double> cd;

inline bool is_h_like(const double* m) {  // s * [[1, 1], [1, -1]], s real: exact check only
  for (int i = 0; i < 4; i++)
    if (m[2 * i + 1] != 0.0) return false;
  return m[0] == m[2] && m[0] == m[4] && m[6] == -m[0] && m[0] != 0.0;
}

inline bool is_perm4(const double* m, int* perm) {  // 4x4 permutation matrix with exact 1 entries
  for (int r = 0; r < 4; r++) {
    int found = -1;
    for (int c = 0; c < 4; c++) {
      const double re = m[2 * (4 * r + c)], im = m[2 * (4 * r + c) + 1];
      if (im != 0.0) return false;
      if (re == 1.0) {
        if (found >= 0) return false;
        found = c;
      } else if (re != 0.0) {
        return false;
      }
    }
    if (found < 0) return false;
    perm[r] = found;
  }
  return true;
}

struct PGate {  // a gate on tile positions
  int type;
  int a, b;        // positions (U*/PERM) or memory-bit operands (DIAG: -1-mb local, 200/201 const)
  uint32_t pmask;  // tile positions it touches (for dependencies)
  bool diag;
  int src;         // index into the section's gate list (payload source)
  int extra;
};

constexpr int kDiagLocal = -1;  // DIAG operand: -(1 + memory bit)
constexpr int kMaxTile = 13;    // 2^13 amplitudes: 128 KiB fp64 / 64 KiB fp32 of shared memory

// One factor term of a DIAGSET: coef applies where slots S, thread bits J and out bits O are all 1.
struct TermKey {
  int S;
  uint32_t J;
  uint64_t O;
  bool operator<(const TermKey& o) const { return std::tie(S, J, O) < std::tie(o.S, o.J, o.O); }
};

}  // namespace

Status compile_section(const std::vector<sv_gate>& gates, int nL, int rank, int world_log2, int T_default,
                       int swizzle_bits, const std::vector<std::pair<int, int>>& store_swaps, Program& prog) {
  (void)world_log2;
  // ---- tile bits
  uint64_t active = 0;
  for (const sv_gate& g : gates) {
    if (is_diag(g.kind)) continue;
    const int b0 = g.q0, b1 = is_two(g.kind) ? g.q1 : -1;
    if (b0 >= nL || b1 >= nL) return Status::err(SV_EMALFORMED, "internal: section gate on a rank bit");
    active |= 1ull << b0;
    if (b1 >= 0) active |= 1ull << b1;
  }
  // The tile always includes the lowest memory bits (128-byte runs: 8 fp64 / 16 fp32 amplitudes)
  // when they fit; the planner (plan.cpp) arranges that they do.
  PlanLayout lay;
  lay.low_bits = swizzle_bits;
  lay.max_tile = kMaxTile;
  lay.pref_tile = pref_tile_for(swizzle_bits);
  lay.tile_default = T_default;
  const uint64_t tile = choose_tile(active, nL, lay);
  const int T = __builtin_popcountll(tile);
  if (T > kMaxTile) return Status::err(SV_ECAPACITY, "section needs more tile bits than shared memory holds");
  int tile_bits[16], pos_of[64];
  std::fill(pos_of, pos_of + 64, -1);
  int t = 0;
  for (int b = 0; b < 64; b++)
    if ((tile >> b) & 1) {
      pos_of[b] = t;
      tile_bits[t++] = b;
    }
  int load_bits[16];  // tile position -> memory bit on the load (the store side may differ)
  for (int j = 0; j < T; j++) load_bits[j] = tile_bits[j];
  int out_bits[SV_MAX_OUT], n_out = 0;
  for (int b = 0; b < nL; b++)
    if (!((tile >> b) & 1)) {
      if (n_out >= SV_MAX_OUT) return Status::err(SV_ECAPACITY, "too many local bits");
      out_bits[n_out++] = b;
    }
  const int r = std::min(SV_R_BITS, T);

  // ---- gates on positions
  std::vector<PGate> pg;
  pg.reserve(gates.size());
  for (size_t gi = 0; gi < gates.size(); gi++) {
    const sv_gate& g = gates[gi];
    PGate p{};
    p.src = (int)gi;
    switch (g.kind) {
      case SV_U1:
        p.a = pos_of[g.q0];
        p.pmask = 1u << p.a;
        p.type = is_h_like(g.m) ? SV_OP_H1 : SV_OP_U1;
        break;
      case SV_U2: {
        p.a = pos_of[g.q0];
        p.b = pos_of[g.q1];
        p.pmask = (1u << p.a) | (1u << p.b);
        int perm[4];
        if (is_perm4(g.m, perm)) {
          p.type = SV_OP_PERM2;
          p.extra = perm[0] | (perm[1] << 2) | (perm[2] << 4) | (perm[3] << 6);
        } else {
          p.type = SV_OP_U2;
        }
        break;
      }
      case SV_D1:
      case SV_D2: {
        p.diag = true;
        auto operand = [&](int mb) {
          if (mb >= nL) return ((rank >> (mb - nL)) & 1) ? SV_CODE_ONE : SV_CODE_ZERO;  // rank bit: a constant
          return kDiagLocal - mb;
        };
        p.a = operand(g.q0);
        p.b = g.kind == SV_D2 ? operand(g.q1) : SV_CODE_ZERO;
        for (int x : {p.a, p.b})
          if (x < 0 && pos_of[kDiagLocal - x] >= 0) p.pmask |= 1u << pos_of[kDiagLocal - x];
        const double* d = g.m;
        const bool cp = g.kind == SV_D2 && d[0] == 1.0 && d[1] == 0.0 && d[2] == 1.0 && d[3] == 0.0 && d[4] == 1.0 &&
                        d[5] == 0.0;
        p.type = cp ? SV_OP_DIAG_CP : SV_OP_DIAG;
        break;
      }
      default:
        return Status::err(SV_EMALFORMED, "internal: unexpected kind in section");
    }
    pg.push_back(p);
  }

  // ---- phase schedule
  struct Ph {
    std::vector<int> R;
    std::vector<int> ops;
  };
  std::vector<Ph> phases;
  std::vector<int> pending(pg.size());
  for (size_t i = 0; i < pg.size(); i++) pending[i] = (int)i;
  std::vector<int> rest;
  while (!pending.empty()) {
    Ph ph;
    uint32_t rmask = 0, blocked = 0;
    rest.clear();
    for (int gi : pending) {
      const PGate& p = pg[gi];
      if (p.pmask & blocked) {
        blocked |= p.pmask;
        rest.push_back(gi);
        continue;
      }
      if (p.diag) {
        ph.ops.push_back(gi);
        continue;
      }
      const uint32_t need = p.pmask & ~rmask;
      if (__builtin_popcount(rmask) + __builtin_popcount(need) <= r) {
        rmask |= need;
        ph.ops.push_back(gi);
      } else {
        blocked |= p.pmask;
        rest.push_back(gi);
      }
    }
    if (ph.ops.empty()) return Status::err(SV_EINFEASIBLE, "internal: phase schedule made no progress");
    // pad the register set with the highest free positions (keeps low positions as thread bits,
    // so lanes walk contiguous memory)
    for (int pos = T - 1; pos >= 0 && __builtin_popcount(rmask) < r; pos--)
      if (!((rmask >> pos) & 1)) rmask |= 1u << pos;
    for (int pos = 0; pos < T; pos++)
      if ((rmask >> pos) & 1) ph.R.push_back(pos);
    phases.push_back(std::move(ph));
    pending.swap(rest);
  }
  if (phases.empty()) {  // no gates at all: one empty phase keeps the kernel uniform
    Ph ph;
    for (int pos = T - r; pos < T; pos++) ph.R.push_back(pos);
    phases.push_back(ph);
  }

  // Shared-memory swizzle of this section: tile position p -> word (a GF(2)-linear, invertible
  // map; every smem offset is an XOR of words).  p < G keeps 1 << p; p >= G adds a nonzero G-bit
  // vector vec[p] to the low bits.  A 2^G-lane group then covers the 2^G 16- (fp64) or 8-byte
  // (fp32) slots of a 128-byte wavefront exactly when its G lane bits carry independent vectors:
  // the load map's lanes are positions 0..G-1, the store map's are the positions of the lowest
  // store memory bits, and each phase picks G independent thread positions (below).  The vectors
  // are searched so every phase's thread positions span GF(2)^G.
  const int G = swizzle_bits;
  int store_bits[16];
  for (int j = 0; j < T; j++) store_bits[j] = tile_bits[j];
  for (const auto& sw : store_swaps) {  // physical bit swaps fused into the store (plan.cpp)
    const int p1 = sw.first < 64 ? pos_of[sw.first] : -1, p2 = sw.second < 64 ? pos_of[sw.second] : -1;
    if (p1 < 0 || p2 < 0) return Status::err(SV_EMALFORMED, "internal: store swap outside the tile");
    std::swap(store_bits[p1], store_bits[p2]);
  }
  int swz[SV_TMAX];
  {
    const int nseq = (1 << G) - 1;
    auto span_of = [&](const int* v, const std::vector<int>& pos) {
      uint32_t span = 1;
      for (int p : pos) {
        uint32_t g2 = span;
        for (int u = 0; u < (1 << G); u++)
          if ((span >> u) & 1) g2 |= 1u << (u ^ v[p]);
        span = g2;
      }
      return span;
    };
    const uint32_t full = (1u << (1 << G)) - 1;  // all 2^G vectors reachable
    int order[16];
    for (int j = 0; j < T; j++) order[j] = j;
    std::sort(order, order + T, [&](int a, int b) { return store_bits[a] < store_bits[b]; });
    std::vector<int> store_lanes(order, order + std::min(G, T));
    std::vector<std::vector<int>> thread_pos;
    for (const Ph& ph : phases) {
      std::vector<int> tp;
      for (int pos = 0; pos < T; pos++)
        if (std::find(ph.R.begin(), ph.R.end(), pos) == ph.R.end()) tp.push_back(pos);
      thread_pos.push_back(tp);
    }
    auto score = [&](const int* v) {  // constraints met (higher is better)
      int sc = 0;
      if (T - r >= G && span_of(v, store_lanes) == full) sc += 1000;
      for (const auto& tp : thread_pos)
        if ((int)tp.size() >= G && span_of(v, tp) == full) sc++;
      return sc;
    };
    int target = (T - r >= G ? 1000 : 0);
    for (const auto& tp : thread_pos)
      if ((int)tp.size() >= G) target++;
    int vec[SV_TMAX], best[SV_TMAX];
    uint64_t rng = 0x9E3779B97F4A7C15ull ^ ((uint64_t)T << 32) ^ phases.size();
    int best_sc = -1;
    for (int attempt = 0; attempt < 256 && best_sc < target; attempt++) {
      for (int pos = 0; pos < T; pos++) {
        if (pos < G) {
          vec[pos] = 1 << pos;
        } else if (attempt == 0) {
          vec[pos] = 1 + (pos - G) % nseq;  // deterministic first try
        } else {
          rng ^= rng << 13;
          rng ^= rng >> 7;
          rng ^= rng << 17;
          vec[pos] = 1 + (int)(rng % (uint64_t)nseq);
        }
      }
      const int sc = score(vec);
      if (sc > best_sc) {
        best_sc = sc;
        std::copy(vec, vec + T, best);
      }
    }
    for (int pos = 0; pos < T; pos++) swz[pos] = pos < G ? (1 << pos) : ((1 << pos) | best[pos]);
  }
  auto low_vec = [&](int pos) { return swz[pos] & ((1 << G) - 1); };

  // ---- per phase: thread-bit order, then the op items (single ops or fused diagonal runs)
  struct Item {
    int gate = -1;           // single op: index into pg
    std::vector<int> group;  // DIAGSET: indices into pg
  };
  struct PhaseOut {
    std::vector<int> chosen;  // thread bit j -> tile position
    int slot_of[SV_TMAX], thread_of[SV_TMAX];
    std::vector<Item> items;
  };
  std::vector<PhaseOut> pout(phases.size());
  for (size_t pi = 0; pi < phases.size(); pi++) {
    const Ph& ph = phases[pi];
    PhaseOut& po = pout[pi];
    std::fill(po.slot_of, po.slot_of + SV_TMAX, -1);
    std::fill(po.thread_of, po.thread_of + SV_TMAX, -1);
    for (int s = 0; s < r; s++) po.slot_of[ph.R[s]] = s;
    // thread bits: the first G get linearly independent swizzle vectors (lowest positions first,
    // so lanes walk the lowest memory bits where they can: direct HBM boundaries need that)
    std::vector<int> cand;
    for (int pos = 0; pos < T; pos++)
      if (po.slot_of[pos] < 0) cand.push_back(pos);
    // the last phase of a multi-phase section walks the lowest STORE memory bits first (they
    // differ from the load order after fused store swaps): its store can then go straight to HBM
    if (pi + 1 == phases.size() && phases.size() > 1)
      std::stable_sort(cand.begin(), cand.end(), [&](int a, int b) { return store_bits[a] < store_bits[b]; });
    std::vector<bool> taken(cand.size(), false);
    uint32_t span = 1;  // bit v set: vector v is an XOR of chosen vectors (v = 0 always)
    for (size_t i = 0; i < cand.size() && (int)po.chosen.size() < G; i++) {
      const int vec = low_vec(cand[i]);
      if ((span >> vec) & 1) continue;
      uint32_t grown = span;
      for (int u = 0; u < (1 << G); u++)
        if ((span >> u) & 1) grown |= 1u << (u ^ vec);
      span = grown;
      po.chosen.push_back(cand[i]);
      taken[i] = true;
    }
    for (size_t i = 0; i < cand.size(); i++)
      if (!taken[i]) po.chosen.push_back(cand[i]);
    for (size_t j = 0; j < po.chosen.size(); j++) po.thread_of[po.chosen[j]] = (int)j;
    // sink diagonal ops: each waits until a later non-diagonal op shares a tile position
    std::vector<int> sink;
    auto flush = [&](uint32_t mask, bool all) {
      std::vector<int> keep, go;
      for (int gi : sink) ((all || (pg[gi].pmask & mask)) ? go : keep).push_back(gi);
      sink.swap(keep);
      // diagonals whose operands are all register slots / constants stay plain ops (a few
      // complex multiplies on the registers); the rest of the run becomes one DIAGSET
      auto in_tile = [&](int x) { return x >= 0 || pos_of[kDiagLocal - x] >= 0; };
      auto slotish = [&](int x) { return x >= 0 || po.slot_of[pos_of[kDiagLocal - x]] >= 0; };
      Item set;
      for (int gi : go) {
        const PGate& p = pg[gi];
        if (in_tile(p.a) && in_tile(p.b) && slotish(p.a) && slotish(p.b)) {
          Item it;
          it.gate = gi;
          po.items.push_back(it);
        } else {
          set.group.push_back(gi);
        }
      }
      if (!set.group.empty()) po.items.push_back(set);
    };
    for (int gi : ph.ops) {
      if (pg[gi].diag) {
        sink.push_back(gi);
        continue;
      }
      flush(pg[gi].pmask, false);
      Item it;
      it.gate = gi;
      po.items.push_back(it);
    }
    flush(0, true);
    if (const char* dbg = std::getenv("SV_DEBUG_PLAN"); dbg && dbg[0] == '2') {
      std::fprintf(stderr, "[sv]   phase %zu R=%d,%d,%d,%d:", pi, ph.R[0], ph.R[1], ph.R[2], ph.R[3]);
      for (const Item& it : po.items) {
        if (it.group.empty())
          std::fprintf(stderr, " op%d", pg[it.gate].type);
        else
          std::fprintf(stderr, " SET[%zu]", it.group.size());
      }
      std::fprintf(stderr, "\n");
    }
  }

  // ---- sizes
  const int header_ints = sizeof(SvSecHeader) / 4;
  const int phase_ints = sizeof(SvPhase) / 4;
  const int op_ints = sizeof(SvOp) / 4;
  size_t n_items = 0;
  for (const auto& po : pout) n_items += po.items.size();

  // ---- emit
  const size_t base = prog.ints.size();
  const size_t cbase = prog.coefs.size() / 2;
  const size_t abase = prog.aux.size() / 2;
  const size_t ops_end = header_ints + phase_ints * phases.size() + op_ints * n_items;
  prog.ints.resize(base + ops_end, 0);
  auto H = [&]() { return reinterpret_cast<SvSecHeader*>(prog.ints.data() + base); };
  H()->T = T;
  H()->r = r;
  H()->n_out = n_out;
  H()->n_phases = (int)phases.size();
  H()->phase_off = header_ints;
  H()->op_off = header_ints + phase_ints * (int)phases.size();
  H()->n_ops = (int)n_items;
  for (int j = 0; j < T; j++) {
    H()->tile_bits[j] = tile_bits[j];
    H()->store_bits[j] = store_bits[j];
  }
  for (int j = 0; j < n_out; j++) H()->out_bits[j] = out_bits[j];
  auto fill_map = [&](SvMap& m, const int* tpos, const int* R, const int* bits) {
    for (int j = 0; j < T - r; j++) {
      m.tw[j] = swz[tpos[j]];
      m.tmb[j] = bits[tpos[j]];
    }
    for (int s = 0; s < r; s++) {
      m.rw[s] = swz[R[s]];
      m.rmb[s] = bits[R[s]];
    }
  };
  {  // boundary maps: lanes walk the lowest memory bits of the load / store side
    int order[16];
    for (int j = 0; j < T; j++) order[j] = j;
    std::sort(order, order + T, [&](int a, int b) { return load_bits[a] < load_bits[b]; });
    fill_map(H()->load, order, order + (T - r), load_bits);
    for (int j = 0; j < T; j++) order[j] = j;
    std::sort(order, order + T, [&](int a, int b) { return store_bits[a] < store_bits[b]; });
    fill_map(H()->store, order, order + (T - r), tile_bits);
    for (int j = 0; j < T - r; j++) H()->store.tmb[j] = store_bits[order[j]];
    for (int s = 0; s < r; s++) H()->store.rmb[s] = store_bits[order[T - r + s]];
  }
  auto push = [&](const double* m, int count) -> int {
    const int at = (int)(prog.coefs.size() / 2 - cbase);
    prog.coefs.insert(prog.coefs.end(), m, m + 2 * count);
    return at;
  };
  auto push_c = [&](cd c) -> int {
    const double m[2] = {c.real(), c.imag()};
    return push(m, 1);
  };

  // Hadamard scales: every H1 of the section multiplies all amplitudes by its real scale, a global
  // scalar, so all but the last run as unscaled butterflies and the last applies the product.
  int last_h1 = -1;
  double h_scale = 1.0;
  for (const auto& po : pout)
    for (const Item& it : po.items)
      if (it.group.empty() && pg[it.gate].type == SV_OP_H1) {
        last_h1 = it.gate;
        h_scale *= gates[pg[it.gate].src].m[0];
      }
  double fpa = 0.0;  // algorithmic flops per amplitude of the section (DESIGN "Roofline")
  int op_cursor = 0;
  bool lanes_contiguous_first = false, lanes_contiguous_last = false;
  int n_diagset = 0, n_diag_fused = 0;
  for (size_t pi = 0; pi < phases.size(); pi++) {
    SvPhase* P = reinterpret_cast<SvPhase*>(prog.ints.data() + base + H()->phase_off + phase_ints * pi);
    const Ph& ph = phases[pi];
    const PhaseOut& po = pout[pi];
    for (int s = 0; s < r; s++) {
      P->R[s] = ph.R[s];
      P->rw[s] = swz[ph.R[s]];
    }
    for (size_t j = 0; j < po.chosen.size(); j++) {
      P->tpos[j] = po.chosen[j];
      P->tw[j] = swz[po.chosen[j]];
    }
    // a direct HBM boundary needs lane j of each 2^swizzle_bits group on memory bit j (128 B runs);
    // when the tile holds only memory bits 0..L-1 of them (a section with more active qubits than
    // the tile leaves room for), lanes 0..L-1 on those bits (runs of 2^L amplitudes, >= 64 B)
    auto lanes_on_low_bits = [&](const int* bits) {
      if ((int)po.chosen.size() < swizzle_bits) return false;
      int L = 0;
      for (bool found = true; found && L < swizzle_bits;) {
        found = false;
        for (int q = 0; q < T; q++) found = found || bits[q] == L;
        if (found) L++;
      }
      if (L < swizzle_bits - 1) return false;
      for (int j = 0; j < L; j++)
        if (bits[po.chosen[j]] != j) return false;
      return true;
    };
    if (pi == 0) {
      lanes_contiguous_first = lanes_on_low_bits(load_bits);
      fill_map(H()->din, po.chosen.data(), ph.R.data(), load_bits);
    }
    if (pi + 1 == phases.size()) {
      lanes_contiguous_last = lanes_on_low_bits(store_bits);
      fill_map(H()->dout, po.chosen.data(), ph.R.data(), store_bits);
    }
    P = reinterpret_cast<SvPhase*>(prog.ints.data() + base + H()->phase_off + phase_ints * pi);
    P->op_begin = op_cursor;
    P->op_count = (int)po.items.size();

    // operand code in this phase's mapping
    auto code = [&](int x) {
      if (x >= 0) return x;  // constant
      const int mb = kDiagLocal - x;
      const int pos = pos_of[mb];
      if (pos < 0) return SV_CODE_OUT(mb);
      if (po.slot_of[pos] >= 0) return SV_CODE_SLOT(po.slot_of[pos]);
      return SV_CODE_THREAD(po.thread_of[pos]);
    };

    for (const Item& it : po.items) {
      SvOp op{};
      if (!it.group.empty()) {  // ---------------------------------------------------- DIAGSET
        std::map<TermKey, cd> terms;
        auto add = [&](int ca, int cb, cd c, bool need_a, bool need_b) {
          TermKey k{0, 0u, 0ull};
          auto cond = [&](int x) -> bool {  // false: the term never applies
            if (x == SV_CODE_ZERO) return false;
            if (x == SV_CODE_ONE) return true;
            if (x < 4) k.S |= 1 << x;
            else if (x < 100) k.J |= 1u << (x - 32);
            else k.O |= 1ull << (x - 100);
            return true;
          };
          if (need_a && !cond(ca)) return;
          if (need_b && !cond(cb)) return;
          auto f = terms.find(k);
          if (f == terms.end())
            terms[k] = c;
          else
            f->second *= c;
        };
        for (int gi : it.group) {
          const PGate& p = pg[gi];
          const sv_gate& g = gates[p.src];
          const int ca = code(p.a), cb = code(p.b);
          auto cval = [&](int i) { return cd(g.m[2 * i], g.m[2 * i + 1]); };
          if (p.type == SV_OP_DIAG_CP) {
            add(ca, cb, cval(3), true, true);
          } else if (g.kind == SV_D1) {
            add(ca, cb, cval(0), false, false);
            add(ca, cb, cval(1) / cval(0), true, false);
          } else {  // general 2-qubit diagonal: d0 * (d1/d0)^a * (d2/d0)^b * (d3 d0 / (d1 d2))^(ab)
            const cd d0 = cval(0), d1 = cval(1), d2 = cval(2), d3 = cval(3);
            add(ca, cb, d0, false, false);
            add(ca, cb, d1 / d0, true, false);
            add(ca, cb, d2 / d0, false, true);
            add(ca, cb, d3 * d0 / (d1 * d2), true, true);
          }
          n_diag_fused++;
        }
        // Split the terms by register subset: |S| <= 1 (the empty set and the four slots, index
        // si = 0..4) keep per-CTA / per-thread structure; |S| >= 2 terms come from both operands
        // on register slots, so they are constants and fold into a 16-entry table LAMBDA[k].
        const int nthr = 1 << (T - r);
        std::vector<cd> lam(16, cd(1.0, 0.0));
        bool has_lam = false;
        std::vector<std::vector<cd>> tab(5, std::vector<cd>(nthr, cd(1.0, 0.0)));
        std::vector<std::vector<std::pair<uint64_t, cd>>> cta(5);
        std::vector<std::tuple<int, uint32_t, uint64_t, cd>> mixed;
        for (const auto& kv : terms) {
          const TermKey& k = kv.first;
          const int pc = __builtin_popcount(k.S);
          if (pc >= 2) {
            if (k.J || k.O) return Status::err(SV_EMALFORMED, "internal: diagonal term on >2 operands");
            for (int kk = 0; kk < 16; kk++)
              if ((kk & k.S) == k.S) lam[kk] *= kv.second;
            has_lam = true;
            continue;
          }
          const int si = pc == 0 ? 0 : 1 + __builtin_ctz(k.S);
          if (k.O == 0) {  // constant or thread-bit term: tabulated per thread index
            for (int tid = 0; tid < nthr; tid++)
              if (((uint32_t)tid & k.J) == k.J) tab[si][tid] *= kv.second;
          } else if (k.J == 0) {
            cta[si].push_back({k.O, kv.second});
          } else {
            mixed.push_back(std::make_tuple(si, k.J, k.O, kv.second));
          }
        }
        const size_t desc = prog.ints.size() - base;
        const int aux0 = (int)(prog.aux.size() / 2 - abase);
        for (int si = 0; si < 5; si++)
          for (int tid = 0; tid < nthr; tid++) {
            prog.aux.push_back(tab[si][tid].real());
            prog.aux.push_back(tab[si][tid].imag());
          }
        int set_idx = 255;  // per-CTA factors: computed once per CTA in the prologue if a slot is free
        if (H()->n_sets < SV_MAX_SETS) {
          set_idx = H()->n_sets++;
          H()->set_desc[set_idx] = (int)desc;
        }
        int tab_mask = 0;  // subsets whose per-thread table is not all ones (generated kernels skip the rest)
        for (int si = 0; si < 5; si++)
          for (int tid = 0; tid < nthr; tid++)
            if (tab[si][tid] != cd(1.0, 0.0)) {
              tab_mask |= 1 << si;
              break;
            }
        prog.ints.push_back((has_lam ? 1 : 0) | (set_idx << 8) | (tab_mask << 16));
        prog.ints.push_back(aux0);
        const size_t off = prog.ints.size();
        prog.ints.resize(prog.ints.size() + 8, 0);
        for (int si = 0; si < 5; si++) {  // per-CTA terms: (out-bit mask lo, hi, coef)
          prog.ints[off + si] = (int)(prog.ints.size() - base);
          for (const auto& tm : cta[si]) {
            prog.ints.push_back((int)(tm.first & 0xffffffffu));
            prog.ints.push_back((int)(tm.first >> 32));
            prog.ints.push_back(push_c(tm.second));
          }
        }
        prog.ints[off + 5] = (int)(prog.ints.size() - base);
        prog.ints[off + 6] = (int)(prog.ints.size() - base);  // mixed terms: (si, J, O lo, O hi, coef)
        for (const auto& tm : mixed) {
          prog.ints.push_back(std::get<0>(tm));
          prog.ints.push_back((int)std::get<1>(tm));
          prog.ints.push_back((int)(std::get<2>(tm) & 0xffffffffu));
          prog.ints.push_back((int)(std::get<2>(tm) >> 32));
          prog.ints.push_back(push_c(std::get<3>(tm)));
        }
        prog.ints[off + 7] = (int)(prog.ints.size() - base);
        int lam0 = 0;
        if (has_lam) {
          lam0 = (int)(prog.coefs.size() / 2 - cbase);
          for (int kk = 0; kk < 16; kk++) push_c(lam[kk]);
        }
        op.type = SV_OP_DIAGSET;
        op.a = (int)desc;
        op.coef = lam0;
        // flops per amplitude: build the 16 register factors from the five subset factors (~16
        // complex multiplies per thread), apply them (16), LAMBDA (16), per-thread mixed terms
        fpa += (6.0 * (32 + (has_lam ? 16 : 0) + mixed.size() + 5)) / 16.0;
        n_diagset++;
      } else {  // ---------------------------------------------------------------- single op
        const PGate& p = pg[it.gate];
        const sv_gate& g = gates[p.src];
        op.type = p.type;
        op.extra = p.extra;
        switch (p.type) {
          case SV_OP_U2: {
            int sa = po.slot_of[p.a], sb = po.slot_of[p.b];
            double m[32];
            std::memcpy(m, g.m, sizeof(m));
            if (sa > sb) {  // canonical slot order: conjugate by the s=1 <-> s=2 permutation
              static const int sw[4] = {0, 2, 1, 3};
              for (int rr = 0; rr < 4; rr++)
                for (int cc = 0; cc < 4; cc++) {
                  m[2 * (4 * rr + cc)] = g.m[2 * (4 * sw[rr] + sw[cc])];
                  m[2 * (4 * rr + cc) + 1] = g.m[2 * (4 * sw[rr] + sw[cc]) + 1];
                }
              std::swap(sa, sb);
            }
            op.a = sa;
            op.b = sb;
            op.coef = push(m, 16);
            {  // Gauss form for the kernel: (-(re + im), im - re) per entry (section_dev.cuh u2_slots)
              double gm[32];
              for (int e = 0; e < 16; e++) {
                gm[2 * e] = -(m[2 * e] + m[2 * e + 1]);
                gm[2 * e + 1] = m[2 * e + 1] - m[2 * e];
              }
              push(gm, 16);
            }
            fpa += 32.0;
            break;
          }
          case SV_OP_PERM2: {
            int sa = po.slot_of[p.a], sb = po.slot_of[p.b];
            if (sa > sb) {  // canonical slot order: relabel s = bit(a) + 2 bit(b) by swapping its bits
              auto swb = [](int s) { return ((s & 1) << 1) | (s >> 1); };
              int np = 0;
              for (int s2 = 0; s2 < 4; s2++) np |= swb((p.extra >> (2 * swb(s2))) & 3) << (2 * s2);
              op.extra = np;
              std::swap(sa, sb);
            }
            op.a = sa;
            op.b = sb;
            op.coef = 0;
            break;
          }
          case SV_OP_U1:
            op.a = po.slot_of[p.a];
            op.coef = push(g.m, 4);
            fpa += 16.0;
            break;
          case SV_OP_H1: {
            op.a = po.slot_of[p.a];
            if (it.gate == last_h1) {
              const double s[2] = {h_scale, 0.0};
              op.coef = push(s, 1);
              fpa += 4.0;
            } else {
              op.type = SV_OP_H1U;
              op.coef = 0;
              fpa += 2.0;
            }
            break;
          }
          case SV_OP_DIAG:
          case SV_OP_DIAG_CP: {
            int ca = code(p.a), cb = code(p.b);
            double d[8] = {1, 0, 1, 0, 1, 0, 1, 0};
            std::memcpy(d, g.m, sizeof(double) * (g.kind == SV_D2 ? 8 : 4));
            // canonical form for the kernel: a register-slot operand comes first, two slots ascend
            if (cb < 4 && (ca >= 4 || cb < ca)) {
              std::swap(ca, cb);
              std::swap(d[2], d[4]);  // d[s] with s = bit(a) + 2 bit(b): exchange s = 1 and s = 2
              std::swap(d[3], d[5]);
            }
            op.a = ca;
            op.b = cb;
            if (p.type == SV_OP_DIAG_CP) {
              op.coef = push(d + 6, 1);
              fpa += 1.5;
            } else {
              op.coef = push(d, 4);
              fpa += 6.0;
            }
            break;
          }
        }
      }
      std::memcpy(prog.ints.data() + base + H()->op_off + op_ints * op_cursor, &op, sizeof(op));
      op_cursor++;
    }
  }
  H()->flags = (lanes_contiguous_first ? SV_FLAG_FIRST_DIRECT : 0) | (lanes_contiguous_last ? SV_FLAG_LAST_DIRECT : 0);
  H()->nl = nL;
  const size_t total_ints = prog.ints.size() - base;
  const size_t ncoef = prog.coefs.size() / 2 - cbase;
  const size_t coef_cap = swizzle_bits == 3 ? SV_CONST_COEF64 : SV_CONST_COEF32;
  if (total_ints > SV_CONST_INTS || ncoef > coef_cap) {
    prog.ints.resize(base);
    prog.coefs.resize(cbase * 2);
    prog.aux.resize(abase * 2);
    return Status::err(kTooBig, "section program exceeds the constant budget");
  }

  if (std::getenv("SV_DEBUG_PLAN")) {  // per-section compile report (analysis aid)
    std::fprintf(stderr,
                 "[sv] section T=%d phases=%zu items=%zu gates=%zu diagsets=%d fused_diag=%d flags=%d "
                 "flops/amp=%.1f ints=%zu coefs=%zu low-tile-bits=%d%d%d%d\n",
                 T, phases.size(), n_items, gates.size(), n_diagset, n_diag_fused, H()->flags, fpa, total_ints, ncoef,
                 (int)(tile & 1), (int)((tile >> 1) & 1), (int)((tile >> 2) & 1), (int)((tile >> 3) & 1));
  }
  Launch L;
  L.flops_per_amp = fpa;
  L.int_off = base;
  L.int_count = total_ints;
  L.coef_off = cbase;
  L.coef_count = ncoef;
  L.aux_off = abase;
  L.aux_count = prog.aux.size() / 2 - abase;
  L.T = T;
  L.r = r;
  L.n_out = n_out;
  L.n_phases = (int)phases.size();
  L.n_ops = (int)n_items;
  L.flags = H()->flags;
  L.n_sets = H()->n_sets;
  prog.launches.push_back(L);
  // keep every section 16-byte aligned
  while (prog.ints.size() % 4) prog.ints.push_back(0);
  return Status::ok();
}

Status compile_section_split(const std::vector<sv_gate>& gates, int nL, int rank, int world_log2, int T_default,
                             int swizzle_bits, const std::vector<std::pair<int, int>>& store_swaps, Program& prog) {
  const size_t ni = prog.ints.size(), nc = prog.coefs.size(), na = prog.aux.size();
  Status s = compile_section(gates, nL, rank, world_log2, T_default, swizzle_bits, store_swaps, prog);
  if (s.code != kTooBig) return s;
  prog.ints.resize(ni);
  prog.coefs.resize(nc);
  prog.aux.resize(na);
  if (gates.size() < 2) return Status::err(SV_ECAPACITY, "a single gate exceeds the constant budget");
  // Consecutive halves of the in-order gate list: each half is a valid section on its own.
  const size_t h = gates.size() / 2;
  std::vector<sv_gate> a(gates.begin(), gates.begin() + h), b(gates.begin() + h, gates.end());
  if (Status sa = compile_section_split(a, nL, rank, world_log2, T_default, swizzle_bits, {}, prog); !sa.good())
    return sa;
  return compile_section_split(b, nL, rank, world_log2, T_default, swizzle_bits, store_swaps, prog);
}

}  // namespace sv
