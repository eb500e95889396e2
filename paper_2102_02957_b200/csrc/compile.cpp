// compile.cpp — section compiler: memory-frame section -> SvSecHeader/SvPhase/SvOp program.
//
// See program.h for the model.  Phase scheduling is a greedy in-order list schedule over the
// section's gates: a gate joins the current phase if no earlier deferred gate of this phase
// shares a tile position with it and its non-diagonal positions fit the R_BITS register slots;
// diagonal gates join whenever their dependencies allow (they act per amplitude).
// Reordering only qubit-disjoint gates is the same legality rule the pass uses.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <utility>

#include "common.h"
#include "compile.h"

namespace sv {

namespace {

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
  int a, b;        // positions (U*/PERM) or memory-bit codes (DIAG: -1-mb local, 200/201 const)
  uint32_t pmask;  // tile positions it touches (for dependencies)
  bool diag;
  int src;         // index into the section's gate list (payload source)
  int extra;
};

constexpr int kDiagLocal = -1;  // DIAG operand: -(1 + memory bit)
constexpr int kMaxTile = 13;    // 2^13 amplitudes: 128 KiB fp64 / 64 KiB fp32 of shared memory

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
  const int nA = __builtin_popcountll(active);
  // The tile always includes the lowest memory bits (128-byte runs: 8 fp64 / 16 fp32 amplitudes)
  // when they fit; the planner (plan.cpp) arranges that they do.
  PlanLayout lay;
  lay.low_bits = swizzle_bits;
  lay.max_tile = kMaxTile;
  lay.tile_default = T_default;
  const uint64_t tile = choose_tile(active, nL, lay);
  const int T = __builtin_popcountll(tile);
  if (T > kMaxTile) return Status::err(SV_ECAPACITY, "section needs more tile bits than shared memory holds");
  int tile_bits[16], pos_of[64];
  std::fill(pos_of, pos_of + 64, -1);
  int t = 0;
  for (int b = 0; b < nL; b++)
    if ((tile >> b) & 1) {
      pos_of[b] = t;
      tile_bits[t++] = b;
    }
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
  size_t ncoef = 0;
  for (size_t gi = 0; gi < gates.size(); gi++) {
    const sv_gate& g = gates[gi];
    PGate p{};
    p.src = (int)gi;
    switch (g.kind) {
      case SV_U1:
        p.a = pos_of[g.q0];
        p.pmask = 1u << p.a;
        p.type = is_h_like(g.m) ? SV_OP_H1 : SV_OP_U1;
        ncoef += p.type == SV_OP_H1 ? 1 : 4;
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
          ncoef += 16;
        }
        break;
      }
      case SV_D1:
      case SV_D2: {
        p.diag = true;
        auto operand = [&](int mb) {
          if (mb >= nL) return ((rank >> (mb - nL)) & 1) ? SV_CODE_ONE : SV_CODE_ZERO;
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
        ncoef += cp ? 1 : 4;
        break;
      }
      default:
        return Status::err(SV_EMALFORMED, "internal: unexpected kind in section");
    }
    pg.push_back(p);
  }
  const size_t coef_cap = swizzle_bits == 3 ? SV_CONST_COEF64 : SV_CONST_COEF32;
  if (ncoef > coef_cap) return Status::err(kTooBig, "section coefficients exceed the constant budget");

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

  // ---- emit
  const size_t base = prog.ints.size();
  const size_t cbase = prog.coefs.size() / 2;
  const int n_ops = (int)pg.size();
  const int header_ints = sizeof(SvSecHeader) / 4;
  const int phase_ints = sizeof(SvPhase) / 4;
  const int op_ints = sizeof(SvOp) / 4;
  const size_t total_ints = header_ints + phase_ints * phases.size() + op_ints * (size_t)n_ops;
  if (total_ints > SV_CONST_INTS) return Status::err(kTooBig, "section program exceeds the constant budget");
  prog.ints.resize(base + total_ints, 0);
  SvSecHeader* H = reinterpret_cast<SvSecHeader*>(prog.ints.data() + base);
  H->T = T;
  H->r = r;
  H->n_out = n_out;
  H->n_phases = (int)phases.size();
  H->phase_off = header_ints;
  H->op_off = header_ints + phase_ints * (int)phases.size();
  H->n_ops = n_ops;
  int store_bits[16];
  for (int j = 0; j < T; j++) store_bits[j] = tile_bits[j];
  for (const auto& sw : store_swaps) {  // physical bit swaps fused into the store (plan.cpp)
    const int p1 = sw.first < 64 ? pos_of[sw.first] : -1, p2 = sw.second < 64 ? pos_of[sw.second] : -1;
    if (p1 < 0 || p2 < 0) return Status::err(SV_EMALFORMED, "internal: store swap outside the tile");
    std::swap(store_bits[p1], store_bits[p2]);
  }
  for (int j = 0; j < T; j++) {
    H->tile_bits[j] = tile_bits[j];
    H->store_bits[j] = store_bits[j];
  }
  for (int j = 0; j < n_out; j++) H->out_bits[j] = out_bits[j];
  auto fill_map = [&](SvMap& m, const int* tpos, const int* R, const int* bits) {
    for (int j = 0; j < T - r; j++) {
      m.tw[j] = sv_swz_host(1 << tpos[j], swizzle_bits);
      m.tmb[j] = bits[tpos[j]];
    }
    for (int s = 0; s < r; s++) {
      m.rw[s] = sv_swz_host(1 << R[s], swizzle_bits);
      m.rmb[s] = bits[R[s]];
    }
  };
  {  // boundary maps: lanes walk the lowest memory bits of the load / store side
    int order[16];
    for (int j = 0; j < T; j++) order[j] = j;
    fill_map(H->load, order, order + (T - r), tile_bits);
    std::sort(order, order + T, [&](int a, int b) { return store_bits[a] < store_bits[b]; });
    fill_map(H->store, order, order + (T - r), tile_bits);
    for (int j = 0; j < T - r; j++) H->store.tmb[j] = store_bits[order[j]];
    for (int s = 0; s < r; s++) H->store.rmb[s] = store_bits[order[T - r + s]];
  }
  auto push = [&](const double* m, int count) -> int {
    const int at = (int)(prog.coefs.size() / 2 - cbase);
    prog.coefs.insert(prog.coefs.end(), m, m + 2 * count);
    return at;
  };

  int op_cursor = 0;
  bool lanes_contiguous_first = false, lanes_contiguous_last = false;
  for (size_t pi = 0; pi < phases.size(); pi++) {
    SvPhase* P = reinterpret_cast<SvPhase*>(prog.ints.data() + base + H->phase_off + phase_ints * pi);
    const Ph& ph = phases[pi];
    int slot_of[SV_TMAX];
    std::fill(slot_of, slot_of + SV_TMAX, -1);
    for (int s = 0; s < r; s++) {
      P->R[s] = ph.R[s];
      P->rw[s] = sv_swz_host(1 << ph.R[s], swizzle_bits);
      slot_of[ph.R[s]] = s;
    }
    // thread bits: the first `swizzle_bits` get distinct residues mod swizzle_bits so a group of
    // 2^swizzle_bits lanes hits distinct 16-/8-byte bank groups under the XOR-fold swizzle.
    std::vector<int> cand, chosen;
    for (int pos = 0; pos < T; pos++)
      if (slot_of[pos] < 0) cand.push_back(pos);
    uint32_t used_res = 0;
    std::vector<bool> taken(cand.size(), false);
    for (size_t i = 0; i < cand.size() && (int)chosen.size() < swizzle_bits; i++) {
      const int res = cand[i] % swizzle_bits;
      if (!((used_res >> res) & 1)) {
        used_res |= 1u << res;
        chosen.push_back(cand[i]);
        taken[i] = true;
      }
    }
    for (size_t i = 0; i < cand.size(); i++)
      if (!taken[i]) chosen.push_back(cand[i]);
    int thread_of[SV_TMAX];
    std::fill(thread_of, thread_of + SV_TMAX, -1);
    for (size_t j = 0; j < chosen.size(); j++) {
      P->tpos[j] = chosen[j];
      P->tw[j] = sv_swz_host(1 << chosen[j], swizzle_bits);
      thread_of[chosen[j]] = (int)j;
    }
    // a direct HBM boundary needs lane j of each 2^swizzle_bits group on memory bit j (128 B runs)
    auto lanes_on_low_bits = [&](const int* bits) {
      if ((int)chosen.size() < swizzle_bits) return false;
      for (int j = 0; j < swizzle_bits; j++)
        if (bits[chosen[j]] != j) return false;
      return true;
    };
    if (pi == 0) {
      lanes_contiguous_first = lanes_on_low_bits(tile_bits);
      fill_map(H->din, chosen.data(), ph.R.data(), tile_bits);
    }
    if (pi + 1 == phases.size()) {
      lanes_contiguous_last = lanes_on_low_bits(store_bits);
      fill_map(H->dout, chosen.data(), ph.R.data(), store_bits);
    }

    P->op_begin = op_cursor;
    P->op_count = (int)ph.ops.size();
    for (int gi : ph.ops) {
      SvOp* O = reinterpret_cast<SvOp*>(prog.ints.data() + base + H->op_off + op_ints * op_cursor);
      const PGate& p = pg[gi];
      const sv_gate& g = gates[p.src];
      O->type = p.type;
      O->extra = p.extra;
      switch (p.type) {
        case SV_OP_U2: {
          int sa = slot_of[p.a], sb = slot_of[p.b];
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
          O->a = sa;
          O->b = sb;
          O->coef = push(m, 16);
          break;
        }
        case SV_OP_PERM2: {
          int sa = slot_of[p.a], sb = slot_of[p.b];
          if (sa > sb) {  // canonical slot order: relabel s = bit(a) + 2 bit(b) by swapping its bits
            auto swb = [](int s) { return ((s & 1) << 1) | (s >> 1); };
            int np = 0;
            for (int s2 = 0; s2 < 4; s2++) np |= swb((p.extra >> (2 * swb(s2))) & 3) << (2 * s2);
            O->extra = np;
            std::swap(sa, sb);
          }
          O->a = sa;
          O->b = sb;
          O->coef = 0;
          break;
        }
        case SV_OP_U1:
          O->a = slot_of[p.a];
          O->coef = push(g.m, 4);
          break;
        case SV_OP_H1: {
          O->a = slot_of[p.a];
          const double s[2] = {g.m[0], 0.0};
          O->coef = push(s, 1);
          break;
        }
        case SV_OP_DIAG:
        case SV_OP_DIAG_CP: {
          auto code = [&](int x) {
            if (x >= 0) return x;  // constant
            const int mb = kDiagLocal - x;
            const int pos = pos_of[mb];
            if (pos < 0) return SV_CODE_OUT(mb);
            if (slot_of[pos] >= 0) return SV_CODE_SLOT(slot_of[pos]);
            return SV_CODE_THREAD(thread_of[pos]);
          };
          int ca = code(p.a), cb = code(p.b);
          double d[8] = {1, 0, 1, 0, 1, 0, 1, 0};
          std::memcpy(d, g.m, sizeof(double) * (g.kind == SV_D2 ? 8 : 4));
          // canonical form for the kernel: a register-slot operand comes first, two slots ascend
          if (cb < 4 && (ca >= 4 || cb < ca)) {
            std::swap(ca, cb);
            std::swap(d[2], d[4]);  // d[s] with s = bit(a) + 2 bit(b): exchange s = 1 and s = 2
            std::swap(d[3], d[5]);
          }
          O->a = ca;
          O->b = cb;
          if (p.type == SV_OP_DIAG_CP)
            O->coef = push(d + 6, 1);
          else
            O->coef = push(d, 4);
          break;
        }
      }
      op_cursor++;
    }
  }
  H->flags = (lanes_contiguous_first ? SV_FLAG_FIRST_DIRECT : 0) | (lanes_contiguous_last ? SV_FLAG_LAST_DIRECT : 0);

  // algorithmic flops per amplitude: U2 4x4 complex matvec = 32, U1 = 16, H1 = 4, PERM = 0,
  // DIAG = one complex multiply (6), DIAG_CP = one complex multiply on a quarter (1.5)
  double fpa = 0.0;
  for (const PGate& p : pg)
    fpa += p.type == SV_OP_U2 ? 32.0 : p.type == SV_OP_U1 ? 16.0 : p.type == SV_OP_H1 ? 4.0
         : p.type == SV_OP_DIAG ? 6.0 : p.type == SV_OP_DIAG_CP ? 1.5 : 0.0;
  if (std::getenv("SV_DEBUG_PLAN")) {  // per-section compile report (analysis aid)
    int cnt[8] = {0}, diag_kind[3] = {0};  // diag operands: slot-slot, slot-other, other-other
    for (int i = 0; i < n_ops; i++) {
      const SvOp* O = reinterpret_cast<const SvOp*>(prog.ints.data() + base + H->op_off + op_ints * i);
      cnt[O->type]++;
      if (O->type == SV_OP_DIAG || O->type == SV_OP_DIAG_CP) diag_kind[(O->a >= 4) + (O->b >= 4)]++;
    }
    std::fprintf(stderr,
                 "[sv] section T=%d phases=%zu ops=%d U2=%d U1=%d H1=%d PERM=%d DIAG=%d CP=%d (ss=%d so=%d oo=%d) "
                 "flags=%d flops/amp=%.1f low-tile-bits=%d%d%d%d\n",
                 T, phases.size(), n_ops, cnt[SV_OP_U2], cnt[SV_OP_U1], cnt[SV_OP_H1], cnt[SV_OP_PERM2],
                 cnt[SV_OP_DIAG], cnt[SV_OP_DIAG_CP], diag_kind[0], diag_kind[1], diag_kind[2], H->flags, fpa,
                 (int)(tile & 1), (int)((tile >> 1) & 1), (int)((tile >> 2) & 1), (int)((tile >> 3) & 1));
  }
  Launch L;
  L.flops_per_amp = fpa;
  L.int_off = base;
  L.int_count = total_ints;
  L.coef_off = cbase;
  L.coef_count = prog.coefs.size() / 2 - cbase;
  L.T = T;
  L.r = r;
  L.n_out = n_out;
  L.n_phases = (int)phases.size();
  L.n_ops = n_ops;
  L.flags = H->flags;
  prog.launches.push_back(L);
  // keep every section 16-byte aligned
  while (prog.ints.size() % 4) prog.ints.push_back(0);
  return Status::ok();
}

Status compile_section_split(const std::vector<sv_gate>& gates, int nL, int rank, int world_log2, int T_default,
                             int swizzle_bits, const std::vector<std::pair<int, int>>& store_swaps, Program& prog) {
  const size_t ni = prog.ints.size(), nc = prog.coefs.size();
  Status s = compile_section(gates, nL, rank, world_log2, T_default, swizzle_bits, store_swaps, prog);
  if (s.code != kTooBig) return s;
  prog.ints.resize(ni);
  prog.coefs.resize(nc);
  if (gates.size() < 2) return Status::err(SV_ECAPACITY, "a single gate exceeds the constant budget");
  // Consecutive halves of the in-order gate list: each half is a valid section on its own.
  const size_t h = gates.size() / 2;
  std::vector<sv_gate> a(gates.begin(), gates.begin() + h), b(gates.begin() + h, gates.end());
  if (Status sa = compile_section_split(a, nL, rank, world_log2, T_default, swizzle_bits, {}, prog); !sa.good())
    return sa;
  return compile_section_split(b, nL, rank, world_log2, T_default, swizzle_bits, store_swaps, prog);
}

}  // namespace sv
