// compile.cpp — section compiler: memory-frame section -> SvSecHeader/SvPhase/SvOp program.
//
// See program.h for the model.  Phase scheduling is a greedy in-order list schedule over the
// section's gates: a gate joins the current phase if no earlier deferred gate of this phase
// shares a tile position with it and its non-diagonal positions fit the R_BITS register slots;
// diagonal gates join whenever their dependencies allow (they act per amplitude).
// Reordering only qubit-disjoint gates is the same legality rule the pass uses.
#include <algorithm>
#include <cmath>
#include <cstring>

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
  int a, b;          // slots are assigned later; here: positions (U*) or codes (DIAG)
  uint32_t pmask;    // tile positions it touches (for dependencies)
  bool diag;
  int coef;          // offset (in complex numbers) into Program::coefs
  int extra;
};

}  // namespace

Status compile_section(const std::vector<sv_gate>& gates, int nL, int rank, int world_log2, int T_default,
                       int swizzle_bits, Program& prog) {
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
  int T = std::max(std::min(T_default, nL), nA);
  if (T > SV_TMAX) return Status::err(SV_ECAPACITY, "section needs more tile bits than shared memory holds");
  uint64_t tile = active;
  for (int b = 0; b < nL && __builtin_popcountll(tile) < T; b++) tile |= 1ull << b;
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

  auto code_of = [&](int mb) -> int {
    if (mb >= nL) return ((rank >> (mb - nL)) & 1) ? SV_CODE_ONE : SV_CODE_ZERO;
    if (pos_of[mb] >= 0) return SV_CODE_TILE(pos_of[mb]);
    return SV_CODE_OUT(mb);
  };
  auto push_coef = [&](const double* m, int count) -> int {
    const int at = (int)(prog.coefs.size() / 2);
    prog.coefs.insert(prog.coefs.end(), m, m + 2 * count);
    return at;
  };

  // ---- gates on positions
  std::vector<PGate> pg;
  pg.reserve(gates.size());
  for (const sv_gate& g : gates) {
    PGate p{};
    p.extra = 0;
    switch (g.kind) {
      case SV_U1:
        p.a = pos_of[g.q0];
        p.pmask = 1u << p.a;
        if (is_h_like(g.m)) {
          p.type = SV_OP_H1;
          const double s[2] = {g.m[0], 0.0};
          p.coef = push_coef(s, 1);
        } else {
          p.type = SV_OP_U1;
          p.coef = push_coef(g.m, 4);
        }
        break;
      case SV_U2: {
        p.a = pos_of[g.q0];
        p.b = pos_of[g.q1];
        p.pmask = (1u << p.a) | (1u << p.b);
        int perm[4];
        if (is_perm4(g.m, perm)) {
          p.type = SV_OP_PERM2;
          p.extra = perm[0] | (perm[1] << 2) | (perm[2] << 4) | (perm[3] << 6);
          p.coef = 0;
        } else {
          p.type = SV_OP_U2;
          p.coef = push_coef(g.m, 16);
        }
        break;
      }
      case SV_D1:
      case SV_D2: {
        p.diag = true;
        p.a = code_of(g.q0);
        p.b = g.kind == SV_D2 ? code_of(g.q1) : SV_CODE_ZERO;
        p.pmask = 0;
        if (p.a < 100) p.pmask |= 1u << p.a;
        if (p.b < 100) p.pmask |= 1u << p.b;
        double d[8] = {1, 0, 1, 0, 1, 0, 1, 0};
        std::memcpy(d, g.m, sizeof(double) * (g.kind == SV_D2 ? 8 : 4));
        const bool cp = g.kind == SV_D2 && d[0] == 1.0 && d[1] == 0.0 && d[2] == 1.0 && d[3] == 0.0 &&
                        d[4] == 1.0 && d[5] == 0.0;
        if (cp) {
          p.type = SV_OP_DIAG_CP;
          p.coef = push_coef(d + 6, 1);
        } else {
          p.type = SV_OP_DIAG;
          p.coef = push_coef(d, 4);
        }
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
    // pad the register set with the highest free positions (keeps low positions as thread bits)
    for (int pos = T - 1; pos >= 0 && __builtin_popcount(rmask) < r; pos--) rmask |= 1u << pos;
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
  const int n_ops = (int)pg.size();
  const int header_ints = sizeof(SvSecHeader) / 4;
  const int phase_ints = sizeof(SvPhase) / 4;
  const int op_ints = sizeof(SvOp) / 4;
  prog.ints.resize(base + header_ints + phase_ints * phases.size() + op_ints * n_ops, 0);
  SvSecHeader* H = reinterpret_cast<SvSecHeader*>(prog.ints.data() + base);
  H->T = T;
  H->r = r;
  H->n_out = n_out;
  H->n_phases = (int)phases.size();
  H->phase_off = header_ints;
  H->op_off = header_ints + phase_ints * (int)phases.size();
  H->n_ops = n_ops;
  for (int j = 0; j < T; j++) H->tile_bits[j] = tile_bits[j];
  for (int j = 0; j < n_out; j++) H->out_bits[j] = out_bits[j];

  int op_cursor = 0;
  for (size_t pi = 0; pi < phases.size(); pi++) {
    SvPhase* P = reinterpret_cast<SvPhase*>(prog.ints.data() + base + H->phase_off + phase_ints * pi);
    const Ph& ph = phases[pi];
    int slot_of[SV_TMAX];
    std::fill(slot_of, slot_of + SV_TMAX, -1);
    for (int s = 0; s < r; s++) {
      P->R[s] = ph.R[s];
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
    for (size_t j = 0; j < chosen.size(); j++) P->tpos[j] = chosen[j];
    P->op_begin = op_cursor;
    P->op_count = (int)ph.ops.size();
    for (int gi : ph.ops) {
      SvOp* O = reinterpret_cast<SvOp*>(prog.ints.data() + base + H->op_off + op_ints * op_cursor);
      const PGate& p = pg[gi];
      O->type = p.type;
      O->coef = p.coef;
      O->extra = p.extra;
      if (p.diag) {
        O->a = p.a;
        O->b = p.b;
      } else {
        O->a = slot_of[p.a];
        O->b = (p.type == SV_OP_U2 || p.type == SV_OP_PERM2) ? slot_of[p.b] : -1;
      }
      op_cursor++;
    }
  }
  // algorithmic flops per amplitude: U2 4x4 complex matvec = 32, U1 = 16, H1 = 4, PERM = 0,
  // DIAG = one complex multiply (6), DIAG_CP = one complex multiply on a quarter (1.5)
  double fpa = 0.0;
  for (const PGate& p : pg)
    fpa += p.type == SV_OP_U2 ? 32.0 : p.type == SV_OP_U1 ? 16.0 : p.type == SV_OP_H1 ? 4.0
         : p.type == SV_OP_DIAG ? 6.0 : p.type == SV_OP_DIAG_CP ? 1.5 : 0.0;
  Launch L;
  L.flops_per_amp = fpa;
  L.int_off = base;
  L.T = T;
  L.r = r;
  L.n_out = n_out;
  L.n_phases = (int)phases.size();
  L.n_ops = n_ops;
  prog.launches.push_back(L);
  // keep every section 16-byte aligned
  while (prog.ints.size() % 4) prog.ints.push_back(0);
  return Status::ok();
}

}  // namespace sv
