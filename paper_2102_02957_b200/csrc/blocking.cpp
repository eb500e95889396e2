// blocking.cpp — the cache-blocking transpiler pass (host C++), §IV-A.
//
// Listing 3: repeat { choose the chunk qubits; insert chunk_swaps that bring them
// into the chunk; scan the remaining gates in order, emitting those whose qubits are all in
// the chunk and not blocked, deferring (and blocking the qubits of) the rest }.  The paper
// leaves the selection rule and the eviction order open; this file implements the readings
// fixed in DESIGN.md:
//   R2  all c slots are usable (QB_CHUNK[nc-1] read as the top index of a c-slot array);
//   R2' the deferral branch sets QB_BLOCKED on every qubit of every deferred gate (P:326 prose);
//   R3  selection = in-order, dependency-aware greedy: walk the queue, skip gates touching a
//       blocked qubit (blocking theirs too), skip diagonal gates, admit a gate only whole;
//   R4  chunk_swaps fill the free slots in DESCENDING slot order;
//   R5  diagonal gates are always executable inside a chunk and are never selected;
//   R6  SWAP is an ordinary non-diagonal two-qubit gate — or, with SV_ABSORB_SWAPS (SURVEY Q6,
//       the paper's "bit reordering"), a relabel of pi at the point the section reaches
//       it: selection then sees later gates on the swapped qubits through the same relabel, and
//       a section left with no gate is not emitted.
// Bitmasks over qubits (n <= 40) keep the pass O(gates * sections) with small constants.
#include <algorithm>
#include <cstring>

#include "common.h"

namespace sv {

Status validate_gates(const sv_gate* g, size_t count, int n) {
  for (size_t i = 0; i < count; i++) {
    const sv_gate& r = g[i];
    if (r.kind < SV_U1 || r.kind > SV_SWAP)
      return Status::err(SV_EMALFORMED, "gate " + std::to_string(i) + ": kind " + std::to_string(r.kind) +
                                            " is not an input kind (U1, U2, D1, D2, SWAP)");
    if (r.q0 < 0 || r.q0 >= n) return Status::err(SV_EINVAL, "gate " + std::to_string(i) + ": qubit q0 out of range");
    if (is_two(r.kind)) {
      if (r.q1 < 0 || r.q1 >= n) return Status::err(SV_EINVAL, "gate " + std::to_string(i) + ": qubit q1 out of range");
      if (r.q1 == r.q0) return Status::err(SV_EINVAL, "gate " + std::to_string(i) + ": duplicate qubit");
    }
  }
  return Status::ok();
}

static sv_gate marker(int kind) {
  sv_gate t;
  std::memset(&t, 0, sizeof(t));
  t.kind = kind;
  t.q0 = t.q1 = -1;
  return t;
}

static sv_gate chunk_swap(int sq0, int sq1) {
  sv_gate t = marker(SV_CHUNK_SWAP);
  t.q0 = sq0;
  t.q1 = sq1;
  return t;
}

Status block_pass(const sv_gate* g, size_t count, int n, int c, std::vector<int>& pi, uint32_t flags,
                  std::vector<sv_gate>& tokens) {
  if (n < 1 || n > 63) return Status::err(SV_EINVAL, "n out of range");
  if (c < 1 || c > n) return Status::err(SV_EINVAL, "chunk_bits must satisfy 1 <= c <= n");
  if ((int)pi.size() != n) return Status::err(SV_EINVAL, "pi has wrong length");
  if (Status s = validate_gates(g, count, n); !s.good()) return s;
  if (c < 2)
    for (size_t i = 0; i < count; i++)
      if (is_two(g[i].kind) && !is_diag(g[i].kind))
        return Status::err(SV_EINFEASIBLE, "a non-diagonal two-qubit gate needs chunk_bits >= 2 (P:324)");

  // where[p] = logical qubit at physical position p (inverse of pi)
  std::vector<int> where(n, -1);
  for (int q = 0; q < n; q++) {
    if (pi[q] < 0 || pi[q] >= n || where[pi[q]] != -1) return Status::err(SV_EINVAL, "pi0 is not a permutation");
    where[pi[q]] = q;
  }
  std::vector<uint64_t> masks(count);
  for (size_t i = 0; i < count; i++) masks[i] = qmask(g[i]);

  std::vector<uint32_t> queue(count), next;
  for (size_t i = 0; i < count; i++) queue[i] = (uint32_t)i;
  next.reserve(count);

  const bool absorb = (flags & SV_ABSORB_SWAPS) != 0;
  std::vector<int> chosen;  // QB_CHUNK, in selection order
  std::vector<int> sel(n);  // absorbed swaps during selection: logical q -> the section-start qubit
  while (!queue.empty()) {
    // --- choose QB_CHUNK (R3)
    chosen.clear();
    for (int q = 0; q < n; q++) sel[q] = q;
    uint64_t chosen_mask = 0, blocked = 0;
    for (uint32_t gi : queue) {
      const uint64_t qm = masks[gi];
      if (qm & blocked) {
        blocked |= qm;
        continue;
      }
      if (is_diag(g[gi].kind)) continue;
      if (absorb && g[gi].kind == SV_SWAP) {
        std::swap(sel[g[gi].q0], sel[g[gi].q1]);
        continue;
      }
      uint64_t need = (1ull << sel[g[gi].q0]) | (is_two(g[gi].kind) ? 1ull << sel[g[gi].q1] : 0ull);
      need &= ~chosen_mask;
      if ((int)chosen.size() + __builtin_popcountll(need) <= c) {
        while (need) {  // ascending qubit order
          int q = __builtin_ctzll(need);
          need &= need - 1;
          chosen.push_back(q);
          chosen_mask |= 1ull << q;
        }
      } else {
        blocked |= qm;
      }
      if ((int)chosen.size() == c) break;
    }
    // --- insert chunk_swaps (R4): incoming qubits in selection order, free slots descending
    std::vector<int> free_slots;
    for (int p = c - 1; p >= 0; p--)
      if (!((chosen_mask >> where[p]) & 1)) free_slots.push_back(p);
    size_t fi = 0;
    for (int q : chosen) {
      if (pi[q] < c) continue;
      const int slot = free_slots[fi++];
      const int far = pi[q];
      tokens.push_back(chunk_swap(slot, far));
      const int evicted = where[slot];
      pi[evicted] = far;
      where[far] = evicted;
      pi[q] = slot;
      where[slot] = q;
    }
    // --- emit the section
    const size_t begin_at = tokens.size();
    tokens.push_back(marker(SV_BEGIN));
    uint64_t blk = 0;
    next.clear();
    for (uint32_t gi : queue) {
      const sv_gate& r = g[gi];
      const uint64_t qm = masks[gi];
      if (qm & blk) {
        blk |= qm;
        next.push_back(gi);
        continue;
      }
      if (absorb && r.kind == SV_SWAP) {  // the state of q0 now lives where q1's was, and vice versa
        const int a = pi[r.q0], b = pi[r.q1];
        pi[r.q0] = b;
        pi[r.q1] = a;
        where[a] = r.q1;
        where[b] = r.q0;
        continue;
      }
      bool local = is_diag(r.kind) || (pi[r.q0] < c && (!is_two(r.kind) || pi[r.q1] < c));
      if (local) {
        sv_gate t = r;
        t.q0 = pi[r.q0];
        t.q1 = is_two(r.kind) ? pi[r.q1] : -1;
        t.pad = (int32_t)gi;
        tokens.push_back(t);
      } else {
        blk |= qm;
        next.push_back(gi);
      }
    }
    if (tokens.size() == begin_at + 1)
      tokens.pop_back();  // nothing but absorbed swaps: no section
    else
      tokens.push_back(marker(SV_END));
    queue.swap(next);
  }

  if (flags & SV_RESTORE_ORDER) {  // P:379 case (b): reorder qubits for the output
    for (int p = 0; p < n; p++) {
      const int q = where[p];
      if (q == p) continue;
      const int t = pi[p];  // > p: every position below p already holds its own qubit
      if (t >= c) {
        tokens.push_back(chunk_swap(p, t));
      } else {
        tokens.push_back(marker(SV_BEGIN));
        sv_gate s = marker(SV_SWAP);
        s.q0 = p;
        s.q1 = t;
        s.pad = -1;
        tokens.push_back(s);
        tokens.push_back(marker(SV_END));
      }
      pi[q] = t;
      where[t] = q;
      pi[p] = p;
      where[p] = p;
    }
  }
  return Status::ok();
}

}  // namespace sv
