// common.h — internal helpers shared by the host C++ and CUDA sources of libsv.so.
#pragma once
#include <cstdint>
#include <cstdlib>
#include <string>
#include <utility>
#include <vector>

#include "../../include/sv.h"

namespace sv {

inline bool is_diag(int kind) { return kind == SV_D1 || kind == SV_D2; }
inline bool is_two(int kind) {
  return kind == SV_U2 || kind == SV_D2 || kind == SV_SWAP || kind == SV_CHUNK_SWAP || kind == SV_EXCHANGE;
}
inline bool is_one(int kind) { return kind == SV_U1 || kind == SV_D1; }
inline uint64_t qmask(const sv_gate& g) {
  uint64_t m = 0;
  if (is_one(g.kind)) m = 1ull << g.q0;
  if (is_two(g.kind)) m = (1ull << g.q0) | (1ull << g.q1);
  return m;
}

// Status carried through the host code; converted to an int + message at the ABI.
struct Status {
  int code = SV_OK;
  std::string msg;
  static Status ok() { return {}; }
  static Status err(int c, std::string m) {
    Status s;
    s.code = c;
    s.msg = std::move(m);
    return s;
  }
  bool good() const { return code == SV_OK; }
};

// Validate input gate records (kinds SV_U1..SV_SWAP, qubits in range and distinct).
Status validate_gates(const sv_gate* g, size_t count, int n);

// ---- blocking pass (blocking.cpp): Listing 3 of the paper, DESIGN readings R2-R6 ----------
// tokens: SV_CHUNK_SWAP(q0<q1), SV_BEGIN, SV_END, and gates on physical qubits with pad = index.
Status block_pass(const sv_gate* g, size_t count, int n, int c, std::vector<int>& pi, uint32_t flags,
                  std::vector<sv_gate>& tokens);

// ---- executor plan (plan.cpp) ---------------------------------------------------------------
struct ExPair {
  int m;  // local memory bit
  int b;  // rank memory bit (>= nL)
};
struct Step {
  enum Type { EXCHANGE = 0, SECTION = 1, GATE = 2, COMPACT = 3 } type;
  std::vector<ExPair> ex;        // EXCHANGE
  std::vector<sv_gate> gates;    // SECTION / GATE: memory-frame gates (no SWAP inside SECTION)
  // SECTION: memory-bit transpositions fused into the section's store (both bits in its tile);
  // COMPACT: memory-bit transpositions done by a standalone swap pass (local bits).
  std::vector<std::pair<int, int>> swaps;
};
struct PlanCounters {
  uint64_t sections = 0, chunk_swaps = 0, exchanges = 0, exchange_batches = 0, compactions = 0, store_swaps = 0;
};
// Layout policy knobs of the planner (plan.cpp).
struct PlanLayout {
  int low_bits = 3;    // memory bits every section tile should contain (3: 128-byte fp64 runs)
  int max_tile = 13;   // largest tile (bits) one CTA holds
  int tile_default = 11;  // small sections pad to 11 bits (32 KiB fp64 tiles, 4 CTAs per SM): more
                          // independent CTAs overlap HBM phases and barriers better than 12-bit tiles
                          // (QFT30 c=8 35.6 vs 40.2 ms; QV33 c=9 1724 vs 1842 ms); 10 bits gains
                          // ~1-2% on QV but loses 15% on QFT (round-1 measurements)
  int pref_tile = 13;  // largest tile worth its coalescing bits (fp64: a T=13 tile is 128 KiB of
                      // smem, one CTA per SM, slower than a T=12 tile with 64-byte runs)
  bool free_initial = false;  // the state is a basis state: choose the initial sigma freely (NEXT-2)
};

// Preferred largest tile for swizzle width G (3: fp64, 4: fp32).
inline int pref_tile_for(int G) { return G == 3 ? 12 : 13; }
// Tile policy of a layout whose low_bits is set: preferred maximum and default size.
inline void apply_tile_prefs(PlanLayout& L) {
  L.pref_tile = pref_tile_for(L.low_bits);
  if (L.tile_default > L.pref_tile) L.tile_default = L.pref_tile;
}

// The tile a section runs on (memory-bit mask), shared by the planner and the compiler: the
// active bits, plus the lowest `low_bits` memory bits when that still fits max_tile, padded with
// the lowest remaining local bits up to tile_default.
inline uint64_t choose_tile(uint64_t active, int nL, const PlanLayout& L) {
  const int nlow = L.low_bits < nL ? L.low_bits : nL;
  uint64_t want = active | ((1ull << nlow) - 1);
  if (__builtin_popcountll(want) > L.max_tile) {
    want = active;
  } else if (__builtin_popcountll(want) > L.pref_tile && __builtin_popcountll(active) <= L.pref_tile) {
    want = active;  // fewer coalescing bits (shorter runs) instead of the next tile size
    for (int b = 0; b < nlow && __builtin_popcountll(want) < L.pref_tile; b++) want |= 1ull << b;
  }
  const int td = L.tile_default < nL ? L.tile_default : nL;
  for (int b = 0; b < nL && __builtin_popcountll(want) < td; b++) want |= 1ull << b;
  return want;
}
// Runs the pass (unless SV_UNBLOCKED) and maps it onto memory bits: every chunk_swap / SWAP is a
// relabel of sigma; data moves only where a section needs a rank bit (DESIGN "Executor mapping").
Status make_plan(const sv_gate* g, size_t count, int n, int c, int world_log2, std::vector<int>& pi,
                 std::vector<int>& sigma, uint32_t flags, std::vector<Step>& steps, PlanCounters& ctr,
                 const PlanLayout& layout = PlanLayout(), std::vector<int>* sigma_initial = nullptr);

}  // namespace sv
