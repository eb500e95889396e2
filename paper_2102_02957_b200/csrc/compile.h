// compile.h — section compiler interface (host).
#pragma once
#include <utility>
#include <vector>

#include "common.h"
#include "program.h"

namespace sv {

constexpr int kTooBig = -100;  // internal: section exceeds the __constant__ budget (split it)

struct Launch {
  size_t int_off;     // start of the section's SvSecHeader in Program::ints
  size_t int_count;   // ints of header + phases + ops
  size_t coef_off;    // first coefficient (complex index) of the section in Program::coefs
  size_t coef_count;  // coefficients of the section
  size_t aux_off;     // first complex of the section's DIAGSET factor tables in Program::aux
  size_t aux_count;
  int T, r, n_out, n_phases, n_ops, flags, n_sets;
  double flops_per_amp;  // algorithmic flops per amplitude of the section (DESIGN "Roofline")
};

struct Program {
  std::vector<int> ints;       // headers, phases, ops of every section, concatenated
  std::vector<double> coefs;   // complex coefficients (re, im) in fp64 (-> __constant__)
  std::vector<double> aux;     // DIAGSET per-thread factor tables (re, im) in fp64 (-> global)
  std::vector<Launch> launches;
  void clear() {
    ints.clear();
    coefs.clear();
    aux.clear();
    launches.clear();
  }
};

// Compile one memory-frame section for this rank.  T_default: tile bits when the section needs
// fewer; swizzle_bits: log2(amplitudes per 128-byte smem row) (3 for fp64, 4 for fp32).
// compile_section_split splits sections whose program or coefficients exceed the __constant__
// budget into consecutive in-order pieces (each its own launch).
// store_swaps: memory-bit transpositions (both bits in the tile) fused into the final store.
Status compile_section(const std::vector<sv_gate>& gates, int nL, int rank, int world_log2, int T_default,
                       int swizzle_bits, const std::vector<std::pair<int, int>>& store_swaps, Program& prog);
Status compile_section_split(const std::vector<sv_gate>& gates, int nL, int rank, int world_log2, int T_default,
                             int swizzle_bits, const std::vector<std::pair<int, int>>& store_swaps, Program& prog);

}  // namespace sv
