// compile.h — section compiler interface (host).
#pragma once
#include <vector>

#include "common.h"
#include "program.h"

namespace sv {

struct Launch {
  size_t int_off;  // start of the section's SvSecHeader in Program::ints
  int T, r, n_out, n_phases, n_ops;
  double flops_per_amp;  // algorithmic flops per amplitude of the section (DESIGN "Roofline")
};

struct Program {
  std::vector<int> ints;       // headers, phases, ops of every section, concatenated
  std::vector<double> coefs;   // complex coefficients (re, im) in fp64
  std::vector<Launch> launches;
  void clear() {
    ints.clear();
    coefs.clear();
    launches.clear();
  }
};

// Compile one memory-frame section for this rank.  T_default: tile bits when the section needs
// fewer; swizzle_bits: log2(amplitudes per 128-byte smem row) (3 for fp64, 4 for fp32).
Status compile_section(const std::vector<sv_gate>& gates, int nL, int rank, int world_log2, int T_default,
                       int swizzle_bits, Program& prog);

}  // namespace sv
