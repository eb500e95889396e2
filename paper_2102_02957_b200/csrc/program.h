// program.h — the per-section "program" the host compiles and the section kernel (K1) runs.
//
// A section (begin_blocking..end_blocking) is compiled into:
//   * a TILE: T memory bits (the bits its non-diagonal gates touch, padded with the lowest free
//     local bits so every tile is a union of >= 128-byte runs); one CTA owns one tile per launch
//     and the grid enumerates the other local bits (out_bits);
//   * PHASES: runs of gates whose non-diagonal qubits fit R_BITS "register" positions.  In a
//     phase each thread holds 2^R_BITS amplitudes that differ only in those positions and applies
//     the phase's gates in registers; shared memory is touched once per phase boundary, and the
//     first / last phase read / write HBM directly when their lane bits are the tile's low bits;
//   * OPS: U2 / U1 / H1 / PERM on register slots, DIAG on any bit (register slot, thread bit,
//     out-of-tile local bit, or a rank bit folded to a constant on the host).
// The program and the section's coefficients are copied into __constant__ memory before each
// launch, so every warp reads them through uniform registers (LDCU) — matrices never occupy
// vector registers or the LSU.
#pragma once

#define SV_R_BITS 4           // register positions per phase (16 amplitudes per thread)
#define SV_TMAX 14            // max tile bits (fp64 T=13 -> 128 KiB smem)
#define SV_MAX_OUT 48         // max out-of-tile local bits
#define SV_MAX_SETS 6         // DIAGSETs per section with prologue-computed per-CTA factors (6 x 5 lanes)

// __constant__ budget per section launch
#define SV_CONST_INTS 4096    // 16 KiB of program
#define SV_CONST_COEF64 2048  // 32 KiB of fp64 complex coefficients
#define SV_CONST_COEF32 1024  // 8 KiB of fp32 complex coefficients

// op types
#define SV_OP_U2 1      // a = slot0 < b = slot1, coef -> 16 complex (row-major, s = bit(a) + 2 bit(b))
#define SV_OP_U1 2      // a = slot, coef -> 4 complex (row-major)
#define SV_OP_H1 3      // a = slot, coef -> 1 complex (scale s, real):  (x, y) -> (s(x+y), s(x-y))
#define SV_OP_H1U 8     // a = slot: unscaled butterfly (x, y) -> (x+y, x-y); the section's product of
                        // Hadamard scales is applied once, by its last H1 op (a global scalar)
#define SV_OP_PERM2 4   // a = slot0, b = slot1, extra = packed permutation out[s] = in[(extra >> 2s) & 3]
#define SV_OP_DIAG 5    // a = code0, b = code1, coef -> 4 complex d[s], s = bit(code0) + 2 bit(code1)
#define SV_OP_DIAG_CP 6 // like DIAG with d0 = d1 = d2 = 1: only s == 3 is multiplied (coef -> d3)
#define SV_OP_DIAGSET 7 // fused run of diagonal gates: a = descriptor offset (ints from the header),
                        // coef -> LAMBDA[16] (if flag bit 0); descriptor:
                        //   [0] flags (bit 0: LAMBDA present)   [1] aux offset of 5 thread tables
                        //   [2+i] / [7] per-CTA terms of subset i (i = 0: empty set, 1+s: slot s),
                        //               3 ints each: out-bit mask lo, hi, coef (apply if set)
                        //   [8] / [9]   per-thread mixed terms, 5 ints: i, thread mask, out lo, hi, coef
                        // register k is multiplied by LAMBDA[k] * F_0 * prod_{s in k} F_{1+s},
                        // F_i = (per-CTA terms) * table_i[tid] * (matching mixed terms)

// DIAG bit codes (per phase)
#define SV_CODE_SLOT(s) (s)           // register slot s (0..3): bit = (k >> s) & 1
#define SV_CODE_THREAD(j) (32 + (j))  // thread-index bit j: bit = (tid >> j) & 1
#define SV_CODE_OUT(mb) (100 + (mb))  // local memory bit mb outside the tile (per-CTA constant)
#define SV_CODE_ZERO 200              // constant 0 (rank bit folded on the host, or unused)
#define SV_CODE_ONE 201               // constant 1

#define SV_FLAG_FIRST_DIRECT 1        // first phase loads straight from HBM
#define SV_FLAG_LAST_DIRECT 2         // last phase stores straight to HBM

// A thread/register <-> tile mapping used at a tile boundary: smem offsets (swizzled) and the
// HBM memory bit of every thread bit j and register slot s.
struct SvMap {
  int tw[16];
  int rw[SV_R_BITS];
  int tmb[16];
  int rmb[SV_R_BITS];
};

struct SvSecHeader {
  int T;          // tile bits
  int r;          // register bits per phase (== SV_R_BITS)
  int n_out;      // local memory bits outside the tile (grid = 2^n_out CTAs)
  int n_phases;
  int phase_off;  // int offset of the first SvPhase from the header
  int op_off;     // int offset of the first SvOp from the header
  int n_ops;
  int flags;      // SV_FLAG_*
  int tile_bits[16];        // tile position -> memory bit on LOAD (ascending)
  int store_bits[16];       // tile position -> memory bit on STORE (a permutation of tile_bits)
  int out_bits[SV_MAX_OUT]; // out-of-tile local memory bits (ascending) <- CTA index bits
  SvMap load;               // non-direct initial load: lanes walk the lowest load memory bits
  SvMap store;              // non-direct final store: lanes walk the lowest store memory bits
  SvMap din;                // direct first phase: phase-0 mapping, load memory bits
  SvMap dout;               // direct last phase: last-phase mapping, store memory bits
  int n_sets;               // DIAGSETs whose per-CTA factors the CTA prologue computes (<= SV_MAX_SETS)
  int set_desc[SV_MAX_SETS];  // their descriptor offsets; factors go to smem after the tile
  int pad_sets[1];
};

// XOR-fold swizzle of a tile element index (host and device): the low G bits are XORed with
// every higher G-bit group.  GF(2)-linear, so swz(a | b) = swz(a) ^ swz(b) for disjoint a, b.
inline int sv_swz_host(int i, int G) {
  int x = i >> G, f = 0;
  for (int j = 0; j < 6; j++) {
    f ^= x;
    x >>= G;
  }
  return i ^ (f & ((1 << G) - 1));
}

struct SvPhase {
  int R[SV_R_BITS];    // register slot -> tile position
  int rw[SV_R_BITS];   // swz(1 << R[s]): smem offset contribution of register slot s
  int op_begin, op_count, pad0, pad1;
  int tpos[16];        // thread-index bit j -> tile position (T - r entries used)
  int tw[16];          // swz(1 << tpos[j])
};

struct SvOp {
  int type, a, b, coef;  // coef: index into the section's coefficients
  int extra, pad0, pad1, pad2;
};

static_assert(sizeof(SvSecHeader) % 16 == 0, "header alignment");
static_assert(sizeof(SvPhase) % 16 == 0, "phase alignment");
static_assert(sizeof(SvOp) % 16 == 0, "op alignment");
