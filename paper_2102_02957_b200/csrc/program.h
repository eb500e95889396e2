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
#define SV_OP_U2 1      // a = slot0 < b = slot1, coef -> 16 complex (row-major, s = bit(a) + 2 bit(b)),
                        // then 16 more: (-(re + im), im - re) of each entry (3-multiply form)
#define SV_OP_U1 2      // a = slot, coef -> 4 complex (row-major)
#define SV_OP_H1 3      // a = slot, coef -> 1 complex (scale s, real):  (x, y) -> (s(x+y), s(x-y))
#define SV_OP_H1U 8     // a = slot: unscaled butterfly (x, y) -> (x+y, x-y); the section's product of
                        // Hadamard scales is applied once, by its last H1 op (a global scalar)
#define SV_OP_PERM2 4   // a = slot0, b = slot1, extra = packed permutation out[s] = in[(extra >> 2s) & 3]
#define SV_OP_DIAG 5    // a = code0, b = code1, coef -> 4 complex d[s], s = bit(code0) + 2 bit(code1)
#define SV_OP_DIAG_CP 6 // like DIAG with d0 = d1 = d2 = 1: only s == 3 is multiplied (coef -> d3)
#define SV_OP_DIAGSET 7 // fused run of diagonal gates: a = descriptor offset (ints from the header),
                        // coef -> LAMBDA[16] (if flag bit 0); descriptor:
                        //   [0] flags (bit 0: LAMBDA present; bits 8..15 prologue factor set or
                        //       255; bits 16..20: subset i's thread table is not all ones)
                        //   [1] aux offset of 5 thread tables
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
  int nl;                   // local memory bits (memory bits >= nl in the maps are rank bits)
};

#ifndef __CUDACC_RTC__
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
#endif

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

// Field offsets in ints, for device code (NVRTC has no offsetof): checked against the structs.
constexpr int kH_T = 0, kH_R = 1, kH_NOUT = 2, kH_NPH = 3, kH_PHOFF = 4, kH_OPOFF = 5, kH_NOPS = 6, kH_FLAGS = 7;
constexpr int kH_TILE = 8, kH_STOREB = 24, kH_OUT = 40, kH_LOAD = 88, kH_STORE = 128, kH_DIN = 168, kH_DOUT = 208;
constexpr int kH_NSETS = 248, kH_SETS = 249;
constexpr int kM_TW = 0, kM_RW = 16, kM_TMB = 20, kM_RMB = 36;
constexpr int kP_RW = 4, kP_OPB = 8, kP_OPC = 9, kP_TW = 28;
constexpr int kPhaseInts = sizeof(SvPhase) / 4, kOpInts = sizeof(SvOp) / 4;
#ifndef __CUDACC_RTC__
#include <cstddef>
#define SV_OFF(S, f) (int)(offsetof(S, f) / 4)
static_assert(SV_OFF(SvSecHeader, T) == kH_T && SV_OFF(SvSecHeader, r) == kH_R && SV_OFF(SvSecHeader, n_out) == kH_NOUT &&
                  SV_OFF(SvSecHeader, n_phases) == kH_NPH && SV_OFF(SvSecHeader, phase_off) == kH_PHOFF &&
                  SV_OFF(SvSecHeader, op_off) == kH_OPOFF && SV_OFF(SvSecHeader, n_ops) == kH_NOPS &&
                  SV_OFF(SvSecHeader, flags) == kH_FLAGS,
              "header scalars");
static_assert(SV_OFF(SvSecHeader, tile_bits) == kH_TILE && SV_OFF(SvSecHeader, store_bits) == kH_STOREB &&
                  SV_OFF(SvSecHeader, out_bits) == kH_OUT && SV_OFF(SvSecHeader, load) == kH_LOAD &&
                  SV_OFF(SvSecHeader, store) == kH_STORE && SV_OFF(SvSecHeader, din) == kH_DIN &&
                  SV_OFF(SvSecHeader, dout) == kH_DOUT && SV_OFF(SvSecHeader, n_sets) == kH_NSETS &&
                  SV_OFF(SvSecHeader, set_desc) == kH_SETS,
              "header arrays");
static_assert(SV_OFF(SvMap, tw) == kM_TW && SV_OFF(SvMap, rw) == kM_RW && SV_OFF(SvMap, tmb) == kM_TMB &&
                  SV_OFF(SvMap, rmb) == kM_RMB,
              "map");
static_assert(SV_OFF(SvPhase, rw) == kP_RW && SV_OFF(SvPhase, op_begin) == kP_OPB &&
                  SV_OFF(SvPhase, op_count) == kP_OPC && SV_OFF(SvPhase, tw) == kP_TW,
              "phase");
#undef SV_OFF
#endif
