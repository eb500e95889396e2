// section.cu — K1, the section kernel: one HBM read + one HBM write of the shard per blocked
// section (Listing 4 "for all chunks: apply gates of the blocking section").
//
// One CTA owns one 2^T-amplitude tile (a gather over the section's memory bits, program.h).
// Each thread holds 16 amplitudes in registers that differ in the phase's 4 register positions
// and applies every gate of the phase there; phases are separated by one shared-memory round
// trip (XOR-fold swizzled, conflict-free for the lane groups the host chose); the first and last
// phase talk to HBM directly when their lane bits are the tile's low memory bits.  The program
// and the matrices live in __constant__ memory and reach the FMA pipe through uniform registers.
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "cplx.cuh"
#include "kernels.cuh"
#include "program.h"

namespace sv {

__constant__ int c_prog[SV_CONST_INTS];
__constant__ double2 c_coef64[SV_CONST_COEF64];
__constant__ float2 c_coef32[SV_CONST_COEF32];

namespace {

template <typename V>
__device__ __forceinline__ V cc(int i);
template <>
__device__ __forceinline__ double2 cc<double2>(int i) {
  return c_coef64[i];
}
template <>
__device__ __forceinline__ float2 cc<float2>(int i) {
  return c_coef32[i];
}

// XOR-fold swizzle of a tile element index: the low G bits are XORed with every higher G-bit
// group.  GF(2)-linear, so swz(a | b) = swz(a) ^ swz(b) for disjoint a, b.
template <int G>
__device__ __forceinline__ int swz(int i) {
  int x = i >> G, f = 0;
#pragma unroll
  for (int j = 0; j < 5; j++) {
    f ^= x;
    x >>= G;
  }
  return i ^ (f & ((1 << G) - 1));
}

// ---------------------------------------------------------------- gates on register slots
template <int S0, int S1, typename V>
__device__ __forceinline__ void u2_slots(V (&v)[16], int cb) {
#pragma unroll
  for (int q = 0; q < 16; q++) {
    if (((q >> S0) & 1) || ((q >> S1) & 1)) continue;
    const int i0 = q, i1 = q | (1 << S0), i2 = q | (1 << S1), i3 = q | (1 << S0) | (1 << S1);
    const V a0 = v[i0], a1 = v[i1], a2 = v[i2], a3 = v[i3];
#pragma unroll
    for (int rr = 0; rr < 4; rr++) {
      V acc = cmul(cc<V>(cb + 4 * rr + 0), a0);
      acc = cfma(cc<V>(cb + 4 * rr + 1), a1, acc);
      acc = cfma(cc<V>(cb + 4 * rr + 2), a2, acc);
      acc = cfma(cc<V>(cb + 4 * rr + 3), a3, acc);
      v[rr == 0 ? i0 : (rr == 1 ? i1 : (rr == 2 ? i2 : i3))] = acc;
    }
  }
}

template <int S, typename V>
__device__ __forceinline__ void u1_slot(V (&v)[16], int cb) {
#pragma unroll
  for (int q = 0; q < 16; q++) {
    if ((q >> S) & 1) continue;
    const V a0 = v[q], a1 = v[q | (1 << S)];
    v[q] = cfma(cc<V>(cb + 1), a1, cmul(cc<V>(cb), a0));
    v[q | (1 << S)] = cfma(cc<V>(cb + 3), a1, cmul(cc<V>(cb + 2), a0));
  }
}

template <int S, typename V, typename R>
__device__ __forceinline__ void h1_slot(V (&v)[16], R s) {
#pragma unroll
  for (int q = 0; q < 16; q++) {
    if ((q >> S) & 1) continue;
    h_ip(v[q], v[q | (1 << S)], s);
  }
}

template <int S, typename V>
__device__ __forceinline__ void hu_slot(V (&v)[16]) {
#pragma unroll
  for (int q = 0; q < 16; q++) {
    if ((q >> S) & 1) continue;
    hu_ip(v[q], v[q | (1 << S)]);
  }
}

template <int S0, int S1, typename V>
__device__ __forceinline__ void perm_slots(V (&v)[16], int perm) {
  const int p0 = perm & 3, p1 = (perm >> 2) & 3, p2 = (perm >> 4) & 3, p3 = (perm >> 6) & 3;
#pragma unroll
  for (int q = 0; q < 16; q++) {
    if (((q >> S0) & 1) || ((q >> S1) & 1)) continue;
    const int i0 = q, i1 = q | (1 << S0), i2 = q | (1 << S1), i3 = q | (1 << S0) | (1 << S1);
    const V a0 = v[i0], a1 = v[i1], a2 = v[i2], a3 = v[i3];
    v[i0] = sel4(p0, a0, a1, a2, a3);
    v[i1] = sel4(p1, a0, a1, a2, a3);
    v[i2] = sel4(p2, a0, a1, a2, a3);
    v[i3] = sel4(p3, a0, a1, a2, a3);
  }
}

// diagonal factors on register slots
template <int S, typename V>
__device__ __forceinline__ void d1_slot(V (&v)[16], V d0, V d1) {
#pragma unroll
  for (int k = 0; k < 16; k++) cmul_ip(v[k], ((k >> S) & 1) ? d1 : d0);
}
template <int S0, int S1, typename V>
__device__ __forceinline__ void d2_slots(V (&v)[16], V d0, V d1, V d2, V d3) {
#pragma unroll
  for (int k = 0; k < 16; k++) cmul_ip(v[k], sel4(((k >> S0) & 1) | (((k >> S1) & 1) << 1), d0, d1, d2, d3));
}
template <int S0, int S1, typename V>
__device__ __forceinline__ void cp_slots(V (&v)[16], V d3) {
#pragma unroll
  for (int k = 0; k < 16; k++)
    if (((k >> S0) & 1) && ((k >> S1) & 1)) cmul_ip(v[k], d3);
}
template <int S, typename V>
__device__ __forceinline__ void cp_slot(V (&v)[16], V d3) {
#pragma unroll
  for (int k = 0; k < 16; k++)
    if ((k >> S) & 1) cmul_ip(v[k], d3);
}
template <typename V>
__device__ __forceinline__ void scale_all(V (&v)[16], V f) {
#pragma unroll
  for (int k = 0; k < 16; k++) cmul_ip(v[k], f);
}

// dispatch on a canonical slot pair a < b (6 cases) / a single slot (4 cases)
#define SV_PAIR_SWITCH(a, b, CALL)        \
  switch ((a) * 4 + (b)) {                \
    case 1: CALL(0, 1); break;            \
    case 2: CALL(0, 2); break;            \
    case 3: CALL(0, 3); break;            \
    case 6: CALL(1, 2); break;            \
    case 7: CALL(1, 3); break;            \
    case 11: CALL(2, 3); break;           \
    default: break;                       \
  }
#define SV_SLOT_SWITCH(a, CALL) \
  switch (a) {                  \
    case 0: CALL(0); break;     \
    case 1: CALL(1); break;     \
    case 2: CALL(2); break;     \
    case 3: CALL(3); break;     \
    default: break;             \
  }

// multiply every register k that contains slot subset S by f
template <int S, typename V>
__device__ __forceinline__ void scale_subset(V (&v)[16], V f) {
#pragma unroll
  for (int k = 0; k < 16; k++)
    if ((k & S) == S) v[k] = cmul(v[k], f);
}

template <typename V>
__device__ __forceinline__ V shfl_c(V x, int src) {
  x.x = __shfl_sync(0xffffffffu, x.x, src);
  x.y = __shfl_sync(0xffffffffu, x.y, src);
  return x;
}

__device__ __forceinline__ uint64_t mask64(int lo, int hi) { return (uint64_t)(uint32_t)lo | ((uint64_t)(uint32_t)hi << 32); }

// Fused diagonal run (SV_OP_DIAGSET, program.h).  The five subset factors F_i (empty set and the
// four register slots) are: per-CTA out-bit terms (lanes 0..4 of each warp, broadcast by shuffle)
// x the host-built per-thread table x rare mixed terms; the 16 register factors are products of
// them built as A[k & 3] * B[k >> 2] with no branches, so v stays in place.
template <typename V>
__device__ __forceinline__ V cta_factor(int b, int e, uint64_t tile_off) {
  V f = cone<V>();
  for (int t = b; t < e; t += 3) {
    const uint64_t O = mask64(c_prog[t], c_prog[t + 1]);
    const V c = cc<V>(c_prog[t + 2]);
    if ((tile_off & O) == O) f = cmul(f, c);
  }
  return f;
}

template <typename V>
__device__ __forceinline__ void diagset(V (&v)[16], int desc, int cb, int tid, uint64_t tile_off,
                                        const V* __restrict__ aux, const V* ctaf) {
  const int flags = c_prog[desc];
  const V* tab = aux + c_prog[desc + 1];
  const int nthr = blockDim.x;
  const int lane = tid & 31;
  const int set = (flags >> 8) & 255;
  V F[5];
  if (set != 255) {  // per-CTA factors computed once by the CTA prologue
#pragma unroll
    for (int i = 0; i < 5; i++) F[i] = cmul(ctaf[5 * set + i], tab[i * nthr + tid]);
  } else if (blockDim.x >= 32) {
    V mine = cone<V>();
    if (lane < 5) mine = cta_factor<V>(c_prog[desc + 2 + lane], c_prog[desc + 3 + lane], tile_off);
#pragma unroll
    for (int i = 0; i < 5; i++) F[i] = cmul(shfl_c(mine, i), tab[i * nthr + tid]);
  } else {  // tiny tiles (T < 9): fewer than 32 threads, every thread walks the terms itself
#pragma unroll
    for (int i = 0; i < 5; i++)
      F[i] = cmul(cta_factor<V>(c_prog[desc + 2 + i], c_prog[desc + 3 + i], tile_off), tab[i * nthr + tid]);
  }
  const int me = c_prog[desc + 9];
  for (int t = c_prog[desc + 8]; t < me; t += 5) {
    const int si = c_prog[t], J = c_prog[t + 1];
    const uint64_t O = mask64(c_prog[t + 2], c_prog[t + 3]);
    const V c = cc<V>(c_prog[t + 4]);
    if ((tid & J) == J && (tile_off & O) == O) {
#pragma unroll
      for (int i = 0; i < 5; i++)
        if (si == i) F[i] = cmul(F[i], c);
    }
  }
  // A[lo] = F_0 * prod_{s in lo} F_{1+s} (slots 0, 1); B[hi] = prod_{s in hi} F_{3+s} (slots 2, 3)
  const V A0 = F[0], A1 = cmul(F[0], F[1]), A2 = cmul(F[0], F[2]), A3 = cmul(A1, F[2]);
  const V B1 = F[3], B2 = F[4], B3 = cmul(F[3], F[4]);
  if (flags & 1) {
#pragma unroll
    for (int k = 0; k < 16; k++) {
      const V a = (k & 3) == 0 ? A0 : (k & 3) == 1 ? A1 : (k & 3) == 2 ? A2 : A3;
      const V f = (k >> 2) == 0 ? a : cmul(a, (k >> 2) == 1 ? B1 : (k >> 2) == 2 ? B2 : B3);
      cmul_ip(v[k], cmul(f, cc<V>(cb + k)));
    }
  } else {
#pragma unroll
    for (int k = 0; k < 16; k++) {
      const V a = (k & 3) == 0 ? A0 : (k & 3) == 1 ? A1 : (k & 3) == 2 ? A2 : A3;
      const V f = (k >> 2) == 0 ? a : cmul(a, (k >> 2) == 1 ? B1 : (k >> 2) == 2 ? B2 : B3);
      cmul_ip(v[k], f);
    }
  }
}

// value of a non-slot DIAG bit code for this thread / tile
__device__ __forceinline__ int code_val(int code, int tid, uint64_t tile_off) {
  if (code < 100) return (tid >> (code - 32)) & 1;
  if (code < 200) return (int)((tile_off >> (code - 100)) & 1ull);
  return code - 200;
}

template <typename V, typename R>
__device__ __forceinline__ void run_op(V (&v)[16], int oi, int tid, uint64_t tile_off, const V* __restrict__ aux,
                                       const V* ctaf) {
  const int type = c_prog[oi], a = c_prog[oi + 1], b = c_prog[oi + 2], cb = c_prog[oi + 3];
  switch (type) {
    case SV_OP_U2: {
#define CALL_U2(x, y) u2_slots<x, y>(v, cb)
      SV_PAIR_SWITCH(a, b, CALL_U2)
#undef CALL_U2
      break;
    }
    case SV_OP_U1: {
#define CALL_U1(x) u1_slot<x>(v, cb)
      SV_SLOT_SWITCH(a, CALL_U1)
#undef CALL_U1
      break;
    }
    case SV_OP_H1: {
      const R s = cc<V>(cb).x;
#define CALL_H1(x) h1_slot<x>(v, s)
      SV_SLOT_SWITCH(a, CALL_H1)
#undef CALL_H1
      break;
    }
    case SV_OP_PERM2: {
      const int perm = c_prog[oi + 4];
#define CALL_P(x, y) perm_slots<x, y>(v, perm)
      SV_PAIR_SWITCH(a, b, CALL_P)
#undef CALL_P
      break;
    }
    case SV_OP_DIAG: {
      const V d0 = cc<V>(cb), d1 = cc<V>(cb + 1), d2 = cc<V>(cb + 2), d3 = cc<V>(cb + 3);
      if (a < 4 && b < 4) {
#define CALL_D2(x, y) d2_slots<x, y>(v, d0, d1, d2, d3)
        SV_PAIR_SWITCH(a, b, CALL_D2)
#undef CALL_D2
      } else if (a < 4) {
        const int tb = code_val(b, tid, tile_off);
        const V e0 = tb ? d2 : d0, e1 = tb ? d3 : d1;
#define CALL_D1(x) d1_slot<x>(v, e0, e1)
        SV_SLOT_SWITCH(a, CALL_D1)
#undef CALL_D1
      } else {
        const int s = code_val(a, tid, tile_off) | (code_val(b, tid, tile_off) << 1);
        scale_all(v, sel4(s, d0, d1, d2, d3));
      }
      break;
    }
    case SV_OP_DIAG_CP: {
      const V d3 = cc<V>(cb);
      if (a < 4 && b < 4) {
#define CALL_CP2(x, y) cp_slots<x, y>(v, d3)
        SV_PAIR_SWITCH(a, b, CALL_CP2)
#undef CALL_CP2
      } else if (a < 4) {
        if (code_val(b, tid, tile_off)) {
#define CALL_CP1(x) cp_slot<x>(v, d3)
          SV_SLOT_SWITCH(a, CALL_CP1)
#undef CALL_CP1
        }
      } else if (code_val(a, tid, tile_off) & code_val(b, tid, tile_off)) {
        scale_all(v, d3);
      }
      break;
    }
    case SV_OP_DIAGSET:
      diagset(v, a, cb, tid, tile_off, aux, ctaf);
      break;
    case SV_OP_H1U: {
#define CALL_HU(x) hu_slot<x>(v)
      SV_SLOT_SWITCH(a, CALL_HU)
#undef CALL_HU
      break;
    }
    default:
      break;
  }
}

// header / phase / map field offsets (ints)
constexpr int kH_T = offsetof(SvSecHeader, T) / 4, kH_NOUT = offsetof(SvSecHeader, n_out) / 4;
constexpr int kH_NPH = offsetof(SvSecHeader, n_phases) / 4, kH_PHOFF = offsetof(SvSecHeader, phase_off) / 4;
constexpr int kH_OPOFF = offsetof(SvSecHeader, op_off) / 4, kH_OUT = offsetof(SvSecHeader, out_bits) / 4;
constexpr int kH_LOAD = offsetof(SvSecHeader, load) / 4, kH_STORE = offsetof(SvSecHeader, store) / 4;
constexpr int kH_DIN = offsetof(SvSecHeader, din) / 4, kH_DOUT = offsetof(SvSecHeader, dout) / 4;
constexpr int kM_TW = offsetof(SvMap, tw) / 4, kM_RW = offsetof(SvMap, rw) / 4;
constexpr int kM_TMB = offsetof(SvMap, tmb) / 4, kM_RMB = offsetof(SvMap, rmb) / 4;
constexpr int kP_RW = offsetof(SvPhase, rw) / 4, kP_OPB = offsetof(SvPhase, op_begin) / 4;
constexpr int kP_OPC = offsetof(SvPhase, op_count) / 4, kP_TW = offsetof(SvPhase, tw) / 4;
constexpr int kPhaseInts = sizeof(SvPhase) / 4, kOpInts = sizeof(SvOp) / 4;
constexpr int kH_NSETS = offsetof(SvSecHeader, n_sets) / 4, kH_SETS = offsetof(SvSecHeader, set_desc) / 4;

// x ^ (the XOR of w[s] over the set bits s of the compile-time register index k)
template <int K>
__device__ __forceinline__ int xk(int x, const int (&w)[SV_R_BITS]) {
#pragma unroll
  for (int s = 0; s < SV_R_BITS; s++)
    if ((K >> s) & 1) x ^= w[s];
  return x;
}

// Swizzled shared-memory offsets of this thread's register-0 amplitude (x) and of each register
// slot (w) under the mapping whose thread-bit offsets start at c_prog[tw] and slot offsets at
// c_prog[rw].
__device__ __forceinline__ void smem_map(int tw, int rw, int nt_log, int tid, int& x, int (&w)[SV_R_BITS]) {
  x = 0;
  for (int j = 0; j < nt_log; j++) x ^= ((tid >> j) & 1) ? c_prog[tw + j] : 0;
#pragma unroll
  for (int s = 0; s < SV_R_BITS; s++) w[s] = c_prog[rw + s];
}

// HBM element offset of this thread's register-0 amplitude under map M (tile base included)
__device__ __forceinline__ uint64_t hbm_base(int M, int nt_log, int tid, uint64_t tile_off) {
  uint64_t mb = tile_off;
  for (int j = 0; j < nt_log; j++) mb |= (uint64_t)((tid >> j) & 1) << c_prog[M + kM_TMB + j];
  return mb;
}

template <typename V>
__device__ __forceinline__ void hbm_load(V (&v)[16], const V* __restrict__ src, int M) {
  int64_t ro[SV_R_BITS];
#pragma unroll
  for (int s = 0; s < SV_R_BITS; s++) ro[s] = (int64_t)1 << c_prog[M + kM_RMB + s];
#pragma unroll
  for (int k = 0; k < 16; k++) {
    int64_t o = 0;
#pragma unroll
    for (int s = 0; s < SV_R_BITS; s++)
      if ((k >> s) & 1) o |= ro[s];
    v[k] = src[o];
  }
}

template <typename V>
__device__ __forceinline__ void hbm_store(const V (&v)[16], V* __restrict__ dst, int M) {
  int64_t ro[SV_R_BITS];
#pragma unroll
  for (int s = 0; s < SV_R_BITS; s++) ro[s] = (int64_t)1 << c_prog[M + kM_RMB + s];
#pragma unroll
  for (int k = 0; k < 16; k++) {
    int64_t o = 0;
#pragma unroll
    for (int s = 0; s < SV_R_BITS; s++)
      if ((k >> s) & 1) o |= ro[s];
    dst[o] = v[k];
  }
}

template <typename V, int G, int NT, int MINB, bool FIRST, bool LAST>
__global__ void __launch_bounds__(NT, MINB) k_section(V* __restrict__ sv, const V* __restrict__ aux) {
  using R = decltype(V().x);
  constexpr int RB = SV_R_BITS;  // the host guarantees T >= RB, so every phase has RB register slots
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* sm = reinterpret_cast<V*>(smem_raw);
  const int T = c_prog[kH_T], n_out = c_prog[kH_NOUT], nph = c_prog[kH_NPH];
  const int phoff = c_prog[kH_PHOFF], opoff = c_prog[kH_OPOFF];
  const int nt_log = T - RB;
  const int tid = threadIdx.x;

  uint64_t tile_off = 0;
  {
    const uint64_t bid = blockIdx.x;
    for (int j = 0; j < n_out; j++) tile_off |= ((bid >> j) & 1ull) << c_prog[kH_OUT + j];
  }

  // per-CTA DIAGSET factors (out-of-tile terms), computed once per CTA by warp 0 into smem
  V* ctaf = reinterpret_cast<V*>(smem_raw + (sizeof(V) << T));
  const int n_sets = c_prog[kH_NSETS];
  if (n_sets > 0) {
    if (tid < 5 * n_sets) {
      const int d = c_prog[kH_SETS + tid / 5], i = tid % 5;
      ctaf[tid] = cta_factor<V>(c_prog[d + 2 + i], c_prog[d + 3 + i], tile_off);
    }
    __syncthreads();
  }

  V v[16];
  if constexpr (FIRST) {  // phase 0 reads HBM directly in its own register mapping
    hbm_load(v, sv + hbm_base(kH_DIN, nt_log, tid, tile_off), kH_DIN);
  } else {  // lanes walk the lowest load memory bits; scatter into the swizzled tile
    hbm_load(v, sv + hbm_base(kH_LOAD, nt_log, tid, tile_off), kH_LOAD);
    int x, w[RB];
    smem_map(kH_LOAD + kM_TW, kH_LOAD + kM_RW, nt_log, tid, x, w);
#define SV_STS(K) sm[xk<K>(x, w)] = v[K];
    SV_STS(0) SV_STS(1) SV_STS(2) SV_STS(3) SV_STS(4) SV_STS(5) SV_STS(6) SV_STS(7)
    SV_STS(8) SV_STS(9) SV_STS(10) SV_STS(11) SV_STS(12) SV_STS(13) SV_STS(14) SV_STS(15)
#undef SV_STS
    __syncthreads();
  }

  for (int ph = 0; ph < nph; ph++) {
    const int P = phoff + ph * kPhaseInts;
    const bool direct_in = FIRST && ph == 0;
    const bool direct_out = LAST && ph == nph - 1;
    int pb, w[RB];
    smem_map(P + kP_TW, P + kP_RW, nt_log, tid, pb, w);
    if (!direct_in) {
#define SV_LDS(K) v[K] = sm[xk<K>(pb, w)];
      SV_LDS(0) SV_LDS(1) SV_LDS(2) SV_LDS(3) SV_LDS(4) SV_LDS(5) SV_LDS(6) SV_LDS(7)
      SV_LDS(8) SV_LDS(9) SV_LDS(10) SV_LDS(11) SV_LDS(12) SV_LDS(13) SV_LDS(14) SV_LDS(15)
#undef SV_LDS
    }
    const int ob = c_prog[P + kP_OPB], oc = c_prog[P + kP_OPC];
    for (int o = 0; o < oc; o++) run_op<V, R>(v, opoff + (ob + o) * kOpInts, tid, tile_off, aux, ctaf);
    if (direct_out) {  // the last phase writes HBM directly (store memory bits, same mapping)
      hbm_store(v, sv + hbm_base(kH_DOUT, nt_log, tid, tile_off), kH_DOUT);
    } else {
#define SV_STS(K) sm[xk<K>(pb, w)] = v[K];
      SV_STS(0) SV_STS(1) SV_STS(2) SV_STS(3) SV_STS(4) SV_STS(5) SV_STS(6) SV_STS(7)
      SV_STS(8) SV_STS(9) SV_STS(10) SV_STS(11) SV_STS(12) SV_STS(13) SV_STS(14) SV_STS(15)
#undef SV_STS
      __syncthreads();
    }
  }

  if constexpr (!LAST) {  // gather in store order (lanes walk the lowest store memory bits)
    int x, w[RB];
    smem_map(kH_STORE + kM_TW, kH_STORE + kM_RW, nt_log, tid, x, w);
#define SV_LDS(K) v[K] = sm[xk<K>(x, w)];
    SV_LDS(0) SV_LDS(1) SV_LDS(2) SV_LDS(3) SV_LDS(4) SV_LDS(5) SV_LDS(6) SV_LDS(7)
    SV_LDS(8) SV_LDS(9) SV_LDS(10) SV_LDS(11) SV_LDS(12) SV_LDS(13) SV_LDS(14) SV_LDS(15)
#undef SV_LDS
    hbm_store(v, sv + hbm_base(kH_STORE, nt_log, tid, tile_off), kH_STORE);
  }
}

template <typename V, int G, int NT, int MINB, bool FIRST, bool LAST>
cudaError_t launch_v(V* sv, const V* aux, int T, int n_out, size_t smem, cudaStream_t st) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(k_section<V, G, NT, MINB, FIRST, LAST>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)((sizeof(V) << 13) + 5 * SV_MAX_SETS * sizeof(V)));
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int threads = 1 << (T - SV_R_BITS);
  k_section<V, G, NT, MINB, FIRST, LAST><<<(unsigned)(1ull << n_out), threads, smem, st>>>(sv, aux);
  return cudaGetLastError();
}

// Direct-HBM boundary phases are compile-time variants.  (first direct, last via smem) is run as
// the all-smem variant: ptxas keeps the coefficient loads on the uniform datapath in the other
// three shapes only (checked by tests/test_sass.py).
template <typename V, int G, int NT, int MINB>
cudaError_t launch_t(V* sv, const V* aux, int T, int n_out, int flags, size_t smem, cudaStream_t st) {
  const bool f = flags & SV_FLAG_FIRST_DIRECT, l = flags & SV_FLAG_LAST_DIRECT;
  if (f && l) return launch_v<V, G, NT, MINB, true, true>(sv, aux, T, n_out, smem, st);
  if (l) return launch_v<V, G, NT, MINB, false, true>(sv, aux, T, n_out, smem, st);
  return launch_v<V, G, NT, MINB, false, false>(sv, aux, T, n_out, smem, st);
}

}  // namespace

cudaError_t launch_section(bool dbl, void* sv, const int* prog_dev, size_t int_count, const void* coef_dev,
                           size_t coef_count, const void* aux_dev, int T, int n_out, int n_phases, int flags,
                           int n_sets, cudaStream_t st) {
  if (int_count > SV_CONST_INTS) return cudaErrorInvalidValue;
  cudaError_t e = cudaMemcpyToSymbolAsync(c_prog, prog_dev, int_count * sizeof(int), 0, cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return e;
  if (coef_count) {
    if (dbl) {
      if (coef_count > SV_CONST_COEF64) return cudaErrorInvalidValue;
      e = cudaMemcpyToSymbolAsync(c_coef64, coef_dev, coef_count * sizeof(double2), 0, cudaMemcpyDeviceToDevice, st);
    } else {
      if (coef_count > SV_CONST_COEF32) return cudaErrorInvalidValue;
      e = cudaMemcpyToSymbolAsync(c_coef32, coef_dev, coef_count * sizeof(float2), 0, cudaMemcpyDeviceToDevice, st);
    }
    if (e != cudaSuccess) return e;
  }
  if (T < SV_R_BITS) return cudaErrorInvalidValue;  // tiny shards run per-gate kernels instead
  const bool no_smem = n_phases == 1 && (flags & SV_FLAG_FIRST_DIRECT) && (flags & SV_FLAG_LAST_DIRECT);
  if (dbl) {
    const size_t smem = n_sets ? (sizeof(double2) << T) + 5 * SV_MAX_SETS * sizeof(double2)
                               : (no_smem ? 0 : sizeof(double2) << T);
    if (T <= 12) return launch_t<double2, 3, 256, 2>((double2*)sv, (const double2*)aux_dev, T, n_out, flags, smem, st);
    if (T == 13) return launch_t<double2, 3, 512, 1>((double2*)sv, (const double2*)aux_dev, T, n_out, flags, smem, st);
    return cudaErrorInvalidValue;
  }
  const size_t smem = n_sets ? (sizeof(float2) << T) + 5 * SV_MAX_SETS * sizeof(float2)
                             : (no_smem ? 0 : sizeof(float2) << T);
  if (T <= 12) return launch_t<float2, 4, 256, 2>((float2*)sv, (const float2*)aux_dev, T, n_out, flags, smem, st);
  if (T == 13) return launch_t<float2, 4, 512, 1>((float2*)sv, (const float2*)aux_dev, T, n_out, flags, smem, st);
  return cudaErrorInvalidValue;
}

}  // namespace sv
