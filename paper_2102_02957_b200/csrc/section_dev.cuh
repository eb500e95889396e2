// section_dev.cuh — device building blocks of the section kernel (K1), shared by the program
// interpreter (section.cu) and the per-section kernels generated at run time (jit.cpp, NVRTC).
// Everything here is plain CUDA C++ that NVRTC can compile on its own: no host headers.
#pragma once
#ifdef __CUDACC_RTC__
typedef unsigned long long uint64_t;
typedef long long int64_t;
typedef unsigned int uint32_t;

#else
#include <cstddef>
#include <cstdint>
#endif

#include "cplx.cuh"
#include "program.h"

namespace sv {

// The section program.  A generated kernel (jit.cpp) bakes its own program into its module's
// constant bank (SV_JIT_PROG: the program's ints, which are also the kernel's cache key), so no
// copy precedes its launches and handles on different streams never share mutable constants; the
// interpreter (section.cu) copies each section's program in before its launch.
#ifdef SV_JIT_PROG
__constant__ int c_prog[SV_CONST_INTS] = {SV_JIT_PROG};
#else
__constant__ int c_prog[SV_CONST_INTS];
__constant__ double2 c_coef64[SV_CONST_COEF64];
__constant__ float2 c_coef32[SV_CONST_COEF32];
#endif

namespace {

// Coefficient accessors: the interpreter reads the section's coefficients from the __constant__
// bank (CoefBank); the generated kernels get them as a __grid_constant__ kernel parameter
// (CoefParam), so every FMA takes its matrix element straight from the parameter bank, or — for
// the rare section whose coefficients exceed the 32 KiB parameter space — through a pointer to
// the handle's device copy (CoefPtr, read-only cached loads).
#ifndef SV_JIT_PROG
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
template <typename V>
struct CoefBank {
  __device__ __forceinline__ V operator()(int i) const { return cc<V>(i); }
};
#else
template <typename V>
struct CoefBank;  // generated kernels have no coefficient bank
#endif
template <typename V, int N>
struct CoefParam {
  V c[N];
  __device__ __forceinline__ V operator()(int i) const { return c[i]; }
};
template <typename V>
struct CoefPtr {
  const V* p;
  __device__ __forceinline__ V operator()(int i) const { return __ldg(p + i); }
};

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
// 4x4 complex matrix on the register pairs of slots S0 < S1, three real products per complex
// multiply-add: with s = x + y of each input, out.re = T + R and out.im = T + I where
// T = sum m.re s, R = sum -(m.re + m.im) y, I = sum (m.im - m.re) x (the host stores the two
// derived coefficients after the matrix).  Chained form (default): the R and I chains start from
// T, so the sums need no separate adds — 52 instead of 64 FP64 operations per 4 amplitudes (4 adds
// for s, per output row one multiply and 11 FMAs).  SPLIT form (60 operations: R and I on their own,
// then T added): shorter dependency chains, used where the inputs come straight from HBM.
template <int S0, int S1, bool SPLIT = false, typename V, typename CF = CoefBank<V>>
__device__ __forceinline__ void u2_slots(V (&v)[16], int cb, const CF& cf = CF()) {
  using R = decltype(V().x);
#pragma unroll
  for (int q = 0; q < 16; q++) {
    if (((q >> S0) & 1) || ((q >> S1) & 1)) continue;
    const int i0 = q, i1 = q | (1 << S0), i2 = q | (1 << S1), i3 = q | (1 << S0) | (1 << S1);
    const V a[4] = {v[i0], v[i1], v[i2], v[i3]};
    R s[4];
#pragma unroll
    for (int c = 0; c < 4; c++) s[c] = a[c].x + a[c].y;
#pragma unroll
    for (int rr = 0; rr < 4; rr++) {
      R t = cf(cb + 4 * rr).x * s[0];
#pragma unroll
      for (int c = 1; c < 4; c++) t = fma(cf(cb + 4 * rr + c).x, s[c], t);
      R re, im;
      if constexpr (SPLIT) {
        re = cf(cb + 16 + 4 * rr).x * a[0].y;
        im = cf(cb + 16 + 4 * rr).y * a[0].x;
#pragma unroll
        for (int c = 1; c < 4; c++) {
          re = fma(cf(cb + 16 + 4 * rr + c).x, a[c].y, re);
          im = fma(cf(cb + 16 + 4 * rr + c).y, a[c].x, im);
        }
        re += t;
        im += t;
      } else {
        re = t;
        im = t;
#pragma unroll
        for (int c = 0; c < 4; c++) {
          re = fma(cf(cb + 16 + 4 * rr + c).x, a[c].y, re);
          im = fma(cf(cb + 16 + 4 * rr + c).y, a[c].x, im);
        }
      }
      V o;
      o.x = re;
      o.y = im;
      v[rr == 0 ? i0 : (rr == 1 ? i1 : (rr == 2 ? i2 : i3))] = o;
    }
  }
}

template <int S, typename V, typename CF = CoefBank<V>>
__device__ __forceinline__ void u1_slot(V (&v)[16], int cb, const CF& cf = CF()) {
#pragma unroll
  for (int q = 0; q < 16; q++) {
    if ((q >> S) & 1) continue;
    const V a0 = v[q], a1 = v[q | (1 << S)];
    v[q] = cfma(cf(cb + 1), a1, cmul(cf(cb), a0));
    v[q | (1 << S)] = cfma(cf(cb + 3), a1, cmul(cf(cb + 2), a0));
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
template <typename V, typename CF = CoefBank<V>>
__device__ __forceinline__ V cta_factor(int b, int e, uint64_t tile_off, const CF& cf = CF()) {
  V f = cone<V>();
  for (int t = b; t < e; t += 3) {
    const uint64_t O = mask64(c_prog[t], c_prog[t + 1]);
    const V c = cf(c_prog[t + 2]);
    if ((tile_off & O) == O) f = cmul(f, c);
  }
  return f;
}

template <typename V, typename CF = CoefBank<V>>
__device__ __forceinline__ void diagset(V (&v)[16], int desc, int cb, int tid, int nthr, uint64_t tile_off,
                                        const V* __restrict__ aux, const V* ctaf, const CF& cf = CF()) {
  const int flags = c_prog[desc];
  const V* tab = aux + c_prog[desc + 1];
  const int lane = tid & 31;
  const int set = (flags >> 8) & 255;
  V F[5];
  if (set != 255) {  // per-CTA factors computed once by the CTA prologue
#pragma unroll
    for (int i = 0; i < 5; i++) F[i] = cmul(ctaf[5 * set + i], tab[i * nthr + tid]);
  } else if (nthr >= 32) {
    V mine = cone<V>();
    if (lane < 5) mine = cta_factor<V>(c_prog[desc + 2 + lane], c_prog[desc + 3 + lane], tile_off, cf);
#pragma unroll
    for (int i = 0; i < 5; i++) F[i] = cmul(shfl_c(mine, i), tab[i * nthr + tid]);
  } else {  // tiny tiles (T < 9): fewer than 32 threads, every thread walks the terms itself
#pragma unroll
    for (int i = 0; i < 5; i++)
      F[i] = cmul(cta_factor<V>(c_prog[desc + 2 + i], c_prog[desc + 3 + i], tile_off, cf), tab[i * nthr + tid]);
  }
  const int me = c_prog[desc + 9];
  for (int t = c_prog[desc + 8]; t < me; t += 5) {
    const int si = c_prog[t], J = c_prog[t + 1];
    const uint64_t O = mask64(c_prog[t + 2], c_prog[t + 3]);
    const V c = cf(c_prog[t + 4]);
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
      cmul_ip(v[k], cmul(f, cf(cb + k)));
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

// header / phase / map field offsets (ints)
// field offsets (ints): program.h (kH_*, kM_*, kP_*, checked against offsetof on the host)

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

// ---------------------------------------------------------------- TMA tile loads (sm_90+ / sm_100a)
// The tensor-map variant of the generated kernel (jit.cpp gen_source_tma) streams each CTA's
// next tiles into a ring of shared-memory slots with cp.async.bulk.tensor (UTMALDG), completion
// counted on an mbarrier per slot, while the CTA computes the current tile.  SvTmap is the
// opaque 128-byte CUtensorMap, passed as a __grid_constant__ kernel parameter.
struct alignas(64) SvTmap {
  unsigned long long w[16];
};
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tSV_WAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra SV_WAIT_%=;\n\t}" ::"r"(
          smem_u32(b)),
      "r"(parity)
      : "memory");
}
// generic-proxy writes of a slot (the previous tile's phases) before the async proxy refills it
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
template <int D>
__device__ __forceinline__ void tma_load(void* dst, const SvTmap* tm, int c0, int c1, int c2, int c3, int c4, uint64_t* bar) {
  const int c[5] = {c0, c1, c2, c3, c4};
  const unsigned long long t = reinterpret_cast<unsigned long long>(tm);
  if constexpr (D == 1)
    asm volatile("cp.async.bulk.tensor.1d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];" ::"r"(
                     smem_u32(dst)), "l"(t), "r"(c[0]), "r"(smem_u32(bar))
                 : "memory");
  else if constexpr (D == 2)
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                     smem_u32(dst)), "l"(t), "r"(c[0]), "r"(c[1]), "r"(smem_u32(bar))
                 : "memory");
  else if constexpr (D == 3)
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            smem_u32(dst)), "l"(t), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(smem_u32(bar))
        : "memory");
  else if constexpr (D == 4)
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(
            smem_u32(dst)), "l"(t), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(smem_u32(bar))
        : "memory");
  else
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(
            smem_u32(dst)), "l"(t), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(smem_u32(bar))
        : "memory");
}

// Tile index of launch block b when the launch covers only the tiles whose out-bit indices
// (split & 255) have the value ((split >> 8) & 1); split = 0: all tiles.  Lower index first.
__device__ __forceinline__ uint64_t expand_tile(uint64_t b, int split_a, int split_b) {
  if (split_a) {
    const int p = split_a & 255;
    const uint64_t lo = b & ((1ull << p) - 1);
    b = ((b - lo) << 1) | ((uint64_t)((split_a >> 8) & 1) << p) | lo;
  }
  if (split_b) {
    const int p = split_b & 255;
    const uint64_t lo = b & ((1ull << p) - 1);
    b = ((b - lo) << 1) | ((uint64_t)((split_b >> 8) & 1) << p) | lo;
  }
  return b;
}

// DIAGSET with its structure as template arguments (generated kernels): subsets without a
// thread table (TABM) or per-CTA terms (CTAM) are identically one and cost nothing; the register
// factors are products of the non-trivial subset factors (the compiler shares common prefixes).
// Requires the per-CTA factors in smem (SET != 255) and no mixed terms.
template <int LAM, int SET, int TABM, int CTAM, typename V, typename CF>
__device__ __forceinline__ void diagset_c(V (&v)[16], int desc, int cb, int tid, int nthr, const V* __restrict__ aux,
                                          const V* ctaf, const CF& cf) {
  const V* tab = aux + c_prog[desc + 1];
  V F[5];
#pragma unroll
  for (int i = 0; i < 5; i++) {
    if ((TABM >> i) & 1) {
      F[i] = __ldg(tab + i * nthr + tid);  // small per-thread tables: keep them in L1
      if ((CTAM >> i) & 1) F[i] = cmul(F[i], ctaf[5 * SET + i]);
    } else if ((CTAM >> i) & 1) {
      F[i] = ctaf[5 * SET + i];
    } else {
      F[i] = cone<V>();
    }
  }
  constexpr int NT = TABM | CTAM;
#pragma unroll
  for (int k = 0; k < 16; k++) {
    V f = cone<V>();
    bool one = true;
    if (NT & 1) {
      f = F[0];
      one = false;
    }
#pragma unroll
    for (int s = 0; s < 4; s++)
      if (((k >> s) & 1) && ((NT >> (1 + s)) & 1)) {
        f = one ? F[1 + s] : cmul(f, F[1 + s]);
        one = false;
      }
    if (LAM) {
      f = one ? cf(cb + k) : cmul(f, cf(cb + k));
      one = false;
    }
    if (!one) cmul_ip(v[k], f);
  }
}

// Compile-time op (generated kernels): the same gate code as the interpreter's run_op, with the
// op fields as template arguments, so slots and coefficient offsets are immediates.
template <int TYPE, int A, int B, int CB, int X, typename V, typename CF>
__device__ __forceinline__ void op_c(V (&v)[16], int tid, int nthr, uint64_t tile_off, const V* __restrict__ aux,
                                     const V* ctaf, const CF& cf) {
  if constexpr (TYPE == SV_OP_U2) {
    u2_slots<A, B, X == 1>(v, CB, cf);
  } else if constexpr (TYPE == SV_OP_U1) {
    u1_slot<A>(v, CB, cf);
  } else if constexpr (TYPE == SV_OP_H1) {
    h1_slot<A>(v, cf(CB).x);
  } else if constexpr (TYPE == SV_OP_H1U) {
    hu_slot<A>(v);
  } else if constexpr (TYPE == SV_OP_PERM2) {
    perm_slots<A, B>(v, X);
  } else if constexpr (TYPE == SV_OP_DIAG) {
    if constexpr (A < 4 && B < 4) {
      d2_slots<A, B>(v, cf(CB), cf(CB + 1), cf(CB + 2), cf(CB + 3));
    } else if constexpr (A < 4) {
      const int tb = code_val(B, tid, tile_off);
      d1_slot<A>(v, tb ? cf(CB + 2) : cf(CB), tb ? cf(CB + 3) : cf(CB + 1));
    } else {
      const int s = code_val(A, tid, tile_off) | (code_val(B, tid, tile_off) << 1);
      scale_all(v, sel4(s, cf(CB), cf(CB + 1), cf(CB + 2), cf(CB + 3)));
    }
  } else if constexpr (TYPE == SV_OP_DIAG_CP) {
    if constexpr (A < 4 && B < 4) {
      cp_slots<A, B>(v, cf(CB));
    } else if constexpr (A < 4) {
      if (code_val(B, tid, tile_off)) cp_slot<A>(v, cf(CB));
    } else {
      if (code_val(A, tid, tile_off) & code_val(B, tid, tile_off)) scale_all(v, cf(CB));
    }
  } else if constexpr (TYPE == SV_OP_DIAGSET) {
    diagset(v, A, CB, tid, nthr, tile_off, aux, ctaf, cf);
  }
}

}  // namespace
}  // namespace sv
