// section.cu — K1, the section kernel: one HBM read + one HBM write of the shard per blocked
// section (Listing 4 "for all chunks: apply gates of the blocking section").
//
// One CTA owns one 2^T-amplitude tile (a gather over the section's memory bits, program.h).
// Each thread holds 16 amplitudes in registers that differ in the phase's 4 register positions
// and applies every gate of the phase there; phases are separated by one shared-memory round
// trip (XOR-fold swizzled, conflict-free for the lane groups the host chose); the first and last
// phase talk to HBM directly when their lane bits are the tile's low memory bits.  The program
// and the matrices live in __constant__ memory and reach the FMA pipe through uniform registers.
#include <cstdlib>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <mutex>

#include "kernels.cuh"
#include "section_dev.cuh"

namespace sv {

namespace {

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
      diagset(v, a, cb, tid, (int)blockDim.x, tile_off, aux, ctaf);
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

template <typename V, int G, int NT, int MINB, bool FIRST, bool LAST>
__global__ void __launch_bounds__(NT, MINB) k_section(V* __restrict__ sv, const V* __restrict__ aux, int split_a,
                                                     int split_b) {
  using R = decltype(V().x);
  constexpr int RB = SV_R_BITS;  // the host guarantees T >= RB, so every phase has RB register slots
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* sm = reinterpret_cast<V*>(smem_raw);
  const int T = c_prog[kH_T], n_out = c_prog[kH_NOUT], nph = c_prog[kH_NPH];
  const int phoff = c_prog[kH_PHOFF], opoff = c_prog[kH_OPOFF];
  const int nt_log = T - RB;
  const int tid = threadIdx.x;
  const uint64_t n_tiles = 1ull << (n_out - (split_a ? 1 : 0) - (split_b ? 1 : 0));
  V* ctaf = reinterpret_cast<V*>(smem_raw + (sizeof(V) << T));
  const int n_sets = c_prog[kH_NSETS];

  (void)G;  // the swizzle width is baked into the host's maps
  // one tile per CTA (a grid-stride loop only if the launch ever exceeds the grid limit)
  for (uint64_t blk = blockIdx.x; blk < n_tiles; blk += gridDim.x) {
    uint64_t tile_off = 0;
    const uint64_t tb = expand_tile(blk, split_a, split_b);
    for (int j = 0; j < n_out; j++) tile_off |= ((tb >> j) & 1ull) << c_prog[kH_OUT + j];

    // per-CTA DIAGSET factors (out-of-tile terms), computed once per tile into smem
    if (n_sets > 0) {
      for (int f = tid; f < 5 * n_sets; f += (int)blockDim.x) {  // tiny tiles have fewer threads than factors
        const int d = c_prog[kH_SETS + f / 5], i = f % 5;
        ctaf[f] = cta_factor<V>(c_prog[d + 2 + i], c_prog[d + 3 + i], tile_off);
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
    __syncthreads();  // the next tile reuses the shared-memory tile and factors
  }
}

constexpr int kMaxDev = 64;

template <typename V, int G, int NT, int MINB, bool FIRST, bool LAST>
cudaError_t launch_v(V* sv, const V* aux, int T, int n_out, size_t smem, cudaStream_t st, int split_a, int split_b) {
  static bool attr_set[kMaxDev] = {};  // cudaFuncSetAttribute applies to the current device only
  auto kern = k_section<V, G, NT, MINB, FIRST, LAST>;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= kMaxDev) return cudaErrorInvalidDevice;
  if (!attr_set[dev]) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)((sizeof(V) << 13) + 5 * SV_MAX_SETS * sizeof(V)));
    if (e != cudaSuccess) return e;
    attr_set[dev] = true;
  }
  const int threads = 1 << (T - SV_R_BITS);
  const uint64_t tiles = 1ull << (n_out - (split_a ? 1 : 0) - (split_b ? 1 : 0));
  const unsigned grid = (unsigned)(tiles < 0x7fffffffull ? tiles : 0x7fffffffull);
  kern<<<grid, threads, smem, st>>>(sv, aux, split_a, split_b);
  return cudaGetLastError();
}

// Direct-HBM boundary phases are compile-time variants.  (first direct, last via smem) is run as
// the all-smem variant: ptxas keeps the coefficient loads on the uniform datapath in the other
// three shapes only (checked by tests/test_sass.py).
template <typename V, int G, int NT, int MINB>
cudaError_t launch_t(V* sv, const V* aux, int T, int n_out, int flags, size_t smem, cudaStream_t st, int sa, int sb) {
  const bool f = flags & SV_FLAG_FIRST_DIRECT, l = flags & SV_FLAG_LAST_DIRECT;
  if (f && l) return launch_v<V, G, NT, MINB, true, true>(sv, aux, T, n_out, smem, st, sa, sb);
  if (l) return launch_v<V, G, NT, MINB, false, true>(sv, aux, T, n_out, smem, st, sa, sb);
  return launch_v<V, G, NT, MINB, false, false>(sv, aux, T, n_out, smem, st, sa, sb);
}

}  // namespace

namespace {
cudaError_t launch_section_locked(bool dbl, void* sv, const int* prog_dev, size_t int_count, const void* coef_dev,
                                  size_t coef_count, const void* aux_dev, int T, int n_out, int n_phases, int flags,
                                  int n_sets, cudaStream_t st, int split_a, int split_b);
}  // namespace

cudaError_t launch_section(bool dbl, void* sv, const int* prog_dev, size_t int_count, const void* coef_dev,
                           size_t coef_count, const void* aux_dev, int T, int n_out, int n_phases, int flags,
                           int n_sets, cudaStream_t st, int split_a, int split_b) {
  if (int_count > SV_CONST_INTS) return cudaErrorInvalidValue;
  // The interpreter's program and coefficients live in this module's __constant__ bank, one per
  // device and shared by every handle.  Handles on different streams (several ranks of a local
  // world, a host-tier handle beside a device handle) are serialised: each copy + launch waits for
  // the previous user's launch (an event chain per device, under a process-wide lock).
  static std::mutex mu;
  static cudaEvent_t last[kMaxDev] = {};
  std::lock_guard<std::mutex> lk(mu);
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= kMaxDev) return cudaErrorInvalidDevice;
  if (!last[dev] && (e = cudaEventCreateWithFlags(&last[dev], cudaEventDisableTiming)) != cudaSuccess) return e;
  if ((e = cudaStreamWaitEvent(st, last[dev], 0)) != cudaSuccess) return e;
  e = launch_section_locked(dbl, sv, prog_dev, int_count, coef_dev, coef_count, aux_dev, T, n_out, n_phases, flags,
                            n_sets, st, split_a, split_b);
  if (e != cudaSuccess) return e;
  return cudaEventRecord(last[dev], st);
}

namespace {
cudaError_t launch_section_locked(bool dbl, void* sv, const int* prog_dev, size_t int_count, const void* coef_dev,
                                  size_t coef_count, const void* aux_dev, int T, int n_out, int n_phases, int flags,
                                  int n_sets, cudaStream_t st, int split_a, int split_b) {
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
    if (T <= 12) return launch_t<double2, 3, 256, 2>((double2*)sv, (const double2*)aux_dev, T, n_out, flags, smem, st, split_a, split_b);
    if (T == 13) return launch_t<double2, 3, 512, 1>((double2*)sv, (const double2*)aux_dev, T, n_out, flags, smem, st, split_a, split_b);
    return cudaErrorInvalidValue;
  }
  const size_t smem = n_sets ? (sizeof(float2) << T) + 5 * SV_MAX_SETS * sizeof(float2)
                             : (no_smem ? 0 : sizeof(float2) << T);
  if (T <= 12) return launch_t<float2, 4, 256, 2>((float2*)sv, (const float2*)aux_dev, T, n_out, flags, smem, st, split_a, split_b);
  if (T == 13) return launch_t<float2, 4, 512, 1>((float2*)sv, (const float2*)aux_dev, T, n_out, flags, smem, st, split_a, split_b);
  return cudaErrorInvalidValue;
}

}  // namespace

}  // namespace sv
