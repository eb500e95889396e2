// kernels.cu — sm_100a kernels of the cache-blocked state-vector path.
//
//   (K1, the section kernel, is in section.cu)
//   K2 k_gate_*       per-gate baseline: one pass per gate with the pair addressing of Listing 2
//                     (P:242-254), 64-bit indices (the listing's 32-bit int would overflow).
//   K5 reductions     norm, marginal probabilities, block masses and shot resolution.
//   K6 k_set_basis    |k>.
//   K7 k_gather       amplitude gather.
//   exchange          peer-memory swap of local bit(s) with rank bit(s) over NVLink.
#include <cstdlib>
#include <cuda_runtime.h>

#include <cstdint>
#include <algorithm>
#include <cstring>
#include <utility>

#include "cplx.cuh"
#include "kernels.cuh"
#include "program.h"

namespace sv {
namespace {

constexpr int kRedBlocks = 148 * 8;  // fixed grid for deterministic reductions
constexpr int kRedThreads = 256;

// ------------------------------------------------------------------ K2: per-gate baseline
template <typename V>
struct Mat16 {
  V m[16];
};

__device__ __forceinline__ uint64_t insert_zero(uint64_t x, int p) {
  const uint64_t lo = x & ((1ull << p) - 1);
  return ((x - lo) << 1) | lo;
}

template <typename V>
__global__ void k_gate_u1(V* __restrict__ sv, uint64_t npairs, int q, V m0, V m1, V m2, V m3) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < npairs; i += stride) {
    const uint64_t i0 = insert_zero(i, q), i1 = i0 | (1ull << q);  // Listing 2
    const V a0 = sv[i0], a1 = sv[i1];
    sv[i0] = cfma(m1, a1, cmul(m0, a0));
    sv[i1] = cfma(m3, a1, cmul(m2, a0));
  }
}

template <typename V>
__global__ void k_gate_u2(V* __restrict__ sv, uint64_t nquads, int q0, int q1, Mat16<V> M) {
  const int lo = q0 < q1 ? q0 : q1, hi = q0 < q1 ? q1 : q0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nquads; i += stride) {
    const uint64_t b = insert_zero(insert_zero(i, lo), hi);
    const uint64_t i0 = b, i1 = b | (1ull << q0), i2 = b | (1ull << q1), i3 = i1 | (1ull << q1);
    const V a0 = sv[i0], a1 = sv[i1], a2 = sv[i2], a3 = sv[i3];
    V o[4];
#pragma unroll
    for (int rr = 0; rr < 4; rr++)
      o[rr] = cfma(M.m[4 * rr + 3], a3, cfma(M.m[4 * rr + 2], a2, cfma(M.m[4 * rr + 1], a1, cmul(M.m[4 * rr], a0))));
    sv[i0] = o[0];
    sv[i1] = o[1];
    sv[i2] = o[2];
    sv[i3] = o[3];
  }
}

template <typename V>
__global__ void k_gate_diag(V* __restrict__ sv, uint64_t N, int c0, int c1, V d0, V d1, V d2, V d3) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < N; x += stride) {
    const int b0 = c0 < 100 ? (int)((x >> c0) & 1) : c0 - 200;
    const int b1 = c1 < 100 ? (int)((x >> c1) & 1) : c1 - 200;
    const V f = sel4(b0 | (b1 << 1), d0, d1, d2, d3);
    if (f.x != 1 || f.y != 0) sv[x] = cmul(sv[x], f);  // untouched amplitudes are not read (CP: 1/4)
  }
}

template <typename V>
__global__ void k_gate_swap(V* __restrict__ sv, uint64_t nquads, int q0, int q1) {
  const int lo = q0 < q1 ? q0 : q1, hi = q0 < q1 ? q1 : q0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nquads; i += stride) {
    const uint64_t b = insert_zero(insert_zero(i, lo), hi);
    const uint64_t x = b | (1ull << q0), y = b | (1ull << q1);
    const V t = sv[x];
    sv[x] = sv[y];
    sv[y] = t;
  }
}

// ------------------------------------------------------------------ K6 / K7
template <typename V>
__global__ void k_set_one(V* sv, int64_t off) {
  sv[off] = cone<V>();
}

template <typename V>
__global__ void k_set_amp(V* sv, int64_t off, double re) {
  V x = czero<V>();
  x.x = re;
  sv[off] = x;
}

template <typename V>
__global__ void k_gather(const V* __restrict__ sv, const uint64_t* __restrict__ offs, size_t cnt, V* __restrict__ out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < cnt; i += (size_t)gridDim.x * blockDim.x) {
    const uint64_t o = offs[i];
    out[i] = o == ~0ull ? czero<V>() : sv[o];
  }
}

// ------------------------------------------------------------------ K5: reductions
__device__ __forceinline__ double block_sum(double x, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = x;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); i++) s += red[i];
  __syncthreads();
  return s;  // valid in thread 0
}

template <typename V>
__global__ void k_norm_partial(const V* __restrict__ sv, uint64_t N, double* __restrict__ partial) {
  __shared__ double red[32];
  double acc = 0.0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < N; i += stride) acc += abs2(sv[i]);
  const double s = block_sum(acc, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

__global__ void k_sum_partials(const double* __restrict__ partial, int count, double* __restrict__ out) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < count; i += blockDim.x) acc += partial[i];
  const double s = block_sum(acc, red);
  if (threadIdx.x == 0) *out = s;
}

struct QBits {
  int b[24];
};

// Marginal probabilities, task form: a warp task fixes every memory bit except the 5 lane bits
// (consecutive amplitudes: coalesced) and up to 6 "iteration" bits that are not marginal bits,
// so each lane's bin is fixed for the whole task and it accumulates in a register; lanes then
// reduce over their non-marginal lane bits by shuffles and one lane per bin adds to the
// histogram (shared memory per CTA, or global for > 12 bits).  One atomic per bin per task.
struct MargPlan {
  int nq, nit, ntb;
  uint32_t lane_q;  // lane bits (0..4) that are marginal bits
  int qb[24];       // bin bit i <- memory bit qb[i]
  int it_b[8];      // iteration bits (not marginal, >= 5)
  int task_b[64];   // all other bits >= 5
};

template <typename V>
__global__ void k_marginal_tasks(const V* __restrict__ sv, MargPlan p, double* __restrict__ dst, int use_smem) {
  extern __shared__ double hist[];
  __shared__ uint64_t offs[64];  // memory offset of each iteration index (deposit into it_b)
  const int bins = 1 << p.nq;
  const int niter = 1 << p.nit;
  for (int it = threadIdx.x; it < niter; it += blockDim.x) {
    uint64_t x = 0;
    for (int j = 0; j < p.nit; j++) x |= (uint64_t)((it >> j) & 1) << p.it_b[j];
    offs[it] = x;
  }
  if (use_smem)
    for (int i = threadIdx.x; i < bins; i += blockDim.x) hist[i] = 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  int y_lane = 0;
  for (int i = 0; i < p.nq; i++)
    if (p.qb[i] < 5) y_lane |= ((lane >> p.qb[i]) & 1) << i;
  const uint32_t nonq = ~p.lane_q & 31u;
  const uint64_t ntasks = 1ull << p.ntb;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t t = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < ntasks; t += nwarps) {
    uint64_t x0 = (uint64_t)lane;
    for (int j = 0; j < p.ntb; j++) x0 |= ((t >> j) & 1ull) << p.task_b[j];
    int y = y_lane;
    for (int i = 0; i < p.nq; i++)
      if (p.qb[i] >= 5) y |= (int)((x0 >> p.qb[i]) & 1ull) << i;
    double acc0 = 0.0, acc1 = 0.0;
    const V* base = sv + x0;
#pragma unroll 8
    for (int it = 0; it < niter; it += 2) {  // niter is a power of two >= 2 here
      acc0 += abs2(base[offs[it]]);
      acc1 += abs2(base[offs[it + 1]]);
    }
    double acc = acc0 + acc1;
#pragma unroll
    for (int j = 0; j < 5; j++)
      if ((nonq >> j) & 1) acc += __shfl_xor_sync(0xffffffffu, acc, 1 << j);
    if ((lane & nonq) == 0) atomicAdd(&(use_smem ? hist : dst)[y], acc);
  }
  if (use_smem) {
    __syncthreads();
    for (int i = threadIdx.x; i < bins; i += blockDim.x) dst[(size_t)blockIdx.x * bins + i] = hist[i];
  }
}

template <typename V>
__global__ void k_marginal_small(const V* __restrict__ sv, uint64_t N, QBits q, int nq, double* __restrict__ out) {
  for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < N; x += (uint64_t)gridDim.x * blockDim.x) {
    int y = 0;
    for (int i = 0; i < nq; i++) y |= (int)((x >> q.b[i]) & 1) << i;
    atomicAdd(&out[y], abs2(sv[x]));
  }
}

__global__ void k_reduce_bins(const double* __restrict__ partial, int blocks, int bins, double* __restrict__ out) {
  for (int y = blockIdx.x * blockDim.x + threadIdx.x; y < bins; y += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int bk = 0; bk < blocks; bk++) s += partial[(size_t)bk * bins + y];
    out[y] = s;
  }
}

template <typename V>
__global__ void k_block_sums(const V* __restrict__ sv, int B, double* __restrict__ out) {
  __shared__ double red[32];
  const uint64_t base = (uint64_t)blockIdx.x << B;
  const int len = 1 << B;
  double acc = 0.0;
  for (int i = threadIdx.x; i < len; i += blockDim.x) acc += abs2(sv[base + i]);
  const double s = block_sum(acc, red);
  if (threadIdx.x == 0) out[blockIdx.x] = s;
}

// items: (block, first shot, count) triples.  The block's |a|^2 is scanned in a fixed order
// (per-thread sequential runs, then a sequential scan of the run totals).
template <typename V>
__global__ void k_sample_resolve(const V* __restrict__ sv, int B, const int64_t* __restrict__ items,
                                 const double* __restrict__ resid, uint64_t* __restrict__ out_off) {
  extern __shared__ double cum[];
  __shared__ double run_tot[1024];
  const int64_t blk = items[3 * blockIdx.x], first = items[3 * blockIdx.x + 1], cnt = items[3 * blockIdx.x + 2];
  const int len = 1 << B;
  const int per = (len + blockDim.x - 1) / blockDim.x;
  const uint64_t base = (uint64_t)blk << B;
  const int lo = threadIdx.x * per;
  double s = 0.0;
  for (int i = lo; i < lo + per && i < len; i++) {
    s += abs2(sv[base + i]);
    cum[i] = s;
  }
  run_tot[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double acc = 0.0;
    for (int t = 0; t < (int)blockDim.x; t++) {
      const double v = run_tot[t];
      run_tot[t] = acc;
      acc += v;
    }
  }
  __syncthreads();
  const double off = run_tot[threadIdx.x];
  for (int i = lo; i < lo + per && i < len; i++) cum[i] += off;
  __syncthreads();
  for (int64_t sidx = threadIdx.x; sidx < cnt; sidx += blockDim.x) {
    const double u = resid[first + sidx];
    int a = 0, b = len;  // first i with cum[i] > u
    while (a < b) {
      const int mid = (a + b) >> 1;
      if (cum[mid] > u)
        b = mid;
      else
        a = mid + 1;
    }
    if (a >= len) {  // u at/after the block total (rounding): last element with mass
      a = len - 1;
      while (a > 0 && cum[a] == cum[a - 1]) a--;
    }
    out_off[first + sidx] = base + (uint64_t)a;
  }
}

// ------------------------------------------------------------------ exchange
__device__ __forceinline__ uint64_t insert_bit(uint64_t x, int p, int v) {
  const uint64_t lo = x & ((1ull << p) - 1);
  return ((x - lo) << 1) | ((uint64_t)v << p) | lo;
}

// Pack / unpack of an exchanged block: element j of a block (compact index over the local bits that
// are not exchanged) lives at the index with the exchanged bits inserted (values fixed per block);
// consecutive j are consecutive amplitudes below the lowest inserted bit.  Pack writes the block
// contiguously (into a local send slot, or straight into a peer's receive slot over NVLink: remote
// stores only, full lines); unpack scatters a received slot into place.
struct InsDev {
  int nins;
  int pos[11];  // ascending
  int val[11];
  uint64_t limit;  // SV_CHECK=1: trap on an index >= limit (0: unchecked)
};
// Eight elements per thread per iteration: eight loads in flight per thread before any store, so
// a small grid (the exchange leaves most SMs to the concurrent section) still keeps enough bytes in
// flight for NVLink (one element per thread topped out near 0.5 of the link).
template <typename V, bool PACK>
__global__ void k_pack_bits(V* __restrict__ sv, V* __restrict__ stage, uint64_t first, uint64_t count, InsDev e) {
  constexpr int U = 8;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  auto at = [&](uint64_t i) {
    uint64_t x = first + i;
    for (int k = 0; k < e.nins; k++) x = insert_bit(x, e.pos[k], e.val[k]);
    if (e.limit && x >= e.limit) __trap();
    return x;
  };
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < count; i += U * stride) {
    uint64_t x[U];
    V t[U];
#pragma unroll
    for (int u = 0; u < U; u++) x[u] = at(i + u * stride);
#pragma unroll
    for (int u = 0; u < U; u++) t[u] = PACK ? sv[x[u]] : stage[i + u * stride];
#pragma unroll
    for (int u = 0; u < U; u++) {
      if (PACK)
        stage[i + u * stride] = t[u];
      else
        sv[x[u]] = t[u];
    }
  }
  for (; i < count; i += stride) {
    const uint64_t x = at(i);
    if (PACK)
      stage[i] = sv[x];
    else
      sv[x] = stage[i];
  }
}

// ------------------------------------------------------------------ host helpers
inline unsigned grid_for(uint64_t work, int threads) {
  uint64_t b = (work + threads - 1) / threads;
  const uint64_t cap = 148ull * 16;
  if (b > cap) b = cap;
  if (b == 0) b = 1;
  return (unsigned)b;
}

template <typename V>
V to_v(const double* c);
template <>
double2 to_v<double2>(const double* c) {
  return make_double2(c[0], c[1]);
}
template <>
float2 to_v<float2>(const double* c) {
  return make_float2((float)c[0], (float)c[1]);
}

template <typename V>
cudaError_t launch_gate_t(V* sv, int nL, const GateArgs& g, cudaStream_t st) {
  const int th = 256;
  const uint64_t N = 1ull << nL;
  switch (g.type) {
    case SV_OP_U1:
      k_gate_u1<V><<<grid_for(N / 2, th), th, 0, st>>>(sv, N / 2, g.q0, to_v<V>(g.m), to_v<V>(g.m + 2),
                                                       to_v<V>(g.m + 4), to_v<V>(g.m + 6));
      break;
    case SV_OP_U2: {
      Mat16<V> M;
      for (int i = 0; i < 16; i++) M.m[i] = to_v<V>(g.m + 2 * i);
      k_gate_u2<V><<<grid_for(N / 4, th), th, 0, st>>>(sv, N / 4, g.q0, g.q1, M);
      break;
    }
    case SV_OP_DIAG:
      k_gate_diag<V><<<grid_for(N, th), th, 0, st>>>(sv, N, g.q0, g.q1, to_v<V>(g.m), to_v<V>(g.m + 2),
                                                     to_v<V>(g.m + 4), to_v<V>(g.m + 6));
      break;
    case 7:
      k_gate_swap<V><<<grid_for(N / 4, th), th, 0, st>>>(sv, N / 4, g.q0, g.q1);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace

// ------------------------------------------------------------------ public wrappers
cudaError_t launch_gate(bool dbl, void* sv, int nL, const GateArgs& g, cudaStream_t st) {
  return dbl ? launch_gate_t<double2>((double2*)sv, nL, g, st) : launch_gate_t<float2>((float2*)sv, nL, g, st);
}

cudaError_t launch_set_basis(bool dbl, void* sv, int nL, int64_t off, cudaStream_t st) {
  const size_t bytes = (dbl ? 16 : 8) * (size_t(1) << nL);
  cudaError_t e = cudaMemsetAsync(sv, 0, bytes, st);
  if (e != cudaSuccess || off < 0) return e;
  if (dbl)
    k_set_one<double2><<<1, 1, 0, st>>>((double2*)sv, off);
  else
    k_set_one<float2><<<1, 1, 0, st>>>((float2*)sv, off);
  return cudaGetLastError();
}

cudaError_t launch_set_amp(bool dbl, void* sv, int64_t off, double re, cudaStream_t st) {
  if (dbl)
    k_set_amp<double2><<<1, 1, 0, st>>>((double2*)sv, off, re);
  else
    k_set_amp<float2><<<1, 1, 0, st>>>((float2*)sv, off, re);
  return cudaGetLastError();
}

size_t norm_scratch_doubles() { return kRedBlocks; }

cudaError_t launch_norm(bool dbl, const void* sv, int nL, double* scratch, double* out_dev, cudaStream_t st) {
  const uint64_t N = 1ull << nL;
  if (dbl)
    k_norm_partial<double2><<<kRedBlocks, kRedThreads, 0, st>>>((const double2*)sv, N, scratch);
  else
    k_norm_partial<float2><<<kRedBlocks, kRedThreads, 0, st>>>((const float2*)sv, N, scratch);
  k_sum_partials<<<1, 1024, 0, st>>>(scratch, kRedBlocks, out_dev);
  return cudaGetLastError();
}

static constexpr int kMargBlocks = 148 * 2;
static constexpr int kMargSmemBits = 12;

size_t marginal_scratch_doubles(int nq) { return nq <= kMargSmemBits ? (size_t)kMargBlocks << nq : 0; }

cudaError_t launch_marginal(bool dbl, const void* sv, int nL, const int* qbits, int nq, double* scratch,
                            double* out_dev, cudaStream_t st) {
  if (nq > 24) return cudaErrorInvalidValue;
  const uint64_t N = 1ull << nL;
  const int bins = 1 << nq;
  int nit_avail = 0;  // non-marginal bits >= 5 (the task form needs at least one)
  for (int b = 5; b < nL; b++) {
    bool q = false;
    for (int i = 0; i < nq; i++) q |= qbits[i] == b;
    nit_avail += q ? 0 : 1;
  }
  if (nL < 11 || nit_avail == 0) {  // tiny shards: one atomic per amplitude
    QBits q;
    for (int i = 0; i < nq; i++) q.b[i] = qbits[i];
    cudaError_t e = cudaMemsetAsync(out_dev, 0, sizeof(double) * bins, st);
    if (e != cudaSuccess) return e;
    if (dbl)
      k_marginal_small<double2><<<grid_for(N, 256), 256, 0, st>>>((const double2*)sv, N, q, nq, out_dev);
    else
      k_marginal_small<float2><<<grid_for(N, 256), 256, 0, st>>>((const float2*)sv, N, q, nq, out_dev);
    return cudaGetLastError();
  }
  MargPlan p{};
  p.nq = nq;
  uint64_t qmask = 0;
  for (int i = 0; i < nq; i++) {
    p.qb[i] = qbits[i];
    qmask |= 1ull << qbits[i];
  }
  p.lane_q = (uint32_t)(qmask & 31u);
  for (int b = 5; b < nL; b++) {
    if (!((qmask >> b) & 1) && p.nit < 6)
      p.it_b[p.nit++] = b;
    else
      p.task_b[p.ntb++] = b;
  }
  const bool smem = nq <= kMargSmemBits;
  if (!smem) {
    cudaError_t e = cudaMemsetAsync(out_dev, 0, sizeof(double) * bins, st);
    if (e != cudaSuccess) return e;
  }
  double* dst = smem ? scratch : out_dev;
  const size_t shm = smem ? sizeof(double) * bins : 0;
  if (dbl)
    k_marginal_tasks<double2><<<kMargBlocks, 512, shm, st>>>((const double2*)sv, p, dst, smem ? 1 : 0);
  else
    k_marginal_tasks<float2><<<kMargBlocks, 512, shm, st>>>((const float2*)sv, p, dst, smem ? 1 : 0);
  if (smem) k_reduce_bins<<<grid_for(bins, 256), 256, 0, st>>>(scratch, kMargBlocks, bins, out_dev);
  return cudaGetLastError();
}

cudaError_t launch_block_sums(bool dbl, const void* sv, int nL, int B, double* out_dev, cudaStream_t st) {
  const unsigned blocks = (unsigned)(1ull << (nL - B));
  if (dbl)
    k_block_sums<double2><<<blocks, 256, 0, st>>>((const double2*)sv, B, out_dev);
  else
    k_block_sums<float2><<<blocks, 256, 0, st>>>((const float2*)sv, B, out_dev);
  return cudaGetLastError();
}

cudaError_t launch_sample_resolve(bool dbl, const void* sv, int B, const int64_t* items, int n_items,
                                  const double* resid, uint64_t* out_off, cudaStream_t st) {
  if (n_items == 0) return cudaSuccess;
  const size_t smem = sizeof(double) << B;
  static bool attr[64] = {};  // cudaFuncSetAttribute applies to the current device only
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  if (!attr[dev]) {
    if ((e = cudaFuncSetAttribute(k_sample_resolve<double2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024)) != cudaSuccess ||
        (e = cudaFuncSetAttribute(k_sample_resolve<float2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024)) != cudaSuccess)
      return e;
    attr[dev] = true;
  }
  if (dbl)
    k_sample_resolve<double2><<<n_items, 256, smem, st>>>((const double2*)sv, B, items, resid, out_off);
  else
    k_sample_resolve<float2><<<n_items, 256, smem, st>>>((const float2*)sv, B, items, resid, out_off);
  return cudaGetLastError();
}

cudaError_t launch_gather(bool dbl, const void* sv, const uint64_t* offs, size_t cnt, void* out, cudaStream_t st) {
  if (cnt == 0) return cudaSuccess;
  if (dbl)
    k_gather<double2><<<grid_for(cnt, 256), 256, 0, st>>>((const double2*)sv, offs, cnt, (double2*)out);
  else
    k_gather<float2><<<grid_for(cnt, 256), 256, 0, st>>>((const float2*)sv, offs, cnt, (float2*)out);
  return cudaGetLastError();
}

cudaError_t launch_pack_bits(bool dbl, bool pack, void* sv, void* stage, uint64_t first, uint64_t count, int nins,
                             const int* pos, const int* val, uint64_t shard_amps, cudaStream_t st, unsigned max_blocks) {
  if (nins > 11) return cudaErrorInvalidValue;
  InsDev e{};
  e.nins = nins;
  static const bool check = [] {
    const char* v = std::getenv("SV_CHECK");
    return v && v[0] == '1';
  }();
  if (check) e.limit = shard_amps;
  for (int i = 0; i < nins; i++) {  // ascending positions (insert_bit order)
    e.pos[i] = pos[i];
    e.val[i] = val[i];
  }
  for (int i = 1; i < nins; i++)
    for (int j = i; j > 0 && e.pos[j] < e.pos[j - 1]; j--) {
      std::swap(e.pos[j], e.pos[j - 1]);
      std::swap(e.val[j], e.val[j - 1]);
    }
  unsigned g = grid_for(count, 256);
  if (max_blocks && g > max_blocks) g = max_blocks;
  if (dbl) {
    if (pack)
      k_pack_bits<double2, true><<<g, 256, 0, st>>>((double2*)sv, (double2*)stage, first, count, e);
    else
      k_pack_bits<double2, false><<<g, 256, 0, st>>>((double2*)sv, (double2*)stage, first, count, e);
  } else {
    if (pack)
      k_pack_bits<float2, true><<<g, 256, 0, st>>>((float2*)sv, (float2*)stage, first, count, e);
    else
      k_pack_bits<float2, false><<<g, 256, 0, st>>>((float2*)sv, (float2*)stage, first, count, e);
  }
  return cudaGetLastError();
}

// Copy-engine form of pack / unpack (no SM): when every inserted bit is >= lo and runs of 2^lo
// elements are at least min_run elements long, a block piece is a few strided 2-D copies (rows of
// 2^lo elements; the pitch is constant up to the next inserted bit that is not adjacent to lo's
// group).  stage may be a peer's receive slot (CUDA IPC / same device): the rows then go over NVLink
// straight from the state, without a local send slot.  Returns cudaErrorNotSupported when the
// piece does not have that shape (the caller packs with k_pack_bits instead).
cudaError_t copy_bits_ce(bool pack, void* sv, void* stage, uint64_t first, uint64_t count, int nins, const int* pos,
                         const int* val, size_t amp, uint64_t min_run, cudaStream_t st, int* copies) {
  *copies = 0;
  if (nins < 1 || nins > 11 || count == 0) return cudaErrorNotSupported;
  int P[11], Vv[11];
  for (int i = 0; i < nins; i++) P[i] = pos[i], Vv[i] = val[i];
  for (int i = 1; i < nins; i++)
    for (int j = i; j > 0 && P[j] < P[j - 1]; j--) std::swap(P[j], P[j - 1]), std::swap(Vv[j], Vv[j - 1]);
  const int lo = P[0];
  const uint64_t run = 1ull << lo;
  if (run < min_run) return cudaErrorNotSupported;
  auto addr = [&](uint64_t x) {  // compact index -> element index (insert_bit, ascending)
    for (int k = 0; k < nins; k++) {
      const uint64_t l = x & ((1ull << P[k]) - 1);
      x = ((x - l) << 1) | ((uint64_t)Vv[k] << P[k]) | l;
    }
    return x;
  };
  char* S = (char*)sv;
  char* G = (char*)stage;
  if (count <= run) {  // inside one run: one contiguous copy
    if ((first >> lo) != ((first + count - 1) >> lo)) return cudaErrorNotSupported;
    const uint64_t a = addr(first);
    *copies = 1;
    return pack ? cudaMemcpyAsync(G, S + a * amp, count * amp, cudaMemcpyDeviceToDevice, st)
                : cudaMemcpyAsync(S + a * amp, G, count * amp, cudaMemcpyDeviceToDevice, st);
  }
  if ((first & (run - 1)) || (count & (run - 1))) return cudaErrorNotSupported;
  int a = 1;
  while (a < nins && P[a] == lo + a) a++;
  const size_t width = run * amp, pitch = (1ull << (lo + a)) * amp;
  const uint64_t seg_rows = a < nins ? 1ull << (P[a] - lo - a) : ~0ull;  // rows of constant pitch
  const uint64_t r0 = first >> lo, r1 = (first + count) >> lo;
  const bool rows_1d = pitch > (size_t)INT32_MAX;
  if (rows_1d && r1 - r0 > 64) return cudaErrorNotSupported;
  for (uint64_t r = r0; r < r1;) {
    const uint64_t e = seg_rows == ~0ull ? r1 : std::min(r1, (r / seg_rows + 1) * seg_rows);
    char* sp = S + addr(r << lo) * amp;
    char* gp = G + ((r - r0) << lo) * amp;
    cudaError_t err = cudaSuccess;
    if (rows_1d) {
      for (uint64_t i = 0; i < e - r && err == cudaSuccess; i++, (*copies)++)
        err = pack ? cudaMemcpyAsync(gp + i * width, sp + i * pitch, width, cudaMemcpyDeviceToDevice, st)
                   : cudaMemcpyAsync(sp + i * pitch, gp + i * width, width, cudaMemcpyDeviceToDevice, st);
    } else {
      err = pack ? cudaMemcpy2DAsync(gp, width, sp, pitch, width, e - r, cudaMemcpyDeviceToDevice, st)
                 : cudaMemcpy2DAsync(sp, pitch, gp, width, width, e - r, cudaMemcpyDeviceToDevice, st);
      (*copies)++;
    }
    if (err != cudaSuccess) return err;
    r = e;
  }
  return cudaSuccess;
}

// State to state: the rows of a block piece (inserted bits valued vsrc) of src go to the same rows
// of dst with the inserted bits valued vdst — the in-place form of the exchange, dst a peer's
// state.  dry: only check the shape.  cudaErrorNotSupported as copy_bits_ce.
cudaError_t copy_bits_ce_xx(void* src, const int* vsrc, void* dst, const int* vdst, uint64_t first, uint64_t count,
                            int nins, const int* pos, size_t amp, uint64_t min_run, cudaStream_t st, int* copies,
                            bool dry) {
  *copies = 0;
  if (nins < 1 || nins > 11 || count == 0) return cudaErrorNotSupported;
  int P[11], Vs[11], Vd[11];
  for (int i = 0; i < nins; i++) P[i] = pos[i], Vs[i] = vsrc[i], Vd[i] = vdst[i];
  for (int i = 1; i < nins; i++)
    for (int j = i; j > 0 && P[j] < P[j - 1]; j--)
      std::swap(P[j], P[j - 1]), std::swap(Vs[j], Vs[j - 1]), std::swap(Vd[j], Vd[j - 1]);
  const int lo = P[0];
  const uint64_t run = 1ull << lo;
  if (run < min_run) return cudaErrorNotSupported;
  auto addr = [&](uint64_t x, const int* V) {
    for (int k = 0; k < nins; k++) {
      const uint64_t l = x & ((1ull << P[k]) - 1);
      x = ((x - l) << 1) | ((uint64_t)V[k] << P[k]) | l;
    }
    return x;
  };
  char* S = (char*)src;
  char* D = (char*)dst;
  if (count <= run) {
    if ((first >> lo) != ((first + count - 1) >> lo)) return cudaErrorNotSupported;
    if (dry) return cudaSuccess;
    *copies = 1;
    return cudaMemcpyAsync(D + addr(first, Vd) * amp, S + addr(first, Vs) * amp, count * amp, cudaMemcpyDeviceToDevice, st);
  }
  if ((first & (run - 1)) || (count & (run - 1))) return cudaErrorNotSupported;
  int a = 1;
  while (a < nins && P[a] == lo + a) a++;
  const size_t width = run * amp, pitch = (1ull << (lo + a)) * amp;
  const uint64_t seg_rows = a < nins ? 1ull << (P[a] - lo - a) : ~0ull;
  const uint64_t r0 = first >> lo, r1 = (first + count) >> lo;
  const bool rows_1d = pitch > (size_t)INT32_MAX;
  if (rows_1d && r1 - r0 > 64) return cudaErrorNotSupported;
  if (dry) return cudaSuccess;
  for (uint64_t r = r0; r < r1;) {
    const uint64_t e = seg_rows == ~0ull ? r1 : std::min(r1, (r / seg_rows + 1) * seg_rows);
    char* sp = S + addr(r << lo, Vs) * amp;
    char* dp = D + addr(r << lo, Vd) * amp;
    cudaError_t err = cudaSuccess;
    if (rows_1d) {
      for (uint64_t i = 0; i < e - r && err == cudaSuccess; i++, (*copies)++)
        err = cudaMemcpyAsync(dp + i * pitch, sp + i * pitch, width, cudaMemcpyDeviceToDevice, st);
    } else {
      err = cudaMemcpy2DAsync(dp, pitch, sp, pitch, width, e - r, cudaMemcpyDeviceToDevice, st);
      (*copies)++;
    }
    if (err != cudaSuccess) return err;
    r = e;
  }
  return cudaSuccess;
}

}  // namespace sv
