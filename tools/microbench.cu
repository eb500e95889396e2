// Microbenchmarks that fill the peaks MEASURED_PEAKS.json lacks (SURVEY §8(d) protocol items 1-3):
//   * DFMA / FFMA / DMMA issue rate, measured in SM cycles (clock64 inside the kernel), so the
//     per-clock rate is independent of the clock the GPU happens to hold; the per-second rate at
//     the observed clock is printed beside it (the clock itself: nvidia-smi sampled by the caller);
//   * shared-memory LDS.128 bandwidth per SM cycle;
//   * HBM streaming copy of complex128 (plain LDG/STG), and the same copy with the loads done by
//     cp.async.bulk (UBLKCP) into a two-slot mbarrier-guarded shared-memory ring, in runs of 128 B
//     and 1 KiB (the section kernel's tile gathers are unions of such runs).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda.h>
#include <cudaTypedefs.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ unsigned long long g_cyc[4096];

template <int CH>
__global__ void dfma_kernel(double* out, double a, double b, int iters) {
  double x[CH];
#pragma unroll
  for (int i = 0; i < CH; i++) x[i] = threadIdx.x * 1e-3 + i;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < CH; i++) x[i] = fma(x[i], a, b);
  }
  __syncthreads();
  if (threadIdx.x == 0) g_cyc[blockIdx.x] = clock64() - t0;
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; i++) s += x[i];
  if (s == 123.456) out[0] = s;
}
template <int CH>
__global__ void ffma_kernel(float* out, float a, float b, int iters) {
  float x[CH];
#pragma unroll
  for (int i = 0; i < CH; i++) x[i] = threadIdx.x * 1e-3f + i;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < CH; i++) x[i] = fmaf(x[i], a, b);
  }
  __syncthreads();
  if (threadIdx.x == 0) g_cyc[blockIdx.x] = clock64() - t0;
  float s = 0;
#pragma unroll
  for (int i = 0; i < CH; i++) s += x[i];
  if (s == 123.456f) out[0] = s;
}
__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 0.5;
  double c[4][2];
  for (int i = 0; i < 4; i++) { c[i][0] = 0; c[i][1] = 0; }
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 4; i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  __syncthreads();
  if (threadIdx.x == 0) g_cyc[blockIdx.x] = clock64() - t0;
  double s = 0;
  for (int i = 0; i < 4; i++) s += c[i][0] + c[i][1];
  if (s == 123.456) out[0] = s;
}

__global__ void smem_kernel(double* out, int iters) {
  extern __shared__ double2 sm[];
  int n = 4096;
  for (int i = threadIdx.x; i < n; i += blockDim.x) sm[i] = make_double2(i, i);
  __syncthreads();
  double2 acc = make_double2(0, 0);
  int idx = threadIdx.x;
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int u = 0; u < 8; u++) {
      double2 v = sm[(idx + u * 256) & (n - 1)];
      acc.x += v.x; acc.y += v.y;
    }
    idx += 1;
  }
  __syncthreads();
  if (threadIdx.x == 0) g_cyc[blockIdx.x] = clock64() - t0;
  if (acc.x == 123.456) out[0] = acc.x + acc.y;
}
__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) b[i] = a[i];
}

// ---- cp.async.bulk streaming copy: persistent CTAs, tiles of TILE complex128 in a two-slot ring
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile("{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(sa(b)),
               "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(dst)),
               "l"(src), "r"(bytes), "r"(sa(b)) : "memory");
}
template <int TILE, int RUN>
__global__ void __launch_bounds__(TILE / 16) bulk_copy_kernel(const double2* __restrict__ a, double2* __restrict__ b,
                                                              size_t ntiles) {
  extern __shared__ __align__(128) unsigned char raw[];
  double2* slot = reinterpret_cast<double2*>(raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(raw + 2 * TILE * 16);
  constexpr int NT = TILE / 16, RUNS = TILE / RUN;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](size_t t, int s) {
    if (threadIdx.x < 32) {
      if (threadIdx.x == 0) mbar_expect(&bar[s], TILE * 16);
      __syncwarp();
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      for (int r = threadIdx.x; r < RUNS; r += 32)
        bulk_g2s(slot + s * TILE + r * RUN, a + t * TILE + (size_t)r * RUN, RUN * 16, &bar[s]);
    }
  };
  size_t t = blockIdx.x;
  if (t < ntiles) issue(t, 0);
  for (int j = 0; t < ntiles; t += gridDim.x, j++) {
    const int s = j & 1;
    if (t + gridDim.x < ntiles) issue(t + gridDim.x, s ^ 1);
    mbar_wait(&bar[s], (j >> 1) & 1);
    double2* src = slot + s * TILE;
#pragma unroll
    for (int k = 0; k < 16; k++) b[t * TILE + k * NT + threadIdx.x] = src[k * NT + threadIdx.x];
    __syncthreads();
  }
}


// ---- tile-gather streaming (the section kernel's access pattern): tiles of 2^11 complex128 over
// memory bits {0,1,2} u {5,6} u {10,11} u {15,16} u {20,21} of a 2^30-amplitude state, read and
// written back in place.  (a) plain LDG/STG, 16 amplitudes per thread; (b) loads by one TMA tensor
// copy per tile (5-D box of 128-byte rows) into an S-slot mbarrier ring, stores by STG.
__device__ __forceinline__ uint64_t tile_base(uint64_t t) {
  return ((t & 3) << 3) | (((t >> 2) & 7) << 7) | (((t >> 5) & 7) << 12) | (((t >> 8) & 7) << 17) | ((t >> 11) << 22);
}
__device__ __forceinline__ uint64_t tile_pos(int i) {
  return (uint64_t)(i & 7) | ((uint64_t)((i >> 3) & 3) << 5) | ((uint64_t)((i >> 5) & 3) << 10) |
         ((uint64_t)((i >> 7) & 3) << 15) | ((uint64_t)((i >> 9) & 3) << 20);
}
__global__ void __launch_bounds__(128) gather_ldg_kernel(double2* __restrict__ a, int dummy) {
  extern __shared__ double2 pad[];
  if (dummy) pad[0] = make_double2(0, 0);
  const uint64_t b = tile_base(blockIdx.x);
  double2 v[16];
#pragma unroll
  for (int k = 0; k < 16; k++) v[k] = a[b + tile_pos(k * 128 + threadIdx.x)];
#pragma unroll
  for (int k = 0; k < 16; k++) { v[k].x += 1.0; a[b + tile_pos(k * 128 + threadIdx.x)] = v[k]; }
}
template <int S>
__global__ void __launch_bounds__(128) gather_tma_kernel(double2* __restrict__ a, const __grid_constant__ CUtensorMap tm,
                                                         uint64_t ntiles) {
  extern __shared__ __align__(128) unsigned char raw[];
  double2* slot = reinterpret_cast<double2*>(raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(raw + S * 2048 * 16);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; s++) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](uint64_t t, int s) {
    if (threadIdx.x == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect(&bar[s], 2048 * 16);
      const int c0 = 16 * (int)(t & 3), c1 = 4 * (int)((t >> 2) & 7), c2 = 4 * (int)((t >> 5) & 7),
                c3 = 4 * (int)((t >> 8) & 7), c4 = 4 * (int)(t >> 11);
      asm volatile(
          "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(
              sa(slot + s * 2048)),
          "l"(reinterpret_cast<uint64_t>(&tm)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(sa(&bar[s]))
          : "memory");
    }
  };
  uint64_t t = blockIdx.x;
  for (int s = 0; s < S - 1; s++)
    if (t + s * gridDim.x < ntiles) issue(t + s * gridDim.x, s);
  for (int j = 0; t < ntiles; t += gridDim.x, j++) {
    const int s = j % S;
    if (t + (S - 1) * gridDim.x < ntiles) issue(t + (S - 1) * gridDim.x, (j + S - 1) % S);
    mbar_wait(&bar[s], (j / S) & 1);
    const double2* src = slot + s * 2048;
    const uint64_t b = tile_base(t);
#pragma unroll
    for (int k = 0; k < 16; k++) {
      double2 v = src[k * 128 + threadIdx.x];
      v.x += 1.0;
      a[b + tile_pos(k * 128 + threadIdx.x)] = v;
    }
    __syncthreads();
  }
}

static double median_cycles(int blocks) {
  static unsigned long long h[4096];
  cudaMemcpyFromSymbol(h, g_cyc, sizeof(unsigned long long) * blocks);
  // insertion sort is fine for <= 4096
  for (int i = 1; i < blocks; i++)
    for (int j = i; j > 0 && h[j] < h[j - 1]; j--) { unsigned long long t = h[j]; h[j] = h[j - 1]; h[j - 1] = t; }
  return (double)h[blocks / 2];
}

template <int TILE, int RUN>
int run_bulk(const double2* a, double2* b, size_t n, int sms, int ctas_per_sm, cudaEvent_t e0, cudaEvent_t e1) {
  const size_t smem = 2 * TILE * 16 + 64;
  CK(cudaFuncSetAttribute(bulk_copy_kernel<TILE, RUN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const size_t ntiles = n / TILE;
  float ms = 0, best = 1e30f;
  for (int rep = 0; rep < 4; rep++) {
    cudaEventRecord(e0);
    bulk_copy_kernel<TILE, RUN><<<sms * ctas_per_sm, TILE / 16, smem>>>(a, b, ntiles);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep && ms < best) best = ms;
  }
  printf("{\"bench\":\"hbm_bulk_copy_c128\",\"tile_bytes\":%d,\"run_bytes\":%d,\"ctas_per_sm\":%d,\"ms\":%.3f,\"GBps_rw\":%.1f}\n",
         TILE * 16, RUN * 16, ctas_per_sm, best, 2.0 * n * 16 / (best * 1e-3) / 1e9);
  return 0;
}


template <int S>
int run_tma(double2* a, int sms, int ctas_per_sm, const CUtensorMap& tm, cudaEvent_t e0, cudaEvent_t e1) {
  const size_t smem = S * 2048 * 16 + 64;
  CK(cudaFuncSetAttribute(gather_tma_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const uint64_t ntiles = 1ull << 19;
  float ms = 0, best = 1e30f;
  for (int rep = 0; rep < 4; rep++) {
    cudaEventRecord(e0);
    gather_tma_kernel<S><<<sms * ctas_per_sm, 128, smem>>>(a, tm, ntiles);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep && ms < best) best = ms;
  }
  printf("{\"bench\":\"tile_gather_tma\",\"slots\":%d,\"ctas_per_sm\":%d,\"ms\":%.3f,\"GBps_rw\":%.1f}\n", S, ctas_per_sm, best,
         2.0 * (1ull << 30) * 16 / (best * 1e-3) / 1e9);
  return 0;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("{\"gpu\":\"%s\",\"sms\":%d,\"smem_per_block_optin\":%zu,\"smem_per_sm\":%zu,\"regs_per_sm\":%d,\"l2_bytes\":%d,\"mem_bytes\":%zu,\"clock_khz\":%d}\n",
         p.name, p.multiProcessorCount, p.sharedMemPerBlockOptin, p.sharedMemPerMultiprocessor, p.regsPerMultiprocessor, p.l2CacheSize, p.totalGlobalMem, clk_khz);
  double* dout; CK(cudaMalloc(&dout, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int sms = p.multiProcessorCount;
  float ms;
  // per-SM cycle rates: 4 CTAs x 256 threads resident on every SM; rate/clk/SM = work per CTA x
  // 4 / cycles of one CTA; the implied clock = cycles / event time
  for (int rep = 0; rep < 3; rep++) {
    const int iters = 40000, blocks = sms * 4, threads = 256;
    cudaEventRecord(e0);
    dfma_kernel<8><<<blocks, threads>>>(dout, 0.999, 1e-3, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    const double cyc = median_cycles(blocks);
    const double per_clk = 4.0 * threads * iters * 8 / cyc;
    const double fmas = (double)blocks * threads * iters * 8;
    printf("{\"bench\":\"dfma\",\"ms\":%.3f,\"dfma_per_clk_sm\":%.2f,\"dfma_per_s\":%.4e,\"implied_mhz\":%.0f}\n", ms, per_clk,
           fmas / (ms * 1e-3), cyc / (ms * 1e-3) / 1e6);
  }
  for (int rep = 0; rep < 2; rep++) {
    const int iters = 40000, blocks = sms * 4, threads = 256;
    cudaEventRecord(e0);
    ffma_kernel<8><<<blocks, threads>>>((float*)dout, 0.999f, 1e-3f, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    const double cyc = median_cycles(blocks);
    const double fmas = (double)blocks * threads * iters * 8;
    printf("{\"bench\":\"ffma\",\"ms\":%.3f,\"ffma_per_clk_sm\":%.2f,\"ffma_per_s\":%.4e,\"implied_mhz\":%.0f}\n", ms,
           4.0 * threads * iters * 8 / cyc, fmas / (ms * 1e-3), cyc / (ms * 1e-3) / 1e6);
  }
  for (int rep = 0; rep < 2; rep++) {
    const int iters = 20000, blocks = sms * 4, threads = 256;
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(dout, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    const double cyc = median_cycles(blocks);
    const double per_cta = (double)(threads / 32) * iters * 4 * 256.0;  // m8n8k4 = 256 FMA per warp-instr
    printf("{\"bench\":\"dmma_m8n8k4\",\"ms\":%.3f,\"fma_per_clk_sm\":%.2f,\"tflops\":%.2f}\n", ms, 4.0 * per_cta / cyc,
           2 * per_cta * blocks / (ms * 1e-3) / 1e12);
  }
  CK(cudaFuncSetAttribute(smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  for (int rep = 0; rep < 2; rep++) {
    const int iters = 20000, blocks = sms * 3, threads = 256;
    cudaEventRecord(e0);
    smem_kernel<<<blocks, threads, 65536>>>(dout, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    const double cyc = median_cycles(blocks);
    printf("{\"bench\":\"smem_lds128\",\"ms\":%.3f,\"bytes_per_clk_sm\":%.2f}\n", ms, 3.0 * threads * iters * 8 * 16 / cyc);
  }
  const size_t n = (size_t)1 << 30;  // 16 GiB complex128 each way (the QFT30 state size)
  double2 *a, *b; CK(cudaMalloc(&a, n * 16)); CK(cudaMalloc(&b, n * 16));
  cudaMemset(a, 0, n * 16); cudaMemset(b, 0, n * 16);
  for (int rep = 0; rep < 4; rep++) {
    cudaEventRecord(e0);
    copy_kernel<<<sms * 8, 512>>>(a, b, n);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"bench\":\"hbm_copy_c128\",\"ms\":%.3f,\"GBps_rw\":%.1f}\n", ms, 2.0 * n * 16 / (ms * 1e-3) / 1e9);
  }
  run_bulk<2048, 8>(a, b, n, sms, 3, e0, e1);
  run_bulk<2048, 8>(a, b, n, sms, 2, e0, e1);
  run_bulk<2048, 64>(a, b, n, sms, 3, e0, e1);
  run_bulk<1024, 8>(a, b, n, sms, 6, e0, e1);
  run_bulk<4096, 8>(a, b, n, sms, 1, e0, e1);

  // tile-gather patterns (in place on a)
  for (int smem_kb : {0, 32, 40}) {
    CK(cudaFuncSetAttribute(gather_ldg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kb * 1024));
    float best = 1e30f;
    for (int rep = 0; rep < 4; rep++) {
      cudaEventRecord(e0);
      gather_ldg_kernel<<<1u << 19, 128, smem_kb * 1024>>>(a, 0);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      if (rep && ms < best) best = ms;
    }
    printf("{\"bench\":\"tile_gather_ldg\",\"smem_kb\":%d,\"ms\":%.3f,\"GBps_rw\":%.1f}\n", smem_kb, best, 2.0 * n * 16 / (best * 1e-3) / 1e9);
  }
  {
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
    CUtensorMap tm;
    cuuint64_t dims[5] = {64, 32, 32, 32, 1024};
    cuuint64_t strides[4] = {512, 16384, 524288, 16777216};
    cuuint32_t box[5] = {16, 4, 4, 4, 4}, es[5] = {1, 1, 1, 1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, a, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("{\"bench\":\"tensor_map_encode\",\"rc\":%d}\n", (int)r);
    if (r == CUDA_SUCCESS) {
      run_tma<2>(a, sms, 3, tm, e0, e1);
      run_tma<3>(a, sms, 2, tm, e0, e1);
      run_tma<2>(a, sms, 2, tm, e0, e1);
      run_tma<4>(a, sms, 1, tm, e0, e1);
    }
  }
  // sustained DFMA: back to back for ~4 s (the FP64 rate a long section step sees under the power cap)
  {
    const int iters = 40000, blocks = sms * 4, threads = 256;
    float tot = 0;
    int launches = 0;
    cudaEventRecord(e0);
    while (tot < 4000.0f) {
      for (int r2 = 0; r2 < 50; r2++) dfma_kernel<8><<<blocks, threads>>>(dout, 0.999, 1e-3, iters);
      launches += 50;
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&tot, e0, e1);
    }
    const double fmas = (double)blocks * threads * iters * 8 * launches;
    printf("{\"bench\":\"dfma_sustained\",\"s\":%.2f,\"dfma_per_s\":%.4e,\"tflops\":%.2f}\n", tot / 1e3, fmas / (tot * 1e-3),
           2 * fmas / (tot * 1e-3) / 1e12);
  }
  CK(cudaGetLastError());
  return 0;
}
