// Microbenchmarks that fill the peaks MEASURED_PEAKS.json lacks (SURVEY §8(d) protocol items 1-3):
// DFMA / FFMA / DMMA issue rate, shared-memory LDS.128 bandwidth, HBM streaming copy of complex128.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int CH>
__global__ void dfma_kernel(double* out, double a, double b, int iters) {
  double x[CH];
#pragma unroll
  for (int i = 0; i < CH; i++) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < CH; i++) x[i] = fma(x[i], a, b);
  }
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
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < CH; i++) x[i] = fmaf(x[i], a, b);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < CH; i++) s += x[i];
  if (s == 123.456f) out[0] = s;
}
__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 0.5;
  double c[4][2];
  for (int i = 0; i < 4; i++) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 4; i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 4; i++) s += c[i][0] + c[i][1];
  if (s == 123.456) out[0] = s;
}
// DMMA and DFMA interleaved: if the FP64 tensor path and the FMA pipe are separate units, the
// combined FMA rate exceeds either alone.
__global__ void mixed_kernel(double* out, int iters, double a0, double b0) {
  double a = threadIdx.x * 1e-3, b = 0.5;
  double c[4][2];
  double x[8];
  for (int i = 0; i < 4; i++) { c[i][0] = 0; c[i][1] = 0; }
  for (int i = 0; i < 8; i++) x[i] = threadIdx.x + i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 4; i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
#pragma unroll
    for (int j = 0; j < 4; j++)
#pragma unroll
      for (int i = 0; i < 8; i++) x[i] = fma(x[i], a0, b0);
  }
  double s = 0;
  for (int i = 0; i < 4; i++) s += c[i][0] + c[i][1];
  for (int i = 0; i < 8; i++) s += x[i];
  if (s == 123.456) out[0] = s;
}

__global__ void smem_kernel(double* out, int iters) {
  extern __shared__ double2 sm[];
  int n = 4096;
  for (int i = threadIdx.x; i < n; i += blockDim.x) sm[i] = make_double2(i, i);
  __syncthreads();
  double2 acc = make_double2(0, 0);
  int idx = threadIdx.x;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int u = 0; u < 8; u++) {
      double2 v = sm[(idx + u * 256) & (n - 1)];
      acc.x += v.x; acc.y += v.y;
    }
    idx += 1;
  }
  if (acc.x == 123.456) out[0] = acc.x + acc.y;
}
__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) b[i] = a[i];
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("{\"gpu\":\"%s\",\"sms\":%d,\"smem_per_block_optin\":%zu,\"smem_per_sm\":%zu,\"regs_per_sm\":%d,\"l2_bytes\":%d,\"mem_bytes\":%zu,\"clock_khz\":%d}\n",
         p.name, p.multiProcessorCount, p.sharedMemPerBlockOptin, p.sharedMemPerMultiprocessor, p.regsPerMultiprocessor, p.l2CacheSize, p.totalGlobalMem, p.clockRate);
  double* dout; CK(cudaMalloc(&dout, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  float ms;
  // DFMA
  for (int rep = 0; rep < 3; rep++) {
    int iters = 20000, blocks = sms * 4, threads = 256;
    cudaEventRecord(e0);
    dfma_kernel<8><<<blocks, threads>>>(dout, 0.999, 1e-3, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double fmas = (double)blocks * threads * iters * 8;
    printf("{\"bench\":\"dfma\",\"ms\":%.3f,\"dfma_per_s\":%.4e,\"dfma_per_clk_sm_at_1965\":%.2f}\n", ms, fmas / (ms * 1e-3), fmas / (ms * 1e-3) / (sms * 1.965e9));
  }
  for (int rep = 0; rep < 2; rep++) {
    int iters = 20000, blocks = sms * 4, threads = 256;
    cudaEventRecord(e0);
    ffma_kernel<8><<<blocks, threads>>>((float*)dout, 0.999f, 1e-3f, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double fmas = (double)blocks * threads * iters * 8;
    printf("{\"bench\":\"ffma\",\"ms\":%.3f,\"ffma_per_s\":%.4e,\"ffma_per_clk_sm_at_1965\":%.2f}\n", ms, fmas / (ms * 1e-3), fmas / (ms * 1e-3) / (sms * 1.965e9));
  }
  for (int rep = 0; rep < 2; rep++) {
    int iters = 20000, blocks = sms * 4, threads = 256;
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(dout, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double fmas = (double)blocks * (threads / 32) * iters * 4 * 256.0;
    printf("{\"bench\":\"dmma_m8n8k4\",\"ms\":%.3f,\"fma_per_s\":%.4e,\"tflops\":%.2f}\n", ms, fmas / (ms * 1e-3), 2 * fmas / (ms * 1e-3) / 1e12);
  }
  for (int rep = 0; rep < 2; rep++) {
    int iters = 20000, blocks = sms * 4, threads = 256;
    cudaEventRecord(e0);
    mixed_kernel<<<blocks, threads>>>(dout, iters, 0.999, 1e-3);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double mma_fmas = (double)blocks * (threads / 32) * iters * 4 * 256.0;
    double dfmas = (double)blocks * threads * iters * 32;
    printf("{\"bench\":\"dmma+dfma\",\"ms\":%.3f,\"total_fma_per_s\":%.4e,\"mma_share\":%.2f}\n", ms, (mma_fmas + dfmas) / (ms * 1e-3), mma_fmas / (mma_fmas + dfmas));
  }
  CK(cudaFuncSetAttribute(smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  for (int rep = 0; rep < 2; rep++) {
    int iters = 20000, blocks = sms * 3, threads = 256;
    cudaEventRecord(e0);
    smem_kernel<<<blocks, threads, 65536>>>(dout, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double bytes = (double)blocks * threads * iters * 8 * 16;
    printf("{\"bench\":\"smem_lds128\",\"ms\":%.3f,\"bytes_per_s\":%.4e,\"bytes_per_clk_sm_at_1965\":%.2f}\n", ms, bytes / (ms * 1e-3), bytes / (ms * 1e-3) / (sms * 1.965e9));
  }
  size_t n = (size_t)1 << 28;  // 4 GiB complex128
  double2 *a, *b; CK(cudaMalloc(&a, n * 16)); CK(cudaMalloc(&b, n * 16));
  cudaMemset(a, 0, n * 16); cudaMemset(b, 0, n * 16);
  for (int rep = 0; rep < 4; rep++) {
    cudaEventRecord(e0);
    copy_kernel<<<sms * 8, 512>>>(a, b, n);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"bench\":\"hbm_copy_c128\",\"ms\":%.3f,\"GBps_rw\":%.1f}\n", ms, 2.0 * n * 16 / (ms * 1e-3) / 1e9);
  }
  CK(cudaGetLastError());
  return 0;
}
