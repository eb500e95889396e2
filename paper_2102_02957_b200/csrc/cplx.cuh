// cplx.cuh — complex double2 / float2 helpers shared by the device kernels.
#pragma once
#include <cuda_runtime.h>

namespace sv {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
// acc + m * a
__device__ __forceinline__ double2 cfma(double2 m, double2 a, double2 acc) {
  acc.x = fma(m.x, a.x, acc.x);
  acc.x = fma(-m.y, a.y, acc.x);
  acc.y = fma(m.x, a.y, acc.y);
  acc.y = fma(m.y, a.x, acc.y);
  return acc;
}
__device__ __forceinline__ float2 cfma(float2 m, float2 a, float2 acc) {
  acc.x = fmaf(m.x, a.x, acc.x);
  acc.x = fmaf(-m.y, a.y, acc.x);
  acc.y = fmaf(m.x, a.y, acc.y);
  acc.y = fmaf(m.y, a.x, acc.y);
  return acc;
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
__device__ __forceinline__ double abs2(double2 a) { return fma(a.x, a.x, a.y * a.y); }
__device__ __forceinline__ double abs2(float2 a) { return (double)a.x * a.x + (double)a.y * a.y; }
template <typename V> __device__ __forceinline__ V czero();
template <> __device__ __forceinline__ double2 czero<double2>() { return make_double2(0.0, 0.0); }
template <> __device__ __forceinline__ float2 czero<float2>() { return make_float2(0.f, 0.f); }
template <typename V> __device__ __forceinline__ V cone();
template <> __device__ __forceinline__ double2 cone<double2>() { return make_double2(1.0, 0.0); }
template <> __device__ __forceinline__ float2 cone<float2>() { return make_float2(1.f, 0.f); }

template <typename V>
__device__ __forceinline__ V sel4(int s, V a0, V a1, V a2, V a3) {
  return s == 0 ? a0 : (s == 1 ? a1 : (s == 2 ? a2 : a3));
}

}  // namespace sv
