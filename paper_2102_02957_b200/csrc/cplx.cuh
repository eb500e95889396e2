// cplx.cuh — complex double2 / float2 helpers shared by the device kernels.
#pragma once
#ifndef __CUDACC_RTC__
#include <cuda_runtime.h>
#endif

namespace sv {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}

// In-place register updates written in PTX with tied operands: the results land in the input
// registers, so a register-resident amplitude array needs no moves after the op (ptxas otherwise
// allocates fresh registers and copies them back at every dynamic-dispatch merge point).
// v <- v * f, same rounding as cmul(v, f).
__device__ __forceinline__ void cmul_ip(double2& v, double2 f) {
  asm("{\n\t.reg .f64 t1, t2;\n\t"
      "mul.f64 t1, %1, %3;\n\t"
      "mul.f64 t2, %1, %2;\n\t"
      "fma.rn.f64 %1, %0, %3, t2;\n\t"
      "neg.f64 t1, t1;\n\t"
      "fma.rn.f64 %0, %0, %2, t1;\n\t}"
      : "+d"(v.x), "+d"(v.y)
      : "d"(f.x), "d"(f.y));
}
__device__ __forceinline__ void cmul_ip(float2& v, float2 f) {
  asm("{\n\t.reg .f32 t1, t2;\n\t"
      "mul.f32 t1, %1, %3;\n\t"
      "mul.f32 t2, %1, %2;\n\t"
      "fma.rn.f32 %1, %0, %3, t2;\n\t"
      "neg.f32 t1, t1;\n\t"
      "fma.rn.f32 %0, %0, %2, t1;\n\t}"
      : "+f"(v.x), "+f"(v.y)
      : "f"(f.x), "f"(f.y));
}
// (a, b) <- (a + b, a - b)
__device__ __forceinline__ void hu_ip(double2& a, double2& b) {
  asm("{\n\t.reg .f64 t1, t2;\n\t"
      "sub.f64 t1, %0, %2;\n\t"
      "sub.f64 t2, %1, %3;\n\t"
      "add.f64 %0, %0, %2;\n\t"
      "add.f64 %1, %1, %3;\n\t"
      "mov.f64 %2, t1;\n\t"
      "mov.f64 %3, t2;\n\t}"
      : "+d"(a.x), "+d"(a.y), "+d"(b.x), "+d"(b.y));
}
__device__ __forceinline__ void hu_ip(float2& a, float2& b) {
  asm("{\n\t.reg .f32 t1, t2;\n\t"
      "sub.f32 t1, %0, %2;\n\t"
      "sub.f32 t2, %1, %3;\n\t"
      "add.f32 %0, %0, %2;\n\t"
      "add.f32 %1, %1, %3;\n\t"
      "mov.f32 %2, t1;\n\t"
      "mov.f32 %3, t2;\n\t}"
      : "+f"(a.x), "+f"(a.y), "+f"(b.x), "+f"(b.y));
}
// (a, b) <- (s (a + b), s (a - b))
__device__ __forceinline__ void h_ip(double2& a, double2& b, double s) {
  asm("{\n\t.reg .f64 t1, t2;\n\t"
      "sub.f64 t1, %0, %2;\n\t"
      "sub.f64 t2, %1, %3;\n\t"
      "add.f64 %0, %0, %2;\n\t"
      "add.f64 %1, %1, %3;\n\t"
      "mul.f64 %0, %0, %4;\n\t"
      "mul.f64 %1, %1, %4;\n\t"
      "mul.f64 %2, t1, %4;\n\t"
      "mul.f64 %3, t2, %4;\n\t}"
      : "+d"(a.x), "+d"(a.y), "+d"(b.x), "+d"(b.y)
      : "d"(s));
}
__device__ __forceinline__ void h_ip(float2& a, float2& b, float s) {
  asm("{\n\t.reg .f32 t1, t2;\n\t"
      "sub.f32 t1, %0, %2;\n\t"
      "sub.f32 t2, %1, %3;\n\t"
      "add.f32 %0, %0, %2;\n\t"
      "add.f32 %1, %1, %3;\n\t"
      "mul.f32 %0, %0, %4;\n\t"
      "mul.f32 %1, %1, %4;\n\t"
      "mul.f32 %2, t1, %4;\n\t"
      "mul.f32 %3, t2, %4;\n\t}"
      : "+f"(a.x), "+f"(a.y), "+f"(b.x), "+f"(b.y)
      : "f"(s));
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
