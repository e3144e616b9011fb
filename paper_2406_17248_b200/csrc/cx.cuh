// cx.cuh — complex128 helpers on double2 (re, im) shared by the kernels.
#pragma once
#include <cuda_runtime.h>

namespace sv {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a*b + c
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c) {
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}
// Re(conj(a) * b)
__device__ __forceinline__ double re_conj_mul(double2 a, double2 b) { return fma(a.x, b.x, a.y * b.y); }

__device__ __forceinline__ double2 csel(bool c, double2 a, double2 b) { return c ? a : b; }

}  // namespace sv
