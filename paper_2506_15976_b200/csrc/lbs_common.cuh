// Shared device helpers for the lbscan_b200 kernels (sm_100a only).
#pragma once
#include <type_traits>

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/lbscan_b200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "lbscan_b200 targets sm_100a (B200) only"
#endif

namespace lbs {

constexpr float kLog2e = 1.4426950408889634f;

// ---------------------------------------------------------------------------
// packed fp32x2 arithmetic: FFMA2 / FMUL2 / FADD2 on sm_100a (two lanes of
// state per instruction — the scan's FP32 pipe work is paired over n).
struct __align__(8) f2 {
  float x, y;
};

__device__ __forceinline__ f2 mk2(float a, float b) { return f2{a, b}; }
__device__ __forceinline__ f2 bc2(float a) { return f2{a, a}; }

__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
  f2 r;
  asm("{.reg .b64 ra,rb,rc,rd;\n\t"
      "mov.b64 ra,{%2,%3}; mov.b64 rb,{%4,%5}; mov.b64 rc,{%6,%7};\n\t"
      "fma.rn.f32x2 rd,ra,rb,rc; mov.b64 {%0,%1},rd;}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return r;
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
  f2 r;
  asm("{.reg .b64 ra,rb,rd;\n\t"
      "mov.b64 ra,{%2,%3}; mov.b64 rb,{%4,%5};\n\t"
      "mul.rn.f32x2 rd,ra,rb; mov.b64 {%0,%1},rd;}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
__device__ __forceinline__ f2 add2(f2 a, f2 b) {
  f2 r;
  asm("{.reg .b64 ra,rb,rd;\n\t"
      "mov.b64 ra,{%2,%3}; mov.b64 rb,{%4,%5};\n\t"
      "add.rn.f32x2 rd,ra,rb; mov.b64 {%0,%1},rd;}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}

// MUFU.EX2 (2^x, ftz); rel. error ~2^-22
__device__ __forceinline__ float ex2(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float lg2(float x) {
  float r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float rcp(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// softplus(x) = log(1 + e^x)  (nn.py:21-22); 2 MUFU, exact-enough fp32
__device__ __forceinline__ float softplus_f(float x) {
  float t = ex2(x * kLog2e);
  float s = lg2(1.0f + t) * (1.0f / kLog2e);
  s = (x > 15.0f) ? x : s;
  return (x < -15.0f) ? t : s;
}
// sigmoid(x) = 1 / (1 + e^-x); silu(x) = x * sigmoid(x)  (nn.py:16-26)
// (a MUFU-free Newton reciprocal measured 1-13 % slower in the scan and the conv)
__device__ __forceinline__ float sigmoid_f(float x) { return rcp(1.0f + ex2(-x * kLog2e)); }
__device__ __forceinline__ float silu_f(float x) { return x * sigmoid_f(x); }
// SiLU of a value that is stored as T (the gate at the output store).  A one-MUFU
// form, 0.5 + 0.5 tanh.approx(x/2) for 16-bit outputs, measured 2.6 % faster in the
// LBVim-Ti layer; not kept for its absolute error near z << 0 (2^-11 |z| / 2)
// (profiles/r02_fwd_experiments.txt, vb3 tanh).
template <typename T>
__device__ __forceinline__ float silu_out(float x) {
  return silu_f(x);
}

// ---------------------------------------------------------------------------
// typed loads / stores (fp32 compute, io in fp32 / bf16 / fp16)
template <typename T>
__device__ __forceinline__ float ld(const T* p);
template <>
__device__ __forceinline__ float ld<float>(const float* p) { return __ldg(p); }
template <>
__device__ __forceinline__ float ld<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat162float(__ldg(p));
}
template <>
__device__ __forceinline__ float ld<__half>(const __half* p) { return __half2float(__ldg(p)); }

__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
__device__ __forceinline__ float to_f(__half x) { return __half2float(x); }

template <typename T>
__device__ __forceinline__ T from_f(float v) {
  if constexpr (sizeof(T) == 4) return v;
  else if constexpr (std::is_same<T, __nv_bfloat16>::value) return __float2bfloat16_rn(v);
  else return __float2half_rn(v);
}

template <typename T>
__device__ __forceinline__ void st(T* p, float v);
template <>
__device__ __forceinline__ void st<float>(float* p, float v) { *p = v; }
template <>
__device__ __forceinline__ void st<__nv_bfloat16>(__nv_bfloat16* p, float v) {
  *p = __float2bfloat16_rn(v);
}
template <>
__device__ __forceinline__ void st<__half>(__half* p, float v) { *p = __float2half_rn(v); }

}  // namespace lbs
