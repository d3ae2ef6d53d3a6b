// cx2.cuh — packed complex FP32 arithmetic on the sm_100a f32x2 instructions.
//
// A complex value lives in one 64-bit register pair (re = low half, im = high half), and
// `fma.rn.f32x2` / `add.rn.f32x2` / `mul.rn.f32x2` (SASS FFMA2/FADD2/FMUL2) operate on both
// halves in one issue slot.  FFMA2 accepts a scalar operand broadcast to both halves
// (`R.F32`) and half swizzles, so a complex multiply-add a·b + c with b pre-split into
// (b, j·b) is two FFMA2:  c + re(a)·b + im(a)·(j·b).  The FP32 pipe rate is unchanged
// (measured: FFMA 70.4, FFMA2 67.5 TFLOP/s on one B200, tools/microbench.cu); what it buys
// is issue slots, the limiter of the demod kernel (ncu: issue slots 85% busy).
#pragma once

#include <cuda_runtime.h>

namespace bos {

typedef unsigned long long cx2;

__device__ __forceinline__ cx2 cx2_make(float re, float im) {
    cx2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(re), "f"(im));
    return r;
}
__device__ __forceinline__ float cx2_re(cx2 a) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a));
    return lo;
}
__device__ __forceinline__ float cx2_im(cx2 a) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a));
    return hi;
}
__device__ __forceinline__ float2 cx2_f2(cx2 a) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a));
    return make_float2(lo, hi);
}
__device__ __forceinline__ cx2 f2_cx2(float2 a) { return cx2_make(a.x, a.y); }
__device__ __forceinline__ cx2 cx2_bcast(float s) { return cx2_make(s, s); }

__device__ __forceinline__ cx2 fma2(cx2 a, cx2 b, cx2 c) {
    cx2 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ cx2 add2(cx2 a, cx2 b) {
    cx2 d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ cx2 sub2(cx2 a, cx2 b) {
    cx2 d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ cx2 mul2(cx2 a, cx2 b) {
    cx2 d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
// j·b = (−im b, re b)
__device__ __forceinline__ cx2 cx2_jmul(cx2 b) { return cx2_make(-cx2_im(b), cx2_re(b)); }
// complex a·b + c, with bj = j·b precomputed (two FFMA2)
__device__ __forceinline__ cx2 cmad2(cx2 a, cx2 b, cx2 bj, cx2 c) {
    return fma2(cx2_bcast(cx2_re(a)), b, fma2(cx2_bcast(cx2_im(a)), bj, c));
}
__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

}  // namespace bos
