// hs_f2.cuh -- packed FP32x2 complex arithmetic (FFMA2, sm_100a).
//
// A complex value lives in one 64-bit register pair (re, im).  The complex
// multiply-accumulate acc += v * x with v given as two scalars is two FFMA2:
//
//   acc += (vr, vr) * (xr, xi)          FFMA2 acc, vr.F32, x, acc
//   acc += (-xi, xr) * (vi, vi)         FFMA2 acc, -x.LO_HI.NP, vi.F32, acc
//
// ptxas folds the scalar broadcast (.F32), the half swap (.LO_HI) and the
// low-half negation (.NP) into the instruction, so a complex MAC costs two
// issue slots instead of four FFMA (same FMA-pipe work, half the issue
// pressure; tools/ffma2_probe.cu: 68 TFLOP/s with a broadcast operand).
// Each lane computes fmaf(a, b, c) exactly (round-to-nearest), so results
// equal the scalar FFMA formulation with the same operation order.
#pragma once

#include <stdint.h>

namespace hs {

typedef unsigned long long f2x;

__device__ __forceinline__ f2x f2_pack(float lo, float hi)
{
    f2x r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}

__device__ __forceinline__ float f2_lo(f2x v)
{
    float lo;
    asm("{ .reg .f32 t;\n mov.b64 {%0, t}, %1; }" : "=f"(lo) : "l"(v));
    return lo;
}

__device__ __forceinline__ float f2_hi(f2x v)
{
    float hi;
    asm("{ .reg .f32 t;\n mov.b64 {t, %0}, %1; }" : "=f"(hi) : "l"(v));
    return hi;
}

__device__ __forceinline__ void f2_fma(f2x &acc, f2x a, f2x b)
{
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(a), "l"(b));
}

// acc += (vr + i vi) * x
__device__ __forceinline__ void f2_cmac(f2x &acc, float vr, float vi, f2x x)
{
    float xl, xh;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(xl), "=f"(xh) : "l"(x));
    f2_fma(acc, f2_pack(vr, vr), x);
    f2_fma(acc, f2_pack(-xh, xl), f2_pack(vi, vi));
}

// The same complex MAC as one asm statement: the broadcast packs and the
// swapped, negated x live inside the statement, so the compiler cannot
// hoist or share them across MACs as materialised register pairs (which
// costs moves and registers); ptxas folds them into the two FFMA2.
__device__ __forceinline__ void f2_cmac1(f2x &acc, float vr, float vi, f2x x)
{
    asm("{\n .reg .b64 vv, ww, xs;\n .reg .f32 xl, xh;\n"
        " mov.b64 vv, {%1, %1};\n"
        " fma.rn.f32x2 %0, vv, %3, %0;\n"
        " mov.b64 {xl, xh}, %3;\n"
        " neg.f32 xh, xh;\n"
        " mov.b64 xs, {xh, xl};\n"
        " mov.b64 ww, {%2, %2};\n"
        " fma.rn.f32x2 %0, xs, ww, %0;\n}"
        : "+l"(acc)
        : "f"(vr), "f"(vi), "l"(x));
}

}  // namespace hs
