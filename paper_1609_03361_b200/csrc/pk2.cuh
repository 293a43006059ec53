// pk2.cuh — packed fp32x2 arithmetic for the vector stencil kernels (sm_100a).
//
// Blackwell issues FMUL2 / FFMA2: one instruction, two independent IEEE fp32
// operations on a 64-bit register pair, each rounded exactly like the scalar
// FMUL / FADD. The FP32 pipe does the same number of operations per clock
// either way (tools/f32x2_probe.cu measured 37 Tops/s for both at 1965 MHz),
// but every packed instruction takes ONE issue slot for two operations. The
// stencils carry four consecutive a2 points per lane, i.e. two pairs, so the
// reference's exact operation sequence can run at half the issue cost; the
// shared-memory loads, queue moves and barriers then share the freed slots.
//
// Rounding contract (kernels must stay bitwise equal to the reference's
// -ffp-contract=off C): ptxas contracts `mul.rn.f32x2` feeding
// `add.rn.f32x2` into FFMA2 even under --fmad=false. So products are
// `mul.rn.f32x2` and sums are `fma.rn.f32x2(a, ONE, b)` with ONE = (1.0f,
// 1.0f) held in a kernel parameter: ptxas cannot prove it is 1.0, so it can
// neither fold the product into it nor rewrite the sum. a*1 + b is exact in
// the product and rounds once, exactly like a + b (checked bitwise on 2^25
// random pairs including NaN/inf/denormals by the probe; the stencil parity
// tests check the kernels end to end).
#pragma once

#include <cstdint>

namespace sfb {

typedef unsigned long long f2;  // .x in the low word, .y in the high word

__host__ __device__ inline f2 f2_splat_host(float v) {
    uint32_t b;
    __builtin_memcpy(&b, &v, 4);
    return (static_cast<f2>(b) << 32) | b;
}

__device__ __forceinline__ f2 pk(float lo, float hi) {
    f2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}

__device__ __forceinline__ void upk(f2 v, float& lo, float& hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}

__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
    f2 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}

// a + b, rounded once (see the contract above; `one` must be the opaque
// (1.0f, 1.0f) parameter)
__device__ __forceinline__ f2 add2(f2 a, f2 b, f2 one) {
    f2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(one), "l"(b));
    return r;
}

// acc + k * v with two roundings (the reference's `acc + k*v` term)
__device__ __forceinline__ f2 mac2(f2 acc, f2 k, f2 v, f2 one) {
    return add2(acc, mul2(k, v), one);
}

// 16-byte shared/global load as two pairs (LDS.128 / LDG.128)
__device__ __forceinline__ ulonglong2 ld2x2(const float* p) {
    return *reinterpret_cast<const ulonglong2*>(p);
}

__device__ __forceinline__ ulonglong2 ldg2x2(const float* p) {
    return __ldg(reinterpret_cast<const ulonglong2*>(p));
}

} // namespace sfb
