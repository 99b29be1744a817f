// Packed float32 pairs for the FFMA2 / FMUL2 / FADD2 instructions of sm_100a.
//
// A pair lives in ONE 64-bit register (PTX .b64) so the compiler keeps it in an
// aligned register pair for its whole lifetime; the float2 intrinsics let it
// re-assemble pairs from scalars at every use (a MOV per operand). Packed ops
// round each lane exactly like the scalar fma.rn / mul.rn / add.rn, so a pair
// of cells computes bit-for-bit what the scalar code computes for each.
#pragma once

typedef unsigned long long wl2;

__device__ __forceinline__ wl2 wl_pk(float lo, float hi) {
    wl2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
// The same pair, produced by an arithmetic instruction (x + -0 = x for every
// x, signed zeros included): ptxas otherwise re-assembles a pair from its two
// scalar halves with two MOVs before EVERY use (it prefers re-materialising to
// keeping both the scalars and the pair live). Use for pairs read many times.
__device__ __forceinline__ wl2 wl_pk_keep(float lo, float hi) {
    wl2 r;
    asm volatile(
        "{\n\t.reg .b64 t, z;\n\t"
        "mov.b64 t, {%1, %2};\n\t"
        "mov.b64 z, 0x8000000080000000;\n\t"
        "add.rn.f32x2 %0, t, z;\n\t}"
        : "=l"(r)
        : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ float wl_lo(wl2 p) {
    float lo;
    asm("{\n\t.reg .b32 h;\n\tmov.b64 {%0, h}, %1;\n\t}" : "=f"(lo) : "l"(p));
    return lo;
}
__device__ __forceinline__ float wl_hi(wl2 p) {
    float hi;
    asm("{\n\t.reg .b32 l;\n\tmov.b64 {l, %0}, %1;\n\t}" : "=f"(hi) : "l"(p));
    return hi;
}
// c * x + acc per lane, c broadcast (folds to the immediate form of FFMA2)
__device__ __forceinline__ wl2 wl_fma2(float c, wl2 x, wl2 acc) {
    wl2 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(x), "l"(wl_pk(c, c)), "l"(acc));
    return d;
}
__device__ __forceinline__ wl2 wl_mul2(float c, wl2 x) {
    wl2 d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(x), "l"(wl_pk(c, c)));
    return d;
}
__device__ __forceinline__ wl2 wl_add2(wl2 a, wl2 b) {
    wl2 d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
