// Counter-based noise for the EnSF particles, regenerated in registers.
//
// The reference draws particle noise from RngStream(seed, ensf_particles,
// (cycle << 32) | i) (proj/src/ensf.cpp:174-175): Philox4x32-10 blocks
// (proj/src/rng.cpp:8-31) turned into 53-bit uniforms (rng.cpp:67-70) and
// Box-Muller pairs whose sin half is cached (rng.cpp:72-84).  Because the
// stream is a pure function of its position, normal #n of particle i is
// half of the pair built from Philox block n >> 1: even n -> r cos a,
// odd n -> r sin a.  The kernels therefore never touch a host noise buffer;
// they evaluate the block for (entity, n >> 1) on the spot.
#pragma once
#include <cstdint>

#include "philox_keys.h"

namespace tb200 {

struct PhiloxOut {
    uint32_t w0, w1, w2, w3;
};

// Philox4x32-10 of counter (q_lo, q_hi, e_lo, e_hi) under key (k0, k1).
__device__ __forceinline__ PhiloxOut philox_block(uint64_t q, uint32_t e_lo, uint32_t e_hi,
                                                  uint32_t k0, uint32_t k1) {
    uint32_t c0 = uint32_t(q), c1 = uint32_t(q >> 32), c2 = e_lo, c3 = e_hi;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        // one IMAD.WIDE.U32 per product yields both halves
        const uint64_t p0 = uint64_t(c0) * 0xD2511F53u;
        const uint64_t p1 = uint64_t(c2) * 0xCD9E8D57u;
        c0 = uint32_t(p1 >> 32) ^ c1 ^ k0;
        c2 = uint32_t(p0 >> 32) ^ c3 ^ k1;
        c1 = uint32_t(p1);
        c3 = uint32_t(p0);
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return {c0, c1, c2, c3};
}

__device__ __forceinline__ PhiloxOut philox_block_rk(uint64_t q, uint32_t e_lo, uint32_t e_hi,
                                                     const PhiloxKeys& rk) {
    uint32_t c0 = uint32_t(q), c1 = uint32_t(q >> 32), c2 = e_lo, c3 = e_hi;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = uint64_t(c0) * 0xD2511F53u;
        const uint64_t p1 = uint64_t(c2) * 0xCD9E8D57u;
        c0 = uint32_t(p1 >> 32) ^ c1 ^ rk.k[2 * r];
        c2 = uint32_t(p0 >> 32) ^ c3 ^ rk.k[2 * r + 1];
        c1 = uint32_t(p1);
        c3 = uint32_t(p0);
    }
    return {c0, c1, c2, c3};
}

// --- fp64: bit-level restatement of RngStream::uniform / normal ------------
__device__ __forceinline__ double u53(uint32_t lo, uint32_t hi) {
    const uint64_t v = uint64_t(lo) | (uint64_t(hi) << 32);
    return (double(v >> 11) + 0.5) * 0x1.0p-53;
}

__device__ __forceinline__ void box_muller_f64(const PhiloxOut& w, double& c, double& s) {
    const double u1 = u53(w.w0, w.w1);
    const double u2 = u53(w.w2, w.w3);
    const double r = sqrt(-2.0 * log(u1));
    const double a = 2.0 * 3.14159265358979323846 * u2;
    double sa, ca;
    sincos(a, &sa, &ca);
    c = r * ca;
    s = r * sa;
}

// --- fp32 fast path --------------------------------------------------------
// u1 keeps ~46 significant bits before the final fp32 rounding, so -2 ln u1
// is accurate to fp32 precision even for tiny u1; built from mantissa bit
// tricks so it stays on the FMA/ALU pipes (no I2F).
__device__ __forceinline__ float u1_f32(uint32_t lo, uint32_t hi) {
    const float a = __uint_as_float(0x3F800000u | (hi >> 9)) - 1.0f;              // bits 63..41
    const float b = __uint_as_float(0x3F800000u | ((hi & 0x1FFu) << 14) | (lo >> 18)) - 1.0f;  // 40..18
    return fmaf(b, 0x1.0p-23f, a + 0x1.0p-54f);
}

__device__ __forceinline__ float u2_f32(uint32_t hi) {
    // 23 leading bits + half-ulp offset; MUFU sin/cos limits accuracy anyway
    return (__uint_as_float(0x3F800000u | (hi >> 9)) - 1.0f) + 0x1.0p-24f;
}

__device__ __forceinline__ float2 box_muller_f32(const PhiloxOut& w) {
    const float u1 = u1_f32(w.w0, w.w1);
    const float u2 = u2_f32(w.w3);
    // -2 ln u1 = -2 ln2 * log2(u1); MUFU.SQRT (no IEEE slow path)
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(-1.3862943611198906f * __log2f(u1)));
    float s, c;
    __sincosf(6.283185307179586f * u2, &s, &c);
    return make_float2(r * c, r * s);
}

// Normals #n0 and #n0+1 of one particle stream.  When n0 is even they are
// the (cos, sin) pair of a single block; when odd they straddle two blocks.
__device__ __forceinline__ float2 normal_pair_f32(uint64_t n0, uint32_t e_lo, uint32_t e_hi,
                                                  uint32_t k0, uint32_t k1) {
    if ((n0 & 1u) == 0) return box_muller_f32(philox_block(n0 >> 1, e_lo, e_hi, k0, k1));
    const float2 a = box_muller_f32(philox_block(n0 >> 1, e_lo, e_hi, k0, k1));
    const float2 b = box_muller_f32(philox_block((n0 >> 1) + 1, e_lo, e_hi, k0, k1));
    return make_float2(a.y, b.x);
}

__device__ __forceinline__ float2 normal_pair_f32(uint64_t n0, uint32_t e_lo, uint32_t e_hi,
                                                  const PhiloxKeys& rk) {
    if ((n0 & 1u) == 0) return box_muller_f32(philox_block_rk(n0 >> 1, e_lo, e_hi, rk));
    const float2 a = box_muller_f32(philox_block_rk(n0 >> 1, e_lo, e_hi, rk));
    const float2 b = box_muller_f32(philox_block_rk((n0 >> 1) + 1, e_lo, e_hi, rk));
    return make_float2(a.y, b.x);
}

__device__ __forceinline__ double2 normal_pair_f64(uint64_t n0, uint32_t e_lo, uint32_t e_hi,
                                                   uint32_t k0, uint32_t k1) {
    double c, s;
    box_muller_f64(philox_block(n0 >> 1, e_lo, e_hi, k0, k1), c, s);
    if ((n0 & 1u) == 0) return make_double2(c, s);
    double c2, s2;
    box_muller_f64(philox_block((n0 >> 1) + 1, e_lo, e_hi, k0, k1), c2, s2);
    return make_double2(s, c2);
}

__device__ __forceinline__ double normal_f64(uint64_t n, uint32_t e_lo, uint32_t e_hi,
                                             uint32_t k0, uint32_t k1) {
    double c, s;
    box_muller_f64(philox_block(n >> 1, e_lo, e_hi, k0, k1), c, s);
    return (n & 1u) ? s : c;
}

}  // namespace tb200
