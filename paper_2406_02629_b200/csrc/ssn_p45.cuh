// ssn_p45.cuh -- arithmetic in the default field p = 2^45 - 55 (S/field.py:21) shared by the
// fused chain kernels and the specialised elementwise kernels: compile-time pseudo-Mersenne fold,
// lazy representatives below 2^46, and small-rational linear combinations (SRow).
#pragma once
#include <cstdint>
#include "ssn_field.cuh"
#include "ssn_lincomb.cuh"

namespace ssn45 {

template <int M>
struct SRow {            // sum_j n[j] x_j / D  (dinv = D^-1 mod p, one = (D == 1))
    uint32_t nn[M];      // n[j] + off >= 0 (< 2^14): sum_j n_j x_j = sum_j nn_j x_j - off * sum_j x_j
    uint32_t off;
    int32_t one;
    u64 dinv;
};

// ---- arithmetic in the default field p = 2^45 - 55 (S/field.py:21) with compile-time fold
constexpr int PS = 45;
constexpr u64 PC = 55;
constexpr u64 PP = (1ull << PS) - PC;
constexpr u64 PMASK = (1ull << PS) - 1;
constexpr u64 PHALF = (PP - 1) / 2;

// Intermediates are kept LAZY: any representative below 2^46 (not necessarily < p); only
// compared and stored values are canonicalised.
// lz: any x < 2^64 -> < 2^46, since (x >> 45) * 55 < 2^25.
// The fold multiplies q = x >> 45 (< 2^19) by 55 in ONE 32-bit IMAD and adds with an
// add/add-with-carry pair: the u64 form compiles to IMAD.WIDE, which occupies the FMA-heavy pipe
// (the chain kernels' bottleneck) twice as long.
__device__ __forceinline__ u64 lz(u64 x) {
    uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32);
    const uint32_t t = (hi >> (PS - 32)) * (uint32_t)PC;
    hi &= (1u << (PS - 32)) - 1;
    asm("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, %1, 0;" : "+r"(lo), "+r"(hi) : "r"(t));
    return ((u64)hi << 32) | lo;
}
// canon: x < 2^64 -> [0, p) ((x >> 45) * 55 + low < 2^45 + 2^25 < 2p)
__device__ __forceinline__ u64 canon(u64 x) {
    const u64 t = lz(x);
    return t >= PP ? t - PP : t;
}
__device__ __forceinline__ u64 red64(u64 x) { return canon(x); }
__device__ __forceinline__ u64 addm(u64 a, u64 b) {
    const u64 s = a + b;
    return s >= PP ? s - PP : s;
}
// a, b < 2^52 (a * b < 2^103): q = prod >> 45 < 2^58, q*55 + low < 2^64 -> lazy result
// Schoolbook on 32-bit halves: three 32x32->64 products for a, b < 2^52 (the middle pair summed
// in one u64, < 2^53) instead of the 64x64 low half plus __umul64hi.
__device__ __forceinline__ u64 mulm(u64 a, u64 b) {
    const uint32_t al = (uint32_t)a, ah = (uint32_t)(a >> 32), bl = (uint32_t)b, bh = (uint32_t)(b >> 32);
    const u64 p0 = (u64)al * bl;
    const u64 p1 = (u64)al * bh + (u64)ah * bl;
    const u64 p2 = (u64)ah * bh;
    const u64 lo = p0 + (p1 << 32);
    const u64 hi = p2 + (p1 >> 32) + (lo < p0);
    const u64 q = (hi << (64 - PS)) | (lo >> PS);
    return lz(q * PC + (lo & PMASK));
}
// mulm for a * b < 2^96 (e.g. a < 2^45 and b < 2^51, or both < 2^48): the product's top word
// fits 32 bits, so its partial products are three 32x32->64 multiplies and one 32-bit
// multiply-add-with-carry, and the fold is  (lo mod 2^45) + 55 (lo >> 45) + 55 * 2^19 * hi.
// Written in PTX: the C form compiled to ~30% more FMA-heavy pipe work (extra VIADD/IMAD.MOV).
template <bool FOLD = true>
__device__ __forceinline__ u64 mulm_hs(u64 a, u64 b) {
    const uint32_t al = (uint32_t)a, ah = (uint32_t)(a >> 32), bl = (uint32_t)b, bh = (uint32_t)(b >> 32);
    uint32_t lo_lo, lo_hi, hi;
    asm("{\n\t.reg .u32 p0l, p0h, p1l, p1h, p2;\n\t.reg .u64 p0, p1;\n\t"
        "mul.wide.u32 p0, %3, %5;\n\t"
        "mul.wide.u32 p1, %3, %6;\n\t"
        "mad.wide.u32 p1, %4, %5, p1;\n\t"
        "mul.lo.u32 p2, %4, %6;\n\t"
        "mov.b64 {p0l, p0h}, p0;\n\t"
        "mov.b64 {p1l, p1h}, p1;\n\t"
        "mov.u32 %0, p0l;\n\t"
        "add.cc.u32 %1, p0h, p1l;\n\t"
        "addc.u32 %2, p1h, p2;\n\t}"
        : "=r"(lo_lo), "=r"(lo_hi), "=r"(hi)
        : "r"(al), "r"(ah), "r"(bl), "r"(bh));
    const uint32_t t1 = (lo_hi >> (PS - 32)) * (uint32_t)PC;                 // 55 (lo >> 45) < 2^25
    const u64 t2 = (u64)hi * (PC << (64 - PS));                             // 55 2^19 hi < 2^57
    const u64 low = ((u64)(lo_hi & ((1u << (PS - 32)) - 1)) << 32) | lo_lo;  // lo mod 2^45
    // FOLD = false: the unreduced low + t1 + t2 < 2^45 + 2^25 + 55 * 2^19 * (a * b >> 64),
    // e.g. below 2^56 for a * b < 2^95
    if constexpr (!FOLD) return low + t1 + t2;
    return lz(low + t1 + t2);
}

// a * b mod p (lazy) for a < 2^64 / b < 2^32 with a * b < 2^96: two 32x32->64 multiplies, the
// mulm_hs fold
__device__ __forceinline__ u64 mulm_s32(u64 a, uint32_t b) {
    const uint32_t al = (uint32_t)a, ah = (uint32_t)(a >> 32);
    uint32_t lo_lo, lo_hi, hi;
    asm("{\n\t.reg .u32 p0l, p0h, p1l, p1h;\n\t.reg .u64 p0, p1;\n\t"
        "mul.wide.u32 p0, %3, %5;\n\t"
        "mul.wide.u32 p1, %4, %5;\n\t"
        "mov.b64 {p0l, p0h}, p0;\n\t"
        "mov.b64 {p1l, p1h}, p1;\n\t"
        "mov.u32 %0, p0l;\n\t"
        "add.cc.u32 %1, p0h, p1l;\n\t"
        "addc.u32 %2, p1h, 0;\n\t}"
        : "=r"(lo_lo), "=r"(lo_hi), "=r"(hi)
        : "r"(al), "r"(ah), "r"(b));
    const uint32_t t1 = (lo_hi >> (PS - 32)) * (uint32_t)PC;
    const u64 t2 = (u64)hi * (PC << (64 - PS));
    const u64 low = ((u64)(lo_hi & ((1u << (PS - 32)) - 1)) << 32) | lo_lo;
    return lz(low + t1 + t2);
}

// sum_j n_j x_j / D for lazy x_j (< 2^46), |n_j| < 2^13, M <= 7.  With non-negative
// nn_j = n_j + off the products split into 32-bit halves: sum nn_j lo_j (< 2^49, one
// IMAD.WIDE each) + (sum nn_j hi_j) << 32 (hi < 2^14, < 2^31) -- then subtract off * sum x_j.
template <int M>
__device__ __forceinline__ u64 lin_s(const u64 (&x)[M], u64 xsum, const SRow<M> &r) {
    u64 lo = 0;
    uint32_t hi = 0;
#pragma unroll
    for (int j = 0; j < M; j++) {
        lo += (u64)(uint32_t)x[j] * r.nn[j];
        hi += (uint32_t)(x[j] >> 32) * r.nn[j];
    }
    // pos < M * 2^60 <= 7 * 2^60 < 2^63 and neg < 2^62 < 2^18 * p, so pos + 2^18 p - neg is a
    // non-negative u64 below 2^64: ONE fold for the whole signed combination
    const u64 pos = lo + ((u64)hi << 32);
    const u64 neg = mul_small(xsum, r.off);
    const u64 v = lz(pos + (PP << 18) - neg);            // < 2^46
    return r.one ? v : mulm(v, r.dinv);
}
template <int M>
__device__ __forceinline__ u64 xsum_of(const u64 (&x)[M]) {
    u64 s = 0;
#pragma unroll
    for (int j = 0; j < M; j++) s += x[j];
    return s;
}
template <int M>
__device__ __forceinline__ u64 lin(const u64 (&x)[M], const SRow<M> &r) {
    return lin_s<M>(x, xsum_of<M>(x), r);
}

template <int MM>
static int make_srow(SRow<MM> &s, const u64 *w, int m, u64 p) {
    LinRow r;
    u64 row[SSN_MAXJ] = {0};
    for (int j = 0; j < m; j++) row[j] = w[j];
    const int ok = make_row(r, row, m, p);
    int32_t off = 0;
    for (int j = 0; j < m; j++)
        if (-r.n[j] > off) off = -r.n[j];
    for (int j = 0; j < MM; j++) s.nn[j] = j < m ? (uint32_t)(r.n[j] + off) : 0;
    s.off = (uint32_t)off;
    s.one = r.one;
    s.dinv = r.dinv;
    return ok;
}

}  // namespace ssn45
