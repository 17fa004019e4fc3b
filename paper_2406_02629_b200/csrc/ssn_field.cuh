// ssn_field.cuh -- prime-field arithmetic and counter-based randomness on sm_100a.
//
// Field elements are canonical uint64 in [0, p), p < 2^62 (the reference caps p at 57
// bits, S/field.py:64-75).  Two exact reductions of the 128-bit product:
//   * pseudo-Mersenne fold for p = 2^s - c with small c and s <= 50 (the default
//     p = 2^45 - 55, S/field.py:21): x = q*2^s + r == q*c + r, folded twice;
//   * Barrett for any other p (e.g. the F_11 worked examples of the reference tests).
// The choice is a warp-uniform branch on SsnField::pm.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

typedef uint64_t u64;
typedef int64_t i64;
typedef uint32_t u32;

struct SsnField {
    u64 p;      // modulus
    u64 mu;     // floor(2^(2s) / p)            (Barrett)
    u64 c;      // 2^s - p                        (pseudo-Mersenne)
    u64 mask;   // 2^s - 1
    u64 half;   // (p-1)/2, signed decode threshold (S/field.py:74)
    int s;      // bit length of p
    int pm;     // 1: use the pseudo-Mersenne fold
    int near;   // 1: 2^s - p < 2^(s-24): uniform draws by masking (stat. distance < 2^-24)
};

static inline SsnField ssn_make_field(u64 p) {
    SsnField f;
    f.p = p;
    int s = 0;
    while (s < 64 && (p >> s)) s++;
    f.s = s;
    unsigned __int128 num = ((unsigned __int128)1) << (2 * s);
    f.mu = (u64)(num / p);
    f.mask = (s >= 64) ? ~0ull : ((1ull << s) - 1);
    f.c = f.mask + 1 - p;
    f.half = (p - 1) / 2;
    f.pm = (s >= 24 && s <= 50 && f.c < (1ull << 12)) ? 1 : 0;
    f.near = (s >= 32 && f.c < (1ull << (s - 24))) ? 1 : 0;
    return f;
}

#ifdef __CUDACC__
__device__ __forceinline__ u64 ssn_addmod(u64 a, u64 b, u64 p) {
    u64 s = a + b;
    return s >= p ? s - p : s;
}
__device__ __forceinline__ u64 ssn_submod(u64 a, u64 b, u64 p) {
    return a >= b ? a - b : a + (p - b);
}

// Barrett reduction of x = hi*2^64 + lo < 2^(2s).
__device__ __forceinline__ u64 ssn_barrett(u64 hi, u64 lo, const SsnField &f) {
    const int s = f.s;
    u64 q1 = (hi << (65 - s)) | (lo >> (s - 1));          // x >> (s-1), < 2^(s+1)
    u64 q2lo = q1 * f.mu, q2hi = __umul64hi(q1, f.mu);
    u64 q3 = (q2hi << (63 - s)) | (q2lo >> (s + 1));       // (q1*mu) >> (s+1)
    u64 r = lo - q3 * f.p;                                 // true r < 3p
    if (r >= f.p) r -= f.p;
    if (r >= f.p) r -= f.p;
    return r;
}

// Pseudo-Mersenne fold of x = hi*2^64 + lo < 2^(2s), s <= 50, c < 2^12.
__device__ __forceinline__ u64 ssn_pmfold(u64 hi, u64 lo, const SsnField &f) {
    const int s = f.s;
    u64 q = (hi << (64 - s)) | (lo >> s);                  // < 2^s
    u64 t = q * f.c + (lo & f.mask);                       // < 2^(s+12) + 2^s
    t = (t >> s) * f.c + (t & f.mask);                     // < 2^s + 2^25
    return t >= f.p ? t - f.p : t;
}

__device__ __forceinline__ u64 ssn_reduce_wide(u64 hi, u64 lo, const SsnField &f) {
    return f.pm ? ssn_pmfold(hi, lo, f) : ssn_barrett(hi, lo, f);
}

__device__ __forceinline__ u64 ssn_mulmod(u64 a, u64 b, const SsnField &f) {
    return ssn_reduce_wide(__umul64hi(a, b), a * b, f);
}

// 128-bit accumulator helpers
struct u128s { u64 lo, hi; };
__device__ __forceinline__ void ssn_mac(u128s &acc, u64 a, u64 b) {
    u64 lo = a * b, hi = __umul64hi(a, b);
    acc.lo += lo;
    acc.hi += hi + (acc.lo < lo);
}
// reduce any 64-bit value mod p (exact for all x when s >= 32)
__device__ __forceinline__ u64 ssn_reduce64(u64 x, const SsnField &f) {
    return f.s >= 32 ? ssn_reduce_wide(0, x, f) : x % f.p;
}
// reduce an arbitrary 128-bit value mod p: hi*2^64 + lo == (hi mod p)*r64 + lo (mod p).
__device__ __forceinline__ u64 ssn_reduce128(u128s x, const SsnField &f, u64 r64) {
    if (f.s >= 32 && x.hi < (1ull << (2 * f.s - 64))) return ssn_reduce_wide(x.hi, x.lo, f);
    u64 t = ssn_mulmod(ssn_reduce64(x.hi, f), r64, f);
    return ssn_addmod(t, ssn_reduce64(x.lo, f), f.p);
}

__device__ __forceinline__ u64 ssn_powmod(u64 a, u64 e, const SsnField &f) {
    u64 r = 1 % f.p;
    while (e) {
        if (e & 1) r = ssn_mulmod(r, a, f);
        a = ssn_mulmod(a, a, f);
        e >>= 1;
    }
    return r;
}

// ---- Philox4x32-10 counter-based generator (device speed mode) ----
struct ssn_u4 { u32 x, y, z, w; };
__device__ __forceinline__ ssn_u4 ssn_philox(u32 c0, u32 c1, u32 c2, u32 c3, u32 k0, u32 k1) {
#pragma unroll
    for (int i = 0; i < 10; i++) {
        u32 hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
        u32 hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
        u32 n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
    }
    return ssn_u4{c0, c1, c2, c3};
}

__device__ __forceinline__ ssn_u4 ssn_philox_at(u64 seed, u64 stream, u64 i, u32 j) {
    return ssn_philox((u32)i, (u32)(i >> 32) ^ (j << 20), (u32)stream, (u32)(stream >> 32), (u32)seed,
                      (u32)(seed >> 32));
}

// floor(r96 * range / 2^96) for r96 = (r64 << 32) | r32: uniform in [0, range),
// statistical distance from uniform < range / 2^96.
__device__ __forceinline__ u64 ssn_bounded(u64 r64, u32 r32, u64 range) {
    u64 lo1 = r64 * range, hi1 = __umul64hi(r64, range);
    u64 ulo = (u64)r32 * range, uhi = __umul64hi((u64)r32, range);
    u64 a0 = lo1 & 0xffffffffull, a1 = lo1 >> 32;
    u64 b1 = ulo >> 32;
    u64 carry1 = (a0 + b1) >> 32;
    return hi1 + ((a1 + uhi + carry1) >> 32);
}

// Draw number `j` for element `i` of stream `stream`: uniform in [0, range) (one Philox call).
__device__ __forceinline__ u64 ssn_rand_range(u64 seed, u64 stream, u64 i, u32 j, u64 range) {
    ssn_u4 r = ssn_philox_at(seed, stream, i, j);
    return ssn_bounded(((u64)r.x << 32) | r.y, r.z, range);
}

// Process-wide count of kernels this library launched (ssn_kernel_launches()); one shared
// instance across translation units (inline function, static local).
inline unsigned long long &ssn_launch_counter() {
    static unsigned long long c = 0;
    return c;
}
#define SSN_COUNT_LAUNCH() (++ssn_launch_counter())

// Kernels that run beside the persistent share GEMM (chains, plane packing) ask for the
// max-shared-memory L1 carveout: an SM configured for a small carveout must drain every resident
// block before it can switch and host a GEMM CTA (~185 KB of shared memory), which serialises
// the two CUDA streams the bench overlaps.  Call once per kernel (host side).
template <typename KernT>
inline void ssn_prefer_max_smem(KernT kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
}

// Two uniform field elements (coefficients 2*jp and 2*jp+1) from one Philox call when p is
// within 2^-24 of a power of two (masked 64-bit words; the default prime is 2^-39 close);
// otherwise the bounded 96-bit method, one call each.
__device__ __forceinline__ void ssn_rand_field2(u64 seed, u64 stream, u64 i, u32 jp, const SsnField &f, u64 &x0,
                                                u64 &x1) {
    if (f.near) {
        ssn_u4 r = ssn_philox_at(seed, stream, i, 0x800u | jp);
        x0 = (((u64)r.x << 32) | r.y) & f.mask;
        x1 = (((u64)r.z << 32) | r.w) & f.mask;
        if (x0 >= f.p) x0 -= f.p;
        if (x1 >= f.p) x1 -= f.p;
    } else {
        x0 = ssn_rand_range(seed, stream, i, 2 * jp, f.p);
        x1 = ssn_rand_range(seed, stream, i, 2 * jp + 1, f.p);
    }
}
#endif
