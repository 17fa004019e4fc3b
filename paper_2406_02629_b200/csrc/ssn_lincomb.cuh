// ssn_lincomb.cuh -- constant linear combinations over the field (Lagrange weights, the reducing
// matrix R, Reed-Solomon extrapolation rows, party-id powers) with the small-integer fast path,
// and the Shamir share evaluation helpers shared by the elementwise and fused-chain kernels.
#pragma once
#include "ssn_field.cuh"

#define SSN_MAXJ 16      // parties / share ids
#define SSN_MAXP 9       // points of one reconstruction (2k-1 <= 9)
#define SSN_MAXK 8       // polynomial coefficients k-1

// ---------------------------------------------------------------- small linear combinations
// Every constant linear combination on the protocol path -- Lagrange weights at 0 (rec),
// the reducing matrix R (reshare step 2), RS extrapolation rows and party-id powers (gen) --
// is a ratio of small integers for the default party ids 1..n (e.g. rec over ids 1..5 at 0
// has weights 5,-10,10,-5,1).  The host finds N_j / D with |N_j| < 2^13 by rational
// reconstruction; the device then evaluates D^-1 * sum N_j x_j with 32-bit multiplies and a
// single reduction instead of one full 64x64 mulmod per term.  Any other constant set falls
// back to full mulmods (flag ok = 0).
struct LinRow {
    u64 w[SSN_MAXJ];        // full field constants (fallback)
    int32_t n[SSN_MAXJ];    // small signed numerators
    u64 dinv;               // D^-1 mod p
    int one;                // D == 1
};

static inline int ratrec(u64 w, u64 p, long long &a, long long &b) {
    // a/b == w (mod p) with |a|, |b| <= 2^15 (half extended Euclid)
    const long long A = 1 << 15;
    __int128 r0 = p, r1 = w % p, t0 = 0, t1 = 1;
    while (r1 > A) {
        __int128 q = r0 / r1, r2 = r0 - q * r1, t2 = t0 - q * t1;
        r0 = r1; r1 = r2; t0 = t1; t1 = t2;
    }
    a = (long long)r1;
    b = (long long)t1;
    if (b < 0) { a = -a; b = -b; }
    return b > 0 && b <= A;
}

static inline long long gcdll(long long x, long long y) {
    if (x < 0) x = -x;
    while (y) { long long t = x % y; x = y; y = t; }
    return x;
}

static inline u64 inv_host(u64 a, u64 p) {
    __int128 lm = 1, hm = 0, low = a % p, high = p;
    while (low > 1) {
        __int128 r = high / low, nm = hm - lm * r, nw = high - low * r;
        hm = lm; high = low; lm = nm; low = nw;
    }
    __int128 v = lm % (__int128)p;
    if (v < 0) v += p;
    return (u64)v;
}

// returns 1 if the row has a small representation
static inline int make_row(LinRow &r, const u64 *w, int m, u64 p) {
    long long a[SSN_MAXJ], b[SSN_MAXJ], D = 1;
    for (int j = 0; j < SSN_MAXJ; j++) { r.w[j] = 0; r.n[j] = 0; }
    for (int j = 0; j < m; j++) r.w[j] = w[j] % p;
    r.dinv = 1;
    r.one = 1;
    // 16 terms of x * |N| with x < p < 2^47 and |N| < 2^13 stay below 2^64
    int ok = p > (1ull << 32) && p < (1ull << 47);
    for (int j = 0; j < m && ok; j++) {
        ok = ratrec(r.w[j], p, a[j], b[j]);
        if (ok) {
            D = D / gcdll(D, b[j]) * b[j];
            ok = D < (1 << 15);
        }
    }
    for (int j = 0; j < m && ok; j++) {
        long long nj = a[j] * (D / b[j]);
        ok = nj > -(1 << 13) && nj < (1 << 13);
        r.n[j] = (int32_t)nj;
    }
    if (ok) {
        r.dinv = inv_host((u64)D, p);
        r.one = D == 1;
    }
    return ok;
}

struct Weights { LinRow r; int small; };
struct RTable { LinRow r[SSN_MAXJ]; int small; };
struct ExtTable { LinRow r[SSN_MAXP]; int small; };
struct PowTable {            // row t: ids[t]^(j+1) mod p, j < km1
    LinRow r[SSN_MAXJ];
    int small;
};

static inline Weights make_weights(const u64 *w, int m, u64 p) {
    Weights W;
    W.small = make_row(W.r, w, m, p);
    return W;
}

static inline PowTable make_pows(const u64 *ids, int nids, int km1, u64 p) {
    PowTable t;
    t.small = 1;
    for (int a = 0; a < SSN_MAXJ; a++) {
        u64 row[SSN_MAXK] = {0};
        unsigned __int128 acc = 1;
        if (a < nids)
            for (int j = 0; j < km1; j++) {
                acc = acc * (ids[a] % p) % p;
                row[j] = (u64)acc;
            }
        int ok = make_row(t.r[a], row, km1, p);
        if (a < nids) {
            // gen accumulates only positive terms: require D == 1 and non-negative numerators
            for (int j = 0; j < km1; j++) ok = ok && t.r[a].n[j] >= 0;
            t.small = t.small && ok && t.r[a].one;
        }
    }
    return t;
}

__device__ __forceinline__ u64 mul_small(u64 x, uint32_t c) {
    // x < 2^62, c < 2^13: (xh*c << 32) + xl*c with two 32x32 products
    return ((u64)(uint32_t)(x >> 32) * c << 32) + (u64)(uint32_t)x * c;
}

// sum_j coef_j * x_j over j < m (coefficients of row r)
template <int MAXM>
__device__ __forceinline__ u64 lincomb(const u64 (&x)[MAXM], const LinRow &r, int small, int m,
                                       const SsnField &f) {
    if (small) {
        u64 pos = 0, neg = 0;
#pragma unroll
        for (int j = 0; j < MAXM; j++)
            if (j < m) {
                const int32_t c = r.n[j];
                if (c >= 0) pos += mul_small(x[j], (uint32_t)c);
                else neg += mul_small(x[j], (uint32_t)(-c));
            }
        const u64 v = ssn_submod(ssn_reduce64(pos, f), ssn_reduce64(neg, f), f.p);
        return r.one ? v : ssn_mulmod(v, r.dinv, f);
    }
    u64 acc = 0;
#pragma unroll
    for (int j = 0; j < MAXM; j++)
        if (j < m) acc = ssn_addmod(acc, ssn_mulmod(x[j], r.w[j], f), f.p);
    return acc;
}

// Polynomial coefficients c_0..c_{km1-1} for element i: host-fed or Philox pairs.
__device__ __forceinline__ void load_coeffs(u64 (&c)[SSN_MAXK], const u64 *__restrict__ coeffs, u64 n, u64 i,
                                            int km1, u64 seed, u64 stream, const SsnField &f) {
    if (coeffs) {
#pragma unroll
        for (int j = 0; j < SSN_MAXK; j++)
            if (j < km1) c[j] = coeffs[(u64)j * n + i];
    } else {
#pragma unroll
        for (int jp = 0; jp < SSN_MAXK / 2; jp++)
            if (2 * jp < km1) ssn_rand_field2(seed, stream, i, jp, f, c[2 * jp], c[2 * jp + 1]);
    }
}

// share at id t: s + sum_j c_j * ids[t]^(j+1)
__device__ __forceinline__ u64 horner_at(u64 s, const u64 (&c)[SSN_MAXK], const PowTable &pw, int t, int km1,
                                         const SsnField &f) {
    if (pw.small) {
        u64 acc = s;
#pragma unroll
        for (int j = 0; j < SSN_MAXK; j++)
            if (j < km1) acc += mul_small(c[j], (uint32_t)pw.r[t].n[j]);
        return ssn_reduce64(acc, f);
    }
    u64 acc = s;
#pragma unroll
    for (int j = 0; j < SSN_MAXK; j++)
        if (j < km1) acc = ssn_addmod(acc, ssn_mulmod(c[j], pw.r[t].w[j], f), f.p);
    return acc;
}


__device__ __forceinline__ i64 ssn_floordiv(i64 a, i64 b) {
    i64 q = a / b;
    if ((a % b != 0) && ((a < 0) != (b < 0))) q -= 1;
    return q;
}

// Elite side of sss_truncation on the reconstructed masked value v (S/layers.py:300-308):
// window decode into [lo, lo + p) with lo = -value_bound + r*d (S/layers.py:231-233,288),
// floor division by r (Python //), round_half_away by d (S/model.py:44-50), back into F_p.
__device__ __forceinline__ u64 ssn_trunc_value(u64 v, i64 lo, u64 neglo_mod, i64 r, int rshift, i64 d,
                                               const SsnField &f) {
    const u64 u = ssn_addmod(v, neglo_mod, f.p);
    const i64 shifted = (i64)u + lo;
    i64 t = rshift >= 0 ? (shifted >> rshift) : ssn_floordiv(shifted, r);   // arithmetic shift == floor
    if (d > 1) {
        const i64 a = t < 0 ? -t : t;
        const i64 qd = (2 * a + d) / (2 * d);
        t = t < 0 ? -qd : qd;
    }
    if (t >= 0) return ssn_reduce64((u64)t, f);
    const u64 mneg = ssn_reduce64((u64)(-t), f);
    return mneg ? f.p - mneg : 0;
}
