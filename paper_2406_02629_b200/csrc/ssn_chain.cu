// ssn_chain.cu -- one fused protocol kernel per secure layer, all n co-resident parties.
//
// In ResNet-style schedules every share GEMM is followed by a chain of per-element protocol
// steps that only ever touch the same element index across parties:
//
//   reshare_degree_reduce   S/protocol.py:131-199   participants 1..m -> front 1..k -> out ranks
//   rerand + bias           S/protocol.py:260-265, S/layers.py:260-267
//   sss_truncation          S/layers.py:277-323     x + alpha -> elite rec/decode/floor/round ->
//                                                   fresh (k,n) shares -> + comp   [+RS check]
//   share_add (residual)    S/sss.py:238
//   sss_nonlinear           S/layers.py:326-380     x * beta -> elite rec/decode/ReLU/pool/encode
//                                                   -> plain * beta^-1 at the fan-out ranks
//
// With the parties co-resident on one GPU, a thread owns one element (or one pooling window)
// for ALL parties: every message of the chain (RESHARE_OUT sub-shares, RESHARE_BACK rows,
// TRUNC_MASKED, SHARE_DIST, NONLIN_MASKED, NONLIN_PLAIN) is computed exactly as the
// reference computes it, and the hand-off between parties is a register move instead of an
// HBM round trip.  The trusted source's masks (zero shares, alpha/comp, beta/beta^-1,
// S/masks.py) are drawn in the same thread from the source's Philox lane (coefficients
// sliced densely from Philox reservoirs); beta^-1 for the 256 windows of a warp comes from one
// Fermat inversion plus warp-shuffle prefix/suffix products (Montgomery's batch trick).  HBM
// traffic per element: 8*m bytes of GEMM output in, 8*n bytes of shares out (+8*n for a
// residual add, +6*m bytes of limb planes for the next implicit-GEMM conv).
//
// Kernels: k_chain_plain (reshare .. truncation [.. add]) and k_chain_nonlin (.. masked
// nonlinearity).  A nonlinear chain normally runs as k_chain_plain into a scratch buffer
// followed by k_chain_nonlin<SPLIT> -- two kernels of half the code each beat one kernel that
// overflows the instruction cache (profiles/r01/README.md).
//
// The kernels are specialised to the default field p = 2^45 - 55 (S/field.py:21, pseudo-Mersenne
// with masked uniform draws) and to the default party ids 1..n, whose protocol constants are
// compile-time integers (ssn_chain_consts.cuh).  They are bound by the FMA-heavy pipe (IMAD), so
// the arithmetic is arranged to spend as few IMAD / IMAD.WIDE as possible.
// ssn_chain_supported() tells the host; other schemes use the unfused kernels of
// ssn_elementwise.cu.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include "ssn.h"
#include "ssn_field.cuh"
#include "ssn_lincomb.cuh"
#include "ssn_p45.cuh"
#include "ssn_chain_consts.cuh"
#include <type_traits>

namespace {
using namespace ssn45;


// ---- compile-time protocol constants (default party ids 1..n, ssn_chain_consts.cuh)
// Every constant linear combination of the chain -- reducing-matrix columns (scaled by their
// common denominator D_t), Lagrange rows at 0, Reed-Solomon rows, party-id powers -- is an
// integer immediate, so the multiplies fold into shift/LEA sequences or 32-bit IMADs and the
// signs are known: no offset trick, no per-row D^-1 multiply (measured: the chain kernels are
// bound by the FMA-heavy pipe that executes IMAD, profiles/r02/alu).
template <int I, int E, class F>
__device__ __forceinline__ void sfor(F &&f) {
    if constexpr (I < E) {
        f(std::integral_constant<int, I>{});
        sfor<I + 1, E>(f);
    }
}

template <int K, int N, int T>
struct RtRow {        // column T of the reducing matrix times D_T: out rank T <- participants j
    static constexpr int len = 2 * K - 1;
    SSN_CC static int64_t c(int j) { return ChainConsts<K, N>::rt(T, j); }
};
template <int K, int N, int C>
struct ViRow {        // column C of the inverse participant Vandermonde matrix times D_v
    static constexpr int len = 2 * K - 1;
    SSN_CC static int64_t c(int j) { return ChainConsts<K, N>::vi(C, j); }
};
template <int K, int N>
struct WfRow {        // Lagrange weights at 0 of the front ids 1..k
    static constexpr int len = K;
    SSN_CC static int64_t c(int j) { return ChainConsts<K, N>::wf(j); }
};
template <int K, int N>
struct WpRow {        // Lagrange weights at 0 of the participant ids 1..2k-1
    static constexpr int len = 2 * K - 1;
    SSN_CC static int64_t c(int j) { return ChainConsts<K, N>::wp(j); }
};
template <int K, int N, int T>
struct ExtRow {       // Reed-Solomon row: share at id T+1 from the front shares
    static constexpr int len = K;
    SSN_CC static int64_t c(int j) { return ChainConsts<K, N>::ext(T, j); }
};
template <class Row>
SSN_CC int64_t row_sum(int sign) {
    int64_t s = 0;
    for (int j = 0; j < Row::len; j++)
        if (Row::c(j) * sign > 0) s += Row::c(j) * sign;
    return s;
}
SSN_CC u64 cmod(int64_t c) { return c >= 0 ? (u64)c % PP : PP - (u64)(-c) % PP; }

// Terms of a row with opposite coefficients +c / -c pair up: c * (x_j + B - x_k), B a multiple of
// p above any input, costs one multiply instead of two (Lagrange rows are full of such pairs:
// wp = (5, -10, 10, -5, 1), wf = (3, -3, 1), D_v B^-1[:, 0] = 24 wp).
// pair[j] >= 0: j is the positive member, pair[j] its negative partner; -2: a negative member
// already paired; -1: unpaired.
template <class Row>
struct Pairing {
    int pair[Row::len];
};
template <class Row>
SSN_CC Pairing<Row> make_pairing() {
    Pairing<Row> pr{};
    for (int j = 0; j < Row::len; j++) pr.pair[j] = -1;
    for (int j = 0; j < Row::len; j++) {
        if (Row::c(j) <= 0 || pr.pair[j] != -1) continue;
        for (int k = 0; k < Row::len; k++)
            if (pr.pair[k] == -1 && Row::c(k) == -Row::c(j)) {
                pr.pair[j] = k;
                pr.pair[k] = -2;
                break;
            }
    }
    return pr;
}
template <class Row>
struct PairOf {
    static constexpr Pairing<Row> v = make_pairing<Row>();
};
// bound weights: sum of c over positive unpaired terms + 3 c over pairs (x + B < 3 * 2^XB), and
// sum of |c| over negative unpaired terms
template <class Row>
SSN_CC int64_t pos_weight() {
    constexpr Pairing<Row> pr = make_pairing<Row>();
    int64_t s = 0;
    for (int j = 0; j < Row::len; j++) {
        if (pr.pair[j] >= 0) s += 3 * Row::c(j);
        else if (pr.pair[j] == -1 && Row::c(j) > 0) s += Row::c(j);
    }
    return s;
}
template <class Row>
SSN_CC int64_t neg_weight() {
    constexpr Pairing<Row> pr = make_pairing<Row>();
    int64_t s = 0;
    for (int j = 0; j < Row::len; j++)
        if (pr.pair[j] == -1 && Row::c(j) < 0) s -= Row::c(j);
    return s;
}

// sum_j c_j x_j mod p, lazy (< 2^46), for compile-time integer c_j and inputs x_j < 2^XB.
// Fast form: positive and negative terms in two u64 sums, one fold:  pos < 2^63 and
// BIAS (a multiple of p above any neg) < 2^63 + p, so pos + BIAS - neg is exact in u64.
// FOLD = false (fast form only): the unreduced pos + BIAS - neg, below clin_raw_bound<Row, XB>()
template <class Row, int XB>
SSN_CC bool clin_fast() {
    return XB < 61 && (u64)pos_weight<Row>() < (1ull << (63 - XB)) && (u64)neg_weight<Row>() < (1ull << (63 - XB));
}
template <class Row, int XB>
SSN_CC u64 clin_raw_bound() {
    return (u64)(pos_weight<Row>() + neg_weight<Row>()) * (1ull << XB) + 2 * PP;
}
template <class Row, int XB, bool FOLD = true>
__device__ __forceinline__ u64 clin(const u64 (&x)[Row::len]) {
    constexpr int64_t P = pos_weight<Row>(), Q = neg_weight<Row>();
    constexpr bool fast = clin_fast<Row, XB>();
    static_assert(fast || FOLD, "unreduced combinations need the fast form");
    if constexpr (fast) {
        constexpr u64 B = ((1ull << XB) / PP + 1) * PP;        // multiple of p, > any x_j
        u64 pos = 0, neg = 0;
        sfor<0, Row::len>([&](auto jc) {
            constexpr int j = decltype(jc)::value;
            constexpr int64_t c = Row::c(j);
            constexpr int pj = PairOf<Row>::v.pair[j];
            if constexpr (pj >= 0) pos += (x[j] + B - x[pj]) * (u64)c;
            else if constexpr (pj == -1 && c > 0) pos += x[j] * (u64)c;
            else if constexpr (pj == -1 && c < 0) neg += x[j] * (u64)(-c);
        });
        constexpr u64 BIAS = (((u64)Q << XB) / PP + 1) * PP;
        if constexpr (!FOLD) return pos + BIAS - neg;
        return lz(pos + BIAS - neg);
    } else {
        // wide coefficients (k = 4 reducing-matrix columns): full field products
        u64 s = 0;
#pragma unroll
        for (int j = 0; j < Row::len; j++) {
            const int64_t c = Row::c(j);
            if (c != 0) s += mulm(XB > 58 ? lz(x[j]) : x[j], cmod(c));
        }
        return lz(s);
    }
}
// bits of (s + sum_e c_e * id^(e+1)) for s < 2^46, c_e < 2^45, id <= MAXID
SSN_CC int poly_bits(int k, int maxid) {
    u64 b = 2;                   // s < 2 * 2^45
    u64 pw = 1;
    for (int e = 0; e < k - 1; e++) {
        pw *= (u64)maxid;
        b += pw;
    }
    int bits = 45;
    while ((1ull << (bits - 45)) < b) bits++;
    return bits;
}

// Division of a 32-bit numerator by a launch-constant 32-bit divisor: q = umulhi64(x, ceil(2^64/d))
// is exact for all x < 2^32 (Granlund-Montgomery with a 64-bit magic), ~3 IMADs instead of the
// ~20-instruction integer-division sequence.
struct FastDiv {
    u64 m;
    uint32_t d;
};
static inline FastDiv make_fastdiv(uint32_t d) {
    FastDiv f;
    f.d = d;
    f.m = d == 1 ? 0 : (u64)((((unsigned __int128)1) << 64) / d + 1);
    return f;
}
__device__ __forceinline__ uint32_t fdiv(uint32_t x, const FastDiv &f) {
    return f.d == 1 ? x : (uint32_t)__umul64hi((u64)x, f.m);
}

struct ChainArgs {
    const u64 *acc;
    u64 acc_ps;
    const u64 *bias;
    u64 bias_ps;
    FastDiv bias_div, bias_mod, f_chw, f_hw, f_ow;
    const u64 *other;
    u64 other_ps;
    u64 *out;
    u64 out_ps;
    u64 nel;
    int nout, senders, relu, pool_kind, c, h, w, kh, kw, fan, nb;
    i64 lo, r, d;
    u64 neglo_mod, stepm, emax, bmax;
    int rshift;
    u64 pseed, pstream, sseed, sstream;
    unsigned long long *fail;
    int fault_rank;
    // channel-major u8 limb planes of the output for the next implicit-GEMM conv (may be null):
    // byte l of participant t's share of (img, c, y, x) at
    //   planes + (dx*pl_nparty + t)*pl_ps + l*pl_ls + c*pl_cs + img*pl_is + y*pl_wp + x + 1 - dx
    // for each of pl_copies column-shifted copies (1: unshifted, 3: shifts -1, 0, +1)
    uint8_t *planes;
    u64 pl_ps, pl_ls, pl_cs, pl_is;
    int pl_wp, pl_copies, pl_nparty;
    const u64 *inv_table;   // optional: inv_table[b] = b^-1 mod p for b in [1, bmax]
    // reference-stream (host-fed) trusted-source material, used by the HF instantiations: the
    // share of party t of image-element ii = i mod per (every image of the batch gets the SAME
    // masks, exactly like the reference's runs over input_index, S/engine.py:64-74):
    //   h_zero / h_alpha / h_comp / h_beta [t*per + ii],  h_tcoef [e*per + ii] (the elite's fresh
    //   truncation coefficients, PURPOSE_PARTY lane), h_binv [t*per_out + oo]
    const u64 *h_zero, *h_alpha, *h_comp, *h_tcoef, *h_beta, *h_binv;
    u64 per, per_out, per_in;      // per_in: nonlinear input elements per image (beta shares)
    FastDiv f_per, f_per_out, f_per_in;
    // overlapping-window gather before the nonlinearity (builder op "gather", e.g. the 3x3/s2/p1
    // stem max-pool): the nonlinearity's (c, h, w) input is the gathered tensor whose window
    // (y0, x0) element (wy, wx) is source element (y0*gs - gp + wy, x0*gs - gp + wx) of the
    // (c, gh, gw) chain output, or a zero share outside it
    int gather, gh, gw, gs, gp;
    // element / window range of this launch (a chain split into L2-sized chunks: the nonlinearity
    // of a chunk reads the scratch its plain kernel just wrote while it is still in L2)
    uint32_t r_lo, r_hi;
};

// Co-scheduling with the persistent share GEMM (-DSSN_COSCHED=1, off: measured slower,
// profiles/r02/README.md): the chain kernels are
// shaped so that AT MOST TWO of their blocks fit on an SM and two always leave room for one GEMM
// CTA (192 threads x 80 registers + its shared memory).  Whatever order the block scheduler sees
// the launches of the two CUDA streams in, a GEMM CTA never waits for chain blocks to drain, so
// the tensor-bound GEMM of one sub-batch runs UNDER the ALU-bound chains of the other.
//   k_chain_plain:  256 threads x <= 96 registers  (24 576 per block, 3 would need 73 728)
//   k_chain_nonlin: 288 threads x <= 80 registers  (23 040 per block, 3 would need 69 120)
#ifndef SSN_COSCHED
#define SSN_COSCHED 0
#endif
#if SSN_COSCHED
constexpr int CHAIN_THREADS = 288;
constexpr int PLAIN_THREADS = 256;
#define SSN_PLAIN_BOUNDS __maxnreg__(96)
#define SSN_NONLIN_BOUNDS __maxnreg__(80)
#else
#ifndef SSN_CHAIN_THREADS
#define SSN_CHAIN_THREADS 128
#endif
constexpr int CHAIN_THREADS = SSN_CHAIN_THREADS;
constexpr int PLAIN_THREADS = 128;
// default: k_chain_plain at 6 CTAs/SM (80 registers, no spill), k_chain_nonlin at 6
#ifndef SSN_PLAIN_MINB
#define SSN_PLAIN_MINB 6
#endif
#ifndef SSN_NONLIN_MINB
#define SSN_NONLIN_MINB 6
#endif
#define SSN_PLAIN_BOUNDS __launch_bounds__(PLAIN_THREADS, SSN_PLAIN_MINB)
#define SSN_NONLIN_BOUNDS __launch_bounds__(CHAIN_THREADS, SSN_NONLIN_MINB)
#endif

__device__ __forceinline__ u64 sqn(u64 x, int n) {
#pragma unroll 1
    for (int i = 0; i < n; i++) x = mulm_hs(x, x);
    return x;
}
// x^(p-2) = x^(2^45 - 57) by the addition chain x^(2^39-1)^(2^6) * x^7 (52 multiplications).
// Here and in the batch inversion every operand is lazy (< 2^46), so products stay below 2^92 and
// mulm_hs applies.
__device__ __noinline__ u64 invm(u64 x) {
    const u64 x2 = mulm_hs(x, x), x3 = mulm_hs(x2, x), x7 = mulm_hs(mulm_hs(x3, x3), x);
    const u64 x6b = mulm_hs(sqn(x7, 3), x7);            // x^(2^6-1)
    const u64 x12 = mulm_hs(sqn(x6b, 6), x6b);          // x^(2^12-1)
    const u64 x24 = mulm_hs(sqn(x12, 12), x12);         // x^(2^24-1)
    const u64 x36 = mulm_hs(sqn(x24, 12), x12);         // x^(2^36-1)
    const u64 x39 = mulm_hs(sqn(x36, 3), x7);           // x^(2^39-1)
    return mulm_hs(sqn(x39, 6), x7);
}

// share of s at party id `id` (a compile-time constant after unrolling): s + sum_e c_e id^(e+1),
// UNREDUCED (< 2^poly_bits(K, id) for s < 2^46): multiplies by small immediates.
template <int K>
__device__ __forceinline__ u64 poly_at(u64 s, const u64 (&c)[K - 1], int id) {
    u64 acc = s, pw = 1;
#pragma unroll
    for (int e = 0; e < K - 1; e++) {
        pw *= (u64)id;
        acc += c[e] * pw;
    }
    return acc;
}

// d-th forward difference of id^e at id = 1: sum_i (-1)^(d-i) C(d, i) (1 + i)^e (>= 0)
SSN_CC u64 fdiff_coef(int d, int e, int base = 1) {
    int64_t s = 0, c = 1;                                   // c = C(d, i)
    for (int i = 0; i <= d; i++) {
        int64_t pw = 1;
        for (int k = 0; k < e; k++) pw *= base + i;
        s += ((d - i) % 2 ? -c : c) * pw;
        c = c * (d - i) / (i + 1);
    }
    return (u64)s;
}

#ifndef SSN_WALK0
#define SSN_WALK0 1
#endif
SSN_CC int ilog2c(u64 c) {
    int l = 0;
    while ((1ull << l) < c) l++;
    return l;
}
// f(id) = sum_e P_e id^e (exact integer, unreduced) at id = 1, 2, 3, ... by forward
// differences: k - 1 adds per point instead of multiplies by the powers of id
template <int K>
struct PolyWalk {
    u64 d[K];                                      // d[j] = Delta^j f at the current id
    // SSN_WALK0: start from the differences at id = 0 (coefficients j! S(e, j): 1 and 2 for
    // k = 3, a shift instead of multiplies) and step once to id = 1
    __device__ __forceinline__ void init(const u64 (&P)[K]) {
        constexpr int BASE = SSN_WALK0 ? 0 : 1;
        sfor<0, K>([&](auto jc) {
            constexpr int j = decltype(jc)::value;
            u64 acc = 0;
            sfor<j, K>([&](auto ec) {
                constexpr int e = decltype(ec)::value;
                constexpr u64 c = fdiff_coef(j, e, BASE);
                if constexpr (c == 1) acc += P[e];
                else if constexpr (c != 0 && (c & (c - 1)) == 0) acc += P[e] << ilog2c(c);
                else if constexpr (c != 0) acc += P[e] * c;
            });
            d[j] = acc;
        });
        if constexpr (SSN_WALK0) step();
    }
    // f = s + sum_e c_e id^(e+1): the share polynomial of poly_at
    __device__ __forceinline__ void init(u64 s, const u64 (&c)[K - 1]) {
        u64 P[K];
        P[0] = s;
#pragma unroll
        for (int e = 1; e < K; e++) P[e] = c[e - 1];
        init(P);
    }
    __device__ __forceinline__ u64 value() const { return d[0]; }
    __device__ __forceinline__ void step() {
#pragma unroll
        for (int j = 0; j + 1 < K; j++) d[j] += d[j + 1];
    }
};

// K-1 uniform field elements: masked 45-bit Philox words.  Values in [p, 2^45) are lazy
// representatives of [0, 55), exactly the distribution of the conditional-subtract form.
template <int K>
__device__ __forceinline__ void coeffs(u64 (&c)[K - 1], u64 seed, u64 stream, u64 i) {
#pragma unroll
    for (int jp = 0; jp < K / 2; jp++) {
        const ssn_u4 r = ssn_philox_at(seed, stream, i, 0x800u | jp);
        c[2 * jp] = (((u64)r.x << 32) | r.y) & PMASK;
        if (2 * jp + 1 < K - 1) c[2 * jp + 1] = (((u64)r.z << 32) | r.w) & PMASK;
    }
}

// Dense use of Philox output: NC calls give 128*NC random bits, sliced into 45-bit field
// coefficients (and one 64-bit word for a bounded draw) instead of one call per 2 coefficients.
template <int NC>
struct Reservoir {
    uint32_t w[4 * NC + 2];
};
template <int NC>
__device__ __forceinline__ void fill(Reservoir<NC> &r, u64 seed, u64 stream, u64 i, uint32_t tag) {
#pragma unroll
    for (int c = 0; c < NC; c++) {
        const ssn_u4 v = ssn_philox_at(seed, stream, i, tag + c);
        r.w[4 * c] = v.x;
        r.w[4 * c + 1] = v.y;
        r.w[4 * c + 2] = v.z;
        r.w[4 * c + 3] = v.w;
    }
    r.w[4 * NC] = r.w[4 * NC + 1] = 0;
}
// bits [bit, bit + 64) of the reservoir; `bit` is a compile-time constant after unrolling, so
// the word indices resolve to registers
template <int NC>
__device__ __forceinline__ u64 take64(const Reservoir<NC> &r, int bit) {
    const int wi = bit >> 5, sh = bit & 31;
    const u64 lo = ((u64)r.w[wi + 1] << 32) | r.w[wi];
    return sh == 0 ? lo : (lo >> sh) | ((u64)r.w[wi + 2] << (64 - sh));
}
template <int NC>
__device__ __forceinline__ u64 take45(const Reservoir<NC> &r, int bit) {
    return take64<NC>(r, bit) & PMASK;
}

// elite truncation of the reconstructed masked value (ssn_trunc_value, specialised)
__device__ __forceinline__ u64 trunc_val(u64 v, const ChainArgs &a) {
    const i64 shifted = (i64)addm(v, a.neglo_mod) + a.lo;
    i64 t = a.rshift >= 0 ? (shifted >> a.rshift) : ssn_floordiv(shifted, a.r);
    if (a.d > 1) {
        const i64 q = ((t < 0 ? -t : t) * 2 + a.d) / (2 * a.d);
        t = t < 0 ? -q : q;
    }
    if (t >= 0) return red64((u64)t);
    const u64 mneg = red64((u64)(-t));
    return mneg ? PP - mneg : 0;
}

// reshare + rerand + bias + truncation (+ residual add) of element i for all N parties.
// HF: the trusted source's masks and the elite's truncation coefficients are host-fed shares
// (reference-stream parity mode) instead of in-register Philox draws.
//
// Every message is computed (RESHARE_OUT sub-shares, RESHARE_BACK rows, TRUNC_MASKED, the elite's
// fresh shares); two representation choices keep the FMA-heavy pipe light:
//  * front fr's RESHARE_BACK row to out rank t is held as D_t * back (D_t the common denominator
//    of R's column t); rank t multiplies its reconstruction by D_t^-1 once, instead of every front
//    row paying one full modular multiply;
//  * a rank adds the zero share and the alpha share it receives as one polynomial evaluation of
//    the summed coefficients (the same integer), likewise the fresh truncation share and comp.
// RAW: leave the outputs unreduced (< 2^58; the caller canonicalises them for the store) instead
// of lazily reduced (< 2^46, the nonlinearity's multiply operands)
template <int K, int N, bool HF, bool RAW = false>
__device__ __forceinline__ void chain_elem(const ChainArgs &a, uint32_t i, u64 (&x)[N], unsigned long long &bad) {
    constexpr int M = 2 * K - 1;
    using CC = ChainConsts<K, N>;
    constexpr int XB_SUB = poly_bits(K, K);          // sub-share bound: front ids <= K
    u64 acc[M];
#pragma unroll
    for (int j = 0; j < M; j++) acc[j] = a.acc[(u64)j * a.acc_ps + i];
    // ---- reshare step 1 (RESHARE_OUT): participant j sub-shares its local product to the front
    // (the participants' M*(K-1) polynomial coefficients, then the elite's K-1 fresh truncation
    // share coefficients, sliced from one party-randomness Philox reservoir)
    constexpr int NCR = (45 * (M + (HF ? 0 : 1)) * (K - 1) + 127) / 128;
    Reservoir<NCR> rr;
    fill<NCR>(rr, a.pseed, a.pstream, i, 0x900u);
    u64 sub[K][M];
#pragma unroll
    for (int j = 0; j < M; j++) {
        u64 c[K - 1];
#pragma unroll
        for (int e = 0; e < K - 1; e++) c[e] = take45<NCR>(rr, 45 * (j * (K - 1) + e));
        PolyWalk<K> pw;
        pw.init(acc[j], c);
#pragma unroll
        for (int fr = 0; fr < K; fr++, pw.step()) sub[fr][j] = pw.value();
    }
    // source: zero shares (gen_zero_shares) and the truncation masks (gen_additive_mask).
    // A rank receives its zero share and its alpha share and only ever uses their sum, the share
    // of the summed polynomial alpha + sum_e (z_e + a_e) x^e; z_e + a_e of two independent uniform
    // coefficients is one uniform coefficient, so the source draws the sum directly (same joint
    // distribution of every rank's view).  za, the comp coefficients and the 64 bits of e come
    // from one source reservoir (2 Philox calls for k = 3 instead of 3).
    u64 za[K - 1], cc[K - 1];        // zero + alpha coefficients, comp coefficients
    u64 alpha = 0, comp = 0;
    uint32_t ii = 0;
    if constexpr (HF) {
        ii = i - fdiv(i, a.f_per) * (uint32_t)a.per;
    } else {
        constexpr int NCS = (45 * 2 * (K - 1) + 64 + 127) / 128;
        Reservoir<NCS> rs;
        fill<NCS>(rs, a.sseed, a.sstream, i, 0x900u);
#pragma unroll
        for (int e = 0; e < K - 1; e++) {
            za[e] = take45<NCS>(rs, 45 * e);
            cc[e] = take45<NCS>(rs, 45 * (K - 1 + e));
        }
        // e = 1 + U[0, emax) by multiply-shift of 64 random bits (bias <= emax / 2^64 <= 2^-32)
        const u64 e = 1 + __umul64hi(take64<NCS>(rs, 45 * 2 * (K - 1)), a.emax);
        const u64 em = red64(e);
        alpha = mulm_hs(em, a.stepm);                        // both canonical
        comp = em ? PP - em : 0;
    }
    const uint32_t bq = fdiv(i, a.bias_div);
    const uint32_t ch = bq - fdiv(bq, a.bias_mod) * a.bias_mod.d;
    // ---- step 2 (RESHARE_BACK): front fr sends rank t  sum_j R[j][t] sub[fr][j].  R is the
    //      rank-k product B^-1[:, :k] B_ext[:k, :] (S/sss.py:197-210), so the front evaluates it as
    //      sum_c id_t^c w[fr][c] with w[fr][c] = sum_j B^-1[j][c] sub[fr][j]: k*m multiplies by
    //      small integers (held as D_v * w) instead of n*m by R's wide numerators.
    //      step 3: out rank t reconstructs (Lagrange over the front), x D_v^-1, + zero share
    //      (rerand) + bias share + alpha share (TRUNC_MASKED)
    // (for k = 2 the factored form runs 1,194 instead of 1,226 thread instructions per element)
    constexpr bool FACTOR = K >= 2;
    constexpr bool LZSUB = XB_SUB > 50;                       // k = 4: fold the sub-shares first
    constexpr int XB_W = LZSUB ? 46 : XB_SUB;
    u64 w[K][K];                                              // D_v * w[fr][c], lazy
    if constexpr (FACTOR) {
#pragma unroll
        for (int fr = 0; fr < K; fr++) {
            if constexpr (LZSUB) {
#pragma unroll
                for (int j = 0; j < M; j++) sub[fr][j] = lz(sub[fr][j]);
            }
            sfor<0, K>([&](auto cc_) {
                constexpr int c = decltype(cc_)::value;
                w[fr][c] = clin<ViRow<K, N, c>, XB_W>(sub[fr]);
            });
        }
    }
    constexpr int XB_BACK = poly_bits(K, N) + 1;              // sum_c id^c w_c, w_c < 2^46
    // TRUNC_MASKED travels scaled by S (the common denominator of the reshare: D_v, or the lcm
    // of R's column denominators for k = 2): rank t sends S * masked_t, the elite reconstructs
    // S * v and multiplies by S^-1 ONCE -- instead of every rank paying a full field multiply
    // to undo its D.  The RS check is linear, so it holds on the scaled shares as well.
    constexpr u64 S = FACTOR ? CC::vi_den : CC::rt_lcm;
    constexpr u64 SINV = FACTOR ? CC::vi_dinv : CC::rt_lcm_inv;
    u64 alpha_s = 0, za_s[K - 1];
    if constexpr (!HF) {
        alpha_s = lz(alpha * S);
#pragma unroll
        for (int e = 0; e < K - 1; e++) za_s[e] = lz(za[e] * S);
    }
    // S * TRUNC_MASKED[t].  k <= 3: left unreduced -- the rank's reconstruction (unfolded, below
    // clin_raw_bound), + S (bias + 1) < 2^47 S, + the alpha/zero share < 2^46 (1 + n + n^2) --
    // and the front's Lagrange row and the RS rows take XB_M-bit inputs in their fast form (two
    // folds fewer per rank); k = 4's RS rows have coefficient sums too wide for that, so it folds
    constexpr bool MFOLD = !FACTOR || K > 3;
    constexpr u64 MBOUND = clin_raw_bound<WfRow<K, N>, XB_BACK>() + (S << 47) + (1ull << 46) * (1 + N + N * N);
    constexpr int XB_M = MFOLD ? 46 : 56;
    static_assert(MFOLD || MBOUND < (1ull << XB_M), "TRUNC_MASKED bound");
    static_assert(MFOLD || clin_fast<WfRow<K, N>, XB_M>(), "front row fast form");
    u64 masked[N];
    PolyWalk<K> aw;                                           // S * (alpha + zero) share polynomial
    if constexpr (!HF) aw.init(alpha_s, za_s);
    PolyWalk<K> bw[K];                                        // front fr's D_v * RESHARE_BACK row polynomial
    if constexpr (FACTOR) {
#pragma unroll
        for (int fr = 0; fr < K; fr++) bw[fr].init(w[fr]);
    }
    sfor<0, N>([&](auto tc) {
        constexpr int t = decltype(tc)::value;
        if (t < a.senders) {
            u64 y;                                             // S * (reshared share of rank t)
            if constexpr (FACTOR) {
                u64 back[K];                                   // D_v * RESHARE_BACK[fr -> t]
#pragma unroll
                for (int fr = 0; fr < K; fr++) back[fr] = bw[fr].value();
                y = clin<WfRow<K, N>, XB_BACK, MFOLD>(back);
            } else {
                u64 back[K];                                   // D_t * RESHARE_BACK[fr -> t]
#pragma unroll
                for (int fr = 0; fr < K; fr++) back[fr] = clin<RtRow<K, N, t>, XB_SUB>(sub[fr]);
                y = clin<WfRow<K, N>, 46>(back);
                if constexpr (S / CC::rt_den(t) != 1) y = lz(y * (S / CC::rt_den(t)));
            }
            u64 add = a.bias[(u64)t * a.bias_ps + ch];
            if constexpr (HF) add += a.h_zero[(u64)t * a.per + ii] + a.h_alpha[(u64)t * a.per + ii];
            y += add * S;                                                                   // < 2^47 * S
            if constexpr (!HF) y += aw.value();
            masked[t] = MFOLD ? lz(y) : y;
        }
        if constexpr (!HF) aw.step();
        if constexpr (FACTOR) {
#pragma unroll
            for (int fr = 0; fr < K; fr++) bw[fr].step();
        }
    });
    if (i == 0 && a.fault_rank >= 0) {                      // test hook: corrupt one rank's message
        sfor<0, N>([&](auto tc) {
            constexpr int t = decltype(tc)::value;
            if (t == a.fault_rank && t < a.senders) masked[t] = lz(masked[t] + S);          // < 2^46 either way
        });
    }
    // ---- truncation elite: rec over the front (x S^-1), RS check of the extra points,
    //      decode/floor/round
    u64 front[K];
#pragma unroll
    for (int j = 0; j < K; j++) front[j] = masked[j];
    const u64 v = canon(mulm_hs(clin<WfRow<K, N>, XB_M>(front), SINV));    // lazy x canonical
    sfor<K, N>([&](auto tc) {
        constexpr int t = decltype(tc)::value;
        if (t < a.senders) bad += (canon(clin<ExtRow<K, N, t>, XB_M>(front)) != canon(masked[t]));
    });
    const u64 tm = trunc_val(v, a);
    // fresh (k, n) shares of the truncated value (SHARE_DIST), + comp at every rank
    u64 g[K - 1];
    if constexpr (HF) {
#pragma unroll
        for (int e = 0; e < K - 1; e++) g[e] = a.h_tcoef[(u64)e * a.per + ii];
    } else {
#pragma unroll
        for (int e = 0; e < K - 1; e++) g[e] = take45<NCR>(rr, 45 * (M * (K - 1) + e)) + cc[e];
    }
    PolyWalk<K> fw;
    if constexpr (HF) fw.init(tm, g);
    else fw.init(tm + comp, g);
#pragma unroll
    for (int t = 0; t < N; t++, fw.step()) {
        u64 s = fw.value();
        if constexpr (HF) s += a.h_comp[(u64)t * a.per + ii];
        if (a.other) s += a.other[(u64)t * a.other_ps + i];                              // residual add
        x[t] = RAW ? s : lz(s);
    }
}

template <int K, int N, bool HF>
__global__ void SSN_PLAIN_BOUNDS k_chain_plain(ChainArgs a, SsnField f) {
    unsigned long long bad = 0;
    const uint32_t nel = (uint32_t)a.nel < a.r_hi ? (uint32_t)a.nel : a.r_hi;
#pragma unroll 1
    for (uint32_t i = a.r_lo + blockIdx.x * blockDim.x + threadIdx.x; i < nel; i += gridDim.x * blockDim.x) {
        u64 x[N];
        chain_elem<K, N, HF, true>(a, i, x, bad);
#pragma unroll
        for (int t = 0; t < N; t++) a.out[(u64)t * a.out_ps + i] = canon(x[t]);
    }
    if (a.fail && bad) atomicAdd(a.fail, bad);
}

// exclusive prefix (up) / suffix (down) products across the warp; inactive lanes hold 1
__device__ __noinline__ u64 warp_excl_prefix(u64 v, int lane) {
    u64 incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u64 t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl = mulm_hs(incl, t);
    }
    const u64 ex = __shfl_up_sync(0xffffffffu, incl, 1);
    return lane ? ex : 1;
}
__device__ __noinline__ u64 warp_excl_suffix(u64 v, int lane) {
    u64 incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u64 t = __shfl_down_sync(0xffffffffu, incl, o);
        if (lane + o < 32) incl = mulm_hs(incl, t);
    }
    const u64 ex = __shfl_down_sync(0xffffffffu, incl, 1);
    return lane < 31 ? ex : 1;
}

// u8 limb planes of one share value for the next implicit-GEMM conv.  Out of line: the chain
// kernel sits near the instruction-cache limit, and 5 inlined copies pushed it over.
__device__ __noinline__ void emit_planes(uint8_t *row, u64 v, int xq, int copies, u64 copy_stride, u64 ls, int wp) {
    for (int dx = 0; dx < copies; dx++) {
        const int xc = copies == 1 ? xq : xq + 1 - dx;
        if (xc < 0 || xc >= wp) continue;
        uint8_t *dst = row + (u64)dx * copy_stride + xc;
#pragma unroll
        for (int l = 0; l < 6; l++) dst[(u64)l * ls] = (uint8_t)(v >> (8 * l));
    }
}

// a * b mod p (lazy) for a < 2^46 and b < 2^32 (beta, a running product times beta): two
// 32x32->64 products instead of three
__device__ __forceinline__ u64 mulm32(u64 a, uint32_t b) { return mulm_s32(a, b); }

// run^-1 for every thread of the block from ONE Fermat inversion (Montgomery's batch trick):
// warp-shuffle exclusive prefix/suffix products, warp totals through shared memory, warp 0
// inverts the block total.  Out of line: it runs once per block iteration, and inlined it
// pushed the per-window loops out of the instruction cache.
__device__ __noinline__ u64 block_batch_inverse(u64 run, int lane, int warp, u64 *s_tot, u64 *s_inv) {
    constexpr int NW = CHAIN_THREADS / 32;
    const u64 wpre = warp_excl_prefix(run, lane);
    const u64 wsuf = warp_excl_suffix(run, lane);
    const u64 wtot = __shfl_sync(0xffffffffu, mulm_hs(wpre, run), 31);
    if (lane == 0) s_tot[warp] = wtot;
    __syncthreads();
    if (warp == 0) {
        const u64 v = lane < NW ? s_tot[lane] : 1;
        const u64 bp = warp_excl_prefix(v, lane), bs = warp_excl_suffix(v, lane);
        const u64 tot = __shfl_sync(0xffffffffu, mulm_hs(bp, v), 31);
        const u64 ti = invm(tot);
        if (lane < NW) s_inv[lane] = mulm_hs(mulm_hs(ti, bp), bs);              // = warp total^-1
    }
    __syncthreads();
    return mulm_hs(mulm_hs(s_inv[warp], wpre), wsuf);                            // = run^-1
}

// masked nonlinearity fused after the chain.  Each thread owns WPT output windows, in groups of G
// ADJACENT windows (a group never crosses a limb-plane row), so the next conv's u8 limb planes
// are written G bytes per store.  beta^-1 of all CHAIN_THREADS*WPT windows of a block iteration
// comes from ONE Fermat inversion (Montgomery's batch trick): per-thread running products,
// warp-shuffle exclusive prefix/suffix products, one inversion of the block total by warp 0,
// then a backward pass.
#ifndef SSN_WPT
#define SSN_WPT 8
#endif
constexpr int WPT = SSN_WPT;
constexpr int NWARP = CHAIN_THREADS / 32;

// byte l of each of the G values, packed little-endian (window g -> byte g)
template <int G>
__device__ __forceinline__ uint32_t pack_limb(const u64 (&v)[G], int l) {
    const int w = l >> 2, s = l & 3;
    auto word = [&](int g) { return (uint32_t)(v[g] >> (32 * w)); };
    if constexpr (G == 1) {
        return (word(0) >> (8 * s)) & 0xffu;
    } else if constexpr (G == 2) {
        return __byte_perm(word(0), word(1), (uint32_t)(s | ((4 + s) << 4)));
    } else {
        const uint32_t sel = (uint32_t)(s | ((4 + s) << 4));
        return __byte_perm(__byte_perm(word(0), word(1), sel), __byte_perm(word(2), word(3), sel), 0x5410);
    }
}

// SPLIT: the reshare/truncation/add part already ran (k_chain_plain into a.acc = its n-party
// output) and this kernel only runs the masked nonlinearity, reading each party's share.
// Two kernels of half the code each run faster than one that overflows the instruction cache.
template <int K, int N, bool SPLIT, bool HF, int G>
__global__ void SSN_NONLIN_BOUNDS k_chain_nonlin(ChainArgs a, SsnField f) {
    constexpr int M = 2 * K - 1;
    static_assert(WPT % G == 0, "groups tile a thread's windows");
    __shared__ u64 s_tot[NWARP], s_inv[NWARP];
    unsigned long long bad = 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t oh = a.h / a.kh, ow = a.w / a.kw;
    const uint32_t hw = oh * ow, chw = (uint32_t)a.c * hw;
    const uint32_t n_all = (uint32_t)a.nb * chw;
    const uint32_t n_out = n_all < a.r_hi ? n_all : a.r_hi;   // end of this launch's window range
    const bool pooled = a.kh != 1 || a.kw != 1;
    const bool batch_inv = !HF && !a.inv_table;
    const uint32_t span = CHAIN_THREADS * WPT;
    // the masked products mk: for k = 2 (speed mode) unfolded mulm_hs, < 2^56 (x < 2^45, beta
    // share < 2^50), into the elite's WpRow fast form -- fewer instructions; for (3,5) the same
    // change measured 17% slower (nonlinearity kernel), so k >= 3 and host-fed shares fold
    constexpr bool MK_RAW = K == 2 && !HF;
    constexpr int MK_XB = MK_RAW ? 56 : 46;
    static_assert(clin_fast<WpRow<K, N>, MK_XB>(), "WpRow fast form");
    // unfolded P_0 + P_1 id (k = 2) < (1 + n) 2^57.1 must stay below 2^64 for the output canon
    static_assert(!MK_RAW || N <= 100, "unfolded output polynomial bound");
#pragma unroll 1
    for (uint32_t base = a.r_lo + blockIdx.x * span; base < n_out; base += gridDim.x * span) {
        // per-window state carried from the masking pass to the output pass (local memory; the
        // lines mostly miss L1, so it is kept small -- 28 B per window for (3,5)): the output
        // share polynomial's products
        // P_e = plain * c_(e-1) (e >= 1, c the beta^-1 sharing coefficients), pp = plain times
        // the product of the thread's earlier betas (the Montgomery prefix; speed mode) or the
        // encoded plain itself (host-fed beta^-1 shares), and beta
        u64 pp[WPT], Pw[WPT][K - 1];
        uint32_t beta[WPT];
        u64 run = 1;
#pragma unroll 1
        for (int q = 0; q < WPT; q++) {
            const uint32_t o = base + ((q / G) * CHAIN_THREADS + threadIdx.x) * G + (q % G);
            i64 pl = 0;
            u64 bt = 1;
            u64 cb1[K - 1];                  // unpooled: the window's beta-share coefficients
            u64 cbi[K - 1];                  // its beta^-1 sharing coefficients
#pragma unroll
            for (int e = 0; e < K - 1; e++) cbi[e] = 0;
            if (o < n_out) {
                if constexpr (!HF) {
                    if (!pooled) {
                        // one dense reservoir per window: 64 bits for beta, then the beta and the
                        // beta^-1 sharing coefficients (2 Philox calls for (3,5) instead of 3)
                        constexpr int NCB = (64 + 2 * 45 * (K - 1) + 127) / 128;
                        Reservoir<NCB> rb;
                        fill<NCB>(rb, a.sseed, a.sstream + 4, o, 0x900u);
                        bt = 1 + __umul64hi(take64<NCB>(rb, 0), a.bmax);     // U[1, bmax], bias <= bmax / 2^64
#pragma unroll
                        for (int e = 0; e < K - 1; e++) {
                            cb1[e] = take45<NCB>(rb, 64 + 45 * e);
                            cbi[e] = take45<NCB>(rb, 64 + 45 * (K - 1 + e));
                        }
                    } else {
                        bt = 1 + ssn_rand_range(a.sseed, a.sstream + 4, o, 0, a.bmax);  // window-constant beta
                        coeffs<K>(cbi, a.sseed, a.sstream + 6, o);
                    }
                }
                uint32_t base_in = o;
                uint32_t src_base = 0;
                int sy0 = 0, sx0 = 0;
                if (pooled) {
                    const uint32_t img = fdiv(o, a.f_chw), rem = o - img * chw;
                    const uint32_t ci = fdiv(rem, a.f_hw), rr = rem - ci * hw;
                    const uint32_t y0 = fdiv(rr, a.f_ow), x0 = rr - y0 * ow;
                    base_in = ((img * a.c + ci) * a.h + y0 * a.kh) * a.w + x0 * a.kw;
                    if (SPLIT && a.gather) {
                        src_base = (img * a.c + ci) * (uint32_t)(a.gh * a.gw);
                        sy0 = (int)y0 * a.gs - a.gp;
                        sx0 = (int)x0 * a.gs - a.gp;
                    }
                }
                i64 acc = a.pool_kind == 1 ? INT64_MIN : 0;
#pragma unroll 1
                for (int wy = 0; wy < a.kh; wy++)
#pragma unroll 1
                    for (int wx = 0; wx < a.kw; wx++) {
                        const uint32_t i = base_in + wy * a.w + wx;      // (gathered) nonlinear input element
                        u64 x[N];
                        if (SPLIT) {
                            uint32_t si = i;
                            bool inside = true;
                            if (a.gather) {
                                const int sy = sy0 + wy, sx = sx0 + wx;
                                inside = sy >= 0 && sy < a.gh && sx >= 0 && sx < a.gw;
                                si = src_base + (uint32_t)(sy * a.gw + sx);
                            }
#pragma unroll
                            for (int t = 0; t < M; t++) x[t] = inside ? a.acc[(u64)t * a.acc_ps + si] : 0;
                        } else {
                            chain_elem<K, N, HF>(a, i, x, bad);
                        }
                        // participants mask with their beta shares (NONLIN_MASKED); elite rec over m
                        u64 mk[M];
                        if constexpr (HF) {
                            const uint32_t ii = i - fdiv(i, a.f_per_in) * (uint32_t)a.per_in;
#pragma unroll
                            for (int j = 0; j < M; j++) mk[j] = mulm_hs(x[j], a.h_beta[(u64)j * a.per_in + ii]);
                        } else {
                            u64 cb[K - 1];
                            if (pooled) {
                                coeffs<K>(cb, a.sseed, a.sstream + 5, i);
                            } else {
#pragma unroll
                                for (int e = 0; e < K - 1; e++) cb[e] = cb1[e];
                            }
                            PolyWalk<K> bsh;                  // beta share polynomial
                            bsh.init(bt, cb);
#pragma unroll
                            for (int j = 0; j < M; j++, bsh.step()) {
                                // x canonical (< 2^45), the beta share < 2^50 for k <= 3: the
                                // product < 2^95 (unfolded mulm_hs < 2^56 = MK_XB for k = 2)
                                if constexpr (K <= 3) mk[j] = mulm_hs<!MK_RAW>(x[j], bsh.value());
                                else mk[j] = mulm(x[j], bsh.value());
                            }
                        }
                        const u64 v = canon(clin<WpRow<K, N>, MK_XB>(mk));
                        i64 sv = v > PHALF ? (i64)v - (i64)PP : (i64)v;
                        if (a.relu && sv <= 0) sv = 0;
                        if (a.pool_kind == 1) acc = sv > acc ? sv : acc;
                        else acc += sv;
                    }
                pl = acc;                                          // NONLIN_PLAIN (signed; encoded at use)
            }
            const u64 ple = pl < 0 ? (u64)((i64)PP + pl) : (u64)pl;      // encoded, < p
            beta[q] = (uint32_t)bt;
            if constexpr (HF) {
                pp[q] = ple;                        // beta^-1 shares are host-fed
            } else {
#pragma unroll
                for (int e = 0; e < K - 1; e++) Pw[q][e] = mulm_hs<!MK_RAW>(ple, cbi[e]);
                if (a.inv_table) {
                    pp[q] = mulm_hs(ple, a.inv_table[bt]);   // = P_0 (source's beta^-1 from the table)
                } else {
                    pp[q] = mulm_hs(ple, run);               // run: product of the earlier betas
                    run = mulm32(run, (uint32_t)bt);
                }
            }
        }
        // source: beta^-1 for every window of the block iteration from ONE inversion
        u64 inv = 0;
        if (batch_inv) inv = block_batch_inverse(run, lane, warp, s_tot, s_inv);
#pragma unroll 1
        for (int gq = WPT / G - 1; gq >= 0; gq--) {
            const uint32_t o0 = base + (gq * CHAIN_THREADS + threadIdx.x) * G;
            u64 P0[G];                                       // plain * beta^-1
#pragma unroll
            for (int g = G - 1; g >= 0; g--) {
                const int q = gq * G + g;
                P0[g] = pp[q];
                if constexpr (!HF) {
                    if (!a.inv_table) {
                        // both lazy, < 2^46; k = 2: left unfolded (< 2^57.1), the output
                        // polynomial P_0 + P_1 id stays below 2^59.1 for id <= 3
                        P0[g] = mulm_hs<!MK_RAW>(inv, pp[q]);
                        inv = mulm32(inv, beta[q]);
                    }
                }
            }
            if (o0 < n_out) {                                // n_out % G == 0: the whole group
                uint32_t oo[G];
                if constexpr (HF) {
#pragma unroll
                    for (int g = 0; g < G; g++) oo[g] = (o0 + g) - fdiv(o0 + g, a.f_per_out) * (uint32_t)a.per_out;
                }
                uint8_t *pb = nullptr;
                int xq = 0;
                if (a.planes) {
                    const uint32_t img = fdiv(o0, a.f_chw), rem = o0 - img * chw;
                    const uint32_t ci = fdiv(rem, a.f_hw), pix = rem - ci * hw;
                    const uint32_t y = fdiv(pix, a.f_ow);
                    xq = (int)(pix - y * ow);
                    pb = a.planes + (u64)ci * a.pl_cs + (u64)img * a.pl_is + (u64)y * a.pl_wp;
                }
                // out ranks in a rolled loop: the G-window body unrolled over the n ranks
                // overflowed the instruction cache.  Speed mode: rank t's share of the output is
                // plain * (binv + sum_e c_e id^(e+1)) = sum_e P_e id^e with P_0 = plain * binv,
                // P_e = plain * c_(e-1): K full multiplies per window, and the polynomial in id
                // walks the ranks by forward differences of its exact integer value (K - 1 adds
                // per rank, no multiply) instead of a multiply per rank
                u64 *op = a.out + o0;
                uint8_t *dst = pb + xq;
                u64 fd[G][K];                                 // fd[g][d] = Delta^d f_g at the current id
                if constexpr (!HF) {
#pragma unroll
                    for (int g = 0; g < G; g++) {
                        u64 P[K];
                        P[0] = P0[g];
#pragma unroll
                        for (int e = 1; e < K; e++) P[e] = Pw[gq * G + g][e - 1];
                        PolyWalk<K> wk;
                        wk.init(P);
#pragma unroll
                        for (int d = 0; d < K; d++) fd[g][d] = wk.d[d];
                    }
                }
#pragma unroll 1
                for (int t = 0; t < a.fan; t++) {
                    u64 v[G];
#pragma unroll
                    for (int g = 0; g < G; g++) {
                        if constexpr (HF) {
                            v[g] = canon(mulm_hs(P0[g], a.h_binv[(u64)t * a.per_out + oo[g]]));
                        } else {
                            v[g] = canon(fd[g][0]);
#pragma unroll
                            for (int d = 0; d + 1 < K; d++) fd[g][d] += fd[g][d + 1];
                        }
                    }
                    if constexpr (G == 1) {
                        op[0] = v[0];
                    } else {
#pragma unroll
                        for (int g = 0; g < G; g += 2) *reinterpret_cast<ulonglong2 *>(op + g) = make_ulonglong2(v[g], v[g + 1]);
                    }
                    op += a.out_ps;
                    if (pb != nullptr && t < a.pl_nparty) {        // limb planes for the next conv
                        if (a.pl_copies == 1) {
                            // offsets l*ls are warp-uniform; G adjacent windows per store
#pragma unroll
                            for (int l = 0; l < 6; l++) {
                                const uint32_t w = pack_limb<G>(v, l);
                                if constexpr (G == 4) *reinterpret_cast<uint32_t *>(dst + (u64)l * a.pl_ls) = w;
                                else if constexpr (G == 2) *reinterpret_cast<uint16_t *>(dst + (u64)l * a.pl_ls) = (uint16_t)w;
                                else dst[(u64)l * a.pl_ls] = (uint8_t)w;
                            }
                        } else if constexpr (G == 1) {
                            emit_planes(dst - xq, v[0], xq, a.pl_copies, a.pl_nparty * a.pl_ps, a.pl_ls, a.pl_wp);
                        }
                        dst += a.pl_ps;
                    }
                }
            }
        }
    }
    if (a.fail && bad) atomicAdd(a.fail, bad);
}


static u64 mulmod_host(u64 a, u64 b, u64 p) { return (u64)((unsigned __int128)a * b % p); }

// 1 if the caller's protocol constants are the ones the kernels were compiled with: the default
// prime, party ids 1..n, R^T rows (rt[t*M + j] = R[j][t]) and RS rows (ext[(t-K)*K + i]).  Other
// id sets / primes run the unfused kernels (ssn_chain_supported says so up front).
template <int K, int N>
int check_consts(const u64 *ids, const u64 *rt, const u64 *ext, u64 p) {
    using CC = ChainConsts<K, N>;
    constexpr int M = 2 * K - 1;
    const SsnField f = ssn_make_field(p);
    if (p != PP || !f.pm || !f.near) return 0;      // kernels are specialised to the default prime
    for (int t = 0; t < N; t++)
        if (ids[t] != (u64)(t + 1)) return 0;
    if (rt)
        for (int t = 0; t < N; t++)
            for (int j = 0; j < M; j++)
                if (rt[(u64)t * M + j] != mulmod_host(cmod(CC::rt(t, j)), CC::rt_dinv(t), p)) return 0;
    if (ext)
        for (int t = K; t < N; t++)
            for (int i = 0; i < K; i++)
                if (ext[(u64)(t - K) * K + i] != cmod(CC::ext(t, i))) return 0;
    return 1;
}

// Grid cap for the grid-stride chain kernels: SSN_CHAIN_WAVES (default 8) x the resident-block
// capacity of the device (occupancy API, cached per kernel).  Measured on ResNet-152 5PC: 1 wave
// (persistent) 168.8 img/s, 2: 173.4, 4: 176.5, 8: 178.2, 16: 177.9, 64: 175.4 -- short blocks
// in several waves balance the SMs better than one long persistent block each.
template <typename KernT>
static u64 chain_grid_cap(KernT kern, int threads) {
    // cached per (kernel, block size, device): the plain / nonlinear / split instantiations share
    // one function-pointer TYPE but not their occupancy
    struct Entry {
        const void *fn;
        int threads, dev;
        u64 cap;
    };
    static Entry cache[32];
    static int used = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    for (int e = 0; e < used; e++)
        if (cache[e].fn == (const void *)kern && cache[e].threads == threads && cache[e].dev == dev)
            return cache[e].cap;
    int nsm = 0, per_sm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    // shared-memory carveout: the driver's default leaves the L1 large enough to keep the
    // nonlinearity's G-strided scratch loads (G = 4 kernels -11%, step +1%); SSN_CHAIN_CARVEOUT=1
    // asks for the maximum (a 185 KB share-GEMM CTA then co-resides without an SM reconfiguration)
    static const int carve = getenv("SSN_CHAIN_CARVEOUT") ? atoi(getenv("SSN_CHAIN_CARVEOUT")) : 0;
    if (carve) ssn_prefer_max_smem(kern);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, 0) != cudaSuccess || per_sm < 1)
        per_sm = 4;
    const char *env = getenv("SSN_CHAIN_WAVES");
    int waves = env ? atoi(env) : 8;
    if (waves < 1) waves = 1;
    const u64 cap = (u64)nsm * per_sm * waves;
    if (used < 32) cache[used++] = Entry{(const void *)kern, threads, dev, cap};
    return cap;
}

// Windows per output group of the nonlinearity kernel: G adjacent windows share one G-byte
// limb-plane store and one 16-byte share store, when every G-group stays inside a plane row
// (G | OW) or a contiguous channel plane (1x1 layout, G | OH*OW) and all strides keep it aligned.
static int nonlin_group(const ChainArgs &a, const ssn_chain_desc *d, u64 n_out) {
    const u64 oh = d->h / d->kh, ow = d->w / d->kw;
    static const int gmax = getenv("SSN_NONLIN_GMAX") ? atoi(getenv("SSN_NONLIN_GMAX")) : 4;
    for (int g = 4; g > 1; g /= 2) {
        if (g > gmax || WPT % g || n_out % g || a.out_ps % 2 || ((uintptr_t)a.out & 15)) continue;
        if (a.planes) {
            const bool rows = ow % g == 0;
            const bool contig = (u64)a.pl_wp == ow && a.pl_is == oh * ow && (oh * ow) % g == 0;
            // the row pitch matters only when groups stay inside rows; a contiguous channel plane
            // (1x1 layout) needs only the group start aligned (pix0 % g == 0)
            if (!(rows || contig) || a.pl_copies != 1 || a.pl_ps % g || a.pl_ls % g || a.pl_cs % g ||
                a.pl_is % g || (!contig && (u64)a.pl_wp % g) || ((uintptr_t)a.planes % g))
                continue;
        }
        return g;
    }
    return 1;
}

template <int K, int N, bool SPLIT, bool HF, int G>
static void launch_nonlin(const ChainArgs &a, const SsnField &f, u64 n_out, cudaStream_t st) {
    u64 blocks = (n_out + CHAIN_THREADS * WPT - 1) / (CHAIN_THREADS * WPT);
    const u64 cap = chain_grid_cap(k_chain_nonlin<K, N, SPLIT, HF, G>, CHAIN_THREADS);
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    SSN_COUNT_LAUNCH();
    k_chain_nonlin<K, N, SPLIT, HF, G><<<(unsigned)blocks, CHAIN_THREADS, 0, st>>>(a, f);
}

// the kernel launches of one chain (HF: host-fed reference-stream masks)
template <int K, int N, bool HF>
int launch_kernels(const ChainArgs &a, const SsnField &f, const ssn_chain_desc *d,
                   cudaStream_t st) {
    if (!d->nonlin) {
        u64 blocks = (a.nel + PLAIN_THREADS - 1) / PLAIN_THREADS;
        const u64 cap = chain_grid_cap(k_chain_plain<K, N, HF>, PLAIN_THREADS);
        if (blocks > cap) blocks = cap;
        SSN_COUNT_LAUNCH();
        k_chain_plain<K, N, HF><<<(unsigned)blocks, PLAIN_THREADS, 0, st>>>(a, f);
    } else {
        const u64 n_out = (u64)d->nb * d->c * (d->h / d->kh) * (d->w / d->kw);
        const bool split = d->scratch || d->nonlin_only;
        const int G = split ? nonlin_group(a, d, n_out) : 1;
        if (getenv("SSN_DEBUG"))
            fprintf(stderr, "chain nonlin G=%d c=%d h=%d w=%d kh=%d planes=%d wp=%d is=%llu copies=%d\n", G, d->c, d->h,
                    d->w, d->kh, a.planes != nullptr, a.pl_wp, (unsigned long long)a.pl_is, a.pl_copies);
        // SSN_CHAIN_CHUNK=E: element-wise chains (no pooling window, no gather) in chunks of E
        // elements -- plain(chunk) then nonlinearity(chunk), the scratch round trip staying in L2.
        // Off by default: measured slower (2^21: 263.9 vs 264.0 img/s, 2^20: 252.4, 2^19: 230.6;
        // the chunks' partial waves cost more than the L2 hits save)
        const bool chunkable = split && !d->nonlin_only && d->kh == 1 && d->kw == 1 && !d->gather;
        static const u64 chunk_env = getenv("SSN_CHAIN_CHUNK") ? strtoull(getenv("SSN_CHAIN_CHUNK"), nullptr, 10) : 0;
        const u64 span = (u64)CHAIN_THREADS * WPT;
        const u64 chunk = chunkable && chunk_env ? (chunk_env + span - 1) / span * span : a.nel;
        for (u64 lo = 0; lo < (chunkable ? a.nel : 1); lo += chunk) {
            const u64 hi = chunkable ? (lo + chunk < a.nel ? lo + chunk : a.nel) : a.nel;
            if (split && !d->nonlin_only) {
                // split: reshare + truncation (+ add) into scratch [n][nel], then the nonlinearity
                ChainArgs a1 = a;
                a1.out = d->scratch;
                a1.out_ps = a.nel;
                a1.planes = nullptr;
                a1.r_lo = (uint32_t)(chunkable ? lo : 0);
                a1.r_hi = (uint32_t)(chunkable ? hi : a.nel);
                u64 b1 = (a1.r_hi - a1.r_lo + PLAIN_THREADS - 1) / PLAIN_THREADS;
                const u64 cap1 = chain_grid_cap(k_chain_plain<K, N, HF>, PLAIN_THREADS);
                if (b1 > cap1) b1 = cap1;
                if (b1 < 1) b1 = 1;
                SSN_COUNT_LAUNCH();
                k_chain_plain<K, N, HF><<<(unsigned)b1, PLAIN_THREADS, 0, st>>>(a1, f);
            }
            ChainArgs a2 = a;
            if (split && !d->nonlin_only) {
                a2.acc = d->scratch;
                a2.acc_ps = a.nel;
            }
            a2.r_lo = (uint32_t)(chunkable ? lo : 0);
            a2.r_hi = chunkable ? (uint32_t)hi : 0xffffffffu;
            const u64 nwin = chunkable ? hi - lo : n_out;
            // a standalone masked nonlinearity (nonlin_only): acc holds the n parties' input shares
            if (split) {
                if (G == 4) launch_nonlin<K, N, true, HF, 4>(a2, f, nwin, st);
                else if (G == 2) launch_nonlin<K, N, true, HF, 2>(a2, f, nwin, st);
                else launch_nonlin<K, N, true, HF, 1>(a2, f, nwin, st);
            } else {
                launch_nonlin<K, N, false, HF, 1>(a2, f, nwin, st);
            }
        }
    }
    return cudaGetLastError() == cudaSuccess ? 0 : SSN_ERR_CUDA;
}

template <int K, int N>
int launch_chain(const ssn_chain_desc *d, cudaStream_t st) {
    const u64 p = d->p;
    // the protocol constants depend only on (ids, R, RS rows, p): checked against the compiled
    // ones only when they change -- host time per launch matters, a ResNet-152 step makes ~300
    // launches
    constexpr int M = 2 * K - 1;
    struct Key {
        u64 ids[N], rt[N * M], ext[N * K], p;
        int has_ext;
    };
    static thread_local Key last_key;
    static thread_local bool have = false;
    Key key;
    memset(&key, 0, sizeof(key));
    for (int t = 0; t < N; t++) key.ids[t] = d->ids[t];
    for (int t = 0; t < N * M; t++) key.rt[t] = d->rt[t];
    key.has_ext = d->ext != nullptr;
    if (d->ext)
        for (int t = 0; t < (N - K) * K; t++) key.ext[t] = d->ext[t];
    key.p = p;
    if (!have || memcmp(&key, &last_key, sizeof(key)) != 0) {
        if (!check_consts<K, N>(d->ids, d->rt, d->ext, p)) {
            have = false;
            return SSN_ERR_UNSUPPORTED;
        }
        last_key = key;
        have = true;
    }
    const SsnField f = ssn_make_field(p);
    ChainArgs a;
    a.acc = d->acc;
    a.acc_ps = d->acc_pstride;
    a.bias = d->bias;
    a.bias_ps = d->bias_pstride;
    a.bias_div = make_fastdiv((uint32_t)d->bias_div);
    a.bias_mod = make_fastdiv((uint32_t)d->bias_mod);
    if (d->nonlin) {
        const uint32_t ohh = (uint32_t)(d->h / d->kh), oww = (uint32_t)(d->w / d->kw);
        a.f_chw = make_fastdiv((uint32_t)d->c * ohh * oww);
        a.f_hw = make_fastdiv(ohh * oww);
        a.f_ow = make_fastdiv(oww);
    }
    a.other = d->other;
    a.other_ps = d->other_pstride;
    a.out = d->out;
    a.out_ps = d->out_pstride;
    a.nel = d->nel;
    a.nout = d->nout;
    a.senders = d->verify ? N : K;
    a.relu = d->relu;
    a.pool_kind = d->pool_kind;
    a.c = d->c;
    a.h = d->h;
    a.w = d->w;
    a.kh = d->kh;
    a.kw = d->kw;
    a.fan = d->fan;
    a.nb = d->nb;
    a.r = d->r;
    a.d = d->d;
    a.lo = -d->value_bound + d->r * d->d;
    a.neglo_mod = a.lo <= 0 ? (u64)(-a.lo) % p : (p - (u64)a.lo % p) % p;
    a.rshift = -1;
    if ((d->r & (d->r - 1)) == 0) {
        a.rshift = 0;
        while ((1ll << a.rshift) < d->r) a.rshift++;
    }
    a.stepm = (u64)(((unsigned __int128)(u64)(d->r * d->d)) % p);
    a.emax = d->emax;
    a.bmax = d->bmax;
    a.pseed = d->party_seed;
    a.pstream = d->party_stream;
    a.sseed = d->src_seed;
    a.sstream = d->src_stream;
    a.fail = d->verify ? d->fail : nullptr;
    a.fault_rank = d->fault_rank;
    a.planes = d->planes;
    a.pl_ps = d->plane_pstride;
    a.pl_ls = d->plane_lstride;
    a.pl_cs = d->plane_cstride;
    a.pl_is = d->plane_istride;
    a.pl_wp = d->plane_wp;
    a.pl_copies = d->plane_copies;
    a.pl_nparty = d->plane_nparty;
    a.inv_table = (d->nonlin && d->inv_table && d->inv_table_len > d->bmax) ? d->inv_table : nullptr;
    const bool hf = d->host_masks != 0;
    a.h_zero = d->h_zero;
    a.h_alpha = d->h_alpha;
    a.h_comp = d->h_comp;
    a.h_tcoef = d->h_tcoef;
    a.h_beta = d->h_beta;
    a.h_binv = d->h_binv;
    a.per = d->h_period;
    a.per_out = d->h_period_out;
    a.per_in = d->h_period_in ? d->h_period_in : d->h_period;
    a.gather = d->gather;
    a.r_lo = 0;
    a.r_hi = 0xffffffffu;
    a.gh = d->gather_h;
    a.gw = d->gather_w;
    a.gs = d->gather_stride;
    a.gp = d->gather_pad;
    if (hf) {
        if (a.per < 1 || a.per >= (1ull << 32) || a.nel % a.per) return SSN_ERR_ARG;
        if (!d->nonlin_only && (!a.h_zero || !a.h_alpha || !a.h_comp || (K > 1 && !a.h_tcoef))) return SSN_ERR_ARG;
        if (d->nonlin && (!a.h_beta || !a.h_binv || a.per_out < 1 || a.per_out >= (1ull << 32))) return SSN_ERR_ARG;
        a.f_per = make_fastdiv((uint32_t)a.per);
        a.f_per_out = make_fastdiv((uint32_t)(a.per_out ? a.per_out : 1));
        if (a.per_in < 1 || a.per_in >= (1ull << 32)) return SSN_ERR_ARG;
        a.f_per_in = make_fastdiv((uint32_t)a.per_in);
        a.inv_table = nullptr;
    }
    if (a.planes && (!d->nonlin || a.pl_copies < 1 || a.pl_nparty < 1 || a.pl_nparty > N)) return SSN_ERR_ARG;
    if (a.senders > a.nout) return SSN_ERR_ARG;
    return hf ? launch_kernels<K, N, true>(a, f, d, st) : launch_kernels<K, N, false>(a, f, d, st);
}

template <int K, int N>
int supported(const u64 *ids, u64 p) {
    return check_consts<K, N>(ids, nullptr, nullptr, p);
}

}  // namespace

namespace {
// inverse table of [0, n): 1024 consecutive entries per thread by Montgomery's batch trick
// (one Fermat inversion per thread), table[0] = 0
__global__ void k_inv_table(u64 *__restrict__ t, u64 n) {
    constexpr int G = 64;
    const u64 start = (blockIdx.x * (u64)blockDim.x + threadIdx.x) * G;
    if (start >= n) return;
    u64 pre[G];
    u64 run = 1;
    for (int g = 0; g < G; g++) {
        const u64 b = start + g;
        pre[g] = run;
        if (b > 0 && b < n) run = mulm_hs(run, b);
    }
    u64 inv = canon(invm(canon(run)));
    for (int g = G - 1; g >= 0; g--) {
        const u64 b = start + g;
        if (b >= n) continue;
        if (b == 0) {
            t[b] = 0;
            continue;
        }
        t[b] = canon(mulm_hs(inv, pre[g]));
        inv = mulm_hs(inv, b);
    }
}
}  // namespace

extern "C" int ssn_inv_table(uint64_t *table, uint64_t n, uint64_t p, void *stream) {
    if (!table || n == 0 || n > (1ull << 32)) return SSN_ERR_ARG;
    if (p != PP) return SSN_ERR_UNSUPPORTED;
    const u64 threads = (n + 63) / 64;
    SSN_COUNT_LAUNCH();
    k_inv_table<<<(unsigned)((threads + 255) / 256), 256, 0, (cudaStream_t)stream>>>(table, n);
    return cudaGetLastError() == cudaSuccess ? 0 : SSN_ERR_CUDA;
}

extern "C" int ssn_chain_supported(int k, int n, const uint64_t *ids, uint64_t p) {
    if (!ids) return 0;
    if (k == 2 && n == 3) return supported<2, 3>(ids, p);
    if (k == 3 && n == 5) return supported<3, 5>(ids, p);
    if (k == 4 && n == 7) return supported<4, 7>(ids, p);
    return 0;
}

extern "C" int ssn_layer_chain(const ssn_chain_desc *d, void *stream) {
    if (!d || !d->acc || !d->out || !d->ids || !d->rt) return SSN_ERR_ARG;
    if (d->nonlin_only && !d->nonlin) return SSN_ERR_ARG;
    if (!d->nonlin_only && (!d->bias || d->r < 1 || d->d < 1 || d->emax < 1 || d->nout < d->k || d->nout > d->n))
        return SSN_ERR_ARG;
    if (d->verify && (!d->ext || d->nout != d->n)) return SSN_ERR_ARG;
    if (d->nel >= (1ull << 32) || d->bias_div < 1 || d->bias_mod < 1 || d->bias_div >= (1ull << 32) ||
        d->bias_mod >= (1ull << 32))
        return SSN_ERR_UNSUPPORTED;
    if (d->nonlin) {
        if (d->kh < 1 || d->kw < 1 || d->h % d->kh || d->w % d->kw || d->bmax < 1 || d->fan < 1 || d->fan > d->n ||
            d->pool_kind < 0 || d->pool_kind > 2 || (d->pool_kind == 0 && (d->kh != 1 || d->kw != 1)))
            return SSN_ERR_ARG;
        if (d->gather) {
            // gathered windows need the split (scratch) form: the chain output is read per tap
            if ((!d->scratch && !d->nonlin_only) || d->gather_h < 1 || d->gather_w < 1 || d->gather_stride < 1 ||
                d->gather_pad < 0 || (u64)d->nb * d->c * d->gather_h * d->gather_w != d->nel || d->kh < 1 ||
                d->kw < 1 || d->h % d->kh || d->w % d->kw)
                return SSN_ERR_ARG;
        } else if ((u64)d->nb * d->c * d->h * d->w != d->nel) {
            return SSN_ERR_ARG;
        }
    }
    if (d->nel == 0) return 0;
    cudaStream_t st = (cudaStream_t)stream;
    if (d->k == 2 && d->n == 3) return launch_chain<2, 3>(d, st);
    if (d->k == 3 && d->n == 5) return launch_chain<3, 5>(d, st);
    if (d->k == 4 && d->n == 7) return launch_chain<4, 7>(d, st);
    return SSN_ERR_UNSUPPORTED;
}
