/*
 * ssn_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C CPU restatement of the SSNet reference's hot-path arithmetic
 * (reference = /root/reference/pkg/src/ssnet, a pure-Python numpy package;
 * paths below are relative to that directory).  It exists to CHECK the CUDA
 * product path, never to be it: only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.
 *
 * Parity pinning: every function here is checked against golden vectors
 * produced by importing the reference itself (tests/golden/make_golden.py ->
 * tests/golden/*.npz) in tests/test_oracle.py.
 *
 * Field elements are canonical uint64 in [0, p) with p < 2^57
 * (S/field.py:64-75 enforces p < 2^64 and 2*bits+13 <= 128).  All products use
 * unsigned __int128 so every intermediate is exact, like the reference's Python
 * bignums inside dtype=object arrays (S/field.py:1-16).
 */
#include <stdint.h>
#include <stddef.h>
#include <string.h>
#include <stdlib.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef uint64_t u64;
typedef int64_t i64;
typedef unsigned __int128 u128;

static inline u64 mulmod(u64 a, u64 b, u64 p) { return (u64)(((u128)a * b) % p); }
static inline u64 addmod(u64 a, u64 b, u64 p) { u64 s = a + b; return s >= p ? s - p : s; }
static inline u64 submod(u64 a, u64 b, u64 p) { return a >= b ? a - b : a + p - b; }

/* Python floor division / floor modulo on int64 (S/layers.py:305 uses `//`). */
static inline i64 floordiv(i64 a, i64 b) {
    i64 q = a / b;
    if ((a % b != 0) && ((a < 0) != (b < 0))) q -= 1;
    return q;
}

int ssn_o_version(void) { return 1; }

/* PrimeField.mul (S/field.py:98-99), scalar. */
u64 ssn_o_mulmod(u64 a, u64 b, u64 p) { return mulmod(a % p, b % p, p); }

/* PrimeField._inv_int (S/field.py:104-116): extended Euclid. 0 -> returns 0 (caller raises). */
u64 ssn_o_inv(u64 a, u64 p) {
    a %= p;
    if (a == 0) return 0;
    __int128 lm = 1, hm = 0, low = a, high = p;
    while (low > 1) {
        __int128 r = high / low;
        __int128 nm = hm - lm * r, nw = high - low * r;
        hm = lm; high = low; lm = nm; low = nw;
    }
    __int128 v = lm % (__int128)p;
    if (v < 0) v += p;
    return (u64)v;
}

/* Elementwise add/sub/mul with optional scalar broadcast of b (b_len==1).
 * share_add/share_sub/share_mul (S/sss.py:238-276), PrimeField.add/sub/mul (S/field.py:89-99). */
void ssn_o_ewise(int op, const u64 *a, const u64 *b, size_t b_len, u64 *out, size_t n, u64 p) {
#ifdef _OPENMP
#pragma omp parallel for schedule(static) if (n > 4096)
#endif
    for (size_t i = 0; i < n; i++) {
        u64 x = a[i], y = b[b_len == 1 ? 0 : i];
        out[i] = op == 0 ? addmod(x, y, p) : op == 1 ? submod(x, y, p) : mulmod(x, y, p);
    }
}

/* SssScheme.gen with explicit coefficients (S/sss.py:118-147):
 * share(id) = s + sum_j c_j * id^j, coefficient tensors in draw order c_1..c_{k-1}.
 * coeffs: (km1, n) row-major; ids: nids party ids; out: (nids, n). */
void ssn_o_gen(const u64 *secret, const u64 *coeffs, int km1, const u64 *ids, int nids,
               u64 *out, size_t n, u64 p) {
    for (int t = 0; t < nids; t++) {
        u64 pid = ids[t] % p;
#ifdef _OPENMP
#pragma omp parallel for schedule(static) if (n > 4096)
#endif
        for (size_t i = 0; i < n; i++) {
            u64 acc = secret[i], pw = 1;
            for (int j = 0; j < km1; j++) {
                pw = mulmod(pw, pid, p);
                acc = addmod(acc, mulmod(coeffs[(size_t)j * n + i], pw, p), p);
            }
            out[(size_t)t * n + i] = acc;
        }
    }
}

/* SssScheme.rec (S/sss.py:172-194): sum_i w_i * s_i over the first m shares.
 * shares: (m, n); weights: m Lagrange weights for the shares' party ids. */
void ssn_o_rec(const u64 *shares, const u64 *w, int m, u64 *out, size_t n, u64 p) {
#ifdef _OPENMP
#pragma omp parallel for schedule(static) if (n > 4096)
#endif
    for (size_t i = 0; i < n; i++) {
        u64 acc = 0;
        for (int j = 0; j < m; j++) acc = addmod(acc, mulmod(shares[(size_t)j * n + i], w[j], p), p);
        out[i] = acc;
    }
}

/* reshare_degree_reduce step 2 (S/protocol.py:176-178): rows = R^T[:out] @ stack mod p.
 * stack: (m, n) sub-shares ascending by source rank; Rt: (nout, m) = R^T rows; out: (nout, n). */
void ssn_o_reduce_apply(const u64 *stack, const u64 *Rt, int m, int nout, u64 *out, size_t n, u64 p) {
    for (int t = 0; t < nout; t++)
#ifdef _OPENMP
#pragma omp parallel for schedule(static) if (n > 4096)
#endif
        for (size_t i = 0; i < n; i++) {
            u128 acc = 0;
            for (int j = 0; j < m; j++) acc += (u128)Rt[t * m + j] * stack[(size_t)j * n + i];
            out[(size_t)t * n + i] = (u64)(acc % p);
        }
}

/* sss_linear's local product (S/layers.py:245-255): C(M,N) = A(M,K) @ B(K,N) mod p,
 * exact, with a u128 accumulator reduced every 2^12 terms (products < 2^114). */
/* OpenMP team size for every later parallel region (torchrun exports OMP_NUM_THREADS=1 to
 * each rank; the CPU baseline should use all host cores); returns the effective size */
int ssn_o_set_threads(int threads) {
    if (threads > 0) omp_set_num_threads(threads);
    return omp_get_max_threads();
}

void ssn_o_gemm(const u64 *A, const u64 *B, u64 *C, int M, int N, int K, u64 p, int threads) {
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (int i = 0; i < M; i++) {
        u128 *acc = (u128 *)calloc((size_t)N, sizeof(u128));
        const u64 *arow = A + (size_t)i * K;
        for (int k = 0; k < K; k++) {
            u64 a = arow[k];
            if (a == 0) continue;
            const u64 *brow = B + (size_t)k * N;
            for (int j = 0; j < N; j++) acc[j] += (u128)a * brow[j];
            if ((k & 4095) == 4095)
                for (int j = 0; j < N; j++) acc[j] %= p;
        }
        for (int j = 0; j < N; j++) C[(size_t)i * N + j] = (u64)(acc[j] % p);
        free(acc);
    }
}

/* im2col (S/model.py:354-371): unfold (c,h,w) into (c*kh*kw, oh*ow) with zero padding.
 * Works on uint64 field elements or int64 plaintext (same bit width). */
void ssn_o_im2col(const u64 *x, int c, int h, int w, int kh, int kw, int stride, int pad, u64 *cols) {
    int oh = (h + 2 * pad - kh) / stride + 1, ow = (w + 2 * pad - kw) / stride + 1;
    for (int ci = 0; ci < c; ci++)
        for (int i = 0; i < kh; i++)
            for (int j = 0; j < kw; j++) {
                size_t row = ((size_t)ci * kh + i) * kw + j;
                for (int y = 0; y < oh; y++)
                    for (int xx = 0; xx < ow; xx++) {
                        int sy = y * stride + i - pad, sx = xx * stride + j - pad;
                        u64 v = 0;
                        if (sy >= 0 && sy < h && sx >= 0 && sx < w) v = x[((size_t)ci * h + sy) * w + sx];
                        cols[row * (size_t)(oh * ow) + (size_t)y * ow + xx] = v;
                    }
            }
}

/* round_half_away (S/model.py:44-50). */
static inline i64 round_half_away1(i64 v, i64 d) {
    i64 a = v < 0 ? -v : v;
    i64 q = floordiv(2 * a + d, 2 * d);
    return v < 0 ? -q : q;
}
void ssn_o_round_half_away(const i64 *v, i64 d, i64 *out, size_t n) {
    for (size_t i = 0; i < n; i++) out[i] = round_half_away1(v[i], d);
}

/* Elite side of sss_truncation (S/layers.py:277-315): from the k masked shares (ranks 1..k,
 * front ids, weights w) reconstruct v, window-decode into [lo, lo+p) with
 * lo = -value_bound + r*d (S/layers.py:231-233,288), floor-divide by r, round half away by d
 * when d>1, and return t mod p (the secret the elite re-shares). */
void ssn_o_trunc_elite(const u64 *masked, const u64 *w, int k, i64 value_bound, i64 r, i64 d,
                       u64 *t_out, size_t n, u64 p) {
    i64 lo = -value_bound + r * d;
#ifdef _OPENMP
#pragma omp parallel for schedule(static) if (n > 4096)
#endif
    for (size_t i = 0; i < n; i++) {
        u64 v = 0;
        for (int j = 0; j < k; j++) v = addmod(v, mulmod(masked[(size_t)j * n + i], w[j], p), p);
        /* ((v - lo) mod p) + lo, v in [0,p), -lo may be up to ~2^44 */
        __int128 s = ((__int128)v - lo) % (__int128)p;
        if (s < 0) s += p;
        i64 shifted = (i64)s + lo;
        i64 t = floordiv(shifted, r);
        if (d > 1) t = round_half_away1(t, d);
        __int128 tm = (__int128)t % (__int128)p;
        if (tm < 0) tm += p;
        t_out[i] = (u64)tm;
    }
}

/* Elite side of sss_nonlinear (S/layers.py:345-364): reconstruct from m = 2k-1 masked
 * product shares, decode_signed (S/field.py:130-134), ReLU, non-overlapping window max or sum
 * over (c, h/kh, kh, w/kw, kw) (S/model.py:374-377), encode_signed.
 * pool_kind: 0 none, 1 max, 2 sum.  in shape (c,h,w) (c*h*w == n_in when pooling).
 * plain_out has n_out elements. */
void ssn_o_nonlin_elite(const u64 *masked, const u64 *w, int m, int relu, int pool_kind,
                        int c, int h, int wd, int kh, int kw, size_t n_in, u64 *plain_out, u64 p) {
    u64 half = (p - 1) / 2;
    i64 *ints = (i64 *)malloc(n_in * sizeof(i64));
    for (size_t i = 0; i < n_in; i++) {
        u64 v = 0;
        for (int j = 0; j < m; j++) v = addmod(v, mulmod(masked[(size_t)j * n_in + i], w[j], p), p);
        i64 s = v > half ? (i64)v - (i64)p : (i64)v;
        if (relu && s <= 0) s = 0;
        ints[i] = s;
    }
    if (pool_kind == 0) {
        for (size_t i = 0; i < n_in; i++) plain_out[i] = ints[i] < 0 ? (u64)((i64)p + ints[i]) : (u64)ints[i];
    } else {
        int oh = h / kh, ow = wd / kw;
        for (int ci = 0; ci < c; ci++)
            for (int y = 0; y < oh; y++)
                for (int x = 0; x < ow; x++) {
                    i64 acc = pool_kind == 1 ? INT64_MIN : 0;
                    for (int i = 0; i < kh; i++)
                        for (int j = 0; j < kw; j++) {
                            i64 v = ints[((size_t)ci * h + y * kh + i) * wd + x * kw + j];
                            if (pool_kind == 1) { if (v > acc) acc = v; } else acc += v;
                        }
                    size_t o = ((size_t)ci * oh + y) * ow + x;
                    plain_out[o] = acc < 0 ? (u64)((i64)p + acc) : (u64)acc;
                }
    }
    free(ints);
}

/* Plaintext integer engine pieces (S/model.py:380-421), int64. */
void ssn_o_plain_gemm_i64(const i64 *A, const i64 *B, i64 *C, int M, int N, int K, int threads) {
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (int i = 0; i < M; i++) {
        i64 *crow = C + (size_t)i * N;
        memset(crow, 0, (size_t)N * sizeof(i64));
        for (int k = 0; k < K; k++) {
            i64 a = A[(size_t)i * K + k];
            if (!a) continue;
            const i64 *brow = B + (size_t)k * N;
            for (int j = 0; j < N; j++) crow[j] += a * brow[j];
        }
    }
}

/* plaintext truncation step (S/model.py:406-410): floor(x / r), then round_half_away(., d). */
void ssn_o_plain_trunc(const i64 *x, i64 r, i64 d, i64 *out, size_t n) {
    for (size_t i = 0; i < n; i++) {
        i64 t = floordiv(x[i], r);
        out[i] = d > 1 ? round_half_away1(t, d) : t;
    }
}

/* Vectorised PrimeField.inv (S/field.py:101-116) for the trusted-source beta^-1. */
void ssn_o_inv_vec(const u64 *a, u64 *out, size_t n, u64 p) {
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
    for (size_t i = 0; i < n; i++) out[i] = ssn_o_inv(a[i], p);
}
