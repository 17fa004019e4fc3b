// ssn_elementwise.cu -- HBM-bound field kernels of the SSNet hot path (sm_100a) + C-ABI.
//
// Every kernel is a grid-stride loop with one thread per element per iteration (coalesced
// u64 loads/stores); multi-party operands are strided 2-D views base + b*stride_b + j*stride_j
// so one launch covers all co-resident parties.  Loops over parties / points / coefficients
// are fully unrolled against compile-time maxima with runtime guards, so every per-element
// temporary lives in registers (no local-memory stack).
// Reference functions restated (paths relative to /root/reference/pkg/src/ssnet):
//   ssn_ewise            share_add/sub/mul, PrimeField.add/sub/mul     S/sss.py:238-276, S/field.py:89-99
//   ssn_gen              SssScheme.gen (Horner over party ids)         S/sss.py:118-147
//   ssn_rec              SssScheme.rec (Lagrange weighted sum)          S/sss.py:172-194
//   ssn_reduce_apply     reshare step 2, R^T @ stack                    S/protocol.py:165-185
//   ssn_reshare_finish   reshare step 3 + rerand + bias (+ trunc mask)  S/protocol.py:187-198, S/layers.py:260-267,290-293
//   ssn_trunc_elite      masked truncation at the elite (+ fresh shares, + RS check)  S/layers.py:295-315
//   ssn_nonlin_elite     masked ReLU / max / sum pool at the elite      S/layers.py:345-364
//   ssn_mask_*           trusted-source masks                           S/masks.py:39-96, S/protocol.py:354-388
#include <cstdlib>
#include "ssn_field.cuh"
#include "ssn.h"
#include "ssn_lincomb.cuh"
#include "ssn_p45.cuh"

// blocks per SM of the grid-stride elementwise kernels (SSN_EW_BLOCKS_PER_SM, default 64:
// 16 -> 64 measured +2-5% on gen / R-apply / the elites)
static u64 ssn_ew_cap() {
    static u64 cap = 0;
    if (!cap) {
        const char *e = getenv("SSN_EW_BLOCKS_PER_SM");
        const int per = e && atoi(e) > 0 ? atoi(e) : 64;
        cap = 148ull * per;
    }
    return cap;
}

static int ssn_blocks(u64 n, int threads = 256) {
    u64 b = (n + threads - 1) / threads;
    const u64 cap = ssn_ew_cap();
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return (int)b;
}

// 2-D grid: y = batch (party / front rank), x = grid-stride over the n elements of one batch
static dim3 ssn_grid2(u64 n, int nb) {
    u64 x = (n + 255) / 256;
    u64 cap = ssn_ew_cap() / (u64)nb;
    if (cap < 1) cap = 1;
    if (x > cap) x = cap;
    if (x < 1) x = 1;
    return dim3((unsigned)x, (unsigned)nb);
}

static inline int ssn_check_launch() {
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : SSN_ERR_CUDA;
}

// ------------------------------------------------------------------ ewise
__global__ void k_ewise(int op, int mode, const u64 *__restrict__ a, const u64 *__restrict__ b,
                        u64 *__restrict__ out, u64 n, u64 b_div, u64 b_mod, u64 b_div2, u64 b_mul2, SsnField f) {
    const u64 row0 = mode == 2 ? (u64)blockIdx.y * b_mod : 0;     // cyclic mode: one row per grid.y
    const u64 lim = mode == 2 ? row0 + b_mod : n;
    for (u64 i = row0 + blockIdx.x * (u64)blockDim.x + threadIdx.x; i < lim; i += (u64)gridDim.x * blockDim.x) {
        u64 x = a[i];
        u64 y;
        if (mode == 0) y = b[i];                                   // full
        else if (mode == 1) y = b[0];                              // scalar
        else if (mode == 2) y = b[i - row0];                       // cyclic: row blockIdx.y
        else if (mode == 3) y = 0;                                 // neg
        else y = b[(i / b_div) % b_mod + (i / b_div2) * b_mul2];   // general strided broadcast
        u64 r;
        if (op == 0) r = ssn_addmod(x, y, f.p);
        else if (op == 1) r = ssn_submod(x, y, f.p);
        else if (op == 2) r = ssn_mulmod(x, y, f);
        else r = x ? f.p - x : 0;
        out[i] = r;
    }
}

extern "C" int ssn_ewise(int op, const u64 *a, const u64 *b, u64 *out, u64 n, u64 b_div, u64 b_mod,
                         u64 b_div2, u64 b_mul2, u64 p, void *stream) {
    if (op < 0 || op > 3 || b_div == 0 || b_mod == 0 || b_div2 == 0) return SSN_ERR_ARG;
    if (n == 0) return 0;
    int mode = 4;
    if (op == 3) mode = 3;
    else if (b_mul2 == 0 && b_div == 1 && b_mod >= n) mode = 0;
    else if (b_mul2 == 0 && b_mod == 1) mode = 1;
    else if (b_mul2 == 0 && b_div == 1 && n % b_mod == 0 && n / b_mod <= 65535) mode = 2;
    dim3 grid = mode == 2 ? ssn_grid2(b_mod, (int)(n / b_mod)) : dim3(ssn_blocks(n));
    SSN_COUNT_LAUNCH();
    k_ewise<<<grid, 256, 0, (cudaStream_t)stream>>>(op, mode, a, b, out, n, b_div, b_mod, b_div2, b_mul2,
                                                    ssn_make_field(p));
    return ssn_check_launch();
}

// ------------------------------------------------------------------ p = 2^45 - 55 fast paths
// rec / R-apply / reshare step 3 with compile-time row lengths and the chain kernels' arithmetic
// (ssn_p45.cuh): non-negative small-rational rows, ONE pseudo-Mersenne fold per row, no sign
// branches.  Same canonical outputs as the generic kernels; taken when every row is small.
template <int M, int NO>
struct P45Rows {
    ssn45::SRow<M> r[NO];
};

template <int M>
__global__ void k_rec_p45(const u64 *__restrict__ pts, u64 p_b, u64 p_j, P45Rows<M, 1> w, u64 *__restrict__ out,
                          u64 o_b, u64 n) {
    const u64 b = blockIdx.y;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u64 *base = pts + b * p_b + i;
        u64 x[M];
#pragma unroll
        for (int j = 0; j < M; j++) x[j] = base[j * p_j];
        out[b * o_b + i] = ssn45::canon(ssn45::lin<M>(x, w.r[0]));
    }
}

template <int M, int NO>
__global__ void k_reduce_apply_p45(const u64 *__restrict__ pts, u64 p_b, u64 p_j, P45Rows<M, NO> R,
                                   u64 *__restrict__ out, u64 o_b, u64 o_t, u64 n) {
    const u64 b = blockIdx.y;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u64 *base = pts + b * p_b + i;
        u64 v[M];
#pragma unroll
        for (int j = 0; j < M; j++) v[j] = base[j * p_j];
        const u64 vs = ssn45::xsum_of<M>(v);
#pragma unroll
        for (int t = 0; t < NO; t++) out[b * o_b + t * o_t + i] = ssn45::canon(ssn45::lin_s<M>(v, vs, R.r[t]));
    }
}

template <int K>
__global__ void k_reshare_finish_p45(const u64 *__restrict__ pts, u64 p_b, u64 p_j, P45Rows<K, 1> w,
                                     const u64 *__restrict__ zero, u64 z_b, const u64 *__restrict__ bias, u64 bi_b,
                                     u64 bias_div, u64 bias_mod, const u64 *__restrict__ alpha, u64 a_b,
                                     u64 *__restrict__ out, u64 o_b, u64 n) {
    const u64 b = blockIdx.y;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u64 *base = pts + b * p_b + i;
        u64 x[K];
#pragma unroll
        for (int j = 0; j < K; j++) x[j] = base[j * p_j];
        u64 acc = ssn45::lin<K>(x, w.r[0]);                      // lazy, < 2^46
        if (zero) acc += zero[b * z_b + i];
        if (bias) {
            const u64 ch = n < (1ull << 32) ? (u64)(((uint32_t)i / (uint32_t)bias_div) % (uint32_t)bias_mod)
                                            : (i / bias_div) % bias_mod;
            acc += bias[b * bi_b + ch];
        }
        if (alpha) acc += alpha[b * a_b + i];
        out[b * o_b + i] = ssn45::canon(acc);                      // < 2^46 + 3 * 2^45
    }
}

// gen with compile-time (k-1, |ids|): the same coefficients as k_gen (host-fed, or the same
// Philox draws), shares s + sum_j c_j id^(j+1) with small id powers, one fold each
template <int KM1, int NIDS>
struct P45Pows {
    uint32_t pw[NIDS][KM1 > 0 ? KM1 : 1];
};

template <int KM1, int NIDS>
__global__ void k_gen_p45(const u64 *__restrict__ secret, u64 s_b, const u64 *__restrict__ coeffs, u64 c_b, u64 seed,
                          u64 stream, P45Pows<KM1, NIDS> pw, u64 *__restrict__ out, u64 o_b, u64 o_t, u64 n,
                          SsnField f) {
    const u64 b = blockIdx.y;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u64 s = secret ? secret[b * s_b + i] : 0;
        u64 c[SSN_MAXK];
        load_coeffs(c, coeffs ? coeffs + b * c_b : nullptr, n, i, KM1, seed, stream + b, f);
#pragma unroll
        for (int t = 0; t < NIDS; t++) {
            u64 acc = s;                                           // < p + 2^45 * sum id^j < 2^64
#pragma unroll
            for (int j = 0; j < KM1; j++) acc += mul_small(c[j], pw.pw[t][j]);
            out[b * o_b + t * o_t + i] = ssn45::canon(acc);
        }
    }
}

// rows[t*m + j] -> small-rational p45 rows; 0 if any row has no small form
template <int M, int NO>
static int p45_rows(P45Rows<M, NO> &R, const u64 *rows, u64 p) {
    if (p != ssn45::PP) return 0;
    for (int t = 0; t < NO; t++)
        if (!ssn45::make_srow<M>(R.r[t], rows + (u64)t * M, M, p)) return 0;
    return 1;
}

// ------------------------------------------------------------------ gen
// out[b][t][i] = secret[b][i] + sum_j c_j[b][i] * ids[t]^(j+1)
__global__ void k_gen(const u64 *__restrict__ secret, u64 s_b, const u64 *__restrict__ coeffs, u64 c_b, u64 seed,
                      u64 stream, int km1, PowTable pw, int nids, u64 *__restrict__ out, u64 o_b, u64 o_t, u64 n,
                      int nb, SsnField f) {
    const u64 b = blockIdx.y;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u64 s = secret ? secret[b * s_b + i] : 0;
        u64 c[SSN_MAXK];
        load_coeffs(c, coeffs ? coeffs + b * c_b : nullptr, n, i, km1, seed, stream + b, f);
#pragma unroll
        for (int t = 0; t < SSN_MAXJ; t++)
            if (t < nids) out[b * o_b + t * o_t + i] = horner_at(s, c, pw, t, km1, f);
    }
}

extern "C" int ssn_gen(const u64 *secret, u64 secret_bstride, const u64 *coeffs, u64 coeff_bstride, u64 seed,
                       u64 stream, int km1, const u64 *ids, int nids, u64 *out, u64 out_bstride, u64 out_tstride,
                       u64 n, int nbatch, u64 p, void *strm) {
    if (km1 < 0 || km1 > SSN_MAXK || nids < 1 || nids > SSN_MAXJ || nbatch < 1) return SSN_ERR_ARG;
    if (n == 0) return 0;
    PowTable pw = make_pows(ids, nids, km1, p);
#define SSN_GEN_P45(KK, NN)                                                                               \
    if (km1 == KK && nids == NN && pw.small && p == ssn45::PP) {                                          \
        P45Pows<KK, NN> q;                                                                                \
        for (int t = 0; t < NN; t++)                                                                      \
            for (int j = 0; j < KK; j++) q.pw[t][j] = (uint32_t)pw.r[t].n[j];                             \
        SSN_COUNT_LAUNCH();                                                                               \
        k_gen_p45<KK, NN><<<ssn_grid2(n, nbatch), 256, 0, (cudaStream_t)strm>>>(                           \
            secret, secret_bstride, coeffs, coeff_bstride, seed, stream, q, out, out_bstride, out_tstride, n, \
            ssn_make_field(p));                                                                           \
        return ssn_check_launch();                                                                        \
    }
    SSN_GEN_P45(1, 2)
    SSN_GEN_P45(1, 3)
    SSN_GEN_P45(2, 3)
    SSN_GEN_P45(2, 5)
#undef SSN_GEN_P45
    SSN_COUNT_LAUNCH();
    k_gen<<<ssn_grid2(n, nbatch), 256, 0, (cudaStream_t)strm>>>(secret, secret_bstride, coeffs, coeff_bstride,
                                                                  seed, stream, km1, pw, nids, out, out_bstride,
                                                                  out_tstride, n, nbatch, ssn_make_field(p));
    return ssn_check_launch();
}

// ------------------------------------------------------------------ rec
__global__ void k_rec(const u64 *__restrict__ pts, u64 p_b, u64 p_j, Weights w, int m, u64 *__restrict__ out,
                      u64 o_b, u64 n, int nb, SsnField f) {
    const u64 b = blockIdx.y;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u64 *base = pts + b * p_b + i;
        u64 x[SSN_MAXJ];
#pragma unroll
        for (int j = 0; j < SSN_MAXJ; j++)
            if (j < m) x[j] = base[j * p_j];
        out[b * o_b + i] = lincomb<SSN_MAXJ>(x, w.r, w.small, m, f);
    }
}

extern "C" int ssn_rec(const u64 *pts, u64 pts_bstride, u64 pts_jstride, const u64 *w, int m, u64 *out,
                       u64 out_bstride, u64 n, int nbatch, u64 p, void *strm) {
    if (m < 1 || m > SSN_MAXJ || nbatch < 1) return SSN_ERR_ARG;
    if (n == 0) return 0;
#define SSN_REC_P45(MM)                                                                                   \
    if (m == MM) {                                                                                        \
        P45Rows<MM, 1> R;                                                                                 \
        if (p45_rows<MM, 1>(R, w, p)) {                                                                   \
            SSN_COUNT_LAUNCH();                                                                           \
            k_rec_p45<MM><<<ssn_grid2(n, nbatch), 256, 0, (cudaStream_t)strm>>>(pts, pts_bstride, pts_jstride, \
                                                                              R, out, out_bstride, n);      \
            return ssn_check_launch();                                                                    \
        }                                                                                                 \
    }
    SSN_REC_P45(2)
    SSN_REC_P45(3)
    SSN_REC_P45(5)
#undef SSN_REC_P45
    Weights W = make_weights(w, m, p);
    SSN_COUNT_LAUNCH();
    k_rec<<<ssn_grid2(n, nbatch), 256, 0, (cudaStream_t)strm>>>(pts, pts_bstride, pts_jstride, W, m, out,
                                                                  out_bstride, n, nbatch, ssn_make_field(p));
    return ssn_check_launch();
}

// ------------------------------------------------------------------ reduce apply (reshare step 2)
// out[b][t][i] = sum_j Rt[t][j] * pts[b][j][i]  -- b = front rank, j = sub-share source, t = out rank
__global__ void k_reduce_apply(const u64 *__restrict__ pts, u64 p_b, u64 p_j, RTable R, int m, int nout,
                               u64 *__restrict__ out, u64 o_b, u64 o_t, u64 n, int nb, SsnField f) {
    const u64 b = blockIdx.y;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u64 *base = pts + b * p_b + i;
        u64 v[SSN_MAXP];
#pragma unroll
        for (int j = 0; j < SSN_MAXP; j++)
            if (j < m) v[j] = base[j * p_j];
#pragma unroll
        for (int t = 0; t < SSN_MAXJ; t++)
            if (t < nout) out[b * o_b + t * o_t + i] = lincomb<SSN_MAXP>(v, R.r[t], R.small, m, f);
    }
}

extern "C" int ssn_reduce_apply(const u64 *pts, u64 pts_bstride, u64 pts_jstride, int m, const u64 *rt, int nout,
                                u64 *out, u64 out_bstride, u64 out_tstride, u64 n, int nbatch, u64 p, void *strm) {
    if (m < 1 || m > SSN_MAXP || nout < 1 || nout > SSN_MAXJ || nbatch < 1) return SSN_ERR_ARG;
    if (n == 0) return 0;
#define SSN_RA_P45(MM, NN)                                                                                \
    if (m == MM && nout == NN) {                                                                          \
        P45Rows<MM, NN> Q;                                                                                \
        if (p45_rows<MM, NN>(Q, rt, p)) {                                                                 \
            SSN_COUNT_LAUNCH();                                                                           \
            k_reduce_apply_p45<MM, NN><<<ssn_grid2(n, nbatch), 256, 0, (cudaStream_t)strm>>>(              \
                pts, pts_bstride, pts_jstride, Q, out, out_bstride, out_tstride, n);                       \
            return ssn_check_launch();                                                                    \
        }                                                                                                 \
    }
    SSN_RA_P45(3, 2)
    SSN_RA_P45(3, 3)
    SSN_RA_P45(5, 3)
    SSN_RA_P45(5, 5)
#undef SSN_RA_P45
    RTable R;
    R.small = 1;
    for (int t = 0; t < SSN_MAXJ; t++) {
        u64 row[SSN_MAXJ] = {0};
        if (t < nout)
            for (int j = 0; j < m; j++) row[j] = rt[t * m + j];
        int ok = make_row(R.r[t], row, m, p);
        if (t < nout) R.small = R.small && ok;
    }
    SSN_COUNT_LAUNCH();
    k_reduce_apply<<<ssn_grid2(n, nbatch), 256, 0, (cudaStream_t)strm>>>(pts, pts_bstride, pts_jstride, R, m, nout,
                                                                           out, out_bstride, out_tstride, n, nbatch,
                                                                           ssn_make_field(p));
    return ssn_check_launch();
}

// ------------------------------------------------------------------ reshare step 3 (+rerand, +bias, +alpha)
__global__ void k_reshare_finish(const u64 *__restrict__ pts, u64 p_b, u64 p_j, Weights w, int k,
                                 const u64 *__restrict__ zero, u64 z_b, const u64 *__restrict__ bias, u64 bi_b,
                                 u64 bias_div, u64 bias_mod, const u64 *__restrict__ alpha, u64 a_b,
                                 u64 *__restrict__ out, u64 o_b, u64 n, int nb, SsnField f) {
    const u64 b = blockIdx.y;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u64 *base = pts + b * p_b + i;
        u64 x[SSN_MAXP];
#pragma unroll
        for (int j = 0; j < SSN_MAXP; j++)
            if (j < k) x[j] = base[j * p_j];
        u64 acc = lincomb<SSN_MAXP>(x, w.r, w.small, k, f);
        if (zero) acc = ssn_addmod(acc, zero[b * z_b + i], f.p);
        if (bias) {
            const u64 ch = n < (1ull << 32) ? (u64)(((uint32_t)i / (uint32_t)bias_div) % (uint32_t)bias_mod)
                                            : (i / bias_div) % bias_mod;
            acc = ssn_addmod(acc, bias[b * bi_b + ch], f.p);
        }
        if (alpha) acc = ssn_addmod(acc, alpha[b * a_b + i], f.p);
        out[b * o_b + i] = acc;
    }
}

extern "C" int ssn_reshare_finish(const u64 *pts, u64 pts_bstride, u64 pts_jstride, const u64 *w, int k,
                                  const u64 *zero, u64 zero_bstride, const u64 *bias, u64 bias_bstride,
                                  u64 bias_div, u64 bias_mod, const u64 *alpha, u64 alpha_bstride, u64 *out,
                                  u64 out_bstride, u64 n, int nbatch, u64 p, void *strm) {
    if (k < 1 || k > SSN_MAXP || nbatch < 1 || bias_div == 0 || bias_mod == 0) return SSN_ERR_ARG;
    if (n == 0) return 0;
#define SSN_RF_P45(KK)                                                                                    \
    if (k == KK) {                                                                                        \
        P45Rows<KK, 1> Q;                                                                                 \
        if (p45_rows<KK, 1>(Q, w, p)) {                                                                   \
            SSN_COUNT_LAUNCH();                                                                           \
            k_reshare_finish_p45<KK><<<ssn_grid2(n, nbatch), 256, 0, (cudaStream_t)strm>>>(                \
                pts, pts_bstride, pts_jstride, Q, zero, zero_bstride, bias, bias_bstride, bias_div, bias_mod, \
                alpha, alpha_bstride, out, out_bstride, n);                                               \
            return ssn_check_launch();                                                                    \
        }                                                                                                 \
    }
    SSN_RF_P45(2)
    SSN_RF_P45(3)
#undef SSN_RF_P45
    Weights W = make_weights(w, k, p);
    SSN_COUNT_LAUNCH();
    k_reshare_finish<<<ssn_grid2(n, nbatch), 256, 0, (cudaStream_t)strm>>>(
        pts, pts_bstride, pts_jstride, W, k, zero, zero_bstride, bias, bias_bstride, bias_div, bias_mod, alpha,
        alpha_bstride, out, out_bstride, n, nbatch, ssn_make_field(p));
    return ssn_check_launch();
}

// ------------------------------------------------------------------ truncation elite
__global__ void k_trunc_elite(const u64 *__restrict__ pts, u64 p_j, int npts, int k, Weights w, ExtTable ext,
                              i64 lo, u64 neglo_mod, i64 r, int rshift, i64 d, const u64 *__restrict__ coeffs,
                              u64 seed, u64 stream, int km1, PowTable pw, int nids, u64 *__restrict__ out, u64 o_t,
                              unsigned long long *__restrict__ fail, u64 n, SsnField f) {
    unsigned long long bad_local = 0;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        u64 s[SSN_MAXP];
#pragma unroll
        for (int j = 0; j < SSN_MAXP; j++)
            if (j < npts) s[j] = pts[j * p_j + i];
        const u64 v = lincomb<SSN_MAXP>(s, w.r, w.small, k, f);
#pragma unroll
        for (int q = 1; q < SSN_MAXP; q++) {                       // RS checks of points k..npts-1
            if (q >= k && q < npts) bad_local += (lincomb<SSN_MAXP>(s, ext.r[q - k], ext.small, k, f) != s[q]);
        }
        const u64 tm = ssn_trunc_value(v, lo, neglo_mod, r, rshift, d, f);
        if (nids == 0) {
            out[i] = tm;
            continue;
        }
        u64 c[SSN_MAXK];
        load_coeffs(c, coeffs, n, i, km1, seed, stream, f);
#pragma unroll
        for (int tt = 0; tt < SSN_MAXJ; tt++)
            if (tt < nids) out[tt * o_t + i] = horner_at(tm, c, pw, tt, km1, f);
    }
    if (fail && bad_local) atomicAdd(fail, bad_local);
}

// p45 truncation elite: compile-time k, extra RS points NX and output ids NIDS (0: the truncated
// value only); same coefficient draws and canonical outputs as k_trunc_elite
template <int K, int NX, int NIDS>
__global__ void k_trunc_elite_p45(const u64 *__restrict__ pts, u64 p_j, P45Rows<K, 1> w,
                                  P45Rows<K, (NX > 0 ? NX : 1)> ext, i64 lo, u64 neglo_mod, i64 r, int rshift, i64 d,
                                  const u64 *__restrict__ coeffs, u64 seed, u64 stream,
                                  P45Pows<K - 1, (NIDS > 0 ? NIDS : 1)> pw, u64 *__restrict__ out, u64 o_t,
                                  unsigned long long *__restrict__ fail, u64 n, SsnField f) {
    unsigned long long bad_local = 0;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        u64 s[K + NX];
#pragma unroll
        for (int j = 0; j < K + NX; j++) s[j] = pts[j * p_j + i];
        u64 front[K];
#pragma unroll
        for (int j = 0; j < K; j++) front[j] = s[j];
        const u64 v = ssn45::canon(ssn45::lin<K>(front, w.r[0]));
#pragma unroll
        for (int q = 0; q < NX; q++) bad_local += (ssn45::canon(ssn45::lin<K>(front, ext.r[q])) != s[K + q]);
        const u64 tm = ssn_trunc_value(v, lo, neglo_mod, r, rshift, d, f);
        if (NIDS == 0) {
            out[i] = tm;
            continue;
        }
        u64 c[SSN_MAXK];
        load_coeffs(c, coeffs, n, i, K - 1, seed, stream, f);
#pragma unroll
        for (int t = 0; t < NIDS; t++) {
            u64 acc = tm;
#pragma unroll
            for (int j = 0; j < K - 1; j++) acc += mul_small(c[j], pw.pw[t][j]);
            out[t * o_t + i] = ssn45::canon(acc);
        }
    }
    if (fail && bad_local) atomicAdd(fail, bad_local);
}

extern "C" int ssn_trunc_elite(const u64 *pts, u64 pts_jstride, int npts, int k, const u64 *w, const u64 *ext,
                               i64 value_bound, i64 r, i64 d, const u64 *coeffs, u64 seed, u64 stream, int km1,
                               const u64 *ids, int nids, u64 *out, u64 out_tstride, unsigned long long *fail, u64 n,
                               u64 p, void *strm) {
    if (k < 1 || k > SSN_MAXP || npts < k || npts > SSN_MAXP || r < 1 || d < 1 || km1 < 0 || km1 > SSN_MAXK ||
        nids < 0 || nids > SSN_MAXJ)
        return SSN_ERR_ARG;
    if (n == 0) return 0;
    Weights W = make_weights(w, k, p);
    ExtTable E;
    E.small = 1;
    for (int e = 0; e < SSN_MAXP; e++) {
        u64 row[SSN_MAXJ] = {0};
        if (e < npts - k && ext)
            for (int j = 0; j < k; j++) row[j] = ext[e * k + j];
        int ok = make_row(E.r[e], row, k, p);
        if (e < npts - k) E.small = E.small && ok;
    }
    PowTable pw = make_pows(ids, nids, km1, p);
    const i64 lo = -value_bound + r * d;
    const u64 neglo_mod = lo <= 0 ? (u64)(-lo) % p : (p - (u64)lo % p) % p;
    int rshift = -1;
    if ((r & (r - 1)) == 0) {
        rshift = 0;
        while ((1ll << rshift) < r) rshift++;
    }
#define SSN_TE_P45(KK, XX, NN)                                                                            \
    if (k == KK && npts - k == XX && nids == NN && km1 == KK - 1 && p == ssn45::PP && pw.small) {          \
        P45Rows<KK, 1> qw;                                                                                \
        P45Rows<KK, (XX > 0 ? XX : 1)> qe;                                                                \
        P45Pows<KK - 1, (NN > 0 ? NN : 1)> qp;                                                            \
        int ok = p45_rows<KK, 1>(qw, w, p);                                                               \
        for (int e = 0; e < XX && ok; e++) ok = ssn45::make_srow<KK>(qe.r[e], ext + (u64)e * KK, KK, p);  \
        for (int t = 0; t < NN; t++)                                                                      \
            for (int j = 0; j < KK - 1; j++) qp.pw[t][j] = (uint32_t)pw.r[t].n[j];                        \
        if (ok) {                                                                                         \
            SSN_COUNT_LAUNCH();                                                                           \
            k_trunc_elite_p45<KK, XX, NN><<<ssn_blocks(n), 256, 0, (cudaStream_t)strm>>>(                  \
                pts, pts_jstride, qw, qe, lo, neglo_mod, r, rshift, d, coeffs, seed, stream, qp, out,      \
                out_tstride, fail, n, ssn_make_field(p));                                                 \
            return ssn_check_launch();                                                                    \
        }                                                                                                 \
    }
    SSN_TE_P45(2, 0, 0)
    SSN_TE_P45(2, 0, 3)
    SSN_TE_P45(2, 1, 0)
    SSN_TE_P45(2, 1, 3)
    SSN_TE_P45(3, 0, 0)
    SSN_TE_P45(3, 0, 5)
    SSN_TE_P45(3, 2, 0)
    SSN_TE_P45(3, 2, 5)
#undef SSN_TE_P45
    SSN_COUNT_LAUNCH();
    k_trunc_elite<<<ssn_blocks(n), 256, 0, (cudaStream_t)strm>>>(pts, pts_jstride, npts, k, W, E, lo, neglo_mod, r,
                                                                 rshift, d, coeffs, seed, stream, km1, pw, nids, out,
                                                                 out_tstride, fail, n, ssn_make_field(p));
    return ssn_check_launch();
}

// ------------------------------------------------------------------ nonlinear elite
// One thread per OUTPUT element (window).  Input viewed as nb x (c, h, wd); pool_kind 0 = none
// (kh = kw = 1), 1 = max, 2 = sum.  plain[o] = encode_signed(pool(relu(decode(rec(pts)))))
__global__ void k_nonlin_elite(const u64 *__restrict__ pts, u64 p_j, int m, Weights w, int relu, int pool_kind,
                               int c, int h, int wd, int kh, int kw, u64 *__restrict__ plain, u64 n_out,
                               SsnField f) {
    const int oh = h / kh, ow = wd / kw;
    for (u64 o = blockIdx.x * (u64)blockDim.x + threadIdx.x; o < n_out; o += (u64)gridDim.x * blockDim.x) {
        u64 base_in;
        if (pool_kind == 0) {
            base_in = o;
        } else {
            const uint32_t o32 = (uint32_t)o, chw = (uint32_t)(c * oh * ow), hw = (uint32_t)(oh * ow);
            const uint32_t img = o32 / chw, rem = o32 - img * chw;
            const uint32_t ci = rem / hw, rr = rem - ci * hw;
            const uint32_t y = rr / (uint32_t)ow, x = rr - y * (uint32_t)ow;
            base_in = (((u64)img * c + ci) * (u64)h + (u64)(y * kh)) * wd + (u64)(x * kw);
        }
        i64 acc = pool_kind == 1 ? INT64_MIN : 0;
        for (int a = 0; a < kh; a++)
            for (int bq = 0; bq < kw; bq++) {
                const u64 i = base_in + (u64)a * wd + bq;
                u64 x[SSN_MAXP];
#pragma unroll
                for (int j = 0; j < SSN_MAXP; j++)
                    if (j < m) x[j] = pts[j * p_j + i];
                const u64 v = lincomb<SSN_MAXP>(x, w.r, w.small, m, f);
                i64 sv = v > f.half ? (i64)v - (i64)f.p : (i64)v;
                if (relu && sv <= 0) sv = 0;
                if (pool_kind == 1) acc = sv > acc ? sv : acc;
                else acc += sv;
            }
        plain[o] = acc < 0 ? (u64)((i64)f.p + acc) : (u64)acc;
    }
}

template <int M>
__global__ void k_nonlin_elite_p45(const u64 *__restrict__ pts, u64 p_j, P45Rows<M, 1> w, int relu, int pool_kind,
                                   int c, int h, int wd, int kh, int kw, u64 *__restrict__ plain, u64 n_out) {
    const int oh = h / kh, ow = wd / kw;
    for (u64 o = blockIdx.x * (u64)blockDim.x + threadIdx.x; o < n_out; o += (u64)gridDim.x * blockDim.x) {
        u64 base_in;
        if (pool_kind == 0) {
            base_in = o;
        } else {
            const uint32_t o32 = (uint32_t)o, chw = (uint32_t)(c * oh * ow), hw = (uint32_t)(oh * ow);
            const uint32_t img = o32 / chw, rem = o32 - img * chw;
            const uint32_t ci = rem / hw, rr = rem - ci * hw;
            const uint32_t y = rr / (uint32_t)ow, x = rr - y * (uint32_t)ow;
            base_in = (((u64)img * c + ci) * (u64)h + (u64)(y * kh)) * wd + (u64)(x * kw);
        }
        i64 acc = pool_kind == 1 ? INT64_MIN : 0;
        for (int a = 0; a < kh; a++)
            for (int bq = 0; bq < kw; bq++) {
                const u64 i = base_in + (u64)a * wd + bq;
                u64 x[M];
#pragma unroll
                for (int j = 0; j < M; j++) x[j] = pts[j * p_j + i];
                const u64 v = ssn45::canon(ssn45::lin<M>(x, w.r[0]));
                i64 sv = v > ssn45::PHALF ? (i64)v - (i64)ssn45::PP : (i64)v;
                if (relu && sv <= 0) sv = 0;
                if (pool_kind == 1) acc = sv > acc ? sv : acc;
                else acc += sv;
            }
        plain[o] = acc < 0 ? (u64)((i64)ssn45::PP + acc) : (u64)acc;
    }
}

extern "C" int ssn_nonlin_elite(const u64 *pts, u64 pts_jstride, int m, const u64 *w, int relu, int pool_kind,
                                int nb, int c, int h, int wd, int kh, int kw, u64 *plain, u64 p, void *strm) {
    if (m < 1 || m > SSN_MAXP || pool_kind < 0 || pool_kind > 2 || kh < 1 || kw < 1 || h % kh || wd % kw)
        return SSN_ERR_ARG;
    if (pool_kind == 0 && (kh != 1 || kw != 1)) return SSN_ERR_ARG;
    Weights W = make_weights(w, m, p);
    const u64 n_out = (u64)nb * c * (h / kh) * (wd / kw);
    if (n_out == 0) return 0;
    if (n_out >= (1ull << 32)) return SSN_ERR_UNSUPPORTED;
#define SSN_NE_P45(MM)                                                                                    \
    if (m == MM) {                                                                                        \
        P45Rows<MM, 1> q;                                                                                 \
        if (p45_rows<MM, 1>(q, w, p)) {                                                                   \
            SSN_COUNT_LAUNCH();                                                                           \
            k_nonlin_elite_p45<MM><<<ssn_blocks(n_out), 256, 0, (cudaStream_t)strm>>>(                     \
                pts, pts_jstride, q, relu, pool_kind, c, h, wd, kh, kw, plain, n_out);                    \
            return ssn_check_launch();                                                                    \
        }                                                                                                 \
    }
    SSN_NE_P45(3)
    SSN_NE_P45(5)
#undef SSN_NE_P45
    SSN_COUNT_LAUNCH();
    k_nonlin_elite<<<ssn_blocks(n_out), 256, 0, (cudaStream_t)strm>>>(pts, pts_jstride, m, W, relu, pool_kind, c, h,
                                                                      wd, kh, kw, plain, n_out, ssn_make_field(p));
    return ssn_check_launch();
}

// ------------------------------------------------------------------ signed embedding, inverse, random
__global__ void k_encode(const i64 *__restrict__ x, u64 *__restrict__ out, u64 n, SsnField f,
                         unsigned long long *overflow) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const i64 v = x[i];
        const u64 mag = v < 0 ? (u64)(-v) : (u64)v;
        if (mag > f.half && overflow) atomicAdd(overflow, 1ull);
        out[i] = v < 0 ? f.p - mag : mag;
    }
}
extern "C" int ssn_encode_signed(const i64 *x, u64 *out, u64 n, unsigned long long *overflow, u64 p, void *strm) {
    if (n == 0) return 0;
    SSN_COUNT_LAUNCH();
    k_encode<<<ssn_blocks(n), 256, 0, (cudaStream_t)strm>>>(x, out, n, ssn_make_field(p), overflow);
    return ssn_check_launch();
}

__global__ void k_decode(const u64 *__restrict__ v, i64 *__restrict__ out, u64 n, SsnField f) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u64 x = v[i];
        out[i] = x > f.half ? (i64)x - (i64)f.p : (i64)x;
    }
}
extern "C" int ssn_decode_signed(const u64 *v, i64 *out, u64 n, u64 p, void *strm) {
    if (n == 0) return 0;
    SSN_COUNT_LAUNCH();
    k_decode<<<ssn_blocks(n), 256, 0, (cudaStream_t)strm>>>(v, out, n, ssn_make_field(p));
    return ssn_check_launch();
}

__global__ void k_inv(const u64 *__restrict__ a, u64 *__restrict__ out, u64 n, SsnField f) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        out[i] = ssn_powmod(a[i], f.p - 2, f);   // Fermat; 0 -> 0
}
extern "C" int ssn_inv(const u64 *a, u64 *out, u64 n, u64 p, void *strm) {
    if (n == 0) return 0;
    SSN_COUNT_LAUNCH();
    k_inv<<<ssn_blocks(n), 256, 0, (cudaStream_t)strm>>>(a, out, n, ssn_make_field(p));
    return ssn_check_launch();
}

__global__ void k_rand(u64 *__restrict__ out, u64 n, u64 lo, u64 range, u64 seed, u64 stream) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        out[i] = lo + ssn_rand_range(seed, stream, i, 0, range);
}
extern "C" int ssn_rand(u64 *out, u64 n, u64 lo, u64 range, u64 seed, u64 stream, void *strm) {
    if (range == 0) return SSN_ERR_ARG;
    if (n == 0) return 0;
    SSN_COUNT_LAUNCH();
    k_rand<<<ssn_blocks(n), 256, 0, (cudaStream_t)strm>>>(out, n, lo, range, seed, stream);
    return ssn_check_launch();
}

// ------------------------------------------------------------------ trusted source (device speed mode)
// Additive mask (S/masks.py:39-54): e = 1 + U[0, emax); alpha = e*step; comp = -e; both shared.
// Philox draw j = 0 is e; alpha / comp coefficients come from streams stream+1 / stream+2.
__global__ void k_mask_trunc(u64 n, u64 step, u64 emax, u64 seed, u64 stream, int km1, PowTable pw, int nids,
                             u64 *__restrict__ alpha, u64 *__restrict__ comp, u64 o_t, SsnField f) {
    const u64 stepm = ssn_reduce64(step, f);
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u64 e = 1 + ssn_rand_range(seed, stream, i, 0, emax);
        const u64 em = ssn_reduce64(e, f);
        const u64 a = ssn_mulmod(em, stepm, f);
        const u64 cm = em ? f.p - em : 0;
        u64 ca[SSN_MAXK], cc[SSN_MAXK];
        load_coeffs(ca, nullptr, n, i, km1, seed, stream + 1, f);
        load_coeffs(cc, nullptr, n, i, km1, seed, stream + 2, f);
#pragma unroll
        for (int t = 0; t < SSN_MAXJ; t++)
            if (t < nids) {
                alpha[t * o_t + i] = horner_at(a, ca, pw, t, km1, f);
                comp[t * o_t + i] = horner_at(cm, cc, pw, t, km1, f);
            }
    }
}

extern "C" int ssn_mask_trunc(u64 n, u64 step, u64 emax, u64 seed, u64 stream, int km1, const u64 *ids, int nids,
                              u64 *alpha, u64 *comp, u64 out_tstride, u64 p, void *strm) {
    if (emax < 1 || km1 < 0 || km1 > SSN_MAXK || nids < 1 || nids > SSN_MAXJ) return SSN_ERR_ARG;
    if (n == 0) return 0;
    PowTable pw = make_pows(ids, nids, km1, p);
    SSN_COUNT_LAUNCH();
    k_mask_trunc<<<ssn_blocks(n), 256, 0, (cudaStream_t)strm>>>(n, step, emax, seed, stream, km1, pw, nids, alpha,
                                                                comp, out_tstride, ssn_make_field(p));
    return ssn_check_launch();
}

// Multiplicative mask (S/masks.py:67-90).  Each thread owns WPT windows spaced a grid
// apart (coalesced); beta = 1 + U[0, bmax) per window, the WPT inverses by Montgomery's
// batch trick (one Fermat exponentiation per thread instead of per window), beta shared per
// input element of the window (streams stream+1), beta^-1 shared per window (stream+2).
#define SSN_WPT 8
__global__ void __launch_bounds__(256, 1) k_mask_beta(int c, int h, int wd, int kh, int kw, u64 n_out, u64 bmax,
                                                   u64 seed, u64 stream, int km1, PowTable pw, int nids,
                                                   u64 *__restrict__ beta, u64 b_t, u64 *__restrict__ binv,
                                                   u64 bi_t, SsnField f) {
    const int oh = h / kh, ow = wd / kw;
    const u64 T = (u64)gridDim.x * blockDim.x;
    for (u64 o0 = blockIdx.x * (u64)blockDim.x + threadIdx.x; o0 < n_out; o0 += T * SSN_WPT) {
        u64 bt[SSN_WPT], pre[SSN_WPT];
        u64 run = 1;
#pragma unroll
        for (int q = 0; q < SSN_WPT; q++) {
            const u64 o = o0 + (u64)q * T;
            bt[q] = o < n_out ? 1 + ssn_rand_range(seed, stream, o, 0, bmax) : 1;
            run = ssn_mulmod(run, bt[q], f);
            pre[q] = run;
        }
        u64 inv = ssn_powmod(run, f.p - 2, f);
#pragma unroll
        for (int q = SSN_WPT - 1; q >= 0; q--) {
            const u64 bi = q ? ssn_mulmod(inv, pre[q - 1], f) : inv;
            inv = ssn_mulmod(inv, bt[q], f);
            pre[q] = bi;                                    // reuse: beta^-1 of window q
        }
#pragma unroll
        for (int q = 0; q < SSN_WPT; q++) {
            const u64 o = o0 + (u64)q * T;
            if (o >= n_out) continue;
            u64 cc[SSN_MAXK];
            load_coeffs(cc, nullptr, n_out, o, km1, seed, stream + 2, f);
#pragma unroll
            for (int t = 0; t < SSN_MAXJ; t++)
                if (t < nids) binv[t * bi_t + o] = horner_at(pre[q], cc, pw, t, km1, f);
            u64 base_in;
            if (kh == 1 && kw == 1) {
                base_in = o;
            } else {
                const uint32_t o32 = (uint32_t)o, chw = (uint32_t)(c * oh * ow), hw = (uint32_t)(oh * ow);
                const uint32_t img = o32 / chw, rem = o32 - img * chw;
                const uint32_t ci = rem / hw, rr = rem - ci * hw;
                const uint32_t y0 = rr / (uint32_t)ow, x0 = rr - y0 * (uint32_t)ow;
                base_in = (((u64)img * c + ci) * (u64)h + (u64)(y0 * kh)) * wd + (u64)(x0 * kw);
            }
            for (int a = 0; a < kh; a++)
                for (int b = 0; b < kw; b++) {
                    const u64 i = base_in + (u64)a * wd + b;
                    u64 ca[SSN_MAXK];
                    load_coeffs(ca, nullptr, 0, i, km1, seed, stream + 1, f);
#pragma unroll
                    for (int t = 0; t < SSN_MAXJ; t++)
                        if (t < nids) beta[t * b_t + i] = horner_at(bt[q], ca, pw, t, km1, f);
                }
        }
    }
}

extern "C" int ssn_mask_beta(int nb, int c, int h, int wd, int kh, int kw, u64 bmax, u64 seed, u64 stream, int km1,
                             const u64 *ids, int nids, u64 *beta, u64 beta_tstride, u64 *binv, u64 binv_tstride,
                             u64 p, void *strm) {
    if (bmax < 1 || kh < 1 || kw < 1 || h % kh || wd % kw || km1 < 0 || km1 > SSN_MAXK || nids < 1 ||
        nids > SSN_MAXJ)
        return SSN_ERR_ARG;
    const u64 n_out = (u64)nb * c * (h / kh) * (wd / kw);
    if (n_out == 0) return 0;
    if (n_out >= (1ull << 32)) return SSN_ERR_UNSUPPORTED;
    PowTable pw = make_pows(ids, nids, km1, p);
    u64 blocks = (n_out + 256 * SSN_WPT - 1) / (256 * SSN_WPT);
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (blocks < 1) blocks = 1;
    SSN_COUNT_LAUNCH();
    k_mask_beta<<<(unsigned)blocks, 256, 0, (cudaStream_t)strm>>>(c, h, wd, kh, kw, n_out, bmax, seed, stream, km1,
                                                                  pw, nids, beta, beta_tstride, binv, binv_tstride,
                                                                  ssn_make_field(p));
    return ssn_check_launch();
}

// Repeat a (nb, c, h/kh, w/kw) block tensor over kh x kw windows (host-fed parity mode beta).
__global__ void k_pool_expand(const u64 *__restrict__ blk, u64 *__restrict__ out, int c, int h, int wd, int kh,
                              int kw, u64 n) {
    const int oh = h / kh, ow = wd / kw;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        const u64 x = i % wd, y = (i / wd) % h, rest = i / ((u64)wd * h);   // rest = img*c + ci
        out[i] = blk[(rest * oh + y / kh) * ow + x / kw];
    }
}
extern "C" int ssn_pool_expand(const u64 *blk, u64 *out, int nb, int c, int h, int wd, int kh, int kw, void *strm) {
    if (kh < 1 || kw < 1 || h % kh || wd % kw) return SSN_ERR_ARG;
    const u64 n = (u64)nb * c * h * wd;
    if (n == 0) return 0;
    SSN_COUNT_LAUNCH();
    k_pool_expand<<<ssn_blocks(n), 256, 0, (cudaStream_t)strm>>>(blk, out, c, h, wd, kh, kw, n);
    return ssn_check_launch();
}

// overlapping-window gather (builder op "gather"): one thread per gathered element
__global__ void k_window_gather(const u64 *__restrict__ x, u64 *__restrict__ out, int h, int w, int kh, int kw,
                                int stride, int pad, int oh, int ow, u64 n) {
    const int gw = ow * kw, gh = oh * kh;
    for (u64 o = blockIdx.x * (u64)blockDim.x + threadIdx.x; o < n; o += (u64)gridDim.x * blockDim.x) {
        const u64 plane = o / ((u64)gh * gw);
        const int rem = (int)(o - plane * (u64)gh * gw);
        const int Y = rem / gw, X = rem - Y * gw;
        const int oy = Y / kh, dy = Y - oy * kh, ox = X / kw, dx = X - ox * kw;
        const int sy = oy * stride - pad + dy, sx = ox * stride - pad + dx;
        out[o] = (sy >= 0 && sy < h && sx >= 0 && sx < w) ? x[plane * (u64)h * w + (u64)sy * w + sx] : 0;
    }
}
extern "C" int ssn_window_gather(const u64 *x, u64 *out, int nb, int c, int h, int w, int kh, int kw, int stride,
                                 int pad, void *strm) {
    if (!x || !out || nb < 0 || c < 0 || kh < 1 || kw < 1 || stride < 1 || pad < 0 || h + 2 * pad < kh ||
        w + 2 * pad < kw)
        return SSN_ERR_ARG;
    const int oh = (h + 2 * pad - kh) / stride + 1, ow = (w + 2 * pad - kw) / stride + 1;
    const u64 n = (u64)nb * c * oh * kh * ow * kw;
    if (n == 0) return 0;
    SSN_COUNT_LAUNCH();
    k_window_gather<<<ssn_blocks(n), 256, 0, (cudaStream_t)strm>>>(x, out, h, w, kh, kw, stride, pad, oh, ow, n);
    return ssn_check_launch();
}

extern "C" int ssn_version(void) { return SSN_ABI_VERSION; }
extern "C" unsigned long long ssn_kernel_launches(void) { return ssn_launch_counter(); }
