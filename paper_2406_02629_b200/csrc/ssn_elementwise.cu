// ssn_elementwise.cu -- HBM-bound field kernels of the SSNet hot path (sm_100a) + C-ABI.
//
// Every kernel is a grid-stride loop over elements with one thread per element per
// iteration (coalesced u64 loads/stores); multi-party operands are addressed as strided
// 2-D views base + b*stride_b + j*stride_j so one launch covers all co-resident parties.
// Reference functions restated (paths relative to /root/reference/pkg/src/ssnet):
//   ssn_ewise            share_add/sub/mul, PrimeField.add/sub/mul   S/sss.py:238-276, S/field.py:89-99
//   ssn_gen              SssScheme.gen (Horner over party ids)      S/sss.py:118-147
//   ssn_rec              SssScheme.rec (Lagrange weighted sum)       S/sss.py:172-194
//   ssn_reduce_apply     reshare step 2, R^T @ stack                 S/protocol.py:165-185
//   ssn_reshare_finish   reshare step 3 + rerand + bias (+ trunc mask) S/protocol.py:187-198, S/layers.py:260-267,290-293
//   ssn_trunc_elite      masked truncation at the elite (+ fresh shares, + RS check)  S/layers.py:295-315
//   ssn_nonlin_elite     masked ReLU / max / sum pool at the elite   S/layers.py:345-364
//   ssn_mask_*           trusted-source masks                        S/masks.py:39-96, S/protocol.py:354-388
#include "ssn_field.cuh"
#include "ssn.h"

#define SSN_MAXJ 16
#define SSN_MAXK 8

static int ssn_blocks(u64 n, int threads = 256) {
    u64 b = (n + threads - 1) / threads;
    const u64 cap = 148ull * 16;
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return (int)b;
}

static inline int ssn_check_launch() {
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : SSN_ERR_CUDA;
}

struct PowTable {            // pw[t][j] = ids[t]^(j+1) mod p
    u64 pw[SSN_MAXJ][SSN_MAXK];
};

static PowTable make_pows(const u64 *ids, int nids, int km1, u64 p) {
    PowTable t;
    for (int a = 0; a < nids; a++) {
        unsigned __int128 acc = 1;
        for (int j = 0; j < km1; j++) {
            acc = acc * (ids[a] % p) % p;
            t.pw[a][j] = (u64)acc;
        }
    }
    return t;
}

struct Weights { u64 w[SSN_MAXJ]; };

// ------------------------------------------------------------------ ewise
__global__ void k_ewise(int op, const u64 *__restrict__ a, const u64 *__restrict__ b, u64 *__restrict__ out,
                        u64 n, u64 b_div, u64 b_mod, u64 b_div2, u64 b_mul2, SsnField f) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        u64 x = a[i];
        u64 y = op == 3 ? 0 : b[(i / b_div) % b_mod + (i / b_div2) * b_mul2];
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
    k_ewise<<<ssn_blocks(n), 256, 0, (cudaStream_t)stream>>>(op, a, b, out, n, b_div, b_mod, b_div2, b_mul2,
                                                            ssn_make_field(p));
    return ssn_check_launch();
}

// ------------------------------------------------------------------ gen
// out[b][t][i] = secret[b][i] + sum_j c_j[b][i] * ids[t]^(j+1)
// coeffs[b][j][i] when host-fed, else Philox(seed, stream + b, i, j).
__global__ void k_gen(const u64 *__restrict__ secret, u64 s_b, const u64 *__restrict__ coeffs, u64 c_b, u64 seed,
                      u64 stream, int km1, PowTable pw, int nids, u64 *__restrict__ out, u64 o_b, u64 o_t, u64 n,
                      int nb, SsnField f) {
    u64 total = n * (u64)nb;
    for (u64 g = blockIdx.x * (u64)blockDim.x + threadIdx.x; g < total; g += (u64)gridDim.x * blockDim.x) {
        u64 b = g / n, i = g - b * n;
        u64 s = secret ? secret[b * s_b + i] : 0;
        u64 c[SSN_MAXK];
#pragma unroll
        for (int j = 0; j < SSN_MAXK; j++) {
            if (j < km1)
                c[j] = coeffs ? coeffs[b * c_b + (u64)j * n + i] : ssn_rand_range(seed, stream + b, i, j, f.p);
        }
        for (int t = 0; t < nids; t++) {
            u64 acc = s;
#pragma unroll
            for (int j = 0; j < SSN_MAXK; j++)
                if (j < km1) acc = ssn_addmod(acc, ssn_mulmod(c[j], pw.pw[t][j], f), f.p);
            out[b * o_b + t * o_t + i] = acc;
        }
    }
}

extern "C" int ssn_gen(const u64 *secret, u64 secret_bstride, const u64 *coeffs, u64 coeff_bstride, u64 seed,
                       u64 stream, int km1, const u64 *ids, int nids, u64 *out, u64 out_bstride, u64 out_tstride,
                       u64 n, int nbatch, u64 p, void *strm) {
    if (km1 < 0 || km1 > SSN_MAXK || nids < 1 || nids > SSN_MAXJ || nbatch < 1) return SSN_ERR_ARG;
    if (n == 0) return 0;
    PowTable pw = make_pows(ids, nids, km1, p);
    k_gen<<<ssn_blocks(n * nbatch), 256, 0, (cudaStream_t)strm>>>(secret, secret_bstride, coeffs, coeff_bstride,
                                                                  seed, stream, km1, pw, nids, out, out_bstride,
                                                                  out_tstride, n, nbatch, ssn_make_field(p));
    return ssn_check_launch();
}

// ------------------------------------------------------------------ rec
// out[b][i] = sum_j w[j] * pts[b][j][i]
__global__ void k_rec(const u64 *__restrict__ pts, u64 p_b, u64 p_j, Weights w, int m, u64 *__restrict__ out,
                      u64 o_b, u64 n, int nb, SsnField f) {
    u64 total = n * (u64)nb;
    for (u64 g = blockIdx.x * (u64)blockDim.x + threadIdx.x; g < total; g += (u64)gridDim.x * blockDim.x) {
        u64 b = g / n, i = g - b * n;
        const u64 *base = pts + b * p_b + i;
        u64 acc = 0;
        for (int j = 0; j < m; j++) acc = ssn_addmod(acc, ssn_mulmod(base[j * p_j], w.w[j], f), f.p);
        out[b * o_b + i] = acc;
    }
}

extern "C" int ssn_rec(const u64 *pts, u64 pts_bstride, u64 pts_jstride, const u64 *w, int m, u64 *out,
                       u64 out_bstride, u64 n, int nbatch, u64 p, void *strm) {
    if (m < 1 || m > SSN_MAXJ || nbatch < 1) return SSN_ERR_ARG;
    if (n == 0) return 0;
    Weights W;
    for (int j = 0; j < m; j++) W.w[j] = w[j] % p;
    k_rec<<<ssn_blocks(n * nbatch), 256, 0, (cudaStream_t)strm>>>(pts, pts_bstride, pts_jstride, W, m, out,
                                                                  out_bstride, n, nbatch, ssn_make_field(p));
    return ssn_check_launch();
}

// ------------------------------------------------------------------ reduce apply (reshare step 2)
// out[b][t][i] = sum_j Rt[t][j] * pts[b][j][i]  -- b = front rank, j = sub-share source, t = out rank
struct RTable { u64 r[SSN_MAXJ][SSN_MAXJ]; };

__global__ void k_reduce_apply(const u64 *__restrict__ pts, u64 p_b, u64 p_j, RTable R, int m, int nout,
                               u64 *__restrict__ out, u64 o_b, u64 o_t, u64 n, int nb, SsnField f, u64 r64) {
    u64 total = n * (u64)nb;
    for (u64 g = blockIdx.x * (u64)blockDim.x + threadIdx.x; g < total; g += (u64)gridDim.x * blockDim.x) {
        u64 b = g / n, i = g - b * n;
        const u64 *base = pts + b * p_b + i;
        u64 v[SSN_MAXJ];
        for (int j = 0; j < m; j++) v[j] = base[j * p_j];
        for (int t = 0; t < nout; t++) {
            u128s acc = {0, 0};
            for (int j = 0; j < m; j++) ssn_mac(acc, v[j], R.r[t][j]);
            out[b * o_b + t * o_t + i] = ssn_reduce128(acc, f, r64);
        }
    }
}

static u64 r64_of(u64 p) { return (u64)((((unsigned __int128)1) << 64) % p); }

extern "C" int ssn_reduce_apply(const u64 *pts, u64 pts_bstride, u64 pts_jstride, int m, const u64 *rt, int nout,
                                u64 *out, u64 out_bstride, u64 out_tstride, u64 n, int nbatch, u64 p, void *strm) {
    if (m < 1 || m > SSN_MAXJ || nout < 1 || nout > SSN_MAXJ || nbatch < 1) return SSN_ERR_ARG;
    if (n == 0) return 0;
    RTable R;
    for (int t = 0; t < nout; t++)
        for (int j = 0; j < m; j++) R.r[t][j] = rt[t * m + j] % p;
    k_reduce_apply<<<ssn_blocks(n * nbatch), 256, 0, (cudaStream_t)strm>>>(pts, pts_bstride, pts_jstride, R, m, nout,
                                                                           out, out_bstride, out_tstride, n, nbatch,
                                                                           ssn_make_field(p), r64_of(p));
    return ssn_check_launch();
}

// ------------------------------------------------------------------ reshare step 3 (+rerand, +bias, +alpha)
// out[b][i] = sum_j w[j]*pts[b][j][i] + zero[b][i] + bias[b][(i / bias_div) % bias_mod] (+ alpha[b][i])
__global__ void k_reshare_finish(const u64 *__restrict__ pts, u64 p_b, u64 p_j, Weights w, int k,
                                 const u64 *__restrict__ zero, u64 z_b, const u64 *__restrict__ bias, u64 bi_b,
                                 u64 bias_div, u64 bias_mod, const u64 *__restrict__ alpha, u64 a_b,
                                 u64 *__restrict__ out, u64 o_b, u64 n, int nb, SsnField f) {
    u64 total = n * (u64)nb;
    for (u64 g = blockIdx.x * (u64)blockDim.x + threadIdx.x; g < total; g += (u64)gridDim.x * blockDim.x) {
        u64 b = g / n, i = g - b * n;
        const u64 *base = pts + b * p_b + i;
        u64 acc = 0;
        for (int j = 0; j < k; j++) acc = ssn_addmod(acc, ssn_mulmod(base[j * p_j], w.w[j], f), f.p);
        if (zero) acc = ssn_addmod(acc, zero[b * z_b + i], f.p);
        if (bias) acc = ssn_addmod(acc, bias[b * bi_b + (i / bias_div) % bias_mod], f.p);
        if (alpha) acc = ssn_addmod(acc, alpha[b * a_b + i], f.p);
        out[b * o_b + i] = acc;
    }
}

extern "C" int ssn_reshare_finish(const u64 *pts, u64 pts_bstride, u64 pts_jstride, const u64 *w, int k,
                                  const u64 *zero, u64 zero_bstride, const u64 *bias, u64 bias_bstride,
                                  u64 bias_div, u64 bias_mod, const u64 *alpha, u64 alpha_bstride, u64 *out,
                                  u64 out_bstride, u64 n, int nbatch, u64 p, void *strm) {
    if (k < 1 || k > SSN_MAXJ || nbatch < 1 || bias_div == 0 || bias_mod == 0) return SSN_ERR_ARG;
    if (n == 0) return 0;
    Weights W;
    for (int j = 0; j < k; j++) W.w[j] = w[j] % p;
    k_reshare_finish<<<ssn_blocks(n * nbatch), 256, 0, (cudaStream_t)strm>>>(
        pts, pts_bstride, pts_jstride, W, k, zero, zero_bstride, bias, bias_bstride, bias_div, bias_mod, alpha,
        alpha_bstride, out, out_bstride, n, nbatch, ssn_make_field(p));
    return ssn_check_launch();
}

// ------------------------------------------------------------------ truncation elite
// v = sum_{j<k} w[j]*pts[j][i]; RS check of pts[k..npts) against Lagrange extrapolation;
// shifted = ((v - lo) mod p) + lo, lo = -value_bound + r*d; t = floor(shifted / r);
// d > 1: t = round_half_away(t, d); then fresh shares out[tt][i] = gen(t mod p) at ids.
struct ExtTable { u64 e[SSN_MAXJ][SSN_MAXK]; };

__device__ __forceinline__ i64 ssn_floordiv(i64 a, i64 b) {
    i64 q = a / b;
    if ((a % b != 0) && ((a < 0) != (b < 0))) q -= 1;
    return q;
}

__global__ void k_trunc_elite(const u64 *__restrict__ pts, u64 p_j, int npts, int k, Weights w, ExtTable ext,
                              i64 lo, i64 r, i64 d, const u64 *__restrict__ coeffs, u64 seed, u64 stream, int km1,
                              PowTable pw, int nids, u64 *__restrict__ out, u64 o_t,
                              unsigned long long *__restrict__ fail, u64 n, SsnField f) {
    unsigned long long bad_local = 0;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        u64 s[SSN_MAXJ];
        for (int j = 0; j < npts; j++) s[j] = pts[j * p_j + i];
        u64 v = 0;
        for (int j = 0; j < k; j++) v = ssn_addmod(v, ssn_mulmod(s[j], w.w[j], f), f.p);
        for (int e = k; e < npts; e++) {
            u64 pred = 0;
            for (int j = 0; j < k; j++) pred = ssn_addmod(pred, ssn_mulmod(s[j], ext.e[e - k][j], f), f.p);
            bad_local += (pred != s[e]);
        }
        // window decode: u = (v - lo) mod p with -lo >= 0 (lo may be negative or positive)
        u64 neglo_mod = lo <= 0 ? ssn_reduce64((u64)(-lo), f) : (f.p - ssn_reduce64((u64)lo, f)) % f.p;
        u64 u = ssn_addmod(v, neglo_mod, f.p);
        i64 shifted = (i64)u + lo;
        i64 t = ssn_floordiv(shifted, r);
        if (d > 1) {
            i64 a = t < 0 ? -t : t;
            i64 q = ssn_floordiv(2 * a + d, 2 * d);
            t = t < 0 ? -q : q;
        }
        u64 tm = t >= 0 ? ssn_reduce64((u64)t, f) : (f.p - ssn_reduce64((u64)(-t), f)) % f.p;
        if (nids == 0) {
            out[i] = tm;
            continue;
        }
        u64 c[SSN_MAXK];
#pragma unroll
        for (int j = 0; j < SSN_MAXK; j++)
            if (j < km1) c[j] = coeffs ? coeffs[(u64)j * n + i] : ssn_rand_range(seed, stream, i, j, f.p);
        for (int tt = 0; tt < nids; tt++) {
            u64 acc = tm;
#pragma unroll
            for (int j = 0; j < SSN_MAXK; j++)
                if (j < km1) acc = ssn_addmod(acc, ssn_mulmod(c[j], pw.pw[tt][j], f), f.p);
            out[tt * o_t + i] = acc;
        }
    }
    if (fail && bad_local) atomicAdd(fail, bad_local);
}

extern "C" int ssn_trunc_elite(const u64 *pts, u64 pts_jstride, int npts, int k, const u64 *w, const u64 *ext,
                               i64 value_bound, i64 r, i64 d, const u64 *coeffs, u64 seed, u64 stream, int km1,
                               const u64 *ids, int nids, u64 *out, u64 out_tstride, unsigned long long *fail, u64 n,
                               u64 p, void *strm) {
    if (k < 1 || npts < k || npts > SSN_MAXJ || npts - k > SSN_MAXJ || r < 1 || d < 1 || km1 < 0 ||
        km1 > SSN_MAXK || nids < 0 || nids > SSN_MAXJ)
        return SSN_ERR_ARG;
    if (n == 0) return 0;
    Weights W;
    for (int j = 0; j < k; j++) W.w[j] = w[j] % p;
    ExtTable E = {};
    if (npts > k && ext)
        for (int e = 0; e < npts - k; e++)
            for (int j = 0; j < k; j++) E.e[e][j] = ext[e * k + j] % p;
    PowTable pw = nids ? make_pows(ids, nids, km1, p) : PowTable{};
    i64 lo = -value_bound + r * d;
    k_trunc_elite<<<ssn_blocks(n), 256, 0, (cudaStream_t)strm>>>(pts, pts_jstride, npts, k, W, E, lo, r, d, coeffs,
                                                                 seed, stream, km1, pw, nids, out, out_tstride, fail,
                                                                 n, ssn_make_field(p));
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
        u64 img = o / ((u64)c * oh * ow);
        u64 rem = o - img * ((u64)c * oh * ow);
        int ci = (int)(rem / ((u64)oh * ow));
        int rr = (int)(rem % ((u64)oh * ow));
        int y = rr / ow, x = rr % ow;
        i64 acc = pool_kind == 1 ? INT64_MIN : 0;
        for (int a = 0; a < kh; a++)
            for (int bq = 0; bq < kw; bq++) {
                u64 i = ((img * c + ci) * (u64)h + (u64)(y * kh + a)) * wd + (u64)(x * kw + bq);
                u64 v = 0;
                for (int j = 0; j < m; j++) v = ssn_addmod(v, ssn_mulmod(pts[j * p_j + i], w.w[j], f), f.p);
                i64 sv = v > f.half ? (i64)v - (i64)f.p : (i64)v;
                if (relu && sv <= 0) sv = 0;
                if (pool_kind == 1) acc = sv > acc ? sv : acc;
                else acc += sv;
            }
        plain[o] = acc < 0 ? (u64)((i64)f.p + acc) : (u64)acc;
    }
}

extern "C" int ssn_nonlin_elite(const u64 *pts, u64 pts_jstride, int m, const u64 *w, int relu, int pool_kind,
                                int nb, int c, int h, int wd, int kh, int kw, u64 *plain, u64 p, void *strm) {
    if (m < 1 || m > SSN_MAXJ || pool_kind < 0 || pool_kind > 2 || kh < 1 || kw < 1 || h % kh || wd % kw)
        return SSN_ERR_ARG;
    if (pool_kind == 0 && (kh != 1 || kw != 1)) return SSN_ERR_ARG;
    Weights W;
    for (int j = 0; j < m; j++) W.w[j] = w[j] % p;
    u64 n_out = (u64)nb * c * (h / kh) * (wd / kw);
    if (n_out == 0) return 0;
    k_nonlin_elite<<<ssn_blocks(n_out), 256, 0, (cudaStream_t)strm>>>(pts, pts_jstride, m, W, relu, pool_kind, c, h,
                                                                      wd, kh, kw, plain, n_out, ssn_make_field(p));
    return ssn_check_launch();
}

// ------------------------------------------------------------------ signed embedding, inverse, random
__global__ void k_encode(const i64 *__restrict__ x, u64 *__restrict__ out, u64 n, SsnField f,
                         unsigned long long *overflow) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        i64 v = x[i];
        u64 mag = v < 0 ? (u64)(-v) : (u64)v;
        if (mag > f.half && overflow) atomicAdd(overflow, 1ull);
        out[i] = v < 0 ? f.p - mag : mag;
    }
}
extern "C" int ssn_encode_signed(const i64 *x, u64 *out, u64 n, unsigned long long *overflow, u64 p, void *strm) {
    if (n == 0) return 0;
    k_encode<<<ssn_blocks(n), 256, 0, (cudaStream_t)strm>>>(x, out, n, ssn_make_field(p), overflow);
    return ssn_check_launch();
}

__global__ void k_decode(const u64 *__restrict__ v, i64 *__restrict__ out, u64 n, SsnField f) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        u64 x = v[i];
        out[i] = x > f.half ? (i64)x - (i64)f.p : (i64)x;
    }
}
extern "C" int ssn_decode_signed(const u64 *v, i64 *out, u64 n, u64 p, void *strm) {
    if (n == 0) return 0;
    k_decode<<<ssn_blocks(n), 256, 0, (cudaStream_t)strm>>>(v, out, n, ssn_make_field(p));
    return ssn_check_launch();
}

__global__ void k_inv(const u64 *__restrict__ a, u64 *__restrict__ out, u64 n, SsnField f) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
        out[i] = ssn_powmod(a[i], f.p - 2, f);   // Fermat; 0 -> 0
}
extern "C" int ssn_inv(const u64 *a, u64 *out, u64 n, u64 p, void *strm) {
    if (n == 0) return 0;
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
    k_rand<<<ssn_blocks(n), 256, 0, (cudaStream_t)strm>>>(out, n, lo, range, seed, stream);
    return ssn_check_launch();
}

// ------------------------------------------------------------------ trusted source (device speed mode)
// Zero shares: out[t][i] = sum_j c_j(i) id_t^(j+1)   (gen_zero_shares, S/masks.py:93-96)
// is ssn_gen with secret = NULL.
//
// Additive mask (S/masks.py:39-54): e = 1 + U[0, emax); alpha = e*step; comp = -e;
// alpha/comp shared over all ids.  Philox draw j = 0 is e, 1..km1 alpha coeffs,
// km1+1..2km1 comp coeffs.
__global__ void k_mask_trunc(u64 n, u64 step, u64 emax, u64 seed, u64 stream, int km1, PowTable pw, int nids,
                             u64 *__restrict__ alpha, u64 *__restrict__ comp, u64 o_t, SsnField f) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        u64 e = 1 + ssn_rand_range(seed, stream, i, 0, emax);
        u64 a = ssn_mulmod(ssn_reduce64(e, f), ssn_reduce64(step, f), f);
        u64 cm = ssn_reduce64(e, f);
        cm = cm ? f.p - cm : 0;
        u64 ca[SSN_MAXK], cc[SSN_MAXK];
#pragma unroll
        for (int j = 0; j < SSN_MAXK; j++)
            if (j < km1) {
                ca[j] = ssn_rand_range(seed, stream, i, 1 + j, f.p);
                cc[j] = ssn_rand_range(seed, stream, i, 1 + km1 + j, f.p);
            }
        for (int t = 0; t < nids; t++) {
            u64 x = a, y = cm;
#pragma unroll
            for (int j = 0; j < SSN_MAXK; j++)
                if (j < km1) {
                    x = ssn_addmod(x, ssn_mulmod(ca[j], pw.pw[t][j], f), f.p);
                    y = ssn_addmod(y, ssn_mulmod(cc[j], pw.pw[t][j], f), f.p);
                }
            alpha[t * o_t + i] = x;
            comp[t * o_t + i] = y;
        }
    }
}

extern "C" int ssn_mask_trunc(u64 n, u64 step, u64 emax, u64 seed, u64 stream, int km1, const u64 *ids, int nids,
                              u64 *alpha, u64 *comp, u64 out_tstride, u64 p, void *strm) {
    if (emax < 1 || km1 < 0 || km1 > SSN_MAXK || nids < 1 || nids > SSN_MAXJ) return SSN_ERR_ARG;
    if (n == 0) return 0;
    PowTable pw = make_pows(ids, nids, km1, p);
    k_mask_trunc<<<ssn_blocks(n), 256, 0, (cudaStream_t)strm>>>(n, step, emax, seed, stream, km1, pw, nids, alpha,
                                                                comp, out_tstride, ssn_make_field(p));
    return ssn_check_launch();
}

// Multiplicative mask (S/masks.py:67-90): one thread per window (output element): beta =
// 1 + U[0, bmax) constant over the kh x kw window, beta^-1 by Fermat, beta shared at every
// input element of the window (own coefficients per element), beta^-1 shared at the window.
// Philox: stream s draws: window o: j=0 beta, 1..km1 beta_inv coeffs; stream s+1 input
// element i: j=0..km1-1 beta coeffs.
__global__ void k_mask_beta(int c, int h, int wd, int kh, int kw, u64 n_out, u64 bmax, u64 seed, u64 stream,
                            int km1, PowTable pw, int nids, u64 *__restrict__ beta, u64 b_t,
                            u64 *__restrict__ binv, u64 bi_t, SsnField f) {
    const int oh = h / kh, ow = wd / kw;
    for (u64 o = blockIdx.x * (u64)blockDim.x + threadIdx.x; o < n_out; o += (u64)gridDim.x * blockDim.x) {
        u64 bt = 1 + ssn_rand_range(seed, stream, o, 0, bmax);
        u64 bi = ssn_powmod(bt, f.p - 2, f);
        u64 cc[SSN_MAXK];
#pragma unroll
        for (int j = 0; j < SSN_MAXK; j++)
            if (j < km1) cc[j] = ssn_rand_range(seed, stream, o, 1 + j, f.p);
        for (int t = 0; t < nids; t++) {
            u64 y = bi;
#pragma unroll
            for (int j = 0; j < SSN_MAXK; j++)
                if (j < km1) y = ssn_addmod(y, ssn_mulmod(cc[j], pw.pw[t][j], f), f.p);
            binv[t * bi_t + o] = y;
        }
        u64 img = o / ((u64)c * oh * ow);
        u64 rem = o - img * ((u64)c * oh * ow);
        int ci = (int)(rem / ((u64)oh * ow));
        int rr = (int)(rem % ((u64)oh * ow));
        int y0 = rr / ow, x0 = rr % ow;
        for (int a = 0; a < kh; a++)
            for (int b = 0; b < kw; b++) {
                u64 i = ((img * c + ci) * (u64)h + (u64)(y0 * kh + a)) * wd + (u64)(x0 * kw + b);
                u64 ca[SSN_MAXK];
#pragma unroll
                for (int j = 0; j < SSN_MAXK; j++)
                    if (j < km1) ca[j] = ssn_rand_range(seed, stream + 1, i, j, f.p);
                for (int t = 0; t < nids; t++) {
                    u64 x = bt;
#pragma unroll
                    for (int j = 0; j < SSN_MAXK; j++)
                        if (j < km1) x = ssn_addmod(x, ssn_mulmod(ca[j], pw.pw[t][j], f), f.p);
                    beta[t * b_t + i] = x;
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
    u64 n_out = (u64)nb * c * (h / kh) * (wd / kw);
    if (n_out == 0) return 0;
    PowTable pw = make_pows(ids, nids, km1, p);
    k_mask_beta<<<ssn_blocks(n_out), 256, 0, (cudaStream_t)strm>>>(c, h, wd, kh, kw, n_out, bmax, seed, stream, km1,
                                                                   pw, nids, beta, beta_tstride, binv, binv_tstride,
                                                                   ssn_make_field(p));
    return ssn_check_launch();
}

// Repeat a (nb, c, h/kh, w/kw) block tensor over kh x kw windows (host-fed parity mode beta).
__global__ void k_pool_expand(const u64 *__restrict__ blk, u64 *__restrict__ out, int c, int h, int wd, int kh,
                              int kw, u64 n) {
    const int oh = h / kh, ow = wd / kw;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
        u64 x = i % wd, y = (i / wd) % h, rest = i / ((u64)wd * h);   // rest = img*c + ci
        out[i] = blk[(rest * oh + y / kh) * ow + x / kw];
    }
}
extern "C" int ssn_pool_expand(const u64 *blk, u64 *out, int nb, int c, int h, int wd, int kh, int kw, void *strm) {
    if (kh < 1 || kw < 1 || h % kh || wd % kw) return SSN_ERR_ARG;
    u64 n = (u64)nb * c * h * wd;
    if (n == 0) return 0;
    k_pool_expand<<<ssn_blocks(n), 256, 0, (cudaStream_t)strm>>>(blk, out, c, h, wd, kh, kw, n);
    return ssn_check_launch();
}

extern "C" int ssn_version(void) { return SSN_ABI_VERSION; }
