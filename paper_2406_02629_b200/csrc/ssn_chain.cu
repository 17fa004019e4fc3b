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
// S/masks.py) are drawn in the same thread from the source's Philox lane.  HBM traffic per
// element: 8*m bytes of GEMM output in, 8*n bytes of shares out (+8*n for a residual add).
#include "ssn.h"
#include "ssn_field.cuh"
#include "ssn_lincomb.cuh"

namespace {

template <int N>
struct ChainTables {
    LinRow wf;          // Lagrange weights of the front ids at 0 (k entries)
    LinRow wp;          // Lagrange weights of the participant ids at 0 (m entries)
    LinRow rt[N];       // R^T rows: out rank t <- participants j (m entries)
    LinRow ext[N];      // Reed-Solomon rows: id t (t >= k) <- front ids (k entries)
    LinRow pw[N];       // id_t^(e+1), e < k-1
    int small_wf, small_wp, small_rt, small_ext, small_pw;
};

struct ChainArgs {
    const u64 *acc;
    u64 acc_ps;
    const u64 *bias;
    u64 bias_ps, bias_div, bias_mod;
    const u64 *other;
    u64 other_ps;
    u64 *out;
    u64 out_ps;
    u64 nel;
    int nout, senders, nonlin, relu, pool_kind, c, h, w, kh, kw, fan, nb;
    i64 lo, r, d;
    u64 neglo_mod, stepm, emax, bmax;
    int rshift;
    u64 pseed, pstream, sseed, sstream;
    unsigned long long *fail;
    int fault_rank;
};

// share of `s` for rank t with coefficients c (K-1 of them)
template <int K>
__device__ __forceinline__ u64 share_at(u64 s, const u64 (&c)[SSN_MAXK], const LinRow &pw, int small,
                                        const SsnField &f) {
    if (small) {
        u64 acc = s;
#pragma unroll
        for (int j = 0; j < K - 1; j++) acc += mul_small(c[j], (uint32_t)pw.n[j]);
        return ssn_reduce64(acc, f);
    }
    u64 acc = s;
#pragma unroll
    for (int j = 0; j < K - 1; j++) acc = ssn_addmod(acc, ssn_mulmod(c[j], pw.w[j], f), f.p);
    return acc;
}

template <int K>
__device__ __forceinline__ void coeffs(u64 (&c)[SSN_MAXK], u64 seed, u64 stream, u64 i, const SsnField &f) {
#pragma unroll
    for (int jp = 0; jp < (K - 1 + 1) / 2; jp++) ssn_rand_field2(seed, stream, i, jp, f, c[2 * jp], c[2 * jp + 1]);
}

// reshare + rerand + bias + truncation (+ residual add) of element i for all N parties.
template <int K, int N>
__device__ __forceinline__ void chain_elem(const ChainArgs &a, const ChainTables<N> &tb, u64 i, u64 (&x)[N],
                                           unsigned long long &bad, const SsnField &f) {
    constexpr int M = 2 * K - 1;
    // ---- reshare step 1 (RESHARE_OUT): participant j sub-shares its local product to the front
    u64 sub[K][SSN_MAXP];
#pragma unroll
    for (int j = 0; j < M; j++) {
        const u64 v = a.acc[(u64)j * a.acc_ps + i];
        u64 c[SSN_MAXK];
        coeffs<K>(c, a.pseed, a.pstream + j, i, f);
#pragma unroll
        for (int fr = 0; fr < K; fr++) sub[fr][j] = share_at<K>(v, c, tb.pw[fr], tb.small_pw, f);
    }
    // ---- step 2 (RESHARE_BACK): front fr applies R^T; step 3: out rank t reconstructs
    u64 back[N][SSN_MAXP];
#pragma unroll
    for (int fr = 0; fr < K; fr++)
#pragma unroll
        for (int t = 0; t < N; t++)
            if (t < a.nout) back[t][fr] = lincomb<SSN_MAXP>(sub[fr], tb.rt[t], tb.small_rt, M, f);
    // source: zero shares (gen_zero_shares) and the truncation masks (gen_additive_mask)
    u64 z[SSN_MAXK], ca[SSN_MAXK], cc[SSN_MAXK];
    coeffs<K>(z, a.sseed, a.sstream + 0, i, f);
    const u64 e = 1 + ssn_rand_range(a.sseed, a.sstream + 1, i, 0, a.emax);
    const u64 em = ssn_reduce64(e, f);
    const u64 alpha = ssn_mulmod(em, a.stepm, f);
    const u64 comp = em ? f.p - em : 0;
    coeffs<K>(ca, a.sseed, a.sstream + 2, i, f);
    coeffs<K>(cc, a.sseed, a.sstream + 3, i, f);
    const u64 ch = (a.bias_div == 1 ? i : i / a.bias_div) % a.bias_mod;
    u64 masked[N];
#pragma unroll
    for (int t = 0; t < N; t++) {
        if (t < a.senders) {
            u64 y = lincomb<SSN_MAXP>(back[t], tb.wf, tb.small_wf, K, f);
            y = ssn_addmod(y, share_at<K>(0, z, tb.pw[t], tb.small_pw, f), f.p);          // rerand
            y = ssn_addmod(y, a.bias[(u64)t * a.bias_ps + ch], f.p);                       // + bias
            if (t == a.fault_rank && i == 0) y = ssn_addmod(y, 1, f.p);                   // test hook
            masked[t] = ssn_addmod(y, share_at<K>(alpha, ca, tb.pw[t], tb.small_pw, f), f.p);  // + alpha
        }
    }
    // ---- truncation elite (TRUNC_MASKED from actives): rec, RS check, decode, floor, round
    u64 front[SSN_MAXP];
#pragma unroll
    for (int j = 0; j < K; j++) front[j] = masked[j];
    const u64 v = lincomb<SSN_MAXP>(front, tb.wf, tb.small_wf, K, f);
#pragma unroll
    for (int t = K; t < N; t++)
        if (t < a.senders) bad += (lincomb<SSN_MAXP>(front, tb.ext[t], tb.small_ext, K, f) != masked[t]);
    const u64 tm = ssn_trunc_value(v, a.lo, a.neglo_mod, a.r, a.rshift, a.d, f);
    // fresh (k, n) shares of the truncated value (SHARE_DIST), + comp at every rank
    u64 g[SSN_MAXK];
    coeffs<K>(g, a.pseed, a.pstream + M, i, f);
#pragma unroll
    for (int t = 0; t < N; t++) {
        u64 s = share_at<K>(tm, g, tb.pw[t], tb.small_pw, f);
        s = ssn_addmod(s, share_at<K>(comp, cc, tb.pw[t], tb.small_pw, f), f.p);
        if (a.other) s = ssn_addmod(s, a.other[(u64)t * a.other_ps + i], f.p);         // residual add
        x[t] = s;
    }
}

template <int K, int N>
__global__ void __launch_bounds__(128) k_chain_plain(ChainArgs a, const __grid_constant__ ChainTables<N> tb,
                                                     SsnField f) {
    unsigned long long bad = 0;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < a.nel; i += (u64)gridDim.x * blockDim.x) {
        u64 x[N];
        chain_elem<K, N>(a, tb, i, x, bad, f);
#pragma unroll
        for (int t = 0; t < N; t++) a.out[(u64)t * a.out_ps + i] = x[t];
    }
    if (a.fail && bad) atomicAdd(a.fail, bad);
}

// masked nonlinearity fused after the chain: one thread per output window, WPT windows
// per thread (spaced a grid apart, coalesced) so beta^-1 costs one Fermat inversion per WPT
// windows (Montgomery batch inversion).
constexpr int WPT = 4;

template <int K, int N>
__global__ void __launch_bounds__(128) k_chain_nonlin(ChainArgs a, const __grid_constant__ ChainTables<N> tb,
                                                      SsnField f) {
    constexpr int M = 2 * K - 1;
    unsigned long long bad = 0;
    const int oh = a.h / a.kh, ow = a.w / a.kw;
    const u64 n_out = (u64)a.nb * a.c * oh * ow;
    const u64 T = (u64)gridDim.x * blockDim.x;
    for (u64 o0 = blockIdx.x * (u64)blockDim.x + threadIdx.x; o0 < n_out; o0 += T * WPT) {
        u64 plain[WPT], beta[WPT], pre[WPT];
        u64 run = 1;
#pragma unroll
        for (int q = 0; q < WPT; q++) {
            const u64 o = o0 + (u64)q * T;
            plain[q] = 0;
            beta[q] = 1;
            if (o < n_out) {
                beta[q] = 1 + ssn_rand_range(a.sseed, a.sstream + 4, o, 0, a.bmax);   // window-constant beta
                u64 base_in = o;
                if (a.kh != 1 || a.kw != 1) {
                    const uint32_t o32 = (uint32_t)o, chw = (uint32_t)(a.c * oh * ow), hw = (uint32_t)(oh * ow);
                    const uint32_t img = o32 / chw, rem = o32 - img * chw;
                    const uint32_t ci = rem / hw, rr = rem - ci * hw;
                    const uint32_t y0 = rr / (uint32_t)ow, x0 = rr - y0 * (uint32_t)ow;
                    base_in = (((u64)img * a.c + ci) * (u64)a.h + (u64)(y0 * a.kh)) * a.w + (u64)(x0 * a.kw);
                }
                i64 acc = a.pool_kind == 1 ? INT64_MIN : 0;
                for (int wy = 0; wy < a.kh; wy++)
                    for (int wx = 0; wx < a.kw; wx++) {
                        const u64 i = base_in + (u64)wy * a.w + wx;
                        u64 x[N];
                        chain_elem<K, N>(a, tb, i, x, bad, f);
                        // participants mask with their beta shares (NONLIN_MASKED), elite rec over m
                        u64 cb[SSN_MAXK];
                        coeffs<K>(cb, a.sseed, a.sstream + 5, i, f);
                        u64 mk[SSN_MAXP];
#pragma unroll
                        for (int j = 0; j < M; j++)
                            mk[j] = ssn_mulmod(x[j], share_at<K>(beta[q], cb, tb.pw[j], tb.small_pw, f), f);
                        const u64 v = lincomb<SSN_MAXP>(mk, tb.wp, tb.small_wp, M, f);
                        i64 sv = v > f.half ? (i64)v - (i64)f.p : (i64)v;
                        if (a.relu && sv <= 0) sv = 0;
                        if (a.pool_kind == 1) acc = sv > acc ? sv : acc;
                        else acc += sv;
                    }
                plain[q] = acc < 0 ? (u64)((i64)f.p + acc) : (u64)acc;      // encode_signed (NONLIN_PLAIN)
            }
            run = ssn_mulmod(run, beta[q], f);
            pre[q] = run;
        }
        u64 inv = ssn_powmod(run, f.p - 2, f);
#pragma unroll
        for (int q = WPT - 1; q >= 0; q--) {
            const u64 bi = q ? ssn_mulmod(inv, pre[q - 1], f) : inv;
            inv = ssn_mulmod(inv, beta[q], f);
            pre[q] = bi;                                     // beta^-1 of window q
        }
#pragma unroll
        for (int q = 0; q < WPT; q++) {
            const u64 o = o0 + (u64)q * T;
            if (o >= n_out) continue;
            u64 cbi[SSN_MAXK];
            coeffs<K>(cbi, a.sseed, a.sstream + 6, o, f);
#pragma unroll
            for (int t = 0; t < N; t++)
                if (t < a.fan)
                    a.out[(u64)t * a.out_ps + o] =
                        ssn_mulmod(plain[q], share_at<K>(pre[q], cbi, tb.pw[t], tb.small_pw, f), f);
        }
    }
    if (a.fail && bad) atomicAdd(a.fail, bad);
}

template <int K, int N>
int launch_chain(const ssn_chain_desc *d, cudaStream_t st) {
    constexpr int M = 2 * K - 1;
    const u64 p = d->p;
    ChainTables<N> tb;
    u64 row[SSN_MAXJ];
    // Lagrange weights at 0 of ids[0..cnt)
    auto lagrange = [&](int cnt) {
        for (int i = 0; i < SSN_MAXJ; i++) row[i] = 0;
        for (int i = 0; i < cnt; i++) {
            unsigned __int128 num = 1, den = 1;
            for (int j = 0; j < cnt; j++)
                if (j != i) {
                    num = num * (d->ids[j] % p) % p;
                    den = den * ((d->ids[j] + p - d->ids[i] % p) % p) % p;
                }
            row[i] = (u64)(num * inv_host((u64)den, p) % p);
        }
    };
    lagrange(K);
    tb.small_wf = make_row(tb.wf, row, K, p);
    lagrange(M);
    tb.small_wp = make_row(tb.wp, row, M, p);
    tb.small_rt = tb.small_ext = tb.small_pw = 1;
    for (int t = 0; t < N; t++) {
        for (int j = 0; j < SSN_MAXJ; j++) row[j] = 0;
        for (int j = 0; j < M; j++) row[j] = d->rt[t * M + j];
        tb.small_rt &= make_row(tb.rt[t], row, M, p);
        for (int j = 0; j < SSN_MAXJ; j++) row[j] = 0;
        if (t >= K) {
            for (int j = 0; j < K; j++) row[j] = d->ext[(t - K) * K + j];
            tb.small_ext &= make_row(tb.ext[t], row, K, p);
        } else {
            make_row(tb.ext[t], row, K, p);
        }
        for (int j = 0; j < SSN_MAXJ; j++) row[j] = 0;
        unsigned __int128 acc = 1;
        for (int j = 0; j < K - 1; j++) {
            acc = acc * (d->ids[t] % p) % p;
            row[j] = (u64)acc;
        }
        int ok = make_row(tb.pw[t], row, K - 1, p);
        for (int j = 0; j < K - 1; j++) ok = ok && tb.pw[t].n[j] >= 0;
        tb.small_pw &= ok && tb.pw[t].one;
    }
    const SsnField f = ssn_make_field(p);
    ChainArgs a;
    a.acc = d->acc;
    a.acc_ps = d->acc_pstride;
    a.bias = d->bias;
    a.bias_ps = d->bias_pstride;
    a.bias_div = d->bias_div;
    a.bias_mod = d->bias_mod;
    a.other = d->other;
    a.other_ps = d->other_pstride;
    a.out = d->out;
    a.out_ps = d->out_pstride;
    a.nel = d->nel;
    a.nout = d->nout;
    a.senders = d->verify ? N : K;
    a.nonlin = d->nonlin;
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
    if (a.senders > a.nout) return SSN_ERR_ARG;
    if (!d->nonlin) {
        u64 blocks = (a.nel + 127) / 128;
        if (blocks > 148ull * 12) blocks = 148ull * 12;
        k_chain_plain<K, N><<<(unsigned)blocks, 128, 0, st>>>(a, tb, f);
    } else {
        const u64 n_out = (u64)d->nb * d->c * (d->h / d->kh) * (d->w / d->kw);
        if (n_out >= (1ull << 32)) return SSN_ERR_UNSUPPORTED;
        u64 blocks = (n_out + 128 * WPT - 1) / (128 * WPT);
        if (blocks > 148ull * 12) blocks = 148ull * 12;
        if (blocks < 1) blocks = 1;
        k_chain_nonlin<K, N><<<(unsigned)blocks, 128, 0, st>>>(a, tb, f);
    }
    return cudaGetLastError() == cudaSuccess ? 0 : SSN_ERR_CUDA;
}

}  // namespace

extern "C" int ssn_layer_chain(const ssn_chain_desc *d, void *stream) {
    if (!d || !d->acc || !d->bias || !d->out || !d->ids || !d->rt) return SSN_ERR_ARG;
    if (d->r < 1 || d->d < 1 || d->emax < 1 || d->nout < d->k || d->nout > d->n) return SSN_ERR_ARG;
    if (d->verify && (!d->ext || d->nout != d->n)) return SSN_ERR_ARG;
    if (d->nonlin) {
        if (d->kh < 1 || d->kw < 1 || d->h % d->kh || d->w % d->kw || d->bmax < 1 || d->fan < 1 || d->fan > d->n ||
            d->pool_kind < 0 || d->pool_kind > 2 || (d->pool_kind == 0 && (d->kh != 1 || d->kw != 1)))
            return SSN_ERR_ARG;
        if ((u64)d->nb * d->c * d->h * d->w != d->nel) return SSN_ERR_ARG;
    }
    if (d->nel == 0) return 0;
    cudaStream_t st = (cudaStream_t)stream;
    if (d->k == 2 && d->n == 3) return launch_chain<2, 3>(d, st);
    if (d->k == 3 && d->n == 5) return launch_chain<3, 5>(d, st);
    if (d->k == 4 && d->n == 7) return launch_chain<4, 7>(d, st);
    return SSN_ERR_UNSUPPORTED;
}
