// ssn_gemm_simt.cu -- exact mod-p share GEMM / implicit-im2col conv on CUDA cores.
//
// The local product of sss_linear (S/layers.py:245-255):
//   conv:  acc(O, OH*OW) = W(O, C*kh*kw) @ im2col(x)   (im2col: S/model.py:354-371)
//   dense: acc(O,)       = W(O, K) @ x.ravel()
// computed exactly: 64-bit operands, 128-bit accumulators (two u64 registers), one
// reduction mod p per output.  Batched over parties (independent W and x per party) and
// images (N = images * OH * OW).  This is the small-shape / any-p path; the tensor-core
// path for large conv/dense tiles is ssn_gemm_tc.cu.
#include "ssn_field.cuh"
#include "ssn.h"

#define TM 64
#define TN 64
#define TK 16

struct ConvGeom {
    int C, H, W, kh, kw, stride, pad, OH, OW;
};

// B(k, n): conv -> x[img][c][oy*s+i-pad][ox*s+j-pad] (zero outside); dense -> x[img][k]
template <bool CONV>
__device__ __forceinline__ u64 load_b(const u64 *__restrict__ x, const ConvGeom &g, int K, int k, u64 n,
                                      u64 nimg_pix) {
    if (CONV) {
        u64 ohw = (u64)g.OH * g.OW;
        u64 img = n / ohw;
        int pix = (int)(n - img * ohw);
        int oy = pix / g.OW, ox = pix - oy * g.OW;
        int c = k / (g.kh * g.kw);
        int r = k - c * g.kh * g.kw;
        int i = r / g.kw, j = r - i * g.kw;
        int sy = oy * g.stride + i - g.pad, sx = ox * g.stride + j - g.pad;
        if (sy < 0 || sy >= g.H || sx < 0 || sx >= g.W) return 0;
        return x[((img * g.C + c) * g.H + sy) * (u64)g.W + sx];
    } else {
        return x[n * (u64)K + k];
    }
}

template <bool CONV>
__global__ void __launch_bounds__(256) k_gemm_simt(const u64 *__restrict__ A, u64 a_b, const u64 *__restrict__ X,
                                                   u64 x_b, u64 *__restrict__ out, u64 o_b, int M, int K, u64 N,
                                                   u64 ohw, ConvGeom g, SsnField f, u64 r64, int fold_every) {
    __shared__ u64 sA[TK][TM + 1];
    __shared__ u64 sB[TK][TN + 1];
    const int party = blockIdx.z;
    A += party * a_b;
    X += party * x_b;
    out += party * o_b;
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const int m0 = blockIdx.y * TM;
    const u64 n0 = (u64)blockIdx.x * TN;
    u128s acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; a++)
#pragma unroll
        for (int b = 0; b < 4; b++) acc[a][b] = {0, 0};

    int since_fold = 0;
    for (int k0 = 0; k0 < K; k0 += TK) {
#pragma unroll
        for (int l = 0; l < 4; l++) {
            int e = threadIdx.x + l * 256;      // 0..1023
            int mm = e / TK, kk = e % TK;       // A tile: 64 rows x 16 k
            int gm = m0 + mm, gk = k0 + kk;
            sA[kk][mm] = (gm < M && gk < K) ? A[(u64)gm * K + gk] : 0;
            int kb = e / TN, nn = e % TN;       // B tile: 16 k x 64 cols
            u64 gn = n0 + nn;
            int gkb = k0 + kb;
            sB[kb][nn] = (gn < N && gkb < K) ? load_b<CONV>(X, g, K, gkb, gn, ohw) : 0;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < TK; kk++) {
            u64 av[4], bv[4];
#pragma unroll
            for (int a = 0; a < 4; a++) av[a] = sA[kk][ty + 16 * a];
#pragma unroll
            for (int b = 0; b < 4; b++) bv[b] = sB[kk][tx + 16 * b];
#pragma unroll
            for (int a = 0; a < 4; a++)
#pragma unroll
                for (int b = 0; b < 4; b++) ssn_mac(acc[a][b], av[a], bv[b]);
        }
        __syncthreads();
        since_fold += TK;
        if (since_fold >= fold_every) {
            since_fold = 0;
#pragma unroll
            for (int a = 0; a < 4; a++)
#pragma unroll
                for (int b = 0; b < 4; b++) acc[a][b] = {ssn_reduce128(acc[a][b], f, r64), 0};
        }
    }
#pragma unroll
    for (int a = 0; a < 4; a++) {
        int gm = m0 + ty + 16 * a;
        if (gm >= M) continue;
#pragma unroll
        for (int b = 0; b < 4; b++) {
            u64 gn = n0 + tx + 16 * b;
            if (gn >= N) continue;
            u64 img = gn / ohw, pix = gn - img * ohw;
            out[(img * M + gm) * ohw + pix] = ssn_reduce128(acc[a][b], f, r64);
        }
    }
}

static int fold_period(u64 p) {
    int s = 0;
    while (s < 64 && (p >> s)) s++;
    // products < 2^(2s); keep sum < 2^127
    int room = 127 - 2 * s;
    if (room >= 20) return 1 << 20;
    if (room < 5) return TK;
    return (1 << room) / TK * TK;
}

// Direct conv for few output channels (LeNet's 1->6 and 6->16 5x5 layers): one thread per
// output pixel computes all O <= OMAX channels, the party's weights broadcast from shared
// memory (k-major), 128-bit accumulators, one reduction per output.  The tiled kernel above
// would spend 64 - O of its 64 weight rows on zeros, and the tensor-core path needs an im2col
// expansion of 6*Kpad bytes per output pixel.
template <int OMAX>
__global__ void __launch_bounds__(128) k_conv_direct(const u64 *__restrict__ Wt, u64 w_b, const u64 *__restrict__ X,
                                                     u64 x_b, u64 *__restrict__ out, u64 o_b, int O, int K, u64 N,
                                                     ConvGeom g, SsnField f, u64 r64) {
    extern __shared__ u64 sw[];                       // [K][OMAX]
    const int party = blockIdx.y;
    Wt += party * w_b;
    X += party * x_b;
    out += party * o_b;
    for (int e = threadIdx.x; e < K * OMAX; e += blockDim.x) {
        const int k = e / OMAX, o = e - k * OMAX;
        sw[e] = o < O ? Wt[(u64)o * K + k] : 0;
    }
    __syncthreads();
    const u64 ohw = (u64)g.OH * g.OW;
    const u64 chw = (u64)g.C * g.H * g.W;
    for (u64 n = blockIdx.x * (u64)blockDim.x + threadIdx.x; n < N; n += (u64)gridDim.x * blockDim.x) {
        const u64 img = n / ohw;
        const int pix = (int)(n - img * ohw);
        const int oy = pix / g.OW, ox = pix - (pix / g.OW) * g.OW;
        u128s acc[OMAX];
#pragma unroll
        for (int o = 0; o < OMAX; o++) acc[o] = {0, 0};
        const u64 *xi = X + img * chw;
        int k = 0;
        for (int c = 0; c < g.C; c++)
            for (int i = 0; i < g.kh; i++) {
                const int sy = oy * g.stride + i - g.pad;
                const bool rowok = sy >= 0 && sy < g.H;
                for (int j = 0; j < g.kw; j++, k++) {
                    const int sx = ox * g.stride + j - g.pad;
                    if (!rowok || sx < 0 || sx >= g.W) continue;
                    const u64 v = xi[((u64)c * g.H + sy) * g.W + sx];
                    const u64 *wk = sw + k * OMAX;
#pragma unroll
                    for (int o = 0; o < OMAX; o++) ssn_mac(acc[o], v, wk[o]);
                }
            }
#pragma unroll
        for (int o = 0; o < OMAX; o++)
            if (o < O) out[(img * O + o) * ohw + pix] = ssn_reduce128(acc[o], f, r64);
    }
}

// conv: W [parties][O][C*kh*kw], x [parties][nimg][C][H][W] -> out [parties][nimg][O][OH*OW]
extern "C" int ssn_conv_simt(const u64 *w, u64 w_pstride, const u64 *x, u64 x_pstride, u64 *out, u64 out_pstride,
                             int nparty, int nimg, int O, int C, int H, int W, int kh, int kw, int stride, int pad,
                             u64 p, void *strm) {
    if (nparty < 1 || nimg < 1 || O < 1 || C < 1 || kh < 1 || kw < 1 || stride < 1 || pad < 0) return SSN_ERR_ARG;
    ConvGeom g;
    g.C = C; g.H = H; g.W = W; g.kh = kh; g.kw = kw; g.stride = stride; g.pad = pad;
    g.OH = (H + 2 * pad - kh) / stride + 1;
    g.OW = (W + 2 * pad - kw) / stride + 1;
    if (g.OH < 1 || g.OW < 1) return SSN_ERR_ARG;
    int K = C * kh * kw;
    u64 ohw = (u64)g.OH * g.OW;
    u64 N = ohw * nimg;
    dim3 grid((unsigned)((N + TN - 1) / TN), (unsigned)((O + TM - 1) / TM), (unsigned)nparty);
    SsnField f = ssn_make_field(p);
    u64 r64 = (u64)((((unsigned __int128)1) << 64) % p);
    // few output channels and no mid-sum folding needed: the direct kernel
    if (O <= 16 && (u64)K * 16 * 8 <= 48 * 1024 && fold_period(p) >= K && N < (1ull << 40)) {
        u64 blocks = (N + 127) / 128;
        if (blocks > 148ull * 32) blocks = 148ull * 32;
        SSN_COUNT_LAUNCH();
        if (O <= 8)
            k_conv_direct<8><<<dim3((unsigned)blocks, (unsigned)nparty), 128, (size_t)K * 8 * 8, (cudaStream_t)strm>>>(
                w, w_pstride, x, x_pstride, out, out_pstride, O, K, N, g, f, r64);
        else
            k_conv_direct<16><<<dim3((unsigned)blocks, (unsigned)nparty), 128, (size_t)K * 16 * 8, (cudaStream_t)strm>>>(
                w, w_pstride, x, x_pstride, out, out_pstride, O, K, N, g, f, r64);
        return cudaGetLastError() == cudaSuccess ? 0 : SSN_ERR_CUDA;
    }
    SSN_COUNT_LAUNCH();
    k_gemm_simt<true><<<grid, 256, 0, (cudaStream_t)strm>>>(w, w_pstride, x, x_pstride, out, out_pstride, O, K, N,
                                                            ohw, g, f, r64, fold_period(p));
    return cudaGetLastError() == cudaSuccess ? 0 : SSN_ERR_CUDA;
}

// dense: W [parties][O][K], x [parties][nimg][K] -> out [parties][nimg][O]
extern "C" int ssn_dense_simt(const u64 *w, u64 w_pstride, const u64 *x, u64 x_pstride, u64 *out, u64 out_pstride,
                              int nparty, int nimg, int O, int K, u64 p, void *strm) {
    if (nparty < 1 || nimg < 1 || O < 1 || K < 1) return SSN_ERR_ARG;
    ConvGeom g = {};
    dim3 grid((unsigned)((nimg + TN - 1) / TN), (unsigned)((O + TM - 1) / TM), (unsigned)nparty);
    SsnField f = ssn_make_field(p);
    u64 r64 = (u64)((((unsigned __int128)1) << 64) % p);
    SSN_COUNT_LAUNCH();
    k_gemm_simt<false><<<grid, 256, 0, (cudaStream_t)strm>>>(w, w_pstride, x, x_pstride, out, out_pstride, O, K,
                                                             (u64)nimg, 1, g, f, r64, fold_period(p));
    return cudaGetLastError() == cudaSuccess ? 0 : SSN_ERR_CUDA;
}
