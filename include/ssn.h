/*
 * ssn.h -- C ABI of the B200-native SSNet secure-inference hot path (libssn_b200.so).
 *
 * The reference (SSNet, /root/reference/pkg/src/ssnet) is a pure-Python package with no
 * FFI: its "plugin boundary" is the Python API (ssnet.*).  These entry points are what a
 * maintainer would bind (ctypes / cffi) to replace the numpy
 * dtype=object expressions on that path; each declaration cites the reference code it
 * replaces.  The Python mirror of the ssnet API lives in paper_2406_02629_b200/ and calls
 * nothing else.
 *
 * Conventions
 *   - field elements: canonical uint64 in [0, p), p prime, p < 2^62 (reference: p < 2^57,
 *     S/field.py:64-75); signed plaintext: int64.
 *   - every pointer named like a tensor is a caller-owned DEVICE pointer; `ids`, `w`,
 *     `rt`, `ext` are small HOST arrays baked into kernel parameters.
 *   - multi-party / multi-image operands are strided views: element (b, j, i) of a
 *     "pts" view lives at pts[b*bstride + j*jstride + i].
 *   - `stream` is a cudaStream_t; calls are asynchronous and reentrant per stream;
 *     no hidden allocation.
 *   - return 0 on success, < 0 on error (SSN_ERR_*); the Python layer maps errors to the
 *     reference's exception types.
 */
#ifndef SSN_H
#define SSN_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SSN_ABI_VERSION 1
#define SSN_OK 0
#define SSN_ERR_ARG (-1)
#define SSN_ERR_CUDA (-2)
#define SSN_ERR_UNSUPPORTED (-3)

int ssn_version(void);

/* Kernels this library has launched in this process (every entry point counts each of its
 * launches; bench.py reports the per-step difference as gpu_launches). */
unsigned long long ssn_kernel_launches(void);

/* out[i] = a[i] OP b[bidx(i)], bidx(i) = (i / b_div) % b_mod + (i / b_div2) * b_mul2.
 * op: 0 add, 1 sub, 2 mul, 3 neg (b unused).
 * Replaces share_add/share_sub/share_mul (S/sss.py:238-276), PrimeField.add/sub/mul/neg
 * (S/field.py:89-99), the bias broadcast `vals + b[:, None]` (S/layers.py:261-265),
 * the masks `x * beta` (S/layers.py:341) and the unmask `plain * beta_inv` (S/layers.py:379). */
int ssn_ewise(int op, const uint64_t *a, const uint64_t *b, uint64_t *out, uint64_t n, uint64_t b_div,
              uint64_t b_mod, uint64_t b_div2, uint64_t b_mul2, uint64_t p, void *stream);

/* Shamir share generation, SssScheme.gen (S/sss.py:118-147):
 * out[b][t][i] = secret[b][i] + sum_{j<km1} c_j[b][i] * ids[t]^(j+1) mod p.
 * Coefficients: coeffs[b][j][i] (host-fed, draw order c_1..c_{k-1}: parity mode) or, when
 * coeffs == NULL, Philox4x32-10(seed, stream + b, i, j) uniform in [0, p) (speed mode).
 * secret == NULL shares zero (gen_zero_shares, S/masks.py:93-96). ids: host, <= 16. */
int ssn_gen(const uint64_t *secret, uint64_t secret_bstride, const uint64_t *coeffs, uint64_t coeff_bstride,
            uint64_t seed, uint64_t stream, int km1, const uint64_t *ids, int nids, uint64_t *out,
            uint64_t out_bstride, uint64_t out_tstride, uint64_t n, int nbatch, uint64_t p, void *strm);

/* Lagrange reconstruction, SssScheme.rec (S/sss.py:172-194):
 * out[b][i] = sum_{j<m} w[j] * pts[b][j][i] mod p.  w: host Lagrange weights (S/sss.py:151-170). */
int ssn_rec(const uint64_t *pts, uint64_t pts_bstride, uint64_t pts_jstride, const uint64_t *w, int m,
            uint64_t *out, uint64_t out_bstride, uint64_t n, int nbatch, uint64_t p, void *strm);

/* Reshare step 2, reshare_degree_reduce (S/protocol.py:165-185): for front rank b,
 * out[b][t][i] = sum_{j<m} rt[t*m + j] * pts[b][j][i] mod p, rt = R^T[:nout] (host). */
int ssn_reduce_apply(const uint64_t *pts, uint64_t pts_bstride, uint64_t pts_jstride, int m, const uint64_t *rt,
                     int nout, uint64_t *out, uint64_t out_bstride, uint64_t out_tstride, uint64_t n, int nbatch,
                     uint64_t p, void *strm);

/* Reshare step 3 + rerand + bias (+ truncation front mask), fused:
 * out[b][i] = sum_{j<k} w[j]*pts[b][j][i] + zero[b][i] + bias[b][(i/bias_div)%bias_mod] + alpha[b][i].
 * zero/bias/alpha may be NULL.  Replaces S/protocol.py:187-198 (rec of RESHARE_BACK points),
 * rerand (S/protocol.py:260-265), the bias add (S/layers.py:261-267) and, when the next op is
 * a truncation, `share_add(x, alpha)` (S/layers.py:293). */
int ssn_reshare_finish(const uint64_t *pts, uint64_t pts_bstride, uint64_t pts_jstride, const uint64_t *w, int k,
                       const uint64_t *zero, uint64_t zero_bstride, const uint64_t *bias, uint64_t bias_bstride,
                       uint64_t bias_div, uint64_t bias_mod, const uint64_t *alpha, uint64_t alpha_bstride,
                       uint64_t *out, uint64_t out_bstride, uint64_t n, int nbatch, uint64_t p, void *strm);

/* Elite side of the masked truncation, sss_truncation (S/layers.py:295-315):
 * v = rec(pts[0..k)); optional Reed-Solomon check of pts[k..npts) against the Lagrange
 * extrapolation ext[(e-k)*k + j] (failures added to *fail, device counter, may be NULL);
 * shifted = ((v - lo) mod p) + lo with lo = -value_bound + r*d (S/layers.py:231-233,288);
 * t = floor(shifted / r); if d > 1 t = round_half_away(t, d) (S/model.py:44-50);
 * then fresh (k,n) shares of t mod p at ids written to out[t_idx*out_tstride + i]
 * (nids == 0: out[i] = t mod p).  Coefficients as in ssn_gen. */
int ssn_trunc_elite(const uint64_t *pts, uint64_t pts_jstride, int npts, int k, const uint64_t *w,
                    const uint64_t *ext, int64_t value_bound, int64_t r, int64_t d, const uint64_t *coeffs,
                    uint64_t seed, uint64_t stream, int km1, const uint64_t *ids, int nids, uint64_t *out,
                    uint64_t out_tstride, unsigned long long *fail, uint64_t n, uint64_t p, void *strm);

/* Elite side of the masked nonlinearity, sss_nonlinear (S/layers.py:345-364):
 * v = rec over m = 2k-1 product shares, decode_signed (S/field.py:130-134), ReLU, window
 * max (pool_kind 1) / sum (2) over non-overlapping kh x kw windows of nb x (c,h,wd) images
 * (pool_blocks, S/model.py:374-377), encode_signed.  pool_kind 0: kh = kw = 1. */
int ssn_nonlin_elite(const uint64_t *pts, uint64_t pts_jstride, int m, const uint64_t *w, int relu, int pool_kind,
                     int nb, int c, int h, int wd, int kh, int kw, uint64_t *plain, uint64_t p, void *strm);

/* Signed embedding (S/field.py:120-134). encode counts |x| > (p-1)/2 into *overflow. */
int ssn_encode_signed(const int64_t *x, uint64_t *out, uint64_t n, unsigned long long *overflow, uint64_t p,
                      void *strm);
int ssn_decode_signed(const uint64_t *v, int64_t *out, uint64_t n, uint64_t p, void *strm);

/* Multiplicative inverse (Fermat), PrimeField.inv (S/field.py:101-116); 0 -> 0. */
int ssn_inv(const uint64_t *a, uint64_t *out, uint64_t n, uint64_t p, void *strm);

/* out[i] = lo + Philox uniform in [0, range) (device speed-mode randomness). */
int ssn_rand(uint64_t *out, uint64_t n, uint64_t lo, uint64_t range, uint64_t seed, uint64_t stream, void *strm);

/* Trusted source, additive mask (gen_additive_mask, S/masks.py:39-54): e = 1 + U[0, emax),
 * alpha = e*step, comp = -e, both shared at ids: alpha[t][i], comp[t][i].
 * Consumes THREE Philox streams: e from `stream`, the alpha / comp sharing coefficients from
 * `stream + 1` / `stream + 2` -- callers reserve all three (DeviceRng.next_stream(3)). */
int ssn_mask_trunc(uint64_t n, uint64_t step, uint64_t emax, uint64_t seed, uint64_t stream, int km1,
                   const uint64_t *ids, int nids, uint64_t *alpha, uint64_t *comp, uint64_t out_tstride, uint64_t p,
                   void *strm);

/* Trusted source, multiplicative mask (gen_multiplicative_mask, S/masks.py:67-90): beta
 * constant per kh x kw window in [1, bmax], shared per input element; beta^-1 shared per
 * window.  Consumes THREE Philox streams: beta from `stream`, the beta sharing coefficients from
 * `stream + 1`, the beta^-1 sharing coefficients from `stream + 2` -- callers reserve all three. */
int ssn_mask_beta(int nb, int c, int h, int wd, int kh, int kw, uint64_t bmax, uint64_t seed, uint64_t stream,
                  int km1, const uint64_t *ids, int nids, uint64_t *beta, uint64_t beta_tstride, uint64_t *binv,
                  uint64_t binv_tstride, uint64_t p, void *strm);

/* Overlapping-window gather of share tensors (builder op "gather"; e.g. ResNet's 3x3/s2/p1 stem
 * max-pool as the reference's non-overlapping pool over gathered windows, S/model.py:374-377):
 * x [nb][c][h][w] -> out [nb][c][OH*kh][OW*kw], OH = (h + 2 pad - kh) / stride + 1, with
 * out[.., oy*kh + dy, ox*kw + dx] = x[.., oy*stride - pad + dy, ox*stride - pad + dx] or 0 (a
 * valid share of 0) outside.  Local: every party gathers its own share. */
int ssn_window_gather(const uint64_t *x, uint64_t *out, int nb, int c, int h, int w, int kh, int kw, int stride,
                      int pad, void *strm);

/* Repeat a (nb, c, h/kh, wd/kw) block over windows (np.repeat twice, S/masks.py:84). */
int ssn_pool_expand(const uint64_t *blk, uint64_t *out, int nb, int c, int h, int wd, int kh, int kw, void *strm);

/* Local share product of sss_linear (S/layers.py:245-255), exact mod p on CUDA cores:
 * conv  W[party][O][C*kh*kw] x im2col(x[party][img][C][H][W]) -> out[party][img][O][OH*OW]
 * dense W[party][O][K] x x[party][img][K] -> out[party][img][O]. */
int ssn_conv_simt(const uint64_t *w, uint64_t w_pstride, const uint64_t *x, uint64_t x_pstride, uint64_t *out,
                  uint64_t out_pstride, int nparty, int nimg, int O, int C, int H, int W, int kh, int kw, int stride,
                  int pad, uint64_t p, void *strm);
int ssn_dense_simt(const uint64_t *w, uint64_t w_pstride, const uint64_t *x, uint64_t x_pstride, uint64_t *out,
                   uint64_t out_pstride, int nparty, int nimg, int O, int K, uint64_t p, void *strm);

/* Tensor-core field GEMM (tcgen05.mma kind::i8, TMEM accumulators, TMA-fed), the same
 * contraction as ssn_conv_simt/ssn_dense_simt (S/layers.py:252,254):
 *  - ssn_limb_split: x[party][rows][K] u64 -> planes[party][L][rows][Kpad] u8 (little-endian
 *    limbs, zero padded to Kpad % 16 == 0);  used for weights (once) and dense activations.
 *  - ssn_im2col_limbs: conv unfold (S/model.py:354-371) fused with the limb split:
 *    x[party][img][C][H][W] -> planes[party][L][img*OH*OW][Kpad], k = (c, i, j).
 *  - ssn_gemm_tc: out[party][img][O][ohw] (row = img*ohw + pix) = A . B^T mod p with
 *    A planes [party][L][M][Kpad], B planes [party][L][O][Kpad]; L in {6,7,8};
 *    requires L * Kpad * 255^2 < 2^32. */
int ssn_limb_split(const uint64_t *x, uint64_t rows, uint64_t K, uint64_t Kpad, int L, uint8_t *planes,
                   uint64_t x_pstride, int nparty, void *stream);
int ssn_im2col_limbs(const uint64_t *x, int nparty, int nimg, int C, int H, int W, int kh, int kw, int stride,
                     int pad, int L, uint8_t *planes, uint64_t Kpad, uint64_t x_pstride, void *stream);
int ssn_gemm_tc(const uint8_t *a_planes, const uint8_t *b_planes, int nparty, int L, int M, int O, uint64_t Kpad,
                uint64_t ohw, uint64_t *out, uint64_t out_pstride, uint64_t p, void *stream);

/* Implicit-GEMM convolution on the tensor cores from CHANNEL-MAJOR limb planes (the A operand
 * is M-major: TMA loads 128 consecutive output pixels x 64 channels per limb; p = 2^45 - 55):
 *  mode 1 (1x1, stride 1, pad 0): a_planes [party][L][C][nimg*H*W];
 *  mode 2 (3x3, stride 1, pad 1): a_planes [3][party][L][C][nimg][H][Wp], Wp >= W, Wp % 16 == 0:
 *    copy dx holds the rows shifted by dx - 1 columns, zero where the shift leaves the image
 *    (that and TMA's out-of-range zero fill for rows are the convolution's zero padding).
 * b_planes [party][L][O][taps*C] with k = tap*C + c (tap = dy*3 + dx; weights (O,C,kh,kw)
 * permuted to (O,kh,kw,C)).  out as ssn_gemm_tc with ohw = H*W.  C % 64 == 0.
 * Replaces im2col + GEMM of sss_linear (S/model.py:354-371, S/layers.py:252). */
int ssn_gemm_tc_conv(const uint8_t *a_planes, int mode, int nimg, int C, int H, int W, int Wp, const uint8_t *b_planes,
                     int nparty, int O, uint64_t *out, uint64_t out_pstride, uint64_t p, void *stream);
/* x [party][img][C][H][W] -> channel-major limb planes [copies][party][L][C][img][H][Wp].
 * copies == 1 (Wp == W: the contiguous mode-1 layout) or 3 (mode 2: copy dx at column x+1-dx);
 * unwritten bytes are untouched -- the caller zeroes the buffer once. */
int ssn_planes_cn(const uint64_t *x, int nparty, int nimg, int C, int H, int W, int Wp, int L, uint8_t *planes,
                  uint64_t x_pstride, int copies, void *stream);
/* Fill mode-2 copies 0 and 2 from copy 1 (planes [3][rows][Wp], rows = party*L*C*img*H): the
 * +-1 column shifts, 16-byte vectorised. */
int ssn_planes_shift(uint8_t *planes, uint64_t rows, int Wp, void *stream);

/* Fused per-layer protocol chain for co-resident parties (one launch per secure layer after
 * its share GEMM).  Per element i of the linear op's output, for all n parties at once:
 *   reshare_degree_reduce (S/protocol.py:131-199): participant j (j < m = 2k-1) sub-shares
 *     acc[j][i] to the k front ranks (RESHARE_OUT), front ranks apply R^T (RESHARE_BACK),
 *     out rank t (t < nout) reconstructs;  + zero share (rerand, S/protocol.py:260-265)
 *     + bias share (S/layers.py:260-267);
 *   sss_truncation (S/layers.py:277-323): + alpha share, elite rec over the k front ranks,
 *     [verify: Reed-Solomon check of the n-k extra masked shares -> *fail], window decode,
 *     floor(/r), round_half_away(/d), fresh (k,n) shares (SHARE_DIST), + comp share;
 *   [other != NULL] share_add of a residual input (S/sss.py:238);
 *   [nonlin] sss_nonlinear (S/layers.py:326-380): * beta shares (window-constant beta),
 *     elite rec over m, decode, ReLU, max/sum over kh x kw windows, encode (NONLIN_PLAIN),
 *     * beta^-1 shares at ranks t < fan.
 * Masks are the trusted source's (S/masks.py:39-96), drawn from Philox lane (src_seed,
 * src_stream + 0..6); protocol randomness from (party_seed, party_stream + 0..m).
 * Layouts: acc [m][nel] at acc_pstride; bias [n][O] at bias_pstride with channel
 * (i / bias_div) % bias_mod; other [n][nel]; out [n][nel or n_out] at out_pstride.
 * Host arrays: ids[n] (party ids), rt[n*m] (R^T rows for all n ranks), ext[(n-k)*k]
 * (Lagrange extrapolation from the front ids to ids[k..n)).  Supported (k, n): (2,3),
 * (3,5), (4,7). */
typedef struct ssn_chain_desc {
    const uint64_t *acc;
    uint64_t acc_pstride;
    const uint64_t *bias;
    uint64_t bias_pstride, bias_div, bias_mod;
    const uint64_t *other;
    uint64_t other_pstride;
    uint64_t *out;
    uint64_t out_pstride;
    uint64_t nel;
    int nout;
    int64_t value_bound, r, d;
    uint64_t emax;
    int verify;
    unsigned long long *fail;
    int nonlin, relu, pool_kind, nb, c, h, w, kh, kw, fan;
    uint64_t bmax;
    uint64_t party_seed, party_stream, src_seed, src_stream;
    int k, n;
    const uint64_t *ids, *rt, *ext;
    uint64_t p;
    int fault_rank;   /* test hook: < 0 off; else rank's reshared share of element 0 is corrupted */
    /* optional (nonlin chains): channel-major u8 limb planes of the output for the next
     * implicit-GEMM conv (ssn_gemm_tc_conv), participants t < plane_nparty, 6 limbs:
     * planes[(dx*plane_nparty + t)*plane_pstride + l*plane_lstride + c*plane_cstride
     *        + img*plane_istride + y*plane_wp + x + 1 - dx] for plane_copies copies (1: x). */
    uint8_t *planes;
    uint64_t plane_pstride, plane_lstride, plane_cstride, plane_istride;
    int plane_wp, plane_copies, plane_nparty;
    /* optional (nonlin chains): scratch [n][nel] -> run as two kernels (reshare/truncation/add
     * into scratch, then the masked nonlinearity); same results */
    uint64_t *scratch;
    /* optional (nonlin chains): the trusted source's beta^-1 from a table inv_table[b] =
     * b^-1 mod p, b < inv_table_len (must exceed bmax) instead of batch inversion */
    const uint64_t *inv_table;
    uint64_t inv_table_len;
    /* 1: only the masked nonlinearity (sss_nonlinear) of the n parties' input shares in acc
     * (a nonlinear op outside a linear chain, e.g. the global pool); reshare fields unused */
    int nonlin_only;
    /* 1: reference-stream (host-fed) masks, the parity mode of S/engine.py's purpose lanes:
     * instead of Philox draws, party t's share of the trusted source's material for element i
     * is read at image-element ii = i mod h_period (every image of the batch sees the same
     * bundle, like the reference's runs over input_index, S/engine.py:64-74):
     *   h_zero  [n][h_period]  zero shares of the linear op (gen_zero_shares, S/masks.py:93-96)
     *   h_alpha [n][h_period], h_comp [n][h_period]  (gen_additive_mask, S/masks.py:39-54)
     *   h_tcoef [k-1][h_period] the elite's fresh truncation coefficients (its PURPOSE_PARTY
     *           stream, S/layers.py:308, drawn after its reshare sub-share draws)
     *   h_beta  [n][h_period]  beta shares per nonlinear input element (S/masks.py:67-90)
     *   h_binv  [n][h_period_out] beta^-1 shares per nonlinear output element.
     * For nonlin_only launches h_period is the nonlinear input size per image. */
    int host_masks;
    const uint64_t *h_zero, *h_alpha, *h_comp, *h_tcoef, *h_beta, *h_binv;
    uint64_t h_period, h_period_out;
    uint64_t h_period_in;   /* beta shares per image (0: h_period); the gathered size with gather */
    /* 1: an overlapping-window gather (ssn_window_gather, builder op "gather") sits between the
     * chain output (nb, c, gather_h, gather_w) and the nonlinearity, whose (c, h, w) input is
     * the gathered (c, OH*kh, OW*kw) tensor: window (y0, x0) tap (wy, wx) reads source
     * (y0*stride - pad + wy, x0*stride - pad + wx), zero outside.  Needs the split form. */
    int gather, gather_h, gather_w, gather_stride, gather_pad;
} ssn_chain_desc;

int ssn_layer_chain(const ssn_chain_desc *desc, void *stream);
/* table[b] = b^-1 mod p for b in [1, n), table[0] = 0 (batch inversion, p = 2^45 - 55):
 * gen_multiplicative_mask's beta^-1 (S/masks.py:67-90) for beta <= 2^28 by lookup. */
int ssn_inv_table(uint64_t *table, uint64_t n, uint64_t p, void *stream);
/* 1 if ssn_layer_chain supports (k, n, ids, p): a pseudo-Mersenne prime within 2^-24 of a
 * power of two (masked uniform draws) and small-rational protocol constants; else 0. */
int ssn_chain_supported(int k, int n, const uint64_t *ids, uint64_t p);

/* sss_linear's local product fused with reshare step 1 (S/layers.py:245-255 then
 * S/protocol.py:154-164, RESHARE_OUT): the tcgen05 share GEMM of ssn_gemm_tc (p = 2^45 - 55,
 * K-major limb planes, Kpad within one exact pass) whose epilogue, instead of the product y of
 * party `pt`, writes its nf sub-shares  y + sum_{e<km1} c_e * front_ids[f]^(e+1)  to
 *   sub[pt * party_stride + f * front_stride + (img*O + o)*ohw + pix]
 * -- the per-destination send buffers of the first reshare hop.  c_e are drawn exactly as
 * ssn_gen draws them for (seed, stream + pt) (bit-identical to GEMM + ssn_gen). */
typedef struct {
    uint64_t *sub;
    uint64_t party_stride, front_stride;
    uint64_t seed, stream;
    int km1, nf;
    const uint64_t *front_ids;
} ssn_subshare_desc;

int ssn_gemm_tc_subshares(const uint8_t *a_planes, const uint8_t *b_planes, int nparty, int M, int O, uint64_t Kpad,
                          uint64_t ohw, const ssn_subshare_desc *desc, uint64_t p, void *stream);

/* Measurement only (no reference counterpart): the dense int8 tensor-pipe rate.  `ctas` CTAs
 * (one per SM) each issue `iters` back-to-back tcgen05.mma.kind::i8 of 128 x 256 x 32 from
 * resident shared-memory tiles; *ms = device time of that launch, *int8_ops = 2*M*N*K*iters*ctas.
 * The share GEMM's roofline (bench.py) divides by this measured peak.  Synchronises `stream`. */
int ssn_mma_peak(int iters, int ctas, float *ms, double *int8_ops, void *stream);
/* Measurement only: the share GEMM's MMA issue pattern from resident shared memory (mode 0: one
 * 128 x n x 32 MMA back to back; mode 1: 6 A limb tiles x stacked B, D at column 32 i, as in
 * k_gemm_p45w).  Same outputs as ssn_mma_peak. */
int ssn_mma_probe(int mode, int n, int iters, int ctas, float *ms, double *int8_ops, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SSN_H */
