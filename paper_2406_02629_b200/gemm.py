"""Field GEMM / conv dispatch: the local share product of sss_linear (S/layers.py:245-255).

All paths are exact mod p.
* tensor-core path (csrc/ssn_gemm_tc.cu): u8 limb planes, tcgen05.mma kind::i8 with the
  2L-1 limb-diagonal accumulators in TMEM, TMA-fed; used whenever the shape fills a
  128-row tile and the prime has 6..8 limbs (the default p = 2^45 - 55 has L = 6).
* CUDA-core path (csrc/ssn_gemm_simt.cu): 64-bit multiply, 128-bit accumulate; small or
  odd shapes and tiny test primes.
"""

import ctypes

import torch

from . import _lib

TC_MIN_ROWS = 128


def limbs(p):
    return (p.bit_length() + 7) // 8


def kpad(K):
    return (K + 15) // 16 * 16


def tc_supported(p, K):
    L = limbs(p)
    return 6 <= L <= 8 and L * kpad(K) * 65025 < (1 << 32)


def weight_planes(w, p, nparty=1):
    """(nparty, O, K) u64 field weights -> (nparty, L, O, Kpad) u8 limb planes."""
    w2 = w.reshape(nparty, w.shape[-2], w.shape[-1]).contiguous()
    O, K = w2.shape[-2:]
    L, Kp = limbs(p), kpad(K)
    planes = torch.empty((nparty, L, O, Kp), dtype=torch.uint8, device=w.device)
    _lib.call("ssn_limb_split", _lib.ptr(w2), O, K, Kp, L, _lib.ptr(planes), O * K, nparty, _lib.stream_ptr())
    return planes


def conv_planes_supported(p):
    """Implicit-GEMM convs from channel-major planes (ssn_gemm_tc_conv): default prime only."""
    return p == (1 << 45) - 55


def gemm_kernel_name(p, L, rows):
    """The kernel ssn_gemm_tc dispatches to (csrc/ssn_gemm_tc.cu)."""
    return "k_gemm_p45w<0>" if (L == 6 and p == (1 << 45) - 55) else f"k_gemm_tc<{L}>"


def use_tc(p, rows, K, O):
    # the persistent p45 kernel zero-fills (TMA out-of-range) a partial 128-row tile, so small
    # row counts (e.g. the classifier's batch rows) still run on the tensor cores
    if p == (1 << 45) - 55:
        # p45 kernel: TMA zero-fills partial 128-row tiles, 32-channel tiles and the K tail, so
        # any shape runs exactly -- e.g. LeNet's 1-channel 5x5 conv (K = 25, O = 6)
        return rows >= 1 and O >= 1 and K >= 1 and tc_supported(p, K)
    return rows >= TC_MIN_ROWS and O >= 16 and K >= 32 and tc_supported(p, K)


def _ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


def direct_conv(p, O, K):
    """Few-output-channel convs (LeNet's 1->6 and 6->16 5x5) run faster as the direct CUDA-core
    kernel inside ssn_conv_simt (all O channels per output pixel, no im2col) than as im2col +
    tensor-core GEMM with 32-wide channel tiles mostly empty."""
    # measured: LeNet-28 conv1 (K = 25, O = 6) and the reference model's convs win; conv2
    # (K = 150, O = 16: 2,400 64-bit MACs per pixel) is faster on the tensor cores
    return p == (1 << 45) - 55 and O <= 16 and K * O <= 256


class SubShares:
    """Reshare step 1 fused into the share GEMM's epilogue (ssn_gemm_tc_subshares): instead of
    the product, write each party's k RESHARE_OUT sub-shares (S/protocol.py:154-164) into
    out[party][f][element] -- bit-identical to the GEMM followed by ssn_gen(seed, stream + party)
    over the front ids."""

    def __init__(self, out, seed, stream, km1, front_ids):
        self.out, self.seed, self.stream, self.km1 = out, seed, stream, km1
        self.front_ids = list(front_ids)

    def call(self, a_planes, b_planes, nparty, rows, O, Kp, ohw, p):
        nf = len(self.front_ids)
        N = self.out.shape[-1]
        ids = _lib.u64_array(self.front_ids)            # alive for the duration of the call
        d = _lib.SubshareDesc(_lib.ptr(self.out).value, nf * N, N, self.seed, self.stream, self.km1, nf,
                              ctypes.cast(ids, ctypes.c_void_p).value)
        _lib.call("ssn_gemm_tc_subshares", _lib.ptr(a_planes), _lib.ptr(b_planes), nparty, rows, O, Kp, ohw,
                  ctypes.byref(d), p, _lib.stream_ptr())


def fused_subshares_supported(p, K):
    return p == (1 << 45) - 55 and kpad(K) <= max_k_chunk(p)


def field_conv(w, x, stride, padding, p, nimg=1, nparty=1, planes=None, force=None, timing=None, sub=None):
    """w: (nparty, O, C, kh, kw), x: (nparty, nimg, C, H, W) -> (nparty, nimg, O, OH, OW)
    (leading unit dims squeezed when nparty == nimg == 1).  timing: optional dict that
    receives CUDA events around the operand-prep and GEMM launches.  sub: a SubShares -- the
    tensor-core GEMM then emits the RESHARE_OUT sub-shares instead (returns None)."""
    O, C, kh, kw = w.shape[-4:]
    H, W = x.shape[-2:]
    OH = (H + 2 * padding - kh) // stride + 1
    OW = (W + 2 * padding - kw) // stride + 1
    K = C * kh * kw
    x = x.contiguous()
    out = torch.empty((nparty, nimg, O, OH, OW) if (nparty > 1 or nimg > 1) else (O, OH, OW),
                      dtype=torch.int64, device=x.device)
    rows = nimg * OH * OW
    tc = use_tc(p, rows, K, O) and not direct_conv(p, O, K) if force is None else force == "tc"
    if tc:
        L, Kp = limbs(p), kpad(K)
        if planes is None:
            planes = weight_planes(w.reshape(nparty, O, K), p, nparty)
        a = torch.empty((nparty, L, rows, Kp), dtype=torch.uint8, device=x.device)
        e0 = _ev() if timing is not None else None
        _lib.call("ssn_im2col_limbs", _lib.ptr(x), nparty, nimg, C, H, W, kh, kw, stride, padding, L, _lib.ptr(a),
                  Kp, nimg * C * H * W, _lib.stream_ptr())
        e1 = _ev() if timing is not None else None
        if sub is not None:
            sub.call(a, planes, nparty, rows, O, Kp, OH * OW, p)
        else:
            _lib.call("ssn_gemm_tc", _lib.ptr(a), _lib.ptr(planes), nparty, L, rows, O, Kp, OH * OW, _lib.ptr(out),
                      nimg * O * OH * OW, p, _lib.stream_ptr())
        if timing is not None:
            timing["prep"] = (e0, e1, "k_im2col_limbs")
            timing["gemm"] = (e1, _ev(), gemm_kernel_name(p, L, rows))
        return None if sub is not None else out
    if sub is not None:
        raise ValueError("fused sub-shares need the tensor-core path")
    w = w.contiguous()
    e0 = _ev() if timing is not None else None
    _lib.call("ssn_conv_simt", _lib.ptr(w), O * C * kh * kw, _lib.ptr(x), nimg * C * H * W, _lib.ptr(out),
              nimg * O * OH * OW, nparty, nimg, O, C, H, W, kh, kw, stride, padding, p, _lib.stream_ptr())
    if timing is not None:
        timing["gemm"] = (e0, _ev(), "k_conv_simt")
    return out


def field_dense(w, x, p, nimg=1, nparty=1, planes=None, force=None, timing=None, sub=None):
    """w: (nparty, O, K), x: (nparty, nimg, K) -> (nparty, nimg, O) (squeezed for 1 x 1).
    sub: as field_conv."""
    O, K = w.shape[-2:]
    x = x.contiguous()
    out = torch.empty((nparty, nimg, O) if (nparty > 1 or nimg > 1) else (O,), dtype=torch.int64,
                      device=x.device)
    tc = use_tc(p, nimg, K, O) if force is None else force == "tc"
    if sub is not None and not (tc and fused_subshares_supported(p, K)):
        raise ValueError("fused sub-shares need the single-pass tensor-core path")
    if tc and kpad(K) > max_k_chunk(p):
        # split-K: exact partial products over K chunks (each within the int32 limb budget),
        # added mod p
        chunk = max_k_chunk(p)
        for k0 in range(0, K, chunk):
            k1 = min(K, k0 + chunk)
            part = field_dense(w[..., k0:k1].contiguous(), x[..., k0:k1].contiguous(), p, nimg=nimg, nparty=nparty,
                               force="tc")
            if k0 == 0:
                out.copy_(part)
            else:
                _lib.call("ssn_ewise", 0, _lib.ptr(out), _lib.ptr(part), _lib.ptr(out), out.numel(), 1, out.numel(),
                          1 << 62, 0, p, _lib.stream_ptr())
        return out
    if tc:
        L, Kp = limbs(p), kpad(K)
        if planes is None:
            planes = weight_planes(w.reshape(nparty, O, K), p, nparty)
        a = torch.empty((nparty, L, nimg, Kp), dtype=torch.uint8, device=x.device)
        e0 = _ev() if timing is not None else None
        _lib.call("ssn_limb_split", _lib.ptr(x), nimg, K, Kp, L, _lib.ptr(a), nimg * K, nparty, _lib.stream_ptr())
        e1 = _ev() if timing is not None else None
        if sub is not None:
            sub.call(a, planes, nparty, nimg, O, Kp, 1, p)
        else:
            _lib.call("ssn_gemm_tc", _lib.ptr(a), _lib.ptr(planes), nparty, L, nimg, O, Kp, 1, _lib.ptr(out),
                      nimg * O, p, _lib.stream_ptr())
        if timing is not None:
            timing["prep"] = (e0, e1, "k_limb_split")
            timing["gemm"] = (e1, _ev(), gemm_kernel_name(p, L, nimg))
        return None if sub is not None else out
    w = w.contiguous()
    e0 = _ev() if timing is not None else None
    _lib.call("ssn_dense_simt", _lib.ptr(w), O * K, _lib.ptr(x), nimg * K, _lib.ptr(out), nimg * O, nparty,
              nimg, O, K, p, _lib.stream_ptr())
    if timing is not None:
        timing["gemm"] = (e0, _ev(), "k_dense_simt")
    return out


# Largest K per tensor-core pass: L * Kpad * 255^2 < 2^32 keeps every limb-diagonal int32
# accumulator exact (L = 6: Kpad <= 11008).  Larger K is split and the partial products are
# added mod p.
def conv_row_pitch(W):
    """Row pitch of the mode-2 (3x3) channel-major planes: W rounded up to 16 bytes (TMA needs
    16-byte-aligned row shifts; the shifted copies' never-written edge bytes are the zero
    padding, so no extra pad column is needed)."""
    return (W + 15) // 16 * 16


def max_k_chunk(p):
    L = limbs(p)
    return ((1 << 32) - 1) // (L * 65025) // 64 * 64


def field_matmul(a_planes, b_planes, M, N, K, p, out=None, timing=None):
    """C[N-major] = A (M x K) . B (N x K)^T mod p from pre-split u8 limb planes
    a_planes [L][M][Kp], b_planes [L][N][Kp] (Kp = kpad(K)); C is (N, M) row-major = (M x N)^T,
    i.e. out[n*M + m] -- the conv output layout with ohw = M.  Split-K above max_k_chunk."""
    L, Kp = limbs(p), kpad(K)
    out = torch.empty((N, M), dtype=torch.int64, device=a_planes.device) if out is None else out
    chunk = max_k_chunk(p)
    if Kp <= chunk:
        e0 = _ev() if timing is not None else None
        _lib.call("ssn_gemm_tc", _lib.ptr(a_planes), _lib.ptr(b_planes), 1, L, M, N, Kp, M, _lib.ptr(out), M * N, p,
                  _lib.stream_ptr())
        if timing is not None:
            timing.append((e0, _ev()))
        return out
    part = torch.empty_like(out)
    first = True
    for k0 in range(0, Kp, chunk):
        kc = min(chunk, Kp - k0)
        a = a_planes[:, :, k0:k0 + kc].contiguous()
        b = b_planes[:, :, k0:k0 + kc].contiguous()
        dst = out if first else part
        e0 = _ev() if timing is not None else None
        _lib.call("ssn_gemm_tc", _lib.ptr(a), _lib.ptr(b), 1, L, M, N, kc, M, _lib.ptr(dst), M * N, p,
                  _lib.stream_ptr())
        if not first:
            _lib.call("ssn_ewise", 0, _lib.ptr(out), _lib.ptr(part), _lib.ptr(out), M * N, 1, M * N, 1 << 62, 0, p,
                      _lib.stream_ptr())
        if timing is not None:
            timing.append((e0, _ev()))
        first = False
    return out
