"""Field GEMM / conv dispatch: the local share product of sss_linear (S/layers.py:245-255).

All paths are exact mod p.  Large conv/dense tiles go to the tcgen05 int8 limb GEMM
(csrc/ssn_gemm_tc.cu) once it is available for the shape; everything else to the CUDA-core
kernel (csrc/ssn_gemm_simt.cu).
"""

import torch

from . import _lib


def field_conv(w, x, stride, padding, p, nimg=1, nparty=1):
    """w: (O, C, kh, kw) [per party], x: (C, H, W) [per party/image] -> (O, OH, OW)."""
    O, C, kh, kw = w.shape[-4:]
    H, W = x.shape[-2:]
    OH = (H + 2 * padding - kh) // stride + 1
    OW = (W + 2 * padding - kw) // stride + 1
    w = w.contiguous()
    x = x.contiguous()
    out = torch.empty((nparty, nimg, O, OH, OW) if (nparty > 1 or nimg > 1) else (O, OH, OW),
                      dtype=torch.int64, device=x.device)
    _lib.call("ssn_conv_simt", _lib.ptr(w), O * C * kh * kw, _lib.ptr(x), nimg * C * H * W, _lib.ptr(out),
              nimg * O * OH * OW, nparty, nimg, O, C, H, W, kh, kw, stride, padding, p, _lib.stream_ptr())
    return out


def field_dense(w, x, p, nimg=1, nparty=1):
    """w: (O, K), x: (K,) -> (O,)."""
    O, K = w.shape[-2:]
    w = w.contiguous()
    x = x.contiguous()
    out = torch.empty((nparty, nimg, O) if (nparty > 1 or nimg > 1) else (O,), dtype=torch.int64,
                      device=x.device)
    _lib.call("ssn_dense_simt", _lib.ptr(w), O * K, _lib.ptr(x), nimg * K, _lib.ptr(out), nimg * O, nparty,
              nimg, O, K, p, _lib.stream_ptr())
    return out
