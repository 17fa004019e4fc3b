"""Offline mask material for masked truncation and nonlinear steps -- mirror of S/masks.py.

numpy Generator (parity mode): e / beta are drawn on the host with the reference's exact
calls and order (S/masks.py:49,76,83), then shared by ssn_gen; beta^-1 is computed on the
device (unique, so bit-identical to the reference's extended Euclid).
DeviceRng (speed mode): the whole mask -- draw, scale, inverse and (k,n) sharing -- is one
fused kernel (ssn_mask_trunc / ssn_mask_beta) writing every party's share.
"""

import numpy as np
import torch

from . import _lib
from .field import as_device, device
from .rng import DeviceRng
from .sss import ShareTensor

E_BUDGET = 1 << 32
BETA_BITS = 28


def additive_mask_bound(field, step: int, value_bound: int) -> int:
    """S/masks.py:24-36."""
    if step < 1 or value_bound < 0:
        raise ValueError("bad mask parameters")
    emax = min(E_BUDGET // step, (field.p - 1 - 2 * value_bound) // step + 1)
    if emax < 1:
        raise ValueError(f"no mask fits: step {step}, value bound {value_bound}, p {field.p}")
    return emax


def multiplicative_mask_bound(field, value_bound: int) -> int:
    """S/masks.py:57-64."""
    if value_bound < 1:
        raise ValueError("value bound must be positive")
    bmax = min(1 << BETA_BITS, field.half // value_bound)
    if bmax < 1:
        raise ValueError(f"no positive factor fits: value bound {value_bound}, p {field.p}")
    return bmax


def _wrap(out, scheme):
    return [ShareTensor(pid, scheme.k - 1, out[t], scheme) for t, pid in enumerate(scheme.party_ids)]


def gen_additive_mask(shape, r: int, divisor: int, scheme, rng, value_bound: int):
    """alpha = e*r*divisor and comp = -e shared over the scheme (S/masks.py:39-54).
    Returns (alpha_shares, comp_shares, e) -- e is None in device mode."""
    f = scheme.field
    step = r * divisor
    emax = additive_mask_bound(f, step, value_bound)
    shape = tuple(shape)
    if isinstance(rng, DeviceRng):
        n = int(np.prod(shape)) if shape else 1
        alpha = torch.empty((scheme.n,) + shape, dtype=torch.int64, device=device())
        comp = torch.empty_like(alpha)
        _lib.call("ssn_mask_trunc", n, step, emax, rng.seed, rng.next_stream(3), scheme.k - 1,
                  _lib.u64_array(scheme.party_ids), scheme.n, _lib.ptr(alpha), _lib.ptr(comp), n, f.p,
                  _lib.stream_ptr())
        return _wrap(alpha, scheme), _wrap(comp, scheme), None
    e = rng.integers(1, emax + 1, size=shape, dtype=np.int64)
    alpha = np.mod(e.astype(object) * step, f.p).astype(np.int64) if e.ndim else (int(e) * step) % f.p
    comp = np.mod(-e, f.p)
    alpha_shares = scheme.gen(as_device(np.asarray(alpha, dtype=np.int64)), rng)
    comp_shares = scheme.gen(as_device(np.asarray(comp, dtype=np.int64)), rng)
    return alpha_shares, comp_shares, e


def gen_multiplicative_mask(shape, scheme, rng, pool=None, value_bound: int = (1 << 15) - 1):
    """beta >= 1 (constant per pooling window) and its inverse (S/masks.py:67-90).
    Returns (beta_shares, inv_shares, beta_plain) -- beta_plain is None in device mode."""
    f = scheme.field
    bmax = multiplicative_mask_bound(f, value_bound)
    shape = tuple(shape)
    if pool is not None:
        kh, kw = pool
        c, h, w = shape
        if h % kh or w % kw:
            raise ValueError(f"pool {kh}x{kw} does not tile {shape}")
        out_shape = (c, h // kh, w // kw)
    else:
        kh = kw = 1
        out_shape = shape
    if isinstance(rng, DeviceRng):
        if pool is not None:
            nb, c, h, w = 1, shape[0], shape[1], shape[2]
        else:
            nb, c, h, w = 1, int(np.prod(shape)) if shape else 1, 1, 1
        beta = torch.empty((scheme.n,) + shape, dtype=torch.int64, device=device())
        binv = torch.empty((scheme.n,) + out_shape, dtype=torch.int64, device=device())
        _lib.call("ssn_mask_beta", nb, c, h, w, kh, kw, bmax, rng.seed, rng.next_stream(3), scheme.k - 1,
                  _lib.u64_array(scheme.party_ids), scheme.n, _lib.ptr(beta), beta[0].numel(),
                  _lib.ptr(binv), binv[0].numel(), f.p, _lib.stream_ptr())
        return _wrap(beta, scheme), _wrap(binv, scheme), None
    if pool is None:
        beta = rng.integers(1, bmax + 1, size=shape, dtype=np.int64)
        out = beta
    else:
        out = rng.integers(1, bmax + 1, size=out_shape, dtype=np.int64)
        beta = np.repeat(np.repeat(out, kh, axis=1), kw, axis=2)
    beta_inv = f.inv(as_device(out))
    beta_shares = scheme.gen(as_device(beta), rng)
    inv_shares = scheme.gen(beta_inv, rng)
    return beta_shares, inv_shares, beta


def gen_zero_shares(shape, scheme, rng):
    """Fresh sharing of the all-zero tensor (S/masks.py:93-96)."""
    return scheme.gen(torch.zeros(tuple(shape), dtype=torch.int64, device=device()), rng)
