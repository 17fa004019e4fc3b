"""Batched lockstep engine: every party and a batch of images per kernel launch.

This is the throughput path (bench.py).  It runs the same protocol as engine.py -- the same
messages are produced and consumed in HBM, one kernel boundary per protocol hop -- but with
all n co-resident parties in one launch and a batch of B images folded into the element
dimension.  Tensors are party-major: value[t] for rank t+1, each (B, *shape) contiguous.

Per op (reference in parentheses, paths relative to /root/reference/pkg/src/ssnet):
  linear      GEMM for the 2k-1 participants (S/layers.py:245-255)      field GEMM kernel
              reshare step 1: sub-shares to the front  (S/protocol.py:154-163)   ssn_gen, nbatch = 2k-1
              step 2: R^T at the k front ranks          (S/protocol.py:165-185)   ssn_reduce_apply, nbatch = k
              step 3: rec + zero + bias [+ alpha of the next truncation]           ssn_reshare_finish
  truncation  elite rec / window-decode / floor / round / re-share [+RS check]     ssn_trunc_elite
              (S/layers.py:277-323); every rank + comp                              ssn_ewise
  nonlinear   x * beta at the participants (S/layers.py:338-342)                   ssn_ewise
              elite rec / decode / ReLU / pool / encode (S/layers.py:345-364)      ssn_nonlin_elite
              plain * beta^-1 at the receivers (S/layers.py:379-380)                ssn_ewise (broadcast)
  add         local share add (residual, S/sss.py:238)                             ssn_ewise
  gather      local overlapping-window gather (builder op; 3x3/s2 stem pool)       ssn_window_gather
  output      rec at the elite + decode (S/protocol.py:289-305)                    ssn_rec, ssn_decode_signed
Masks come from a device-side trusted source, generated per op just before use
(S/protocol.py:354-388, S/masks.py): ssn_gen (zero), ssn_mask_trunc, ssn_mask_beta.
Randomness: rng_mode="device" (speed mode, the bench) draws everything from device Philox;
decoded outputs are RNG-independent, so they equal the reference / plaintext exactly.
rng_mode="host" is the reference-stream parity mode: weight shares (lane 1), input shares
(lane 3, input_index = image position), the trusted source's bundle (lane 4) and the elite's
truncation coefficients (lane 5, rank 1) are drawn with the reference's numpy calls and fed to
the SAME kernels (ssn_chain.cu HF instantiations), so every party's share of every op output
equals the reference's run of that image bit for bit (tests/test_gpu_parity_batched.py).
"""

import ctypes
import os
import time

import numpy as np
import torch

from . import _lib
from . import gemm as gemm_mod
from .gemm import field_conv, field_dense
from .layers import comm_estimate, consumers, plan_schedule, window_gather
from .masks import additive_mask_bound, multiplicative_mask_bound
from .protocol import VerificationError, extrapolation_coeffs
from .rng import DeviceRng


def _count(shape):
    n = 1
    for d in shape:
        n *= int(d)
    return n


class BatchedEngine:
    def __init__(self, model, scheme, batch, seed=7, rng_mode="device", verify=False, ordering="ltn",
                 profile=False, fuse=True, share_weights_with=None, implicit=True):
        if rng_mode not in ("device", "host"):
            raise ValueError(f"unknown rng mode {rng_mode!r}")
        self.host = rng_mode == "host"
        if self.host and share_weights_with is not None:
            raise ValueError("reference-stream mode deals its own weight shares")
        self.model = model
        self.scheme = scheme
        self.batch = int(batch)
        self.seed = seed
        self.verify = verify
        self.profile = profile
        self.p = scheme.field.p
        self.ops, self.digest = plan_schedule(model, scheme, ordering, verify=verify)
        self.cons = consumers(self.ops)
        self.dev = torch.device("cuda", torch.cuda.current_device())
        k, n = scheme.k, scheme.n
        self.k, self.n, self.m = k, n, 2 * k - 1
        self.w_front = scheme.lagrange_weights(scheme.front_ids)
        self.w_part = scheme.lagrange_weights(scheme.party_ids[:self.m])
        R = scheme.reducing_matrix()
        self.rt = {nout: [R[i][t] for t in range(nout) for i in range(self.m)] for nout in (k, n)}
        self.ext = [v for row in extrapolation_coeffs(scheme, scheme.front_ids, scheme.party_ids[k:]) for v in row]
        self.ids_all = _lib.u64_array(scheme.party_ids)
        self.ids_front = _lib.u64_array(scheme.front_ids)
        self.runs = 0
        self.fail = torch.zeros(1, dtype=torch.int64, device=self.dev)
        if share_weights_with is not None:      # same dealt weight shares / limb planes (read-only)
            self.W, self._planes = share_weights_with.W, share_weights_with._planes
        else:
            self._planes = {}
            self._deal_weights_host() if self.host else self._deal_weights()
        self.hm = self._host_source() if self.host else None
        self.kernel_launches = 0
        self.fault = None
        self.fuse = fuse
        self.chains = self._plan_chains() if fuse else {}
        self._chain_cache = {}
        self._chain_member = {i: start for start, ch in self.chains.items() for i in ch[1:]}
        self._rt_all = _lib.u64_array([R[i][t] for t in range(n) for i in range(self.m)])
        self._plan_implicit_convs(implicit)
        # chain kernels emit the next conv's limb planes (else ssn_planes_cn does, per conv)
        self.chain_planes = os.environ.get("SSN_CHAIN_PLANES", "1") != "0"
        # nonlinear chains as two kernels (reshare/truncation, then nonlinearity)
        self.split_chain = os.environ.get("SSN_SPLIT_CHAIN", "1") != "0"
        self._ext_host = _lib.u64_array(self.ext) if self.ext else None

    # ------------------------------------------------------------------ setup
    def _deal_weights(self):
        """Weight shares dealt once from lane 1 and reused across runs (S/engine.py:40-49)."""
        rng = DeviceRng(self.seed, 1)
        values = self.model.weight_values() if hasattr(self.model, "weight_values") else \
            {name: qt.values for name, qt in self.model.weights.items()}
        self.W = {}
        for name in sorted(values):
            v = torch.as_tensor(np.asarray(values[name], dtype=np.int64), device=self.dev).contiguous()
            enc = self._encode(v)
            out = torch.empty((self.n,) + tuple(v.shape), dtype=torch.int64, device=self.dev)
            nel = v.numel()
            _lib.call("ssn_gen", _lib.ptr(enc), 0, None, 0, rng.seed, rng.next_stream(), self.k - 1, self.ids_all,
                      self.n, _lib.ptr(out), 0, nel, nel, 1, self.p, _lib.stream_ptr())
            self.W[name] = out

    def _deal_weights_host(self):
        """Reference-stream weight shares: lane 1, sorted names (S/engine.py:40-49)."""
        from .engine import deal_weight_shares
        values = self.model.weight_values() if hasattr(self.model, "weight_values") else \
            {name: qt.values for name, qt in self.model.weights.items()}
        per_rank = deal_weight_shares(values, self.scheme, self.seed, "host")
        self.W = {name: torch.stack([per_rank[r][name].values for r in range(1, self.n + 1)]).contiguous()
                  for name in sorted(values)}

    def _host_source(self):
        """Reference-stream trusted-source material, drawn once (the reference deals the same
        bundle and the same party streams for every input_index, S/engine.py:64-74,166-171):
          (idx, name) -> [n][numel]  shares of zero / alpha / comp / beta / beta_inv
                         (trusted_source_prepare on lane 4, S/protocol.py:354-388);
          (idx, "tcoef") -> [k-1][numel] the elite's fresh truncation coefficients: rank 1's
                         PURPOSE_PARTY stream replayed -- each linear op first draws its reshare
                         sub-share coefficients (S/protocol.py:158, values never matter), each
                         truncation then its k-1 coefficient tensors (S/layers.py:308)."""
        from .engine import PURPOSE_MASKS, PURPOSE_PARTY, seeded_rng
        from .protocol import trusted_source_prepare
        n, k, p = self.n, self.k, self.p
        bundles, _ = trusted_source_prepare(self.ops, self.scheme, seeded_rng(self.seed, PURPOSE_MASKS))
        hm = {key: torch.stack([bundles[r].entries[key].values.reshape(-1) for r in range(1, n + 1)]).contiguous()
              for key in bundles[1].entries}
        rng = seeded_rng(self.seed, PURPOSE_PARTY, 1)
        for idx, op in enumerate(self.ops):
            if k == 1:
                break
            if op.kind == "linear":
                for _ in range(k - 1):
                    rng.integers(0, p, size=_count(op.out_shape), dtype=np.int64)
            elif op.kind == "truncation":
                draws = np.stack([rng.integers(0, p, size=_count(op.in_shape), dtype=np.int64) for _ in range(k - 1)])
                hm[(idx, "tcoef")] = torch.as_tensor(draws, device=self.dev).contiguous()
        return hm

    def _hb(self, idx, name):
        """Host-fed material of op idx broadcast over the batch: [rows][B * numel] (the
        unfused kernels index the batch directly)."""
        t = self.hm[(idx, name)]
        return t.view(t.shape[0], 1, -1).expand(t.shape[0], self.batch, t.shape[1]).reshape(t.shape[0], -1) \
            .contiguous()

    def _encode(self, v):
        out = torch.empty_like(v)
        ovf = torch.zeros(1, dtype=torch.int64, device=self.dev)
        _lib.call("ssn_encode_signed", _lib.ptr(v), _lib.ptr(out), v.numel(), _lib.ptr(ovf), self.p,
                  _lib.stream_ptr())
        return out

    # ------------------------------------------------------------------ implicit-GEMM convs
    IMPLICIT_MIN_W = 14          # 3x3 row-padded tiles waste (Wp - W)/Wp; below 14x14 use im2col (8x8 measured slower)

    def _plan_implicit_convs(self, enabled):
        """Convs whose A operand is read straight from channel-major limb planes (no im2col):
        1x1/stride 1 (mode 1) and 3x3/stride 1/pad 1 (mode 2).  The planes are emitted by the
        producing chain kernel, or by ssn_planes_cn from the u64 shares otherwise."""
        self._conv_mode, self._plane_src, self._plane_buf, self._planes_ready = {}, {}, {}, set()
        if not enabled or not gemm_mod.conv_planes_supported(self.p):
            return
        B = self.batch
        wants = {}
        for idx, op in enumerate(self.ops):
            if op.kind != "linear":
                continue
            w = self.W[op.weight + ".w"]
            if w.dim() != 5 or len(op.in_shape) != 3:
                continue
            C, H, Wd = op.in_shape
            kh = int(w.shape[-1])
            if C % 64 or B * H * Wd >= (1 << 31) or not gemm_mod.use_tc(self.p, B * H * Wd, C * kh * kh,
                                                                     op.out_shape[0]):
                continue
            if kh == 1 and op.stride == 1 and op.padding == 0 and (B * H * Wd) % 16 == 0:
                mode = (1, Wd, 1)
            elif kh == 3 and op.stride == 1 and op.padding == 1 and Wd >= self.IMPLICIT_MIN_W:
                mode = (2, gemm_mod.conv_row_pitch(Wd), 3)
            else:
                continue
            src = idx - 1 if op.src is None else op.src
            wants.setdefault(src, []).append((idx, mode, (C, H, Wd)))
        for src, lst in wants.items():
            if len({m for _, m, _ in lst}) != 1:      # consumers disagree on the layout: im2col
                continue
            for idx, mode, _ in lst:
                self._conv_mode[idx] = (src,) + mode
            self._plane_src[src] = lst[0][1] + lst[0][2]

    def _plane_buffer(self, src):
        """Persistent zeroed planes [copies][m][L][C][B][H][Wp] for producer `src` (pad bytes
        are never written, so they stay zero across runs)."""
        buf = self._plane_buf.get(src)
        if buf is None:
            mode, Wp, copies, C, H, Wd = self._plane_src[src]
            L = gemm_mod.limbs(self.p)
            buf = self._plane_buf[src] = torch.zeros((copies, self.m, L, C, self.batch, H, Wp), dtype=torch.uint8,
                                                     device=self.dev)
        return buf

    def _conv_weight_planes(self, op, mode):
        key = (op.weight, "cn", mode)
        pl = self._planes.get(key)
        if pl is None:
            w = self.W[op.weight + ".w"][:self.m]
            O, C, kh, kw = w.shape[1:]
            wt = w.permute(0, 1, 3, 4, 2).contiguous().reshape(self.m, O, kh * kw * C)   # k = (tap, c)
            pl = self._planes[key] = gemm_mod.weight_planes(wt, self.p, self.m)
        return pl

    def _gemm_implicit(self, idx, op, X):
        src, mode, Wp, copies = self._conv_mode[idx]
        B, m, p = self.batch, self.m, self.p
        C, H, Wd = op.in_shape
        O = op.out_shape[0]
        buf = self._plane_buffer(src)
        prof = self._prof is not None
        if src not in self._planes_ready:                 # producer was not a plane-emitting chain
            e0 = self._event() if prof else None
            _lib.call("ssn_planes_cn", _lib.ptr(X), m, B, C, H, Wd, Wp, gemm_mod.limbs(p), _lib.ptr(buf),
                      B * C * H * Wd, copies, _lib.stream_ptr())
            if prof:
                self._record("im2col", e0, self._event(), (8 + 6 * copies) * m * B * C * H * Wd, "k_planes_cn")
            self._planes_ready.add(src)
        bpl = self._conv_weight_planes(op, mode)
        out = torch.empty((m, B, O, H, Wd), dtype=torch.int64, device=self.dev)
        e0 = self._event() if prof else None
        _lib.call("ssn_gemm_tc_conv", _lib.ptr(buf), mode, B, C, H, Wd, Wp, _lib.ptr(bpl), m, O, _lib.ptr(out),
                  B * O * H * Wd, p, _lib.stream_ptr())
        if prof:
            K = C * (9 if mode == 2 else 1)
            self._record("gemm", e0, self._event(), m * B * H * Wd * O * K, f"k_gemm_p45w<{mode}>")
        return out

    # ------------------------------------------------------------------ beta^-1 table
    _INV_TABLES = {}                       # device -> table (shared by every engine)
    INV_TABLE_MAX = 1 << 28                # gen_multiplicative_mask caps beta at 2^28 (S/masks.py:57-64)

    def _inv_table(self, bmax):
        """The trusted source's beta^-1 by lookup: table[b] = b^-1 mod p for b <= bmax, built
        once per device by batch inversion (2 GiB for the 2^28 cap).  Opt-in (SSN_INV_TABLE=1):
        measured no faster than the in-kernel per-warp batch inversion, which is the default."""
        if os.environ.get("SSN_INV_TABLE", "0") != "1" or self.p != (1 << 45) - 55 or bmax > self.INV_TABLE_MAX:
            return None
        tab = self._INV_TABLES.get(self.dev)
        if tab is None or tab.numel() <= bmax:
            n = self.INV_TABLE_MAX + 1
            tab = torch.empty(n, dtype=torch.int64, device=self.dev)
            _lib.call("ssn_inv_table", _lib.ptr(tab), n, self.p, _lib.stream_ptr())
            self._INV_TABLES[self.dev] = tab
        return tab

    # ------------------------------------------------------------------ fused chains
    CHAIN_SCHEMES = ((2, 3), (3, 5), (4, 7))

    def _srcs(self, idx):
        op = self.ops[idx]
        s = [idx - 1 if op.src is None else op.src]
        if op.kind == "add":
            s.append(op.src2)
        return s

    def _plan_chains(self):
        """Group linear -> truncation [-> add] [-> gather] [-> nonlinear] runs whose intermediates
        have a single consumer into one fused protocol launch (csrc/ssn_chain.cu)."""
        if (self.k, self.n) not in self.CHAIN_SCHEMES:
            return {}
        if not _lib.load(require_cuda=False).ssn_chain_supported(self.k, self.n, self.ids_all, self.p):
            return {}
        ops, cons = self.ops, self.cons
        chains = {}
        for idx, op in enumerate(ops):
            c = cons.get(idx, [])
            if op.kind != "linear" or len(c) != 1 or ops[c[0]].kind != "truncation":
                continue
            chain = [idx, c[0]]
            cur = c[0]
            nxt = cons.get(cur, [])
            if len(nxt) == 1 and ops[nxt[0]].kind == "add":
                a = nxt[0]
                others = [s for s in self._srcs(a) if s != cur]
                if len(others) == 1 and others[0] < idx:
                    chain.append(a)
                    cur = a
                    nxt = cons.get(cur, [])
            if (len(nxt) == 1 and ops[nxt[0]].kind == "gather" and len(cons.get(nxt[0], [])) == 1
                    and ops[cons[nxt[0]][0]].kind == "nonlinear" and ops[cons[nxt[0]][0]].pool is not None):
                g = nxt[0]
                chain.append(g)
                cur = g
                nxt = cons.get(cur, [])
            if len(nxt) == 1 and ops[nxt[0]].kind == "nonlinear" and self._srcs(nxt[0]) == [cur]:
                chain.append(nxt[0])
            chains[idx] = chain
        return chains

    def _chain_static(self, chain):
        """The launch-invariant part of a chain's descriptor (geometry, mask bounds, bias,
        constants, plane buffer), built once per chain: host time per launch matters."""
        B, n, k, m, p = self.batch, self.n, self.k, self.m, self.p
        lin, tr = self.ops[chain[0]], self.ops[chain[1]]
        add = next((self.ops[i] for i in chain[2:] if self.ops[i].kind == "add"), None)
        nl = next((self.ops[i] for i in chain[2:] if self.ops[i].kind == "nonlinear"), None)
        gat = next((self.ops[i] for i in chain[2:] if self.ops[i].kind == "gather"), None)
        last = self.ops[chain[-1]]
        O = lin.out_shape[0]
        ohw = _count(lin.out_shape[1:]) if len(lin.out_shape) > 1 else 1
        nel = B * _count(lin.out_shape)
        n_out = B * _count(last.out_shape)
        d = _lib.ChainDesc()
        d.acc_pstride = nel
        bias = self.W[lin.weight + ".b"]
        d.bias, d.bias_pstride, d.bias_div, d.bias_mod = bias.data_ptr(), O, ohw, O
        other = None
        if add is not None:
            other = [s for s in self._srcs(chain[2]) if s != chain[1]][0]
            d.other_pstride = nel
        d.out_pstride = n_out
        d.nel = nel
        d.nout = n if lin.passive_out else k
        d.value_bound, d.r, d.d = tr.value_bound, tr.r, tr.divisor
        d.emax = additive_mask_bound(self.scheme.field, tr.r * tr.divisor, tr.value_bound)
        d.verify = int(bool(self.verify))
        d.fail = self.fail.data_ptr()
        if nl is not None:
            if nl.pool_kind is not None:
                (c, h, w), (kh, kw) = nl.in_shape, nl.pool
                kind = 1 if nl.pool_kind == "max" else 2
            elif len(nl.in_shape) == 3:
                (c, h, w), kh, kw, kind = nl.in_shape, 1, 1, 0
            else:
                c, h, w, kh, kw, kind = _count(nl.in_shape), 1, 1, 1, 1, 0
            d.nonlin, d.relu, d.pool_kind = 1, int(bool(nl.relu)), kind
            d.nb, d.c, d.h, d.w, d.kh, d.kw = B, c, h, w, kh, kw
            if gat is not None:
                d.gather, d.gather_h, d.gather_w = 1, gat.in_shape[1], gat.in_shape[2]
                d.gather_stride, d.gather_pad = gat.stride, gat.padding
            d.fan = n if nl.passive_out else k
            d.bmax = multiplicative_mask_bound(self.scheme.field, nl.value_bound)
            tab = self._inv_table(d.bmax)
            if tab is not None:
                d.inv_table, d.inv_table_len = tab.data_ptr(), tab.numel()
        d.k, d.n = k, n
        d.ids, d.rt = ctypes.addressof(self.ids_all), ctypes.addressof(self._rt_all)
        d.ext = ctypes.addressof(self._ext_host) if self._ext_host is not None else None
        d.p = p
        if self.host:
            hm = self.hm
            d.host_masks = 1
            d.h_zero = hm[(chain[0], "zero")].data_ptr()
            d.h_alpha = hm[(chain[1], "alpha")].data_ptr()
            d.h_comp = hm[(chain[1], "comp")].data_ptr()
            d.h_tcoef = hm[(chain[1], "tcoef")].data_ptr() if k > 1 else None
            d.h_period = _count(lin.out_shape)
            if nl is not None:
                nidx = next(i for i in chain[2:] if self.ops[i].kind == "nonlinear")
                d.h_beta = hm[(nidx, "beta")].data_ptr()
                d.h_binv = hm[(nidx, "beta_inv")].data_ptr()
                d.h_period_out = _count(last.out_shape)
                d.h_period_in = _count(nl.in_shape)
        shift = None
        ps = self._plane_src.get(chain[-1])
        if ps is not None and nl is not None and self.chain_planes and tuple(last.out_shape) == tuple(ps[3:]):
            _, Wp, copies, C2, H2, W2 = ps
            buf = self._plane_buffer(chain[-1])
            # the chain writes the unshifted copy (index 1 of 3 for mode 2); ssn_planes_shift
            # derives the +-1 column copies with 16-byte vector moves
            d.planes = buf[1 if copies == 3 else 0].data_ptr()
            d.plane_istride = H2 * Wp
            d.plane_cstride = B * H2 * Wp
            d.plane_lstride = C2 * B * H2 * Wp
            d.plane_pstride = gemm_mod.limbs(p) * C2 * B * H2 * Wp
            d.plane_wp, d.plane_copies, d.plane_nparty = Wp, 1, m
            if copies == 3:
                shift = (buf.data_ptr(), m * gemm_mod.limbs(p) * C2 * B * H2, Wp)
        nbytes = 8 * m * nel + (8 * n * nel if add is not None else 0)
        nbytes += 8 * (d.fan * n_out if nl is not None else n * nel)
        return {"d": d, "lin": lin, "last": last, "other": other, "nl": nl is not None, "nel": nel,
                "shift": shift, "planes": bool(d.planes), "nbytes": nbytes, "gather": gat is not None}

    def _chain(self, chain, vals, src_rng, party_rng):
        """One fused launch: reshare + rerand + bias + truncation [+ add] [+ nonlinear]."""
        B, n, m = self.batch, self.n, self.m
        st = self._chain_cache.get(chain[0])
        if st is None:
            st = self._chain_cache[chain[0]] = self._chain_static(chain)
        d = st["d"]
        acc = self._gemm(chain[0], st["lin"], vals[self._srcs(chain[0])[0]])
        Y = torch.empty((n, B) + tuple(st["last"].out_shape), dtype=torch.int64, device=self.dev)
        d.acc = acc.data_ptr()
        if st["other"] is not None:
            d.other = vals[st["other"]].data_ptr()
        d.out = Y.data_ptr()
        d.party_seed, d.party_stream = party_rng.seed, party_rng.next_stream(m + 1)
        d.src_seed, d.src_stream = src_rng.seed, src_rng.next_stream(7)
        d.fault_rank = self.fault[1] if (self.fault is not None and self.fault[0] == chain[0]) else -1
        scratch = None
        if st["nl"] and (self.split_chain or st["gather"]):      # gathered windows read a scratch
            scratch = torch.empty((n, st["nel"]), dtype=torch.int64, device=self.dev)
            d.scratch = scratch.data_ptr()
        else:
            d.scratch = None
        if st["planes"]:
            self._planes_ready.add(chain[-1])
        e0 = self._event() if self._prof is not None else None
        _lib.call("ssn_layer_chain", ctypes.byref(d), _lib.stream_ptr())
        if st["shift"] is not None:
            _lib.call("ssn_planes_shift", *st["shift"], _lib.stream_ptr())
        if e0 is not None:
            self._record("chain", e0, self._event(), st["nbytes"],
                         "k_chain_nonlin" if st["nl"] else "k_chain_plain", elems=st["nel"])
        self.kernel_launches += 1
        return Y

    # ------------------------------------------------------------------ helpers
    def _ew(self, op, a, b, out, n, b_mod=None):
        """out[:n] = a OP b; b broadcast cyclically with period b_mod (default: full)."""
        bm = n if b_mod is None else b_mod
        _lib.call("ssn_ewise", op, _lib.ptr(a), _lib.ptr(b), _lib.ptr(out), n, 1, bm, 1 << 62, 0, self.p,
                  _lib.stream_ptr())
        self.kernel_launches += 1

    # ------------------------------------------------------------------ instrumentation
    # Per kernel class, CUDA events recorded on the launching stream around every launch of
    # the timed steps, with the launch's algorithmic work (bench roofline):
    #   gemm    field MACs (x L^2 u8 limb products on the tensor pipe)    k_gemm_p45 / k_gemm_tc
    #   chain   algorithmic HBM bytes (8*m in + 8*n out [+ 8*n add])      k_chain_*
    #   im2col  algorithmic HBM bytes (8 B per input share read once + limb-plane bytes written)
    _prof = None

    def enable_profiling(self):
        self._prof = {}
        return self._prof

    def disable_profiling(self):
        self._prof = None

    def _record(self, cls, e0, e1, work, kernel, elems=0):
        if self._prof is not None:
            self._prof.setdefault(cls, []).append((e0, e1, work, kernel, elems))

    @staticmethod
    def _event():
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        return e

    def profile_summary(self, steps):
        torch.cuda.synchronize()
        out = {}
        for cls, rec in (self._prof or {}).items():
            ms = [r[0].elapsed_time(r[1]) for r in rec]
            work = [r[2] for r in rec]
            elems = [r[4] for r in rec]
            nl = len(rec)
            out[cls] = {"launches_per_step": nl / max(steps, 1), "ms_per_step": sum(ms) / max(steps, 1),
                        "ms_per_launch": sum(ms) / nl if nl else 0.0, "work_per_launch": sum(work) / nl if nl else 0.0,
                        "elems_per_launch": sum(elems) / nl if nl else 0.0,
                        "kernel": ",".join(sorted({r[3] for r in rec}))}
        return out

    def limb_products(self):
        L = (self.p.bit_length() + 7) // 8
        return L * L

    def out_shape(self):
        return tuple(self.ops[-1].out_shape)

    def comm_per_image(self):
        """Online elements exchanged per image (reference closed forms, S/layers.py:193-225)."""
        est = comm_estimate(self.ops, self.scheme, verify=self.verify)
        online = sum(r["elements"] for r in est if r["kind"] != "offline")
        offline = next(r["elements"] for r in est if r["kind"] == "offline")
        return online, offline

    # ------------------------------------------------------------------ run
    def run(self, x_int, timings=None):
        """One secure inference of a batch.  x_int: int64 (B, *input_shape), numpy or device.
        Returns the decoded int64 outputs (numpy, shape (B, *out))."""
        out = self.run_device(x_int, timings)
        return out.cpu().numpy()

    def _reveal(self, Y, shape):
        """Test helper: reconstruct an op output from the front ranks' shares (decoded int64)."""
        N = self.batch * _count(shape)
        v = torch.empty(N, dtype=torch.int64, device=self.dev)
        _lib.call("ssn_rec", _lib.ptr(Y), 0, N, _lib.u64_array(self.w_front), self.k, _lib.ptr(v), 0, N, 1,
                  self.p, _lib.stream_ptr())
        out = torch.empty_like(v)
        _lib.call("ssn_decode_signed", _lib.ptr(v), _lib.ptr(out), N, self.p, _lib.stream_ptr())
        return out.reshape((self.batch,) + tuple(shape)).cpu().numpy()

    def run_device(self, x_int, timings=None, capture=None, capture_shares=None, input_indices=None):
        """capture: {idx: decoded op output} (test helper); capture_shares: {idx: [n][B][...]
        every party's share of each materialised op output (fused chains: the chain's last op;
        the output op: its input shares)}; input_indices: the reference input_index of each
        image for the reference-stream input shares (default 0..B-1)."""
        B, n, k, m, p = self.batch, self.n, self.k, self.m, self.p
        run_id = self.runs
        self.runs += 1
        src_rng = DeviceRng(self.seed, 4, run_id)          # trusted source lane
        party_rng = DeviceRng(self.seed, 5, run_id)        # online protocol lane
        if isinstance(x_int, torch.Tensor):
            x = x_int.to(device=self.dev, dtype=torch.int64).contiguous()
        else:
            x = torch.as_tensor(np.asarray(x_int, dtype=np.int64), device=self.dev).contiguous()
        if x.shape[0] != B:
            raise ValueError(f"batch {x.shape[0]} != engine batch {B}")
        ev = [] if timings is not None else None

        def mark(label):
            if ev is not None:
                e = torch.cuda.Event(enable_timing=True)
                e.record()
                ev.append((label, e))

        mark("start")
        # input dealing (S/engine.py:52-54), lane 3
        if self.host:
            from .engine import deal_input_shares
            idxs = list(range(B)) if input_indices is None else [int(i) for i in input_indices]
            xh = x.cpu().numpy()
            X = torch.stack([torch.stack([st.values for st in deal_input_shares(xh[b], self.scheme, self.seed, idxs[b],
                                                                                  "host")])
                             for b in range(B)], dim=1).contiguous()
        else:
            enc = self._encode(x)
            X = torch.empty((n,) + tuple(x.shape), dtype=torch.int64, device=self.dev)
            irng = DeviceRng(self.seed, 3, run_id)
            nel = x.numel()
            _lib.call("ssn_gen", _lib.ptr(enc), 0, None, 0, irng.seed, irng.next_stream(), k - 1, self.ids_all, n,
                      _lib.ptr(X), 0, nel, nel, 1, p, _lib.stream_ptr())
        vals = {-1: X}
        masked_for = {}          # linear idx -> True when its output already carries alpha
        remaining = {i: len(c) for i, c in self.cons.items()}
        result = None
        pending = {}
        self._planes_ready = set()
        for idx, op in enumerate(self.ops):
            src = idx - 1 if op.src is None else op.src
            xin = vals.get(src)
            if idx in self.chains:
                chain = self.chains[idx]
                pending[chain[-1]] = self._chain(chain, vals, src_rng, party_rng)
                y = None
            elif idx in self._chain_member:
                y = pending.pop(idx, None)
            elif op.kind == "linear":
                y = self._linear(idx, op, xin, src_rng, party_rng)
                masked_for[idx] = getattr(self, "_fused_alpha", False)
            elif op.kind == "truncation":
                y = self._truncation(idx, op, xin, masked_for.get(src, False), src_rng, party_rng)
            elif op.kind == "nonlinear":
                y = (self._nonlinear_fused(idx, op, xin, src_rng) if self.chains
                     else self._nonlinear(idx, op, xin, src_rng))
            elif op.kind == "add":
                other = vals[op.src2]
                nn = _count(op.out_shape) * B
                y = torch.empty((n, B) + tuple(op.out_shape), dtype=torch.int64, device=self.dev)
                self._ew(0, xin, other, y, n * nn)
            elif op.kind == "gather":
                kh, kw = op.pool
                y = window_gather(xin, op.in_shape, kh, kw, op.stride, op.padding, nbatch=n * B) \
                    .reshape((n, B) + tuple(op.out_shape))
                self.kernel_launches += 1
            elif op.kind == "output":
                if capture_shares is not None:
                    capture_shares[idx] = xin.clone()
                result = self._output(op, xin)
                y = None
            else:
                raise ValueError(op.kind)
            if y is not None:
                vals[idx] = y
                if capture_shares is not None and not masked_for.get(idx, False):   # not: y + next alpha
                    capture_shares[idx] = y.clone()
            if self.fault is not None and self.fault[0] == idx and y is not None and not self.chains:
                y[self.fault[1]].view(-1)[0] += 1              # test hook: corrupt one share
            if capture is not None and y is not None and op.kind != "linear" and idx not in self.chains:
                capture[idx] = self._reveal(y, op.out_shape)
            mark("chain" if (idx in self.chains or idx in self._chain_member) else op.kind)
            # release inputs no longer needed
            for s in ([src] + ([op.src2] if op.kind == "add" else [])):
                remaining[s] -= 1
                if remaining[s] <= 0 and s in vals:
                    del vals[s]
        if timings is not None:
            torch.cuda.synchronize()
            for (lab0, e0), (lab1, e1) in zip(ev[:-1], ev[1:]):
                timings[lab1] = timings.get(lab1, 0.0) + e0.elapsed_time(e1)
        return result

    # ------------------------------------------------------------------ ops
    def _gemm(self, idx, op, X):
        """Local share products of the m participants (S/layers.py:245-255): acc [m][B][O][ohw]."""
        if idx in self._conv_mode:
            return self._gemm_implicit(idx, op, X)
        B, m, p = self.batch, self.m, self.p
        w = self.W[op.weight + ".w"]
        O = op.out_shape[0]
        conv = w.dim() == 5
        timing = {} if self._prof is not None else None
        K = _count(w.shape[2:])
        ohw = _count(op.out_shape[1:]) if conv else 1
        tc = gemm_mod.use_tc(p, B * ohw, K, O) and not (conv and gemm_mod.direct_conv(p, O, K))
        planes = None
        if tc:
            planes = self._planes.get(op.weight)
            if planes is None:
                planes = self._planes[op.weight] = gemm_mod.weight_planes(w[:m].reshape(m, O, K), p, m)
        if conv:
            C, H, Wd = op.in_shape
            acc = field_conv(w[:m], X[:m].reshape(m, B, C, H, Wd), op.stride, op.padding, p, nimg=B, nparty=m,
                             planes=planes, force="tc" if tc else "simt", timing=timing)
        else:
            acc = field_dense(w[:m], X[:m].reshape(m, B, -1), p, nimg=B, nparty=m, planes=planes,
                              force="tc" if tc else "simt", timing=timing)
        if timing:
            L = gemm_mod.limbs(p)
            macs = m * B * ohw * O * K
            e0, e1, kname = timing["gemm"]
            self._record("gemm" if tc else "gemm_simt", e0, e1, macs, kname)
            if "prep" in timing:
                e0, e1, kname = timing["prep"]
                in_el = m * B * _count(op.in_shape)
                self._record("im2col", e0, e1, 8 * in_el + L * m * B * ohw * gemm_mod.kpad(K), kname)
        return acc

    def _linear(self, idx, op, X, src_rng, party_rng):
        B, n, k, m, p = self.batch, self.n, self.k, self.m, self.p
        b = self.W[op.weight + ".b"]
        O = op.out_shape[0]
        ohw = _count(op.out_shape[1:]) if len(op.out_shape) > 1 else 1
        acc = self._gemm(idx, op, X)
        N = B * O * ohw
        nout = n if op.passive_out else k
        # source: zero shares for every rank (gen_zero_shares)
        if self.host:
            Z = self._hb(idx, "zero")
        else:
            Z = torch.empty((n, N), dtype=torch.int64, device=self.dev)
            _lib.call("ssn_gen", None, 0, None, 0, src_rng.seed, src_rng.next_stream(), k - 1, self.ids_all, n,
                      _lib.ptr(Z), 0, N, N, 1, p, _lib.stream_ptr())
        # fuse the next truncation's alpha into step 3 when the truncation is the sole consumer
        nxt = self.cons[idx]
        alpha = None
        self._fused_alpha = False
        if len(nxt) == 1 and self.ops[nxt[0]].kind == "truncation":
            alpha = self._trunc_masks(nxt[0], self.ops[nxt[0]], src_rng)
            self._fused_alpha = True
        # step 1 (RESHARE_OUT): participant i -> front j
        SUB = torch.empty((m, k, N), dtype=torch.int64, device=self.dev)
        _lib.call("ssn_gen", _lib.ptr(acc), N, None, 0, party_rng.seed, party_rng.next_stream(m), k - 1,
                  self.ids_front, k, _lib.ptr(SUB), k * N, N, N, m, p, _lib.stream_ptr())
        # step 2 (RESHARE_BACK): front j applies R^T to its m sub-shares
        BACK = torch.empty((k, nout, N), dtype=torch.int64, device=self.dev)
        _lib.call("ssn_reduce_apply", _lib.ptr(SUB), N, k * N, m, _lib.u64_array(self.rt[nout]), nout,
                  _lib.ptr(BACK), nout * N, N, N, k, p, _lib.stream_ptr())
        del SUB
        # step 3: out rank t reconstructs from the k fronts, + zero + bias (+ alpha)
        Y = torch.empty((n, B) + tuple(op.out_shape), dtype=torch.int64, device=self.dev)
        _lib.call("ssn_reshare_finish", _lib.ptr(BACK), N, nout * N, _lib.u64_array(self.w_front), k,
                  _lib.ptr(Z), N, _lib.ptr(b), O, ohw, O, _lib.ptr(alpha[0] if alpha is not None else None), N,
                  _lib.ptr(Y), N, N, nout, p, _lib.stream_ptr())
        self.kernel_launches += 5
        return Y

    def _trunc_masks(self, idx, op, src_rng):
        """Source: alpha / comp shares for truncation idx (gen_additive_mask), cached."""
        if not hasattr(self, "_mask_cache"):
            self._mask_cache = {}
        got = self._mask_cache.get(idx)
        if got is not None:
            return got
        B, n, p = self.batch, self.n, self.p
        N = B * _count(op.in_shape)
        step = op.r * op.divisor
        emax = additive_mask_bound(self.scheme.field, step, op.value_bound)
        if self.host:
            got = self._mask_cache[idx] = (self._hb(idx, "alpha"), self._hb(idx, "comp"))
            return got
        A = torch.empty((n, N), dtype=torch.int64, device=self.dev)
        Cm = torch.empty((n, N), dtype=torch.int64, device=self.dev)
        _lib.call("ssn_mask_trunc", N, step, emax, src_rng.seed, src_rng.next_stream(3), self.k - 1, self.ids_all, n,
                  _lib.ptr(A), _lib.ptr(Cm), N, p, _lib.stream_ptr())
        self.kernel_launches += 1
        self._mask_cache[idx] = (A, Cm)
        return A, Cm

    def _truncation(self, idx, op, X, fused, src_rng, party_rng):
        B, n, k, p = self.batch, self.n, self.k, self.p
        N = B * _count(op.in_shape)
        A, Cm = self._trunc_masks(idx, op, src_rng)
        self._mask_cache.pop(idx, None)
        senders = n if self.verify else k
        if fused:
            masked = X
        else:
            masked = torch.empty((senders, N), dtype=torch.int64, device=self.dev)
            self._ew(0, X, A, masked, senders * N)
        FR = torch.empty((n, N), dtype=torch.int64, device=self.dev)
        tco = self._hb(idx, "tcoef") if (self.host and k > 1) else None
        _lib.call("ssn_trunc_elite", _lib.ptr(masked), N, senders, k, _lib.u64_array(self.w_front),
                  _lib.u64_array(self.ext), op.value_bound, op.r, op.divisor, _lib.ptr(tco), party_rng.seed,
                  party_rng.next_stream(), k - 1, self.ids_all, n, _lib.ptr(FR), N,
                  _lib.ptr(self.fail) if self.verify else None, N, p, _lib.stream_ptr())
        Y = torch.empty((n, B) + tuple(op.out_shape), dtype=torch.int64, device=self.dev)
        self._ew(0, FR, Cm, Y, n * N)
        self.kernel_launches += 1
        return Y

    def _nonlinear_fused(self, idx, op, X, src_rng):
        """A nonlinear op outside a linear chain (e.g. the global pool) as ONE launch of the
        chain kernel's masked-nonlinearity stage (mask, elite rec/ReLU/pool, beta^-1 output)."""
        B, n, k, m, p = self.batch, self.n, self.k, self.m, self.p
        n_in, n_out = B * _count(op.in_shape), B * _count(op.out_shape)
        if op.pool_kind is not None:
            (c, h, w), (kh, kw) = op.in_shape, op.pool
            kind = 1 if op.pool_kind == "max" else 2
        elif len(op.in_shape) == 3:
            (c, h, w), kh, kw, kind = op.in_shape, 1, 1, 0
        else:
            c, h, w, kh, kw, kind = _count(op.in_shape), 1, 1, 1, 1, 0
        Y = torch.empty((n, B) + tuple(op.out_shape), dtype=torch.int64, device=self.dev)
        d = _lib.ChainDesc()
        d.acc, d.acc_pstride = X.data_ptr(), n_in
        d.out, d.out_pstride = Y.data_ptr(), n_out
        d.nel = n_in
        d.nonlin, d.nonlin_only, d.relu, d.pool_kind = 1, 1, int(bool(op.relu)), kind
        d.nb, d.c, d.h, d.w, d.kh, d.kw = B, c, h, w, kh, kw
        d.fan = n if op.passive_out else k
        d.bmax = multiplicative_mask_bound(self.scheme.field, op.value_bound)
        d.nout, d.r, d.d, d.emax = n, 1, 1, 1
        d.bias_div, d.bias_mod = 1, 1
        d.src_seed, d.src_stream = src_rng.seed, src_rng.next_stream(7)
        d.k, d.n = k, n
        d.ids, d.rt = ctypes.addressof(self.ids_all), ctypes.addressof(self._rt_all)
        d.ext = ctypes.addressof(self._ext_host) if self._ext_host is not None else None
        d.p = p
        d.fault_rank = -1
        if self.host:
            d.host_masks = 1
            d.h_beta = self.hm[(idx, "beta")].data_ptr()
            d.h_binv = self.hm[(idx, "beta_inv")].data_ptr()
            d.h_period, d.h_period_out = _count(op.in_shape), _count(op.out_shape)
        _lib.call("ssn_layer_chain", ctypes.byref(d), _lib.stream_ptr())
        self.kernel_launches += 1
        return Y

    def _nonlinear(self, idx, op, X, src_rng):
        B, n, k, m, p = self.batch, self.n, self.k, self.m, self.p
        n_in, n_out = B * _count(op.in_shape), B * _count(op.out_shape)
        if op.pool_kind is not None:
            c, h, w = op.in_shape
            kh, kw = op.pool
            kind = 1 if op.pool_kind == "max" else 2
        elif len(op.in_shape) == 3:
            (c, h, w), kh, kw, kind = op.in_shape, 1, 1, 0
        else:
            c, h, w, kh, kw, kind = _count(op.in_shape), 1, 1, 1, 1, 0
        bmax = multiplicative_mask_bound(self.scheme.field, op.value_bound)
        if self.host:
            BETA, BINV = self._hb(idx, "beta"), self._hb(idx, "beta_inv")
        else:
            BETA = torch.empty((n, n_in), dtype=torch.int64, device=self.dev)
            BINV = torch.empty((n, n_out), dtype=torch.int64, device=self.dev)
            _lib.call("ssn_mask_beta", B, c, h, w, kh, kw, bmax, src_rng.seed, src_rng.next_stream(3), k - 1,
                      self.ids_all, n, _lib.ptr(BETA), n_in, _lib.ptr(BINV), n_out, p, _lib.stream_ptr())
        MASKED = torch.empty((m, n_in), dtype=torch.int64, device=self.dev)
        self._ew(2, X, BETA, MASKED, m * n_in)
        plain = torch.empty(n_out, dtype=torch.int64, device=self.dev)
        _lib.call("ssn_nonlin_elite", _lib.ptr(MASKED), n_in, m, _lib.u64_array(self.w_part), int(bool(op.relu)),
                  kind, B, c, h, w, kh, kw, _lib.ptr(plain), p, _lib.stream_ptr())
        fan = n if op.passive_out else k
        Y = torch.empty((n, B) + tuple(op.out_shape), dtype=torch.int64, device=self.dev)
        self._ew(2, BINV, plain, Y, fan * n_out, b_mod=n_out)
        self.kernel_launches += 2
        return Y

    def _output(self, op, X):
        B, n, k, p = self.batch, self.n, self.k, self.p
        N = B * _count(op.out_shape)
        if self.verify:
            scratch = torch.empty(N, dtype=torch.int64, device=self.dev)
            _lib.call("ssn_trunc_elite", _lib.ptr(X), N, n, k, _lib.u64_array(self.w_front),
                      _lib.u64_array(self.ext), 0, 1, 1, None, 0, 0, 0, None, 0, _lib.ptr(scratch), 0,
                      _lib.ptr(self.fail), N, p, _lib.stream_ptr())
        v = torch.empty(N, dtype=torch.int64, device=self.dev)
        _lib.call("ssn_rec", _lib.ptr(X), 0, N, _lib.u64_array(self.w_front), k, _lib.ptr(v), 0, N, 1, p,
                  _lib.stream_ptr())
        out = torch.empty_like(v)
        _lib.call("ssn_decode_signed", _lib.ptr(v), _lib.ptr(out), N, p, _lib.stream_ptr())
        self.kernel_launches += 2
        if self.verify and not self.defer_verify:
            self._check_failures()
        return out.reshape((B,) + tuple(op.out_shape))

    # defer_verify: the Reed-Solomon checks still run inside every step's kernels, but the host
    # reads the device failure counter only in check_verification() -- no per-step sync, so the
    # host enqueues step i+1 while the GPU runs step i
    defer_verify = False

    def check_verification(self):
        """Raise VerificationError if any deferred check failed since the last call."""
        self._check_failures()

    def _check_failures(self):
        bad = int(self.fail.item())
        if bad:
            self.fail.zero_()
            raise VerificationError(f"{bad} share(s) failed the Reed-Solomon check")


class StreamPipelinedEngine:
    """S BatchedEngines on S CUDA streams, each on 1/S of the batch.  The share GEMMs are
    tensor-pipe bound and the fused protocol chains integer-ALU bound, so kernels of different
    streams co-reside on the SMs (the persistent GEMM leaves registers for a chain block) and
    overlap.  Weight shares and limb planes are shared.  Same outputs as one engine."""

    def __init__(self, model, scheme, batch, streams=2, seed=7, verify=False, **kw):
        if batch % streams:
            raise ValueError(f"batch {batch} not divisible by {streams} streams")
        self.batch, self.nstreams = batch, streams
        if kw.get("rng_mode", "device") != "device":
            raise ValueError("the stream-pipelined engine runs in speed mode (device randomness)")
        first = BatchedEngine(model, scheme, batch // streams, seed=seed, verify=verify, **kw)
        self.engines = [first] + [BatchedEngine(model, scheme, batch // streams, seed=seed + 1000 * i, verify=verify,
                                                share_weights_with=first, **kw) for i in range(1, streams)]
        self.streams = [torch.cuda.Stream() for _ in range(streams)]
        self.scheme, self.ops = scheme, first.ops
        self._warm = False

    def __getattr__(self, name):                  # out_shape, comm_per_image, limb_products, ...
        return getattr(self.engines[0], name)

    def run(self, x_int, timings=None):
        return self.run_device(x_int).cpu().numpy()

    def run_device(self, x_int, timings=None, serial=False):
        """serial=True runs the sub-batches back to back (each stream waits for the previous
        one): same results, no kernel overlap -- bench.py times its per-kernel roofline step so."""
        if not isinstance(x_int, torch.Tensor):
            x_int = torch.as_tensor(np.asarray(x_int, dtype=np.int64))
        x = x_int.to(device=self.engines[0].dev, dtype=torch.int64)
        cur = torch.cuda.current_stream()
        parts = x.chunk(self.nstreams)
        if not self._warm:
            # the weight limb planes are built lazily by the first GEMM that needs them and are
            # shared by all sub-batches: the first run goes stream after stream, so no sub-batch
            # reads planes another stream has not finished writing
            serial, self._warm = True, True
        outs = []
        prev = cur
        for eng, st, xp in zip(self.engines, self.streams, parts):
            st.wait_stream(prev if serial else cur)
            with torch.cuda.stream(st):
                outs.append(eng.run_device(xp))
            if serial:
                prev = st
        for st, o in zip(self.streams, outs):
            cur.wait_stream(st)
            o.record_stream(cur)
        return torch.cat(outs)

    def enable_profiling(self):
        for e in self.engines:
            e.enable_profiling()

    def disable_profiling(self):
        for e in self.engines:
            e.disable_profiling()

    def profile_summary(self, steps):
        merged = {}
        for e in self.engines:
            for cls, rec in (e._prof or {}).items():
                merged.setdefault(cls, []).extend(rec)
        e0 = self.engines[0]
        saved, e0._prof = e0._prof, merged
        try:
            return e0.profile_summary(steps)
        finally:
            e0._prof = saved
