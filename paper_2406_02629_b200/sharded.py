"""Party-per-GPU batched secure inference: one process (GPU) per protocol rank, share
exchange over torch.distributed point-to-point (NCCL send/recv over NVLink on a multi-GPU
node; gloo, host-staged, when several ranks share one GPU).

The same protocol as the co-resident engines (engine.py, batched.py) and the reference
(S/engine.py:77-102, S/layers.py:236-380, S/protocol.py:131-305), but every rank computes
ONLY its own party's shares, and every message crosses a process boundary:

  rank 0 (trusted source)   draws every mask with the device kernels (ssn_gen zero shares,
                            ssn_mask_trunc alpha/comp, ssn_mask_beta beta/beta^-1) and streams
                            each party its row, per op, ahead of use (MASK_DIST,
                            S/protocol.py:354-388).
  ranks 1..n (parties)      linear: local share GEMM -> RESHARE_OUT to the k front ranks ->
                            R^T at the fronts -> RESHARE_BACK -> rec + zero + bias
                            (S/protocol.py:131-199); truncation: TRUNC_MASKED to the elite,
                            elite truncates and SHARE_DIST's fresh shares (S/layers.py:277-323);
                            nonlinear: NONLIN_MASKED to the elite, NONLIN_PLAIN back
                            (S/layers.py:326-380); output: OUTPUT_SHARE (S/protocol.py:289-305).

Each protocol hop is one grouped batch_isend_irecv (ncclGroupStart / ncclSend / ncclRecv /
ncclGroupEnd) over all of the rank's peers for that hop.  The elite role of the masked
truncations and nonlinearities rotates over the front ranks op by op (rotate_elite, default on;
any front rank can reconstruct over the same front ids, S/sss.py:172-194), so the elite's
extra receives, reconstructions and fan-out sends -- and its NVLink ingress -- are spread
over k GPUs instead of landing on rank 1; the final output is still collected at rank 1.  A world of G*(n+1) ranks runs G
independent groups, each on its own image batch (data parallel over images, SURVEY.md
section 8e placement 2).  Decoded outputs equal the reference / integer plaintext exactly.
"""

import os

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from . import gemm as gemm_mod
from .batched import _count
from .gemm import field_conv, field_dense
from .layers import consumers, plan_schedule, window_gather
from .masks import additive_mask_bound, multiplicative_mask_bound
from .protocol import VerificationError, extrapolation_coeffs
from .rng import DeviceRng


class PartyShardedEngine:
    def __init__(self, model, scheme, batch, seed=7, verify=False, ordering="ltn", group=0, rotate_elite=True):
        self.model, self.scheme, self.batch, self.seed, self.verify = model, scheme, int(batch), seed, verify
        self.rotate_elite = rotate_elite
        # reshare step 1 in the share GEMM's epilogue (ssn_gemm_tc_subshares, bit-identical to the
        # GEMM + ssn_gen pair).  Opt-in (SSN_FUSED_SUBSHARES=1): measured slower on every ResNet
        # layer class (profiles/r02/fused_subshares_probe.json) -- the single-buffered 352-column
        # TMEM accumulator makes the longer epilogue the critical path on small-K layers
        self.fuse_subshares = os.environ.get("SSN_FUSED_SUBSHARES", "0") == "1"
        self.k, self.n = scheme.k, scheme.n
        self.m = 2 * self.k - 1
        self.p = scheme.field.p
        self.size = self.n + 1
        self.base = group * self.size
        self.role = dist.get_rank() - self.base            # 0 = source, 1..n = party id
        if not 0 <= self.role < self.size:
            raise ValueError(f"rank {dist.get_rank()} is not in group {group}")
        self.t = self.role - 1                             # party index (ids[t])
        self.nccl = dist.get_backend() == "nccl"
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self.ops, self.digest = plan_schedule(model, scheme, ordering, verify=verify)
        self.cons = consumers(self.ops)
        k, n, m = self.k, self.n, self.m
        self.w_front = scheme.lagrange_weights(scheme.front_ids)
        self.w_part = scheme.lagrange_weights(scheme.party_ids[:m])
        R = scheme.reducing_matrix()
        self.rt = {nout: [R[i][t] for t in range(nout) for i in range(m)] for nout in (k, n)}
        self.ext = [v for row in extrapolation_coeffs(scheme, scheme.front_ids, scheme.party_ids[k:]) for v in row]
        self.ids_all = _lib.u64_array(scheme.party_ids)
        self.ids_front = _lib.u64_array(scheme.front_ids)
        self.fail = torch.zeros(1, dtype=torch.int64, device=self.dev)
        self.runs = 0
        self._pending = []
        self._planes = {}
        if self.role > 0:
            self._deal_weights()

    # ------------------------------------------------------------------ plumbing
    def _g(self, role):
        return self.base + role

    def _exchange(self, sends, recvs):
        """One grouped hop: sends [(role, tensor)], recvs [(role, out_tensor)]."""
        if not sends and not recvs:
            return
        ops, staged = [], []
        for role, t in sends:
            tt = t.contiguous() if self.nccl else t.contiguous().cpu()
            ops.append(dist.P2POp(dist.isend, tt, self._g(role)))
            staged.append(tt)
        for role, t in recvs:
            buf = t if self.nccl else torch.empty(t.shape, dtype=t.dtype)
            ops.append(dist.P2POp(dist.irecv, buf, self._g(role)))
            staged.append((buf, t))
        for w in dist.batch_isend_irecv(ops):
            w.wait()
        if not self.nccl:
            for item in staged[len(sends):]:
                item[1].copy_(item[0])

    def _post(self, role, tensor):
        """Source: non-blocking send, kept alive until completion."""
        tt = tensor.contiguous() if self.nccl else tensor.contiguous().cpu()
        self._pending.append((dist.isend(tt, self._g(role)), tt))
        if len(self._pending) > 256:
            self._pending[0][0].wait()
            self._pending = [(w, x) for (w, x) in self._pending if not w.is_completed()]

    def _recv_new(self, role, shape):
        out = torch.empty(shape, dtype=torch.int64, device=self.dev)
        self._exchange([], [(role, out)])
        return out

    # ------------------------------------------------------------------ setup
    def _deal_weights(self):
        """Own row of the weight shares dealt from lane 1 (S/engine.py:40-49)."""
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
            self.W[name] = out[self.t:self.t + 1].clone()

    def _encode(self, v):
        out = torch.empty_like(v)
        ovf = torch.zeros(1, dtype=torch.int64, device=self.dev)
        _lib.call("ssn_encode_signed", _lib.ptr(v), _lib.ptr(out), v.numel(), _lib.ptr(ovf), self.p,
                  _lib.stream_ptr())
        return out

    def _ew(self, op, a, b, out, n, b_mod=None):
        bm = n if b_mod is None else b_mod
        _lib.call("ssn_ewise", op, _lib.ptr(a), _lib.ptr(b), _lib.ptr(out), n, 1, bm, 1 << 62, 0, self.p,
                  _lib.stream_ptr())

    # ------------------------------------------------------------------ run
    def run(self, x_int):
        """One secure inference of this group's batch.  Every rank of the group calls it; the
        elite (role 1) returns the decoded int64 outputs, every other rank None."""
        out = self.run_device(x_int)
        return None if out is None else out.cpu().numpy()

    def run_device(self, x_int):
        run_id = self.runs
        self.runs += 1
        if self.role == 0:
            self._source(run_id)
            return None
        return self._party(x_int, run_id)

    # ------------------------------------------------------------------ trusted source
    def _source(self, run_id):
        B, n, k, p = self.batch, self.n, self.k, self.p
        rng = DeviceRng(self.seed, 4, run_id)
        for idx, op in enumerate(self.ops):
            if op.kind == "linear":
                N = B * _count(op.out_shape)
                Z = torch.empty((n, N), dtype=torch.int64, device=self.dev)
                _lib.call("ssn_gen", None, 0, None, 0, rng.seed, rng.next_stream(), k - 1, self.ids_all, n,
                          _lib.ptr(Z), 0, N, N, 1, p, _lib.stream_ptr())
                rows = [Z]
            elif op.kind == "truncation":
                N = B * _count(op.in_shape)
                step = op.r * op.divisor
                emax = additive_mask_bound(self.scheme.field, step, op.value_bound)
                A = torch.empty((n, N), dtype=torch.int64, device=self.dev)
                C = torch.empty((n, N), dtype=torch.int64, device=self.dev)
                _lib.call("ssn_mask_trunc", N, step, emax, rng.seed, rng.next_stream(3), k - 1, self.ids_all, n,
                          _lib.ptr(A), _lib.ptr(C), N, p, _lib.stream_ptr())
                rows = [A, C]
            elif op.kind == "nonlinear":
                c, h, w, kh, kw, _ = self._nl_geom(op)
                n_in, n_out = B * _count(op.in_shape), B * _count(op.out_shape)
                bmax = multiplicative_mask_bound(self.scheme.field, op.value_bound)
                BETA = torch.empty((n, n_in), dtype=torch.int64, device=self.dev)
                BINV = torch.empty((n, n_out), dtype=torch.int64, device=self.dev)
                _lib.call("ssn_mask_beta", B, c, h, w, kh, kw, bmax, rng.seed, rng.next_stream(3), k - 1,
                          self.ids_all, n, _lib.ptr(BETA), n_in, _lib.ptr(BINV), n_out, p, _lib.stream_ptr())
                rows = [BETA, BINV]
            else:
                continue
            for T in rows:                      # MASK_DIST: party t gets row t
                for t in range(n):
                    self._post(t + 1, T[t])
        for w, _ in self._pending:
            w.wait()
        self._pending = []

    @staticmethod
    def _nl_geom(op):
        if op.pool_kind is not None:
            (c, h, w), (kh, kw) = op.in_shape, op.pool
            return c, h, w, kh, kw, (1 if op.pool_kind == "max" else 2)
        if len(op.in_shape) == 3:
            c, h, w = op.in_shape
            return c, h, w, 1, 1, 0
        return _count(op.in_shape), 1, 1, 1, 1, 0

    # ------------------------------------------------------------------ party
    def _party(self, x_int, run_id):
        B, n, k, t, p = self.batch, self.n, self.k, self.t, self.p
        prng = DeviceRng(self.seed, 5, run_id, self.role)
        if isinstance(x_int, torch.Tensor):
            x = x_int.to(device=self.dev, dtype=torch.int64).contiguous()
        else:
            x = torch.as_tensor(np.asarray(x_int, dtype=np.int64), device=self.dev).contiguous()
        # input dealing (S/engine.py:52-54), lane 3: every rank derives the same sharing, keeps its row
        enc = self._encode(x)
        X = torch.empty((n,) + tuple(x.shape), dtype=torch.int64, device=self.dev)
        irng = DeviceRng(self.seed, 3, run_id)
        nel = x.numel()
        _lib.call("ssn_gen", _lib.ptr(enc), 0, None, 0, irng.seed, irng.next_stream(), k - 1, self.ids_all, n,
                  _lib.ptr(X), 0, nel, nel, 1, p, _lib.stream_ptr())
        vals = {-1: X[t].clone()}
        del X
        remaining = {i: len(c) for i, c in self.cons.items()}
        result = None
        masked_ops = 0
        for idx, op in enumerate(self.ops):
            src = idx - 1 if op.src is None else op.src
            xin = vals.get(src)
            if op.kind in ("truncation", "nonlinear"):
                e = masked_ops % k if self.rotate_elite else 0          # this op's elite (front index)
                masked_ops += 1
            if op.kind == "linear":
                y = self._linear(op, xin, prng)
            elif op.kind == "truncation":
                y = self._truncation(op, xin, prng, e)
            elif op.kind == "nonlinear":
                y = self._nonlinear(op, xin, e)
            elif op.kind == "add":
                other = vals.get(op.src2)
                y = None
                if xin is not None and other is not None:
                    y = torch.empty_like(xin)
                    self._ew(0, xin, other, y, y.numel())
            elif op.kind == "gather":               # local: this party's share only
                y = None
                if xin is not None:
                    kh, kw = op.pool
                    y = window_gather(xin, op.in_shape, kh, kw, op.stride, op.padding, nbatch=B) \
                        .reshape((B,) + tuple(op.out_shape))
            elif op.kind == "output":
                result = self._output(op, xin)
                y = None
            else:
                raise ValueError(op.kind)
            if y is not None:
                vals[idx] = y
            for s in ([src] + ([op.src2] if op.kind == "add" else [])):
                remaining[s] -= 1
                if remaining[s] <= 0:
                    vals.pop(s, None)
        return result

    def _linear(self, op, X, prng):
        B, n, k, m, t, p = self.batch, self.n, self.k, self.m, self.t, self.p
        O = op.out_shape[0]
        ohw = _count(op.out_shape[1:]) if len(op.out_shape) > 1 else 1
        N = B * O * ohw
        nout = n if op.passive_out else k
        Z = self._recv_new(0, (N,))                                      # MASK_DIST: zero share
        SUB = None
        if t < m:                                                        # participant: local product
            w = self.W[op.weight + ".w"]
            K = _count(w.shape[2:])
            tc = gemm_mod.use_tc(p, B * ohw, K, O)
            planes = None
            if tc:
                planes = self._planes.get(op.weight)
                if planes is None:
                    planes = self._planes[op.weight] = gemm_mod.weight_planes(w.reshape(1, O, K), p, 1)
            SUB = torch.empty((k, N), dtype=torch.int64, device=self.dev)    # step 1 sub-shares
            stream = prng.next_stream()
            # reshare step 1 fused into the GEMM epilogue: the sub-shares are written straight into
            # the RESHARE_OUT send buffers (bit-identical to GEMM + ssn_gen)
            fused = self.fuse_subshares and tc and gemm_mod.fused_subshares_supported(p, K)
            sub = gemm_mod.SubShares(SUB, prng.seed, stream, k - 1, self.scheme.front_ids) if fused else None
            if w.dim() == 5:
                C, H, Wd = op.in_shape
                acc = field_conv(w, X.reshape(1, B, C, H, Wd), op.stride, op.padding, p, nimg=B, nparty=1,
                                 planes=planes, force="tc" if tc else "simt", sub=sub)
            else:
                acc = field_dense(w, X.reshape(1, B, -1), p, nimg=B, nparty=1, planes=planes,
                                  force="tc" if tc else "simt", sub=sub)
            if not fused:
                _lib.call("ssn_gen", _lib.ptr(acc), N, None, 0, prng.seed, stream, k - 1, self.ids_front, k,
                          _lib.ptr(SUB), N, N, N, 1, p, _lib.stream_ptr())
        # hop 1 (RESHARE_OUT): participant -> every other front rank
        PTS = torch.empty((m, N), dtype=torch.int64, device=self.dev) if t < k else None
        sends = [(f + 1, SUB[f]) for f in range(k) if f != t] if SUB is not None else []
        recvs = [(j + 1, PTS[j]) for j in range(m) if j != t] if t < k else []
        self._exchange(sends, recvs)
        BACK = None
        if t < k:
            PTS[t].copy_(SUB[t])
            BACK = torch.empty((nout, N), dtype=torch.int64, device=self.dev)           # step 2: R^T
            _lib.call("ssn_reduce_apply", _lib.ptr(PTS), 0, N, m, _lib.u64_array(self.rt[nout]), nout,
                      _lib.ptr(BACK), 0, N, N, 1, p, _lib.stream_ptr())
        # hop 2 (RESHARE_BACK): front -> every other out rank
        BK = torch.empty((k, N), dtype=torch.int64, device=self.dev) if t < nout else None
        sends = [(o + 1, BACK[o]) for o in range(nout) if o != t] if BACK is not None else []
        recvs = [(f + 1, BK[f]) for f in range(k) if f != t] if t < nout else []
        self._exchange(sends, recvs)
        if t >= nout:
            return None
        if t < k:
            BK[t].copy_(BACK[t])
        Y = torch.empty((B,) + tuple(op.out_shape), dtype=torch.int64, device=self.dev)   # step 3
        bias = self.W[op.weight + ".b"]
        _lib.call("ssn_reshare_finish", _lib.ptr(BK), 0, N, _lib.u64_array(self.w_front), k, _lib.ptr(Z), 0,
                  _lib.ptr(bias), 0, ohw, O, None, 0, _lib.ptr(Y), 0, N, 1, p, _lib.stream_ptr())
        return Y

    def _truncation(self, op, X, prng, e=0):
        """S/layers.py:277-323 with front rank e+1 as the elite."""
        B, n, k, t, p = self.batch, self.n, self.k, self.t, self.p
        N = B * _count(op.in_shape)
        A = self._recv_new(0, (N,))
        Cm = self._recv_new(0, (N,))
        senders = n if self.verify else k
        masked = None
        if t < senders:
            masked = torch.empty(N, dtype=torch.int64, device=self.dev)
            self._ew(0, X, A, masked, N)
        FR = torch.empty((n if t == e else 1, N), dtype=torch.int64, device=self.dev)
        if t == e:                                                       # elite
            PTS = torch.empty((senders, N), dtype=torch.int64, device=self.dev)   # points in id order
            self._exchange([], [(j + 1, PTS[j]) for j in range(senders) if j != e])
            PTS[e].copy_(masked)
            _lib.call("ssn_trunc_elite", _lib.ptr(PTS), N, senders, k, _lib.u64_array(self.w_front),
                      _lib.u64_array(self.ext), op.value_bound, op.r, op.divisor, None, prng.seed,
                      prng.next_stream(), k - 1, self.ids_all, n, _lib.ptr(FR), N,
                      _lib.ptr(self.fail) if self.verify else None, N, p, _lib.stream_ptr())
            self._exchange([(o + 1, FR[o]) for o in range(n) if o != e], [])     # SHARE_DIST
            own = FR[e]
        else:
            self._exchange([(e + 1, masked)] if masked is not None else [], [])   # TRUNC_MASKED
            self._exchange([], [(e + 1, FR[0])])
            own = FR[0]
        Y = torch.empty((B,) + tuple(op.out_shape), dtype=torch.int64, device=self.dev)
        self._ew(0, own, Cm, Y, N)
        return Y

    def _nonlinear(self, op, X, e=0):
        """S/layers.py:326-380 with participant e+1 (a front rank) as the elite."""
        B, n, k, m, t, p = self.batch, self.n, self.k, self.m, self.t, self.p
        n_in, n_out = B * _count(op.in_shape), B * _count(op.out_shape)
        BETA = self._recv_new(0, (n_in,))
        BINV = self._recv_new(0, (n_out,))
        c, h, w, kh, kw, kind = self._nl_geom(op)
        fan = n if op.passive_out else k
        MK = None
        if t < m:
            MK = torch.empty(n_in, dtype=torch.int64, device=self.dev)
            self._ew(2, X, BETA, MK, n_in)
        plain = torch.empty(n_out, dtype=torch.int64, device=self.dev)
        if t == e:
            PTS = torch.empty((m, n_in), dtype=torch.int64, device=self.dev)
            self._exchange([], [(j + 1, PTS[j]) for j in range(m) if j != e])   # NONLIN_MASKED
            PTS[e].copy_(MK)
            _lib.call("ssn_nonlin_elite", _lib.ptr(PTS), n_in, m, _lib.u64_array(self.w_part), int(bool(op.relu)),
                      kind, B, c, h, w, kh, kw, _lib.ptr(plain), p, _lib.stream_ptr())
            self._exchange([(o + 1, plain) for o in range(fan) if o != e], [])  # NONLIN_PLAIN
        else:
            self._exchange([(e + 1, MK)] if MK is not None else [], [])
            if t < fan:
                self._exchange([], [(e + 1, plain)])
        if t >= fan:
            return None
        Y = torch.empty((B,) + tuple(op.out_shape), dtype=torch.int64, device=self.dev)
        self._ew(2, BINV, plain, Y, n_out)
        return Y

    def _output(self, op, X):
        B, n, k, t, p = self.batch, self.n, self.k, self.t, self.p
        N = B * _count(op.out_shape)
        senders = n if self.verify else k
        if t != 0:
            self._exchange([(1, X.reshape(-1))] if t < senders else [], [])  # OUTPUT_SHARE
            return None
        PTS = torch.empty((senders, N), dtype=torch.int64, device=self.dev)
        self._exchange([], [(j + 1, PTS[j]) for j in range(1, senders)])
        PTS[0].copy_(X.reshape(-1))
        if self.verify:
            scratch = torch.empty(N, dtype=torch.int64, device=self.dev)
            _lib.call("ssn_trunc_elite", _lib.ptr(PTS), N, senders, k, _lib.u64_array(self.w_front),
                      _lib.u64_array(self.ext), 0, 1, 1, None, 0, 0, 0, None, 0, _lib.ptr(scratch), 0,
                      _lib.ptr(self.fail), N, p, _lib.stream_ptr())
        v = torch.empty(N, dtype=torch.int64, device=self.dev)
        _lib.call("ssn_rec", _lib.ptr(PTS), 0, N, _lib.u64_array(self.w_front), k, _lib.ptr(v), 0, N, 1, p,
                  _lib.stream_ptr())
        out = torch.empty_like(v)
        _lib.call("ssn_decode_signed", _lib.ptr(v), _lib.ptr(out), N, p, _lib.stream_ptr())
        if self.verify:
            bad = int(self.fail.item())
            if bad:
                self.fail.zero_()
                raise VerificationError(f"{bad} share(s) failed the Reed-Solomon check")
        return out.reshape((B,) + tuple(op.out_shape))
