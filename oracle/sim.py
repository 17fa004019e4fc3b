"""Lockstep CPU restatement of the reference secure-inference run -- TEST ONLY.

Restates simulate_schedule (S/engine.py:145-193) with every party advanced in
lockstep on one thread instead of one thread per rank.  Each rank owns its own
numpy Generator (S/engine.py:166-171), so per-rank draw order -- and therefore
every share value -- matches the threaded reference exactly.  The arithmetic
runs through oracle/ssn_oracle.c.

What it reproduces (pinned by tests/test_oracle.py against the reference):
  * decoded output at the elite (output_collect, S/protocol.py:289-305)
  * every party's share of every op output
  * the SimHub canonical transcript (S/transport.py:68-80) and its sha256
  * per-op element counts (S/metrics.py:46-60)

Schedule ops are the reference's ScheduledOp.meta() dicts (S/layers.py:63-73).
Two builder extensions, used by the ResNet models and marked as such:
  * "src"/"src2": producer op index (-1 = model input); default = previous op.
  * kind "add": local share_add of two degree-(k-1) shares (S/sss.py:238).
  * kind "gather": local overlapping-window gather of every party's share (zero fill), so the
    following reference nonlinear op's non-overlapping pool is an overlapping pool (ResNet's
    3x3/s2/p1 stem max-pool).  Fields: pool = (kh, kw), stride, padding.
  * verify=True: masked-value Reed-Solomon check at the truncation elite and
    at output collection; never changes outputs.
"""

import hashlib
import json
import struct

import numpy as np

from . import (DEFAULT_PRIME, decode_signed, encode_signed, ewise, gemm, gen, im2col,
               lagrange_weights, nonlin_elite, reducing_matrix, rec, reduce_apply,
               trunc_elite, window_gather)

# Phase tags (S/wire.py:32-41)
MASK_DIST, SHARE_DIST, RESHARE_OUT, RESHARE_BACK = 2, 3, 4, 5
TRUNC_MASKED, NONLIN_MASKED, NONLIN_PLAIN, OUTPUT_SHARE = 6, 7, 8, 9

E_BUDGET = 1 << 32      # S/masks.py:20
BETA_BITS = 28          # S/masks.py:21


def seeded_rng(seed, *path):
    """S/engine.py:31-32."""
    return np.random.default_rng([int(seed)] + [int(x) for x in path])


class Scheme:
    def __init__(self, k, n, party_ids=None, p=DEFAULT_PRIME):
        self.k, self.n, self.p = k, n, p
        self.party_ids = tuple(party_ids or range(1, n + 1))
        self.front_ids = self.party_ids[:k]
        self.part_ids = self.party_ids[:2 * k - 1]
        self.half = (p - 1) // 2

    def rand(self, rng, shape):
        """PrimeField.rand (S/field.py:138-142)."""
        return rng.integers(0, self.p, size=shape, dtype=np.int64).astype(np.uint64)

    def share(self, secret, rng, ids=None):
        """SssScheme.gen (S/sss.py:118-147): coefficients drawn c_1..c_{k-1} in order."""
        secret = np.asarray(secret, dtype=np.uint64)
        coeffs = [self.rand(rng, secret.shape) for _ in range(self.k - 1)]
        return gen(secret, coeffs, ids or self.party_ids, self.p)


class Transcript:
    """SimHub channel transcript (S/transport.py:49-84) + CommMetrics element counts."""

    def __init__(self, n, record):
        self.record = record
        self.frames = {(s, d): [] for s in range(n + 1) for d in range(n + 1) if s != d}
        self.elements = {}

    def send(self, label, src, dst, phase, payload_fn, elements):
        key = label
        self.elements[key] = self.elements.get(key, 0) + int(elements)
        if self.record:
            payload = payload_fn()
            self.frames[(src, dst)].append(
                struct.pack("<4sHHI", b"SSN1", src, phase, len(payload)) + payload)

    def canonical(self):
        parts = []
        for key in sorted(self.frames):
            fr = self.frames[key]
            parts.append(struct.pack("<HHI", key[0], key[1], len(fr)))
            parts.extend(fr)
        return b"".join(parts)

    def digest(self):
        return hashlib.sha256(self.canonical()).hexdigest()


def _share_payload(pid, degree, vals):
    """encode_share_tensor (S/wire.py:104-107)."""
    v = np.asarray(vals, dtype=np.uint64)
    hdr = struct.pack(f"<QHB{v.ndim}I", pid, degree, v.ndim, *v.shape)
    return hdr + v.astype("<u8").tobytes()


def _plain_payload(vals):
    """encode_plain_tensor (S/wire.py:95-98)."""
    v = np.asarray(vals, dtype=np.uint64)
    return struct.pack(f"<B{v.ndim}I", v.ndim, *v.shape) + v.astype("<u8").tobytes()


def _bundle_payload(entries):
    """MaskBundle.encode (S/protocol.py:324-333); entries {(idx,name): (pid, deg, vals)}."""
    meta, blobs = [], []
    for key in sorted(entries):
        pid, deg, vals = entries[key]
        meta.append({"op": key[0], "name": key[1], "party_id": pid, "degree": deg,
                     "shape": list(vals.shape)})
        blobs.append(np.asarray(vals, dtype=np.uint64).astype("<u8").tobytes())
    head = json.dumps(meta, sort_keys=True).encode()
    return struct.pack("<I", len(head)) + head + b"".join(blobs)


def additive_mask_bound(p, step, value_bound):
    """S/masks.py:24-36."""
    emax = min(E_BUDGET // step, (p - 1 - 2 * value_bound) // step + 1)
    if emax < 1:
        raise ValueError("no mask fits")
    return emax


def multiplicative_mask_bound(p, value_bound):
    """S/masks.py:57-64."""
    bmax = min(1 << BETA_BITS, ((p - 1) // 2) // value_bound)
    if bmax < 1:
        raise ValueError("no positive factor fits")
    return bmax


def _inv_vec(x, p):
    from . import inv_vec
    return inv_vec(np.asarray(x, dtype=np.uint64), p).reshape(np.shape(x))


def source_masks(ops, sch, rng, record_plain=False):
    """trusted_source_prepare (S/protocol.py:354-388) with S/masks.py draws.

    Returns bundles {rank: {(idx, name): (pid, degree, values)}} and plain masks."""
    p, k = sch.p, sch.k
    bundles = {r: {} for r in range(1, sch.n + 1)}
    plain = {}

    def spread(idx, name, shares):
        for r in range(1, sch.n + 1):
            bundles[r][(idx, name)] = (sch.party_ids[r - 1], k - 1, shares[r - 1])

    for idx, op in enumerate(ops):
        kind = op["kind"]
        if kind == "linear":
            spread(idx, "zero", sch.share(np.zeros(tuple(op["out_shape"]), np.uint64), rng))
        elif kind == "truncation":
            step = op["r"] * op["divisor"]
            emax = additive_mask_bound(p, step, op["value_bound"])
            e = rng.integers(1, emax + 1, size=tuple(op["in_shape"]), dtype=np.int64)
            alpha = ((e * step) % p).astype(np.uint64)      # e*step < 2^52: exact in int64
            comp = ((-e) % p).astype(np.uint64)
            spread(idx, "alpha", sch.share(alpha, rng))
            spread(idx, "comp", sch.share(comp, rng))
            plain[idx] = {"e": e}
        elif kind == "nonlinear":
            bmax = multiplicative_mask_bound(p, op["value_bound"])
            shape = tuple(op["in_shape"])
            if op.get("pool") is None:
                beta = rng.integers(1, bmax + 1, size=shape, dtype=np.int64)
                out = beta
            else:
                kh, kw = op["pool"]
                c, h, w = shape
                out = rng.integers(1, bmax + 1, size=(c, h // kh, w // kw), dtype=np.int64)
                beta = np.repeat(np.repeat(out, kh, axis=1), kw, axis=2)
            beta_inv = _inv_vec(out, p)
            spread(idx, "beta", sch.share(beta.astype(np.uint64), rng))
            spread(idx, "beta_inv", sch.share(beta_inv, rng))
            plain[idx] = {"beta": beta}
        elif kind in ("output", "add", "gather"):
            pass
        else:
            raise ValueError(f"unknown op kind {kind!r}")
    return bundles, plain


def _src(op, idx, key="src"):
    return op.get(key, idx - 1)


def simulate(ops, sch, seed, input_int, weight_values, input_index=0, record=False,
             verify=False, return_shares=False, corrupt=None):
    """One secure inference, lockstep.  Returns a dict with output, transcript digest,
    per-op element counts, per-rank final shares (when return_shares) and, with
    verify=True, the number of failed Reed-Solomon checks."""
    p, k, n = sch.p, sch.k, sch.n
    m = 2 * k - 1
    tr = Transcript(n, record)
    w_front = lagrange_weights(sch.front_ids, p)
    w_part = lagrange_weights(sch.part_ids, p)
    R = reducing_matrix(k, n, sch.party_ids, p)
    checks_failed = 0

    # dealing (S/engine.py:40-54): weights lane 1 in sorted name order, input lane 3
    wrng = seeded_rng(seed, 1)
    wsh = {}
    for name in sorted(weight_values):
        wsh[name] = sch.share(encode_signed(weight_values[name], p), wrng)
    xin = sch.share(encode_signed(np.asarray(input_int, dtype=np.int64), p),
                    seeded_rng(seed, 3, input_index))

    # offline phase (S/engine.py:64-74): one MASK_DIST frame per rank
    bundles, _ = source_masks(ops, sch, seeded_rng(seed, 4))
    for r in range(1, n + 1):
        count = sum(v[2].size for v in bundles[r].values())
        tr.send(("offline", -1), 0, r, MASK_DIST, lambda r=r: _bundle_payload(bundles[r]), count)
    prng = {r: seeded_rng(seed, 5, r) for r in range(1, n + 1)}

    # values[i] = {rank: (degree, ndarray)} output of op i; -1 = input
    values = {-1: {r: (k - 1, xin[r - 1]) for r in range(1, n + 1)}}
    out = None
    for idx, op in enumerate(ops):
        kind = op["kind"]
        label = (op["name"], op["layer"])
        x = values.get(_src(op, idx), {})
        res = {}
        pid = lambda r: sch.party_ids[r - 1]
        if kind == "linear":
            w = wsh[op["weight"] + ".w"]
            b = wsh[op["weight"] + ".b"]
            prod = {}
            for r in range(1, m + 1):
                deg, xv = x[r]
                wr = w[r - 1]
                if wr.ndim == 4:
                    cols = im2col(xv.reshape(tuple(op["in_shape"])), wr.shape[2], wr.shape[3],
                                  op["stride"], op["padding"])
                    acc = gemm(wr.reshape(wr.shape[0], -1), cols, p)
                else:
                    acc = gemm(wr, xv.reshape(-1, 1), p).reshape(-1)
                prod[r] = (deg + (k - 1), acc)
            out_ranks = list(range(1, (n if op["passive_out"] else k) + 1))
            if k == 1:
                reduced = {r: prod[r] for r in out_ranks if r in prod}
            else:
                # step 1 (S/protocol.py:154-163)
                subs = {}
                for i in range(1, m + 1):
                    yv = prod[i][1]
                    sh = sch.share(yv, prng[i], ids=sch.front_ids)
                    subs[i] = sh
                    for j in range(1, k + 1):
                        if j != i:
                            tr.send(label, i, j, RESHARE_OUT,
                                    lambda s=sh[j - 1], j=j: _share_payload(pid(j), k - 1, s),
                                    yv.size)
                # step 2 (S/protocol.py:165-185)
                rows = {}
                rt = np.array([[R[i][t] for i in range(m)] for t in range(len(out_ranks))],
                              dtype=np.uint64)
                for j in range(1, k + 1):
                    stack = np.stack([subs[i][j - 1].reshape(-1) for i in range(1, m + 1)])
                    rj = reduce_apply(stack, rt, p)
                    rows[j] = rj
                    for t in out_ranks:
                        if t != j:
                            shp = prod[1][1].shape
                            tr.send(label, j, t, RESHARE_BACK,
                                    lambda v=rj[t - 1].reshape(shp), j=j: _share_payload(pid(j), k - 1, v),
                                    rj[t - 1].size)
                # step 3 (S/protocol.py:187-198)
                reduced = {}
                for t in out_ranks:
                    pts = np.stack([rows[j][t - 1] for j in range(1, k + 1)])
                    reduced[t] = (k - 1, rec(pts, w_front, p).reshape(prod[1][1].shape))
            # rerand + bias (S/layers.py:260-267)
            for t in out_ranks:
                deg, v = reduced[t]
                z = bundles[t].pop((idx, "zero"))[2].reshape(v.shape)
                v = ewise("add", v, z, p)
                bv = b[t - 1]
                if len(op["out_shape"]) == 3:
                    v = ewise("add", v, np.repeat(bv, v.shape[1]).reshape(v.shape), p)
                else:
                    v = ewise("add", v, bv, p)
                res[t] = (deg, v.reshape(tuple(op["out_shape"])))
        elif kind == "truncation":
            step = op["r"] * op["divisor"]
            masked = {}
            senders = range(1, (n if verify else k) + 1)
            for r in senders:
                deg, xv = x[r]
                a = bundles[r].pop((idx, "alpha"))[2]
                masked[r] = ewise("add", xv, a, p)
                if corrupt is not None and corrupt == (idx, r):
                    masked[r] = masked[r].copy()
                    masked[r].flat[0] = (int(masked[r].flat[0]) + 1) % p
                if r != 1:
                    tr.send(label, r, 1, TRUNC_MASKED,
                            lambda v=masked[r], r=r: _share_payload(pid(r), deg, v), xv.size)
            for r in range(k + 1 if not verify else n + 1, n + 1):
                bundles[r].pop((idx, "alpha"))
            pts = np.stack([masked[r] for r in range(1, k + 1)])
            if verify:
                checks_failed += _rs_check(np.stack([masked[r] for r in range(1, n + 1)]),
                                           sch, p)
            t_val = trunc_elite(pts, w_front, op["value_bound"], op["r"], op["divisor"], p)
            fresh = sch.share(t_val, prng[1])
            for r in range(2, n + 1):
                tr.send(label, 1, r, SHARE_DIST,
                        lambda v=fresh[r - 1], r=r: _share_payload(pid(r), k - 1, v), t_val.size)
            for r in range(1, n + 1):
                c = bundles[r].pop((idx, "comp"))[2]
                res[r] = (k - 1, ewise("add", fresh[r - 1], c, p))
        elif kind == "nonlinear":
            masked = {}
            for r in range(1, m + 1):
                deg, xv = x[r]
                bt = bundles[r][(idx, "beta")][2]
                masked[r] = (deg + k - 1, ewise("mul", xv, bt, p))
                if r != 1:
                    tr.send(label, r, 1, NONLIN_MASKED,
                            lambda v=masked[r], r=r: _share_payload(pid(r), v[0], v[1]),
                            xv.size)
            pts = np.stack([masked[r][1].reshape(-1) for r in range(1, m + 1)])
            plain = nonlin_elite(pts, w_part, op["relu"], op.get("pool_kind"),
                                 tuple(op["in_shape"]), op.get("pool"), p)
            plain = plain.reshape(tuple(op["out_shape"]))
            fan = n if op["passive_out"] else k
            for r in range(2, fan + 1):
                tr.send(label, 1, r, NONLIN_PLAIN, lambda: _plain_payload(plain), plain.size)
            for r in range(1, n + 1):
                bundles[r].pop((idx, "beta"))
                bi = bundles[r].pop((idx, "beta_inv"))[2]
                if r <= fan:
                    res[r] = (k - 1, ewise("mul", plain, bi.reshape(plain.shape), p))
        elif kind == "add":
            y = values[_src(op, idx, "src2")]
            for r in range(1, n + 1):
                if r in x and r in y:
                    res[r] = (x[r][0], ewise("add", x[r][1], y[r][1], p))
        elif kind == "gather":
            kh, kw = op["pool"]
            for r, (deg, xv) in x.items():
                res[r] = (deg, window_gather(np.asarray(xv).reshape(tuple(op["in_shape"])), kh, kw,
                                             op["stride"], op["padding"]))
        elif kind == "output":
            senders = range(2, (n if verify else k) + 1)
            for r in senders:
                tr.send(label, r, 1, OUTPUT_SHARE,
                        lambda v=x[r][1], r=r: _share_payload(pid(r), x[r][0], v), x[r][1].size)
            if verify:
                checks_failed += _rs_check(np.stack([x[r][1] for r in range(1, n + 1)]), sch, p)
            v = rec(np.stack([x[r][1] for r in range(1, k + 1)]), w_front, p)
            out = decode_signed(v, p)
            res = x
        else:
            raise ValueError(kind)
        values[idx] = res

    result = {"output": out, "elements": tr.elements, "checks_failed": checks_failed}
    if record:
        result["transcript_digest"] = tr.digest()
    if return_shares:
        result["values"] = values
    return result


def _rs_check(points, sch, p):
    """Reed-Solomon consistency of n points of a degree-(k-1) sharing: every point beyond
    the first k must equal the Lagrange extrapolation of the first k (builder-defined
    verification).  Returns the count of bad elements."""
    k, n = sch.k, sch.n
    bad = np.zeros(points.shape[1:], dtype=bool)
    base = sch.front_ids
    for j in range(k, n):
        xj = sch.party_ids[j]
        coeffs = []
        for i, xi in enumerate(base):
            num, den = 1, 1
            for jj, xm in enumerate(base):
                if jj != i:
                    num = num * (xj - xm) % p
                    den = den * (xi - xm) % p
            coeffs.append(num * pow(den, p - 2, p) % p)
        pred = rec(points[:k], coeffs, p)
        bad |= pred != points[j]
    return int(bad.sum())


def plaintext(ops, input_int, weight_values, threads=0):
    """Integer plaintext engine over a schedule (S/model.py:380-421, merged mode),
    extended with residual "add".  Returns the final int64 tensor."""
    from . import plain_gemm_i64, plain_trunc
    vals = {-1: np.asarray(input_int, dtype=np.int64)}
    out = None
    for idx, op in enumerate(ops):
        x = vals.get(_src(op, idx))
        kind = op["kind"]
        if kind == "linear":
            w = np.asarray(weight_values[op["weight"] + ".w"], dtype=np.int64)
            b = np.asarray(weight_values[op["weight"] + ".b"], dtype=np.int64)
            if w.ndim == 4:
                cols = im2col(x.reshape(tuple(op["in_shape"])), w.shape[2], w.shape[3],
                              op["stride"], op["padding"])
                acc = plain_gemm_i64(w.reshape(w.shape[0], -1), cols, threads) + b[:, None]
            else:
                acc = plain_gemm_i64(w, x.reshape(-1, 1), threads).reshape(-1) + b
            y = acc.reshape(tuple(op["out_shape"]))
        elif kind == "truncation":
            y = plain_trunc(x, op["r"], op["divisor"])
        elif kind == "nonlinear":
            y = np.maximum(x, 0) if op["relu"] else x
            if op.get("pool_kind"):
                kh, kw = op["pool"]
                c, h, w_ = y.shape
                blk = y.reshape(c, h // kh, kh, w_ // kw, kw)
                y = blk.max(axis=(2, 4)) if op["pool_kind"] == "max" else blk.sum(axis=(2, 4))
        elif kind == "add":
            y = x + vals[_src(op, idx, "src2")]
        elif kind == "gather":
            kh, kw = op["pool"]
            y = window_gather(x.reshape(tuple(op["in_shape"])), kh, kw, op["stride"], op["padding"])
        elif kind == "output":
            out = x
            y = x
        vals[idx] = y
    return out, vals
