"""Model and share files in the reference's sealed container format (S/wire.py:129-153,
S/model.py:327-347, S/model.py:519-557), plus the share-file consistency check
(S/cli.py:458-475) run on the GPU.

  SSNM  model file: arch meta + quantized weights (i64 LE blobs)
  SSNS  one party's share file: scheme, rank, binding model digest (+ dealing metadata),
        share tensors as u64 LE blobs

Files written here are byte-identical to the reference's for the same content, and files the
reference wrote load here (tests/test_wire_tcp.py, tests/test_gpu_containers_tcp.py).  Share tensors come off / go onto the
GPU as one copy per tensor.
"""

import os

import numpy as np
import torch

from . import wire
from .model import ModelGraph, QuantizedTensor, layers_from_meta

MODEL_MAGIC = b"SSNM"
SHARE_MAGIC = b"SSNS"


def _model_payload(model):
    header = model.arch_meta()
    header["tensors"] = []
    blobs = []
    for name in sorted(model.weights):
        qt = model.weights[name]
        header["tensors"].append({"name": name, "scale_bits": qt.scale_bits, "bits": qt.bits,
                                  "shape": list(qt.values.shape)})
        blobs.append(np.ascontiguousarray(qt.values, dtype="<i8").tobytes())
    return header, b"".join(blobs)


def save_model(path, model):
    """S/model.py:327-330.  Returns the model digest."""
    header, blob = _model_payload(model)
    wire.write_container(path, MODEL_MAGIC, header, blob)
    return model.digest()


def load_model(path):
    """S/model.py:333-347."""
    header, blob, _ = wire.read_container(path, MODEL_MAGIC)
    weights, off = {}, 0
    for item in header["tensors"]:
        shape = tuple(item["shape"])
        count = int(np.prod(shape)) if shape else 1
        vals = np.frombuffer(blob, dtype="<i8", count=count, offset=off).astype(np.int64).reshape(shape)
        off += 8 * count
        weights[item["name"]] = QuantizedTensor(vals, item["scale_bits"], item["bits"])
    return ModelGraph(header["name"], header["input_shape"], layers_from_meta(header["layers"]), weights,
                      header["input_scale_bits"])


def _host_u64(values):
    if isinstance(values, torch.Tensor):
        return values.detach().contiguous().cpu().numpy().view(np.uint64)
    return np.ascontiguousarray(values, dtype=np.uint64)


def save_shares(path, scheme, rank, model_digest, entries, extra=None):
    """One party's share file (S/model.py:519-534): {name: ShareTensor} (device values; any
    object with party_id / degree / values works)."""
    header = {"k": scheme.k, "n": scheme.n, "p": scheme.field.p, "party_ids": list(scheme.party_ids),
              "rank": rank, "model_digest": model_digest, "tensors": []}
    if extra:
        header.update(extra)
    blobs = []
    for name in sorted(entries):
        st = entries[name]
        vals = _host_u64(st.values)
        header["tensors"].append({"name": name, "party_id": st.party_id, "degree": st.degree,
                                  "shape": list(vals.shape)})
        blobs.append(wire.encode_elements(vals))
    wire.write_container(path, SHARE_MAGIC, header, b"".join(blobs))


def read_share_file(path):
    """Host side of load_shares: -> (header, {name: (party_id, degree, uint64 ndarray)}).
    Elements outside [0, p) raise ProtocolError."""
    header, blob, _ = wire.read_container(path, SHARE_MAGIC)
    entries, off = {}, 0
    for item in header["tensors"]:
        shape = tuple(item["shape"])
        count = int(np.prod(shape)) if shape else 1
        vals = wire.decode_elements(blob, count, off).reshape(shape)
        off += 8 * count
        if count and int(vals.max()) >= header["p"]:
            raise wire.ProtocolError(f"{item['name']}: element outside field range")
        entries[item["name"]] = (item["party_id"], item["degree"], vals)
    if off != len(blob):
        raise wire.ProtocolError("share file blob length mismatch")
    return header, entries


def load_shares(path, scheme=None, device=None):
    """-> (header, scheme, {name: ShareTensor}) with values on `device` (default: the current
    CUDA device) (S/model.py:537-557)."""
    from .field import PrimeField
    from .sss import ShareTensor, SssScheme
    header, raw = read_share_file(path)
    if scheme is None:
        scheme = SssScheme(PrimeField(header["p"]), header["k"], header["n"], party_ids=tuple(header["party_ids"]))
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    entries = {name: ShareTensor(pid, deg, torch.from_numpy(vals.view(np.int64).copy()).to(device), scheme)
               for name, (pid, deg, vals) in raw.items()}
    return header, scheme, entries


def load_share_dir(shares_dir, n=None, device=None):
    """Every party file of a dealing (S/cli.py:148-166): -> (header, scheme, {rank: {name: st}},
    [input share per rank]).  Ranks, digests, ordering, seed and scheme must agree."""
    if n is None:
        n = read_share_file(os.path.join(shares_dir, "party1.shares"))[0]["n"]
    preshared, inputs, headers, scheme = {}, [], [], None
    for rank in range(1, n + 1):
        path = os.path.join(shares_dir, f"party{rank}.shares")
        header, scheme, entries = load_shares(path, scheme, device)
        if header["rank"] != rank:
            raise ValueError(f"{path} holds rank {header['rank']}, expected {rank}")
        inputs.append(entries.pop("input"))
        preshared[rank] = entries
        headers.append(header)
    for key in ("model_digest", "schedule_digest", "ordering", "seed", "k", "n"):
        if len({str(h.get(key)) for h in headers}) != 1:
            raise ValueError(f"share files disagree on {key}")
    return headers[0], scheme, preshared, inputs


def deal_share_files(model, scheme, seed, out_dir, ordering="ltn", input_index=0, rng_mode="host"):
    """The dealer side (S/cli.py:115-145): weight and input shares of every party, one SSNS
    file each, plus the source's bundle file.  Host mode reproduces the reference's files."""
    from .engine import deal_input_shares, deal_weight_shares
    from .layers import plan_schedule
    from .model import random_input
    mdig = model.digest()
    _, sdig = plan_schedule(model, scheme, ordering)
    weight_values = {name: qt.values for name, qt in model.weights.items()}
    per_rank = deal_weight_shares(weight_values, scheme, seed, rng_mode)
    x, _ = random_input(seed, model, index=input_index)
    inputs = deal_input_shares(x, scheme, seed, input_index, rng_mode)
    os.makedirs(out_dir, exist_ok=True)
    extra = {"arch": model.arch_meta(), "ordering": ordering, "seed": seed, "input_index": input_index,
             "schedule_digest": sdig.hex()}
    paths = []
    for rank in range(1, scheme.n + 1):
        entries = dict(per_rank[rank])
        entries["input"] = inputs[rank - 1]
        path = os.path.join(out_dir, f"party{rank}.shares")
        save_shares(path, scheme, rank, mdig, entries, extra=extra)
        paths.append(path)
    bundle = os.path.join(out_dir, "source.bundle")
    save_shares(bundle, scheme, 0, mdig, {}, extra=extra)
    return paths + [bundle]


def check_share_files(shares_dir, device=None):
    """Reconstruct every dealt tensor from two different k-subsets of the party files (the
    first k and the last k ranks) on the GPU; a single corrupted share makes them disagree
    (S/cli.py:458-475).  -> {"tensors": count, "rec_mismatch": [names]}."""
    header, scheme, preshared, inputs = load_share_dir(shares_dir, device=device)
    n, k = header["n"], header["k"]
    names = sorted(preshared[1]) + ["input"]
    bad = []
    for name in names:
        shares = inputs if name == "input" else [preshared[r][name] for r in range(1, n + 1)]
        lo = scheme.rec(shares[:k], m=k)
        hi = scheme.rec(shares[n - k:], m=k)
        if not torch.equal(torch.as_tensor(lo), torch.as_tensor(hi)):
            bad.append(name)
    return {"tensors": len(names), "rec_mismatch": bad}
