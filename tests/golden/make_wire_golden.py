"""Golden wire/container fixtures made by the REFERENCE itself (S/wire.py, S/protocol.py
MaskBundle, S/model.py save_model / save_shares, S/cli.py cmd_share's dealing).

Run in the build container (where /root/reference exists):
    python tests/golden/make_wire_golden.py
Writes tests/golden/wire.json (hex of small frames / payloads / files, sha256 of the dealt
party share files and the reference's decoded TCP-run output) and tests/golden/wire_files/
(one small model file and one party share file).  Nothing on the GPU box reads the reference.
"""

import hashlib
import json
import os
import shutil
import socket
import sys
import tempfile
import threading

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from ssnet import wire  # noqa: E402
from ssnet.cli import check_share_files  # noqa: E402
from ssnet.engine import (deal_input_shares, deal_weight_shares, run_tcp_party, run_tcp_source,  # noqa: E402
                          simulate_inference)
from ssnet.field import PrimeField  # noqa: E402
from ssnet.layers import plan_schedule  # noqa: E402
from ssnet.model import build_reference_model, random_input, save_model, save_shares  # noqa: E402
from ssnet.protocol import MaskBundle  # noqa: E402
from ssnet.sss import SssScheme  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
FILES = os.path.join(OUT, "wire_files")


def free_ports(n):
    socks = [socket.socket() for _ in range(n)]
    for s in socks:
        s.bind(("127.0.0.1", 0))
    ports = [s.getsockname()[1] for s in socks]
    for s in socks:
        s.close()
    return ports


def main():
    g = {}
    F = PrimeField()
    s35 = SssScheme(F, 3, 5)
    g["frame"] = wire.encode_frame(3, wire.Phase.RESHARE_OUT, b"\x01\x02\x03").hex()
    g["hello"] = wire.encode_hello(3, 5, 2, bytes(range(32)), bytes(range(32, 64))).hex()
    vals = np.array([[0, 1, F.p - 1], [12345678901, 2, 3]], dtype=object)
    g["plain_payload"] = wire.encode_plain_tensor(vals).hex()
    sh = s35.gen(np.array([5, 6, 7], dtype=object), coeffs=[np.array([1, 2, 3], dtype=object),
                                                            np.array([4, 5, 6], dtype=object)])
    g["share_payload"] = wire.encode_share_tensor(sh[3]).hex()
    g["share_payload_values"] = [int(v) for v in sh[3].values]
    b = MaskBundle()
    b.put(0, "zero", sh[0])
    b.put(2, "alpha", sh[1])
    g["mask_bundle"] = b.encode().hex()

    os.makedirs(FILES, exist_ok=True)
    model, _ = build_reference_model(7)
    mpath = os.path.join(FILES, "reference_model.ssnm")
    g["model_digest"] = save_model(mpath, model)
    g["model_file_sha256"] = hashlib.sha256(open(mpath, "rb").read()).hexdigest()

    # the reference's `ssnet share` dealing (S/cli.py:115-145), (2,3), seed 7, input 0
    s23 = SssScheme(F, 2, 3)
    ops, sdig = plan_schedule(model, s23, "ltn")
    weight_values = {name: qt.values for name, qt in model.weights.items()}
    per_rank = deal_weight_shares(weight_values, s23, 7)
    x, _ = random_input(7, model, index=0)
    inputs = deal_input_shares(x, s23, 7, 0)
    extra = {"arch": model.arch_meta(), "ordering": "ltn", "seed": 7, "input_index": 0,
             "schedule_digest": sdig.hex()}
    tmp = tempfile.mkdtemp()
    g["share_files_sha256"] = {}
    for rank in range(1, 4):
        entries = dict(per_rank[rank])
        entries["input"] = inputs[rank - 1]
        path = os.path.join(tmp, f"party{rank}.shares")
        save_shares(path, s23, rank, model.digest(), entries, extra=extra)
        g["share_files_sha256"][f"party{rank}.shares"] = hashlib.sha256(open(path, "rb").read()).hexdigest()
    save_shares(os.path.join(tmp, "source.bundle"), s23, 0, model.digest(), {}, extra=extra)
    g["share_files_sha256"]["source.bundle"] = hashlib.sha256(
        open(os.path.join(tmp, "source.bundle"), "rb").read()).hexdigest()
    shutil.copy(os.path.join(tmp, "party2.shares"), os.path.join(FILES, "party2.shares"))
    g["check_share_files"] = check_share_files(tmp)
    shutil.rmtree(tmp)

    # one full reference run over localhost TCP (run-party / run-source), decoded output
    ports = free_ports(3)
    peers = [("127.0.0.1", pt) for pt in ports]
    mdig = model.digest()
    outs = {}

    def party(r):
        outs[r] = run_tcp_party(r, peers, ops, sdig, s23, mdig, 7, per_rank[r], inputs[r - 1])[0]
    th = [threading.Thread(target=party, args=(r,)) for r in (1, 2, 3)]
    for t in th:
        t.start()
    run_tcp_source(peers, ops, sdig, s23, mdig, 7)
    for t in th:
        t.join()
    g["tcp_output"] = [int(v) for v in np.asarray(outs[1]).ravel()]
    g["sim_output"] = [int(v) for v in np.asarray(simulate_inference(model, s23, 7, x).output).ravel()]
    with open(os.path.join(OUT, "wire.json"), "w") as fh:
        json.dump(g, fh, indent=1, sort_keys=True)
    print("wrote", os.path.join(OUT, "wire.json"), "and", FILES)


if __name__ == "__main__":
    main()
