"""Share files, the share-file check and cross-host TCP runs on the GPU, against fixtures the
reference made itself (tests/golden/make_wire_golden.py):

* dealing (S/cli.py:115-145) in host-RNG mode writes party files byte-identical to the
  reference's, and check_share_files (S/cli.py:458-475) passes on them and flags a corrupted
  share;
* a full secure inference over localhost TCP with this package's source and parties
  (tcp.run_source_tcp / run_party_tcp) decodes the reference's output;
* a MIXED deployment -- this package's party 1 on the GPU, the unmodified reference's parties
  2, 3 and trusted source (baseline/_ref) -- completes the protocol and decodes the same output.
"""
import hashlib
import json
import os
import socket
import sys
import threading

import numpy as np
import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2406_02629_b200 import containers  # noqa: E402
from paper_2406_02629_b200.field import PrimeField  # noqa: E402
from paper_2406_02629_b200.model import build_reference_model, random_input  # noqa: E402
from paper_2406_02629_b200.sss import SssScheme  # noqa: E402
from paper_2406_02629_b200 import tcp  # noqa: E402

pytestmark = pytest.mark.gpu
G = json.load(open(os.path.join(ROOT, "tests", "golden", "wire.json")))


def _ports(n):
    socks = [socket.socket() for _ in range(n)]
    for s in socks:
        s.bind(("127.0.0.1", 0))
    ports = [s.getsockname()[1] for s in socks]
    for s in socks:
        s.close()
    return [("127.0.0.1", p) for p in ports]


def test_dealt_share_files_match_reference_and_check(tmp_path):
    model, _ = build_reference_model(7)
    s23 = SssScheme(PrimeField(), 2, 3)
    paths = containers.deal_share_files(model, s23, 7, str(tmp_path), rng_mode="host")
    got = {os.path.basename(p): hashlib.sha256(open(p, "rb").read()).hexdigest() for p in paths}
    assert got == G["share_files_sha256"]
    assert containers.check_share_files(str(tmp_path)) == G["check_share_files"]
    # corrupt ONE element of party 2's input share: the two k-subsets now disagree
    header, scheme, entries = containers.load_shares(str(tmp_path / "party2.shares"))
    bad = entries["input"].values.clone()
    bad.view(-1)[5] = (bad.view(-1)[5] + 1) % scheme.field.p
    entries["input"] = type(entries["input"])(entries["input"].party_id, entries["input"].degree, bad, scheme)
    extra = {kk: header[kk] for kk in ("arch", "ordering", "seed", "input_index", "schedule_digest")}
    containers.save_shares(str(tmp_path / "party2.shares"), scheme, 2, header["model_digest"], entries, extra)
    assert containers.check_share_files(str(tmp_path))["rec_mismatch"] == ["input"]


def _run_mesh(party_fns, source_fn):
    outs, errs = {}, []

    def wrap(r, fn):
        try:
            outs[r] = fn()
        except Exception as exc:          # noqa: BLE001 (re-raised by the assert below)
            errs.append((r, exc))
    th = [threading.Thread(target=wrap, args=(r, fn)) for r, fn in party_fns.items()]
    for t in th:
        t.start()
    wrap(0, source_fn)
    for t in th:
        t.join(300)
    assert not errs, errs
    return outs


def test_full_inference_over_tcp_matches_reference():
    model, _ = build_reference_model(7)
    s23 = SssScheme(PrimeField(), 2, 3)
    x, _ = random_input(7, model, 0)
    peers = _ports(3)
    dev = torch.device("cuda", 0)
    outs = _run_mesh({r: (lambda r=r: tcp.run_party_tcp(r, peers, model, s23, 7, x, dev)) for r in (1, 2, 3)},
                     lambda: tcp.run_source_tcp(peers, model, s23, 7))
    assert outs[1].ravel().tolist() == G["tcp_output"] == G["sim_output"]
    assert outs[2] is None and outs[3] is None


def test_mixed_deployment_b200_party_with_reference_parties():
    sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
    try:
        import ssnet
        from ssnet.engine import deal_input_shares, deal_weight_shares, run_tcp_party, run_tcp_source
        from ssnet.layers import plan_schedule
    except ImportError:
        pytest.skip("reference not installed in baseline/_ref (tools/install_reference.sh)")
    rmodel, _ = ssnet.build_reference_model(7)
    rs = ssnet.SssScheme(ssnet.PrimeField(), 2, 3)
    ops, sdig = plan_schedule(rmodel, rs, "ltn")
    wv = {name: qt.values for name, qt in rmodel.weights.items()}
    per_rank = deal_weight_shares(wv, rs, 7)
    rx, _ = ssnet.random_input(7, rmodel, index=0)
    rin = deal_input_shares(rx, rs, 7, 0)
    model, _ = build_reference_model(7)
    assert model.digest() == rmodel.digest()
    x, _ = random_input(7, model, 0)
    peers = _ports(3)
    fns = {1: lambda: tcp.run_party_tcp(1, peers, model, SssScheme(PrimeField(), 2, 3), 7, x, torch.device("cuda", 0))}
    for r in (2, 3):
        fns[r] = (lambda r=r: run_tcp_party(r, peers, ops, sdig, rs, rmodel.digest(), 7, per_rank[r], rin[r - 1])[0])
    outs = _run_mesh(fns, lambda: run_tcp_source(peers, ops, sdig, rs, rmodel.digest(), 7))
    assert outs[1].ravel().tolist() == G["tcp_output"]
