"""The batched lockstep engine (the bench path) against the oracle: decoded outputs
(parity tier T1) and every op's reconstructed value (tier T2) equal the integer plaintext;
verification detects a corrupted share.  GPU only."""

import numpy as np
import pytest
import torch

from oracle import sim

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ssn():
    import paper_2406_02629_b200 as pkg
    pkg._lib.load()
    return pkg


def _plain_batch(ops, xb, weights):
    outs, inter = [], []
    for i in range(xb.shape[0]):
        o, vals = sim.plaintext(ops, xb[i], weights)
        outs.append(o)
        inter.append(vals)
    return np.stack(outs), inter


def test_reference_model_batched_matches_plaintext(ssn):
    from paper_2406_02629_b200.batched import BatchedEngine
    model, _ = ssn.build_reference_model(7, pool="max")
    weights = {name: qt.values for name, qt in model.weights.items()}
    F = ssn.PrimeField()
    for k, n in ((2, 3), (3, 5)):
        scheme = ssn.SssScheme(F, k, n)
        B = 8
        xb = np.stack([ssn.random_input(7, model, index=i)[0] for i in range(B)])
        for fuse in (False, True):
            eng = BatchedEngine(model, scheme, batch=B, seed=9, fuse=fuse)
            ops = [op.meta() for op in eng.ops]
            want, _ = _plain_batch(ops, xb, weights)
            for _ in range(2):                       # second run uses fresh randomness
                assert np.array_equal(eng.run(xb), want)


@pytest.mark.parametrize("verify", [False, True])
def test_lnt_ordering_batched_matches_plaintext(ssn, verify):
    """ordering="lnt" (nonlinear before truncation, S/layers.py:164-184) through the batched
    engine, fused and unfused: decoded outputs equal the integer plaintext of that schedule."""
    from paper_2406_02629_b200.batched import BatchedEngine
    model, _ = ssn.build_reference_model(7, pool="max")
    weights = {name: qt.values for name, qt in model.weights.items()}
    F = ssn.PrimeField()
    for k, n in ((2, 3), (3, 5)):
        scheme = ssn.SssScheme(F, k, n)
        B = 6
        xb = np.stack([ssn.random_input(7, model, index=i)[0] for i in range(B)])
        for fuse in (False, True):
            eng = BatchedEngine(model, scheme, batch=B, seed=5, fuse=fuse, ordering="lnt", verify=verify)
            ops = [op.meta() for op in eng.ops]
            assert [o["kind"] for o in ops] != [o.kind for o in BatchedEngine(
                model, scheme, batch=B, seed=5, fuse=False).ops]          # the schedule did change
            want, _ = _plain_batch(ops, xb, weights)
            assert np.array_equal(eng.run(xb), want)
            if verify:
                assert int(eng.fail.item()) == 0


def test_avg_pool_chain_model(ssn):
    from paper_2406_02629_b200.batched import BatchedEngine
    model, _ = ssn.build_reference_model(7, pool="avg")
    weights = {name: qt.values for name, qt in model.weights.items()}
    scheme = ssn.SssScheme(ssn.PrimeField(), 2, 3)
    xb = np.stack([ssn.random_input(8, model, index=i)[0] for i in range(4)])
    want = np.stack([ssn.plaintext_infer(model, xb[i]) for i in range(4)])
    for fuse in (False, True):
        eng = BatchedEngine(model, scheme, batch=4, seed=2, fuse=fuse)
        assert np.array_equal(eng.run(xb), want)


@pytest.mark.parametrize("fuse", [False, True])
@pytest.mark.parametrize("k,n", [(2, 3), (3, 5)])
def test_tiny_resnet_every_op_reconstructs_to_plaintext(ssn, k, n, fuse):
    from paper_2406_02629_b200 import resnet
    from paper_2406_02629_b200.batched import BatchedEngine
    net = resnet.tiny_resnet(seed=3)
    scheme = ssn.SssScheme(ssn.PrimeField(), k, n)
    B = 3
    xb = net.random_inputs(seed=5, batch=B)
    eng = BatchedEngine(net, scheme, batch=B, seed=11, fuse=fuse)
    assert bool(eng.chains) == fuse
    ops = [op.meta() for op in eng.ops]
    want, inter = _plain_batch(ops, xb, net.weight_values())
    cap = {}
    out = eng.run_device(xb, capture=cap).cpu().numpy()
    assert np.array_equal(out, want)
    for idx, got in cap.items():
        ref = np.stack([inter[b][idx] for b in range(B)])
        assert np.array_equal(got, ref.reshape(got.shape)), (idx, eng.ops[idx].name)
    # independent checker: float64 exact plaintext of the DAG
    pf, _ = resnet.plaintext_forward(net, xb)
    assert np.array_equal(out, pf)


def test_cifar_resnet18_batched_matches_plaintext(ssn):
    from paper_2406_02629_b200 import resnet
    from paper_2406_02629_b200.batched import BatchedEngine
    net = resnet.cifar_resnet18(seed=7)
    scheme = ssn.SssScheme(ssn.PrimeField(), 2, 3)
    xb = net.random_inputs(seed=1, batch=2)
    eng = BatchedEngine(net, scheme, batch=2, seed=3)
    want, _ = resnet.plaintext_forward(net, xb)
    assert np.array_equal(eng.run(xb), want)


@pytest.mark.parametrize("fuse", [False, True])
def test_verification_detects_corruption(ssn, fuse):
    from paper_2406_02629_b200 import resnet
    from paper_2406_02629_b200.batched import BatchedEngine
    from paper_2406_02629_b200.protocol import VerificationError
    net = resnet.tiny_resnet(seed=3)
    scheme = ssn.SssScheme(ssn.PrimeField(), 3, 5)
    xb = net.random_inputs(seed=6, batch=2)
    eng = BatchedEngine(net, scheme, batch=2, seed=4, verify=True, fuse=fuse)
    want, _ = resnet.plaintext_forward(net, xb)
    assert np.array_equal(eng.run(xb), want)
    first_linear = next(i for i, op in enumerate(eng.ops) if op.kind == "linear")
    eng.fault = (first_linear, 4)            # a passive rank's share of a linear output
    with pytest.raises(VerificationError):
        eng.run(xb)
    eng.fault = None
    assert np.array_equal(eng.run(xb), want)


def test_implicit_conv_path_resnet50_small(ssn):
    """Bottleneck ResNet-50 at 64x64: 1x1 stride-1 convs read channel-major planes (mode 1),
    3x3 pad-1 convs on 16x16 maps use the implicit GEMM with pre-shifted copies (mode 2); the
    planes come from the chain kernels.  Outputs equal the im2col path and the plaintext."""
    from paper_2406_02629_b200 import resnet
    from paper_2406_02629_b200.batched import BatchedEngine
    net = resnet.imagenet_resnet(50, image=64)
    scheme = ssn.SssScheme(ssn.PrimeField(), 3, 5)
    xb = net.random_inputs(seed=2, batch=2)
    want, _ = resnet.plaintext_forward(net, xb)
    eng = BatchedEngine(net, scheme, batch=2, seed=5, verify=True)
    modes = {m[1] for m in eng._conv_mode.values()}
    assert modes == {1, 2}, modes
    assert np.array_equal(eng.run(xb), want)
    ref = BatchedEngine(net, scheme, batch=2, seed=5, verify=True, implicit=False)
    assert not ref._conv_mode
    assert np.array_equal(ref.run(xb), want)


@pytest.mark.parametrize("k,n", [(2, 3), (3, 5)])
def test_lenet28_config1(ssn, k, n):
    """Config 1 (LeNet-style CNN on 1x28x28, built from the reference's layer kinds): the
    reference-API simulation and the batched engine both equal plaintext_infer exactly."""
    from paper_2406_02629_b200.batched import BatchedEngine
    from paper_2406_02629_b200.model import build_lenet28
    model, _ = build_lenet28(7)
    scheme = ssn.SssScheme(ssn.PrimeField(), k, n)
    xb = np.stack([ssn.random_input(7, model, index=i)[0] for i in range(4)])
    want = np.stack([ssn.plaintext_infer(model, xb[i]) for i in range(4)])
    got = ssn.simulate_inference(model, scheme, seed=7, input_int=xb[0])
    assert np.array_equal(got.output, want[0])
    eng = BatchedEngine(model, scheme, batch=4, seed=3)
    assert np.array_equal(eng.run(xb), want)


@pytest.mark.parametrize("split,planes,table", [(False, True, False), (True, False, False), (True, True, True)])
def test_chain_variants_agree(ssn, split, planes, table, monkeypatch):
    """The fused chain's variants -- one kernel vs reshare/nonlinearity split, limb planes from
    the chain vs ssn_planes_cn, beta^-1 by per-warp batch inversion vs the inverse table --
    all reproduce the plaintext (ResNet-50 bottlenecks at 64x64, 5 parties, verification)."""
    from paper_2406_02629_b200 import resnet
    from paper_2406_02629_b200.batched import BatchedEngine
    monkeypatch.setenv("SSN_SPLIT_CHAIN", "1" if split else "0")
    monkeypatch.setenv("SSN_CHAIN_PLANES", "1" if planes else "0")
    monkeypatch.setenv("SSN_INV_TABLE", "1" if table else "0")
    net = resnet.imagenet_resnet(50, image=64)
    scheme = ssn.SssScheme(ssn.PrimeField(), 3, 5)
    xb = net.random_inputs(seed=4, batch=2)
    want, _ = resnet.plaintext_forward(net, xb)
    eng = BatchedEngine(net, scheme, batch=2, seed=6, verify=True)
    assert eng.split_chain == split and eng.chain_planes == planes
    assert np.array_equal(eng.run(xb), want)


def test_resnet152_5pc_full_size_matches_plaintext(ssn):
    """The headline configuration at full size (ResNet-152, 224x224, 5 parties, t=2,
    verification on): decoded logits equal the exact integer plaintext, no RS failures."""
    from paper_2406_02629_b200 import resnet
    from paper_2406_02629_b200.batched import BatchedEngine
    net = resnet.imagenet_resnet(152)
    xb = net.random_inputs(seed=8, batch=2)
    eng = BatchedEngine(net, ssn.SssScheme(ssn.PrimeField(), 3, 5), batch=2, seed=13, verify=True)
    want, _ = resnet.plaintext_forward(net, xb, device="cuda")
    assert np.array_equal(eng.run(xb), want)
    assert int(eng.fail.item()) == 0
    # and the oracle's integer plaintext over the schedule (oracle/sim.py, pinned to the
    # reference's plaintext_infer and the reference-composed residual fixture)
    import oracle
    from oracle import sim
    oracle.set_threads(0)
    ops = net.op_dicts()
    for b in range(2):
        got, _ = sim.plaintext(ops, xb[b], net.weight_values())
        assert np.array_equal(got, want[b]), b


@pytest.mark.parametrize("streams", [2, 3])
def test_stream_pipelined_engine_matches_plaintext(ssn, streams):
    """bench.py --streams S: the batch split over S engines on S CUDA streams (shared weight
    shares and limb planes) decodes to the same integer plaintext as one engine."""
    from paper_2406_02629_b200 import resnet
    from paper_2406_02629_b200.batched import StreamPipelinedEngine
    net = resnet.tiny_resnet(seed=3)
    scheme = ssn.SssScheme(ssn.PrimeField(), 3, 5)
    B = 2 * streams
    xb = net.random_inputs(seed=9, batch=B)
    eng = StreamPipelinedEngine(net, scheme, batch=B, streams=streams, seed=4, verify=True)
    want, _ = resnet.plaintext_forward(net, xb)
    for _ in range(2):
        assert np.array_equal(eng.run(xb), want)
    assert all(int(e.fail.item()) == 0 for e in eng.engines)
