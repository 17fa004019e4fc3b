"""INTEGRATION.md route B, executed: the ctypes stub a reference maintainer would add
(`ssnet/_b200.py`, taken verbatim from INTEGRATION.md) computes the field contraction of
sss_linear (S/layers.py:252) on the tensor cores, and the UNMODIFIED reference
(baseline/_ref, tools/install_reference.sh) run with that contraction routed through the stub
gives the same decoded outputs and the same SimHub transcript as the stock reference."""
import ctypes
import glob
import os
import re
import sys

import numpy as np
import pytest

import paper_2406_02629_b200 as P
from paper_2406_02629_b200 import _lib

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


def _cudart():
    import torch
    cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib",
                                   "libcudart.so*"))
    cands += glob.glob("/usr/local/cuda/lib64/libcudart.so*")
    if not cands:
        pytest.skip("no libcudart found")
    return sorted(cands)[0]


def _stub():
    """The ```python block of INTEGRATION.md that starts with '# ssnet/_b200.py', with the two
    library names pointed at this checkout's files."""
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    blocks = re.findall(r"```python\n(.*?)```", text, re.S)
    code = next(b for b in blocks if b.startswith("# ssnet/_b200.py"))
    _lib.load()
    code = code.replace('ctypes.CDLL("libssn_b200.so")', f'ctypes.CDLL({_lib.LIB_PATH!r})')
    code = code.replace('ctypes.CDLL("libcudart.so.12")', f'ctypes.CDLL({_cudart()!r})')
    ns = {}
    exec(compile(code, "INTEGRATION.md:ssnet/_b200.py", "exec"), ns)
    return ns


def test_stub_field_matmul_exact():
    stub = _stub()
    p = P.PrimeField().p
    rng = np.random.default_rng(3)
    for O, K, N in ((7, 75, 33), (16, 400, 129), (5, 9, 1)):
        w = rng.integers(0, p, size=(O, K), dtype=np.uint64)
        cols = rng.integers(0, p, size=(K, N), dtype=np.uint64)
        got = stub["field_matmul"](w, cols, p)
        want = (w.astype(object) @ cols.astype(object)) % p
        assert got.dtype == object and np.array_equal(got, want), (O, K, N)


def _reference():
    if not os.path.isdir(os.path.join(REF, "ssnet")):
        pytest.skip("baseline/_ref not installed (tools/install_reference.sh)")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import ssnet
    return ssnet


@pytest.mark.parametrize("k,n", [(2, 3), (3, 5)])
def test_reference_sss_linear_through_stub(k, n):
    ssnet = _reference()
    import ssnet.layers as L
    stub = _stub()
    F = ssnet.PrimeField()
    scheme = ssnet.SssScheme(F, k, n)
    model, _ = ssnet.build_reference_model(7, pool="max")
    x, _ = ssnet.random_input(7, model, index=0)
    stock = ssnet.simulate_inference(model, scheme, 7, x)

    calls = []

    class Cols(np.ndarray):
        """im2col's object matrix; `w @ cols` in sss_linear dispatches here (subclass
        reflected operand) and runs the stub's tensor-core contraction."""

        def __rmatmul__(self, w):
            calls.append(w.shape)
            return stub["field_matmul"](np.asarray(w).astype(np.uint64), np.asarray(self).astype(np.uint64), F.p)

    orig = L.im2col
    L.im2col = lambda *a, **kw: orig(*a, **kw).view(Cols)
    try:
        routed = ssnet.simulate_inference(model, scheme, 7, x)
    finally:
        L.im2col = orig
    assert calls, "the stub was never called"
    assert np.array_equal(np.asarray(routed.output), np.asarray(stock.output))
    assert routed.transcript_digest() == stock.transcript_digest()
