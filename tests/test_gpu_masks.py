"""Trusted-source mask randomness on the device (speed mode): every sharing the source deals
must use its own polynomial coefficients.  If two sharings reused one Philox stream, a party
could subtract its two shares and the difference would be the SAME at every party -- i.e. a
public function of the two secrets (e.g. zero - beta^-1 = -beta^-1 would leak beta).
Reference: trusted_source_prepare S/protocol.py:354-388, S/masks.py:39-96 (numpy draws are
independent by construction there)."""

import itertools

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import paper_2406_02629_b200 as P
    P._lib.load()
    return P


def _schedule(P):
    from paper_2406_02629_b200.layers import ScheduledOp
    shp = (4, 8, 8)
    return [ScheduledOp("linear", 0, "c1", (2, 8, 8), shp, value_bound=2 ** 40, weight="c1"),
            ScheduledOp("truncation", 1, "div1", shp, shp, r=1 << 12, value_bound=2 ** 40),
            ScheduledOp("nonlinear", 2, "nl2", shp, shp, relu=True, value_bound=2 ** 15 + 8),
            ScheduledOp("linear", 3, "c3", shp, shp, value_bound=2 ** 40, weight="c3"),
            ScheduledOp("truncation", 4, "div4", shp, shp, r=1 << 12, value_bound=2 ** 40),
            ScheduledOp("nonlinear", 5, "nl5", shp, (4, 4, 4), relu=True, pool=(2, 2), pool_kind="max",
                        value_bound=2 ** 15 + 8),
            ScheduledOp("output", -1, "output", (4, 4, 4), (4, 4, 4))]


@pytest.mark.parametrize("k,n", [(2, 3), (3, 5)])
def test_device_source_sharings_use_independent_coefficients(pkg, k, n):
    from paper_2406_02629_b200.protocol import trusted_source_prepare
    from paper_2406_02629_b200.rng import DeviceRng
    scheme = pkg.SssScheme(pkg.PrimeField(), k, n)
    p = scheme.field.p
    bundles, _ = trusted_source_prepare(_schedule(pkg), scheme, DeviceRng(7, 4))
    keys = sorted(bundles[1].entries)
    sharings = {key: np.stack([bundles[r].entries[key].values.reshape(-1).cpu().numpy().astype(object)
                               for r in range(1, n + 1)]) for key in keys}
    checked = 0
    for ka, kb in itertools.combinations(keys, 2):
        a, b = sharings[ka], sharings[kb]
        m = min(a.shape[1], b.shape[1])
        diff = (a[:, :m] - b[:, :m]) % p                   # party t: (sA - sB) + sum (cA - cB) id_t^j
        const = np.all(diff == diff[0:1], axis=0)
        # independent coefficients: the difference is constant across parties with prob ~ 2^-45
        assert const.sum() == 0, f"{ka} and {kb} share polynomial coefficients on {const.sum()}/{m} elements"
        checked += 1
    assert checked >= 20
