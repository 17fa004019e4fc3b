"""The fused chain kernels' compile-time protocol constants (csrc/ssn_chain_consts.cuh) are the
generator's output for the current SssScheme (tools/gen_chain_consts.py checks R against
SssScheme.reducing_matrix while rendering), and their scaled rationals equal the field values
the kernels' host check compares against (check_consts in csrc/ssn_chain.cu)."""
import importlib.util
import os
from fractions import Fraction

import paper_2406_02629_b200 as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gen():
    spec = importlib.util.spec_from_file_location("gen_chain_consts", os.path.join(ROOT, "tools", "gen_chain_consts.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_committed_header_is_generator_output():
    gen = _gen()
    with open(gen.PATH) as fh:
        assert fh.read() == gen.render(), "regenerate with python tools/gen_chain_consts.py"


def test_factored_reshare_equals_reducing_matrix():
    """R = B^-1[:, :k] B_ext[:k, :]: the fronts' factored evaluation (vi columns, id powers)
    reproduces every entry of the reference's reducing matrix."""
    gen = _gen()
    F = P.PrimeField()
    p = F.p
    for k, n in gen.SCHEMES:
        m = 2 * k - 1
        inv = gen.inverse_vandermonde(m)
        R = P.SssScheme(F, k, n).reducing_matrix()
        for j in range(m):
            for t in range(n):
                v = sum(inv[j][c] * Fraction(t + 1) ** c for c in range(k))
                assert R[j][t] == v.numerator % p * pow(v.denominator % p, p - 2, p) % p
