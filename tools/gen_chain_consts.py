"""Generate paper_2406_02629_b200/csrc/ssn_chain_consts.cuh: the protocol constants of the fused
chain kernels for the default party ids 1..n, as exact rationals (compile-time immediates).

  wf[i]      Lagrange weight at 0 of front id i+1 over ids 1..k            (S/sss.py:151-170)
  wp[j]      Lagrange weight at 0 of participant id j+1 over ids 1..2k-1
  rt[t][j]   D_t * R[j][t]: column t of the reducing matrix (S/sss.py:197-210) scaled by its
             common denominator D_t; rt_dinv[t] = D_t^-1 mod p
  vi[c][j]   D_v * B^-1[j][c] (c < k): the first k columns of the inverse Vandermonde matrix of
             the participant ids, scaled by their common denominator D_v (vi_dinv = D_v^-1 mod p).
             R = B^-1[:, :k] @ B_ext[:k, :] (S/sss.py:197-210), so a front's RESHARE_BACK row to
             rank t is  sum_c id_t^c * (sum_j B^-1[j][c] sub_j)
  ext[t][i]  Reed-Solomon row: share at id t+1 (t >= k) from the front shares (Lagrange basis of
             ids 1..k evaluated at t+1)

All of them are integers for consecutive ids; the script checks that, and checks R against the
product package's SssScheme.reducing_matrix.  Usage: python tools/gen_chain_consts.py"""
import os
import sys
from fractions import Fraction
from math import lcm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
P45 = (1 << 45) - 55
SCHEMES = ((2, 3), (3, 5), (4, 7))


def lagrange_at(ids, x):
    out = []
    for i, xi in enumerate(ids):
        w = Fraction(1)
        for j, xj in enumerate(ids):
            if j != i:
                w *= Fraction(x - xj, xi - xj)
        out.append(w)
    return out


def as_int(v):
    assert v.denominator == 1, v
    return int(v)


def inverse_vandermonde(m):
    """B^-1 over Q for B[i][j] = id_j^i, ids 1..m."""
    ids = list(range(1, m + 1))
    # B[i][j] = id_j^i; B^-1 by Gauss-Jordan over Q
    B = [[Fraction(pid) ** i for pid in ids] for i in range(m)]
    inv = [[Fraction(int(i == j)) for j in range(m)] for i in range(m)]
    A = [row[:] for row in B]
    for col in range(m):
        piv = next(r for r in range(col, m) if A[r][col] != 0)
        A[col], A[piv] = A[piv], A[col]
        inv[col], inv[piv] = inv[piv], inv[col]
        f = A[col][col]
        A[col] = [v / f for v in A[col]]
        inv[col] = [v / f for v in inv[col]]
        for r in range(m):
            if r != col and A[r][col] != 0:
                g = A[r][col]
                A[r] = [a - g * b for a, b in zip(A[r], A[col])]
                inv[r] = [a - g * b for a, b in zip(inv[r], inv[col])]
    return inv


def reducing_columns(k, n):
    """R[j][t] = sum_{c<k} Binv[j][c] * id_t^c (Vandermonde of the 2k-1 participant ids)."""
    m = 2 * k - 1
    inv = inverse_vandermonde(m)
    return [[sum(inv[j][c] * Fraction(t + 1) ** c for c in range(k)) for t in range(n)] for j in range(m)]


def check_against_package(k, n, R):
    try:
        import paper_2406_02629_b200 as P
    except Exception:                                   # generator still works standalone
        return
    F = P.PrimeField()
    S = P.SssScheme(F, k, n)
    Rp = S.reducing_matrix()
    for j in range(2 * k - 1):
        for t in range(n):
            v = R[j][t]
            want = v.numerator % P45 * pow(v.denominator % P45, P45 - 2, P45) % P45
            assert Rp[j][t] == want, (k, n, j, t)


def emit(k, n):
    m = 2 * k - 1
    wf = [as_int(v) for v in lagrange_at(list(range(1, k + 1)), 0)]
    wp = [as_int(v) for v in lagrange_at(list(range(1, m + 1)), 0)]
    R = reducing_columns(k, n)
    check_against_package(k, n, R)
    rt, dens = [], []
    for t in range(n):
        D = lcm(*[R[j][t].denominator for j in range(m)])
        rt.append([as_int(R[j][t] * D) for j in range(m)])
        dens.append(D)
    inv = inverse_vandermonde(m)
    Dv = lcm(*[inv[j][c].denominator for j in range(m) for c in range(k)])
    vi = [[as_int(inv[j][c] * Dv) for j in range(m)] for c in range(k)]
    ext = []
    for t in range(n):
        ext.append([as_int(v) for v in lagrange_at(list(range(1, k + 1)), t + 1)] if t >= k else [0] * k)

    def arr(v):
        return "{" + ", ".join(str(x) for x in v) + "}"

    lines = [f"template <> struct ChainConsts<{k}, {n}> {{"]
    lines.append(f"    static constexpr int M = {m};")
    lines.append(f"    SSN_CC static int64_t wf(int i) {{ constexpr int64_t a[{k}] = {arr(wf)}; return a[i]; }}")
    lines.append(f"    SSN_CC static int64_t wp(int j) {{ constexpr int64_t a[{m}] = {arr(wp)}; return a[j]; }}")
    lines.append(f"    SSN_CC static int64_t rt(int t, int j) {{")
    lines.append(f"        constexpr int64_t a[{n}][{m}] = {{{', '.join(arr(r) for r in rt)}}};")
    lines.append("        return a[t][j];")
    lines.append("    }")
    lines.append(f"    SSN_CC static uint64_t rt_den(int t) {{ constexpr uint64_t a[{n}] = {arr(dens)}; return a[t]; }}")
    dinv = [pow(D, P45 - 2, P45) for D in dens]
    lines.append(f"    SSN_CC static uint64_t rt_dinv(int t) {{")
    lines.append(f"        constexpr uint64_t a[{n}] = {{{', '.join(f'{x}ull' for x in dinv)}}};")
    lines.append("        return a[t];")
    lines.append("    }")
    Dr = lcm(*dens)
    lines.append(f"    static constexpr uint64_t rt_lcm = {Dr};             // common denominator of R's columns")
    lines.append(f"    static constexpr uint64_t rt_lcm_inv = {pow(Dr, P45 - 2, P45)}ull;")
    lines.append(f"    SSN_CC static int64_t vi(int c, int j) {{")
    lines.append(f"        constexpr int64_t a[{k}][{m}] = {{{', '.join(arr(r) for r in vi)}}};")
    lines.append("        return a[c][j];")
    lines.append("    }")
    lines.append(f"    static constexpr uint64_t vi_den = {Dv};")
    lines.append(f"    static constexpr uint64_t vi_dinv = {pow(Dv, P45 - 2, P45)}ull;")
    lines.append(f"    SSN_CC static int64_t ext(int t, int i) {{")
    lines.append(f"        constexpr int64_t a[{n}][{k}] = {{{', '.join(arr(r) for r in ext)}}};")
    lines.append("        return a[t][i];")
    lines.append("    }")
    lines.append("};")
    return "\n".join(lines)


def render():
    body = [
        "// ssn_chain_consts.cuh -- GENERATED by tools/gen_chain_consts.py; do not edit.",
        "// Protocol constants of the fused chain kernels for the default party ids 1..n as exact",
        "// integers (Lagrange rows) and scaled reducing-matrix columns D_t * R[:, t] (S/sss.py:151-210).",
        "#pragma once",
        "#include <cstdint>",
        "#define SSN_CC __host__ __device__ __forceinline__ constexpr",
        "namespace ssn45 {",
        "template <int K, int N> struct ChainConsts;",
    ]
    for k, n in SCHEMES:
        body.append(emit(k, n))
    body.append("}  // namespace ssn45")
    return "\n".join(body) + "\n"


PATH = os.path.join(ROOT, "paper_2406_02629_b200", "csrc", "ssn_chain_consts.cuh")


def main():
    with open(PATH, "w") as f:
        f.write(render())
    print("wrote", PATH)


if __name__ == "__main__":
    main()
