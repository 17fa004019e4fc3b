"""Time the two p45 GEMM kernels (SSN_GEMM_VARIANT=0: 128x16 double-buffered TMEM;
1: 128x32 wide) on conv-like shapes: python tools/gemm_variant_probe.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_02629_b200 import _lib, gemm as G  # noqa: E402

p = (1 << 45) - 55
L = G.limbs(p)
for (M, N, K) in [(15680 * 2, 1024, 256), (250880, 256, 64), (15680 * 2, 256, 1024), (15680 * 2, 256, 2304)]:
    a = torch.empty(M * K, dtype=torch.int64, device="cuda")
    b = torch.empty(N * K, dtype=torch.int64, device="cuda")
    _lib.call("ssn_rand", _lib.ptr(a), a.numel(), 0, p, 1, 1, _lib.stream_ptr())
    _lib.call("ssn_rand", _lib.ptr(b), b.numel(), 0, p, 2, 2, _lib.stream_ptr())
    A = torch.empty((L, M, G.kpad(K)), dtype=torch.uint8, device="cuda")
    B = torch.empty((L, N, G.kpad(K)), dtype=torch.uint8, device="cuda")
    _lib.call("ssn_limb_split", _lib.ptr(a), M, K, G.kpad(K), L, _lib.ptr(A), M * K, 1, _lib.stream_ptr())
    _lib.call("ssn_limb_split", _lib.ptr(b), N, K, G.kpad(K), L, _lib.ptr(B), N * K, 1, _lib.stream_ptr())
    out = torch.empty((N, M), dtype=torch.int64, device="cuda")
    for _ in range(3):
        G.field_matmul(A, B, M, N, K, p, out=out)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        G.field_matmul(A, B, M, N, K, p, out=out)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 10
    print(f"variant={os.environ.get('SSN_GEMM_VARIANT', '1')} M={M} N={N} K={K}: {t:.3f} ms, "
          f"{36 * 2 * M * N * K / t / 1e9:.0f} int8 TOP/s")
