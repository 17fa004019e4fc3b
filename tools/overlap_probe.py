"""Can a tensor-bound share GEMM and an ALU-bound field kernel run concurrently on one B200?
Times (a) the GEMM alone, (b) an ALU-heavy ssn_gen alone, (c) both on two streams at once.
Usage: python tools/overlap_probe.py [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_02629_b200 import _lib, gemm  # noqa: E402

P = (1 << 45) - 55
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
_lib.load()
dev = torch.device("cuda")
M, N, K = 16384, 2048, 2304
L, Kp = gemm.limbs(P), gemm.kpad(K)
a = torch.randint(0, 256, (L, M, Kp), dtype=torch.uint8, device=dev)
b = torch.randint(0, 256, (L, N, Kp), dtype=torch.uint8, device=dev)
out = torch.empty((N, M), dtype=torch.int64, device=dev)
nel = 1 << 26
sec = torch.randint(0, P, (nel,), dtype=torch.int64, device=dev)
ids = _lib.u64_array([1, 2, 3, 4, 5])
gout = torch.empty((5, nel), dtype=torch.int64, device=dev)


def g():
    for _ in range(reps):
        gemm.field_matmul(a, b, M, N, K, P, out=out)


def e():
    for _ in range(reps * 3):
        _lib.call("ssn_gen", _lib.ptr(sec), 0, None, 0, 7, 11, 6, ids, 5, _lib.ptr(gout), 0, nel, nel, 1, P,
                  _lib.stream_ptr())


def timed(fn):
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    fn()
    t1.record()
    torch.cuda.synchronize()
    return t0.elapsed_time(t1)


s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        g()
    with torch.cuda.stream(s2):
        e()
    cur.wait_stream(s1)
    cur.wait_stream(s2)


for f in (g, e, both):
    f()
tg, te, tb = timed(g), timed(e), timed(both)
print(f"gemm alone {tg:.2f} ms, ALU kernel alone {te:.2f} ms, both concurrently {tb:.2f} ms "
      f"(sum {tg + te:.2f}, max {max(tg, te):.2f})")
