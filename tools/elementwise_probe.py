"""Launch the elementwise field kernels once on 4096^2-element inputs (for ncu captures):
python tools/elementwise_probe.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_02629_b200 import _lib  # noqa: E402
from paper_2406_02629_b200.field import PrimeField  # noqa: E402
from paper_2406_02629_b200.sss import SssScheme  # noqa: E402

p = PrimeField().p
k, n = 3, 5
sch = SssScheme(PrimeField(), k, n)
E = 4096 * 4096
x = torch.empty((n, E), dtype=torch.int64, device="cuda")
_lib.call("ssn_rand", _lib.ptr(x), x.numel(), 0, p, 99, 7, _lib.stream_ptr())
out = torch.empty((n, E), dtype=torch.int64, device="cuda")
ids = _lib.u64_array(list(sch.party_ids))
for _ in range(2):
    _lib.call("ssn_gen", _lib.ptr(x), E, None, 0, 5, 11, k - 1, ids, n, _lib.ptr(out), n * E, E, E, 1, p,
              _lib.stream_ptr())
torch.cuda.synchronize()
print("ok")
