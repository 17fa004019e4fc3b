import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2406_02629_b200 as P
from paper_2406_02629_b200 import resnet, _lib, gemm as G
from paper_2406_02629_b200.batched import BatchedEngine
net = resnet.cifar_resnet18(seed=7)
scheme = P.SssScheme(P.PrimeField(), 2, 3)
xb = net.random_inputs(seed=1, batch=2)
e = BatchedEngine(net, scheme, batch=2, seed=3)
orig = e._gemm_implicit
def patched(idx, op, X):
    src, mode, Wp, copies = e._conv_mode[idx]
    if src in e._planes_ready:
        buf = e._plane_buffer(src)
        C, H, W = op.in_shape
        ref = torch.zeros_like(buf)
        _lib.call("ssn_planes_cn", _lib.ptr(X), e.m, e.batch, C, H, W, Wp, 6, _lib.ptr(ref), e.batch * C * H * W, copies, _lib.stream_ptr())
        torch.cuda.synchronize()
        d = (buf != ref)
        if d.any():
            nz = d.nonzero()
            print("op", idx, op.name, "mode", mode, "Wp", Wp, "mismatch", d.float().mean().item(), "shape", tuple(buf.shape))
            b = buf[0, 0, 0, 0, 0, 0, :40].tolist(); r = ref[0, 0, 0, 0, 0, 0, :40].tolist()
            print("  chain", b); print("  ref  ", r)
            b = buf[1, 0, 0, 0, 0, 0, :40].tolist(); r = ref[1, 0, 0, 0, 0, 0, :40].tolist()
            print("  chain1", b); print("  ref1  ", r)
            for c in range(3):
                print("  copy", c, "mismatch", d[c].float().mean().item(), "party", [d[c, t].float().mean().item() for t in range(3)])
            raise SystemExit
        else:
            print("op", idx, op.name, "planes ok")
    return orig(idx, op, X)
e._gemm_implicit = patched
e.run(xb)
