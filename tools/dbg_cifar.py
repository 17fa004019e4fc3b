import sys, numpy as np
sys.path.insert(0, '.')
import paper_2406_02629_b200 as P
from paper_2406_02629_b200 import resnet
from paper_2406_02629_b200.batched import BatchedEngine
net = resnet.cifar_resnet18(seed=7)
for k, n in ((2, 3), (3, 5)):
    scheme = P.SssScheme(P.PrimeField(), k, n)
    xb = net.random_inputs(seed=1, batch=2)
    want, _ = resnet.plaintext_forward(net, xb)
    for fuse in (False, True):
        e = BatchedEngine(net, scheme, batch=2, seed=3, fuse=fuse)
        ok = np.array_equal(e.run(xb), want)
        print(k, n, "fuse", fuse, "implicit convs", len(e._conv_mode), "ok", ok)
    e0 = BatchedEngine(net, scheme, batch=2, seed=3, implicit=False, fuse=False)
    e1 = BatchedEngine(net, scheme, batch=2, seed=3, fuse=False)
    c0, c1 = {}, {}
    e0.run_device(xb, capture=c0); e1.run_device(xb, capture=c1)
    for idx in sorted(c0):
        if idx in c1 and not np.array_equal(c0[idx], c1[idx]):
            op = e0.ops[idx]; print("first diff at", idx, op.kind, op.name, op.in_shape); break
