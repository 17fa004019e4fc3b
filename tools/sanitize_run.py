"""compute-sanitizer workload: the tiny residual net for (2,3) and (3,5) in device and host-fed
randomness with verification, and a 64x64 ResNet-50 through the implicit-GEMM (mode 1 / 2, 2-CTA
cluster) path, each checked against the plaintext.  Usage:
  compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2406_02629_b200 as P
from paper_2406_02629_b200 import batched, resnet
from oracle import sim
F = P.PrimeField()
for k, n in ((2, 3), (3, 5)):
    net = resnet.tiny_resnet(seed=3)
    for host in ("device", "host"):
        eng = batched.BatchedEngine(net, P.SssScheme(F, k, n), batch=3, seed=11, rng_mode=host, verify=True)
        xb = net.random_inputs(seed=5, batch=3)
        out = eng.run(xb)
        ref = np.stack([sim.plaintext(net.op_dicts(P.SssScheme(F, k, n)), xb[i], net.weight_values())[0] for i in range(3)])
        assert np.array_equal(out, ref), (k, n, host)
# a small implicit-conv ResNet-50 slice (mode 1 / mode 2 GEMMs with 2-CTA clusters)
net = resnet.imagenet_resnet(50, image=64)
xb = net.random_inputs(seed=2, batch=2)
want, _ = resnet.plaintext_forward(net, xb)
eng = batched.BatchedEngine(net, P.SssScheme(F, 3, 5), batch=2, seed=5, verify=True)
assert np.array_equal(eng.run(xb), want)
print("sanitize run ok")
