"""Residual networks expressed in the reference's layer vocabulary (configs 2-4).

The reference graph is a chain of conv/dense/truncation/nonlinear layers (S/model.py:148-149)
and cannot express residual adds; SURVEY.md section 7 prescribes composing the reference's
own secure ops with share_add for the shortcut.  This module builds such DAGs:

  conv  -> Truncation(12)                                  (BN folded into the conv)
  relu  -> NonLinear(relu)                                 (masked, S/layers.py:326-380)
  add   -> local share_add of two degree-(k-1) shares      (S/sss.py:238)
  stem max-pool 3x3/s2/p1 -> gather -> NonLinear(relu, max 3x3)
        "gather" is a local op on every party's share: window (oy, ox) of the overlapping pool
        becomes a non-overlapping 3x3 block (zero shares outside the image), so the reference's
        own masked max-pool (window-constant beta, S/layers.py:326-380, S/masks.py:67-90) runs
        unchanged on it.  After ReLU every value is >= 0, so zero fill == -inf padding.
  global avg-pool 7x7 (4x4) -> NonLinear(relu, sum 7x7) -> Truncation(r=1, divisor=49)
        a true average, round_half_away(sum / 49) -- the reference's merged-divisor rounding
        (S/layers.py:300-308, S/model.py:44-50) with r = 1 (the sum is >= 0 after ReLU).

Value bounds follow the reference's planner rules (S/layers.py:94-135, S/model.py:239-252)
generalised to the DAG: an add doubles the bound, a sum pool multiplies it by the window.
Weights are random (He-style uniform, quantized at 2^12 like S/model.py:452-490) with the
last conv of every residual branch damped so 16-bit activations neither overflow nor vanish
through 152 layers; biases are small.  The data path is synthetic.
"""

from dataclasses import dataclass, field

import numpy as np

from .layers import ScheduledOp
from .model import (ACCUMULATOR_BUDGET_BITS, ACTIVATION_BITS, BIAS_BITS, WEIGHT_BITS, QuantizedTensor,
                    quantize)

W_SCALE = 12
B_SCALE = W_SCALE + 7
ACT_BOUND = (1 << (ACTIVATION_BITS - 1)) + 8
RES_BOUND = ACT_BOUND   # residual sums stay 16-bit (a 17-bit stream overflows 3x3x512 fan-in at 2^43)
W_MAX = (1 << (WEIGHT_BITS - 1)) - 1
B_MAX = (1 << (BIAS_BITS - 1)) - 1


@dataclass
class Node:
    kind: str                  # conv | dense | trunc | relu | gather | add | output
    name: str
    src: int                   # producer node index (-1 = input)
    src2: int = None
    out_channels: int = 0
    kernel: int = 1
    stride: int = 1
    padding: int = 0
    shift: int = 0
    pool: tuple = None
    pool_kind: str = None
    relu: bool = True
    divisor: int = 1           # trunc: extra round_half_away divisor (average pooling)


@dataclass
class ResNetGraph:
    name: str
    input_shape: tuple
    nodes: list = field(default_factory=list)
    weights: dict = field(default_factory=dict)
    input_scale_bits: int = 7

    # -- construction helpers --
    def _add(self, node):
        self.nodes.append(node)
        return len(self.nodes) - 1

    def conv_trunc(self, src, name, cout, k, stride=1, pad=0):
        c = self._add(Node("conv", name, src, out_channels=cout, kernel=k, stride=stride, padding=pad))
        return self._add(Node("trunc", f"div.{name}", c, shift=W_SCALE))

    def relu(self, src, name, pool=None, pool_kind=None):
        return self._add(Node("relu", name, src, pool=pool, pool_kind=pool_kind))

    # -- shapes / bounds / schedule --
    def shapes(self):
        shp = {-1: tuple(self.input_shape)}
        for i, nd in enumerate(self.nodes):
            s = shp[nd.src]
            if nd.kind == "conv":
                c, h, w = s
                oh = (h + 2 * nd.padding - nd.kernel) // nd.stride + 1
                ow = (w + 2 * nd.padding - nd.kernel) // nd.stride + 1
                shp[i] = (nd.out_channels, oh, ow)
            elif nd.kind == "dense":
                shp[i] = (nd.out_channels,)
            elif nd.kind == "relu" and nd.pool is not None:
                c, h, w = s
                shp[i] = (c, h // nd.pool[0], w // nd.pool[1])
            elif nd.kind == "gather":
                c, h, w = s
                oh = (h + 2 * nd.padding - nd.kernel) // nd.stride + 1
                ow = (w + 2 * nd.padding - nd.kernel) // nd.stride + 1
                shp[i] = (c, oh * nd.kernel, ow * nd.kernel)
            else:
                shp[i] = s
        return shp

    def plan_ops(self, scheme=None):
        """ScheduledOps with DAG producers (src/src2) and propagated value bounds."""
        shp = self.shapes()
        bound = {-1: ACT_BOUND}
        ops = []
        for i, nd in enumerate(self.nodes):
            s_in, s_out = shp[nd.src], shp[i]
            src = None if nd.src == i - 1 else nd.src
            if nd.kind in ("conv", "dense"):
                fan = (s_in[0] * nd.kernel * nd.kernel) if nd.kind == "conv" else int(np.prod(s_in))
                acc = fan * bound[nd.src] * W_MAX + B_MAX
                if acc >= (1 << ACCUMULATOR_BUDGET_BITS):
                    raise ValueError(f"{nd.name}: accumulator bound 2**{acc.bit_length()} too wide")
                bound[i] = acc
                ops.append(ScheduledOp("linear", i, nd.name, s_in, s_out, stride=nd.stride, padding=nd.padding,
                                       value_bound=acc, weight=nd.name, src=src))
            elif nd.kind == "trunc":
                prev = self.nodes[nd.src] if nd.src >= 0 else None
                vb = bound[nd.src] if prev is not None and prev.kind in ("conv", "dense") else bound[nd.src]
                bound[i] = ACT_BOUND
                ops.append(ScheduledOp("truncation", i, nd.name, s_in, s_out, r=1 << nd.shift, divisor=nd.divisor,
                                       value_bound=vb, src=src))
            elif nd.kind == "relu":
                vb = bound[nd.src]
                if nd.pool_kind == "sum":
                    vb = vb * nd.pool[0] * nd.pool[1]
                bound[i] = vb
                ops.append(ScheduledOp("nonlinear", i, nd.name, s_in, s_out, relu=nd.relu, pool=nd.pool,
                                       pool_kind=nd.pool_kind, value_bound=vb, src=src))
            elif nd.kind == "gather":
                bound[i] = bound[nd.src]
                ops.append(ScheduledOp("gather", i, nd.name, s_in, s_out, pool=(nd.kernel, nd.kernel), stride=nd.stride,
                                       padding=nd.padding, src=src))
            elif nd.kind == "add":
                # residual stream re-bounded to 16 bits (checked by check_bounds on plaintext,
                # like the reference's 16-bit activation check, S/model.py:409-410)
                bound[i] = RES_BOUND
                ops.append(ScheduledOp("add", i, nd.name, s_in, s_out, src=src, src2=nd.src2))
            else:
                raise ValueError(nd.kind)
        last = len(self.nodes) - 1
        final = shp[last]
        ops.append(ScheduledOp("output", -1, "output", final, final))
        return ops

    def op_dicts(self, scheme=None):
        from .layers import _flag_passive
        return [op.meta() for op in _flag_passive(self.plan_ops(scheme), False)]

    def weight_values(self):
        return {name: qt.values for name, qt in self.weights.items()}

    def macs(self):
        shp = self.shapes()
        total = 0
        for i, nd in enumerate(self.nodes):
            if nd.kind == "conv":
                total += int(np.prod(shp[i])) * shp[nd.src][0] * nd.kernel * nd.kernel
            elif nd.kind == "dense":
                total += int(np.prod(shp[nd.src])) * nd.out_channels
        return total

    def random_inputs(self, seed, batch):
        """Quantized inputs uniform in (-1, 1) at 2^7 (S/model.py:493-497 style)."""
        out = []
        for i in range(batch):
            rng = np.random.default_rng([int(seed), 2, int(i)])
            out.append(quantize(rng.uniform(-1.0, 1.0, size=self.input_shape), self.input_scale_bits))
        return np.stack(out)

    # -- weights --
    def init_weights(self, seed, branch_gain=0.25, gain=1.0):
        rng = np.random.default_rng([int(seed), 1])
        shp = self.shapes()
        damp = {nd.src for nd in self.nodes if nd.kind == "add"}   # trunc feeding an add (branch end)
        for i, nd in enumerate(self.nodes):
            if nd.kind not in ("conv", "dense"):
                continue
            cin = shp[nd.src][0]
            if nd.kind == "conv":
                wshape = (nd.out_channels, cin, nd.kernel, nd.kernel)
                fan = cin * nd.kernel * nd.kernel
            else:
                wshape = (nd.out_channels, int(np.prod(shp[nd.src])))
                fan = wshape[1]
            g = gain * (branch_gain if (i + 1) in damp else 1.0)
            limit = np.sqrt(6.0 / fan) * g
            w = rng.uniform(-limit, limit, size=wshape)
            b = rng.uniform(-0.05, 0.05, size=(nd.out_channels,))
            self.weights[nd.name + ".w"] = QuantizedTensor(quantize(w, W_SCALE, WEIGHT_BITS), W_SCALE, WEIGHT_BITS)
            self.weights[nd.name + ".b"] = QuantizedTensor(quantize(b, B_SCALE, BIAS_BITS), B_SCALE, BIAS_BITS)
        return self


def _bottleneck(g, x, name, width, stride, downsample):
    a = g.conv_trunc(x, f"{name}.conv1", width, 1)
    a = g.relu(a, f"{name}.relu1")
    a = g.conv_trunc(a, f"{name}.conv2", width, 3, stride=stride, pad=1)
    a = g.relu(a, f"{name}.relu2")
    a = g.conv_trunc(a, f"{name}.conv3", width * 4, 1)
    sc = g.conv_trunc(x, f"{name}.down", width * 4, 1, stride=stride) if downsample else x
    s = g._add(Node("add", f"{name}.add", a, src2=sc))
    return g.relu(s, f"{name}.relu3")


def _basic(g, x, name, width, stride, downsample):
    a = g.conv_trunc(x, f"{name}.conv1", width, 3, stride=stride, pad=1)
    a = g.relu(a, f"{name}.relu1")
    a = g.conv_trunc(a, f"{name}.conv2", width, 3, pad=1)
    sc = g.conv_trunc(x, f"{name}.down", width, 1, stride=stride) if downsample else x
    s = g._add(Node("add", f"{name}.add", a, src2=sc))
    return g.relu(s, f"{name}.relu2")


def _stem_pool(g, x):
    """3x3 / stride 2 / pad 1 max-pool over ReLU: gathered windows + the reference's pool."""
    x = g._add(Node("gather", "stem.gather", x, kernel=3, stride=2, padding=1))
    return g.relu(x, "stem.pool", pool=(3, 3), pool_kind="max")


def _head(g, x, pool_hw, classes):
    """Global average pool: ReLU + window sum, then round_half_away(sum / pool_hw^2)."""
    x = g.relu(x, "gpool", pool=(pool_hw, pool_hw), pool_kind="sum")
    x = g._add(Node("trunc", "div.gpool", x, shift=0, divisor=pool_hw * pool_hw))
    return _dense(g, x, "fc", classes)


def _dense(g, x, name, classes):
    d = g._add(Node("dense", name, x, out_channels=classes))
    return g._add(Node("trunc", f"div.{name}", d, shift=W_SCALE))


def imagenet_resnet(depth, seed=7, classes=1000, image=224):
    """ResNet-50/101/152 (bottleneck [3,4,6,3] / [3,4,23,3] / [3,8,36,3]) at 224x224."""
    blocks = {50: [3, 4, 6, 3], 101: [3, 4, 23, 3], 152: [3, 8, 36, 3]}[depth]
    g = ResNetGraph(f"resnet{depth}-ss", (3, image, image))
    x = g.conv_trunc(-1, "stem", 64, 7, stride=2, pad=3)
    x = _stem_pool(g, x)
    for si, (nb, width) in enumerate(zip(blocks, (64, 128, 256, 512))):
        for bi in range(nb):
            stride = 2 if (bi == 0 and si > 0) else 1
            x = _bottleneck(g, x, f"s{si + 1}.b{bi}", width, stride, downsample=(bi == 0))
    _head(g, x, image // 32, classes)
    return g.init_weights(seed)


def cifar_resnet18(seed=7, classes=10):
    g = ResNetGraph("resnet18-cifar-ss", (3, 32, 32))
    x = g.conv_trunc(-1, "stem", 64, 3, pad=1)
    x = g.relu(x, "stem.relu")
    for si, width in enumerate((64, 128, 256, 512)):
        for bi in range(2):
            stride = 2 if (bi == 0 and si > 0) else 1
            x = _basic(g, x, f"s{si + 1}.b{bi}", width, stride, downsample=(bi == 0 and si > 0))
    _head(g, x, 4, classes)
    return g.init_weights(seed)


def tiny_resnet(seed=3, classes=10):
    """Small residual net for smoke / parity tests (both block kinds, a downsample, both pools)."""
    g = ResNetGraph("tiny-resnet-ss", (3, 16, 16))
    x = g.conv_trunc(-1, "stem", 8, 3, pad=1)
    x = _stem_pool(g, x)
    x = _basic(g, x, "s1.b0", 8, 1, downsample=False)
    x = _bottleneck(g, x, "s2.b0", 4, 2, downsample=True)
    _head(g, x, 4, classes)
    return g.init_weights(seed)


def plaintext_forward(graph, x, device="cpu", check=True):
    """Exact integer forward of a ResNetGraph (the DAG analogue of plaintext_infer,
    S/model.py:380-421): float64 convolutions are exact here because every partial sum is an
    integer below 2^43 < 2^53.  x: int64 (B, C, H, W).  Raises on activation overflow of the
    planned bounds (|activation| <= 2^15 + 8, like S/model.py:409-410).
    Returns (logits int64 (B, classes), max |activation| seen)."""
    import torch
    import torch.nn.functional as F
    vals = {-1: torch.as_tensor(np.asarray(x), dtype=torch.float64, device=device)}
    peak = 0
    for i, nd in enumerate(graph.nodes):
        t = vals[nd.src]
        if nd.kind == "conv":
            w = torch.as_tensor(graph.weights[nd.name + ".w"].values, dtype=torch.float64, device=device)
            b = torch.as_tensor(graph.weights[nd.name + ".b"].values, dtype=torch.float64, device=device)
            y = F.conv2d(t, w, b, stride=nd.stride, padding=nd.padding)
        elif nd.kind == "dense":
            w = torch.as_tensor(graph.weights[nd.name + ".w"].values, dtype=torch.float64, device=device)
            b = torch.as_tensor(graph.weights[nd.name + ".b"].values, dtype=torch.float64, device=device)
            y = t.reshape(t.shape[0], -1) @ w.T + b
        elif nd.kind == "trunc":
            y = torch.floor(t / float(1 << nd.shift))
            if nd.divisor > 1:                      # round_half_away (S/model.py:44-50)
                y = torch.sign(y) * torch.floor((2 * y.abs() + nd.divisor) / (2 * nd.divisor))
        elif nd.kind == "gather":
            B, c, h, w_ = t.shape
            k, s_, pd = nd.kernel, nd.stride, nd.padding
            cols = F.unfold(t.reshape(B * c, 1, h, w_), k, padding=pd, stride=s_)   # (B*c, k*k, OH*OW)
            oh, ow = (h + 2 * pd - k) // s_ + 1, (w_ + 2 * pd - k) // s_ + 1
            y = cols.reshape(B, c, k, k, oh, ow).permute(0, 1, 4, 2, 5, 3).reshape(B, c, oh * k, ow * k)
        elif nd.kind == "relu":
            y = torch.clamp(t, min=0) if nd.relu else t
            if nd.pool is not None:
                B, c, h, w_ = y.shape
                blk = y.reshape(B, c, h // nd.pool[0], nd.pool[0], w_ // nd.pool[1], nd.pool[1])
                y = blk.amax(dim=(3, 5)) if nd.pool_kind == "max" else blk.sum(dim=(3, 5))
        elif nd.kind == "add":
            y = t + vals[nd.src2]
        else:
            raise ValueError(nd.kind)
        if nd.kind in ("trunc", "add") or (nd.kind == "relu" and nd.pool_kind != "sum"):
            m = float(y.abs().max())
            peak = max(peak, m)
            if check and m > ACT_BOUND:
                raise ValueError(f"activation overflow after {nd.name}: {m:.0f} > {ACT_BOUND}")
        vals[i] = y
    return vals[len(graph.nodes) - 1].to(torch.int64).cpu().numpy(), peak
