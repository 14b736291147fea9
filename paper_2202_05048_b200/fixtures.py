"""Deterministic model generators (host side; not the hot path).

Two families:

* the reference's three 32x32 toy presets, ``generate_fixture(recipe, seed)``
  with recipe in {"lenet-ish", "resnet-toy", "mobile-toy"}.  Node/tensor/
  weight naming and the RNG draw order follow the reference builder
  (/root/reference/pkg/src/ptqtune/fixtures.py:128-265), so the graphs are
  bit-identical to the reference's (pinned by tests/test_host_mirror.py
  against golden hashes produced by the reference itself);
* 224x224 ImageNet-shaped stand-ins for the BASELINE.json configs:
  ``build_model("resnet50"|"resnet18"|"mobilenet_v2"|"squeezenet", seed)``.
  The reference IR has no batch-norm, no pooling padding and no ReLU6
  (ir.py:31-33, :150), so these follow SURVEY.md section 0.4: BN is folded
  away (He-normal conv weights, N(0, 0.01^2) biases), the ResNet stem max-pool
  is k2 s2, MobileNet-v2 uses ReLU.  ShuffleNet needs channel shuffle and
  grouped convs, which the IR cannot express, so it is not offered.

Every generator ends with the reference's "planted head" idea
(fixtures.py:231-252): the last fully-connected layer's rows are the
normalised features of the class templates propagated through the random
stack ahead of it, which makes the fp32 model a template matcher.
"""

from __future__ import annotations

import numpy as np
from numpy.lib.stride_tricks import sliding_window_view

from .dataset import IMAGE_SHAPE, N_CLASSES, class_templates
from .ir import INPUT_TENSOR, Graph, Node, tensor_shapes, validate

IMAGENET_SHAPE = (3, 224, 224)


class _GraphWriter:
    """Sequential graph writer; ``cur`` is the running tensor."""

    def __init__(self, name: str, seed: int, shape=IMAGE_SHAPE):
        self.name = name
        self.rng = np.random.default_rng(seed)
        self.in_shape = tuple(shape)
        self.chw = tuple(shape)
        self.cur = INPUT_TENSOR
        self.nodes: list[Node] = []
        self.weights: dict[str, np.ndarray] = {}
        self.count = 0

    # -- parameters ---------------------------------------------------------
    def _param(self, prefix: str, shape, std: float) -> str:
        key = f"w_{prefix}{len(self.weights)}"
        self.weights[key] = (std * self.rng.standard_normal(shape)).astype(np.float32)
        return key

    def _node(self, kind: str, inputs, attrs=None) -> str:
        nid = f"{kind[:4]}{self.count}"
        self.count += 1
        out = "t_" + nid
        self.nodes.append(Node(nid, kind, list(inputs), out, dict(attrs or {})))
        self.cur = out
        return out

    def at(self, tensor: str, chw) -> "_GraphWriter":
        self.cur, self.chw = tensor, tuple(chw)
        return self

    # -- layers -------------------------------------------------------------
    def conv(self, cout: int, k: int, stride: int = 1, pad: int = 0) -> str:
        cin, h, w = self.chw
        wk = self._param("conv", (cout, cin, k, k), np.sqrt(2.0 / (cin * k * k)))
        bk = self._param("bias", (cout,), 0.01)
        self.chw = (cout, (h + 2 * pad - k) // stride + 1, (w + 2 * pad - k) // stride + 1)
        return self._node("conv2d", [self.cur, wk, bk], {"stride": stride, "padding": pad})

    def dwconv(self, k: int = 3, stride: int = 1, pad: int = 1) -> str:
        c, h, w = self.chw
        wk = self._param("dw", (c, 1, k, k), np.sqrt(2.0 / (k * k)))
        bk = self._param("bias", (c,), 0.01)
        self.chw = (c, (h + 2 * pad - k) // stride + 1, (w + 2 * pad - k) // stride + 1)
        return self._node("depthwise_conv2d", [self.cur, wk, bk],
                          {"stride": stride, "padding": pad})

    def pwconv(self, cout: int) -> str:
        cin, h, w = self.chw
        wk = self._param("pw", (cout, cin, 1, 1), np.sqrt(2.0 / cin))
        bk = self._param("bias", (cout,), 0.01)
        self.chw = (cout, h, w)
        return self._node("pointwise_conv2d", [self.cur, wk, bk], {"stride": 1, "padding": 0})

    def fc(self, nout: int = N_CLASSES) -> str:
        d = int(np.prod(self.chw))
        wk = self._param("fc", (nout, d), np.sqrt(1.0 / d))
        self.chw = (nout,)
        return self._node("fully_connected", [self.cur, wk])

    def relu(self) -> str:
        return self._node("relu", [self.cur])

    def _pool(self, kind: str, k: int, stride: int | None) -> str:
        s = stride or k
        c, h, w = self.chw
        self.chw = (c, (h - k) // s + 1, (w - k) // s + 1)
        return self._node(kind, [self.cur], {"kernel": k, "stride": s})

    def maxpool(self, k: int, stride: int | None = None) -> str:
        return self._pool("maxpool", k, stride)

    def avgpool(self, k: int, stride: int | None = None) -> str:
        return self._pool("avgpool", k, stride)

    def add(self, other: str) -> str:
        return self._node("add", [self.cur, other])

    def concat(self, parts: list[str], chws) -> str:
        self.chw = (sum(p[0] for p in chws),) + tuple(chws[0][1:])
        return self._node("concat", list(parts))

    def softmax(self) -> str:
        return self._node("softmax", [self.cur])

    def finish(self) -> Graph:
        g = Graph(self.name, self.nodes, self.weights, self.in_shape, N_CLASSES)
        validate(g)
        _plant_head(g)
        return g


# --------------------------------------------------------------------------
# reference toy presets (fixtures.py:211-248)

def _toy_lenet(b: _GraphWriter) -> None:
    for cout in (6, 16):
        b.conv(cout, 5)
        b.relu()
        b.maxpool(2)
    b.fc()


def _toy_resnet(b: _GraphWriter) -> None:
    b.conv(8, 3, pad=1)
    skip = b.relu()
    b.conv(8, 3, pad=1)
    b.add(skip)
    b.relu()
    b.maxpool(2)
    b.conv(16, 3, stride=2, pad=1)
    b.relu()
    b.avgpool(4)
    b.fc()
    b.softmax()


def _toy_mobile(b: _GraphWriter) -> None:
    b.conv(8, 3, pad=1)
    b.relu()
    for cout, pool in ((16, b.maxpool), (32, b.avgpool)):
        b.dwconv()
        b.relu()
        b.pwconv(cout)
        b.relu()
        pool(4)
    b.fc()


TOY_RECIPES = {"lenet-ish": _toy_lenet, "resnet-toy": _toy_resnet, "mobile-toy": _toy_mobile}


def generate_fixture(recipe: str, seed: int) -> Graph:
    if recipe not in TOY_RECIPES:
        raise ValueError(f"unknown fixture recipe {recipe!r}; have {sorted(TOY_RECIPES)}")
    b = _GraphWriter(f"{recipe}-s{seed}", seed)
    TOY_RECIPES[recipe](b)
    return b.finish()


# --------------------------------------------------------------------------
# ImageNet-shaped stand-ins

def _resnet(b: _GraphWriter, blocks, bottleneck: bool) -> None:
    b.conv(64, 7, stride=2, pad=3)
    b.relu()
    b.maxpool(2)
    widths = (64, 128, 256, 512)
    expand = 4 if bottleneck else 1
    for stage, (nblk, width) in enumerate(zip(blocks, widths)):
        for i in range(nblk):
            stride = 2 if (stage > 0 and i == 0) else 1
            x, xchw = b.cur, b.chw
            cout = width * expand
            if bottleneck:
                b.pwconv(width)
                b.relu()
                b.conv(width, 3, stride=stride, pad=1)
                b.relu()
                b.pwconv(cout)
            else:
                b.conv(width, 3, stride=stride, pad=1)
                b.relu()
                b.conv(width, 3, pad=1)
            main, mchw = b.cur, b.chw
            if stride != 1 or xchw[0] != cout:
                b.at(x, xchw)
                if stride == 1:
                    skip = b.pwconv(cout)
                else:
                    skip = b.conv(cout, 1, stride=stride)
                b.at(main, mchw)
            else:
                skip = x
            b.add(skip)
            b.relu()
    b.avgpool(b.chw[1])
    b.fc()


def _mobilenet_v2(b: _GraphWriter) -> None:
    b.conv(32, 3, stride=2, pad=1)
    b.relu()
    cin = 32
    for t, c, n, s in ((1, 16, 1, 1), (6, 24, 2, 2), (6, 32, 3, 2), (6, 64, 4, 2),
                       (6, 96, 3, 1), (6, 160, 3, 2), (6, 320, 1, 1)):
        for i in range(n):
            stride = s if i == 0 else 1
            x = b.cur
            if t != 1:
                b.pwconv(cin * t)
                b.relu()
            b.dwconv(3, stride=stride, pad=1)
            b.relu()
            b.pwconv(c)
            if stride == 1 and cin == c:
                b.add(x)
            cin = c
    b.pwconv(1280)
    b.relu()
    b.avgpool(b.chw[1])
    b.fc()


def _squeezenet(b: _GraphWriter) -> None:
    b.conv(96, 7, stride=2)
    b.relu()
    b.maxpool(3, 2)
    fires = [(16, 64), (16, 64), (32, 128), "pool", (32, 128), (48, 192), (48, 192),
             (64, 256), "pool", (64, 256)]
    for f in fires:
        if f == "pool":
            b.maxpool(3, 2)
            continue
        sq, ex = f
        b.pwconv(sq)
        s = b.relu()
        schw = b.chw
        b.pwconv(ex)
        e1 = b.relu()
        e1chw = b.chw
        b.at(s, schw)
        b.conv(ex, 3, pad=1)
        e3 = b.relu()
        b.concat([e1, e3], [e1chw, b.chw])
    b.pwconv(1000)
    b.relu()
    b.avgpool(b.chw[1])
    b.fc()


IMAGENET_MODELS = {
    "resnet18": lambda b: _resnet(b, (2, 2, 2, 2), bottleneck=False),
    "resnet50": lambda b: _resnet(b, (3, 4, 6, 3), bottleneck=True),
    "mobilenet_v2": _mobilenet_v2,
    "squeezenet": _squeezenet,
}


def build_model(name: str, seed: int = 0, shape=IMAGENET_SHAPE) -> Graph:
    if name in TOY_RECIPES:
        return generate_fixture(name, seed)
    if name not in IMAGENET_MODELS:
        raise ValueError(f"unknown model {name!r}; have {sorted(IMAGENET_MODELS) + sorted(TOY_RECIPES)}")
    b = _GraphWriter(f"{name}-s{seed}", seed, shape)
    IMAGENET_MODELS[name](b)
    return b.finish()


def macs_per_image(g) -> int:
    """Multiply-accumulates of the weighted layers for one image."""
    shapes = tensor_shapes(g)
    total = 0
    for n in g.nodes:
        if n.kind in ("conv2d", "pointwise_conv2d", "depthwise_conv2d"):
            o, ci, kh, kw = g.weights[n.inputs[1]].shape
            c, h, w = shapes[n.output]
            total += c * h * w * ci * kh * kw
        elif n.kind == "fully_connected":
            total += int(np.prod(g.weights[n.inputs[1]].shape))
    return total


def int8_traffic_per_image(g) -> int:
    """Minimal HBM bytes of one image's int8 forward (SURVEY.md 8(d) whole-path roofline): every
    weighted layer reads its int8 input and writes its int8 output once, a residual add's second
    operand is read once (in the producing conv's epilogue), pools / concats read their inputs
    and write their output once, and the fp32 image is read once (4 bytes per value)."""
    shapes = tensor_shapes(g)

    def el(t):
        return int(np.prod(shapes[t]))
    b = 0
    for n in g.nodes:
        if n.kind in ("conv2d", "pointwise_conv2d", "depthwise_conv2d", "fully_connected"):
            b += el(n.inputs[0]) + el(n.output)
        elif n.kind == "add":
            b += el(n.inputs[1])
        elif n.kind in ("maxpool", "avgpool", "concat"):
            b += sum(el(t) for t in n.inputs) + el(n.output)
    return b + 3 * int(np.prod(g.input_shape))          # fp32 image: 4 bytes, 1 already counted


# --------------------------------------------------------------------------
# planted head: host fp32 forward of the class templates (model construction
# only; the evaluator's own fp32 forward runs on the GPU)

def _host_windows(x, k, stride, pad):
    if pad:
        x = np.pad(x, ((0, 0), (0, 0), (pad, pad), (pad, pad)))
    return sliding_window_view(x, (k, k), axis=(2, 3))[:, :, ::stride, ::stride]


def _host_forward_until(g, batch: np.ndarray, target: str) -> np.ndarray:
    env = {INPUT_TENSOR: batch}
    if target == INPUT_TENSOR:
        return batch
    for n in g.nodes:
        x = env[n.inputs[0]]
        if n.kind in ("conv2d", "pointwise_conv2d"):
            w, b = g.weights[n.inputs[1]], g.weights[n.inputs[2]] if len(n.inputs) > 2 else None
            s, p = int(n.attrs.get("stride", 1)), int(n.attrs.get("padding", 0))
            win = _host_windows(x, w.shape[2], s, p)
            nb, _, oh, ow = win.shape[:4]
            cols = np.ascontiguousarray(win.transpose(0, 2, 3, 1, 4, 5).reshape(nb * oh * ow, -1))
            y = cols @ w.reshape(w.shape[0], -1).T
            if b is not None:
                y = y + b
            y = y.reshape(nb, oh, ow, w.shape[0]).transpose(0, 3, 1, 2)
        elif n.kind == "depthwise_conv2d":
            w, b = g.weights[n.inputs[1]], g.weights[n.inputs[2]] if len(n.inputs) > 2 else None
            s, p = int(n.attrs.get("stride", 1)), int(n.attrs.get("padding", 0))
            win = _host_windows(x, w.shape[2], s, p)
            y = np.einsum("nchwij,cij->nchw", win, w[:, 0], dtype=x.dtype)
            if b is not None:
                y = y + b[None, :, None, None]
        elif n.kind == "fully_connected":
            w, b = g.weights[n.inputs[1]], g.weights[n.inputs[2]] if len(n.inputs) > 2 else None
            y = x.reshape(x.shape[0], -1) @ w.T
            if b is not None:
                y = y + b
        elif n.kind == "relu":
            y = np.maximum(x, np.float32(0))
        elif n.kind == "maxpool":
            k = int(n.attrs["kernel"])
            y = _host_windows(x, k, int(n.attrs.get("stride", k)), 0).max(axis=(-1, -2))
        elif n.kind == "avgpool":
            k = int(n.attrs["kernel"])
            y = _host_windows(x, k, int(n.attrs.get("stride", k)), 0).mean(axis=(-1, -2), dtype=x.dtype)
        elif n.kind == "add":
            y = x + env[n.inputs[1]]
        elif n.kind == "concat":
            y = np.concatenate([env[t] for t in n.inputs], axis=1)
        elif n.kind == "softmax":
            z = np.exp(x - x.max(axis=-1, keepdims=True))
            y = z / z.sum(axis=-1, keepdims=True)
        else:
            raise ValueError(n.kind)
        env[n.output] = y.astype(np.float32, copy=False)
        if n.output == target:
            return env[n.output]
    raise KeyError(target)


def _plant_head(g: Graph) -> None:
    fcs = [n for n in g.nodes if n.kind == "fully_connected"]
    if not fcs:
        return
    head = fcs[-1]
    feats = _host_forward_until(g, class_templates(g.output_classes, g.input_shape),
                                head.inputs[0])
    feats = feats.reshape(g.output_classes, -1).astype(np.float64)
    norms = np.linalg.norm(feats, axis=1, keepdims=True)
    norms[norms == 0] = 1.0
    g.weights[head.inputs[1]] = (feats / norms).astype(np.float32)
